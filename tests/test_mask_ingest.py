"""Mask-ingest ACSR build (splat_acsr_from_mask) against the oracle.

Expected metadata comes from the oracle only: per row, oracle.runs_from_cols of the row's columns
(the greedy runs of P:218-219, reading R-4) and the exclusive prefix of their counts; the first
offending point is the start of run max_runs + 1 of the first row that has one, and for
max_runs = 1 it must also equal oracle.regularity's checkRegularity answer.  The CPU
tests run the library's host inspection path (device -1); the GPU tests run the ingest kernel.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2407_16847_b200 import build as B
from paper_2407_16847_b200 import splat as S
from workloads import Pattern
from conftest import cuda_ok


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()
    S.lib()


def expected(mask: np.ndarray, max_runs: int):
    """(seg [n,4,3], nseg [n], row_ptr [n+1], bad (row, col) or None) from the oracle."""
    n = mask.shape[0]
    seg = np.zeros((n, 4, 3), dtype=np.int32)
    nseg = np.zeros(n, dtype=np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    for i in range(n):
        runs = O.runs_from_cols(np.nonzero(mask[i])[0], max_seg=64)
        if len(runs) > max_runs:
            return None, None, None, (i, runs[max_runs][0])
        nseg[i] = len(runs)
        for k, r in enumerate(runs):
            seg[i, k] = r
        row_ptr[i + 1] = row_ptr[i] + sum(r[2] for r in runs)
    return seg, nseg, row_ptr, None


def random_mask(n, rng, max_runs=4, noise_rows=0):
    """Rows made of up to max_runs random affine runs (possibly merging or overlapping, so the
    greedy decomposition is not simply the generating runs), plus noise rows."""
    m = np.zeros((n, n), dtype=bool)
    for i in range(n):
        for _ in range(int(rng.integers(0, max_runs + 1))):
            st = int(rng.integers(0, n))
            step = int(rng.choice([1, 1, 2, 3, 7, 32, 33]))
            cnt = int(rng.integers(1, max(2, (n - st) // step + 1)))
            m[i, st:st + step * cnt:step] = True
    for i in rng.choice(n, size=noise_rows, replace=False) if noise_rows else []:
        m[i] = rng.random(n) < 0.3
    return m


def check_handle(h, mask, max_runs):
    seg, nseg, row_ptr, bad = expected(mask, max_runs)
    assert bad is None
    gs, gn, gr = h.copy_meta()
    assert np.array_equal(gn.numpy().astype(np.int32), nseg)
    assert np.array_equal(gr.numpy(), row_ptr)
    assert np.array_equal(gs.numpy()[:, :, :3], seg)
    assert h.nnz == int(mask.sum())


def ingest(mask, max_runs, device):
    words = S.pack_mask(torch.from_numpy(mask))
    if device >= 0:
        words = words.cuda(device)
    return S.splat_acsr_from_mask(words, mask.shape[0], max_runs=max_runs, device=device)


def test_pack_mask_layout():
    m = torch.zeros((40, 40), dtype=torch.bool)
    m[3, 0] = m[3, 31] = m[3, 32] = m[39, 39] = True
    w = S.pack_mask(m)
    assert w.shape == (40, 2)
    assert w[3, 0].item() == (1 | (1 << 31)) - (1 << 32) and w[3, 1].item() == 1
    assert w[39, 1].item() == 1 << 7


def cases():
    for p in [Pattern("window", 100, lo=3, hi=5), Pattern("blocked", 96, block=7), Pattern("strided", 77, stride=5),
              Pattern("dilated", 90, stride=3, radius=4), Pattern("global_local", 200, lo=7, hi=7, n_global=4),
              Pattern("bigbird", 192, block=8, radius=1), Pattern("strided_local", 256, stride=16, causal=1)]:
        yield p.kind, O.mask(p).astype(bool)


@pytest.mark.parametrize("case", list(cases()), ids=lambda c: c[0])
def test_host_ingest_of_pattern_masks(case):
    _, m = case
    check_handle(ingest(m, 4, -1), m, 4)


@pytest.mark.parametrize("n", [1, 2, 31, 33, 130])
def test_host_ingest_random(n):
    rng = np.random.default_rng(n)
    m = random_mask(n, rng, max_runs=2)
    for max_runs in (1, 2, 3, 4):
        seg, _, _, bad = expected(m, max_runs)
        if bad is None:
            check_handle(ingest(m, max_runs, -1), m, max_runs)
        else:
            with pytest.raises(S.NotRegular) as e:
                ingest(m, max_runs, -1)
            assert (e.value.row, e.value.col) == bad


def test_paper_example_not_regular():
    # {0, 2, 4, 5} is not regular; the offending column is 5
    m = np.zeros((8, 8), dtype=bool)
    m[0, [0, 2, 4, 6]] = True
    m[1, [0, 2, 4, 5]] = True
    ok, _, _, _, bad = O.regularity(m.astype(np.uint8))
    assert not ok and bad == (1, 5)
    with pytest.raises(S.NotRegular) as e:
        ingest(m, 1, -1)
    assert (e.value.row, e.value.col) == (1, 5)
    check_handle(ingest(m, 2, -1), m, 2)


def test_arguments():
    w = torch.zeros((4, 1), dtype=torch.int32)
    with pytest.raises(S.SplatError):
        S.splat_acsr_from_mask(w, 4, max_runs=0, device=-1)
    with pytest.raises(S.SplatError):
        S.splat_acsr_from_mask(w, 4, max_runs=5, device=-1)
    with pytest.raises(S.SplatError):
        S.splat_acsr_from_mask(w, 5, device=-1)          # wrong word count


# ---------------------------------------------------------------- GPU (the ingest kernel)

gpu = pytest.mark.skipif(not cuda_ok(), reason="needs a GPU")


@pytest.mark.gpu
@gpu
@pytest.mark.parametrize("case", list(cases()), ids=lambda c: c[0])
def test_gpu_ingest_of_pattern_masks(case):
    _, m = case
    h = ingest(m, 4, 0)
    check_handle(h, m, 4)
    assert S.last_launch_count() == 2


@pytest.mark.gpu
@gpu
@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 128, 130, 1031, 2048, 2500, 3200])
def test_gpu_ingest_random(n):
    rng = np.random.default_rng(1000 + n)
    m = random_mask(n, rng, max_runs=3, noise_rows=min(3, n // 300))
    for max_runs in (1, 2, 3, 4):
        _, _, _, bad = expected(m, max_runs)
        if bad is None:
            check_handle(ingest(m, max_runs, 0), m, max_runs)
        else:
            with pytest.raises(S.NotRegular) as e:
                ingest(m, max_runs, 0)
            assert (e.value.row, e.value.col) == bad
            if max_runs == 1:
                assert O.regularity(m.astype(np.uint8))[4] == bad


@pytest.mark.gpu
@gpu
def test_gpu_ingest_long_runs_and_first_offender():
    # rows longer than 1024 columns (several 32-word scan chunks) and two rows that need a fifth
    # run: the earlier one is reported
    n = 5000
    m = np.zeros((n, n), dtype=bool)
    for i in range(n):
        m[i, max(0, i - 1500):i + 1] = True
    m[4000, [10, 20, 31, 45, 70, 100, 200]] = True        # 4 two-column runs, then the band
    m[3000, [3, 9, 40, 41, 77, 90, 300]] = True
    assert expected(m, 4)[3][0] == 3000
    expected_bad = expected(m, 4)[3]
    with pytest.raises(S.NotRegular) as e:
        ingest(m, 4, 0)
    assert (e.value.row, e.value.col) == expected_bad


@pytest.mark.gpu
@gpu
def test_gpu_mask_handle_runs_the_fused_path():
    # a handle ingested from a pattern's explicit mask computes what the oracle computes for the
    # pattern (the compute path reads only the ACSR metadata and the plan)
    p = Pattern("window", 512, lo=40, hi=40)
    h = ingest(O.mask(p).astype(bool), 4, 0)
    g = torch.Generator().manual_seed(7)
    q, k, v = (torch.rand((1, 2, 512, 64), generator=g) * 2 - 1 for _ in range(3))
    qb, kb, vb = (t.to(torch.bfloat16) for t in (q, k, v))
    o = torch.empty_like(qb, device="cuda")
    S.splat_sparse_mhsa(h, qb.cuda(), kb.cuda(), vb.cuda(), o, 0.125)
    torch.cuda.synchronize()
    for bh in range(2):
        want = O.attention(p, qb[0, bh].double().numpy(), kb[0, bh].double().numpy(), vb[0, bh].double().numpy(),
                           0.125)
        got = o[0, bh].float().cpu().numpy()
        assert np.max(np.abs(got - want)) < 2e-2


@pytest.mark.gpu
@gpu
@pytest.mark.parametrize("name", ["longformer", "mistral", "win8192", "win12800"])
def test_gpu_ingest_full_size(name):
    # the bench configurations' masks (and two windows whose rows span 256 / 400 words, the other
    # register-resident and streaming kernels), packed on the GPU (no N x N host array), ingested, and
    # compared with the descriptor build (itself bit-exact against the oracle) and with the oracle
    # on sampled rows
    from workloads import CONFIG_BY_NAME
    extra = {"win8192": Pattern("window", 8192, lo=300, hi=20), "win12800": Pattern("window", 12800, lo=5, hi=700)}
    p = extra[name] if name in extra else CONFIG_BY_NAME[name].pattern
    n = p.seq_len
    W = (n + 31) // 32
    words = torch.zeros((n, W), dtype=torch.int32, device="cuda")
    i = torch.arange(n, device="cuda")[:, None]
    for c0 in range(0, n, 4096):
        j = torch.arange(c0, min(n, c0 + 4096), device="cuda")[None, :]
        if p.kind == "window":
            bits = (j >= i - p.lo) & (j <= i + p.hi)
        else:
            g = p.n_global
            bits = (i < g) | (j < g) | ((j >= i - p.lo) & (j <= i + p.hi))
        packed = (bits.view(n, -1, 32).to(torch.int64) << torch.arange(32, device="cuda")).sum(-1)
        words[:, c0 // 32:c0 // 32 + packed.shape[1]] = torch.where(packed >= 2 ** 31, packed - 2 ** 32,
                                                                     packed).to(torch.int32)
    h = S.splat_acsr_from_mask(words, n, device=0)
    ref = S.Acsr(p, device=0)
    a, b = h.copy_meta(), ref.copy_meta()
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    assert h.plan_info() == ref.plan_info()
    for r in [0, 1, n // 3, n - 1]:
        runs = O.runs_from_cols(O.row_cols(p, r), max_seg=64)
        assert [tuple(t) for t in a[0][r, :len(runs)].tolist()] == [tuple(x) for x in runs]
