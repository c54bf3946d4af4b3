"""Data-layout reordering (PAPER "Data-layout reordering" P:722, Fig. 15
P:863-874): the transposed (column-compressed) ACSR handle, the value transpose and the R-SpMM that
reads column-compressed P, against the oracle.

CPU: the transposed handle's runs equal the oracle's greedy runs of every column of the explicit
mask (P:218-219 applied to M^T), and the density classification.  GPU: the transposed values equal
an independent reordering of the oracle's P (bit-exact), and O from column-compressed P matches the
oracle within the dtype tolerance."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2407_16847_b200 import splat as S
from workloads import Pattern

PATTERNS = [Pattern("window", 300, lo=20, hi=5), Pattern("strided_local", 512, stride=16, causal=1),
            Pattern("global_local", 256, lo=16, hi=16, n_global=4), Pattern("bigbird", 512, block=32, radius=1),
            Pattern("blocked", 200, block=24), Pattern("dilated", 300, stride=3, radius=20),
            Pattern("strided", 256, stride=8)]


def column_runs(m):
    """Per column j of the explicit mask: greedy runs of its rows (the oracle's routine)."""
    n = m.shape[0]
    out = []
    for j in range(n):
        rows = np.nonzero(m[:, j])[0]
        out.append(O.runs_from_cols(rows, 64) if len(rows) else [])
    return out


@pytest.mark.parametrize("p", PATTERNS, ids=lambda p: p.kind)
def test_transpose_handle_is_column_compressed(p):
    a = S.Acsr(p, device=-1)
    at = S.splat_acsr_transpose(a)
    assert at.n == a.n and at.nnz == a.nnz
    seg, nseg, row_ptr = at.copy_meta()
    m = O.mask(p)
    ref = column_runs(m)
    cnt = np.concatenate([[0], np.cumsum(m.sum(axis=0))])
    assert np.array_equal(row_ptr.numpy(), cnt)
    for j in range(p.seq_len):
        runs = [tuple(int(v) for v in seg[j, s]) for s in range(int(nseg[j]))]
        assert runs == ref[j], (p, j)


def test_transpose_of_symmetric_mask_is_itself():
    p = Pattern("window", 257, lo=7, hi=7)
    a = S.Acsr(p, device=-1)
    at = S.splat_acsr_transpose(a)
    for x, y in zip(a.copy_meta(), at.copy_meta()):
        assert torch.equal(x, y)


def test_layout_choice_is_density_threshold():
    for p in PATTERNS:
        a = S.Acsr(p, device=-1)
        dens = a.nnz / p.seq_len ** 2
        assert S.splat_layout_choice(a) == (1 if dens >= S.ALPHA else 0)
        assert S.splat_layout_choice(a, 0.0) == 1
        assert S.splat_layout_choice(a, 1.01) == 0


def column_order(m, vals):
    """Reorder row-compressed values (ACSR order of M) into column-compressed order of M^T."""
    ii, jj = np.nonzero(m)                      # row-major: the ACSR order
    order = np.lexsort((ii, jj))                # by column, then row
    return vals[..., order]


@pytest.mark.gpu
@pytest.mark.parametrize("dt,d", [("fp32", 16), ("fp32", 64), ("bf16", 64), ("fp32", 200)])
@pytest.mark.parametrize("p", PATTERNS[:5], ids=lambda p: p.kind)
def test_column_compressed_rspmm_matches_oracle(p, dt, d):
    torch.manual_seed(11)
    dtype = torch.float32 if dt == "fp32" else torch.bfloat16
    B, H, n = 1, 2, p.seq_len
    q, k, v = ((torch.rand(B * H, n, d) * 2 - 1).to(dtype) for _ in range(3))
    a = S.Acsr(p)
    at = S.splat_acsr_transpose(a)
    m = O.mask(p).astype(bool)
    Ps, Os = [], []
    for bh in range(B * H):
        o, _, pp = O.attention(p, q[bh], k[bh], v[bh], d ** -0.5, want_sp=True)
        Ps.append(pp)
        Os.append(o)
    P = torch.from_numpy(np.stack(Ps)).to(dtype)          # the kernels' input: P rounded to the dtype
    ref_col = column_order(m, P.float().numpy())
    Pd = P.reshape(-1).cuda().contiguous()
    PT = torch.empty_like(Pd)
    S.splat_transpose_values(a, at, Pd, PT, B, H)
    torch.cuda.synchronize()
    assert np.array_equal(PT.float().cpu().numpy().reshape(B * H, -1), ref_col)
    V = v.reshape(B, H, n, d).cuda()
    Oc = torch.empty_like(V)
    S.splat_rspmm_cc(a, at, PT, V, Oc)
    torch.cuda.synchronize()
    # reference: the oracle's P (rounded as the kernel's input) times V in fp64
    Pdense = np.zeros((B * H, n, n))
    for bh in range(B * H):
        Pdense[bh][m] = P[bh].double().numpy()
    Oref = np.einsum("bij,bjd->bid", Pdense, v.double().numpy())
    err = np.abs(Oc.float().cpu().numpy().reshape(B * H, n, d) - Oref).max()
    tol = 1e-5 if dt == "fp32" else 2e-2
    assert err <= tol, err
    # and against the oracle's attention output (P in fp64): same bound
    err2 = np.abs(Oc.float().cpu().numpy().reshape(B * H, n, d) - np.stack(Os)).max()
    assert err2 <= tol, err2


def test_layout_abi_errors():
    L = S.lib()
    import ctypes as C
    assert L.splat_layout_choice(None, 0.1) == 0
    h = C.c_void_p()
    assert L.splat_acsr_transpose(None, None, C.byref(h)) == 1            # INVALID_ARG
    a = S.Acsr(Pattern("window", 64, lo=2, hi=2), device=-1)
    at = S.splat_acsr_transpose(a)
    # host inspection handles have no compute path (no CPU fallback)
    assert L.splat_transpose_values(a.handle, at.handle, None, None, 1, 1, 1, None) == 1
    assert L.splat_rspmm_cc(a.handle, at.handle, None, None, 1, 1, 1, 16, None, None) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("p", PATTERNS, ids=lambda p: p.kind)
def test_device_transpose_handle_equals_host(p):
    ah, ad = S.Acsr(p, device=-1), S.Acsr(p)
    th, td = S.splat_acsr_transpose(ah), S.splat_acsr_transpose(ad)
    for x, y in zip(th.copy_meta(), td.copy_meta()):
        assert torch.equal(x, y)
