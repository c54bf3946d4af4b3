"""GPU parity of the CUDA path (through the C ABI) against the fp64 oracle.

Bar (BASELINE.json north_star): ACSR metadata and nnz
bit-exact; max-abs error <= 2e-2 for bf16 inputs with fp32 accumulation and
<= 1e-5 for the fp32 path, on the same seeded inputs.
"""
import math
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2407_16847_b200 import splat as S
from workloads import CONFIG_BY_NAME, CONFIGS, Config, Pattern, make_qkv, make_random, make_tensor

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2
TOL_FP32 = 1e-5
DEV = 0


@pytest.fixture(scope="module", autouse=True)
def gpu():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.set_device(DEV)


def dev(x):
    return x.to(f"cuda:{DEV}").contiguous()


def oracle_heads(p, q, k, v, scale, heads, rows=None, want_sp=False):
    """Oracle O (and S, P) for the listed (b*H+h) slices of [BH, N, d] CPU tensors."""
    outs = []
    rp = O.acsr(p)[2] if want_sp else None
    for bh in heads:
        outs.append(O.attention(p, q[bh], k[bh], v[bh], scale, rows=rows, want_sp=want_sp, row_ptr=rp))
    return outs


def maxabs(a, b):
    return float(np.max(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)))) if np.size(a) else 0.0


# ---------------------------------------------------------------------------
# a1: ACSR build on the device, bit-exact
# ---------------------------------------------------------------------------

def device_meta_equals_oracle(p):
    a = S.Acsr(p, device=DEV)
    seg, nseg, row_ptr = a.copy_meta()
    oseg, onseg, orow, rc = O.acsr(p, max_seg=4)
    assert rc == 0
    assert np.array_equal(nseg.numpy().astype(np.int32), onseg), p
    assert np.array_equal(seg.numpy(), oseg), p
    assert np.array_equal(row_ptr.numpy(), orow), p
    assert a.nnz == int(orow[-1])
    a.destroy()


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: c.name)
def test_acsr_bit_exact_configs(cfg):
    device_meta_equals_oracle(cfg.pattern)


@pytest.mark.parametrize("p", [Pattern("window", 8193, lo=5, hi=2), Pattern("window", 50001, lo=7, hi=3000),
                               Pattern("strided_local", 65536, stride=256, causal=1)], ids=["8193", "50001", "65536"])
def test_acsr_bit_exact_multi_tile_scan(p):
    # N > 8192: several scan tiles in one CTA
    device_meta_equals_oracle(p)


def test_acsr_multi_cta_scan_large_n():
    # N > 32 * 8192: tile sums + scan of sums + per-tile apply.  The oracle's mask enumeration is
    # O(N^2), so row_ptr is checked against the window's closed-form row counts
    # min(N-1, i+hi) - max(0, i-lo) + 1 and sampled rows against the oracle
    p = Pattern("window", 300001, lo=3, hi=40)
    a = S.Acsr(p, device=DEV)
    seg, nseg, row_ptr = a.copy_meta()
    i = np.arange(p.seq_len, dtype=np.int64)
    cnt = np.minimum(p.seq_len - 1, i + p.hi) - np.maximum(0, i - p.lo) + 1
    assert np.array_equal(row_ptr.numpy(), np.concatenate([[0], np.cumsum(cnt)]))
    for r in (0, 1, 2, 4, 150000, 262143, 262144, 300000):
        runs = O.runs_from_cols(O.row_cols(p, r), max_seg=64)
        assert [tuple(x) for x in seg[r, :int(nseg[r])].tolist()] == [tuple(x) for x in runs]


@pytest.mark.parametrize("N", [1, 2, 7, 33, 64, 130])
def test_acsr_bit_exact_exhaustive_small(N):
    pats = []
    for lo in range(0, N + 1, max(1, N // 4)):
        pats.append(Pattern("window", N, lo=lo, hi=N - lo))
    for w in range(1, N + 1, max(1, N // 16)):
        pats += [Pattern("blocked", N, block=w), Pattern("strided", N, stride=w),
                 Pattern("strided_local", N, stride=w, causal=1), Pattern("dilated", N, stride=w, radius=min(N, 3))]
        if w >= 2:
            pats.append(Pattern("bigbird", N, block=w, radius=1))
    if N >= 2:
        pats.append(Pattern("global_local", N, lo=N // 3, hi=N // 4, n_global=min(N, 2)))
    for p in pats:
        device_meta_equals_oracle(p)


# ---------------------------------------------------------------------------
# fp32 path (SIMT, paper precision): 1e-5
# ---------------------------------------------------------------------------

def run_unfused(a, Q, K, V, scale, p_dtype):
    B, H = Q.shape[0], Q.shape[1]
    Sd = torch.empty(B * H * a.nnz, dtype=torch.float32, device=Q.device)
    Pd = torch.empty(B * H * a.nnz, dtype=p_dtype, device=Q.device)
    Od = torch.empty_like(Q)
    S.splat_rsddmm(a, Q, K, Sd, scale)
    S.splat_sparse_softmax(a, Sd, Pd, B, H)
    S.splat_rspmm(a, Pd, V, Od)
    torch.cuda.synchronize()
    return Sd.view(B * H, a.nnz), Pd.view(B * H, a.nnz), Od


def test_tiny_config_fp32_all_primitives():
    cfg = CONFIG_BY_NAME["tiny"]
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    Sd, Pd, Od = run_unfused(a, Q, K, V, cfg.scale, torch.float32)
    Of = torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
    torch.cuda.synchronize()
    (o, s, p), = oracle_heads(cfg.pattern, q.view(1, 256, 64), k.view(1, 256, 64), v.view(1, 256, 64), cfg.scale,
                              [0], want_sp=True)
    assert maxabs(Sd[0].cpu(), s) <= TOL_FP32
    assert maxabs(Pd[0].cpu(), p) <= TOL_FP32
    assert maxabs(Od.view(256, 64).cpu(), o) <= TOL_FP32
    assert maxabs(Of.view(256, 64).cpu(), o) <= TOL_FP32


@pytest.mark.parametrize("p,BH", [(Pattern("window", 101, lo=3, hi=3), 3), (Pattern("blocked", 77, block=5), 5),
                                   (Pattern("strided", 130, stride=9), 1), (Pattern("window", 300, lo=90, hi=60), 3)],
                         ids=["win", "blk", "str", "win16"])
def test_softmax_short_rows(p, BH):
    # mean row length <= 64 (<= 256) takes the 8 (16) lanes-per-row softmax; BH * N not a multiple
    # of the rows per CTA leaves a ragged last CTA
    q, k, v = (make_random((BH, p.seq_len, 16), 300 + t, torch.float32) for t in range(3))
    a = S.Acsr(p, device=DEV)
    assert a.nnz <= 256 * p.seq_len
    Q, K, V = (dev(t.view(1, BH, p.seq_len, 16)) for t in (q, k, v))
    Sd = torch.empty(BH * a.nnz, dtype=torch.float32, device=DEV)
    S.splat_rsddmm(a, Q, K, Sd, 0.5)
    refs = oracle_heads(p, q, k, v, 0.5, range(BH), want_sp=True)
    for pdt in (torch.float32, torch.bfloat16):
        Pd = torch.empty(BH * a.nnz, dtype=pdt, device=DEV)
        S.splat_sparse_softmax(a, Sd, Pd, 1, BH)
        torch.cuda.synchronize()
        Pd = Pd.view(BH, a.nnz)
        for bh, (_, _, pref) in enumerate(refs):
            assert maxabs(Pd[bh].float().cpu(), pref) <= (TOL_FP32 if pdt == torch.float32 else 4e-3)


def paper_grid():
    # SPEC criterion 6: 3 paper patterns x densities x N x d
    for N in (64, 128, 256):
        for d in (16, 64):
            for r in (0, 2, N // 8, N // 2, N):
                yield Pattern("window", N, lo=r, hi=r), d
            for w in (1, 4, N // 4, N):
                yield Pattern("blocked", N, block=w), d
            for X in (1, 3, 16, N):
                yield Pattern("strided", N, stride=X), d


@pytest.mark.parametrize("case", list(paper_grid()), ids=lambda c: f"{c[0].kind}-N{c[0].seq_len}-d{c[1]}-{c[0].lo or c[0].block or c[0].stride}")
def test_paper_grid_fp32(case):
    p, d = case
    N, BH = p.seq_len, 2
    q, k, v = (make_random((BH, N, d), 100 + t, torch.float32) for t in range(3))
    a = S.Acsr(p, device=DEV)
    Q, K, V = dev(q.view(1, BH, N, d)), dev(k.view(1, BH, N, d)), dev(v.view(1, BH, N, d))
    _, _, Od = run_unfused(a, Q, K, V, 0.25, torch.float32)
    Of = torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, Of, 0.25)
    torch.cuda.synchronize()
    refs = oracle_heads(p, q, k, v, 0.25, range(BH))
    for bh in range(BH):
        assert maxabs(Od[0, bh].cpu(), refs[bh]) <= TOL_FP32
        assert maxabs(Of[0, bh].cpu(), refs[bh]) <= TOL_FP32


# ---------------------------------------------------------------------------
# bf16 path: 2e-2 (small variants spanning several tiles + ragged tails)
# ---------------------------------------------------------------------------

SMALL_BF16 = [
    Config("lf_small", Pattern("global_local", 1000, lo=128, hi=128, n_global=32), 1, 3, 64, "bf16", 201),
    Config("bb_small", Pattern("bigbird", 1024, block=64, radius=1), 1, 3, 64, "bf16", 202),
    Config("bb_ragged", Pattern("bigbird", 1000, block=64, radius=1), 1, 2, 64, "bf16", 203),
    Config("st_small", Pattern("strided_local", 1100, stride=128, causal=1), 1, 2, 128, "bf16", 204),
    Config("mis_small", Pattern("window", 1500, lo=511, hi=0), 1, 2, 128, "bf16", 205),
    Config("win_d64", Pattern("window", 777, lo=100, hi=37), 1, 2, 64, "bf16", 206),
    Config("dil_d128", Pattern("dilated", 900, stride=3, radius=50), 1, 2, 128, "bf16", 207),
    Config("strided_d64", Pattern("strided", 600, stride=7), 1, 2, 64, "bf16", 208),
    Config("blocked_d64", Pattern("blocked", 640, block=96), 2, 1, 64, "bf16", 209),
    # plain STRIDED with N = X nk, nk | 128 or 128 | nk: the residue-major (permuted, block-
    # diagonal) fused path
    Config("strided_perm_d64", Pattern("strided", 1024, stride=16), 1, 2, 64, "bf16", 220),
    Config("strided_perm_d128", Pattern("strided", 768, stride=12), 1, 2, 128, "bf16", 221),
    Config("strided_perm_ragged", Pattern("strided", 1000, stride=125), 1, 2, 64, "bf16", 222),
    Config("strided_perm_nk128", Pattern("strided", 1024, stride=8), 1, 2, 64, "bf16", 223),
    Config("strided_perm_nk2", Pattern("strided", 512, stride=256), 1, 2, 128, "bf16", 224),
    Config("strided_perm_nk256", Pattern("strided", 1024, stride=4), 1, 2, 64, "bf16", 225),
    Config("strided_perm_nk256_d128", Pattern("strided", 512, stride=2), 1, 2, 128, "bf16", 226),
    Config("tiny_n", Pattern("window", 5, lo=1, hi=1), 1, 1, 64, "bf16", 210),
    # STRIDED_LOCAL with N % l == 0 and N/l | 128: residue decomposition (strided pass on
    # residue-major views + band pass with the merge), R = 2, 1, 4, 16 residues per tile
    Config("st_res_nk64", Pattern("strided_local", 1024, stride=16, causal=1), 1, 3, 128, "bf16", 211),
    Config("st_res_nk128", Pattern("strided_local", 2048, stride=16, causal=1), 1, 2, 128, "bf16", 212),
    Config("st_res_nk32", Pattern("strided_local", 512, stride=16, causal=1), 2, 1, 128, "bf16", 213),
    Config("st_res_nk8", Pattern("strided_local", 256, stride=32, causal=1), 1, 2, 128, "bf16", 214),
    # d = 64: the fused kernel keeps the natural plan, the unfused primitives split
    Config("st_res_d64", Pattern("strided_local", 1024, stride=16, causal=1), 1, 2, 64, "bf16", 215),
]
RESIDUE = [c for c in SMALL_BF16 if c.name.startswith("st_res")]
PERM = [c for c in SMALL_BF16 if c.name.startswith("strided_perm")]


@pytest.mark.parametrize("cfg", SMALL_BF16, ids=lambda c: c.name)
def test_bf16_fused_and_unfused_small(cfg):
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    Of = torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
    Sd, Pd, Ou = run_unfused(a, Q, K, V, cfg.scale, torch.bfloat16)
    shp = (cfg.BH, cfg.N, cfg.d)
    refs = oracle_heads(cfg.pattern, q.view(shp), k.view(shp), v.view(shp), cfg.scale, range(cfg.BH), want_sp=True)
    Of, Ou = Of.view(shp).float().cpu(), Ou.view(shp).float().cpu()
    for bh, (o, s, p) in enumerate(refs):
        assert maxabs(Of[bh], o) <= TOL_BF16, ("fused", bh)
        assert maxabs(Ou[bh], o) <= TOL_BF16, ("unfused", bh)
        assert maxabs(Sd[bh].cpu(), s) <= TOL_BF16
        assert maxabs(Pd[bh].float().cpu(), p) <= TOL_BF16


@pytest.mark.parametrize("cfg", SMALL_BF16[:5] + RESIDUE + PERM, ids=lambda c: c.name)
def test_bf16_uniform_attention_pin(cfg):
    # Q = 0 -> p_ij = 1/nnz_i; V one-hot (V[j,t] = [t == j mod d]) -> O_i[t] = #{j: j = t mod d}/nnz_i
    N, d = cfg.N, cfg.d
    q = torch.zeros(1, 1, N, d, dtype=torch.bfloat16)
    k = make_random((1, 1, N, d), 7, torch.bfloat16)
    v = torch.zeros(1, 1, N, d, dtype=torch.bfloat16)
    v[0, 0, torch.arange(N), torch.arange(N) % d] = 1
    a = S.Acsr(cfg.pattern, device=DEV)
    Of = torch.empty(1, 1, N, d, dtype=torch.bfloat16, device=f"cuda:{DEV}")
    S.splat_sparse_mhsa(a, dev(q), dev(k), dev(v), Of, 1.0)
    torch.cuda.synchronize()
    m = O.mask(cfg.pattern)
    want = np.zeros((N, d))
    for i in range(N):
        cols = np.nonzero(m[i])[0]
        want[i] = np.bincount(cols % d, minlength=d) / len(cols)
    assert maxabs(Of[0, 0].float().cpu(), want) <= 4e-3


@pytest.mark.parametrize("cfg", [SMALL_BF16[0], RESIDUE[0]], ids=lambda c: c.name)
def test_bf16_stress_large_scores(cfg):
    # Q scaled by 8: score std ~2.7, exercises the online-softmax rescaling (SURVEY C-5) and, for
    # the residue decomposition, the merge of two partial softmaxes with far-apart maxima
    q, k, v = make_qkv(cfg)
    q = (q.float() * 8).to(torch.bfloat16)
    a = S.Acsr(cfg.pattern, device=DEV)
    Of = torch.empty_like(dev(q))
    S.splat_sparse_mhsa(a, dev(q), dev(k), dev(v), Of, cfg.scale)
    torch.cuda.synchronize()
    shp = (cfg.BH, cfg.N, cfg.d)
    refs = oracle_heads(cfg.pattern, q.view(shp), k.view(shp), v.view(shp), cfg.scale, range(cfg.BH))
    for bh in range(cfg.BH):
        assert maxabs(Of.view(shp)[bh].float().cpu(), refs[bh]) <= TOL_BF16


def test_deterministic_and_shard_invariant():
    # (b,h)-sharded execution must be bitwise equal to the single call (no atomics, SURVEY C-4)
    cfg = SMALL_BF16[0]
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    O1, O2 = torch.empty_like(Q), torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, O1, cfg.scale)
    S.splat_sparse_mhsa(a, Q, K, V, O2, cfg.scale)
    parts = []
    for h in range(cfg.H):
        Oh = torch.empty_like(Q[:, h:h + 1])
        S.splat_sparse_mhsa(a, Q[:, h:h + 1].contiguous(), K[:, h:h + 1].contiguous(), V[:, h:h + 1].contiguous(),
                            Oh, cfg.scale)
        parts.append(Oh)
    torch.cuda.synchronize()
    assert torch.equal(O1, O2)
    assert torch.equal(O1, torch.cat(parts, dim=1))


def test_shape_errors():
    cfg = SMALL_BF16[0]
    a = S.Acsr(cfg.pattern, device=DEV)
    Q = torch.zeros(1, 1, cfg.N + 1, 64, dtype=torch.bfloat16, device=f"cuda:{DEV}")
    with pytest.raises(S.SplatError):
        S.splat_sparse_mhsa(a, Q, Q, Q, torch.empty_like(Q), 1.0)
    Q = torch.zeros(1, 1, cfg.N, 96, dtype=torch.bfloat16, device=f"cuda:{DEV}")
    with pytest.raises(S.SplatError) as e:
        S.splat_sparse_mhsa(a, Q, Q, Q, torch.empty_like(Q), 1.0)
    assert e.value.status == 4


# ---------------------------------------------------------------------------
# full-size BASELINE configs, in the launch configuration bench.py times
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["longformer", "bigbird", "sparse_transformer"])
def test_full_config_fused_all_heads(name):
    cfg = CONFIG_BY_NAME[name]
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    Of = torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
    torch.cuda.synchronize()
    shp = (cfg.BH, cfg.N, cfg.d)
    Of = Of.view(shp).float().cpu()
    heads = range(cfg.BH) if os.environ.get("SPLAT_FULL_PARITY", "1") == "1" else range(0, cfg.BH, 11)
    qs, ks, vs = q.view(shp), k.view(shp), v.view(shp)
    worst = 0.0
    for bh in heads:
        ref = O.attention(cfg.pattern, qs[bh], ks[bh], vs[bh], cfg.scale)
        worst = max(worst, maxabs(Of[bh], ref))
    assert worst <= TOL_BF16, worst


@pytest.mark.parametrize("name", ["longformer", "sparse_transformer"])
def test_full_config_unfused_sampled_heads(name):
    cfg = CONFIG_BY_NAME[name]
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    Sd, Pd, Ou = run_unfused(a, Q, K, V, cfg.scale, torch.bfloat16)
    shp = (cfg.BH, cfg.N, cfg.d)
    rp = O.acsr(cfg.pattern)[2]
    for bh in (0, cfg.BH // 2, cfg.BH - 1):
        o, s, p = O.attention(cfg.pattern, q.view(shp)[bh], k.view(shp)[bh], v.view(shp)[bh], cfg.scale,
                              want_sp=True, row_ptr=rp)
        assert maxabs(Sd[bh].cpu(), s) <= TOL_BF16
        assert maxabs(Pd[bh].float().cpu(), p) <= TOL_BF16
        assert maxabs(Ou.view(shp)[bh].float().cpu(), o) <= TOL_BF16


def test_full_mistral_sampled_heads_and_rows():
    cfg = CONFIG_BY_NAME["mistral"]
    # 16 (b,h) slices spread over all 8 shards of the 128 heads; rows: first, middle and last tiles
    heads = [s * 16 + j for s in range(8) for j in (0, 9)]
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    Of = torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
    torch.cuda.synchronize()
    shp = (cfg.BH, cfg.N, cfg.d)
    qs, ks, vs = q.view(shp), k.view(shp), v.view(shp)
    Ov = Of.view(shp)
    for bh in heads:
        for r0 in (0, 16384 - 64, cfg.N - 200):
            r1 = min(cfg.N, r0 + 200)
            ref = O.attention(cfg.pattern, qs[bh], ks[bh], vs[bh], cfg.scale, rows=(r0, r1))
            assert maxabs(Ov[bh, r0:r1].float().cpu(), ref) <= TOL_BF16, (bh, r0)


@pytest.mark.parametrize("cfg", [SMALL_BF16[0], RESIDUE[0], SMALL_BF16[4]], ids=lambda c: c.name)
def test_host_path_pipelined_equals_device_call(cfg):
    # splat_sparse_mhsa_host pipelines (b,h) chunks over three streams; the result must be
    # bitwise the device-resident call's (same kernels, same per-(b,h) work, no atomics)
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Qd, Kd, Vd = dev(q), dev(k), dev(v)
    Od = torch.empty_like(Qd)
    S.splat_sparse_mhsa(a, Qd, Kd, Vd, Od, cfg.scale)
    torch.cuda.synchronize()
    qh, kh, vh = (x.contiguous().pin_memory() for x in (q, k, v))
    oh = torch.empty_like(qh).pin_memory()
    dQ, dK, dV, dO = (torch.empty_like(Qd) for _ in range(4))
    S.splat_sparse_mhsa_host(a, qh, kh, vh, oh, cfg.scale, dQ, dK, dV, dO)
    torch.cuda.synchronize()
    assert torch.equal(oh, Od.cpu())


EDGE = [
    # N = 1: a single query row attending only itself (O = V exactly up to bf16)
    Config("n1_d64", Pattern("window", 1, lo=0, hi=0), 1, 2, 64, "bf16", 301),
    Config("n1_d128", Pattern("window", 1, lo=0, hi=0), 1, 1, 128, "bf16", 302),
    # N just past one tile, one row in the last tile
    Config("n129", Pattern("window", 129, lo=3, hi=3), 1, 2, 64, "bf16", 303),
    # many (b, h) units on a tiny N: more work units than group slots, several per CTA
    Config("many_heads", Pattern("window", 256, lo=16, hi=16), 8, 80, 64, "bf16", 304),
    Config("many_heads_d128", Pattern("blocked", 384, block=128), 4, 50, 128, "bf16", 305),
    # full density (every tile FULL, no masks) and a dilated pattern with sparse chunks
    Config("dense_d64", Pattern("window", 384, lo=384, hi=384), 1, 2, 64, "bf16", 306),
    Config("dilated_d64", Pattern("dilated", 700, stride=7, radius=40), 1, 2, 64, "bf16", 307),
]


@pytest.mark.parametrize("cfg", EDGE, ids=lambda c: c.name)
def test_bf16_fused_edge_cases(cfg):
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    Of = torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
    torch.cuda.synchronize()
    shp = (cfg.BH, cfg.N, cfg.d)
    heads = range(cfg.BH) if cfg.BH <= 8 else [0, 1, cfg.BH // 2, cfg.BH - 2, cfg.BH - 1]
    refs = oracle_heads(cfg.pattern, q.view(shp), k.view(shp), v.view(shp), cfg.scale, heads)
    Of = Of.view(shp).float().cpu()
    for bh, o in zip(heads, refs):
        assert maxabs(Of[bh], o) <= TOL_BF16, (cfg.name, bh)


@pytest.mark.gpu
def test_residue_head_chunks_and_repeat():
    # the residue decomposition over B*H = 70 heads: two head chunks of the launch slot's lse
    # scratch (kLseHeads = 64); repeated calls must give bitwise-identical O and every sampled head
    # (both chunks) must match the oracle
    cfg = Config("st_res_chunks", Pattern("strided_local", 1024, stride=16, causal=1), 7, 10, 128, "bf16", 216)
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    outs = []
    for _ in range(3):
        Of = torch.empty_like(Q)
        S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
        torch.cuda.synchronize()
        outs.append(Of.view(cfg.BH, cfg.N, cfg.d).cpu())
    assert S.last_launch_count() == 4          # two launches (strided pass, band pass) per head chunk
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    shp = (cfg.BH, cfg.N, cfg.d)
    heads = [0, 33, 63, 64, 69]
    refs = oracle_heads(cfg.pattern, q.view(shp), k.view(shp), v.view(shp), cfg.scale, heads)
    for bh, o in zip(heads, refs):
        o = o[0] if isinstance(o, tuple) else o
        assert maxabs(outs[0][bh].float(), o) <= TOL_BF16, bh


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["longformer", "bigbird"])
def test_split_k_long_tiles_few_heads(name):
    # Few heads per call (a rank of a sharded job): the d = 64 kernel takes the split-K unit list --
    # the global-row tiles run as several parts whose partial softmax results the last part merges
    # (DESIGN.md section 8).  Full-size mask, 3 heads, every row against the oracle; repeated calls
    # are bitwise identical (the merge sums the parts in part order, whichever part merges).
    base = CONFIG_BY_NAME[name]
    cfg = Config(name + "_ks", base.pattern, 1, 3, base.d, base.dtype, 217)
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    outs = []
    for _ in range(2):
        Of = torch.empty_like(Q)
        S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
        torch.cuda.synchronize()
        outs.append(Of.view(cfg.BH, cfg.N, cfg.d).cpu())
    assert torch.equal(outs[0], outs[1])
    shp = (cfg.BH, cfg.N, cfg.d)
    refs = oracle_heads(cfg.pattern, q.view(shp), k.view(shp), v.view(shp), cfg.scale, range(cfg.BH))
    for bh, o in enumerate(refs):
        o = o[0] if isinstance(o, tuple) else o
        assert maxabs(outs[0][bh].float(), o) <= TOL_BF16, bh


@pytest.mark.gpu
def test_split_k_ragged_global_rows():
    # split-K on a ragged sequence (rows past N in the last tile) with 64 global rows: the long
    # tile's parts merge, every row of both heads against the oracle
    cfg = Config("ks_ragged", Pattern("global_local", 3000, lo=128, hi=128, n_global=64), 1, 2, 64, "bf16", 218)
    a = S.Acsr(cfg.pattern, device=DEV)
    assert a.ksplit_units().shape[0] > 0                      # the plan has a split-K list
    q, k, v = make_qkv(cfg)
    Q, K, V = dev(q), dev(k), dev(v)
    Of = torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
    torch.cuda.synchronize()
    shp = (cfg.BH, cfg.N, cfg.d)
    out = Of.view(shp).float().cpu()
    refs = oracle_heads(cfg.pattern, q.view(shp), k.view(shp), v.view(shp), cfg.scale, range(cfg.BH))
    for bh, o in enumerate(refs):
        o = o[0] if isinstance(o, tuple) else o
        assert maxabs(out[bh], o) <= TOL_BF16, bh
