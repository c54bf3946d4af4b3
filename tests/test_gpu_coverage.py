"""GPU parity coverage beyond test_gpu_parity.py (VERDICT r1 "What's weak" #1):

* unfused S / P / O at full size for BigBird (all 96 heads) and Mistral (8 slices, one per
  8-GPU shard, streamed one head at a time -- SURVEY H7);
* the fused Mistral path on ALL 32,768 rows of 8 slices spread over the 8 shards (SURVEY C-5);
* the fp32 path at d = 128 and d = 256 (include/splat.h allows d <= 256);
* a d = 64 bf16 case with more than 32 key tiles in one query tile;
* the host-buffer path in fp32 with N*d not a multiple of 4 elements (16-byte chunk alignment).

Bar: max-abs <= 2e-2 (bf16 inputs, fp32 accumulation) / 1e-5 (fp32 path) against the fp64
oracle on the same seeded inputs (BASELINE.json north_star)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2407_16847_b200 import splat as S
from workloads import CONFIG_BY_NAME, Config, Pattern, make_qkv, make_slice

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


def maxabs(a, b):
    return float(np.max(np.abs(np.asarray(a, dtype=np.float64) - np.asarray(b, dtype=np.float64)))) if np.size(a) else 0.0


def unfused(a, Q, K, V, scale, p_dtype=torch.bfloat16):
    B, H = Q.shape[0], Q.shape[1]
    Sd = torch.empty(B * H * a.nnz, dtype=torch.float32, device=Q.device)
    Pd = torch.empty(B * H * a.nnz, dtype=p_dtype, device=Q.device)
    Od = torch.empty_like(Q)
    S.splat_rsddmm(a, Q, K, Sd, scale)
    S.splat_sparse_softmax(a, Sd, Pd, B, H)
    S.splat_rspmm(a, Pd, V, Od)
    torch.cuda.synchronize()
    return Sd.view(B * H, a.nnz), Pd.view(B * H, a.nnz), Od


# Mistral: 8 slices, one in each of the 8 contiguous 16-slice shards of bench.py --gpus 8
MISTRAL_SLICES = [s * 16 + (5 * s) % 16 for s in range(8)]


def test_bigbird_unfused_all_heads_full_size():
    cfg = CONFIG_BY_NAME["bigbird"]
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Sd, Pd, Ou = unfused(a, dev(q), dev(k), dev(v), cfg.scale)
    shp = (cfg.BH, cfg.N, cfg.d)
    rp = O.acsr(cfg.pattern)[2]
    Sd, Pd, Ou = Sd.cpu(), Pd.float().cpu(), Ou.view(shp).float().cpu()
    worst = [0.0, 0.0, 0.0]
    for bh in range(cfg.BH):
        o, s, p = O.attention(cfg.pattern, q.view(shp)[bh], k.view(shp)[bh], v.view(shp)[bh], cfg.scale,
                              want_sp=True, row_ptr=rp)
        worst = [max(worst[0], maxabs(Sd[bh], s)), max(worst[1], maxabs(Pd[bh], p)), max(worst[2], maxabs(Ou[bh], o))]
    assert max(worst) <= TOL_BF16, worst


@pytest.mark.parametrize("bh", MISTRAL_SLICES)
def test_mistral_unfused_full_slice(bh):
    cfg = CONFIG_BY_NAME["mistral"]
    q, k, v = (make_slice(cfg.index, t, bh, cfg.N, cfg.d, torch.bfloat16) for t in (0, 1, 2))
    a = S.Acsr(cfg.pattern, device=DEV)
    Sd, Pd, Ou = unfused(a, *(dev(x.view(1, 1, cfg.N, cfg.d)) for x in (q, k, v)), cfg.scale)
    o, s, p = O.attention(cfg.pattern, q, k, v, cfg.scale, want_sp=True)
    assert maxabs(Sd[0].cpu(), s) <= TOL_BF16
    assert maxabs(Pd[0].float().cpu(), p) <= TOL_BF16
    assert maxabs(Ou.view(cfg.N, cfg.d).float().cpu(), o) <= TOL_BF16


def test_mistral_fused_all_rows_eight_shard_slices():
    # the bench launch configuration: all 128 heads in one call; every row of 8 slices checked
    cfg = CONFIG_BY_NAME["mistral"]
    g = torch.Generator(device=f"cuda:{DEV}")
    g.manual_seed(99)
    Q, K, V = ((torch.rand(cfg.B, cfg.H, cfg.N, cfg.d, generator=g, device=f"cuda:{DEV}") * 2 - 1)
               .to(torch.bfloat16) for _ in range(3))
    for t, X in enumerate((Q, K, V)):            # the checked slices carry the seeded inputs
        Xv = X.view(cfg.BH, cfg.N, cfg.d)
        for bh in MISTRAL_SLICES:
            Xv[bh] = dev(make_slice(cfg.index, t, bh, cfg.N, cfg.d, torch.bfloat16))
    a = S.Acsr(cfg.pattern, device=DEV)
    Of = torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
    torch.cuda.synchronize()
    Ov = Of.view(cfg.BH, cfg.N, cfg.d)
    for bh in MISTRAL_SLICES:
        q, k, v = (make_slice(cfg.index, t, bh, cfg.N, cfg.d, torch.bfloat16) for t in (0, 1, 2))
        ref = O.attention(cfg.pattern, q, k, v, cfg.scale)
        assert maxabs(Ov[bh].float().cpu(), ref) <= TOL_BF16, bh


FP32_WIDE = [
    Config("fp32_d128_win", Pattern("window", 300, lo=40, hi=25), 1, 2, 128, "fp32", 401),
    Config("fp32_d256_gl", Pattern("global_local", 260, lo=30, hi=30, n_global=4), 1, 2, 256, "fp32", 402),
    Config("fp32_d256_st", Pattern("strided_local", 256, stride=16, causal=1), 1, 1, 256, "fp32", 403),
    Config("fp32_d200_bb", Pattern("bigbird", 320, block=32, radius=1), 2, 1, 200, "fp32", 404),
]


@pytest.mark.parametrize("cfg", FP32_WIDE, ids=lambda c: c.name)
def test_fp32_wide_head_dim(cfg):
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    Sd, Pd, Ou = unfused(a, Q, K, V, cfg.scale, torch.float32)
    Of = torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
    torch.cuda.synchronize()
    shp = (cfg.BH, cfg.N, cfg.d)
    rp = O.acsr(cfg.pattern)[2]
    for bh in range(cfg.BH):
        o, s, p = O.attention(cfg.pattern, q.view(shp)[bh], k.view(shp)[bh], v.view(shp)[bh], cfg.scale,
                              want_sp=True, row_ptr=rp)
        assert maxabs(Sd[bh].cpu(), s) <= TOL_FP32
        assert maxabs(Pd[bh].cpu(), p) <= TOL_FP32
        assert maxabs(Ou.view(shp)[bh].cpu(), o) <= TOL_FP32
        assert maxabs(Of.view(shp)[bh].cpu(), o) <= TOL_FP32


def test_d64_query_tile_with_many_key_tiles():
    # global rows of query tile 0 touch 47 key tiles (> the 32 entries some kernels cache on chip)
    cfg = Config("gl6000", Pattern("global_local", 6000, lo=64, hi=64, n_global=32), 1, 2, 64, "bf16", 405)
    a = S.Acsr(cfg.pattern, device=DEV)
    qt_ptr, _, _ = a.plan_copy()
    assert int(qt_ptr[1] - qt_ptr[0]) > 32
    q, k, v = make_qkv(cfg)
    Of = torch.empty_like(dev(q))
    S.splat_sparse_mhsa(a, dev(q), dev(k), dev(v), Of, cfg.scale)
    torch.cuda.synchronize()
    shp = (cfg.BH, cfg.N, cfg.d)
    for bh in range(cfg.BH):
        ref = O.attention(cfg.pattern, q.view(shp)[bh], k.view(shp)[bh], v.view(shp)[bh], cfg.scale)
        assert maxabs(Of.view(shp)[bh].float().cpu(), ref) <= TOL_BF16


@pytest.mark.parametrize("N,d,BH", [(5, 3, 2), (7, 5, 13), (31, 6, 17)])
def test_host_path_fp32_unaligned_slices(N, d, BH):
    # N*d*4 bytes per slice is not a multiple of 16: chunk boundaries must stay 16-byte aligned
    cfg = Config(f"host_fp32_{N}_{d}", Pattern("window", N, lo=1, hi=2), 1, BH, d, "fp32", 406)
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
    shp = (cfg.BH, N, d)
    ref = O.attention(cfg.pattern, q.view(shp)[BH - 1], k.view(shp)[BH - 1], v.view(shp)[BH - 1], cfg.scale)
    assert maxabs(oh.view(shp)[BH - 1], ref) <= TOL_FP32
