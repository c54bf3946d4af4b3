"""The C-ABI contract of SURVEY §8(b) on the GPU: compute calls never allocate, and one handle is
safe on concurrent streams (per-call launch slots, event-ordered reuse; include/splat.h)."""
import pytest
import torch

from paper_2407_16847_b200 import splat as S
from workloads import Config, Pattern, make_qkv

pytestmark = pytest.mark.gpu
DEV = 0

CASES = [
    # d = 64 split kernel (dynamic work counter of the launch slot)
    Config("lf_small", Pattern("global_local", 1024, lo=128, hi=128, n_global=16), 2, 4, 64, "bf16", 501),
    # residue decomposition (lse scratch of the launch slot) -- Sparse-TF shape at small N
    Config("st_small", Pattern("strided_local", 2048, stride=32, causal=1), 1, 3, 128, "bf16", 502),
    # plain STRIDED on the permuted handle
    Config("str_perm", Pattern("strided", 1024, stride=16), 1, 2, 64, "bf16", 503),
    # fp32 SIMT path
    Config("fp32", Pattern("window", 256, lo=32, hi=32), 1, 2, 64, "fp32", 504),
]


@pytest.fixture(scope="module", autouse=True)
def gpu():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    torch.cuda.set_device(DEV)


def dev(x):
    return x.to(f"cuda:{DEV}").contiguous()


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: c.name)
def test_compute_calls_never_allocate(cfg):
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern, device=DEV)
    Q, K, V = dev(q), dev(k), dev(v)
    B, H = cfg.B, cfg.H
    Sd = torch.empty(B * H * a.nnz, dtype=torch.float32, device=Q.device)
    Pd = torch.empty(B * H * a.nnz, dtype=cfg.torch_dtype, device=Q.device)
    Od = torch.empty_like(Q)
    qh, kh, vh = (x.contiguous().pin_memory() for x in (q, k, v))
    oh = torch.empty_like(qh).pin_memory()
    dQ, dK, dV, dO = (torch.empty_like(Q) for _ in range(4))
    torch.cuda.synchronize()
    before = S.device_alloc_count()
    for _ in range(3):
        S.splat_rsddmm(a, Q, K, Sd, cfg.scale)
        S.splat_sparse_softmax(a, Sd, Pd, B, H)
        S.splat_rspmm(a, Pd, V, Od)
        S.splat_sparse_mhsa(a, Q, K, V, Od, cfg.scale)
        S.splat_sparse_mhsa_host(a, qh, kh, vh, oh, cfg.scale, dQ, dK, dV, dO)
    torch.cuda.synchronize()
    assert S.device_alloc_count() == before
    # and a new handle does allocate (the counter is live)
    b = S.Acsr(cfg.pattern, device=DEV)
    assert S.device_alloc_count() > before
    b.destroy()
    a.destroy()


@pytest.mark.parametrize("cfg", CASES[:3], ids=lambda c: c.name)
def test_one_handle_on_concurrent_streams(cfg):
    # two streams share one handle, each with its own inputs, many calls in flight at once: every
    # result equals the same call made alone (bitwise -- same kernels, no atomics on the data)
    a = S.Acsr(cfg.pattern, device=DEV)
    ins = []
    for s in range(2):
        q, k, v = make_qkv(Config(cfg.name, cfg.pattern, cfg.B, cfg.H, cfg.d, cfg.dtype, cfg.index + 10 * s))
        ins.append((dev(q), dev(k), dev(v)))
    ref = []
    for Q, K, V in ins:
        O = torch.empty_like(Q)
        S.splat_sparse_mhsa(a, Q, K, V, O, cfg.scale)
        ref.append(O)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(device=DEV) for _ in range(2)]
    outs = [[torch.empty_like(ins[s][0]) for _ in range(12)] for s in range(2)]
    torch.cuda.synchronize()
    for it in range(12):
        for s in range(2):
            with torch.cuda.stream(streams[s]):
                S.splat_sparse_mhsa(a, *ins[s], outs[s][it], cfg.scale, streams[s])
    torch.cuda.synchronize()
    for s in range(2):
        for it in range(12):
            assert torch.equal(outs[s][it], ref[s]), (s, it)
    a.destroy()
