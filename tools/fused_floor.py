"""Fused-kernel small-problem floor: time vs number of work units at N = 1024 (d = 64, bf16),
blocked-4 / blocked-128 / window-64, B*H from 8 to 2048 (CUDA events, L2 flushed before each
launch).  Separates the fixed cost of a launch from the steady per-unit cost.

    python tools/fused_floor.py
"""
import sys, torch
sys.path.insert(0, '.')
from paper_2407_16847_b200 import splat as S
from workloads import Pattern, make_random
N, D = 1024, 64
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=0)
for kind, p in (("blocked4", Pattern("blocked", N, block=4)), ("blocked128", Pattern("blocked", N, block=128)), ("window64", Pattern("window", N, lo=64, hi=64))):
    h = S.Acsr(p, device=0)
    for BH in (8, 32, 128, 512, 2048):
        Q, K, V = (make_random((1, BH, N, D), seed=t).to(torch.bfloat16).cuda() for t in range(3))
        O = torch.empty_like(Q)
        for _ in range(3): S.splat_sparse_mhsa(h, Q, K, V, O, 0.125, st)
        torch.cuda.synchronize()
        ts = []
        for i in range(10):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); S.splat_sparse_mhsa(h, Q, K, V, O, 0.125, st); e1.record(st); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(kind, BH, "units", BH * 8, "us %.1f" % ts[5], "us/unit/SM %.2f" % (ts[5] / (BH * 8 / 148)))
