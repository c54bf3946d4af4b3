"""Per-rank time of the (b, h)-sharded strong-scaling split on ONE GPU: the fused call on B*H/G heads of
a config (what each of G ranks runs, §8(e)), L2 flushed, CUDA events, median.  Predicts the
strong-scaling efficiency t(1) / (G * t(G)) without a multi-GPU box (no inter-rank term: the data
path has no collective)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import CONFIG_BY_NAME  # noqa: E402

cfg = CONFIG_BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "longformer"]
BH = cfg.B * cfg.H
a = S.Acsr(cfg.pattern)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
res = {}
for G in (1, 2, 4, 8):
    nbh = BH // G
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    Q, K, V = ((torch.rand(1, nbh, cfg.N, cfg.d, generator=g, device="cuda") * 2 - 1).to(cfg.torch_dtype) for _ in range(3))
    O = torch.empty_like(Q)
    for _ in range(3):
        S.splat_sparse_mhsa(a, Q, K, V, O, cfg.scale)
    ts = []
    for i in range(20):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        S.splat_sparse_mhsa(a, Q, K, V, O, cfg.scale)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[G] = sorted(ts)[len(ts) // 2] * 1e3
out = {"config": cfg.name, "bh_total": BH, "us_per_rank": {G: round(t, 1) for G, t in res.items()},
       "predicted_strong_efficiency": {G: round(res[1] / (G * res[G]), 3) for G in res}}
print(json.dumps(out))
