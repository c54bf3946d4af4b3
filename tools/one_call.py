"""Debug aid: time a single fused call of a config (with a watchdog-friendly structure)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_16847_b200 import splat as S
from workloads import CONFIG_BY_NAME, make_qkv
cfg = CONFIG_BY_NAME[sys.argv[1]]
BHs = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.BH
q, k, v = make_qkv(cfg, bh_range=range(BHs))
Q, K, V = q.cuda()[None], k.cuda()[None], v.cuda()[None]
O = torch.empty_like(Q)
a = S.Acsr(cfg.pattern)
for i in range(3):
    t = time.time()
    S.splat_sparse_mhsa(a, Q, K, V, O, cfg.scale)
    torch.cuda.synchronize()
    print(cfg.name, BHs, "call", i, f"{(time.time()-t)*1e3:.3f} ms", flush=True)
