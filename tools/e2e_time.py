"""e2e time of splat_sparse_mhsa_host (pinned host buffers, copies + kernels), CUDA events, median of 10:
    [SPLAT_LIB=diag ...] python tools/e2e_time.py [config]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import CONFIG_BY_NAME  # noqa: E402

cfg = CONFIG_BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "longformer"]
a = S.Acsr(cfg.pattern)
shp = (cfg.B, cfg.H, cfg.N, cfg.d)
hq, hk, hv = ((torch.rand(shp) * 2 - 1).to(cfg.torch_dtype).pin_memory() for _ in range(3))
ho = torch.empty(shp, dtype=cfg.torch_dtype).pin_memory()
dq, dk, dv, do = (torch.empty(shp, dtype=cfg.torch_dtype, device="cuda") for _ in range(4))
for _ in range(3):
    S.splat_sparse_mhsa_host(a, hq, hk, hv, ho, cfg.scale, dq, dk, dv, do)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S.splat_sparse_mhsa_host(a, hq, hk, hv, ho, cfg.scale, dq, dk, dv, do)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"{cfg.name} {os.environ.get('TAGV', '')} e2e {sorted(ts)[5]:.3f} ms")
