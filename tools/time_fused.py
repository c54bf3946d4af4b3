"""Time the fused call of a config with the library selected by SPLAT_LIB (diagnostics builds):
    SPLAT_LIB=diag python tools/time_fused.py <config> [steps]
L2 flushed before each call, CUDA events; prints TFLOP/s and us per call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import CONFIG_BY_NAME  # noqa: E402

cfg = CONFIG_BY_NAME[sys.argv[1]]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = torch.Generator(device="cuda")
g.manual_seed(5)
Q, K, V = ((torch.rand(cfg.B, cfg.H, cfg.N, cfg.d, generator=g, device="cuda") * 2 - 1).to(cfg.torch_dtype)
           for _ in range(3))
O = torch.empty_like(Q)
a = S.Acsr(cfg.pattern)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(3):
    S.splat_sparse_mhsa(a, Q, K, V, O, cfg.scale)
torch.cuda.synchronize()
ts = []
for i in range(steps):
    flush.fill_(float(i))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S.splat_sparse_mhsa(a, Q, K, V, O, cfg.scale)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = sorted(ts)[len(ts) // 2]
print(f"{cfg.name} {os.environ.get('TAGV', '')} {a.flops(cfg.B, cfg.H, cfg.d) / ms / 1e9:.1f} TFLOP/s {ms * 1e3:.1f} us (median)")
