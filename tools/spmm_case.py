"""One R-SpMM call on a config's mask with few heads (for compute-sanitizer):
    python tools/spmm_case.py <config> <bh>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import CONFIG_BY_NAME  # noqa: E402

cfg = CONFIG_BY_NAME[sys.argv[1]]
bh = int(sys.argv[2])
a = S.Acsr(cfg.pattern)
V = torch.rand(1, bh, cfg.N, cfg.d, device="cuda").to(cfg.torch_dtype)
P = torch.rand(bh * a.nnz, device="cuda").to(cfg.torch_dtype)
O = torch.empty_like(V)
S.splat_rspmm(a, P, V, O)
torch.cuda.synchronize()
print("ok", O.float().abs().sum().item())
