"""R-SDDMM wait profile (SPLAT_UNF_PROF build): per warp of CTA 0, cycles in each barrier wait."""
import ctypes as C
import os

os.environ.setdefault("SPLAT_LIB", "diag")     # profiling hooks live in libsplat_diag.so
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_16847_b200 import splat as S
from workloads import CONFIG_BY_NAME, make_tensor

cfg = CONFIG_BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "longformer"]
nbh = cfg.B * cfg.H
a = S.Acsr(cfg.pattern)
Q, K = (make_tensor(cfg.index, t, 1, 1, cfg.N, cfg.d, cfg.torch_dtype, range(nbh)).view(1, nbh, cfg.N, cfg.d).cuda()
        for t in (0, 1))
Sb = torch.empty(nbh * a.nnz, dtype=torch.float32, device="cuda")
L = S.lib()
buf = (C.c_ulonglong * (32 * 8))()
for it in range(3):
    S.splat_rsddmm(a, Q, K, Sb, cfg.scale)
    torch.cuda.synchronize()
    L.splat_debug_unf_prof(buf)
names = ["q_empty(prod)", "k_empty(prod)", "q_full(mma)", "k_full(mma)", "s_empty(mma)", "s_full(epi)", "-", "total"]
for w in range(18):
    row = [buf[w * 8 + k] for k in range(8)]
    tot = row[7]
    if not tot:
        continue
    print(f"warp {w:2d} total {tot:9d} " + " ".join(f"{names[k]}={100 * row[k] / tot:5.1f}%" for k in range(6) if row[k]))
