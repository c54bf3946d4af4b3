"""R-SDDMM wait profile (SPLAT_UNF_PROF diagnostics build): per warp of CTA 0, cycles in each barrier
wait, plus a span of the epilogue's per-tile metadata phase (mask / row-offset loads, publish)."""
import ctypes as C
import os

os.environ.setdefault("SPLAT_LIB", "diag")
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_16847_b200 import splat as S
from workloads import CONFIG_BY_NAME, make_tensor

cfg = CONFIG_BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "longformer"]
nbh = cfg.B * cfg.H
a = S.Acsr(cfg.pattern)
Q = make_tensor(cfg.index, 0, 1, 1, cfg.N, cfg.d, cfg.torch_dtype, range(nbh)).view(1, nbh, cfg.N, cfg.d).cuda()
K = make_tensor(cfg.index, 1, 1, 1, cfg.N, cfg.d, cfg.torch_dtype, range(nbh)).view(1, nbh, cfg.N, cfg.d).cuda()
Sd = torch.empty(nbh * a.nnz, device="cuda")
L = S.lib()
buf = (C.c_ulonglong * (32 * 8))()
for it in range(3):
    S.splat_rsddmm(a, Q, K, Sd, cfg.scale)
    torch.cuda.synchronize()
    L.splat_debug_unf_prof(buf)
roles = {0: "Q/K TMA", 1: "MMA"}
names = ["q_empty", "k_empty", "q_full", "k_full", "s_empty", "s_full", "meta", "total"]
for w in range(18):
    row = [buf[w * 8 + k] for k in range(8)]
    tot = row[7]
    if not tot:
        continue
    print(f"warp {w:2d} {roles.get(w, 'epilogue'):9s} total {tot:9d} " +
          " ".join(f"{names[k]}={100 * row[k] / tot:5.1f}%" for k in range(7) if row[k]))
