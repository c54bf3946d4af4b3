"""Split-kernel wait profile (SPLAT_FUSED_PROF build): per warp of CTA 0, % of cycles per wait site."""
import ctypes as C
import os

os.environ.setdefault("SPLAT_LIB", "diag")     # profiling hooks live in libsplat_diag.so
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_16847_b200 import splat as S
from workloads import CONFIG_BY_NAME, make_qkv

cfg = CONFIG_BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "longformer"]
q, k, v = make_qkv(cfg)
Q, K, V = q.cuda(), k.cuda(), v.cuda()
O = torch.empty_like(Q)
a = S.Acsr(cfg.pattern)
L = S.lib()
buf = (C.c_ulonglong * (12 * 16))()
for it in range(3):
    S.splat_sparse_mhsa(a, Q, K, V, O, cfg.scale)
    torch.cuda.synchronize()
    L.splat_debug_fused_prof(buf)
names = {0: "s_full", 1: "pv_done", 2: "epi", 3: "q_full", 4: "k_full", 5: "s_empty", 6: "p_full", 7: "v_full",
         8: "q_empty", 9: "k_empty", 10: "v_empty", 11: "q_full(mma)"}
for w in range(12):
    row = [buf[w * 16 + k] for k in range(16)]
    tot = row[15]
    if not tot:
        continue
    print(f"warp {w:2d} total {tot:9d} " + " ".join(f"{names[k]}={100 * row[k] / tot:4.1f}%" for k in range(12) if row[k]))
