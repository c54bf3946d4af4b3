"""R-SpMM wait profile (SPLAT_UNF_PROF build): per warp of CTA 0, cycles in each barrier wait."""
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
V = make_tensor(cfg.index, 2, 1, 1, cfg.N, cfg.d, cfg.torch_dtype, range(nbh)).view(1, nbh, cfg.N, cfg.d).cuda()
P = torch.rand(nbh * a.nnz, device="cuda").to(torch.bfloat16)
O = torch.empty_like(V)
L = S.lib()
buf = (C.c_ulonglong * (32 * 8))()
for it in range(3):
    S.splat_rspmm(a, P, V, O)
    torch.cuda.synchronize()
    L.splat_debug_unf_prof(buf)
# wait sites of rspmm_tc_kernel by role (warp -> role); slot 7 = warp total
roles = {0: "V TMA", 1: "MMA", 4: "epilogue", 5: "epilogue", 6: "epilogue", 7: "epilogue"}
roles.update({w: "P producer" for w in range(8, 16)})
roles.update({w: "expander" for w in range(16, 24)})
names = ["v_empty", "o_empty", "v_full", "p_full|exp-rows|prod-unit", "stg_empty|exp-fence", "stg_full|prod-copy", "p_empty/o_full", "total"]
for w in range(24):
    row = [buf[w * 8 + k] for k in range(8)]
    tot = row[7]
    if not tot:
        continue
    print(f"warp {w:2d} {roles.get(w, '-'):10s} total {tot:9d} " +
          " ".join(f"{names[k]}={100 * row[k] / tot:5.1f}%" for k in range(7) if row[k]))
