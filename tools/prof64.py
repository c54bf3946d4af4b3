"""Per-phase cycle breakdown of the d = 64 fused kernel (diagnostics build with -DSPLAT_FUSED_PROF):
    SPLAT_EXTRA_NVCC_FLAGS=-DSPLAT_FUSED_PROF python -m paper_2407_16847_b200.build --diag
    python tools/prof64.py [config]
Prints, per role, the share of each phase in the warps' cycles (summed over all CTAs)."""
import ctypes as C
import os
import sys

os.environ.setdefault("SPLAT_LIB", "diag")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import CONFIG_BY_NAME, make_qkv  # noqa: E402

cfg = CONFIG_BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "longformer"]
q, k, v = make_qkv(cfg)
Q, K, V = q.cuda(), k.cuda(), v.cuda()
O = torch.empty_like(Q)
a = S.Acsr(cfg.pattern)
L = S.lib()
buf = (C.c_ulonglong * (20 * 16))()
for it in range(3):
    L.splat_debug_prof64(buf)
    S.splat_sparse_mhsa(a, Q, K, V, O, cfg.scale)
    torch.cuda.synchronize()
L.splat_debug_prof64(buf)
names = {
    "producer": {1: "m_empty wait", 2: "k_empty wait", 3: "v_empty wait", 0: "work"},
    "mma": {1: "k_full wait", 2: "s_empty wait", 3: "o_empty wait", 4: "p_full wait", 5: "v_full wait", 0: "work"},
    "softmax": {11: "metadata (m_full)", 0: "meta->s_full", 1: "s_full wait", 2: "S ld+wait", 3: "mask+max",
                4: "max exchange", 5: "bump+exps", 6: "epilogue", 7: "pv_done wait", 8: "O rescale", 9: "P st+arrive"},
}
for w in range(int(os.environ.get("NWARPS", "12"))):
    row = [buf[w * 16 + k] for k in range(16)]
    tot = row[15]
    if not tot:
        continue
    role = os.environ.get("ROLES", "p,m").split(",")[w] if w < len(os.environ.get("ROLES", "p,m").split(",")) else "s"
    role = {"p": "producer", "m": "mma", "s": "softmax"}[role]
    parts = ", ".join(f"{n}={100 * row[k] / tot:.1f}%" for k, n in names[role].items() if row[k])
    print(f"warp {w:2d} {role:8s} total {tot / 1e6:8.1f} Mcyc: {parts}")
