"""Debug aid: pipeline timeline of CTA 0 of the fused kernel (SPLAT_TC_DEBUG=4)."""
import ctypes as C
import os

os.environ.setdefault("SPLAT_LIB", "diag")     # profiling hooks live in libsplat_diag.so
import sys

os.environ["SPLAT_TC_DEBUG"] = str(4 | int(os.environ.get("SPLAT_TC_DEBUG_EXTRA", "0")))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2407_16847_b200 import splat as S
from workloads import CONFIG_BY_NAME, make_qkv

cfg = CONFIG_BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "longformer"]
q, k, v = make_qkv(cfg)
Q, K, V = q.cuda(), k.cuda(), v.cuda()
O = torch.empty_like(Q)
a = S.Acsr(cfg.pattern)
L = S.lib()
buf = (C.c_ulonglong * (6 * 2048))()
cnt = (C.c_int * 6)()
for it in range(3):
    S.splat_sparse_mhsa(a, Q, K, V, O, cfg.scale)
    torch.cuda.synchronize()
    L.splat_debug_trace(buf, cnt)
arr = np.frombuffer(buf, dtype=np.uint64).reshape(6, 2048)
names = {0: "producer", 1: "mmaA", 2: "softmaxA", 3: "softmaxB", 4: "mmaB", 5: "vprod"}
t0 = min(int(arr[r][0] & 0xffffffffffff) for r in range(6) if cnt[r] > 0)
for r in range(6):
    n = min(cnt[r], 2048)
    ev = [(int(x >> 48), int(x & 0xffffffffffff) - t0) for x in arr[r][:n]]
    print(names[r], "events", cnt[r])
    print("  ", " ".join(f"{tag}@{t}" for tag, t in ev))
