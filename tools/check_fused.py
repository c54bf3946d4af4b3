"""Parity spot-check of the fused call with the library selected by SPLAT_LIB (diagnostics builds):
    SPLAT_LIB=diag SPLAT_TC_PAIRED64=3 python tools/check_fused.py
Compares a few configurations against the fp64 oracle (max-abs error, bf16 bar 2e-2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import CONFIG_BY_NAME, Config, Pattern, make_qkv  # noqa: E402

cases = [
    Config("gl_small", Pattern("global_local", 1500, lo=100, hi=60, n_global=16), 2, 3, 64, "bf16", 701),
    Config("bb_small", Pattern("bigbird", 1024, block=64, radius=1), 1, 4, 64, "bf16", 702),
    Config("win_ragged", Pattern("window", 777, lo=100, hi=37), 1, 2, 64, "bf16", 703),
    Config("many_heads", Pattern("window", 256, lo=16, hi=16), 8, 40, 64, "bf16", 704),
    Config("gl6000", Pattern("global_local", 6000, lo=64, hi=64, n_global=32), 1, 2, 64, "bf16", 705),
]
worst_all = 0.0
for cfg in cases + [CONFIG_BY_NAME["longformer"], CONFIG_BY_NAME["bigbird"]]:
    q, k, v = make_qkv(cfg)
    a = S.Acsr(cfg.pattern)
    Q, K, V = q.cuda(), k.cuda(), v.cuda()
    Of = torch.empty_like(Q)
    S.splat_sparse_mhsa(a, Q, K, V, Of, cfg.scale)
    torch.cuda.synchronize()
    shp = (cfg.BH, cfg.N, cfg.d)
    Of = Of.view(shp).float().cpu()
    heads = range(cfg.BH) if cfg.BH <= 12 else [0, 1, cfg.BH // 2, cfg.BH - 1]
    worst = 0.0
    for bh in heads:
        ref = O.attention(cfg.pattern, q.view(shp)[bh], k.view(shp)[bh], v.view(shp)[bh], cfg.scale)
        worst = max(worst, float(np.max(np.abs(Of[bh].numpy() - ref))))
    worst_all = max(worst_all, worst)
    print(f"{cfg.name:12s} max-abs {worst:.2e} {'OK' if worst <= 2e-2 else 'FAIL'}", flush=True)
print("ALL OK" if worst_all <= 2e-2 else "FAILED")
