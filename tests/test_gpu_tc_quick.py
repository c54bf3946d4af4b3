"""Quick GPU checks of the tcgen05 fused kernel on small shapes (one tile, a
few tiles, ragged) -- run first when iterating on the kernel."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2407_16847_b200 import splat as S
from workloads import Pattern, make_random

pytestmark = pytest.mark.gpu

CASES = [
    (Pattern("window", 128, lo=128, hi=128), 64),        # one full tile
    (Pattern("window", 128, lo=5, hi=9), 64),            # one partial tile
    (Pattern("window", 256, lo=256, hi=256), 64),        # 2x2 full tiles (multi-tile accumulate)
    (Pattern("window", 128, lo=128, hi=128), 128),
    (Pattern("window", 300, lo=40, hi=40), 128),          # ragged
    (Pattern("strided", 384, stride=5), 64),             # strided partial tiles
    (Pattern("global_local", 640, lo=64, hi=64, n_global=8), 64),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0].kind}-{c[0].seq_len}-d{c[1]}")
def test_tc_small(case):
    p, d = case
    N, BH = p.seq_len, 3
    q, k, v = (make_random((1, BH, N, d), 500 + t, torch.bfloat16) for t in range(3))
    a = S.Acsr(p, device=0)
    Od = torch.empty(1, BH, N, d, dtype=torch.bfloat16, device="cuda")
    S.splat_sparse_mhsa(a, q.cuda(), k.cuda(), v.cuda(), Od, 0.125)
    torch.cuda.synchronize()
    for bh in range(BH):
        ref = O.attention(p, q[0, bh], k[0, bh], v[0, bh], 0.125)
        err = np.max(np.abs(Od[0, bh].float().cpu().numpy() - ref))
        assert err <= 2e-2, (bh, err)
