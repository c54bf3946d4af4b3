"""Debug aid: per-(bh, row) error map of the fused kernel vs the oracle for one small case."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import oracle as O
from paper_2407_16847_b200 import splat as S
from workloads import Pattern, make_random

p = Pattern("window", int(sys.argv[1]), lo=int(sys.argv[2]), hi=int(sys.argv[2]))
d = int(sys.argv[3])
N, BH = p.seq_len, 3
q, k, v = (make_random((1, BH, N, d), 500 + t, torch.bfloat16) for t in range(3))
a = S.Acsr(p, device=0)
Od = torch.empty(1, BH, N, d, dtype=torch.bfloat16, device="cuda")
S.splat_sparse_mhsa(a, q.cuda(), k.cuda(), v.cuda(), Od, 0.125)
torch.cuda.synchronize()
for bh in range(BH):
    ref = O.attention(p, q[0, bh], k[0, bh], v[0, bh], 0.125)
    err = np.abs(Od[0, bh].float().cpu().numpy() - ref).max(axis=1)
    bad = np.nonzero(err > 2e-2)[0]
    print("bh", bh, "max", err.max(), "bad rows", len(bad), bad[:10], bad[-10:] if len(bad) else "")
