"""Per-region stall summary of an ncu --page source --csv --print-source sass dump.

    python tools/sass_regions.py src.csv
Groups instructions by execution count (a proxy for the loop / role an instruction
belongs to) and prints each group's share of the warp-stall samples and top reasons.
"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
ia, isrc = h.index("Address"), h.index("Source")
iss, iex = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = {c: h.index(c) for c in reasons}
tot = sum(int(r[iss]) for r in data)
print("total samples", tot)
byex = defaultdict(lambda: [0, Counter(), 0, None])
for k, r in enumerate(data):
    e = int(r[iex] or 0)
    b = byex[e]
    b[0] += int(r[iss])
    b[2] += 1
    if b[3] is None:
        b[3] = r[ia][-5:]
    for c in reasons:
        b[1][c] += int(r[ri[c]] or 0)
for e, (s, c, n, a0) in sorted(byex.items(), key=lambda x: -x[1][0])[:25]:
    print(f"exec={e:8d} ninstr={n:4d} first={a0} samples={s:6d} ({100*s/tot:4.1f}%)",
          ", ".join(f"{k[6:]}={v}" for k, v in c.most_common(4)))
