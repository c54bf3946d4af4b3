"""Summarise a tools/trace.py dump: per role, mean gap between consecutive tag pairs."""
import sys
from collections import defaultdict
lines = open(sys.argv[1]).read().splitlines()
for i in range(0, len(lines) - 1, 2):
    name = lines[i].split()[0]
    evs = [tuple(map(int, e.split("@"))) for e in lines[i + 1].split()]
    gaps = defaultdict(list)
    for (t0, c0), (t1, c1) in zip(evs, evs[1:]):
        gaps[(t0, t1)].append(c1 - c0)
    print(name, "events", len(evs), "span", evs[-1][1] - evs[0][1] if evs else 0)
    for k, v in sorted(gaps.items(), key=lambda x: -sum(x[1]))[:12]:
        print(f"   {k[0]:>2}->{k[1]:<2} n={len(v):4d} mean={sum(v)/len(v):8.1f} total={sum(v)}")
