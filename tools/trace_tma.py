"""TMA latency from a split-kernel trace: j-th K issue (producer tag 31) -> j-th k_full seen (MMA tag 11)."""
import sys
lines = open(sys.argv[1]).read().splitlines()
ev = {}
for i in range(0, len(lines) - 1, 2):
    ev[lines[i].split()[0]] = [tuple(map(int, e.split("@"))) for e in lines[i + 1].split()]
iss = [c for t, c in ev["producer"] if t == 31]
seen = [c for t, c in ev["mmaA"] if t == 11]
lat = [b - a for a, b in zip(iss, seen)]
lat.sort()
n = len(lat)
print("K loads", n, "latency issue->k_full seen: min", lat[0], "median", lat[n // 2], "p90", lat[int(n * 0.9)], "max", lat[-1])
