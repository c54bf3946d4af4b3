"""Fig. 12 analogue: thread blocks used by poset tiling vs the naive tiling at N = 1024,
over every density of the window (radius r = 0..N-1) and block-diagonal (w | N) masks, through the
library's host tiling analysis (splat_poset_tile / splat_naive_tile).  Also counts, for the bench
configurations (N <= 8192), the 128 x 128 tcgen05 tiles our planner issues against poset and naive
tilings with 128 x 128 blocks.  Writes one JSON document (default profiles/r01h_fig12.json).

    python tools/fig12.py [--out FILE] [--shapes 16x16,32x8,...]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import CONFIGS, Pattern  # noqa: E402


def sweep(kind, N, m, n):
    vals = range(N) if kind == "window" else [w for w in range(1, N + 1) if N % w == 0]
    rows = []
    for v in vals:
        p = Pattern("window", N, lo=v, hi=v) if kind == "window" else Pattern("blocked", N, block=v)
        _, cp = S.splat_poset_tile(p, m, n)
        _, cn = S.splat_naive_tile(p, m, n)
        rows.append({"param": v, "density": cp["points"] / N / N, "poset": cp["lambda"], "naive": cn["lambda"]})
    ratios = [r["naive"] / r["poset"] for r in rows]
    k = max(range(len(rows)), key=lambda i: ratios[i])
    return {"kind": kind, "m": m, "n": n, "avg_reduction": sum(ratios) / len(ratios), "max_reduction": ratios[k],
            "max_at": rows[k]["param"], "threads_saved_at_max": (rows[k]["naive"] - rows[k]["poset"]) * m * n,
            "n_worse": sum(1 for x in ratios if x < 1), "points": rows}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01h_fig12.json"))
    ap.add_argument("--shapes", default="16x16,32x32,32x8,8x32,64x16")
    a = ap.parse_args()
    N = 1024
    t0 = time.time()
    doc = {"N": N, "sweeps": [], "bench_configs_128": []}
    for sh in a.shapes.split(","):
        m, n = (int(x) for x in sh.split("x"))
        for kind in ("window", "blocked"):
            r = sweep(kind, N, m, n)
            doc["sweeps"].append(r)
            print(f"{kind:8s} {m:3d}x{n:<3d} avg {r['avg_reduction']:.3f}  max {r['max_reduction']:.3f} "
                  f"(param {r['max_at']}, {r['threads_saved_at_max']} threads)  poset worse at {r['n_worse']}")
    for c in CONFIGS:
        if c.pattern.seq_len > 8192:
            continue
        h = S.Acsr(c.pattern, device=-1)
        bm, bn, nq, ne = h.plan_info()
        _, cp = S.splat_poset_tile(c.pattern, bm, bn)
        _, cn = S.splat_naive_tile(c.pattern, bm, bn)
        row = {"config": c.name, "tile": [bm, bn], "planner_tiles": ne, "poset": cp["lambda"], "poset_stretch": cp["stretch"],
               "naive": cn["lambda"], "nnz": cp["points"]}
        doc["bench_configs_128"].append(row)
        print(f"{c.name:20s} planner {ne:6d}  poset {cp['lambda']:6d} (s={cp['stretch']})  naive {cn['lambda']:6d}")
    doc["seconds"] = time.time() - t0
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
