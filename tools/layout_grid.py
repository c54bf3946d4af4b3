"""Fig. 15 analogue (PAPER "Data-Layout Exploration" P:863-874): R-SpMM with
row-compressed & row-major P against transpose + R-SpMM with column-compressed & column-major P,
over the paper's density grid of the window pattern at N = 1024 (radius 2^k and 1023 =
dense), B = 8, H = 16, d = 64.

Two precisions: fp32 (the paper's: both R-SpMMs are SIMT kernels -- row layout: a warp per
row, lanes over d; column layout: a warp per 32 rows, lane = row, one coalesced load per column) and
bf16 (the tensor-core row-layout R-SpMM of the bench path against transpose + the SIMT column
kernel).  Per point: launch times with L2 flushed before each launch (CUDA events on the launching
stream), the transpose time separately, the two outputs' max difference, and the layout the
density classification (alpha = 0.10) picks.  Summary: geomean speedup of the column layout
(transpose included, as in the paper's figure) for density < 10 % and >= 10 %.

    python tools/layout_grid.py [--iters 20] [--out profiles/r02_layout_grid.json]
"""
import argparse
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import Pattern  # noqa: E402

N, B, H, D = 1024, 8, 16, 64


def timer(stream, flush, iters):
    def run(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        tot = 0.0
        for i in range(iters):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        return tot / iters
    return run


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_layout_grid.json"))
    a = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    run = timer(stream, flush, a.iters)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    points = []
    for r in (2, 4, 8, 16, 32, 64, 128, 256, 512, 1023):
        p = Pattern("window", N, lo=r, hi=r)
        acsr = S.Acsr(p)
        at = S.splat_acsr_transpose(acsr)
        for dt in ("fp32", "bf16"):
            dtype = torch.float32 if dt == "fp32" else torch.bfloat16
            V = (torch.rand(B, H, N, D, generator=g, device="cuda") * 2 - 1).to(dtype)
            P = torch.rand(B * H * acsr.nnz, generator=g, device="cuda").to(dtype)
            PT = torch.empty_like(P)
            Or, Oc = torch.empty_like(V), torch.empty_like(V)
            t_row = run(lambda: S.splat_rspmm(acsr, P, V, Or))
            t_tr = run(lambda: S.splat_transpose_values(acsr, at, P, PT, B, H))
            t_cc = run(lambda: S.splat_rspmm_cc(acsr, at, PT, V, Oc))
            torch.cuda.synchronize()
            diff = (Or.float() - Oc.float()).abs().max().item()
            pt = {"pattern": "window", "radius": r, "density": acsr.density, "dtype": dt,
                  "row_ms": t_row, "transpose_ms": t_tr, "col_ms": t_cc, "col_total_ms": t_tr + t_cc,
                  "speedup_col_total_vs_row": t_row / (t_tr + t_cc), "speedup_col_kernel_vs_row": t_row / t_cc,
                  "max_abs_diff": diff, "alpha_choice": "column" if S.splat_layout_choice(acsr) else "row"}
            points.append(pt)
            print(json.dumps(pt), flush=True)
    summary = {}
    for dt in ("fp32", "bf16"):
        for name, sel in (("sparse_lt_10pct", lambda x: x < 0.10), ("dense_ge_10pct", lambda x: x >= 0.10)):
            sp = [q["speedup_col_total_vs_row"] for q in points if q["dtype"] == dt and sel(q["density"])]
            summary[f"{dt}_{name}_geomean_col_over_row"] = math.exp(sum(map(math.log, sp)) / len(sp))
    doc = {"what": "Fig. 15 analogue: row-compressed vs column-compressed P for R-SpMM (window, N=1024)",
           "B": B, "H": H, "d": D, "iters": a.iters, "points": points, "summary": summary,
           "paper": "column layout: 1.6x geomean for density >= 10%, row layout 1.37x for < 10% (A100, FP32)"}
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
