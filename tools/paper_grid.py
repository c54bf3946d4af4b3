"""Paper-grid microbenchmarks (a Fig. 9 / Fig. 10 analogue on B200).

The paper's density grid [0.4, 0.8, 1.6, 3, 6, 12, 24, 44, 75, 100] % at N = 1024 over
its three patterns, tuned by "the width of the stride, the size of the window, or the size of the
block": window radius r = 2^k (2..512, plus 1023 = dense), block w = 2^k (4..1024),
stride X = 2^k (256..1); SURVEY's derived reading of the grid.  B, H and d are not stated
(SURVEY E-table): B = 8, H = 16, d = 64, bf16 inputs, fp32 accumulation (our path; the paper's
numbers are FP32 on an A100).

Per point: R-SDDMM, softmax and R-SpMM launch times (the unfused primitives, Fig. 9) and the
fused sparse MHSA (Fig. 10), CUDA events on the launching stream with L2 flushed before every
launch; dense context = torch SDPA (bf16, flash) on the same Q, K, V and torch.matmul QK^T.
Each point also checks the fused output of one (b, h) slice against the fp64 oracle (max abs
error, bf16 tolerance 2e-2).  Writes one JSON document (default profiles/r01h_paper_grid.json).

    python tools/paper_grid.py [--iters 20] [--out FILE]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402  (parity check of each point only)
from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import Pattern, make_random  # noqa: E402

N, B, H, D = 1024, 8, 16, 64


def grid():
    for r in (2, 4, 8, 16, 32, 64, 128, 256, 512, 1023):
        yield "window", r, Pattern("window", N, lo=r, hi=r)
    for w in (4, 8, 16, 32, 64, 128, 256, 512, 1024):
        yield "blocked", w, Pattern("blocked", N, block=w)
    for X in (256, 128, 64, 32, 16, 8, 4, 2, 1):
        yield "strided", X, Pattern("strided", N, stride=X)


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
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01h_paper_grid.json"))
    ap.add_argument("--ablate", type=int, default=0,
                    help="span-specialisation ablation (SPLAT_PLAN_ABLATE): 1 = no FULL tiles / chunks, "
                         "2 = also no span (every key tile, every chunk)")
    ap.add_argument("--patterns", default="window,blocked,strided")
    a = ap.parse_args()
    if a.ablate:
        os.environ["SPLAT_PLAN_ABLATE"] = str(a.ablate)
        os.environ["SPLAT_LIB"] = "diag"          # the ablation knob exists only in libsplat_diag.so
    dev = 0
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    run = timer(stream, flush, a.iters)
    scale = 1.0 / np.sqrt(D)
    Q, K, V = (make_random((B, H, N, D), seed=11 + t).to(torch.bfloat16).to(dev) for t in range(3))
    O_ = torch.empty_like(Q)
    dense_ms = run(lambda: torch.nn.functional.scaled_dot_product_attention(Q, K, V, scale=scale))
    mm_ms = run(lambda: torch.matmul(Q, K.transpose(-1, -2)))
    doc = {"N": N, "B": B, "H": H, "d": D, "dtype": "bf16", "iters": a.iters, "ablate": a.ablate,
           "dense_sdpa_ms": dense_ms, "dense_qkT_matmul_ms": mm_ms, "points": []}
    print(f"dense SDPA {dense_ms * 1e3:.1f} us, QK^T matmul {mm_ms * 1e3:.1f} us")
    for kind, param, p in grid():
        if kind not in a.patterns.split(","):
            continue
        h = S.Acsr(p, device=dev)
        nnz = h.nnz
        Sb = torch.empty(B * H * nnz, dtype=torch.float32, device=dev)
        Pb = torch.empty(B * H * nnz, dtype=torch.bfloat16, device=dev)
        t = {
            "rsddmm": run(lambda: S.splat_rsddmm(h, Q, K, Sb, scale, stream)),
            "softmax": run(lambda: S.splat_sparse_softmax(h, Sb, Pb, B, H, stream)),
            "rspmm": run(lambda: S.splat_rspmm(h, Pb, V, O_, stream)),
            "fused": run(lambda: S.splat_sparse_mhsa(h, Q, K, V, O_, scale, stream)),
        }
        torch.cuda.synchronize()
        want = O.attention(p, Q[0, 0].double().cpu().numpy(), K[0, 0].double().cpu().numpy(),
                           V[0, 0].double().cpu().numpy(), scale)
        err = float(np.max(np.abs(O_[0, 0].float().cpu().numpy() - want)))
        fl = 4.0 * nnz * D * B * H
        pt = {"pattern": kind, "param": param, "density_pct": 100.0 * nnz / N / N,
              "ms": t, "fused_tflops": fl / (t["fused"] * 1e-3) / 1e12,
              "unfused_total_ms": t["rsddmm"] + t["softmax"] + t["rspmm"],
              "fused_vs_sdpa": dense_ms / t["fused"], "max_abs_err_vs_oracle": err}
        doc["points"].append(pt)
        print(f"{kind:8s} {param:5d} {pt['density_pct']:7.2f}%  sddmm {t['rsddmm'] * 1e3:8.1f}  "
              f"softmax {t['softmax'] * 1e3:8.1f}  spmm {t['rspmm'] * 1e3:8.1f}  fused {t['fused'] * 1e3:7.1f} us "
              f"({pt['fused_tflops']:6.1f} TF/s, {pt['fused_vs_sdpa']:5.2f}x SDPA)  err {err:.1e}", flush=True)
        assert err < 2e-2, (kind, param, err)
        del Sb, Pb
        h.destroy()
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
