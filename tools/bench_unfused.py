"""Diagnostic timing of the three unfused primitives per config.

Prints one JSON line per config with each kernel's average launch time (CUDA events on the
launching stream, L2 flushed before each launch) and its algorithmic HBM traffic:
  R-SDDMM  : Q + K read (2 N d bytes each per head, bf16) + S written (4 B per non-zero)
  softmax  : S read (4 B / nnz) + P written (2 B / nnz for bf16)
  R-SpMM   : P read (2 B / nnz) + V read + O written (2 N d bytes each per head)
Also the ACSR build + plan wall time (rows a1/a2, once per pattern).
Not part of the bench contract; the fused kernel is the hot path bench.py times.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from workloads import CONFIGS, CONFIG_BY_NAME, make_tensor  # noqa: E402
from paper_2407_16847_b200 import splat as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="longformer,bigbird,sparse_transformer,mistral")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--max-bh", type=int, default=0, help="cap heads (memory); 0 = all")
    args = ap.parse_args()
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        peaks = {"hbm_gbs": 6650.0}     # B200_PROFILING.md fallback
    hbm = None
    for k, v in peaks.items():
        if "hbm" in k.lower() and isinstance(v, (int, float)):
            hbm = v
            break
    dev = 0
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for name in args.configs.split(","):
        cfg = CONFIG_BY_NAME[name]
        nbh = cfg.B * cfg.H
        if cfg.dtype != "bf16":
            continue
        # row a1/a2: ACSR build + tile plan (synchronous, once per pattern): wall time of the call,
        # median of 5 (device kernels + host planner + metadata upload)
        import time
        tb = []
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a = S.Acsr(cfg.pattern, device=dev)
            tb.append(time.perf_counter() - t0)
            a.destroy()
        build_ms = sorted(tb)[2] * 1e3
        a = S.Acsr(cfg.pattern, device=dev)
        # keep S (fp32) under ~60 GB
        cap = max(1, int(60e9 // (a.nnz * 6)))
        if args.max_bh:
            cap = min(cap, args.max_bh)
        nbh = min(nbh, cap)
        bh = range(nbh)
        Q, K, V = (make_tensor(cfg.index, t, 1, 1, cfg.N, cfg.d, cfg.torch_dtype, bh).view(1, nbh, cfg.N, cfg.d).to(dev)
                   for t in (0, 1, 2))
        Sb = torch.empty(nbh * a.nnz, dtype=torch.float32, device=dev)
        Pb = torch.empty(nbh * a.nnz, dtype=torch.bfloat16, device=dev)
        O = torch.empty_like(Q)
        calls = {
            "rsddmm": lambda: S.splat_rsddmm(a, Q, K, Sb, cfg.scale, stream),
            "softmax": lambda: S.splat_sparse_softmax(a, Sb, Pb, 1, nbh, stream),
            "rspmm": lambda: S.splat_rspmm(a, Pb, V, O, stream),
        }
        qkv = cfg.N * cfg.d * 2 * nbh
        byts = {"rsddmm": 2 * qkv + 4 * a.nnz * nbh, "softmax": 6 * a.nnz * nbh,
                "rspmm": 2 * a.nnz * nbh + 2 * qkv}
        out = {"config": name, "bh": nbh, "nnz_per_head": a.nnz, "acsr_build_ms": build_ms,
               "acsr_meta_bytes": 81 * cfg.N}
        for k, fn in calls.items():
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            tot = 0.0
            for i in range(args.iters):
                flush.fill_(float(i))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn()
                e1.record(stream)
                torch.cuda.synchronize()
                tot += e0.elapsed_time(e1)
            ms = tot / args.iters
            gbs = byts[k] / (ms * 1e-3) / 1e9
            out[k] = {"ms": ms, "GB/s": gbs, "frac_hbm": gbs / hbm if hbm else None,
                      "TFLOP/s": (2.0 * a.nnz * cfg.d * nbh) / (ms * 1e-3) / 1e12 if k != "softmax" else None}
        print(json.dumps(out), flush=True)
        del Sb, Pb, Q, K, V, O
        a.destroy()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
