#!/usr/bin/env python
"""Benchmark of the fused SPLAT sparse-MHSA hot path on B200 (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1)

Metric (BASELINE.json): fused sparse-MHSA nnz-counted TFLOP/s (4*nnz*d per
(b, h), SURVEY A-14) and its fraction of the B200 roofline.  A step is one
splat_sparse_mhsa call (rows a1/a2 -- ACSR + plan -- are built once per
pattern, outside the step, exactly as the paper's compile-once/launch-many
workflow, Listing 4) over one batch of synthetic Q/K/V of the
config's shape (workloads.py), resident in HBM.  L2 is flushed (a 256 MiB
write) before every timed step, and each step is timed with CUDA events on
the launching stream; ms_per_step is the mean over the K steps, max over
ranks.  Multi-GPU: one process per GPU, every rank runs its own batch of
independent (b, h) units (weak scaling, no collective on the data path;
NCCL only for the barrier and the max-over-ranks time).

``e2e`` is the same metric through splat_sparse_mhsa_host with pinned host
buffers: H2D of Q, K, V, the kernel and D2H of O inside the timed region.
``cpu_baseline`` is the fp64 oracle (oracle/) timed on the host's cores on a
bounded sample of the same workload (rank 0, N=1 only).
``--impl reference`` times that oracle as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import math

import numpy as np
import os
import statistics
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import CONFIG_BY_NAME, CONFIGS, make_tensor  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                  "sm_max_mhz": 1965.0}
DEFAULT_CONFIG = "longformer"          # BASELINE.json configs[1]


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f), "measured"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# clocks sampler (NVML) -- runs during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
               "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device_index: int, period_s: float = 0.002):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period_s
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def sample(self):
        if self.nv is None:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for name, bit in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(self.period)

    def __enter__(self):
        self.sample()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()
        self.sample()

    def result(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU oracle (cpu_baseline / reference arm)
# ---------------------------------------------------------------------------
def oracle_sample(cfg, seconds_target: float = 15.0):
    """Bounded sample of the workload for the oracle: the first H_s (b,h) slices
    (all rows), plus rows [0, R) of one more slice, sized so the fp64 oracle
    needs about ``seconds_target`` s at ~1 GFLOP/s per thread (measured rate of
    the oracle on the GPU box).  Returns (full_heads, extra_rows, flops, threads)."""
    from oracle import oracle as O
    threads = O.default_threads()
    budget = seconds_target * 1.0e9 * threads
    if cfg.N <= 8192:
        row_ptr = O.acsr(cfg.pattern)[2]
    else:                     # nnz per row from the (causal) window bound, exact for WINDOW(lo, 0)
        per = np.minimum(np.arange(cfg.N) + 1, cfg.pattern.lo + 1)
        row_ptr = np.concatenate([[0], np.cumsum(per)])
    per_head = 4.0 * cfg.d * float(row_ptr[-1])
    full = int(min(cfg.BH, budget // per_head))
    rows = 0
    if full < cfg.BH:
        rest = budget - full * per_head
        for r in range(0, cfg.N + 1, 64):
            if 4.0 * cfg.d * float(row_ptr[r]) > rest:
                break
            rows = r
    flops = full * per_head + 4.0 * cfg.d * float(row_ptr[rows])
    return full, rows, flops, threads


def time_oracle(cfg, full: int, rows: int, threads: int, reps: int = 1):
    from oracle import oracle as O
    n_sl = full + (1 if rows else 0)
    qkv = [make_tensor(cfg.index, t, 1, 1, cfg.N, cfg.d, cfg.torch_dtype, range(0, n_sl)) for t in (0, 1, 2)]
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for bh in range(full):
            O.attention(cfg.pattern, qkv[0][bh], qkv[1][bh], qkv[2][bh], cfg.scale, nthreads=threads)
        if rows:
            O.attention(cfg.pattern, qkv[0][full], qkv[1][full], qkv[2][full], cfg.scale, rows=(0, rows),
                        nthreads=threads)
        ts.append(time.perf_counter() - t0)
    return ts


def sample_text(cfg, full, rows, threads):
    s = f"{full} of {cfg.BH} (b,h) slices of {cfg.name} (N={cfg.N}, d={cfg.d}), all rows"
    if rows:
        s += f", + rows [0,{rows}) of slice {full}"
    return s + f"; fp64 oracle, {threads} threads"


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    full, rows, flops, threads = oracle_sample(cfg, seconds_target=min(8.0, 150.0 / max(1, args.steps + args.warmup)))
    ts = time_oracle(cfg, full, rows, threads, reps=args.steps + args.warmup)
    ts = ts[args.warmup:]
    sec = sum(ts) / len(ts)
    value = flops / sec / 1e12
    sample = sample_text(cfg, full, rows, threads)
    line = {
        "impl": "reference", "metric": "fused sparse-MHSA nnz-counted TFLOP/s", "value": value,
        "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "B": cfg.B, "H": cfg.H, "N": cfg.N, "d": cfg.d,
                   "pattern": cfg.pattern.__dict__, "sample": sample},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def load_traffic(cfg_name: str):
    """dram bytes per launch of the fused kernel from the committed ncu summary (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(cfg_name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def run_ours(args, cfg):
    import torch.distributed as dist
    from paper_2407_16847_b200 import splat as S

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

    from paper_2407_16847_b200.shard import bh_range
    B, H = cfg.B, cfg.H
    bh = bh_range(B * H, rank, ws, args.scaling if ws > 1 else "weak")
    nbh = len(bh)
    dt = cfg.torch_dtype
    host = [make_tensor(cfg.index, t, 1, 1, cfg.N, cfg.d, dt, bh).view(1, nbh, cfg.N, cfg.d).pin_memory()
            for t in (0, 1, 2)]
    Q, K, V = (h.to(dev, non_blocking=True) for h in host)
    O = torch.empty_like(Q)
    acsr = S.Acsr(cfg.pattern, device=dev)
    flops = acsr.flops(1, nbh, cfg.d)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        S.splat_sparse_mhsa(acsr, Q, K, V, O, cfg.scale, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = S.last_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for i in range(args.steps):
            if not args.no_flush:
                flush.fill_(float(i))                       # evict L2 (256 MiB > 126 MB)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    ms = [a.elapsed_time(b) for a, b in ev]
    ms_step = sum(ms) / len(ms)
    if not torch.isfinite(O.float()).all():
        raise RuntimeError("non-finite output")

    # e2e through the C ABI with pinned host buffers (H2D + kernel + D2H per step)
    Oh = torch.empty_like(host[0]).pin_memory()
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]

    def e2e_step():
        S.splat_sparse_mhsa_host(acsr, host[0], host[1], host[2], Oh, cfg.scale, Q, K, V, O, stream)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    for i in range(args.steps):
        e2e_ev[i][0].record(stream)
        e2e_step()
        e2e_ev[i][1].record(stream)
    torch.cuda.synchronize()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev) / args.steps
    h2d = sum(h.numel() * h.element_size() for h in host)
    d2h = Oh.numel() * Oh.element_size()

    t = torch.tensor([ms_step, e2e_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step, e2e_ms = float(t[0]), float(t[1])
    total_flops = flops * ws
    value = total_flops / (ms_step * 1e-3) / 1e12

    peaks, peak_src = load_peaks()
    kernel_tflops = flops / (ms_step * 1e-3) / 1e12          # per-GPU, per launch
    if cfg.dtype == "bf16":
        ai = 4.0 * acsr.nnz * cfg.d / (4.0 * cfg.N * cfg.d * 2)  # FLOP per compulsory byte
        ridge = peaks["bf16_tflops"] * 1e3 / peaks["hbm_gbs"]
        if ai >= ridge:
            roof = {"bound": "tensor", "achieved": kernel_tflops, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s"}
        else:
            gbs = 4.0 * cfg.N * cfg.d * 2 * nbh / (ms_step * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
    else:
        alu_peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12   # SIMT fp32 FFMA
        roof = {"bound": "alu", "achieved": kernel_tflops, "peak": alu_peak, "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["peak_source"] = peak_src
    roof["traffic"] = load_traffic(cfg.name)

    line = {
        "metric": "fused sparse-MHSA nnz-counted TFLOP/s", "value": value, "unit": "TFLOP/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak" if args.scaling == "weak" or ws == 1 else "strong",
        "vs_baseline": None, "dtype": cfg.dtype if cfg.dtype != "fp32" else "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "B": B, "H": H, "N": cfg.N, "d": cfg.d, "bh_per_rank": nbh,
                   "pattern": cfg.pattern.__dict__, "nnz_per_head": acsr.nnz, "density": acsr.density,
                   "l2": "warm (diagnostic --no-flush)" if args.no_flush else "flushed before every timed step (256 MiB write)", "parallelism": f"bh-shard x{ws}"},
        "roofline": roof,
        "e2e": {"value": total_flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.result(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        full, rows, oflops, threads = oracle_sample(cfg, seconds_target=args.cpu_seconds)
        ts = time_oracle(cfg, full, rows, threads, reps=1)
        line["cpu_baseline"] = {
            "value": oflops / ts[0] / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
            "sample": sample_text(cfg, full, rows, threads) + f"; {ts[0]:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    acsr.destroy()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=[c.name for c in CONFIGS])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="diagnostics only: keep L2 warm between steps")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIG_BY_NAME[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
