#!/usr/bin/env python
"""Benchmark of the fused SPLAT sparse-MHSA hot path on B200 (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

Metric (BASELINE.json): fused sparse-MHSA nnz-counted TFLOP/s (4*nnz*d per
(b, h), SURVEY A-14) and its fraction of the B200 roofline.  A step is one
splat_sparse_mhsa call (rows a1/a2 -- ACSR + plan -- are built once per
pattern, outside the step, as the paper's compile-once/launch-many workflow,
Listing 4) over one batch of synthetic Q/K/V of the config's shape
(workloads.py), resident in HBM.  L2 is flushed (a 256 MiB write) before every
timed step, and each step is timed with CUDA events on the launching stream;
ms_per_step is the mean over the K steps, max over ranks.

Multi-GPU: ``--gpus N`` launches N ranks (torch.distributed.run,
one process per GPU, NCCL) when the script is not already running under a
launcher.  The config's B*H (b, h) units are split into contiguous blocks of
B*H/N per rank (strong scaling; ``--scaling weak`` gives every rank a full
batch).  No collective on the data path; outside the timed region O is
all-gathered over NCCL and every rank's first and last slices are compared
BITWISE with a one-device recomputation, and sampled rows with the fp64 oracle.

``e2e`` is the same metric through splat_sparse_mhsa_host with pinned host
buffers: H2D of Q, K, V, the kernel and D2H of O inside the timed region.
``per_config`` (N = 1) measures the other BASELINE configs in the same run.
``cpu_baseline`` is the fp64 oracle (oracle/) timed on the host's cores on a
bounded sample of the same workload (rank 0, N=1 only).  ``--impl reference``
times that oracle as the reference arm.

The library is the product build (libsplat.so): the script refuses to run when
any SPLAT_* environment variable is set (those select diagnostics builds or
knobs), and records that in the line.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import CONFIG_BY_NAME, CONFIGS, make_tensor  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                  "sm_max_mhz": 1965.0}
DEFAULT_CONFIG = "longformer"          # BASELINE.json configs[1]
METRIC = "fused sparse-MHSA nnz-counted TFLOP/s"


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def refuse_knobs():
    bad = sorted(k for k in os.environ if k.startswith("SPLAT_"))
    if bad:
        sys.stderr.write(f"bench.py: refusing to run with {bad} set (diagnostics knobs / builds are not "
                         "product runs); unset them\n")
        sys.exit(2)


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(n: int) -> int:
    """Re-run this script under torch.distributed.run with n ranks on this node."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def oracle_sample(cfg, seconds_target: float = 15.0, threads: int | None = None):
    """Bounded sample of the workload for the oracle: the first H_s (b,h) slices (all rows),
    plus rows [0, R) of one more slice, sized so the fp64 oracle needs about ``seconds_target`` s
    at ~1 GFLOP/s per thread.  Returns (full_heads, extra_rows, flops, threads)."""
    from oracle import oracle as O
    threads = threads or O.default_threads()
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


def cpu_baseline(cfg, seconds: float) -> dict:
    full, rows, oflops, threads = oracle_sample(cfg, seconds_target=seconds)
    ts = time_oracle(cfg, full, rows, threads, reps=1)
    tiny = CONFIG_BY_NAME["tiny"]
    t1 = time_oracle(tiny, 1, 0, 1, reps=1)[0]             # single-thread tiny time
    return {"value": oflops / ts[0] / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": "oracle",
            "sample": sample_text(cfg, full, rows, threads) + f"; {ts[0]:.1f} s",
            "cpu_model": cpu_model(), "tiny_single_thread_s": t1}


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
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "TFLOP/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "B": cfg.B, "H": cfg.H, "N": cfg.N, "d": cfg.d,
                   "pattern": cfg.pattern.__dict__, "sample": sample},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def load_traffic(cfg_name: str):
    """DRAM bytes per launch of the fused kernel from the committed ncu --set full summary (or None)."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(cfg_name, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def roofline(cfg, nnz: int, nbh: int, ms: float, peaks: dict, peak_src: str) -> dict:
    """Dominant-kernel roofline for one launch over nbh (b,h) slices taking ms milliseconds."""
    kernel_tflops = 4.0 * nnz * cfg.d * nbh / (ms * 1e-3) / 1e12
    if cfg.dtype == "bf16":
        ai = 4.0 * nnz * cfg.d / (4.0 * cfg.N * cfg.d * 2)       # FLOP per compulsory byte (Q, K, V, O once)
        ridge = peaks["bf16_tflops"] * 1e3 / peaks["hbm_gbs"]
        if ai >= ridge:
            r = {"bound": "tensor", "achieved": kernel_tflops, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s"}
        else:
            gbs = 4.0 * cfg.N * cfg.d * 2 * nbh / (ms * 1e-3) / 1e9
            r = {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s"}
        r["arith_intensity"] = ai
    else:
        alu_peak = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12   # SIMT fp32 FFMA
        r = {"bound": "alu", "achieved": kernel_tflops, "peak": alu_peak, "unit": "TFLOP/s"}
    r["frac"] = r["achieved"] / r["peak"]
    r["peak_source"] = peak_src
    return r


def time_steps(step, stream, steps: int, warmup: int, flush, dev: int, sync_ranks=None):
    """CUDA-event time of `steps` calls of step() after `warmup`, L2 flushed before each timed call."""
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if sync_ranks:
        sync_ranks()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for i in range(steps):
            if flush is not None:
                flush.fill_(float(i))                       # evict L2 (256 MiB > 126 MB)
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    if sync_ranks:
        sync_ranks()
    ms = [a.elapsed_time(b) for a, b in ev]
    return sum(ms) / len(ms), clk.result()


def device_inputs(cfg, nbh: int, dev, seed: int):
    """Seeded uniform [-1, 1) Q, K, V generated on the device (per_config timing only)."""
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    out = []
    for _ in range(3):
        x = torch.rand((1, nbh, cfg.N, cfg.d), generator=g, device=dev, dtype=torch.float32) * 2 - 1
        out.append(x.to(cfg.torch_dtype))
    return out


def plan_stats(acsr, d: int = 0) -> dict:
    """Tile plan of the handle; for d = 64 also the split-group kernel's own plan (row classes and
    composite windows: the (tile, window) entries that kernel actually walks per head)."""
    bm, bn, nq, ne = acsr.plan_info()
    out = {"tile": [bm, bn], "query_tiles": nq, "entries_per_head": ne,
           "tile_efficiency": acsr.nnz / float(max(1, ne) * bm * bn)}
    if d == 64:
        rc, nse = acsr.split_info()
        out["fused_d64"] = {"row_classes": rc, "entries_per_head": nse,
                            "tile_efficiency": acsr.nnz / float(max(1, nse) * bm * bn)}
    return out


def per_config_line(S, cfg, dev, stream, flush, peaks, peak_src, steps: int) -> dict:
    """One BASELINE config on this GPU (all B*H slices, device-generated inputs)."""
    acsr = S.Acsr(cfg.pattern, device=dev)
    Q, K, V = device_inputs(cfg, cfg.BH, dev, 7 + cfg.index)
    O = torch.empty_like(Q)

    def step():
        S.splat_sparse_mhsa(acsr, Q, K, V, O, cfg.scale, stream)

    ms, clk = time_steps(step, stream, steps, 3, flush, dev)
    launches = S.last_launch_count()
    ok = bool(torch.isfinite(O.float()).all())
    flops = acsr.flops(1, cfg.BH, cfg.d)
    line = {"value": flops / (ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms, "steps": steps,
            "B": cfg.B, "H": cfg.H, "N": cfg.N, "d": cfg.d, "dtype": cfg.dtype, "nnz_per_head": acsr.nnz,
            "density": acsr.density, "plan": plan_stats(acsr, cfg.d if cfg.dtype == "bf16" else 0), "launches_per_step": launches,
            "roofline": roofline(cfg, acsr.nnz, cfg.BH, ms, peaks, peak_src), "clocks": clk, "finite": ok,
            "data": "synthetic, device-generated uniform [-1, 1)"}
    acsr.destroy()
    del Q, K, V, O
    torch.cuda.empty_cache()
    return line


def oracle_rows_check(cfg, host, O_host, bh_global, n_slices: int = 2, rows: int = 64) -> float:
    """Max-abs error of the first `rows` rows of `n_slices` slices against the fp64 oracle."""
    from oracle import oracle as O
    err = 0.0
    for i in range(min(n_slices, O_host.shape[1])):
        ref = O.attention(cfg.pattern, host[0][0, i], host[1][0, i], host[2][0, i], cfg.scale, rows=(0, rows))
        got = O_host[0, i, :rows].float().numpy()
        err = max(err, float(np.max(np.abs(got - ref))))
    return err


def run_ours(args, cfg):
    import torch.distributed as dist
    from paper_2407_16847_b200 import splat as S
    from paper_2407_16847_b200.shard import bh_range, gather_and_check

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.cuda.current_device()
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    sync_ranks = dist.barrier if ws > 1 else None

    B, H = cfg.B, cfg.H
    scaling = args.scaling if ws > 1 else "strong"
    bh = bh_range(B * H, rank, ws, scaling)
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

    ms_step, clocks = time_steps(step, stream, args.steps, args.warmup, None if args.no_flush else flush, dev,
                                 sync_ranks)
    launches_per_step = S.last_launch_count()
    if not torch.isfinite(O.float()).all():
        raise RuntimeError("non-finite output")

    # e2e through the C ABI with pinned host buffers (H2D + kernel + D2H per step)
    Oh = torch.empty_like(host[0]).pin_memory()

    def e2e_step():
        S.splat_sparse_mhsa_host(acsr, host[0], host[1], host[2], Oh, cfg.scale, Q, K, V, O, stream)

    e2e_ms, _ = time_steps(e2e_step, stream, args.steps, max(1, args.warmup), None, dev, sync_ranks)
    h2d = sum(h.numel() * h.element_size() for h in host)
    d2h = Oh.numel() * Oh.element_size()

    t = torch.tensor([ms_step, e2e_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step, e2e_ms = float(t[0]), float(t[1])
    total_flops = flops * ws
    value = total_flops / (ms_step * 1e-3) / 1e12

    # ---- validation (outside the timed region)
    S.splat_sparse_mhsa(acsr, Q, K, V, O, cfg.scale, stream)
    torch.cuda.synchronize()
    validation = {}
    if ws > 1 and scaling == "strong":
        def recompute(idx):
            qkv = [make_tensor(cfg.index, t, 1, 1, cfg.N, cfg.d, dt, idx).view(1, len(idx), cfg.N, cfg.d).to(dev)
                   for t in (0, 1, 2)]
            o = torch.empty_like(qkv[0])
            S.splat_sparse_mhsa(acsr, qkv[0], qkv[1], qkv[2], o, cfg.scale, stream)
            torch.cuda.synchronize()
            return o[0]
        validation.update(gather_and_check(O[0], recompute))
    validation["oracle_rows_maxabs"] = oracle_rows_check(cfg, host, O.cpu(), bh)
    validation["oracle_rows_checked"] = "rows [0, 64) of this rank's first 2 slices"
    validation["tolerance"] = 2e-2 if cfg.dtype == "bf16" else 1e-5
    validation["ok"] = validation["oracle_rows_maxabs"] <= validation["tolerance"] and \
        validation.get("bitwise_equal_to_one_device", True)

    peaks, peak_src = load_peaks()
    roof = roofline(cfg, acsr.nnz, nbh, ms_step, peaks, peak_src)
    roof["traffic"] = load_traffic(cfg.name)
    roof["traffic_source"] = "profiles/ncu_summary.json (ncu --set full, dram read+write per launch)"

    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": scaling,
        "vs_baseline": None, "dtype": cfg.dtype if cfg.dtype != "fp32" else "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "B": B, "H": H, "N": cfg.N, "d": cfg.d, "bh_per_rank": nbh,
                   "pattern": cfg.pattern.__dict__, "nnz_per_head": acsr.nnz, "density": acsr.density,
                   "plan": plan_stats(acsr, cfg.d if cfg.dtype == "bf16" else 0),
                   "l2": "warm (diagnostic --no-flush)" if args.no_flush else "flushed before every timed step (256 MiB write)",
                   "parallelism": f"(b,h)-shard x{ws} ({scaling})"},
        "roofline": roof,
        "e2e": {"value": total_flops / (e2e_ms * 1e-3) / 1e12, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks,
        "validation": validation,
        "library": {"so": os.path.basename(S.LIB_PATH), "knobs": "none (SPLAT_* refused)"},
    }
    acsr.destroy()
    del Q, K, V, O
    torch.cuda.empty_cache()
    if ws == 1 and not args.no_per_config:
        line["per_config"] = {}
        for c in CONFIGS:
            if c.name == cfg.name:
                continue
            line["per_config"][c.name] = per_config_line(S, c, dev, stream, flush, peaks, peak_src,
                                                         5 if c.name == "mistral" else 20)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0 if validation["ok"] else 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=[c.name for c in CONFIGS])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="diagnostics only: keep L2 warm between steps")
    args = ap.parse_args()
    refuse_knobs()
    if args.warmup < 3:
        args.warmup = 3
    ws, _, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args.gpus)
    if ws != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
        return 2
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")            # communicator logs: rank count on stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cfg = CONFIG_BY_NAME[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
