"""Mask-ingest kernel bandwidth (splat_acsr_from_mask's scan).

Builds the explicit bit mask of a configuration on the GPU (Mistral by default: N = 32768,
134 MB of mask words, larger than L2), then times the ingest kernels alone (row scan + row_ptr
scan, through the library's timing hook) with CUDA events on the launching stream, and reports
algorithmic bytes (the mask words read once + the metadata written) / time against the measured
HBM peak.  Also times the full synchronous splat_acsr_from_mask call (plan build included).

    python tools/bench_mask_ingest.py [--config mistral] [--iters 20]
"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_16847_b200 import splat as S  # noqa: E402
from workloads import CONFIG_BY_NAME  # noqa: E402


def mask_words(p):
    n = p.seq_len
    W = (n + 31) // 32
    words = torch.zeros((n, W), dtype=torch.int32, device="cuda")
    i = torch.arange(n, device="cuda")[:, None]
    sh = torch.arange(32, device="cuda")
    for c0 in range(0, n, 4096):
        j = torch.arange(c0, min(n, c0 + 4096), device="cuda")[None, :]
        if p.kind == "window":
            bits = (j >= i - p.lo) & (j <= i + p.hi)
        elif p.kind == "global_local":
            g = p.n_global
            bits = (i < g) | (j < g) | ((j >= i - p.lo) & (j <= i + p.hi))
        else:
            raise SystemExit(f"no GPU mask generator for {p.kind}")
        packed = (bits.view(n, -1, 32).to(torch.int64) << sh).sum(-1)
        words[:, c0 // 32:c0 // 32 + packed.shape[1]] = torch.where(packed >= 2 ** 31, packed - 2 ** 32,
                                                                     packed).to(torch.int32)
    return words


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mistral")
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    p = CONFIG_BY_NAME[a.config].pattern
    n = p.seq_len
    words = mask_words(p)
    L = S.lib()
    L.splat_debug_mask_ingest.argtypes = [C.c_void_p, C.c_int, C.c_int] + [C.c_void_p] * 5
    seg = torch.empty((n, 16), dtype=torch.int32, device="cuda")
    nseg = torch.empty(n, dtype=torch.uint8, device="cuda")
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    bad = torch.empty(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    args = [words.data_ptr(), n, 4, seg.data_ptr(), nseg.data_ptr(), row_ptr.data_ptr(), bad.data_ptr(),
            st.cuda_stream]
    for _ in range(3):
        assert L.splat_debug_mask_ingest(*args) == 0
    torch.cuda.synchronize()
    ms = []
    for _ in range(a.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        L.splat_debug_mask_ingest(*args)
        e1.record(st)
        e1.synchronize()
        ms.append(e0.elapsed_time(e1))
    ms.sort()
    med = ms[len(ms) // 2]
    mask_bytes = words.numel() * 4
    meta_bytes = n * (64 + 1 + 8) + 8
    gbs = (mask_bytes + meta_bytes) / (med * 1e-3) / 1e9
    peak, src = 6650.0, "fallback"
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        d = json.load(open(pk))
        for k in ("hbm_gbs_burst", "hbm_copy_gbs", "hbm_gbs"):
            if k in d:
                peak, src = float(d[k]), k
                break
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    h = S.splat_acsr_from_mask(words, n, device=0)
    e1.record(st)
    e1.synchronize()
    full_ms = e0.elapsed_time(e1)
    ref = S.Acsr(p, device=0)
    same = all(torch.equal(x, y) for x, y in zip(h.copy_meta(), ref.copy_meta()))
    print(json.dumps({"config": a.config, "n": n, "mask_bytes": mask_bytes, "kernel_ms_median": med,
                      "kernel_ms_min": ms[0], "achieved_gbs": gbs, "peak_gbs": peak, "peak_source": src,
                      "frac": gbs / peak, "full_call_ms": full_ms, "meta_equals_descriptor_build": same}))


if __name__ == "__main__":
    main()
