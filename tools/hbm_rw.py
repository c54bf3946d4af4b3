"""HBM bandwidth by direction on this GPU (torch kernels, 2 GiB buffers, CUDA events, median of 20):
read-only (sum), write-only (fill_), copy (read + write).  Context for the unfused primitives'
roofline: R-SDDMM writes ~9x what it reads, R-SpMM / softmax mostly read."""
import json
import torch

n = 512 * 1024 * 1024      # floats = 2 GiB
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
a.fill_(1.0)


def t(fn, reps=20):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return sorted(ts)[len(ts) // 2]


nb = n * 4
out = {"read_GBps": nb / t(lambda: a.sum()) / 1e9,
       "write_GBps": nb / t(lambda: b.fill_(2.0)) / 1e9,
       "copy_GBps_rw": 2 * nb / t(lambda: b.copy_(a)) / 1e9,
       "buffer_bytes": nb}
print(json.dumps(out))

# host <-> device over PCIe: pinned 151 MB (one Longformer step's Q, K, V) each way, and both at once
h = torch.empty(151 * 1024 * 1024 // 4, dtype=torch.float32).pin_memory()
d = torch.empty_like(h, device="cuda")
h2 = torch.empty_like(h).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(b[: h.numel()], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


hb = h.numel() * 4
print(json.dumps({"h2d_GBps": hb / t(lambda: d.copy_(h, non_blocking=True)) / 1e9,
                  "d2h_GBps": hb / t(lambda: h2.copy_(d, non_blocking=True)) / 1e9,
                  "duplex_GBps_each": hb / t(both) / 1e9}))
