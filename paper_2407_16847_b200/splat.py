"""Thin ctypes binding of the C ABI in include/splat.h (libsplat.so).

Argument marshalling only: names follow the C entry points; torch tensors are
passed as raw device pointers together with the current CUDA stream.  Every
step of the hot path runs in the library's CUDA kernels.  There is no CPU
fallback: if libsplat.so is missing or fails to load, every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# SPLAT_LIB=diag selects the diagnostics build (profiling / ablation knobs; tools/ only -- bench.py
# refuses to run with any SPLAT_* variable set).  Default: the product library.
LIB_PATH = os.path.join(_PKG, "libsplat.so")
DIAG_LIB_PATH = os.path.join(_PKG, "libsplat_diag.so")

SPLAT_MAX_SEGS = 4
STATUS = {0: "SPLAT_OK", 1: "SPLAT_ERR_INVALID_ARG", 2: "SPLAT_ERR_NOT_REGULAR", 3: "SPLAT_ERR_SHAPE",
          4: "SPLAT_ERR_UNSUPPORTED", 5: "SPLAT_ERR_CUDA", 6: "SPLAT_ERR_OOM"}
SPLAT_BF16, SPLAT_FP32 = 0, 1
KINDS = {"window": 0, "blocked": 1, "strided": 2, "dilated": 3, "global_local": 4, "bigbird": 5,
         "strided_local": 6}

# every symbol include/splat.h declares (tests check the library exports them all)
EXPORTS = ("splat_acsr_build", "splat_acsr_info", "splat_acsr_copy_meta", "splat_plan_info",
           "splat_plan_copy", "splat_plan_split_info", "splat_plan_sizes", "splat_plan_split_copy", "splat_plan_ksplit_copy", "splat_acsr_destroy", "splat_rsddmm", "splat_sparse_softmax", "splat_rspmm",
           "splat_sparse_mhsa", "splat_sparse_mhsa_host", "splat_acsr_from_mask", "splat_poset_tile", "splat_naive_tile",
           "splat_tiling_cost_eval", "splat_acsr_transpose", "splat_transpose_values", "splat_rspmm_cc",
           "splat_layout_choice", "splat_flops", "splat_last_launch_count", "splat_device_alloc_count",
           "splat_last_error")


class SplatError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class splat_tiling_cost(C.Structure):
    _fields_ = [("lambda_", C.c_int64), ("points", C.c_int64), ("phi_td", C.c_int64), ("phi_r", C.c_int64),
                ("phi_ru", C.c_double), ("phi_cmr", C.c_double), ("cost", C.c_double), ("stretch", C.c_int32),
                ("m", C.c_int32), ("n", C.c_int32), ("reserved", C.c_int32)]

    def as_dict(self) -> dict:
        return {"lambda": self.lambda_, "points": self.points, "phi_td": self.phi_td, "phi_r": self.phi_r,
                "phi_ru": self.phi_ru, "phi_cmr": self.phi_cmr, "cost": self.cost, "stretch": self.stretch,
                "m": self.m, "n": self.n}


class splat_pattern(C.Structure):
    _fields_ = [("kind", C.c_int32), ("seq_len", C.c_int32), ("lo", C.c_int32), ("hi", C.c_int32),
                ("block", C.c_int32), ("n_global", C.c_int32), ("stride", C.c_int32), ("radius", C.c_int32),
                ("causal", C.c_int32), ("reserved", C.c_int32 * 7)]


_lib = None


def lib():
    """Load libsplat.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is None:
        path = DIAG_LIB_PATH if os.environ.get("SPLAT_LIB") == "diag" else LIB_PATH
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built: run `python -m paper_2407_16847_b200.build`")
        L = C.CDLL(path)
        vp, i32, i64, f32 = C.c_void_p, C.c_int32, C.c_int64, C.c_float
        P = C.POINTER
        L.splat_acsr_build.argtypes = [P(splat_pattern), C.c_int, vp, P(vp)]
        L.splat_acsr_info.argtypes = [vp, P(i32), P(i64), P(i32), P(C.c_double)]
        L.splat_acsr_copy_meta.argtypes = [vp, vp, vp, vp]
        L.splat_plan_info.argtypes = [vp, P(i32), P(i32), P(i32), P(i32)]
        L.splat_plan_copy.argtypes = [vp, vp, vp, vp]
        L.splat_plan_split_info.argtypes = [vp, P(i32), P(i32)]
        L.splat_plan_sizes.argtypes = [vp, i32]
        L.splat_plan_sizes.restype = i64
        L.splat_plan_split_copy.argtypes = [vp, vp, vp, vp, vp]
        L.splat_plan_ksplit_copy.argtypes = [vp, vp]
        L.splat_acsr_destroy.argtypes = [vp]
        L.splat_rsddmm.argtypes = [vp, vp, vp, C.c_int, i32, i32, i32, f32, vp, vp]
        L.splat_sparse_softmax.argtypes = [vp, vp, vp, C.c_int, i32, i32, vp]
        L.splat_rspmm.argtypes = [vp, vp, vp, C.c_int, i32, i32, i32, vp, vp]
        L.splat_sparse_mhsa.argtypes = [vp, vp, vp, vp, C.c_int, i32, i32, i32, f32, vp, vp]
        L.splat_sparse_mhsa_host.argtypes = [vp, vp, vp, vp, C.c_int, i32, i32, i32, f32, vp, vp, vp, vp, vp,
                                             vp]
        L.splat_acsr_from_mask.argtypes = [vp, i32, i32, C.c_int, vp, P(vp), P(i32), P(i32)]
        L.splat_poset_tile.argtypes = [P(splat_pattern), i32, i32, i32, vp, i64, P(splat_tiling_cost)]
        L.splat_naive_tile.argtypes = [P(splat_pattern), i32, i32, vp, i64, P(splat_tiling_cost)]
        L.splat_tiling_cost_eval.argtypes = [P(splat_pattern), i32, i32, i32, vp, i64, P(splat_tiling_cost)]
        L.splat_acsr_transpose.argtypes = [vp, vp, P(vp)]
        L.splat_transpose_values.argtypes = [vp, vp, vp, vp, C.c_int, i32, i32, vp]
        L.splat_rspmm_cc.argtypes = [vp, vp, vp, vp, C.c_int, i32, i32, i32, vp, vp]
        L.splat_layout_choice.argtypes = [vp, C.c_double]
        L.splat_layout_choice.restype = i32
        L.splat_flops.argtypes = [vp, i32, i32, i32]
        L.splat_flops.restype = C.c_double
        L.splat_last_launch_count.restype = i32
        L.splat_last_error.restype = C.c_char_p
        for name in EXPORTS:
            if name not in ("splat_flops", "splat_last_error", "splat_last_launch_count", "splat_layout_choice",
                            "splat_plan_sizes"):
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise SplatError(st, lib().splat_last_error().decode())


def to_c_pattern(p) -> splat_pattern:
    """workloads.Pattern (or any object with its fields) -> splat_pattern."""
    return splat_pattern(KINDS[p.kind], p.seq_len, p.lo, p.hi, p.block, p.n_global, p.stride, p.radius,
                         p.causal)


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return SPLAT_BF16
    if t.dtype == torch.float32:
        return SPLAT_FP32
    raise SplatError(1, f"unsupported dtype {t.dtype}")


class Acsr:
    """Owning wrapper of a ``splat_acsr`` handle (splat_acsr_build / _from_mask / _destroy)."""

    def __init__(self, pattern, device: int = 0, stream=None, _handle=None):
        self.pattern = pattern
        self.device = device
        h = C.c_void_p()
        if _handle is not None:
            h = _handle
        else:
            st = 0 if device < 0 else _stream(stream) if torch.cuda.is_available() else 0
            _check(lib().splat_acsr_build(C.byref(to_c_pattern(pattern)), device, C.c_void_p(st), C.byref(h)))
        self.handle = h
        n, nnz, ms, dens = C.c_int32(), C.c_int64(), C.c_int32(), C.c_double()
        _check(lib().splat_acsr_info(h, C.byref(n), C.byref(nnz), C.byref(ms), C.byref(dens)))
        self.n, self.nnz, self.max_segs, self.density = n.value, nnz.value, ms.value, dens.value

    def copy_meta(self):
        """(seg [N,4,3] int32, nseg [N] uint8, row_ptr [N+1] int64) as CPU tensors."""
        seg = torch.zeros((self.n, SPLAT_MAX_SEGS, 3), dtype=torch.int32)
        nseg = torch.zeros(self.n, dtype=torch.uint8)
        row_ptr = torch.zeros(self.n + 1, dtype=torch.int64)
        _check(lib().splat_acsr_copy_meta(self.handle, seg.data_ptr(), nseg.data_ptr(), row_ptr.data_ptr()))
        return seg, nseg, row_ptr

    def plan_info(self):
        bm, bn, nq, ne = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().splat_plan_info(self.handle, C.byref(bm), C.byref(bn), C.byref(nq), C.byref(ne)))
        return bm.value, bn.value, nq.value, ne.value

    def split_info(self):
        """(row_classes, entries per (b, h)) of the d = 64 split-group kernel's plan."""
        rc, ne = C.c_int32(), C.c_int32()
        _check(lib().splat_plan_split_info(self.handle, C.byref(rc), C.byref(ne)))
        return rc.value, ne.value

    def split_plan_copy(self):
        """The split kernel's units, entries (kv, mask ids) and masks as CPU tensors."""
        L = lib()
        nu, ne, nm = (L.splat_plan_sizes(self.handle, w) for w in (0, 1, 2))
        units = torch.zeros((nu, 4), dtype=torch.int32)
        kv = torch.zeros(max(ne, 1), dtype=torch.int32)
        mid = torch.zeros(max(ne, 1), dtype=torch.int32)
        masks = torch.zeros((max(nm, 1), 128, 4), dtype=torch.int64).to(torch.int32)
        _check(L.splat_plan_split_copy(self.handle, units.data_ptr(), kv.data_ptr(), mid.data_ptr(), masks.data_ptr()))
        return units, kv[:ne], mid[:ne], masks[:nm]

    def ksplit_units(self):
        """The split-K unit list [n][4] (tile, j0, j1, part | parts << 8 | sid << 16); empty if none."""
        L = lib()
        n = L.splat_plan_sizes(self.handle, 3)
        units = torch.zeros((max(n, 1), 4), dtype=torch.int32)
        _check(L.splat_plan_ksplit_copy(self.handle, units.data_ptr()))
        return units[:n]

    def plan_copy(self):
        _, _, nq, ne = self.plan_info()
        qt_ptr = torch.zeros(nq + 1, dtype=torch.int32)
        kv = torch.zeros(max(ne, 1), dtype=torch.int32)
        order = torch.zeros(nq, dtype=torch.int32)
        _check(lib().splat_plan_copy(self.handle, qt_ptr.data_ptr(), kv.data_ptr(), order.data_ptr()))
        return qt_ptr, kv[:ne], order

    def flops(self, B: int, H: int, d: int) -> float:
        return lib().splat_flops(self.handle, B, H, d)

    def destroy(self):
        if self.handle:
            lib().splat_acsr_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def splat_acsr_build(pattern, device: int = 0, stream=None) -> Acsr:
    return Acsr(pattern, device, stream)


class NotRegular(SplatError):
    def __init__(self, status: int, msg: str, row: int, col: int):
        super().__init__(status, msg)
        self.row, self.col = row, col


def pack_mask(mask: torch.Tensor) -> torch.Tensor:
    """[n, n] bool -> [n, ceil(n/32)] int32 words, column j at bit j % 32 (LSB first).  Marshalling
    of the caller's mask into the ABI's layout (the metadata itself is computed by the library)."""
    n = mask.shape[0]
    W = (n + 31) // 32
    m = torch.zeros((n, W * 32), dtype=torch.int64, device=mask.device)
    m[:, :n] = mask.to(torch.int64)
    w = (m.view(n, W, 32) << torch.arange(32, device=mask.device, dtype=torch.int64)).sum(-1)
    return torch.where(w >= 2 ** 31, w - 2 ** 32, w).to(torch.int32).contiguous()


def splat_acsr_from_mask(words: torch.Tensor, n: int, max_runs: int = SPLAT_MAX_SEGS, device: int = 0,
                         stream=None) -> Acsr:
    """ACSR handle from a packed bit mask (see pack_mask): CUDA tensor -> GPU ingest on `device`;
    CPU tensor with device=-1 -> host inspection handle.  Raises NotRegular with (row, col)."""
    if not words.is_contiguous() or words.dtype != torch.int32 or words.numel() != n * ((n + 31) // 32):
        raise SplatError(1, "words must be contiguous int32 [n, ceil(n/32)]")
    if (device >= 0) != words.is_cuda:
        raise SplatError(1, "device >= 0 needs a CUDA mask, device -1 a CPU mask")
    h = C.c_void_p()
    br, bc = C.c_int32(), C.c_int32()
    st = _stream(stream) if device >= 0 else 0
    rc = lib().splat_acsr_from_mask(words.data_ptr(), n, max_runs, device, C.c_void_p(st), C.byref(h),
                                    C.byref(br), C.byref(bc))
    if rc == 2:
        raise NotRegular(rc, lib().splat_last_error().decode(), br.value, bc.value)
    _check(rc)
    return Acsr(None, device, _handle=h)


def _bhnd(x: torch.Tensor):
    if x.dim() == 4:
        return x.shape
    if x.dim() == 3:
        return (1,) + tuple(x.shape)
    raise SplatError(3, f"expected [B,H,N,d] or [BH,N,d], got {tuple(x.shape)}")


def _check_qkv(a: Acsr, *ts):
    B, H, N, d = _bhnd(ts[0])
    for t in ts:
        if tuple(_bhnd(t)) != (B, H, N, d) or not t.is_contiguous() or not t.is_cuda:
            raise SplatError(3, "tensors must be contiguous CUDA tensors of one [B,H,N,d] shape")
        if t.dtype != ts[0].dtype:
            raise SplatError(1, "dtype mismatch")
    if N != a.n:
        raise SplatError(3, f"N={N} differs from the handle's {a.n}")
    return B, H, d


def splat_rsddmm(a: Acsr, Q, K, S, scale: float, stream=None):
    B, H, d = _check_qkv(a, Q, K)
    if S.dtype != torch.float32 or S.numel() != B * H * a.nnz or not S.is_contiguous():
        raise SplatError(3, "S must be contiguous float32 [B,H,nnz]")
    _check(lib().splat_rsddmm(a.handle, Q.data_ptr(), K.data_ptr(), _dt(Q), B, H, d, scale, S.data_ptr(),
                              C.c_void_p(_stream(stream))))
    return S


def splat_sparse_softmax(a: Acsr, S, P, B: int, H: int, stream=None):
    if S.dtype != torch.float32 or S.numel() != B * H * a.nnz or P.numel() != S.numel():
        raise SplatError(3, "S float32 and P of B*H*nnz elements")
    _check(lib().splat_sparse_softmax(a.handle, S.data_ptr(), P.data_ptr(), _dt(P), B, H,
                                      C.c_void_p(_stream(stream))))
    return P


def splat_rspmm(a: Acsr, P, V, O, stream=None):
    B, H, d = _check_qkv(a, V, O)
    if P.dtype != V.dtype or P.numel() != B * H * a.nnz:
        raise SplatError(3, "P must have V's dtype and B*H*nnz elements")
    _check(lib().splat_rspmm(a.handle, P.data_ptr(), V.data_ptr(), _dt(V), B, H, d, O.data_ptr(),
                             C.c_void_p(_stream(stream))))
    return O


ALPHA = 0.10     # the paper's density threshold for the column-compressed layout


def splat_acsr_transpose(a: Acsr, stream=None) -> Acsr:
    """Handle of M^T (column-compressed ACSR of a's mask), on a's device."""
    h = C.c_void_p()
    st = _stream(stream) if a.device >= 0 else 0
    _check(lib().splat_acsr_transpose(a.handle, C.c_void_p(st), C.byref(h)))
    return Acsr(None, a.device, _handle=h)


def splat_transpose_values(a: Acsr, at: Acsr, X, Y, B: int, H: int, stream=None):
    if X.dtype != Y.dtype or X.numel() != B * H * a.nnz or Y.numel() != X.numel():
        raise SplatError(3, "X and Y: same dtype, B*H*nnz elements")
    _check(lib().splat_transpose_values(a.handle, at.handle, X.data_ptr(), Y.data_ptr(), _dt(X), B, H,
                                        C.c_void_p(_stream(stream))))
    return Y


def splat_rspmm_cc(a: Acsr, at: Acsr, PT, V, O, stream=None):
    B, H, d = _check_qkv(a, V, O)
    if PT.dtype != V.dtype or PT.numel() != B * H * a.nnz:
        raise SplatError(3, "PT must have V's dtype and B*H*nnz elements")
    _check(lib().splat_rspmm_cc(a.handle, at.handle, PT.data_ptr(), V.data_ptr(), _dt(V), B, H, d, O.data_ptr(),
                                C.c_void_p(_stream(stream))))
    return O


def splat_layout_choice(a: Acsr, alpha: float = ALPHA) -> int:
    """1 = column-compressed (density >= alpha), 0 = row-compressed."""
    return int(lib().splat_layout_choice(a.handle, alpha))


def splat_sparse_mhsa(a: Acsr, Q, K, V, O, scale: float, stream=None):
    B, H, d = _check_qkv(a, Q, K, V, O)
    _check(lib().splat_sparse_mhsa(a.handle, Q.data_ptr(), K.data_ptr(), V.data_ptr(), _dt(Q), B, H, d, scale,
                                   O.data_ptr(), C.c_void_p(_stream(stream))))
    return O


def splat_sparse_mhsa_host(a: Acsr, Qh, Kh, Vh, Oh, scale: float, dQ, dK, dV, dO, stream=None):
    """Host-buffer variant: Qh/Kh/Vh/Oh are (pinned) CPU tensors, dQ.. device staging buffers."""
    B, H, N, d = _bhnd(Qh)
    for t in (Qh, Kh, Vh, Oh):
        if t.is_cuda or not t.is_contiguous() or tuple(_bhnd(t)) != (B, H, N, d):
            raise SplatError(3, "host tensors must be contiguous CPU tensors of one shape")
    _check_qkv(a, dQ, dK, dV, dO)
    _check(lib().splat_sparse_mhsa_host(a.handle, Qh.data_ptr(), Kh.data_ptr(), Vh.data_ptr(), _dt(Qh), B, H, d,
                                        scale, Oh.data_ptr(), dQ.data_ptr(), dK.data_ptr(), dV.data_ptr(),
                                        dO.data_ptr(), C.c_void_p(_stream(stream))))
    return Oh


def _tiling(fn, pattern, m: int, n: int, *pre):
    cost = splat_tiling_cost()
    pat = to_c_pattern(pattern)
    _check(fn(C.byref(pat), m, n, *pre, None, 0, C.byref(cost)))
    anchors = torch.zeros((max(cost.lambda_, 1), 2), dtype=torch.int32)
    _check(fn(C.byref(pat), m, n, *pre, anchors.data_ptr(), cost.lambda_, C.byref(cost)))
    return anchors[:cost.lambda_], cost.as_dict()


def splat_poset_tile(pattern, m: int, n: int, stretch: int = 0):
    """Poset tiling (Alg. 1) of the pattern's point set: (anchors [lambda,2] int32 (x, y), cost dict).
    Host-only analysis; stretch 0 = Sec. 7.3.1 selection."""
    return _tiling(lib().splat_poset_tile, pattern, m, n, stretch)


def splat_naive_tile(pattern, m: int, n: int):
    """App. C naive tiling: (anchors [lambda,2] int32 (x, y), cost dict)."""
    return _tiling(lib().splat_naive_tile, pattern, m, n)


def splat_tiling_cost_eval(pattern, m: int, n: int, stretch: int, anchors) -> dict:
    """Def. 3/4 cost report of a given uniform-stretch arrangement (anchors: [k,2] (x, y))."""
    a = torch.as_tensor(anchors, dtype=torch.int32).reshape(-1, 2).contiguous()
    cost = splat_tiling_cost()
    _check(lib().splat_tiling_cost_eval(C.byref(to_c_pattern(pattern)), m, n, stretch, a.data_ptr(), a.shape[0],
                                        C.byref(cost)))
    return cost.as_dict()


def device_alloc_count() -> int:
    """Device allocations the library has made so far (build time only)."""
    L = lib()
    L.splat_device_alloc_count.restype = C.c_int64
    return int(L.splat_device_alloc_count())


def last_launch_count() -> int:
    return lib().splat_last_launch_count()
