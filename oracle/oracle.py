"""ctypes wrapper around oracle/splat_oracle.c (fp64 CPU oracle).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this module.
It never imports the product package (paper_2407_16847_b200) and the product
never imports it.  Argument marshalling only: every step of the oracle's
arithmetic lives in splat_oracle.c, each step citing PAPER.md.

Pinning: every function here is pinned by ``tests/test_oracle_pins.py``
(worked examples of the paper, closed forms, textbook/library special cases,
brute force on tiny inputs); see DESIGN.md "Oracle pins".
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "splat_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

KIND_IDS = {"window": 0, "blocked": 1, "strided": 2, "dilated": 3,
            "global_local": 4, "bigbird": 5, "strided_local": 6}


class _Pattern(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("kind", "n", "lo", "hi", "block", "n_global", "stride", "radius", "causal")]


def build(force: bool = False) -> str:
    """Compile splat_oracle.c with gcc (plain -O2, IEEE fp64; no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-pthread", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.POINTER
        L.or_pred.argtypes = [P(_Pattern), C.c_int, C.c_int]
        L.or_pred.restype = C.c_int
        L.or_row_cols.argtypes = [P(_Pattern), C.c_int, C.c_void_p]
        L.or_row_cols.restype = C.c_int
        L.or_runs_from_cols.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int]
        L.or_runs_from_cols.restype = C.c_int
        L.or_acsr.argtypes = [P(_Pattern), C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.or_acsr.restype = C.c_int
        L.or_regularity.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                    C.c_void_p, P(C.c_int32), P(C.c_int32)]
        L.or_regularity.restype = C.c_int
        L.or_softmax_rows.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.or_softmax_rows.restype = None
        L.or_attention.argtypes = [P(_Pattern), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                   C.c_double, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_int]
        L.or_attention.restype = C.c_int
        L.or_mask.argtypes = [P(_Pattern), C.c_void_p]
        L.or_mask.restype = None
        L.or_fast_index.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.or_fast_index.restype = C.c_int
        _lib = L
    return _lib


def _pat(p) -> _Pattern:
    """Any object with the workloads.Pattern fields -> the oracle's own struct."""
    return _Pattern(KIND_IDS[p.kind], p.seq_len, p.lo, p.hi, p.block, p.n_global,
                    p.stride, p.radius, p.causal)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(x) -> np.ndarray:
    """torch / numpy array -> contiguous float64 numpy (exact upcast of bf16/fp32)."""
    if hasattr(x, "detach"):
        x = x.detach().to("cpu").double().numpy()
    return np.ascontiguousarray(x, dtype=np.float64)


def pred(p, i: int, j: int) -> bool:
    return bool(lib().or_pred(C.byref(_pat(p)), i, j))


def fast_index(start: int, step: int, count: int, c: int) -> int:
    """Sparse index of dense column c in run (start, step, count), or -1 (reading A-7)."""
    return int(lib().or_fast_index(start, step, count, c))


def mask(p) -> np.ndarray:
    """Explicit [N, N] uint8 mask (row i = query, column j = key; reading A-8)."""
    n = p.seq_len
    out = np.zeros((n, n), dtype=np.uint8)
    lib().or_mask(C.byref(_pat(p)), _ptr(out))
    return out


def row_cols(p, i: int) -> np.ndarray:
    buf = np.zeros(max(p.seq_len, 1), dtype=np.int32)
    c = lib().or_row_cols(C.byref(_pat(p)), i, _ptr(buf))
    return buf[:c].copy()


def runs_from_cols(cols, max_seg: int = 64):
    """Greedy affine runs (start, step, count) of an ascending column list."""
    cols = np.ascontiguousarray(np.asarray(cols, dtype=np.int32))
    seg = np.zeros(3 * max_seg, dtype=np.int32)
    ns = lib().or_runs_from_cols(_ptr(cols), len(cols), _ptr(seg), max_seg)
    return [tuple(int(v) for v in seg[3 * s:3 * s + 3]) for s in range(min(ns, max_seg))]


def acsr(p, max_seg: int = 4):
    """ACSR metadata: seg [N, max_seg, 3] int32, nseg [N] int32, row_ptr [N+1] int64, rc."""
    n = p.seq_len
    seg = np.zeros((n, max_seg, 3), dtype=np.int32)
    nseg = np.zeros(n, dtype=np.int32)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    rc = lib().or_acsr(C.byref(_pat(p)), max_seg, _ptr(seg), _ptr(nseg), _ptr(row_ptr))
    return seg, nseg, row_ptr, rc


def regularity(m: np.ndarray):
    """Paper's checkRegularity on an explicit mask -> (regular, a, b, nnzs, (bad_row, bad_col))."""
    m = np.ascontiguousarray(m, dtype=np.uint8)
    rows, ncols = m.shape
    a = np.zeros(rows)
    b = np.zeros(rows)
    nnzs = np.zeros(rows, dtype=np.int32)
    br, bc = C.c_int32(-1), C.c_int32(-1)
    ok = lib().or_regularity(_ptr(m), rows, ncols, _ptr(a), _ptr(b), _ptr(nnzs), C.byref(br), C.byref(bc))
    return bool(ok), a, b, nnzs, (br.value, bc.value)


def softmax_rows(S, row_ptr) -> np.ndarray:
    S = _f64(S)
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    P = np.zeros_like(S)
    lib().or_softmax_rows(_ptr(S), _ptr(row_ptr), len(row_ptr) - 1, _ptr(P))
    return P


def default_threads() -> int:
    return os.cpu_count() or 1


def attention(p, q, k, v, scale: float, rows=None, want_sp: bool = False,
              nthreads: int | None = None, row_ptr=None):
    """Masked attention of one (b, h) slice.

    q, k, v: [N, d] (torch or numpy, any float dtype; upcast exactly to fp64).
    rows: (row0, row1) half-open; default all rows.
    Returns O [(row1-row0), d] and, if want_sp, S and P in ACSR order for those rows.
    """
    n = p.seq_len
    q, k, v = _f64(q), _f64(k), _f64(v)
    assert q.shape[0] == n and k.shape[0] == n and v.shape[0] == n
    d = q.shape[1]
    r0, r1 = (0, n) if rows is None else rows
    O = np.zeros((r1 - r0, d))
    S = P = None
    if want_sp:
        if row_ptr is None:
            row_ptr = acsr(p, max_seg=64)[2]
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        tot = int(row_ptr[r1] - row_ptr[r0])
        S = np.zeros(tot)
        P = np.zeros(tot)
    nt = nthreads or default_threads()
    rc = lib().or_attention(C.byref(_pat(p)), _ptr(q), _ptr(k), _ptr(v), d, float(scale), r0, r1,
                            _ptr(row_ptr) if want_sp else None, _ptr(S), _ptr(P), _ptr(O), nt)
    assert rc == 0
    return (O, S, P) if want_sp else O
