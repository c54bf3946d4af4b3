"""Oracle of the paper's thread-block tiling model.

TEST INFRASTRUCTURE ONLY (same rule as oracle/oracle.py): only tests/, ``__graft_entry__`` and
bench.py's baseline legs may import this module; it never imports the product package.

Plain numpy / Python restatement of PAPER.md Sec. 7.2-7.3 and App. A-C, step by step:

  P        the mask's point set, a bool grid ``P[y, x]`` (query row y attends key column x),
           enumerated by the fp64 oracle's mask (oracle.mask).
  comp     Def. 2: Comp(TB) = {t + (c s, r s)}, r < m (rows), c < n (columns)
           -- DESIGN.md reading T-1 fixes m = thread rows (the App. C patches are "m consecutive
           rows"), n = thread columns.
  top      Def. 5: the uncovered points no other uncovered point comes before
           (q <- p iff q.x <= p.x and q.y <= p.y, q != p).
  poset    Alg. 1: while points remain, anchor a block at every point of ⊤ (computed
           once per iteration), then remove each block's Comp from Rem (reading T-2).
  stretch  Sec. 7.3.1: polygonal -> 1 (App. A); strided with row stride X -> the
           divisor of X of least Def. 4 cost (App. B); else s in [1, min(N, 64)] (reading T-4);
           ties -> fewer blocks (reading T-3).
  naive    App. C Def. 8.
  cost     Def. 3 and Def. 4, exact rationals.
  closed forms   App. B cover count f(kappa) and App. C lambda_naive
           (P:1008-1017).

Pinned by tests/test_tiling_oracle.py (the paper's Fig. 6 numbers, the appendix closed forms,
brute-force optimal covers on tiny masks).
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

from . import oracle as O

GENERIC_STRETCH_CAP = 64


def points(pattern) -> np.ndarray:
    """P[y, x] for a pattern descriptor (oracle.mask: row i attends column j)."""
    return np.asarray(O.mask(pattern), dtype=bool)


def structured_polygon(r: int, l: int, h: int, lp: int) -> np.ndarray:
    """App. C Def. 7: P = {(floor(y/h) l' + t, y) : t < l, y < r h}, as a grid wide
    enough to hold every point."""
    rows = r * h
    width = (rows - 1) // h * lp + l
    P = np.zeros((rows, width), dtype=bool)
    for y in range(rows):
        for t in range(l):
            P[y, (y // h) * lp + t] = True
    return P


def comp(anchor, s: int, m: int, n: int) -> set:
    """Def. 2: the m x n stretched lattice of a block, as (x, y) points."""
    x, y = anchor
    return {(x + c * s, y + r * s) for r in range(m) for c in range(n)}


def top(rem: np.ndarray) -> np.ndarray:
    """Def. 5: rem & (no other remaining point in the rectangle [0, x] x [0, y]).

    The number of remaining points q with q.x <= x and q.y <= y is the 2-D prefix count of rem;
    a remaining point is minimal iff that count is 1 (itself)."""
    cnt = np.cumsum(np.cumsum(rem.astype(np.int64), axis=0), axis=1)
    return rem & (cnt == 1)


def poset_tile(P: np.ndarray, m: int, n: int, s: int) -> list:
    """Alg. 1 with a fixed stretch: the anchors (x, y) in placement order."""
    rem = P.copy()
    anchors = []
    while rem.any():                                   # line 4: until P is covered
        ys, xs = np.nonzero(top(rem))                  # line 5: ⊤ of the uncovered points
        tcur = list(zip(xs.tolist(), ys.tolist()))     # row-major: ascending y
        anchors.extend(tcur)                           # line 6
        for (x, y) in tcur:                            # lines 7-8: Rem <- Rem \ Comp
            rem[y:y + m * s:s, x:x + n * s:s] = False
    return anchors


def row_classes(P: np.ndarray):
    """(polygonal, X): polygonal iff every row's columns are contiguous; X = the common difference
    of every multi-column row when each such row is one arithmetic progression with difference > 1
    and no row is contiguous with two or more columns (else X = None)."""
    polygonal, diffs, contiguous = True, set(), False
    for y in range(P.shape[0]):
        xs = np.nonzero(P[y])[0]
        if len(xs) < 2:
            continue
        d = np.unique(np.diff(xs))
        if len(d) == 1 and d[0] == 1:
            contiguous = True
            continue
        polygonal = False
        if len(d) == 1:
            diffs.add(int(d[0]))
        else:
            diffs.add(None)
    X = None
    if not polygonal and not contiguous and len(diffs) == 1 and None not in diffs:
        X = diffs.pop()
    return polygonal, X


def cost(P: np.ndarray, anchors, stretches, m: int, n: int) -> dict:
    """Def. 3 and Def. 4 for an arrangement (one stretch per block).  Raises if the covers do
    not union to P.  Comp points outside the mask grid are not in P (they count in phi_TD)."""
    if isinstance(stretches, int):
        stretches = [stretches] * len(anchors)
    lam = len(anchors)
    H, W = P.shape
    ext_y = max([H] + [y + (m - 1) * s + 1 for (x, y), s in zip(anchors, stretches)])
    ext_x = max([W] + [x + (n - 1) * s + 1 for (x, y), s in zip(anchors, stretches)])
    U = np.zeros((ext_y, ext_x), dtype=bool)           # ∪ Comp(TB_i)
    for (x, y), s in zip(anchors, stretches):
        U[y:y + m * s:s, x:x + n * s:s] = True
    Pe = np.zeros_like(U)
    Pe[:H, :W] = P
    if np.any(Pe & ~U):
        yy, xx = np.nonzero(Pe & ~U)
        raise ValueError(f"arrangement does not cover P: ({xx[0]}, {yy[0]}) uncovered")
    size_p = int(P.sum())
    phi_td = int((U & ~Pe).sum())                      # |(∪ Comp) \ P|
    phi_r = lam * m * n - size_p - phi_td
    phi_ru = Fraction(size_p, lam * m * n) if lam else Fraction(0)
    phi_cmr = sum((Fraction(1, s) for s in stretches), Fraction(0)) / lam if lam else Fraction(1)
    return {"lambda": lam, "points": size_p, "phi_td": phi_td, "phi_r": phi_r, "phi_ru": phi_ru,
            "phi_cmr": phi_cmr, "cost": Fraction(lam) / phi_cmr}


def stretch_candidates(P: np.ndarray) -> list:
    polygonal, X = row_classes(P)
    if polygonal:
        return [1]                                     # App. A
    if X is not None:
        return [d for d in range(1, X + 1) if X % d == 0]   # App. B: factors(X)
    return list(range(1, min(P.shape[0], GENERIC_STRETCH_CAP) + 1))


def select_stretch(P: np.ndarray, m: int, n: int) -> int:
    """Sec. 7.3.1: argmin over the candidates of lambda^s / phi_CMR^s; ties -> fewer blocks."""
    best = None
    for s in stretch_candidates(P):
        lam = len(poset_tile(P, m, n, s))
        c = Fraction(lam) / Fraction(1, s)
        if best is None or (c, lam) < (best[0], best[1]):
            best = (c, lam, s)
    return best[2]


def poset(P: np.ndarray, m: int, n: int, stretch: int = 0):
    """Alg. 1 with line 3's stretch selection (stretch 0) or a forced stretch: (anchors, s)."""
    s = stretch or select_stretch(P, m, n)
    return poset_tile(P, m, n, s), s


def naive_tile(P: np.ndarray, m: int, n: int) -> list:
    """App. C Def. 8: patches of m consecutive rows, tiled left to right with unit-stretch m x n
    blocks from the patch's leftmost non-zero column until its rightmost one is covered."""
    anchors = []
    for y0 in range(0, P.shape[0], m):
        cols = np.nonzero(P[y0:y0 + m].any(axis=0))[0]
        if len(cols) == 0:
            continue
        lo, hi = int(cols[0]), int(cols[-1])
        anchors.extend((x, y0) for x in range(lo, hi + 1, n))
    return anchors


def cover_count_direct(m: int, n: int, X: int, s: int) -> int:
    """App. B (stronger form P:967-977): |{(i, j) in Z_n x Z_m : kappa | (j - i)}|,
    kappa = X / gcd(s, X)."""
    kappa = X // math.gcd(s, X)
    return sum(1 for i in range(n) for j in range(m) if (j - i) % kappa == 0)


def _cover_sections(m: int, n: int, kappa: int, floor_limits: bool):
    ceil = lambda a, b: -(-a // b)
    up = (lambda a, b: a // b) if floor_limits else ceil
    pink = [ceil(m - n + 1, kappa) * n]
    blue = [m - k * kappa for k in range(ceil(m - n + 1, kappa), up(m - 1, kappa) + 1)]
    green = [n - k * kappa for k in range(1, up(n - 1, kappa) + 1)]
    return pink + blue + green


def cover_count_closed(m: int, n: int, kappa: int, floor_limits: bool = False) -> int:
    """App. B's f(kappa): the pink, blue and green sections, with the paper's
    ceiling upper limits (or floor limits, reading T-5)."""
    return sum(_cover_sections(m, n, kappa, floor_limits))


def cover_count_terms_nonnegative(m: int, n: int, kappa: int) -> bool:
    return all(t >= 0 for t in _cover_sections(m, n, kappa, False))


def naive_lambda_closed(r: int, l: int, h: int, lp: int, m: int, n: int) -> Fraction:
    """App. C Theorem: lambda_naive of a structured dense polygon (r, l, h, l')."""
    kappa = math.gcd(m, h)
    tau_m, tau_h = m // kappa, h // kappa
    alpha, beta = divmod(tau_m, tau_h)
    ceil = lambda a, b: -(-a // b)
    if beta == 0:
        per = tau_h * ceil(l + (alpha - 1) * lp, n)
    else:
        per = (beta - 1) * ceil(l + (alpha + 1) * lp, n) + (tau_h - beta + 1) * ceil(l + alpha * lp, n)
    return Fraction(r, tau_m) * per


def optimal_bruteforce(P: np.ndarray, m: int, n: int, stretches, budget: int = 2_000_000) -> dict:
    """Least-cost total cover (Def. 4) over anchors in P and one stretch from `stretches`
    (the SPEC's acceptance oracle): exhaustive branch and bound.  Tiny masks only."""
    pts = {(int(x), int(y)) for y, x in zip(*np.nonzero(P))}
    order = sorted(pts, key=lambda p: (p[1], p[0]))
    best = None
    for s in stretches:
        covers = {a: comp(a, s, m, n) & pts for a in order}
        bound = [None]
        steps = [0]

        def search(unc, k):
            steps[0] += 1
            if steps[0] > budget:
                raise RuntimeError("brute-force budget exceeded")
            if not unc:
                if bound[0] is None or k < bound[0]:
                    bound[0] = k
                return
            if bound[0] is not None and k + -(-len(unc) // (m * n)) >= bound[0]:
                return
            first = min(unc, key=lambda p: (p[1], p[0]))
            for a in order:
                if first in covers[a]:
                    search(unc - covers[a], k + 1)

        search(frozenset(pts), 0)
        c = Fraction(bound[0]) * s                     # lambda / phi_CMR with phi_CMR = 1/s
        if best is None or (c, bound[0]) < (best["cost"], best["lambda"]):
            best = {"cost": c, "lambda": bound[0], "stretch": s}
    return best


__all__ = ["points", "structured_polygon", "comp", "top", "poset_tile", "poset", "select_stretch",
           "stretch_candidates", "row_classes", "naive_tile", "cost", "cover_count_direct",
           "cover_count_closed", "cover_count_terms_nonnegative", "naive_lambda_closed", "optimal_bruteforce"]
