"""Pins of the tiling oracle (oracle/tiling.py) to the paper, not to itself.

Each test names what fixes the expected value: a number the paper prints for Fig. 6 (Sec. 7.2,
P:283-314), an appendix closed form checked against enumeration (App. B, App. C
P:997-1017), a brute-force least-cost cover on a tiny mask (Theorem 1 P:333-336 and App. C.2
P:1106-1111), or a statement of the paper (App. A, Sec. 7.3.1).
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import tiling as T
from workloads import Pattern


def strided_grid(N, X):
    y, x = np.mgrid[0:N, 0:N]
    return (x - y) % X == 0


def test_comp_fig6g():
    # Sec. 7.2: Cov(TB_0) = {(0,0),(0,2),(2,0),(2,2)}, Cov(TB_1) = {(1,1),(3,1),(1,3),(3,3)}
    assert T.comp((0, 0), 2, 2, 2) == {(0, 0), (0, 2), (2, 0), (2, 2)}
    assert T.comp((1, 1), 2, 2, 2) == {(1, 1), (3, 1), (1, 3), (3, 3)}
    assert T.comp((0, 0), 1, 2, 2) == {(0, 0), (1, 0), (0, 1), (1, 1)}


def test_fig6_g_and_h_costs():
    # reuse of (g) = 1 and of (h) = (2x2 - 8/4 - 0)/(2x2) = 1/2; coalescing (g) = 1/2,
    # (h) = 1 -- both 4x4 strided (X = 2) arrangements with 2x2 blocks; (h) uses 4 blocks
    P = strided_grid(4, 2)
    g = T.cost(P, [(0, 0), (1, 1)], 2, 2, 2)
    assert (g["phi_ru"], g["phi_cmr"], g["lambda"], g["cost"]) == (1, Fraction(1, 2), 2, 4)
    h_anchors, s = T.poset(P, 2, 2, stretch=1)
    h = T.cost(P, h_anchors, s, 2, 2)
    assert (h["lambda"], h["phi_td"], h["phi_r"]) == (4, 8, 0)          # phi_TD / lambda = 8/4
    assert (h["phi_ru"], h["phi_cmr"], h["cost"]) == (Fraction(1, 2), 1, 4)
    # Sec. 7.3.1: stretch 2 turns the 4-block arrangement into the 2-block one of (g)
    anchors, s = T.poset(P, 2, 2)
    assert s == 2 and sorted(anchors) == [(0, 0), (1, 1)]


def test_top_definition_cases():
    g = np.zeros((4, 4), dtype=bool)
    g[0, 1] = g[1, 0] = True                             # incomparable: both minimal
    assert set(zip(*np.nonzero(T.top(g)))) == {(0, 1), (1, 0)}
    g[:] = False
    g[0, 0] = g[1, 1] = True                             # (0,0) comes before (1,1)
    assert set(zip(*np.nonzero(T.top(g)))) == {(0, 0)}
    g[:] = False
    g[2:4, 2:4] = True
    assert set(zip(*np.nonzero(T.top(g)))) == {(2, 2)}
    # brute-force definition on random sets
    rng = np.random.default_rng(5)
    for _ in range(20):
        r = rng.random((9, 7)) < 0.3
        pts = [(x, y) for y, x in zip(*np.nonzero(r))]
        want = {(x, y) for (x, y) in pts
                if not any((q != (x, y)) and q[0] <= x and q[1] <= y for q in pts)}
        got = {(int(x), int(y)) for y, x in zip(*np.nonzero(T.top(r)))}
        assert got == want


def test_poset_blocked_4x4_is_optimal():
    P = T.points(Pattern("blocked", 4, block=2))
    anchors, s = T.poset(P, 2, 2)
    assert s == 1 and anchors == [(0, 0), (2, 2)]
    assert T.optimal_bruteforce(P, 2, 2, [1])["lambda"] == 2


def test_single_point():
    P = np.zeros((8, 8), dtype=bool)
    P[7, 5] = True
    assert T.poset(P, 2, 2)[0] == [(5, 7)]


@pytest.mark.parametrize("m,n", [(1, 1), (2, 2), (3, 2), (2, 3), (4, 4)])
def test_cover_count_direct_matches_enumeration(m, n):
    # App. B (P:943-955 and the stronger form P:967-977): a block anchored on the strided mask,
    # stretch s, covers f(kappa) points, kappa = X / gcd(s, X) -- counted here by enumerating Comp ∩ P
    for X in range(1, 7):
        P = strided_grid(40, X)
        for s in range(1, 7):
            for ax, ay in [(0, 0), (1, 1), (3, 0), (0, X)]:
                if not P[ay, ax]:
                    continue
                got = sum(1 for (x, y) in T.comp((ax, ay), s, m, n) if P[y, x])
                assert got == T.cover_count_direct(m, n, X, s), (m, n, X, s, ax, ay)


def test_cover_count_closed_form():
    # App. B's f(kappa) against enumeration of {(i, j) in Z_n x Z_m : kappa | (j - i)}, for
    # m >= n (the pink section j - i in {0..m-n} needs it).  The upper limits ceil((m-1)/kappa) and
    # ceil((n-1)/kappa) add one negative term when kappa does not divide m-1 (n-1); the formula
    # holds wherever every term is non-negative (reading T-5), and always with floor limits
    hits = 0
    for m in range(1, 10):
        for n in range(1, m + 1):
            for kappa in range(1, 10):
                want = sum(1 for i in range(n) for j in range(m) if (j - i) % kappa == 0)
                assert T.cover_count_closed(m, n, kappa, floor_limits=True) == want, (m, n, kappa)
                if T.cover_count_terms_nonnegative(m, n, kappa):
                    assert T.cover_count_closed(m, n, kappa) == want, (m, n, kappa)
                    hits += 1
    assert hits > 100


def test_cover_count_stretch_X_full():
    # P:963 reasoning: stretch = X (kappa = 1) makes every thread of the block hit the pattern
    for m, n, X in [(2, 2, 2), (3, 4, 4), (4, 4, 6)]:
        assert T.cover_count_direct(m, n, X, X) == m * n


@pytest.mark.parametrize("r,l,h,lp,m,n", [
    (4, 4, 2, 2, 2, 2),      # SPEC example: blocked staircase -> 8 blocks
    (8, 3, 1, 1, 2, 2),      # window (h = l' = 1, l = 2w + 1) -> 8
    (12, 5, 1, 1, 4, 2), (12, 8, 2, 2, 4, 4), (6, 8, 4, 4, 2, 4), (12, 6, 3, 3, 2, 2),
    (12, 6, 3, 3, 4, 2), (24, 9, 3, 3, 6, 4), (20, 16, 8, 8, 4, 4), (30, 10, 5, 5, 3, 4),
    (18, 5, 2, 2, 6, 3), (16, 7, 3, 2, 4, 5), (15, 4, 2, 2, 5, 3),
])
def test_naive_lambda_closed_form(r, l, h, lp, m, n):
    # App. C Theorem against Def. 8 applied to the Def. 7 polygon
    P = T.structured_polygon(r, l, h, lp)
    kappa = math.gcd(m, h)
    if r % (m // kappa):
        pytest.skip("r not a multiple of tau_m")
    assert Fraction(len(T.naive_tile(P, m, n))) == T.naive_lambda_closed(r, l, h, lp, m, n)


def test_naive_spec_examples():
    assert len(T.naive_tile(T.points(Pattern("window", 8, lo=1, hi=1)), 2, 2)) == 8
    assert len(T.naive_tile(np.ones((4, 4), dtype=bool), 2, 2)) == 4


def _window_block_masks(N):
    for r in range(N):
        yield T.points(Pattern("window", N, lo=r, hi=r))
    for w in range(1, N + 1):
        yield T.points(Pattern("blocked", N, block=w))


@pytest.mark.parametrize("N", [4, 5, 6])
def test_theorem1_bound_bruteforce(N):
    # Theorem 1: Cost(poset) / Cost(opt) <= 1 + m / l, l = most points in a row
    m = n = 2
    for P in _window_block_masks(N):
        anchors, s = T.poset(P, m, n)
        c = T.cost(P, anchors, s, m, n)["cost"]
        opt = T.optimal_bruteforce(P, m, n, [1, 2])["cost"]
        l = int(P.sum(axis=1).max())
        assert opt <= c <= opt * (1 + Fraction(m, l))


@pytest.mark.parametrize("N,X", [(4, 2), (6, 2), (6, 3), (8, 2), (8, 4)])
def test_strided_optimality_bruteforce(N, X):
    # App. C.2: for the strided pattern the selected-stretch poset cost is optimal
    P = strided_grid(N, X)
    anchors, s = T.poset(P, 2, 2)
    c = T.cost(P, anchors, s, 2, 2)["cost"]
    divisors = [d for d in range(1, X + 1) if X % d == 0]
    assert c == T.optimal_bruteforce(P, 2, 2, divisors)["cost"]


def _cov_gain(P, m, n, smax):
    """anchors of P whose block covers more points at some s > 1 than at s = 1"""
    pts = {(int(x), int(y)) for y, x in zip(*np.nonzero(P))}
    out = []
    for a in sorted(pts):
        c1 = len(T.comp(a, 1, m, n) & pts)
        if any(len(T.comp(a, s, m, n) & pts) > c1 for s in range(2, smax + 1)):
            out.append(a)
    return out


def test_appendix_a_stretching_polygons_shrinks_cover():
    # App. A: for a polygonal mask and an anchor in P, |Cov| is largest at s = 1.
    # True for an axis-aligned rectangle (the proof's "right or bottom edge" case) ...
    P = np.zeros((12, 12), dtype=bool)
    P[2:9, 3:11] = True
    assert _cov_gain(P, 3, 3, 4) == []
    # ... and for every window band ...
    for r in range(10):
        assert _cov_gain(T.points(Pattern("window", 10, lo=r, hi=r)), 3, 3, 4) == []
    # ... but the block-diagonal mask is a union of squares: a stretched block anchored near the
    # corner of one square reaches into the next one (reading T-6)
    assert (3, 0) in _cov_gain(T.points(Pattern("blocked", 10, block=4)), 3, 3, 4)


def test_stretch_one_is_best_for_polygons():
    # the consequence Sec. 7.3.1 draws from App. A: for windowed and blocked masks poset
    # tiling uses the fewest blocks at stretch 1
    for N in (8, 12):
        for P in _window_block_masks(N):
            l1 = len(T.poset_tile(P, 2, 2, 1))
            assert all(l1 <= len(T.poset_tile(P, 2, 2, s)) for s in range(2, 5))


def test_appendix_b_lambda_depends_on_gcd_and_falls():
    # App. B: lambda^s decreases as gcd(s, X) increases.  The proof's count
    # lambda^s = |P| / f(kappa) ignores the mask's edges and f(kappa) is flat once kappa >= m, n
    # (a 2x2 block then covers its diagonal only), so compare stretches whose per-block cover
    # differs, on a mask large enough for the interior to dominate
    for X in (2, 3, 4, 6):
        P = strided_grid(48, X)
        lam = {s: len(T.poset_tile(P, 2, 2, s)) for s in range(1, X + 1)}
        for s1 in lam:
            for s2 in lam:
                g1, g2 = math.gcd(s1, X), math.gcd(s2, X)
                f1, f2 = T.cover_count_direct(2, 2, X, s1), T.cover_count_direct(2, 2, X, s2)
                if g1 < g2 and g2 % g1 == 0 and f2 > f1:
                    assert lam[s2] < lam[s1], (X, s1, s2, lam)


def test_poset_total_cover_and_anchors_in_p():
    rng = np.random.default_rng(11)
    for _ in range(10):
        P = rng.random((12, 12)) < 0.35
        for m, n in [(2, 2), (3, 2), (1, 4)]:
            anchors, s = T.poset(P, m, n, stretch=1)
            T.cost(P, anchors, s, m, n)                  # raises unless the covers union to P
            assert all(P[y, x] for x, y in anchors)
