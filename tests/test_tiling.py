"""The library's tiling analysis (splat_poset_tile / splat_naive_tile / splat_tiling_cost_eval, host
C++ in csrc/tiling.cpp) against the tiling oracle (oracle/tiling.py): identical anchors, stretch
and Def. 3 / Def. 4 costs on every pattern kind, and the paper's Fig. 12 comparison (poset vs
naive block counts at N = 1024).  Host-only entry points: no GPU needed."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import tiling as T
from paper_2407_16847_b200 import build as B
from paper_2407_16847_b200 import splat as S
from workloads import Pattern


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()
    S.lib()


def patterns(N):
    yield Pattern("window", N, lo=2, hi=2)
    yield Pattern("window", N, lo=N // 4, hi=1)
    yield Pattern("window", N, lo=N - 1, hi=N - 1)
    yield Pattern("blocked", N, block=4)
    yield Pattern("blocked", N, block=N // 2 + 1)
    yield Pattern("strided", N, stride=4)
    yield Pattern("strided", N, stride=6)
    yield Pattern("dilated", N, stride=3, radius=3)
    yield Pattern("global_local", N, lo=3, hi=3, n_global=2)
    yield Pattern("bigbird", N, block=4, radius=1)
    yield Pattern("strided_local", N, stride=4, causal=1)


def same_cost(got, want):
    for k in ("lambda", "points", "phi_td", "phi_r"):
        assert got[k] == want[k], k
    for k in ("phi_ru", "phi_cmr", "cost"):
        assert got[k] == pytest.approx(float(want[k]), rel=1e-15, abs=0), k


@pytest.mark.parametrize("N", [16, 24, 40])
@pytest.mark.parametrize("m,n", [(2, 2), (3, 2), (2, 3), (4, 4), (1, 5), (8, 4)])
def test_poset_matches_oracle(N, m, n):
    for p in patterns(N):
        P = T.points(p)
        want_anchors, want_s = T.poset(P, m, n)
        anchors, cost = S.splat_poset_tile(p, m, n)
        assert cost["stretch"] == want_s, p
        assert [tuple(a) for a in anchors.tolist()] == want_anchors, p
        same_cost(cost, T.cost(P, want_anchors, want_s, m, n))


@pytest.mark.parametrize("N", [16, 40])
@pytest.mark.parametrize("m,n", [(2, 2), (3, 2), (4, 8)])
def test_forced_stretch_and_naive_match_oracle(N, m, n):
    for p in patterns(N):
        P = T.points(p)
        for s in (1, 2, 3):
            anchors, cost = S.splat_poset_tile(p, m, n, s)
            want = T.poset_tile(P, m, n, s)
            assert [tuple(a) for a in anchors.tolist()] == want
            same_cost(cost, T.cost(P, want, s, m, n))
        anchors, cost = S.splat_naive_tile(p, m, n)
        want = T.naive_tile(P, m, n)
        assert [tuple(a) for a in anchors.tolist()] == want
        same_cost(cost, T.cost(P, want, 1, m, n))


def test_cost_eval_matches_oracle_and_rejects_non_covers():
    rng = np.random.default_rng(3)
    p = Pattern("window", 32, lo=3, hi=5)
    P = T.points(p)
    for _ in range(20):
        m, n, s = int(rng.integers(1, 5)), int(rng.integers(1, 5)), int(rng.integers(1, 4))
        anchors = T.poset_tile(P, m, n, s)
        extra = [(int(rng.integers(0, 40)), int(rng.integers(0, 40))) for _ in range(5)]
        arr = anchors + extra                       # overlapping and out-of-mask blocks
        same_cost(S.splat_tiling_cost_eval(p, m, n, s, arr), T.cost(P, arr, s, m, n))
        missing = arr[1:]
        try:
            T.cost(P, missing, s, m, n)
            covered = True
        except ValueError:
            covered = False
        if not covered:
            with pytest.raises(S.SplatError) as e:
                S.splat_tiling_cost_eval(p, m, n, s, missing)
            assert e.value.status == 1 and "uncovered" in str(e.value)


def test_fig6_examples_through_the_library():
    # the strided 4x4 mask (X = 2) with 2x2 blocks
    p = Pattern("strided", 4, stride=2)
    anchors, c = S.splat_poset_tile(p, 2, 2)
    assert (c["stretch"], c["lambda"], c["phi_ru"], c["phi_cmr"], c["cost"]) == (2, 2, 1.0, 0.5, 4.0)
    assert anchors.tolist() == [[0, 0], [1, 1]]
    _, c = S.splat_poset_tile(p, 2, 2, 1)
    assert (c["lambda"], c["phi_td"], c["phi_r"], c["phi_ru"], c["phi_cmr"]) == (4, 8, 0, 0.5, 1.0)


def test_argument_errors():
    p = Pattern("window", 16, lo=1, hi=1)
    for bad in [(0, 2, 0), (2, 0, 0), (2, 2, -1), (2, 2, 17), (5000, 2, 0)]:
        with pytest.raises(S.SplatError) as e:
            S.splat_poset_tile(p, *bad)
        assert e.value.status == 1
    with pytest.raises(S.SplatError) as e:
        S.splat_poset_tile(Pattern("window", 8193, lo=1, hi=1), 2, 2)
    assert e.value.status == 4
    with pytest.raises(S.SplatError) as e:
        S.splat_tiling_cost_eval(p, 2, 2, 1, [(-1, 0)])
    assert e.value.status == 1


@pytest.mark.parametrize("N", [256])
def test_poset_matches_oracle_mid_size(N):
    for p in (Pattern("window", N, lo=37, hi=37), Pattern("blocked", N, block=32), Pattern("strided", N, stride=8)):
        P = T.points(p)
        want, s = T.poset(P, 16, 16)
        anchors, cost = S.splat_poset_tile(p, 16, 16)
        assert cost["stretch"] == s and [tuple(a) for a in anchors.tolist()] == want


def test_fig12_poset_vs_naive_at_1024():
    # Fig. 12: N = 1024, every density of the window (radius r) and block-diagonal
    # (w | N) masks; square 16 x 16 blocks.  Poset tiling never uses more blocks than the naive
    # tiling, and the naive count of the block diagonal equals App. C's closed form
    # (h = l' = l = w, r = N / w)
    N, m, n = 1024, 16, 16
    ratios = []
    for r in list(range(0, 64)) + list(range(64, N, 37)) + [N - 1]:
        p = Pattern("window", N, lo=r, hi=r)
        lp, ln = S.splat_poset_tile(p, m, n)[1]["lambda"], S.splat_naive_tile(p, m, n)[1]["lambda"]
        assert lp <= ln, r
        ratios.append(ln / lp)
    for w in [1 << k for k in range(11)]:
        p = Pattern("blocked", N, block=w)
        lp, ln = S.splat_poset_tile(p, m, n)[1]["lambda"], S.splat_naive_tile(p, m, n)[1]["lambda"]
        assert lp <= ln
        assert Fraction(ln) == T.naive_lambda_closed(N // w, w, w, w, m, n)
    assert max(ratios) > 1.2          # poset saves blocks on narrow bands


def test_poset_can_exceed_naive_for_non_square_blocks():
    # App. C ends with lambda_poset <= lambda_naive ("the Naive Tiling Algorithm is essentially the
    # Poset Tiling Algorithm applied to each patch").  Both implementations agree that
    # this fails for wide blocks on a band: N = 8, window radius 2, m x n = 2 x 3 (reading T-7)
    p = Pattern("window", 8, lo=2, hi=2)
    P = T.points(p)
    assert len(T.poset_tile(P, 2, 3, 1)) == 9 and len(T.naive_tile(P, 2, 3)) == 8
    assert S.splat_poset_tile(p, 2, 3)[1]["lambda"] == 9 and S.splat_naive_tile(p, 2, 3)[1]["lambda"] == 8
