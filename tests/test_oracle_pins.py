"""Pins for the fp64 CPU oracle (oracle/), runnable without a GPU.

Each test ties the oracle to something other than itself: a worked example
printed in the paper or SPEC (tests/golden/paper_examples.json, cited), a
closed form, a textbook/library special case (torch SDPA in fp64), or brute
force on tiny inputs.  A plausible mistake anywhere in the oracle (wrong sign
or index in a predicate, a dropped term in the softmax, a transposed operand
in the scores or the output sum) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from workloads import CONFIG_BY_NAME, CONFIGS, Pattern, make_random

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def triplet_to_run(a, b, nnzs):
    """Paper affine indices (a, b, nnzs) -> (start, step, count); a = 1/step, b = -start/step."""
    step = round(1.0 / a)
    return (round(-b * step), step, nnzs)


# --------------------------------------------------------------------------
# Worked examples of the paper / SPEC
# --------------------------------------------------------------------------

def test_affine_compressible_example():
    for ex in GOLD["affine_compressible"]:
        runs = O.runs_from_cols(ex["cols"])
        assert runs == [triplet_to_run(ex["a"], ex["b"], ex["nnzs"])], ex["cite"]
        m = np.zeros((1, max(ex["cols"]) + 1), np.uint8)
        m[0, ex["cols"]] = 1
        ok, a, b, nnzs, _ = O.regularity(m)
        assert ok and a[0] == ex["a"] and b[0] == ex["b"] and nnzs[0] == ex["nnzs"]


def test_not_compressible_example():
    for ex in GOLD["not_compressible"]:
        m = np.zeros((1, max(ex["cols"]) + 1), np.uint8)
        m[0, ex["cols"]] = 1
        ok, _, _, _, bad = O.regularity(m)
        assert not ok and bad == (0, ex["bad_col"]), ex["cite"]
        assert len(O.runs_from_cols(ex["cols"])) == 2


def test_value14_example():
    ex = GOLD["value14"]
    start, step, count = triplet_to_run(ex["a"], ex["b"], ex["nnzs"])
    cols = [start + step * s for s in range(count)]
    assert O.runs_from_cols(cols) == [(start, step, count)]
    # (sparse_i - b) / a = dense column
    assert start + step * ex["sparse_i"] == ex["dense"] == (ex["sparse_i"] - ex["b"]) / ex["a"]
    assert O.fast_index(start, step, count, ex["dense"]) == ex["sparse_i"]


def test_fast_index_examples():
    for ex in GOLD["fast_index"]:
        start, step, count = triplet_to_run(ex["a"], ex["b"], ex["nnzs"])
        got = O.fast_index(start, step, count, ex["dense"])
        assert got == (-1 if ex["sparse"] is None else ex["sparse"]), ex["cite"]
    for ex in GOLD["sparse_to_dense"]:
        start, step, _ = triplet_to_run(ex["a"], ex["b"], 1)
        assert start + step * ex["sparse"] == ex["dense"], ex["cite"]


def test_fast_index_is_inverse_of_decode():
    # dense<->sparse maps are mutually inverse on every row of every pattern
    for p in [Pattern("strided", 40, stride=3), Pattern("window", 40, lo=3, hi=5),
              Pattern("dilated", 40, stride=4, radius=3)]:
        seg, nseg, _, _ = O.acsr(p)
        for i in range(p.seq_len):
            start, step, count = seg[i, 0]
            for c in range(p.seq_len):
                s = O.fast_index(int(start), int(step), int(count), c)
                assert (s >= 0) == O.pred(p, i, c)
                if s >= 0:
                    assert start + step * s == c


def test_softmax_examples():
    for ex in GOLD["softmax"]:
        x = np.array(ex["in"])
        P = O.softmax_rows(x, np.array([0, len(x)]))
        assert np.max(np.abs(P - np.array(ex["out"]))) <= ex["tol"], ex["cite"]


def test_spec_pattern_examples():
    for ex in GOLD["patterns"]:
        p = Pattern(**ex["pattern"])
        want = np.array([[int(ch) for ch in row] for row in ex["mask"]], np.uint8)
        assert np.array_equal(O.mask(p), want), ex["cite"]


@pytest.mark.parametrize("name", ["tiny", "longformer", "bigbird", "sparse_transformer", "mistral"])
def test_config_nnz_closed_forms(name):
    ex = next(e for e in GOLD["config_nnz"] if e["config"] == name)
    p = CONFIG_BY_NAME[name].pattern
    _, nseg, row_ptr, rc = O.acsr(p)
    assert rc == 0 and int(row_ptr[-1]) == ex["nnz"], ex["cite"]


@pytest.mark.parametrize("N", [8, 12, 16, 32, 64])
def test_paper_grid_closed_forms(N):
    # window radius r: N(2r+1) - r(r+1) (r < N); blocked w | N: N*w; strided X | N: N^2/X
    for r in range(0, N):
        _, _, rp, _ = O.acsr(Pattern("window", N, lo=r, hi=r))
        assert rp[-1] == N * (2 * r + 1) - r * (r + 1)
    for w in [w for w in range(1, N + 1) if N % w == 0]:
        assert O.acsr(Pattern("blocked", N, block=w))[2][-1] == N * w
        assert O.acsr(Pattern("strided", N, stride=w))[2][-1] == N * N // w


# --------------------------------------------------------------------------
# Closed-form canonical segments, an independent derivation
# of the same runs, vs the oracle's enumerate-then-greedy construction.
# --------------------------------------------------------------------------

def closed_form_segments(p, i):
    N = p.seq_len
    out = []

    def add(start, step, count):
        if count <= 0:
            return
        out.append((start, 1 if count == 1 else step, count))

    if p.kind == "window":
        s, e = max(0, i - p.lo), min(N - 1, i + p.hi)
        add(s, 1, e - s + 1)
    elif p.kind == "blocked":
        b0 = (i // p.block) * p.block
        add(b0, 1, min(p.block, N - b0))
    elif p.kind == "strided":
        r = i % p.stride
        add(r, p.stride, (N - 1 - r) // p.stride + 1)
    elif p.kind == "dilated":
        dl, rho = p.stride, p.radius
        start = i - dl * min(rho, i // dl)
        end = i + dl * min(rho, (N - 1 - i) // dl)
        add(start, dl, (end - start) // dl + 1)
    elif p.kind == "global_local":
        g = p.n_global
        s, e = max(0, i - p.lo), min(N - 1, i + p.hi)
        if i < g:
            add(0, 1, N)
        elif s <= g:
            add(0, 1, max(e, g - 1) + 1)
        else:
            add(0, 1, g)
            add(s, 1, e - s + 1)
    elif p.kind == "bigbird":
        bs, r = p.block, p.radius
        nb = -(-N // bs)
        qb = i // bs
        if qb in (0, nb - 1):
            add(0, 1, N)
        else:
            blocks = sorted({0, nb - 1} | {b for b in range(qb - r, qb + r + 1) if 0 <= b < nb})
            runs = []
            for b in blocks:
                if runs and runs[-1][1] == b - 1:
                    runs[-1][1] = b
                else:
                    runs.append([b, b])
            for b0, b1 in runs:
                c0, c1 = b0 * bs, min(N, (b1 + 1) * bs)
                add(c0, 1, c1 - c0)
    elif p.kind == "strided_local":
        l = p.stride
        if i < l or l == 1:
            add(0, 1, i + 1)
        elif i // l == 1:
            add(i - l, 1, l + 1)
        else:
            add(i % l, l, i // l)
            add(i - l + 1, 1, l)
    return out


def small_patterns(N):
    for lo in range(0, N + 1, max(1, N // 6)):
        for hi in range(0, N + 1, max(1, N // 5)):
            yield Pattern("window", N, lo=lo, hi=hi)
    for w in range(1, N + 1):
        yield Pattern("blocked", N, block=w)
        yield Pattern("strided", N, stride=w)
        yield Pattern("strided_local", N, stride=w, causal=1)
    for dl in range(1, N + 1, 2):
        for rho in range(0, N // dl + 1, max(1, N // (3 * dl) or 1)):
            yield Pattern("dilated", N, stride=dl, radius=rho)
    for g in [0, 2, 3, N // 2]:
        for lo in range(0, N, max(1, N // 4)):
            yield Pattern("global_local", N, lo=lo, hi=lo, n_global=g)
    for bs in range(2, N + 1):
        for r in (0, 1, 2):
            yield Pattern("bigbird", N, block=bs, radius=r)


@pytest.mark.parametrize("N", [1, 2, 5, 16, 23, 32])
def test_closed_form_segments_equal_greedy(N):
    for p in small_patterns(N):
        seg, nseg, row_ptr, rc = O.acsr(p, max_seg=8)
        assert rc == 0, p
        for i in range(N):
            got = [tuple(int(v) for v in seg[i, s]) for s in range(nseg[i])]
            assert got == closed_form_segments(p, i), (p, i)
            assert row_ptr[i + 1] - row_ptr[i] == sum(c for _, _, c in got)


def test_degenerate_greedy_cases_documented():
    # g = 1 global+local and bs = 1 BigBird: greedy pairs an isolated column with
    # the next one (reading A-11) -> the library rejects them as UNSUPPORTED.
    p = Pattern("global_local", 16, lo=2, hi=2, n_global=1)
    seg, nseg, _, _ = O.acsr(p, max_seg=8)
    assert tuple(seg[8, 0]) == (0, 6, 2)       # {0, 6} paired with step 6
    p = Pattern("bigbird", 16, block=1, radius=1)
    assert O.acsr(p, max_seg=8)[1].max() >= 2


def test_paper_kinds_are_regular():
    # every generated paper pattern is regular (Def. 1)
    for N in (7, 16, 33):
        for w in range(1, N + 1):
            for p in (Pattern("window", N, lo=w, hi=w), Pattern("blocked", N, block=w),
                      Pattern("strided", N, stride=w)):
                ok, a, b, nnzs, _ = O.regularity(O.mask(p))
                assert ok, p
                seg, nseg, _, _ = O.acsr(p, max_seg=4)
                assert nseg.max() == 1
                for i in range(N):
                    assert triplet_to_run(a[i], b[i], int(nnzs[i])) == tuple(seg[i, 0])


def test_regularity_rejects_flipped_interior_bit():
    # flipping off one interior bit of a run makes the row irregular
    p = Pattern("window", 16, lo=3, hi=3)
    m = O.mask(p)
    m[9, 8] = 0
    ok, _, _, _, bad = O.regularity(m)
    assert not ok and bad == (9, 9)


# --------------------------------------------------------------------------
# Attention: brute force dense fp64 (torch) and library special cases
# --------------------------------------------------------------------------

def dense_masked_attention(q, k, v, m, scale):
    """SPEC S:439-447 dense_reference_mhsa in torch fp64 (masked -> -inf, empty row -> 0)."""
    s = scale * (q @ k.T)
    mm = torch.from_numpy(m.astype(bool))
    s = s.masked_fill(~mm, float("-inf"))
    p = torch.softmax(s, dim=-1)
    p = torch.nan_to_num(p, nan=0.0)
    return p @ v, s, p


PIN_PATTERNS = [
    Pattern("window", 64, lo=5, hi=9),
    Pattern("blocked", 48, block=16),
    Pattern("strided", 40, stride=6),
    Pattern("dilated", 50, stride=3, radius=4),
    Pattern("global_local", 64, lo=7, hi=7, n_global=4),
    Pattern("bigbird", 64, block=8, radius=1),
    Pattern("strided_local", 64, stride=8, causal=1),
]


@pytest.mark.parametrize("p", PIN_PATTERNS, ids=lambda p: p.kind)
def test_attention_matches_dense_brute_force(p):
    N, d = p.seq_len, 16
    q = make_random((N, d), 11, torch.float64)
    k = make_random((N, d), 12, torch.float64)
    v = make_random((N, d), 13, torch.float64)
    scale = 1 / math.sqrt(d)
    o, S, P = O.attention(p, q, k, v, scale, want_sp=True, nthreads=3)
    m = O.mask(p)
    o_ref, s_ref, p_ref = dense_masked_attention(q, k, v, m, scale)
    assert np.max(np.abs(o - o_ref.numpy())) < 1e-12
    # S and P in ACSR (row-compressed row-major, Fig. 5(b)) order
    idx = np.nonzero(m)
    assert np.max(np.abs(S - s_ref.numpy()[idx])) < 1e-12
    assert np.max(np.abs(P - p_ref.numpy()[idx])) < 1e-12
    # softmax step alone agrees with the fused evaluation; rows sum to 1
    _, _, row_ptr, _ = O.acsr(p, max_seg=8)
    assert np.max(np.abs(O.softmax_rows(S, row_ptr) - P)) < 1e-15
    sums = np.add.reduceat(P, row_ptr[:-1])
    assert np.max(np.abs(sums - 1)) < 1e-12


def test_attention_not_symmetric_in_q_k():
    # a transposed score operand (k q^T) would pass symmetric masks only
    p = Pattern("strided_local", 32, stride=4, causal=1)
    q = make_random((32, 8), 1, torch.float64)
    k = make_random((32, 8), 2, torch.float64)
    v = make_random((32, 8), 3, torch.float64)
    o = O.attention(p, q, k, v, 0.5)
    o_ref, _, _ = dense_masked_attention(q, k, v, O.mask(p), 0.5)
    assert np.max(np.abs(o - o_ref.numpy())) < 1e-12


@pytest.mark.parametrize("p", [Pattern("window", 40, lo=40, hi=40), Pattern("strided", 40, stride=1),
                               Pattern("blocked", 40, block=40)], ids=["window", "strided", "blocked"])
def test_full_density_is_library_attention(p):
    # full mask == dense attention (torch SDPA, fp64)
    N, d = 40, 24
    q = make_random((N, d), 21, torch.float64, 3.0)
    k = make_random((N, d), 22, torch.float64)
    v = make_random((N, d), 23, torch.float64)
    o = O.attention(p, q, k, v, 0.3)
    ref = torch.nn.functional.scaled_dot_product_attention(q[None], k[None], v[None], scale=0.3)[0]
    assert np.max(np.abs(o - ref.numpy())) < 1e-12


def test_diagonal_mask_returns_v():
    # diagonal mask -> one-hot softmax -> O = V exactly
    p = Pattern("window", 30, lo=0, hi=0)
    v = make_random((30, 8), 5, torch.float64)
    o = O.attention(p, make_random((30, 8), 6, torch.float64), make_random((30, 8), 7, torch.float64), v, 1.0)
    assert np.array_equal(o, v.numpy())


@pytest.mark.parametrize("p", PIN_PATTERNS, ids=lambda p: p.kind)
def test_uniform_attention_counts_columns(p):
    # Q = 0 -> p_ij = 1/nnz_i ; V one-hot V[j,t] = [t == j mod d]
    #   -> O_i[t] = #{j in cols(i): j = t mod d} / nnz_i   (exact rational)
    N, d = p.seq_len, 8
    q = torch.zeros(N, d, dtype=torch.float64)
    k = make_random((N, d), 9, torch.float64)
    v = torch.zeros(N, d, dtype=torch.float64)
    v[torch.arange(N), torch.arange(N) % d] = 1.0
    o = O.attention(p, q, k, v, 1.0)
    m = O.mask(p)
    for i in range(N):
        cols = np.nonzero(m[i])[0]
        want = np.bincount(cols % d, minlength=d) / len(cols)
        assert np.max(np.abs(o[i] - want)) < 1e-15


def test_row_block_and_threads_do_not_change_results():
    p = CONFIG_BY_NAME["tiny"].pattern
    q, k, v = (make_random((256, 64), s, torch.float32) for s in (1, 2, 3))
    a = O.attention(p, q, k, v, 0.125, nthreads=1)
    b = O.attention(p, q, k, v, 0.125, nthreads=7)
    c = O.attention(p, q, k, v, 0.125, rows=(100, 180), nthreads=2)
    assert np.array_equal(a, b) and np.array_equal(a[100:180], c)
