"""Host-side pins of the residue decomposition of strided rows.

The fused and unfused kernels run STRIDED_LOCAL(l) as two components -- the causal band
WINDOW(l-1, 0) in natural row order and the stride keys i - l m (m >= 1) as a dense strictly
causal block per residue class rho = i mod l in residue-major order (the paper's row classes
of equal residue) -- and address S / P of each component in the NATURAL ACSR order.
These tests re-derive that arithmetic independently and check it against the oracle's explicit
mask and ACSR (oracle/, fp64 enumeration), for every (N, l) shape the decomposition accepts.
"""
import numpy as np
import pytest

from oracle import oracle as O
from workloads import Pattern

SHAPES = [(1024, 16), (2048, 16), (512, 16), (256, 32), (8192, 128), (768, 12)]


def applicable(N, l):
    return l >= 2 and N % l == 0 and 2 <= N // l <= 128 and 128 % (N // l) == 0


@pytest.mark.parametrize("N,l", SHAPES)
def test_band_and_stride_partition_the_mask(N, l):
    if N > 2048:
        pytest.skip("explicit N x N mask too large for a quick CPU test")
    m = O.mask(Pattern("strided_local", N, stride=l, causal=1))
    i = np.arange(N)[:, None]
    j = np.arange(N)[None, :]
    band = (j <= i) & (i - j < l)
    stride = (j < i) & ((i - j) % l == 0) & (i - j >= l)
    assert not np.any(band & stride)
    assert np.array_equal(band | stride, m)


@pytest.mark.parametrize("N,l", SHAPES)
def test_residue_major_block_is_the_stride_component(N, l):
    if not applicable(N, l):
        pytest.skip("decomposition not applicable (N % l or N / l does not divide 128)")
    nk = N // l
    R = 128 // nk
    # permuted row r' = rho * nk + k is natural row rho + l k; its keys (internal pattern
    # kind 100) are permuted columns rho * nk + m, m < k
    rows, cols = [], []
    for rp in range(N):
        rho, k = divmod(rp, nk)
        i = rho + l * k
        for m in range(k):
            rows.append(i)
            cols.append(rho + l * m)
    got = np.zeros((N, N), dtype=bool)
    got[rows, cols] = True
    i = np.arange(N)[:, None]
    j = np.arange(N)[None, :]
    want = (j < i) & ((i - j) % l == 0)
    assert np.array_equal(got, want)
    # a 128-row tile of the residue-major order holds R whole classes, and its keys stay in the
    # same tile (one plan entry per query tile)
    for t in range(N // 128):
        rps = np.arange(128 * t, 128 * t + 128)
        assert set(np.unique(rps // nk)) == set(range(R * t, R * t + R))


@pytest.mark.parametrize("N,l", [s for s in SHAPES if s[0] <= 2048])
def test_component_offsets_in_natural_acsr(N, l):
    # stride key i - l (k - m) of row i sits at offset m of the natural ACSR row (k = i // l stride
    # entries first), band key j at offset k + rank of j in [max(0, i-l+1), i]
    p = Pattern("strided_local", N, stride=l, causal=1)
    _, _, row_ptr, rc = O.acsr(p, max_seg=4)
    assert rc == 0
    for i in list(range(0, min(N, 3 * l))) + list(range(N - 3, N)):
        cols = O.row_cols(p, i)
        k = i // l
        rho = i % l
        for m in range(k):
            assert cols[m] == rho + l * m
        lo = max(0, i - l + 1)
        for x, j in enumerate(range(lo, i + 1)):
            assert cols[k + x] == j
        assert len(cols) == k + (i - lo + 1) == row_ptr[i + 1] - row_ptr[i]
