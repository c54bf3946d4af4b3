"""CPU tests of the C-ABI library: it loads, exports every symbol of
include/splat.h, validates descriptors, and its host logic (closed-form ACSR
runs -- the same function the GPU build kernel evaluates -- and the tile
planner) agrees bit-exactly with the oracle.  No compute calls (no GPU)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_2407_16847_b200 import build as B
from paper_2407_16847_b200 import splat as S
from workloads import CONFIGS, Pattern

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()
    S.lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "splat.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(splat_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    declared = header_symbols()
    assert set(declared) == set(S.EXPORTS)
    out = subprocess.check_output(["nm", "-D", "--defined-only", S.LIB_PATH]).decode()
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for name in declared:
        assert name in exported, name
        assert hasattr(ctypes.CDLL(S.LIB_PATH), name)


def test_library_has_sm100a_code():
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", S.LIB_PATH]).decode()
    assert "sm_100a" in out


def _err(pattern):
    with pytest.raises(S.SplatError) as e:
        S.Acsr(pattern, device=-1)
    return e.value.status


def test_descriptor_validation():
    assert _err(Pattern("window", 0, lo=1, hi=1)) == 1               # N < 1
    assert _err(Pattern("window", 16, lo=17, hi=1)) == 1              # > N
    assert _err(Pattern("blocked", 16, block=0)) == 1                 # <= 0
    assert _err(Pattern("strided", 16, stride=3, block=2)) == 1       # unused field set
    assert _err(Pattern("global_local", 16, lo=2, hi=2, n_global=1)) == 4   # degenerate greedy (R-11)
    assert _err(Pattern("bigbird", 16, block=1, radius=1)) == 4
    assert _err(Pattern("strided_local", 16, stride=4, causal=0)) == 4


def test_host_handle_rejects_compute():
    a = S.Acsr(Pattern("window", 64, lo=2, hi=2), device=-1)
    L = S.lib()
    st = L.splat_sparse_mhsa(a.handle, 16, 16, 16, 0, 1, 1, 64, 1.0, 16, None)
    assert st == 1 and b"no CPU fallback" in L.splat_last_error()


def compare_meta_with_oracle(p):
    a = S.Acsr(p, device=-1)
    seg, nseg, row_ptr = a.copy_meta()
    oseg, onseg, orow, rc = O.acsr(p, max_seg=4)
    assert rc == 0
    assert np.array_equal(nseg.numpy().astype(np.int32), onseg), p
    assert np.array_equal(seg.numpy(), oseg), p
    assert np.array_equal(row_ptr.numpy(), orow), p
    assert a.nnz == orow[-1] and a.max_segs == onseg.max()
    return a


@pytest.mark.parametrize("cfg", CONFIGS[:4], ids=lambda c: c.name)
def test_closed_form_meta_bit_exact_configs(cfg):
    compare_meta_with_oracle(cfg.pattern)


def small_patterns(N):
    for lo in range(0, N + 1, max(1, N // 5)):
        for hi in range(0, N + 1, max(1, N // 4)):
            yield Pattern("window", N, lo=lo, hi=hi)
    for w in range(1, N + 1):
        yield Pattern("blocked", N, block=w)
        yield Pattern("strided", N, stride=w)
        yield Pattern("strided_local", N, stride=w, causal=1)
        if w >= 2:
            yield Pattern("bigbird", N, block=w, radius=1)
    for dl in range(1, N + 1, 3):
        yield Pattern("dilated", N, stride=dl, radius=min(2, N))
    for g in (0, min(2, N), N // 3):
        if g != 1:
            yield Pattern("global_local", N, lo=min(3, N), hi=min(5, N), n_global=g)


@pytest.mark.parametrize("N", [1, 3, 17, 64])
def test_closed_form_meta_bit_exact_exhaustive(N):
    for p in small_patterns(N):
        compare_meta_with_oracle(p)


def plan_reference(m, bm, bn, unit=64):
    """Key windows / FULL from the oracle's explicit mask (independent of the planner): per query
    tile, the 64-column blocks holding a non-zero of any row, covered greedily from the left by
    bn-wide windows starting at a block boundary (the fewest such windows); FULL = every row holds
    every column of the window.  Entries are (start / 64, full)."""
    N, NC = m.shape
    out = []
    for t in range((N + bm - 1) // bm):
        rows = m[t * bm:(t + 1) * bm]
        live = [bool(rows[:, b * unit:(b + 1) * unit].any()) for b in range((NC + unit - 1) // unit)]
        ents, b = [], 0
        while b < len(live):
            if not live[b]:
                b += 1
                continue
            blk = rows[:, b * unit:b * unit + bn]
            full = b * unit + bn <= NC and bool(blk.all())
            ents.append((b, full))
            b += bn // unit
        out.append(ents)
    return out


def test_plan_reference_greedy_is_minimal():
    """Brute force on small masks: no set of fewer 64-aligned windows covers the live blocks."""
    import itertools
    rng = np.random.default_rng(7)
    for _ in range(200):
        nb = int(rng.integers(1, 9))
        live = rng.random(nb) < 0.5
        m = np.zeros((1, nb * 64), dtype=bool)
        for b in range(nb):
            m[0, b * 64] = live[b]
        greedy = len(plan_reference(m, 1, 128)[0])
        need = [b for b in range(nb) if live[b]]
        best = 0 if not need else min(k for k in range(1, nb + 1) for c in itertools.combinations(range(nb), k)
                                      if all(any(s <= b <= s + 1 for s in c) for b in need))
        assert greedy == best


@pytest.mark.parametrize("p", [Pattern("window", 700, lo=64, hi=64), Pattern("global_local", 1000, lo=128, hi=128, n_global=32),
                               Pattern("bigbird", 1024, block=64, radius=1), Pattern("strided_local", 1100, stride=128, causal=1),
                               Pattern("strided", 600, stride=7), Pattern("dilated", 900, stride=3, radius=50),
                               Pattern("blocked", 640, block=96), Pattern("window", 300, lo=299, hi=0),
                               Pattern("bigbird", 4096, block=64, radius=1)],
                         ids=lambda p: p.kind)
def test_tile_plan_matches_mask(p):
    a = S.Acsr(p, device=-1)
    bm, bn, nq, ne = a.plan_info()
    qt_ptr, kv, order = a.plan_copy()
    ref = plan_reference(O.mask(p), bm, bn)
    assert nq == len(ref)
    for t in range(nq):
        ents = [(int(e) & 0xFFFFFF, not (int(e) >> 24) & 1) for e in kv[qt_ptr[t]:qt_ptr[t + 1]]]
        assert ents == ref[t], (p, t)
    # LPT order: a permutation, by non-increasing number of key tiles
    cnt = (qt_ptr[1:] - qt_ptr[:-1]).numpy()
    assert sorted(order.tolist()) == list(range(nq))
    assert all(cnt[order[i]] >= cnt[order[i + 1]] for i in range(nq - 1))


def test_density_and_flops():
    p = CONFIGS[1].pattern
    a = S.Acsr(p, device=-1)
    assert abs(a.density - a.nnz / p.seq_len ** 2) < 1e-15
    assert a.flops(8, 12, 64) == 4.0 * a.nnz * 64 * 96


# ---------------------------------------------------------------------------
# product build hygiene: no environment knobs, no debug exports, every
# device allocation through the counted wrapper (build time only)
# ---------------------------------------------------------------------------
CSRC = os.path.join(ROOT, "paper_2407_16847_b200", "csrc")


def _sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".cu", ".cpp", ".h", ".cuh"))]


def test_no_getenv_outside_the_diagnostics_helper():
    for f in _sources():
        txt = open(f).read()
        for m in re.finditer(r"\bgetenv\s*\(", txt):
            pre = txt[:m.start()]
            # the only getenv is diag_env's, compiled under #ifdef SPLAT_DIAG
            assert os.path.basename(f) == "splat_internal.h", f
            assert pre.rfind("#ifdef SPLAT_DIAG") > pre.rfind("#endif"), f


def test_every_device_allocation_is_counted():
    for f in _sources():
        txt = open(f).read()
        n = len(re.findall(r"\bcudaMalloc(Async)?\s*\(", txt))
        if os.path.basename(f) == "api.cu":
            assert n == 2, n          # the two wrappers themselves
        else:
            assert n == 0, f


def test_product_library_has_no_debug_exports():
    out = subprocess.check_output(["nm", "-D", "--defined-only", S.LIB_PATH]).decode()
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for name in ("splat_debug_trace", "splat_debug_fused_prof", "splat_debug_hang", "splat_debug_prof64",
                 "splat_debug_unf_prof"):
        assert name not in exported, name


def split_plan_coverage(p):
    """Times each (row, column) is covered by the split kernel's plan (its units' two 64-row
    segments x key windows x row masks) -- must equal the oracle's explicit mask."""
    a = S.Acsr(p, device=-1)
    rc, ne = a.split_info()
    units, kv, mid, masks = a.split_plan_copy()
    N = p.seq_len
    nseg = (N + 63) // 64
    cover = np.zeros((N, N), dtype=np.int32)
    masks = masks.numpy().astype(np.int64) & 0xFFFFFFFF
    for t, j0, j1, _ in units.tolist():
        sa, sb = (t & 0xFFFF, t >> 16) if rc else (2 * t, 2 * t + 1)
        rows = np.array([s * 64 + r if s < nseg and s * 64 + r < N else -1 for s in (sa, sb) for r in range(64)])
        ok = rows >= 0
        for e in range(j0, j1):
            ent = int(kv[e])
            if (ent >> 25) & 1:                      # composite window: key blocks a (cols 0-63), b (64-127)
                ba, bb = ent & 0xFFF, (ent >> 12) & 0xFFF
            else:
                ba = ent & 0xFFFFFF
                bb = ba + 1
            pos = np.arange(128)
            keys = np.where(pos < 64, ba * 64 + pos, bb * 64 + pos - 64)
            keep = keys < N
            pos, cols = pos[keep], keys[keep]
            if (ent >> 24) & 1:
                w = masks[int(mid[e])]                                   # [128, 4]
                bits = (w[:, pos >> 5] >> (pos & 31)) & 1
            else:
                bits = np.ones((128, len(cols)), dtype=np.int64)
            cover[np.ix_(rows[ok], cols)] += bits[ok].astype(np.int32)
    return cover, rc, ne


@pytest.mark.parametrize("p", [Pattern("bigbird", 4096, block=64, radius=1), Pattern("bigbird", 1000, block=64, radius=1),
                               Pattern("bigbird", 520, block=32, radius=1),
                               Pattern("global_local", 1000, lo=128, hi=128, n_global=32),
                               Pattern("window", 700, lo=64, hi=64), Pattern("strided_local", 1100, stride=128, causal=1),
                               Pattern("strided", 600, stride=7)], ids=lambda p: f"{p.kind}{p.seq_len}")
def test_split_plan_covers_mask_exactly_once(p):
    cover, rc, ne = split_plan_coverage(p)
    assert np.array_equal(cover, O.mask(p).astype(np.int32)), p
    if p.kind == "bigbird" and p.seq_len == 4096:
        assert rc == 1 and ne == 125          # row classes (global blocks share a tile) + composite windows


@pytest.mark.parametrize("p", [Pattern("global_local", 4096, lo=256, hi=256, n_global=32),
                               Pattern("bigbird", 4096, block=64, radius=1),
                               Pattern("global_local", 2000, lo=64, hi=64, n_global=40)], ids=lambda p: f"{p.kind}{p.seq_len}")
def test_ksplit_units_partition_long_tiles(p):
    # The split-K list: every whole-tile unit with more than 8 entries becomes
    # parts with contiguous entry ranges that partition it (each <= 8 entries, part order = entry
    # order, one split-tile index per tile); the other units are unchanged -- so the list still
    # covers the oracle mask exactly once.
    a = S.Acsr(p, device=-1)
    units, kv, mid, masks = a.split_plan_copy()
    ks = a.ksplit_units()
    whole = {(int(t), int(j0), int(j1)) for t, j0, j1, _ in units.tolist()}
    long_tiles = {u for u in whole if u[2] - u[1] > 8}
    assert long_tiles, "a global-row tile is long"
    assert ks.shape[0] > 0
    parts = {}
    for t, j0, j1, sp in ks.tolist():
        if sp == 0:
            assert (t, j0, j1) in whole and j1 - j0 <= 8
            continue
        part, npart, sid = sp & 0xFF, (sp >> 8) & 0xFF, sp >> 16
        assert 0 < j1 - j0 <= 8 and part < npart
        parts.setdefault((t, sid, npart), []).append((part, j0, j1))
    assert len(parts) == len(long_tiles)
    sids = set()
    for (t, sid, npart), lst in parts.items():
        lst.sort()
        assert [q for q, _, _ in lst] == list(range(npart))
        for (_, _, e1), (_, s0, _) in zip(lst, lst[1:]):
            assert e1 == s0                      # contiguous
        assert (t, lst[0][1], lst[-1][2]) in long_tiles
        sids.add(sid)
    assert sids == set(range(len(parts)))
    # whole units that are not long appear unchanged
    short = {(int(t), int(j0), int(j1)) for t, j0, j1, sp in ks.tolist() if sp == 0}
    assert short == whole - long_tiles
