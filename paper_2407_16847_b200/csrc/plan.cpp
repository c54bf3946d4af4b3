// plan.cpp -- host tile planner.
//
// From the ACSR runs of every row it derives, per 128-row query tile, the
// 128-column key windows (starting on 64-column boundaries) that cover the
// columns touched by any row of the tile.  This is the B200
// form of the paper's span specialisation (a row group only iterates
// over [min start, max end] of its rows) applied at tile granularity, and of
// the R-SDDMM thread-block arrangement (Sec. 7.2): every plan
// entry is one dense 128x128 tcgen05 tile, FULL when every row of the query
// tile contains every column of the key tile (no fast-index masking needed,
// P:237) and PARTIAL otherwise.  Query tiles are ordered longest first
// (LPT) for the persistent kernels.  The planner works on O(rows) metadata
// only, never on per-nnz data.
#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <stdexcept>
#include <unordered_map>

#include "splat_internal.h"

namespace splat {

void build_plan(splat_acsr_s &a)
{
    Plan &P = a.plan;
    const int N = a.n, bm = P.bm, bn = P.bn;
    // Ablation knob for the span-specialisation study (the paper's Fig. 13),
    // diagnostics build only: SPLAT_PLAN_ABLATE=1 drops the FULL flags (every tile masked), =2 also
    // drops the span (every query tile visits every key tile).  Product build: always 0.
    const int ablate = diag_env("SPLAT_PLAN_ABLATE");
    // Key windows are bn = 128 columns wide and start on a multiple of kKvUnit = 64 columns (kv =
    // start / 64); kv_align = 2 keeps them 128-aligned (sub-handles whose tiles are residue-major
    // views).  Per query tile, the 64-column blocks holding a non-zero of any row are covered
    // greedily from the left -- a window at the first uncovered live block -- which uses the fewest
    // windows of that width (interval covering); with 128-aligned windows only, BigBird's
    // three-block band (192 columns at 64-column block offsets) would need three.
    const int align = P.kv_align, nb = (N + kKvUnit - 1) / kKvUnit, wb = bn / kKvUnit;
    P.n_qt = (N + bm - 1) / bm;
    P.n_kt = (N + bn - 1) / bn;
    P.qt_ptr.assign(P.n_qt + 1, 0);
    P.kv.clear();
    std::vector<int32_t> stamp(nb, -1);
    for (int t = 0; t < P.n_qt; ++t) {
        const int r0 = t * bm, r1 = std::min(N, r0 + bm), nrows = r1 - r0;
        auto mark = [&](int blk) { stamp[blk] = t; };
        for (int i = r0; i < r1; ++i) {
            const int32_t *sg = &a.seg_h[(size_t)i * 16];
            for (int s = 0; s < a.nseg_h[i]; ++s) {
                const int start = sg[4 * s], step = sg[4 * s + 1], count = sg[4 * s + 2];
                const int last = start + step * (count - 1);
                if (step < kKvUnit) {
                    for (int j = start / kKvUnit; j <= last / kKvUnit; ++j) mark(j);
                } else {
                    for (int x = 0; x < count; ++x) mark((start + step * x) / kKvUnit);
                }
            }
        }
        if (ablate >= 2)
            for (int j = 0; j < nb; ++j) mark(j);
        for (int j = 0; j < nb;) {
            if (stamp[j] != t) { ++j; continue; }
            const int kv = j - j % align;                       // window [64 kv, 64 kv + bn)
            const int c0 = kv * kKvUnit, c1 = std::min(N, c0 + bn) - 1;
            // FULL: every row of the query tile holds every column of the window (one step-1 run)
            bool full = ablate == 0 && c0 + bn <= N;
            for (int i = r0; i < r1 && full; ++i) {
                const int32_t *sg = &a.seg_h[(size_t)i * 16];
                bool row_full = false;
                for (int s = 0; s < a.nseg_h[i] && !row_full; ++s) {
                    const int start = sg[4 * s], step = sg[4 * s + 1], count = sg[4 * s + 2];
                    row_full = (step == 1 || count == 1) && start <= c0 && c1 <= start + step * (count - 1);
                }
                full = row_full;
            }
            (void)nrows;
            P.kv.push_back(kv | (full ? 0 : kPartialBit));
            j = kv + wb;
        }
        if (P.kv.size() > (size_t)0x7fffffff) throw std::length_error("tile plan exceeds 2^31 entries");
        P.qt_ptr[t + 1] = (int32_t)P.kv.size();
    }
    P.n_entries = (int)P.kv.size();
    P.order.resize(P.n_qt);
    std::iota(P.order.begin(), P.order.end(), 0);
    std::stable_sort(P.order.begin(), P.order.end(), [&](int x, int y) {
        return (P.qt_ptr[x + 1] - P.qt_ptr[x]) > (P.qt_ptr[y + 1] - P.qt_ptr[y]);
    });

    // ---- pairs of adjacent query tiles (2p, 2p+1): union of the two sorted key-tile
    // lists, each entry flagged with which tile uses it and whether it is PARTIAL there.
    P.n_pairs = (P.n_qt + 1) / 2;
    P.pair_ptr.assign(P.n_pairs + 1, 0);
    P.pair_ent.clear();
    std::vector<int32_t> qent_of_pair_ent[2];   // pair entry -> query-tile entry index of tile A / B
    qent_of_pair_ent[0].clear();
    qent_of_pair_ent[1].clear();
    for (int p = 0; p < P.n_pairs; ++p) {
        const int ta = 2 * p, tb = 2 * p + 1;
        int ia = P.qt_ptr[ta], ea = P.qt_ptr[ta + 1];
        int ib = tb < P.n_qt ? P.qt_ptr[tb] : 0, eb = tb < P.n_qt ? P.qt_ptr[tb + 1] : 0;
        while (ia < ea || ib < eb) {
            const int ka = ia < ea ? (P.kv[ia] & kKvMask) : 0x7fffffff;
            const int kb = ib < eb ? (P.kv[ib] & kKvMask) : 0x7fffffff;
            const int k = std::min(ka, kb);
            int ent = k;
            int qa = -1, qb = -1;
            if (ka == k) { ent |= kUseA | ((P.kv[ia] & kPartialBit) ? kPartA : 0); qa = ia; ++ia; }
            if (kb == k) { ent |= kUseB | ((P.kv[ib] & kPartialBit) ? kPartB : 0); qb = ib; ++ib; }
            P.pair_ent.push_back(ent);
            qent_of_pair_ent[0].push_back(qa);
            qent_of_pair_ent[1].push_back(qb);
        }
        P.pair_ptr[p + 1] = (int32_t)P.pair_ent.size();
    }
    P.n_pair_entries = (int)P.pair_ent.size();
    // order: cost buckets (floor(log2(union length))) longest first; the persistent
    // kernel walks the units of a bucket head-major so K/V of one (b,h) stay in L2.
    auto bucket = [&](int p) {
        int len = P.pair_ptr[p + 1] - P.pair_ptr[p], b = 0;
        while (len > 1) { len >>= 1; ++b; }
        return b;
    };
    P.pair_order.resize(P.n_pairs);
    std::iota(P.pair_order.begin(), P.pair_order.end(), 0);
    std::stable_sort(P.pair_order.begin(), P.pair_order.end(),
                     [&](int x, int y) { return bucket(x) > bucket(y); });
    P.bucket_start.clear();
    for (int i = 0; i < P.n_pairs; ++i)
        if (i == 0 || bucket(P.pair_order[i]) != bucket(P.pair_order[i - 1])) P.bucket_start.push_back(i);
    P.bucket_start.push_back(P.n_pairs);
    P.n_buckets = (int)P.bucket_start.size() - 1;
    // pair_info: (pair, e0, e1, jA0), (jA1, jB1, 0, 0) -- the union range and the two query
    // tiles' own entry ranges [jA0, jA1) and [jA1, jB1) (adjacent tiles: jB0 == jA1).
    P.pair_info.assign((size_t)P.n_pairs * 8, 0);
    for (int k = 0; k < P.n_pairs; ++k) {
        const int p = P.pair_order[k];
        const int ta = 2 * p, tb = std::min(2 * p + 1, P.n_qt);
        P.pair_info[8 * k + 0] = p;
        P.pair_info[8 * k + 1] = P.pair_ptr[p];
        P.pair_info[8 * k + 2] = P.pair_ptr[p + 1];
        P.pair_info[8 * k + 3] = P.qt_ptr[ta];
        P.pair_info[8 * k + 4] = P.qt_ptr[ta + 1];
        P.pair_info[8 * k + 5] = P.qt_ptr[std::min(tb + 1, P.n_qt)];
    }

    // ---- per-row column masks of the PARTIAL (tile, key tile) entries (fast-index predicate
    // of reading A-7 evaluated once per pattern, shared by every (b, h)), and per-warp chunk
    // liveness of every entry.
    P.pair_mask.assign((size_t)P.n_pair_entries * 2, -1);
    // qt_bits per query-tile entry: bit 4 quad + w = chunk w (32 key columns) has a valid entry
    // in some row of warp quad; bit 16 + 4 quad + w = every row of the warp has all 32 columns
    // (the softmax skips the fast-index mask there).
    P.qt_bits.assign(P.n_entries, 0xFFFFFFFFu);
    P.masks.clear();
    // masks are deduplicated by content (a strided or windowed pattern repeats a few row masks
    // across its tiles): hash -> mask ids with that hash
    std::unordered_map<uint64_t, std::vector<int32_t>> seen;
    std::vector<uint32_t> mbuf(128 * 4);
    for (int p = 0; p < P.n_pairs; ++p) {
        for (int e = P.pair_ptr[p]; e < P.pair_ptr[p + 1]; ++e) {
            const int ent = P.pair_ent[e], c0 = (ent & kKvMask) * kKvUnit;
            for (int g = 0; g < 2; ++g) {
                const int t = 2 * p + g;
                if (!(ent & (g == 0 ? kUseA : kUseB))) continue;
                if (!(ent & (g == 0 ? kPartA : kPartB))) continue;
                std::fill(mbuf.begin(), mbuf.end(), 0u);
                uint32_t *m = mbuf.data();
                for (int r = 0; r < 128; ++r) {
                    const int i = t * bm + r;
                    if (i >= N) continue;
                    const int32_t *sg = &a.seg_h[(size_t)i * 16];
                    for (int s = 0; s < a.nseg_h[i]; ++s) {
                        const int start = sg[4 * s], step = sg[4 * s + 1], count = sg[4 * s + 2];
                        const int last = start + step * (count - 1);
                        const int lo = std::max(start, c0), hi = std::min(last, c0 + bn - 1);
                        if (lo > hi) continue;
                        const int first = start + ((lo - start + step - 1) / step) * step;
                        for (int c = first; c <= hi; c += step) m[4 * r + ((c - c0) >> 5)] |= 1u << ((c - c0) & 31);
                    }
                }
                uint64_t h = 1469598103934665603ull;                 // FNV-1a over the 512 words
                for (uint32_t x : mbuf) h = (h ^ x) * 1099511628211ull;
                int32_t id = -1;
                auto &cand = seen[h];
                for (int32_t c : cand)
                    if (std::equal(mbuf.begin(), mbuf.end(), P.masks.begin() + (size_t)c * 128 * 4)) { id = c; break; }
                if (id < 0) {
                    id = (int32_t)(P.masks.size() / (128 * 4));
                    P.masks.insert(P.masks.end(), mbuf.begin(), mbuf.end());
                    cand.push_back(id);
                }
                P.pair_mask[(size_t)e * 2 + g] = id;
                uint32_t bits = 0;
                for (int q = 0; q < 4; ++q)
                    for (int w = 0; w < 4; ++w) {
                        bool any = false, all = true;
                        for (int r = 32 * q; r < 32 * q + 32; ++r) {
                            any |= m[4 * r + w] != 0u;
                            all &= m[4 * r + w] == ~0u;
                        }
                        if (any || ablate >= 2) bits |= 1u << (4 * q + w);   // ablation 2: no dead-chunk skip
                        if (all && ablate == 0) bits |= 1u << (16 + 4 * q + w);   // ablation >= 1: always mask
                    }
                P.qt_bits[qent_of_pair_ent[g][e]] = bits;
            }
        }
    }
    P.n_masks = (int)(P.masks.size() / (128 * 4));
    P.kv_mask.assign(P.n_entries, -1);
    for (int e = 0; e < P.n_pair_entries; ++e)
        for (int g = 0; g < 2; ++g)
            if (qent_of_pair_ent[g][e] >= 0) P.kv_mask[qent_of_pair_ent[g][e]] = P.pair_mask[(size_t)e * 2 + g];

    // ---- row classes of the split-group kernel (d = 64): a query tile is two 64-row segments.
    // Rows are grouped by the key blocks they touch (the paper's row classes by segment shape,
    // alignment P:575-576): segments whose rows touch nearly every key block (global rows) share
    // tiles, the others keep their natural order, so a band segment is not dragged across every
    // key window by a global segment (BigBird: the first and last blocks are global rows).  Used
    // only when it needs fewer plan entries than the natural tiles; the classed entries are
    // appended after the natural ones (kv / kv_mask / qt_bits), which every other kernel uses.
    const int nseg = (N + 63) / 64;
    std::vector<int> seg_a, seg_b;          // per split-kernel tile
    std::vector<int32_t> tj0, tj1;          // its entry range
    for (int t = 0; t < P.n_qt; ++t) {      // natural: segments 2t, 2t + 1
        seg_a.push_back(2 * t);
        seg_b.push_back(2 * t + 1 < nseg ? 2 * t + 1 : nseg);
        tj0.push_back(P.qt_ptr[t]);
        tj1.push_back(P.qt_ptr[t + 1]);
    }
    if (ablate == 0 && N <= 65536 && nseg >= 4) {
        const int W = (nb + 63) / 64;
        std::vector<uint64_t> foot((size_t)nseg * W, 0ull);
        std::vector<int> fsz(nseg, 0);
        for (int sg = 0; sg < nseg; ++sg) {
            uint64_t *f = &foot[(size_t)sg * W];
            for (int i = sg * 64; i < std::min(N, sg * 64 + 64); ++i) {
                const int32_t *rs = &a.seg_h[(size_t)i * 16];
                for (int q = 0; q < a.nseg_h[i]; ++q) {
                    const int start = rs[4 * q], step = rs[4 * q + 1], count = rs[4 * q + 2];
                    const int last = start + step * (count - 1);
                    if (step < kKvUnit) {
                        for (int j = start / kKvUnit; j <= last / kKvUnit; ++j) f[j >> 6] |= 1ull << (j & 63);
                    } else {
                        for (int x = 0; x < count; ++x) {
                            const int j = (start + step * x) / kKvUnit;
                            f[j >> 6] |= 1ull << (j & 63);
                        }
                    }
                }
            }
            for (int w = 0; w < W; ++w) fsz[sg] += __builtin_popcountll(f[w]);
        }
        std::vector<int> full, rest;
        for (int sg = 0; sg < nseg; ++sg) (4 * fsz[sg] >= 3 * nb ? full : rest).push_back(sg);
        if (full.size() >= 2) {
            std::vector<int> order = full;
            order.insert(order.end(), rest.begin(), rest.end());
            std::vector<int> ca, cb;
            for (size_t k = 0; k < order.size(); k += 2) {
                ca.push_back(order[k]);
                cb.push_back(k + 1 < order.size() ? order[k + 1] : nseg);
            }
            // windows of a classed tile: greedy cover of its rows' live 64-column blocks
            std::vector<int32_t> ckv, cj0, cj1;
            std::vector<uint64_t> u(W);
            for (size_t t = 0; t < ca.size(); ++t) {
                cj0.push_back((int32_t)(P.kv.size() + ckv.size()));
                for (int w = 0; w < W; ++w)
                    u[w] = foot[(size_t)ca[t] * W + w] | (cb[t] < nseg ? foot[(size_t)cb[t] * W + w] : 0ull);
                auto live = [&](int j) { return j < nb && ((u[j >> 6] >> (j & 63)) & 1ull); };
                // composite windows: two half-live windows (one live 64-column block each -- BigBird's
                // first and last key blocks) become one window of two 64-row K / V boxes (kCompBit,
                // blocks a | b << 12): one plan entry instead of two
                std::vector<int32_t> half;
                for (int j = 0; j < nb;) {
                    if (!live(j)) { ++j; continue; }
                    const int kv = j - j % P.kv_align;
                    if (bn == 2 * kKvUnit && live(kv) != live(kv + 1)) half.push_back(live(kv) ? kv : kv + 1);
                    else ckv.push_back(kv);
                    j = kv + bn / kKvUnit;
                }
                for (size_t h = 0; h + 1 < half.size(); h += 2) ckv.push_back(half[h] | (half[h + 1] << 12) | kCompBit);
                if (half.size() & 1) ckv.push_back(half.back() - half.back() % P.kv_align);
                cj1.push_back((int32_t)(P.kv.size() + ckv.size()));
            }
            if ((long long)ckv.size() < (long long)P.n_entries) {
                // adopt: FULL flags, masks, chunk bits of the classed entries (rows in tile order)
                for (size_t t = 0; t < ca.size(); ++t) {
                    int rows[128];
                    for (int r = 0; r < 128; ++r) {
                        const int sg = r < 64 ? ca[t] : cb[t];
                        const int i = sg * 64 + (r & 63);
                        rows[r] = sg < nseg && i < N ? i : -1;
                    }
                    for (int e = cj0[t]; e < cj1[t]; ++e) {
                        const int32_t ent = ckv[e - P.n_entries];
                        const bool comp = (ent & kCompBit) != 0;
                        // the window's two 64-column halves: key blocks ba (columns 0-63), bb (64-127)
                        const int ba = comp ? (ent & 0xFFF) : ent, bb = comp ? ((ent >> 12) & 0xFFF) : ent + 1;
                        std::fill(mbuf.begin(), mbuf.end(), 0u);
                        bool full_all = (ba + 1) * kKvUnit <= N && (bb + 1) * kKvUnit <= N;
                        for (int r = 0; r < 128; ++r) {
                            const int i = rows[r];
                            if (i < 0) continue;
                            const int32_t *rs = &a.seg_h[(size_t)i * 16];
                            for (int q = 0; q < a.nseg_h[i]; ++q) {
                                const int start = rs[4 * q], step = rs[4 * q + 1], count = rs[4 * q + 2];
                                const int last = start + step * (count - 1);
                                for (int hf = 0; hf < 2; ++hf) {
                                    const int k0 = (hf ? bb : ba) * kKvUnit;      // keys [k0, k0 + 64) -> columns 64 hf + ...
                                    const int lo = std::max(start, k0), hi = std::min(last, k0 + kKvUnit - 1);
                                    if (lo > hi) continue;
                                    const int first = start + ((lo - start + step - 1) / step) * step;
                                    for (int c = first; c <= hi; c += step) {
                                        const int pcol = kKvUnit * hf + (c - k0);
                                        mbuf[4 * r + (pcol >> 5)] |= 1u << (pcol & 31);
                                    }
                                }
                            }
                            for (int w = 0; w < 4; ++w) full_all &= mbuf[4 * r + w] == ~0u;
                        }
                        for (int r = 0; r < 128; ++r)
                            if (rows[r] < 0) full_all = false;
                        int32_t id = -1;
                        uint32_t bits = 0xFFFFFFFFu;
                        if (!full_all) {
                            uint64_t h = 1469598103934665603ull;
                            for (uint32_t x : mbuf) h = (h ^ x) * 1099511628211ull;
                            auto &cand = seen[h];
                            for (int32_t c : cand)
                                if (std::equal(mbuf.begin(), mbuf.end(), P.masks.begin() + (size_t)c * 128 * 4)) { id = c; break; }
                            if (id < 0) {
                                id = (int32_t)(P.masks.size() / (128 * 4));
                                P.masks.insert(P.masks.end(), mbuf.begin(), mbuf.end());
                                cand.push_back(id);
                            }
                            bits = 0;
                            for (int q = 0; q < 4; ++q)
                                for (int w = 0; w < 4; ++w) {
                                    bool any = false, all = true;
                                    for (int r = 32 * q; r < 32 * q + 32; ++r) {
                                        any |= mbuf[4 * r + w] != 0u;
                                        all &= mbuf[4 * r + w] == ~0u;
                                    }
                                    if (any) bits |= 1u << (4 * q + w);
                                    if (all) bits |= 1u << (16 + 4 * q + w);
                                }
                        }
                        P.kv.push_back(ent | (full_all ? 0 : kPartialBit));
                        P.kv_mask.push_back(id);
                        P.qt_bits.push_back(bits);
                    }
                }
                seg_a = ca;
                seg_b = cb;
                tj0 = cj0;
                tj1 = cj1;
                P.row_classes = 1;
            }
        }
    }
    P.n_masks = (int)(P.masks.size() / (128 * 4));

    // ---- split-kernel work units: its tiles in cost buckets (floor(log2(entries))), longest
    // first, walked head-major inside a bucket; (tile or segments a | b << 16, j0, j1, split).
    // Two lists: whole tiles (t_info), and the same with split-K of long tiles (t_info_ks): a tile
    // with more than kSplitMax entries (the global-row tiles) becomes np parts with contiguous entry
    // ranges, split = part | np << 8 | sid << 16 (sid = the tile's index among the split tiles of a
    // head); the kernel merges the parts' partial softmax results (the last part to finish).  The
    // launch takes the split list when a long tile would outlast the average work of a tile group
    // (few heads per GPU: DESIGN.md section 8).
    {
        auto emit = [&](bool ksplit, std::vector<int32_t> &info, std::vector<int32_t> &bstart, int &nbk, int &n_split,
                        int &pmax) {
            std::vector<int32_t> ut, uj0, uj1, usp;
            n_split = 0;
            pmax = 0;
            // only outliers are split: tiles longer than kSplitMax AND twice the mean (the global-row
            // tiles; a window pattern whose tiles are all long -- Mistral -- gains nothing from parts)
            long long tot = 0;
            for (size_t t = 0; t < seg_a.size(); ++t) tot += tj1[t] - tj0[t];
            const double mean = seg_a.empty() ? 0.0 : (double)tot / (double)seg_a.size();
            for (size_t t = 0; t < seg_a.size(); ++t) {
                const int32_t tt = P.row_classes ? (seg_a[t] | (seg_b[t] << 16)) : (int32_t)t;
                const int n = tj1[t] - tj0[t];
                if (ksplit && n > kSplitMax && n > 2.0 * mean) {
                    const int np = std::min((n + kSplitMax - 1) / kSplitMax, kSplitPartsMax);
                    for (int q = 0; q < np; ++q) {
                        ut.push_back(tt);
                        uj0.push_back(tj0[t] + (int)((long long)n * q / np));
                        uj1.push_back(tj0[t] + (int)((long long)n * (q + 1) / np));
                        usp.push_back(q | (np << 8) | (n_split << 16));
                    }
                    pmax = std::max(pmax, np);
                    ++n_split;
                } else {
                    ut.push_back(tt);
                    uj0.push_back(tj0[t]);
                    uj1.push_back(tj1[t]);
                    usp.push_back(0);
                }
            }
            const int nt = (int)ut.size();
            auto tb = [&](int t) {
                int len = uj1[t] - uj0[t], b = 0;
                while (len > 1) { len >>= 1; ++b; }
                return b;
            };
            std::vector<int> to(nt);
            std::iota(to.begin(), to.end(), 0);
            std::stable_sort(to.begin(), to.end(), [&](int x, int y) { return tb(x) > tb(y); });
            bstart.clear();
            for (int i = 0; i < nt; ++i)
                if (i == 0 || tb(to[i]) != tb(to[i - 1])) bstart.push_back(i);
            bstart.push_back(nt);
            nbk = (int)bstart.size() - 1;
            info.assign((size_t)nt * 4, 0);
            for (int k = 0; k < nt; ++k) {
                // natural tiles: the tile index (segments 2t, 2t + 1); classed (N <= 65536): packed segments
                info[4 * k + 0] = ut[to[k]];
                info[4 * k + 1] = uj0[to[k]];
                info[4 * k + 2] = uj1[to[k]];
                info[4 * k + 3] = usp[to[k]];
            }
        };
        int ns0 = 0, pm0 = 0;
        emit(false, P.t_info, P.t_bucket_start, P.t_n_buckets, ns0, pm0);
        P.n_split_tiles = (int)(P.t_info.size() / 4);
        P.t_max_len = 0;
        for (size_t k = 0; k < P.t_info.size(); k += 4) P.t_max_len = std::max(P.t_max_len, P.t_info[k + 2] - P.t_info[k + 1]);
        if (ablate == 0 && P.t_max_len > kSplitMax && (int)P.t_bucket_start.size() <= kMaxBuckets + 1) {
            emit(true, P.t_info_ks, P.t_bucket_start_ks, P.t_n_buckets_ks, P.n_ksplit, P.ksplit_pmax);
            if (P.n_ksplit == 0) P.t_info_ks.clear();
        } else {
            P.t_info_ks.clear();
            P.n_ksplit = 0;
            P.ksplit_pmax = 0;
        }
    }
    // R-SpMM row records of every PARTIAL mask: per row and 8-column group g the live columns left
    // of the group (low byte) and the group's 8 mask bits (high byte), and per row the live count
    P.mask_rec.assign((size_t)P.n_masks * 128 * 16, 0);
    P.mask_cnt.assign((size_t)P.n_masks * 128, 0);
    for (int m = 0; m < P.n_masks; ++m)
        for (int r = 0; r < 128; ++r) {
            const uint32_t *w = &P.masks[((size_t)m * 128 + r) * 4];
            int pre = 0;
            for (int g = 0; g < 16; ++g) {
                const uint32_t byte = (w[g >> 2] >> (8 * (g & 3))) & 0xFFu;
                P.mask_rec[((size_t)m * 128 + r) * 16 + g] = (uint16_t)(pre | (byte << 8));
                pre += __builtin_popcount(byte);
            }
            P.mask_cnt[(size_t)m * 128 + r] = (uint8_t)(pre > 255 ? 255 : pre);   // <= 128
        }
}

}  // namespace splat
