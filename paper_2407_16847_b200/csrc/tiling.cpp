// tiling.cpp -- thread-block tilings of the R-SDDMM point set.
//
// The paper's Sec. 7.2-7.3 model of an R-SDDMM launch: a mask's non-zeros form a point set P of
// (x = key column, y = query row) points; a thread block of m x n threads with anchor t and
// stretch s computes Comp = {t + (c s, r s) : r < m, c < n} (Def. 2; m = thread rows
// = y extent, n = thread columns = x extent, reading T-1) and covers Comp ∩ P.  This
// file implements, on the host, for P given by a pattern descriptor:
//   - the four-factor cost model (Def. 3) and Cost = lambda / phi_CMR (Def. 4);
//   - poset tiling (Def. 5, Alg. 1): repeatedly anchor one block at every
//     minimal uncovered point (the set ⊤ under the comes-before order) until P is covered;
//   - stretch-factor selection (Sec. 7.3.1): 1 for polygonal masks (App. A), the
//     cheapest divisor of the row stride X for strided masks (App. B), else a bounded search;
//   - the naive tiling of App. C (Def. 8): m-row patches tiled left to right.
// The tcgen05 kernels do not launch these arrangements (their tiles are 128 x 128 and aligned,
// DESIGN.md §9 "Poset tiling"); this is the planner the paper's SIMT R-SDDMM would use, exposed
// so its block counts (Fig. 12) can be reproduced and compared with ours.
#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

#include "splat_internal.h"

namespace {

using namespace splat;

constexpr int kMaxTilingN = 8192;       // bitset of P: N * N / 8 bytes (8 MB at the cap)
constexpr int kGenericStretchCap = 64;  // bounded search for masks that are neither (T-4)

// P as one bit per point, row y = query row, bit x = key column.
struct Points {
    int N = 0, W = 0;
    std::vector<uint64_t> bits;
    int64_t count = 0;
    bool polygonal = true;   // every row's columns are contiguous (App. A)
    int stride = 0;          // common step of every multi-column row (strided masks), else -1
    uint64_t *row(int y) { return bits.data() + (size_t)y * W; }
    const uint64_t *row(int y) const { return bits.data() + (size_t)y * W; }
    bool test(int x, int y) const { return (row(y)[x >> 6] >> (x & 63)) & 1ull; }
};

void set_range(uint64_t *r, int a, int b)   // bits [a, b)
{
    while (a < b) {
        int w = a >> 6, o = a & 63, k = std::min(64 - o, b - a);
        uint64_t msk = (k == 64) ? ~0ull : (((1ull << k) - 1) << o);
        r[w] |= msk;
        a += k;
    }
}

int clear_range(uint64_t *r, int a, int b)  // clears bits [a, b), returns how many were set
{
    int n = 0;
    while (a < b) {
        int w = a >> 6, o = a & 63, k = std::min(64 - o, b - a);
        uint64_t msk = (k == 64) ? ~0ull : (((1ull << k) - 1) << o);
        n += __builtin_popcountll(r[w] & msk);
        r[w] &= ~msk;
        a += k;
    }
    return n;
}

int first_set(const uint64_t *r, int W, int from)  // first set bit >= from, or INT_MAX
{
    for (int w = from >> 6; w < W; ++w) {
        uint64_t v = r[w];
        if (w == (from >> 6)) v &= ~0ull << (from & 63);
        if (v) return w * 64 + __builtin_ctzll(v);
    }
    return INT_MAX;
}

Points make_points(const splat_pattern &p)
{
    Points P;
    P.N = p.seq_len;
    P.W = (P.N + 63) / 64;
    P.bits.assign((size_t)P.N * P.W, 0ull);
    Seg s[SPLAT_MAX_SEGS];
    bool contig = false;
    for (int i = 0; i < P.N; ++i) {
        int ns = row_segments(p, i, s);
        uint64_t *r = P.row(i);
        for (int k = 0; k < ns; ++k) {
            if (s[k].step == 1) {
                set_range(r, s[k].start, s[k].start + s[k].count);
            } else {
                for (int c = 0; c < s[k].count; ++c) {
                    int x = s[k].start + c * s[k].step;
                    r[x >> 6] |= 1ull << (x & 63);
                }
            }
            P.count += s[k].count;
            if (s[k].count > 1 && s[k].step > 1) {
                P.polygonal = false;
                if (ns > 1 || (P.stride != 0 && P.stride != s[k].step)) P.stride = -1;
                else if (P.stride == 0) P.stride = s[k].step;
            }
        }
        for (int k = 0; k < ns; ++k) contig |= s[k].count > 1 && s[k].step == 1;
        if (ns > 1) {
            P.polygonal = false;   // a gap between runs
            P.stride = -1;
        }
    }
    if (!P.polygonal && contig) P.stride = -1;   // mixes contiguous and strided rows
    return P;
}

// Alg. 1 with the stretch fixed.  Rem is a copy of P's bits; rowmin[y] is the first
// uncovered column of row y.  A point is in ⊤ (Def. 5) iff it is its row's first uncovered point
// and every earlier row's first uncovered column is larger (a point (x', y') with x' <= x and
// y' <= y would come before it).  Every block of one iteration is anchored at a ⊤ point computed
// before any of them is placed (lines 5-8), and then removes its Comp from Rem (reading T-2).
int64_t poset(const Points &P, int m, int n, int s, std::vector<int32_t> *anchors)
{
    const int N = P.N, W = P.W;
    std::vector<uint64_t> rem(P.bits);
    std::vector<int> rowmin(N);
    for (int y = 0; y < N; ++y) rowmin[y] = first_set(rem.data() + (size_t)y * W, W, 0);
    int64_t left = P.count, lambda = 0;
    std::vector<int> top_x, top_y;
    while (left > 0) {
        top_x.clear();
        top_y.clear();
        int best = INT_MAX;
        for (int y = 0; y < N; ++y)
            if (rowmin[y] < best) {
                best = rowmin[y];
                top_x.push_back(best);
                top_y.push_back(y);
            }
        for (size_t t = 0; t < top_x.size(); ++t) {
            const int x = top_x[t], y = top_y[t];
            ++lambda;
            if (anchors) {
                anchors->push_back(x);
                anchors->push_back(y);
            }
            for (int r = 0; r < m; ++r) {
                long long yy = (long long)y + (long long)r * s;
                if (yy >= N) break;
                uint64_t *row = rem.data() + (size_t)yy * W;
                if (s == 1) {
                    left -= clear_range(row, x, std::min<long long>(N, (long long)x + n));
                } else {
                    for (int c = 0; c < n; ++c) {
                        long long xx = (long long)x + (long long)c * s;
                        if (xx >= N) break;
                        uint64_t b = 1ull << (xx & 63);
                        if (row[xx >> 6] & b) {
                            row[xx >> 6] &= ~b;
                            --left;
                        }
                    }
                }
                if (rowmin[yy] != INT_MAX) rowmin[yy] = first_set(row, W, rowmin[yy]);
            }
        }
    }
    return lambda;
}

// App. C Def. 8: patches of m consecutive rows (from row 0); each non-empty patch is tiled left to
// right by unit-stretch blocks from its leftmost non-zero column until its rightmost is reached.
int64_t naive(const Points &P, int m, int n, std::vector<int32_t> *anchors)
{
    int64_t lambda = 0;
    for (int y0 = 0; y0 < P.N; y0 += m) {
        int lo = INT_MAX, hi = -1;
        for (int y = y0; y < std::min(P.N, y0 + m); ++y) {
            const uint64_t *r = P.row(y);
            for (int w = 0; w < P.W; ++w)
                if (r[w]) {
                    lo = std::min(lo, w * 64 + __builtin_ctzll(r[w]));
                    break;
                }
            for (int w = P.W - 1; w >= 0; --w)
                if (r[w]) {
                    hi = std::max(hi, w * 64 + 63 - __builtin_clzll(r[w]));
                    break;
                }
        }
        if (hi < 0) continue;
        for (int x = lo; x <= hi; x += n) {
            ++lambda;
            if (anchors) {
                anchors->push_back(x);
                anchors->push_back(y0);
            }
        }
    }
    return lambda;
}

// Def. 3 / Def. 4 for a uniform-stretch arrangement.  Comp sets are unioned row by row: in row
// yy a block contributes the lattice {x + c s : c < n}, i.e. the index interval [x div s,
// x div s + n) of residue class x mod s, so the union is a merge of intervals per (row, class).
// Points outside the N x N mask count as divergent threads (they are not in P).  Fails with the
// first uncovered point if the union of the covers is not P.
splat_status evaluate(const Points &P, int m, int n, int s, const int32_t *anc, int64_t lambda,
                      splat_tiling_cost *c)
{
    struct E { long long y; long long res, lo, hi; };
    std::vector<E> ev;
    ev.reserve((size_t)lambda * m);
    for (int64_t b = 0; b < lambda; ++b) {
        long long x = anc[2 * b], y = anc[2 * b + 1];
        if (x < 0 || y < 0) return set_error(SPLAT_ERR_INVALID_ARG, "anchor %lld has a negative coordinate", (long long)b);
        for (int r = 0; r < m; ++r) ev.push_back({y + (long long)r * s, x % s, x / s, x / s + n});
    }
    std::sort(ev.begin(), ev.end(), [](const E &a, const E &b) {
        return a.y != b.y ? a.y < b.y : a.res != b.res ? a.res < b.res : a.lo < b.lo;
    });
    long long uni = 0;
    std::vector<uint64_t> cov(P.W);
    size_t i = 0;
    long long next_row = 0;   // rows of P not yet checked
    auto check_row = [&](long long y, bool has) -> bool {
        const uint64_t *pr = P.row((int)y);
        for (int w = 0; w < P.W; ++w) {
            uint64_t miss = pr[w] & ~(has ? cov[w] : 0ull);
            if (miss) {
                set_error(SPLAT_ERR_INVALID_ARG, "arrangement does not cover P: point (x=%d, y=%lld) uncovered",
                          w * 64 + __builtin_ctzll(miss), y);
                return false;
            }
        }
        return true;
    };
    while (i < ev.size()) {
        const long long y = ev[i].y;
        for (; next_row < std::min<long long>(y, P.N); ++next_row)
            if (!check_row(next_row, false)) return SPLAT_ERR_INVALID_ARG;
        std::fill(cov.begin(), cov.end(), 0ull);
        size_t j = i;
        while (j < ev.size() && ev[j].y == y) {
            const long long res = ev[j].res, lo = ev[j].lo;
            long long hi = ev[j].hi;
            for (++j; j < ev.size() && ev[j].y == y && ev[j].res == res && ev[j].lo <= hi; ++j)
                hi = std::max(hi, ev[j].hi);
            uni += hi - lo;
            if (y >= P.N) continue;
            if (s == 1) {
                if (lo < P.N) set_range(cov.data(), (int)lo, (int)std::min<long long>(P.N, hi));
                continue;
            }
            for (long long k = lo; k < hi; ++k) {
                long long x = k * s + res;
                if (x >= P.N) break;
                cov[x >> 6] |= 1ull << (x & 63);
            }
        }
        if (y < P.N) {
            if (!check_row(y, true)) return SPLAT_ERR_INVALID_ARG;
            next_row = y + 1;
        }
        i = j;
    }
    for (; next_row < P.N; ++next_row)
        if (!check_row(next_row, false)) return SPLAT_ERR_INVALID_ARG;
    c->lambda = lambda;
    c->points = P.count;
    c->phi_td = uni - P.count;   // P ⊆ ∪Comp, so |∪Comp \ P| = |∪Comp| - |P|
    c->phi_r = lambda * (int64_t)m * n - P.count - c->phi_td;
    c->phi_ru = lambda ? (double)P.count / ((double)lambda * m * n) : 0.0;
    c->phi_cmr = 1.0 / s;        // (1/λ) Σ 1/Str(TB_i) with one stretch for every block
    c->cost = (double)lambda / c->phi_cmr;
    c->stretch = s;
    c->m = m;
    c->n = n;
    c->reserved = 0;
    return SPLAT_OK;
}

// Sec. 7.3.1: candidates {1} for polygonal masks (App. A: stretching only shrinks a block's
// cover), the divisors of the row stride X for strided masks (App. B: lambda^s depends on
// gcd(s, X) only and falls as it grows), otherwise s in [1, min(N, 64)] (reading T-4).  The
// cheapest arrangement under Def. 4 wins; ties go to fewer blocks (reading T-3).
int select_stretch(const Points &P, int m, int n)
{
    if (P.polygonal) return 1;
    std::vector<int> cand;
    if (P.stride > 1) {
        for (int d = 1; d <= P.stride; ++d)
            if (P.stride % d == 0) cand.push_back(d);
    } else {
        for (int d = 1; d <= std::min(P.N, kGenericStretchCap); ++d) cand.push_back(d);
    }
    int best_s = 1;
    long double best_cost = 0;
    int64_t best_l = 0;
    for (size_t k = 0; k < cand.size(); ++k) {
        int64_t l = poset(P, m, n, cand[k], nullptr);
        long double cost = (long double)l * cand[k];   // lambda / phi_CMR, phi_CMR = 1/s
        if (k == 0 || cost < best_cost || (cost == best_cost && l < best_l)) {
            best_s = cand[k];
            best_cost = cost;
            best_l = l;
        }
    }
    return best_s;
}

splat_status check_args(const splat_pattern *p, int32_t m, int32_t n, int64_t cap, const void *anchors,
                        const splat_tiling_cost *cost)
{
    if (!p || !cost) return set_error(SPLAT_ERR_INVALID_ARG, "null pattern or cost pointer");
    splat_status st = validate_pattern(*p);
    if (st != SPLAT_OK) return st;
    if (m < 1 || n < 1 || m > 4096 || n > 4096)
        return set_error(SPLAT_ERR_INVALID_ARG, "block shape %d x %d outside [1, 4096]^2", m, n);
    if (cap < 0 || (cap > 0 && !anchors)) return set_error(SPLAT_ERR_INVALID_ARG, "bad anchor buffer");
    if (p->seq_len > kMaxTilingN)
        return set_error(SPLAT_ERR_UNSUPPORTED, "tiling analysis supports seq_len <= %d", kMaxTilingN);
    return SPLAT_OK;
}

splat_status finish(const Points &P, int m, int n, int s, const std::vector<int32_t> &anc,
                    int32_t *anchors, int64_t cap, splat_tiling_cost *cost)
{
    const int64_t lambda = (int64_t)anc.size() / 2;
    splat_status st = evaluate(P, m, n, s, anc.data(), lambda, cost);
    if (st != SPLAT_OK) return st;   // cannot happen for poset / naive arrangements
    if (cap > 0) std::memcpy(anchors, anc.data(), sizeof(int32_t) * 2 * (size_t)std::min(cap, lambda));
    return SPLAT_OK;
}

}  // namespace

extern "C" {

splat_status splat_poset_tile(const splat_pattern *p, int32_t m, int32_t n, int32_t stretch,
                              int32_t *anchors, int64_t cap, splat_tiling_cost *cost)
{
    clear_error();
    splat_status st = check_args(p, m, n, cap, anchors, cost);
    if (st != SPLAT_OK) return st;
    if (stretch < 0 || stretch > p->seq_len)
        return set_error(SPLAT_ERR_INVALID_ARG, "stretch %d outside [0, seq_len]", stretch);
    Points P = make_points(*p);
    const int s = stretch > 0 ? stretch : select_stretch(P, m, n);
    std::vector<int32_t> anc;
    poset(P, m, n, s, &anc);
    return finish(P, m, n, s, anc, anchors, cap, cost);
}

splat_status splat_naive_tile(const splat_pattern *p, int32_t m, int32_t n, int32_t *anchors, int64_t cap,
                              splat_tiling_cost *cost)
{
    clear_error();
    splat_status st = check_args(p, m, n, cap, anchors, cost);
    if (st != SPLAT_OK) return st;
    Points P = make_points(*p);
    std::vector<int32_t> anc;
    naive(P, m, n, &anc);
    return finish(P, m, n, 1, anc, anchors, cap, cost);
}

splat_status splat_tiling_cost_eval(const splat_pattern *p, int32_t m, int32_t n, int32_t stretch,
                                    const int32_t *anchors, int64_t n_blocks, splat_tiling_cost *cost)
{
    clear_error();
    splat_status st = check_args(p, m, n, 0, nullptr, cost);
    if (st != SPLAT_OK) return st;
    if (stretch < 1 || stretch > p->seq_len)
        return set_error(SPLAT_ERR_INVALID_ARG, "stretch %d outside [1, seq_len]", stretch);
    if (n_blocks < 0 || (n_blocks > 0 && !anchors)) return set_error(SPLAT_ERR_INVALID_ARG, "bad anchor list");
    Points P = make_points(*p);
    return evaluate(P, m, n, stretch, anchors, n_blocks, cost);
}

}  // extern "C"
