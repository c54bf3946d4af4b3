/*
 * splat_oracle.c -- plain, slow, obviously-correct CPU oracle for the SPLAT
 * sparse-MHSA hot path (arXiv 2407.16847).  fp64 throughout.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2407_16847_b200/csrc); it defines its own descriptor struct.
 *
 * What it computes (Eq. 1, and §6):
 *     O = softmax( M (x) scale * Q K^T ) V      per (batch, head),
 * where the softmax of each row runs over the row's mask non-zeros only
 * (reading R-1 in DESIGN.md: the masked-out entries are excluded, not
 * zeros; "masked positions set to -inf").
 *
 * Steps, each following the passage cited beside it:
 *   1. mask      : or_pred()          -- SURVEY §8(c) C-2 predicates
 *   2. row cols  : or_row_cols()      -- point-set of row i
 *   3. ACSR      : or_runs_from_cols() -- 2x2 solve + consecutive
 *                  check, restarted greedily at the first failing
 *                  column (reading A-11); row_ptr = exclusive prefix
 *   4. regularity: or_regularity()    -- P:218-219 on an explicit mask, with
 *                  the first offending (row, col)
 *   5. scores    : s_ij = scale * sum_t q[i,t] k[j,t], t ascending (R-SDDMM,
 *                  P:241; Listing 1 K-loop P:424-426)
 *   6. softmax   : m = max_j s_ij, e = exp(s - m), l = sum_j e, p = e / l
 *                  ("computing the softmax for each input row";
 *                  SPEC S:405-407)
 *   7. output    : o_i = sum_j p_ij v_j, j ascending (R-SpMM)
 * Empty rows give o_i = 0.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- descriptor (oracle's own copy; kinds numbered as in SURVEY §8(b)) ---- */
enum { OR_WINDOW = 0, OR_BLOCKED = 1, OR_STRIDED = 2, OR_DILATED = 3,
       OR_GLOBAL_LOCAL = 4, OR_BIGBIRD = 5, OR_STRIDED_LOCAL = 6 };

typedef struct {
    int32_t kind, n;          /* pattern kind, sequence length N */
    int32_t lo, hi;           /* window: columns [i-lo, i+hi] */
    int32_t block;            /* BLOCKED / BIGBIRD block size */
    int32_t n_global;         /* GLOBAL_LOCAL: first g rows and columns global */
    int32_t stride;           /* STRIDED X, DILATED delta, STRIDED_LOCAL l */
    int32_t radius;           /* DILATED rho, BIGBIRD sliding radius in blocks */
    int32_t causal;           /* STRIDED_LOCAL: 1 = keys j <= i only */
} or_pattern;

static int iabs(int x) { return x < 0 ? -x : x; }

/* Step 1: M[i][j] for the descriptor. */
int or_pred(const or_pattern *p, int i, int j)
{
    switch (p->kind) {
    case OR_WINDOW:                      /* "Windowed(w)" S:47, Fig. 2 */
        return (i - p->lo <= j) && (j <= i + p->hi);
    case OR_BLOCKED:                     /* block diagonal, S:48 (reading A-5) */
        return (i / p->block) == (j / p->block);
    case OR_STRIDED:                     /* x = y (mod X), App. B */
        return (i % p->stride) == (j % p->stride);
    case OR_DILATED:                     /* |i-j| <= rho*delta and i = j (mod delta) */
        return iabs(i - j) <= p->radius * p->stride && ((i - j) % p->stride) == 0;
    case OR_GLOBAL_LOCAL:                /* Longformer: global rows/cols + window */
        return i < p->n_global || j < p->n_global ||
               ((i - p->lo <= j) && (j <= i + p->hi));
    case OR_BIGBIRD: {                   /* first/last blocks global + sliding blocks */
        int bs = p->block;
        int nb = (p->n + bs - 1) / bs;
        int qb = i / bs, kb = j / bs;
        return qb == 0 || qb == nb - 1 || kb == 0 || kb == nb - 1 ||
               iabs(qb - kb) <= p->radius;
    }
    case OR_STRIDED_LOCAL: {             /* Sparse Transformer strided (local band + every l-th key) */
        int l = p->stride, dlt = i - j;
        if (p->causal)
            return j <= i && (dlt < l || dlt % l == 0);
        return iabs(dlt) < l || dlt % l == 0;
    }
    }
    return 0;
}

/* Step 2: the point-set of row i, columns in ascending order. */
int or_row_cols(const or_pattern *p, int i, int32_t *cols)
{
    int c = 0;
    for (int j = 0; j < p->n; ++j)
        if (or_pred(p, i, j)) cols[c++] = j;
    return c;
}

/*
 * Step 3: affine runs of one row.
 * For the first two unconsumed columns i0 < i1 the paper solves
 *     [i0 1; i1 1] [a b]^T = [0 1]^T   =>  a = 1/(i1-i0),  b = -i0/(i1-i0)
 * and then checks i_x*a + b == i_{x-1}*a + b + 1 for the following columns.
 * Multiplying that check by (i1 - i0) > 0 gives the exact integer test
 *     i_x - i_{x-1} == i1 - i0 ,
 * which is what we evaluate (reading A-9: exact integers, no float round()).
 * The run is stored as (start = i0 = -b/a, step = 1/a = i1-i0, count = nnzs).
 * A run that fails the check ends there and a new run starts at the failing
 * column (reading A-11, canonical greedy).  A lone column is (c, 1, 1)
 * (SPEC S:96).  Returns the number of runs; writes at most max_seg of them
 * as (start, step, count) triplets.
 */
int or_runs_from_cols(const int32_t *cols, int n, int32_t *seg, int max_seg)
{
    int ns = 0, x = 0;
    while (x < n) {
        int32_t i0 = cols[x], step = 1, count = 1;
        if (x + 1 < n) {
            int32_t i1 = cols[x + 1];
            step = i1 - i0;                      /* = 1/a */
            count = 2;
            while (x + count < n && cols[x + count] - cols[x + count - 1] == step)
                ++count;
        }
        if (ns < max_seg) {
            seg[3 * ns + 0] = i0;
            seg[3 * ns + 1] = step;
            seg[3 * ns + 2] = count;
        }
        ++ns;
        x += count;
    }
    return ns;
}

/*
 * ACSR metadata of the whole mask: seg[N][max_seg][3], nseg[N], row_ptr[N+1]
 * (row_ptr = exclusive prefix sum of the per-row nnzs, Fig. 5(b)).
 * Returns 0, or -(i+1) for the first row i needing more than max_seg runs
 * (that row's nseg is still the true count).
 */
int or_acsr(const or_pattern *p, int max_seg, int32_t *seg, int32_t *nseg, int64_t *row_ptr)
{
    int32_t *cols = (int32_t *)malloc(sizeof(int32_t) * (size_t)(p->n > 0 ? p->n : 1));
    int rc = 0;
    row_ptr[0] = 0;
    for (int i = 0; i < p->n; ++i) {
        int c = or_row_cols(p, i, cols);
        memset(seg + (size_t)i * max_seg * 3, 0, sizeof(int32_t) * 3 * (size_t)max_seg);
        int ns = or_runs_from_cols(cols, c, seg + (size_t)i * max_seg * 3, max_seg);
        nseg[i] = ns;
        if (ns > max_seg && rc == 0) rc = -(i + 1);
        row_ptr[i + 1] = row_ptr[i] + c;
    }
    free(cols);
    return rc;
}

/*
 * Step 4: the paper's regularity check on an explicit rows x cols mask
 * (Listing 4 checkRegularity P:682).  For every row with >= 2
 * non-zeros: a = 1/(i1-i0), b = -i0/(i1-i0); every later non-zero must
 * satisfy i_x*a + b = i_{x-1}*a + b + 1.  A lone column gets a = 1, b = -c
 * and an empty row a = 1, b = 0, nnzs = 0.
 * Outputs a, b (as doubles, for reporting) and nnzs per row.  Returns 1 if
 * regular; 0 otherwise with bad_row, bad_col = the first offending point in
 * row-major scan order.
 */
int or_regularity(const uint8_t *mask, int rows, int ncols, double *a, double *b,
                  int32_t *nnzs, int32_t *bad_row, int32_t *bad_col)
{
    for (int y = 0; y < rows; ++y) {
        const uint8_t *m = mask + (size_t)y * ncols;
        int cnt = 0, i0 = -1, i1 = -1, prev = -1;
        for (int x = 0; x < ncols; ++x) {
            if (!m[x]) continue;
            if (cnt == 0) i0 = x;
            else if (cnt == 1) i1 = x;
            else if (x - prev != i1 - i0) {      /* i_x*a+b != i_{x-1}*a+b+1 */
                *bad_row = y; *bad_col = x;
                return 0;
            }
            prev = x;
            ++cnt;
        }
        nnzs[y] = cnt;
        if (cnt >= 2) { a[y] = 1.0 / (double)(i1 - i0); b[y] = -(double)i0 / (double)(i1 - i0); }
        else if (cnt == 1) { a[y] = 1.0; b[y] = -(double)i0; }
        else { a[y] = 1.0; b[y] = 0.0; }
    }
    *bad_row = -1; *bad_col = -1;
    return 1;
}

/* Step 6 alone: softmax of each row of an ACSR value array. */
void or_softmax_rows(const double *S, const int64_t *row_ptr, int nrows, double *P)
{
    for (int i = 0; i < nrows; ++i) {
        int64_t b = row_ptr[i], e = row_ptr[i + 1];
        if (e <= b) continue;                       /* empty row: no-op */
        double m = S[b];
        for (int64_t t = b + 1; t < e; ++t) if (S[t] > m) m = S[t];
        double l = 0.0;
        for (int64_t t = b; t < e; ++t) l += exp(S[t] - m);
        for (int64_t t = b; t < e; ++t) P[t] = exp(S[t] - m) / l;
    }
}

/* ---- steps 2, 5, 6, 7 for a block of rows of one (b, h) slice ---- */
typedef struct {
    const or_pattern *p;
    const double *q, *k, *v;
    int d;
    double scale;
    int row0, row1;
    const int64_t *row_ptr;   /* may be NULL when S and P are NULL */
    double *S, *P, *O;        /* S, P indexed by row_ptr[i] - row_ptr[row0]; O by (i-row0)*d */
    int tid, nthreads;
} or_job;

static void or_attention_row(const or_job *jb, int i, int32_t *cols, double *s)
{
    const int d = jb->d;
    int c = or_row_cols(jb->p, i, cols);
    double *o = jb->O + (size_t)(i - jb->row0) * d;
    for (int t = 0; t < d; ++t) o[t] = 0.0;
    if (c == 0) return;
    for (int x = 0; x < c; ++x) {                         /* step 5 */
        const double *qi = jb->q + (size_t)i * d, *kj = jb->k + (size_t)cols[x] * d;
        double acc = 0.0;
        for (int t = 0; t < d; ++t) acc += qi[t] * kj[t];
        s[x] = jb->scale * acc;
    }
    double m = s[0];                                      /* step 6 */
    for (int x = 1; x < c; ++x) if (s[x] > m) m = s[x];
    double l = 0.0;
    for (int x = 0; x < c; ++x) l += exp(s[x] - m);
    int64_t base = jb->row_ptr ? jb->row_ptr[i] - jb->row_ptr[jb->row0] : 0;
    for (int x = 0; x < c; ++x) {
        double pij = exp(s[x] - m) / l;
        if (jb->S) jb->S[base + x] = s[x];
        if (jb->P) jb->P[base + x] = pij;
        const double *vj = jb->v + (size_t)cols[x] * d;   /* step 7 */
        for (int t = 0; t < d; ++t) o[t] += pij * vj[t];
    }
}

static void *or_attention_worker(void *arg)
{
    const or_job *jb = (const or_job *)arg;
    int32_t *cols = (int32_t *)malloc(sizeof(int32_t) * (size_t)jb->p->n);
    double *s = (double *)malloc(sizeof(double) * (size_t)jb->p->n);
    /* rows are dealt in blocks of 64, round-robin over threads; every output
       element is written by exactly one thread, so results are deterministic */
    for (int blk = jb->row0 + 64 * jb->tid; blk < jb->row1; blk += 64 * jb->nthreads)
        for (int i = blk; i < blk + 64 && i < jb->row1; ++i)
            or_attention_row(jb, i, cols, s);
    free(cols);
    free(s);
    return NULL;
}

/*
 * Masked attention for rows [row0, row1) of one (b, h) slice.
 * q, k, v: [N][d] row-major fp64.  O: [(row1-row0)][d].  S, P (optional,
 * NULL to skip): ACSR order, element (i, x-th column of row i) at
 * row_ptr[i] - row_ptr[row0] + x (Fig. 5(b)).  nthreads <= 0 means 1.
 */
int or_attention(const or_pattern *p, const double *q, const double *k, const double *v,
                 int d, double scale, int row0, int row1, const int64_t *row_ptr,
                 double *S, double *P, double *O, int nthreads)
{
    if (nthreads <= 0) nthreads = 1;
    if ((S || P) && !row_ptr) return -1;
    or_job *jobs = (or_job *)malloc(sizeof(or_job) * (size_t)nthreads);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        or_job jb = { p, q, k, v, d, scale, row0, row1, row_ptr, S, P, O, t, nthreads };
        jobs[t] = jb;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, or_attention_worker, &jobs[t]);
    or_attention_worker(&jobs[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
    return 0;
}

/* The explicit 0/1 mask, row-major [N][N] (oracle-side only; the GPU path
   never materialises M). */
void or_mask(const or_pattern *p, uint8_t *out)
{
    for (int i = 0; i < p->n; ++i)
        for (int j = 0; j < p->n; ++j)
            out[(size_t)i * p->n + j] = (uint8_t)or_pred(p, i, j);
}

/*
 * Fast O(1) index of one affine run ("Fast indexing", P:504-505 guard),
 * in the complete form of reading A-7: dense column c is the s-th stored
 * non-zero of the run (start, step, count) iff (c - start) is a multiple of
 * step and 0 <= s = (c - start)/step < count.  (In the paper's notation
 * a = 1/step, b = -start/step and s = c*a + b.)  Returns s, or -1 when c is a
 * structural zero of the run.
 */
int or_fast_index(int32_t start, int32_t step, int32_t count, int32_t c)
{
    int32_t off = c - start;
    if (off < 0 || off % step != 0) return -1;
    if (off / step >= count) return -1;
    return off / step;
}
