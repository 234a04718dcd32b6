/*
 * CPU oracle kernels for the bounded-Katz hot path -- TEST INFRASTRUCTURE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load this library, and only as the checker or the timed CPU
 * baseline. The product path (paper_1807_03847_b200) never links it.
 *
 * Restated algorithms (no reference source copied):
 *
 *  oracle_csr_matvec
 *      The reference computes y = A @ x with A = Graph.out_csr(), a 0/1 CSR
 *      whose rows are sorted ascending (/root/reference/pkg/src/katzbounds/
 *      graph.py:177-197) and whose data are fp64 ones (graph.py:193). The
 *      arithmetic lives in the third-party scipy `_sparsetools::csr_matvec`
 *      (scipy, pinned only as >=1.10 by pkg/pyproject.toml:13; 1.18.1 in this
 *      image): for every row i, sum = 0; for jj in [indptr[i], indptr[i+1]):
 *      sum += data[jj] * x[indices[jj]]; y[i] = sum -- a strict sequential
 *      sum in stored (ascending-column) order. data == 1.0 so the product is
 *      exact and FMA contraction cannot change the result.
 *      Threading restates KatzState._matvec (engine.py:181-208): with t > 1
 *      and n >= 2t the rows are cut at np.linspace(0, n, t+1) (engine.py:195)
 *      and each chunk is computed independently -- bitwise identical.
 *
 *  oracle_pcg64_*
 *      numpy's PCG64 bit generator (numpy >= 1.24, not vendored by the
 *      reference; used through np.random.default_rng(seed) in
 *      generate.py:68): 128-bit LCG state' = state * M + inc, output
 *      XSL-RR of the *new* state; Generator.random() = (raw >> 11) * 2^-53.
 *      The jump-ahead is the standard LCG advance (Brown 1994).
 *
 *  oracle_rmat_pairs
 *      generate.py:55-81: for each of `scale` bits, one draw per sampled
 *      pair (draw index = bit * m + e), src_bit = draw >= ab,
 *      dst_bit = (draw >= a && draw < ab) || draw >= abc, shifted in MSB
 *      first; then lo = min, hi = max, keep lo != hi, packed = lo * n + hi.
 *      The caller (numpy) does np.unique of the packed keys (generate.py:80).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef unsigned __int128 u128;

#define PCG_MULT ((((u128)2549297995355413924ULL) << 64) | (u128)4865540595714422341ULL)

static inline uint64_t pcg_out(u128 s) {
    uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    uint64_t x = hi ^ lo;
    unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

static inline u128 pcg_advance(u128 state, u128 delta, u128 mult, u128 inc) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = mult, cur_plus = inc;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

static inline u128 mk128(uint64_t hi, uint64_t lo) { return (((u128)hi) << 64) | lo; }

/* raw 64-bit outputs number [skip, skip+count) of a generator whose current
 * state is (state_hi, state_lo) with increment (inc_hi, inc_lo). */
void oracle_pcg64_raw(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                      uint64_t inc_lo, uint64_t skip, int64_t count,
                      uint64_t *out) {
    u128 inc = mk128(inc_hi, inc_lo);
    u128 s = pcg_advance(mk128(state_hi, state_lo), skip, PCG_MULT, inc);
    for (int64_t i = 0; i < count; i++) {
        s = s * PCG_MULT + inc;
        out[i] = pcg_out(s);
    }
}

/* ---------------- csr matvec ---------------- */

static void matvec_rows(int64_t lo, int64_t hi, const int64_t *indptr,
                        const int32_t *indices, const double *x, double *y) {
    for (int64_t i = lo; i < hi; i++) {
        double sum = 0.0;
        for (int64_t jj = indptr[i]; jj < indptr[i + 1]; jj++)
            sum += x[indices[jj]];
        y[i] = sum;
    }
}

typedef struct {
    int64_t lo, hi;
    const int64_t *indptr;
    const int32_t *indices;
    const double *x;
    double *y;
} mv_job;

static void *mv_worker(void *p) {
    mv_job *j = (mv_job *)p;
    matvec_rows(j->lo, j->hi, j->indptr, j->indices, j->x, j->y);
    return NULL;
}

/* np.linspace(0, n, t+1, dtype=int64): start + i*step truncated toward 0. */
static int64_t linspace_bound(int64_t n, int t, int i) {
    if (i == t) return n;
    double step = (double)n / (double)t;
    return (int64_t)((double)i * step);
}

int oracle_csr_matvec(int64_t n, const int64_t *indptr, const int32_t *indices,
                      const double *x, double *y, int threads) {
    if (threads <= 1 || n < 2 * (int64_t)threads) {
        matvec_rows(0, n, indptr, indices, x, y);
        return 0;
    }
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    mv_job *jobs = (mv_job *)malloc(sizeof(mv_job) * threads);
    for (int i = 0; i < threads; i++) {
        jobs[i].lo = linspace_bound(n, threads, i);
        jobs[i].hi = linspace_bound(n, threads, i + 1);
        jobs[i].indptr = indptr;
        jobs[i].indices = indices;
        jobs[i].x = x;
        jobs[i].y = y;
        pthread_create(&tid[i], NULL, mv_worker, &jobs[i]);
    }
    for (int i = 0; i < threads; i++) pthread_join(tid[i], NULL);
    free(tid);
    free(jobs);
    return 0;
}

/* ---------------- rmat sampling ---------------- */

typedef struct {
    u128 state0, inc;
    int scale;
    int64_t m, e0, e1;
    double a, ab, abc;
    int64_t *src, *dst;
} rmat_job;

static void *rmat_worker(void *p) {
    rmat_job *j = (rmat_job *)p;
    int64_t cnt = j->e1 - j->e0;
    if (cnt <= 0) return NULL;
    memset(j->src + j->e0, 0, sizeof(int64_t) * cnt);
    memset(j->dst + j->e0, 0, sizeof(int64_t) * cnt);
    for (int bit = 0; bit < j->scale; bit++) {
        u128 s = pcg_advance(j->state0, (u128)((uint64_t)bit * (uint64_t)j->m + (uint64_t)j->e0),
                             PCG_MULT, j->inc);
        for (int64_t e = j->e0; e < j->e1; e++) {
            s = s * PCG_MULT + j->inc;
            double draw = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
            int64_t sb = draw >= j->ab;
            int64_t db = ((draw >= j->a) & (draw < j->ab)) | (draw >= j->abc);
            j->src[e] = (j->src[e] << 1) | sb;
            j->dst[e] = (j->dst[e] << 1) | db;
        }
    }
    return NULL;
}

/* Samples the m = n*edge_factor endpoint pairs of generate.py:66-76 and
 * writes packed = lo*n + hi for every non-loop pair into `packed`; returns
 * the number written (order = sample order; caller uniques). src/dst are
 * caller scratch of length m. */
int64_t oracle_rmat_pairs(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                          uint64_t inc_lo, int scale, int64_t m, double a,
                          double ab, double abc, int threads, int64_t *src,
                          int64_t *dst, int64_t *packed) {
    if (threads < 1) threads = 1;
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    rmat_job *jobs = (rmat_job *)malloc(sizeof(rmat_job) * threads);
    for (int i = 0; i < threads; i++) {
        jobs[i].state0 = mk128(state_hi, state_lo);
        jobs[i].inc = mk128(inc_hi, inc_lo);
        jobs[i].scale = scale;
        jobs[i].m = m;
        jobs[i].e0 = m * i / threads;
        jobs[i].e1 = m * (i + 1) / threads;
        jobs[i].a = a;
        jobs[i].ab = ab;
        jobs[i].abc = abc;
        jobs[i].src = src;
        jobs[i].dst = dst;
        pthread_create(&tid[i], NULL, rmat_worker, &jobs[i]);
    }
    for (int i = 0; i < threads; i++) pthread_join(tid[i], NULL);
    free(tid);
    free(jobs);
    int64_t n = (int64_t)1 << scale, w = 0;
    for (int64_t e = 0; e < m; e++) {
        int64_t s = src[e], d = dst[e];
        if (s == d) continue;
        int64_t lo = s < d ? s : d, hi = s < d ? d : s;
        packed[w++] = lo * n + hi;
    }
    return w;
}

/* Same draw stream as oracle_rmat_pairs, but without the two m-long src/dst
 * scratch arrays: each thread walks its sample range in blocks of B samples,
 * replays the `scale` per-bit draws of the block (jump-ahead per bit), and
 * appends the block's non-loop packed keys to its own slice of `packed`.
 * The slices are then compacted in thread order.  Peak memory is the m-long
 * `packed` array alone, which is what makes scale 27 (m = 2^31) fit a 64 GB
 * host.  Key ORDER differs from oracle_rmat_pairs (block-major per thread);
 * the caller sorts, so the unique key set is identical. */
typedef struct {
    u128 state0, inc;
    int scale;
    int64_t m, e0, e1, n_out;
    double a, ab, abc;
    int64_t *packed;
} rmat_lm_job;

#define RMAT_BLOCK 65536

static void *rmat_lm_worker(void *p) {
    rmat_lm_job *j = (rmat_lm_job *)p;
    int64_t src[RMAT_BLOCK], dst[RMAT_BLOCK];
    int64_t w = j->e0, n = (int64_t)1 << j->scale;
    for (int64_t b0 = j->e0; b0 < j->e1; b0 += RMAT_BLOCK) {
        int64_t cnt = j->e1 - b0 < RMAT_BLOCK ? j->e1 - b0 : RMAT_BLOCK;
        memset(src, 0, sizeof(int64_t) * cnt);
        memset(dst, 0, sizeof(int64_t) * cnt);
        for (int bit = 0; bit < j->scale; bit++) {
            u128 s = pcg_advance(j->state0, (u128)((uint64_t)bit * (uint64_t)j->m + (uint64_t)b0),
                                 PCG_MULT, j->inc);
            for (int64_t e = 0; e < cnt; e++) {
                s = s * PCG_MULT + j->inc;
                double draw = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
                int64_t sb = draw >= j->ab;
                int64_t db = ((draw >= j->a) & (draw < j->ab)) | (draw >= j->abc);
                src[e] = (src[e] << 1) | sb;
                dst[e] = (dst[e] << 1) | db;
            }
        }
        for (int64_t e = 0; e < cnt; e++) {
            int64_t s = src[e], d = dst[e];
            if (s == d) continue;
            int64_t lo = s < d ? s : d, hi = s < d ? d : s;
            j->packed[w++] = lo * n + hi;
        }
    }
    j->n_out = w - j->e0;
    return NULL;
}

int64_t oracle_rmat_packed_lowmem(uint64_t state_hi, uint64_t state_lo,
                                  uint64_t inc_hi, uint64_t inc_lo, int scale,
                                  int64_t m, double a, double ab, double abc,
                                  int threads, int64_t *packed) {
    if (threads < 1) threads = 1;
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    rmat_lm_job *jobs = (rmat_lm_job *)malloc(sizeof(rmat_lm_job) * threads);
    for (int i = 0; i < threads; i++) {
        jobs[i].state0 = mk128(state_hi, state_lo);
        jobs[i].inc = mk128(inc_hi, inc_lo);
        jobs[i].scale = scale;
        jobs[i].m = m;
        jobs[i].e0 = m * i / threads;
        jobs[i].e1 = m * (i + 1) / threads;
        jobs[i].a = a;
        jobs[i].ab = ab;
        jobs[i].abc = abc;
        jobs[i].packed = packed;
        pthread_create(&tid[i], NULL, rmat_lm_worker, &jobs[i]);
    }
    for (int i = 0; i < threads; i++) pthread_join(tid[i], NULL);
    int64_t w = 0;
    for (int i = 0; i < threads; i++) {
        if (w != jobs[i].e0)
            memmove(packed + w, packed + jobs[i].e0, sizeof(int64_t) * jobs[i].n_out);
        w += jobs[i].n_out;
    }
    free(tid);
    free(jobs);
    return w;
}

/* ---------------- undirected CSR from sorted unique packed edges ----------
 * packed: sorted unique lo*n+hi with lo<hi. Builds the symmetric CSR with
 * each row sorted ascending (graph.py:191-192 canonical order). */
int oracle_csr_from_packed(int64_t n, int64_t ne, const int64_t *packed,
                           int64_t *indptr, int32_t *indices) {
    memset(indptr, 0, sizeof(int64_t) * (n + 1));
    for (int64_t i = 0; i < ne; i++) {
        int64_t lo = packed[i] / n, hi = packed[i] % n;
        indptr[lo + 1]++;
        indptr[hi + 1]++;
    }
    for (int64_t v = 0; v < n; v++) indptr[v + 1] += indptr[v];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * n);
    memcpy(fill, indptr, sizeof(int64_t) * n);
    /* Row v's neighbours: all lo<v with (lo,v) -- these come first in packed
     * order as lo increases -- then all hi>v with (v,hi). Scanning packed in
     * ascending order appends, for row hi, the lo's ascending; for row lo the
     * hi's ascending; and every lo-neighbour (< v) of row v is appended
     * before any hi-neighbour (> v) only if we do two passes. */
    for (int64_t i = 0; i < ne; i++) { /* pass 1: smaller neighbours */
        int64_t lo = packed[i] / n, hi = packed[i] % n;
        indices[fill[hi]++] = (int32_t)lo;
    }
    for (int64_t i = 0; i < ne; i++) { /* pass 2: larger neighbours */
        int64_t lo = packed[i] / n, hi = packed[i] % n;
        indices[fill[lo]++] = (int32_t)hi;
    }
    free(fill);
    return 0;
}

/* In-place np.unique of a sorted array (generate.py:80); returns the new
 * length.  Used by the low-memory scale-27 golden build. */
int64_t oracle_unique_sorted_inplace(int64_t cnt, int64_t *a) {
    if (cnt == 0) return 0;
    int64_t w = 1;
    for (int64_t i = 1; i < cnt; i++)
        if (a[i] != a[w - 1]) a[w++] = a[i];
    return w;
}
