// K1: fused walk-count SpMV + bound refresh (iterate_once, engine.py:296-319).
//
// One pull step  w_r(v) = alpha * sum_{u in N+(v)} w_{r-1}(u)  over the
// SELL-32 layout of kb_ingest.cu, fused with
//     katz += w; tail = alpha*w; lower = katz + tail (undirected) | katz;
//     upper = katz + tail*gamma
// in exactly numpy's operation order with every multiply and add rounded
// separately (no FMA contraction: __dmul_rn/__dadd_rn), so every row whose
// length is <= the split threshold is bit-identical to scipy's sequential
// csr_matvec (each lane folds its own row in ascending original column
// order).  Rows longer than the threshold are cut into fixed segments whose
// partial sums are combined in segment order by k_heavy_combine: a
// deterministic, hardware-independent order that differs from the pure
// sequential sum only by rounding (<= ~1e-15 relative; north-star tolerance
// 1e-12).
//
// Memory plan per iteration (C2: n=16.8M, nnz=521M):
//   column stream  4 B/slot, read once, L1::no_allocate + L2::evict_first
//   x = w_{r-1}    gathered; the `hot` leading entries (the highest-degree
//                  vertices after relabelling) are staged in shared memory
//                  once per CTA, the rest read through L1/L2
//   katz r+w, w/lower/upper w  (coalesced: lanes own consecutive rows)
#include "kb_internal.cuh"

namespace kb {

namespace {

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ int4 ld_stream_i4(const int32_t *p, uint64_t pol) {
    int4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ int32_t ld_stream_i1(const int32_t *p, uint64_t pol) {
    int32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
        : "=r"(r) : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ void st_stream(double *p, double v) {
    asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

struct IterArgs {
    const int32_t *cols;
    const int64_t *slice_off;
    const int32_t *slice_w;
    const int32_t *vlen;
    int64_t nslices, nvr, nseg, nh;
    int64_t ncols;                  // id space (columns < ncols; checked build)
    int64_t nwide;                  // slices >= nwide are narrow: 4 per grab
    const double *x;
    double *w, *katz, *lower, *upper, *seg_sum;
    double alpha, gamma;
    int undirected;
    int level_only;                 // write w only (dynamic level repair)
    int seg_only;                   // heavy-row segment sums only (no row epilogue)
    int lazy_bounds;                // leave lower/upper to materialize_bounds
    // fused exchange: every w store also goes to the other ranks' buffers
    int npeer;
    double *peer[KB_MAX_PEERS];
    const int32_t *hrow, *vrow;     // explicit row maps (nullptr: implicit)
    int hot;
    int warm;                       // XL 3/4 tier boundary (ids < warm: L1 evict_last)
    // sharded graphs: the hot set is the head of every rank's block of the
    // exchange layout (hot_per entries each, blocks of 2^hot_shift ids)
    int hot_per, hot_shift;
    unsigned long long *counter;
    const unsigned long long *abort;  // speculative launch: exit if set
    // fused cached-pair test (RANKING chain, k_sell_narrow_tma): the last CTA
    // evaluates k_pair_refutes_pub's rule on the level just written
    unsigned long long *pair_done;
    int32_t pair_q, pair_x;
    double pair_eps;
    const int32_t *pair_perm;
    unsigned long long *pair_out, *pair_abort, *pair_pub, *pair_k1c;
    int64_t pair_level;
    int fresh = 0;                  // ones step on a lazily initialised state: katz is 0
};

__device__ __forceinline__ bool aborted(const IterArgs &A) {
    return A.abort && *(const volatile unsigned long long *)A.abort != 0;
}

struct HotMap {
    int hot, per, shift;
    uint32_t mask;
    int warm;     // XL 3/4: ids in [hot, warm) are the L1-resident tier
    int rank;     // ST >= 2 (cluster hot set): this CTA's rank in the cluster
    uint32_t sbase;  // shared::cta address of hot_s
};

template <int ST>
struct Log2 { static constexpr int v = ST <= 1 ? 0 : 1 + Log2<ST / 2>::v; };
template <>
struct Log2<1> { static constexpr int v = 0; };

// XL: 0 = ld.global.nc (read-only path, L1 allocate), 1 = ld.global.cg
// (L2 only), 2 = ld.global.ca with an L2 evict_last hint
template <int XL>
__device__ __forceinline__ double ldx(const double *p) {
    if (XL == 0) return __ldg(p);
    double r;
    if (XL == 1) asm("ld.global.cg.f64 %0, [%1];" : "=d"(r) : "l"(p));
    else asm("{ .reg .b64 pol; createpolicy.fractional.L2::evict_last.b64 pol, 1.0;\n"
             "  ld.global.nc.L2::cache_hint.f64 %0, [%1], pol; }" : "=d"(r) : "l"(p));
    return r;
}

// XL 3: ids in [hot, warm) load with L1::evict_last, colder ones with
// L1::no_allocate (they never displace the warm tier); XL 4: evict_last /
// evict_first
template <int XL>
__device__ __forceinline__ double ldx_tier(const double *p, bool warm) {
    double r;
    if (warm) {
        asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(r) : "l"(p));
    } else if (XL == 3) {
        asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    } else {
        asm("ld.global.nc.L1::evict_first.f64 %0, [%1];" : "=d"(r) : "l"(p));
    }
    return r;
}

template <int XL, int ST>
__device__ __forceinline__ double fetch(const double *__restrict__ hot_s, const HotMap &hm,
                                        const double *__restrict__ x, int32_t c) {
    if (ST >= 2) {
        // cluster hot set: the hm.hot hottest ids are dealt round-robin over
        // the ST CTAs of the cluster (id c lives in CTA c mod ST, slot c / ST);
        // a local slot is a shared-memory load, a remote one a DSMEM load
        // over the cluster network -- off the L1->L2 request path
        if (c >= hm.hot) return ldx<XL>(x + c);
        const int owner = c & (ST - 1);
        const uint32_t la = hm.sbase + ((uint32_t)(c >> Log2<ST>::v) << 3);
        if (owner == hm.rank) return hot_s[c >> Log2<ST>::v];
        uint32_t ra;
        asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(owner));
        double r;
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(r) : "r"(ra));
        return r;
    }
    if (XL >= 3 && !ST) return (c < hm.hot) ? hot_s[c] : ldx_tier<XL>(x + c, c < hm.warm);
    if (!ST) return (c < hm.hot) ? hot_s[c] : ldx<XL>(x + c);
    const int j = (int)((uint32_t)c & hm.mask);
    return (j < hm.per) ? hot_s[(c >> hm.shift) * hm.per + j] : ldx<XL>(x + c);
}

__device__ __forceinline__ void epilogue(const IterArgs &A, int64_t v, double s) {
    KB_DCHECK(v >= 0 && v < A.ncols);
    const double w = __dmul_rn(A.alpha, s);          // engine.py:306
    for (int q = 0; q < A.npeer; q++) A.peer[q][v] = w;  // NVLink stores to the peers
    if (A.level_only) {
        A.w[v] = w;
        return;
    }
    const double k = __dadd_rn(A.katz[v], w);        // :308
    const double t = __dmul_rn(A.alpha, w);          // :309
    A.katz[v] = k;
    A.w[v] = w;                                      // :317
    if (A.lazy_bounds) return;
    st_stream(A.lower + v, A.undirected ? __dadd_rn(k, t) : k);  // :313/:315
    st_stream(A.upper + v, __dadd_rn(k, __dmul_rn(t, A.gamma)));  // :316
}

// Gather of one batch of 8 column slots (two int4 groups) of a lane's row;
// slots at or beyond the row length read as +0.0 without touching memory.
template <int XL, int ST>
__device__ __forceinline__ void gather8(const double *__restrict__ hot_s, const HotMap &hm,
                                        const double *__restrict__ x, int4 ca, int4 cb,
                                        int jb, int len, double v[8], int64_t ncols) {
    const int32_t c[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
#pragma unroll
    for (int q = 0; q < 8; q++) KB_DCHECK(jb + q >= len || (c[q] >= 0 && c[q] < ncols));
    (void)ncols;
#pragma unroll
    for (int q = 0; q < 8; q++)
        v[q] = (jb + q < len) ? fetch<XL, ST>(hot_s, hm, x, c[q]) : 0.0;
}

// epilogue with katz already loaded (narrow-slice path)
__device__ __forceinline__ void epilogue_k(const IterArgs &A, int64_t v, double s, double kv) {
    const double w = __dmul_rn(A.alpha, s);
    for (int q = 0; q < A.npeer; q++) A.peer[q][v] = w;
    if (A.level_only) {
        A.w[v] = w;
        return;
    }
    const double k = __dadd_rn(kv, w);
    const double t = __dmul_rn(A.alpha, w);
    A.katz[v] = k;
    A.w[v] = w;
    if (A.lazy_bounds) return;
    st_stream(A.lower + v, A.undirected ? __dadd_rn(k, t) : k);
    st_stream(A.upper + v, __dadd_rn(k, __dmul_rn(t, A.gamma)));
}

// Persistent kernel: each warp takes 32-row slices off a global counter.
// Slices are ordered by descending length so the longest chains start first.
// DEPTH batches of 8 gathers per lane are kept in flight (software pipeline):
// the loads of batch i+1..i+DEPTH-1 are issued before batch i is folded, so
// the in-order dependent add chain never waits on a single batch's latency.
// four narrow slices (width <= 4) from slice s0 on, folded per lane
template <int XL, int ST, int Q = 4>
__device__ __forceinline__ void narrow_group(const IterArgs &A, int64_t s0, int lane,
                                             const double *__restrict__ hot_s,
                                             const HotMap &hm, const double *__restrict__ x,
                                             uint64_t pol) {
    int len[Q], w[Q];
    const int32_t *base[Q];
    int64_t row[Q];
    double kz[Q];
#pragma unroll
    for (int q = 0; q < Q; q++) {
        const int64_t sq = s0 + q;
        const int64_t vq = sq * 32 + lane;
        const bool ok = sq < A.nslices && vq < A.nvr;
        len[q] = ok ? A.vlen[vq] : 0;
        w[q] = sq < A.nslices ? A.slice_w[sq] : 0;
        base[q] = A.cols + (sq < A.nslices ? A.slice_off[sq] : 0);
        row[q] = -1;
        if (ok && vq >= A.nseg)
            row[q] = A.vrow ? A.vrow[vq - A.nseg] : A.nh + (vq - A.nseg);
        kz[q] = (row[q] >= 0 && !A.level_only) ? A.katz[row[q]] : 0.0;
    }
    int32_t cc[Q][4];
#pragma unroll
    for (int q = 0; q < Q; q++)
#pragma unroll
        for (int j = 0; j < 4; j++)
            cc[q][j] = (j < w[q]) ? ld_stream_i1(base[q] + j * 32 + lane, pol) : 0;
    double v[Q][4];
#pragma unroll
    for (int q = 0; q < Q; q++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
            KB_DCHECK(j >= len[q] || (cc[q][j] >= 0 && cc[q][j] < A.ncols));
            v[q][j] = (j < len[q]) ? fetch<XL, ST>(hot_s, hm, x, cc[q][j]) : 0.0;
        }
#pragma unroll
    for (int q = 0; q < Q; q++) {
        double sum = 0.0;
#pragma unroll
        for (int j = 0; j < 4; j++) sum = __dadd_rn(sum, v[q][j]);
        const int64_t vq = (s0 + q) * 32 + lane;
        if (s0 + q < A.nslices && vq < A.nvr) {
            if (vq < A.nseg) A.seg_sum[vq] = sum;
            else if (!A.seg_only) epilogue_k(A, row[q], sum, kz[q]);
        }
    }
}

template <int DEPTH, int XL, int ST = 0>
__global__ void __launch_bounds__(1024, 1) k_sell_iterate(IterArgs A) {
    if (aborted(A)) return;
    extern __shared__ double hot_s[];
    unsigned crank = 0;
    if (ST >= 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const HotMap hm{A.hot, A.hot_per, A.hot_shift, (1u << A.hot_shift) - 1u, A.warm, (int)crank,
                    (uint32_t)__cvta_generic_to_shared(hot_s)};
    // The hot set is one contiguous range (or, for a shard, the head of
    // every rank's block): TMA bulk copies global -> shared, completing on
    // an mbarrier, while the CTA's threads only wait.
    const int nseg_hot = ST == 1 ? (A.hot_per > 0 ? A.hot / A.hot_per : 0) : 1;
    const int seg_len = ST == 1 ? A.hot_per : A.hot;
    if (ST >= 2) {
        // this CTA's share of the cluster hot set: ids crank, crank+ST, ...
        constexpr int CS = ST >= 2 ? ST : 1;
        for (int i = threadIdx.x; i < A.hot / CS; i += blockDim.x)
            hot_s[i] = A.x[(int64_t)i * CS + crank];
        // every CTA's share is in place before any remote read
        asm volatile("barrier.cluster.arrive.release.aligned;\n"
                     "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (A.hot > 0 && (seg_len & 1) == 0 && nseg_hot >= 1) {
        __shared__ __align__(8) unsigned long long bar;
        const unsigned sbar = (unsigned)__cvta_generic_to_shared(&bar);
        const unsigned sdst = (unsigned)__cvta_generic_to_shared(hot_s);
        const unsigned bytes = (unsigned)seg_len * 8u;
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                         ::"r"(sbar), "r"(bytes * (unsigned)nseg_hot) : "memory");
            for (int r = 0; r < nseg_hot; r++) {
                const double *src = ST == 1 ? A.x + ((int64_t)r << A.hot_shift) : A.x;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
                             "[%0], [%1], %2, [%3];"
                             ::"r"(sdst + (unsigned)r * bytes), "l"(src), "r"(bytes), "r"(sbar)
                             : "memory");
            }
        }
        unsigned done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
                         "  selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(sbar) : "memory");
    } else if (ST == 1) {
        for (int i = threadIdx.x; i < A.hot; i += blockDim.x) {
            const int r = i / A.hot_per, j = i - r * A.hot_per;
            hot_s[i] = A.x[((int64_t)r << A.hot_shift) + j];
        }
    } else {
        for (int i = threadIdx.x; i < A.hot; i += blockDim.x) hot_s[i] = A.x[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const double *__restrict__ x = A.x;
    const uint64_t pol = evict_first_policy();
    const int4 zero4 = make_int4(0, 0, 0, 0);
    const int64_t nwide_grabs = A.nwide;
    const int64_t grabs = A.nwide + (A.nslices - A.nwide + 3) / 4;
    for (;;) {
        unsigned long long c = 0;
        if (lane == 0) c = atomicAdd(A.counter, 1ULL);
        c = __shfl_sync(0xffffffffu, c, 0);
        if ((int64_t)c >= grabs) break;
        if ((int64_t)c >= nwide_grabs) {
            // four narrow slices (width <= 4) at once: their loads overlap
            narrow_group<XL, ST>(A, A.nwide + ((int64_t)c - nwide_grabs) * 4, lane, hot_s, hm,
                                 x, pol);
            continue;
        }
        const int64_t s = (int64_t)c;
        const int64_t vr = (int64_t)s * 32 + lane;
        const int len = (vr < A.nvr) ? A.vlen[vr] : 0;
        const int w = A.slice_w[s];
        const int32_t *base = A.cols + A.slice_off[s];
        double sum = 0.0;
        if (w <= 4) {
            int32_t c[4];
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (j < w) c[j] = ld_stream_i1(base + j * 32 + lane, pol);
#pragma unroll
            for (int j = 0; j < 4; j++)
                if (j < len) sum = __dadd_rn(sum, fetch<XL, ST>(hot_s, hm, x, c[j]));
        } else {
            const int32_t *p = base + lane * 4;
            const int w4 = w >> 2;             // int4 groups per lane
            const int nb = (w4 + 1) >> 1;      // batches of 8 slots
            double v[DEPTH][8];
#pragma unroll
            for (int d = 0; d < DEPTH; d++) {
                if (d < nb) {
                    const int g0 = 2 * d;
                    const int4 ca = ld_stream_i4(p + (int64_t)g0 * 128, pol);
                    const int4 cb = (g0 + 1 < w4) ? ld_stream_i4(p + (int64_t)(g0 + 1) * 128, pol)
                                                  : zero4;
                    gather8<XL, ST>(hot_s, hm, x, ca, cb, g0 * 4, len, v[d], A.ncols);
                }
            }
            for (int b = 0; b < nb; b += DEPTH) {
#pragma unroll
                for (int d = 0; d < DEPTH; d++) {
                    if (b + d < nb) {
#pragma unroll
                        for (int q = 0; q < 8; q++) sum = __dadd_rn(sum, v[d][q]);
                        const int bn = b + d + DEPTH;  // refill this slot
                        if (bn < nb) {
                            const int g0 = 2 * bn;
                            const int4 ca = ld_stream_i4(p + (int64_t)g0 * 128, pol);
                            const int4 cb = (g0 + 1 < w4)
                                                ? ld_stream_i4(p + (int64_t)(g0 + 1) * 128, pol)
                                                : zero4;
                            gather8<XL, ST>(hot_s, hm, x, ca, cb, g0 * 4, len, v[d], A.ncols);
                        }
                    }
                }
            }
        }
        if (vr < A.nvr) {
            if (vr < A.nseg) A.seg_sum[vr] = sum;
            else if (!A.seg_only) epilogue(A, A.vrow ? A.vrow[vr - A.nseg] : A.nh + (vr - A.nseg), sum);
        }
    }
    if (A.npeer) __threadfence_system();  // peer stores visible before the next collective
    if (ST >= 2)   // no CTA leaves while the others may still read its share
        asm volatile("barrier.cluster.arrive.release.aligned;\n"
                     "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Graphs whose slices are all narrow (width <= 4: grids, meshes): no hot
// set, fewer registers, two CTAs per SM and a static slice-group schedule,
// so twice the warps keep loads in flight (K1 on C4 is latency-bound).
template <int Q>
__global__ void __launch_bounds__(1024, 2) k_sell_narrow(IterArgs A) {
    if (aborted(A)) return;
    const int lane = threadIdx.x & 31;
    const uint64_t pol = evict_first_policy();
    const HotMap hm{0, 0, 0, 0u, 0};
    const int64_t groups = (A.nslices + Q - 1) / Q;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t gi = wid; gi < groups; gi += nw)
        narrow_group<0, false, Q>(A, gi * Q, lane, nullptr, hm, A.x, pol);
    if (A.npeer) __threadfence_system();
}


// All-narrow graphs, software-pipelined: a static schedule of Q-slice groups
// per warp where the next group's row metadata, katz and column ids are
// loaded before the current group's gathers are consumed, so the three
// dependent round trips of a group (metadata -> columns -> omega) overlap
// with the previous group's.
template <int Q>
struct NarrowStage {
    int len[Q];
    int64_t row[Q];
    double kz[Q];
    int32_t cc[Q][4];
};

template <int Q>
__device__ __forceinline__ void narrow_load(const IterArgs &A, int64_t s0, int lane, uint64_t pol,
                                            NarrowStage<Q> &S) {
#pragma unroll
    for (int q = 0; q < Q; q++) {
        const int64_t sq = s0 + q;
        const int64_t vq = sq * 32 + lane;
        const bool ok = sq < A.nslices && vq < A.nvr;
        S.len[q] = ok ? A.vlen[vq] : 0;
        const int w = sq < A.nslices ? A.slice_w[sq] : 0;
        const int32_t *base = A.cols + (sq < A.nslices ? A.slice_off[sq] : 0);
        S.row[q] = -1;
        if (ok && vq >= A.nseg) S.row[q] = A.vrow ? A.vrow[vq - A.nseg] : A.nh + (vq - A.nseg);
        S.kz[q] = (S.row[q] >= 0 && !A.level_only) ? A.katz[S.row[q]] : 0.0;
#pragma unroll
        for (int j = 0; j < 4; j++) S.cc[q][j] = (j < w) ? ld_stream_i1(base + j * 32 + lane, pol) : 0;
    }
}

template <int Q>
__global__ void __launch_bounds__(1024, 1) k_sell_narrow_pf(IterArgs A) {
    if (aborted(A)) return;
    const int lane = threadIdx.x & 31;
    const uint64_t pol = evict_first_policy();
    const HotMap hm{0, 0, 0, 0u, 0, 0, 0u};
    const int64_t groups = (A.nslices + Q - 1) / Q;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (wid >= groups) return;
    NarrowStage<Q> cur;
    narrow_load<Q>(A, wid * Q, lane, pol, cur);
    for (int64_t gi = wid; gi < groups; gi += nw) {
        NarrowStage<Q> nxt;
        const int64_t gn = gi + nw;
        if (gn < groups) narrow_load<Q>(A, gn * Q, lane, pol, nxt);
        double v[Q][4];
#pragma unroll
        for (int q = 0; q < Q; q++)
#pragma unroll
            for (int j = 0; j < 4; j++) {
                KB_DCHECK(j >= cur.len[q] || (cur.cc[q][j] >= 0 && cur.cc[q][j] < A.ncols));
                v[q][j] = (j < cur.len[q]) ? fetch<0, 0>(nullptr, hm, A.x, cur.cc[q][j]) : 0.0;
            }
#pragma unroll
        for (int q = 0; q < Q; q++) {
            double sum = 0.0;
#pragma unroll
            for (int j = 0; j < 4; j++) sum = __dadd_rn(sum, v[q][j]);
            const int64_t vq = (gi * Q + q) * 32 + lane;
            if (gi * Q + q < A.nslices && vq < A.nvr) {
                if (vq < A.nseg) A.seg_sum[vq] = sum;
                else if (!A.seg_only) epilogue_k(A, cur.row[q], sum, cur.kz[q]);
            }
        }
        if (gn < groups) cur = nxt;
    }
    if (A.npeer) __threadfence_system();
}

// All-narrow graphs with the streams moved by TMA: one producer thread per
// CTA bulk-copies chunks of NB_CH consecutive slices -- their column slots,
// row lengths and katz rows, all contiguous -- into a ring of NB_ST
// shared-memory stages (mbarrier complete_tx), and 31 consumer warps take
// two slices of a landed chunk each: column ids come from shared memory, so
// a slice's only global round trip is its omega gather, and the streams stay
// in flight however long the gathers take.  Chunks go round-robin over the
// CTAs; the slices past the last whole chunk are read directly.  Needs
// implicit rows and no segments (nh = 0), which every all-narrow layout has.
constexpr int NB_CH = 62;          // slices per chunk (two per consumer warp)
constexpr int NB_ST = 3;           // stages
constexpr int NB_COLS_B = NB_CH * 32 * 4 * 4;   // up to width 4
constexpr int NB_VLEN_B = NB_CH * 32 * 4;
constexpr int NB_KATZ_B = NB_CH * 32 * 8;
constexpr int NB_STAGE_B = NB_COLS_B + NB_VLEN_B + NB_KATZ_B;
constexpr size_t NB_SMEM = (size_t)NB_ST * NB_STAGE_B;

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     "  selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
}

__device__ __forceinline__ void bulk_g2s(unsigned dst, const void *src, unsigned bytes,
                                         unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
                 "[%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

// one slice of a narrow layout, its column ids and lengths given
__device__ __forceinline__ double narrow_slice_sum(const double *__restrict__ x, const int32_t c[4],
                                                   int len) {
    double v[4];
#pragma unroll
    for (int j = 0; j < 4; j++) v[j] = (j < len) ? __ldg(x + c[j]) : 0.0;
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < 4; j++) sum = __dadd_rn(sum, v[j]);
    return sum;
}

// k_pair_refutes_pub's rule (kb_check.cu) on the level this launch wrote, by
// the last CTA to finish (its stores fenced device-wide before it counts in)
__device__ void fused_pair_test(const IterArgs &A) {
    const int32_t q = A.pair_q, x = A.pair_x;
    const double tq = __dmul_rn(A.alpha, __ldcg(A.w + q));
    const double tx = __dmul_rn(A.alpha, __ldcg(A.w + x));
    const double kq = __ldcg(A.katz + q), kx = __ldcg(A.katz + x);
    const double lq = A.undirected ? __dadd_rn(kq, tq) : kq;
    const double lx = A.undirected ? __dadd_rn(kx, tx) : kx;
    const double uq = __dadd_rn(kq, __dmul_rn(tq, A.gamma));
    const bool above = lx > lq || (lx == lq && A.pair_perm[x] < A.pair_perm[q]);
    const bool ref = above && lx <= __dsub_rn(uq, A.pair_eps);
    A.pair_out[0] = ref ? 1ull : 0ull;
    A.pair_abort[0] = ref ? 0ull : 1ull;
    A.pair_k1c[0] = 0ull;
    A.pair_pub[0] = ref ? 1ull : 0ull;
    A.pair_pub[3] = (unsigned long long)A.pair_level;
}

__global__ void __launch_bounds__(1024, 1) k_sell_narrow_tma(IterArgs A, int64_t nfull) {
    if (aborted(A)) return;
    extern __shared__ int4 nb_smem4[];                   // 16-byte aligned (bulk copies)
    unsigned char *nb_smem = (unsigned char *)nb_smem4;
    __shared__ __align__(8) unsigned long long full[NB_ST], empty[NB_ST];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ncw = (int)(blockDim.x >> 5) - 1;          // consumer warps
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(nb_smem);
    const unsigned fbar = (unsigned)__cvta_generic_to_shared(full);
    const unsigned ebar = (unsigned)__cvta_generic_to_shared(empty);
    if (threadIdx.x == 0) {
        for (int i = 0; i < NB_ST; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fbar + 8 * i));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ebar + 8 * i), "r"(ncw));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t G = gridDim.x;
    const int64_t nmine = nfull > blockIdx.x ? (nfull - 1 - blockIdx.x) / G + 1 : 0;
    const double *__restrict__ x = A.x;
    if (warp == 0) {
        if (lane == 0) {
            for (int64_t k = 0; k < nmine; k++) {
                const int st = (int)(k % NB_ST);
                const unsigned r = (unsigned)(k / NB_ST);
                const int64_t s0 = (blockIdx.x + k * G) * NB_CH;
                const int64_t off0 = A.slice_off[s0], off1 = A.slice_off[s0 + NB_CH];
                const unsigned colsB = (unsigned)((off1 - off0) * 4);
                const unsigned katzB = A.level_only ? 0u : (unsigned)NB_KATZ_B;
                mbar_wait(ebar + 8 * st, (r & 1) ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             ::"r"(fbar + 8 * st), "r"(colsB + NB_VLEN_B + katzB) : "memory");
                const unsigned d = sbase + (unsigned)st * NB_STAGE_B;
                if (colsB) bulk_g2s(d, A.cols + off0, colsB, fbar + 8 * st);
                bulk_g2s(d + NB_COLS_B, A.vlen + s0 * 32, NB_VLEN_B, fbar + 8 * st);
                if (katzB) bulk_g2s(d + NB_COLS_B + NB_VLEN_B, A.katz + s0 * 32, katzB,
                                    fbar + 8 * st);
            }
        }
    } else {
        const int cw = warp - 1;
        for (int64_t k = 0; k < nmine; k++) {
            const int st = (int)(k % NB_ST);
            const unsigned r = (unsigned)(k / NB_ST);
            const int64_t s0 = (blockIdx.x + k * G) * NB_CH;
            // this warp's two slices and their column offsets in the chunk
            // (exclusive prefix of 32 * width over the chunk's slices)
            const int qa = cw, qb = cw + ncw;
            const int wa_l = lane < NB_CH ? A.slice_w[s0 + lane] : 0;
            const int wb_l = lane + 32 < NB_CH ? A.slice_w[s0 + lane + 32] : 0;
            int pa = wa_l, pb = wb_l;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int ta = __shfl_up_sync(0xffffffffu, pa, o);
                const int tb = __shfl_up_sync(0xffffffffu, pb, o);
                if (lane >= o) { pa += ta; pb += tb; }
            }
            const int tota = __shfl_sync(0xffffffffu, pa, 31);
            pb += tota;                                   // inclusive over 0..lane+32
            const int ea = (pa - wa_l) * 32, eb = (pb - wb_l) * 32;   // exclusive, in ints
            const int w_a = __shfl_sync(0xffffffffu, qa < 32 ? wa_l : wb_l, qa & 31);
            const int o_a = __shfl_sync(0xffffffffu, qa < 32 ? ea : eb, qa & 31);
            const int w_b = __shfl_sync(0xffffffffu, qb < 32 ? wa_l : wb_l, qb & 31);
            const int o_b = __shfl_sync(0xffffffffu, qb < 32 ? ea : eb, qb & 31);
            mbar_wait(fbar + 8 * st, r & 1);
            const unsigned char *stg = nb_smem + (size_t)st * NB_STAGE_B;
            const int32_t *cs = (const int32_t *)stg;
            const int32_t *vs = (const int32_t *)(stg + NB_COLS_B);
            const double *ks = (const double *)(stg + NB_COLS_B + NB_VLEN_B);
            const bool hb = qb < NB_CH;
            int32_t ca[4], cb[4];
#pragma unroll
            for (int j = 0; j < 4; j++) {
                ca[j] = j < w_a ? cs[o_a + j * 32 + lane] : 0;
                cb[j] = (hb && j < w_b) ? cs[o_b + j * 32 + lane] : 0;
            }
            const int la = vs[qa * 32 + lane];
            const int lb = hb ? vs[qb * 32 + lane] : 0;
            const double ka = A.level_only ? 0.0 : ks[qa * 32 + lane];
            const double kb2 = (hb && !A.level_only) ? ks[qb * 32 + lane] : 0.0;
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ebar + 8 * st)
                             : "memory");
#pragma unroll
            for (int j = 0; j < 4; j++) {
                KB_DCHECK(j >= la || (ca[j] >= 0 && ca[j] < A.ncols));
                KB_DCHECK(j >= lb || (cb[j] >= 0 && cb[j] < A.ncols));
            }
            const double sa = narrow_slice_sum(x, ca, la);
            const double sb = narrow_slice_sum(x, cb, lb);
            epilogue_k(A, (s0 + qa) * 32 + lane, sa, ka);
            if (hb) epilogue_k(A, (s0 + qb) * 32 + lane, sb, kb2);
        }
        // the slices past the last whole chunk: direct loads
        const int64_t gw = (int64_t)blockIdx.x * ncw + cw, nwarps = G * ncw;
        const uint64_t pol = evict_first_policy();
        for (int64_t s = nfull * NB_CH + gw; s < A.nslices; s += nwarps) {
            const int64_t vq = s * 32 + lane;
            const int w = A.slice_w[s];
            const int32_t *base = A.cols + A.slice_off[s];
            int32_t c[4];
#pragma unroll
            for (int j = 0; j < 4; j++) c[j] = j < w ? ld_stream_i1(base + j * 32 + lane, pol) : 0;
            const int len = vq < A.nvr ? A.vlen[vq] : 0;
            const double sum = narrow_slice_sum(x, c, len);
            if (vq < A.nvr) epilogue_k(A, vq, sum, A.level_only ? 0.0 : A.katz[vq]);
        }
    }
    if (A.npeer) __threadfence_system();
    if (A.pair_done) {
        __threadfence();                       // this thread's row stores
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(A.pair_done, 1ull) == gridDim.x - 1) {
            __threadfence();
            fused_pair_test(A);
            *A.pair_done = 0ull;               // ready for the next launch
        }
    }
}

// First iteration: x = levels[0] = ones, so every sequential row (or segment)
// sum is exactly its length -- the same bits K1 would produce -- and no
// gather is needed: w_1 = alpha * deg.
__global__ void k_ones_step(IterArgs A) {
    const int64_t vr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (vr >= A.nvr) return;
    const double s = (double)A.vlen[vr];
    if (vr < A.nseg) {
        A.seg_sum[vr] = s;
    } else {
        const int64_t v = A.vrow ? A.vrow[vr - A.nseg] : A.nh + (vr - A.nseg);
        if (A.fresh) epilogue_k(A, v, s, 0.0);   // katz_0 = 0 (not written yet)
        else epilogue(A, v, s);
    }
    if (A.npeer) __threadfence_system();
}

// the rows without arcs after the first step of a lazily initialised state:
// katz = lower = upper = 0 (engine.py:148-149, then the collapse of :313-316)
__global__ void k_fresh_tail(double *katz, double *lower, double *upper, int64_t nv,
                             int64_t n) {
    const int64_t i = nv + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    katz[i] = 0.0;
    lower[i] = 0.0;
    upper[i] = 0.0;
}

// heavy row h = combine its segment sums in segment order, then epilogue
__global__ void k_heavy_combine(IterArgs A, const int32_t *seg_ptr,
                                const int32_t *seg_list) {
    int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (h >= A.nh || aborted(A)) return;
    double s = 0.0;
    for (int q = seg_ptr[h]; q < seg_ptr[h + 1]; q++) {
        KB_DCHECK(seg_list[q] >= 0 && seg_list[q] < A.nseg);
        s = __dadd_rn(s, A.seg_sum[seg_list[q]]);
    }
    epilogue(A, A.hrow ? A.hrow[h] : h, s);
}

// The same fold, a warp per heavy row: the lanes load 32 segment sums at a
// time (independent loads in flight) and lane 0 adds them in segment order.
// A thread per row left the hub rows' ~200 dependent load pairs as the tail
// of every level (26 us at C2).
// Rows [0, nwarp) take a warp each (the long ones: fresh layouts order heavy
// rows by descending length), the rest a thread each.
__global__ void k_heavy_combine_w(IterArgs A, const int32_t *seg_ptr, const int32_t *seg_list,
                                  int64_t nwarp) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (aborted(A)) return;
    if (t >= nwarp * 32) {
        const int64_t h = nwarp + (t - nwarp * 32);
        if (h >= A.nh) return;
        double s = 0.0;
        for (int q = seg_ptr[h]; q < seg_ptr[h + 1]; q++) {
            KB_DCHECK(seg_list[q] >= 0 && seg_list[q] < A.nseg);
            s = __dadd_rn(s, A.seg_sum[seg_list[q]]);
        }
        epilogue(A, A.hrow ? A.hrow[h] : h, s);
        return;
    }
    const int64_t h = t >> 5;
    const int lane = threadIdx.x & 31;
    const int q0 = seg_ptr[h], q1 = seg_ptr[h + 1];
    double s = 0.0;
    // up to 8 x 32 segment sums loaded at once (one round of latency for the
    // hubs' ~200 segments), then folded in order by lane 0
    constexpr int R = 8;
    for (int b0 = q0; b0 < q1; b0 += 32 * R) {
        double v[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int q = b0 + r * 32 + lane;
            v[r] = 0.0;
            if (q < q1) {
                KB_DCHECK(seg_list[q] >= 0 && seg_list[q] < A.nseg);
                v[r] = A.seg_sum[seg_list[q]];
            }
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int b = b0 + r * 32;
            const int cnt = max(0, min(32, q1 - b));
            for (int j = 0; j < cnt; j++) {
                const double t = __shfl_sync(0xffffffffu, v[r], j);
                if (lane == 0) s = __dadd_rn(s, t);
            }
        }
    }
    if (lane == 0) epilogue(A, A.hrow ? A.hrow[h] : h, s);
}

// rows without out-arcs: w = 0, katz unchanged (0), bounds collapse to katz
__global__ void k_empty_rows(double *upper, double *lower, const double *katz,
                             int64_t nv, int64_t n) {
    int64_t i = nv + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    lower[i] = katz[i];
    upper[i] = katz[i];
}

// Overflow rows (dynamic batches that outgrew their SELL lane): recomputed
// from the canonical CSR with K1's summation order -- one sequential chain,
// or split-sized segments combined in order -- after K1 left them at +0.
// One warp per row.
__global__ void k_ovf_rows(IterArgs A, const int32_t *rows, int64_t nr, const int32_t *perm,
                           const int32_t *iperm, const int64_t *indptr, const int32_t *rlen,
                           const int32_t *indices, int64_t split, double *sums = nullptr) {
    if (aborted(A)) return;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= nr) return;
    const int32_t v = rows[warp];
    const int32_t o = perm[v];
    const int32_t *row = indices + indptr[o];
    const int64_t L = rlen[o];
    if (L > OVF_LONG) return;  // k_ovf_long
    const double *__restrict__ x = A.x;
    double s = 0.0;
    if (L <= split) {
        for (int64_t base = 0; base < L; base += 32) {
            const int64_t j = base + lane;
            const double val = j < L ? x[iperm[row[j]]] : 0.0;
            const int cnt = (int)min((int64_t)32, L - base);
            for (int q = 0; q < cnt; q++) {
                const double t = __shfl_sync(0xffffffffu, val, q);
                if (lane == 0) s = __dadd_rn(s, t);
            }
        }
    } else {
        const int64_t nseg = (L + split - 1) / split;
        for (int64_t g0 = 0; g0 < nseg; g0 += 32) {
            const int64_t sg = g0 + lane;
            double ss = 0.0;
            if (sg < nseg) {
                const int64_t a = sg * split, b = min(L, a + split);
                for (int64_t j = a; j < b; j++) ss = __dadd_rn(ss, x[iperm[row[j]]]);
            }
            const int cnt = (int)min((int64_t)32, nseg - g0);
            for (int q = 0; q < cnt; q++) {
                const double t = __shfl_sync(0xffffffffu, ss, q);
                if (lane == 0) s = __dadd_rn(s, t);
            }
        }
    }
    if (lane == 0) {
        if (sums) sums[warp] = s;      // side-stream mode: k_ovf_merge applies it
        else epilogue(A, v, s);
    }
}

// Long overflow rows, a block each.  A row of at most split arcs is one
// serial chain: warps 1.. gather the next 2048 values into shared memory
// while thread 0 folds the current ones, so the chain never waits on a
// gather.  A segmented row (> split arcs) folds up to 8 segments at once, a
// warp each (lanes gather 256 values ahead while lane 0 folds), and thread
// 0 combines the segment sums in order -- K1's order in both cases.
constexpr int OVF_CHUNK = 2048;
constexpr int OVF_WCHUNK = 256;

__global__ void __launch_bounds__(256) k_ovf_long(IterArgs A, const int32_t *rows,
                                                  const int32_t *perm, const int32_t *iperm,
                                                  const int64_t *indptr, const int32_t *rlen,
                                                  const int32_t *indices, int64_t split,
                                                  double *sums = nullptr) {
    if (aborted(A)) return;
    __shared__ double buf[2][OVF_CHUNK];
    __shared__ double segsum[8];
    const int32_t v = rows[blockIdx.x];
    const int32_t o = perm[v];
    const int32_t *row = indices + indptr[o];
    const int64_t L = rlen[o];
    const double *__restrict__ x = A.x;
    const int tid = threadIdx.x;
    double s = 0.0;
    if (L <= split) {
        const int64_t nchunks = (L + OVF_CHUNK - 1) / OVF_CHUNK;
        auto stage = [&](int64_t c, int nthreads, int t0) {
            const int64_t a = c * OVF_CHUNK, b = min(L, a + OVF_CHUNK);
            double *d = buf[c & 1];
            for (int64_t j = a + (tid - t0); j < b; j += nthreads) d[j - a] = x[iperm[row[j]]];
        };
        stage(0, blockDim.x, 0);
        __syncthreads();
        for (int64_t c = 0; c < nchunks; c++) {
            if (tid >= 32) {
                if (c + 1 < nchunks) stage(c + 1, blockDim.x - 32, 32);
            } else if (tid == 0) {
                const int n = (int)(min(L, (c + 1) * OVF_CHUNK) - c * OVF_CHUNK);
                const double *d = buf[c & 1];
#pragma unroll 8
                for (int j = 0; j < n; j++) s = __dadd_rn(s, d[j]);
            }
            __syncthreads();
        }
    } else {
        const int warp = tid >> 5, lane = tid & 31;
        double *wb = &buf[0][0] + warp * 2 * OVF_WCHUNK;   // 2 x 256 per warp
        const int64_t nseg = (L + split - 1) / split;
        for (int64_t g0 = 0; g0 < nseg; g0 += 8) {
            const int64_t sg = g0 + warp;
            if (sg < nseg) {
                const int64_t a = sg * split, b = min(L, a + split);
                const int64_t nch = (b - a + OVF_WCHUNK - 1) / OVF_WCHUNK;
                double val[OVF_WCHUNK / 32];
                auto gather = [&](int64_t c) {
#pragma unroll
                    for (int q = 0; q < OVF_WCHUNK / 32; q++) {
                        const int64_t j = a + c * OVF_WCHUNK + q * 32 + lane;
                        val[q] = j < b ? x[iperm[row[j]]] : 0.0;
                    }
                };
                gather(0);
                double ss = 0.0;
                for (int64_t c = 0; c < nch; c++) {
                    double *d = wb + (c & 1) * OVF_WCHUNK;
#pragma unroll
                    for (int q = 0; q < OVF_WCHUNK / 32; q++) d[q * 32 + lane] = val[q];
                    __syncwarp();
                    if (c + 1 < nch) gather(c + 1);   // in flight during the fold
                    if (lane == 0) {
                        const int n = (int)min((int64_t)OVF_WCHUNK, b - a - c * OVF_WCHUNK);
#pragma unroll 8
                        for (int j = 0; j < n; j++) ss = __dadd_rn(ss, d[j]);
                    }
                    __syncwarp();
                }
                if (lane == 0) segsum[warp] = ss;
            }
            __syncthreads();
            if (tid == 0) {
                const int cnt = (int)min((int64_t)8, nseg - g0);
                for (int q = 0; q < cnt; q++) s = __dadd_rn(s, segsum[q]);
            }
            __syncthreads();
        }
    }
    if (tid == 0) {
        if (sums) sums[blockIdx.x] = s;
        else epilogue(A, v, s);
    }
}

// Side-stream mode: the overflow rows' sums were computed concurrently with
// K1 (which left those rows at +0 and katz unchanged: katz + 0.0 is katz);
// applying the epilogue now gives the same bits as the serial passes.
__global__ void k_ovf_merge(IterArgs A, const int32_t *rows, int64_t nr, const int32_t *perm,
                            const int32_t *rlen, const double *sums,
                            const int32_t *long_rows, int64_t nlong,
                            const double *long_sums) {
    if (aborted(A)) return;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < nr) {
        const int32_t v = rows[t];
        if (rlen[perm[v]] <= OVF_LONG) epilogue(A, v, sums[t]);
    } else if (t < nr + nlong) {
        epilogue(A, long_rows[t - nr], long_sums[t - nr]);
    }
}

// explicit empty rows (after updates): w = 0 and the bounds collapse to katz
__global__ void k_zero_rows(const int32_t *zrows, int64_t nz, double *w, double *lower,
                            double *upper, const double *katz, int level_only) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nz) return;
    const int32_t v = zrows[i];
    w[v] = 0.0;
    if (!level_only) {
        lower[v] = katz[v];
        upper[v] = katz[v];
    }
}

__global__ void k_gather(const int32_t *iperm, const double *src, double *dst,
                         int64_t n) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    dst[i] = src[iperm[i]];
}

}  // namespace

void gather_to_original(const Graph &g, const double *src_new, double *dst_orig,
                        cudaStream_t st) {
    if (!g.n) return;
    k_gather<<<(unsigned)((g.n + 255) / 256), 256, 0, st>>>(g.iperm.p, src_new,
                                                           dst_orig, g.n); note_launch();
    KB_CUDA(cudaGetLastError());
}

void collect_k1_times(State &s) {
    for (; s.k1_read + 2 <= s.k1_used; s.k1_read += 2) {
        float ms = 0;
        KB_CUDA(cudaEventSynchronize(s.k1_ev[s.k1_read + 1]));
        KB_CUDA(cudaEventElapsedTime(&ms, s.k1_ev[s.k1_read], s.k1_ev[s.k1_read + 1]));
        s.spmv_ms += ms;
        s.spmv_launches += 1;
    }
    if (s.k1_read == s.k1_used) s.k1_read = s.k1_used = 0;  // recycle the pool
}

// One SpMV step w = alpha * A x (+ the fused bound refresh unless
// level_only) over the current SELL layout.
void run_spmv(State &s, cudaStream_t st, const double *x, double *w, bool level_only) {
    Graph &g = *s.g;
    const int64_t n = g.n;
    if (g.sell_dirty) build_sell(g, false);
    IterArgs A;
    A.cols = g.sell.cols.p;
    A.slice_off = g.sell.slice_off.p;
    A.slice_w = g.sell.slice_w.p;
    A.vlen = g.sell.vlen.p;
    A.nslices = g.sell.nslices;
    A.nvr = g.sell.nvr;
    A.nseg = g.sell.nseg;
    A.nh = g.nh;
    A.ncols = n;
    A.nwide = tune_get("k1.narrow4", 1) ? g.sell.nwide : g.sell.nslices;
    A.x = x;
    A.w = w;
    A.katz = s.katz.p;
    A.lower = s.lower.p;
    A.upper = s.upper.p;
    A.seg_sum = s.seg_sum.p;
    A.alpha = s.alpha;
    A.gamma = s.gamma;
    A.undirected = s.undirected;
    A.level_only = level_only;
    A.seg_only = 0;
    A.hrow = g.implicit_rows ? nullptr : g.hrow.p;
    A.vrow = g.implicit_rows ? nullptr : g.vrow.p;
    A.hot = (int)std::min<int64_t>(tune_get("k1.hot", g.hot), n);
    A.warm = (int)std::min<int64_t>(tune_get("k1.warm", 0), n);
    A.hot_per = 0;
    A.hot_shift = 0;
    const bool strided = g.hot_per > 0 && tune_get("k1.shard_hot", 1);
    if (strided) {
        const int64_t P = n >> g.hot_shift;
        A.hot_per = (int)std::min<int64_t>(g.hot_per, (int64_t)1 << g.hot_shift);
        A.hot_shift = g.hot_shift;
        A.hot = (int)(A.hot_per * P);
    }
    A.counter = s.work_counter.p;
    A.abort = s.spec_abort ? s.abort_flag.p : nullptr;
    A.pair_done = nullptr;
    if (s.pair_fuse.want && !level_only) {
        if (!s.pair_done.p) {
            s.pair_done.alloc(1);
            KB_CUDA(cudaMemsetAsync(s.pair_done.p, 0, sizeof(unsigned long long), st));
        }
        const auto &f = s.pair_fuse;
        A.pair_done = s.pair_done.p;
        A.pair_q = f.q;
        A.pair_x = f.x;
        A.pair_eps = f.eps;
        A.pair_perm = f.perm;
        A.pair_out = f.out;
        A.pair_abort = f.abort;
        A.pair_pub = f.pub;
        A.pair_k1c = f.k1c;
        A.pair_level = s.r + 1;
    }
    A.lazy_bounds = (s.lazy_bounds && !level_only) ? 1 : 0;
    A.npeer = 0;
    if (s.exch_on && w == g.exch[s.exch_parity]) {
        const auto &pp = g.exch_peer[s.exch_parity];
        A.npeer = (int)std::min<size_t>(pp.size(), KB_MAX_PEERS);
        for (int q = 0; q < A.npeer; q++) A.peer[q] = pp[q];
    }
    if (A.lazy_bounds) s.bounds_stale = true;
    if (s.seg_sum.n < (size_t)std::max<int64_t>(1, g.sell.nseg)) {
        s.seg_sum.alloc(std::max<int64_t>(1, g.sell.nseg));
        A.seg_sum = s.seg_sum.p;
    }
    if (g.implicit_rows) {
        // rows without arcs: w = 0 (bounds collapse once, see k_empty_rows)
        KB_CUDA(cudaMemsetAsync(w + g.nv, 0, (n + 1 - g.nv) * sizeof(double), st));
    } else {
        KB_CUDA(cudaMemsetAsync(w + n, 0, sizeof(double), st));
    }
    if (s.k1_used + 2 > s.k1_ev.size()) {
        for (int q = 0; q < 2; q++) {
            cudaEvent_t e;
            KB_CUDA(cudaEventCreate(&e));
            s.k1_ev.push_back(e);
        }
    }
    const bool ones = !s.levels.empty() && s.level_base == 0 && x == s.levels[0].p &&
                      tune_get("k1.ones_shortcut", 1);
    // lazily initialised state: the ones step writes katz, lower and upper
    // itself (katz_0 = 0); any other first K1 needs the initial vectors
    const bool fresh = s.init_pending && ones && !level_only && g.implicit_rows && !s.exch_on;
    if (s.init_pending && !fresh) ensure_init(s);
    if (s.ones_pending && !ones && !s.levels.empty() && s.level_base == 0 &&
        x == s.levels[0].p)
        ensure_ones(s);
    A.fresh = fresh ? 1 : 0;
    if (fresh && g.nh)     // heavy rows fold in k_heavy_combine, which adds to katz
        KB_CUDA(cudaMemsetAsync(s.katz.p, 0, g.nh * sizeof(double), st));
    // host-side setup first, so the events bracket only device work
    const int depth = (int)tune_get("k1.depth", 1);
    const int xl = (int)tune_get("k1.xload", 0);
    const int threads = (int)tune_get("k1.threads", 1024);
    const int ctas = (int)tune_get("k1.ctas_per_sm", 1);
    auto kern = k_sell_iterate<2, 0>;
    if (depth == 1)
        kern = xl == 1 ? k_sell_iterate<1, 1> : xl == 2 ? k_sell_iterate<1, 2>
             : xl == 3 ? k_sell_iterate<1, 3> : xl == 4 ? k_sell_iterate<1, 4>
                       : k_sell_iterate<1, 0>;
    else if (depth == 3) kern = xl == 1 ? k_sell_iterate<3, 1> : xl == 2 ? k_sell_iterate<3, 2> : k_sell_iterate<3, 0>;
    else kern = xl == 1 ? k_sell_iterate<2, 1> : xl == 2 ? k_sell_iterate<2, 2> : k_sell_iterate<2, 0>;
    if (strided)
        kern = depth == 3 ? k_sell_iterate<3, 0, 1>
             : depth == 2 ? k_sell_iterate<2, 0, 1> : k_sell_iterate<1, 0, 1>;
    static bool attr_done[64][16] = {};
    const int kid = strided ? 9 + (depth - 1) : xl >= 3 ? 12 + (xl - 3) : (depth - 1) * 3 + xl;
    if (!attr_done[g.device][kid]) {
        KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     227 * 1024 - 64));
        attr_done[g.device][kid] = true;
    }
    const size_t smem = (size_t)A.hot * sizeof(double);
    // k1.cluster = 2/4/8: the hot set spans a thread-block cluster (DSMEM)
    const int cl = strided ? 0 : (int)tune_get("k1.cluster", 0);
    auto ckern = cl == 4 ? k_sell_iterate<1, 0, 4> : cl == 8 ? k_sell_iterate<1, 0, 8>
                                                   : k_sell_iterate<1, 0, 2>;
    size_t csmem = 0;
    if (cl >= 2 && !ones) {
        const int64_t per = std::min<int64_t>(tune_get("k1.hot", g.hot), n / cl);
        A.hot = (int)(per * cl);
        csmem = (size_t)per * sizeof(double);
    }
    if (A.nslices && !ones && !s.counter_zeroed)
        KB_CUDA(cudaMemsetAsync(s.work_counter.p, 0, sizeof(unsigned long long), st));
    s.counter_zeroed = false;
    KB_CUDA(cudaEventRecord(s.k1_ev[s.k1_used], st));
    // overflow rows (dynamic batches): their sums on a side stream while K1
    // runs, the epilogue applied after it (k_ovf_merge)
    const bool ovf_side = g.n_ovf > 0 && !ones && tune_get("k1.ovf_side", 1);
    if (ovf_side) {
        if (!g.side_stream) {
            KB_CUDA(cudaStreamCreateWithFlags(&g.side_stream, cudaStreamNonBlocking));
            KB_CUDA(cudaEventCreateWithFlags(&g.side_fork, cudaEventDisableTiming));
            KB_CUDA(cudaEventCreateWithFlags(&g.side_join, cudaEventDisableTiming));
        }
        if (g.ovf_sum.n < (size_t)(g.n_ovf + g.n_ovf_long))
            g.ovf_sum.alloc(g.n_ovf + g.n_ovf_long);
        KB_CUDA(cudaEventRecord(g.side_fork, st));
        KB_CUDA(cudaStreamWaitEvent(g.side_stream, g.side_fork, 0));
        k_ovf_rows<<<(unsigned)((g.n_ovf * 32 + 255) / 256), 256, 0, g.side_stream>>>(
            A, g.ovf.p, g.n_ovf, g.perm.p, g.iperm.p, g.indptr.p, g.rlen.p, g.indices.p,
            g.split, g.ovf_sum.p);
        note_launch();
        if (g.n_ovf_long) {
            k_ovf_long<<<(unsigned)g.n_ovf_long, 256, 0, g.side_stream>>>(
                A, g.ovf_long.p, g.perm.p, g.iperm.p, g.indptr.p, g.rlen.p, g.indices.p, g.split,
                g.ovf_sum.p + g.n_ovf);
            note_launch();
        }
        KB_CUDA(cudaGetLastError());
        KB_CUDA(cudaEventRecord(g.side_join, g.side_stream));
    }
    if (A.nslices && ones) {
        k_ones_step<<<(unsigned)((A.nvr + 255) / 256), 256, 0, st>>>(A);
        note_launch();
        KB_CUDA(cudaGetLastError());
    } else if (A.nslices && g.sell.nwide == 0 && A.nseg == 0 &&
               (!A.lazy_bounds || tune_get("k1.narrow_lazy", 0) || tune_get("k1.narrow_pf", 9)) &&
               tune_get("k1.narrow_kernel", 1)) {
        // C4 (4096^2 grid) per launch with lazy bounds: TMA-staged narrow
        // kernel 0.149 ms; register-pipelined 0.1825 (0.223 with the bound
        // stores); unpipelined 0.1954 (0.250); the persistent kernel 0.1929
        const int pf = (int)tune_get("k1.narrow_pf", 9);
        if (pf == 9 && A.nh == 0 && !A.vrow && A.nseg == 0) {
            static bool attr[64] = {};
            if (!attr[g.device]) {
                KB_CUDA(cudaFuncSetAttribute(k_sell_narrow_tma,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)NB_SMEM));
                attr[g.device] = true;
            }
            const int64_t nfull = A.nvr / (32 * NB_CH);
            k_sell_narrow_tma<<<g.sm_count, 1024, NB_SMEM, st>>>(A, nfull);
            if (A.pair_done) s.pair_fuse.done = true;
        } else if (pf == 1) k_sell_narrow_pf<1><<<g.sm_count, 1024, 0, st>>>(A);
        else if (pf == 2 || pf == 9) k_sell_narrow_pf<2><<<g.sm_count, 1024, 0, st>>>(A);
        else if (pf == 4) k_sell_narrow_pf<4><<<g.sm_count, 1024, 0, st>>>(A);
        else if (tune_get("k1.narrow_q", 2) == 4) k_sell_narrow<4><<<g.sm_count * 2, 1024, 0, st>>>(A);
        else k_sell_narrow<2><<<g.sm_count * 2, 1024, 0, st>>>(A);
        note_launch();
        KB_CUDA(cudaGetLastError());
    } else if (A.nslices && cl >= 2) {
        // cluster hot set: cl CTAs share cl x hot ids over DSMEM
        static int max_clusters[64][4] = {};
        const int ci = cl == 2 ? 0 : cl == 4 ? 1 : 2;
        if (!max_clusters[g.device][ci]) {
            KB_CUDA(cudaFuncSetAttribute(ckern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024 - 64));
            cudaLaunchConfig_t q = {};
            q.gridDim = dim3((unsigned)(g.sm_count / cl * cl));
            q.blockDim = dim3(1024);
            q.dynamicSmemBytes = csmem;
            cudaLaunchAttribute qa[1];
            qa[0].id = cudaLaunchAttributeClusterDimension;
            qa[0].val.clusterDim.x = (unsigned)cl;
            qa[0].val.clusterDim.y = 1;
            qa[0].val.clusterDim.z = 1;
            q.attrs = qa;
            q.numAttrs = 1;
            int mc = 0;
            KB_CUDA(cudaOccupancyMaxActiveClusters(&mc, ckern, &q));
            max_clusters[g.device][ci] = std::max(1, mc);
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(max_clusters[g.device][ci] * cl));
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = csmem;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        KB_CUDA(cudaLaunchKernelEx(&cfg, ckern, A));
        note_launch();
    } else if (A.nslices) {
        kern<<<g.sm_count * ctas, threads, smem, st>>>(A); note_launch();
        KB_CUDA(cudaGetLastError());
    }
    if (A.nslices && g.nh) {
        if (tune_get("k1.combine_warp", 1)) {
            const int64_t nwarp = g.nh_long >= 0 && !A.hrow ? g.nh_long : g.nh;
            const int64_t threads = nwarp * 32 + (g.nh - nwarp);
            k_heavy_combine_w<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
                A, g.seg_ptr.p, g.seg_list.p, nwarp);
        }
        else
            k_heavy_combine<<<(unsigned)((g.nh + 127) / 128), 128, 0, st>>>(
                A, g.seg_ptr.p, g.seg_list.p);
        note_launch();
        KB_CUDA(cudaGetLastError());
    }
    if (!g.implicit_rows && g.nzero) {
        k_zero_rows<<<(unsigned)((g.nzero + 255) / 256), 256, 0, st>>>(
            g.zrows.p, g.nzero, w, s.lower.p, s.upper.p, s.katz.p, level_only);
        note_launch();
        KB_CUDA(cudaGetLastError());
    }
    if (fresh) {
        k_fresh_tail<<<(unsigned)((n + 1 - g.nv + 255) / 256), 256, 0, st>>>(
            s.katz.p, s.lower.p, s.upper.p, g.nv, n); note_launch();
        KB_CUDA(cudaGetLastError());
        s.init_pending = false;           // levels[0] stays pending (ones_pending)
    } else if (g.implicit_rows && s.r == 0 && !level_only && n > g.nv) {
        // rows without arcs: bounds collapse to katz (= 0) after the first step
        k_empty_rows<<<(unsigned)((n - g.nv + 255) / 256), 256, 0, st>>>(
            s.upper.p, s.lower.p, s.katz.p, g.nv, n); note_launch();
        KB_CUDA(cudaGetLastError());
    }
    if (ovf_side) {
        KB_CUDA(cudaStreamWaitEvent(st, g.side_join, 0));
        k_ovf_merge<<<(unsigned)((g.n_ovf + g.n_ovf_long + 255) / 256), 256, 0, st>>>(
            A, g.ovf.p, g.n_ovf, g.perm.p, g.rlen.p, g.ovf_sum.p, g.ovf_long.p, g.n_ovf_long,
            g.ovf_sum.p + g.n_ovf);
        note_launch();
        KB_CUDA(cudaGetLastError());
    } else if (g.n_ovf) {
        k_ovf_rows<<<(unsigned)((g.n_ovf * 32 + 255) / 256), 256, 0, st>>>(
            A, g.ovf.p, g.n_ovf, g.perm.p, g.iperm.p, g.indptr.p, g.rlen.p, g.indices.p,
            g.split);
        note_launch();
        KB_CUDA(cudaGetLastError());
    }
    if (g.n_ovf_long && !ovf_side) {
        k_ovf_long<<<(unsigned)g.n_ovf_long, 256, 0, st>>>(A, g.ovf_long.p, g.perm.p, g.iperm.p,
                                                          g.indptr.p, g.rlen.p, g.indices.p,
                                                          g.split);
        note_launch();
        KB_CUDA(cudaGetLastError());
    }
    KB_CUDA(cudaEventRecord(s.k1_ev[s.k1_used + 1], st));
    // the gather-free first step is not a K1 launch: keep it out of the
    // K1 timing (bench roofline) but count it in the run
    if (!level_only && !ones) s.k1_used += 2;
}

// The heavy-row segment sums alone (seg_sum, K1's folds) over the slices
// that hold segments -- the dynamic path's dense recompute of heavy rows.
void run_segments(State &s, cudaStream_t st, const double *x) {
    Graph &g = *s.g;
    if (g.sell_dirty || g.sell.nseg == 0) return;
    IterArgs A{};
    A.cols = g.sell.cols.p;
    A.slice_off = g.sell.slice_off.p;
    A.slice_w = g.sell.slice_w.p;
    A.vlen = g.sell.vlen.p;
    A.nslices = (g.sell.nseg + 31) / 32;
    A.nvr = g.sell.nvr;
    A.nseg = g.sell.nseg;
    A.nh = g.nh;
    A.ncols = g.n;
    A.nwide = std::min<int64_t>(g.sell.nwide, A.nslices);
    A.x = x;
    A.seg_sum = s.seg_sum.p;
    A.level_only = 1;
    A.seg_only = 1;
    A.lazy_bounds = 0;
    A.npeer = 0;
    A.hrow = g.implicit_rows ? nullptr : g.hrow.p;
    A.vrow = g.implicit_rows ? nullptr : g.vrow.p;
    A.hot = (int)std::min<int64_t>(tune_get("k1.hot", g.hot), g.n);
    A.counter = s.work_counter.p;
    if (s.seg_sum.n < (size_t)std::max<int64_t>(1, g.sell.nseg)) {
        s.seg_sum.alloc(std::max<int64_t>(1, g.sell.nseg));
        A.seg_sum = s.seg_sum.p;
    }
    auto kern = k_sell_iterate<1, 0>;
    static bool attr_done[64] = {};
    if (!attr_done[g.device]) {
        KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     227 * 1024 - 64));
        attr_done[g.device] = true;
    }
    KB_CUDA(cudaMemsetAsync(s.work_counter.p, 0, sizeof(unsigned long long), st));
    s.counter_zeroed = false;   // this launch leaves the counter non-zero
    kern<<<g.sm_count, 1024, (size_t)A.hot * sizeof(double), st>>>(A);
    note_launch();
    KB_CUDA(cudaGetLastError());
}

// lower/upper of every row from katz and the last level, with the epilogue's
// exact operations (engine.py:309-316): the bits K1 would have stored
__global__ void k_bounds_from(const double *katz, const double *w, int64_t n, double alpha,
                              double gamma, int undirected, double *lower, double *upper) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    const double k = katz[v];
    const double t = __dmul_rn(alpha, w[v]);
    lower[v] = undirected ? __dadd_rn(k, t) : k;
    upper[v] = __dadd_rn(k, __dmul_rn(t, gamma));
}

void materialize_bounds(State &s, cudaStream_t st) {
    if (!s.bounds_stale) return;
    const int64_t n = s.g->n;
    if (n) {
        k_bounds_from<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
            s.katz.p, s.x_level(), n, s.alpha, s.gamma, s.undirected, s.lower.p, s.upper.p);
        note_launch();
        KB_CUDA(cudaGetLastError());
    }
    s.bounds_stale = false;
}

void launch_iterate(State &s, cudaStream_t st) {
    NvtxRange nv("K1 level", (long long)s.r + 1);
    Graph &g = *s.g;
    const int64_t n = g.n;
    DBuf<double> wnew;
    if (s.exch_on) {           // the level goes to the exchange buffer of its parity
        s.exch_parity = (int)((s.r + 1) & 1);
        wnew.borrow(g.exch[s.exch_parity], g.exch_n);
    } else {
        wnew.alloc(n + 1);
    }
    run_spmv(s, st, s.x_level(), wnew.p, false);
    s.levels.push_back(std::move(wnew));
    s.r += 1;
    if (!s.keep_all && s.levels.size() > 2) {
        s.levels.erase(s.levels.begin());
        s.level_base += 1;
    }
}

}  // namespace kb
