// K2: the stopping rule (check_converged, engine.py:333-379) on the device.
//
// TOPK (k <= KMAX): one cooperative kernel over the active set
//   1. radix-select the k-th largest lower bound: 8 passes of 8-bit digits
//      over the IEEE bits of lower (lower >= +0, so the bit pattern orders
//      like the value); histograms are block-privatised in shared memory;
//   2. ties at the cut are broken by the smallest original id (a 4-pass
//      radix select on the id among the keys equal to the threshold) --
//      numpy's argpartition (engine.py:359) breaks them arbitrarily;
//   3. order-preserving compaction: the k winners go to a prefix buffer, the
//      losers with fl(upper - eps) >= threshold survive (engine.py:368-373);
// then a one-block kernel sorts the prefix by (-lower, id) in shared memory
// (engine.py:365) and evaluates |active| > k and the adjacent separations
// fl(upper[p_i] - eps) < lower[p_{i-1}] (engine.py:374-378).
//
// RANKING, or TOPK with k > KMAX: O(n) certificates first (SURVEY.md 7
// "exact O(n) fast paths"), and a full stable radix sort by (-lower, id)
// only when they cannot decide.
// SCORE: max(upper-lower) < eps (:344-345).  PAIR: scalar test (:346-353).
#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_partition.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <cub/block/block_reduce.cuh>

#include <algorithm>

#include "kb_internal.cuh"

namespace cg = cooperative_groups;

namespace kb {

namespace {

constexpr int KMAX = 4096;
constexpr int CHK_THREADS = 512;
constexpr int NCAND = 8;

__device__ __forceinline__ uint64_t key_of(const double *lower, int32_t id) {
    return (uint64_t)__double_as_longlong(lower[id]);
}

struct TopkArgs {
    const double *lower, *upper;
    const int32_t *perm;
    const int32_t *act_in;
    int64_t m;
    int dense;
    int32_t *act_out;
    int64_t k;
    double eps;
    unsigned int *hist;             // HIST_WORDS
    unsigned long long *blk;        // 2 * gridDim + 2
    int32_t *prefix_buf;            // k
    int32_t *cand;                  // capacity m: positions matching the 24-bit prefix
    uint64_t *stK;                  // staged keys / uppers / ids (non-dense sets)
    double *stU;
    int32_t *stI;
    unsigned long long *out;        // [0]=new m, [1]=converged, [2]=#prefix, [3]=kstar,
                                    // [4]=istar, [5]=winners, [6]=survivors, [7]=m in
    // device-driven runs: m is read from *m_dev (the previous check's count)
    // and this launch only acts when m_lo < m <= m_hi (one launch per grid
    // size; the others exit), and not at all once *abort (converged) is set
    const unsigned long long *m_dev = nullptr;
    int64_t m_lo = -1, m_hi = INT64_MAX;
    const unsigned long long *abort = nullptr;
    // fused split: winners -> prefix_buf, survivors -> act_out + k, in
    // active-set order, counts into out[0], out[2], out[5], out[6]
    int split = 0;
    // SURVEY.md 8(c) rule 4: losers that tie the k-th lower bound exactly and
    // are dropped (gap < eps) -- where numpy's arbitrary argpartition choice
    // (engine.py:359) could have kept them -- are counted here
    unsigned long long *ties = nullptr;
    int64_t act_cap = INT64_MAX;    // capacity of act_out (checked build)
    // sharded cut: the (global) cut is given in out[3], out[4] -- no
    // selection, only the split; winners to win_out and survivors to
    // surv_out when set (else prefix_buf and act_out + k)
    int cut_given = 0;
    int early_cut = (int)tune_get("k2.early_cut", 1);  // compact after one digit when small
    int32_t *win_out = nullptr, *surv_out = nullptr;
};

__device__ __forceinline__ bool flag_set(const unsigned long long *f) {
    return f && *(const volatile unsigned long long *)f != 0;
}

// The check's verdict, published by the kernel that finishes the check (one
// thread, after the result words are final): the abort flag for the K1s
// queued behind (they exit when it is set), that K1's work counter reset,
// the new |active| as the next check's input, and the result words written
// straight into page-locked host memory (no separate copy).
// (The host reads the published words only after an event synchronisation
// on the stream: no system-scope fence is needed.)
struct Publish {
    unsigned long long *abort, *k1_counter;
    volatile unsigned long long *host;
    int64_t level;
    int fence = 0;   // kb_tune chk.sys_fence: the old fenced publish
};

__device__ __forceinline__ void publish(const Publish &p, unsigned long long *out) {
    if (!p.abort) return;
    *p.abort = out[1];
    if (p.k1_counter) *p.k1_counter = 0ull;
    out[7] = out[0];
    p.host[0] = out[0];   // pub_words(): the device mirror or h_flags
    p.host[1] = out[1];
    p.host[2] = out[2];
    p.host[3] = (unsigned long long)p.level;
    if (p.fence) __threadfence_system();
}

// digit plan: two 12-bit digits over all elements, then the survivors of the
// 24-bit prefix are compacted and five 8-bit digits finish on them; ties at
// the cut take four 8-bit digits of the original id
constexpr int HIST_WORDS = 2 * 4096 + 5 * 256 + 4 * 256;

// Shared-memory histogram increment with warp aggregation: lanes hitting the
// same bin (common for the exponent digit) elect one leader that adds the
// group's count, so a warp costs at most one atomic per distinct bin.
__device__ __forceinline__ void hist_add(unsigned int *sh, unsigned bin, bool active) {
    const unsigned mask = __ballot_sync(0xffffffffu, active);
    if (!active) return;
    const unsigned peers = __match_any_sync(mask, bin);
    if ((threadIdx.x & 31) == (__ffs(peers) - 1)) atomicAdd(&sh[bin], __popc(peers));
}

// Find the bin where the running count (from the top, or from the bottom)
// first reaches `need`; every block computes it identically from the global
// histogram.  Block-parallel: bins are staged in shared memory and scanned
// with cub::BlockScan over per-thread runs.
__device__ __forceinline__ void select_digit(unsigned int *sh, const unsigned int *gh, int nbins,
                                             int64_t &need, int &sel, bool from_top) {
    typedef cub::BlockScan<unsigned long long, CHK_THREADS> BS;
    __shared__ typename BS::TempStorage bs_tmp;
    __shared__ unsigned long long s_res[2];
    for (int b = threadIdx.x; b < nbins; b += blockDim.x) sh[b] = gh[b];
    __syncthreads();
    const int per = (nbins + CHK_THREADS - 1) / CHK_THREADS;
    unsigned long long mine = 0;
    for (int q = 0; q < per; q++) {
        const int bp = threadIdx.x * per + q;  // position in scan order
        if (bp < nbins) mine += sh[from_top ? nbins - 1 - bp : bp];
    }
    unsigned long long before;
    BS(bs_tmp).ExclusiveSum(mine, before);
    unsigned long long cum = before;
    for (int q = 0; q < per; q++) {
        const int bp = threadIdx.x * per + q;
        if (bp >= nbins) break;
        const int bin = from_top ? nbins - 1 - bp : bp;
        const unsigned long long c = sh[bin];
        if (cum < (unsigned long long)need && cum + c >= (unsigned long long)need) {
            s_res[0] = (unsigned long long)bin;
            s_res[1] = cum;
        }
        cum += c;
    }
    __syncthreads();
    sel = (int)s_res[0];
    need -= (int64_t)s_res[1];
    __syncthreads();
}

constexpr int UNR = 4;  // elements per thread per tile (memory-level parallelism)
constexpr int CSORT = 2048;  // candidate sets up to this size are sorted in shared memory

// Block-wide bitonic sort of P (a power of two) (key, label) pairs ascending,
// carrying x when given.  Callers pad with (~0, ~0).
__device__ __forceinline__ void bitonic_kl(uint64_t *key, uint32_t *lab, int32_t *x, int P) {
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const bool gt = key[i] > key[j] || (key[i] == key[j] && lab[i] > lab[j]);
                    if (gt == up) {
                        const uint64_t tk = key[i]; key[i] = key[j]; key[j] = tk;
                        const uint32_t tl = lab[i]; lab[i] = lab[j]; lab[j] = tl;
                        if (x) { const int32_t tx = x[i]; x[i] = x[j]; x[j] = tx; }
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(CHK_THREADS, 2) k_topk_select(TopkArgs A) {
    if (flag_set(A.abort)) return;
    const int64_t m = A.m_dev ? (int64_t)*(const volatile unsigned long long *)A.m_dev : A.m;
    if (m <= A.m_lo || m > A.m_hi) return;     // another launch's size class
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned int sh[4096];
    const int64_t G = gridDim.x;
    const int64_t TILE = (int64_t)CHK_THREADS * UNR;
    const int64_t chunk = ((m + G - 1) / G + TILE - 1) / TILE * TILE;
    const int64_t i0 = min(m, blockIdx.x * chunk), i1 = min(m, i0 + chunk);
    unsigned long long *ncand = A.blk + 2 * G;
    // Element views: dense -> lower/upper by position; otherwise the active
    // ids are first staged into contiguous key/upper/id arrays so that every
    // later pass streams instead of gathering.
    const bool dense = A.dense;
    auto id_at = [&](int64_t i) -> int32_t { return dense ? (int32_t)i : A.act_in[i]; };

    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < HIST_WORDS; i += blockDim.x) A.hist[i] = 0;
        if (threadIdx.x == 0) *ncand = 0;
    }
    grid.sync();

    // with m <= k every element is a winner (engine.py:361-363): kstar = 0,
    // istar = max admits every key >= +0
    uint64_t kstar = 0;
    uint32_t istar = 0xFFFFFFFFu;
    if (A.cut_given) {
        kstar = A.out[3];
        istar = (uint32_t)A.out[4];
    } else if (m > A.k) {
    // ---- 1a. two 12-bit digits over the whole active set
    uint64_t prefix = 0, mask = 0;
    int64_t kk = A.k;
    for (int p = 0; p < 2; p++) {
        const int shift = 52 - 12 * p;
        unsigned int *gh = A.hist + p * 4096;
        for (int b = threadIdx.x; b < 4096; b += blockDim.x) sh[b] = 0;
        __syncthreads();
        for (int64_t t = i0; t < i1; t += TILE) {
            uint64_t key[UNR];
#pragma unroll
            for (int q = 0; q < UNR; q++) {
                const int64_t i = t + q * CHK_THREADS + threadIdx.x;
                key[q] = i < i1 ? key_of(A.lower, id_at(i)) : 0;
            }
#pragma unroll
            for (int q = 0; q < UNR; q++) {
                const int64_t i = t + q * CHK_THREADS + threadIdx.x;
                const bool on = i < i1 && (key[q] & mask) == prefix;
                hist_add(sh, (unsigned)((key[q] >> shift) & 4095), on);
            }
        }
        __syncthreads();
        for (int b = threadIdx.x; b < 4096; b += blockDim.x)
            if (sh[b]) atomicAdd(&gh[b], sh[b]);
        grid.sync();
        int sel;
        select_digit(sh, gh, 4096, kk, sel, true);
        prefix |= (uint64_t)sel << shift;
        mask |= (uint64_t)0xFFF << shift;
        // the cut's bin after the first digit is already small (the usual
        // case: it is the top exponent band): compact it now, skipping the
        // second pass over the whole set (same decision in every block)
        if (p == 0 && gh[sel] <= (unsigned)CSORT && A.early_cut) break;
    }
    // ---- 1b. compact the positions carrying the 12- or 24-bit prefix
    for (int64_t t = i0; t < i1; t += TILE) {
        uint64_t key[UNR];
#pragma unroll
        for (int q = 0; q < UNR; q++) {
            const int64_t i = t + q * CHK_THREADS + threadIdx.x;
            key[q] = i < i1 ? key_of(A.lower, id_at(i)) : 0;
        }
#pragma unroll
        for (int q = 0; q < UNR; q++) {
            const int64_t i = t + q * CHK_THREADS + threadIdx.x;
            const bool on = i < i1 && (key[q] & mask) == prefix;
            const unsigned bal = __ballot_sync(0xffffffffu, on);
            if (bal) {
                unsigned long long base = 0;
                const int lane = threadIdx.x & 31;
                if (lane == __ffs(bal) - 1) base = atomicAdd(ncand, (unsigned long long)__popc(bal));
                base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
                if (on) A.cand[base + __popc(bal & ((1u << lane) - 1))] = (int32_t)i;
            }
        }
    }
    grid.sync();
    const int64_t nc = (int64_t)*ncand;
    if (nc <= CSORT) {
        // few keys carry the 24-bit prefix (the usual case): every block
        // sorts them by (-key, label) in shared memory and reads the cut at
        // rank kk -- no further grid-wide digit passes
        __shared__ uint64_t ck[CSORT];
        __shared__ uint32_t cl[CSORT];
        int P = 1;
        while (P < nc) P <<= 1;
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
            if (i < nc) {
                const int32_t id = id_at(A.cand[i]);
                ck[i] = ~key_of(A.lower, id);
                cl[i] = (uint32_t)A.perm[id];
            } else {
                ck[i] = ~0ull;
                cl[i] = 0xFFFFFFFFu;
            }
        }
        __syncthreads();
        bitonic_kl(ck, cl, nullptr, P);
        kstar = ~ck[kk - 1];
        istar = cl[kk - 1];
        __syncthreads();
    } else {
    const int64_t cchunk = (nc + G - 1) / G;
    const int64_t c0 = min(nc, blockIdx.x * cchunk), c1 = min(nc, c0 + cchunk);
    // ---- 1c. five 8-bit digits over the candidates
    for (int p = 0; p < 5; p++) {
        const int shift = 32 - 8 * p;
        unsigned int *gh = A.hist + 2 * 4096 + p * 256;
        for (int b = threadIdx.x; b < 256; b += blockDim.x) sh[b] = 0;
        __syncthreads();
        for (int64_t i0w = c0; i0w < c1; i0w += blockDim.x) {
            const int64_t i = i0w + threadIdx.x;
            bool on = i < c1;
            uint64_t key = 0;
            if (on) key = key_of(A.lower, id_at(A.cand[i]));
            on = on && (key & mask) == prefix;
            hist_add(sh, (unsigned)((key >> shift) & 255), on);
        }
        __syncthreads();
        for (int b = threadIdx.x; b < 256; b += blockDim.x)
            if (sh[b]) atomicAdd(&gh[b], sh[b]);
        grid.sync();
        int sel;
        select_digit(sh, gh, 256, kk, sel, true);
        prefix |= (uint64_t)sel << shift;
        mask |= (uint64_t)0xFF << shift;
    }
    kstar = prefix;
    const int64_t count_eq = A.hist[2 * 4096 + 4 * 256 + (int)(kstar & 255)];

    // ---- 2. ties at the cut: the kk smallest original ids among key == kstar
    if (kk < count_eq) {
        uint32_t ipre = 0, imask = 0;
        int64_t need = kk;
        for (int p = 0; p < 4; p++) {
            const int shift = 24 - 8 * p;
            unsigned int *gh = A.hist + 2 * 4096 + 5 * 256 + p * 256;
            for (int b = threadIdx.x; b < 256; b += blockDim.x) sh[b] = 0;
            __syncthreads();
            for (int64_t i0w = c0; i0w < c1; i0w += blockDim.x) {
                const int64_t i = i0w + threadIdx.x;
                bool on = i < c1;
                uint32_t o = 0;
                if (on) {
                    const int32_t pos = A.cand[i];
                    on = key_of(A.lower, id_at(pos)) == kstar;
                    if (on) o = (uint32_t)A.perm[id_at(pos)];
                }
                on = on && (o & imask) == ipre;
                hist_add(sh, (o >> shift) & 255, on);
            }
            __syncthreads();
            for (int b = threadIdx.x; b < 256; b += blockDim.x)
                if (sh[b]) atomicAdd(&gh[b], sh[b]);
            grid.sync();
            int sel;
            select_digit(sh, gh, 256, need, sel, false);
            ipre |= (uint32_t)sel << shift;
            imask |= 0xFFu << shift;
        }
        istar = ipre;
    }
    }   // nc > CSORT
    }   // m > k
    if (blockIdx.x == 0 && threadIdx.x == 0 && !A.cut_given) {
        A.out[3] = kstar;
        A.out[4] = istar;
    }
    if (!A.split) return;

    // ---- 3. the split (engine.py:359-373), fused: winners (the k best by
    // (-lower, id)) to prefix_buf, survivors (the rest with fl(upper - eps) >=
    // threshold) to act_out + k, both in active-set order.  Each warp owns a
    // contiguous run of the block's chunk: pass A classifies its elements
    // (loads kept in flight, one class byte each in the staging buffer) and
    // counts them with ballots; one grid barrier publishes the block counts;
    // pass B streams the class bytes and ids and writes every kept id at its
    // rank (ballot + popc), so nothing is gathered twice.
    const double thr = __longlong_as_double((long long)kstar);
    // class bytes go to the staging buffer, not the candidate list: in the
    // shared-memory cut other blocks may still be reading the candidates
    // (no grid barrier separates that read from this pass)
    uint8_t *cls = (uint8_t *)A.stK;
    constexpr int NW = CHK_THREADS / 32;
    __shared__ unsigned long long s_wcnt[NW];
    __shared__ unsigned long long s_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t sub = ((i1 - i0 + NW - 1) / NW + 31) / 32 * 32;
    const int64_t a_w = min(i1, i0 + warp * sub), b_w = min(i1, a_w + sub);
    unsigned long long wc = 0;                 // (winners << 32) | survivors
    for (int64_t t = a_w; t < b_w; t += 4 * 32) {
        int32_t id[4];
        uint64_t key[4];
        double up[4];
        bool in[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int64_t i = t + q * 32 + lane;
            in[q] = i < b_w;
            id[q] = in[q] ? id_at(i) : 0;
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
            key[q] = in[q] ? key_of(A.lower, id[q]) : 0;
            up[q] = (in[q] && key[q] <= kstar) ? A.upper[id[q]] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
            uint8_t c = 0;
            if (in[q]) {
                if (key[q] > kstar || (key[q] == kstar && (uint32_t)A.perm[id[q]] <= istar))
                    c = 2;
                else if (__dsub_rn(up[q], A.eps) >= thr)
                    c = 1;
                else if (key[q] == kstar && A.ties)
                    atomicAdd(A.ties, 1ull);
                cls[t + q * 32 + lane] = c;
            }
            const unsigned bw = __ballot_sync(0xffffffffu, c == 2);
            const unsigned bs = __ballot_sync(0xffffffffu, c == 1);
            wc += ((unsigned long long)__popc(bw) << 32) + (unsigned long long)__popc(bs);
        }
    }
    if (lane == 0) s_wcnt[warp] = wc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long tot = 0;
        for (int w = 0; w < NW; w++) tot += s_wcnt[w];
        A.blk[blockIdx.x] = tot;
    }
    grid.sync();
    if (threadIdx.x < 32) {                    // this block's base and the grid total
        unsigned long long before = 0, total = 0;
        for (int64_t b = threadIdx.x; b < G; b += 32) {
            const unsigned long long c = A.blk[b];
            total += c;
            if (b < blockIdx.x) before += c;
        }
        for (int o = 16; o > 0; o >>= 1) {
            before += __shfl_down_sync(0xffffffffu, before, o);
            total += __shfl_down_sync(0xffffffffu, total, o);
        }
        if (threadIdx.x == 0) {
            s_base = before;
            if (blockIdx.x == 0) {
                const unsigned long long W = total >> 32, S = total & 0xFFFFFFFFull;
                A.out[0] = W + S;       // |active| after the cut
                A.out[2] = W;           // winners in the prefix buffer
                A.out[5] = W;
                A.out[6] = S;
            }
        }
    }
    __syncthreads();
    unsigned long long base = s_base;
    for (int w = 0; w < warp; w++) base += s_wcnt[w];
    unsigned long long ow = base >> 32, os = base & 0xFFFFFFFFull;
    for (int64_t t = a_w; t < b_w; t += 32) {
        const int64_t i = t + lane;
        const bool in = i < b_w;
        const uint8_t c = in ? cls[i] : 0;
        const unsigned bw = __ballot_sync(0xffffffffu, c == 2);
        const unsigned bs = __ballot_sync(0xffffffffu, c == 1);
        KB_DCHECK(c != 2 || ow + __popc(bw & lt) < (unsigned long long)A.k);
        KB_DCHECK(c != 1 || A.k + (int64_t)(os + __popc(bs & lt)) < A.act_cap);
        if (c == 2) (A.win_out ? A.win_out : A.prefix_buf)[ow + __popc(bw & lt)] = id_at(i);
        else if (c == 1) {
            const int64_t q = (int64_t)(os + __popc(bs & lt));
            if (A.surv_out) A.surv_out[q] = id_at(i);
            else A.act_out[A.k + q] = id_at(i);
        }
        ow += __popc(bw);
        os += __popc(bs);
    }
}

// Three-way split of the active set once the cut (kstar, istar) is known:
// winners (the k best by (-lower, id)) and survivors (the rest with
// fl(upper - eps) >= threshold, engine.py:368-373) in active-set order.
struct IsWinner {
    const double *lower;
    const int32_t *perm;
    const unsigned long long *cut;
    __device__ bool operator()(int32_t id) const {
        const uint64_t key = key_of(lower, id), kstar = cut[3];
        return key > kstar || (key == kstar && (uint32_t)perm[id] <= (uint32_t)cut[4]);
    }
};
struct IsSurvivor {
    const double *lower, *upper;
    const unsigned long long *cut;
    double eps;
    __device__ bool operator()(int32_t id) const {
        const double thr = __longlong_as_double((long long)cut[3]);
        return __dsub_rn(upper[id], eps) >= thr;
    }
};

// Sort the prefix by (-lower, original id), write it to act_out[0..cnt), and
// evaluate the stopping rule.  One block; cnt <= KMAX.
__global__ void __launch_bounds__(1024) k_topk_finish(const double *lower, const double *upper,
                                                      const int32_t *perm, const int32_t *src,
                                                      int dense_src, int32_t *act_out,
                                                      unsigned long long *out, double eps,
                                                      int64_t k,
                                                      const unsigned long long *abort = nullptr,
                                                      const unsigned long long *m_dev = nullptr,
                                                      int64_t m_min = -1, Publish pub = {}) {
    if (flag_set(abort)) return;
    if (m_dev && (int64_t)*(const volatile unsigned long long *)m_dev <= m_min) return;
    extern __shared__ unsigned char smem[];
    const int64_t cnt = (int64_t)out[2];
    const int64_t mnew = (int64_t)out[0];
    KB_DCHECK(cnt >= 0 && cnt <= k);
    int P = 1;
    while (P < cnt) P <<= 1;
    uint64_t *hi = (uint64_t *)smem;            // ~key  (ascending = lower desc)
    uint32_t *lo = (uint32_t *)(hi + P);        // original id
    int32_t *nid = (int32_t *)(lo + P);         // new id
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        if (i < cnt) {
            const int32_t id = dense_src ? i : src[i];
            hi[i] = ~key_of(lower, id);
            lo[i] = (uint32_t)perm[id];
            nid[i] = id;
        } else {
            hi[i] = ~0ull;
            lo[i] = 0xFFFFFFFFu;
            nid[i] = -1;
        }
    }
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const bool gt = hi[i] > hi[j] || (hi[i] == hi[j] && lo[i] > lo[j]);
                    if (gt == up) {
                        uint64_t th = hi[i]; hi[i] = hi[j]; hi[j] = th;
                        uint32_t tl = lo[i]; lo[i] = lo[j]; lo[j] = tl;
                        int32_t tn = nid[i]; nid[i] = nid[j]; nid[j] = tn;
                    }
                }
            }
            __syncthreads();
        }
    }
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        act_out[i] = nid[i];
        if (i >= 1 && !(__dsub_rn(upper[nid[i]], eps) < lower[nid[i - 1]])) bad = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out[1] = (mnew <= k) && !bad;
        publish(pub, out);
    }
}

// The TOPK check at level 1 of a fresh degree-relabelled layout, in one
// thread.  After the first iteration every bound is a function of the row
// length alone -- lower_1 = fl(a*d) + fl(a*fl(a*d)) (undirected; katz_1 for
// directed), upper_1 = fl(a*d) + fl(fl(a*fl(a*d))*gamma), both
// non-decreasing in d and strictly increasing for distinct integer d < 2^52
// -- and new ids order rows by (length desc, original id asc).  So the
// order by (-lower, id) is the new-id order: the winners are [0, k), the
// threshold is lower[k-1], and since upper is non-increasing in the new id
// the survivors fl(upper - eps) >= threshold are [k, S), found by bisection.
// The active set becomes exactly [0, S): the next check reads it densely.
// Boundary ties (lower == threshold, dropped) are [S, end of the equal run).
__global__ void k_topk_level1(const double *lower, const double *upper, int64_t nv, int64_t k,
                              double eps, const int32_t *perm, int32_t *act_out,
                              unsigned long long *out, unsigned long long *ties,
                              Publish pub) {
    if (flag_set(pub.abort)) return;
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const double T = lower[k - 1];
    // warp-wide 32-ary searches for the first v in [k, nv) failing a monotone
    // predicate (true on a prefix): five rounds at C2 instead of 24 probes
    auto first_fail = [&](auto pred) {
        int64_t lo = k, hi = nv;      // pred true on [k, lo), false on [hi, nv)
        while (hi - lo > 0) {
            const int64_t len = hi - lo;
            const int64_t step = (len + 31) / 32;
            const int64_t p = lo + (int64_t)lane * step;
            const bool ok = p < hi ? pred(p) : false;
            const unsigned bal = __ballot_sync(0xffffffffu, ok);
            const int c = __popc(bal);        // lanes [0, c) pass (prefix)
            const int64_t nlo = lo + (int64_t)c * step;
            if (c == 0) { hi = lo; break; }
            lo = c == 32 ? lo + 31 * step + 1 : lo + (int64_t)(c - 1) * step + 1;
            hi = min(hi, nlo);
            if (step == 1) { lo = hi = min(nlo, hi); break; }
        }
        return lo;
    };
    const int64_t S = first_fail([&](int64_t v) { return __dsub_rn(upper[v], eps) >= T; });
    const int64_t a = first_fail([&](int64_t v) { return lower[v] >= T; });
    if (lane != 0) return;
    if (ties && a > S) atomicAdd(ties, (unsigned long long)(a - S));
    bool conv = false;
    if (S <= k) {                     // |active| <= k: the adjacent separations
        bool bad = false;
        for (int64_t i = 1; i < S && !bad; i++) bad = !(__dsub_rn(upper[i], eps) < lower[i - 1]);
        conv = !bad;
        for (int64_t i = 0; i < S; i++) act_out[i] = (int32_t)i;   // also as a list
    }
    out[0] = (unsigned long long)S;
    out[1] = conv ? 1ull : 0ull;
    out[2] = (unsigned long long)k;
    out[3] = (unsigned long long)__double_as_longlong(T);
    out[4] = (unsigned long long)(uint32_t)perm[k - 1];
    out[5] = (unsigned long long)k;
    out[6] = (unsigned long long)(S - k);
    publish(pub, out);
}

// The whole TOPK check for a small active set (m <= SMALL_M, the last
// iterations of every R-MAT run: C2 ends at |active| 254 -> 100) in one
// block: the set is sorted by (-lower, label) in shared memory, the first
// min(m, k) are the sorted prefix (engine.py:359-366), the cut is read off,
// survivors are compacted in active-set order (engine.py:367-373) and the
// stopping rule is evaluated (engine.py:374-378).  Writes out[0..2] like
// k_topk_select + k_topk_finish.
__global__ void __launch_bounds__(1024) k_topk_small(const double *lower, const double *upper,
                                                     const int32_t *perm, const int32_t *act_in,
                                                     int dense, int64_t m_host,
                                                     const unsigned long long *m_dev, int64_t m_max,
                                                     int32_t *act_out, unsigned long long *out,
                                                     double eps, int64_t k,
                                                     const unsigned long long *abort,
                                                     unsigned long long *ties, Publish pub) {
    if (flag_set(abort)) return;
    const int64_t m = m_dev ? (int64_t)*(const volatile unsigned long long *)m_dev : m_host;
    if (m > m_max) return;
    if (m == 0) {
        if (threadIdx.x == 0) { out[0] = 0; out[1] = 1; out[2] = 0; publish(pub, out); }
        return;
    }
    extern __shared__ unsigned char smem[];
    int P = 1;
    while (P < m) P <<= 1;
    uint64_t *key = (uint64_t *)smem;
    uint32_t *lab = (uint32_t *)(key + P);
    int32_t *nid = (int32_t *)(lab + P);
    __shared__ unsigned int s_cnt[32];
    __shared__ int bad;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        if (i < m) {
            const int32_t id = dense ? i : act_in[i];
            key[i] = ~key_of(lower, id);
            lab[i] = (uint32_t)perm[id];
            nid[i] = id;
        } else {
            key[i] = ~0ull;
            lab[i] = 0xFFFFFFFFu;
            nid[i] = -1;
        }
    }
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    bitonic_kl(key, lab, nid, P);
    const int64_t W = m < k ? m : k;
    const uint64_t kstar = ~key[W - 1];
    const uint32_t istar = lab[W - 1];
    const double thr = __longlong_as_double((long long)kstar);
    for (int64_t i = threadIdx.x; i < W; i += blockDim.x) {
        act_out[i] = nid[i];
        if (i >= 1 && !(__dsub_rn(upper[nid[i]], eps) < lower[nid[i - 1]])) bad = 1;
    }
    // survivors, in active-set order
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int64_t base = W;
    for (int64_t t = 0; t < (m > k ? m : 0); t += blockDim.x) {
        const int64_t i = t + threadIdx.x;
        bool sv = false;
        int32_t id = 0;
        if (i < m) {
            id = dense ? (int32_t)i : act_in[i];
            const uint64_t kx = key_of(lower, id);
            const bool win = kx > kstar || (kx == kstar && (uint32_t)perm[id] <= istar);
            sv = !win && __dsub_rn(upper[id], eps) >= thr;
            if (!win && !sv && kx == kstar && ties) atomicAdd(ties, 1ull);
        }
        const unsigned b = __ballot_sync(0xffffffffu, sv);
        if (lane == 0) s_cnt[warp] = __popc(b);
        __syncthreads();
        int64_t off = base;
        for (int w = 0; w < warp; w++) off += s_cnt[w];
        KB_DCHECK(!sv || off + __popc(b & ((1u << lane) - 1u)) < m);
        if (sv) act_out[off + __popc(b & ((1u << lane) - 1u))] = id;
        int64_t tile = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) tile += s_cnt[w];
        base += tile;
        __syncthreads();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out[0] = (unsigned long long)base;          // |active| after the cut
        out[1] = (base <= k) && !bad;
        out[2] = (unsigned long long)W;
        publish(pub, out);
    }
}

// ---------------------------------------------------------------- reductions
__global__ void k_gap(const double *lower, const double *upper, int64_t n,
                      unsigned long long *out) {
    typedef cub::BlockReduce<unsigned long long, 256> Red;
    __shared__ typename Red::TempStorage tmp;
    unsigned long long best = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double d = __dsub_rn(upper[i], lower[i]);
        // map doubles to order-preserving unsigned keys (d may be -0/neg)
        const unsigned long long b = (unsigned long long)__double_as_longlong(d);
        const unsigned long long key = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
        best = max(best, key);
    }
    best = Red(tmp).Reduce(best, cub::Max());
    if (threadIdx.x == 0) atomicMax(out, best);
}

__global__ void k_pair(const double *lower, const double *upper, const int32_t *iperm,
                       int64_t u, int64_t v, double eps, unsigned long long *out) {
    const int32_t nu = iperm[u], nv = iperm[v];
    const double lu = lower[nu], lv = lower[nv];
    int64_t w, x;
    int32_t nw, nx;
    // (lu, -u) >= (lv, -v)  (engine.py:349)
    if (lu > lv || (lu == lv && -u >= -v)) { w = u; x = v; nw = nu; nx = nv; }
    else { w = v; x = u; nw = nv; nx = nu; }
    (void)w; (void)x;
    out[1] = lower[nw] > __dsub_rn(upper[nx], eps);
}

// ---------------------------------------------------------------- ranking
// violators of the self test fl(upper[q]-eps) < lower[q]; count them and keep,
// per block, the one with the widest excess (ties: smallest original id)
struct Cand {
    unsigned long long key;  // order-preserving bits of excess
    int32_t id;              // new id
};

__device__ __forceinline__ unsigned long long ord_bits(double d) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(d);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(256, 4) k_rank_violators(const double *lower, const double *upper, const int32_t *perm,
                                 const int32_t *act, int dense, int64_t m, double eps,
                                 unsigned long long *count, unsigned long long *blk_key,
                                 int32_t *blk_id) {
    __shared__ unsigned long long sk[256];
    __shared__ int32_t sid[256];
    unsigned long long bk = 0, c = 0;
    int32_t bid = -1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < m; i0 += 4 * stride) {
        int32_t q[4];
        double lo[4], up[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const int64_t i = i0 + t * stride;
            q[t] = i < m ? (dense ? (int32_t)i : act[i]) : -1;
        }
#pragma unroll
        for (int t = 0; t < 4; t++) {
            lo[t] = q[t] >= 0 ? lower[q[t]] : 0.0;
            up[t] = q[t] >= 0 ? upper[q[t]] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 4; t++) {
            if (q[t] < 0) continue;
            const double um = __dsub_rn(up[t], eps);
            if (!(um < lo[t])) {
                c++;
                const unsigned long long k = ord_bits(__dsub_rn(um, lo[t]));
                if (bid < 0 || k > bk || (k == bk && perm[q[t]] < perm[bid])) {
                    bk = k;
                    bid = q[t];
                }
            }
        }
    }
    sk[threadIdx.x] = bk;
    sid[threadIdx.x] = bid;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const unsigned long long k2 = sk[threadIdx.x + s];
            const int32_t i2 = sid[threadIdx.x + s];
            const int32_t i1 = sid[threadIdx.x];
            if (i2 >= 0 && (i1 < 0 || k2 > sk[threadIdx.x] ||
                            (k2 == sk[threadIdx.x] && perm[i2] < perm[i1]))) {
                sk[threadIdx.x] = k2;
                sid[threadIdx.x] = i2;
            }
        }
        __syncthreads();
    }
    typedef cub::BlockReduce<unsigned long long, 256> Red;
    __shared__ typename Red::TempStorage tmp;
    unsigned long long tot = Red(tmp).Sum(c);
    if (threadIdx.x == 0) {
        if (tot) atomicAdd(count, tot);
        blk_key[blockIdx.x] = sk[0];
        blk_id[blockIdx.x] = sid[0];
    }
}

// predecessor search for up to NCAND candidates: for each q the element x
// ranked immediately before it in (-lower, id) order, i.e. the minimum of
// (lower[x], -id[x]) over {x : (lower[x], -id[x]) > (lower[q], -id[q])}.
// Packed into one 64-bit key per block-candidate for a min reduction:
// we reduce on (lower bits, ~id) with atomicMin over two words via a
// 128-bit emulation -- done here as per-block arrays + host-free final pass.
__global__ void __launch_bounds__(256, 4) k_rank_pred(const double *lower, const int32_t *perm,
                                                     const int32_t *act, int dense, int64_t m,
                                                     const int32_t *cand, int ncand_max,
                                                     const unsigned long long *meta,
                                                     unsigned long long *pred_key,
                                                     unsigned int *pred_id) {
    const int ncand = meta ? (int)min((unsigned long long)ncand_max, *meta) : ncand_max;
    // candidates sorted by rank order R = (lower, -label) ascending; sidx maps
    // back to the caller's candidate slot
    __shared__ uint64_t ck[NCAND];
    __shared__ uint32_t co[NCAND];
    __shared__ int sidx[NCAND];
    if (threadIdx.x == 0) {
        for (int c = 0; c < ncand; c++) {
            const uint64_t k = key_of(lower, cand[c]);
            const uint32_t o = (uint32_t)perm[cand[c]];
            int p = c;
            while (p > 0 && (ck[p - 1] > k || (ck[p - 1] == k && co[p - 1] < o))) {
                ck[p] = ck[p - 1]; co[p] = co[p - 1]; sidx[p] = sidx[p - 1];
                p--;
            }
            ck[p] = k; co[p] = o; sidx[p] = c;
        }
    }
    __syncthreads();
    // x can only be the predecessor of the highest-ranked-below candidate:
    // every candidate is itself an element, so it pre-empts x for the rest
    uint64_t bk[NCAND];
    uint32_t bo[NCAND];
#pragma unroll
    for (int c = 0; c < NCAND; c++) { bk[c] = ~0ull; bo[c] = 0; }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < m; i0 += 4 * stride) {
        int32_t xs[4];
        uint64_t ks[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const int64_t i = i0 + t * stride;
            xs[t] = i < m ? (dense ? (int32_t)i : act[i]) : -1;
        }
#pragma unroll
        for (int t = 0; t < 4; t++) ks[t] = xs[t] >= 0 ? key_of(lower, xs[t]) : 0;
#pragma unroll
        for (int t = 0; t < 4; t++) {
            if (xs[t] < 0) continue;
            const uint64_t kx = ks[t];
            if (ncand == 0 || kx < ck[0]) continue;   // below every candidate
            uint32_t ox = 0;
            bool have = false;
            int js = -1;
            for (int j = ncand - 1; j >= 0; j--) {
                bool before = kx > ck[j];
                if (!before && kx == ck[j]) {
                    if (!have) { ox = (uint32_t)perm[xs[t]]; have = true; }
                    before = ox < co[j];
                }
                if (before) { js = j; break; }
            }
            if (js < 0) continue;
            if (!have) { ox = (uint32_t)perm[xs[t]]; have = true; }
#pragma unroll
            for (int c = 0; c < NCAND; c++)
                if (c == js && (kx < bk[c] || (kx == bk[c] && ox > bo[c]))) { bk[c] = kx; bo[c] = ox; }
        }
    }
    __shared__ uint64_t rk[256];
    __shared__ uint32_t ro[256];
#pragma unroll
    for (int c = 0; c < NCAND; c++) {
        if (c >= ncand) break;
        rk[threadIdx.x] = bk[c];
        ro[threadIdx.x] = bo[c];
        __syncthreads();
        for (int sft = 128; sft > 0; sft >>= 1) {
            if (threadIdx.x < sft) {
                const uint64_t k2 = rk[threadIdx.x + sft];
                const uint32_t o2 = ro[threadIdx.x + sft];
                if (k2 < rk[threadIdx.x] || (k2 == rk[threadIdx.x] && o2 > ro[threadIdx.x])) {
                    rk[threadIdx.x] = k2;
                    ro[threadIdx.x] = o2;
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            pred_key[blockIdx.x * NCAND + sidx[c]] = rk[0];
            pred_id[blockIdx.x * NCAND + sidx[c]] = ro[0];
        }
        __syncthreads();
    }
}

__global__ void k_orig_keys(const double *lower, const int32_t *iperm, const int32_t *act,
                            int dense, int64_t m, uint32_t *okey, int32_t *nid) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    // dense: walk original ids in order; else the active new ids
    if (dense) { okey[i] = (uint32_t)i; nid[i] = iperm[i]; }
    else { nid[i] = act[i]; }
}

__global__ void k_perm_keys(const int32_t *perm, const int32_t *nid, int64_t m, uint32_t *okey) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    okey[i] = (uint32_t)perm[nid[i]];
}

__global__ void k_lower_keys(const double *lower, const int32_t *nid, int64_t m, uint64_t *key) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    key[i] = ~key_of(lower, nid[i]);
}

// after the (-lower, id) sort: keep the first k, and the rest whose
// fl(upper - eps) >= lower of the k-th (engine.py:367-373); count adjacent
// separation failures inside the prefix (engine.py:376-378)
__global__ void k_cut_flags(const double *lower, const double *upper, const int32_t *order,
                            int64_t m, int64_t k, double eps, unsigned char *flag,
                            unsigned long long *bad) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t pk = (m < k ? m : k) - 1;
    const double thr = lower[order[pk]];
    if (i <= pk) {
        flag[i] = 1;
        if (i >= 1 && !(__dsub_rn(upper[order[i]], eps) < lower[order[i - 1]]))
            atomicAdd(bad, 1ull);
    } else {
        flag[i] = __dsub_rn(upper[order[i]], eps) >= thr;
    }
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

int coop_grid(int sm_count) {
    static int per_sm = 0;
    if (!per_sm) {
        KB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_topk_select,
                                                              CHK_THREADS, 0));
        per_sm = std::max(1, std::min(per_sm, 2));
    }
    return sm_count * per_sm;
}

// Where device-driven checks publish their verdict words: a device mirror
// copied to the page-locked h_flags once per batch (publish_copy) -- a
// kernel that writes page-locked memory itself ends only after those PCIe
// writes land (~3 us per check) -- or, with kb_tune chk.pub_host, h_flags
// directly.
unsigned long long *pub_words(State &s) {
    if (tune_get("chk.pub_host", 0)) return s.h_flags;
    if (!s.pub_dev.p) s.pub_dev.alloc(4);
    return s.pub_dev.p;
}

void publish_copy(State &s, cudaStream_t st) {
    if (tune_get("chk.pub_host", 0) || !s.pub_dev.p) return;
    KB_CUDA(cudaMemcpyAsync(s.h_flags, s.pub_dev.p, 4 * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, st));
}

void sync_read(State &s, cudaStream_t st, const unsigned long long *dev, int count) {
    KB_CUDA(cudaMemcpyAsync(s.h_flags, dev, count * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
}

// Generic rule by full sort: order the active set by (-lower, original id)
// with two stable radix sorts, cut at k, compact the survivors in sorted
// order.  Used for RANKING when the O(n) certificates cannot decide and for
// TOPK with k > KMAX.
bool sorted_check(State &s, cudaStream_t st, int64_t k) {
    Graph &g = *s.g;
    s.check_full_sorts++;
    const int64_t m = s.m_host;
    DBuf<uint32_t> ok_in, ok_out;
    DBuf<int32_t> id_in, id_out;
    DBuf<uint64_t> lk_in, lk_out;
    ok_in.alloc(m); ok_out.alloc(m); id_in.alloc(m); id_out.alloc(m);
    lk_in.alloc(m); lk_out.alloc(m);
    const int32_t *act = s.act[s.cur].p;
    k_orig_keys<<<nblk(m, 256), 256, 0, st>>>(s.lower.p, g.iperm.p, act, s.act_dense, m,
                                              ok_in.p, id_in.p); note_launch();
    const int32_t *by_orig = id_in.p;
    size_t tb = 0;
    if (!s.act_dense) {
        k_perm_keys<<<nblk(m, 256), 256, 0, st>>>(g.labels(), id_in.p, m, ok_in.p); note_launch();
        KB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, ok_in.p, ok_out.p, id_in.p,
                                                id_out.p, (int)m, 0, 32, st));
        ensure_cub_tmp(s, tb);
        KB_CUDA(cub::DeviceRadixSort::SortPairs(s.cub_tmp.p, tb, ok_in.p, ok_out.p, id_in.p,
                                                id_out.p, (int)m, 0, 32, st)); note_launch();
        by_orig = id_out.p;
    }
    k_lower_keys<<<nblk(m, 256), 256, 0, st>>>(s.lower.p, by_orig, m, lk_in.p); note_launch();
    int32_t *sorted = s.act_dense ? id_out.p : id_in.p;
    tb = 0;
    KB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, lk_in.p, lk_out.p, by_orig, sorted,
                                            (int)m, 0, 64, st));
    ensure_cub_tmp(s, tb);
    KB_CUDA(cub::DeviceRadixSort::SortPairs(s.cub_tmp.p, tb, lk_in.p, lk_out.p, by_orig, sorted,
                                            (int)m, 0, 64, st)); note_launch();
    unsigned char *flag = (unsigned char *)lk_in.p;  // reuse
    unsigned long long *u = s.scratch_u64.p;          // [0]=bad, [1]=selected count
    KB_CUDA(cudaMemsetAsync(u, 0, 2 * sizeof(unsigned long long), st));
    k_cut_flags<<<nblk(m, 256), 256, 0, st>>>(s.lower.p, s.upper.p, sorted, m, k, s.eps, flag, u); note_launch();
    const int nxt = s.cur ^ 1;
    tb = 0;
    KB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, sorted, flag, s.act[nxt].p, u + 1, (int)m,
                                       st));
    ensure_cub_tmp(s, tb);
    KB_CUDA(cub::DeviceSelect::Flagged(s.cub_tmp.p, tb, sorted, flag, s.act[nxt].p, u + 1,
                                       (int)m, st)); note_launch();
    sync_read(s, st, u, 2);
    s.cur = nxt;
    s.act_dense = false;
    s.m_host = (int64_t)s.h_flags[1];
    s.rank_order_pending = false;
    return s.m_host <= k && s.h_flags[0] == 0;
}

// the cached pair test for a speculative run: out[0] = refutes; the queued
// K1 of the next level runs only if it does (abort = !refutes)
__global__ void k_pair_refutes_pub(const double *katz, const double *w, double alpha, double gamma,
                                   int undirected, const int32_t *perm, int32_t q, int32_t x,
                                   double eps, unsigned long long *out,
                                   unsigned long long *abort, volatile unsigned long long *host,
                                   unsigned long long *k1_counter, int64_t level = -1,
                                   int fence = 0) {
    // in a device-driven chain, a test behind a failed one does nothing
    if (level >= 0 && *(volatile unsigned long long *)abort) return;
    // the two nodes' bounds from katz and the level, as the K1 epilogue forms them
    const double tq = __dmul_rn(alpha, w[q]), tx = __dmul_rn(alpha, w[x]);
    const double lq = undirected ? __dadd_rn(katz[q], tq) : katz[q];
    const double lx = undirected ? __dadd_rn(katz[x], tx) : katz[x];
    const double uq = __dadd_rn(katz[q], __dmul_rn(tq, gamma));
    const bool above = lx > lq || (lx == lq && perm[x] < perm[q]);
    const bool ref = above && lx <= __dsub_rn(uq, eps);
    out[0] = ref ? 1ull : 0ull;
    abort[0] = ref ? 0ull : 1ull;
    k1_counter[0] = 0ull;      // the queued K1's work counter (no separate memset)
    host[0] = ref ? 1ull : 0ull;  // pub_words(): the device mirror or h_flags
    if (level >= 0) host[3] = (unsigned long long)level;
    if (fence) __threadfence_system();   // see Publish
}

// candidates: the NCAND block winners with the widest excess (ties: the
// smaller label), chosen identically on the device by NCAND rounds of a
// block-wide arg-max
__global__ void __launch_bounds__(256) k_pick_cands(const unsigned long long *blk_key,
                                                    const int32_t *blk_id, int nb,
                                                    const int32_t *perm, int32_t *cand,
                                                    unsigned long long *meta) {
    __shared__ unsigned long long rk[256];
    __shared__ int32_t rb[256];
    __shared__ int32_t chosen[NCAND];
    int nc = 0;
    for (int round = 0; round < NCAND; round++) {
        unsigned long long bk = 0;
        int32_t bb = -1;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            const int32_t id = blk_id[b];
            if (id < 0) continue;
            bool taken = false;
            for (int t = 0; t < nc; t++) taken |= chosen[t] == b;
            if (taken) continue;
            const unsigned long long k = blk_key[b];
            if (bb < 0 || k > bk || (k == bk && perm[id] < perm[blk_id[bb]])) { bk = k; bb = b; }
        }
        rk[threadIdx.x] = bk;
        rb[threadIdx.x] = bb;
        __syncthreads();
        for (int sft = 128; sft > 0; sft >>= 1) {
            if (threadIdx.x < sft) {
                const int32_t b2 = rb[threadIdx.x + sft], b1 = rb[threadIdx.x];
                const unsigned long long k2 = rk[threadIdx.x + sft];
                if (b2 >= 0 && (b1 < 0 || k2 > rk[threadIdx.x] ||
                                (k2 == rk[threadIdx.x] && perm[blk_id[b2]] < perm[blk_id[b1]]))) {
                    rk[threadIdx.x] = k2;
                    rb[threadIdx.x] = b2;
                }
            }
            __syncthreads();
        }
        const int32_t win = rb[0];
        __syncthreads();
        if (win < 0) break;
        if (threadIdx.x == 0) {
            chosen[nc] = win;
            cand[nc] = blk_id[win];
        }
        nc++;
        __syncthreads();
    }
    if (threadIdx.x == 0) meta[0] = (unsigned long long)nc;
}

// per candidate: the exact predecessor over all blocks, then the verdict
// out[0]: 0 converged, 1 certified not converged, 2 undecided
__global__ void __launch_bounds__(256) k_rank_decide(
    const unsigned long long *count, const unsigned long long *meta, const int32_t *cand,
    const unsigned long long *pred_key, const unsigned int *pred_id, int nb,
    const double *upper, double eps, unsigned long long *out) {
    __shared__ uint64_t rk[256];
    __shared__ uint32_t ro[256];
    __shared__ int s_bad, s_ok;
    const unsigned long long nviol = *count;
    if (nviol == 0) {
        if (threadIdx.x == 0) out[0] = 0;
        return;
    }
    const int nc = (int)min((unsigned long long)NCAND, meta[0]);
    if (threadIdx.x == 0) { s_bad = 0; s_ok = 0; }
    __syncthreads();
    for (int c = 0; c < nc; c++) {
        uint64_t bestk = ~0ull;
        uint32_t besto = 0;
        for (int b = threadIdx.x; b < nb; b += blockDim.x) {
            const uint64_t k2 = pred_key[(size_t)b * NCAND + c];
            const uint32_t o2 = pred_id[(size_t)b * NCAND + c];
            if (k2 < bestk || (k2 == bestk && o2 > besto)) { bestk = k2; besto = o2; }
        }
        rk[threadIdx.x] = bestk;
        ro[threadIdx.x] = besto;
        __syncthreads();
        for (int sft = 128; sft > 0; sft >>= 1) {
            if (threadIdx.x < sft) {
                const uint64_t k2 = rk[threadIdx.x + sft];
                const uint32_t o2 = ro[threadIdx.x + sft];
                if (k2 < rk[threadIdx.x] || (k2 == rk[threadIdx.x] && o2 > ro[threadIdx.x])) {
                    rk[threadIdx.x] = k2;
                    ro[threadIdx.x] = o2;
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            if (rk[0] == ~0ull) s_ok++;  // q is ranked first
            else if (!(__dsub_rn(upper[cand[c]], eps) < __longlong_as_double((long long)rk[0])))
                s_bad = 1;
            else s_ok++;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        out[0] = s_bad ? 1 : ((unsigned long long)s_ok == nviol ? 0 : 2);
}

// Candidate q fails its adjacent-separation test iff some x ranked above q
// (lower[x] > lower[q], or equal with the smaller label) has
// lower[x] <= fl(upper[q] - eps): the predecessor has the smallest lower of
// all elements above q.  One pass tests that for every candidate at once
// and stops every block as soon as any candidate is refuted (the verdict is
// then "not converged"); only a converging check reads the whole set.
__global__ void __launch_bounds__(256, 4) k_rank_refute(const double *lower, const double *upper,
                                                       const int32_t *perm, const int32_t *act,
                                                       int dense, int64_t m,
                                                       const int32_t *cand,
                                                       const unsigned long long *meta,
                                                       double eps, unsigned long long *fail,
                                                       unsigned long long *pair) {
    __shared__ double cl[NCAND], ct[NCAND];
    __shared__ int32_t cq[NCAND], co[NCAND];
    const int nc = (int)min((unsigned long long)NCAND, *meta);
    if (threadIdx.x < nc) {
        const int32_t q = cand[threadIdx.x];
        cq[threadIdx.x] = q;
        cl[threadIdx.x] = lower[q];
        ct[threadIdx.x] = __dsub_rn(upper[q], eps);
        co[threadIdx.x] = perm[q];
    }
    __syncthreads();
    if (nc == 0) return;
    const volatile unsigned long long *vf = fail;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int it = 0;
    // block-uniform trip count (the early-exit vote is a block barrier)
    for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x; b0 < m; b0 += 4 * stride) {
        const int64_t i0 = b0 + threadIdx.x;
        if ((++it & 3) == 0 && __syncthreads_or(*vf != 0)) return;
        int32_t xs[4];
        double lx[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const int64_t i = i0 + t * stride;
            xs[t] = i < m ? (dense ? (int32_t)i : act[i]) : -1;
        }
#pragma unroll
        for (int t = 0; t < 4; t++) lx[t] = xs[t] >= 0 ? lower[xs[t]] : -1.0;
        bool hit = false;
        unsigned long long rec = 0;
#pragma unroll
        for (int t = 0; t < 4; t++) {
            if (xs[t] < 0) continue;
            for (int c = 0; c < nc; c++) {
                const double l = lx[t];
                if (l > ct[c] || l < cl[c]) continue;     // outside [lower_q, upper_q - eps]
                if (l > cl[c] || (xs[t] != cq[c] && perm[xs[t]] < co[c])) {
                    hit = true;
                    rec = ((unsigned long long)(uint32_t)cq[c] << 32) | (uint32_t)xs[t];
                }
            }
        }
        // one atomic pair per warp (a refuted check on a graph with many
        // exact ties, e.g. the grid, has a hit in almost every lane)
        const unsigned hm = __ballot_sync(0xffffffffu, hit);
        if (hm && (threadIdx.x & 31) == __ffs(hm) - 1) {
            atomicOr(fail, 1ull);
            if (*(volatile unsigned long long *)pair == ~0ull) atomicCAS(pair, ~0ull, rec);
        }
    }
}

// does the cached pair (q, x) still refute q's adjacent-separation test?
__global__ void k_pair_refutes(const double *lower, const double *upper, const int32_t *perm,
                               int32_t q, int32_t x, double eps, unsigned long long *out) {
    const double lq = lower[q], lx = lower[x];
    const bool above = lx > lq || (lx == lq && perm[x] < perm[q]);
    out[0] = (above && lx <= __dsub_rn(upper[q], eps)) ? 1ull : 0ull;
}

// candidates: the NCAND block winners with the widest excess (ties: the
// smaller label); one warp-synchronous arg-max per round, no block barriers
__global__ void __launch_bounds__(1024) k_pick_cands_fast(const unsigned long long *blk_key,
                                                         const int32_t *blk_id, int nb,
                                                         const int32_t *perm, int32_t *cand,
                                                         unsigned long long *meta) {
    __shared__ unsigned long long wk[32];
    __shared__ int32_t wb[32], wl[32];
    __shared__ int32_t win_b;
    extern __shared__ unsigned char taken[];
    for (int b = threadIdx.x; b < nb; b += blockDim.x) taken[b] = 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // every thread owns <= 2 block results (nb <= 2048)
    unsigned long long k0 = 0, k1 = 0;
    int32_t b0 = -1, b1 = -1, l0 = 0, l1 = 0;
    {
        const int a = threadIdx.x, c = threadIdx.x + blockDim.x;
        if (a < nb && blk_id[a] >= 0) { b0 = a; k0 = blk_key[a]; l0 = perm[blk_id[a]]; }
        if (c < nb && blk_id[c] >= 0) { b1 = c; k1 = blk_key[c]; l1 = perm[blk_id[c]]; }
    }
    __syncthreads();
    int nc = 0;
    for (int round = 0; round < NCAND; round++) {
        // local best among untaken
        unsigned long long bk = 0;
        int32_t bb = -1, bl = 0;
        if (b0 >= 0 && !taken[b0]) { bk = k0; bb = b0; bl = l0; }
        if (b1 >= 0 && !taken[b1] &&
            (bb < 0 || k1 > bk || (k1 == bk && l1 < bl))) { bk = k1; bb = b1; bl = l1; }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const unsigned long long ok = __shfl_down_sync(0xffffffffu, bk, o);
            const int32_t ob = __shfl_down_sync(0xffffffffu, bb, o);
            const int32_t ol = __shfl_down_sync(0xffffffffu, bl, o);
            if (ob >= 0 && (bb < 0 || ok > bk || (ok == bk && ol < bl))) { bk = ok; bb = ob; bl = ol; }
        }
        if (lane == 0) { wk[warp] = bk; wb[warp] = bb; wl[warp] = bl; }
        __syncthreads();
        if (warp == 0) {
            const int nw = blockDim.x >> 5;
            bk = lane < nw ? wk[lane] : 0;
            bb = lane < nw ? wb[lane] : -1;
            bl = lane < nw ? wl[lane] : 0;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const unsigned long long ok = __shfl_down_sync(0xffffffffu, bk, o);
                const int32_t ob = __shfl_down_sync(0xffffffffu, bb, o);
                const int32_t ol = __shfl_down_sync(0xffffffffu, bl, o);
                if (ob >= 0 && (bb < 0 || ok > bk || (ok == bk && ol < bl))) { bk = ok; bb = ob; bl = ol; }
            }
            if (lane == 0) {
                win_b = bb;
                if (bb >= 0) {
                    taken[bb] = 1;
                    cand[nc] = blk_id[bb];
                }
            }
        }
        __syncthreads();
        if (win_b < 0) break;
        nc++;
    }
    if (threadIdx.x == 0) meta[0] = (unsigned long long)nc;
}

bool check_ranking(State &s, cudaStream_t st) {
    NvtxRange nv("K2 ranking check", (long long)s.r);
    Graph &g = *s.g;
    // the reference leaves active sorted by (-lower, id) after every ranking
    // check (engine.py:362-372 with k = n); the certificates below decide
    // without sorting, so the order is produced on demand
    // (materialize_rank_order) unless the full sort runs anyway
    s.rank_order_pending = true;
    const int64_t n = s.m_host;
    const int32_t *act = s.act[s.cur].p;
    const int dense = s.act_dense;
    const int nb = 8 * g.sm_count;
    unsigned long long *u = s.scratch_u64.p;   // [0]=count [1]=ncand [2]=verdict [4..) blocks
    unsigned long long *bkey = u + 4;
    unsigned long long *pk = bkey + nb;
    int32_t *ids = s.scratch_i32.p;            // [0..nb) block ids, [nb..nb+8) candidates
    int32_t *cand = ids + nb;
    unsigned int *po = (unsigned int *)(cand + NCAND);
    if (s.rk_q >= 0 && tune_get("check.pair_cache", 1)) {
        k_pair_refutes<<<1, 1, 0, st>>>(s.lower.p, s.upper.p, g.labels(), s.rk_q, s.rk_x, s.eps, u);
        note_launch();
        sync_read(s, st, u, 1);
        if (s.h_flags[0]) return false;          // still refuted: not converged
        s.rk_q = s.rk_x = -1;
    }
    KB_CUDA(cudaMemsetAsync(u, 0, 4 * sizeof(unsigned long long), st));
    KB_CUDA(cudaMemsetAsync(u + 3, 0xff, sizeof(unsigned long long), st));   // refuting pair
    k_rank_violators<<<nb, 256, 0, st>>>(s.lower.p, s.upper.p, g.labels(), act, dense, n, s.eps,
                                         u, bkey, ids);
    if (tune_get("check.refute", 1) && nb <= 2048) {
        k_pick_cands_fast<<<1, 1024, nb, st>>>(bkey, ids, nb, g.labels(), cand, u + 1);
        k_rank_refute<<<nb, 256, 0, st>>>(s.lower.p, s.upper.p, g.labels(), act, dense, n, cand,
                                          u + 1, s.eps, u + 2, u + 3);
        note_launch(3);
        KB_CUDA(cudaGetLastError());
        sync_read(s, st, u, 4);
        const unsigned long long nviol = s.h_flags[0], ncand = s.h_flags[1],
                                 refuted = s.h_flags[2];
        if (nviol == 0) return true;            // every node passes its self test
        if (refuted) {                           // a candidate fails: not converged
            if (s.h_flags[3] != ~0ull) {
                s.rk_q = (int32_t)(s.h_flags[3] >> 32);
                s.rk_x = (int32_t)(uint32_t)s.h_flags[3];
            }
            return false;
        }
        if (nviol <= ncand) return true;         // every violator checked and passes
        return sorted_check(s, st, g.n);
    }
    k_pick_cands<<<1, 256, 0, st>>>(bkey, ids, nb, g.labels(), cand, u + 1);
    k_rank_pred<<<nb, 256, 0, st>>>(s.lower.p, g.labels(), act, dense, n, cand, NCAND, u + 1, pk,
                                    po);
    k_rank_decide<<<1, 256, 0, st>>>(u, u + 1, cand, pk, po, nb, s.upper.p, s.eps, u + 2);
    note_launch(4);
    KB_CUDA(cudaGetLastError());
    sync_read(s, st, u + 2, 1);
    const unsigned long long verdict = s.h_flags[0];
    if (verdict == 0) return true;
    if (verdict == 1) return false;
    return sorted_check(s, st, g.n);
}

}  // namespace

void materialize_rank_order(State &s, cudaStream_t st) {
    if (!s.rank_order_pending || s.kind != KB_RANKING) return;
    sorted_check(s, st, s.g->n);    // k = n: keeps every node, sorted
    s.check_full_sorts--;           // not a check the certificates missed
}

void ensure_cub_tmp(State &s, size_t bytes) {
    if (s.cub_tmp.n < bytes) s.cub_tmp.alloc(bytes);
}

double run_gap(State &s, cudaStream_t st) {
    Graph &g = *s.g;
    unsigned long long *u = s.scratch_u64.p;
    KB_CUDA(cudaMemsetAsync(u, 0, sizeof(unsigned long long), st));
    const int64_t lo = g.own_lo, hi = g.own_hi < 0 ? g.n : g.own_hi;
    if (hi > lo)
        k_gap<<<2 * g.sm_count, 256, 0, st>>>(s.lower.p + lo, s.upper.p + lo, hi - lo, u); note_launch();
    sync_read(s, st, u, 1);
    unsigned long long key = s.h_flags[0];
    unsigned long long b = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
    double d;
    memcpy(&d, &b, sizeof(double));
    return g.n ? d : 0.0;
}

// RANKING run with a cached refuting pair, the loop on the device: the test
// of the pair at the current level, then up to `batch` - 1 more levels, each
// a K1 (lazy bounds) followed by the pair's test, all queued with no host
// read; a test that no longer refutes sets the abort flag and every kernel
// behind it exits.  One host wait per chain; the levels queued past the
// last test that ran are dropped.  Returns true while the pair still
// refutes at s.r (not converged, caller iterates on), false when it stopped
// refuting at s.r (the full check decides).  C4: 95 of 99 checks.
bool ranking_pair_chain(State &s, cudaStream_t st) {
    NvtxRange nv("K2 ranking pair chain from level", (long long)s.r);
    Graph &g = *s.g;
    s.rank_order_pending = true;
    if (!s.abort_flag.p) s.abort_flag.alloc(1);
    if (!s.chk_ev) KB_CUDA(cudaEventCreateWithFlags(&s.chk_ev, cudaEventDisableTiming));
    if (!s.chk_ev2) KB_CUDA(cudaEventCreateWithFlags(&s.chk_ev2, cudaEventDisableTiming));
    KB_CUDA(cudaMemsetAsync(s.abort_flag.p, 0, sizeof(unsigned long long), st));
    const int64_t batch = std::max<int64_t>(1, tune_get("run.rank_batch", 8));
    const bool fuse = tune_get("chk.pair_fuse", 1) != 0;
    const bool pub_host = tune_get("chk.pub_host", 0) != 0;
    // two batches in flight: the next is queued before the host waits on the
    // current one, so the GPU never idles through a host read; a batch
    // queued behind a test that stopped refuting exits kernel by kernel on
    // the abort flag, and its levels are dropped here
    const bool pipe = tune_get("run.rank_pipe", 1) != 0 && !pub_host;
    struct Inflight {
        int64_t r_last;
        const unsigned long long *words;
        cudaEvent_t ev;
    };
    Inflight q[2];
    int nq = 0, slot = 0;
    cudaEvent_t evs[2] = {s.chk_ev, s.chk_ev2};
    unsigned long long *hb[2] = {s.h_flags + 16, s.h_flags + 24};
    bool first = true;
    s.pair_fuse = State::PairFuse{};
    auto enqueue = [&] {
        for (int64_t j = 0; j < batch; j++) {
            if (!(first && j == 0)) {
                if (s.r >= s.max_iter) break;
                if (fuse) {
                    s.pair_fuse.want = true;
                    s.pair_fuse.q = s.rk_q;
                    s.pair_fuse.x = s.rk_x;
                    s.pair_fuse.eps = s.eps;
                    s.pair_fuse.perm = g.labels();
                    s.pair_fuse.out = s.scratch_u64.p;
                    s.pair_fuse.abort = s.abort_flag.p;
                    s.pair_fuse.pub = pub_words(s);
                    s.pair_fuse.k1c = s.work_counter.p;
                }
                s.spec_abort = true;   // exits once a test before it stopped refuting
                launch_iterate(s, st);
                s.spec_abort = false;
                s.pair_fuse.want = false;
            }
            // the test of level s.r: already run by the tail of the K1 that
            // produced it (the TMA-staged narrow kernel), else a one-thread
            // launch
            if (!s.pair_fuse.done) {
                k_pair_refutes_pub<<<1, 1, 0, st>>>(s.katz.p, s.x_level(), s.alpha, s.gamma,
                                                    s.undirected, g.labels(), s.rk_q, s.rk_x,
                                                    s.eps, s.scratch_u64.p, s.abort_flag.p,
                                                    pub_words(s), s.work_counter.p, s.r,
                                                    (int)tune_get("chk.sys_fence", 0));
                note_launch();
            }
            s.pair_fuse = State::PairFuse{};
            s.counter_zeroed = true;
        }
        first = false;
        KB_CUDA(cudaGetLastError());
        const unsigned long long *words = s.h_flags;
        if (!pub_host) {      // this batch's closing words to its own host slot
            KB_CUDA(cudaMemcpyAsync(hb[slot], s.pub_dev.p, 4 * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, st));
            words = hb[slot];
        }
        KB_CUDA(cudaEventRecord(evs[slot], st));
        q[nq++] = Inflight{s.r, words, evs[slot]};
        slot ^= 1;
    };
    const int64_t r0 = s.r;
    enqueue();
    for (;;) {
        if (pipe && nq < 2 && s.r < s.max_iter) enqueue();
        const Inflight b = q[0];
        q[0] = q[1];
        nq -= 1;
        KB_CUDA(cudaEventSynchronize(b.ev));
        const bool refutes = b.words[0] != 0;
        const int64_t last = (int64_t)b.words[3];   // level of the last test that ran
        KB_REQUIRE(last >= r0 && last <= b.r_last, KB_ECUDA, "device loop lost its verdict");
        if (!refutes) {
            while (s.r > last) {      // levels queued behind the test that stopped refuting
                s.levels.pop_back();
                s.r -= 1;
                if (s.k1_used >= 2) s.k1_used -= 2;
            }
            return false;
        }
        KB_REQUIRE(last == b.r_last, KB_ECUDA, "device loop lost its verdict");
        if (nq == 0) {
            if (s.r >= s.max_iter) return true;
            enqueue();
        }
    }
}

bool run_check(State &s, cudaStream_t st) {
    Graph &g = *s.g;
    KB_REQUIRE(s.r >= 1, KB_ESTATE, "check_converged needs at least one iteration");
    if (s.kind == KB_SCORE) return run_gap(s, st) < s.eps;
    if (s.kind == KB_PAIR) {
        k_pair<<<1, 1, 0, st>>>(s.lower.p, s.upper.p, g.iperm.p, s.u, s.v, s.eps,
                                s.scratch_u64.p); note_launch();
        sync_read(s, st, s.scratch_u64.p, 2);
        return s.h_flags[1] != 0;
    }
    const int64_t k = (s.kind == KB_RANKING) ? g.n : s.k;
    if (s.kind == KB_RANKING) return check_ranking(s, st);
    if (k > KMAX) return sorted_check(s, st, k);
    const int nxt = topk_check_enqueue(s, st);
    KB_CUDA(cudaEventSynchronize(s.chk_ev));
    return topk_check_finish(s, nxt);
}

namespace {
// size classes of the device-driven select: one cooperative launch each,
// only the one whose class holds the runtime |active| does any work
constexpr int64_t SMALL_M = 4096, MID_M = 1 << 18, MID_G = 32;
}  // namespace

// Enqueue one TOPK check (engine.py:333-379) with no host read.  m_host >= 0:
// |active| is known on the host (grid sized for it); m_host < 0: it is the
// previous check's count, read on the device (device-driven run).  The
// active set moves from act[cur] to act[cur ^ 1]; the kernel that finishes the
// check publishes the verdict tagged with `level`.  Returns the new index.
int topk_check_enqueue_dev(State &s, cudaStream_t st, int64_t m_host, bool dense, int cur,
                           int64_t level, bool level1 = false) {
    NvtxRange nv("K2 topk check", (long long)level);
    Graph &g = *s.g;
    const int64_t k = s.k;
    unsigned long long *out = s.scratch_u64.p;  // [0..8)
    const int nxt = cur ^ 1;
    if (!s.abort_flag.p) {
        s.abort_flag.alloc(1);
        KB_CUDA(cudaMemsetAsync(s.abort_flag.p, 0, sizeof(unsigned long long), st));
    }
    TopkArgs A;
    A.lower = s.lower.p;
    A.upper = s.upper.p;
    A.perm = g.labels();
    A.act_in = s.act[cur].p;
    A.dense = dense ? 1 : 0;
    A.act_out = s.act[nxt].p;
    A.k = k;
    A.eps = s.eps;
    A.hist = (unsigned int *)(s.scratch_u64.p + 8);
    A.blk = s.scratch_u64.p + 8 + HIST_WORDS;
    A.prefix_buf = s.scratch_i32.p;
    A.cand = s.cand.p;
    A.stK = s.stK.p;
    A.stU = s.stU.p;
    A.stI = s.stI.p;
    A.out = out;
    A.abort = s.abort_flag.p;
    A.split = 1;
    A.ties = s.tie_count.p;
    A.act_cap = (int64_t)s.act[nxt].n;
    void *args[] = {&A};
    const int Gmax = coop_grid(g.sm_count);
    int P = 1;
    while (P < k) P <<= 1;
    const size_t smem = (size_t)P * 16;
    static bool attr_done[64] = {};
    static size_t attr_smem[64] = {};
    if (!attr_done[g.device] || attr_smem[g.device] < smem) {
        KB_CUDA(cudaFuncSetAttribute(k_topk_finish, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(smem, 1)));
        KB_CUDA(cudaFuncSetAttribute(k_topk_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(SMALL_M * 16)));
        attr_done[g.device] = true;
        attr_smem[g.device] = smem;
    }
    const Publish pub{s.abort_flag.p, s.work_counter.p, pub_words(s), level,
                      (int)tune_get("chk.sys_fence", 0)};
    auto small = [&](int64_t mh, const unsigned long long *md) {
        int Ps = 1;
        while (Ps < (mh >= 0 ? mh : SMALL_M)) Ps <<= 1;
        k_topk_small<<<1, 1024, (size_t)Ps * 16, st>>>(s.lower.p, s.upper.p, g.labels(),
                                                       s.act[cur].p, dense ? 1 : 0, mh, md,
                                                       SMALL_M, s.act[nxt].p, out, s.eps, k,
                                                       s.abort_flag.p, s.tie_count.p, pub);
        note_launch();
    };
    auto finish = [&](const unsigned long long *md) {
        k_topk_finish<<<1, 1024, smem, st>>>(s.lower.p, s.upper.p, g.labels(), A.prefix_buf, 0,
                                             s.act[nxt].p, out, s.eps, k, s.abort_flag.p, md,
                                             SMALL_M, pub);
        note_launch();
    };
    if (level1) {
        k_topk_level1<<<1, 32, 0, st>>>(s.lower.p, s.upper.p, s.g->nv, k, s.eps, g.labels(),
                                        s.act[nxt].p, out, s.tie_count.p, pub);
        note_launch();
    } else if (m_host >= 0) {
        // in the dense first check, rows without out-arcs (new ids >= nv) have
        // lower == upper == 0 < every other lower: when k <= nv they can be
        // neither winners nor survivors, so they are dropped unread
        A.m = (dense && k <= s.tail_zero_from) ? s.tail_zero_from : m_host;
        if (A.m <= SMALL_M) {
            small(A.m, nullptr);
        } else {
            const int G = (int)std::max<int64_t>(1, std::min<int64_t>(Gmax, (A.m + 8191) / 8192));
            KB_CUDA(cudaLaunchCooperativeKernel((void *)k_topk_select, G, CHK_THREADS, args, 0,
                                                st));
            note_launch();
            finish(nullptr);
        }
    } else {
        A.m_dev = out + 7;
        small(-1, out + 7);
        const int64_t lo[2] = {SMALL_M, MID_M}, hi[2] = {MID_M, INT64_MAX};
        const int G[2] = {(int)std::min<int64_t>(MID_G, Gmax), Gmax};
        for (int c = 0; c < 2; c++) {
            A.m_lo = lo[c];
            A.m_hi = hi[c];
            KB_CUDA(cudaLaunchCooperativeKernel((void *)k_topk_select, G[c], CHK_THREADS, args,
                                                0, st));
            note_launch();
        }
        finish(out + 7);
    }
    KB_CUDA(cudaGetLastError());
    s.counter_zeroed = true;
    return nxt;
}

// k_topk_level1 applies: the check right after the first iteration of a
// fresh single-GPU degree-relabelled layout, with the whole node set active
bool level1_shortcut_ok(const State &s) {
    const Graph &g = *s.g;
    return tune_get("chk.level1", 1) && s.kind == KB_TOPK && s.r == 1 && s.act_dense &&
           s.m_host == g.n && g.relabel && !g.mutated && g.implicit_rows && !s.exch_on &&
           g.own_lo == 0 && (g.own_hi < 0 || g.own_hi == g.n) && s.k >= 1 && s.k <= g.nv &&
           s.k <= KMAX && s.tail_zero_from == g.nv && s.level_base == 0;
}

int topk_check_enqueue(State &s, cudaStream_t st) {
    if (!s.abort_flag.p) s.abort_flag.alloc(1);
    // a stand-alone check acts whatever an earlier run left in the flag
    KB_CUDA(cudaMemsetAsync(s.abort_flag.p, 0, sizeof(unsigned long long), st));
    const int nxt = topk_check_enqueue_dev(s, st, s.m_host, s.act_dense, s.cur, s.r);
    publish_copy(s, st);
    if (!s.chk_ev) KB_CUDA(cudaEventCreateWithFlags(&s.chk_ev, cudaEventDisableTiming));
    KB_CUDA(cudaEventRecord(s.chk_ev, st));
    return nxt;
}

bool topk_check_finish(State &s, int nxt) {
    s.cur = nxt;
    s.act_dense = false;
    s.m_host = (int64_t)s.h_flags[0];
    return s.h_flags[1] != 0;
}

// engine.run (engine.py:382-396) for TOPK with the loop on the device: the
// host queues up to `batch` levels of K1 + check back to back with no host
// read in between -- each check's count feeds the next on the device, and a
// converged check's flag makes every kernel queued behind it exit -- then
// waits once.  C2 (r = 7) and C3 (r = 6) certify in one batch: one host
// synchronisation per run.  Returns converged (false: the cap was reached).
bool topk_run_device(State &s, cudaStream_t st) {
    if (!s.abort_flag.p) s.abort_flag.alloc(1);
    KB_CUDA(cudaMemsetAsync(s.abort_flag.p, 0, sizeof(unsigned long long), st));
    if (!s.chk_ev) KB_CUDA(cudaEventCreateWithFlags(&s.chk_ev, cudaEventDisableTiming));
    const int64_t batch = std::max<int64_t>(1, tune_get("run.batch", 8));
    for (;;) {
        const int64_t r0 = s.r, B = std::min<int64_t>(batch, s.max_iter - s.r);
        const int cur0 = s.cur;
        int cur = cur0;
        bool dense_next = false;
        for (int64_t j = 0; j < B; j++) {
            s.spec_abort = true;      // exits once a check before it has converged
            launch_iterate(s, st);
            s.spec_abort = false;
            const bool l1 = j == 0 && level1_shortcut_ok(s);
            cur = topk_check_enqueue_dev(s, st, j == 0 ? s.m_host : -1,
                                         (j == 0 && s.act_dense) || dense_next, cur, s.r, l1);
            dense_next = l1;          // the level-1 check leaves active = [0, S)
        }
        publish_copy(s, st);
        KB_CUDA(cudaEventRecord(s.chk_ev, st));
        KB_CUDA(cudaEventSynchronize(s.chk_ev));
        const bool conv = s.h_flags[1] != 0;
        const int64_t last = (int64_t)s.h_flags[3];   // level of the last check that ran
        KB_REQUIRE(last > r0 && last <= r0 + B, KB_ECUDA, "device loop lost its verdict");
        for (int64_t r = r0 + B; r > last; r--) {     // levels queued behind convergence
            s.levels.pop_back();
            s.r -= 1;
            if (s.k1_used >= 2) s.k1_used -= 2;
        }
        s.cur = cur0 ^ (int)((last - r0) & 1);
        s.act_dense = false;
        s.m_host = (int64_t)s.h_flags[0];
        (void)cur;
        if (conv) return true;
        if (s.r >= s.max_iter) return false;
    }
}


// ---------------------------------------------------------------- multi-GPU

namespace {

__global__ void __launch_bounds__(1024) k_sort_cands(const double *lower, const double *upper,
                                                     const int32_t *labels, const int32_t *src,
                                                     int dense, int64_t cnt, uint64_t *keys_out,
                                                     int64_t *labels_out, double *uppers_out,
                                                     unsigned long long *count_out) {
    extern __shared__ unsigned char smem[];
    if (count_out && threadIdx.x == 0) *count_out = (unsigned long long)cnt;
    int P = 1;
    while (P < cnt) P <<= 1;
    uint64_t *hi = (uint64_t *)smem;
    uint32_t *lo = (uint32_t *)(hi + P);
    int32_t *nid = (int32_t *)(lo + P);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        if (i < cnt) {
            const int32_t id = dense ? i : src[i];
            hi[i] = ~key_of(lower, id);
            lo[i] = (uint32_t)labels[id];
            nid[i] = id;
        } else {
            hi[i] = ~0ull;
            lo[i] = 0xFFFFFFFFu;
            nid[i] = -1;
        }
    }
    __syncthreads();
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const bool gt = hi[i] > hi[j] || (hi[i] == hi[j] && lo[i] > lo[j]);
                    if (gt == up) {
                        uint64_t th = hi[i]; hi[i] = hi[j]; hi[j] = th;
                        uint32_t tl = lo[i]; lo[i] = lo[j]; lo[j] = tl;
                        int32_t tn = nid[i]; nid[i] = nid[j]; nid[j] = tn;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        keys_out[i] = ~hi[i];
        labels_out[i] = (int64_t)lo[i];
        uppers_out[i] = upper[nid[i]];
    }
}

__global__ void k_global_cut(const uint64_t *keys, const int64_t *labels, const double *uppers,
                             const int32_t *order, int64_t kk, double eps,
                             unsigned long long *out) {
    // order: candidate indices sorted by (key desc, label asc)
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    for (int64_t i = 1 + threadIdx.x; i < kk; i += blockDim.x) {
        const double lprev = __longlong_as_double((long long)keys[order[i - 1]]);
        if (!(__dsub_rn(uppers[order[i]], eps) < lprev)) bad = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out[0] = keys[order[kk - 1]];
        out[1] = (unsigned long long)labels[order[kk - 1]];
        out[2] = !bad;
    }
}

__global__ void k_neg_keys(const uint64_t *keys, int64_t n, uint64_t *nk, int32_t *iota) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) { nk[i] = ~keys[i]; iota[i] = (int32_t)i; }
}

__global__ void k_gather_u64(const uint64_t *src, const int32_t *idx, int64_t n, uint64_t *dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}

template <typename F>
void cub_go(State *s, F &&f) {
    size_t tb = 0;
    KB_CUDA(f(nullptr, tb));
    DBuf<unsigned char> tmp;
    tmp.alloc(tb);
    KB_CUDA(f(tmp.p, tb));
    note_launch();
}

// three-way split of the active set under the cut stored in out[3], out[4]
int64_t partition_cut(State &s, cudaStream_t st, int32_t *win_out, int32_t *surv_out,
                      int64_t *nwin) {
    Graph &g = *s.g;
    unsigned long long *out = s.scratch_u64.p;
    IsWinner win{s.lower.p, g.labels(), out};
    IsSurvivor sur{s.lower.p, s.upper.p, out, s.eps};
    unsigned long long *nsel = out + 5;
    const int64_t m = s.m_host;
    auto run_part = [&](auto in) {
        cub_go(&s, [&](void *t, size_t &b) {
            return cub::DevicePartition::If(t, b, in, win_out, surv_out, s.stI.p, nsel, (int)m,
                                            win, sur, st);
        });
    };
    if (s.act_dense) run_part(cub::CountingInputIterator<int32_t>(0));
    else run_part((const int32_t *)s.act[s.cur].p);
    unsigned long long h[2];
    KB_CUDA(cudaMemcpyAsync(h, nsel, sizeof(h), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    *nwin = (int64_t)h[0];
    return (int64_t)h[1];
}

}  // namespace

void local_topk(State &s, cudaStream_t st, int64_t k, uint64_t *keys, int64_t *labels,
                double *uppers, int64_t *count) {
    Graph &g = *s.g;
    KB_REQUIRE(k <= KMAX, KB_EPARAM, "sharded top-k supports k <= 4096");
    const int64_t m = s.m_host;
    const int32_t *src = s.act[s.cur].p;
    int dense = s.act_dense;
    int64_t cnt = m;
    if (m > k) {
        TopkArgs A;
        A.lower = s.lower.p;
        A.upper = s.upper.p;
        A.perm = g.labels();
        A.act_in = s.act[s.cur].p;
        A.m = m;
        A.dense = s.act_dense;
        A.act_out = s.act[s.cur ^ 1].p;
        A.k = k;
        A.eps = s.eps;
        A.hist = (unsigned int *)(s.scratch_u64.p + 8);
        const int G = (int)std::max<int64_t>(
            1, std::min<int64_t>(coop_grid(g.sm_count), (A.m + 8191) / 8192));
        A.blk = s.scratch_u64.p + 8 + HIST_WORDS;
        A.prefix_buf = s.scratch_i32.p;
        A.cand = s.cand.p;
        A.stK = s.stK.p;
        A.stU = s.stU.p;
        A.stI = s.stI.p;
        A.out = s.scratch_u64.p;
        void *args[] = {&A};
        KB_CUDA(cudaLaunchCooperativeKernel((void *)k_topk_select, G, CHK_THREADS, args, 0, st));
        note_launch();
        int64_t nw = 0;
        DBuf<int32_t> surv;
        surv.alloc(m);
        partition_cut(s, st, s.scratch_i32.p, surv.p, &nw);
        cnt = nw;
        src = s.scratch_i32.p;
        dense = 0;
    }
    DBuf<uint64_t> dk;
    DBuf<int64_t> dl;
    DBuf<double> du;
    dk.alloc(std::max<int64_t>(1, cnt));
    dl.alloc(std::max<int64_t>(1, cnt));
    du.alloc(std::max<int64_t>(1, cnt));
    if (cnt) {
        int P = 1;
        while (P < cnt) P <<= 1;
        const size_t smem = (size_t)P * 16;
        KB_CUDA(cudaFuncSetAttribute(k_sort_cands, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        k_sort_cands<<<1, 1024, smem, st>>>(s.lower.p, s.upper.p, g.labels(), src, dense, cnt,
                                            dk.p, dl.p, du.p, nullptr);
        note_launch();
        KB_CUDA(cudaMemcpyAsync(keys, dk.p, cnt * 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaMemcpyAsync(labels, dl.p, cnt * 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaMemcpyAsync(uppers, du.p, cnt * 8, cudaMemcpyDeviceToHost, st));
    }
    KB_CUDA(cudaStreamSynchronize(st));
    *count = cnt;
}

void apply_cut(State &s, cudaStream_t st, uint64_t kstar, int64_t istar) {
    unsigned long long cut[2] = {kstar, (unsigned long long)istar};
    KB_CUDA(cudaMemcpyAsync(s.scratch_u64.p + 3, cut, sizeof(cut), cudaMemcpyHostToDevice, st));
    const int nxt = s.cur ^ 1;
    DBuf<int32_t> surv;
    surv.alloc(std::max<int64_t>(1, s.m_host));
    int64_t nw = 0;
    const int64_t ns = partition_cut(s, st, s.act[nxt].p, surv.p, &nw);
    if (ns)
        KB_CUDA(cudaMemcpyAsync(s.act[nxt].p + nw, surv.p, ns * sizeof(int32_t),
                                cudaMemcpyDeviceToDevice, st));
    KB_CUDA(cudaStreamSynchronize(st));
    s.cur = nxt;
    s.act_dense = false;
    s.m_host = nw + ns;
}

void select_global(int device, const uint64_t *keys, const int64_t *labels, const double *uppers,
                   int64_t ncand, int64_t k, double eps, uint64_t *kstar, int64_t *istar,
                   int *prefix_ok) {
    (void)device;
    cudaStream_t st = device_stream();
    DBuf<uint64_t> dk, nk, nk2;
    DBuf<int64_t> dl, l2;
    DBuf<double> du;
    DBuf<int32_t> i0, i1, i2;
    DBuf<unsigned long long> out;
    dk.alloc(ncand); nk.alloc(ncand); nk2.alloc(ncand); dl.alloc(ncand); l2.alloc(ncand);
    du.alloc(ncand); i0.alloc(ncand); i1.alloc(ncand); i2.alloc(ncand); out.alloc(3);
    KB_CUDA(cudaMemcpyAsync(dk.p, keys, ncand * 8, cudaMemcpyHostToDevice, st));
    KB_CUDA(cudaMemcpyAsync(dl.p, labels, ncand * 8, cudaMemcpyHostToDevice, st));
    KB_CUDA(cudaMemcpyAsync(du.p, uppers, ncand * 8, cudaMemcpyHostToDevice, st));
    k_neg_keys<<<nblk(ncand, 256), 256, 0, st>>>(dk.p, ncand, nk.p, i0.p);
    note_launch();
    // stable: by label ascending, then by key descending
    cub_go(nullptr, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, dl.p, l2.p, i0.p, i1.p, (int)ncand, 0, 64,
                                               st);
    });
    k_gather_u64<<<nblk(ncand, 256), 256, 0, st>>>(nk.p, i1.p, ncand, nk2.p);
    note_launch();
    cub_go(nullptr, [&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, nk2.p, nk.p, i1.p, i2.p, (int)ncand, 0, 64,
                                               st);
    });
    const int64_t kk = std::min(k, ncand);
    k_global_cut<<<1, 256, 0, st>>>(dk.p, dl.p, du.p, i2.p, kk, eps, out.p);
    note_launch();
    unsigned long long h[3];
    KB_CUDA(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    *kstar = h[0];
    *istar = (int64_t)h[1];
    *prefix_ok = (int)h[2];
}

// ------------------------------------------- device-resident shard protocol
//
// The TOPK check of a sharded run without host round trips: every rank
// writes its k proposals into a fixed-size device block, the blocks are
// all-gathered by NCCL on the same stream, every rank derives the same
// global cut on its device and splits its active set; only the new local
// count leaves the device (after the count all-reduce).  Block layout, in
// 64-bit words: [count, keys[k], labels[k], uppers[k] (f64 bits)].

namespace {

__global__ void k_unpack_blocks(const unsigned long long *blocks, int64_t P, int64_t k,
                                uint64_t *keys, int64_t *labels, double *uppers, uint64_t *nk,
                                int32_t *iota) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= P * k) return;
    const int64_t b = i / k, j = i - b * k;
    const unsigned long long *blk = blocks + b * (1 + 3 * k);
    uint64_t key = 0;
    int64_t lab = INT64_MAX;  // padding sorts after every real candidate
    double up = 0.0;
    if (j < (int64_t)blk[0]) {
        key = blk[1 + j];
        lab = (int64_t)blk[1 + k + j];
        up = __longlong_as_double((long long)blk[1 + 2 * k + j]);
    }
    keys[i] = key;
    labels[i] = lab;
    uppers[i] = up;
    nk[i] = ~key;
    iota[i] = (int32_t)i;
}

// the global cut (k-th of the merged proposals) and the adjacent-separation
// test of the merged top-k prefix; cut[3], cut[4] feed IsWinner/IsSurvivor
// the P*k proposals ordered by (key desc, label asc) in one block (nc <=
// 4096): a shared-memory bitonic sort instead of two device radix sorts
__global__ void __launch_bounds__(1024) k_order_cands(const uint64_t *nk, const int64_t *labels,
                                                      int64_t nc, int32_t *order) {
    extern __shared__ unsigned char smem[];
    int P = 1;
    while (P < nc) P <<= 1;
    uint64_t *key = (uint64_t *)smem;
    uint32_t *lab = (uint32_t *)(key + P);
    int32_t *idx = (int32_t *)(lab + P);
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        if (i < nc) {
            key[i] = nk[i];
            lab[i] = labels[i] >= 0 && labels[i] < 0xFFFFFFFFll ? (uint32_t)labels[i] : 0xFFFFFFFFu;
            idx[i] = i;
        } else {
            key[i] = ~0ull;
            lab[i] = 0xFFFFFFFFu;
            idx[i] = -1;
        }
    }
    __syncthreads();
    bitonic_kl(key, lab, idx, P);
    for (int i = threadIdx.x; i < nc; i += blockDim.x) order[i] = idx[i];
}

__global__ void k_global_cut_dev(const uint64_t *keys, const int64_t *labels,
                                 const double *uppers, const int32_t *order,
                                 const unsigned long long *blocks, int64_t P, int64_t k,
                                 double eps, unsigned long long *cut) {
    __shared__ int bad;
    __shared__ int64_t kk;
    if (threadIdx.x == 0) {
        bad = 0;
        int64_t tot = 0;
        for (int64_t b = 0; b < P; b++) tot += (int64_t)blocks[b * (1 + 3 * k)];
        kk = tot < k ? tot : k;
    }
    __syncthreads();
    for (int64_t i = 1 + threadIdx.x; i < kk; i += blockDim.x) {
        const double lprev = __longlong_as_double((long long)keys[order[i - 1]]);
        if (!(__dsub_rn(uppers[order[i]], eps) < lprev)) bad = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (kk == 0) {  // no active node anywhere: nothing wins or survives
            cut[3] = ~0ull;
            cut[4] = 0;
        } else {
            cut[3] = keys[order[kk - 1]];
            cut[4] = (unsigned long long)labels[order[kk - 1]];
        }
        cut[7] = !bad;
    }
}

// winners stay first, survivors follow; word = [m_local, m_local, prefix_ok]
__global__ void k_append_survivors(const int32_t *surv, const unsigned long long *cut,
                                   int32_t *act, long long *word) {
    const unsigned long long nw = cut[5], ns = cut[6];
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < (int64_t)ns) act[nw + i] = surv[i];
    if (i == 0) {
        word[0] = (long long)(nw + ns);
        word[1] = (long long)(nw + ns);
        word[2] = (long long)cut[7];
    }
}

}  // namespace

void shard_propose(State &s, cudaStream_t st, int64_t k, unsigned long long *blk) {
    Graph &g = *s.g;
    KB_REQUIRE(k >= 1 && k <= KMAX, KB_EPARAM, "sharded top-k supports 1 <= k <= 4096");
    KB_REQUIRE(s.m_host >= 0, KB_ESTATE, "active count pending: kb_shard_commit first");
    const int64_t m = s.m_host;
    const int32_t *src = s.act[s.cur].p;
    int dense = s.act_dense;
    const int64_t cnt = std::min(m, k);
    if (m > k) {
        TopkArgs A;
        A.lower = s.lower.p;
        A.upper = s.upper.p;
        A.perm = g.labels();
        A.act_in = s.act[s.cur].p;
        A.m = m;
        A.dense = s.act_dense;
        A.act_out = s.act[s.cur ^ 1].p;
        A.k = k;
        A.eps = s.eps;
        A.hist = (unsigned int *)(s.scratch_u64.p + 8);
        const int G = (int)std::max<int64_t>(
            1, std::min<int64_t>(coop_grid(g.sm_count), (A.m + 8191) / 8192));
        A.blk = s.scratch_u64.p + 8 + HIST_WORDS;
        A.prefix_buf = s.scratch_i32.p;
        A.cand = s.cand.p;
        A.stK = s.stK.p;
        A.stU = s.stU.p;
        A.stI = s.stI.p;
        A.out = s.scratch_u64.p;
        // the fused split writes the k local winners (labels are unique, so
        // exactly k) to the prefix buffer; its survivors land in the spare
        // active buffer, which the cut overwrites
        A.split = 1;
        A.act_cap = (int64_t)s.act[s.cur ^ 1].n;
        void *args[] = {&A};
        KB_CUDA(cudaLaunchCooperativeKernel((void *)k_topk_select, G, CHK_THREADS, args, 0, st));
        note_launch();
        src = s.scratch_i32.p;
        dense = 0;
    }
    int P = 1;
    while (P < std::max<int64_t>(1, cnt)) P <<= 1;
    const size_t smem = (size_t)P * 16;
    KB_CUDA(cudaFuncSetAttribute(k_sort_cands, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    k_sort_cands<<<1, 1024, smem, st>>>(s.lower.p, s.upper.p, g.labels(), src, dense, cnt,
                                        (uint64_t *)(blk + 1), (int64_t *)(blk + 1 + k),
                                        (double *)(blk + 1 + 2 * k), blk);
    note_launch();
}

void shard_cut(State &s, cudaStream_t st, const unsigned long long *blocks, int64_t P, int64_t k,
               long long *word) {
    KB_REQUIRE(P >= 1 && k >= 1 && k <= KMAX, KB_EPARAM, "bad proposal blocks");
    KB_REQUIRE(s.m_host >= 0, KB_ESTATE, "active count pending: kb_shard_commit first");
    const int64_t nc = P * k;
    DBuf<uint64_t> dk, nk, nk2;
    DBuf<int64_t> dl, l2;
    DBuf<double> du;
    DBuf<int32_t> i0, i1, i2, surv;
    dk.alloc(nc); nk.alloc(nc); nk2.alloc(nc); dl.alloc(nc); l2.alloc(nc);
    du.alloc(nc); i0.alloc(nc); i1.alloc(nc); i2.alloc(nc);
    k_unpack_blocks<<<nblk(nc, 256), 256, 0, st>>>(blocks, P, k, dk.p, dl.p, du.p, nk.p, i0.p);
    note_launch();
    if (nc <= 4096) {
        // (key desc, label asc) in one block
        int Pp = 1;
        while (Pp < nc) Pp <<= 1;
        const size_t smem = (size_t)Pp * 16;
        KB_CUDA(cudaFuncSetAttribute(k_order_cands, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)std::max<size_t>(smem, 1)));
        k_order_cands<<<1, 1024, smem, st>>>(nk.p, dl.p, nc, i2.p);
        note_launch();
    } else {
        // (key desc, label asc): stable sort by label, then by inverted key
        cub_go(nullptr, [&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortPairs(t, b, dl.p, l2.p, i0.p, i1.p, (int)nc, 0, 64,
                                                   st);
        });
        k_gather_u64<<<nblk(nc, 256), 256, 0, st>>>(nk.p, i1.p, nc, nk2.p);
        note_launch();
        cub_go(nullptr, [&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortPairs(t, b, nk2.p, nk.p, i1.p, i2.p, (int)nc, 0, 64,
                                                   st);
        });
    }
    unsigned long long *cut = s.scratch_u64.p;
    k_global_cut_dev<<<1, 256, 0, st>>>(dk.p, dl.p, du.p, i2.p, blocks, P, k, s.eps, cut);
    note_launch();
    // three-way split of the local active set under the global cut
    Graph &g = *s.g;
    const int64_t m = s.m_host;
    const int nxt = s.cur ^ 1;
    surv.alloc(std::max<int64_t>(1, m));
    if (m) {
        // winners (under the global cut) to act[nxt], survivors to surv, both
        // in active-set order: the select kernel's fused split with the cut
        // given (counts into cut[5], cut[6])
        TopkArgs A;
        A.lower = s.lower.p;
        A.upper = s.upper.p;
        A.perm = g.labels();
        A.act_in = s.act[s.cur].p;
        A.m = m;
        A.dense = s.act_dense;
        A.act_out = s.act[nxt].p;
        A.k = k;
        A.eps = s.eps;
        A.hist = (unsigned int *)(s.scratch_u64.p + 8);
        A.blk = s.scratch_u64.p + 8 + HIST_WORDS;
        A.prefix_buf = s.scratch_i32.p;
        A.cand = s.cand.p;
        A.stK = s.stK.p;
        A.stU = s.stU.p;
        A.stI = s.stI.p;
        A.out = cut;
        A.split = 1;
        A.cut_given = 1;
        A.win_out = s.act[nxt].p;
        A.surv_out = surv.p;
        const int G = (int)std::max<int64_t>(
            1, std::min<int64_t>(coop_grid(g.sm_count), (m + 8191) / 8192));
        void *args[] = {&A};
        KB_CUDA(cudaLaunchCooperativeKernel((void *)k_topk_select, G, CHK_THREADS, args, 0, st));
        note_launch();
    } else {
        KB_CUDA(cudaMemsetAsync(cut + 5, 0, 16, st));
    }
    k_append_survivors<<<nblk(std::max<int64_t>(1, m), 256), 256, 0, st>>>(surv.p, cut,
                                                                          s.act[nxt].p, word);
    note_launch();
    s.cur = nxt;
    s.act_dense = false;
    s.m_host = -1;  // known after the count all-reduce: kb_shard_commit
}

void shard_commit(State &s, int64_t m) {
    KB_REQUIRE(s.m_host < 0, KB_ESTATE, "no cut pending");
    KB_REQUIRE(m >= 0 && m <= s.g->n, KB_EPARAM, "bad active count");
    s.m_host = m;
}

}  // namespace kb
