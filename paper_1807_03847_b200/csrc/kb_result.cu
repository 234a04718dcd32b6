// K3: ranking_result + separated_fraction (engine.py:399-427) on the device.
//
// order = lexsort((arange(n), -lower))  (engine.py:401): nodes with lower > 0
// are stably radix-sorted on ~bits(lower) in ascending original-id order, so
// equal bounds keep ascending ids; nodes with lower == +0 (no out-arcs) are
// appended in id order -- the same permutation as a full sort, with half the
// keys at C2.
// separated pairs = sum_v #{w : lower[w] > upper[v]}  (engine.py:423-426):
// one binary search per node in the descending lower array, reduced as an
// exact 64-bit integer.
#include <cub/block/block_reduce.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>

#include "kb_internal.cuh"

namespace kb {

namespace {

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

__global__ void k_pos_flags(const double *lower, const int32_t *iperm, int64_t n,
                            unsigned char *pos, unsigned char *zero, int32_t *iota) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool p = lower[iperm[i]] > 0.0;
    pos[i] = p;
    zero[i] = !p;
    iota[i] = (int32_t)i;
}

__global__ void k_sort_keys(const double *lower, const int32_t *iperm, const int32_t *ids,
                            int64_t npos, uint64_t *keys, int32_t *nids) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= npos) return;
    const int32_t v = iperm[ids[i]];
    keys[i] = ~(uint64_t)__double_as_longlong(lower[v]);
    nids[i] = v;
}

// the same, with each block's key range to part[2 * block] (a grid-wide
// atomic pair per warp serialised at C2), reduced by k_range_reduce
__global__ void k_sort_keys_range(const double *lower, const int32_t *iperm, const int32_t *ids,
                                  int64_t npos, uint64_t *keys, int32_t *nids,
                                  unsigned long long *part) {
    __shared__ unsigned long long slo[32], shi[32];
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long lo = ~0ull, hi = 0ull;
    if (i < npos) {
        const int32_t v = iperm[ids[i]];
        const unsigned long long k = ~(uint64_t)__double_as_longlong(lower[v]);
        keys[i] = k;
        nids[i] = v;
        lo = hi = k;
    }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) { slo[w] = lo; shi[w] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < nw; q++) { lo = min(lo, slo[q]); hi = max(hi, shi[q]); }
        part[2 * blockIdx.x] = lo;
        part[2 * blockIdx.x + 1] = hi;
    }
}

__global__ void k_range_reduce(const unsigned long long *part, int64_t nb,
                               unsigned long long *mm) {
    __shared__ unsigned long long slo[32], shi[32];
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) {
        lo = min(lo, part[2 * b]);
        hi = max(hi, part[2 * b + 1]);
    }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) { slo[w] = lo; shi[w] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < nw; q++) { lo = min(lo, slo[q]); hi = max(hi, shi[q]); }
        mm[0] = lo;
        mm[1] = hi;
    }
}

// keys already offset by a host-known floor K0 = ~bits(alpha * gamma): every
// lower bound is <= the initial upper bound alpha * gamma (engine.py:151), so
// every key is >= K0; a key below it (rounding at a bound that tight) sets
// the fallback flag and the caller redoes the full sort
__global__ void k_sort_keys_off(const double *lower, const int32_t *iperm, const int32_t *ids,
                                int64_t npos, uint64_t *keys, int32_t *nids, uint64_t K0,
                                uint64_t K1, unsigned long long *mm) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i == 0) mm[0] = K0;
    if (i >= npos) return;
    const int32_t v = iperm[ids[i]];
    const uint64_t k = ~(uint64_t)__double_as_longlong(lower[v]);
    if (k < K0 || k > K1) atomicOr(&mm[3], 1ull);   // outside the bounds: fall back
    keys[i] = k - K0;
    nids[i] = v;
}

__global__ void k_offset_keys(uint64_t *keys, int64_t n, const unsigned long long *mm) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) keys[i] -= mm[0];
}

// After a stable sort on bits [shift, 64) of the offset keys, a run of equal
// prefixes is in input (ascending id) order, which is the final order unless
// its low bits disagree.  Each run holding such a disagreement is found once
// (by its first element), listed, and put in order by one thread: an
// insertion sort on the full offset key that only moves past strictly
// greater keys, so equal keys keep ascending ids.  Runs longer than FIX_MAX
// (or walks past it) set the fallback flag.
constexpr int FIX_MAX = 512;

__global__ void k_fix_find(const uint64_t *k, int64_t n, int shift, unsigned int *claimed,
                           int64_t *runs, int64_t cap, unsigned long long *nruns,
                           unsigned long long *fallback, const int32_t *ids = nullptr,
                           const int32_t *perm = nullptr, int32_t *order = nullptr) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (order && i < n) order[i] = perm[ids[i]];   // the id map, fused (runs re-map theirs)
    if (i < 1 || i >= n) return;
    if ((k[i - 1] >> shift) != (k[i] >> shift) || k[i - 1] <= k[i]) return;
    const uint64_t p = k[i] >> shift;
    int64_t a = i - 1;
    while (a > 0 && (k[a - 1] >> shift) == p) {
        if (i - a > FIX_MAX) { atomicExch(fallback, 1ull); return; }
        a--;
    }
    // claim the run by its first element (one flag bit per element)
    const unsigned int bit = 1u << (a & 31);
    if (atomicOr(&claimed[a >> 5], bit) & bit) return;
    int64_t b = i + 1;
    while (b < n && (k[b] >> shift) == p) {
        if (b - a > FIX_MAX) { atomicExch(fallback, 1ull); return; }
        b++;
    }
    const unsigned long long slot = atomicAdd(nruns, 1ull);
    if ((int64_t)slot >= cap) { atomicExch(fallback, 1ull); return; }
    runs[2 * slot] = a;
    runs[2 * slot + 1] = b;
}

// one warp per listed run: (key, position) pairs into shared memory, a
// bitonic sort there (the position keeps equal keys in input order), back
constexpr int FIX_WARPS = 4;

__global__ void __launch_bounds__(32 * FIX_WARPS) k_fix_runs(uint64_t *k, int32_t *ids,
                                                             const int64_t *runs, int64_t cap,
                                                             const unsigned long long *nruns,
                                                             const int32_t *perm = nullptr,
                                                             int32_t *order = nullptr) {
    __shared__ uint64_t sk[FIX_WARPS][FIX_MAX];
    __shared__ int32_t sp[FIX_WARPS][FIX_MAX];
    __shared__ int32_t si[FIX_WARPS][FIX_MAX];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned long long nr = min(*nruns, (unsigned long long)cap);
    for (unsigned long long r = (unsigned long long)blockIdx.x * FIX_WARPS + w; r < nr;
         r += (unsigned long long)gridDim.x * FIX_WARPS) {
        const int64_t a = runs[2 * r];
        const int L = (int)(runs[2 * r + 1] - a);
        int P = 1;
        while (P < L) P <<= 1;
        for (int i = lane; i < P; i += 32) {
            sk[w][i] = i < L ? k[a + i] : ~0ull;
            sp[w][i] = i < L ? i : 0x7fffffff;
            si[w][i] = i < L ? ids[a + i] : 0;
        }
        __syncwarp();
        for (int size = 2; size <= P; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = lane; i < P; i += 32) {
                    const int j = i ^ stride;
                    if (j > i) {
                        const bool up = (i & size) == 0;
                        const bool gt = sk[w][i] > sk[w][j] ||
                                        (sk[w][i] == sk[w][j] && sp[w][i] > sp[w][j]);
                        if (gt == up) {
                            const uint64_t tk = sk[w][i]; sk[w][i] = sk[w][j]; sk[w][j] = tk;
                            const int32_t tp = sp[w][i]; sp[w][i] = sp[w][j]; sp[w][j] = tp;
                            const int32_t ti = si[w][i]; si[w][i] = si[w][j]; si[w][j] = ti;
                        }
                    }
                }
                __syncwarp();
            }
        for (int i = lane; i < L; i += 32) {
            k[a + i] = sk[w][i];
            ids[a + i] = si[w][i];
            if (order) order[a + i] = perm[si[w][i]];
        }
        __syncwarp();
    }
}



__global__ void k_new_to_orig(const int32_t *perm, const int32_t *nids, int64_t n, int32_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) KB_DCHECK(nids[i] >= 0);
    if (i < n) out[i] = perm[nids[i]];
}

// Separated pairs counted by rank: the node at rank t (descending lower) has
// upper >= lower, so every w with lower[w] > upper[v] ranks before it and the
// count is the first rank j <= t with sorted[j] <= upper[v].  Bounds are
// tight, so j is found by galloping down from t inside a small window that
// neighbouring threads share (coalesced, cache resident).
__global__ void k_sep_pairs_rank(const uint64_t *skeys, const int32_t *snids, int64_t npos,
                                 const double *upper, unsigned long long *total,
                                 const unsigned long long *koff) {
    typedef cub::BlockReduce<unsigned long long, 256> Red;
    __shared__ typename Red::TempStorage tmp;
    unsigned long long acc = 0;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < npos) {
        const double u = upper[snids[t]];
        const unsigned long long off = koff ? *koff : 0ull;
        auto val = [&](int64_t j) { return __longlong_as_double((long long)~(skeys[j] + off)); };
        // invariant: val(hi) <= u ; find smallest j in [0, hi] with val(j) <= u
        int64_t hi = t, step = 1, lo = t;
        while (true) {
            lo = hi - step;
            if (lo < 0) { lo = -1; break; }
            if (val(lo) > u) break;
            hi = lo;
            step <<= 1;
        }
        // val(lo) > u (or lo == -1), val(hi) <= u
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (val(mid) > u) lo = mid; else hi = mid;
        }
        acc = (unsigned long long)hi;
    }
    acc = Red(tmp).Sum(acc);
    if (threadIdx.x == 0 && acc) atomicAdd(total, acc);
}

// The same count with a search table for far answers (graphs with many
// unseparated pairs, e.g. the grid, where galloping walks far): a few
// galloping steps near t first (R-MAT's answers are near), then a bisection
// of a shared-memory sample of every S-th sorted key, then one of the
// S-long window it selects.
constexpr int SEP_TAB = 4096;
constexpr int SEP_GALLOP = 6;

__global__ void k_sep_tab(const uint64_t *skeys, int64_t npos, int64_t S, uint64_t *tab) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < SEP_TAB) tab[i] = skeys[min(i * S, npos - 1)];
}

__global__ void __launch_bounds__(256) k_sep_pairs_tab(const uint64_t *skeys,
                                                       const int32_t *snids, int64_t npos,
                                                       const double *upper,
                                                       const uint64_t *__restrict__ tab, int64_t S,
                                                       unsigned long long *total,
                                                       const unsigned long long *koff) {
    typedef cub::BlockReduce<unsigned long long, 256> Red;
    __shared__ typename Red::TempStorage tmp;
    unsigned long long acc = 0;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < npos) {
        // lower(j) <= u  <=>  skeys[j] >= ~bits(u)  (keys ascend as lower descends);
        // keys offset by koff (the prefix sort): compare against ku - koff,
        // which is 0 -- below every key -- when ku < koff
        uint64_t ku = ~(uint64_t)__double_as_longlong(upper[snids[t]]);
        if (koff) ku = ku < *koff ? 0ull : ku - *koff;
        int64_t hi = t, lo = -1, step = 1;
        bool found = false;
        for (int g = 0; g < SEP_GALLOP; g++) {
            const int64_t c = hi - step;
            if (c < 0) { lo = -1; found = true; break; }
            if (skeys[c] < ku) { lo = c; found = true; break; }
            hi = c;
            step <<= 1;
        }
        if (!found) {
            // first sample i with tab[i] >= ku among samples at or below hi
            // (the 32 KB table stays in L1/L2: every thread reads it)
            int a = 0, b = (int)min((int64_t)SEP_TAB, hi / S + 1);
            while (a < b) {
                const int mid = (a + b) >> 1;
                if (__ldg(tab + mid) >= ku) b = mid; else a = mid + 1;
            }
            lo = a == 0 ? -1 : (int64_t)(a - 1) * S;
            hi = min(hi, (int64_t)a * S);
        }
        while (hi - lo > 1) {            // keys[lo] < ku (or lo = -1), keys[hi] >= ku
            const int64_t mid = (lo + hi) >> 1;
            if (skeys[mid] < ku) lo = mid; else hi = mid;
        }
        acc = (unsigned long long)hi;
    }
    acc = Red(tmp).Sum(acc);
    if (threadIdx.x == 0 && acc) atomicAdd(total, acc);
}

__global__ void k_widen(const int32_t *src, int64_t n, int64_t *dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i];
}

}  // namespace


// separated pairs of the sorted positive part (ties and zero bounds are
// handled by the callers): galloping for near answers, a table for far ones
static void sep_pairs(const uint64_t *skeys, const int32_t *snids, int64_t npos,
                      const double *upper, unsigned long long *total, int sms,
                      cudaStream_t st, const unsigned long long *koff = nullptr) {
    if (npos <= 0) return;
    if (!tune_get("result.sep_table", 1) || npos < 4 * SEP_TAB) {
        k_sep_pairs_rank<<<nblk(npos, 256), 256, 0, st>>>(skeys, snids, npos, upper, total,
                                                          koff);
        note_launch();
        return;
    }
    const int64_t S = (npos + SEP_TAB - 1) / SEP_TAB;
    DBuf<uint64_t> tab;
    tab.alloc(SEP_TAB);
    k_sep_tab<<<nblk(SEP_TAB, 256), 256, 0, st>>>(skeys, npos, S, tab.p);
    k_sep_pairs_tab<<<nblk(npos, 256), 256, 0, st>>>(skeys, snids, npos, upper, tab.p, S, total,
                                                     koff);
    (void)sms;
    note_launch(2);
    KB_CUDA(cudaGetLastError());
}

namespace {
template <typename F>
void cub_do(F &&f) {
    size_t tb = 0;
    KB_CUDA(f(nullptr, tb));
    DBuf<unsigned char> tmp;
    tmp.alloc(tb);
    KB_CUDA(f(tmp.p, tb));
    note_launch();
}
}  // namespace

// Stable ascending sort of 64-bit keys with an int32 payload (input in id
// order, so equal keys keep ascending ids): CUB onesweep radix sort.  (A
// 32-bit leading-bits sort plus in-run fix-up was measured slower at C2:
// 2.1 vs 1.1 ms, because R-MAT bounds cluster densely.)
void sort_keys_stable(const uint64_t *kin, const int32_t *nids, int64_t m, uint64_t *kout,
                      int32_t *snids, cudaStream_t st) {
    if (m == 0) return;
    cub_do([&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, kin, kout, nids, snids, m, 0, 64, st);
    });
}

// positive-bound nodes by ascending original id, and the rest, from the
// flags of the current lower bounds (after dynamic updates; static runs read
// the lists precomputed at ingest, Graph::orig_pos / orig_zero, in place)
static void split_positive(State &s, cudaStream_t st, DBuf<int32_t> &ids, int32_t *zero_out,
                           int64_t &npos) {
    Graph &g = *s.g;
    const int64_t n = g.n;
    DBuf<unsigned char> fpos, fzero;
    DBuf<int32_t> iota;
    fpos.alloc(n); fzero.alloc(n); iota.alloc(n);
    unsigned long long *u = s.scratch_u64.p + 16;
    KB_CUDA(cudaMemsetAsync(u, 0, 2 * sizeof(unsigned long long), st));
    k_pos_flags<<<nblk(n, 256), 256, 0, st>>>(s.lower.p, g.iperm.p, n, fpos.p, fzero.p, iota.p);
    note_launch();
    size_t tb = 0;
    KB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, fpos.p, ids.p, u, (int)n, st));
    ensure_cub_tmp(s, tb);
    KB_CUDA(cub::DeviceSelect::Flagged(s.cub_tmp.p, tb, iota.p, fpos.p, ids.p, u, (int)n, st));
    note_launch();
    unsigned long long hcnt = 0;
    KB_CUDA(cudaMemcpyAsync(&hcnt, u, sizeof(hcnt), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    npos = (int64_t)hcnt;
    tb = 0;
    KB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, fzero.p, zero_out, u + 1, (int)n, st));
    ensure_cub_tmp(s, tb);
    KB_CUDA(cub::DeviceSelect::Flagged(s.cub_tmp.p, tb, iota.p, fzero.p, zero_out, u + 1, (int)n,
                                       st));
    note_launch();
}

// ranking_result on the device: order (int64 original ids), lower and upper
// by original id, and the exact separated-pair count
// The ranking order with fewer radix passes (round 2): the keys are offset
// by their minimum, so they vary in B low bits; a stable CUB sort on the top
// min(B, 40) of them -- 5 onesweep passes instead of 8 at C2, where B = 57 --
// is followed by the fix-up of the equal-prefix runs whose low bits disagree
// (C2: ~12K runs of <= 97 keys).  B <= 56 (the grid) sorts every varying
// bit, with no fix-up.  Writes kout (full keys, ascending), snids and the
// order; false = not applicable / fall back (run too long, too many runs).
static bool sort_prefix_core(const double *lower, const int32_t *iperm, const int32_t *pos_ids,
                             int64_t npos, DBuf<uint64_t> &kin, DBuf<int32_t> &nids,
                             DBuf<uint64_t> &kout, DBuf<int32_t> &snids, unsigned long long *mm,
                             int sms, cudaStream_t st, double alpha = 0, double gamma = 0,
                             const int32_t *perm = nullptr, int32_t *order = nullptr) {
    // perm/order: also write order = perm[snids] (fused into the fix-up
    // passes when there is one; returns whether it was written)
    // mm (device, 4 words): key offset (minimum), maximum, fix-up run count,
    // fallback
    KB_CUDA(cudaMemsetAsync(mm + 2, 0, 16, st));
    unsigned long long d;
    const double ag = alpha * gamma;
    if (alpha > 0 && ag >= alpha && tune_get("result.prefix_bound", 1)) {
        // the key range from bounds the host knows, no device reduction, no
        // host read: lower <= alpha * gamma (the initial upper bound) and
        // every positive lower >= alpha (katz_1 of a row with an arc)
        uint64_t bg, ba;
        memcpy(&bg, &ag, 8);
        memcpy(&ba, &alpha, 8);
        const uint64_t K0 = ~bg, K1 = ~ba;
        k_sort_keys_off<<<nblk(npos, 256), 256, 0, st>>>(lower, iperm, pos_ids, npos, kin.p,
                                                         nids.p, K0, K1, mm);
        note_launch();
        d = K1 - K0;
    } else {
        const int64_t nb = (int64_t)nblk(npos, 256);
        DBuf<unsigned long long> part;
        part.alloc(2 * nb);
        k_sort_keys_range<<<(unsigned)nb, 256, 0, st>>>(lower, iperm, pos_ids, npos, kin.p,
                                                        nids.p, part.p);
        k_range_reduce<<<1, 1024, 0, st>>>(part.p, nb, mm);
        note_launch(2);
        unsigned long long h[2];
        KB_CUDA(cudaMemcpyAsync(h, mm, sizeof(h), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        d = h[1] - h[0];
        k_offset_keys<<<nblk(npos, 256), 256, 0, st>>>(kin.p, npos, mm);
        note_launch();
    }
    int B = 0;
    while (B < 64 && (d >> B)) B++;
    // prefix width: ~16 bits above log2(npos), in whole 8-bit passes (C2,
    // 8.9M keys: 40 bits -- 12.5K short runs to fix; C3, 63M keys: 48 bits,
    // where 40 would leave runs of 4K keys)
    int lg = 1;
    while (lg < 62 && ((int64_t)1 << lg) < npos) lg++;
    int HB = (int)tune_get("result.prefix_bits", 0);        // <= 0: the default
    if (HB <= 0) HB = std::min(56, (lg + 16 + 7) / 8 * 8);
    const int exact = (int)tune_get("result.prefix_exact_bits", 56);  // sort all bits up to this
    const int shift = B <= exact ? 0 : std::max(0, B - HB);
    if (B == 0) {
        KB_CUDA(cudaMemcpyAsync(kout.p, kin.p, npos * 8, cudaMemcpyDeviceToDevice, st));
        KB_CUDA(cudaMemcpyAsync(snids.p, nids.p, npos * 4, cudaMemcpyDeviceToDevice, st));
    } else {
        cub_do([&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortPairs(t, b, kin.p, kout.p, nids.p, snids.p, npos,
                                                   shift, B, st);
        });
    }
    if (shift > 0) {
        const int64_t cap = std::min<int64_t>(npos, (int64_t)1 << 20);
        DBuf<unsigned int> claimed;
        DBuf<int64_t> runs;
        claimed.alloc((npos + 31) / 32);
        runs.alloc(2 * cap);
        KB_CUDA(cudaMemsetAsync(claimed.p, 0, claimed.bytes(), st));
        k_fix_find<<<nblk(npos, 256), 256, 0, st>>>(kout.p, npos, shift, claimed.p, runs.p, cap,
                                                    mm + 2, mm + 3, snids.p, perm, order);
        k_fix_runs<<<8 * sms, 32 * FIX_WARPS, 0, st>>>(kout.p, snids.p, runs.p, cap, mm + 2,
                                                      perm, order);
        note_launch(2);
        // mm[3] (a run too long, too many runs) is read with the pair count;
        // the caller then redoes the ranking with the full sort
        KB_CUDA(cudaGetLastError());
        return order != nullptr;
    }
    KB_CUDA(cudaGetLastError());
    return false;     // kout stays offset by mm[0]: sep_pairs compares against ku - mm[0]
}

// The ranking order with fewer radix passes (round 2): the keys are offset
// by their minimum, so they vary in B low bits; a stable CUB sort on the top
// ~log2(n) + 16 of them (whole 8-bit passes) is followed by the fix-up of
// the equal-prefix runs whose low bits disagree.  Keys varying in <= 56 bits
// (the grid) are sorted on all of them with no fix-up.
static bool sort_prefix(State &s, cudaStream_t st, const int32_t *pos_ids, int64_t npos,
                        DBuf<uint64_t> &kin, DBuf<int32_t> &nids, DBuf<uint64_t> &kout,
                        DBuf<int32_t> &snids, int32_t *order) {
    Graph &g = *s.g;
    if (!sort_prefix_core(s.lower.p, g.iperm.p, pos_ids, npos, kin, nids, kout, snids,
                          s.scratch_u64.p + 32, g.sm_count, st, s.alpha, s.gamma, g.perm.p,
                          order)) {
        k_new_to_orig<<<nblk(npos, 256), 256, 0, st>>>(g.perm.p, snids.p, npos, order);
        note_launch();
    }
    return true;
}

void result_device(State &s, cudaStream_t st, DBuf<int64_t> *order64, DBuf<double> *lower,
                   DBuf<double> *upper, int64_t *h_pairs) {
    NvtxRange nv("K3 ranking_result");
    Graph &g = *s.g;
    const int64_t n = g.n;
    KB_REQUIRE(s.r >= 1, KB_ESTATE, "separated_fraction needs at least one iteration");
    DBuf<int32_t> ids, order, nids, snids;
    DBuf<uint64_t> kin, kout;
    order.alloc(n);
    int64_t npos = 0;
    const int32_t *pos_ids = nullptr;           // positive-bound nodes, ascending id
    if (s.zero_tail_exact && g.orig_pos.p) {
        // static runs: exactly the rows with out-arcs are positive, and their
        // lists were laid out at ingest -- read in place, zero part copied once
        npos = g.nv;
        pos_ids = g.orig_pos.p;
        if (n > npos)
            KB_CUDA(cudaMemcpyAsync(order.p + npos, g.orig_zero.p, (n - npos) * sizeof(int32_t),
                                    cudaMemcpyDeviceToDevice, st));
    } else {
        ids.alloc(n);
        split_positive(s, st, ids, order.p, npos);  // zero part lands at order[0..)
        pos_ids = ids.p;
        if (n > npos) {                             // shift it behind the positive part
            DBuf<int32_t> zero_part;
            zero_part.alloc(n - npos);
            KB_CUDA(cudaMemcpyAsync(zero_part.p, order.p, (n - npos) * sizeof(int32_t),
                                    cudaMemcpyDeviceToDevice, st));
            KB_CUDA(cudaMemcpyAsync(order.p + npos, zero_part.p,
                                    (n - npos) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        }
    }
    unsigned long long *u = s.scratch_u64.p;  // [2]=pairs
    KB_CUDA(cudaMemsetAsync(u + 2, 0, sizeof(unsigned long long), st));
    // +4: the own sort loads tiles in 16-byte chunks (kb_sort.cu)
    kin.alloc(npos + 4); kout.alloc(npos + 4); nids.alloc(npos + 4); snids.alloc(npos + 4);
    bool sorted = false;
    if (npos >= (1 << 16) && npos < ((int64_t)1 << 31) && tune_get("result.prefix_sort", 1) &&
        !tune_get("result.own_sort", 0))
        sorted = sort_prefix(s, st, pos_ids, npos, kin, nids, kout, snids, order.p);
    if (npos && !sorted) {
        k_sort_keys<<<nblk(npos, 256), 256, 0, st>>>(s.lower.p, g.iperm.p, pos_ids, npos, kin.p,
                                                     nids.p);
        note_launch();
        if (!tune_get("result.own_sort", 0)) {
            sort_keys_stable(kin.p, nids.p, npos, kout.p, snids.p, st);
        } else if (!radix_sort_pairs(kin.p, nids.p, kout.p, snids.p, npos, g.device, st)) {
            std::swap(kin, kout);                       // sorted pairs ended in (kin, nids)
            std::swap(nids, snids);
        }
        k_new_to_orig<<<nblk(npos, 256), 256, 0, st>>>(g.perm.p, snids.p, npos, order.p);
        note_launch();
    }
    if (n >= 2 && npos) {
        sep_pairs(kout.p, snids.p, npos, s.upper.p, u + 2, g.sm_count, st,
                  sorted ? s.scratch_u64.p + 32 : nullptr);
    }
    if (order64) {
        order64->alloc(n);
        k_widen<<<nblk(n, 256), 256, 0, st>>>(order.p, n, order64->p); note_launch();
    }
    if (lower) {
        lower->alloc(n);
        gather_to_original(g, s.lower.p, lower->p, st);
    }
    if (upper) {
        upper->alloc(n);
        gather_to_original(g, s.upper.p, upper->p, st);
    }
    unsigned long long pairs = 0, fallback = 0;
    KB_CUDA(cudaMemcpyAsync(&pairs, u + 2, sizeof(pairs), cudaMemcpyDeviceToHost, st));
    if (sorted) KB_CUDA(cudaMemcpyAsync(&fallback, u + 35, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    if (fallback) {   // the prefix sort's fix-up gave up: the full sort, redone
        k_sort_keys<<<nblk(npos, 256), 256, 0, st>>>(s.lower.p, g.iperm.p, pos_ids, npos, kin.p,
                                                     nids.p);
        note_launch();
        sort_keys_stable(kin.p, nids.p, npos, kout.p, snids.p, st);
        k_new_to_orig<<<nblk(npos, 256), 256, 0, st>>>(g.perm.p, snids.p, npos, order.p);
        note_launch();
        KB_CUDA(cudaMemsetAsync(u + 2, 0, sizeof(unsigned long long), st));
        if (n >= 2) sep_pairs(kout.p, snids.p, npos, s.upper.p, u + 2, g.sm_count, st);
        if (order64) {
            k_widen<<<nblk(n, 256), 256, 0, st>>>(order.p, n, order64->p); note_launch();
        }
        KB_CUDA(cudaMemcpyAsync(&pairs, u + 2, sizeof(pairs), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
    }
    // zero-bound nodes have upper == 0: every positive lower separates them
    pairs += (unsigned long long)(n - npos) * (unsigned long long)npos;
    if (h_pairs) *h_pairs = (int64_t)pairs;
}

static bool host_pinned(const void *p) {
    cudaPointerAttributes a{};
    const bool ok = p && cudaPointerGetAttributes(&a, p) == cudaSuccess &&
                    a.type == cudaMemoryTypeHost;
    (void)cudaGetLastError();
    return ok;
}

// ranking_result to host arrays.  With page-locked destinations the bound
// vectors are gathered first and downloaded on the copy stream while the
// order is sorted on the device stream.
void run_result(State &s, cudaStream_t st, int64_t *h_order, double *h_lower, double *h_upper,
                int64_t *h_pairs) {
    const int64_t n = s.g->n;
    DBuf<int64_t> o;
    DBuf<double> lo, up;
    const bool early = (h_lower || h_upper) && (!h_lower || host_pinned(h_lower)) &&
                       (!h_upper || host_pinned(h_upper));
    cudaStream_t cs = nullptr;
    cudaEvent_t ev = nullptr;
    if (early) {
        cs = copy_stream();
        if (h_lower) {
            lo.alloc(n);
            gather_to_original(*s.g, s.lower.p, lo.p, st);
        }
        if (h_upper) {
            up.alloc(n);
            gather_to_original(*s.g, s.upper.p, up.p, st);
        }
        KB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        KB_CUDA(cudaEventRecord(ev, st));
        KB_CUDA(cudaStreamWaitEvent(cs, ev, 0));
        if (h_lower) KB_CUDA(cudaMemcpyAsync(h_lower, lo.p, n * 8, cudaMemcpyDeviceToHost, cs));
        if (h_upper) KB_CUDA(cudaMemcpyAsync(h_upper, up.p, n * 8, cudaMemcpyDeviceToHost, cs));
    }
    try {
        result_device(s, st, h_order ? &o : nullptr, (h_lower && !early) ? &lo : nullptr,
                      (h_upper && !early) ? &up : nullptr, h_pairs);
        if (h_order) download_d2h(h_order, o.p, n * 8, st);
        if (!early) {
            if (h_lower) download_d2h(h_lower, lo.p, n * 8, st);
            if (h_upper) download_d2h(h_upper, up.p, n * 8, st);
        }
        KB_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
        if (cs) cudaStreamSynchronize(cs);
        if (ev) cudaEventDestroy(ev);
        throw;
    }
    if (cs) {
        KB_CUDA(cudaStreamSynchronize(cs));
        KB_CUDA(cudaEventDestroy(ev));
    }
}

namespace {
__global__ void k_iota32(int64_t n, int32_t *a) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = (int32_t)i;
}
}  // namespace

// ranking_result + separated pairs on caller vectors indexed by node id
// (the multi-GPU path gathers the shard bounds and ranks them here)
namespace {
__global__ void k_scatter_by_label(const double *lo_x, const double *up_x, const int32_t *label,
                                   int64_t N, int64_t n, double *lo, double *up) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= N) return;
    const int32_t v = label[e];
    if (v >= 0 && v < n) {
        lo[v] = lo_x[e];
        up[v] = up_x[e];
    }
}
}  // namespace

// ranking_result + separated pairs on device vectors indexed by node id
static void rank_bounds_core(cudaStream_t st, int64_t n, const double *lo, const double *up,
                             int64_t *h_order, int64_t *h_pairs) {
    DBuf<int32_t> iota, ids, order, zero_part, nids, snids;
    DBuf<unsigned char> fpos, fzero;
    DBuf<uint64_t> kin, kout;
    DBuf<unsigned long long> u;
    iota.alloc(n); ids.alloc(n); order.alloc(n); fpos.alloc(n); fzero.alloc(n); u.alloc(8);
    KB_CUDA(cudaMemsetAsync(u.p, 0, 8 * 8, st));
    k_iota32<<<nblk(n, 256), 256, 0, st>>>(n, iota.p);
    k_pos_flags<<<nblk(n, 256), 256, 0, st>>>(lo, iota.p, n, fpos.p, fzero.p, ids.p);
    note_launch(2);
    auto sel = [&](unsigned char *fl, int32_t *outp, unsigned long long *cnt) {
        size_t tb = 0;
        KB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, fl, outp, cnt, (int)n, st));
        DBuf<unsigned char> t;
        t.alloc(tb);
        KB_CUDA(cub::DeviceSelect::Flagged(t.p, tb, iota.p, fl, outp, cnt, (int)n, st));
        note_launch();
    };
    sel(fpos.p, ids.p, u.p);
    zero_part.alloc(n);
    sel(fzero.p, zero_part.p, u.p + 1);
    unsigned long long hc[2];
    KB_CUDA(cudaMemcpyAsync(hc, u.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    const int64_t npos = (int64_t)hc[0];
    // +4: the own sort loads tiles in 16-byte chunks (kb_sort.cu)
    kin.alloc(npos + 4); kout.alloc(npos + 4); nids.alloc(npos + 4); snids.alloc(npos + 4);
    int dev = 0, sms = 148;
    KB_CUDA(cudaGetDevice(&dev));
    KB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // the prefix sort (sort_prefix_core) when large enough, as on one GPU
    // (measured slower here than the full sort on the sharded C2 result,
    // 13.4 vs 12.9 ms per step: kept behind result.prefix_gathered)
    const bool prefix = npos >= (1 << 16) && npos < ((int64_t)1 << 31) &&
                        tune_get("result.prefix_sort", 1) != 0 &&
                        tune_get("result.prefix_gathered", 0) != 0;
    auto full_sort = [&] {
        k_sort_keys<<<nblk(npos, 256), 256, 0, st>>>(lo, iota.p, ids.p, npos, kin.p, nids.p);
        note_launch();
        sort_keys_stable(kin.p, nids.p, npos, kout.p, snids.p, st);
        KB_CUDA(cudaMemcpyAsync(order.p, snids.p, npos * 4, cudaMemcpyDeviceToDevice, st));
        if (n >= 2) sep_pairs(kout.p, snids.p, npos, up, u.p + 2, sms, st);
    };
    if (npos && prefix) {
        sort_prefix_core(lo, iota.p, ids.p, npos, kin, nids, kout, snids, u.p + 4, sms, st);
        KB_CUDA(cudaMemcpyAsync(order.p, snids.p, npos * 4, cudaMemcpyDeviceToDevice, st));
        if (n >= 2) sep_pairs(kout.p, snids.p, npos, up, u.p + 2, sms, st, u.p + 4);
    } else if (npos) {
        full_sort();
    }
    if (n > npos)
        KB_CUDA(cudaMemcpyAsync(order.p + npos, zero_part.p, (n - npos) * 4,
                                cudaMemcpyDeviceToDevice, st));
    if (h_order) {
        DBuf<int64_t> wide;
        wide.alloc(n);
        k_widen<<<nblk(n, 256), 256, 0, st>>>(order.p, n, wide.p);
        note_launch();
        download_d2h(h_order, wide.p, n * 8, st);
    }
    unsigned long long pairs = 0, fallback = 0;
    KB_CUDA(cudaMemcpyAsync(&pairs, u.p + 2, 8, cudaMemcpyDeviceToHost, st));
    if (npos && prefix) KB_CUDA(cudaMemcpyAsync(&fallback, u.p + 7, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    if (fallback) {   // the prefix sort's fix-up gave up: the full sort, redone
        KB_CUDA(cudaMemsetAsync(u.p + 2, 0, 8, st));
        full_sort();
        if (h_order) {
            DBuf<int64_t> wide;
            wide.alloc(n);
            k_widen<<<nblk(n, 256), 256, 0, st>>>(order.p, n, wide.p);
            note_launch();
            download_d2h(h_order, wide.p, n * 8, st);
        }
        KB_CUDA(cudaMemcpyAsync(&pairs, u.p + 2, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
    }
    pairs += (unsigned long long)(n - npos) * (unsigned long long)npos;
    if (h_pairs) *h_pairs = (int64_t)pairs;
}

void rank_bounds(int device, int64_t n, const double *h_lower, const double *h_upper,
                 int64_t *h_order, int64_t *h_pairs) {
    (void)device;
    cudaStream_t st = device_stream();
    DBuf<double> lo, up;
    lo.alloc(n); up.alloc(n);
    KB_CUDA(cudaMemcpyAsync(lo.p, h_lower, n * 8, cudaMemcpyHostToDevice, st));
    KB_CUDA(cudaMemcpyAsync(up.p, h_upper, n * 8, cudaMemcpyHostToDevice, st));
    rank_bounds_core(st, n, lo.p, up.p, h_order, h_pairs);
}

// The multi-GPU result: the state's lower/upper hold every shard's block
// (exchange layout) after the all-gather; the graph labels map exchange ids
// to node ids (>= n: padding).  Everything stays on the device.
void rank_gathered(State &s, int64_t n, int64_t *h_order, double *h_lower, double *h_upper,
                   int64_t *h_pairs) {
    Graph &g = *s.g;
    cudaStream_t st = g.stream;
    DBuf<double> lo, up;
    lo.alloc(n); up.alloc(n);
    k_scatter_by_label<<<nblk(g.n, 256), 256, 0, st>>>(s.lower.p, s.upper.p, g.labels(), g.n, n,
                                                      lo.p, up.p);
    note_launch();
    if (h_lower) download_d2h(h_lower, lo.p, n * 8, st);
    if (h_upper) download_d2h(h_upper, up.p, n * 8, st);
    rank_bounds_core(st, n, lo.p, up.p, h_order, h_pairs);
}

}  // namespace kb
