// Stable LSD radix sort of (uint64 key, int32 value) pairs: K3's order
// (ranking_result, engine.py:399-408: lexsort((arange(n), -lower)) as a
// stable sort of ~bits(lower) over ids in ascending order).
//
// One pass over the keys builds the 256-bin histograms of all eight bytes;
// byte positions whose keys all share one digit are skipped (their pass is
// the identity).  Each remaining pass is reduce-then-scan:
//   * upsweep: every 4096-key tile counts its digits (bin-major counts);
//   * scan: one block per digit turns its column of tile counts into the
//     tiles' global offsets (plus the digit's base from the histogram);
//   * downsweep: each tile ranks its keys warp by warp (__match_any_sync
//     groups the lanes of a digit; per-warp digit counters in shared memory
//     keep element order: warp, then item, then lane), reorders the tile by
//     digit in shared memory and writes it out in runs, so consecutive
//     threads store consecutive addresses.
// Measured at C2 (8.9M pairs, 8 passes): upsweep 39 us + offsets 7 us +
// downsweep 111 us per pass, against 82 us for CUB's onesweep -- the
// downsweep is latency-bound (3 blocks/SM, every warp waiting on its tile's
// key loads before ranking).  A persistent variant loading the next tile
// with cp.async while ranking the current one (one 256-thread CTA per SM)
// measured 127 us: the per-warp ranking chain (16 items, each waiting on
// the previous item's shared counter update) then binds.  A single-pass onesweep variant with decoupled
// look-back measured 120-135 us per pass.  So K3 keeps CUB's sort by default
// and this one runs with kb_tune("result.own_sort", 1) (bit-identical
// order; tests/test_gpu_fullsize.py digests pass with either).
#include <algorithm>
#include <mutex>

#include "kb_internal.cuh"

namespace kb {

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;   // 4096
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_BINS = 256;

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// histograms of all 8 byte positions: hist[p * 256 + d]
__global__ void __launch_bounds__(256) k_rs_hist(const uint64_t *keys, int64_t n,
                                                 unsigned long long *hist) {
    __shared__ unsigned int sh[8 * RS_BINS];
    for (int i = threadIdx.x; i < 8 * RS_BINS; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t k = keys[i];
#pragma unroll
        for (int p = 0; p < 8; p++) atomicAdd(&sh[p * RS_BINS + ((k >> (8 * p)) & 255)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 8 * RS_BINS; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

// exclusive scan of each byte's histogram into base[p * 256 + d]; skip[p] = 1
// when one digit holds every key
__global__ void __launch_bounds__(RS_BINS) k_rs_scan(const unsigned long long *hist, int64_t n,
                                                     unsigned long long *base, int *skip) {
    __shared__ unsigned long long s[RS_BINS];
    const int p = blockIdx.x, d = threadIdx.x;
    const unsigned long long c = hist[p * RS_BINS + d];
    s[d] = c;
    __syncthreads();
    for (int off = 1; off < RS_BINS; off <<= 1) {      // inclusive Hillis-Steele
        const unsigned long long v = d >= off ? s[d - off] : 0ull;
        __syncthreads();
        s[d] += v;
        __syncthreads();
    }
    base[p * RS_BINS + d] = s[d] - c;
    if (c == (unsigned long long)n) skip[p] = 1;
}

// the lanes of the warp holding the same 8-bit digit (d < 256; lanes with
// d = 256 -- out of range -- never match a real digit): 8 ballots
__device__ __forceinline__ unsigned digit_peers(int d, bool valid) {
    unsigned m = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < 8; b++) {
        const unsigned bb = __ballot_sync(0xffffffffu, (d >> b) & 1);
        m &= ((d >> b) & 1) ? bb : ~bb;
    }
    return valid ? m : 0u;
}

// per-tile digit counts, bin-major: counts[d * tiles + tile]
__global__ void __launch_bounds__(256) k_rs_upsweep(const uint64_t *__restrict__ kin, int64_t n,
                                                    int shift, int64_t tiles,
                                                    unsigned int *counts) {
    __shared__ unsigned int sh[RS_BINS];
    const int t = threadIdx.x;
    sh[t] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * RS_TILE;
#pragma unroll 4
    for (int i = 0; i < RS_TILE / 256; i++) {
        const int64_t idx = base + i * 256 + t;
        const bool in = idx < n;
        const int d = in ? (int)((kin[idx] >> shift) & 255) : 0;
        const unsigned peers = digit_peers(d, in);
        if (in && (t & 31) == __ffs(peers) - 1) atomicAdd(&sh[d], __popc(peers));
    }
    __syncthreads();
    counts[(int64_t)t * tiles + blockIdx.x] = sh[t];
}

// one block per digit: exclusive scan of its tile counts + the digit's base
__global__ void __launch_bounds__(1024) k_rs_offsets(unsigned int *counts, int64_t tiles,
                                                     const unsigned long long *bin_base,
                                                     unsigned long long *offsets) {
    __shared__ unsigned long long wsum[32];
    __shared__ unsigned long long carry;
    const int d = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    if (t == 0) carry = bin_base[d];
    __syncthreads();
    for (int64_t c0 = 0; c0 < tiles; c0 += 1024) {
        const int64_t i = c0 + t;
        const unsigned long long c = i < tiles ? counts[(int64_t)d * tiles + i] : 0ull;
        unsigned long long v = c;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane == 31) wsum[warp] = v;
        __syncthreads();
        if (warp == 0) {
            unsigned long long w = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            wsum[lane] = w;                       // inclusive over warps
        }
        __syncthreads();
        const unsigned long long before = (warp ? wsum[warp - 1] : 0ull) + v - c;
        if (i < tiles) offsets[(int64_t)d * tiles + i] = carry + before;
        __syncthreads();
        if (t == 1023) carry += before + c;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(RS_THREADS, 3) k_rs_downsweep(
    const uint64_t *__restrict__ kin, const int32_t *__restrict__ vin, uint64_t *kout,
    int32_t *vout, int64_t n, int shift, int64_t tiles,
    const unsigned long long *__restrict__ offsets) {
    __shared__ unsigned int wcnt[RS_WARPS][RS_BINS];   // per-warp digit counters -> prefixes
    __shared__ unsigned int lofs[RS_BINS];              // tile-local start of each digit
    __shared__ unsigned long long gofs[RS_BINS];        // global start of each digit's run
    __shared__ unsigned wtot[RS_BINS / 32];
    extern __shared__ __align__(16) unsigned char rs_smem[];   // the tile, reordered
    uint64_t *skey = (uint64_t *)rs_smem;
    int32_t *sval = (int32_t *)(skey + RS_TILE);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < RS_WARPS * RS_BINS; i += RS_THREADS) (&wcnt[0][0])[i] = 0;
    const int64_t tile = blockIdx.x;
    const int64_t base = tile * RS_TILE;
    if (t < RS_BINS) gofs[t] = offsets[(int64_t)t * tiles + tile];
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
    // ---- load (warp-striped: warp w owns [base + 512 w, +512)) and rank
    uint64_t key[RS_ITEMS];
    int32_t val[RS_ITEMS];
    unsigned short rank[RS_ITEMS];
    const int64_t wbase = base + warp * (RS_ITEMS * 32) + lane;
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++) {
        const int64_t idx = wbase + i * 32;
        const bool in = idx < n;
        key[i] = in ? kin[idx] : 0ull;
        val[i] = in ? vin[idx] : 0;
    }
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++) {
        const bool in = wbase + i * 32 < n;
        const int d = in ? (int)((key[i] >> shift) & 255) : RS_BINS;
        const unsigned peers = digit_peers(d & 255, in);
        unsigned before = 0;
        if (d < RS_BINS) before = wcnt[warp][d];
        __syncwarp();
        if (d < RS_BINS && lane == __ffs(peers) - 1) wcnt[warp][d] = before + __popc(peers);
        __syncwarp();
        rank[i] = (unsigned short)(before + __popc(peers & lt));
    }
    __syncthreads();
    // ---- per digit: warp prefixes, tile-local digit starts
    if (t < RS_BINS) {
        unsigned cnt = 0;
#pragma unroll
        for (int w = 0; w < RS_WARPS; w++) {
            const unsigned c = wcnt[w][t];
            wcnt[w][t] = cnt;
            cnt += c;
        }
        unsigned v = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += y;
        }
        if (lane == 31) wtot[warp] = v;
        lofs[t] = v - cnt;
    }
    __syncthreads();
    if (t < RS_BINS) {
        unsigned add = 0;
        for (int w = 0; w < warp; w++) add += wtot[w];
        lofs[t] += add;
    }
    __syncthreads();
    // ---- reorder the tile by digit in shared memory (stable)
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++) {
        if (wbase + i * 32 < n) {
            const int d = (int)((key[i] >> shift) & 255);
            const unsigned pos = lofs[d] + wcnt[warp][d] + rank[i];
            skey[pos] = key[i];
            sval[pos] = val[i];
        }
    }
    __syncthreads();
    const int tile_n = (int)(n - base < RS_TILE ? n - base : RS_TILE);
    for (int j = t; j < tile_n; j += RS_THREADS) {
        const uint64_t k = skey[j];
        const int d = (int)((k >> shift) & 255);
        const unsigned long long pos = gofs[d] + (unsigned long long)(j - (int)lofs[d]);
        KB_DCHECK(pos < (unsigned long long)n);
        kout[pos] = k;
        vout[pos] = sval[j];
    }
}

}  // namespace

// Sorts n pairs stably by key.  (k0, v0) hold the input; (k1, v1) are
// scratch of the same size.  Returns true if the result is in (k1, v1),
// false if it is in (k0, v0).
bool radix_sort_pairs(uint64_t *k0, int32_t *v0, uint64_t *k1, int32_t *v1, int64_t n,
                      int device, cudaStream_t st) {
    if (n <= 1) return false;
    KB_REQUIRE(n < ((int64_t)1 << 31), KB_EPARAM, "radix sort supports < 2^31 keys");
    const int64_t tiles = (n + RS_TILE - 1) / RS_TILE;
    DBuf<unsigned long long> hist;                 // [0, 2048) histograms, [2048, 4096) bases
    DBuf<int> skip;
    DBuf<unsigned int> counts;
    DBuf<unsigned long long> offsets;
    hist.alloc(2 * 8 * RS_BINS);
    skip.alloc(8);
    counts.alloc((size_t)tiles * RS_BINS);
    offsets.alloc((size_t)tiles * RS_BINS);
    KB_CUDA(cudaMemsetAsync(hist.p, 0, 8 * RS_BINS * sizeof(unsigned long long), st));
    KB_CUDA(cudaMemsetAsync(skip.p, 0, 8 * sizeof(int), st));
    int sms = 0;
    KB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    constexpr size_t tile_smem = (size_t)RS_TILE * (sizeof(uint64_t) + sizeof(int32_t));
    static bool attr_done[64] = {};
    if (!attr_done[device]) {
        KB_CUDA(cudaFuncSetAttribute(k_rs_downsweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)tile_smem));
        attr_done[device] = true;
    }
    k_rs_hist<<<(unsigned)std::min<int64_t>(4 * sms, nblk(n, 256)), 256, 0, st>>>(k0, n, hist.p);
    k_rs_scan<<<8, RS_BINS, 0, st>>>(hist.p, n, hist.p + 8 * RS_BINS, skip.p);
    note_launch(2);
    int h_skip[8];
    KB_CUDA(cudaMemcpyAsync(h_skip, skip.p, sizeof(h_skip), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    uint64_t *ka = k0, *kb = k1;
    int32_t *va = v0, *vb = v1;
    bool in1 = false;
    for (int p = 0; p < 8; p++) {
        if (h_skip[p]) continue;
        const int shift = 8 * p;
        k_rs_upsweep<<<(unsigned)tiles, 256, 0, st>>>(ka, n, shift, tiles, counts.p);
        k_rs_offsets<<<RS_BINS, 1024, 0, st>>>(counts.p, tiles, hist.p + 8 * RS_BINS + p * RS_BINS,
                                               offsets.p);
        k_rs_downsweep<<<(unsigned)tiles, RS_THREADS, tile_smem, st>>>(ka, va, kb, vb, n, shift,
                                                                        tiles, offsets.p);
        note_launch(3);
        std::swap(ka, kb);
        std::swap(va, vb);
        in1 = !in1;
    }
    KB_CUDA(cudaGetLastError());
    return in1;
}

}  // namespace kb
