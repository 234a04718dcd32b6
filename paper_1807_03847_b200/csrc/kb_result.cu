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
                            int64_t npos, uint64_t *keys) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= npos) return;
    keys[i] = ~(uint64_t)__double_as_longlong(lower[iperm[ids[i]]]);
}

// count_v = #{i < npos : sorted_desc[i] > upper[v]} where sorted_desc holds
// ~keys.  Every 1024th key is staged in shared memory, so the search touches
// global memory only inside one 1024-key window.  Nodes with upper == 0
// (no out-arcs) count every positive lower bound without a search.
constexpr int SEP_SAMPLES = 12288;  // 96 KB of shared memory

__global__ void __launch_bounds__(512) k_sep_pairs(const uint64_t *skeys, int64_t npos,
                                                   const double *upper, int64_t n,
                                                   int64_t SEP_STRIDE,
                                                   unsigned long long *total) {
    extern __shared__ double samp[];
    const int64_t ns = (npos + SEP_STRIDE - 1) / SEP_STRIDE;
    for (int64_t t = threadIdx.x; t < ns; t += blockDim.x)
        samp[t] = __longlong_as_double((long long)~skeys[t * SEP_STRIDE]);
    __syncthreads();
    typedef cub::BlockReduce<unsigned long long, 512> Red;
    __shared__ typename Red::TempStorage tmp;
    unsigned long long acc = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
         v += (int64_t)gridDim.x * blockDim.x) {
        const double u = upper[v];
        if (u == 0.0) { acc += (unsigned long long)npos; continue; }
        // sample level: first sample index t with samp[t] <= u
        int64_t lo = 0, hi = ns;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (samp[mid] > u) lo = mid + 1; else hi = mid;
        }
        // answer lies in ((lo-1)*S, lo*S]
        int64_t a = lo == 0 ? 0 : (lo - 1) * SEP_STRIDE + 1;
        int64_t b = lo * SEP_STRIDE < npos ? lo * SEP_STRIDE : npos;
        while (a < b) {
            const int64_t mid = (a + b) >> 1;
            const double val = __longlong_as_double((long long)~skeys[mid]);
            if (val > u) a = mid + 1; else b = mid;
        }
        acc += (unsigned long long)a;
    }
    acc = Red(tmp).Sum(acc);
    if (threadIdx.x == 0 && acc) atomicAdd(total, acc);
}

__global__ void k_widen(const int32_t *src, int64_t n, int64_t *dst) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i];
}

}  // namespace

void run_result(State &s, cudaStream_t st, int64_t *h_order, double *h_lower, double *h_upper,
                int64_t *h_pairs) {
    Graph &g = *s.g;
    const int64_t n = g.n;
    KB_REQUIRE(s.r >= 1, KB_ESTATE, "separated_fraction needs at least one iteration");
    DBuf<unsigned char> fpos, fzero;
    DBuf<int32_t> iota, ids, order;
    DBuf<uint64_t> kin, kout;
    fpos.alloc(n); fzero.alloc(n); iota.alloc(n); ids.alloc(n); order.alloc(n);
    unsigned long long *u = s.scratch_u64.p;  // [0]=npos, [1]=nzero, [2]=pairs
    KB_CUDA(cudaMemsetAsync(u, 0, 3 * sizeof(unsigned long long), st));
    k_pos_flags<<<nblk(n, 256), 256, 0, st>>>(s.lower.p, g.iperm.p, n, fpos.p, fzero.p, iota.p); note_launch();
    size_t tb = 0;
    KB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, fpos.p, ids.p, u, (int)n, st));
    ensure_cub_tmp(s, tb);
    KB_CUDA(cub::DeviceSelect::Flagged(s.cub_tmp.p, tb, iota.p, fpos.p, ids.p, u, (int)n, st)); note_launch();
    unsigned long long hcnt[1];
    KB_CUDA(cudaMemcpyAsync(hcnt, u, sizeof(hcnt), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    const int64_t npos = (int64_t)hcnt[0];
    // zero-bound nodes go last, in id order
    tb = 0;
    KB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, fzero.p, order.p + npos, u + 1,
                                       (int)n, st));
    ensure_cub_tmp(s, tb);
    KB_CUDA(cub::DeviceSelect::Flagged(s.cub_tmp.p, tb, iota.p, fzero.p, order.p + npos, u + 1,
                                       (int)n, st)); note_launch();
    kin.alloc(npos); kout.alloc(npos);
    if (npos) {
        k_sort_keys<<<nblk(npos, 256), 256, 0, st>>>(s.lower.p, g.iperm.p, ids.p, npos, kin.p); note_launch();
        tb = 0;
        KB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.p, kout.p, ids.p, order.p,
                                                (int)npos, 0, 64, st));
        ensure_cub_tmp(s, tb);
        KB_CUDA(cub::DeviceRadixSort::SortPairs(s.cub_tmp.p, tb, kin.p, kout.p, ids.p, order.p,
                                                (int)npos, 0, 64, st)); note_launch();
    }
    if (n >= 2) {
        int64_t stride = 1024;
        while ((npos + stride - 1) / stride > SEP_SAMPLES) stride *= 2;
        const size_t smem = SEP_SAMPLES * sizeof(double);
        KB_CUDA(cudaFuncSetAttribute(k_sep_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        k_sep_pairs<<<2 * g.sm_count, 512, smem, st>>>(kout.p, npos, s.upper.p, n, stride, u + 2);
        note_launch();
    }
    if (h_order) {
        DBuf<int64_t> wide;
        wide.alloc(n);
        k_widen<<<nblk(n, 256), 256, 0, st>>>(order.p, n, wide.p); note_launch();
        KB_CUDA(cudaMemcpyAsync(h_order, wide.p, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
    }
    if (h_lower || h_upper) {
        DBuf<double> tmpv;
        tmpv.alloc(n);
        if (h_lower) {
            gather_to_original(g, s.lower.p, tmpv.p, st);
            KB_CUDA(cudaMemcpyAsync(h_lower, tmpv.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
            KB_CUDA(cudaStreamSynchronize(st));
        }
        if (h_upper) {
            gather_to_original(g, s.upper.p, tmpv.p, st);
            KB_CUDA(cudaMemcpyAsync(h_upper, tmpv.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
            KB_CUDA(cudaStreamSynchronize(st));
        }
    }
    unsigned long long pairs = 0;
    KB_CUDA(cudaMemcpyAsync(&pairs, u + 2, sizeof(pairs), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    if (h_pairs) *h_pairs = (int64_t)pairs;
}

}  // namespace kb
