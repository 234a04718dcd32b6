// Ranking agreement for the compare command:
// concordant_fraction(order_a, order_b) = 1 - inversions(pos_a[order_b]) /
// (n(n-1)/2)  (cli.py:349-360; the reference counts inversions with a
// pure-Python merge sort, cli.py:363-386).
//
// Device algorithm: seq is a permutation of 0..n-1.  An inverted pair
// (i < j, seq[i] > seq[j]) is decided by the highest bit k where the two
// values differ: seq[i] has a 1 there, seq[j] a 0, and they agree above k.
// So, MSB first, keep seq stably sorted by the bits above k; inside each
// group of equal upper bits count, for every element with bit k = 0, the
// elements with bit k = 1 before it; then stably split each group by bit k.
// Because seq is a permutation, the group of upper-prefix p spans exactly
// positions [p*2^(k+1), min(n, (p+1)*2^(k+1))) and holds min(n, start+2^k)
// - start zeros, so one exclusive scan of the bit per level is all the
// bookkeeping: ceil(log2 n) levels of scan + scatter, O(n log n) work,
// exact 64-bit integer count.
#include "kb_internal.cuh"

#include <cub/cub.cuh>

namespace kb {

namespace {

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

__global__ void k_perm_check(const int64_t *ord, int64_t n, int32_t *pos,
                             unsigned long long *bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t v = ord[i];
    if (v < 0 || v >= n) {
        atomicOr(bad, 1ull);
        return;
    }
    pos[v] = (int32_t)i;  // duplicates leave some slot unwritten (-1): caught below
}

__global__ void k_seq(const int64_t *ord_b, const int32_t *pos_a, int64_t n, int32_t *seq,
                      unsigned long long *bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t v = ord_b[i];
    if (v < 0 || v >= n) {
        atomicOr(bad, 1ull);
        return;
    }
    const int32_t p = pos_a[v];
    if (p < 0) atomicOr(bad, 1ull);
    seq[i] = p;
}

__global__ void k_mark_seen(const int32_t *seq, int64_t n, int32_t *seen) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && seq[i] >= 0) seen[seq[i]] = 1;
}

__global__ void k_count_unseen(const int32_t *seen, int64_t n, unsigned long long *bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n && !seen[i]) atomicOr(bad, 1ull);
}

struct BitOf {
    const int32_t *seq;
    int k;
    __device__ int32_t operator()(int64_t i) const { return (seq[i] >> k) & 1; }
};

__global__ void k_split_level(const int32_t *__restrict__ seq, const int32_t *__restrict__ ones,
                              int64_t n, int k, int32_t *__restrict__ out,
                              unsigned long long *inv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long c = 0;
    if (i < n) {
        const int32_t x = seq[i];
        const int64_t span = 1ll << (k + 1);
        const int64_t gs = (i / span) * span;                  // group start
        const int64_t ones_before = (int64_t)ones[i] - (int64_t)ones[gs];
        const int64_t half_end = gs + (span >> 1);
        const int64_t zeros = (half_end < n ? half_end : n) - gs;
        int64_t dst;
        if ((x >> k) & 1) {
            dst = gs + zeros + ones_before;
        } else {
            dst = gs + (i - gs - ones_before);
            c = (unsigned long long)ones_before;                 // 1s before this 0
        }
        out[dst] = x;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(inv, c);
}

}  // namespace

int64_t count_inversions(const int64_t *h_order_a, const int64_t *h_order_b, int64_t n) {
    cudaStream_t st = device_stream();
    if (n < 2) return 0;
    KB_REQUIRE(n < (1ll << 31) - 1, KB_EPARAM, "rankings longer than 2^31 - 1");
    DBuf<int64_t> a, b;
    DBuf<int32_t> pos, seq, tmp, ones, seen;
    DBuf<unsigned long long> flags;
    a.alloc(n); b.alloc(n); pos.alloc(n); seq.alloc(n); tmp.alloc(n); ones.alloc(n + 1);
    seen.alloc(n); flags.alloc(2);
    KB_CUDA(cudaMemcpyAsync(a.p, h_order_a, n * 8, cudaMemcpyHostToDevice, st));
    KB_CUDA(cudaMemcpyAsync(b.p, h_order_b, n * 8, cudaMemcpyHostToDevice, st));
    KB_CUDA(cudaMemsetAsync(flags.p, 0, 16, st));
    KB_CUDA(cudaMemsetAsync(pos.p, 0xff, n * 4, st));
    KB_CUDA(cudaMemsetAsync(seen.p, 0, n * 4, st));
    k_perm_check<<<nblk(n, 256), 256, 0, st>>>(a.p, n, pos.p, flags.p);
    k_seq<<<nblk(n, 256), 256, 0, st>>>(b.p, pos.p, n, seq.p, flags.p);
    k_mark_seen<<<nblk(n, 256), 256, 0, st>>>(seq.p, n, seen.p);
    k_count_unseen<<<nblk(n, 256), 256, 0, st>>>(seen.p, n, flags.p);
    note_launch(4);
    unsigned long long hb = 0;
    KB_CUDA(cudaMemcpyAsync(&hb, flags.p, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    KB_REQUIRE(!hb, KB_EPARAM, "orders must be permutations of 0..n-1");
    int L = 0;
    while ((1ll << L) < n) L++;
    size_t tb = 0;
    {
        cub::CountingInputIterator<int64_t> it(0);
        cub::TransformInputIterator<int32_t, BitOf, cub::CountingInputIterator<int64_t>> bits(
            it, BitOf{seq.p, 0});
        KB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, bits, ones.p, (int)n, st));
    }
    DBuf<unsigned char> cubtmp;
    cubtmp.alloc(tb);
    for (int k = L - 1; k >= 0; k--) {
        cub::CountingInputIterator<int64_t> it(0);
        cub::TransformInputIterator<int32_t, BitOf, cub::CountingInputIterator<int64_t>> bits(
            it, BitOf{seq.p, k});
        KB_CUDA(cub::DeviceScan::ExclusiveSum(cubtmp.p, tb, bits, ones.p, (int)n, st));
        k_split_level<<<nblk(n, 256), 256, 0, st>>>(seq.p, ones.p, n, k, tmp.p, flags.p + 1);
        note_launch(2);
        std::swap(seq, tmp);
    }
    unsigned long long inv = 0;
    KB_CUDA(cudaMemcpyAsync(&inv, flags.p + 1, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    return (int64_t)inv;
}

}  // namespace kb
