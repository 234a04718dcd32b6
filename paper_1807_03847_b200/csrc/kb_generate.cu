// Device graph generators: bit-identical replicas of katzbounds.generate
// (generate.py:38-103), so benchmark inputs at scale 24..27 are produced in
// milliseconds on the GPU instead of hours of numpy.
//
// R-MAT (generate.py:55-81): numpy's Generator(PCG64) stream -- 128-bit LCG
// s' = s*M + inc, output XSL-RR of the new state, random() = (raw>>11)*2^-53.
// Draw (bit b, pair e) is raw number b*m + e of the stream; thread e jumps to
// s_e with the LCG advance and then hops by m per bit with a precomputed
// affine jump, so every thread is independent and exact.  Then
// lo=min,hi=max, drop loops, sort+unique lo*n+hi (np.unique), and build the
// canonical symmetric CSR (Graph.from_edges(..., undirected=True) +
// out_csr, graph.py:101-116, :177-197) with rows ascending.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>

#include "kb_internal.cuh"

namespace kb {

namespace {

typedef unsigned __int128 u128;

__host__ __device__ inline u128 mk(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

__host__ __device__ inline u128 pcg_mult() {
    return mk(2549297995355413924ULL, 4865540595714422341ULL);
}

__host__ __device__ inline uint64_t pcg_out(u128 s) {
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

// affine map of `delta` LCG steps: s -> A*s + C
__host__ __device__ inline void pcg_jump(u128 delta, u128 inc, u128 &A, u128 &C) {
    u128 am = 1, ap = 0, cm = pcg_mult(), cp = inc;
    while (delta > 0) {
        if (delta & 1) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        delta >>= 1;
    }
    A = am;
    C = ap;
}

struct RmatArgs {
    uint64_t s_hi, s_lo, inc_hi, inc_lo;
    uint64_t jm_a_hi, jm_a_lo, jm_c_hi, jm_c_lo;  // jump by m
    int scale;
    int64_t m;
    double a, ab, abc;
    uint64_t *packed;
};

__global__ void k_rmat_pairs(RmatArgs R) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= R.m) return;
    const u128 inc = mk(R.inc_hi, R.inc_lo);
    u128 A, C;
    pcg_jump((u128)e, inc, A, C);
    u128 s = A * mk(R.s_hi, R.s_lo) + C;  // state after e steps
    const u128 JA = mk(R.jm_a_hi, R.jm_a_lo), JC = mk(R.jm_c_hi, R.jm_c_lo);
    const u128 M = pcg_mult();
    uint64_t src = 0, dst = 0;
    for (int b = 0; b < R.scale; b++) {
        const u128 t = s * M + inc;  // the draw's state: b*m + e + 1 steps
        const double draw = (double)(pcg_out(t) >> 11) * (1.0 / 9007199254740992.0);
        const uint64_t sb = draw >= R.ab;
        const uint64_t db = ((draw >= R.a) & (draw < R.ab)) | (draw >= R.abc);
        src = (src << 1) | sb;
        dst = (dst << 1) | db;
        s = JA * s + JC;  // advance m steps to bit b+1
    }
    const uint64_t lo = src < dst ? src : dst, hi = src < dst ? dst : src;
    R.packed[e] = (lo != hi) ? ((lo << R.scale) | hi) : ~0ull;
}

__global__ void k_row_starts(const uint64_t *keys, int64_t ne, int64_t n, int scale,
                             int64_t *start) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v > n) return;
    const uint64_t target = (uint64_t)v << scale;
    int64_t lo = 0, hi = ne;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    start[v] = lo;
}

__global__ void k_swap_key(const uint64_t *in, int64_t ne, int scale, uint64_t *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ne) return;
    const uint64_t mask = (1ull << scale) - 1;
    const uint64_t k = in[i];
    out[i] = ((k & mask) << scale) | (k >> scale);
}

__global__ void k_csr_degree(const int64_t *sa, const int64_t *sb, int64_t n, int64_t *deg) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    deg[v] = (sa[v + 1] - sa[v]) + (sb[v + 1] - sb[v]);
}

// row v = [lo-neighbours from the (hi,lo)-sorted list] ++ [hi-neighbours from
// the (lo,hi)-sorted list] -- ascending overall
__global__ void k_csr_fill_a(const uint64_t *keys_a, int64_t ne, int scale, const int64_t *sa,
                             const int64_t *sb, const int64_t *indptr, int32_t *indices) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= ne) return;
    const uint64_t mask = (1ull << scale) - 1;
    const int64_t lo = (int64_t)(keys_a[i] >> scale), hi = (int64_t)(keys_a[i] & mask);
    indices[indptr[lo] + (sb[lo + 1] - sb[lo]) + (i - sa[lo])] = (int32_t)hi;
}

__global__ void k_csr_fill_b(const uint64_t *keys_b, int64_t ne, int scale, const int64_t *sb,
                             const int64_t *indptr, int32_t *indices) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= ne) return;
    const uint64_t mask = (1ull << scale) - 1;
    const int64_t hi = (int64_t)(keys_b[j] >> scale), lo = (int64_t)(keys_b[j] & mask);
    indices[indptr[hi] + (j - sb[hi])] = (int32_t)lo;
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

template <typename F>
void cub_call(F &&f, cudaStream_t st) {
    size_t tb = 0;
    KB_CUDA(f(nullptr, tb));
    DBuf<unsigned char> tmp;
    tmp.alloc(tb);
    KB_CUDA(f(tmp.p, tb));
    (void)st;
}

}  // namespace

// Generates the canonical symmetric CSR of generate("rmat", 2^scale, seed,
// edge_factor) loaded undirected, into device buffers indptr/indices.
void rmat_device_csr(int scale, int64_t edge_factor, const uint64_t state[4], double a,
                     double ab, double abc, DBuf<int64_t> &indptr, DBuf<int32_t> &indices,
                     int64_t &nnz_out) {
    cudaStream_t st = device_stream();
    KB_REQUIRE(scale >= 1 && scale <= 30, KB_EPARAM, "rmat scale must be in [1, 30]");
    const int64_t n = (int64_t)1 << scale;
    const int64_t m = n * edge_factor;
    KB_REQUIRE(m <= ((int64_t)1 << 33), KB_EPARAM, "rmat: n*edge_factor too large");
    const u128 inc = mk(state[2], state[3]);
    u128 JA, JC;
    pcg_jump((u128)m, inc, JA, JC);
    RmatArgs R;
    R.s_hi = state[0]; R.s_lo = state[1]; R.inc_hi = state[2]; R.inc_lo = state[3];
    R.jm_a_hi = (uint64_t)(JA >> 64); R.jm_a_lo = (uint64_t)JA;
    R.jm_c_hi = (uint64_t)(JC >> 64); R.jm_c_lo = (uint64_t)JC;
    R.scale = scale; R.m = m; R.a = a; R.ab = ab; R.abc = abc;
    DBuf<uint64_t> keys, keys2;
    keys.alloc(m);
    keys2.alloc(m);
    R.packed = keys.p;
    k_rmat_pairs<<<nblk(m, 256), 256, 0, st>>>(R); note_launch();
    KB_CUDA(cudaGetLastError());
    // valid keys are < n*n - 1; the loop sentinel ~0 has all low 2*scale bits
    // set, so sorting only those bits still puts it last
    cub_call([&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortKeys(t, b, keys.p, keys2.p, m, 0, 2 * scale, st);
    }, st);
    DBuf<int64_t> cnt;
    cnt.alloc(1);
    cub_call([&](void *t, size_t &b) {
        return cub::DeviceSelect::Unique(t, b, keys2.p, keys.p, cnt.p, m, st);
    }, st);
    int64_t nu = 0;
    KB_CUDA(cudaMemcpyAsync(&nu, cnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    // drop the loop sentinel (sorted last) if present
    uint64_t last = 0;
    if (nu) {
        KB_CUDA(cudaMemcpyAsync(&last, keys.p + nu - 1, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        if (last == ~0ull) nu--;
    }
    const int64_t ne = nu;
    // list A = keys.p[0..ne) sorted by (lo,hi); list B sorted by (hi,lo)
    k_swap_key<<<nblk(ne, 256), 256, 0, st>>>(keys.p, ne, scale, keys2.p); note_launch();
    DBuf<uint64_t> keys_b;
    keys_b.alloc(ne);
    cub_call([&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortKeys(t, b, keys2.p, keys_b.p, ne, 0, 2 * scale, st);
    }, st);
    keys2.release();
    DBuf<int64_t> sa, sb, deg;
    sa.alloc(n + 1); sb.alloc(n + 1); deg.alloc(n + 1);
    k_row_starts<<<nblk(n + 1, 256), 256, 0, st>>>(keys.p, ne, n, scale, sa.p); note_launch();
    k_row_starts<<<nblk(n + 1, 256), 256, 0, st>>>(keys_b.p, ne, n, scale, sb.p); note_launch();
    k_csr_degree<<<nblk(n, 256), 256, 0, st>>>(sa.p, sb.p, n, deg.p); note_launch();
    KB_CUDA(cudaMemsetAsync(deg.p + n, 0, sizeof(int64_t), st));
    indptr.alloc(n + 1);
    cub_call([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, deg.p, indptr.p, (int)(n + 1), st);
    }, st);
    nnz_out = 2 * ne;
    indices.alloc(nnz_out);
    k_csr_fill_a<<<nblk(ne, 256), 256, 0, st>>>(keys.p, ne, scale, sa.p, sb.p, indptr.p,
                                                 indices.p); note_launch();
    k_csr_fill_b<<<nblk(ne, 256), 256, 0, st>>>(keys_b.p, ne, scale, sb.p, indptr.p, indices.p); note_launch();
    KB_CUDA(cudaGetLastError());
    KB_CUDA(cudaStreamSynchronize(st));
}

// grid_edges (generate.py:38-52) loaded undirected: row-major ids, floor(sqrt
// n) columns, right and down neighbours; row v ascending = up, left, right, down
namespace {
__global__ void k_grid_deg(int64_t n, int64_t cols, int64_t *deg) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t d = 0;
    if (i - cols >= 0) d++;                                         // up: (i-cols, i)
    if (i >= 1 && (i % cols) != 0) d++;                             // left: (i-1, i)
    if ((i + 1) % cols != 0 && i + 1 < n) d++;                      // right
    if (i + cols < n) d++;                                          // down
    deg[i] = d;
}
__global__ void k_grid_fill(int64_t n, int64_t cols, const int64_t *indptr, int32_t *idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t p = indptr[i];
    if (i - cols >= 0) idx[p++] = (int32_t)(i - cols);
    if (i >= 1 && (i % cols) != 0) idx[p++] = (int32_t)(i - 1);
    if ((i + 1) % cols != 0 && i + 1 < n) idx[p++] = (int32_t)(i + 1);
    if (i + cols < n) idx[p++] = (int32_t)(i + cols);
}
}  // namespace

void grid_device_csr(int64_t n, DBuf<int64_t> &indptr, DBuf<int32_t> &indices,
                     int64_t &nnz_out) {
    cudaStream_t st = device_stream();
    int64_t cols = 1;
    while ((cols + 1) * (cols + 1) <= n) cols++;  // math.isqrt, >= 1
    DBuf<int64_t> deg;
    deg.alloc(n + 1);
    k_grid_deg<<<nblk(n, 256), 256, 0, st>>>(n, cols, deg.p); note_launch();
    KB_CUDA(cudaMemsetAsync(deg.p + n, 0, sizeof(int64_t), st));
    indptr.alloc(n + 1);
    cub_call([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, deg.p, indptr.p, (int)(n + 1), st);
    }, st);
    KB_CUDA(cudaMemcpyAsync(&nnz_out, indptr.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    indices.alloc(nnz_out);
    k_grid_fill<<<nblk(n, 256), 256, 0, st>>>(n, cols, indptr.p, indices.p); note_launch();
    KB_CUDA(cudaGetLastError());
    KB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace kb
