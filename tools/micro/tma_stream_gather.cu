// Microbenchmark: does moving K1's column-id stream from LDG to TMA bulk
// copies free L1->XBAR request bandwidth for the omega gathers?
//
// Both kernels read the same int32 index stream (K1's column slots) and
// gather x[idx] (8-byte, random over a 134 MB vector like C2's omega):
//   mode 0: warps load their indices with 128-bit LDG (L1::no_allocate),
//   mode 1: one producer thread per CTA bulk-copies index chunks into a
//           3-stage shared-memory ring (mbarrier complete_tx) and 31
//           consumer warps read indices from shared memory.
// Prints the time per launch and gathers per SM-cycle.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int CHUNK = 8192;                // indices per stage (32 KB)
constexpr int ST = 3;

__global__ void k_ldg(const int32_t *__restrict__ idx, int64_t m, const double *__restrict__ x,
                      double *out) {
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    double acc = 0.0;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < m;
         i += nthreads * 4) {
        int4 c;
        asm("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
            : "=r"(c.x), "=r"(c.y), "=r"(c.z), "=r"(c.w) : "l"(idx + i));
        acc += __ldg(x + c.x) + __ldg(x + c.y) + __ldg(x + c.z) + __ldg(x + c.w);
    }
    if (acc == 12345.0) out[0] = acc;
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    unsigned done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                     "  selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(bar), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(1024, 1) k_tma(const int32_t *__restrict__ idx, int64_t m,
                                                 const double *__restrict__ x, double *out) {
    extern __shared__ int4 sm4[];
    int32_t *ring = (int32_t *)sm4;
    __shared__ __align__(8) unsigned long long full[ST], empty[ST];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ncw = (blockDim.x >> 5) - 1;
    const unsigned fbar = (unsigned)__cvta_generic_to_shared(full);
    const unsigned ebar = (unsigned)__cvta_generic_to_shared(empty);
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(ring);
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; i++) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(fbar + 8 * i));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(ebar + 8 * i), "r"(ncw));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t nchunks = m / CHUNK, G = gridDim.x;
    const int64_t nmine = nchunks > blockIdx.x ? (nchunks - 1 - blockIdx.x) / G + 1 : 0;
    double acc = 0.0;
    if (warp == 0) {
        if (lane == 0)
            for (int64_t k = 0; k < nmine; k++) {
                const int s = (int)(k % ST);
                const unsigned r = (unsigned)(k / ST);
                mbar_wait(ebar + 8 * s, (r & 1) ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                             ::"r"(fbar + 8 * s), "r"(CHUNK * 4) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
                             "[%0], [%1], %2, [%3];"
                             ::"r"(sbase + s * CHUNK * 4),
                               "l"(idx + (blockIdx.x + k * G) * CHUNK), "r"(CHUNK * 4),
                               "r"(fbar + 8 * s) : "memory");
            }
    } else {
        const int cw = warp - 1;
        for (int64_t k = 0; k < nmine; k++) {
            const int s = (int)(k % ST);
            const unsigned r = (unsigned)(k / ST);
            mbar_wait(fbar + 8 * s, r & 1);
            const int32_t *c = ring + s * CHUNK;
            // this warp's share: CHUNK / 31 rounded, 8 indices per lane per step
            int32_t v[8];
            const int per = (CHUNK + ncw - 1) / ncw;
            const int a = cw * per, b = min(CHUNK, a + per);
            double part = 0.0;
            for (int base = a; base < b; base += 256) {
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const int j = base + q * 32 + lane;
                    v[q] = j < b ? c[j] : -1;
                }
                __syncwarp();
#pragma unroll
                for (int q = 0; q < 8; q++) part += v[q] >= 0 ? __ldg(x + v[q]) : 0.0;
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"
                                        ::"r"(ebar + 8 * s) : "memory");
            acc += part;
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

int main(int argc, char **argv) {
    // omega size: 2^24 doubles (C2's 134 MB) by default; smaller sizes keep
    // the gathers L2-resident like C2's skewed columns (74% L2 hits)
    const int64_t n = (int64_t)1 << (argc > 1 ? atoi(argv[1]) : 24);
    const int64_t m = (int64_t)CHUNK * 148 * 200;   // ~242M gathers
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::vector<int32_t> h(m);
    uint64_t s = 88172645463325252ull;
    for (int64_t i = 0; i < m; i++) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        h[i] = (int32_t)(s % (uint64_t)n);
    }
    int32_t *idx; double *x, *out;
    CK(cudaMalloc(&idx, m * 4)); CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&out, 8));
    CK(cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(x, 0, n * 8));
    const size_t smem = (size_t)ST * CHUNK * 4;
    CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    int clk = 0;
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    for (int mode = 0; mode < 2; mode++) {
        float best = 1e9f;
        for (int rep = 0; rep < 6; rep++) {
            CK(cudaEventRecord(e0));
            if (mode == 0) k_ldg<<<sms * 2, 1024>>>(idx, m, x, out);
            else k_tma<<<sms, 1024, smem>>>(idx, m, x, out);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rep) best = ms < best ? ms : best;
        }
        CK(cudaGetLastError());
        const double cyc = best * 1e-3 * clk * 1e3 * sms;
        printf("omega 2^%d doubles, mode %s: %.3f ms for %.0fM gathers, %.3f gathers per "
               "SM-cycle\n", argc > 1 ? atoi(argv[1]) : 24, mode ? "tma-stream" : "ldg-stream",
               best, m / 1e6, m / cyc);
    }
    return 0;
}
