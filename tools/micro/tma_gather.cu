// Random 8-byte gathers from a 128 MiB vector: LDG (one lane per element,
// the K1 path) against TMA tile::gather4 (one instruction fetches four
// 16-byte rows into shared memory).  Question: does the TMA engine sustain
// more random rows per SM-cycle than the L1/TEX wavefront queue (~1/cycle)?
//
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -o tma_gather tma_gather.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                            \
        }                                                                       \
    } while (0)

__global__ void k_ldg(const double *__restrict__ x, const int32_t *__restrict__ idx, int64_t m,
                      double *out) {
    double s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        s += x[idx[i]];
    if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(tx)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int r0, int r1, int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}

constexpr int G = 32;        // gather4 ops per stage (128 rows, 2 KiB)
constexpr int S = 8;         // stages
constexpr int CONS = 8;      // consumer warps

__global__ void __launch_bounds__(32 * (CONS + 1))
    k_tma(const __grid_constant__ CUtensorMap map, const int32_t *__restrict__ idx, int64_t m,
          double *out) {
    __shared__ __align__(128) double buf[S][G * 16];  // 4 rows x 2 doubles per op, 128 B apart
    __shared__ uint64_t full[S], empty[S];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CONS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t per_stage = 4 * G;
    const int64_t nst = m / per_stage;
    // stage t of this CTA: global stage blockIdx.x + t * gridDim.x
    if (warp == CONS) {
        // the whole producer warp: lane q loads 4 indices and issues gather4 q
        int64_t t = 0;
        int64_t gs = blockIdx.x;
        int4 r = gs < nst ? ((const int4 *)(idx + gs * per_stage))[lane] : make_int4(0, 0, 0, 0);
        for (; gs < nst; gs += gridDim.x, t++) {
            const int s = (int)(t % S);
            const int64_t nx = gs + gridDim.x;
            const int4 rn = nx < nst ? ((const int4 *)(idx + nx * per_stage))[lane] : r;
            if (t >= S) mbar_wait(&empty[s], (uint32_t)(((t / S) - 1) & 1));
            if (lane == 0) mbar_expect(&full[s], G * 64);
            __syncwarp();
            tma_gather4(&buf[s][lane * 16], &map, &full[s], r.x >> 1, r.y >> 1, r.z >> 1,
                        r.w >> 1);
            r = rn;
        }
        return;
    }
    double acc = 0;
    int64_t t = 0;
    for (int64_t gs = blockIdx.x; gs < nst; gs += gridDim.x, t++) {
        const int s = (int)(t % S);
        mbar_wait(&full[s], (uint32_t)((t / S) & 1));
        // each consumer warp folds a quarter... every warp reads one slot
        acc += buf[s][(warp * 32 + lane) % (G * 16)];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 12345.678) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                             const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                             const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
    // log2 of the vector length (default 24: 128 MiB, DRAM-bound); 22 keeps
    // it L2-resident like C2's hot columns; "mix" runs LDG and TMA gather4
    // kernels concurrently on split index sets
    const int64_t n = 1ll << (argc > 1 ? atoi(argv[1]) : 24), m = 1ll << 26;
    double *x;
    int32_t *idx;
    double *out;
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&idx, m * 4));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(x, 0, n * 8));
    std::vector<int32_t> h(m);
    std::mt19937_64 rng(1);
    for (auto &v : h) v = (int32_t)(rng() % n);
    CK(cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int clk = 0;
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int thr : {256, 1024}) {
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(a);
            k_ldg<<<sms * (2048 / thr), thr>>>(x, idx, m, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2)
                printf("LDG  %4d thr: %.3f ms, %.3f gathers/SM/cycle (at %d MHz)\n", thr, ms,
                       m / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        }
    }
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap map;
    cuuint64_t dims[2] = {2, (cuuint64_t)(n / 2)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {2, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box,
                                es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        return 1;
    }
    for (int ctas : {1, 2, 4, 6}) {
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(a);
            k_tma<<<sms * ctas, 32 * (CONS + 1)>>>(map, idx, m, out);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep == 2)
                printf("TMA gather4 %d CTA/SM: %.3f ms, %.3f rows/SM/cycle\n", ctas, ms,
                       m / (ms * 1e-3) / sms / (clk * 1e3));
        }
    }
    // concurrent: LDG (768 threads/SM) on a fraction f of the indices, TMA
    // gather4 (4 CTAs/SM) on the rest, on two streams
    cudaStream_t s1, s2;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    for (double f : {1.0, 0.9, 0.8, 0.7, 0.6}) {
        const int64_t ml = ((int64_t)(m * f) / 512) * 512, mt = m - ml;
        float best = 1e9f;
        for (int rep = 0; rep < 4; rep++) {
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            CK(cudaStreamWaitEvent(s1, a, 0));
            CK(cudaStreamWaitEvent(s2, a, 0));
            if (mt) k_tma<<<sms * 4, 32 * (CONS + 1), 0, s2>>>(map, idx + ml, mt, out);
            k_ldg<<<sms, 768, 0, s1>>>(x, idx, ml, out);
            cudaEvent_t e1, e2;
            cudaEventCreate(&e1); cudaEventCreate(&e2);
            cudaEventRecord(e1, s1); cudaEventRecord(e2, s2);
            CK(cudaStreamWaitEvent(0, e1, 0)); CK(cudaStreamWaitEvent(0, e2, 0));
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep && ms < best) best = ms;
        }
        printf("mix LDG %.0f%% / TMA %.0f%%: %.3f ms, %.3f gathers/SM/cycle\n", f * 100,
               (1 - f) * 100, best, m / (best * 1e-3) / sms / (clk * 1e3));
    }
    return 0;
}
