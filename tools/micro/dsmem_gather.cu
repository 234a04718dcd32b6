// Microbenchmark: random 8-byte gathers from (a) local shared memory,
// (b) cluster-distributed shared memory (DSMEM), (c) an L2-resident global
// array, to size the K1 hot-vertex cache.  Prints gathers per SM-cycle.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void k_gather(const double *g, int64_t gsize, int H, int iters, double *out,
                         unsigned long long *cyc) {
    extern __shared__ double sm[];
    cg::cluster_group cl = cg::this_cluster();
    for (int i = threadIdx.x; i < H; i += blockDim.x) sm[i] = (double)(i + blockIdx.x);
    cl.sync();
    const int csize = cl.num_blocks();
    uint32_t st = hash32(blockIdx.x * blockDim.x + threadIdx.x + 1);
    double acc = 0;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            st = hash32(st + q);
            if (MODE == 0) v[q] = sm[st % H];
            else if (MODE >= 3 && (MODE == 3 ? (q & 1) : (q & 3) == 3)) {
                // mixed: a share of the loads go to the cluster's DSMEM, the
                // rest to the global array (both paths in flight together)
                const uint32_t idx = st % (uint32_t)(H * csize);
                const double *rp = cl.map_shared_rank(sm, idx / H);
                v[q] = rp[idx % H];
            } else if (MODE >= 3) {
                v[q] = __ldg(g + (st % (uint32_t)gsize));
            } else if (MODE == 1) {
                const uint32_t idx = st % (uint32_t)(H * csize);
                const double *rp = cl.map_shared_rank(sm, idx / H);
                v[q] = rp[idx % H];
            } else v[q] = __ldg(g + (st % (uint32_t)gsize));
        }
#pragma unroll
        for (int q = 0; q < 8; q++) acc += v[q];
    }
    unsigned long long t1 = clock64();
    cl.sync();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int H = 24576, threads = 1024, iters = 200;
    int64_t gsize = (int64_t)(getenv("GSIZE") ? atoll(getenv("GSIZE")) : (8 << 20));
    double *g, *out;
    unsigned long long *cyc;
    cudaMalloc(&g, gsize * 8);
    cudaMemset(g, 0, gsize * 8);
    cudaMalloc(&out, (size_t)sms * 2 * threads * 8);
    cudaMalloc(&cyc, 8);
    for (int mode = 0; mode < 5; mode++) {
        for (int cs : {1, 2, 4, 8}) {
            if ((mode == 0 || mode == 2) && cs > 1) continue;
            if (mode >= 3 && cs == 1) continue;
            int grid = (sms / cs) * cs;
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = grid;
            cfg.blockDim = threads;
            cfg.dynamicSmemBytes = H * 8;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            auto kern = mode == 0 ? k_gather<0> : mode == 1 ? k_gather<1> : mode == 2 ? k_gather<2>
                      : mode == 3 ? k_gather<3> : k_gather<4>;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, H * 8);
            cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            for (int rep = 0; rep < 2; rep++) {
                cudaMemset(cyc, 0, 8);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                cudaError_t err = cudaLaunchKernelEx(&cfg, kern, (const double *)g, gsize, H, iters, out, cyc);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                unsigned long long c = 0;
                cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
                double gathers = (double)grid * threads * iters * 8;
                double cyc_per_block = (double)c / grid;
                if (rep == 1)
                    printf("mode=%s cluster=%d err=%s time=%.3f ms gathers/SM-cycle=%.3f (Ggathers/s %.1f)\n",
                           mode == 0 ? "local-smem" : mode == 1 ? "dsmem" : mode == 2 ? "global"
                           : mode == 3 ? "1:1 dsmem+global" : "1:3 dsmem+global", cs,
                           cudaGetErrorString(err), ms,
                           gathers / grid / cyc_per_block, gathers / (ms * 1e-3) / 1e9);
            }
        }
    }
    return 0;
}
