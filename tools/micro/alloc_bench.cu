// Allocation cost on this B200: cudaMalloc vs stream-ordered pool growth vs
// pool reuse, for GB-sized buffers (why does a new state/graph sometimes
// stall for hundreds of ms?).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdint>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

int main() {
    cudaFree(0);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaMemPool_t pool;
    cudaDeviceGetDefaultMemPool(&pool, 0);
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    const size_t GB = 1ull << 30;
    for (size_t sz : {GB / 4, GB, 2 * GB, 4 * GB}) {
        void *p;
        double t = now();
        cudaMalloc(&p, sz);
        double t1 = now();
        cudaMemsetAsync(p, 0, sz, st);
        cudaStreamSynchronize(st);
        double t2 = now();
        cudaFree(p);
        double t3 = now();
        printf("cudaMalloc %5.2f GB: alloc %7.2f ms, first memset %7.2f ms, free %7.2f ms\n",
               sz / (double)GB, 1e3 * (t1 - t), 1e3 * (t2 - t1), 1e3 * (t3 - t2));
    }
    for (size_t sz : {GB / 4, GB, 2 * GB, 4 * GB}) {
        void *p;
        double t = now();
        cudaMallocAsync(&p, sz, st);
        cudaStreamSynchronize(st);
        double t1 = now();
        cudaMemsetAsync(p, 0, sz, st);
        cudaStreamSynchronize(st);
        double t2 = now();
        cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
        double t3 = now();
        cudaMallocAsync(&p, sz, st);
        cudaStreamSynchronize(st);
        double t4 = now();
        cudaFreeAsync(p, st);
        cudaStreamSynchronize(st);
        printf("pool grow  %5.2f GB: alloc %7.2f ms, first memset %7.2f ms, free %7.2f ms, "
               "re-alloc %7.2f ms\n",
               sz / (double)GB, 1e3 * (t1 - t), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3));
    }
    // fragmentation: many mid-size live blocks, free every other, then a big one
    {
        void *blk[64];
        for (int i = 0; i < 64; i++) cudaMallocAsync(&blk[i], 128ull << 20, st);
        for (int i = 0; i < 64; i += 2) cudaFreeAsync(blk[i], st);
        cudaStreamSynchronize(st);
        void *p;
        double t = now();
        cudaMallocAsync(&p, 3 * GB, st);
        cudaStreamSynchronize(st);
        printf("fragmented pool, 3 GB alloc: %7.2f ms\n", 1e3 * (now() - t));
        cudaFreeAsync(p, st);
        for (int i = 1; i < 64; i += 2) cudaFreeAsync(blk[i], st);
        cudaStreamSynchronize(st);
    }
    uint64_t r = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r);
    printf("pool reserved %.2f GB\n", r / (double)GB);
    return 0;
}
