// Can one warp fold a hub row in exact sequential order inside K1's window?
// (1) dependent DADD latency; (2) one warp gathering a 406,877-arc row from a
// 128 MiB vector with a prefetch ring and folding it in order, bit-identical
// to a host sequential sum.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

__global__ void k_chain(double *out, int iters, double a) {
    double s = threadIdx.x * 1e-3;
    for (int i = 0; i < iters; i++) s = __dadd_rn(s, a);
    if (s == 1234.5) out[0] = s;
    out[1 + threadIdx.x] = s;
}

// one warp: RING chunks of 32 gathers in flight; lane 0 folds in order via shfl
template <int RING>
__global__ void k_fold(const double *__restrict__ x, const int32_t *__restrict__ cols, int64_t L,
                       double *out) {
    const int lane = threadIdx.x & 31;
    double ring[RING];
    const int64_t nchunk = (L + 31) / 32;
#pragma unroll
    for (int r = 0; r < RING; r++) {
        const int64_t j = (int64_t)r * 32 + lane;
        ring[r] = (r < nchunk && j < L) ? __ldg(x + cols[j]) : 0.0;
    }
    double s = 0.0;
    for (int64_t c = 0; c < nchunk; c += RING) {
#pragma unroll
        for (int r = 0; r < RING; r++) {
            const double v = ring[r];
            const int64_t cc = c + r;
            // refill this slot with chunk cc + RING
            const int64_t j = (cc + RING) * 32 + lane;
            ring[r] = (cc + RING < nchunk && j < L) ? __ldg(x + cols[j]) : 0.0;
            const int64_t base = cc * 32;
#pragma unroll
            for (int q = 0; q < 32; q++) {
                const double t = __shfl_sync(0xffffffffu, v, q);
                if (base + q < L) s = __dadd_rn(s, t);
            }
        }
    }
    if (lane == 0) out[0] = s;
}

int main() {
    double *d_out;
    cudaMalloc(&d_out, 4096 * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 1 << 22;
    k_chain<<<1, 32>>>(d_out, 1000, 1.0);
    cudaEventRecord(a);
    k_chain<<<1, 32>>>(d_out, iters, 1.0000001);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("dependent DADD: %.2f cycles each (%d MHz)\n", ms * 1e-3 * clk * 1e3 / iters, clk / 1000);

    const int64_t n = 1 << 24, L = 406877;
    std::vector<double> hx(n);
    std::mt19937_64 rng(3);
    std::uniform_real_distribution<double> U(0, 1e-3);
    for (auto &v : hx) v = U(rng);
    std::vector<int32_t> hc(L);
    for (auto &c : hc) c = (int32_t)(rng() % n);
    std::sort(hc.begin(), hc.end());
    double ref = 0.0;
    for (int64_t j = 0; j < L; j++) ref = ref + hx[hc[j]];
    double *dx;
    int32_t *dc;
    cudaMalloc(&dx, n * 8);
    cudaMalloc(&dc, L * 4);
    cudaMemcpy(dx, hx.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, hc.data(), L * 4, cudaMemcpyHostToDevice);
    auto run = [&](auto kern, const char *name) {
        kern<<<1, 32>>>(dx, dc, L, d_out);
        cudaEventRecord(a);
        kern<<<1, 32>>>(dx, dc, L, d_out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float t;
        cudaEventElapsedTime(&t, a, b);
        double got;
        cudaMemcpy(&got, d_out, 8, cudaMemcpyDeviceToHost);
        printf("%s: %.3f ms for %lld arcs (%.2f cycles/arc), exact=%d\n", name, t, (long long)L,
               t * 1e-3 * clk * 1e3 / L, got == ref);
    };
    run(k_fold<8>, "fold ring 8");
    run(k_fold<16>, "fold ring 16");
    run(k_fold<32>, "fold ring 32");
    return 0;
}
