// The paper's comparison methods on the K1 SpMV:
//
//   foster   c <- alpha*A*c + 1 from all ones until the sup-norm change drops
//            below tol; returns c - 1                (baselines.py:36-68)
//   cg_katz  plain conjugate gradient on (I - alpha*A) z = 1 from z = 1,
//            absolute 2-norm stop on the recursive residual; returns
//            alpha*A*z                                 (baselines.py:71-129)
//
// Both reuse run_spmv (level_only: w = alpha*A*x, one sequential ascending
// chain per row) on a scratch State, so the matvec is the engine's own.
// Every elementwise operation is rounded separately as numpy does; Foster is
// therefore bit-identical to the reference wherever K1 is (rows up to the
// split threshold).  CG's inner products are deterministic fixed-order tree
// sums, not BLAS ddot: they agree with numpy to rounding, not bit for bit.
#include "kb_internal.cuh"

#include <cmath>
#include <cstring>

namespace kb {

namespace {

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

constexpr int RB = 592;  // reduction grid: 4 x 148 SMs
constexpr int RT = 256;

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[RT / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < RT / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    }
    return v;  // valid in thread 0
}

__global__ void k_ones_pad(double *c, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) c[i] = 1.0;
    else if (i == n) c[n] = 0.0;
}

// nxt = alpha*A*c + 1 (w holds alpha*A*c, overwritten by nxt);
// delta = max |nxt - c| as ordered bits (nonnegative; NaN sorts above inf)
__global__ void k_foster_step(const double *__restrict__ c, double *__restrict__ w, int64_t n,
                              unsigned long long *dmax) {
    unsigned long long m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double nxt = __dadd_rn(w[i], 1.0);               // baselines.py:58
        w[i] = nxt;
        const unsigned long long b =
            (unsigned long long)__double_as_longlong(fabs(__dsub_rn(nxt, c[i])));  // :59
        m = b > m ? b : m;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_down_sync(0xffffffffu, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(dmax, m);
}

__global__ void k_minus_one(const double *c, double *out, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = __dsub_rn(c[i], 1.0);                  // :61
    else if (i == n) out[n] = 0.0;
}

// --- conjugate gradient (scal: 0 rs, 1 denom, 2 step, 3 rs_next, 4 bad)

// r = 1 - (x - alpha*A*x); partial r.r
__global__ void k_cg_init(const double *__restrict__ x, const double *__restrict__ w,
                          double *__restrict__ r, double *__restrict__ p, int64_t n,
                          double *part) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double ri = __dsub_rn(1.0, __dsub_rn(x[i], w[i]));  // :100, system() :97
        r[i] = ri;
        p[i] = ri;                                               // :104
        acc = __dadd_rn(acc, __dmul_rn(ri, ri));
    }
    const double b = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = b;
}

// Ap = p - alpha*A*p; partial p.Ap
__global__ void k_cg_ap(const double *__restrict__ p, const double *__restrict__ w,
                        double *__restrict__ ap, int64_t n, double *part) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double a = __dsub_rn(p[i], w[i]);                 // :106
        ap[i] = a;
        acc = __dadd_rn(acc, __dmul_rn(p[i], a));
    }
    const double b = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = b;
}

// fixed-order sum of the RB partials into scal[slot]; after the p.Ap sum
// also the step rs/denom and the breakdown flag (baselines.py:107-111)
__global__ void k_cg_reduce(const double *part, double *scal, int slot) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < RB; i += RT) acc = __dadd_rn(acc, part[i]);
    const double s = block_sum(acc);
    if (threadIdx.x == 0) {
        scal[slot] = s;
        if (slot == 1) {
            const bool bad = !(s > 0.0) || !isfinite(s);
            scal[4] = bad ? 1.0 : 0.0;
            scal[2] = bad ? 0.0 : scal[0] / s;
        }
    }
}

// x += step*p; r -= step*Ap; partial r.r (skipped after a breakdown)
__global__ void k_cg_update(double *__restrict__ x, double *__restrict__ r,
                            const double *__restrict__ p, const double *__restrict__ ap,
                            int64_t n, const double *scal, double *part) {
    if (scal[4] != 0.0) return;
    const double step = scal[2];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        x[i] = __dadd_rn(x[i], __dmul_rn(step, p[i]));          // :112
        const double ri = __dsub_rn(r[i], __dmul_rn(step, ap[i]));  // :113
        r[i] = ri;
        acc = __dadd_rn(acc, __dmul_rn(ri, ri));
    }
    const double b = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = b;
}

// p = r + beta*p
__global__ void k_cg_dir(const double *__restrict__ r, double *__restrict__ p, int64_t n,
                         double beta) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = __dadd_rn(r[i], __dmul_rn(beta, p[i]));          // :119
}

// A scratch State that only carries what run_spmv needs (level_only)
struct SpmvCtx {
    State s;
    explicit SpmvCtx(Graph &g, double alpha) {
        s.g = &g;
        s.alpha = alpha;
        s.work_counter.alloc(2);
        s.seg_sum.alloc(std::max<int64_t>(1, g.sell.nseg));
    }
    ~SpmvCtx() {
        for (cudaEvent_t e : s.k1_ev) cudaEventDestroy(e);
    }
    void spmv(const double *x, double *w) { run_spmv(s, s.g->stream, x, w, true); }
};

void to_host_original(Graph &g, const double *src_new, double *h_out, cudaStream_t st) {
    DBuf<double> orig;
    orig.alloc(std::max<int64_t>(1, g.n));
    gather_to_original(g, src_new, orig.p, st);
    KB_CUDA(cudaMemcpyAsync(h_out, orig.p, g.n * sizeof(double), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

bool foster(Graph &g, double alpha, double tol, int64_t max_iter, double *h_values,
            int64_t *iterations, double *residual) {
    const int64_t n = g.n;
    cudaStream_t st = g.stream;
    SpmvCtx ctx(g, alpha);
    DBuf<double> c, w;
    DBuf<unsigned long long> dmax;
    c.alloc(n + 1);
    w.alloc(n + 1);
    dmax.alloc(1);
    k_ones_pad<<<nblk(n + 1, 256), 256, 0, st>>>(c.p, n);       // :56
    note_launch();
    unsigned long long h[1] = {0};
    double delta = INFINITY;
    bool done = false;
    int64_t it = 0;
    while (it < max_iter) {
        it += 1;
        ctx.spmv(c.p, w.p);                                      // :58 alpha*(A@c)
        KB_CUDA(cudaMemsetAsync(dmax.p, 0, sizeof(unsigned long long), st));
        k_foster_step<<<RB, RT, 0, st>>>(c.p, w.p, n, dmax.p);
        note_launch();
        KB_CUDA(cudaMemcpyAsync(h, dmax.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                st));
        KB_CUDA(cudaStreamSynchronize(st));
        double dv;
        memcpy(&dv, h, sizeof(dv));
        delta = n ? dv : 0.0;
        std::swap(c, w);                                         // :60 c = nxt
        if (delta < tol) {                                       // :61
            done = true;
            break;
        }
    }
    k_minus_one<<<nblk(n + 1, 256), 256, 0, st>>>(c.p, w.p, n);
    note_launch();
    to_host_original(g, w.p, h_values, st);
    *iterations = it;
    *residual = delta;
    return done;
}

// returns 0 converged, 1 not converged (cap), 2 breakdown
int cg_katz(Graph &g, double alpha, double residual_tol, int64_t max_iter, double *h_values,
            int64_t *iterations, double *residual) {
    const int64_t n = g.n;
    cudaStream_t st = g.stream;
    SpmvCtx ctx(g, alpha);
    DBuf<double> x, r, p, ap, w, part, scal;
    x.alloc(n + 1); r.alloc(n + 1); p.alloc(n + 1); ap.alloc(n + 1); w.alloc(n + 1);
    part.alloc(RB);
    scal.alloc(8);
    KB_CUDA(cudaMemsetAsync(scal.p, 0, 8 * sizeof(double), st));
    KB_CUDA(cudaMemsetAsync(p.p, 0, (n + 1) * sizeof(double), st));
    k_ones_pad<<<nblk(n + 1, 256), 256, 0, st>>>(x.p, n);       // :99 x = 1
    note_launch();
    ctx.spmv(x.p, w.p);
    k_cg_init<<<RB, RT, 0, st>>>(x.p, w.p, r.p, p.p, n, part.p);
    k_cg_reduce<<<1, RT, 0, st>>>(part.p, scal.p, 0);            // :101 rs = r.r
    note_launch(2);
    double hs[5];
    KB_CUDA(cudaMemcpyAsync(hs, scal.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    double rs = hs[0];
    int64_t it = 0;
    int status = 0;
    if (std::sqrt(rs) >= residual_tol) {                         // :103
        status = 1;
        while (it < max_iter) {
            ctx.spmv(p.p, w.p);
            k_cg_ap<<<RB, RT, 0, st>>>(p.p, w.p, ap.p, n, part.p);
            k_cg_reduce<<<1, RT, 0, st>>>(part.p, scal.p, 1);   // denom, step
            k_cg_update<<<RB, RT, 0, st>>>(x.p, r.p, p.p, ap.p, n, scal.p, part.p);
            k_cg_reduce<<<1, RT, 0, st>>>(part.p, scal.p, 3);   // rs_next
            note_launch(4);
            KB_CUDA(cudaMemcpyAsync(hs, scal.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
            KB_CUDA(cudaStreamSynchronize(st));
            if (hs[4] != 0.0) {                                  // :107-110
                status = 2;
                break;
            }
            const double rs_next = hs[3];
            it += 1;
            if (std::sqrt(rs_next) < residual_tol) {             // :116
                rs = rs_next;
                status = 0;
                break;
            }
            k_cg_dir<<<RB, RT, 0, st>>>(r.p, p.p, n, rs_next / rs);  // :119
            note_launch();
            rs = rs_next;
            KB_CUDA(cudaMemcpyAsync(scal.p, &rs, sizeof(double), cudaMemcpyHostToDevice, st));
        }
    }
    *iterations = it;
    *residual = std::sqrt(rs);
    if (status == 2) return 2;
    ctx.spmv(x.p, w.p);                                          // :129 alpha*(A@x)
    to_host_original(g, w.p, h_values, st);
    return status;
}

}  // namespace kb
