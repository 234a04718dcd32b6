// K4: dynamic edge-batch update (dynamic.update_batch, dynamic.py:126-211).
//
// 1. The batch is applied to the device CSR-with-slack in place: every edited
//    row is rebuilt by one warp as (old row - deletions) merged with the
//    sorted insertions.  Rows whose capacity would overflow trigger one
//    re-spread of the whole CSR with fresh slack.
// 2. Levels 1..r are repaired on the post-batch graph.  The rows recomputed
//    at level i are R_i = seeds U in-neighbours of the rows whose level i-1
//    changed bit-wise -- the reference's affected-set growth
//    (dynamic.py:94-103) -- so UpdateStats follow it.  Each row is recomputed
//    by pull with exactly K1's summation order (sequential per row, or per
//    split-sized segment combined in order), so repaired levels are
//    bit-identical to a fresh static run.  Past theta*n affected nodes the
//    remaining levels are recomputed whole with K1 (dynamic.py:78-88).
// 3. katz is re-summed from the stored levels in order, the bounds are
//    refreshed under the new tail factor (dynamic.py:181-187), nodes that may
//    contend again are reactivated (:190-197), and the run resumes (:203-210).
#include <cub/block/block_reduce.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kb_internal.cuh"

namespace kb {

namespace {

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

template <typename F>
void cub_run(F &&f) {
    size_t tb = 0;
    KB_CUDA(f(nullptr, tb));
    DBuf<unsigned char> tmp;
    tmp.alloc(tb);
    KB_CUDA(f(tmp.p, tb));
    note_launch();
}

// ---------------------------------------------------------------- slack CSR

__global__ void k_capacity(const int32_t *rlen, const int32_t *extra, int64_t n, int64_t *cap) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v > n) return;
    if (v == n) { cap[v] = 0; return; }
    const int64_t need = (int64_t)rlen[v] + (extra ? extra[v] : 0);
    cap[v] = need + max((int64_t)2, need / 8);
}

__global__ void k_cap32(const int64_t *cap, int64_t n, int32_t *rcap) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v < n) rcap[v] = (int32_t)min(cap[v], (int64_t)INT32_MAX);
}


// Row copy old -> new layout.  Short rows: a block takes 256 consecutive
// rows, scans their lengths in shared memory and copies the concatenated
// elements with every thread busy (a warp per row would idle most lanes on
// R-MAT's ~30-arc rows).  Rows longer than LONG_ROW get a block each.
constexpr int COPY_ROWS = 256;
constexpr int LONG_ROW = 1024;

__global__ void __launch_bounds__(COPY_ROWS) k_copy_short(const int64_t *old_ip,
                                                          const int32_t *old_ix,
                                                          const int32_t *rlen, int64_t n,
                                                          const int64_t *new_ip,
                                                          int32_t *new_ix) {
    __shared__ int64_t a[COPY_ROWS], b[COPY_ROWS];
    __shared__ int off[COPY_ROWS + 1];
    const int64_t r0 = (int64_t)blockIdx.x * COPY_ROWS;
    const int t = threadIdx.x;
    int len = 0;
    if (r0 + t < n) {
        len = rlen[r0 + t];
        if (len > LONG_ROW) len = 0;
        a[t] = old_ip[r0 + t];
        b[t] = new_ip[r0 + t];
    }
    // exclusive scan of the lengths (block-wide, Hillis-Steele in smem)
    off[t + 1] = len;
    if (t == 0) off[0] = 0;
    __syncthreads();
    for (int d = 1; d < COPY_ROWS; d <<= 1) {
        const int v = (t + 1 > d) ? off[t + 1 - d] : 0;
        __syncthreads();
        off[t + 1] += v;
        __syncthreads();
    }
    const int total = off[COPY_ROWS];
    for (int e = t; e < total; e += COPY_ROWS) {
        int lo = 0, hi = COPY_ROWS;              // last row with off[row] <= e
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (off[mid] <= e) lo = mid; else hi = mid;
        }
        const int k = e - off[lo];
        new_ix[b[lo] + k] = old_ix[a[lo] + k];
    }
}

__global__ void k_copy_long(const int32_t *rows, const int64_t *old_ip, const int32_t *old_ix,
                            const int32_t *rlen, const int64_t *new_ip, int32_t *new_ix) {
    const int32_t r = rows[blockIdx.x];
    const int64_t L = rlen[r], a = old_ip[r], b = new_ip[r];
    for (int64_t j = threadIdx.x; j < L; j += blockDim.x) new_ix[b + j] = old_ix[a + j];
}

struct IsLongRow {
    const int32_t *rlen;
    __device__ bool operator()(int32_t r) const { return rlen[r] > LONG_ROW; }
};

}  // namespace

static void copy_rows(const int64_t *old_ip, const int32_t *old_ix, const int32_t *rlen, int64_t n,
               const int64_t *new_ip, int32_t *new_ix, cudaStream_t st) {
    if (n <= 0) return;
    k_copy_short<<<nblk(n, COPY_ROWS), COPY_ROWS, 0, st>>>(old_ip, old_ix, rlen, n, new_ip,
                                                         new_ix);
    note_launch();
    DBuf<int32_t> longs;
    DBuf<int64_t> cnt;
    longs.alloc(n);
    cnt.alloc(1);
    cub::CountingInputIterator<int32_t> it(0);
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceSelect::If(t, b, it, longs.p, cnt.p, (int)n, IsLongRow{rlen}, st);
    });
    int64_t nl = 0;
    KB_CUDA(cudaMemcpyAsync(&nl, cnt.p, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    if (nl) {
        k_copy_long<<<(unsigned)nl, 256, 0, st>>>(longs.p, old_ip, old_ix, rlen, new_ip, new_ix);
        note_launch();
    }
}

namespace {

__global__ void k_compact_len(const int32_t *rlen, int64_t n, int64_t *len) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v > n) return;
    len[v] = v < n ? rlen[v] : 0;
}

}  // namespace

// The slack layout for the current row lengths (+extra): capacity = len
// (+extra) + max(2, len/8), row starts nip, the column array nix with 1/16
// tail room (rows that later outgrow their slack are relocated there instead
// of re-spreading the whole graph) and g.rcap.  Rows are not copied.
void slack_layout(Graph &g, const int32_t *extra, DBuf<int64_t> &nip, DBuf<int32_t> &nix,
                  int64_t &total) {
    cudaStream_t st = g.stream;
    const int64_t n = g.n;
    DBuf<int64_t> cap;
    cap.alloc(n + 1);
    nip.alloc(n + 1);
    k_capacity<<<nblk(n + 1, 256), 256, 0, st>>>(g.rlen.p, extra, n, cap.p);
    note_launch();
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, cap.p, nip.p, (int)(n + 1), st);
    });
    total = 0;
    KB_CUDA(cudaMemcpyAsync(&total, nip.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    const int64_t room = std::max<int64_t>(total / 16, tune_get("dyn.tail_room", 1 << 20));
    nix.alloc(total + room);
    g.rcap.alloc(std::max<int64_t>(1, n));
    k_cap32<<<nblk(n, 256), 256, 0, st>>>(cap.p, n, g.rcap.p);
    note_launch();
}

namespace {

// Rebuild the slack layout and copy every row into it.
void respread(Graph &g, const int32_t *extra) {
    DBuf<int64_t> nip;
    DBuf<int32_t> nix;
    int64_t total = 0;
    slack_layout(g, extra, nip, nix, total);
    copy_rows(g.indptr.p, g.indices.p, g.rlen.p, g.n, nip.p, nix.p, g.stream);
    g.indptr = std::move(nip);
    g.indices = std::move(nix);
    g.tail = total;
    g.slack = true;
}

}  // namespace

// the slack layout the dynamic path edits in place, built once at ingest so
// the first update does not re-spread (and regrow the memory pool) inside it
void make_slack(Graph &g) {
    if (!g.slack) respread(g, nullptr);
}

namespace {

// ---------------------------------------------------------------- batch edits

// Edited row e: original id rows[e], deletions del[dptr[e]..dptr[e+1]),
// insertions ins[iptr[e]..iptr[e+1]) (both ascending).  One warp per row
// writes the merged row to tmp[toff[e] ..) and then back in place.
__device__ __forceinline__ int64_t lower_bound32(const int32_t *a, int64_t n, int32_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void k_apply_edits(const int32_t *rows, int64_t ne, const int64_t *dptr,
                              const int32_t *del, const int64_t *iptr, const int32_t *ins,
                              const int64_t *toff, int32_t *tmp, const int64_t *indptr,
                              int32_t *indices, int32_t *rlen, const int32_t *rcap = nullptr,
                              int64_t cap_total = INT64_MAX) {
    const int64_t e = blockIdx.x;  // a block per edited row (hub rows are long)
    const int t = threadIdx.x, nt = blockDim.x;
    if (e >= ne) return;
    const int32_t v = rows[e];
    const int32_t *row = indices + indptr[v];
    const int64_t L = rlen[v];
    const int32_t *D = del + dptr[e];
    const int64_t nd = dptr[e + 1] - dptr[e];
    const int32_t *I = ins + iptr[e];
    const int64_t ni = iptr[e + 1] - iptr[e];
    int32_t *out = tmp + toff[e];
    for (int64_t j = t; j < L; j += nt) {
        const int32_t c = row[j];
        const int64_t dl = lower_bound32(D, nd, c);
        if (dl < nd && D[dl] == c) continue;  // deleted
        out[j - dl + lower_bound32(I, ni, c)] = c;
    }
    for (int64_t q = t; q < ni; q += nt) {
        const int32_t x = I[q];
        out[lower_bound32(row, L, x) - lower_bound32(D, nd, x) + q] = x;
    }
    __syncthreads();
    const int64_t nl = L - nd + ni;
    // the edited row fits its slot (capacity planned on the host) and the array
    KB_DCHECK(nl >= 0 && (!rcap || nl <= rcap[v]) && indptr[v] + nl <= cap_total);
    (void)rcap; (void)cap_total;
    for (int64_t j = t; j < nl; j += nt) indices[indptr[v] + j] = out[j];
    if (t == 0) rlen[v] = (int32_t)nl;
}



// ---------------------------------------------------------------- transpose

__global__ void k_arc_keys_t(const int64_t *indptr, const int32_t *indices, const int32_t *rlen,
                             int64_t n, const int64_t *cidx, uint64_t *keys) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const int64_t base = cidx[warp];
    for (int64_t j = lane; j < rlen[warp]; j += 32)
        keys[base + j] = ((uint64_t)(uint32_t)indices[indptr[warp] + j] << 32) | (uint32_t)warp;
}

__global__ void k_row_count_t(const uint64_t *keys, int64_t m, int64_t n, int64_t *ip) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v > n) return;
    const uint64_t target = (uint64_t)v << 32;
    int64_t lo = 0, hi = m;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    ip[v] = lo;
}

__global__ void k_low32(const uint64_t *keys, int64_t m, int32_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) out[i] = (int32_t)(keys[i] & 0xffffffffu);
}

// ---------------------------------------------------------------- frontier

// add the rows of `list` to R (deduplicated with a per-level stamp)
__global__ void k_mark_list(const int32_t *list, int64_t m, int32_t *stamp, int32_t level,
                            int32_t *R, unsigned long long *rcount, unsigned char *touched) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int32_t v = list[i];
    if (atomicExch(&stamp[v], level) != level) {
        R[atomicAdd(rcount, 1ull)] = v;
        touched[v] = 1;
    }
}

// cumulative affected set: byte flags, count of first-time insertions
__global__ void k_affect(const int32_t *list, int64_t m, unsigned int *aff_words,
                         unsigned long long *affcount) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int32_t v = list[i];
    const unsigned bit = 1u << (v & 31);
    atomicOr(&aff_words[v >> 5], bit);
    (void)affcount;
}

constexpr int EXPAND_SPLIT = 16;

// in-neighbours of the changed rows (new ids) -> R (stamped) and affected
__global__ void k_expand(const int32_t *changed, int64_t nc, const int64_t *in_ip,
                         const int32_t *in_len, const int32_t *in_ix, const int32_t *perm,
                         const int32_t *iperm, int32_t *stamp, int32_t level, int32_t *R,
                         unsigned long long *rcount, unsigned int *aff_words,
                         unsigned long long *affcount, unsigned char *touched) {
    // EXPAND_SPLIT warps per changed row, each taking every EXPAND_SPLIT-th
    // 32-arc step: a hub's in-neighbours (10^5 arcs) do not serialise on one
    // warp's atomics
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t warp = gw / EXPAND_SPLIT;
    const int part = (int)(gw % EXPAND_SPLIT);
    if (warp >= nc) return;
    const int32_t o = perm[changed[warp]];
    const int64_t a = in_ip[o];
    const int64_t L = in_len ? in_len[o] : in_ip[o + 1] - a;
    (void)affcount;
    for (int64_t j0 = (int64_t)part * 32; j0 < L; j0 += 32 * EXPAND_SPLIT) {
        const int64_t j = j0 + lane;
        bool fresh = false;
        int32_t u = 0;
        if (j < L) {
            u = iperm[in_ix[a + j]];
            atomicOr(&aff_words[u >> 5], 1u << (u & 31));
            fresh = atomicExch(&stamp[u], level) != level;
            if (fresh) touched[u] = 1;
        }
        // one counter update per warp step: the list position of each new row
        const unsigned b = __ballot_sync(0xffffffffu, fresh);
        if (b) {
            unsigned long long base = 0;
            if (lane == __ffs(b) - 1) base = atomicAdd(rcount, (unsigned long long)__popc(b));
            base = __shfl_sync(0xffffffffu, base, __ffs(b) - 1);
            if (fresh) R[base + __popc(b & ((1u << lane) - 1u))] = u;
        }
    }
}

// |affected| = population count of the bitmap (one pass over n/32 words;
// the marking kernels set bits without counting)
__global__ void k_popc_count(const unsigned int *words, int64_t nw, unsigned long long *count) {
    unsigned long long c = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw;
         i += (int64_t)gridDim.x * blockDim.x)
        c += __popc(words[i]);
#pragma unroll
    for (int k = 16; k; k >>= 1) c += __shfl_down_sync(0xffffffffu, c, k);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// total in-degree of the changed rows: the work an expansion would do
__global__ void k_work_sum(const int32_t *changed, int64_t nc, const int64_t *in_ip,
                           const int32_t *in_len, const int32_t *perm,
                           unsigned long long *work) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long w = 0;
    if (i < nc) {
        const int32_t o = perm[changed[i]];
        w = (unsigned long long)(in_len ? in_len[o] : in_ip[o + 1] - in_ip[o]);
    }
#pragma unroll
    for (int k = 16; k; k >>= 1) w += __shfl_down_sync(0xffffffffu, w, k);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(work, w);
}

// ---------------------------------------------------------------- recompute

// w_level[v] = alpha * sum_{c in row(v)} x[iperm[c]] with K1's order: one
// sequential chain per row of length <= split, else split-sized segments
// summed sequentially and combined in segment order.  One warp per row.
__global__ void k_recompute(const int32_t *R, int64_t nr, const int32_t *perm,
                            const int32_t *iperm, const int64_t *indptr, const int32_t *rlen,
                            const int32_t *indices, const double *x, double *w, double alpha,
                            int64_t split, int32_t *changed, unsigned long long *nchanged,
                            const int32_t *h_of_row, const int32_t *ovf_flag,
                            int32_t *heavy_out, unsigned long long *nheavy) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= nr) return;
    const int32_t v = R[warp];
    const int32_t o = perm[v];
    const int32_t *row = indices + indptr[o];
    const int64_t L = rlen[o];
    if (heavy_out && L > split && h_of_row[v] >= 0 && !(ovf_flag && ovf_flag[v])) {
        // a heavy row with current SELL segments: k_heavy_rows_fold
        if (lane == 0) heavy_out[atomicAdd(nheavy, 1ull)] = v;
        return;
    }
    double s = 0.0;
    if (L <= split) {
        // lanes gather 32 consecutive slots; lane 0 folds them in order
        for (int64_t base = 0; base < L; base += 32) {
            const int64_t j = base + lane;
            const double val = j < L ? x[iperm[row[j]]] : 0.0;
            const int cnt = (int)min((int64_t)32, L - base);
            for (int q = 0; q < cnt; q++) {
                const double t = __shfl_sync(0xffffffffu, val, q);
                if (lane == 0) s = __dadd_rn(s, t);
            }
        }
    } else {
        const int64_t nseg = (L + split - 1) / split;
        for (int64_t g0 = 0; g0 < nseg; g0 += 32) {
            const int64_t sg = g0 + lane;
            double ss = 0.0;
            if (sg < nseg) {
                const int64_t a = sg * split, b = min(L, a + split);
                for (int64_t j = a; j < b; j++) ss = __dadd_rn(ss, x[iperm[row[j]]]);
            }
            const int cnt = (int)min((int64_t)32, nseg - g0);
            for (int q = 0; q < cnt; q++) {
                const double t = __shfl_sync(0xffffffffu, ss, q);
                if (lane == 0) s = __dadd_rn(s, t);
            }
        }
    }
    if (lane == 0) {
        const double nw = __dmul_rn(alpha, s);
        const double old = w[v];
        if (__double_as_longlong(nw) != __double_as_longlong(old)) {
            changed[atomicAdd(nchanged, 1ull)] = v;
            w[v] = nw;
        }
    }
}

// Heavy rows of a sparse level, recomputed from their SELL segments with
// K1's own folds (each lane one segment, ascending slots, gathers issued 16
// ahead) and k_heavy_combine's segment order, so the bits are K1's.  A block
// per row: a hub's ~200 segments fold in parallel instead of one warp
// walking them.
__global__ void __launch_bounds__(256) k_heavy_rows_fold(
    const int32_t *rows, const double *x, double *w, double alpha, const int32_t *h_of_row,
    const int32_t *seg_ptr, const int32_t *seg_list, const int64_t *slice_off,
    const int32_t *slice_w, const int32_t *vlen, const int32_t *cols, int32_t *changed,
    unsigned long long *nchanged) {
    __shared__ double part[256];
    const int32_t v = rows[blockIdx.x];
    const int32_t h = h_of_row[v];
    const int q0 = seg_ptr[h], nq = seg_ptr[h + 1] - q0;
    double s = 0.0;  // thread 0's running row sum
    for (int b = 0; b < nq; b += blockDim.x) {
        const int q = b + threadIdx.x;
        double ss = 0.0;
        if (q < nq) {
            const int32_t vr = seg_list[q0 + q];
            const int64_t sl = vr >> 5;
            const int ln = vr & 31;
            const int len = vlen[vr];
            const int32_t *p = cols + slice_off[sl] + ln * 4;
            (void)slice_w;
            // batches of 32 slots: the next batch's column groups are loaded
            // before this batch's gathers are folded
            int4 cn[8];
#pragma unroll
            for (int g4 = 0; g4 < 8; g4++)
                cn[g4] = (g4 * 4 < len) ? *(const int4 *)(p + (int64_t)g4 * 128)
                                        : make_int4(0, 0, 0, 0);
            for (int j0 = 0; j0 < len; j0 += 32) {
                int4 c[8];
#pragma unroll
                for (int g4 = 0; g4 < 8; g4++) c[g4] = cn[g4];
#pragma unroll
                for (int g4 = 0; g4 < 8; g4++) {
                    const int j = j0 + 32 + g4 * 4;
                    cn[g4] = (j < len) ? *(const int4 *)(p + (int64_t)(j >> 2) * 128)
                                       : make_int4(0, 0, 0, 0);
                }
                double t[32];
#pragma unroll
                for (int g4 = 0; g4 < 8; g4++) {
                    const int j = j0 + g4 * 4;
                    t[g4 * 4 + 0] = j + 0 < len ? x[c[g4].x] : 0.0;
                    t[g4 * 4 + 1] = j + 1 < len ? x[c[g4].y] : 0.0;
                    t[g4 * 4 + 2] = j + 2 < len ? x[c[g4].z] : 0.0;
                    t[g4 * 4 + 3] = j + 3 < len ? x[c[g4].w] : 0.0;
                }
#pragma unroll
                for (int u = 0; u < 32; u++)
                    if (j0 + u < len) ss = __dadd_rn(ss, t[u]);
            }
        }
        part[threadIdx.x] = ss;
        __syncthreads();
        if (threadIdx.x == 0) {
            const int cnt = min((int)blockDim.x, nq - b);
            for (int u = 0; u < cnt; u++) s = __dadd_rn(s, part[u]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double nw = __dmul_rn(alpha, s);
        if (__double_as_longlong(nw) != __double_as_longlong(w[v])) {
            changed[atomicAdd(nchanged, 1ull)] = v;
            w[v] = nw;
        }
    }
}

// heavy row rows[i] = its segment sums combined in order (warp per row)
__global__ void k_heavy_finish(const int32_t *rows, int64_t m, double *w, double alpha,
                               const int32_t *h_of_row, const int32_t *seg_ptr,
                               const int32_t *seg_list, const double *seg_sum,
                               int32_t *changed, unsigned long long *nchanged) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= m) return;
    const int32_t v = rows[i];
    const int32_t h = h_of_row[v];
    const int q0 = seg_ptr[h], q1 = seg_ptr[h + 1];
    double s = 0.0;
    for (int b = q0; b < q1; b += 32) {
        const double val = (b + lane < q1) ? seg_sum[seg_list[b + lane]] : 0.0;
        const int cnt = min(32, q1 - b);
        for (int q = 0; q < cnt; q++) {
            const double t = __shfl_sync(0xffffffffu, val, q);
            if (lane == 0) s = __dadd_rn(s, t);
        }
    }
    if (lane == 0) {
        const double nw = __dmul_rn(alpha, s);
        if (__double_as_longlong(nw) != __double_as_longlong(w[v])) {
            changed[atomicAdd(nchanged, 1ull)] = v;
            w[v] = nw;
        }
    }
}

// katz[v] = ((0 + w_1) + w_2) + ... + w_r, the static accumulation order
__global__ void k_katz_rows(const int32_t *rows, int64_t m, const double *const *levels, int r,
                            double *katz) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t v = rows ? rows[i] : i;
    double k = 0.0;
    for (int l = 1; l <= r; l++) k = __dadd_rn(k, levels[l][v]);
    katz[v] = k;
}

__global__ void k_bounds_rows(const int32_t *rows, int64_t m, const double *katz,
                              const double *wr, double alpha, double gamma, int undirected,
                              double *lower, double *upper) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t v = rows ? rows[i] : i;
    const double k = katz[v];
    const double t = __dmul_rn(alpha, wr[v]);                 // dynamic.py:182
    lower[v] = undirected ? __dadd_rn(k, t) : k;             // :183-186
    upper[v] = __dadd_rn(k, __dmul_rn(t, gamma));            // :187
}

// u joins the affected set when any of its out-neighbours changed
// rows (original id o) with a changed out-neighbour join the affected set;
// chg_bits marks the changed rows by original id (2 MB at C2: L2-resident)
__global__ void k_pull_affect(const int64_t *indptr, const int32_t *rlen, const int32_t *indices,
                              const int32_t *iperm, int64_t n, const unsigned int *chg_bits,
                              unsigned int *aff_words, unsigned long long *affcount) {
    int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (o >= n) return;
    const int32_t u = iperm[o];
    const unsigned bit = 1u << (u & 31);
    if (aff_words[u >> 5] & bit) return;
    const int32_t *row = indices + indptr[o];
    const int32_t L = rlen[o];
    for (int32_t j = 0; j < L; j++) {
        const int32_t c = __ldg(row + j);
        if ((__ldg(chg_bits + (c >> 5)) >> (c & 31)) & 1u) {
            atomicOr(&aff_words[u >> 5], bit);
            (void)affcount;
            return;
        }
    }
}

// sources of every edit, then targets: ends[0..m) and ends[m..2m)
__global__ void k_batch_ends(const int64_t *ins, int64_t ni, const int64_t *dels, int64_t nd,
                             int32_t *ends) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t m = ni + nd;
    if (i >= m) return;
    const int64_t *a = i < ni ? ins + 2 * i : dels + 2 * (i - ni);
    ends[i] = (int32_t)a[0];
    ends[m + i] = (int32_t)a[1];
}

__global__ void k_map_new(const int32_t *orig, int64_t m, const int32_t *iperm, int32_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) out[i] = iperm[orig[i]];
}

__global__ void k_flags_from_list(const int32_t *list, int64_t m, unsigned char *flag) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) flag[list[i]] = 1;
}

// bitmap by original id of a list of new ids
__global__ void k_bits_from_list(const int32_t *list, int64_t m, const int32_t *perm,
                                 unsigned int *bits) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) {
        const int32_t o = perm[list[i]];
        atomicOr(bits + (o >> 5), 1u << (o & 31));
    }
}

__global__ void k_min_lower(const int32_t *act, int64_t m, const double *lower,
                            unsigned long long *out) {
    typedef cub::BlockReduce<unsigned long long, 256> Red;
    __shared__ typename Red::TempStorage tmp;
    unsigned long long best = ~0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        // lower >= +0: the IEEE bits order like the values
        best = min(best, (unsigned long long)__double_as_longlong(lower[act[i]]));
    }
    best = Red(tmp).Reduce(best, cub::Min());
    if (threadIdx.x == 0) atomicMin(out, best);
}

// reactivation flags by original id: not active and fl(upper) >= floor
__global__ void k_reactivate_flags(const int32_t *iperm, int64_t n, const unsigned char *inact,
                                   const double *upper, const unsigned long long *minbits,
                                   double eps, unsigned char *flag) {
    int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (o >= n) return;
    const int32_t v = iperm[o];
    const double floor = __dsub_rn(__longlong_as_double((long long)*minbits), eps);
    flag[o] = !inact[v] && upper[v] >= floor;
}

__global__ void k_has_arcs(const int64_t *arcs, int64_t m, const int64_t *indptr,
                           const int32_t *rlen, const int32_t *indices, unsigned char *present) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t u = arcs[2 * i], v = arcs[2 * i + 1];
    const int32_t *row = indices + indptr[u];
    const int64_t L = rlen[u];
    const int64_t p = lower_bound32(row, L, (int32_t)v);
    present[i] = p < L && row[p] == v;
}

__global__ void k_deg_delta(const int64_t *arcs, int64_t m, int delta, int32_t *deg) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) atomicAdd(&deg[arcs[2 * i]], delta);
}

__global__ void k_max_i32(const int32_t *a, int64_t n, unsigned long long *out) {
    typedef cub::BlockReduce<int, 256> Red;
    __shared__ typename Red::TempStorage tmp;
    int m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, a[i]);
    m = Red(tmp).Reduce(m, cub::Max());
    if (threadIdx.x == 0) atomicMax(out, (unsigned long long)m);
}

__global__ void k_widen_i32(const int32_t *a, int64_t n, int64_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = a[i];
}

}  // namespace

void graph_has_arcs(Graph &g, const int64_t *h_arcs, int64_t m, unsigned char *h_present) {
    cudaStream_t st = g.stream;
    if (m <= 0) return;
    DBuf<int64_t> a;
    DBuf<unsigned char> pr;
    a.alloc(2 * m);
    pr.alloc(m);
    KB_CUDA(cudaMemcpyAsync(a.p, h_arcs, 2 * m * 8, cudaMemcpyHostToDevice, st));
    k_has_arcs<<<nblk(m, 256), 256, 0, st>>>(a.p, m, g.indptr.p, g.rlen.p, g.indices.p, pr.p);
    note_launch();
    KB_CUDA(cudaMemcpyAsync(h_present, pr.p, m, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
}

int64_t graph_max_degree_after(Graph &g, const int64_t *ins, int64_t n_ins, const int64_t *dels,
                               int64_t n_dels) {
    cudaStream_t st = g.stream;
    DBuf<int32_t> deg;
    DBuf<int64_t> a;
    DBuf<unsigned long long> mx;
    deg.alloc(g.n);
    mx.alloc(1);
    KB_CUDA(cudaMemcpyAsync(deg.p, g.rlen.p, g.n * 4, cudaMemcpyDeviceToDevice, st));
    KB_CUDA(cudaMemsetAsync(mx.p, 0, 8, st));
    const int64_t m = std::max(n_ins, n_dels);
    a.alloc(std::max<int64_t>(1, 2 * m));
    if (n_ins) {
        KB_CUDA(cudaMemcpyAsync(a.p, ins, 2 * n_ins * 8, cudaMemcpyHostToDevice, st));
        k_deg_delta<<<nblk(n_ins, 256), 256, 0, st>>>(a.p, n_ins, 1, deg.p);
        note_launch();
    }
    if (n_dels) {
        KB_CUDA(cudaStreamSynchronize(st));
        KB_CUDA(cudaMemcpyAsync(a.p, dels, 2 * n_dels * 8, cudaMemcpyHostToDevice, st));
        k_deg_delta<<<nblk(n_dels, 256), 256, 0, st>>>(a.p, n_dels, -1, deg.p);
        note_launch();
    }
    if (g.n) {
        k_max_i32<<<2 * std::max(1, g.sm_count), 256, 0, st>>>(deg.p, g.n, mx.p);
        note_launch();
    }
    unsigned long long h = 0;
    KB_CUDA(cudaMemcpyAsync(&h, mx.p, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    return (int64_t)h;
}

void graph_out_degrees(Graph &g, int64_t *h_out) {
    cudaStream_t st = g.stream;
    DBuf<int64_t> w;
    w.alloc(std::max<int64_t>(1, g.n));
    if (g.n) k_widen_i32<<<nblk(g.n, 256), 256, 0, st>>>(g.rlen.p, g.n, w.p);
    note_launch();
    KB_CUDA(cudaMemcpyAsync(h_out, w.p, g.n * 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
}

void compact_csr(Graph &g, DBuf<int64_t> &ip, DBuf<int32_t> &ix) {
    cudaStream_t st = g.stream;
    const int64_t n = g.n;
    DBuf<int64_t> len;
    len.alloc(n + 1);
    ip.alloc(n + 1);
    k_compact_len<<<nblk(n + 1, 256), 256, 0, st>>>(g.rlen.p, n, len.p);
    note_launch();
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, len.p, ip.p, (int)(n + 1), st);
    });
    ix.alloc(std::max<int64_t>(1, g.nnz));
    copy_rows(g.indptr.p, g.indices.p, g.rlen.p, n, ip.p, ix.p, st);
    KB_CUDA(cudaStreamSynchronize(st));
}

// in-neighbour CSR of the current arc set (original ids; rows ascending)
static void build_transpose(Graph &g, DBuf<int64_t> &tip, DBuf<int32_t> &tix) {
    cudaStream_t st = g.stream;
    const int64_t n = g.n, m = g.nnz;
    DBuf<int64_t> cip;
    DBuf<int32_t> cix;
    compact_csr(g, cip, cix);
    DBuf<uint64_t> keys, skeys;
    keys.alloc(std::max<int64_t>(1, m));
    skeys.alloc(std::max<int64_t>(1, m));
    k_arc_keys_t<<<nblk(n * 32, 256), 256, 0, st>>>(g.indptr.p, g.indices.p, g.rlen.p, n, cip.p,
                                                    keys.p);
    note_launch();
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortKeys(t, b, keys.p, skeys.p, (int)m, 0, 64, st);
    });
    tip.alloc(n + 1);
    tix.alloc(std::max<int64_t>(1, m));
    k_row_count_t<<<nblk(n + 1, 256), 256, 0, st>>>(skeys.p, m, n, tip.p);
    k_low32<<<nblk(m, 256), 256, 0, st>>>(skeys.p, m, tix.p);
    note_launch(2);
    KB_CUDA(cudaStreamSynchronize(st));
}

namespace {

// ---------------------------------------------------------------- edit grouping
// One 64-bit key per edit: src << 33 | kind << 32 | dst (kind 0 delete,
// 1 insert), so a plain integer sort groups the edits by row with the
// deletions first and the dsts ascending (the order k_apply_edits merges in).
__global__ void k_edit_keys(const int64_t *ins, int64_t ni, const int64_t *dels, int64_t nd,
                            uint64_t *keys) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nd) {
        keys[i] = ((uint64_t)(uint32_t)dels[2 * i] << 33) | (uint32_t)dels[2 * i + 1];
    } else if (i < nd + ni) {
        const int64_t j = i - nd;
        keys[i] = ((uint64_t)(uint32_t)ins[2 * j] << 33) | (1ull << 32) | (uint32_t)ins[2 * j + 1];
    }
}

// packed per-edit counters: (row head) << 32 | (is a deletion)
__global__ void k_edit_flags(const uint64_t *k, int64_t m, uint64_t *fl) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const bool head = i == 0 || (k[i] >> 33) != (k[i - 1] >> 33);
    fl[i] = ((uint64_t)head << 32) | (uint64_t)(((k[i] >> 32) & 1) == 0);
}

// from the exclusive scan of the flags: row e's id and its deletion and
// insertion ranges; the dst lists split by kind (each ascending per row)
__global__ void k_edit_scatter(const uint64_t *k, const uint64_t *sc, int64_t m, int32_t *rows,
                               int64_t *dptr, int64_t *iptr, int32_t *del, int32_t *ins,
                               int64_t *ne_out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const bool head = i == 0 || (k[i] >> 33) != (k[i - 1] >> 33);
    const bool isdel = ((k[i] >> 32) & 1) == 0;
    const int64_t e = (int64_t)(sc[i] >> 32), dc = (int64_t)(sc[i] & 0xffffffffu);
    if (head) {
        rows[e] = (int32_t)(k[i] >> 33);
        dptr[e] = dc;
        iptr[e] = i - dc;
    }
    if (isdel) del[dc] = (int32_t)(uint32_t)k[i];
    else ins[i - dc] = (int32_t)(uint32_t)k[i];
    if (i == m - 1) {
        const int64_t ne = e + head, nd = dc + isdel;
        dptr[ne] = nd;
        iptr[ne] = m - nd;
        *ne_out = ne;
    }
}

// capacity plan per edited row: the merged length, the relocation capacity
// when it outgrows its slack (0 if it fits) and its scratch size
__global__ void k_cap_plan(const int32_t *rows, const int64_t *ne_p, const int64_t *dptr,
                           const int64_t *iptr, const int32_t *rlen, const int32_t *rcap,
                           int64_t *need, int64_t *tsz) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t ne = *ne_p;
    if (e > ne) return;
    if (e == ne) { need[e] = tsz[e] = 0; return; }
    const int32_t v = rows[e];
    const int64_t L = rlen[v];
    const int64_t nl = L - (dptr[e + 1] - dptr[e]) + (iptr[e + 1] - iptr[e]);
    need[e] = nl > rcap[v] ? nl + max((int64_t)2, nl / 8) : 0;
    tsz[e] = max(nl, L);
}

// summary for the host: rows, relocation slots, relocated rows, scratch size
__global__ void k_cap_summary(const int64_t *ne_p, const int64_t *need, const int64_t *need_off,
                              const int64_t *toff, int64_t *out) {
    __shared__ unsigned long long nover;
    const int64_t ne = *ne_p;
    if (threadIdx.x == 0) nover = 0;
    __syncthreads();
    unsigned long long c = 0;
    for (int64_t e = threadIdx.x; e < ne; e += blockDim.x) c += need[e] > 0;
    atomicAdd(&nover, c);
    __syncthreads();
    if (threadIdx.x == 0) {
        out[0] = ne;
        out[1] = need_off[ne];
        out[2] = (int64_t)nover;
        out[3] = toff[ne];
    }
}

// move every row that outgrew its slack to tail + need_off[e]
__global__ void k_relocate_planned(const int32_t *rows, const int64_t *ne_p, const int64_t *need,
                                   const int64_t *need_off, int64_t tail, int64_t *indptr,
                                   const int32_t *rlen, int32_t *rcap, int32_t *indices) {
    const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= *ne_p || need[e] == 0) return;
    const int32_t v = rows[e];
    const int64_t a = indptr[v], b = tail + need_off[e];
    const int64_t L = rlen[v];
    for (int64_t j = lane; j < L; j += 32) indices[b + j] = indices[a + j];
    __syncwarp();
    if (lane == 0) {
        indptr[v] = b;
        rcap[v] = (int32_t)min(need[e], (int64_t)INT32_MAX);
    }
}

// re-spread slack: each edited row gets room for its insertions
__global__ void k_extra_from_edits(const int32_t *rows, const int64_t *ne_p, const int64_t *iptr,
                                   int32_t *extra) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e < *ne_p) extra[rows[e]] = (int32_t)(iptr[e + 1] - iptr[e]);
}

}  // namespace

// Edits already on the device (ins / dels: (m, 2) int64 rows, validated):
// grouped by source row, capacity planned, rows relocated and merged, SELL
// patched -- one small host read (the plan's totals) in the whole call.
void apply_batch_dev(Graph &g, const int64_t *ins, int64_t n_ins, const int64_t *dels,
                     int64_t n_dels) {
    cudaStream_t st = g.stream;
    const int64_t m = n_ins + n_dels;
    if (m == 0) return;
    PhaseTrace tr(st);
    DBuf<uint64_t> ka, kb, fl, sc;
    ka.alloc(m); kb.alloc(m); fl.alloc(m); sc.alloc(m);
    k_edit_keys<<<nblk(m, 256), 256, 0, st>>>(ins, n_ins, dels, n_dels, ka.p);
    note_launch();
    int hi = 1;
    while (hi < 31 && ((int64_t)1 << hi) < g.n) hi++;
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortKeys(t, b, ka.p, kb.p, (int)m, 0, 33 + hi, st);
    });
    k_edit_flags<<<nblk(m, 256), 256, 0, st>>>(kb.p, m, fl.p);
    note_launch();
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, fl.p, sc.p, (int)m, st);
    });
    DBuf<int32_t> drows, ddel, dins;
    DBuf<int64_t> ddptr, diptr, ne_d, need, need_off, tsz, toff, summ;
    drows.alloc(m); ddel.alloc(std::max<int64_t>(1, n_dels)); dins.alloc(std::max<int64_t>(1, n_ins));
    ddptr.alloc(m + 1); diptr.alloc(m + 1); ne_d.alloc(1);
    need.alloc(m + 1); need_off.alloc(m + 1); tsz.alloc(m + 1); toff.alloc(m + 1); summ.alloc(4);
    k_edit_scatter<<<nblk(m, 256), 256, 0, st>>>(kb.p, sc.p, m, drows.p, ddptr.p, diptr.p, ddel.p,
                                                 dins.p, ne_d.p);
    note_launch();
    tr.mark("  group edits");
    // capacity check (slack CSR); re-spread once if any edited row overflows
    if (!g.slack) respread(g, nullptr);
    k_cap_plan<<<nblk(m + 1, 256), 256, 0, st>>>(drows.p, ne_d.p, ddptr.p, diptr.p, g.rlen.p,
                                                 g.rcap.p, need.p, tsz.p);
    note_launch();
    // rows past ne hold garbage; the scans over m + 1 are read up to ne only
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, need.p, need_off.p, (int)(m + 1), st);
    });
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, tsz.p, toff.p, (int)(m + 1), st);
    });
    k_cap_summary<<<1, 1024, 0, st>>>(ne_d.p, need.p, need_off.p, toff.p, summ.p);
    note_launch();
    int64_t hs[4];
    KB_CUDA(cudaMemcpyAsync(hs, summ.p, sizeof(hs), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    const int64_t ne = hs[0], need_total = hs[1], n_over = hs[2], tmp_total = hs[3];
    tr.mark("  capacity check");
    if (n_over && g.tail + need_total <= (int64_t)g.indices.n) {
        k_relocate_planned<<<nblk(ne * 32, 256), 256, 0, st>>>(drows.p, ne_d.p, need.p,
                                                               need_off.p, g.tail, g.indptr.p,
                                                               g.rlen.p, g.rcap.p, g.indices.p);
        note_launch();
        g.tail += need_total;
        tr.mark("  relocate rows");
    } else if (n_over) {
        // the tail is full: re-spread everything (with fresh tail room)
        DBuf<int32_t> dex;
        dex.alloc(g.n);
        KB_CUDA(cudaMemsetAsync(dex.p, 0, g.n * 4, st));
        k_extra_from_edits<<<nblk(ne, 256), 256, 0, st>>>(drows.p, ne_d.p, diptr.p, dex.p);
        note_launch();
        respread(g, dex.p);
        KB_CUDA(cudaStreamSynchronize(st));
        tr.mark("  respread");
    }
    DBuf<int32_t> tmp;
    tmp.alloc(std::max<int64_t>(1, tmp_total));
    k_apply_edits<<<(unsigned)ne, 128, 0, st>>>(drows.p, ne, ddptr.p, ddel.p, diptr.p, dins.p,
                                                toff.p, tmp.p, g.indptr.p, g.indices.p, g.rlen.p,
                                                g.rcap.p, (int64_t)g.indices.n);
    note_launch();
    KB_CUDA(cudaGetLastError());
    tr.mark("  edit rows");
    g.nnz += n_ins - n_dels;
    patch_sell(g, drows.p, ne);
    KB_CUDA(cudaStreamSynchronize(st));
    tr.mark("  patch SELL");
    g.mutated = true;
    g.version += 1;
}

void apply_batch_to_graph(Graph &g, const int64_t *ins, int64_t n_ins, const int64_t *dels,
                          int64_t n_dels) {
    if (n_ins + n_dels == 0) return;
    cudaStream_t st = g.stream;
    DBuf<int64_t> di, dd;
    di.alloc(std::max<int64_t>(1, 2 * n_ins));
    dd.alloc(std::max<int64_t>(1, 2 * n_dels));
    if (n_ins) KB_CUDA(cudaMemcpyAsync(di.p, ins, n_ins * 16, cudaMemcpyHostToDevice, st));
    if (n_dels) KB_CUDA(cudaMemcpyAsync(dd.p, dels, n_dels * 16, cudaMemcpyHostToDevice, st));
    apply_batch_dev(g, di.p, n_ins, dd.p, n_dels);
}

namespace {
struct BitsDiffer {
    const double *a, *b;
    __device__ bool operator()(int32_t v) const {
        return __double_as_longlong(a[v]) != __double_as_longlong(b[v]);
    }
};
}  // namespace

// rows whose value differs bit-wise, ascending, and their count (a device
// select: one decoupled-lookback pass instead of an atomic per warp)
static void diff_changed(const double *old, const double *nw, int64_t n, int32_t *changed,
                         unsigned long long *count, cudaStream_t st) {
    DBuf<int64_t> c64;
    c64.alloc(1);
    cub::CountingInputIterator<int32_t> it(0);
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceSelect::If(t, b, it, changed, c64.p, (int)n, BitsDiffer{old, nw}, st);
    });
    KB_CUDA(cudaMemcpyAsync(count, c64.p, 8, cudaMemcpyDeviceToDevice, st));
}

void update_batch(State &s, const int64_t *ins, int64_t n_ins, const int64_t *dels,
                  int64_t n_dels, double theta, double new_gamma, kb_update_stats *stats) {
    NvtxRange nv("K4 update_batch");
    Graph &g = *s.g;
    cudaStream_t st = g.stream;
    const int64_t n = g.n;
    KB_REQUIRE(s.keep_all, KB_ESTATE, "dynamic updates need keep_all_levels=True");
    KB_REQUIRE(s.r >= 1, KB_ESTATE, "run the static engine before applying updates");
    KB_REQUIRE(g.version == s.graph_version, KB_ESTATE,
               "state does not belong to this graph revision");
    KB_REQUIRE(theta >= 0.0 && theta <= 1.0, KB_EPARAM, "theta must be in [0, 1]");
    kb_update_stats st_out{};
    s.level_sizes.clear();
    st_out.batch_size = n_ins + n_dels;
    st_out.aborted_level = -1;

    // the batch on the device once: seeds (sources) and targets, deduplicated
    // in original-id order and mapped to new ids, and the edits themselves
    const int64_t m = n_ins + n_dels;
    DBuf<int64_t> d_ins, d_dels;
    d_ins.alloc(std::max<int64_t>(1, 2 * n_ins));
    d_dels.alloc(std::max<int64_t>(1, 2 * n_dels));
    if (n_ins) KB_CUDA(cudaMemcpyAsync(d_ins.p, ins, n_ins * 16, cudaMemcpyHostToDevice, st));
    if (n_dels) KB_CUDA(cudaMemcpyAsync(d_dels.p, dels, n_dels * 16, cudaMemcpyHostToDevice, st));
    DBuf<int32_t> dseeds, dtargets;
    int64_t ns = 0, nt = 0;
    {
        DBuf<int32_t> ends, sorted, uniq;
        DBuf<int64_t> cnt2;
        ends.alloc(std::max<int64_t>(1, 2 * m));
        sorted.alloc(std::max<int64_t>(1, 2 * m));
        uniq.alloc(std::max<int64_t>(1, 2 * m));
        cnt2.alloc(2);
        dseeds.alloc(std::max<int64_t>(1, m));
        dtargets.alloc(std::max<int64_t>(1, m));
        KB_CUDA(cudaMemsetAsync(cnt2.p, 0, 16, st));
        if (m) {
            k_batch_ends<<<nblk(m, 256), 256, 0, st>>>(d_ins.p, n_ins, d_dels.p, n_dels, ends.p);
            note_launch();
            int hi = 1;
            while (hi < 31 && ((int64_t)1 << hi) < n) hi++;
            for (int side = 0; side < 2; side++) {
                cub_run([&](void *t, size_t &b) {
                    return cub::DeviceRadixSort::SortKeys(t, b, ends.p + side * m,
                                                          sorted.p + side * m, (int)m, 0, hi, st);
                });
                cub_run([&](void *t, size_t &b) {
                    return cub::DeviceSelect::Unique(t, b, sorted.p + side * m, uniq.p + side * m,
                                                     cnt2.p + side, (int)m, st);
                });
            }
        }
        int64_t hc[2];
        KB_CUDA(cudaMemcpyAsync(hc, cnt2.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        ns = hc[0];
        nt = hc[1];
        if (ns) k_map_new<<<nblk(ns, 256), 256, 0, st>>>(uniq.p, ns, g.iperm.p, dseeds.p);
        if (nt) k_map_new<<<nblk(nt, 256), 256, 0, st>>>(uniq.p + m, nt, g.iperm.p, dtargets.p);
        note_launch(2);
    }
    st_out.seeds = ns;

    PhaseTrace tr(st);
    // 1. the post-batch arc set on the device
    const bool was_sym = g.symmetric == 1;
    apply_batch_dev(g, d_ins.p, n_ins, d_dels.p, n_dels);
    tr.mark("apply batch");
    if (!(was_sym && s.undirected)) g.symmetric = -1;
    // in-neighbours: the CSR itself when undirected (symmetric), else a transpose
    DBuf<int64_t> tip;
    DBuf<int32_t> tix;
    const int64_t *in_ip = g.indptr.p;
    const int32_t *in_len = g.rlen.p;
    const int32_t *in_ix = g.indices.p;
    if (!s.undirected) {
        build_transpose(g, tip, tix);
        in_ip = tip.p;
        in_len = nullptr;
        in_ix = tix.p;
    }

    // 2. level repair
    DBuf<int32_t> stamp, R, C, HR;
    DBuf<unsigned int> aff;
    DBuf<unsigned char> touched;
    DBuf<unsigned long long> cnt;  // [0]=|R|, [1]=|changed|, [2]=|affected|
    stamp.alloc(n); R.alloc(n); C.alloc(n); HR.alloc(std::max<int64_t>(1, g.nh)); aff.alloc((n + 31) / 32 + 1); touched.alloc(n);
    cnt.alloc(4);
    KB_CUDA(cudaMemsetAsync(stamp.p, 0xff, n * 4, st));
    KB_CUDA(cudaMemsetAsync(aff.p, 0, ((n + 31) / 32 + 1) * 4, st));
    KB_CUDA(cudaMemsetAsync(touched.p, 0, n, st));
    KB_CUDA(cudaMemsetAsync(cnt.p, 0, 4 * 8, st));
    if (ns) {
        k_affect<<<nblk(ns, 256), 256, 0, st>>>(dseeds.p, ns, aff.p, cnt.p + 2);
        note_launch();
    }
    int64_t affected = ns;
    const int64_t aff_words = (n + 31) / 32 + 1;
    auto recount_affected = [&] {   // cnt[2] = |affected| from the bitmap
        KB_CUDA(cudaMemsetAsync(cnt.p + 2, 0, 8, st));
        k_popc_count<<<(unsigned)std::min<int64_t>(nblk(aff_words, 256), 4 * g.sm_count), 256, 0,
                       st>>>(aff.p, aff_words, cnt.p + 2);
        note_launch();
    };
    bool aborted = false;
    bool all_touched = false;
    DBuf<unsigned int> chg_bits;
    chg_bits.alloc((n + 31) / 32 + 1);
    int64_t nchanged = 0;
    for (int64_t level = 1; level <= s.r; level++) {
        double *w_prev = s.levels[level - 1 - s.level_base].p;
        double *w_cur = s.levels[level - s.level_base].p;
        if (aborted || (double)affected > theta * (double)n) {  // dynamic.py:58-60, :78
            if (!aborted) {
                aborted = true;
                st_out.aborted_level = level;
            }
            run_spmv(s, st, w_prev, w_cur, true);
            KB_CUDA(cudaStreamSynchronize(st));
            tr.mark("level (full K1)");
            continue;
        }
        if (st_out.n_level_sizes < 64) st_out.level_sizes[st_out.n_level_sizes] = affected;
        st_out.n_level_sizes++;
        s.level_sizes.push_back(affected);
        bool dense = nchanged > n / 256;
        if (!dense && nchanged) {
            // a few hubs can carry most of the arcs: decide by the expansion's
            // arc count (a warp per changed row would serialise on them)
            KB_CUDA(cudaMemsetAsync(cnt.p + 3, 0, 8, st));
            k_work_sum<<<nblk(nchanged, 256), 256, 0, st>>>(C.p, nchanged, in_ip, in_len,
                                                            g.perm.p, cnt.p + 3);
            note_launch();
            unsigned long long work = 0;
            KB_CUDA(cudaMemcpyAsync(&work, cnt.p + 3, 8, cudaMemcpyDeviceToHost, st));
            KB_CUDA(cudaStreamSynchronize(st));
            dense = (int64_t)work > std::max<int64_t>(g.nnz / tune_get("dyn.dense_div", 64), 1 << 20);
            if (tr.on) fprintf(stderr, "[kb]   level %lld: %lld changed rows, %llu in-arcs\n",
                               (long long)level, (long long)nchanged, work);
        }
        if (dense) {
            // Dense level: the expansion would reach most rows, so recompute
            // the whole level with K1 (identical bits for every row) and
            // find the changed rows by comparison.  The affected set grows by
            // the in-neighbours of the previous changed rows, found by a pull
            // over every row's out-arcs (u in N-(v) <=> v in N+(u)).
            KB_CUDA(cudaMemsetAsync(chg_bits.p, 0, chg_bits.bytes(), st));
            k_bits_from_list<<<nblk(nchanged, 256), 256, 0, st>>>(C.p, nchanged, g.perm.p,
                                                                  chg_bits.p);
            k_pull_affect<<<nblk(n, 256), 256, 0, st>>>(g.indptr.p, g.rlen.p, g.indices.p,
                                                        g.iperm.p, n, chg_bits.p, aff.p,
                                                        cnt.p + 2);
            note_launch(2);
            DBuf<double> fresh;
            fresh.alloc(n + 1);
            run_spmv(s, st, w_prev, fresh.p, true);
            diff_changed(w_cur, fresh.p, n, C.p, cnt.p + 1, st);
            std::swap(s.levels[level - s.level_base], fresh);
            recount_affected();
            unsigned long long hc[3];
            KB_CUDA(cudaMemcpyAsync(hc, cnt.p, 3 * 8, cudaMemcpyDeviceToHost, st));
            KB_CUDA(cudaStreamSynchronize(st));
            nchanged = (int64_t)hc[1];
            affected = (int64_t)hc[2];
            all_touched = true;
            tr.mark("level (dense repair)");
            continue;
        }
        // R_level = seeds U in-neighbours(changed at level-1)
        KB_CUDA(cudaMemsetAsync(cnt.p, 0, 2 * 8, st));
        if (ns) {
            k_mark_list<<<nblk(ns, 256), 256, 0, st>>>(dseeds.p, ns, stamp.p, (int32_t)level,
                                                       R.p, cnt.p, touched.p);
            note_launch();
        }
        if (nchanged) {
            k_expand<<<nblk(nchanged * 32 * EXPAND_SPLIT, 256), 256, 0, st>>>(
                C.p, nchanged, in_ip, in_len, in_ix, g.perm.p, g.iperm.p, stamp.p, (int32_t)level,
                R.p, cnt.p, aff.p, cnt.p + 2, touched.p);
            note_launch();
        }
        recount_affected();
        unsigned long long hc[3];
        KB_CUDA(cudaMemcpyAsync(hc, cnt.p, 3 * 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        const int64_t nr = (int64_t)hc[0];
        affected = (int64_t)hc[2];
        if (tr.on) fprintf(stderr, "[kb]   level %lld: frontier %lld rows\n", (long long)level,
                           (long long)nr);
        if (nr > n / 64) {
            // a wide frontier: one K1 level (same bits) is cheaper than a
            // warp per row; the changed rows come from the comparison
            DBuf<double> fresh;
            fresh.alloc(n + 1);
            run_spmv(s, st, w_prev, fresh.p, true);
            diff_changed(w_cur, fresh.p, n, C.p, cnt.p + 1, st);
            std::swap(s.levels[level - s.level_base], fresh);
            unsigned long long hchg = 0;
            KB_CUDA(cudaMemcpyAsync(&hchg, cnt.p + 1, 8, cudaMemcpyDeviceToHost, st));
            KB_CUDA(cudaStreamSynchronize(st));
            nchanged = (int64_t)hchg;
            all_touched = true;
            tr.mark("level (wide frontier)");
            continue;
        }
        // recompute R at this level; the changed list feeds the next level
        KB_CUDA(cudaMemsetAsync(cnt.p + 1, 0, 8, st));
        if (nr) {
            // heavy rows fold their SELL segments (only while the layout is current)
            const bool seg_ok = !g.sell_dirty && g.nh > 0 && g.sell.nseg > 0;
            KB_CUDA(cudaMemsetAsync(cnt.p + 3, 0, 8, st));
            k_recompute<<<nblk(nr * 32, 256), 256, 0, st>>>(
                R.p, nr, g.perm.p, g.iperm.p, g.indptr.p, g.rlen.p, g.indices.p, w_prev, w_cur,
                s.alpha, g.split, C.p, cnt.p + 1, g.h_of_row.p, g.ovf_flag.p,
                seg_ok ? HR.p : nullptr, cnt.p + 3);
            note_launch();
            if (seg_ok) {
                unsigned long long hh = 0;
                KB_CUDA(cudaMemcpyAsync(&hh, cnt.p + 3, 8, cudaMemcpyDeviceToHost, st));
                KB_CUDA(cudaStreamSynchronize(st));
                if ((int64_t)hh > tune_get("dyn.heavy_dense", 256)) {
                    // many heavy rows: all segment sums by K1 (~45% of a
                    // level), then each listed row combined and compared
                    run_segments(s, st, w_prev);
                    k_heavy_finish<<<nblk((int64_t)hh * 32, 256), 256, 0, st>>>(
                        HR.p, (int64_t)hh, w_cur, s.alpha, g.h_of_row.p, g.seg_ptr.p,
                        g.seg_list.p, s.seg_sum.p, C.p, cnt.p + 1);
                    note_launch();
                    tr.mark("heavy rows (segment pass)");
                } else if (hh) {
                    k_heavy_rows_fold<<<(unsigned)hh, 256, 0, st>>>(
                        HR.p, w_prev, w_cur, s.alpha, g.h_of_row.p, g.seg_ptr.p, g.seg_list.p,
                        g.sell.slice_off.p, g.sell.slice_w.p, g.sell.vlen.p, g.sell.cols.p, C.p,
                        cnt.p + 1);
                    note_launch();
                }
            }
        }
        unsigned long long hchg = 0;
        KB_CUDA(cudaMemcpyAsync(&hchg, cnt.p + 1, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        nchanged = (int64_t)hchg;
        tr.mark("level (local repair)");
    }
    // visited = |affected U targets| (dynamic.py:176)
    {
        if (nt) {
            k_affect<<<nblk(nt, 256), 256, 0, st>>>(dtargets.p, nt, aff.p, cnt.p + 2);
            note_launch();
        }
        recount_affected();
        unsigned long long ha = 0;
        KB_CUDA(cudaMemcpyAsync(&ha, cnt.p + 2, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        st_out.visited = (int64_t)ha;
    }

    tr.mark("visited count");
    // 3. katz and bounds (dynamic.py:181-187)
    std::vector<const double *> hl(s.r + 1);
    for (int64_t l = 0; l <= s.r; l++) hl[l] = s.levels[l - s.level_base].p;
    DBuf<const double *> dl;
    dl.alloc(s.r + 1);
    KB_CUDA(cudaMemcpyAsync(dl.p, hl.data(), (s.r + 1) * sizeof(double *), cudaMemcpyHostToDevice,
                            st));
    const bool gamma_changed = new_gamma != s.gamma;
    s.gamma = new_gamma;
    const double *wr = s.levels[s.r - s.level_base].p;
    if (aborted || all_touched) {
        k_katz_rows<<<nblk(n, 256), 256, 0, st>>>(nullptr, n, dl.p, (int)s.r, s.katz.p);
        k_bounds_rows<<<nblk(n, 256), 256, 0, st>>>(nullptr, n, s.katz.p, wr, s.alpha, s.gamma,
                                                    s.undirected, s.lower.p, s.upper.p);
        note_launch(2);
    } else {
        DBuf<int32_t> tl, iota;
        DBuf<int64_t> tn;
        tl.alloc(n); iota.alloc(n); tn.alloc(1);
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceSelect::Flagged(t, b, cub::CountingInputIterator<int32_t>(0),
                                              touched.p, tl.p, tn.p, (int)n, st);
        });
        int64_t ntouch = 0;
        KB_CUDA(cudaMemcpyAsync(&ntouch, tn.p, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        if (ntouch) {
            k_katz_rows<<<nblk(ntouch, 256), 256, 0, st>>>(tl.p, ntouch, dl.p, (int)s.r, s.katz.p);
            note_launch();
        }
        if (gamma_changed) {
            k_bounds_rows<<<nblk(n, 256), 256, 0, st>>>(nullptr, n, s.katz.p, wr, s.alpha,
                                                        s.gamma, s.undirected, s.lower.p,
                                                        s.upper.p);
            note_launch();
        } else if (ntouch) {
            k_bounds_rows<<<nblk(ntouch, 256), 256, 0, st>>>(tl.p, ntouch, s.katz.p, wr, s.alpha,
                                                             s.gamma, s.undirected, s.lower.p,
                                                             s.upper.p);
            note_launch();
        }
    }
    KB_CUDA(cudaGetLastError());

    tr.mark("katz + bounds");
    // 4. reactivation (dynamic.py:190-197)
    if ((s.kind == KB_RANKING || s.kind == KB_TOPK) && !s.act_dense && s.m_host < n) {
        const int64_t m = s.m_host;
        DBuf<unsigned char> inact, flag;
        DBuf<unsigned long long> mn;
        DBuf<int64_t> nb;
        inact.alloc(n); flag.alloc(n); mn.alloc(1); nb.alloc(1);
        KB_CUDA(cudaMemsetAsync(inact.p, 0, n, st));
        KB_CUDA(cudaMemsetAsync(mn.p, 0xff, 8, st));
        if (m) {
            k_flags_from_list<<<nblk(m, 256), 256, 0, st>>>(s.act[s.cur].p, m, inact.p);
            k_min_lower<<<2 * g.sm_count, 256, 0, st>>>(s.act[s.cur].p, m, s.lower.p, mn.p);
            note_launch(2);
        }
        k_reactivate_flags<<<nblk(n, 256), 256, 0, st>>>(g.iperm.p, n, inact.p, s.upper.p, mn.p,
                                                        s.eps, flag.p);
        note_launch();
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceSelect::Flagged(t, b, g.iperm.p, flag.p, s.act[s.cur].p + m, nb.p,
                                              (int)n, st);
        });
        int64_t back = 0;
        KB_CUDA(cudaMemcpyAsync(&back, nb.p, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        s.m_host = m + back;
        st_out.reactivated = back;
    }

    // 5. the relabelling is no longer degree-sorted: no static shortcuts
    s.zero_tail_exact = false;
    s.tail_zero_from = n;
    s.graph_version = g.version;

    tr.mark("reactivation");
    // 6. resume (dynamic.py:203-210)
    for (;;) {
        if (run_check(s, st)) break;
        if (s.r >= s.max_iter) {
            *stats = st_out;
            const double gap = run_gap(s, st);
            char buf[160];
            snprintf(buf, sizeof buf,
                     "stopping rule unmet after resuming to %lld iterations (gap %.3e)",
                     (long long)s.r, gap);
            throw Error{KB_ECONVERGENCE, buf};
        }
        launch_iterate(s, st);
        st_out.resumed_iterations++;
    }
    tr.mark("resume (checks)");
    *stats = st_out;
}

}  // namespace kb
