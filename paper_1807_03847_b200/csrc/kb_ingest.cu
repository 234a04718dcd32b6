// Graph ingest: canonical CSR -> device SELL-32 over degree-relabelled rows
// (replaces Graph.out_csr, graph.py:177-197).
//
// The canonical CSR is kept on the device as a CSR-with-slack: row v owns
// the slots [indptr[v], indptr[v+1]) of `indices` and uses the first rlen[v]
// of them, ascending.  A fresh graph is compact (capacity == length); the
// first dynamic batch spreads it out with per-row slack (kb_dynamic.cu).
// The SELL layout K1 reads is (re)built from it by build_sell().
#include <cub/block/block_reduce.cuh>
#include <cub/cub.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <numeric>

#include "kb_internal.cuh"

namespace kb {

size_t Graph::device_bytes() const {
    return perm.bytes() + iperm.bytes() + deg.bytes() + indptr.bytes() + rlen.bytes() +
           indices.bytes() + sell.cols.bytes() + sell.slice_off.bytes() +
           sell.slice_w.bytes() + sell.vlen.bytes() + seg_ptr.bytes() + seg_list.bytes() +
           hrow.bytes() + vrow.bytes() + zrows.bytes() + orig_pos.bytes() + orig_zero.bytes();
}

namespace {

inline unsigned blocks_for(int64_t n, int t) {
    return (unsigned)std::max<int64_t>(1, (n + t - 1) / t);
}

__global__ void k_rlen_compact(const int64_t *indptr, int64_t n, int32_t *rlen) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v < n) rlen[v] = (int32_t)(indptr[v + 1] - indptr[v]);
}

__global__ void k_degree_key(const int32_t *rlen, int64_t n, uint32_t *key, int32_t *ids) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    key[v] = 0xFFFFFFFFu - (uint32_t)rlen[v];  // ascending key == descending degree
    ids[v] = (int32_t)v;
}

__global__ void k_iota_pair(int64_t n, int32_t *a, int32_t *b) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) a[i] = b[i] = (int32_t)i;
}

__global__ void k_invert(const int32_t *perm, int64_t n, int32_t *iperm) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) iperm[perm[i]] = (int32_t)i;
}

__global__ void k_len_by_new(const int32_t *rlen, const int32_t *perm, int64_t n, int32_t *deg) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) deg[i] = rlen[perm[i]];
}

// first index in the descending array whose value <= bound
__device__ int64_t first_le(const int32_t *a, int64_t n, int64_t bound) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] <= bound) hi = mid; else lo = mid + 1;
    }
    return lo;
}

__global__ void k_counts(const int32_t *sdeg, int64_t n, int64_t split, int64_t *out) {
    out[0] = first_le(sdeg, n, 0);      // rows with arcs
    out[1] = first_le(sdeg, n, split);  // rows longer than split
}

__global__ void k_max(const int32_t *a, int64_t n, unsigned long long *out) {
    typedef cub::BlockReduce<int, 256> Red;
    __shared__ typename Red::TempStorage tmp;
    int m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, a[i]);
    m = Red(tmp).Reduce(m, cub::Max());
    if (threadIdx.x == 0) atomicMax(out, (unsigned long long)m);
}

// classify rows by new id: heavy (len > split), normal (0 < len <= split), empty
__global__ void k_row_class(const int32_t *deg, int64_t n, int64_t split, unsigned char *heavy,
                            unsigned char *normal, unsigned char *zero, int32_t *iota,
                            uint32_t *key, int64_t own_lo, int64_t own_hi) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int d = deg[v];
    heavy[v] = d > split;
    normal[v] = d > 0 && d <= split;
    zero[v] = d == 0 && v >= own_lo && v < own_hi;  // empty rows this device owns
    iota[v] = (int32_t)v;
    key[v] = d <= split ? (uint32_t)(split - d) : 0u;  // normal rows: descending length
}

__global__ void k_gather_keys(const uint32_t *key, const int32_t *ids, int64_t m, uint32_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) out[i] = key[ids[i]];
}

__global__ void k_vlen_normal(const int32_t *deg, const int32_t *vrow, int64_t nh, int64_t nnorm,
                              int64_t nseg, int32_t *vlen) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nnorm) return;
    vlen[nseg + i] = deg[vrow ? vrow[i] : nh + i];
}

__global__ void k_slice_width(const int32_t *vlen, int64_t nvr, int64_t nslices,
                              int32_t *slice_w, int64_t *slice_sz) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nslices) return;
    int w = 0;
    for (int l = 0; l < 32; l++) {
        int64_t vr = s * 32 + l;
        if (vr < nvr) w = max(w, vlen[vr]);
    }
    if (w > 4) w = (w + 3) & ~3;
    slice_w[s] = w;
    slice_sz[s] = (int64_t)w * 32;
}

// one warp per slice: lane l copies virtual row s*32+l into its column slots
__global__ void k_fill(const int64_t *indptr, const int32_t *indices, const int32_t *perm,
                       const int32_t *iperm, const int32_t *vlen, const int32_t *seg_row,
                       const int32_t *seg_start, const int32_t *hrow, const int32_t *vrow,
                       const int32_t *slice_w, const int64_t *slice_off, int64_t nslices,
                       int64_t nvr, int64_t nseg, int64_t nh, int32_t *cols) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= nslices) return;
    int64_t s = warp;
    int64_t vr = s * 32 + lane;
    int len = 0;
    int64_t src = 0;
    if (vr < nvr) {
        len = vlen[vr];
        int64_t row_new, start = 0;
        if (vr < nseg) {
            const int32_t h = seg_row[vr];
            row_new = hrow ? hrow[h] : h;
            start = seg_start[vr];
        } else {
            row_new = vrow ? vrow[vr - nseg] : nh + (vr - nseg);
        }
        src = indptr[perm[row_new]] + start;
    }
    int w = slice_w[s];
    int32_t *base = cols + slice_off[s];
    // eight columns per step with every load issued before the first use:
    // the column ids, then their relabelled ids (a random gather), then the
    // stores -- a step costs two memory latencies instead of sixteen
    for (int j0 = 0; j0 < w; j0 += 8) {
        int32_t r[8], c[8];
#pragma unroll
        for (int q = 0; q < 8; q++) r[q] = (j0 + q < len) ? indices[src + j0 + q] : -1;
#pragma unroll
        for (int q = 0; q < 8; q++) c[q] = r[q] >= 0 ? iperm[r[q]] : 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const int j = j0 + q;
            if (j < w) {
                const int64_t pos = (w <= 4) ? ((int64_t)j * 32 + lane)
                                             : ((int64_t)(j >> 2) * 128 + lane * 4 + (j & 3));
                base[pos] = c[q];
            }
        }
    }
}

__global__ void k_rev_normal(const int32_t *vrow, int64_t nh, int64_t nnorm, int64_t nseg,
                             int32_t *vr_of_row) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nnorm) vr_of_row[vrow ? vrow[i] : nh + i] = (int32_t)(nseg + i);
}

__global__ void k_rev_heavy(const int32_t *hrow, int64_t nh, int32_t *h_of_row) {
    int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (h < nh) h_of_row[hrow ? hrow[h] : h] = (int32_t)h;
}

// One thread per edited row (original id): rewrite its SELL lane in place
// when the new length fits the slice, else turn it into an overflow row
// (its SELL lane / segments contribute 0 and the overflow pass recomputes it)
__global__ void k_patch_rows(const int32_t *rows_orig, int64_t ne, const int32_t *iperm,
                             const int64_t *indptr, const int32_t *rlen, const int32_t *indices,
                             const int32_t *vr_of_row, const int32_t *h_of_row,
                             const int32_t *seg_ptr, const int32_t *seg_list,
                             const int32_t *slice_w, const int64_t *slice_off, int32_t *vlen,
                             int32_t *cols, int32_t *ovf_flag, int32_t *ovf,
                             unsigned long long *ovf_count, int64_t split, int32_t *heavy,
                             unsigned long long *heavy_count) {
    // a warp per edited row: the lanes rewrite a fitting row's slots
    const int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (e >= ne) return;
    const int32_t o = rows_orig[e];
    const int32_t v = iperm[o];
    if (ovf_flag[v]) return;  // already recomputed from the canonical CSR
    const int32_t len = rlen[o];
    const int32_t vr = vr_of_row[v];
    if (vr >= 0) {
        const int64_t s = vr >> 5;
        const int sl = vr & 31;
        const int w = slice_w[s];
        if (len <= w) {
            int32_t *base = cols + slice_off[s];
            const int32_t *row = indices + indptr[o];
            for (int j = lane; j < len; j += 32) {
                const int64_t pos = (w <= 4) ? ((int64_t)j * 32 + sl)
                                             : ((int64_t)(j >> 2) * 128 + sl * 4 + (j & 3));
                base[pos] = iperm[row[j]];
            }
            if (lane == 0) vlen[vr] = len;
            return;
        }
        if (lane == 0) vlen[vr] = 0;
    } else if (h_of_row[v] >= 0) {
        // a heavy row keeps its segments while the count of full ones is
        // unchanged and the remainder fits the partial segment's lane (or
        // is 0): k_patch_heavy rewrites them in place
        const int32_t h = h_of_row[v];
        const int q0 = seg_ptr[h], nq = seg_ptr[h + 1] - q0;
        const int32_t last = seg_list[q0 + nq - 1];
        const int F = vlen[last] < split ? nq - 1 : nq;
        const int64_t rem = (int64_t)len - (int64_t)F * split;
        bool fits = false;
        if (rem >= 0 && rem < split)
            fits = (nq == F + 1) ? rem <= slice_w[last >> 5] : rem == 0;
        if (fits) {
            if (lane == 0) heavy[atomicAdd(heavy_count, 1ull)] = v;
            return;
        }
        for (int q = q0 + lane; q < q0 + nq; q += 32) vlen[seg_list[q]] = 0;
    }
    if (lane == 0 && atomicExch(&ovf_flag[v], 1) == 0) ovf[atomicAdd(ovf_count, 1ull)] = v;
}

// rewrite the SELL segments of an edited heavy row (new id rows[blockIdx.x])
__global__ void k_patch_heavy(const int32_t *rows, const int32_t *perm, const int64_t *indptr,
                              const int32_t *rlen, const int32_t *indices, const int32_t *iperm,
                              const int32_t *h_of_row, const int32_t *seg_ptr,
                              const int32_t *seg_list, const int32_t *slice_w,
                              const int64_t *slice_off, int64_t split, int32_t *vlen,
                              int32_t *cols) {
    const int32_t v = rows[blockIdx.x];
    const int32_t o = perm[v];
    const int32_t h = h_of_row[v];
    const int q0 = seg_ptr[h], nq = seg_ptr[h + 1] - q0;
    const int32_t *row = indices + indptr[o];
    const int64_t L = rlen[o];
    for (int64_t j = threadIdx.x; j < L; j += blockDim.x) {
        const int64_t q = j / split, jj = j - q * split;
        const int32_t vr = seg_list[q0 + q];
        const int64_t s = vr >> 5;
        const int ln = vr & 31;
        const int w = slice_w[s];
        const int64_t pos = (w <= 4) ? jj * 32 + ln : (jj >> 2) * 128 + ln * 4 + (jj & 3);
        cols[slice_off[s] + pos] = iperm[row[j]];
    }
    for (int q = threadIdx.x; q < nq; q += blockDim.x) {
        const int64_t a = (int64_t)q * split;
        vlen[seg_list[q0 + q]] = (int32_t)(L > a ? min(split, L - a) : 0);
    }
}

__global__ void k_ovf_long_list(const int32_t *ovf, int64_t n_ovf, const int32_t *perm,
                                const int32_t *rlen, int32_t *out, unsigned long long *count) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n_ovf && rlen[perm[ovf[i]]] > OVF_LONG) out[atomicAdd(count, 1ull)] = ovf[i];
}

__global__ void k_count_above(const int32_t *deg, int64_t m, int64_t thr,
                              unsigned long long *count) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool above = i < m && deg[i] > thr;
    const unsigned b = __ballot_sync(0xffffffffu, above);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(count, (unsigned long long)__popc(b));
}

// trace only: total and longest length of the overflow rows, rows > split
__global__ void k_ovf_stats(const int32_t *ovf, int64_t n_ovf, const int32_t *perm,
                            const int32_t *rlen, int64_t split, unsigned long long *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_ovf) return;
    const unsigned long long L = (unsigned long long)rlen[perm[ovf[i]]];
    atomicAdd(&out[0], L);
    atomicMax(&out[1], L);
    if ((int64_t)L > split) atomicAdd(&out[2], 1ull);
}

__global__ void k_arc_flags(const int32_t *rlen, int64_t n, unsigned char *fl, int32_t *iota) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    fl[v] = rlen[v] > 0;
    iota[v] = (int32_t)v;
}

__global__ void k_flip(unsigned char *fl, int64_t n) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v < n) fl[v] = !fl[v];
}

template <typename F>
void cub_run(F &&f) {
    size_t tb = 0;
    KB_CUDA(f(nullptr, tb));
    DBuf<unsigned char> tmp;
    tmp.alloc(tb);
    KB_CUDA(f(tmp.p, tb));
    note_launch();
}

// heavy row h: full[h] segments of T arcs plus one partial one if deg % T;
// the sort key orders partial segments by descending remainder (T: none)
__global__ void k_seg_counts(const int32_t *hdeg, int64_t nh, int64_t T, int32_t *full,
                             int32_t *tot, uint32_t *pkey, int32_t *hid) {
    int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (h > nh) return;
    if (h == nh) { full[h] = tot[h] = 0; return; }
    const int64_t d = hdeg[h], f = d / T, r = d % T;
    full[h] = (int32_t)f;
    tot[h] = (int32_t)(f + (r ? 1 : 0));
    pkey[h] = (uint32_t)(r ? T - r : T);
    hid[h] = (int32_t)h;
}

// partial segment ids follow the F full ones in sorted (remainder) order
__global__ void k_seg_rank(const int32_t *hid_sorted, const uint32_t *key_sorted, int64_t nh,
                           int64_t T, const int32_t *fstart, int32_t *pid) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nh && key_sorted[i] < (uint32_t)T) pid[hid_sorted[i]] = fstart[nh] + (int32_t)i;
}

__global__ void k_seg_fill(const int32_t *hdeg, int64_t nh, int64_t T, const int32_t *fstart,
                           const int32_t *seg_ptr, const int32_t *pid, int32_t *seg_row,
                           int32_t *seg_start, int32_t *seg_len, int32_t *seg_list) {
    int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (h >= nh) return;
    const int64_t d = hdeg[h], f = d / T, r = d % T;
    for (int64_t q = 0; q < f; q++) {
        const int32_t sid = fstart[h] + (int32_t)q;
        seg_row[sid] = (int32_t)h;
        seg_start[sid] = (int32_t)(q * T);
        seg_len[sid] = (int32_t)T;
        seg_list[seg_ptr[h] + q] = sid;
    }
    if (r) {
        const int32_t sid = pid[h];
        seg_row[sid] = (int32_t)h;
        seg_start[sid] = (int32_t)(f * T);
        seg_len[sid] = (int32_t)r;
        seg_list[seg_ptr[h] + f] = sid;
    }
}

// 1 + the last slice wider than 4 (0 if none)
__global__ void k_last_wide(const int32_t *slice_w, int64_t nslices, unsigned long long *out) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool wide = s < nslices && slice_w[s] > 4;
    if (__any_sync(0xffffffffu, wide)) {
        unsigned long long v = wide ? (unsigned long long)(s + 1) : 0ull;
        for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((threadIdx.x & 31) == 0) atomicMax(out, v);
    }
}

}  // namespace

// Virtual rows, slices and column slots for the current arc set under the
// current relabelling.  `fresh` means perm sorts rows by descending length,
// so heavy / normal / empty rows are the contiguous new-id ranges
// [0,nh) / [nh,nv) / [nv,n) and no explicit row maps are needed.
void build_sell(Graph &g, bool fresh, bool fill) {
    cudaStream_t st = g.stream;
    PhaseTrace tr(st);
    const int64_t n = g.n;
    if (!g.deg.p) g.deg.alloc(n);
    if (n) k_len_by_new<<<blocks_for(n, 256), 256, 0, st>>>(g.rlen.p, g.perm.p, n, g.deg.p);
    note_launch();
    g.hrow.release();
    g.vrow.release();
    g.zrows.release();
    g.implicit_rows = fresh;
    {
        DBuf<unsigned long long> mx;
        mx.alloc(1);
        KB_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long), st));
        k_max<<<2 * std::max(1, g.sm_count), 256, 0, st>>>(g.deg.p, n, mx.p);
        note_launch();
        unsigned long long hm = 0;
        KB_CUDA(cudaMemcpyAsync(&hm, mx.p, sizeof(hm), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        g.max_deg = (int64_t)hm;
    }
    if (fresh) {
        DBuf<int64_t> cnt;
        cnt.alloc(2);
        k_counts<<<1, 1, 0, st>>>(g.deg.p, n, g.split, cnt.p);
        note_launch();
        int64_t hc[2];
        KB_CUDA(cudaMemcpyAsync(hc, cnt.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        g.nv = hc[0];
        g.nh = hc[1];
        g.nzero = n - g.nv;
        // heavy rows are [0, nh) by descending length: the leading ones with
        // more than 8 segments get a warp each in the segment fold
        {
            DBuf<unsigned long long> c;
            c.alloc(1);
            KB_CUDA(cudaMemsetAsync(c.p, 0, 8, st));
            if (g.nh)
                k_count_above<<<blocks_for(g.nh, 256), 256, 0, st>>>(g.deg.p, g.nh, 8 * g.split,
                                                                   c.p);
            unsigned long long hl = 0;
            KB_CUDA(cudaMemcpyAsync(&hl, c.p, 8, cudaMemcpyDeviceToHost, st));
            KB_CUDA(cudaStreamSynchronize(st));
            g.nh_long = (int64_t)hl;
        }
    } else {
        g.nh_long = -1;
        DBuf<unsigned char> fh, fn, fz;
        DBuf<int32_t> iota, sel;
        DBuf<uint32_t> key, k2, k3;
        DBuf<int64_t> cnt;
        fh.alloc(n); fn.alloc(n); fz.alloc(n); iota.alloc(n); key.alloc(n); cnt.alloc(3);
        k_row_class<<<blocks_for(n, 256), 256, 0, st>>>(g.deg.p, n, g.split, fh.p, fn.p, fz.p,
                                                       iota.p, key.p, g.own_lo,
                                                       g.own_hi < 0 ? n : g.own_hi);
        note_launch();
        g.hrow.alloc(n); g.zrows.alloc(n); sel.alloc(n);
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceSelect::Flagged(t, b, iota.p, fh.p, g.hrow.p, cnt.p, (int)n, st);
        });
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceSelect::Flagged(t, b, iota.p, fn.p, sel.p, cnt.p + 1, (int)n, st);
        });
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceSelect::Flagged(t, b, iota.p, fz.p, g.zrows.p, cnt.p + 2, (int)n,
                                              st);
        });
        int64_t hc[3];
        KB_CUDA(cudaMemcpyAsync(hc, cnt.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        g.nh = hc[0];
        const int64_t nnorm = hc[1];
        g.nzero = hc[2];
        g.nv = g.nh + nnorm;
        // normal rows by descending length (stable in the new id) for balance
        g.vrow.alloc(std::max<int64_t>(1, nnorm));
        k2.alloc(std::max<int64_t>(1, nnorm));
        k3.alloc(std::max<int64_t>(1, nnorm));
        if (nnorm) {
            k_gather_keys<<<blocks_for(nnorm, 256), 256, 0, st>>>(key.p, sel.p, nnorm, k2.p);
            note_launch();
            int kbits = 1;
            while (kbits < 32 && ((int64_t)1 << kbits) <= g.split) kbits++;
            cub_run([&](void *t, size_t &b) {
                return cub::DeviceRadixSort::SortPairs(t, b, k2.p, k3.p, sel.p, g.vrow.p,
                                                       (int)nnorm, 0, kbits, st);
            });
        }
    }
    g.hot = std::min<int64_t>(g.hot, g.n);
    tr.mark("  sell: row classes");

    // ---- heavy rows -> segments, planned on the device (no host round trip
    // while a pipelined upload holds the copy engine).  Full segments come
    // first, row by row; then one partial segment per row with a remainder,
    // longest remainder first (stable in h), so the long chains start early.
    const int64_t T = g.split;
    Sell &S = g.sell;
    DBuf<int32_t> d_seg_row, d_seg_start;
    g.seg_ptr.alloc(g.nh + 1);
    if (g.nh) {
        const int64_t nh = g.nh;
        DBuf<int32_t> hdeg, full, tot, fstart, hid, hid2, pid;
        DBuf<uint32_t> pkey, pkey2;
        const int32_t *hd = g.deg.p;
        if (!fresh) {
            hdeg.alloc(nh);
            k_gather_keys<<<blocks_for(nh, 256), 256, 0, st>>>(
                (const uint32_t *)g.deg.p, g.hrow.p, nh, (uint32_t *)hdeg.p);
            note_launch();
            hd = hdeg.p;
        }
        full.alloc(nh + 1); tot.alloc(nh + 1); fstart.alloc(nh + 1);
        hid.alloc(nh); hid2.alloc(nh); pid.alloc(nh); pkey.alloc(nh); pkey2.alloc(nh);
        k_seg_counts<<<blocks_for(nh + 1, 256), 256, 0, st>>>(hd, nh, T, full.p, tot.p, pkey.p,
                                                             hid.p);
        note_launch();
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceScan::ExclusiveSum(t, b, full.p, fstart.p, (int)(nh + 1), st);
        });
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceScan::ExclusiveSum(t, b, tot.p, g.seg_ptr.p, (int)(nh + 1), st);
        });
        int bits = 1;
        while (((int64_t)1 << bits) <= T) bits++;
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortPairs(t, b, pkey.p, pkey2.p, hid.p, hid2.p, (int)nh,
                                                   0, bits, st);
        });
        int32_t ns = 0;
        KB_CUDA(cudaMemcpyAsync(&ns, g.seg_ptr.p + nh, sizeof(ns), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        S.nseg = ns;
        g.seg_list.alloc(std::max<int64_t>(1, ns));
        d_seg_row.alloc(std::max<int64_t>(1, ns));
        d_seg_start.alloc(std::max<int64_t>(1, ns));
        S.nvr = S.nseg + (g.nv - g.nh);
        S.vlen.alloc(S.nvr);
        k_seg_rank<<<blocks_for(nh, 256), 256, 0, st>>>(hid2.p, pkey2.p, nh, T, fstart.p, pid.p);
        note_launch();
        k_seg_fill<<<blocks_for(nh, 128), 128, 0, st>>>(hd, nh, T, fstart.p, g.seg_ptr.p, pid.p,
                                                        d_seg_row.p, d_seg_start.p, S.vlen.p,
                                                        g.seg_list.p);
        note_launch();
        KB_CUDA(cudaGetLastError());
    } else {
        KB_CUDA(cudaMemsetAsync(g.seg_ptr.p, 0, sizeof(int32_t), st));
        S.nseg = 0;
        g.seg_list.alloc(1);
        d_seg_row.alloc(1);
        d_seg_start.alloc(1);
        S.nvr = g.nv - g.nh;
        S.vlen.alloc(S.nvr);
    }
    S.nslices = (S.nvr + 31) / 32;
    tr.mark("  sell: segment plan");
    const int64_t nnorm = g.nv - g.nh;
    if (nnorm) {
        k_vlen_normal<<<blocks_for(nnorm, 256), 256, 0, st>>>(g.deg.p, g.vrow.p, g.nh, nnorm,
                                                             S.nseg, S.vlen.p);
        note_launch();
    }

    // ---- slice widths and offsets
    S.slice_w.alloc(S.nslices);
    S.slice_off.alloc(S.nslices + 1);
    DBuf<int64_t> sz;
    sz.alloc(S.nslices + 1);
    if (S.nslices) {
        k_slice_width<<<blocks_for(S.nslices, 256), 256, 0, st>>>(S.vlen.p, S.nvr, S.nslices,
                                                                 S.slice_w.p, sz.p);
        note_launch();
    }
    KB_CUDA(cudaMemsetAsync(sz.p + S.nslices, 0, sizeof(int64_t), st));
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, sz.p, S.slice_off.p, (int)(S.nslices + 1), st);
    });
    KB_CUDA(cudaMemcpyAsync(&S.elems, S.slice_off.p + S.nslices, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
    {   // narrow tail: K1 takes those slices four at a time
        DBuf<unsigned long long> lw;
        lw.alloc(1);
        KB_CUDA(cudaMemsetAsync(lw.p, 0, sizeof(unsigned long long), st));
        if (S.nslices) {
            k_last_wide<<<blocks_for(S.nslices, 256), 256, 0, st>>>(S.slice_w.p, S.nslices, lw.p);
            note_launch();
        }
        unsigned long long h = 0;
        KB_CUDA(cudaMemcpyAsync(&h, lw.p, sizeof(h), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        S.nwide = (int64_t)h;
    }
    KB_CUDA(cudaStreamSynchronize(st));
    sz.release();
    tr.mark("  sell: slice widths");

    // ---- fill the column slots (relabelled, original per-row order)
    S.cols.alloc(S.elems + 4);
    if (!fill) {
        // filled row by row as the arcs arrive (pipelined ingest); slots past
        // a row's length read as column 0 like k_fill's padding
        KB_CUDA(cudaMemsetAsync(S.cols.p, 0, S.cols.bytes(), st));
    } else if (S.nslices) {
        const int64_t threads = S.nslices * 32;
        k_fill<<<blocks_for(threads, 256), 256, 0, st>>>(
            g.indptr.p, g.indices.p, g.perm.p, g.iperm.p, S.vlen.p, d_seg_row.p, d_seg_start.p,
            g.hrow.p, g.vrow.p, S.slice_w.p, S.slice_off.p, S.nslices, S.nvr, S.nseg, g.nh,
            S.cols.p);
        note_launch();
        KB_CUDA(cudaGetLastError());
    }
    tr.mark("  sell: cols");
    // reverse maps for in-place patching by dynamic batches
    g.vr_of_row.alloc(std::max<int64_t>(1, n));
    g.h_of_row.alloc(std::max<int64_t>(1, n));
    KB_CUDA(cudaMemsetAsync(g.vr_of_row.p, 0xff, std::max<int64_t>(1, n) * 4, st));
    KB_CUDA(cudaMemsetAsync(g.h_of_row.p, 0xff, std::max<int64_t>(1, n) * 4, st));
    if (g.nv > g.nh) {
        k_rev_normal<<<blocks_for(g.nv - g.nh, 256), 256, 0, st>>>(g.vrow.p, g.nh, g.nv - g.nh,
                                                                  S.nseg, g.vr_of_row.p);
        note_launch();
    }
    if (g.nh) {
        k_rev_heavy<<<blocks_for(g.nh, 256), 256, 0, st>>>(g.hrow.p, g.nh, g.h_of_row.p);
        note_launch();
    }
    g.ovf.release();
    g.ovf_flag.release();
    g.n_ovf = 0;
    g.ovf_long.release();
    g.n_ovf_long = 0;
    KB_CUDA(cudaStreamSynchronize(st));
    g.sell_dirty = false;
}

// Apply the per-row effects of a batch to the SELL layout (after the
// canonical CSR was edited).  Too many overflow rows -> full rebuild later.
void patch_sell(Graph &g, const int32_t *rows_orig, int64_t ne) {
    cudaStream_t st = g.stream;
    if (g.sell_dirty || ne == 0) return;
    const int64_t n = g.n;
    if (!g.ovf.p) {
        g.ovf.alloc(std::max<int64_t>(1, n));
        g.ovf_flag.alloc(std::max<int64_t>(1, n));
        g.ovf_count.alloc(1);
        KB_CUDA(cudaMemsetAsync(g.ovf_flag.p, 0, std::max<int64_t>(1, n) * 4, st));
        KB_CUDA(cudaMemsetAsync(g.ovf_count.p, 0, 8, st));
    }
    Sell &S = g.sell;
    DBuf<int32_t> hv;                 // edited heavy rows patched in place
    DBuf<unsigned long long> hc;
    hv.alloc(std::max<int64_t>(1, std::min<int64_t>(ne, g.nh)));
    hc.alloc(1);
    KB_CUDA(cudaMemsetAsync(hc.p, 0, 8, st));
    k_patch_rows<<<blocks_for(ne * 32, 256), 256, 0, st>>>(
        rows_orig, ne, g.iperm.p, g.indptr.p, g.rlen.p, g.indices.p, g.vr_of_row.p,
        g.h_of_row.p, g.seg_ptr.p, g.seg_list.p, S.slice_w.p, S.slice_off.p, S.vlen.p, S.cols.p,
        g.ovf_flag.p, g.ovf.p, g.ovf_count.p, g.split, hv.p, hc.p);
    note_launch();
    KB_CUDA(cudaGetLastError());
    unsigned long long h[2] = {0, 0};
    KB_CUDA(cudaMemcpyAsync(&h[0], g.ovf_count.p, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaMemcpyAsync(&h[1], hc.p, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    g.n_ovf = (int64_t)h[0];
    if (h[1]) {
        k_patch_heavy<<<(unsigned)h[1], 256, 0, st>>>(
            hv.p, g.perm.p, g.indptr.p, g.rlen.p, g.indices.p, g.iperm.p, g.h_of_row.p,
            g.seg_ptr.p, g.seg_list.p, S.slice_w.p, S.slice_off.p, g.split, S.vlen.p, S.cols.p);
        note_launch();
        KB_CUDA(cudaGetLastError());
    }
    if (g.n_ovf) {
        // long overflow rows get a block each in K1 (a warp's serial chain
        // over thousands of arcs would be the level's tail)
        g.ovf_long.alloc(g.n_ovf);
        KB_CUDA(cudaMemsetAsync(hc.p, 0, 8, st));
        k_ovf_long_list<<<blocks_for(g.n_ovf, 256), 256, 0, st>>>(g.ovf.p, g.n_ovf, g.perm.p,
                                                                g.rlen.p, g.ovf_long.p, hc.p);
        note_launch();
        unsigned long long nl = 0;
        KB_CUDA(cudaMemcpyAsync(&nl, hc.p, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        g.n_ovf_long = (int64_t)nl;
    }
    if (getenv("KB_TRACE") && g.n_ovf) {
        DBuf<unsigned long long> lm;
        lm.alloc(3);
        KB_CUDA(cudaMemsetAsync(lm.p, 0, 24, st));
        k_ovf_stats<<<blocks_for(g.n_ovf, 256), 256, 0, st>>>(g.ovf.p, g.n_ovf, g.perm.p,
                                                            g.rlen.p, g.split, lm.p);
        unsigned long long hl[3];
        KB_CUDA(cudaMemcpyAsync(hl, lm.p, 24, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        fprintf(stderr, "[kb]   overflow rows %lld: %llu arcs, longest %llu, %llu over the split\n",
                (long long)g.n_ovf, hl[0], hl[1], hl[2]);
    }
    // the overflow pass is a warp per row: past a few percent of the rows a
    // rebuild of the layout is cheaper
    if (g.n_ovf > std::max<int64_t>(4096, g.nv / 32)) g.sell_dirty = true;
}

// Row lengths, the degree relabelling and the original-id lists K3 uses:
// everything that depends on g.indptr alone.
static void build_rows(Graph &g) {
    cudaStream_t st = g.stream;
    const int64_t n = g.n;
    g.rlen.alloc(n);
    if (n) k_rlen_compact<<<blocks_for(n, 256), 256, 0, st>>>(g.indptr.p, n, g.rlen.p);
    note_launch();

    // ---- relabel rows by descending degree (stable radix sort on ~deg)
    if (!g.relabel) {
        g.perm.alloc(n); g.iperm.alloc(n);
        if (n) {
            k_iota_pair<<<blocks_for(n, 256), 256, 0, st>>>(n, g.perm.p, g.iperm.p);
            note_launch();
        }
    } else {
        DBuf<uint32_t> key_in, key_out;
        DBuf<int32_t> id_in;
        key_in.alloc(n); key_out.alloc(n); id_in.alloc(n);
        g.perm.alloc(n); g.iperm.alloc(n);
        if (n) k_degree_key<<<blocks_for(n, 256), 256, 0, st>>>(g.rlen.p, n, key_in.p, id_in.p);
        note_launch();
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceRadixSort::SortPairs(t, b, key_in.p, key_out.p, id_in.p, g.perm.p,
                                                   (int)n, 0, 32, st);
        });
        if (n) k_invert<<<blocks_for(n, 256), 256, 0, st>>>(g.perm.p, n, g.iperm.p);
        note_launch();
        KB_CUDA(cudaGetLastError());
    }

    // ---- original ids with / without out-arcs, ascending (for K3)
    {
        DBuf<unsigned char> fl;
        DBuf<int32_t> iota;
        DBuf<int64_t> cntp;
        fl.alloc(n); iota.alloc(n); cntp.alloc(2);
        k_arc_flags<<<blocks_for(n, 256), 256, 0, st>>>(g.rlen.p, n, fl.p, iota.p);
        note_launch();
        g.orig_pos.alloc(n);
        g.orig_zero.alloc(n);
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceSelect::Flagged(t, b, iota.p, fl.p, g.orig_pos.p, cntp.p, (int)n,
                                              st);
        });
        k_flip<<<blocks_for(n, 256), 256, 0, st>>>(fl.p, n);
        note_launch();
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceSelect::Flagged(t, b, iota.p, fl.p, g.orig_zero.p, cntp.p + 1,
                                              (int)n, st);
        });
    }
}

// g.indptr / g.indices hold a compact canonical CSR on the device
void build_graph_device(Graph &g) {
    build_rows(g);
    build_sell(g, g.relabel);
    make_slack(g);
}


namespace {

// ---------------------------------------------------------------- row passes
// Per-arc work over a range of rows of a CSR (row starts ip, lengths rl,
// columns ix).  Rows of at most LONG_ARCS arcs are taken TILE_ROWS at a time
// by one block that scans their lengths and strides over the concatenated
// arcs with every thread busy (R-MAT rows average ~30 arcs); longer rows get
// a block each from a host-side list.
constexpr int TILE_ROWS = 256;
constexpr int LONG_ARCS = 256;   // tiles stay balanced: <= 64K arcs each

enum : int { OP_VALIDATE = 1, OP_COPY = 2, OP_FILL = 4, OP_SCATTER = 8, OP_ORDER = 16 };
enum : unsigned long long { F_ASYM = 1, F_INVALID = 2 };

struct RowOps {
    const int64_t *ip;
    const int32_t *rl;
    const int32_t *ix;
    int64_t n;
    int ops;
    unsigned long long *flags;
    // symmetry buckets: lower arc u -> v (v < u) goes to bkt[ip[v] + k] with
    // k < rl[v] taken from fill[v]
    unsigned int *fill;
    int32_t *bkt;
    // slack copy: row u to nix[nip[u] ..)
    const int64_t *nip;
    int32_t *nix;
    // SELL fill (the plan of build_sell)
    const int32_t *iperm, *vr_of_row, *h_of_row, *seg_ptr, *seg_list, *slice_w;
    const int64_t *slice_off;
    int32_t *cols;
    int64_t split;
};

struct RowCtx {
    int64_t first, dst, base;
    int w, lane, h;
};

__device__ __forceinline__ void row_ctx(const RowOps &A, int64_t u, RowCtx &c) {
    c.first = A.ip[u];
    c.dst = (A.ops & OP_COPY) ? A.nip[u] : 0;
    c.h = -1;
    c.base = 0;
    c.w = 0;
    c.lane = 0;
    if (A.ops & OP_FILL) {
        const int32_t v = A.iperm[u];
        const int32_t vr = A.vr_of_row[v];
        if (vr >= 0) {
            const int64_t s = vr >> 5;
            c.base = A.slice_off[s];
            c.w = A.slice_w[s];
            c.lane = vr & 31;
        } else {
            c.h = A.h_of_row[v];
        }
    }
}

__device__ __forceinline__ int64_t sell_pos(int w, int lane, int64_t j) {
    return (w <= 4) ? j * 32 + lane : (j >> 2) * 128 + lane * 4 + (j & 3);
}

// arc j of row u: validate, copy to the slack layout, place the relabelled
// column in its SELL slot, drop the reversed lower arc into its bucket
__device__ __forceinline__ void arc_ops(const RowOps &A, int64_t u, const RowCtx &c, int64_t j,
                                        bool &asym, bool &bad) {
    const int32_t col = A.ix[c.first + j];
    const bool in_range = col >= 0 && (int64_t)col < A.n;
    if (A.ops & OP_VALIDATE) {
        if (!in_range || ((A.ops & OP_ORDER) && j > 0 && A.ix[c.first + j - 1] >= col))
            bad = true;
    }
    if (A.ops & OP_COPY) A.nix[c.dst + j] = col;
    if (!in_range) return;
    if (A.ops & OP_FILL) {
        const int32_t nc = A.iperm[col];
        if (c.h < 0) {
            A.cols[c.base + sell_pos(c.w, c.lane, j)] = nc;
        } else {
            const int64_t q = j / A.split;
            const int32_t vr = A.seg_list[A.seg_ptr[c.h] + q];
            const int64_t s = vr >> 5;
            A.cols[A.slice_off[s] + sell_pos(A.slice_w[s], vr & 31, j - q * A.split)] = nc;
        }
    }
    if ((A.ops & OP_SCATTER) && (int64_t)col < u) {
        const unsigned k = atomicAdd(A.fill + col, 1u);
        if (k < (unsigned)A.rl[col]) A.bkt[A.ip[col] + k] = (int32_t)u;
        else asym = true;  // more reversed arcs than the row has slots
    }
}

__device__ __forceinline__ void raise_flags(const RowOps &A, bool asym, bool bad) {
    const unsigned long long f = (asym ? F_ASYM : 0ull) | (bad ? F_INVALID : 0ull);
    if (__any_sync(0xffffffffu, f != 0)) {
        if (f) atomicOr(A.flags, f);
    }
}

// index in the block's exclusive offsets of the row holding element e
__device__ __forceinline__ int tile_row(const int *off, int e) {
    int lo = 0, hi = TILE_ROWS;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= e) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(TILE_ROWS) k_rows_tile(RowOps A, int64_t a, int64_t b) {
    typedef cub::BlockScan<int, TILE_ROWS> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int off[TILE_ROWS + 1];
    __shared__ RowCtx ctx[TILE_ROWS];
    const int64_t r0 = a + (int64_t)blockIdx.x * TILE_ROWS;
    const int t = threadIdx.x;
    int cnt = 0;
    if (r0 + t < b) {
        const int L = A.rl[r0 + t];
        if (L <= LONG_ARCS) {
            cnt = L;
            row_ctx(A, r0 + t, ctx[t]);
        }
    }
    int ex, total;
    Scan(tmp).ExclusiveSum(cnt, ex, total);
    off[t] = ex;
    if (t == 0) off[TILE_ROWS] = total;
    __syncthreads();
    bool asym = false, bad = false;
    for (int e = t; e < total; e += TILE_ROWS) {
        const int lo = tile_row(off, e);
        arc_ops(A, r0 + lo, ctx[lo], e - off[lo], asym, bad);
    }
    raise_flags(A, asym, bad);
}

// long rows are cut into items of LONG_ITEM arcs (row, first arc), so a hub
// row spreads over many blocks instead of serialising the pass's tail
constexpr int LONG_ITEM = 2048;

__global__ void k_rows_long(RowOps A, const int32_t *item_row, const int32_t *item_j0) {
    __shared__ RowCtx c;
    const int64_t u = item_row[blockIdx.x];
    if (threadIdx.x == 0) row_ctx(A, u, c);
    __syncthreads();
    const int64_t j0 = item_j0[blockIdx.x];
    const int64_t j1 = min((int64_t)A.rl[u], j0 + LONG_ITEM);
    bool asym = false, bad = false;
    for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) arc_ops(A, u, c, j, asym, bad);
    raise_flags(A, asym, bad);
}

// first index of the ascending row with a column > v
__device__ __forceinline__ int64_t upper_start(const int32_t *row, int64_t L, int64_t v) {
    int64_t lo = 0, hi = L;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)row[mid] <= v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ bool contains(const int32_t *a, int64_t n, int32_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo < n && a[lo] == x;
}

// Row v's bucket holds the sources u > v of the arcs u -> v.  The arc set is
// symmetric iff for every v the bucket has exactly as many entries as v has
// upper arcs v -> w (w > v) and each entry is one of those w: the entries
// are distinct (one per row u, rows strictly ascending), so the bucket then
// equals the upper part and every arc has its reversal.
__global__ void __launch_bounds__(TILE_ROWS) k_verify_tile(RowOps A, int64_t a, int64_t b) {
    typedef cub::BlockScan<int, TILE_ROWS> Scan;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int off[TILE_ROWS + 1];
    __shared__ int64_t first[TILE_ROWS], up[TILE_ROWS];
    __shared__ int hi_n[TILE_ROWS];
    const int64_t r0 = a + (int64_t)blockIdx.x * TILE_ROWS;
    const int t = threadIdx.x;
    int cnt = 0;
    bool asym = false;
    if (r0 + t < b) {
        const int64_t v = r0 + t;
        const int64_t L = A.rl[v];
        const int64_t f = A.ip[v];
        const int64_t u0 = upper_start(A.ix + f, L, v);
        const unsigned got = A.fill[v];
        if ((int64_t)got != L - u0) asym = true;
        first[t] = f;
        up[t] = f + u0;
        hi_n[t] = (int)(L - u0);
        if (L <= LONG_ARCS && !asym) cnt = (int)(L - u0);
    }
    int ex, total;
    Scan(tmp).ExclusiveSum(cnt, ex, total);
    off[t] = ex;
    if (t == 0) off[TILE_ROWS] = total;
    __syncthreads();
    for (int e = t; e < total; e += TILE_ROWS) {
        const int lo = tile_row(off, e);
        const int32_t u = A.bkt[first[lo] + (e - off[lo])];
        if (!contains(A.ix + up[lo], hi_n[lo], u)) asym = true;
    }
    raise_flags(A, asym, false);
}

// A long row's buckets are checked against a sample of its upper part in
// shared memory (every stride-th column, at most VSAMPLES of them): each
// search is a shared-memory bisection plus one short window in global
// memory instead of ~19 dependent loads through L2.
constexpr int VSAMPLES = 4096;

__global__ void __launch_bounds__(256) k_verify_long(RowOps A, const int32_t *item_row,
                                                     const int32_t *item_j0) {
    __shared__ int64_t u0s;
    __shared__ int32_t samp[VSAMPLES];
    const int64_t v = item_row[blockIdx.x];
    const int64_t L = A.rl[v], f = A.ip[v];
    if (threadIdx.x == 0) u0s = upper_start(A.ix + f, L, v);
    __syncthreads();
    const int64_t u0 = u0s, hn = L - u0;
    if ((int64_t)A.fill[v] != hn) return;  // k_verify_tile flagged the row
    const int32_t *U = A.ix + f + u0;
    const int64_t stride = (hn + VSAMPLES - 1) / VSAMPLES;
    const int ns = (int)((hn + stride - 1) / stride);
    for (int i = threadIdx.x; i < ns; i += blockDim.x) samp[i] = U[i * stride];
    __syncthreads();
    const int64_t e0 = item_j0[blockIdx.x], e1 = min(hn, e0 + LONG_ITEM);
    bool asym = false;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const int32_t x = A.bkt[f + e];
        int lo = 0, hi = ns;  // first sample > x
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (samp[mid] <= x) lo = mid + 1; else hi = mid;
        }
        if (lo == 0) { asym = true; continue; }  // below every upper column
        const int64_t w0 = (int64_t)(lo - 1) * stride;
        if (!contains(U + w0, min(stride, hn - w0), x)) asym = true;
    }
    raise_flags(A, asym, false);
}

struct LongRow {
    const int32_t *rl;
    __device__ bool operator()(int32_t r) const { return rl[r] > LONG_ARCS; }
};

__global__ void k_item_counts(const int32_t *len, int64_t m, int32_t *cnt) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) cnt[i] = (len[i] + LONG_ITEM - 1) / LONG_ITEM;
    else if (i == m) cnt[i] = 0;
}

__global__ void k_item_fill(const int32_t *rows, const int32_t *len, const int32_t *pre,
                            int64_t m, int32_t *item_row, int32_t *item_j0) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    for (int32_t k = 0, j = 0; j < len[i]; k++, j += LONG_ITEM) {
        item_row[pre[i] + k] = rows[i];
        item_j0[pre[i] + k] = j;
    }
}

// Work items of the rows of rl longer than LONG_ARCS, ascending by row:
// (row, first arc) every LONG_ITEM arcs.  Host copy of the item rows for the
// per-chunk ranges, device copies for the kernels.
struct LongItems {
    std::vector<int32_t> row;      // host, ascending
    DBuf<int32_t> d_row, d_j0;
    void build(const int32_t *rl, int64_t n, cudaStream_t st) {
        DBuf<int32_t> d, len;
        DBuf<int64_t> cnt;
        d.alloc(std::max<int64_t>(1, n));
        cnt.alloc(1);
        cub::CountingInputIterator<int32_t> it(0);
        cub_run([&](void *t, size_t &b) {
            return cub::DeviceSelect::If(t, b, it, d.p, cnt.p, (int)n, LongRow{rl}, st);
        });
        int64_t m = 0;
        KB_CUDA(cudaMemcpyAsync(&m, cnt.p, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        std::vector<int32_t> rows(m), lens(m);
        if (m) {
            len.alloc(m);
            k_gather_keys<<<blocks_for(m, 256), 256, 0, st>>>((const uint32_t *)rl, d.p, m,
                                                              (uint32_t *)len.p);
            note_launch();
            KB_CUDA(cudaMemcpyAsync(rows.data(), d.p, m * 4, cudaMemcpyDeviceToHost, st));
            KB_CUDA(cudaMemcpyAsync(lens.data(), len.p, m * 4, cudaMemcpyDeviceToHost, st));
            KB_CUDA(cudaStreamSynchronize(st));
        }
        // host mirror of the item rows (for the per-chunk ranges); the device
        // arrays are written by a kernel, so nothing is uploaded
        row.clear();
        for (int64_t i = 0; i < m; i++)
            for (int64_t j = 0; j < lens[i]; j += LONG_ITEM) row.push_back(rows[i]);
        const int64_t ni = (int64_t)row.size();
        d_row.alloc(std::max<int64_t>(1, ni));
        d_j0.alloc(std::max<int64_t>(1, ni));
        if (ni) {
            DBuf<int32_t> cnt_i, pre;
            cnt_i.alloc(m + 1);
            pre.alloc(m + 1);
            k_item_counts<<<blocks_for(m + 1, 256), 256, 0, st>>>(len.p, m, cnt_i.p);
            note_launch();
            cub_run([&](void *t, size_t &b) {
                return cub::DeviceScan::ExclusiveSum(t, b, cnt_i.p, pre.p, (int)(m + 1), st);
            });
            k_item_fill<<<blocks_for(m, 128), 128, 0, st>>>(d.p, len.p, pre.p, m, d_row.p,
                                                            d_j0.p);
            note_launch();
            KB_CUDA(cudaGetLastError());
            KB_CUDA(cudaStreamSynchronize(st));
        }
    }
};

// one pass (arc ops or bucket verification) over rows [a, b)
void rows_pass(const RowOps &A, bool verify, int64_t a, int64_t b, const LongItems &li,
               cudaStream_t st) {
    if (b <= a) return;
    if (verify) k_verify_tile<<<blocks_for(b - a, TILE_ROWS), TILE_ROWS, 0, st>>>(A, a, b);
    else k_rows_tile<<<blocks_for(b - a, TILE_ROWS), TILE_ROWS, 0, st>>>(A, a, b);
    note_launch();
    const auto &R = li.row;
    const int64_t la = std::lower_bound(R.begin(), R.end(), (int32_t)a) - R.begin();
    const int64_t lb = std::lower_bound(R.begin(), R.end(),
                                        (int32_t)std::min<int64_t>(b, INT32_MAX)) - R.begin();
    if (lb > la) {
        if (verify) k_verify_long<<<(unsigned)(lb - la), 256, 0, st>>>(A, li.d_row.p + la,
                                                                        li.d_j0.p + la);
        else k_rows_long<<<(unsigned)(lb - la), 256, 0, st>>>(A, li.d_row.p + la,
                                                              li.d_j0.p + la);
        note_launch();
    }
    KB_CUDA(cudaGetLastError());
}

}  // namespace

// Graph.is_symmetric (graph.py:168-175): the arc set equals its reversal.
// Every lower arc u -> v (v < u) is dropped into v's bucket (k_rows_tile,
// OP_SCATTER); then each bucket must equal v's upper part (k_verify_*).
// Works on the CSR-with-slack as it stands (row starts + lengths).
int graph_is_symmetric(Graph &g) {
    cudaStream_t st = g.stream;
    const int64_t n = g.n;
    if (n == 0 || g.indices.n == 0) return 1;
    DBuf<unsigned int> fill;
    DBuf<int32_t> bkt;
    DBuf<unsigned long long> flags;
    fill.alloc(n);
    bkt.alloc(g.indices.n);
    flags.alloc(1);
    KB_CUDA(cudaMemsetAsync(fill.p, 0, n * sizeof(unsigned int), st));
    KB_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(unsigned long long), st));
    LongItems li;
    li.build(g.rlen.p, n, st);
    RowOps A{};
    A.ip = g.indptr.p;
    A.rl = g.rlen.p;
    A.ix = g.indices.p;
    A.n = n;
    A.ops = OP_SCATTER;
    A.flags = flags.p;
    A.fill = fill.p;
    A.bkt = bkt.p;
    rows_pass(A, false, 0, n, li, st);
    rows_pass(A, true, 0, n, li, st);
    unsigned long long hf = 0;
    KB_CUDA(cudaMemcpyAsync(&hf, flags.p, sizeof(hf), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    return (hf & F_ASYM) ? 0 : 1;
}

// Ingest of a host CSR, pipelined with its upload.  indptr goes first; the
// relabelling, the SELL plan and the slack layout need only the row lengths
// and are computed while the columns stream in.  The columns arrive in
// chunks of whole rows, highest rows first, on a copy stream; as each chunk
// lands, one pass validates it (ids in range, rows strictly ascending),
// copies it into the slack layout, writes its SELL slots and drops its lower
// arcs into the symmetry buckets, and a second pass verifies the buckets of
// its rows -- complete, because every row above it has arrived.  The upload
// is the bound (2.2 GB at C2); the graph and its symmetry flag are ready
// one chunk after the last byte lands.
void build_graph(Graph &g, const int64_t *h_indptr, const int32_t *h_indices) {
    NvtxRange nv("ingest (upload + layout + symmetry)");
    cudaStream_t st = g.stream;
    cudaStream_t cs = copy_stream();
    const int64_t n = g.n, nnz = g.nnz;
    g.indptr.alloc(n + 1);
    DBuf<int32_t> stage;  // the compact columns as uploaded
    stage.alloc(nnz);
    const bool pinned = host_is_pinned(h_indices);
    // chunks of whole rows, ~chunk_arcs arcs each, processed from the top
    // rows down; the last ones (the bottom rows, processed after the final
    // byte lands) shrink geometrically so little work trails the upload
    const int64_t C = std::max<int64_t>(1, tune_get("ingest.chunk_arcs", (int64_t)1 << 25));
    std::vector<int64_t> rb{n};   // descending row boundaries
    while (rb.back() > 0) {
        const int64_t hi = rb.back(), arcs_left = h_indptr[hi];
        const int64_t size = arcs_left > 2 * C ? C : std::max<int64_t>(C / 16, arcs_left / 2);
        int64_t r = std::lower_bound(h_indptr, h_indptr + hi + 1, arcs_left - size) - h_indptr;
        r = std::max<int64_t>(0, std::min<int64_t>(r, hi - 1));
        rb.push_back(r);
    }
    std::reverse(rb.begin(), rb.end());   // ascending: chunk c = [rb[c], rb[c+1])
    const int nch = (int)rb.size() - 1;
    const bool trace = getenv("KB_TRACE") != nullptr;
    std::vector<cudaEvent_t> ev(nch + 2), tev(trace ? nch : 0);
    cudaEvent_t tev0 = nullptr;
    for (auto &e : ev)
        KB_CUDA(cudaEventCreateWithFlags(&e, trace ? cudaEventDefault : cudaEventDisableTiming));
    for (auto &e : tev) KB_CUDA(cudaEventCreate(&e));
    if (trace) KB_CUDA(cudaEventCreate(&tev0));
    auto cleanup = [&] {
        cudaStreamSynchronize(cs);
        for (auto &e : ev) cudaEventDestroy(e);
        for (auto &e : tev) cudaEventDestroy(e);
        if (tev0) cudaEventDestroy(tev0);
    };
    auto copy_chunk = [&](int c) {
        const int64_t a = h_indptr[rb[c]], b = h_indptr[rb[c + 1]];
        if (b > a) upload_h2d(stage.p + a, h_indices + a, (b - a) * sizeof(int32_t), cs);
        KB_CUDA(cudaEventRecord(ev[c], cs));
    };
    try {
        // the buffers may be recycled blocks still in use by queued work
        KB_CUDA(cudaEventRecord(ev[nch], st));
        KB_CUDA(cudaStreamWaitEvent(cs, ev[nch], 0));
        if (trace) KB_CUDA(cudaEventRecord(tev0, cs));
        upload_h2d(g.indptr.p, h_indptr, (n + 1) * sizeof(int64_t), cs);
        KB_CUDA(cudaEventRecord(ev[nch + 1], cs));
        if (pinned)
            for (int c = nch - 1; c >= 0; c--) copy_chunk(c);
        KB_CUDA(cudaStreamWaitEvent(st, ev[nch + 1], 0));

        const auto h0 = std::chrono::steady_clock::now();
        auto mark = [&](const char *what) {
            if (!trace) return;
            KB_CUDA(cudaStreamSynchronize(st));
            fprintf(stderr, "[ingest]   %s at %.2f ms\n", what,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
        };
        build_rows(g);
        mark("rows");
        build_sell(g, g.relabel, false);
        mark("sell plan");
        DBuf<int64_t> nip;
        DBuf<int32_t> nix, bkt;
        int64_t total = 0;
        slack_layout(g, nullptr, nip, nix, total);
        mark("slack layout");
        DBuf<unsigned int> fill;
        DBuf<unsigned long long> flags;
        fill.alloc(n);
        bkt.alloc(nnz);
        flags.alloc(1);
        KB_CUDA(cudaMemsetAsync(fill.p, 0, std::max<int64_t>(1, n) * sizeof(unsigned int), st));
        KB_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(unsigned long long), st));
        LongItems li;
        li.build(g.rlen.p, n, st);

        if (trace) {
            KB_CUDA(cudaStreamSynchronize(st));
            fprintf(stderr, "[ingest] plan (rows, SELL plan, slack layout, long items): %.2f ms host\n",
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
        }
        RowOps A{};
        A.ip = g.indptr.p;
        A.rl = g.rlen.p;
        A.ix = stage.p;
        A.n = n;
        // shard graphs (no relabelling) keep their rows in original-id order
        // over exchange ids: ranges are checked, order and symmetry are not
        A.ops = OP_VALIDATE | OP_COPY | OP_FILL | (g.relabel ? OP_SCATTER | OP_ORDER : 0);
        A.flags = flags.p;
        A.fill = fill.p;
        A.bkt = bkt.p;
        A.nip = nip.p;
        A.nix = nix.p;
        A.iperm = g.iperm.p;
        A.vr_of_row = g.vr_of_row.p;
        A.h_of_row = g.h_of_row.p;
        A.seg_ptr = g.seg_ptr.p;
        A.seg_list = g.seg_list.p;
        A.slice_w = g.sell.slice_w.p;
        A.slice_off = g.sell.slice_off.p;
        A.cols = g.sell.cols.p;
        A.split = g.split;
        for (int c = nch - 1; c >= 0; c--) {
            if (!pinned) copy_chunk(c);
            KB_CUDA(cudaStreamWaitEvent(st, ev[c], 0));
            rows_pass(A, false, rb[c], rb[c + 1], li, st);
            if (A.ops & OP_SCATTER) rows_pass(A, true, rb[c], rb[c + 1], li, st);
            if (trace) KB_CUDA(cudaEventRecord(tev[c], st));
        }
        unsigned long long hf = 0;
        KB_CUDA(cudaMemcpyAsync(&hf, flags.p, sizeof(hf), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        KB_REQUIRE(!(hf & F_INVALID), KB_EPARAM,
                   "indices: every row must be strictly ascending with ids in [0, n)");
        g.symmetric = !(A.ops & OP_SCATTER) ? -1 : (hf & F_ASYM) ? 0 : 1;
        if (trace) {
            float t0 = 0, t1 = 0;
            for (int c = nch - 1; c >= 0; c--) {
                KB_CUDA(cudaEventElapsedTime(&t0, tev0, ev[c]));
                KB_CUDA(cudaEventElapsedTime(&t1, tev0, tev[c]));
                fprintf(stderr, "[ingest] chunk %d rows [%lld, %lld): copied %.2f ms, done %.2f ms\n",
                        c, (long long)rb[c], (long long)rb[c + 1], t0, t1);
            }
        }
        g.indptr = std::move(nip);
        g.indices = std::move(nix);
        g.tail = total;
        g.slack = true;
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
}

}  // namespace kb
