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

#include <algorithm>
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
    key[v] = 0xFFFFFFFFu - (uint32_t)d;
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
    for (int j = 0; j < w; j++) {
        int32_t c = (j < len) ? iperm[indices[src + j]] : 0;
        int64_t pos = (w <= 4) ? ((int64_t)j * 32 + lane)
                               : ((int64_t)(j >> 2) * 128 + lane * 4 + (j & 3));
        base[pos] = c;
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
                             unsigned long long *ovf_count) {
    int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const int32_t o = rows_orig[e];
    const int32_t v = iperm[o];
    if (ovf_flag[v]) return;  // already recomputed from the canonical CSR
    const int32_t len = rlen[o];
    const int32_t vr = vr_of_row[v];
    if (vr >= 0) {
        const int64_t s = vr >> 5;
        const int lane = vr & 31;
        const int w = slice_w[s];
        if (len <= w) {
            int32_t *base = cols + slice_off[s];
            const int32_t *row = indices + indptr[o];
            for (int j = 0; j < len; j++) {
                const int64_t pos = (w <= 4) ? ((int64_t)j * 32 + lane)
                                             : ((int64_t)(j >> 2) * 128 + lane * 4 + (j & 3));
                base[pos] = iperm[row[j]];
            }
            vlen[vr] = len;
            return;
        }
        vlen[vr] = 0;
    } else if (h_of_row[v] >= 0) {
        const int32_t h = h_of_row[v];
        for (int q = seg_ptr[h]; q < seg_ptr[h + 1]; q++) vlen[seg_list[q]] = 0;
    }
    if (atomicExch(&ovf_flag[v], 1) == 0) ovf[atomicAdd(ovf_count, 1ull)] = v;
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

}  // namespace

// Virtual rows, slices and column slots for the current arc set under the
// current relabelling.  `fresh` means perm sorts rows by descending length,
// so heavy / normal / empty rows are the contiguous new-id ranges
// [0,nh) / [nh,nv) / [nv,n) and no explicit row maps are needed.
void build_sell(Graph &g, bool fresh) {
    cudaStream_t st = g.stream;
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
    } else {
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
            cub_run([&](void *t, size_t &b) {
                return cub::DeviceRadixSort::SortPairs(t, b, k2.p, k3.p, sel.p, g.vrow.p,
                                                       (int)nnorm, 0, 32, st);
            });
        }
    }
    g.hot = std::min<int64_t>(g.hot, g.n);

    // ---- heavy rows -> segments (host plan; nh is small)
    std::vector<int32_t> hdeg(g.nh);
    if (g.nh) {
        if (fresh) {
            KB_CUDA(cudaMemcpyAsync(hdeg.data(), g.deg.p, g.nh * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, st));
        } else {
            DBuf<int32_t> hd;
            hd.alloc(g.nh);
            k_gather_keys<<<blocks_for(g.nh, 256), 256, 0, st>>>(
                (const uint32_t *)g.deg.p, g.hrow.p, g.nh, (uint32_t *)hd.p);
            note_launch();
            KB_CUDA(cudaMemcpyAsync(hdeg.data(), hd.p, g.nh * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, st));
            KB_CUDA(cudaStreamSynchronize(st));
        }
        KB_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<int32_t> seg_row, seg_start, seg_len;
    std::vector<std::vector<int32_t>> row_segs(g.nh);
    const int64_t T = g.split;
    for (int64_t h = 0; h < g.nh; h++) {  // full segments, row by row
        const int64_t full = hdeg[h] / T;
        for (int64_t q = 0; q < full; q++) {
            row_segs[h].push_back((int32_t)seg_row.size());
            seg_row.push_back((int32_t)h);
            seg_start.push_back((int32_t)(q * T));
            seg_len.push_back((int32_t)T);
        }
    }
    std::vector<int64_t> partial;
    for (int64_t h = 0; h < g.nh; h++)
        if (hdeg[h] % T) partial.push_back(h);
    std::stable_sort(partial.begin(), partial.end(), [&](int64_t a, int64_t b) {
        return hdeg[a] % T > hdeg[b] % T;
    });
    for (int64_t h : partial) {
        row_segs[h].push_back((int32_t)seg_row.size());
        seg_row.push_back((int32_t)h);
        seg_start.push_back((int32_t)((hdeg[h] / T) * T));
        seg_len.push_back((int32_t)(hdeg[h] % T));
    }
    std::vector<int32_t> sptr(g.nh + 1, 0), slist;
    for (int64_t h = 0; h < g.nh; h++) {
        for (int32_t x : row_segs[h]) slist.push_back(x);
        sptr[h + 1] = (int32_t)slist.size();
    }
    Sell &S = g.sell;
    S.nseg = (int64_t)seg_row.size();
    S.nvr = S.nseg + (g.nv - g.nh);
    S.nslices = (S.nvr + 31) / 32;
    g.seg_ptr.alloc(g.nh + 1);
    g.seg_list.alloc(std::max<size_t>(1, slist.size()));
    KB_CUDA(cudaMemcpyAsync(g.seg_ptr.p, sptr.data(), sptr.size() * sizeof(int32_t),
                            cudaMemcpyHostToDevice, st));
    if (!slist.empty())
        KB_CUDA(cudaMemcpyAsync(g.seg_list.p, slist.data(), slist.size() * sizeof(int32_t),
                                cudaMemcpyHostToDevice, st));
    DBuf<int32_t> d_seg_row, d_seg_start;
    d_seg_row.alloc(std::max<size_t>(1, seg_row.size()));
    d_seg_start.alloc(std::max<size_t>(1, seg_row.size()));
    S.vlen.alloc(S.nvr);
    if (S.nseg) {
        KB_CUDA(cudaMemcpyAsync(d_seg_row.p, seg_row.data(), S.nseg * sizeof(int32_t),
                                cudaMemcpyHostToDevice, st));
        KB_CUDA(cudaMemcpyAsync(d_seg_start.p, seg_start.data(), S.nseg * sizeof(int32_t),
                                cudaMemcpyHostToDevice, st));
        KB_CUDA(cudaMemcpyAsync(S.vlen.p, seg_len.data(), S.nseg * sizeof(int32_t),
                                cudaMemcpyHostToDevice, st));
    }
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
        std::vector<int32_t> hw(S.nslices);
        if (S.nslices)
            KB_CUDA(cudaMemcpyAsync(hw.data(), S.slice_w.p, S.nslices * sizeof(int32_t),
                                    cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        int64_t t = S.nslices;
        while (t > 0 && hw[t - 1] <= 4) t--;
        S.nwide = t;
    }
    KB_CUDA(cudaStreamSynchronize(st));
    sz.release();

    // ---- fill the column slots (relabelled, original per-row order)
    S.cols.alloc(S.elems + 4);
    if (S.nslices) {
        const int64_t threads = S.nslices * 32;
        k_fill<<<blocks_for(threads, 256), 256, 0, st>>>(
            g.indptr.p, g.indices.p, g.perm.p, g.iperm.p, S.vlen.p, d_seg_row.p, d_seg_start.p,
            g.hrow.p, g.vrow.p, S.slice_w.p, S.slice_off.p, S.nslices, S.nvr, S.nseg, g.nh,
            S.cols.p);
        note_launch();
        KB_CUDA(cudaGetLastError());
    }
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
    k_patch_rows<<<blocks_for(ne, 128), 128, 0, st>>>(
        rows_orig, ne, g.iperm.p, g.indptr.p, g.rlen.p, g.indices.p, g.vr_of_row.p,
        g.h_of_row.p, g.seg_ptr.p, g.seg_list.p, S.slice_w.p, S.slice_off.p, S.vlen.p, S.cols.p,
        g.ovf_flag.p, g.ovf.p, g.ovf_count.p);
    note_launch();
    KB_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    KB_CUDA(cudaMemcpyAsync(&h, g.ovf_count.p, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    g.n_ovf = (int64_t)h;
    // the overflow pass is a warp per row: past a few percent of the rows a
    // rebuild of the layout is cheaper
    if (g.n_ovf > std::max<int64_t>(4096, g.nv / 32)) g.sell_dirty = true;
}

void build_graph(Graph &g, const int64_t *h_indptr, const int32_t *h_indices) {
    cudaStream_t st = g.stream;
    g.indptr.alloc(g.n + 1);
    g.indices.alloc(g.nnz);
    KB_CUDA(cudaMemcpyAsync(g.indptr.p, h_indptr, (g.n + 1) * sizeof(int64_t),
                            cudaMemcpyHostToDevice, st));
    if (g.nnz)
        KB_CUDA(cudaMemcpyAsync(g.indices.p, h_indices, g.nnz * sizeof(int32_t),
                                cudaMemcpyHostToDevice, st));
    build_graph_device(g);
}

// g.indptr / g.indices hold a compact canonical CSR on the device
void build_graph_device(Graph &g) {
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
    build_sell(g, g.relabel);
    make_slack(g);
}


namespace {
// per row u: arcs to smaller ids (lower triangle) and to larger ids (upper)
__global__ void k_tri_counts(const int64_t *indptr, const int32_t *rlen, const int32_t *indices,
                             int64_t n, int64_t *lo_cnt, int64_t *hi_cnt) {
    int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u > n) return;
    if (u == n) { lo_cnt[u] = hi_cnt[u] = 0; return; }
    const int32_t *row = indices + indptr[u];
    const int64_t L = rlen[u];
    int64_t a = 0, b = L;  // first slot with col >= u
    while (a < b) { const int64_t m = (a + b) >> 1; if (row[m] < u) a = m + 1; else b = m; }
    const int64_t lo = a;
    const int64_t self = (lo < L && row[lo] == u) ? 1 : 0;
    lo_cnt[u] = lo;
    hi_cnt[u] = L - lo - self;
}

// Arcs of a row range, with every lane busy: a block takes SEG_ROWS rows,
// scans the per-row counts in shared memory and strides over the
// concatenated arcs; rows with more than SEG_LONG arcs are skipped here and
// get a block each (k_*_long).  part(u) = (first slot, count) of the arcs
// of row u the kernel visits.
constexpr int SEG_ROWS = 256;
constexpr int SEG_LONG = 1024;

template <typename Part, typename Visit>
__device__ __forceinline__ void seg_rows(int64_t n, Part part, Visit visit) {
    __shared__ int off[SEG_ROWS + 1];
    __shared__ int64_t first[SEG_ROWS];
    const int64_t r0 = (int64_t)blockIdx.x * SEG_ROWS;
    const int t = threadIdx.x;
    int cnt = 0;
    if (r0 + t < n) {
        int64_t f, c;
        part(r0 + t, f, c);
        first[t] = f;
        cnt = c > SEG_LONG ? 0 : (int)c;
    }
    off[t + 1] = cnt;
    if (t == 0) off[0] = 0;
    __syncthreads();
    for (int d = 1; d < SEG_ROWS; d <<= 1) {
        const int v = (t + 1 > d) ? off[t + 1 - d] : 0;
        __syncthreads();
        off[t + 1] += v;
        __syncthreads();
    }
    const int total = off[SEG_ROWS];
    for (int e = t; e < total; e += SEG_ROWS) {
        int lo = 0, hi = SEG_ROWS;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (off[mid] <= e) lo = mid; else hi = mid;
        }
        visit(r0 + lo, first[lo], e - off[lo]);
    }
}

// lower-triangle arcs u -> v (v < u) as (key v, value u), written in row
// order at lo_off[u]: a stable sort by v then lists each v's u ascending
struct LowerPart {
    const int64_t *lo_cnt;
    __device__ void operator()(int64_t u, int64_t &f, int64_t &c) const { f = 0; c = lo_cnt[u]; }
};

__global__ void __launch_bounds__(SEG_ROWS) k_tri_pairs(const int64_t *indptr,
                                                        const int32_t *indices, int64_t n,
                                                        const int64_t *lo_off,
                                                        const int64_t *lo_cnt, uint32_t *key,
                                                        int32_t *val) {
    seg_rows(n, LowerPart{lo_cnt}, [&](int64_t u, int64_t, int j) {
        const int64_t o = lo_off[u] + j;
        key[o] = (uint32_t)indices[indptr[u] + j];
        val[o] = (int32_t)u;
    });
}

__global__ void k_tri_pairs_long(const int32_t *rows, const int64_t *indptr,
                                 const int32_t *indices, const int64_t *lo_off,
                                 const int64_t *lo_cnt, uint32_t *key, int32_t *val) {
    const int64_t u = rows[blockIdx.x];
    const int64_t c = lo_cnt[u];
    for (int64_t j = threadIdx.x; j < c; j += blockDim.x) {
        key[lo_off[u] + j] = (uint32_t)indices[indptr[u] + j];
        val[lo_off[u] + j] = (int32_t)u;
    }
}

// upper-triangle arcs v -> w (w > v) in row order must equal the sorted
// reversed lower arcs one for one
struct UpperPart {
    const int64_t *lo_cnt, *hi_cnt;
    const int32_t *rlen;
    __device__ void operator()(int64_t v, int64_t &f, int64_t &c) const {
        c = hi_cnt[v];
        f = rlen[v] - c;          // the upper part is the row's tail
    }
};

__global__ void __launch_bounds__(SEG_ROWS) k_tri_match(const int64_t *indptr,
                                                        const int32_t *rlen,
                                                        const int32_t *indices, int64_t n,
                                                        const int64_t *hi_off,
                                                        const int64_t *lo_cnt,
                                                        const int64_t *hi_cnt,
                                                        const uint32_t *skey,
                                                        const int32_t *sval,
                                                        unsigned long long *bad) {
    bool b = false;
    seg_rows(n, UpperPart{lo_cnt, hi_cnt, rlen}, [&](int64_t v, int64_t f, int j) {
        const int64_t o = hi_off[v] + j;
        b |= skey[o] != (uint32_t)v || sval[o] != indices[indptr[v] + f + j];
    });
    if (b) atomicOr(bad, 1ull);
}

__global__ void k_tri_match_long(const int32_t *rows, const int64_t *indptr,
                                 const int32_t *rlen, const int32_t *indices,
                                 const int64_t *hi_off, const int64_t *hi_cnt,
                                 const uint32_t *skey, const int32_t *sval,
                                 unsigned long long *bad) {
    const int64_t v = rows[blockIdx.x];
    const int64_t c = hi_cnt[v], f = rlen[v] - c;
    bool b = false;
    for (int64_t j = threadIdx.x; j < c; j += blockDim.x) {
        const int64_t o = hi_off[v] + j;
        b |= skey[o] != (uint32_t)v || sval[o] != indices[indptr[v] + f + j];
    }
    if (b) atomicOr(bad, 1ull);
}

struct LongOf {
    const int64_t *cnt;
    __device__ bool operator()(int32_t r) const { return cnt[r] > SEG_LONG; }
};
}  // namespace

// Graph.is_symmetric (graph.py:168-175): the arc set equals its reversal.
// Self-loops are their own reversal; every arc u->v with u < v must be
// matched by v->u.  The upper-triangle keys u*2^s+v come out of the
// canonical CSR already sorted, so the set is symmetric iff the sorted
// reversed lower-triangle keys match them one for one (half the arcs sorted).
int graph_is_symmetric(Graph &g) {
    cudaStream_t st = g.stream;
    const int64_t n = g.n, m = g.nnz;
    if (m == 0) return 1;
    int shift = 1;
    while (((int64_t)1 << shift) < n) shift++;
    DBuf<int64_t> lo_cnt, hi_cnt, lo_off, hi_off;
    lo_cnt.alloc(n + 1); hi_cnt.alloc(n + 1); lo_off.alloc(n + 1); hi_off.alloc(n + 1);
    k_tri_counts<<<blocks_for(n + 1, 256), 256, 0, st>>>(g.indptr.p, g.rlen.p, g.indices.p, n,
                                                        lo_cnt.p, hi_cnt.p);
    note_launch();
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, lo_cnt.p, lo_off.p, (int)(n + 1), st);
    });
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceScan::ExclusiveSum(t, b, hi_cnt.p, hi_off.p, (int)(n + 1), st);
    });
    int64_t tot[2];
    KB_CUDA(cudaMemcpyAsync(&tot[0], lo_off.p + n, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaMemcpyAsync(&tot[1], hi_off.p + n, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    if (tot[0] != tot[1]) return 0;
    const int64_t h = tot[0];
    if (h == 0) return 1;
    // (v, u) pairs of the lower triangle in row order, stably sorted by v
    // alone (the u's of each v stay ascending): 32-bit keys, 4 passes at
    // most instead of a 64-bit (v, u) key sort
    DBuf<uint32_t> key, skey;
    DBuf<int32_t> val, sval, longs;
    DBuf<int64_t> nlong;
    key.alloc(h); skey.alloc(h); val.alloc(h); sval.alloc(h); longs.alloc(n); nlong.alloc(2);
    k_tri_pairs<<<blocks_for(n, SEG_ROWS), SEG_ROWS, 0, st>>>(g.indptr.p, g.indices.p, n,
                                                             lo_off.p, lo_cnt.p, key.p, val.p);
    note_launch();
    cub::CountingInputIterator<int32_t> it(0);
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceSelect::If(t, b, it, longs.p, nlong.p, (int)n, LongOf{lo_cnt.p}, st);
    });
    int64_t nl = 0;
    KB_CUDA(cudaMemcpyAsync(&nl, nlong.p, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    if (nl) {
        k_tri_pairs_long<<<(unsigned)nl, 256, 0, st>>>(longs.p, g.indptr.p, g.indices.p,
                                                        lo_off.p, lo_cnt.p, key.p, val.p);
        note_launch();
    }
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceRadixSort::SortPairs(t, b, key.p, skey.p, val.p, sval.p, h, 0, shift,
                                               st);
    });
    DBuf<unsigned long long> bad;
    bad.alloc(1);
    KB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), st));
    k_tri_match<<<blocks_for(n, SEG_ROWS), SEG_ROWS, 0, st>>>(
        g.indptr.p, g.rlen.p, g.indices.p, n, hi_off.p, lo_cnt.p, hi_cnt.p, skey.p, sval.p,
        bad.p);
    note_launch();
    cub_run([&](void *t, size_t &b) {
        return cub::DeviceSelect::If(t, b, it, longs.p, nlong.p + 1, (int)n, LongOf{hi_cnt.p},
                                     st);
    });
    KB_CUDA(cudaMemcpyAsync(&nl, nlong.p + 1, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    if (nl) {
        k_tri_match_long<<<(unsigned)nl, 256, 0, st>>>(longs.p, g.indptr.p, g.rlen.p,
                                                        g.indices.p, hi_off.p, hi_cnt.p, skey.p,
                                                        sval.p, bad.p);
        note_launch();
    }
    KB_CUDA(cudaGetLastError());
    unsigned long long hb = 0;
    KB_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    return hb == 0;
}

}  // namespace kb
