// Graph ingest: canonical host CSR -> device SELL-32 over degree-relabelled
// rows (replaces Graph.out_csr, graph.py:177-197).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <numeric>

#include "kb_internal.cuh"

namespace kb {

size_t Graph::device_bytes() const {
    return perm.bytes() + iperm.bytes() + deg.bytes() + indptr.bytes() +
           indices.bytes() + sell.cols.bytes() + sell.slice_off.bytes() +
           sell.slice_w.bytes() + sell.vlen.bytes() + seg_ptr.bytes() +
           seg_list.bytes();
}

namespace {

__global__ void k_degree(const int64_t *indptr, int64_t n, uint32_t *key,
                         int32_t *ids) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    int64_t d = indptr[v + 1] - indptr[v];
    key[v] = 0xFFFFFFFFu - (uint32_t)d;  // ascending key == descending degree
    ids[v] = (int32_t)v;
}

__global__ void k_finish_perm(const uint32_t *skey, const int32_t *perm,
                              int64_t n, int32_t *iperm, int32_t *sdeg) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    iperm[perm[i]] = (int32_t)i;
    sdeg[i] = (int32_t)(0xFFFFFFFFu - skey[i]);
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

__global__ void k_counts(const int32_t *sdeg, int64_t n, int64_t split,
                         int64_t *out) {
    out[0] = first_le(sdeg, n, 0);      // nv: rows with arcs
    out[1] = first_le(sdeg, n, split);  // nh: rows longer than split
    out[2] = n ? sdeg[0] : 0;
}

__global__ void k_vlen_tail(const int32_t *sdeg, int64_t nh, int64_t nv,
                            int64_t nseg, int32_t *vlen) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nv - nh) return;
    vlen[nseg + i] = sdeg[nh + i];
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
__global__ void k_fill(const int64_t *indptr, const int32_t *indices,
                       const int32_t *perm, const int32_t *iperm,
                       const int32_t *vlen, const int32_t *seg_row,
                       const int32_t *seg_start, const int32_t *slice_w,
                       const int64_t *slice_off, int64_t nslices, int64_t nvr,
                       int64_t nseg, int64_t nh, int32_t *cols) {
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
        if (vr < nseg) { row_new = seg_row[vr]; start = seg_start[vr]; }
        else row_new = nh + (vr - nseg);
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

__global__ void k_arc_flags(const int64_t *indptr, int64_t n, unsigned char *fl, int32_t *iota) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    fl[v] = indptr[v + 1] > indptr[v];
    iota[v] = (int32_t)v;
}

__global__ void k_flip(unsigned char *fl, int64_t n) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v < n) fl[v] = !fl[v];
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

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

// g.indptr / g.indices already hold the canonical CSR on the device
void build_graph_device(Graph &g) {
    cudaStream_t st = g.stream;
    const int64_t n = g.n;

    // ---- relabel rows by descending degree (stable radix sort on ~deg)
    DBuf<uint32_t> key_in, key_out;
    DBuf<int32_t> id_in;
    key_in.alloc(n); key_out.alloc(n); id_in.alloc(n);
    g.perm.alloc(n); g.iperm.alloc(n); g.deg.alloc(n);
    if (n) k_degree<<<blocks_for(n, 256), 256, 0, st>>>(g.indptr.p, n, key_in.p, id_in.p); note_launch();
    KB_CUDA(cudaGetLastError());
    size_t tmp_bytes = 0;
    KB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key_in.p, key_out.p,
                                            id_in.p, g.perm.p, (int)n, 0, 32, st));
    DBuf<unsigned char> tmp;
    tmp.alloc(tmp_bytes);
    KB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, key_in.p, key_out.p,
                                            id_in.p, g.perm.p, (int)n, 0, 32, st)); note_launch();
    if (n) k_finish_perm<<<blocks_for(n, 256), 256, 0, st>>>(key_out.p, g.perm.p, n,
                                                            g.iperm.p, g.deg.p); note_launch();
    KB_CUDA(cudaGetLastError());
    key_in.release(); key_out.release(); id_in.release(); tmp.release();

    DBuf<int64_t> cnt;
    cnt.alloc(3);
    k_counts<<<1, 1, 0, st>>>(g.deg.p, n, g.split, cnt.p); note_launch();
    int64_t hc[3];
    KB_CUDA(cudaMemcpyAsync(hc, cnt.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    g.nv = hc[0];
    g.nh = hc[1];
    g.max_deg = hc[2];
    g.hot = std::min<int64_t>(g.hot, g.n);

    // ---- heavy rows -> segments (host plan; nh is small)
    std::vector<int32_t> hdeg(g.nh);
    if (g.nh)
        KB_CUDA(cudaMemcpy(hdeg.data(), g.deg.p, g.nh * sizeof(int32_t),
                           cudaMemcpyDeviceToHost));
    std::vector<int32_t> seg_row, seg_start, seg_len;
    std::vector<std::vector<int32_t>> row_segs(g.nh);
    const int64_t T = g.split;
    for (int64_t h = 0; h < g.nh; h++) {  // full segments, row by row
        int64_t full = hdeg[h] / T;
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
    if (g.nv > g.nh)
        k_vlen_tail<<<blocks_for(g.nv - g.nh, 256), 256, 0, st>>>(g.deg.p, g.nh, g.nv,
                                                                 S.nseg, S.vlen.p); note_launch();
    KB_CUDA(cudaGetLastError());

    // ---- slice widths and offsets
    S.slice_w.alloc(S.nslices);
    S.slice_off.alloc(S.nslices + 1);
    DBuf<int64_t> sz;
    sz.alloc(S.nslices + 1);
    if (S.nslices)
        k_slice_width<<<blocks_for(S.nslices, 256), 256, 0, st>>>(S.vlen.p, S.nvr, S.nslices,
                                                                 S.slice_w.p, sz.p); note_launch();
    KB_CUDA(cudaMemsetAsync(sz.p + S.nslices, 0, sizeof(int64_t), st));
    tmp_bytes = 0;
    KB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sz.p, S.slice_off.p,
                                          (int)(S.nslices + 1), st));
    tmp.alloc(tmp_bytes);
    KB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, sz.p, S.slice_off.p,
                                          (int)(S.nslices + 1), st)); note_launch();
    KB_CUDA(cudaMemcpyAsync(&S.elems, S.slice_off.p + S.nslices, sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    tmp.release();
    sz.release();

    // ---- original ids with / without out-arcs, ascending (for K3)
    {
        DBuf<unsigned char> fl;
        DBuf<int32_t> iota;
        DBuf<int64_t> cntp;
        fl.alloc(n); iota.alloc(n); cntp.alloc(2);
        k_arc_flags<<<blocks_for(std::max<int64_t>(n, 1), 256), 256, 0, st>>>(g.indptr.p, n, fl.p, iota.p);
        note_launch();
        g.orig_pos.alloc(std::max<int64_t>(1, g.nv));
        g.orig_zero.alloc(std::max<int64_t>(1, n - g.nv));
        size_t tb = 0;
        DBuf<unsigned char> t2;
        // stable selection of both sides (DevicePartition would reverse the
        // rejected side)
        KB_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.p, fl.p, g.orig_pos.p, cntp.p,
                                           (int)n, st));
        t2.alloc(tb);
        KB_CUDA(cub::DeviceSelect::Flagged(t2.p, tb, iota.p, fl.p, g.orig_pos.p, cntp.p, (int)n,
                                           st));
        k_flip<<<blocks_for(std::max<int64_t>(n, 1), 256), 256, 0, st>>>(fl.p, n);
        KB_CUDA(cub::DeviceSelect::Flagged(t2.p, tb, iota.p, fl.p, g.orig_zero.p, cntp.p + 1,
                                           (int)n, st));
        note_launch(3);
    }

    // ---- fill the column slots (relabelled, original per-row order)
    S.cols.alloc(S.elems + 4);
    if (S.nslices) {
        int64_t threads = S.nslices * 32;
        k_fill<<<blocks_for(threads, 256), 256, 0, st>>>(
            g.indptr.p, g.indices.p, g.perm.p, g.iperm.p, S.vlen.p, d_seg_row.p,
            d_seg_start.p, S.slice_w.p, S.slice_off.p, S.nslices, S.nvr, S.nseg,
            g.nh, S.cols.p); note_launch();
        KB_CUDA(cudaGetLastError());
    }
    KB_CUDA(cudaStreamSynchronize(st));
}

namespace {
// arc (u, v) needs u in row v; rows are sorted, so a binary search per arc
__global__ void k_symmetric(const int64_t *indptr, const int32_t *indices, int64_t n,
                            unsigned long long *bad) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const int64_t u = warp;
    for (int64_t e = indptr[u] + lane; e < indptr[u + 1]; e += 32) {
        const int64_t v = indices[e];
        int64_t lo = indptr[v], hi = indptr[v + 1];
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (indices[mid] < u) lo = mid + 1; else hi = mid;
        }
        if (lo >= indptr[v + 1] || indices[lo] != u) { atomicAdd(bad, 1ull); return; }
    }
}
}  // namespace

int graph_is_symmetric(Graph &g) {
    DBuf<unsigned long long> bad;
    bad.alloc(1);
    KB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), g.stream));
    if (g.n)
        k_symmetric<<<blocks_for(g.n * 32, 256), 256, 0, g.stream>>>(g.indptr.p, g.indices.p,
                                                                      g.n, bad.p); note_launch();
    KB_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    KB_CUDA(cudaMemcpyAsync(&h, bad.p, sizeof(h), cudaMemcpyDeviceToHost, g.stream));
    KB_CUDA(cudaStreamSynchronize(g.stream));
    return h == 0;
}

}  // namespace kb
