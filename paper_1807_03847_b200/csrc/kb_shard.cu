// Multi-GPU shard construction on the device.
//
// A rank's shard is built from a device graph that holds the canonical
// CSR (kb_graph_create / the device generators): no host partitioning and no
// host copy of the graph per rank.
//
// Partition (degree-rank round-robin, distributed.ShardPlan restated): the
// node of degree rank q (descending out-degree, stable in the node id) is
// owned by rank q mod P and sits at exchange id
//     e(v) = (q mod P) * n_per + q div P,      n_per = ceil(n / P),
// so rank p's rows are the contiguous block [p*n_per, (p+1)*n_per) and one
// all-gather of the blocks (or K1's fused NVLink stores) rebuilds omega in
// the exchange layout on every rank.  The shard is a KB_GRAPH_NO_RELABEL
// graph over the P*n_per exchange ids whose non-owned rows are empty; each
// owned row keeps its arcs in ascending *original* id order (columns mapped
// to exchange ids), so its K1 sum is the one-GPU sum bit for bit.  Tie-break
// labels are the original ids (padding ids: n, n+1, ... in exchange order).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "kb_internal.cuh"

namespace kb {

namespace {

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

// degree of original row v of a (possibly slack) canonical CSR
__global__ void k_deg_keys(const int32_t *rlen, int64_t n, uint32_t *key, int32_t *id) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    key[v] = 0xFFFFFFFFu - (uint32_t)rlen[v];   // ascending key = descending degree
    id[v] = (int32_t)v;
}

// q(v) from the degree order; exch_of_node / node_of_exch of the plan
__global__ void k_plan(const int32_t *by_rank, int64_t n, int64_t P, int64_t n_per,
                       int32_t *exch_of_node, int32_t *node_of_exch) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int32_t v = by_rank[q];
    const int64_t e = (q % P) * n_per + q / P;
    exch_of_node[v] = (int32_t)e;
    node_of_exch[e] = v;
}

// labels of the shard's ids: the node id, padding -> n + its index among the
// padding ids in exchange order (block p pads [owned(p), n_per))
__global__ void k_labels(const int32_t *node_of_exch, int64_t n, int64_t P, int64_t n_per,
                         int32_t *label) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= P * n_per) return;
    const int32_t v = node_of_exch[e];
    if (v >= 0) { label[e] = v; return; }
    const int64_t p = e / n_per, local = e - p * n_per;
    int64_t before = 0;                          // padding ids in blocks < p
    for (int64_t b = 0; b < p; b++) before += n_per - (n - b + P - 1) / P;
    const int64_t owned = (n - p + P - 1) / P;
    label[e] = (int32_t)(n + before + (local - owned));
}

// row lengths of the shard's CSR (owned rows only)
__global__ void k_local_len(const int32_t *node_of_exch, const int32_t *rlen, int64_t lo,
                            int64_t hi, int64_t N, int64_t *len) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= N) return;
    int64_t l = 0;
    if (e >= lo && e < hi) {
        const int32_t v = node_of_exch[e];
        if (v >= 0) l = rlen[v];
    }
    len[e] = l;
}

// one warp per owned row: copy its columns in stored (ascending original id)
// order, mapped to exchange ids
__global__ void k_local_cols(const int32_t *node_of_exch, const int64_t *ip_full,
                             const int32_t *ix_full, const int32_t *exch_of_node,
                             const int64_t *ip_loc, int64_t lo, int64_t hi, int32_t *ix_loc,
                             int64_t nnz_loc) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t e = lo + warp;
    if (e >= hi) return;
    const int32_t v = node_of_exch[e];
    if (v < 0) return;
    const int64_t src = ip_full[v], dst = ip_loc[e], L = ip_loc[e + 1] - dst;
    KB_DCHECK(dst >= 0 && dst + L <= nnz_loc);
    (void)nnz_loc;
    for (int64_t j = lane; j < L; j += 32) ix_loc[dst + j] = exch_of_node[ix_full[src + j]];
}

// device ids whose tie-break label is one of the m targets (-1 if none)
__global__ void k_find_labels(const int32_t *label, int64_t N, const int64_t *targets, int m,
                              unsigned long long *out) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= N) return;
    const int32_t l = label[e];
    for (int j = 0; j < m; j++)
        if ((int64_t)l == targets[j]) out[j] = (unsigned long long)e;
}

}  // namespace

void find_labels(Graph &g, const int64_t *h_targets, int64_t m, int64_t *h_ids) {
    cudaStream_t st = g.stream;
    KB_REQUIRE(m >= 0 && m <= 64, KB_EPARAM, "at most 64 labels per call");
    if (!m) return;
    DBuf<int64_t> t;
    DBuf<unsigned long long> o;
    t.alloc(m);
    o.alloc(m);
    KB_CUDA(cudaMemcpyAsync(t.p, h_targets, m * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    KB_CUDA(cudaMemsetAsync(o.p, 0xFF, m * sizeof(unsigned long long), st));
    const int32_t *lab = g.labels();
    if (g.n)
        k_find_labels<<<nblk(g.n, 256), 256, 0, st>>>(lab, g.n, t.p, (int)m, o.p);
    note_launch();
    KB_CUDA(cudaMemcpyAsync(h_ids, o.p, m * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
}

// Builds rank `rank`'s shard of `full` into `out` (fresh Graph: device,
// stream, split and hot already set by the caller).  Returns n_per and the
// number of owned rows.
void build_shard(Graph &full, int64_t P, int64_t rank, Graph &out, int64_t *n_per_out,
                 int64_t *owned_out) {
    cudaStream_t st = full.stream;
    const int64_t n = full.n;
    KB_REQUIRE(P >= 1 && rank >= 0 && rank < P, KB_EPARAM, "bad rank / world size");
    KB_REQUIRE(!full.sell_dirty || full.indptr.p, KB_ESTATE, "graph has no canonical CSR");
    const int64_t n_per = std::max<int64_t>(1, (n + P - 1) / P);
    const int64_t N = P * n_per;
    KB_REQUIRE(N < ((int64_t)1 << 31), KB_ENODERANGE, "exchange ids must fit 32 bits");
    // ---- the degree order: a fresh relabelled graph already holds it
    // (perm = new -> original id, new ids by descending degree, stable)
    DBuf<int32_t> by_rank;
    const int32_t *order = nullptr;
    if (full.relabel && !full.mutated) {
        order = full.perm.p;
    } else {
        DBuf<uint32_t> k0, k1;
        DBuf<int32_t> i0;
        k0.alloc(n); k1.alloc(n); i0.alloc(n); by_rank.alloc(n);
        k_deg_keys<<<nblk(n, 256), 256, 0, st>>>(full.rlen.p, n, k0.p, i0.p);
        note_launch();
        size_t tb = 0;
        KB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.p, k1.p, i0.p, by_rank.p, (int)n, 0,
                                                32, st));
        DBuf<unsigned char> tmp;
        tmp.alloc(tb);
        KB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k0.p, k1.p, i0.p, by_rank.p, (int)n, 0,
                                                32, st));
        note_launch();
        order = by_rank.p;
    }
    DBuf<int32_t> eon, noe;
    eon.alloc(n);
    noe.alloc(N);
    KB_CUDA(cudaMemsetAsync(noe.p, 0xFF, N * sizeof(int32_t), st));
    k_plan<<<nblk(n, 256), 256, 0, st>>>(order, n, P, n_per, eon.p, noe.p);
    note_launch();
    // ---- the shard's CSR over exchange ids
    const int64_t lo = rank * n_per, hi = lo + n_per;
    DBuf<int64_t> len;
    len.alloc(N + 1);
    k_local_len<<<nblk(N, 256), 256, 0, st>>>(noe.p, full.rlen.p, lo, hi, N, len.p);
    note_launch();
    KB_CUDA(cudaMemsetAsync(len.p + N, 0, sizeof(int64_t), st));
    out.indptr.alloc(N + 1);
    {
        size_t tb = 0;
        KB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len.p, out.indptr.p, (int)(N + 1), st));
        DBuf<unsigned char> tmp;
        tmp.alloc(tb);
        KB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, len.p, out.indptr.p, (int)(N + 1), st));
        note_launch();
    }
    int64_t nnz_loc = 0;
    KB_CUDA(cudaMemcpyAsync(&nnz_loc, out.indptr.p + N, sizeof(int64_t), cudaMemcpyDeviceToHost,
                            st));
    KB_CUDA(cudaStreamSynchronize(st));
    out.indices.alloc(std::max<int64_t>(1, nnz_loc));
    if (n_per)
        k_local_cols<<<nblk(n_per * 32, 256), 256, 0, st>>>(noe.p, full.indptr.p, full.indices.p,
                                                            eon.p, out.indptr.p, lo, hi,
                                                            out.indices.p, nnz_loc);
    note_launch();
    out.n = N;
    out.nnz = nnz_loc;
    out.relabel = false;
    out.own_lo = lo;
    out.own_hi = hi;
    // the head of every rank's block (its top hubs) in K1's shared-memory hot
    // set when blocks are 2^k ids (kb_graph_create_ex does the same)
    if ((n_per & (n_per - 1)) == 0 && P > 1) {
        int sh = 0;
        while (((int64_t)1 << sh) < n_per) sh++;
        out.hot_shift = sh;
        out.hot_per = std::max<int64_t>(1, out.hot / P);
    }
    build_graph_device(out);
    // a shard inherits the whole graph's (verified) symmetry
    if (full.symmetric < 0) full.symmetric = graph_is_symmetric(full);
    out.symmetric = full.symmetric;
    // labels: node ids by shard id (the shard is not relabelled: perm = id)
    out.label.alloc(N);
    k_labels<<<nblk(N, 256), 256, 0, st>>>(noe.p, n, P, n_per, out.label.p);
    note_launch();
    out.mutated = true;   // no degree-sorted tail shortcuts
    KB_CUDA(cudaStreamSynchronize(st));
    *n_per_out = n_per;
    *owned_out = std::max<int64_t>(0, (n - rank + P - 1) / P);
}

}  // namespace kb
