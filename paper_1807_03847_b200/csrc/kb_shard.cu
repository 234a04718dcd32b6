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
#include <cstring>
#include <vector>

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

// row lengths from a host-uploaded indptr; flags[0] |= 1 if it decreases
__global__ void k_rlen_from_ip(const int64_t *ip, int64_t n, int32_t *rlen,
                               unsigned long long *flags) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= n) return;
    const int64_t l = ip[v + 1] - ip[v];
    if (l < 0 || l > 0x7FFFFFFF) { atomicOr(flags, 1ull); rlen[v] = 0; return; }
    rlen[v] = (int32_t)l;
}

// the owned rows' lengths in exchange order (for the host gather's offsets)
__global__ void k_owned_len(const int32_t *node_of_exch, const int32_t *rlen, int64_t lo,
                            int64_t owned, int64_t *len) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < owned) len[i] = rlen[node_of_exch[lo + i]];
    if (i == owned) len[i] = 0;
}

// one warp per owned row: validate its (gathered, original-id) columns --
// ids in [0, n), strictly ascending (graph.py:191-192) -- and map them to
// exchange ids; flags[0] |= 2 on a bad row
__global__ void k_local_cols_host(const int64_t *ip_loc, int64_t lo, int64_t hi,
                                  const int32_t *cols, const int64_t *src_off,
                                  const int32_t *exch_of_node, int64_t n, int32_t *ix_loc,
                                  unsigned long long *flags) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t e = lo + warp;
    if (e >= hi) return;
    const int64_t dst = ip_loc[e], L = ip_loc[e + 1] - dst, src = src_off[warp];
    bool bad = false;
    for (int64_t j = lane; j < L; j += 32) {
        const int32_t c = cols[src + j];
        if (c < 0 || c >= n || (j > 0 && cols[src + j - 1] >= c)) {
            bad = true;
            ix_loc[dst + j] = 0;
        } else {
            ix_loc[dst + j] = exch_of_node[c];
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, 2ull);
}

// symmetry exchange: the reverse of every local arc (e -> c) as the key
// c * N + e, grouped by the owner of c (rank c / n_per)
__global__ void k_sym_count(const int64_t *ip, const int32_t *ix, int64_t lo, int64_t hi,
                            int64_t n_per, unsigned long long *cnt) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t e = lo + warp;
    if (e >= hi) return;
    // one atomic per distinct destination per warp step (P is small: a
    // per-arc atomic on P counters serialises)
    for (int64_t j0 = ip[e]; j0 < ip[e + 1]; j0 += 32) {
        const int64_t j = j0 + lane;
        const bool in = j < ip[e + 1];
        const int dst = in ? (int)(ix[j] / n_per) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, dst);
        if (in && lane == __ffs(peers) - 1) atomicAdd(&cnt[dst], (unsigned long long)__popc(peers));
    }
}

__global__ void k_sym_scatter(const int64_t *ip, const int32_t *ix, int64_t lo, int64_t hi,
                              int64_t n_per, int64_t N, unsigned long long *pos, int64_t *keys) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t e = lo + warp;
    if (e >= hi) return;
    for (int64_t j0 = ip[e]; j0 < ip[e + 1]; j0 += 32) {
        const int64_t j = j0 + lane;
        const bool in = j < ip[e + 1];
        const int64_t c = in ? ix[j] : 0;
        const int dst = in ? (int)(c / n_per) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, dst);
        const int leader = __ffs(peers) - 1;
        unsigned long long base = 0;
        if (in && lane == leader) base = atomicAdd(&pos[dst], (unsigned long long)__popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (in) keys[base + __popc(peers & ((1u << lane) - 1u))] = c * N + e;
    }
}

// the local arcs as keys e * N + c (row-major: already sorted when rows and
// columns ascend in exchange ids -- not guaranteed, so they are sorted too)
__global__ void k_own_keys(const int64_t *ip, const int32_t *ix, int64_t lo, int64_t hi,
                           int64_t N, int64_t *keys) {
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t e = lo + warp;
    if (e >= hi) return;
    for (int64_t j = ip[e] + lane; j < ip[e + 1]; j += 32) keys[j - ip[lo]] = e * N + ix[j];
}

__global__ void k_keys_differ(const int64_t *a, const int64_t *b, int64_t m,
                              unsigned long long *bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m && a[i] != b[i]) atomicOr(bad, 1ull);
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

// Rank `rank`'s shard straight from a host CSR: only indptr (for the degree
// order) and the rank's own rows travel to its GPU -- the rows are gathered
// on the host into the page-locked upload ring by the pool threads -- so a
// graph larger than one GPU's memory can be sharded.  The columns are
// validated (ids in range, rows strictly ascending) like kb_graph_create's.
void build_shard_host(Graph &out, int64_t n, int64_t nnz, const int64_t *h_ip,
                      const int32_t *h_ix, int64_t P, int64_t rank, int64_t *n_per_out,
                      int64_t *owned_out) {
    cudaStream_t st = out.stream;
    KB_REQUIRE(P >= 1 && rank >= 0 && rank < P, KB_EPARAM, "bad rank / world size");
    KB_REQUIRE(n >= 1 && h_ip && (nnz == 0 || h_ix), KB_EPARAM, "NULL CSR arrays");
    KB_REQUIRE(h_ip[0] == 0 && h_ip[n] == nnz, KB_EPARAM, "indptr must start at 0 and end at nnz");
    const int64_t n_per = std::max<int64_t>(1, (n + P - 1) / P);
    const int64_t N = P * n_per;
    KB_REQUIRE(N < ((int64_t)1 << 31), KB_ENODERANGE, "exchange ids must fit 32 bits");
    const int64_t lo = rank * n_per, hi = lo + n_per;
    const int64_t owned = std::max<int64_t>(0, (n - rank + P - 1) / P);
    DBuf<int64_t> ip;
    DBuf<int32_t> rlen, key_in_id, by_rank;
    DBuf<uint32_t> k0, k1;
    DBuf<unsigned long long> flags;
    ip.alloc(n + 1);
    rlen.alloc(n);
    flags.alloc(1);
    KB_CUDA(cudaMemsetAsync(flags.p, 0, 8, st));
    upload_h2d(ip.p, h_ip, (n + 1) * sizeof(int64_t), st);
    k_rlen_from_ip<<<nblk(n, 256), 256, 0, st>>>(ip.p, n, rlen.p, flags.p);
    note_launch();
    // the degree order (descending, stable in the id) and the plan
    k0.alloc(n); k1.alloc(n); key_in_id.alloc(n); by_rank.alloc(n);
    k_deg_keys<<<nblk(n, 256), 256, 0, st>>>(rlen.p, n, k0.p, key_in_id.p);
    note_launch();
    {
        size_t tb = 0;
        KB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.p, k1.p, key_in_id.p, by_rank.p,
                                                (int)n, 0, 32, st));
        DBuf<unsigned char> tmp;
        tmp.alloc(tb);
        KB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tb, k0.p, k1.p, key_in_id.p, by_rank.p,
                                                (int)n, 0, 32, st));
        note_launch();
    }
    DBuf<int32_t> eon, noe;
    eon.alloc(n);
    noe.alloc(N);
    KB_CUDA(cudaMemsetAsync(noe.p, 0xFF, N * sizeof(int32_t), st));
    k_plan<<<nblk(n, 256), 256, 0, st>>>(by_rank.p, n, P, n_per, eon.p, noe.p);
    note_launch();
    // the owned rows' original ids, in exchange order, and their offsets in
    // the gathered column array (a device scan of their lengths)
    std::vector<int32_t> rows(owned);
    std::vector<int64_t> loc(owned + 1, 0);
    DBuf<int64_t> olen, oloc;
    olen.alloc(owned + 1);
    oloc.alloc(owned + 1);
    k_owned_len<<<nblk(owned + 1, 256), 256, 0, st>>>(noe.p, rlen.p, lo, owned, olen.p);
    note_launch();
    {
        size_t tb = 0;
        KB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, olen.p, oloc.p, (int)(owned + 1), st));
        DBuf<unsigned char> tmp;
        tmp.alloc(tb);
        KB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, olen.p, oloc.p, (int)(owned + 1), st));
        note_launch();
    }
    unsigned long long hflags = 0;
    if (owned)
        KB_CUDA(cudaMemcpyAsync(rows.data(), noe.p + lo, owned * sizeof(int32_t),
                                cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaMemcpyAsync(loc.data(), oloc.p, (owned + 1) * sizeof(int64_t),
                            cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaMemcpyAsync(&hflags, flags.p, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    KB_REQUIRE(!(hflags & 1), KB_EPARAM, "indptr must be non-decreasing");
    const int64_t nnz_loc = loc[owned];
    // gather the owned rows' columns through the upload ring
    DBuf<int32_t> cols;
    cols.alloc(std::max<int64_t>(1, nnz_loc));
    upload_gather_h2d(cols.p, (size_t)nnz_loc * sizeof(int32_t), st,
                      [&](char *slot, size_t off, size_t len, int t, int T) {
                          const int64_t a0 = (int64_t)(off / 4), a1 = (int64_t)((off + len) / 4);
                          const int64_t p0 = a0 + (a1 - a0) * t / T;
                          const int64_t p1 = a0 + (a1 - a0) * (t + 1) / T;
                          if (p1 <= p0) return;
                          int64_t i = std::upper_bound(loc.begin(), loc.end(), p0) - loc.begin() - 1;
                          for (int64_t q = p0; q < p1; i++) {
                              const int64_t end = std::min(loc[i + 1], p1);
                              const int32_t *srcp = h_ix + h_ip[rows[i]] + (q - loc[i]);
                              memcpy(slot + (q - a0) * 4, srcp, (size_t)(end - q) * 4);
                              q = end;
                          }
                      });
    // the shard's CSR over exchange ids (owned rows only)
    DBuf<int64_t> len, src_off;
    len.alloc(N + 1);
    k_local_len<<<nblk(N, 256), 256, 0, st>>>(noe.p, rlen.p, lo, hi, N, len.p);
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
    (void)src_off;
    out.indices.alloc(std::max<int64_t>(1, nnz_loc));
    if (owned)
        k_local_cols_host<<<nblk(owned * 32, 256), 256, 0, st>>>(out.indptr.p, lo, lo + owned,
                                                                cols.p, oloc.p, eon.p, n,
                                                                out.indices.p, flags.p);
    note_launch();
    KB_CUDA(cudaMemcpyAsync(&hflags, flags.p, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    KB_REQUIRE(!(hflags & 2), KB_EPARAM,
               "CSR rows must hold strictly ascending ids in [0, n)");
    cols.release();
    out.n = N;
    out.nnz = nnz_loc;
    out.relabel = false;
    out.own_lo = lo;
    out.own_hi = hi;
    if ((n_per & (n_per - 1)) == 0 && P > 1) {
        int sh = 0;
        while (((int64_t)1 << sh) < n_per) sh++;
        out.hot_shift = sh;
        out.hot_per = std::max<int64_t>(1, out.hot / P);
    }
    out.symmetric = -1;        // decided across the ranks (shard_symmetry_*)
    build_graph_device(out);
    out.label.alloc(N);
    k_labels<<<nblk(N, 256), 256, 0, st>>>(noe.p, n, P, n_per, out.label.p);
    note_launch();
    out.mutated = true;
    out.sym_n_per = n_per;
    KB_CUDA(cudaStreamSynchronize(st));
    *n_per_out = n_per;
    *owned_out = owned;
}

// Exact distributed symmetry check, step 1: the reverse of every local arc,
// keyed c * N + e and grouped by the rank owning c; counts[q] = keys for q.
void shard_symmetry_keys(Graph &g, int64_t P, int64_t *keys, int64_t *h_counts) {
    cudaStream_t st = g.stream;
    const int64_t n_per = g.own_hi - g.own_lo, N = g.n;
    KB_REQUIRE(P >= 1 && N == P * n_per, KB_EPARAM, "not a shard of this world size");
    DBuf<int64_t> cip;                  // the shard's arcs, compact (rows ascending)
    DBuf<int32_t> cix;
    compact_csr(g, cip, cix);
    DBuf<unsigned long long> cnt, pos;
    cnt.alloc(P);
    pos.alloc(P);
    KB_CUDA(cudaMemsetAsync(cnt.p, 0, P * 8, st));
    const int64_t rows = g.own_hi - g.own_lo;
    if (rows)
        k_sym_count<<<nblk(rows * 32, 256), 256, 0, st>>>(cip.p, cix.p, g.own_lo, g.own_hi,
                                                        n_per, cnt.p);
    note_launch();
    std::vector<unsigned long long> c(P), off(P, 0);
    KB_CUDA(cudaMemcpyAsync(c.data(), cnt.p, P * 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    for (int64_t q = 1; q < P; q++) off[q] = off[q - 1] + c[q - 1];
    KB_CUDA(cudaMemcpyAsync(pos.p, off.data(), P * 8, cudaMemcpyHostToDevice, st));
    if (rows)
        k_sym_scatter<<<nblk(rows * 32, 256), 256, 0, st>>>(cip.p, cix.p, g.own_lo, g.own_hi,
                                                          n_per, N, pos.p, keys);
    note_launch();
    KB_CUDA(cudaStreamSynchronize(st));
    for (int64_t q = 0; q < P; q++) h_counts[q] = (int64_t)c[q];
}

// step 2: the reversed arcs every rank sent here must be exactly this
// rank's arc set (as multisets: CSR rows hold distinct columns) -- true on
// every rank iff the whole arc set is closed under reversal
// (Graph.is_symmetric, graph.py:168-175)
int shard_symmetry_verify(Graph &g, const int64_t *recv, int64_t nrecv) {
    cudaStream_t st = g.stream;
    const int64_t m = g.nnz;
    if (nrecv != m) return 0;
    if (!m) return 1;
    DBuf<int64_t> cip, own, own_s, rs, rtmp;
    DBuf<int32_t> cix;
    compact_csr(g, cip, cix);
    own.alloc(m); own_s.alloc(m); rs.alloc(m); rtmp.alloc(m);
    const int64_t rows = g.own_hi - g.own_lo;
    k_own_keys<<<nblk(rows * 32, 256), 256, 0, st>>>(cip.p, cix.p, g.own_lo, g.own_hi, g.n,
                                                     own.p);
    note_launch();
    KB_CUDA(cudaMemcpyAsync(rtmp.p, recv, m * 8, cudaMemcpyDeviceToDevice, st));
    auto sort = [&](int64_t *in, int64_t *outp) {
        size_t tb = 0;
        KB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, in, outp, (int)m, 0, 64, st));
        DBuf<unsigned char> tmp;
        tmp.alloc(tb);
        KB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, in, outp, (int)m, 0, 64, st));
        note_launch();
    };
    sort(own.p, own_s.p);
    sort(rtmp.p, rs.p);
    DBuf<unsigned long long> bad;
    bad.alloc(1);
    KB_CUDA(cudaMemsetAsync(bad.p, 0, 8, st));
    k_keys_differ<<<nblk(m, 256), 256, 0, st>>>(own_s.p, rs.p, m, bad.p);
    note_launch();
    unsigned long long hb = 0;
    KB_CUDA(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    return hb ? 0 : 1;
}

}  // namespace kb
