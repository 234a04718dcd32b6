// Internal structures of the katzb200 engine (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/katzb200.h"

namespace kb {

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);

struct Error {
    int code;
    std::string msg;
};

#define KB_CUDA(call)                                                          \
    do {                                                                       \
        cudaError_t _e = (call);                                               \
        if (_e != cudaSuccess)                                                 \
            throw ::kb::Error{KB_ECUDA, std::string(#call) + ": " +            \
                                            cudaGetErrorString(_e)};           \
    } while (0)

#define KB_REQUIRE(cond, code, msg)                                            \
    do {                                                                       \
        if (!(cond)) throw ::kb::Error{(code), (msg)};                         \
    } while (0)

// ---------------------------------------------------------------- checked build
// `make checked` builds the library with -DKB_CHECKED (into _lib_checked/):
// KB_DCHECK(cond) in a kernel counts a failed invariant (index in range,
// count within capacity) in a per-translation-unit device word and records
// the source line, without faulting the context; every C-ABI call ends by
// reading all those words (dcheck_poll) and returns KB_ECUDA with the
// file:line of the first failure.  This stands in for compute-sanitizer,
// which is closed on the GPU pool.  In the normal build KB_DCHECK is empty.
#ifdef KB_CHECKED
int dcheck_register(void (*read)(unsigned long long *fails, int *line), const char *file);
#define KB_DCHECK(c)                                                           \
    do {                                                                       \
        if (!(c)) {                                                            \
            atomicAdd(&kb_dcheck_fail, 1ull);                                  \
            kb_dcheck_line = __LINE__;                                         \
        }                                                                      \
    } while (0)
namespace {
__device__ unsigned long long kb_dcheck_fail;
__device__ int kb_dcheck_line;
void kb_dcheck_read(unsigned long long *fails, int *line) {
    unsigned long long f = 0;
    int l = 0;
    cudaMemcpyFromSymbol(&f, kb_dcheck_fail, sizeof(f));
    cudaMemcpyFromSymbol(&l, kb_dcheck_line, sizeof(l));
    if (f) {                        // reported once, then re-armed
        const unsigned long long zero = 0;
        cudaMemcpyToSymbol(kb_dcheck_fail, &zero, sizeof(zero));
    }
    *fails = f;
    *line = l;
}
const int kb_dcheck_registered = dcheck_register(kb_dcheck_read, __BASE_FILE__);
}  // namespace
#else
#define KB_DCHECK(c) do { } while (0)
#endif
void dcheck_poll();   // throws Error{KB_ECUDA} if any KB_DCHECK failed (checked build)

// named tuning knobs (kb_tune); default when unset
int64_t tune_get(const char *name, int64_t dflt);

// number of kernel launches issued by the library (bench.py gpu_launches)
void note_launch(int64_t k = 1);
int64_t launch_count();

// KB_TRACE=1: host-side phase times (syncing the stream at each mark)
// overflow rows longer than this are summed by a block each (K1 tail)
constexpr int OVF_LONG = 256;

struct PhaseTrace {
    bool on;
    std::chrono::steady_clock::time_point t0;
    cudaStream_t st;
    explicit PhaseTrace(cudaStream_t s) : on(getenv("KB_TRACE") != nullptr), st(s) {
        t0 = std::chrono::steady_clock::now();
    }
    void mark(const char *what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        auto t1 = std::chrono::steady_clock::now();
        fprintf(stderr, "[kb] %-28s %9.3f ms\n", what,
                std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

// NVTX ranges (SURVEY.md §5 tracing: nsys ranges per iteration): host-side
// enqueue regions of every K1 level, check, result, update and ingest; the
// header-only NVTX3 API costs nothing unless a tool is attached
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    NvtxRange(const char *what, long long level) {
        char buf[64];
        snprintf(buf, sizeof buf, "%s %lld", what, level);
        nvtxRangePushA(buf);
    }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// ---------------------------------------------------------------- device buf
// All device work of a process runs on one non-blocking stream per device.
// Buffers come from dev_alloc: below BIG_ALLOC bytes, stream-ordered
// allocations from the device mempool (release threshold raised at first
// use, so per-iteration scratch costs no cudaMalloc round trip); from
// BIG_ALLOC up, cudaMalloc'd blocks kept in a per-device best-fit cache.
// Measured on B200 (tools/micro/alloc_bench.cu): growing the mempool costs
// 40-140 ms per GB-sized request and a fragmented pool 1.4 s for 3 GB,
// against 3-15 ms for cudaMalloc; cached blocks are reused in stream order
// (one stream per device), so reuse needs no synchronisation.
cudaStream_t device_stream();
cudaStream_t copy_stream();
bool host_is_pinned(const void *p);
void upload_h2d(void *dst, const void *src, size_t bytes, cudaStream_t cs);
void download_d2h(void *dst, const void *src, size_t bytes, cudaStream_t st);
void upload_gather_h2d(void *dst, size_t bytes, cudaStream_t cs,
                       const std::function<void(char *, size_t, size_t, int, int)> &fill);
constexpr size_t BIG_ALLOC = (size_t)64 << 20;
void *dev_alloc(size_t bytes);
void dev_free(void *p, size_t bytes);
void dev_mem_info(int64_t info[6]);

template <typename T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    bool owned = true;  // false: a view of memory owned elsewhere (borrow)
    DBuf() = default;
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), owned(o.owned) {
        o.p = nullptr; o.n = 0; o.owned = true;
    }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; owned = o.owned;
            o.p = nullptr; o.n = 0; o.owned = true;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count == 0) count = 1;
        p = (T *)dev_alloc(count * sizeof(T));
        n = count;
    }
    void borrow(T *q, size_t count) {
        release();
        p = q;
        n = count;
        owned = false;
    }
    void release() {
        if (p && owned) dev_free(p, n * sizeof(T));
        p = nullptr;
        n = 0;
        owned = true;
    }
    size_t bytes() const { return n * sizeof(T); }
};

// ---------------------------------------------------------------- layout
// SELL-32 over "virtual rows":
//   vr in [0, nseg)        : segments of heavy rows (deg > split), length <= split
//   vr in [nseg, nvr)      : ordinary rows, new id = nh + (vr - nseg)
// Rows are relabelled by descending out-degree (stable in the original id),
// so new ids [0, nh) are the heavy rows, [0, nv) the rows with arcs and
// [nv, n) the rows without.  Within a row the column order is the original
// ascending-id order of graph.py:191-192, stored as *new* ids.
// Slice s holds 32 consecutive virtual rows.  If its padded width w <= 4 the
// slot of (step j, lane l) is cols[off + j*32 + l]; otherwise w % 4 == 0 and
// the slot is cols[off + (j/4)*128 + l*4 + j%4] (one int4 per lane per 4
// steps).
struct Sell {
    DBuf<int32_t> cols;
    DBuf<int64_t> slice_off;
    DBuf<int32_t> slice_w;
    DBuf<int32_t> vlen;
    int64_t nslices = 0, nvr = 0, nseg = 0, elems = 0;
    int64_t nwide = 0;  // slices [nwide, nslices) all have width <= 4
};

struct Graph {
    int device = 0;
    int sm_count = 0;
    int64_t n = 0, nnz = 0, nv = 0, nh = 0, nzero = 0, max_deg = 0;
    int64_t nh_long = -1;  // leading heavy rows with > 8 segments (fresh layouts), else -1
    int64_t split = 0, hot = 0;
    // sharded graphs (KB_GRAPH_NO_RELABEL with an owned block of 2^k ids):
    // K1's shared-memory hot set takes the first hot_per ids of each block
    int64_t hot_per = 0;
    int hot_shift = 0;
    int64_t version = 1;
    DBuf<int32_t> perm;    // new -> original id
    DBuf<int32_t> iperm;   // original -> new id
    DBuf<int32_t> deg;     // out-degree by new id
    // canonical CSR-with-slack (original ids, rows ascending): row v starts
    // at indices[indptr[v]] and uses the first rlen[v] slots.  Compact as
    // built (capacity = indptr[v+1] - indptr[v]); after the first update
    // (slack) capacities live in rcap and rows may be relocated to the
    // reserved tail [tail, indices.n) when a batch outgrows them
    DBuf<int64_t> indptr;
    DBuf<int32_t> indices;
    DBuf<int32_t> rlen;
    DBuf<int32_t> rcap;
    int64_t tail = 0;
    bool slack = false;      // rcap/tail valid (after an update)
    // row maps of the SELL layout; empty while implicit_rows (fresh
    // relabelling: heavy [0,nh), normal [nh,nv), empty [nv,n))
    bool implicit_rows = true;
    bool sell_dirty = false; // arcs changed since the SELL build
    int64_t own_lo = 0, own_hi = -1;  // rows this device computes (shards)
    bool relabel = true;     // rows degree-sorted (false: identity, shard graphs)
    DBuf<int32_t> label;     // tie-break/output label by new id (empty: perm)
    const int32_t *labels() const { return label.p ? label.p : perm.p; }
    bool mutated = false;    // a batch was applied: the relabelling is no longer
                             // degree-sorted and empty rows are not a tail
    DBuf<int32_t> hrow, vrow, zrows;
    // dynamic patching of the SELL layout: new id -> normal virtual row /
    // heavy index (-1 if none); rows that no longer fit their slice are
    // "overflow" rows recomputed from the canonical CSR after K1
    DBuf<int32_t> vr_of_row, h_of_row;
    DBuf<int32_t> ovf, ovf_flag;
    DBuf<unsigned long long> ovf_count;
    int64_t n_ovf = 0;
    DBuf<int32_t> ovf_long;           // overflow rows longer than OVF_LONG arcs
    int64_t n_ovf_long = 0;
    DBuf<double> ovf_sum;             // their sums, computed beside K1 (side stream)
    cudaStream_t side_stream = nullptr;
    cudaEvent_t side_fork = nullptr, side_join = nullptr;
    Sell sell;
    // heavy-row combine: segments of heavy row h are seg_list[seg_ptr[h] ..
    // seg_ptr[h+1]) in order (indices into the segment-sum buffer)
    // original ids of the rows with / without out-arcs, ascending
    DBuf<int32_t> orig_pos, orig_zero;
    DBuf<int32_t> seg_ptr;
    DBuf<int32_t> seg_list;
    // fused omega exchange (shards): two full-length level buffers (ping-
    // pong by level parity, cudaMalloc'd so they can be exported through
    // CUDA IPC) and, per parity, the same buffers of the other ranks: K1's
    // epilogue stores every owned row's w into all of them
    double *exch[2] = {nullptr, nullptr};
    size_t exch_n = 0;
    std::vector<double *> exch_peer[2];
    std::vector<void *> exch_opened;  // IPC mappings to close
    cudaStream_t stream = nullptr;
    int symmetric = -1;  // cached result of kb_graph_is_symmetric
    int64_t sym_n_per = 0;  // shards built from a host CSR (symmetry decided across ranks)
    size_t device_bytes() const;
    Graph() = default;
    Graph(const Graph &) = delete;
    Graph &operator=(const Graph &) = delete;
    ~Graph() {
        if (side_stream) {
            cudaStreamSynchronize(side_stream);
            cudaStreamDestroy(side_stream);
            cudaEventDestroy(side_fork);
            cudaEventDestroy(side_join);
        }
        for (void *p : exch_opened) cudaIpcCloseMemHandle(p);
        for (double *&p : exch)
            if (p) { cudaFree(p); p = nullptr; }
    }
};

// ranks a fused omega exchange stores to besides the local one (8 GPUs)
constexpr int KB_MAX_PEERS = 7;

// ---------------------------------------------------------------- state
struct State {
    Graph *g = nullptr;
    double alpha = 0, gamma = 0, eps = 0;
    int undirected = 0, kind = 0, keep_all = 1;
    int64_t k = 0, u = 0, v = 0;
    int64_t r = 0, max_iter = 0;
    int64_t graph_version = 0;
    std::vector<DBuf<double>> levels;  // new-id space, n+1 slots each
    int64_t level_base = 0;            // level index of levels[0]
    DBuf<double> katz, lower, upper;   // new-id space
    DBuf<double> seg_sum;
    // active set (new ids) -- ping-pong buffers; count lives on the device
    DBuf<int32_t> act[2];
    int cur = 0;
    bool act_dense = true;  // active == arange(n) (never materialised)
    int64_t tail_zero_from = 0;  // new ids >= this have lower == upper == 0
    bool zero_tail_exact = true; // and exactly those (no dynamic change yet)
    // lazy initial vectors (engine.py:147-151): init_pending -- katz, lower,
    // upper and levels[0] not written yet (the first K1's ones step writes
    // the first three itself); ones_pending -- levels[0] (ones) not written
    bool init_pending = false, ones_pending = false;
    DBuf<int32_t> cand;          // selection candidates (capacity n)
    DBuf<uint64_t> stK;          // staged keys/uppers/ids of the active set
    DBuf<double> stU;
    DBuf<int32_t> stI;
    int64_t m_host = 0;     // |active| mirrored after each check
    // device scratch for the checks
    DBuf<unsigned long long> scratch_u64;
    DBuf<int32_t> scratch_i32;
    DBuf<double> scratch_f64;
    DBuf<unsigned char> cub_tmp;
    DBuf<unsigned long long> work_counter;
    unsigned long long *h_flags = nullptr;  // pinned host mirror
    DBuf<unsigned long long> pub_dev;       // check verdict words, copied to h_flags per batch
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    double last_check_ms = 0;
    // K1 launch timing: event pairs recorded around each SpMV+bounds step
    std::vector<cudaEvent_t> k1_ev;
    size_t k1_used = 0, k1_read = 0;
    double spmv_ms = 0;
    int64_t spmv_launches = 0;
    int64_t check_full_sorts = 0;   // RANKING checks the certificates could not decide
    // RANKING: the last refuting pair (q, x): x ranked above q with
    // lower[x] <= fl(upper[q] - eps); while it still refutes, a check is
    // "not converged" without a pass over the set
    int32_t rk_q = -1, rk_x = -1;
    // speculative iteration (TOPK runs): K1 of r+1 is queued behind check r
    // and exits at once if that check converged (abort_flag, set on device)
    DBuf<unsigned long long> abort_flag;
    bool spec_abort = false;
    // RANKING chain: the cached pair's test fused into the next K1's tail
    // (k_sell_narrow_tma's last CTA), when that kernel runs the level
    struct PairFuse {
        bool want = false, done = false;
        int32_t q = -1, x = -1;
        double eps = 0;
        const int32_t *perm = nullptr;
        unsigned long long *out = nullptr, *abort = nullptr, *pub = nullptr, *k1c = nullptr;
    } pair_fuse;
    DBuf<unsigned long long> pair_done;     // arrival counter of the fused test
    // RANKING runs skip the per-iteration lower/upper stores (K1 writes w and
    // katz only); materialize_bounds recomputes them, bit for bit, before
    // anything reads them
    bool lazy_bounds = false, bounds_stale = false;
    bool exch_on = false;     // levels live in the graph's exchange buffers
    bool counter_zeroed = false;  // the next K1's work counter was reset on the device
    int exch_parity = 0;      // parity of the level being computed
    cudaEvent_t chk_ev = nullptr;
    cudaEvent_t chk_ev2 = nullptr;   // the second batch in flight (RANKING chain)
    DBuf<unsigned long long> tie_count;  // k-boundary ties dropped with gap < eps (rule 4)
    bool rank_order_pending = false;    // RANKING: active not yet in (-lower, id) order
    std::vector<int64_t> level_sizes;   // UpdateStats.level_sizes of the last update
    const double *x_level() const { return levels.back().p; }
};

// A scanned text file (kb_text.cu): bytes, newline offsets, per-line class
// and ids, anomaly lines and arc lines (indices, ascending)
struct TextScan {
    int device = 0;
    int batches = 0;
    int64_t nbytes = 0, n_nl = 0, n_lines = 0, n_cand = 0, n_arcs = 0;
    int64_t first_arc_line = -1, max_id = -1;
    DBuf<char> buf;
    DBuf<int64_t> nl, cand, arcs;
    DBuf<uint8_t> kind;
    DBuf<int32_t> u, v;
};

// ---------------------------------------------------------------- kernels
void text_scan(TextScan &t, const char *h_bytes, int64_t nbytes, int batches);
void text_candidates(TextScan &t, int64_t *h_out);
void text_lines(TextScan &t, uint8_t *h_kind, int32_t *h_u, int32_t *h_v);
void text_csr(TextScan &t, int64_t n, int undirected, const int64_t *h_extra, int64_t n_extra,
              DBuf<int64_t> &indptr, DBuf<int32_t> &indices, int64_t &nnz);
void launch_iterate(State &s, cudaStream_t st);
// write whatever initial vectors are still pending (ensure_init: all of
// them; ensure_ones: levels[0]) -- before any read outside the first K1
void ensure_init(State &s);
void ensure_ones(State &s);
void run_spmv(State &s, cudaStream_t st, const double *x, double *w, bool level_only);
void collect_k1_times(State &s);
void materialize_bounds(State &s, cudaStream_t st);
void run_segments(State &s, cudaStream_t st, const double *x);
bool run_check(State &s, cudaStream_t st);      // returns converged
// TOPK check split around its one host read: enqueue (kernels, publish the
// verdict to abort_flag, D2H into h_flags, record chk_ev) / finish (after
// chk_ev: adopt the new active set, return converged); -1: not applicable
int topk_check_enqueue(State &s, cudaStream_t st);
bool topk_run_device(State &s, cudaStream_t st);  // TOPK loop, one host sync per batch
bool topk_check_finish(State &s, int nxt);
bool ranking_pair_chain(State &s, cudaStream_t st);   // device-driven cached-pair levels
void materialize_rank_order(State &s, cudaStream_t st);
double run_gap(State &s, cudaStream_t st);
void result_device(State &s, cudaStream_t st, DBuf<int64_t> *order64, DBuf<double> *lower,
                   DBuf<double> *upper, int64_t *h_pairs);
void run_result(State &s, cudaStream_t st, int64_t *order, double *lower,
                double *upper, int64_t *pairs);
void gather_to_original(const Graph &g, const double *src_new, double *dst_orig,
                        cudaStream_t st);
void build_graph(Graph &g, const int64_t *h_indptr, const int32_t *h_indices);
void build_graph_device(Graph &g);
void build_sell(Graph &g, bool fresh, bool fill = true);
void make_slack(Graph &g);
void slack_layout(Graph &g, const int32_t *extra, DBuf<int64_t> &nip, DBuf<int32_t> &nix,
                  int64_t &total);
void compact_csr(Graph &g, DBuf<int64_t> &indptr, DBuf<int32_t> &indices);
void patch_sell(Graph &g, const int32_t *rows_orig, int64_t ne);
void apply_batch_to_graph(Graph &g, const int64_t *ins, int64_t n_ins, const int64_t *dels,
                          int64_t n_dels);
void graph_has_arcs(Graph &g, const int64_t *arcs, int64_t m, unsigned char *present);
int64_t graph_max_degree_after(Graph &g, const int64_t *ins, int64_t n_ins, const int64_t *dels,
                               int64_t n_dels);
void graph_out_degrees(Graph &g, int64_t *out);
void local_topk(State &s, cudaStream_t st, int64_t k, uint64_t *keys, int64_t *labels,
                double *uppers, int64_t *count);
void apply_cut(State &s, cudaStream_t st, uint64_t kstar, int64_t istar);
void select_global(int device, const uint64_t *keys, const int64_t *labels, const double *uppers,
                   int64_t ncand, int64_t k, double eps, uint64_t *kstar, int64_t *istar,
                   int *prefix_ok);
int64_t count_inversions(const int64_t *h_order_a, const int64_t *h_order_b, int64_t n);
bool foster(Graph &g, double alpha, double tol, int64_t max_iter, double *h_values,
            int64_t *iterations, double *residual);
int cg_katz(Graph &g, double alpha, double residual_tol, int64_t max_iter, double *h_values,
            int64_t *iterations, double *residual);
void shard_propose(State &s, cudaStream_t st, int64_t k, unsigned long long *blk);
void shard_cut(State &s, cudaStream_t st, const unsigned long long *blocks, int64_t P, int64_t k,
               long long *word);
void shard_commit(State &s, int64_t m);
void rank_gathered(State &s, int64_t n, int64_t *order, double *lower, double *upper,
                   int64_t *pairs);
void rank_bounds(int device, int64_t n, const double *lower, const double *upper, int64_t *order,
                 int64_t *pairs);
void update_batch(State &s, const int64_t *ins, int64_t n_ins, const int64_t *dels,
                  int64_t n_dels, double theta, double new_gamma, kb_update_stats *stats);
void rmat_device_csr(int scale, int64_t edge_factor, const uint64_t state[4], double a,
                     double ab, double abc, DBuf<int64_t> &indptr, DBuf<int32_t> &indices,
                     int64_t &nnz_out);
void grid_device_csr(int64_t n, DBuf<int64_t> &indptr, DBuf<int32_t> &indices,
                     int64_t &nnz_out);
int graph_is_symmetric(Graph &g);
void find_labels(Graph &g, const int64_t *h_targets, int64_t m, int64_t *h_ids);
void build_shard(Graph &full, int64_t P, int64_t rank, Graph &out, int64_t *n_per_out,
                 int64_t *owned_out);
void build_shard_host(Graph &out, int64_t n, int64_t nnz, const int64_t *h_ip,
                      const int32_t *h_ix, int64_t P, int64_t rank, int64_t *n_per_out,
                      int64_t *owned_out);
void shard_symmetry_keys(Graph &g, int64_t P, int64_t *keys, int64_t *h_counts);
int shard_symmetry_verify(Graph &g, const int64_t *recv, int64_t nrecv);
void ensure_cub_tmp(State &s, size_t bytes);
// stable (uint64 key, int32 value) radix sort (kb_sort.cu); input in (k0, v0),
// scratch (k1, v1); returns true if the sorted pairs are in (k1, v1)
bool radix_sort_pairs(uint64_t *k0, int32_t *v0, uint64_t *k1, int32_t *v1, int64_t n,
                      int device, cudaStream_t st);

}  // namespace kb
