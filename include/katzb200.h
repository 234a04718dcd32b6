/*
 * katzb200 -- C-ABI of the B200-native bounded-Katz ranking engine.
 *
 * The reference (katzbounds, arxiv 1807.03847) is a pure-Python package; it
 * has no FFI of its own.  These entry points are the ones its Python engine
 * would bind to hand the hot path to native code: each one replaces the
 * reference function named beside it (paths under
 * /root/reference/pkg/src/katzbounds/).  All functions return a status code
 * (KB_OK == 0); on failure kb_last_error() gives a message.  Plain pointers
 * and sizes only -- no torch or CUDA types cross this boundary.
 *
 * Id spaces: every array that crosses the ABI is indexed by the caller's
 * (original) node ids.  Internally the device relabels rows by descending
 * out-degree; that is invisible here.
 *
 * Ownership: host arrays are borrowed for the duration of a call; device
 * memory is owned by the handles and freed by the *_destroy calls.
 * Threading: a kb_state is used by one thread at a time; a kb_graph may be
 * shared by many states (read-only) except during kb_update_batch.
 */
#ifndef KATZB200_H
#define KATZB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -> katzbounds.errors classes (errors.py:9-58) */
enum {
    KB_OK = 0,
    KB_EPARAM = 1,        /* ParameterError       errors.py:29 */
    KB_ESTATE = 2,        /* StateError           errors.py:33 */
    KB_ECONVERGENCE = 3,  /* ConvergenceError     errors.py:37-50 */
    KB_ENUMERIC = 4,      /* NumericError         errors.py:57 */
    KB_EBATCH = 5,        /* BatchPreconditionError errors.py:25 */
    KB_ENODERANGE = 6,    /* NodeRangeError       errors.py:21 */
    KB_ECUDA = 7,         /* device failure (no reference analogue) */
    KB_ENOMEM = 8
};

/* Criterion kinds (engine.py:28-31) */
enum { KB_RANKING = 0, KB_TOPK = 1, KB_SCORE = 2, KB_PAIR = 3 };

/* vectors readable through kb_get_vector */
enum { KB_VEC_LEVEL = 0, KB_VEC_KATZ = 1, KB_VEC_LOWER = 2, KB_VEC_UPPER = 3 };

typedef struct kb_graph kb_graph;
typedef struct kb_state kb_state;
typedef struct kb_text kb_text;
typedef struct kb_ranking kb_ranking;

typedef struct {
    int64_t n;                /* node_count                                  */
    int64_t nnz;              /* arcs                                        */
    int64_t max_out_degree;   /* Graph.max_out_degree  graph.py:154-158      */
    int64_t nonisolated;      /* rows with out-degree > 0                    */
    int64_t heavy_rows;       /* rows split into segments (deg > threshold)  */
    int64_t segments;         /* virtual rows covering the heavy rows        */
    int64_t slices;           /* 32-row SELL slices                          */
    int64_t sell_elems;       /* stored column slots incl. padding           */
    int64_t split_threshold;  /* rows longer than this are segmented         */
    int64_t hot_size;         /* leading (hottest) x entries staged in smem  */
    int64_t version;          /* bumped by kb_update_batch                   */
    int64_t device_bytes;     /* device memory held by the graph             */
    int64_t overflow_rows;    /* rows edited past their SELL lane (batches)  */
    int64_t overflow_long;    /* ... of which longer than 256 arcs           */
} kb_graph_info;

typedef struct {
    int64_t r;                /* KatzState.r                                 */
    int64_t active;           /* KatzState.active.size                       */
    int64_t max_iterations;   /* KatzState.max_iterations                    */
    int64_t levels_kept;      /* len(KatzState.levels)                       */
    double  alpha, gamma, epsilon;
    double  last_check_ms;    /* device time of the last kb_check            */
    double  spmv_ms;          /* summed device time of the K1 launches       */
    int64_t spmv_launches;    /* number of K1 iterations timed in spmv_ms    */
    int64_t check_full_sorts; /* ranking checks that needed the full sort    */
    int64_t k_boundary_ties;  /* SURVEY 8(c) rule 4: nodes tied exactly with
                                 the k-th lower bound and dropped with
                                 gap < eps, summed over TOPK checks -- where
                                 argpartition (engine.py:359) may choose
                                 differently; 0 = active and r are the
                                 reference's whatever its tie choice      */
} kb_state_info;

typedef struct {
    int64_t batch_size, seeds, visited, reactivated, resumed_iterations;
    int64_t aborted_level;    /* -1 == None                                  */
    int64_t n_level_sizes;    /* the full count (may exceed 64)              */
    int64_t level_sizes[64];  /* UpdateStats.level_sizes (dynamic.py:35):
                                 the first 64; kb_update_level_sizes has all */
} kb_update_stats;

/* ---- library ---- */
const char *kb_last_error(void);
int kb_version(void);
int kb_device_count(int *count);

/* ---- measurement plumbing (bench.py): device-stream timer, kernel launch
 * counter, page-locking of caller buffers for the host<->device copies */
int kb_timer(int device, int op /* 0 start, 1 stop */, double *elapsed_ms);
int kb_launch_count(int64_t *count);
/* named tuning knobs of the kernels (e.g. "k1.depth", "k1.hot"); defaults
 * apply when unset */
int kb_tune(const char *name, int64_t value);
int kb_host_register(void *ptr, int64_t bytes);
int kb_host_unregister(void *ptr);

/* ---- graph ingest: replaces Graph.out_csr() + the scipy CSR the engine
 * reads (graph.py:177-197) with a device-resident, degree-relabelled SELL-32
 * layout.  indptr: n+1 int64, indices: nnz int32, each row strictly
 * ascending with ids in [0, n) (checked: KB_EPARAM otherwise).  The columns
 * are uploaded in row chunks and laid out while later chunks are in flight;
 * the symmetry flag (kb_graph_is_symmetric) is decided in the same pass.
 * split_threshold <= 0 and hot_size < 0 select the defaults. */
int kb_graph_create(int device, int64_t n, int64_t nnz, const int64_t *indptr,
                    const int32_t *indices, int64_t split_threshold,
                    int64_t hot_size, kb_graph **out);
/* flags for kb_graph_create_ex */
enum { KB_GRAPH_NO_RELABEL = 1, KB_GRAPH_SYMMETRIC = 2 };
/* kb_graph_create with options: KB_GRAPH_NO_RELABEL keeps the caller's row
 * order as the device id space (multi-GPU shards, whose omega blocks must stay
 * contiguous for the all-gather); `labels` (n int32, may be NULL) replaces
 * the node id in every tie-break (engine.py:365, :401) -- shards pass the
 * original ids of the exchange layout.  Rows [own_lo, own_hi) are the ones
 * this device computes (own_hi < 0: all); KatzState.gap covers only them. */
int kb_graph_create_ex(int device, int64_t n, int64_t nnz, const int64_t *indptr,
                       const int32_t *indices, int64_t split_threshold,
                       int64_t hot_size, int flags, const int32_t *labels,
                       int64_t own_lo, int64_t own_hi, kb_graph **out);
/* Rank `rank` of `nranks`' row shard of a device graph, built on that
 * graph's device with no host round trip (the multi-GPU
 * split of KatzState._matvec's rows, engine.py:181-208): rows are dealt by
 * degree rank round-robin, the shard is a KB_GRAPH_NO_RELABEL graph over the
 * exchange layout e(v) = (q mod P)*n_per + q div P whose non-owned rows are
 * empty, each owned row keeps its arcs in ascending original-id order, and
 * the tie-break labels are the node ids (padding: n, n+1, ...).  The shard
 * inherits `full`'s symmetry flag.  Outputs n_per = ceil(n/P) and the number
 * of rows this rank owns (its block's head). */
/* The same shard straight from a host CSR (indptr n+1 int64, indices nnz
 * int32, rows strictly ascending -- checked): only indptr (for the degree
 * order) and this rank's own rows are uploaded to `device` (the rows
 * gathered on the host into a page-locked ring), so graphs larger than one
 * GPU shard too.  The shard's symmetry is decided across the ranks with
 * kb_shard_symmetry_keys / kb_shard_symmetry_verify. */
int kb_graph_create_shard_host(int device, int64_t n, int64_t nnz, const int64_t *indptr,
                               const int32_t *indices, int64_t nranks, int64_t rank,
                               int64_t split_threshold, int64_t hot_size, kb_graph **out,
                               int64_t *n_per, int64_t *owned);
/* Graph.is_symmetric (graph.py:168-175) of a sharded graph, exactly: every
 * rank writes the reverse of each of its arcs as a device key, grouped by the
 * rank owning the reversed arc's row (keys: nnz int64 device buffer;
 * counts[q]: keys for rank q); after an all-to-all of those groups each rank
 * verifies that the keys it received are exactly its own arcs (ok = 1); the
 * graph is symmetric iff every rank says so. */
int kb_shard_symmetry_keys(kb_graph *shard, int64_t nranks, int64_t *keys, int64_t *counts);
int kb_shard_symmetry_verify(kb_graph *shard, const int64_t *recv, int64_t nrecv, int *ok);
/* Device ids of the nodes whose tie-break label is labels[j] (-1: none),
 * m <= 64: a shard's exchange ids of given node ids (sharded PAIR checks,
 * engine.py:346-353). */
int kb_graph_find_labels(kb_graph *g, const int64_t *labels, int64_t m, int64_t *ids);
int kb_graph_create_shard(kb_graph *full, int64_t nranks, int64_t rank,
                          int64_t split_threshold, int64_t hot_size, kb_graph **out,
                          int64_t *n_per, int64_t *owned);
/* Device generators, bit-identical to katzbounds.generate (generate.py:38-103)
 * loaded with undirected=True: R-MAT on n = 2^scale nodes from numpy's PCG64
 * stream whose current state is pcg_state = {state_hi, state_lo, inc_hi,
 * inc_lo} (np.random.default_rng(seed).bit_generator.state); a, ab, abc are
 * the quadrant thresholds exactly as generate.py:73-74 evaluates them. */
int kb_graph_create_rmat(int device, int scale, int64_t edge_factor,
                         const uint64_t *pcg_state, double a, double ab,
                         double abc, int64_t split_threshold, int64_t hot_size,
                         kb_graph **out);
int kb_graph_create_grid(int device, int64_t n, int64_t split_threshold,
                         int64_t hot_size, kb_graph **out);
/* the canonical CSR (original ids, rows ascending): n+1 / nnz entries */
int kb_graph_get_csr(kb_graph *g, int64_t *indptr, int32_t *indices);
/* Graph.has_arc / validate_batch presence test (graph.py:207-220), batched:
 * arcs = m (src,dst) int64 pairs, present = m bytes */
int kb_graph_has_arcs(kb_graph *g, const int64_t *arcs, int64_t m, uint8_t *present);
/* max out-degree after applying a batch (dynamic.py:151-157), on the device */
int kb_graph_max_degree_after(kb_graph *g, const int64_t *ins, int64_t n_ins,
                              const int64_t *dels, int64_t n_dels, int64_t *max_degree);
/* Graph.out_degrees (graph.py:160-161): n int64 */
int kb_graph_out_degrees(kb_graph *g, int64_t *out);
/* Graph.apply_batch (graph.py:201-205) without a state: the device
 * CSR-with-slack is edited in place (the caller validated the batch) */
int kb_graph_apply_batch(kb_graph *g, const int64_t *ins, int64_t n_ins,
                         const int64_t *dels, int64_t n_dels);
int kb_graph_destroy(kb_graph *g);
int kb_graph_info_get(const kb_graph *g, kb_graph_info *info);
/* Graph.is_symmetric (graph.py:168-175), evaluated on the device */
int kb_graph_is_symmetric(kb_graph *g, int *symmetric);

/* ---- state: replaces engine.init (engine.py:248-283).  alpha/gamma/cap are
 * computed by the caller with the reference's own expressions
 * (engine.py:96-119, :286-293) so the device sees bit-identical inputs. */
int kb_state_create(kb_graph *g, double alpha, double gamma, int undirected,
                    int kind, double epsilon, int64_t k, int64_t u, int64_t v,
                    int keep_all_levels, int64_t max_iterations,
                    kb_state **out);
int kb_state_destroy(kb_state *s);
int kb_state_info_get(const kb_state *s, kb_state_info *info);
int kb_state_set_max_iterations(kb_state *s, int64_t max_iterations);

/* iterate_once (engine.py:296-319), `steps` times, no stopping test */
int kb_iterate(kb_state *s, int64_t steps);
/* check_converged (engine.py:333-379); may shrink the active set */
int kb_check(kb_state *s, int *converged);
/* run (engine.py:382-396) without the final ranking_result: iterate+check on
 * the device until converged; KB_ECONVERGENCE at the cap (r, gap via info) */
int kb_run(kb_state *s, int *converged);
/* KatzState.gap (engine.py:172-174) */
int kb_gap(kb_state *s, double *gap);
/* epsilon_separated (engine.py:322-330) */
int kb_epsilon_separated(kb_state *s, int64_t w, int64_t v, int *separated);

/* ranking_result (engine.py:399-408) + separated_fraction (:411-427):
 * order (n int64), lower/upper (n fp64, by node id), and the exact number of
 * separated ordered pairs; any output pointer may be NULL. */
int kb_result(kb_state *s, int64_t *order, double *lower, double *upper,
              int64_t *separated_pairs);
int kb_separated_pairs(kb_state *s, int64_t *separated_pairs);

/* read KatzState vectors (by node id): levels[level], katz, lower, upper */
int kb_get_vector(kb_state *s, int which, int64_t level, double *out);
/* KatzState.active in its current order (node ids); `out` holds >= active */
int kb_get_active(kb_state *s, int64_t *out);

/* ---- multi-GPU building blocks (one process per GPU; the caller moves the
 * omega blocks and candidates with NCCL) */
/* restrict the active set (node ids of this graph) */
int kb_state_set_active(kb_state *s, const int64_t *ids, int64_t m);
/* the same for the contiguous internal id range [lo, hi) of a
 * KB_GRAPH_NO_RELABEL graph (a shard's owned rows), without a host list */
int kb_state_set_active_range(kb_state *s, int64_t lo, int64_t hi);
/* device pointer of a state vector (device id space: node ids for
 * KB_GRAPH_NO_RELABEL graphs) */
int kb_state_vector_ptr(kb_state *s, int which, int64_t level, void **ptr);
int kb_sync(int device);
/* the k best active nodes by (-lower, label) without deactivating anything:
 * raw lower bits, labels and upper bounds, sorted; count <= k */
int kb_check_local_topk(kb_state *s, int64_t k, uint64_t *keys, int64_t *labels,
                        double *uppers, int64_t *count);
/* global top-k of gathered candidates: the cut (k-th key and label) and the
 * adjacent-separation test of the prefix (engine.py:365-378) */
int kb_select_global(int device, const uint64_t *keys, const int64_t *labels,
                     const double *uppers, int64_t ncand, int64_t k, double eps,
                     uint64_t *kstar, int64_t *istar, int *prefix_separated);
/* keep the winners of the global cut and the survivors
 * fl(upper - eps) >= threshold (engine.py:367-373); returns |active| */
int kb_check_apply_cut(kb_state *s, uint64_t kstar, int64_t istar, int64_t *active);
/* Fused omega exchange (B200-native replacement of the per-iteration
 * all-gather).  A shard graph owns two full-length level
 * buffers (parity 0/1, cudaMalloc'd); each rank registers the other ranks'
 * buffers of each parity -- by CUDA IPC handle across processes or by device
 * pointer within one -- and K1's epilogue stores every owned row's w into
 * all of them over NVLink while it computes, followed by a system-scope
 * fence.  The caller's per-check collectives order the ranks' iterations.
 * A state using it keeps two levels (keep_levels = 0). */
int kb_graph_exchange_alloc(kb_graph *g);
int kb_graph_exchange_ptr(kb_graph *g, int parity, void **ptr);
/* 64-byte cudaIpcMemHandle_t of this rank's buffer */
int kb_graph_exchange_handle(kb_graph *g, int parity, void *handle);
/* a peer's buffer of `parity`: IPC handle (opened here) or a device pointer */
int kb_graph_exchange_add_peer(kb_graph *g, int parity, const void *handle, void *ptr);
int kb_state_exchange(kb_state *s, int on);
/* ranking_result + separated pairs on caller vectors indexed by node id */
int kb_rank_bounds(int device, int64_t n, const double *lower, const double *upper,
                   int64_t *order, int64_t *separated_pairs);

/* graph.load_edge_list (graph.py:260-320) / dynamic.load_batches
 * (dynamic.py:216-253), parsed on the device.  scan: copies `bytes` to the
 * device, splits lines at '\n' and classifies each one; info[0..4] =
 * lines, arc lines, anomaly lines, first arc line (-1: none), max arc id.
 * Anomalies (anything outside the plain ASCII grammar, and every "NODES"
 * line) are for the caller to re-read with the reference's exact rules:
 * candidates writes (line index, byte start, byte end) triples in line
 * order.  lines copies the per-line class (edges: 0 skip, 1 arc, 2 header,
 * 3 anomaly; batches: 0 separator, 1 insert, 4 delete, 3 anomaly) and ids.
 * create_text builds the canonical CSR of the arc lines plus `n_extra`
 * caller-resolved (u, v) pairs over [0, n), with reversals if undirected. */
int kb_text_scan(int device, const void *bytes, int64_t nbytes, int batches,
                 kb_text **out, int64_t *info);
int kb_text_candidates(kb_text *t, int64_t *lines);
int kb_text_lines(kb_text *t, uint8_t *kind, int32_t *u, int32_t *v);
int kb_text_destroy(kb_text *t);
int kb_graph_create_text(kb_text *t, int64_t n, int undirected,
                         const int64_t *extra_arcs, int64_t n_extra,
                         int64_t split_threshold, int64_t hot_size,
                         kb_graph **out);

/* baselines.foster (baselines.py:36-68): c <- alpha*A*c + 1 from ones until
 * max|change| < tol; values = c - 1 by original id (n doubles).  At the cap:
 * KB_ECONVERGENCE with values/iterations/residual holding the partial. */
int kb_foster(kb_graph *g, double alpha, double tol, int64_t max_iter,
              double *values, int64_t *iterations, double *residual);

/* baselines.cg_katz (baselines.py:71-129): CG on (I - alpha*A) z = 1 from
 * z = 1; values = alpha*A*z.  KB_ENUMERIC on breakdown, KB_ECONVERGENCE at
 * the cap (values = the partial).  The caller checks symmetry. */
int kb_cg_katz(kb_graph *g, double alpha, double residual_tol, int64_t max_iter,
               double *values, int64_t *iterations, double *residual);

/* cli.concordant_fraction (cli.py:349-386): the number of node pairs the two
 * rankings (permutations of 0..n-1, host arrays) order differently;
 * concordant fraction = 1 - inversions / (n(n-1)/2).  KB_EPARAM unless both
 * are permutations. */
int kb_ranking_inversions(int device, int64_t n, const int64_t *order_a,
                          const int64_t *order_b, int64_t *inversions);

/* engine.ranking_result kept on the device (engine.py:399-408): a snapshot
 * of order (int64 original ids, rank order), lower and upper (by original
 * id) plus the exact separated-pair count; read copies any slice (which: 0
 * order, 1 lower, 2 upper; 8-byte elements) to the host, so a caller that
 * needs only the top k copies k entries. */
int kb_ranking_snapshot(kb_state *s, kb_ranking **out, int64_t *separated_pairs);
int kb_ranking_read(kb_ranking *r, int which, int64_t offset, int64_t count, void *host);
int kb_ranking_destroy(kb_ranking *r);

/* device memory held by the library: info[0..3] = stream-ordered pool
 * (buffers < 64 MiB) reserved bytes, reserved high-water mark, used bytes,
 * used high-water mark; info[4..5] = bytes held in large cached blocks
 * (>= 64 MiB, cudaMalloc'd, reused best-fit) and the part in use.  reserve
 * grows the pool by one allocation of `bytes` returned to it at once. */
int kb_pool_info(int device, int64_t *info);
int kb_pool_reserve(int device, int64_t bytes);

/* the library's stream on `device` (every call above is ordered on it; a
 * caller running collectives on the same stream needs no host sync) */
int kb_stream(int device, void **stream);

/* device-resident sharded TOPK check (no host copies; all async on the
 * library stream).  propose: this rank's k best active nodes into a device
 * block of 1 + 3k 64-bit words [count, lower bit keys, labels, uppers].
 * cut: from the nblocks all-gathered blocks, the global k-th cut and the
 * adjacent-separation test; splits the local active set (winners, then
 * survivors) and writes word[0] = word[1] = new local count, word[2] =
 * prefix ok.  commit: the new local count, read back by the caller after
 * all-reducing word[0] (required before the next propose/cut). */
int kb_shard_propose(kb_state *s, int64_t k, void *block);
int kb_shard_cut(kb_state *s, const void *blocks, int64_t nblocks, int64_t k,
                 void *word);
int kb_shard_commit(kb_state *s, int64_t active);
/* K1 of the next level queued behind a check's device word (after its
 * all-reduce): it exits on the device if the word says converged, so the
 * GPU does not idle through the host read; the caller then drops that
 * level with kb_state_rollback */
int kb_shard_iterate_spec(kb_state *s, const long long *word, int64_t k);
int kb_state_rollback(kb_state *s);

/* ranking_result of a sharded run: the state's lower/upper hold all shards'
 * blocks (exchange layout, after the all-gather) and the graph labels map
 * exchange ids to the n node ids; outputs by node id, any may be NULL */
int kb_rank_gathered(kb_state *s, int64_t n, int64_t *order, double *lower,
                     double *upper, int64_t *separated_pairs);

/* dynamic.update_batch (dynamic.py:126-211): arcs as (src,dst) int64 pairs,
 * already validated by the caller against the host graph. */
/* every entry of the last update's UpdateStats.level_sizes (dynamic.py:35),
 * up to cap; *count receives the full length */
int kb_update_level_sizes(kb_state *state, int64_t *out, int64_t cap, int64_t *count);
int kb_update_batch(kb_state *s, const int64_t *ins, int64_t n_ins,
                    const int64_t *dels, int64_t n_dels, double theta,
                    double new_gamma, kb_update_stats *stats);

#ifdef __cplusplus
}
#endif
#endif /* KATZB200_H */
