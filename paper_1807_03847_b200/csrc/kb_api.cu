// The C-ABI (include/katzb200.h): handle management and the run loop.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "kb_internal.cuh"

#include <map>
#include <unordered_map>

struct kb_graph {
    kb::Graph g;
};
struct kb_state {
    kb::State s;
};
struct kb_text {
    kb::TextScan t;
};
struct kb_ranking {
    int device = 0;
    int64_t n = 0;
    kb::DBuf<int64_t> order;
    kb::DBuf<double> lower, upper;
};

namespace kb {

static thread_local std::string t_err;
static std::atomic<int64_t> g_launches{0};
static std::mutex g_tune_mu;
static std::vector<std::pair<std::string, int64_t>> g_tune;
int64_t tune_get(const char *name, int64_t dflt) {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    for (auto &kv : g_tune)
        if (kv.first == name) return kv.second;
    return dflt;
}
void note_launch(int64_t k) { g_launches += k; }
int64_t launch_count() { return g_launches.load(); }
void set_error(const std::string &msg) { t_err = msg; }

#ifdef KB_CHECKED
namespace {
struct DcheckReader {
    void (*read)(unsigned long long *, int *);
    const char *file;
};
std::vector<DcheckReader> &dcheck_readers() {
    static std::vector<DcheckReader> v;
    return v;
}
}  // namespace
int dcheck_register(void (*read)(unsigned long long *, int *), const char *file) {
    dcheck_readers().push_back({read, file});
    return 1;
}
void dcheck_poll() {
    if (cudaDeviceSynchronize() != cudaSuccess) return;   // the call's own error wins
    for (auto &r : dcheck_readers()) {
        unsigned long long f = 0;
        int line = 0;
        r.read(&f, &line);
        if (f) {
            char buf[256];
            snprintf(buf, sizeof buf, "KB_DCHECK failed %llu time(s), last at %s:%d",
                     f, r.file, line);
            throw Error{KB_ECUDA, buf};
        }
    }
}
#else
void dcheck_poll() {}
#endif

cudaStream_t device_stream() {
    static std::mutex mu;
    static cudaStream_t streams[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!streams[dev]) {
        cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    return streams[dev];
}

// A second non-blocking stream per device for bulk host<->device copies that
// overlap the device stream's kernels (pipelined ingest, result download).
cudaStream_t copy_stream() {
    static std::mutex mu;
    static cudaStream_t streams[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!streams[dev]) KB_CUDA(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
    return streams[dev];
}

namespace {
struct BigCache {
    std::multimap<size_t, void *> idle;      // size -> block
    std::unordered_map<void *, size_t> live;
    size_t held = 0;                          // bytes in live + idle blocks
};
std::mutex g_big_mu;
BigCache g_big[64];

int cur_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

void flush_idle(BigCache &c) {
    if (c.idle.empty()) return;
    cudaStreamSynchronize(device_stream());
    for (auto &kv : c.idle) {
        cudaFree(kv.second);
        c.held -= kv.first;
    }
    c.idle.clear();
}
}  // namespace

void *dev_alloc(size_t bytes) {
    cudaStream_t st = device_stream();
    void *p = nullptr;
    if (bytes < BIG_ALLOC) {
        KB_CUDA(cudaMallocAsync(&p, bytes, st));
        return p;
    }
    std::lock_guard<std::mutex> lk(g_big_mu);
    BigCache &c = g_big[cur_device()];
    // best fit among idle blocks, wasting at most a quarter of the block
    auto it = c.idle.lower_bound(bytes);
    if (it != c.idle.end() && it->first - bytes <= it->first / 4) {
        p = it->second;
        c.live[p] = it->first;
        c.idle.erase(it);
        return p;
    }
    const size_t sz = (bytes + ((size_t)2 << 20) - 1) & ~(((size_t)2 << 20) - 1);
    cudaError_t e = cudaMalloc(&p, sz);
    if (e == cudaErrorMemoryAllocation) {
        (void)cudaGetLastError();
        flush_idle(c);                        // give cached blocks back and retry
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, cur_device()) == cudaSuccess)
            cudaMemPoolTrimTo(pool, 0);
        e = cudaMalloc(&p, sz);
    }
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        throw Error{e == cudaErrorMemoryAllocation ? KB_ENOMEM : KB_ECUDA,
                    std::string("device allocation of ") + std::to_string(sz) + " bytes: " +
                        cudaGetErrorString(e)};
    }
    c.live[p] = sz;
    c.held += sz;
    return p;
}

void dev_free(void *p, size_t bytes) {
    if (!p) return;
    if (bytes < BIG_ALLOC) {
        cudaFreeAsync(p, device_stream());
        return;
    }
    std::lock_guard<std::mutex> lk(g_big_mu);
    BigCache &c = g_big[cur_device()];
    auto it = c.live.find(p);
    if (it == c.live.end()) {
        cudaFreeAsync(p, device_stream());
        return;
    }
    c.idle.emplace(it->second, p);            // reused in stream order
    c.live.erase(it);
}

void dev_mem_info(int64_t info[6]) {
    cudaMemPool_t pool;
    KB_CUDA(cudaDeviceGetDefaultMemPool(&pool, cur_device()));
    const cudaMemPoolAttr at[4] = {cudaMemPoolAttrReservedMemCurrent,
                                   cudaMemPoolAttrReservedMemHigh,
                                   cudaMemPoolAttrUsedMemCurrent, cudaMemPoolAttrUsedMemHigh};
    for (int i = 0; i < 4; i++) {
        uint64_t v = 0;
        KB_CUDA(cudaMemPoolGetAttribute(pool, at[i], &v));
        info[i] = (int64_t)v;
    }
    std::lock_guard<std::mutex> lk(g_big_mu);
    BigCache &c = g_big[cur_device()];
    size_t live = 0;
    for (auto &kv : c.live) live += kv.second;
    info[4] = (int64_t)c.held;
    info[5] = (int64_t)live;
}

// page-locked mirror for small device->host reads; one per host thread, used
// only inside a single synchronous API call
unsigned long long *pinned_flags() {
    static thread_local unsigned long long *p = nullptr;
    if (!p) KB_CUDA(cudaMallocHost(&p, 64 * sizeof(unsigned long long)));
    return p;
}

namespace {

__global__ void k_init_state(double *ones, double *katz, double *lower, double *upper,
                             int64_t n, double ag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    if (ones) ones[i] = i < n ? 1.0 : 0.0;
    if (katz) {
        katz[i] = 0.0;
        lower[i] = 0.0;
        upper[i] = ag;
    }
}

__global__ void k_active_to_orig(const int32_t *act, int dense, int64_t m, const int32_t *perm,
                                 int64_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) out[i] = perm[dense ? (int32_t)i : act[i]];
}

__global__ void k_compose(const int32_t *ul, const int32_t *perm, int64_t n, int32_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = ul[perm[i]];
}

__global__ void k_map_ids(const int64_t *ids, int64_t m, const int32_t *iperm, int64_t n,
                          int32_t *out, unsigned long long *bad) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int64_t v = ids[i];
    if (v < 0 || v >= n) { bad[8] = 1; return; }
    out[i] = iperm[v];
}

__global__ void k_range32(int64_t lo, int64_t m, int32_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) out[i] = (int32_t)(lo + i);
}

// checked build self-test: one failing KB_DCHECK (tests/test_checked_build.py)
__global__ void k_dcheck_selftest(int v) { KB_DCHECK(v == 0); (void)v; }

__global__ void k_sep_one(const double *lower, const double *upper, const int32_t *iperm,
                          int64_t w, int64_t v, double eps, unsigned long long *out) {
    out[0] = lower[iperm[w]] > __dsub_rn(upper[iperm[v]], eps);
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)std::max<int64_t>(1, (n + t - 1) / t); }

template <typename F>
int guarded(F &&f) {
    // a non-sticky error left by an earlier failed runtime call (for example
    // a destructor running during interpreter teardown) must not surface in
    // this call's cudaPeekAtLastError checks (CUB)
    {
        const cudaError_t stale = cudaGetLastError();
        if (stale != cudaSuccess && getenv("KB_TRACE"))
            fprintf(stderr, "[kb] stale CUDA error before API call: %s (last message: %s)\n",
                    cudaGetErrorString(stale), t_err.c_str());
    }
    try {
        f();
        dcheck_poll();
        return KB_OK;
    } catch (const Error &e) {
        set_error(e.msg);
        (void)cudaGetLastError();
        return e.code;
    } catch (const std::bad_alloc &) {
        set_error("host allocation failed");
        return KB_ENOMEM;
    } catch (const std::exception &e) {
        set_error(e.what());
        return KB_ECUDA;
    }
}

void use_device(int dev) { KB_CUDA(cudaSetDevice(dev)); }

}  // namespace

void ensure_init(State &s) {
    // katz, lower, upper (and levels[0] with them) when nothing wrote them yet
    if (!s.init_pending) return;
    const int64_t n = s.g->n;
    k_init_state<<<nblk(n + 1, 256), 256, 0, s.g->stream>>>(
        s.ones_pending && s.level_base == 0 ? s.levels[0].p : nullptr, s.katz.p, s.lower.p,
        s.upper.p, n, s.alpha * s.gamma);
    note_launch();
    KB_CUDA(cudaGetLastError());
    s.init_pending = s.ones_pending = false;
}

void ensure_ones(State &s) {
    // levels[0] (all ones), for the readers of that level only
    ensure_init(s);
    if (!s.ones_pending) return;
    if (s.level_base == 0 && !s.levels.empty()) {
        const int64_t n = s.g->n;
        k_init_state<<<nblk(n + 1, 256), 256, 0, s.g->stream>>>(s.levels[0].p, nullptr, nullptr,
                                                                nullptr, n, 0.0);
        note_launch();
        KB_CUDA(cudaGetLastError());
    }
    s.ones_pending = false;
}

}  // namespace kb

using namespace kb;

extern "C" {

static kb_graph *new_graph(int device, int64_t split_threshold, int64_t hot_size);

const char *kb_last_error(void) { return t_err.c_str(); }

int kb_version(void) { return 10000; }

int kb_device_count(int *count) {
    return guarded([&] { KB_CUDA(cudaGetDeviceCount(count)); });
}

int kb_timer(int device, int op, double *elapsed_ms) {
    return guarded([&] {
        static cudaEvent_t ev[64][2];
        static bool made[64];
        KB_REQUIRE(device >= 0 && device < 64, KB_EPARAM, "bad device");
        use_device(device);
        if (!made[device]) {
            KB_CUDA(cudaEventCreate(&ev[device][0]));
            KB_CUDA(cudaEventCreate(&ev[device][1]));
            made[device] = true;
        }
        cudaStream_t st = device_stream();
        if (op == 0) {
            KB_CUDA(cudaEventRecord(ev[device][0], st));
        } else {
            KB_CUDA(cudaEventRecord(ev[device][1], st));
            KB_CUDA(cudaEventSynchronize(ev[device][1]));
            float ms = 0;
            KB_CUDA(cudaEventElapsedTime(&ms, ev[device][0], ev[device][1]));
            if (elapsed_ms) *elapsed_ms = ms;
        }
    });
}

int kb_tune(const char *name, int64_t value) {
    return guarded([&] {
        KB_REQUIRE(name, KB_EPARAM, "NULL name");
        std::lock_guard<std::mutex> lk(g_tune_mu);
        for (auto &kv : g_tune)
            if (kv.first == name) { kv.second = value; return; }
        g_tune.emplace_back(name, value);
    });
}

int kb_launch_count(int64_t *count) {
    return guarded([&] {
        KB_REQUIRE(count, KB_EPARAM, "NULL argument");
        *count = launch_count();
    });
}

int kb_host_register(void *ptr, int64_t bytes) {
    return guarded([&] {
        if (!ptr || bytes <= 0) return;
        KB_CUDA(cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault));
    });
}

int kb_host_unregister(void *ptr) {
    return guarded([&] {
        if (ptr) KB_CUDA(cudaHostUnregister(ptr));
    });
}

int kb_graph_create(int device, int64_t n, int64_t nnz, const int64_t *indptr,
                    const int32_t *indices, int64_t split_threshold, int64_t hot_size,
                    kb_graph **out) {
    return guarded([&] {
        KB_REQUIRE(out, KB_EPARAM, "out is NULL");
        KB_REQUIRE(n >= 0 && n < ((int64_t)1 << 31), KB_ENODERANGE,
                   "node ids must fit the 32-bit index type");
        KB_REQUIRE(nnz >= 0 && nnz < ((int64_t)1 << 31) * 32, KB_EPARAM, "bad nnz");
        KB_REQUIRE(indptr && (nnz == 0 || indices), KB_EPARAM, "NULL CSR arrays");
        KB_REQUIRE(indptr[0] == 0 && indptr[n] == nnz, KB_EPARAM,
                   "indptr must start at 0 and end at nnz");
        kb_graph *h = new_graph(device, split_threshold, hot_size);
        Graph &g = h->g;
        g.n = n;
        g.nnz = nnz;
        try {
            build_graph(g, indptr, indices);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int kb_graph_create_ex(int device, int64_t n, int64_t nnz, const int64_t *indptr,
                       const int32_t *indices, int64_t split_threshold, int64_t hot_size,
                       int flags, const int32_t *labels, int64_t own_lo, int64_t own_hi,
                       kb_graph **out) {
    return guarded([&] {
        KB_REQUIRE(out, KB_EPARAM, "out is NULL");
        KB_REQUIRE(n >= 0 && n < ((int64_t)1 << 31), KB_ENODERANGE,
                   "node ids must fit the 32-bit index type");
        KB_REQUIRE(indptr && (nnz == 0 || indices), KB_EPARAM, "NULL CSR arrays");
        KB_REQUIRE(indptr[0] == 0 && indptr[n] == nnz, KB_EPARAM,
                   "indptr must start at 0 and end at nnz");
        kb_graph *h = new_graph(device, split_threshold, hot_size);
        Graph &g = h->g;
        g.n = n;
        g.nnz = nnz;
        g.relabel = !(flags & KB_GRAPH_NO_RELABEL);
        KB_REQUIRE(own_lo >= 0 && (own_hi < 0 || (own_hi >= own_lo && own_hi <= n)), KB_EPARAM,
                   "bad owned row range");
        g.own_lo = own_lo;
        g.own_hi = own_hi < 0 ? n : own_hi;
        {
            // a shard of an exchange layout with 2^k-id blocks: K1 keeps the
            // head of every block (the top hubs of each rank) in shared memory
            const int64_t B = g.own_hi - g.own_lo;
            if (!g.relabel && B > 0 && (B & (B - 1)) == 0 && n % B == 0 && own_lo % B == 0 &&
                n / B > 1) {
                int sh = 0;
                while (((int64_t)1 << sh) < B) sh++;
                g.hot_shift = sh;
                g.hot_per = std::max<int64_t>(1, g.hot / (n / B));
            }
        }
        try {
            build_graph(g, indptr, indices);
            if (labels) {
                DBuf<int32_t> ul;
                ul.alloc(std::max<int64_t>(1, n));
                KB_CUDA(cudaMemcpyAsync(ul.p, labels, n * sizeof(int32_t),
                                        cudaMemcpyHostToDevice, g.stream));
                g.label.alloc(std::max<int64_t>(1, n));
                if (n) k_compose<<<nblk(n, 256), 256, 0, g.stream>>>(ul.p, g.perm.p, n, g.label.p);
                note_launch();
                KB_CUDA(cudaStreamSynchronize(g.stream));
            }
            if (flags & KB_GRAPH_SYMMETRIC) g.symmetric = 1;
            if (!g.relabel) g.mutated = true;  // no degree-sorted tail shortcuts
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int kb_graph_create_shard(kb_graph *full, int64_t nranks, int64_t rank, int64_t split_threshold,
                          int64_t hot_size, kb_graph **out, int64_t *n_per, int64_t *owned) {
    return guarded([&] {
        KB_REQUIRE(full && out && n_per && owned, KB_EPARAM, "NULL argument");
        use_device(full->g.device);
        kb_graph *h = new_graph(full->g.device, split_threshold, hot_size);
        try {
            build_shard(full->g, nranks, rank, h->g, n_per, owned);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int kb_graph_create_shard_host(int device, int64_t n, int64_t nnz, const int64_t *indptr,
                               const int32_t *indices, int64_t nranks, int64_t rank,
                               int64_t split_threshold, int64_t hot_size, kb_graph **out,
                               int64_t *n_per, int64_t *owned) {
    return guarded([&] {
        KB_REQUIRE(out && n_per && owned, KB_EPARAM, "NULL argument");
        KB_REQUIRE(n >= 1 && n < ((int64_t)1 << 31), KB_ENODERANGE,
                   "node ids must fit the 32-bit index type");
        kb_graph *h = new_graph(device, split_threshold, hot_size);
        try {
            build_shard_host(h->g, n, nnz, indptr, indices, nranks, rank, n_per, owned);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int kb_shard_symmetry_keys(kb_graph *h, int64_t nranks, int64_t *keys, int64_t *counts) {
    return guarded([&] {
        KB_REQUIRE(h && counts && (keys || h->g.nnz == 0), KB_EPARAM, "NULL argument");
        use_device(h->g.device);
        shard_symmetry_keys(h->g, nranks, keys, counts);
    });
}

int kb_shard_symmetry_verify(kb_graph *h, const int64_t *recv, int64_t nrecv, int *ok) {
    return guarded([&] {
        KB_REQUIRE(h && ok && (recv || nrecv == 0), KB_EPARAM, "NULL argument");
        use_device(h->g.device);
        *ok = shard_symmetry_verify(h->g, recv, nrecv);
    });
}

int kb_graph_find_labels(kb_graph *h, const int64_t *labels, int64_t m, int64_t *ids) {
    return guarded([&] {
        KB_REQUIRE(h && (m == 0 || (labels && ids)), KB_EPARAM, "NULL argument");
        use_device(h->g.device);
        find_labels(h->g, labels, m, ids);
    });
}

int kb_state_set_active(kb_state *h, const int64_t *ids, int64_t m) {
    return guarded([&] {
        KB_REQUIRE(h && (m == 0 || ids), KB_EPARAM, "NULL argument");
        State &s = h->s;
        KB_REQUIRE(m >= 0 && m <= s.g->n, KB_EPARAM, "bad active size");
        use_device(s.g->device);
        ensure_init(h->s);
        cudaStream_t st = s.g->stream;
        DBuf<int64_t> d;
        d.alloc(std::max<int64_t>(1, m));
        KB_CUDA(cudaMemsetAsync(s.scratch_u64.p + 8, 0, 8, st));
        if (m) {
            KB_CUDA(cudaMemcpyAsync(d.p, ids, m * 8, cudaMemcpyHostToDevice, st));
            k_map_ids<<<nblk(m, 256), 256, 0, st>>>(d.p, m, s.g->iperm.p, s.g->n, s.act[s.cur].p,
                                                    s.scratch_u64.p);
            note_launch();
        }
        unsigned long long bad = 0;
        KB_CUDA(cudaMemcpyAsync(&bad, s.scratch_u64.p + 8, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        KB_REQUIRE(!bad, KB_EPARAM, "active id out of range");
        s.act_dense = false;
        s.m_host = m;
    });
}

int kb_state_set_active_range(kb_state *h, int64_t lo, int64_t hi) {
    return guarded([&] {
        KB_REQUIRE(h, KB_EPARAM, "NULL argument");
        State &s = h->s;
        KB_REQUIRE(0 <= lo && lo <= hi && hi <= s.g->n, KB_EPARAM, "bad active range");
        KB_REQUIRE(!s.g->relabel, KB_EPARAM, "active ranges need a KB_GRAPH_NO_RELABEL graph");
        use_device(s.g->device);
        ensure_init(h->s);
        const int64_t m = hi - lo;
        if (m) {
            k_range32<<<nblk(m, 256), 256, 0, s.g->stream>>>(lo, m, s.act[s.cur].p);
            note_launch();
        }
        s.act_dense = false;
        s.m_host = m;
    });
}

int kb_state_vector_ptr(kb_state *h, int which, int64_t level, void **ptr) {
    return guarded([&] {
        KB_REQUIRE(h && ptr, KB_EPARAM, "NULL argument");
        State &s = h->s;
        use_device(s.g->device);
        ensure_ones(s);
        switch (which) {
            case KB_VEC_LEVEL: {
                const int64_t idx = level - s.level_base;
                KB_REQUIRE(idx >= 0 && idx < (int64_t)s.levels.size(), KB_EPARAM,
                           "level not retained");
                *ptr = s.levels[idx].p;
                break;
            }
            case KB_VEC_KATZ: *ptr = s.katz.p; break;
            case KB_VEC_LOWER: *ptr = s.lower.p; break;
            case KB_VEC_UPPER: *ptr = s.upper.p; break;
            default: throw Error{KB_EPARAM, "unknown vector"};
        }
    });
}

int kb_sync(int device) {
    return guarded([&] {
        use_device(device);
        if (tune_get("dcheck.selftest", 0)) {
            k_dcheck_selftest<<<1, 1, 0, device_stream()>>>(1);
            note_launch();
        }
        KB_CUDA(cudaStreamSynchronize(device_stream()));
    });
}

int kb_check_local_topk(kb_state *h, int64_t k, uint64_t *keys, int64_t *labels,
                        double *uppers, int64_t *count) {
    return guarded([&] {
        KB_REQUIRE(h && keys && labels && uppers && count && k >= 1, KB_EPARAM, "bad argument");
        State &s = h->s;
        KB_REQUIRE(s.r >= 1, KB_ESTATE, "check_converged needs at least one iteration");
        use_device(s.g->device);
        ensure_init(h->s);
        local_topk(s, s.g->stream, k, keys, labels, uppers, count);
    });
}

int kb_check_apply_cut(kb_state *h, uint64_t kstar, int64_t istar, int64_t *active) {
    return guarded([&] {
        KB_REQUIRE(h && active, KB_EPARAM, "NULL argument");
        State &s = h->s;
        use_device(s.g->device);
        ensure_init(h->s);
        apply_cut(s, s.g->stream, kstar, istar);
        *active = s.m_host;
    });
}

int kb_select_global(int device, const uint64_t *keys, const int64_t *labels,
                     const double *uppers, int64_t ncand, int64_t k, double eps, uint64_t *kstar,
                     int64_t *istar, int *prefix_separated) {
    return guarded([&] {
        KB_REQUIRE(keys && labels && uppers && kstar && istar && prefix_separated, KB_EPARAM,
                   "NULL argument");
        KB_REQUIRE(ncand >= 1 && k >= 1, KB_EPARAM, "no candidates");
        use_device(device);
        select_global(device, keys, labels, uppers, ncand, k, eps, kstar, istar,
                      prefix_separated);
    });
}

int kb_rank_bounds(int device, int64_t n, const double *lower, const double *upper,
                   int64_t *order, int64_t *separated_pairs) {
    return guarded([&] {
        KB_REQUIRE(lower && upper && n >= 1, KB_EPARAM, "bad argument");
        use_device(device);
        rank_bounds(device, n, lower, upper, order, separated_pairs);
    });
}

int kb_foster(kb_graph *gh, double alpha, double tol, int64_t max_iter, double *values,
              int64_t *iterations, double *residual) {
    return guarded([&] {
        KB_REQUIRE(gh && values && iterations && residual, KB_EPARAM, "NULL argument");
        KB_REQUIRE(std::isfinite(alpha) && alpha > 0, KB_EPARAM, "alpha must be finite and > 0");
        KB_REQUIRE(tol > 0, KB_EPARAM, "tol must be > 0");
        KB_REQUIRE(max_iter >= 1, KB_EPARAM, "max_iter must be >= 1");
        use_device(gh->g.device);
        const bool ok = foster(gh->g, alpha, tol, max_iter, values, iterations, residual);
        KB_REQUIRE(ok, KB_ECONVERGENCE, "foster did not reach tol within max_iter iterations");
    });
}

int kb_cg_katz(kb_graph *gh, double alpha, double residual_tol, int64_t max_iter,
               double *values, int64_t *iterations, double *residual) {
    return guarded([&] {
        KB_REQUIRE(gh && values && iterations && residual, KB_EPARAM, "NULL argument");
        KB_REQUIRE(std::isfinite(alpha) && alpha > 0, KB_EPARAM, "alpha must be finite and > 0");
        KB_REQUIRE(residual_tol > 0, KB_EPARAM, "residual_tol must be > 0");
        KB_REQUIRE(max_iter >= 0, KB_EPARAM, "max_iter must be >= 0");
        use_device(gh->g.device);
        const int st = cg_katz(gh->g, alpha, residual_tol, max_iter, values, iterations,
                               residual);
        KB_REQUIRE(st != 2, KB_ENUMERIC, "conjugate gradient broke down (non-positive curvature)");
        KB_REQUIRE(st == 0, KB_ECONVERGENCE, "cg residual still above residual_tol");
    });
}

int kb_ranking_inversions(int device, int64_t n, const int64_t *order_a,
                          const int64_t *order_b, int64_t *inversions) {
    return guarded([&] {
        KB_REQUIRE(inversions && n >= 0 && (n == 0 || (order_a && order_b)), KB_EPARAM,
                   "NULL argument");
        use_device(device);
        *inversions = count_inversions(order_a, order_b, n);
    });
}

int kb_pool_info(int device, int64_t *info) {
    return guarded([&] {
        KB_REQUIRE(info, KB_EPARAM, "NULL argument");
        use_device(device);
        (void)device_stream();
        dev_mem_info(info);
    });
}

int kb_pool_reserve(int device, int64_t bytes) {
    return guarded([&] {
        KB_REQUIRE(bytes >= 0, KB_EPARAM, "bad size");
        use_device(device);
        cudaStream_t st = device_stream();
        if (!bytes) return;
        void *p = nullptr;
        KB_CUDA(cudaMallocAsync(&p, (size_t)bytes, st));
        KB_CUDA(cudaFreeAsync(p, st));
        KB_CUDA(cudaStreamSynchronize(st));
    });
}

int kb_ranking_snapshot(kb_state *h, kb_ranking **out, int64_t *separated_pairs) {
    return guarded([&] {
        KB_REQUIRE(h && out, KB_EPARAM, "NULL argument");
        State &s = h->s;
        use_device(s.g->device);
        ensure_init(h->s);
        auto *r = new kb_ranking();
        try {
            r->device = s.g->device;
            r->n = s.g->n;
            result_device(s, s.g->stream, &r->order, &r->lower, &r->upper, separated_pairs);
        } catch (...) {
            delete r;
            throw;
        }
        *out = r;
    });
}

int kb_ranking_read(kb_ranking *r, int which, int64_t offset, int64_t count, void *host) {
    return guarded([&] {
        KB_REQUIRE(r && (host || !count), KB_EPARAM, "NULL argument");
        KB_REQUIRE(which >= 0 && which <= 2, KB_EPARAM, "which: 0 order, 1 lower, 2 upper");
        KB_REQUIRE(offset >= 0 && count >= 0 && offset + count <= r->n, KB_EPARAM,
                   "range outside the result");
        use_device(r->device);
        if (!count) return;
        const void *src = which == 0 ? (const void *)(r->order.p + offset)
                        : which == 1 ? (const void *)(r->lower.p + offset)
                                     : (const void *)(r->upper.p + offset);
        cudaStream_t st = device_stream();
        download_d2h(host, src, count * 8, st);
        KB_CUDA(cudaStreamSynchronize(st));
    });
}

int kb_ranking_destroy(kb_ranking *r) {
    return guarded([&] {
        if (!r) return;
        use_device(r->device);
        delete r;
    });
}

int kb_stream(int device, void **stream) {
    return guarded([&] {
        KB_REQUIRE(stream, KB_EPARAM, "NULL argument");
        use_device(device);
        *stream = (void *)device_stream();
    });
}

int kb_shard_propose(kb_state *h, int64_t k, void *block) {
    return guarded([&] {
        KB_REQUIRE(h && block, KB_EPARAM, "NULL argument");
        use_device(h->s.g->device);
        ensure_init(h->s);
        shard_propose(h->s, h->s.g->stream, k, (unsigned long long *)block);
        KB_CUDA(cudaGetLastError());
    });
}

int kb_shard_cut(kb_state *h, const void *blocks, int64_t nblocks, int64_t k, void *word) {
    return guarded([&] {
        KB_REQUIRE(h && blocks && word, KB_EPARAM, "NULL argument");
        use_device(h->s.g->device);
        ensure_init(h->s);
        shard_cut(h->s, h->s.g->stream, (const unsigned long long *)blocks, nblocks, k,
                  (long long *)word);
        KB_CUDA(cudaGetLastError());
    });
}

int kb_shard_commit(kb_state *h, int64_t active) {
    return guarded([&] {
        KB_REQUIRE(h, KB_EPARAM, "NULL state");
        shard_commit(h->s, active);
    });
}

namespace kb {
namespace {
// converged iff |active| over all ranks <= k and the prefix is separated
__global__ void k_shard_publish(const long long *word, int64_t k, unsigned long long *abort) {
    abort[0] = (word[0] <= k && word[2] != 0) ? 1ull : 0ull;
}
}  // namespace
}  // namespace kb

int kb_shard_iterate_spec(kb_state *h, const long long *word, int64_t k) {
    return guarded([&] {
        KB_REQUIRE(h && word && k >= 1, KB_EPARAM, "bad argument");
        State &s = h->s;
        use_device(s.g->device);
        ensure_init(h->s);
        KB_REQUIRE(s.g->version == s.graph_version, KB_ESTATE,
                   "graph changed since init; static iteration would be unsound");
        KB_REQUIRE(s.r < s.max_iter, KB_ECONVERGENCE, "iteration cap reached");
        cudaStream_t st = s.g->stream;
        if (!s.abort_flag.p) s.abort_flag.alloc(1);
        k_shard_publish<<<1, 1, 0, st>>>(word, k, s.abort_flag.p);
        note_launch();
        KB_CUDA(cudaGetLastError());
        s.spec_abort = true;
        try {
            launch_iterate(s, st);
        } catch (...) {
            s.spec_abort = false;
            throw;
        }
        s.spec_abort = false;
    });
}

int kb_state_rollback(kb_state *h) {
    return guarded([&] {
        KB_REQUIRE(h, KB_EPARAM, "NULL state");
        State &s = h->s;
        use_device(s.g->device);
        ensure_init(s);
        KB_REQUIRE(s.r >= 1 && s.levels.size() >= 2, KB_ESTATE, "no level to roll back");
        s.levels.pop_back();
        s.r -= 1;
        if (s.k1_used >= 2) s.k1_used -= 2;
    });
}

int kb_rank_gathered(kb_state *h, int64_t n, int64_t *order, double *lower, double *upper,
                     int64_t *separated_pairs) {
    return guarded([&] {
        KB_REQUIRE(h && n >= 1, KB_EPARAM, "bad argument");
        use_device(h->s.g->device);
        ensure_init(h->s);
        rank_gathered(h->s, n, order, lower, upper, separated_pairs);
    });
}

static kb_graph *new_graph(int device, int64_t split_threshold, int64_t hot_size) {
    use_device(device);
    auto *h = new kb_graph();
    Graph &g = h->g;
    g.device = device;
    KB_CUDA(cudaDeviceGetAttribute(&g.sm_count, cudaDevAttrMultiProcessorCount, device));
    g.stream = device_stream();
    g.split = split_threshold > 0 ? split_threshold : 2048;
    g.split = std::max<int64_t>(4, g.split & ~(int64_t)3);
    g.hot = hot_size >= 0 ? hot_size : 12288;
    return h;
}

int kb_graph_create_rmat(int device, int scale, int64_t edge_factor, const uint64_t *pcg_state,
                         double a, double ab, double abc, int64_t split_threshold,
                         int64_t hot_size, kb_graph **out) {
    return guarded([&] {
        KB_REQUIRE(out && pcg_state, KB_EPARAM, "NULL argument");
        KB_REQUIRE(edge_factor >= 1, KB_EPARAM, "edge_factor must be >= 1");
        kb_graph *h = new_graph(device, split_threshold, hot_size);
        try {
            Graph &g = h->g;
            g.n = (int64_t)1 << scale;
            rmat_device_csr(scale, edge_factor, pcg_state, a, ab, abc, g.indptr, g.indices,
                            g.nnz);
            g.symmetric = 1;
            build_graph_device(g);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int kb_text_scan(int device, const void *bytes, int64_t nbytes, int batches, kb_text **out,
                 int64_t *info) {
    return guarded([&] {
        KB_REQUIRE(out && info && nbytes >= 0 && (nbytes == 0 || bytes), KB_EPARAM,
                   "NULL argument");
        use_device(device);
        auto *t = new kb_text();
        try {
            t->t.device = device;
            text_scan(t->t, (const char *)bytes, nbytes, batches ? 1 : 0);
        } catch (...) {
            delete t;
            throw;
        }
        const TextScan &s = t->t;
        info[0] = s.n_lines;
        info[1] = s.n_arcs;
        info[2] = s.n_cand;
        info[3] = s.first_arc_line;
        info[4] = s.max_id;
        *out = t;
    });
}

int kb_text_candidates(kb_text *t, int64_t *lines) {
    return guarded([&] {
        KB_REQUIRE(t && (lines || !t->t.n_cand), KB_EPARAM, "NULL argument");
        use_device(t->t.device);
        text_candidates(t->t, lines);
    });
}

int kb_text_lines(kb_text *t, uint8_t *kind, int32_t *u, int32_t *v) {
    return guarded([&] {
        KB_REQUIRE(t, KB_EPARAM, "NULL argument");
        use_device(t->t.device);
        text_lines(t->t, kind, u, v);
    });
}

int kb_text_destroy(kb_text *t) {
    return guarded([&] {
        if (!t) return;
        use_device(t->t.device);
        delete t;
    });
}

int kb_graph_create_text(kb_text *t, int64_t n, int undirected, const int64_t *extra_arcs,
                         int64_t n_extra, int64_t split_threshold, int64_t hot_size,
                         kb_graph **out) {
    return guarded([&] {
        KB_REQUIRE(t && out && n_extra >= 0 && (n_extra == 0 || extra_arcs), KB_EPARAM,
                   "NULL argument");
        KB_REQUIRE(n >= 1, KB_EPARAM, "graph must have at least one node");
        kb_graph *h = new_graph(t->t.device, split_threshold, hot_size);
        try {
            Graph &g = h->g;
            g.n = n;
            text_csr(t->t, n, undirected, extra_arcs, n_extra, g.indptr, g.indices, g.nnz);
            g.symmetric = undirected ? 1 : -1;
            build_graph_device(g);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int kb_graph_create_grid(int device, int64_t n, int64_t split_threshold, int64_t hot_size,
                         kb_graph **out) {
    return guarded([&] {
        KB_REQUIRE(out, KB_EPARAM, "NULL argument");
        KB_REQUIRE(n >= 1 && n < ((int64_t)1 << 31), KB_EPARAM, "grid needs 1 <= n < 2^31");
        kb_graph *h = new_graph(device, split_threshold, hot_size);
        try {
            Graph &g = h->g;
            g.n = n;
            grid_device_csr(n, g.indptr, g.indices, g.nnz);
            g.symmetric = 1;
            build_graph_device(g);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int kb_graph_get_csr(kb_graph *h, int64_t *indptr, int32_t *indices) {
    return guarded([&] {
        KB_REQUIRE(h, KB_EPARAM, "NULL graph");
        Graph &g = h->g;
        use_device(g.device);
        DBuf<int64_t> cip;
        DBuf<int32_t> cix;
        const int64_t *ip = g.indptr.p;
        const int32_t *ix = g.indices.p;
        if (g.slack) {  // compact the CSR-with-slack first
            compact_csr(g, cip, cix);
            ip = cip.p;
            ix = cix.p;
        }
        if (indptr) download_d2h(indptr, ip, (g.n + 1) * sizeof(int64_t), g.stream);
        if (indices && g.nnz) download_d2h(indices, ix, g.nnz * sizeof(int32_t), g.stream);
        KB_CUDA(cudaStreamSynchronize(g.stream));
    });
}

int kb_graph_has_arcs(kb_graph *h, const int64_t *arcs, int64_t m, uint8_t *present) {
    return guarded([&] {
        KB_REQUIRE(h && (m == 0 || (arcs && present)), KB_EPARAM, "NULL argument");
        Graph &g = h->g;
        for (int64_t i = 0; i < 2 * m; i++)
            KB_REQUIRE(arcs[i] >= 0 && arcs[i] < g.n, KB_ENODERANGE, "node id outside graph");
        use_device(g.device);
        graph_has_arcs(g, arcs, m, present);
    });
}

int kb_graph_max_degree_after(kb_graph *h, const int64_t *ins, int64_t n_ins,
                              const int64_t *dels, int64_t n_dels, int64_t *out) {
    return guarded([&] {
        KB_REQUIRE(h && out, KB_EPARAM, "NULL argument");
        use_device(h->g.device);
        *out = graph_max_degree_after(h->g, ins, n_ins, dels, n_dels);
    });
}

int kb_graph_out_degrees(kb_graph *h, int64_t *out) {
    return guarded([&] {
        KB_REQUIRE(h && out, KB_EPARAM, "NULL argument");
        use_device(h->g.device);
        graph_out_degrees(h->g, out);
    });
}

int kb_graph_apply_batch(kb_graph *h, const int64_t *ins, int64_t n_ins, const int64_t *dels,
                         int64_t n_dels) {
    return guarded([&] {
        KB_REQUIRE(h, KB_EPARAM, "NULL graph");
        Graph &g = h->g;
        for (int64_t i = 0; i < 2 * n_ins; i++)
            KB_REQUIRE(ins[i] >= 0 && ins[i] < g.n, KB_ENODERANGE, "node id outside graph");
        for (int64_t i = 0; i < 2 * n_dels; i++)
            KB_REQUIRE(dels[i] >= 0 && dels[i] < g.n, KB_ENODERANGE, "node id outside graph");
        use_device(g.device);
        apply_batch_to_graph(g, ins, n_ins, dels, n_dels);
        g.symmetric = -1;
    });
}

// ---- fused omega exchange for shards (replaces the per-iteration NCCL
// all-gather of SURVEY.md 8(e) with K1-epilogue stores over NVLink)
int kb_graph_exchange_alloc(kb_graph *h) {
    return guarded([&] {
        KB_REQUIRE(h, KB_EPARAM, "NULL graph");
        Graph &g = h->g;
        use_device(g.device);
        if (g.exch[0]) return;
        g.exch_n = (size_t)g.n + 1;
        for (int p = 0; p < 2; p++) {
            KB_CUDA(cudaMalloc(&g.exch[p], g.exch_n * sizeof(double)));
            KB_CUDA(cudaMemsetAsync(g.exch[p], 0, g.exch_n * sizeof(double), g.stream));
        }
        KB_CUDA(cudaStreamSynchronize(g.stream));
    });
}

int kb_graph_exchange_ptr(kb_graph *h, int parity, void **ptr) {
    return guarded([&] {
        KB_REQUIRE(h && ptr && (parity == 0 || parity == 1), KB_EPARAM, "bad argument");
        KB_REQUIRE(h->g.exch[parity], KB_ESTATE, "exchange buffers not allocated");
        *ptr = h->g.exch[parity];
    });
}

int kb_graph_exchange_handle(kb_graph *h, int parity, void *handle) {
    return guarded([&] {
        KB_REQUIRE(h && handle && (parity == 0 || parity == 1), KB_EPARAM, "bad argument");
        KB_REQUIRE(h->g.exch[parity], KB_ESTATE, "exchange buffers not allocated");
        use_device(h->g.device);
        cudaIpcMemHandle_t m;
        KB_CUDA(cudaIpcGetMemHandle(&m, h->g.exch[parity]));
        memcpy(handle, &m, sizeof(m));
    });
}

int kb_graph_exchange_add_peer(kb_graph *h, int parity, const void *handle, void *ptr) {
    return guarded([&] {
        KB_REQUIRE(h && (parity == 0 || parity == 1) && (handle || ptr), KB_EPARAM,
                   "bad argument");
        Graph &g = h->g;
        KB_REQUIRE((int)g.exch_peer[parity].size() < KB_MAX_PEERS, KB_EPARAM,
                   "too many exchange peers");
        use_device(g.device);
        double *p = (double *)ptr;
        if (handle) {
            cudaIpcMemHandle_t m;
            memcpy(&m, handle, sizeof(m));
            void *q = nullptr;
            KB_CUDA(cudaIpcOpenMemHandle(&q, m, cudaIpcMemLazyEnablePeerAccess));
            g.exch_opened.push_back(q);
            p = (double *)q;
        }
        g.exch_peer[parity].push_back(p);
    });
}

int kb_state_exchange(kb_state *h, int on) {
    return guarded([&] {
        KB_REQUIRE(h, KB_EPARAM, "NULL state");
        State &s = h->s;
        use_device(s.g->device);
        ensure_init(s);
        if (on) {
            KB_REQUIRE(s.g->exch[0], KB_ESTATE, "exchange buffers not allocated");
            KB_REQUIRE(!s.keep_all, KB_ESTATE, "the exchange keeps two levels: keep_levels=0");
            KB_REQUIRE(s.r == 0, KB_ESTATE, "enable the exchange before the first iteration");
        }
        s.exch_on = on != 0;
    });
}

int kb_graph_destroy(kb_graph *h) {
    return guarded([&] {
        if (!h) return;
        use_device(h->g.device);
        KB_CUDA(cudaStreamSynchronize(h->g.stream));
        delete h;
    });
}

int kb_graph_info_get(const kb_graph *h, kb_graph_info *info) {
    return guarded([&] {
        KB_REQUIRE(h && info, KB_EPARAM, "NULL argument");
        const Graph &g = h->g;
        info->n = g.n;
        info->nnz = g.nnz;
        info->max_out_degree = g.max_deg;
        info->nonisolated = g.nv;
        info->heavy_rows = g.nh;
        info->segments = g.sell.nseg;
        info->slices = g.sell.nslices;
        info->sell_elems = g.sell.elems;
        info->split_threshold = g.split;
        info->hot_size = std::min<int64_t>(g.hot, g.n);
        info->version = g.version;
        info->device_bytes = (int64_t)g.device_bytes();
        info->overflow_rows = g.n_ovf;
        info->overflow_long = g.n_ovf_long;
    });
}

int kb_graph_is_symmetric(kb_graph *h, int *symmetric) {
    return guarded([&] {
        KB_REQUIRE(h && symmetric, KB_EPARAM, "NULL argument");
        use_device(h->g.device);
        if (h->g.symmetric < 0) h->g.symmetric = graph_is_symmetric(h->g);
        *symmetric = h->g.symmetric;
    });
}

int kb_state_create(kb_graph *gh, double alpha, double gamma, int undirected, int kind,
                    double epsilon, int64_t k, int64_t u, int64_t v, int keep_all_levels,
                    int64_t max_iterations, kb_state **out) {
    return guarded([&] {
        KB_REQUIRE(gh && out, KB_EPARAM, "NULL argument");
        Graph &g = gh->g;
        KB_REQUIRE(g.n >= 1, KB_EPARAM, "graph must have at least one node");
        KB_REQUIRE(std::isfinite(alpha) && alpha > 0, KB_EPARAM, "alpha must be finite and > 0");
        KB_REQUIRE(std::isfinite(epsilon) && epsilon > 0, KB_EPARAM,
                   "epsilon must be finite and > 0");
        KB_REQUIRE(kind >= KB_RANKING && kind <= KB_PAIR, KB_EPARAM, "unknown criterion kind");
        KB_REQUIRE(kind != KB_TOPK || (k >= 1 && k <= g.n), KB_EPARAM, "bad k");
        KB_REQUIRE(kind != KB_PAIR || (u >= 0 && v >= 0 && u < g.n && v < g.n && u != v),
                   KB_EPARAM, "pair criterion names a node outside the graph");
        KB_REQUIRE(max_iterations >= 1, KB_EPARAM, "max_iterations must be >= 1");
        use_device(g.device);
        auto *h = new kb_state();
        State &s = h->s;
        s.g = &g;
        s.alpha = alpha;
        s.gamma = gamma;
        s.eps = epsilon;
        s.undirected = undirected;
        s.kind = kind;
        s.k = k;
        s.u = u;
        s.v = v;
        s.keep_all = keep_all_levels;
        s.max_iter = max_iterations;
        s.graph_version = g.version;
        const int64_t n = g.n;
        cudaStream_t st = g.stream;
        s.levels.emplace_back();
        s.levels.back().alloc(n + 1);
        s.katz.alloc(n + 1);
        s.lower.alloc(n + 1);
        s.upper.alloc(n + 1);
        // levels[0] = ones (engine.py:147), katz = lower = 0 (:148-149),
        // upper = alpha * gamma (:151): one pass over the four vectors -- or,
        // on a fresh degree-relabelled layout, none: the first K1 (the ones
        // step) writes katz, lower and upper itself, and every other entry
        // point writes what it would read first (ensure_init / ensure_ones)
        if (tune_get("init.lazy", 1) && g.implicit_rows && !g.mutated) {
            s.init_pending = s.ones_pending = true;
        } else {
            k_init_state<<<nblk(n + 1, 256), 256, 0, st>>>(s.levels.back().p, s.katz.p, s.lower.p,
                                                           s.upper.p, n, alpha * gamma);
            note_launch();
        }
        s.seg_sum.alloc(std::max<int64_t>(1, g.sell.nseg));
        s.act[0].alloc(n);
        s.act[1].alloc(n);
        s.act_dense = true;  // :152 arange(n), materialised on first check
        s.tail_zero_from = g.mutated ? n : g.nv;
        s.zero_tail_exact = !g.mutated;
        s.cand.alloc(n);
        s.stK.alloc(n);
        s.stU.alloc(n);
        s.stI.alloc(n);
        s.m_host = n;
        s.scratch_u64.alloc(1 << 16);
        s.scratch_i32.alloc(1 << 16);
        s.work_counter.alloc(2);
        s.abort_flag.alloc(1);
        KB_CUDA(cudaMemsetAsync(s.abort_flag.p, 0, sizeof(unsigned long long), st));
        s.tie_count.alloc(1);
        KB_CUDA(cudaMemsetAsync(s.tie_count.p, 0, sizeof(unsigned long long), st));
        KB_CUDA(cudaEventCreateWithFlags(&s.chk_ev, cudaEventDisableTiming));
        s.h_flags = pinned_flags();
        KB_CUDA(cudaEventCreate(&s.ev0));
        KB_CUDA(cudaEventCreate(&s.ev1));
        KB_CUDA(cudaGetLastError());
        // no sync: the fills are stream-ordered before any use of the state,
        // and run() can queue its first K1 behind them
        *out = h;
    });
}

int kb_state_destroy(kb_state *h) {
    return guarded([&] {
        if (!h) return;
        use_device(h->s.g->device);
        // a state must not outlive its graph (the Python layer holds the
        // DeviceGraph); sync before the buffers go back to the pool
        KB_CUDA(cudaStreamSynchronize(h->s.g->stream));
        if (h->s.ev0) cudaEventDestroy(h->s.ev0);
        if (h->s.ev1) cudaEventDestroy(h->s.ev1);
        if (h->s.chk_ev) cudaEventDestroy(h->s.chk_ev);
        if (h->s.chk_ev2) cudaEventDestroy(h->s.chk_ev2);
        for (cudaEvent_t e : h->s.k1_ev) cudaEventDestroy(e);
        delete h;
    });
}

int kb_state_info_get(const kb_state *h, kb_state_info *info) {
    return guarded([&] {
        KB_REQUIRE(h && info, KB_EPARAM, "NULL argument");
        const State &s = h->s;
        info->r = s.r;
        info->active = s.m_host;
        info->max_iterations = s.max_iter;
        info->levels_kept = (int64_t)s.levels.size();
        info->alpha = s.alpha;
        info->gamma = s.gamma;
        info->epsilon = s.eps;
        info->last_check_ms = s.last_check_ms;
        collect_k1_times(const_cast<State &>(s));
        info->spmv_ms = s.spmv_ms;
        info->spmv_launches = s.spmv_launches;
        info->check_full_sorts = s.check_full_sorts;
        unsigned long long ties = 0;
        if (s.tie_count.p) {
            KB_CUDA(cudaMemcpyAsync(&ties, s.tie_count.p, sizeof(ties), cudaMemcpyDeviceToHost,
                                    s.g->stream));
            KB_CUDA(cudaStreamSynchronize(s.g->stream));
        }
        info->k_boundary_ties = (int64_t)ties;
    });
}

int kb_state_set_max_iterations(kb_state *h, int64_t m) {
    return guarded([&] {
        KB_REQUIRE(h, KB_EPARAM, "NULL state");
        h->s.max_iter = m;
    });
}

static void check_version(State &s) {
    KB_REQUIRE(s.g->version == s.graph_version, KB_ESTATE,
               "graph changed since init; static iteration would be unsound");
}

int kb_iterate(kb_state *h, int64_t steps) {
    return guarded([&] {
        KB_REQUIRE(h, KB_EPARAM, "NULL state");
        State &s = h->s;
        use_device(s.g->device);
        check_version(s);
        if (steps > 0) materialize_rank_order(s, s.g->stream);
        for (int64_t i = 0; i < steps; i++) launch_iterate(s, s.g->stream);
        KB_CUDA(cudaGetLastError());
    });
}

int kb_check(kb_state *h, int *converged) {
    return guarded([&] {
        KB_REQUIRE(h && converged, KB_EPARAM, "NULL argument");
        State &s = h->s;
        use_device(s.g->device);
        ensure_init(h->s);
        *converged = run_check(s, s.g->stream) ? 1 : 0;
    });
}

int kb_run(kb_state *h, int *converged) {
    return guarded([&] {
        KB_REQUIRE(h && converged, KB_EPARAM, "NULL argument");
        State &s = h->s;
        use_device(s.g->device);
        *converged = 0;
        cudaStream_t st = s.g->stream;
        // TOPK: the loop runs on the device (topk_run_device): levels of K1 +
        // check are queued back to back, each check's count feeding the next,
        // and a converged check stops everything queued behind it
        const bool spec = s.kind == KB_TOPK && s.k <= 4096 && s.keep_all &&
                          tune_get("run.speculate", 1);
        if (spec) {
            check_version(s);
            if (topk_run_device(s, st)) {
                *converged = 1;
                return;
            }
            const double gap = run_gap(s, st);
            char buf[160];
            snprintf(buf, sizeof buf,
                     "stopping rule still unmet after %lld iterations (widest bound "
                     "interval %.3e)", (long long)s.r, gap);
            throw Error{KB_ECONVERGENCE, buf};
        }
        // RANKING: while a cached refuting pair still refutes (95 of C4's 99
        // checks) the check is one tiny kernel; K1 of r+1 is queued behind it
        // and exits on the device when the pair no longer refutes, in which
        // case the level is rolled back and the full check decides
        const bool spec_rank = s.kind == KB_RANKING && s.keep_all &&
                               tune_get("run.speculate", 1);
        if (spec_rank) {
            check_version(s);
            s.lazy_bounds = tune_get("k1.lazy_bounds", 1) != 0;
            struct Restore {   // bounds are materialized however the loop ends
                State &s;
                cudaStream_t st;
                ~Restore() {
                    s.lazy_bounds = false;
                    try { materialize_bounds(s, st); } catch (...) {}
                }
            } restore{s, st};
            launch_iterate(s, st);
            for (;;) {
                if (s.rk_q >= 0 && tune_get("check.pair_cache", 1)) {
                    if (ranking_pair_chain(s, st)) {     // still refuted at s.r
                        if (s.r >= s.max_iter) {
                            materialize_bounds(s, st);
                            const double gap = run_gap(s, st);
                            char buf[160];
                            snprintf(buf, sizeof buf,
                                     "stopping rule still unmet after %lld iterations (widest "
                                     "bound interval %.3e)", (long long)s.r, gap);
                            throw Error{KB_ECONVERGENCE, buf};
                        }
                        launch_iterate(s, st);
                        continue;
                    }
                    s.rk_q = s.rk_x = -1;                 // the full check decides at s.r
                }
                materialize_bounds(s, st);
                if (run_check(s, st)) { *converged = 1; break; }
                if (s.r >= s.max_iter) {
                    const double gap = run_gap(s, st);
                    char buf[160];
                    snprintf(buf, sizeof buf,
                             "stopping rule still unmet after %lld iterations (widest bound "
                             "interval %.3e)", (long long)s.r, gap);
                    throw Error{KB_ECONVERGENCE, buf};
                }
                launch_iterate(s, st);
            }
            return;
        }
        for (;;) {
            check_version(s);
            launch_iterate(s, s.g->stream);
            if (run_check(s, s.g->stream)) { *converged = 1; break; }
            if (s.r >= s.max_iter) {
                const double gap = run_gap(s, s.g->stream);
                char buf[160];
                snprintf(buf, sizeof buf,
                         "stopping rule still unmet after %lld iterations (widest bound "
                         "interval %.3e)", (long long)s.r, gap);
                throw Error{KB_ECONVERGENCE, buf};
            }
        }
    });
}

int kb_gap(kb_state *h, double *gap) {
    return guarded([&] {
        KB_REQUIRE(h && gap, KB_EPARAM, "NULL argument");
        use_device(h->s.g->device);
        ensure_init(h->s);
        *gap = run_gap(h->s, h->s.g->stream);
    });
}

int kb_epsilon_separated(kb_state *h, int64_t w, int64_t v, int *sep) {
    return guarded([&] {
        KB_REQUIRE(h && sep, KB_EPARAM, "NULL argument");
        State &s = h->s;
        KB_REQUIRE(w >= 0 && w < s.g->n, KB_EPARAM, "node id outside graph");
        KB_REQUIRE(v >= 0 && v < s.g->n, KB_EPARAM, "node id outside graph");
        use_device(s.g->device);
        ensure_init(h->s);
        cudaStream_t st = s.g->stream;
        k_sep_one<<<1, 1, 0, st>>>(s.lower.p, s.upper.p, s.g->iperm.p, w, v, s.eps,
                                   s.scratch_u64.p); note_launch();
        KB_CUDA(cudaMemcpyAsync(s.h_flags, s.scratch_u64.p, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
        *sep = s.h_flags[0] != 0;
    });
}

int kb_result(kb_state *h, int64_t *order, double *lower, double *upper, int64_t *pairs) {
    return guarded([&] {
        KB_REQUIRE(h, KB_EPARAM, "NULL state");
        use_device(h->s.g->device);
        ensure_init(h->s);
        run_result(h->s, h->s.g->stream, order, lower, upper, pairs);
    });
}

int kb_separated_pairs(kb_state *h, int64_t *pairs) {
    return guarded([&] {
        KB_REQUIRE(h && pairs, KB_EPARAM, "NULL argument");
        use_device(h->s.g->device);
        ensure_init(h->s);
        run_result(h->s, h->s.g->stream, nullptr, nullptr, nullptr, pairs);
    });
}

int kb_get_vector(kb_state *h, int which, int64_t level, double *out) {
    return guarded([&] {
        KB_REQUIRE(h && out, KB_EPARAM, "NULL argument");
        State &s = h->s;
        use_device(s.g->device);
        ensure_ones(h->s);
        const double *src = nullptr;
        switch (which) {
            case KB_VEC_LEVEL: {
                const int64_t idx = level - s.level_base;
                KB_REQUIRE(idx >= 0 && idx < (int64_t)s.levels.size(), KB_EPARAM,
                           "level not retained");
                src = s.levels[idx].p;
                break;
            }
            case KB_VEC_KATZ: src = s.katz.p; break;
            case KB_VEC_LOWER: src = s.lower.p; break;
            case KB_VEC_UPPER: src = s.upper.p; break;
            default: throw Error{KB_EPARAM, "unknown vector"};
        }
        cudaStream_t st = s.g->stream;
        DBuf<double> tmp;
        tmp.alloc(s.g->n);
        gather_to_original(*s.g, src, tmp.p, st);
        download_d2h(out, tmp.p, s.g->n * sizeof(double), st);
        KB_CUDA(cudaStreamSynchronize(st));
    });
}

int kb_get_active(kb_state *h, int64_t *out) {
    return guarded([&] {
        KB_REQUIRE(h && out, KB_EPARAM, "NULL argument");
        State &s = h->s;
        use_device(s.g->device);
        ensure_init(h->s);
        cudaStream_t st = s.g->stream;
        materialize_bounds(s, st);
        materialize_rank_order(s, st);
        const int64_t m = s.m_host;
        if (!m) return;
        DBuf<int64_t> tmp;
        tmp.alloc(m);
        k_active_to_orig<<<nblk(m, 256), 256, 0, st>>>(s.act[s.cur].p, s.act_dense, m,
                                                       s.g->perm.p, tmp.p); note_launch();
        KB_CUDA(cudaMemcpyAsync(out, tmp.p, m * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
    });
}

int kb_update_level_sizes(kb_state *h, int64_t *out, int64_t cap, int64_t *count) {
    return guarded([&] {
        KB_REQUIRE(h && count && (cap <= 0 || out), KB_EPARAM, "NULL argument");
        const auto &v = h->s.level_sizes;
        *count = (int64_t)v.size();
        for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)v.size()); i++) out[i] = v[i];
    });
}

int kb_update_batch(kb_state *h, const int64_t *ins, int64_t n_ins, const int64_t *dels,
                    int64_t n_dels, double theta, double new_gamma, kb_update_stats *stats) {
    return guarded([&] {
        KB_REQUIRE(h && stats, KB_EPARAM, "NULL argument");
        KB_REQUIRE((n_ins == 0 || ins) && (n_dels == 0 || dels), KB_EPARAM, "NULL arc array");
        State &s = h->s;
        use_device(s.g->device);
        ensure_ones(h->s);
        for (int64_t i = 0; i < 2 * n_ins; i++)
            KB_REQUIRE(ins[i] >= 0 && ins[i] < s.g->n, KB_ENODERANGE, "node id outside graph");
        for (int64_t i = 0; i < 2 * n_dels; i++)
            KB_REQUIRE(dels[i] >= 0 && dels[i] < s.g->n, KB_ENODERANGE, "node id outside graph");
        materialize_rank_order(s, s.g->stream);
        update_batch(s, ins, n_ins, dels, n_dels, theta, new_gamma, stats);
    });
}

}  // extern "C"
