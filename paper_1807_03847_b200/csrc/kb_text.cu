// Text ingestion on the device: load_edge_list
// (graph.py:260-320) and load_batches (dynamic.py:216-253) for SNAP/KONECT-
// scale inputs.
//
// The file bytes are copied to HBM once; newline positions are compacted
// with a flag + select pass; then one thread per line strips and splits it
// (ASCII whitespace as Python's str.isspace) and classifies it:
//
//   edge lists   0 blank / '#' / '%' comment   1 arc "u v"
//                2 "NODES n" candidate          3 anomaly
//   batches      0 blank (batch separator)      1 "+ u v"   4 "- u v"
//                3 anomaly
//
// Only the plain ASCII grammar is decided here: ids are [+]?[0-9]+ up to
// 2^31-1.  Every other line (non-ASCII bytes, signs, underscores, overflow,
// wrong field counts, misplaced headers ...) is an *anomaly*: the host
// re-reads just those lines with the reference's exact rules (UTF-8 decode,
// int(), error messages and line numbers), in file order, so the first error
// is reported exactly as the reference would.  Arcs then go straight into
// the device CSR builder: (u << b | v) keys, radix sort, unique, row starts.
#include "kb_internal.cuh"

#include <cub/cub.cuh>

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

__device__ __forceinline__ bool is_space(unsigned char c) {
    // str.isspace over ASCII: \t \n \v \f \r, \x1c-\x1f, ' '
    return c == ' ' || (c >= 9 && c <= 13) || (c >= 0x1c && c <= 0x1f);
}

struct IsNewline {
    const unsigned char *buf;
    __device__ bool operator()(int64_t i) const { return buf[i] == '\n'; }
};

// [+]?[0-9]+ with value <= 2^31-1; false otherwise (the host decides)
__device__ bool parse_id(const unsigned char *s, int len, int32_t *out) {
    int i = 0;
    if (len && s[0] == '+') i = 1;
    if (i >= len) return false;
    int64_t v = 0;
    for (; i < len; i++) {
        const unsigned c = s[i] - '0';
        if (c > 9) return false;
        v = v * 10 + c;
        if (v > 2147483647ll) return false;
    }
    *out = (int32_t)v;
    return true;
}

__device__ bool is_nodes(const unsigned char *s, int len) {
    const char *w = "NODES";
    if (len != 5) return false;
    for (int i = 0; i < 5; i++) {
        unsigned char c = s[i];
        if (c >= 'a' && c <= 'z') c -= 32;
        if (c != (unsigned char)w[i]) return false;
    }
    return true;
}

__global__ void k_parse_lines(const unsigned char *__restrict__ buf, int64_t nbytes,
                              const int64_t *__restrict__ nl, int64_t n_nl, int64_t n_lines,
                              int batches, uint8_t *kind, int32_t *u, int32_t *v) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_lines) return;
    const int64_t start = i ? nl[i - 1] + 1 : 0;
    const int64_t end = i < n_nl ? nl[i] : nbytes;
    int ntok = 0;
    int64_t ts[3] = {0, 0, 0};
    int tl[3] = {0, 0, 0};
    bool ascii = true, cr = false;
    int64_t p = start;
    while (p < end) {
        while (p < end && is_space(buf[p])) {
            cr |= buf[p] == '\r';
            p++;
        }
        if (p >= end) break;
        const int64_t t0 = p;
        while (p < end && !is_space(buf[p])) {
            ascii &= buf[p] < 0x80;
            p++;
        }
        if (ntok < 3) {
            ts[ntok] = t0;
            tl[ntok] = (p - t0) > (1 << 20) ? (1 << 20) : (int)(p - t0);
        }
        ntok++;
    }
    uint8_t k = 3;
    int32_t a = 0, b = 0;
    if (!ascii) {
        k = 3;                                   // decode + unicode rules: host
    } else if (batches) {
        if (cr) k = 3;                           // text-mode newline translation: host
        else if (ntok == 0) k = 0;
        else if (ntok == 3 && tl[0] == 1 && (buf[ts[0]] == '+' || buf[ts[0]] == '-') &&
                 parse_id(buf + ts[1], tl[1], &a) && parse_id(buf + ts[2], tl[2], &b))
            k = buf[ts[0]] == '+' ? 1 : 4;
    } else {
        if (ntok == 0 || buf[ts[0]] == '#' || buf[ts[0]] == '%') k = 0;
        else if (is_nodes(buf + ts[0], tl[0])) k = (ntok == 2 && parse_id(buf + ts[1], tl[1], &a)) ? 2 : 3;
        else if (ntok == 2 && parse_id(buf + ts[0], tl[0], &a) && parse_id(buf + ts[1], tl[1], &b))
            k = 1;
    }
    kind[i] = k;
    u[i] = a;
    v[i] = b;
}

struct KindIs {
    const uint8_t *kind;
    uint8_t a, b;
    __device__ bool operator()(int64_t i) const { return kind[i] == a || kind[i] == b; }
};

__global__ void k_arc_stats(const uint8_t *kind, const int32_t *u, const int32_t *v, int64_t n,
                            unsigned long long *first_content, unsigned long long *max_id) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long fc = ~0ull, mx = 0;
    if (i < n) {
        if (kind[i] == 1) {
            fc = (unsigned long long)i;
            mx = (unsigned long long)max(u[i], v[i]) + 1;  // +1: 0 means "none"
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        fc = min(fc, __shfl_down_sync(0xffffffffu, fc, o));
        mx = max(mx, __shfl_down_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (fc != ~0ull) atomicMin(first_content, fc);
        if (mx) atomicMax(max_id, mx);
    }
}

__global__ void k_line_bounds(const int64_t *idx, int64_t m, const int64_t *nl, int64_t n_nl,
                              int64_t nbytes, int64_t *out) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int64_t i = idx[j];
    out[3 * j] = i;
    out[3 * j + 1] = i ? nl[i - 1] + 1 : 0;
    out[3 * j + 2] = i < n_nl ? nl[i] : nbytes;
}

// arc keys (u << b) | v, plus the reversal for undirected loads
__global__ void k_arc_keys(const uint8_t *kind, const int32_t *u, const int32_t *v,
                           const int64_t *sel, int64_t m, int b, int undirected,
                           uint64_t *keys) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int64_t i = sel[j];
    const uint64_t a = (uint64_t)u[i], c = (uint64_t)v[i];
    keys[j] = (a << b) | c;
    if (undirected) keys[m + j] = (c << b) | a;
}

__global__ void k_extra_keys(const int64_t *arcs, int64_t m, int b, int undirected,
                             uint64_t *keys) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= m) return;
    const uint64_t a = (uint64_t)arcs[2 * j], c = (uint64_t)arcs[2 * j + 1];
    keys[j] = (a << b) | c;
    if (undirected) keys[m + j] = (c << b) | a;
}

__global__ void k_key_rows(const uint64_t *keys, int64_t ne, int64_t n, int b, int64_t *start) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r > n) return;
    const uint64_t target = (uint64_t)r << b;
    int64_t lo = 0, hi = ne;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    start[r] = lo;
}

__global__ void k_key_cols(const uint64_t *keys, int64_t ne, int b, int32_t *cols) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j < ne) cols[j] = (int32_t)(keys[j] & ((1ull << b) - 1));
}

}  // namespace

void text_scan(TextScan &t, const char *h_bytes, int64_t nbytes, int batches) {
    cudaStream_t st = device_stream();
    t.nbytes = nbytes;
    t.batches = batches;
    t.buf.alloc(std::max<int64_t>(1, nbytes));
    if (nbytes)
        KB_CUDA(cudaMemcpyAsync(t.buf.p, h_bytes, nbytes, cudaMemcpyHostToDevice, st));
    // newline positions
    DBuf<int64_t> cnt;
    cnt.alloc(4);
    t.nl.alloc(std::max<int64_t>(1, nbytes));
    if (nbytes) {
        cub::CountingInputIterator<int64_t> it(0);
        IsNewline pred{(const unsigned char *)t.buf.p};
        cub_run([&](void *tmp, size_t &b) {
            return cub::DeviceSelect::If(tmp, b, it, t.nl.p, cnt.p, nbytes, pred, st);
        });
    } else {
        KB_CUDA(cudaMemsetAsync(cnt.p, 0, 8, st));
    }
    int64_t n_nl = 0;
    KB_CUDA(cudaMemcpyAsync(&n_nl, cnt.p, 8, cudaMemcpyDeviceToHost, st));
    char last = '\n';
    if (nbytes) KB_CUDA(cudaMemcpyAsync(&last, t.buf.p + nbytes - 1, 1, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    t.n_nl = n_nl;
    t.n_lines = n_nl + (last != '\n' ? 1 : 0);
    const int64_t L = t.n_lines;
    t.kind.alloc(std::max<int64_t>(1, L));
    t.u.alloc(std::max<int64_t>(1, L));
    t.v.alloc(std::max<int64_t>(1, L));
    DBuf<unsigned long long> red;
    red.alloc(2);
    const unsigned long long init[2] = {~0ull, 0ull};
    KB_CUDA(cudaMemcpyAsync(red.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    if (L) {
        k_parse_lines<<<nblk(L, 256), 256, 0, st>>>((const unsigned char *)t.buf.p, nbytes,
                                                    t.nl.p, n_nl, L, batches, t.kind.p, t.u.p,
                                                    t.v.p);
        k_arc_stats<<<nblk(L, 256), 256, 0, st>>>(t.kind.p, t.u.p, t.v.p, L, red.p, red.p + 1);
        note_launch(2);
    }
    // anomalies (+ header candidates) and arc lines, each in line order
    t.cand.alloc(std::max<int64_t>(1, L));
    t.arcs.alloc(std::max<int64_t>(1, L));
    KB_CUDA(cudaMemsetAsync(cnt.p, 0, 32, st));
    if (L) {
        cub::CountingInputIterator<int64_t> it(0);
        KindIs anom{t.kind.p, 2, 3};
        KindIs arc{t.kind.p, 1, 4};
        cub_run([&](void *tmp, size_t &b) {
            return cub::DeviceSelect::If(tmp, b, it, t.cand.p, cnt.p, L, anom, st);
        });
        cub_run([&](void *tmp, size_t &b) {
            return cub::DeviceSelect::If(tmp, b, it, t.arcs.p, cnt.p + 1, L, arc, st);
        });
    }
    int64_t hc[2];
    unsigned long long hr[2];
    KB_CUDA(cudaMemcpyAsync(hc, cnt.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaMemcpyAsync(hr, red.p, sizeof(hr), cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
    t.n_cand = hc[0];
    t.n_arcs = hc[1];
    t.first_arc_line = hr[0] == ~0ull ? -1 : (int64_t)hr[0];
    t.max_id = (int64_t)hr[1] - 1;
}

void text_candidates(TextScan &t, int64_t *h_out) {
    if (!t.n_cand) return;
    cudaStream_t st = device_stream();
    DBuf<int64_t> o;
    o.alloc(3 * t.n_cand);
    k_line_bounds<<<nblk(t.n_cand, 256), 256, 0, st>>>(t.cand.p, t.n_cand, t.nl.p, t.n_nl,
                                                      t.nbytes, o.p);
    note_launch();
    KB_CUDA(cudaMemcpyAsync(h_out, o.p, 3 * t.n_cand * 8, cudaMemcpyDeviceToHost, st));
    KB_CUDA(cudaStreamSynchronize(st));
}

void text_lines(TextScan &t, uint8_t *h_kind, int32_t *h_u, int32_t *h_v) {
    cudaStream_t st = device_stream();
    if (t.n_lines) {
        if (h_kind) KB_CUDA(cudaMemcpyAsync(h_kind, t.kind.p, t.n_lines, cudaMemcpyDeviceToHost, st));
        if (h_u) KB_CUDA(cudaMemcpyAsync(h_u, t.u.p, t.n_lines * 4, cudaMemcpyDeviceToHost, st));
        if (h_v) KB_CUDA(cudaMemcpyAsync(h_v, t.v.p, t.n_lines * 4, cudaMemcpyDeviceToHost, st));
    }
    KB_CUDA(cudaStreamSynchronize(st));
}

// canonical CSR (rows ascending, duplicates collapsed) of the scanned arcs
// plus host-resolved extra arcs, over the universe [0, n)
void text_csr(TextScan &t, int64_t n, int undirected, const int64_t *h_extra, int64_t n_extra,
              DBuf<int64_t> &indptr, DBuf<int32_t> &indices, int64_t &nnz) {
    cudaStream_t st = device_stream();
    KB_REQUIRE(n >= 0 && n <= ((int64_t)1 << 31), KB_EPARAM, "node count out of range");
    KB_REQUIRE(t.max_id < n, KB_ENODERANGE, "node id exceeds the declared universe");
    int b = 1;
    while (((int64_t)1 << b) < n) b++;
    const int64_t m1 = t.n_arcs, m2 = n_extra;
    const int mul = undirected ? 2 : 1;
    const int64_t m = mul * (m1 + m2);
    DBuf<uint64_t> keys, sorted;
    keys.alloc(std::max<int64_t>(1, m));
    sorted.alloc(std::max<int64_t>(1, m));
    if (m1) {
        k_arc_keys<<<nblk(m1, 256), 256, 0, st>>>(t.kind.p, t.u.p, t.v.p, t.arcs.p, m1, b,
                                                  undirected, keys.p);
        note_launch();
    }
    if (m2) {
        DBuf<int64_t> ex;
        ex.alloc(2 * m2);
        KB_CUDA(cudaMemcpyAsync(ex.p, h_extra, 2 * m2 * 8, cudaMemcpyHostToDevice, st));
        k_extra_keys<<<nblk(m2, 256), 256, 0, st>>>(ex.p, m2, b, undirected,
                                                    keys.p + mul * m1);
        note_launch();
        KB_CUDA(cudaStreamSynchronize(st));   // ex is released at scope exit
    }
    int64_t ne = 0;
    if (m) {
        cub_run([&](void *tmp, size_t &bb) {
            return cub::DeviceRadixSort::SortKeys(tmp, bb, keys.p, sorted.p, m, 0, 2 * b, st);
        });
        DBuf<int64_t> c;
        c.alloc(1);
        cub_run([&](void *tmp, size_t &bb) {
            return cub::DeviceSelect::Unique(tmp, bb, sorted.p, keys.p, c.p, m, st);
        });
        KB_CUDA(cudaMemcpyAsync(&ne, c.p, 8, cudaMemcpyDeviceToHost, st));
        KB_CUDA(cudaStreamSynchronize(st));
    }
    indptr.alloc(n + 1);
    k_key_rows<<<nblk(n + 1, 256), 256, 0, st>>>(keys.p, ne, n, b, indptr.p);
    note_launch();
    indices.alloc(std::max<int64_t>(1, ne));
    if (ne) {
        k_key_cols<<<nblk(ne, 256), 256, 0, st>>>(keys.p, ne, b, indices.p);
        note_launch();
    }
    KB_CUDA(cudaGetLastError());
    KB_CUDA(cudaStreamSynchronize(st));
    nnz = ne;
}

}  // namespace kb
