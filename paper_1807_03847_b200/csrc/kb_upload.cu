// Host -> device uploads from pageable memory.
//
// A pageable cudaMemcpyAsync is staged by the driver through its own pinned
// buffer with a single-threaded host copy: 11 GB/s on the B200 box (C2's
// 2.2 GB CSR: 200 ms), and page-locking the arrays first costs more
// (cudaHostRegister of 2.2 GB: 170 ms).  Here the bytes go through a ring of
// page-locked slots that a small pool of host threads fills in parallel
// while the copy engine drains the previous slot, so the upload runs near
// the PCIe rate from ordinary numpy arrays too.
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "kb_internal.cuh"

namespace kb {

namespace {

// Parallel memcpy: the caller copies part 0, T-1 workers the rest.  The pool
// lives for the whole process (never destroyed: joinable threads must not be
// torn down at exit).
class CopyPool {
  public:
    explicit CopyPool(int T) : T_(T) {
        for (int i = 1; i < T_; i++) th_.emplace_back([this, i] { worker(i); });
    }
    void copy(void *dst, const void *src, size_t bytes) {
        {
            std::lock_guard<std::mutex> lk(m_);
            d_ = (char *)dst;
            s_ = (const char *)src;
            n_ = bytes;
            fn_ = nullptr;
            pending_ = T_ - 1;
            gen_++;
        }
        cv_.notify_all();
        part(0, (char *)dst, (const char *)src, bytes);
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }
    // fn(i, T) on every pool thread (i = 0 on the caller)
    void parallel(const std::function<void(int, int)> &fn) {
        {
            std::lock_guard<std::mutex> lk(m_);
            fn_ = &fn;
            pending_ = T_ - 1;
            gen_++;
        }
        cv_.notify_all();
        fn(0, T_);
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }

  private:
    void part(int i, char *d, const char *s, size_t n) const {
        const size_t a = (n * i / T_) & ~(size_t)63, b = (i + 1 == T_) ? n : (n * (i + 1) / T_) & ~(size_t)63;
        if (b > a) memcpy(d + a, s + a, b - a);
    }
    void worker(int i) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            char *d = d_;
            const char *s = s_;
            const size_t n = n_;
            const std::function<void(int, int)> *fn = fn_;
            lk.unlock();
            if (fn) (*fn)(i, T_);
            else part(i, d, s, n);
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }
    int T_;
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    char *d_ = nullptr;
    const char *s_ = nullptr;
    size_t n_ = 0;
    const std::function<void(int, int)> *fn_ = nullptr;
    uint64_t gen_ = 0;
    int pending_ = 0;
};

constexpr int RING = 4;
constexpr size_t SLOT = (size_t)32 << 20;

struct Ring {
    void *slot[RING] = {};
    cudaEvent_t ev[RING] = {};
    int next = 0;
};

std::mutex g_up_mu;

CopyPool &pool() {
    static CopyPool *p = new CopyPool(
        (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency())));
    return *p;
}

Ring &ring(int dev) {
    static Ring r[64];
    Ring &x = r[dev];
    if (!x.slot[0]) {
        for (int i = 0; i < RING; i++) {
            KB_CUDA(cudaHostAlloc(&x.slot[i], SLOT, cudaHostAllocPortable));
            KB_CUDA(cudaEventCreateWithFlags(&x.ev[i], cudaEventDisableTiming));
        }
    }
    return x;
}

}  // namespace

bool host_is_pinned(const void *p) {
    cudaPointerAttributes a{};
    const bool ok = p && cudaPointerGetAttributes(&a, p) == cudaSuccess &&
                    a.type == cudaMemoryTypeHost;
    (void)cudaGetLastError();
    return ok;
}

// dst (device) <- src (host), ordered on stream cs.  Page-locked sources are
// a plain async copy; pageable ones go through the ring (the call returns
// once the last byte is staged; the copies complete in stream order).
void upload_h2d(void *dst, const void *src, size_t bytes, cudaStream_t cs) {
    if (!bytes) return;
    if (host_is_pinned(src) || bytes < ((size_t)1 << 20) || !tune_get("upload.ring", 1)) {
        KB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cs));
        return;
    }
    std::lock_guard<std::mutex> lk(g_up_mu);
    int dev = 0;
    KB_CUDA(cudaGetDevice(&dev));
    Ring &R = ring(dev);
    for (size_t off = 0; off < bytes; off += SLOT) {
        const size_t len = std::min(SLOT, bytes - off);
        const int i = R.next;
        R.next = (R.next + 1) % RING;
        KB_CUDA(cudaEventSynchronize(R.ev[i]));   // the slot's previous copy is done
        pool().copy(R.slot[i], (const char *)src + off, len);
        KB_CUDA(cudaMemcpyAsync((char *)dst + off, R.slot[i], len, cudaMemcpyHostToDevice, cs));
        KB_CUDA(cudaEventRecord(R.ev[i], cs));
    }
}

// dst (device) <- a virtual host source of `bytes` bytes that fill(slot, off,
// len, i, T) materialises piece by piece (part i of T on every pool thread)
// into page-locked ring slots, each copied on stream cs while the next is
// filled: a host-side gather (a rank's rows of a host CSR) at the PCIe rate
void upload_gather_h2d(void *dst, size_t bytes, cudaStream_t cs,
                       const std::function<void(char *, size_t, size_t, int, int)> &fill) {
    if (!bytes) return;
    std::lock_guard<std::mutex> lk(g_up_mu);
    int dev = 0;
    KB_CUDA(cudaGetDevice(&dev));
    Ring &R = ring(dev);
    for (size_t off = 0; off < bytes; off += SLOT) {
        const size_t len = std::min(SLOT, bytes - off);
        const int i = R.next;
        R.next = (R.next + 1) % RING;
        KB_CUDA(cudaEventSynchronize(R.ev[i]));
        char *slot = (char *)R.slot[i];
        pool().parallel([&](int t, int T) { fill(slot, off, len, t, T); });
        KB_CUDA(cudaMemcpyAsync((char *)dst + off, slot, len, cudaMemcpyHostToDevice, cs));
        KB_CUDA(cudaEventRecord(R.ev[i], cs));
    }
}

// host dst <- device src after the work queued on st.  Page-locked or small
// destinations: a plain async copy (the caller synchronises).  Pageable
// ones: up to RING slot copies in flight, each drained into dst by the host
// threads as it lands; returns when dst is complete.
void download_d2h(void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (!bytes) return;
    if (host_is_pinned(dst) || bytes < ((size_t)1 << 20) || !tune_get("upload.ring", 1)) {
        KB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        return;
    }
    std::lock_guard<std::mutex> lk(g_up_mu);
    int dev = 0;
    KB_CUDA(cudaGetDevice(&dev));
    Ring &R = ring(dev);
    const size_t npieces = (bytes + SLOT - 1) / SLOT;
    auto issue = [&](size_t k) {
        const size_t off = k * SLOT, len = std::min(SLOT, bytes - off);
        const int i = (int)(k % RING);
        KB_CUDA(cudaMemcpyAsync(R.slot[i], (const char *)src + off, len, cudaMemcpyDeviceToHost,
                                st));
        KB_CUDA(cudaEventRecord(R.ev[i], st));
    };
    // the ring's slots may still feed an upload on another stream
    for (int i = 0; i < RING; i++) KB_CUDA(cudaEventSynchronize(R.ev[i]));
    for (size_t k = 0; k < std::min(npieces, (size_t)RING); k++) issue(k);
    for (size_t k = 0; k < npieces; k++) {
        const int i = (int)(k % RING);
        const size_t off = k * SLOT, len = std::min(SLOT, bytes - off);
        KB_CUDA(cudaEventSynchronize(R.ev[i]));
        pool().copy((char *)dst + off, R.slot[i], len);
        if (k + RING < npieces) issue(k + RING);
    }
}

}  // namespace kb
