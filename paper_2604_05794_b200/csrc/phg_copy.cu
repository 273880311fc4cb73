// phg_copy.cu -- host<->device copies for PAGEABLE host memory (numpy arrays of the drop-in).
//
// cudaMemcpy to/from pageable memory goes through a driver bounce buffer one chunk at a time
// and runs far below PCIe speed.  Here large copies are staged through two pinned chunks owned
// by the library: the DMA of chunk k overlaps a multi-threaded memcpy of chunk k-1 (host side),
// so the transfer runs near the slower of PCIe and host-memcpy bandwidth.  Pinned host memory
// and device memory are copied directly.  Both functions return when the data has arrived.

#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "phg_core.cuh"

namespace phg {
namespace {

constexpr size_t kChunk = 64ull << 20;       // pinned staging chunk
constexpr size_t kDirectBelow = 8ull << 20;  // small copies: plain cudaMemcpy

// Fixed pool of host threads for the parallel memcpy of one chunk.
class MemcpyPool {
  public:
    MemcpyPool() {
        unsigned n = std::thread::hardware_concurrency();
        n = n < 2 ? 1 : (n > 16 ? 16 : n);
        for (unsigned i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
        nthreads_ = n;
    }
    ~MemcpyPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    // dst[0:n) = src[0:n), split across all threads (the caller works too)
    void copy(void* dst, const void* src, size_t n) {
        if (nthreads_ == 1 || n < (4u << 20)) {
            std::memcpy(dst, src, n);
            return;
        }
        const size_t part = (n / nthreads_ + 4095) & ~size_t(4095);
        std::unique_lock<std::mutex> lk(m_);
        pending_ = 0;
        for (unsigned i = 1; i < nthreads_; ++i) {
            const size_t a = part * i;
            if (a >= n) break;
            const size_t b = std::min(n, a + part);
            jobs_.push_back([=] { std::memcpy((char*)dst + a, (const char*)src + a, b - a); });
            ++pending_;
        }
        lk.unlock();
        cv_.notify_all();
        std::memcpy(dst, src, std::min(n, part));
        lk.lock();
        done_.wait(lk, [this] { return pending_ == 0; });
    }

  private:
    void loop() {
        std::unique_lock<std::mutex> lk(m_);
        while (true) {
            cv_.wait(lk, [this] { return stop_ || !jobs_.empty(); });
            if (stop_) return;
            auto job = std::move(jobs_.back());
            jobs_.pop_back();
            lk.unlock();
            job();
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::vector<std::function<void()>> jobs_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    unsigned nthreads_ = 1;
    int pending_ = 0;
    bool stop_ = false;
};

struct Staging {
    std::mutex m;  // one staged copy at a time per process
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    MemcpyPool pool;
    phg_status ensure() {
        if (buf[0]) return PHG_OK;
        for (int k = 0; k < 2; ++k) {
            PHG_CUDA(cudaMallocHost(&buf[k], kChunk));
            PHG_CUDA(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
        }
        return PHG_OK;
    }
};

Staging& staging() {
    static Staging* s = new Staging();  // process lifetime (not destroyed at exit)
    return *s;
}

bool is_pinned_or_device(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice ||
           a.type == cudaMemoryTypeManaged;
}

}  // namespace

phg_status copy_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return PHG_OK;
    if (bytes < kDirectBelow || is_pinned_or_device(src)) {
        PHG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
        PHG_CUDA(cudaStreamSynchronize(st));
        return PHG_OK;
    }
    Staging& S = staging();
    std::lock_guard<std::mutex> g(S.m);
    PHG_TRY(S.ensure());
    const size_t n = (bytes + kChunk - 1) / kChunk;
    for (size_t i = 0; i < n; ++i) {
        const int k = (int)(i & 1);
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        if (i >= 2) PHG_CUDA(cudaEventSynchronize(S.ev[k]));  // chunk i-2's DMA has drained
        S.pool.copy(S.buf[k], (const char*)src + off, len);
        PHG_CUDA(cudaMemcpyAsync((char*)dst + off, S.buf[k], len, cudaMemcpyHostToDevice, st));
        PHG_CUDA(cudaEventRecord(S.ev[k], st));
    }
    PHG_CUDA(cudaStreamSynchronize(st));
    return PHG_OK;
}

phg_status copy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (bytes == 0) return PHG_OK;
    if (bytes < kDirectBelow || is_pinned_or_device(dst)) {
        PHG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st));
        PHG_CUDA(cudaStreamSynchronize(st));
        return PHG_OK;
    }
    Staging& S = staging();
    std::lock_guard<std::mutex> g(S.m);
    PHG_TRY(S.ensure());
    const size_t n = (bytes + kChunk - 1) / kChunk;
    for (size_t i = 0; i <= n; ++i) {
        if (i < n) {  // DMA chunk i while the host unpacks chunk i-1
            const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
            PHG_CUDA(cudaMemcpyAsync(S.buf[i & 1], (const char*)src + off, len,
                                     cudaMemcpyDeviceToHost, st));
            PHG_CUDA(cudaEventRecord(S.ev[i & 1], st));
        }
        if (i > 0) {
            const size_t j = i - 1, off = j * kChunk, len = std::min(kChunk, bytes - off);
            PHG_CUDA(cudaEventSynchronize(S.ev[j & 1]));
            S.pool.copy((char*)dst + off, S.buf[j & 1], len);
        }
    }
    return PHG_OK;
}

}  // namespace phg
