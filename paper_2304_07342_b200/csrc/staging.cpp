// staging.cpp — pageable host memory <-> device at copy-engine speed.
//
// cudaMemcpy[Async] of pageable memory goes through the driver's staging: one
// host thread copies the caller's pages into a small pinned buffer, then the
// DMA moves it, ~10 GB/s on the B200 boxes (bench.py e2e.pageable).  The
// callers of the reference's std::vector API (plz::compress(std::span),
// decompress_bytes) hand us exactly such memory, so large transfers are
// staged here instead: a process-wide pool of host threads copies between
// the caller's pages and one of three pinned slots of the context while the
// copy engine moves another slot.
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>

#include "host_internal.h"

namespace plzhost {

namespace {

constexpr int kSlots = 3;

class CopyPool {
  public:
    static CopyPool& get() {
        static CopyPool* pool = new CopyPool();  // never destroyed (threads outlive statics)
        return *pool;
    }

    void copy(void* dst, const void* src, size_t n) {
        if (n < (size_t(4) << 20) || workers_ == 0) {
            std::memcpy(dst, src, n);
            return;
        }
        std::lock_guard<std::mutex> serial(busy_);  // one multi-threaded copy at a time
        const int parts = workers_ + 1;
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<uint8_t*>(dst);
            src_ = static_cast<const uint8_t*>(src);
            n_ = n;
            parts_ = parts;
            pending_ = workers_;
            ++gen_;
        }
        cv_.notify_all();
        std::memcpy(dst, src, part_end(n, 0, parts));  // part 0 on the calling thread
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
    }

  private:
    CopyPool() {
        const PipelineConfig& cfg = pipeline_config();
        int t = cfg.copy_threads;
        if (t <= 0) {
            const unsigned hc = std::thread::hardware_concurrency();
            t = int(hc > 1 ? hc - 1 : 0);
        }
        workers_ = std::min(t, 15);
        for (int i = 0; i < workers_; ++i) std::thread([this, i] { run(i + 1); }).detach();
    }

    static size_t part_end(size_t n, int k, int parts) {  // end of part k (64-byte aligned cuts)
        return k + 1 == parts ? n : (n / size_t(parts) * size_t(k + 1)) & ~size_t(63);
    }

    void run(int k) {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(mu_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            uint8_t* d = dst_;
            const uint8_t* s = src_;
            const size_t n = n_;
            const int parts = parts_;
            lk.unlock();
            const size_t lo = part_end(n, k - 1, parts), hi = part_end(n, k, parts);
            if (hi > lo) std::memcpy(d + lo, s + lo, hi - lo);
            lk.lock();
            if (--pending_ == 0) done_.notify_one();
        }
    }

    int workers_ = 0;
    std::mutex busy_, mu_;
    std::condition_variable cv_, done_;
    uint64_t gen_ = 0;
    int pending_ = 0, parts_ = 1;
    uint8_t* dst_ = nullptr;
    const uint8_t* src_ = nullptr;
    size_t n_ = 0;
};

// Slot size (a multiple of `unit` when given) and the context's slots.
int ensure_slots(plzgpu_ctx* c, uint64_t unit, uint64_t* slot, plzgpu_error* err) {
    uint64_t s = pipeline_config().pageable_stage;
    if (unit) s = std::max<uint64_t>(1, s / unit) * unit;
    if (c->bounce_cap < s) {
        for (uint8_t*& b : c->bounce) {
            if (b) cudaFreeHost(b);
            b = nullptr;
        }
        c->bounce_cap = 0;
        for (uint8_t*& b : c->bounce) CK(cudaMallocHost(reinterpret_cast<void**>(&b), s));
        c->bounce_cap = s;
    }
    for (cudaEvent_t& ev : c->bounce_ev)
        if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    if (!c->order_ev) CK(cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming));
    if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    *slot = s;
    return PLZGPU_OK;
}

}  // namespace

void pool_memcpy(void* dst, const void* src, size_t n) { CopyPool::get().copy(dst, src, n); }

bool use_staged(const void* host_ptr, uint64_t n) {
    return n >= pipeline_config().pageable_min && !is_pinned_host(host_ptr) && !is_device_ptr(host_ptr);
}

int h2d_pageable(plzgpu_ctx* c, uint8_t* d_dst, const uint8_t* h_src, uint64_t n,
                 cudaStream_t st, bool after_st, const uint32_t* ready, uint64_t seg_bytes,
                 uint32_t epoch, plzgpu_error* err) {
    uint64_t slot = 0;
    int rc = ensure_slots(c, ready ? seg_bytes : 0, &slot, err);
    if (rc) return rc;
    const StreamValue32Fn write_value = stream_write_value32();
    if (ready && !write_value)
        return set_err(err, PLZGPU_CUDA, 0, kNoIndex, kNoIndex, "cuStreamWriteValue32 unavailable");
    if (after_st) {
        CK(cudaEventRecord(c->order_ev, st));
        CK(cudaStreamWaitEvent(c->copy_stream, c->order_ev, 0));
    }
    uint64_t i = 0;
    for (uint64_t off = 0; off < n; off += slot, ++i) {
        const int k = int(i % kSlots);
        const uint64_t len = std::min(slot, n - off);
        if (i >= kSlots) CK(cudaEventSynchronize(c->bounce_ev[k]));  // the slot's last DMA
        pool_memcpy(c->bounce[k], h_src + off, len);
        CK(cudaMemcpyAsync(d_dst + off, c->bounce[k], len, cudaMemcpyHostToDevice, c->copy_stream));
        CK(cudaEventRecord(c->bounce_ev[k], c->copy_stream));
        if (ready) {
            const uint64_t g0 = off / seg_bytes;
            const uint64_t g1 = off + len == n ? (n + seg_bytes - 1) / seg_bytes : (off + len) / seg_bytes;
            for (uint64_t g = g0; g < g1; ++g)
                if (write_value(c->copy_stream, reinterpret_cast<unsigned long long>(ready + g), epoch,
                                0) != 0)
                    return set_err(err, PLZGPU_CUDA, 0, kNoIndex, kNoIndex,
                                   "cuStreamWriteValue32 failed");
        }
    }
    if (!ready) {  // the consumer is the work enqueued on st next
        CK(cudaEventRecord(c->order_ev, c->copy_stream));
        CK(cudaStreamWaitEvent(st, c->order_ev, 0));
    }
    return PLZGPU_OK;
}

int d2h_pageable(plzgpu_ctx* c, uint8_t* h_dst, const uint8_t* d_src, uint64_t n,
                 cudaStream_t st, plzgpu_error* err) {
    uint64_t slot = 0;
    int rc = ensure_slots(c, 0, &slot, err);
    if (rc) return rc;
    CK(cudaEventRecord(c->order_ev, st));
    CK(cudaStreamWaitEvent(c->copy_stream, c->order_ev, 0));
    const uint64_t nslots = (n + slot - 1) / slot;
    auto issue = [&](uint64_t i) -> int {
        const int k = int(i % kSlots);
        const uint64_t off = i * slot, len = std::min(slot, n - off);
        CK(cudaMemcpyAsync(c->bounce[k], d_src + off, len, cudaMemcpyDeviceToHost, c->copy_stream));
        CK(cudaEventRecord(c->bounce_ev[k], c->copy_stream));
        return PLZGPU_OK;
    };
    for (uint64_t i = 0; i < std::min<uint64_t>(kSlots, nslots); ++i)
        if ((rc = issue(i))) return rc;
    for (uint64_t i = 0; i < nslots; ++i) {
        const int k = int(i % kSlots);
        const uint64_t off = i * slot, len = std::min(slot, n - off);
        CK(cudaEventSynchronize(c->bounce_ev[k]));
        pool_memcpy(h_dst + off, c->bounce[k], len);
        if (i + kSlots < nslots && (rc = issue(i + kSlots))) return rc;
    }
    return PLZGPU_OK;
}

}  // namespace plzhost
