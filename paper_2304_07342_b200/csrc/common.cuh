// common.cuh — shared device-side definitions for the sm_100a GPULZ kernels.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.h"

namespace plzgpu {

// Symbol types by width S and the packed (symbol, run) smem cell the matcher
// works on: cell = symbol | min(255, equal-run length) << (8*S).
template <int S> struct Sym;
template <> struct Sym<1> { using T = uint8_t;  using Cell = uint16_t; };
template <> struct Sym<2> { using T = uint16_t; using Cell = uint32_t; };
template <> struct Sym<4> { using T = uint32_t; using Cell = uint64_t; };

template <int S>
__device__ __forceinline__ typename Sym<S>::T cell_sym(typename Sym<S>::Cell c) {
    return static_cast<typename Sym<S>::T>(c);
}
template <int S>
__device__ __forceinline__ uint32_t cell_run(typename Sym<S>::Cell c) {
    return static_cast<uint32_t>(c >> (8 * S));
}
template <int S>
__device__ __forceinline__ typename Sym<S>::Cell make_cell(typename Sym<S>::T v, uint32_t run) {
    using Cell = typename Sym<S>::Cell;
    return static_cast<Cell>(v) | (static_cast<Cell>(run) << (8 * S));
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// ----------------------------------------------------------- async copies
// 1-D TMA bulk copy global -> shared, completion on an mbarrier
// (SASS: UBLKCP.S.G + SYNCS).  dst/src 16-byte aligned, bytes % 16 == 0.
__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* mbar) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    const uint32_t m = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(d),
        "l"(src), "r"(bytes), "r"(m)
        : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
    const uint32_t m = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(m), "r"(phase)
            : "memory");
    }
}

// 1-D TMA bulk copy shared -> global as a bulk group of the issuing thread
// (SASS: UBLKCP.G.S).  dst/src 16-byte aligned, bytes % 16 == 0.  The
// writers of src run fence_proxy_async_smem() + a warp barrier first.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(src));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(s),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Lane 0's bulk stores have read their shared source (the buffer may be
// rewritten); a no-op without outstanding stores.
__device__ __forceinline__ void bulk_store_drain(uint32_t lane) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
}
// Lane 0's bulk stores are complete (visible in global memory).
__device__ __forceinline__ void bulk_store_complete(uint32_t lane) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
}

// Orders this thread's generic-proxy shared-memory accesses before later
// async-proxy (TMA) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ------------------------------------------------------ release / acquire
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Little-endian unaligned loads from global bytes.
__device__ __forceinline__ uint32_t ld_le32(const uint8_t* p) {
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) |
           (uint32_t(p[3]) << 24);
}
__device__ __forceinline__ uint64_t ld_le64(const uint8_t* p) {
    return uint64_t(ld_le32(p)) | (uint64_t(ld_le32(p + 4)) << 32);
}
__device__ __forceinline__ void st_le32(uint8_t* p, uint32_t v) {
    p[0] = uint8_t(v);
    p[1] = uint8_t(v >> 8);
    p[2] = uint8_t(v >> 16);
    p[3] = uint8_t(v >> 24);
}

// Warp-cooperative copy of `len` bytes from a 16-byte-aligned source to an
// arbitrary destination: byte head up to 16-byte alignment, realigned 128-bit
// body stores (funnel shift of two aligned 128-bit loads), byte tail.
// Source bytes up to 16 past `len` may be read (callers pad their buffers).
__device__ __forceinline__ void warp_copy_realign(uint8_t* __restrict__ dst,
                                                  const uint8_t* __restrict__ src, uint64_t len,
                                                  uint32_t lane) {
    if (len == 0) return;
    const uint64_t mis = reinterpret_cast<uintptr_t>(dst) & 15u;
    uint64_t head = (16u - mis) & 15u;
    if (head > len) head = len;
    if (lane < head) dst[lane] = src[lane];
    const uint64_t body = (len - head) >> 4;
    const uint64_t done = head + (body << 4);
    if (body) {
        uint4* d16 = reinterpret_cast<uint4*>(dst + head);
        const uint4* s16 = reinterpret_cast<const uint4*>(src);
        const int h = static_cast<int>(head);  // source misalignment of every body word
        const int q = h >> 2, r = h & 3;
        for (uint64_t i = lane; i < body; i += 32) {
            const uint4 a = __ldg(s16 + i);
            if (h == 0) {
                d16[i] = a;
                continue;
            }
            const uint4 b = __ldg(s16 + i + 1);
            // select the 5 words starting at word q (q uniform per call), then
            // funnel-shift by r bytes: registers only, no local memory
            uint32_t y0, y1, y2, y3, y4;
            switch (q) {
                case 0: y0 = a.x; y1 = a.y; y2 = a.z; y3 = a.w; y4 = b.x; break;
                case 1: y0 = a.y; y1 = a.z; y2 = a.w; y3 = b.x; y4 = b.y; break;
                case 2: y0 = a.z; y1 = a.w; y2 = b.x; y3 = b.y; y4 = b.z; break;
                default: y0 = a.w; y1 = b.x; y2 = b.y; y3 = b.z; y4 = b.w; break;
            }
            uint4 o;
            o.x = __funnelshift_r(y0, y1, 8 * r);
            o.y = __funnelshift_r(y1, y2, 8 * r);
            o.z = __funnelshift_r(y2, y3, 8 * r);
            o.w = __funnelshift_r(y3, y4, 8 * r);
            d16[i] = o;
        }
    }
    for (uint64_t i = done + lane; i < len; i += 32) dst[i] = src[i];
}

}  // namespace plzgpu
