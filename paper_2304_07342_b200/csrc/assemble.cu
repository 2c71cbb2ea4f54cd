// assemble.cu — Kernel III: write the bit-exact PLZ1 image.
//
// Reference: deflate.cpp:10-36 (copy chunk k's payload to
// [payload_offsets[k], payload_offsets[k+1]) and its flags likewise) and
// format.cpp:75-104 (serialise header | payload_offsets | flag_offsets |
// flag_stream | payload_stream | tail, all little-endian), for every container
// of pipeline.cpp:88-99 back to back.
//
// Image geometry straight from Kernel II's u64 prefixes, no host round trip:
// containers 0..j-1 have no tail (only the final block can, partition.cpp:16)
// so container j starts at 26*j + 8*(g0 + j) + P64[g0] + F64[g0] with g0 its
// first chunk.
//
// The kernel is a copy at HBM speed, so it is organised around memory
// round trips:
//  * plz_assemble_tma_kernel (the default when a chunk's slices fit a warp's
//    8 KiB ring): TMA bulk copies stage up to 8 chunks ahead per warp in
//    shared memory, the warp writes them out with realigned 128-bit stores;
//  * plz_assemble_kernel (larger chunks, PLZGPU_ASM_TMA=0): one warp per
//    chunk, its two table entries (byte stores by 8 lanes), its
//    flag slice and payload slice (warp_copy2: every source byte of both
//    loaded before the first store, realigned 128-bit body stores); the next
//    chunk's prefixes are loaded while this chunk's data is in flight;
//  * the shard variant writes its table slices with one thread per aligned
//    4-byte image word (coalesced; straddling entries funnel-shifted).
// The header kernel (one thread per container) writes the 26-byte header,
// the tail and the image length, and flags 4-byte table overflow
// (scan.cpp:43-44).
#include <algorithm>

#include "common.cuh"

namespace plzgpu {
namespace {

// ------------------------------------------------------------ stream copies
// A chunk's flag slice and payload slice are copied by one warp as two jobs:
// a byte head up to the destination's 16-byte alignment, 128-bit body words
// realigned from two aligned source words (funnel shift; the shift is
// uniform per job, so the select is a uniform branch), a byte tail.  Every
// source byte of both jobs (up to 64 body words each) is loaded before the
// first store: one DRAM round trip per chunk instead of one per head, body
// iteration and tail of each slice.
struct Job {
    uint8_t* dst;        // any alignment
    const uint8_t* src;  // 16-byte aligned; readable up to 16 bytes past len
    uint32_t len, head, body, tail;
};

__device__ __forceinline__ Job make_job(uint8_t* dst, const uint8_t* src, uint32_t len) {
    Job j;
    j.dst = dst;
    j.src = src;
    j.len = len;
    const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(dst) & 15u);
    j.head = min((16u - mis) & 15u, len);
    j.body = (len - j.head) >> 4;
    j.tail = len - j.head - 16u * j.body;
    return j;
}

struct JobData {
    uint32_t hb, tb;  // this lane's head / tail byte
    uint4 a[2], b[2];  // body words lane and lane + 32: source words i and i + 1
};

__device__ __forceinline__ uint4 realign(const uint4& a, const uint4& b, uint32_t h) {
    if (h == 0) return a;
    uint32_t y0, y1, y2, y3, y4;
    switch (h >> 2) {
        case 0: y0 = a.x; y1 = a.y; y2 = a.z; y3 = a.w; y4 = b.x; break;
        case 1: y0 = a.y; y1 = a.z; y2 = a.w; y3 = b.x; y4 = b.y; break;
        case 2: y0 = a.z; y1 = a.w; y2 = b.x; y3 = b.y; y4 = b.z; break;
        default: y0 = a.w; y1 = b.x; y2 = b.y; y3 = b.z; y4 = b.w; break;
    }
    const uint32_t r = 8u * (h & 3u);
    uint4 o;
    o.x = __funnelshift_r(y0, y1, r);
    o.y = __funnelshift_r(y1, y2, r);
    o.z = __funnelshift_r(y2, y3, r);
    o.w = __funnelshift_r(y3, y4, r);
    return o;
}

__device__ __forceinline__ void load_job(const Job& j, JobData& d, uint32_t lane) {
    const uint4* s16 = reinterpret_cast<const uint4*>(j.src);
    d.hb = lane < j.head ? j.src[lane] : 0u;
    d.tb = lane < j.tail ? j.src[j.head + 16u * j.body + lane] : 0u;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const uint32_t i = lane + 32u * u;
        if (i < j.body) {
            d.a[u] = __ldg(s16 + i);
            if (j.head) d.b[u] = __ldg(s16 + i + 1);
        }
    }
}

__device__ __forceinline__ void store_job(const Job& j, const JobData& d, uint32_t lane) {
    if (lane < j.head) j.dst[lane] = uint8_t(d.hb);
    uint4* d16 = reinterpret_cast<uint4*>(j.dst + j.head);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
        const uint32_t i = lane + 32u * u;
        if (i < j.body) d16[i] = realign(d.a[u], d.b[u], j.head);
    }
    const uint4* s16 = reinterpret_cast<const uint4*>(j.src);
    for (uint32_t i = lane + 64u; i < j.body; i += 32u)  // bodies past 1 KiB
        d16[i] = realign(__ldg(s16 + i), j.head ? __ldg(s16 + i + 1) : make_uint4(0, 0, 0, 0), j.head);
    if (lane < j.tail) j.dst[j.head + 16u * j.body + lane] = uint8_t(d.tb);
}

__device__ __forceinline__ void warp_copy2(const Job& j0, const Job& j1, uint32_t lane) {
    JobData d0, d1;
    load_job(j0, d0, lane);
    load_job(j1, d1, lane);
    store_job(j0, d0, lane);
    store_job(j1, d1, lane);
}

// ------------------------------------------------------------ offset tables
// Entry i (u32, little-endian) of a table region lands at region + 4i; the
// thread owning aligned image word W composes it from entries e - 1 and e.
template <typename EntryFn>
__device__ __forceinline__ void table_word(uint8_t* region, uint64_t n_entries, uint64_t wi,
                                           EntryFn entry) {
    const uint32_t m = uint32_t(reinterpret_cast<uintptr_t>(region) & 3u);
    uint8_t* at = region - m + 4 * wi;               // aligned word
    const int64_t rel = int64_t(4 * wi) - int64_t(m);  // region byte of its first byte
    const int64_t bytes = int64_t(4 * n_entries);
    uint32_t v;
    if (m == 0) {
        v = entry(wi);
    } else {
        const int64_t e = (rel + 4) >> 2;  // entry holding the word's last bytes
        const uint32_t lo = e >= 1 ? entry(uint64_t(e - 1)) : 0u;
        const uint32_t hi = e < int64_t(n_entries) ? entry(uint64_t(e)) : 0u;
        v = __funnelshift_r(lo, hi, 8u * (4u - m));
    }
    if (rel >= 0 && rel + 4 <= bytes) {
        *reinterpret_cast<uint32_t*>(at) = v;
    } else {
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if (rel + b >= 0 && rel + b < bytes) at[b] = uint8_t(v >> (8 * b));
    }
}

__device__ __forceinline__ uint64_t table_words(const uint8_t* region, uint64_t n_entries) {
    return (uint64_t(reinterpret_cast<uintptr_t>(region) & 3u) + 4 * n_entries + 3) >> 2;
}

// ------------------------------------------------------------------ geometry
struct Geo {
    uint64_t j, g0, n;  // container, its first chunk, its chunk count
};

__device__ __forceinline__ Geo locate(const AssembleArgs& a, uint64_t g) {
    Geo r;
    r.j = g / a.cpb;
    r.g0 = r.j * a.cpb;
    r.n = (r.j + 1 == a.n_blocks) ? a.n_chunks - r.g0 : a.cpb;
    return r;
}

__device__ __forceinline__ uint64_t container_start(const AssembleArgs& a, uint64_t j,
                                                    uint64_t g0) {
    return 26u * j + 8u * (g0 + j) + a.P64[g0] + a.F64[g0];
}

__global__ void __launch_bounds__(128) plz_assemble_kernel(AssembleArgs a) {
    const uint32_t lane = lane_id();
    const uint64_t j_hi = a.j_hi ? a.j_hi : a.n_blocks;
    const uint64_t C = uint64_t(a.C), S = uint64_t(a.S);
    const uint64_t g_lo = a.j_lo * a.cpb;
    const uint64_t g_hi = min(a.n_chunks, j_hi * a.cpb);
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    uint64_t g = g_lo + uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (g >= g_hi) return;
    // per-chunk prefixes and sizes, loaded one chunk ahead
    uint64_t pg = a.P64[g], fg = a.F64[g];
    uint32_t ps = a.psize[g], fs = a.fsize[g];
    uint64_t cj = ~0ull, g0 = 0, n = 0, tabs = 0, pb = 0, fb = 0, ftot = 0;
    for (; g < g_hi; g += warps) {
        const uint64_t gn = g + warps;
        uint64_t pg_n = 0, fg_n = 0;
        uint32_t ps_n = 0, fs_n = 0;
        if (gn < g_hi) {
            pg_n = a.P64[gn];
            fg_n = a.F64[gn];
            ps_n = a.psize[gn];
            fs_n = a.fsize[gn];
        }
        if (cj == ~0ull || g - g0 >= n) {  // container constants, cached while the warp stays in it
            const Geo c = locate(a, g);     // (a 64-bit division)
            cj = c.j;
            g0 = c.g0;
            n = c.n;
            pb = a.P64[g0];
            fb = a.F64[g0];
            ftot = a.F64[g0 + n] - fb;
            tabs = container_start(a, cj, g0) + 26;
        }
        const uint64_t pk = pg - pb, fk = fg - fb, k = g - g0;
        const uint64_t streams = tabs + 8 * (n + 1);
        const Job jf = make_job(a.img + streams + fk, a.flag_slots + g * (C / 8), fs);
        const Job jp = make_job(a.img + streams + ftot + pk, a.pay_slots + g * C * S, ps);
        JobData df, dp;
        load_job(jf, df, lane);
        load_job(jp, dp, lane);
        // table entries k (the header kernel writes entry n)
        if (lane < 4) {
            a.img[tabs + 4 * k + lane] = uint8_t(pk >> (8 * lane));
        } else if (lane < 8) {
            a.img[tabs + 4 * (n + 1) + 4 * k + (lane - 4)] = uint8_t(fk >> (8 * (lane - 4)));
        }
        store_job(jf, df, lane);
        store_job(jp, dp, lane);
        pg = pg_n;
        fg = fg_n;
        ps = ps_n;
        fs = fs_n;
    }
}

// ------------------------------------------------- TMA-staged Kernel III
// plz_assemble_tma_kernel: the same image bytes as plz_assemble_kernel, with
// the loads taken off the registers.  Each warp owns a shared-memory ring
// (kAsmRing bytes, kAsmSlots mbarriers) and walks its chunks g, g + warps,
// ...: lane 0 keeps up to kAsmSlots chunks' flag and payload slices in
// flight as TMA bulk copies (cp.async.bulk, 16-byte rounded, each chunk at
// the ring's next free 16-byte offset; an allocation that would run past
// the ring's end starts at 0, and an empty ring restarts at 0), while the warp writes the oldest
// staged chunk out — byte head to the destination's 16-byte alignment,
// 128-bit body stores realigned from two aligned shared words, byte tail —
// and its two table entries.  Per-chunk sizes and prefixes come 32 chunks at
// a time, one chunk per lane, a batch ahead.  Chunks whose slices exceed the
// ring (C*S + C/8 + 32 > kAsmRing) take plz_assemble_kernel.
// 8 KiB rings: ~24 warps/SM (c5: 1.04 ms, DRAM 48 %; 16 KiB rings with 16
// slots gave 12 warps/SM and 1.32 ms, the register-staged kernel 1.30 ms)
constexpr int kAsmWarps = 4;
constexpr uint32_t kAsmRing = 8192;
constexpr uint32_t kAsmSlots = 8;
constexpr uint32_t kAsmWarpSmem = kAsmRing + 8 * kAsmSlots;

struct AsmMeta {  // one chunk per lane
    uint64_t P, F;
    uint32_t ps, fs;
};

__device__ __forceinline__ AsmMeta load_meta(const AssembleArgs& a, uint64_t g, uint64_t g_hi) {
    AsmMeta m{0, 0, 0, 0};
    if (g < g_hi) {
        m.P = a.P64[g];
        m.F = a.F64[g];
        m.ps = a.psize[g];
        m.fs = a.fsize[g];
    }
    return m;
}

__host__ __device__ __forceinline__ uint32_t r16(uint32_t x) { return (x + 15u) & ~15u; }

__device__ __forceinline__ uint32_t lds_w(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_b(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// Warp copy of len bytes from shared memory (shared-window address src) to
// dst: byte head to dst's 16-byte alignment, 128-bit body stores each built
// from five aligned 4-byte shared loads and four funnel shifts, byte tail.
__device__ __forceinline__ void smem_copy_out(uint8_t* dst, uint32_t src, uint32_t len,
                                              uint32_t lane) {
    const uint32_t mis = uint32_t(reinterpret_cast<uintptr_t>(dst) & 15u);
    const uint32_t head = min((16u - mis) & 15u, len);
    const uint32_t body = (len - head) >> 4;
    const uint32_t tail = len - head - 16u * body;
    if (lane < head) dst[lane] = uint8_t(lds_b(src + lane));
    uint4* d16 = reinterpret_cast<uint4*>(dst + head);
    const uint32_t r = 8u * (head & 3u);
    uint32_t b = src + (head & ~3u) + 16u * lane;
    for (uint32_t i = lane; i < body; i += 32u, b += 512u) {
        const uint32_t w0 = lds_w(b), w1 = lds_w(b + 4), w2 = lds_w(b + 8), w3 = lds_w(b + 12),
                       w4 = lds_w(b + 16);
        d16[i] = make_uint4(__funnelshift_r(w0, w1, r), __funnelshift_r(w1, w2, r),
                            __funnelshift_r(w2, w3, r), __funnelshift_r(w3, w4, r));
    }
    const uint32_t t0 = head + 16u * body;
    if (lane < tail) dst[t0 + lane] = uint8_t(lds_b(src + t0 + lane));
}

__global__ void __launch_bounds__(kAsmWarps * 32) plz_assemble_tma_kernel(AssembleArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    uint8_t* ring = smem + size_t(warp) * kAsmWarpSmem;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(ring + kAsmRing);
    const uint32_t s_ring = static_cast<uint32_t>(__cvta_generic_to_shared(ring));
    const uint64_t j_hi = a.j_hi ? a.j_hi : a.n_blocks;
    const uint64_t C = uint64_t(a.C), S = uint64_t(a.S);
    const uint64_t g_lo = a.j_lo * a.cpb;
    const uint64_t g_hi = min(a.n_chunks, j_hi * a.cpb);
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint64_t g_first = g_lo + uint64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
    if (g_first >= g_hi) return;
    const uint64_t K = (g_hi - g_first + warps - 1) / warps;  // this warp's chunks
    if (lane < kAsmSlots) mbar_init(&mbar[lane], 1);
    __syncwarp();
    // metadata of sequence entries [32b, 32b + 32): cur = the consumer's batch
    AsmMeta cur = load_meta(a, g_first + warps * lane, g_hi);
    AsmMeta nxt = load_meta(a, g_first + warps * (32u + lane), g_hi);
    uint64_t k_issue = 0, k_done = 0;
    uint32_t wr = 0, rd = 0, infl = 0;
    uint64_t cj = ~0ull, g0 = 0, n = 0, tabs = 0, pb = 0, fb = 0, ftot = 0;
    while (k_done < K) {
        // ---- producer: stage chunks ahead while slots and ring space last
        while (k_issue < K && k_issue - k_done < kAsmSlots) {
            const bool in_cur = (k_issue >> 5) == (k_done >> 5);
            const uint32_t src_lane = uint32_t(k_issue & 31u);
            const uint32_t ps = __shfl_sync(0xffffffffu, in_cur ? cur.ps : nxt.ps, src_lane);
            const uint32_t fs = __shfl_sync(0xffffffffu, in_cur ? cur.fs : nxt.fs, src_lane);
            const uint32_t need = r16(fs) + r16(ps);
            const bool wrap = wr + need > kAsmRing;  // the rest of the ring is skipped
            const uint32_t waste = wrap ? kAsmRing - wr : 0u;
            if (infl + waste + need > kAsmRing) break;
            const uint32_t at = wrap ? 0u : wr;
            const uint64_t g = g_first + warps * k_issue;
            fence_proxy_async_smem();  // this warp's earlier reads of the ring before the TMA writes
            __syncwarp();
            if (lane == 0) {
                uint64_t* mb = &mbar[k_issue % kAsmSlots];
                const uint32_t m = static_cast<uint32_t>(__cvta_generic_to_shared(mb));
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(m),
                             "r"(need) : "memory");
                const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(ring + at));
                if (fs)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                        "l"(a.flag_slots + g * (C / 8)), "r"(r16(fs)), "r"(m) : "memory");
                if (ps)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d + r16(fs)),
                        "l"(a.pay_slots + g * C * S), "r"(r16(ps)), "r"(m) : "memory");
            }
            wr = at + need;
            infl += waste + need;
            ++k_issue;
        }
        // ---- consumer: write the oldest staged chunk out
        const uint32_t src_lane = uint32_t(k_done & 31u);
        const uint64_t pg = __shfl_sync(0xffffffffu, cur.P, src_lane);
        const uint64_t fg = __shfl_sync(0xffffffffu, cur.F, src_lane);
        const uint32_t ps = __shfl_sync(0xffffffffu, cur.ps, src_lane);
        const uint32_t fs = __shfl_sync(0xffffffffu, cur.fs, src_lane);
        const uint32_t need = r16(fs) + r16(ps);
        const bool wrap = rd + need > kAsmRing;  // the producer's allocation, replayed
        const uint32_t waste = wrap ? kAsmRing - rd : 0u;
        const uint32_t at = wrap ? 0u : rd;
        const uint64_t g = g_first + warps * k_done;
        if (cj == ~0ull || g - g0 >= n) {  // container constants, cached while the warp stays in it
            const Geo c = locate(a, g);     // (a 64-bit division)
            cj = c.j;
            g0 = c.g0;
            n = c.n;
            pb = a.P64[g0];
            fb = a.F64[g0];
            ftot = a.F64[g0 + n] - fb;
            tabs = container_start(a, cj, g0) + 26;
        }
        const uint64_t pk = pg - pb, fk = fg - fb, k = g - g0;
        const uint64_t streams = tabs + 8 * (n + 1);
        if (lane < 4) {
            a.img[tabs + 4 * k + lane] = uint8_t(pk >> (8 * lane));
        } else if (lane < 8) {
            a.img[tabs + 4 * (n + 1) + 4 * k + (lane - 4)] = uint8_t(fk >> (8 * (lane - 4)));
        }
        mbar_wait(&mbar[k_done % kAsmSlots], uint32_t(k_done / kAsmSlots) & 1u);
        smem_copy_out(a.img + streams + fk, s_ring + at, fs, lane);
        smem_copy_out(a.img + streams + ftot + pk, s_ring + at + r16(fs), ps, lane);
        __syncwarp();
        rd = at + need;
        infl -= waste + need;
        if (infl == 0) wr = rd = 0;  // ring empty: restart at 0 (so any chunk <= kAsmRing fits)
        ++k_done;
        if ((k_done & 31u) == 0u) {  // next batch of metadata
            cur = nxt;
            nxt = load_meta(a, g_first + warps * (k_done + 32u + lane), g_hi);
        }
    }
}

// ------------------------------------------------- batched Kernel III
// plz_assemble_batch_kernel: the same image bytes, with the per-chunk
// bookkeeping done once per run of 32 consecutive chunks, one chunk per
// lane: each lane finds its chunk's container (header geometry, stream
// offsets), writes its two table entries and computes both destinations; a
// warp scan of the staged sizes cuts the run into batches (chunk c joins
// batch floor(excl_c / kAbSplit), so a batch spans at most kAbSplit plus one
// chunk's slices) and each batch is staged by one TMA bulk copy per slice,
// issued by the chunk's own lane on the buffer's mbarrier, then written out
// chunk by chunk (byte head + tail in one predicated pass, 128-bit body
// stores realigned from two aligned 16-byte shared loads).  One buffer per
// warp: the other warps of the SM cover a batch's TMA latency (two buffers,
// batch b + 1 in flight while b is written, fitted fewer warps and measured
// 6 % slower).  The next run's metadata is loaded while this run is written.
constexpr int kAbWarps = 4;
constexpr uint32_t kAbSplit = 4096;  // c5: 2048 / 4096 / 6144 / 8192 -> 0.70 / 0.685 / 0.685 / 0.74 ms
constexpr uint32_t kAbMaxSlices = 4608;  // C*S <= 4 KiB: + C/8 <= 512 B
// a buffer holds kAbSplit + one chunk's largest slices (sized per launch)
constexpr uint32_t kAbBufs = 1;  // staging buffers per warp (2: the next batch in flight)
__host__ __device__ __forceinline__ uint32_t ab_warp_smem(uint32_t buf) { return kAbBufs * buf + 16; }
constexpr uint64_t kAbMinChunks = 1ull << 14;  // below: the TMA ring kernel (c1's 4 Ki chunks: 30 vs 7.5 us;
                                               // c2 / c3 (82 Ki / 64 Ki): 36 / 30 vs 47 / 36 us)

struct AbChunk {  // one chunk per lane
    uint64_t P, F;
    uint32_t ps, fs;
};

__device__ __forceinline__ AbChunk ab_load(const AssembleArgs& a, uint64_t g, uint64_t g_hi) {
    AbChunk m{0, 0, 0, 0};
    if (g < g_hi) {
        m.P = a.P64[g];
        m.F = a.F64[g];
        m.ps = a.psize[g];
        m.fs = a.fsize[g];
    }
    return m;
}

// Warp copy of one staged slice: byte head to dst's 16-byte alignment and
// byte tail in one predicated pass (lanes 0-15 head, 16-31 tail), then the
// body as realigned 128-bit stores.
__device__ __forceinline__ void ab_copy(uint8_t* dst, uint32_t src, uint32_t len, uint32_t lane) {
    const uint32_t head = min((16u - uint32_t(reinterpret_cast<uintptr_t>(dst) & 15u)) & 15u, len);
    const uint32_t body = (len - head) >> 4;
    const uint32_t tail = len - head - 16u * body;
    const uint32_t jb = lane & 15u;
    const uint32_t o = lane < 16u ? jb : head + 16u * body + jb;
    if (jb < (lane < 16u ? head : tail)) dst[o] = uint8_t(lds_b(src + o));
    // body word i = source bytes [head + 16 i, +16): two aligned 16-byte
    // shared loads, the five words from (head >> 2) on (uniform per slice),
    // funnel-shifted by head & 3 bytes
    uint4* d16 = reinterpret_cast<uint4*>(dst + head);
    uint32_t b = src + 16u * lane;
    for (uint32_t i = lane; i < body; i += 32u, b += 512u) {
        uint4 x, y;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "r"(b));
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(y.x), "=r"(y.y), "=r"(y.z), "=r"(y.w) : "r"(b + 16));
        d16[i] = realign(x, y, head);
    }
}

__global__ void __launch_bounds__(kAbWarps * 32) plz_assemble_batch_kernel(AssembleArgs a, uint32_t buf_bytes) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    uint8_t* wbase = smem + size_t(warp) * ab_warp_smem(buf_bytes);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(wbase + kAbBufs * buf_bytes);
    const uint32_t s_buf = static_cast<uint32_t>(__cvta_generic_to_shared(wbase));
    const uint64_t j_hi = a.j_hi ? a.j_hi : a.n_blocks;
    const uint64_t C = uint64_t(a.C), S = uint64_t(a.S);
    const uint64_t g_lo = a.j_lo * a.cpb;
    const uint64_t g_hi = min(a.n_chunks, j_hi * a.cpb);
    const uint64_t n_runs = (g_hi - g_lo + 31) / 32;
    const uint64_t warps = uint64_t(gridDim.x) * kAbWarps;
    uint64_t r = uint64_t(blockIdx.x) * kAbWarps + warp;
    if (r >= n_runs) return;
    if (lane < 2) mbar_init(&mbar[lane], 1);
    __syncwarp();
    uint32_t phase = 0;  // bit i: parity of buffer i's next completion
    uint32_t issued = 0; // batches issued so far (buffer = issued & 1)
    AbChunk cur = ab_load(a, g_lo + 32 * r + lane, g_hi);
    for (; r < n_runs; r += warps) {
        const uint64_t g = g_lo + 32 * r + lane;
        const bool live = g < g_hi;
        AbChunk nxt = ab_load(a, g_lo + 32 * (r + warps) + lane, g_hi);
        // ---- per-lane geometry: container, table entries, destinations
        uint8_t* dst_f = a.img;
        uint8_t* dst_p = a.img;
        if (live) {
            const uint64_t j = g / a.cpb;
            const uint64_t g0 = j * a.cpb;
            const uint64_t n = (j + 1 == a.n_blocks) ? a.n_chunks - g0 : a.cpb;
            const uint64_t pb = a.P64[g0], fb = a.F64[g0];
            const uint64_t ftot = a.F64[g0 + n] - fb;
            const uint64_t tabs = 26u * j + 8u * (g0 + j) + pb + fb + 26u;
            const uint64_t k = g - g0;
            const uint32_t pk = uint32_t(cur.P - pb), fk = uint32_t(cur.F - fb);
            uint8_t* tp = a.img + tabs + 4 * k;
            uint8_t* tf = a.img + tabs + 4 * (n + 1) + 4 * k;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                tp[b] = uint8_t(pk >> (8 * b));
                tf[b] = uint8_t(fk >> (8 * b));
            }
            const uint64_t streams = tabs + 8 * (n + 1);
            dst_f = a.img + streams + (cur.F - fb);
            dst_p = a.img + streams + ftot + (cur.P - pb);
        }
        // ---- batches: exclusive scan of the staged sizes
        const uint32_t z = live ? r16(cur.fs) + r16(cur.ps) : 0u;
        uint32_t incl = z;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t x = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= uint32_t(d)) incl += x;
        }
        const uint32_t excl = incl - z;
        // batch of chunk c: floor(excl_c / kAbSplit); batch values only grow
        // with c but may skip one (a chunk larger than kAbSplit)
        const uint32_t bat = live ? excl / kAbSplit : 0xffffffffu;
        auto issue = [&](uint32_t bv) {  // returns the buffer
            const uint32_t m = __ballot_sync(0xffffffffu, bat == bv);
            const uint32_t c0 = __ffs(m) - 1, c1 = 31 - __clz(m);
            const uint32_t base = __shfl_sync(0xffffffffu, excl, c0);
            const uint32_t total = __shfl_sync(0xffffffffu, incl, c1) - base;
            const uint32_t buf = kAbBufs == 2 ? issued & 1u : 0u;
            const uint32_t s_mb = static_cast<uint32_t>(__cvta_generic_to_shared(&mbar[buf]));
            fence_proxy_async_smem();  // earlier reads of this buffer before the TMA writes
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_mb),
                             "r"(total) : "memory");
            __syncwarp();
            if (bat == bv) {
                const uint32_t d = s_buf + buf * buf_bytes + (excl - base);
                if (cur.fs)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                        "l"(a.flag_slots + g * (C / 8)), "r"(r16(cur.fs)), "r"(s_mb) : "memory");
                if (cur.ps)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d + r16(cur.fs)),
                        "l"(a.pay_slots + g * C * S), "r"(r16(cur.ps)), "r"(s_mb) : "memory");
            }
            ++issued;
            return buf;
        };
        uint32_t bv = __shfl_sync(0xffffffffu, bat, 0);  // lane 0 is always live
        uint32_t buf = issue(bv);
        for (;;) {
            const uint32_t bn = __reduce_min_sync(0xffffffffu, bat > bv ? bat : 0xffffffffu);
            const uint32_t buf_n = kAbBufs == 2 && bn != 0xffffffffu ? issue(bn) : 0u;
            mbar_wait(&mbar[buf], (phase >> buf) & 1u);
            phase ^= 1u << buf;
            uint32_t m = __ballot_sync(0xffffffffu, bat == bv);
            const uint32_t base = __shfl_sync(0xffffffffu, excl, __ffs(m) - 1);
            while (m) {
                const uint32_t c = __ffs(m) - 1;
                m &= m - 1;
                uint8_t* df = reinterpret_cast<uint8_t*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst_f), c));
                uint8_t* dp = reinterpret_cast<uint8_t*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst_p), c));
                const uint32_t fs = __shfl_sync(0xffffffffu, cur.fs, c);
                const uint32_t ps = __shfl_sync(0xffffffffu, cur.ps, c);
                const uint32_t src = s_buf + buf * buf_bytes + __shfl_sync(0xffffffffu, excl, c) - base;
                ab_copy(df, src, fs, lane);
                ab_copy(dp, src + r16(fs), ps, lane);
            }
            __syncwarp();
            if (bn == 0xffffffffu) break;
            bv = bn;
            buf = kAbBufs == 2 ? buf_n : issue(bn);
        }
        cur = nxt;
    }
}

__global__ void plz_headers_kernel(AssembleArgs a) {
    const uint64_t j = a.j_lo + uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= (a.j_hi ? a.j_hi : a.n_blocks)) return;
    const uint64_t g0 = j * a.cpb;
    const uint64_t n = (j + 1 == a.n_blocks) ? a.n_chunks - g0 : a.cpb;
    const uint64_t pb = a.P64[g0], fb = a.F64[g0];
    const uint64_t ptot = a.P64[g0 + n] - pb, ftot = a.F64[g0 + n] - fb;
    if (ptot > 0xffffffffull || ftot > 0xffffffffull) atomicExch(a.overflow, 1u);
    const uint64_t byte_len = (j + 1 == a.n_blocks) ? a.n_bytes - j * a.block_bytes : a.block_bytes;
    const uint32_t tail = uint32_t(byte_len % uint64_t(a.S));
    const uint64_t img0 = container_start(a, j, g0);
    uint8_t* h = a.img + img0;
    h[0] = 'P'; h[1] = 'L'; h[2] = 'Z'; h[3] = '1';
    h[4] = 1;  // format version
    h[5] = uint8_t(a.S);
    h[6] = uint8_t(a.W);
    h[7] = uint8_t(a.I);
    h[8] = 0;  // reserved
    st_le32(h + 9, uint32_t(a.C));
    st_le32(h + 13, uint32_t(byte_len));
    st_le32(h + 17, uint32_t(byte_len >> 32));
    st_le32(h + 21, uint32_t(n));
    h[25] = uint8_t(tail);
    // the final table entries (also written by Kernel III's table pass, which
    // does not run for an input without chunks)
    st_le32(h + 26 + 4 * n, uint32_t(ptot));
    st_le32(h + 26 + 4 * (n + 1) + 4 * n, uint32_t(ftot));
    uint8_t* t = h + 26 + 8 * (n + 1) + ftot + ptot;
    const uint8_t* src = a.in + j * a.block_bytes + byte_len - tail;
    for (uint32_t i = 0; i < tail; ++i) t[i] = src[i];
    if (j + 1 == a.n_blocks) *a.img_len = img0 + 26 + 8 * (n + 1) + ftot + ptot + tail;
}

// Shard variant of Kernel III (multi-GPU): the same table
// words and chunk copies, into a local segment buffer (or straight into the
// root's image) with offsets rebased by the shard's position inside each
// container's streams.
__device__ __forceinline__ uint64_t find_cont(const ShardAssembleArgs& a, uint64_t g) {
    uint64_t c = 0;
    while (c + 1 < a.n_conts && a.conts[c + 1].g_lo <= g) ++c;
    return c;
}

__global__ void __launch_bounds__(256, 4) plz_shard_assemble_kernel(ShardAssembleArgs a) {
    const uint32_t lane = lane_id();
    // ---- table slices: per touched container, its payload-table slice then
    // its flag-table slice, g_hi - g_lo entries each
    {
        uint64_t total = 0;
        for (uint64_t c = 0; c < a.n_conts; ++c) {
            const uint64_t m = a.conts[c].g_hi - a.conts[c].g_lo;
            total += table_words(a.out + a.conts[c].seg_ptab, m) +
                     table_words(a.out + a.conts[c].seg_ftab, m);
        }
        for (uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
             idx += uint64_t(gridDim.x) * blockDim.x) {
            uint64_t rest = idx;
            for (uint64_t c = 0; c < a.n_conts; ++c) {
                const ShardCont& d = a.conts[c];
                const uint64_t m = d.g_hi - d.g_lo;
                uint8_t* rp = a.out + d.seg_ptab;
                uint8_t* rf = a.out + d.seg_ftab;
                const uint64_t wp = table_words(rp, m), wf = table_words(rf, m);
                if (rest < wp) {
                    const uint64_t p0 = a.P64[d.g_lo];
                    table_word(rp, m, rest, [&](uint64_t e) {
                        return uint32_t(d.p_base + a.P64[d.g_lo + e] - p0);
                    });
                    break;
                }
                rest -= wp;
                if (rest < wf) {
                    const uint64_t f0 = a.F64[d.g_lo];
                    table_word(rf, m, rest, [&](uint64_t e) {
                        return uint32_t(d.f_base + a.F64[d.g_lo + e] - f0);
                    });
                    break;
                }
                rest -= wf;
            }
        }
    }
    // ---- streams
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint64_t C = uint64_t(a.C), S = uint64_t(a.S);
    for (uint64_t g = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         g < a.n_chunks; g += warps) {
        const ShardCont& d = a.conts[find_cont(a, g)];
        const uint64_t lp = a.P64[g] - a.P64[d.g_lo], lf = a.F64[g] - a.F64[d.g_lo];
        const uint64_t pk = d.p_base + lp, fk = d.f_base + lf;
        if (lane == 0 && (pk > 0xffffffffull || fk > 0xffffffffull)) atomicExch(a.overflow, 1u);
        const Job jf = make_job(a.out + d.seg_flags + lf, a.flag_slots + g * (C / 8), a.fsize[g]);
        const Job jp = make_job(a.out + d.seg_pay + lp, a.pay_slots + g * C * S, a.psize[g]);
        warp_copy2(jf, jp, lane);
    }
}

__global__ void plz_shard_headers_kernel(const HeaderDesc* descs, uint64_t n_conts, uint8_t* img,
                                         int S, int W, int I, int C) {
    const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_conts) return;
    const HeaderDesc d = descs[j];
    uint8_t* h = img + d.img_off;
    h[0] = 'P'; h[1] = 'L'; h[2] = 'Z'; h[3] = '1';
    h[4] = 1;
    h[5] = uint8_t(S);
    h[6] = uint8_t(W);
    h[7] = uint8_t(I);
    h[8] = 0;
    st_le32(h + 9, uint32_t(C));
    st_le32(h + 13, uint32_t(d.byte_len));
    st_le32(h + 17, uint32_t(d.byte_len >> 32));
    st_le32(h + 21, d.n);
    h[25] = d.tail_len;
    const uint64_t n = d.n;
    st_le32(h + 26 + 4 * n, uint32_t(d.ptot));
    st_le32(h + 26 + 4 * (n + 1) + 4 * n, uint32_t(d.ftot));
    uint8_t* t = h + 26 + 8 * (n + 1) + d.ftot + d.ptot;
    for (uint32_t i = 0; i < d.tail_len; ++i) t[i] = d.tail[i];
}

}  // namespace

void launch_shard_assemble(const ShardAssembleArgs& a, cudaStream_t st) {
    if (a.n_chunks == 0) return;
    uint64_t blocks = (a.n_chunks + 7) / 8;
    if (blocks > 148ull * 8) blocks = 148ull * 8;
    plz_shard_assemble_kernel<<<unsigned(blocks), 256, 0, st>>>(a);
}

void launch_shard_headers(const HeaderDesc* d, uint64_t n_conts, uint8_t* img, int S, int W, int I,
                          int C, cudaStream_t st) {
    if (n_conts == 0) return;
    plz_shard_headers_kernel<<<unsigned((n_conts + 127) / 128), 128, 0, st>>>(d, n_conts, img, S, W,
                                                                              I, C);
}

void launch_assemble(const AssembleArgs& a, cudaStream_t st) {
    if (a.n_chunks == 0) return;
    const uint64_t g_lo = a.j_lo * a.cpb;
    const uint64_t g_hi = a.j_hi ? std::min(a.n_chunks, a.j_hi * a.cpb) : a.n_chunks;
    const uint64_t warps_needed = g_hi - g_lo;
    const uint64_t slices = uint64_t(a.C) * a.S + a.C / 8 + 32;
    const int mode = assemble_mode();
    // batched runs need enough of them to fill the GPU (c5: 65k runs; c1's
    // 128 runs took 30 us against the ring's 7.5 us)
    const uint32_t ab_slices = r16(uint32_t(a.C) * a.S) + r16(uint32_t(a.C) / 8);
    if (mode >= 2 && warps_needed >= kAbMinChunks && ab_slices <= kAbMaxSlices) {
        const uint32_t buf = kAbSplit + ab_slices;
        const size_t smem = size_t(kAbWarps) * ab_warp_smem(buf);
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, plz_assemble_batch_kernel,
                                                      kAbWarps * 32, smem);
        if (per_sm < 1) per_sm = 1;
        int sms = 148;
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const uint64_t runs = (warps_needed + 31) / 32;
        uint64_t blocks = (runs + kAbWarps - 1) / kAbWarps;
        blocks = std::min<uint64_t>(blocks, uint64_t(sms) * per_sm);
        plz_assemble_batch_kernel<<<unsigned(blocks), kAbWarps * 32, smem, st>>>(a, buf);
        return;
    }
    if (mode >= 1 && slices <= kAsmRing) {
        static int per_sm = -1;  // same answer on every B200; computed once
        const size_t smem = size_t(kAsmWarps) * kAsmWarpSmem;
        if (per_sm < 0) {
            int blocks = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, plz_assemble_tma_kernel,
                                                          kAsmWarps * 32, smem);
            per_sm = blocks > 0 ? blocks : 1;
        }
        int sms = 148;
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        uint64_t blocks = (warps_needed + kAsmWarps - 1) / kAsmWarps;
        blocks = std::min<uint64_t>(blocks, uint64_t(sms) * per_sm);
        plz_assemble_tma_kernel<<<unsigned(blocks), kAsmWarps * 32, smem, st>>>(a);
        return;
    }
    uint64_t blocks = (warps_needed + 3) / 4;
    if (blocks > 148ull * 10) blocks = 148ull * 10;
    plz_assemble_kernel<<<unsigned(blocks), 128, 0, st>>>(a);
}

void launch_headers(const AssembleArgs& a, cudaStream_t st) {
    const uint64_t nj = (a.j_hi ? a.j_hi : a.n_blocks) - a.j_lo;
    if (nj == 0) return;
    plz_headers_kernel<<<unsigned((nj + 127) / 128), 128, 0, st>>>(a);
}

void preload_assemble_kernels() {
    preload_kernel(reinterpret_cast<const void*>(plz_assemble_kernel));
    preload_kernel(reinterpret_cast<const void*>(plz_assemble_tma_kernel));
    preload_kernel(reinterpret_cast<const void*>(plz_assemble_batch_kernel));
    preload_kernel(reinterpret_cast<const void*>(plz_headers_kernel));
    preload_kernel(reinterpret_cast<const void*>(plz_shard_assemble_kernel));
    preload_kernel(reinterpret_cast<const void*>(plz_shard_headers_kernel));
}

}  // namespace plzgpu
