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
//  * offset tables: one thread per aligned 4-byte image word (coalesced
//    32-bit stores; an entry straddling two words is funnel-shifted from its
//    neighbours; the region's two edge words are written bytewise);
//  * streams: one warp per chunk, its flag slice and payload slice copied as
//    one job list — every source word the chunk needs is loaded before the
//    first store (one DRAM round trip per chunk, not one per head / body /
//    tail), realigned to the destination with funnel shifts and stored as
//    aligned 128-bit words (edge words bytewise); the next chunk's prefixes
//    are loaded while this chunk's data is in flight.
// The header kernel (one thread per container) writes the 26-byte header,
// the tail and the image length, and flags 4-byte table overflow
// (scan.cpp:43-44).
#include <algorithm>

#include "common.cuh"

namespace plzgpu {
namespace {

// ------------------------------------------------------------ stream copies
struct Job {
    uint8_t* dst;        // any alignment
    const uint8_t* src;  // 16-byte aligned; readable up to 16 bytes past len
    uint32_t len;
};

__device__ __forceinline__ uint32_t job_words(const Job& j) {
    return j.len ? ((uint32_t(reinterpret_cast<uintptr_t>(j.dst) & 15u) + j.len + 15u) >> 4) : 0u;
}

// 128-bit funnel shift: bytes [r, r + 16) of the 32-byte value (hi:lo), r in 0..15
__device__ __forceinline__ uint4 funnel128(const uint4& lo, const uint4& hi, uint32_t r) {
    const uint32_t q = r >> 2, s = 8u * (r & 3u);
    uint32_t y0, y1, y2, y3, y4;
    switch (q) {
        case 0: y0 = lo.x; y1 = lo.y; y2 = lo.z; y3 = lo.w; y4 = hi.x; break;
        case 1: y0 = lo.y; y1 = lo.z; y2 = lo.w; y3 = hi.x; y4 = hi.y; break;
        case 2: y0 = lo.z; y1 = lo.w; y2 = hi.x; y3 = hi.y; y4 = hi.z; break;
        default: y0 = lo.w; y1 = hi.x; y2 = hi.y; y3 = hi.z; y4 = hi.w; break;
    }
    uint4 o;
    o.x = __funnelshift_r(y0, y1, s);
    o.y = __funnelshift_r(y1, y2, s);
    o.z = __funnelshift_r(y2, y3, s);
    o.w = __funnelshift_r(y3, y4, s);
    return o;
}

// Word w of a job: the aligned 16-byte destination word W0 + 16w (W0 = dst
// rounded down); its bytes come from source bytes [16w - m, 16w - m + 16),
// m = dst & 15, i.e. source words w - 1 and w (word -1 reads as zeros: its
// bytes lie before dst and are never stored).  Only the source words are
// kept between the load and the store (registers: 4 words per lane).
__device__ __forceinline__ void load_word(const Job& j, uint32_t w, uint4& lo, uint4& hi) {
    const uint32_t m = uint32_t(reinterpret_cast<uintptr_t>(j.dst) & 15u);
    const uint4* s16 = reinterpret_cast<const uint4*>(j.src);
    hi = __ldg(s16 + w);
    lo = (m && w) ? __ldg(s16 + w - 1) : make_uint4(0, 0, 0, 0);
}

__device__ __forceinline__ void store_word(const Job& j, uint32_t w, const uint4& lo,
                                           const uint4& hi) {
    const uint32_t m = uint32_t(reinterpret_cast<uintptr_t>(j.dst) & 15u);
    uint8_t* at = j.dst - m + 16u * w;
    const int32_t b0 = w == 0 ? int32_t(m) : 0;
    const int32_t end = int32_t(m + j.len) - int32_t(16u * w);
    const int32_t b1 = end < 16 ? end : 16;
    const uint4 v = m ? funnel128(lo, hi, 16u - m) : hi;
    if (b0 == 0 && b1 == 16) {
        *reinterpret_cast<uint4*>(at) = v;
        return;
    }
    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int b = 0; b < 16; ++b)
        if (b >= b0 && b < b1) at[b] = uint8_t(wv[b >> 2] >> (8 * (b & 3)));
}

// One warp copies two jobs (a chunk's flag and payload slices): up to 4
// words per lane per round, all of a round's loads before its stores.
__device__ __forceinline__ void warp_copy2(const Job& j0, const Job& j1, uint32_t lane) {
    const uint32_t n0 = job_words(j0), n = n0 + job_words(j1);
    for (uint32_t base = 0; base < n; base += 128) {
        uint4 lo[4], hi[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t i = base + lane + 32u * u;
            if (i < n) load_word(i < n0 ? j0 : j1, i < n0 ? i : i - n0, lo[u], hi[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t i = base + lane + 32u * u;
            if (i < n) store_word(i < n0 ? j0 : j1, i < n0 ? i : i - n0, lo[u], hi[u]);
        }
    }
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

__global__ void __launch_bounds__(256, 3) plz_assemble_kernel(AssembleArgs a) {
    const uint32_t lane = lane_id();
    const uint64_t j_hi = a.j_hi ? a.j_hi : a.n_blocks;
    // ---- offset tables: both tables of container j are one region of
    // 2(n+1) entries at image byte img0 + 26
    {
        const uint64_t stride = 2 * (a.cpb + 1) + 1;  // words per container, at most
        const uint64_t total = (j_hi - a.j_lo) * stride;
        for (uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
             idx += uint64_t(gridDim.x) * blockDim.x) {
            const uint64_t j = a.j_lo + idx / stride, wi = idx % stride;
            const uint64_t g0 = j * a.cpb;
            const uint64_t n = (j + 1 == a.n_blocks) ? a.n_chunks - g0 : a.cpb;
            uint8_t* region = a.img + container_start(a, j, g0) + 26;
            if (wi >= table_words(region, 2 * (n + 1))) continue;
            const uint64_t pb = a.P64[g0], fb = a.F64[g0];
            table_word(region, 2 * (n + 1), wi, [&](uint64_t e) {
                return e <= n ? uint32_t(a.P64[g0 + e] - pb) : uint32_t(a.F64[g0 + e - (n + 1)] - fb);
            });
        }
    }
    // ---- streams: warp per chunk
    const uint64_t C = uint64_t(a.C), S = uint64_t(a.S);
    const uint64_t g_lo = a.j_lo * a.cpb;
    const uint64_t g_hi = min(a.n_chunks, j_hi * a.cpb);
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    uint64_t g = g_lo + uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (g >= g_hi) return;
    // per-chunk prefixes, loaded one chunk ahead
    uint64_t pg = a.P64[g], fg = a.F64[g];
    uint32_t ps = a.psize[g], fs = a.fsize[g];
    uint64_t cj = ~0ull, streams = 0, pb = 0, fb = 0, ftot = 0;
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
        const Geo c = locate(a, g);
        if (c.j != cj) {
            cj = c.j;
            pb = a.P64[c.g0];
            fb = a.F64[c.g0];
            ftot = a.F64[c.g0 + c.n] - fb;
            streams = container_start(a, c.j, c.g0) + 26 + 8 * (c.n + 1);
        }
        const Job jf{a.img + streams + (fg - fb), a.flag_slots + g * (C / 8), fs};
        const Job jp{a.img + streams + ftot + (pg - pb), a.pay_slots + g * C * S, ps};
        warp_copy2(jf, jp, lane);
        pg = pg_n;
        fg = fg_n;
        ps = ps_n;
        fs = fs_n;
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
        const Job jf{a.out + d.seg_flags + lf, a.flag_slots + g * (C / 8), a.fsize[g]};
        const Job jp{a.out + d.seg_pay + lp, a.pay_slots + g * C * S, a.psize[g]};
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
    uint64_t blocks = (warps_needed + 7) / 8;
    if (blocks > 148ull * 8) blocks = 148ull * 8;
    plz_assemble_kernel<<<unsigned(blocks), 256, 0, st>>>(a);
}

void launch_headers(const AssembleArgs& a, cudaStream_t st) {
    const uint64_t nj = (a.j_hi ? a.j_hi : a.n_blocks) - a.j_lo;
    if (nj == 0) return;
    plz_headers_kernel<<<unsigned((nj + 127) / 128), 128, 0, st>>>(a);
}

void preload_assemble_kernels() {
    preload_kernel(reinterpret_cast<const void*>(plz_assemble_kernel));
    preload_kernel(reinterpret_cast<const void*>(plz_headers_kernel));
    preload_kernel(reinterpret_cast<const void*>(plz_shard_assemble_kernel));
    preload_kernel(reinterpret_cast<const void*>(plz_shard_headers_kernel));
}

}  // namespace plzgpu
