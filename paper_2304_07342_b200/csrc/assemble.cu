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
// first chunk.  One warp per chunk copies its flag and payload slices with
// realigned 128-bit stores; the header kernel (one thread per container)
// writes the 26-byte header, the final table entries, the tail and the image
// length, and flags 4-byte table overflow (scan.cpp:43-44).
#include <algorithm>

#include "common.cuh"

namespace plzgpu {
namespace {

struct Geo {
    uint64_t j, k, g0, n;  // container, chunk within it, its first chunk, its chunk count
};

__device__ __forceinline__ Geo locate(const AssembleArgs& a, uint64_t g) {
    Geo r;
    r.j = g / a.cpb;
    r.k = g - r.j * a.cpb;
    r.g0 = r.j * a.cpb;
    r.n = (r.j + 1 == a.n_blocks) ? a.n_chunks - r.g0 : a.cpb;
    return r;
}

__device__ __forceinline__ uint64_t container_start(const AssembleArgs& a, uint64_t j,
                                                    uint64_t g0) {
    return 26u * j + 8u * (g0 + j) + a.P64[g0] + a.F64[g0];
}

__global__ void __launch_bounds__(256) plz_assemble_kernel(AssembleArgs a) {
    const uint32_t lane = lane_id();
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint64_t C = uint64_t(a.C), S = uint64_t(a.S);
    const uint64_t g_lo = a.j_lo * a.cpb;
    const uint64_t g_hi = a.j_hi ? min(a.n_chunks, a.j_hi * a.cpb) : a.n_chunks;
    for (uint64_t g = g_lo + uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         g < g_hi; g += warps) {
        const Geo c = locate(a, g);
        const uint64_t img0 = container_start(a, c.j, c.g0);
        const uint64_t pb = a.P64[c.g0], fb = a.F64[c.g0];
        const uint64_t pk = a.P64[g] - pb, fk = a.F64[g] - fb;
        const uint64_t ftot = a.F64[c.g0 + c.n] - fb;
        uint8_t* tabs = a.img + img0 + 26;
        // table entries k (the header kernel writes entry n)
        if (lane < 4) {
            tabs[4 * c.k + lane] = uint8_t(pk >> (8 * lane));
        } else if (lane < 8) {
            tabs[4 * (c.n + 1) + 4 * c.k + (lane - 4)] = uint8_t(fk >> (8 * (lane - 4)));
        }
        uint8_t* streams = tabs + 8 * (c.n + 1);
        warp_copy_realign(streams + fk, a.flag_slots + g * (C / 8), a.fsize[g], lane);
        warp_copy_realign(streams + ftot + pk, a.pay_slots + g * C * S, a.psize[g], lane);
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
    st_le32(h + 26 + 4 * n, uint32_t(ptot));
    st_le32(h + 26 + 4 * (n + 1) + 4 * n, uint32_t(ftot));
    uint8_t* t = h + 26 + 8 * (n + 1) + ftot + ptot;
    const uint8_t* src = a.in + j * a.block_bytes + byte_len - tail;
    for (uint32_t i = 0; i < tail; ++i) t[i] = src[i];
    if (j + 1 == a.n_blocks) *a.img_len = img0 + 26 + 8 * (n + 1) + ftot + ptot + tail;
}

// Shard variant of Kernel III (multi-GPU): the same per-chunk
// copies into a local segment buffer with offsets rebased by the shard's
// position inside each container's streams.
__global__ void __launch_bounds__(256) plz_shard_assemble_kernel(ShardAssembleArgs a) {
    const uint32_t lane = lane_id();
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    const uint64_t C = uint64_t(a.C), S = uint64_t(a.S);
    for (uint64_t g = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         g < a.n_chunks; g += warps) {
        uint64_t c = 0;
        while (c + 1 < a.n_conts && a.conts[c + 1].g_lo <= g) ++c;
        const ShardCont& d = a.conts[c];
        const uint64_t i = g - d.g_lo;
        const uint64_t lp = a.P64[g] - a.P64[d.g_lo], lf = a.F64[g] - a.F64[d.g_lo];
        const uint64_t pk = d.p_base + lp, fk = d.f_base + lf;
        if (lane == 0 && (pk > 0xffffffffull || fk > 0xffffffffull)) atomicExch(a.overflow, 1u);
        if (lane < 4) {
            a.out[d.seg_ptab + 4 * i + lane] = uint8_t(pk >> (8 * lane));
        } else if (lane < 8) {
            a.out[d.seg_ftab + 4 * i + (lane - 4)] = uint8_t(fk >> (8 * (lane - 4)));
        }
        warp_copy_realign(a.out + d.seg_flags + lf, a.flag_slots + g * (C / 8), a.fsize[g], lane);
        warp_copy_realign(a.out + d.seg_pay + lp, a.pay_slots + g * C * S, a.psize[g], lane);
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
    if (blocks > 148ull * 16) blocks = 148ull * 16;
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
    if (blocks > 148ull * 16) blocks = 148ull * 16;
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
