// cusz.cu — cuSZ-style dual quantization feeding GPULZ on the device
// (PAPER.md "Use-case of gpuLZ", Table 3).
//
// The paper's improved cuSZ runs gpuLZ on the quantization codes of cuSZ's
// dual-quant step before (out-of-scope) Huffman coding.  This file is that
// producer and its inverse, so a field can go  field -> codes -> GPULZ image
// and back without leaving HBM:
//
//   prequant     q = rint(f * s),  s = float32(1 / (2 eb))   (round half even)
//   Lorenzo      d = Δx Δy Δz q  (3-D; 2-D / 1-D when nz / ny are 1), with
//                q = 0 outside the field
//   codes        code = d + radius if |d| < radius, else 0 (an outlier; its
//                (index, d) is listed in index order)
//   inverse      q = Σx Σy Σz d (three axis scans), f' = float32(q) * float32(2 eb)
//
// |f - f'| <= eb up to float32 rounding of f * s.  HBM-bound kernels: the
// quantizer reads each value once (a z-walking tile keeps the previous
// plane's term in a register) and writes 2 bytes; the scans read and write
// int32 once per axis.
#include "common.cuh"

namespace plzgpu {
namespace {

constexpr int kQuantThreads = 256;
constexpr int kQuantItems = 4;
constexpr int kQuantTile = kQuantThreads * kQuantItems;  // elements per outlier tile

struct Dims {
    uint64_t nx, ny, nz;
};

__device__ __forceinline__ int32_t prequant(const float* __restrict__ f, const Dims& g, int64_t x,
                                            int64_t y, int64_t z, float s) {
    if (x < 0 || y < 0 || z < 0) return 0;
    const float v = __ldg(f + (uint64_t(z) * g.ny + uint64_t(y)) * g.nx + uint64_t(x));
    return static_cast<int32_t>(rintf(__fmul_rn(v, s)));
}

// Lorenzo residual of element i (x fastest).
__device__ __forceinline__ int32_t lorenzo_delta(const float* __restrict__ f, const Dims& g,
                                                 uint64_t i, float s) {
    const int64_t x = int64_t(i % g.nx), y = int64_t((i / g.nx) % g.ny), z = int64_t(i / (g.nx * g.ny));
    const int32_t c = prequant(f, g, x, y, z, s);
    const int32_t a = prequant(f, g, x - 1, y, z, s), b = prequant(f, g, x, y - 1, z, s);
    const int32_t e = prequant(f, g, x, y, z - 1, s);
    const int32_t ab = prequant(f, g, x - 1, y - 1, z, s), ae = prequant(f, g, x - 1, y, z - 1, s);
    const int32_t be = prequant(f, g, x, y - 1, z - 1, s);
    const int32_t abe = prequant(f, g, x - 1, y - 1, z - 1, s);
    return c - a - b - e + ab + ae + be - abe;
}

// codes and per-tile outlier counts
__global__ void __launch_bounds__(kQuantThreads) plz_lorenzo_quant_kernel(
    const float* __restrict__ f, Dims g, uint64_t n, float s, int32_t radius,
    uint16_t* __restrict__ codes, uint32_t* __restrict__ tile_count) {
    __shared__ uint32_t warp_out[kQuantThreads / 32];
    const uint64_t t0 = uint64_t(blockIdx.x) * kQuantTile;
    uint32_t outl = 0;
#pragma unroll
    for (int k = 0; k < kQuantItems; ++k) {
        const uint64_t i = t0 + uint64_t(k) * kQuantThreads + threadIdx.x;
        if (i < n) {
            const int32_t d = lorenzo_delta(f, g, i, s);
            const bool in = d > -radius && d < radius;
            codes[i] = in ? uint16_t(d + radius) : uint16_t(0);
            outl += in ? 0u : 1u;
        }
    }
    outl = __reduce_add_sync(0xffffffffu, outl);
    if ((threadIdx.x & 31u) == 0) warp_out[threadIdx.x >> 5] = outl;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (int w = 0; w < kQuantThreads / 32; ++w) tot += warp_out[w];
        tile_count[blockIdx.x] = tot;
    }
}

// 2-D / 3-D fields: a 32 x 8 thread block owns a (y, x) tile and walks it
// through z.  Each plane's tile plus its y-1 / x-1 halo is prequantised once
// into shared memory; a thread forms its 2-D Lorenzo term of the plane
// (q - q_x - q_y + q_xy) and subtracts the previous plane's, kept in a
// register — every input value is read once (+ the halo), HBM-bound.
// Outliers bump the count of their 1024-element index tile.
constexpr int kTileX = 32, kTileY = 8;

__global__ void __launch_bounds__(kTileX * kTileY) plz_lorenzo_tiled_kernel(
    const float* __restrict__ f, Dims g, float s, int32_t radius, uint16_t* __restrict__ codes,
    uint32_t* __restrict__ tile_count) {
    constexpr int kHalo = (kTileY + 1) * (kTileX + 1);  // tile + row y0-1 + column x0-1
    constexpr int kPlanes = 4;                           // planes loaded per round (in flight)
    __shared__ int32_t qs2[2][kTileY + 1][kTileX + 1];  // double-buffered: one barrier per plane
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t x = int64_t(blockIdx.x) * kTileX + tx, y = int64_t(blockIdx.y) * kTileY + ty;
    const bool in = x < int64_t(g.nx) && y < int64_t(g.ny);
    // this thread's (at most two) halo slots: position in the tile, offset
    // in a plane, and whether it lies in the field (q = 0 outside)
    const int i0 = ty * kTileX + tx, i1 = i0 + kTileX * kTileY;
    int hy[2], hx[2];
    int64_t off[2];
    bool val[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int i = k ? i1 : i0;
        hy[k] = i / (kTileX + 1);
        hx[k] = i % (kTileX + 1);
        const int64_t gy = int64_t(blockIdx.y) * kTileY + hy[k] - 1;
        const int64_t gx = int64_t(blockIdx.x) * kTileX + hx[k] - 1;
        val[k] = i < kHalo && gy >= 0 && gx >= 0 && gy < int64_t(g.ny) && gx < int64_t(g.nx);
        off[k] = val[k] ? gy * int64_t(g.nx) + gx : 0;
    }
    const bool has1 = i1 < kHalo;
    const uint64_t plane_sz = g.ny * g.nx;
    int32_t prev = 0;  // the previous plane's 2-D term at (y, x)
    for (uint64_t z0 = 0; z0 < g.nz; z0 += kPlanes) {
        // kPlanes planes' loads issued together (memory-level parallelism),
        // then each plane: tile into shared memory, 2-D term, z difference
        float v[kPlanes][2];
#pragma unroll
        for (int d = 0; d < kPlanes; ++d)
#pragma unroll
            for (int k = 0; k < 2; ++k)
                v[d][k] = (val[k] && z0 + d < g.nz) ? __ldg(f + (z0 + d) * plane_sz + off[k]) : 0.f;
#pragma unroll
        for (int d = 0; d < kPlanes; ++d) {
            const uint64_t z = z0 + d;
            if (z >= g.nz) break;
            // plane z's tile goes to buffer z & 1: the barrier below also
            // orders every read of plane z-1 (other buffer) before the
            // writes of plane z+1 into it
            int32_t (*qs)[kTileX + 1] = qs2[z & 1];
            qs[hy[0]][hx[0]] = val[0] ? static_cast<int32_t>(rintf(__fmul_rn(v[d][0], s))) : 0;
            if (has1) qs[hy[1]][hx[1]] = val[1] ? static_cast<int32_t>(rintf(__fmul_rn(v[d][1], s))) : 0;
            __syncthreads();
            const int32_t cur = qs[ty + 1][tx + 1] - qs[ty + 1][tx] - qs[ty][tx + 1] + qs[ty][tx];
            if (in) {
                const int32_t dd = cur - prev;
                const uint64_t i = (z * g.ny + uint64_t(y)) * g.nx + uint64_t(x);
                const bool ok = dd > -radius && dd < radius;
                codes[i] = ok ? uint16_t(dd + radius) : uint16_t(0);
                if (!ok) atomicAdd(&tile_count[i / kQuantTile], 1u);
            }
            prev = cur;
        }
    }
}

// outliers (index, d) in index order: each tile compacts its zero codes,
// slab by slab (slab k = elements t0 + k*256 + tid, increasing with tid)
__global__ void __launch_bounds__(kQuantThreads) plz_outlier_write_kernel(
    const float* __restrict__ f, Dims g, uint64_t n, float s, const uint16_t* __restrict__ codes,
    const uint32_t* __restrict__ tile_count, const uint64_t* __restrict__ tile_off,
    uint64_t* __restrict__ out_idx, int32_t* __restrict__ out_val, uint64_t cap) {
    if (tile_count[blockIdx.x] == 0) return;
    constexpr int NWp = kQuantThreads / 32;
    __shared__ uint32_t wcount[NWp], wbase[NWp];
    __shared__ uint64_t base;
    const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) base = tile_off[blockIdx.x];
    const uint64_t t0 = uint64_t(blockIdx.x) * kQuantTile;
    for (int k = 0; k < kQuantItems; ++k) {
        const uint64_t i = t0 + uint64_t(k) * kQuantThreads + threadIdx.x;
        const bool o = i < n && codes[i] == 0;
        const uint32_t m = __ballot_sync(0xffffffffu, o);
        if (lane == 0) wcount[wid] = __popc(m);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t r = 0;
            for (int w = 0; w < NWp; ++w) {
                wbase[w] = r;
                r += wcount[w];
            }
            wcount[0] = r;  // slab total
        }
        __syncthreads();
        if (o) {
            const uint64_t at = base + wbase[wid] + __popc(m & ((1u << lane) - 1u));
            if (at < cap) {
                out_idx[at] = i;
                out_val[at] = lorenzo_delta(f, g, i, s);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) base += wcount[0];
        __syncthreads();
    }
}

// ---- inverse
// the residual of element i: code - radius, or (code 0) the outlier's value,
// found by binary search in the index-ordered outlier list
__device__ __forceinline__ int32_t residual(uint32_t code, uint64_t i, int32_t radius,
                                            const uint64_t* __restrict__ idx,
                                            const int32_t* __restrict__ val, uint64_t m) {
    if (code) return int32_t(code) - radius;
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (idx[mid] < i) lo = mid + 1;
        else hi = mid;
    }
    return lo < m && idx[lo] == i ? val[lo] : 0;
}

// inclusive sums along x straight from the codes (residuals and outliers
// resolved on the fly): one warp per row, 32 elements per step with a carry
__global__ void plz_scan_x_codes_kernel(const uint16_t* __restrict__ codes, int32_t radius,
                                        const uint64_t* __restrict__ idx,
                                        const int32_t* __restrict__ val, uint64_t m,
                                        int32_t* __restrict__ d, uint64_t rows, uint64_t nx) {
    const uint32_t lane = lane_id();
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t r = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows;
         r += warps) {
        const uint16_t* crow = codes + r * nx;
        int32_t* row = d + r * nx;
        int32_t carry = 0;
        uint32_t nxt = lane < nx ? crow[lane] : 1u;
        for (uint64_t x0 = 0; x0 < nx; x0 += 32) {
            const uint64_t x = x0 + lane;
            const uint32_t c = nxt;
            nxt = x + 32 < nx ? crow[x + 32] : 1u;
            int32_t v = x < nx ? residual(c, r * nx + x, radius, idx, val, m) : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t u = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= uint32_t(o)) v += u;
            }
            v += carry;
            if (x < nx) row[x] = v;
            carry = __shfl_sync(0xffffffffu, v, 31);
        }
    }
}

// inclusive sums along a strided axis: thread per (outer, x) column, serial
// over `len` elements `stride` apart (coalesced across x); the last axis
// also dequantises: f = float(q) * two_eb
template <bool kLast>
__global__ void plz_scan_strided_kernel(int32_t* __restrict__ d, uint64_t outer, uint64_t len,
                                        uint64_t stride, uint64_t outer_stride, float two_eb,
                                        float* __restrict__ f) {
    const uint64_t cols = outer * stride;
    for (uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < cols;
         c += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t o = c / stride, x = c % stride;
        const uint64_t b = o * outer_stride + x;
        int32_t run = 0;
        // kBatch loads in flight per thread, then their running sums stored
        constexpr int kBatch = 8;
        uint64_t k = 0;
        for (; k + kBatch <= len; k += kBatch) {
            int32_t v[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) v[j] = d[b + (k + j) * stride];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                run += v[j];
                if constexpr (kLast) f[b + (k + j) * stride] = __fmul_rn(float(run), two_eb);
                else d[b + (k + j) * stride] = run;
            }
        }
        for (; k < len; ++k) {
            run += d[b + k * stride];
            if constexpr (kLast) f[b + k * stride] = __fmul_rn(float(run), two_eb);
            else d[b + k * stride] = run;
        }
    }
}

__global__ void plz_dequant_kernel(const int32_t* __restrict__ q, uint64_t n, float two_eb,
                                   float* __restrict__ f) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        f[i] = __fmul_rn(float(q[i]), two_eb);
}

}  // namespace

uint64_t lorenzo_tiles(uint64_t n) { return (n + kQuantTile - 1) / kQuantTile; }

void launch_lorenzo_quantize(const float* f, uint64_t nx, uint64_t ny, uint64_t nz, float s,
                             int32_t radius, uint16_t* codes, uint32_t* tile_count,
                             cudaStream_t st) {
    const uint64_t n = nx * ny * nz, tiles = lorenzo_tiles(n);
    const Dims g{nx, ny, nz};
    if (ny > 1) {
        cudaMemsetAsync(tile_count, 0, tiles * 4, st);
        const dim3 grid(unsigned((nx + kTileX - 1) / kTileX), unsigned((ny + kTileY - 1) / kTileY));
        plz_lorenzo_tiled_kernel<<<grid, dim3(kTileX, kTileY), 0, st>>>(f, g, s, radius, codes,
                                                                        tile_count);
    } else {
        plz_lorenzo_quant_kernel<<<unsigned(tiles), kQuantThreads, 0, st>>>(f, g, n, s, radius,
                                                                            codes, tile_count);
    }
}

void launch_outlier_write(const float* f, uint64_t nx, uint64_t ny, uint64_t nz, float s,
                          const uint16_t* codes, const uint32_t* tile_count,
                          const uint64_t* tile_off, uint64_t* out_idx, int32_t* out_val,
                          uint64_t cap, cudaStream_t st) {
    const uint64_t n = nx * ny * nz, tiles = lorenzo_tiles(n);
    const Dims g{nx, ny, nz};
    plz_outlier_write_kernel<<<unsigned(tiles), kQuantThreads, 0, st>>>(
        f, g, n, s, codes, tile_count, tile_off, out_idx, out_val, cap);
}

void launch_lorenzo_reconstruct(const uint16_t* codes, const uint64_t* out_idx,
                                const int32_t* out_val, uint64_t n_out, uint64_t nx, uint64_t ny,
                                uint64_t nz, int32_t radius, float two_eb, int32_t* d, float* f,
                                int sms, cudaStream_t st) {
    const uint64_t n = nx * ny * nz;
    const unsigned grid = unsigned(sms) * 8;
    plz_scan_x_codes_kernel<<<grid, 256, 0, st>>>(codes, radius, out_idx, out_val, n_out, d,
                                                  ny * nz, nx);
    // along y within each z-slab, then along z (which also dequantises)
    if (nz > 1) {
        if (ny > 1) plz_scan_strided_kernel<false><<<grid, 256, 0, st>>>(d, nz, ny, nx, nx * ny, two_eb, f);
        plz_scan_strided_kernel<true><<<grid, 256, 0, st>>>(d, 1, nz, nx * ny, 0, two_eb, f);
    } else if (ny > 1) {
        plz_scan_strided_kernel<true><<<grid, 256, 0, st>>>(d, 1, ny, nx, 0, two_eb, f);
    } else {
        plz_dequant_kernel<<<grid, 256, 0, st>>>(d, n, two_eb, f);
    }
}

void preload_cusz_kernels() {
    const void* fs[] = {reinterpret_cast<const void*>(plz_dequant_kernel),
                          reinterpret_cast<const void*>(plz_lorenzo_quant_kernel),
                          reinterpret_cast<const void*>(plz_lorenzo_tiled_kernel),
                          reinterpret_cast<const void*>(plz_outlier_write_kernel),
                          reinterpret_cast<const void*>(plz_scan_strided_kernel<false>),
                          reinterpret_cast<const void*>(plz_scan_strided_kernel<true>),
                          reinterpret_cast<const void*>(plz_scan_x_codes_kernel)};
    for (const void* f : fs) preload_kernel(f);
}

}  // namespace plzgpu
