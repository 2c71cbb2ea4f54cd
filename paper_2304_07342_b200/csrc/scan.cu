// scan.cu — Kernel II: device-wide exclusive scan of per-chunk (payload, flag)
// sizes with decoupled look-back.
//
// Reference: scan.cpp:38-47 (global_exclusive_scan), run twice by
// deflate.cpp:45-46 — offsets[0] = 0, offsets[i+1] = offsets[i] + size[i].
// The reference scans each container separately into u32 tables; here one
// pass scans every chunk of every container into u64 prefixes and Kernel III
// rebases each container's entries (entry = P64[g] - P64[first chunk]) and
// checks the 4-byte range (scan.cpp:43-44).
//
// One CTA per 2048-chunk tile, tiles claimed in launch order through an
// atomic counter so every predecessor is already running.  In-tile: blocked
// loads (8 consecutive sizes per thread, two 128-bit loads), thread-serial
// sums, warp-shuffle scan, smem scan of warp totals.  Across tiles: publish
// the aggregate, walk predecessors (a warp reads 32 tile states per step)
// until an inclusive prefix is found, publish the inclusive prefix.
#include "common.cuh"

namespace plzgpu {
namespace {

struct Pair {
    unsigned long long p, f;
};

__device__ __forceinline__ Pair warp_incl_scan(Pair v, uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long p = __shfl_up_sync(0xffffffffu, v.p, d);
        const unsigned long long f = __shfl_up_sync(0xffffffffu, v.f, d);
        if (lane >= uint32_t(d)) {
            v.p += p;
            v.f += f;
        }
    }
    return v;
}

__global__ void __launch_bounds__(kScanThreads) plz_scan_kernel(ScanArgs a) {
    __shared__ uint32_t s_tile;
    __shared__ Pair s_warp[kScanThreads / 32];
    __shared__ Pair s_prefix;

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(a.tile_counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t first = tile * kScanTile + uint64_t(tid) * kScanItems;

    // ---- blocked load of 8 (payload, flag) sizes
    uint32_t ps[kScanItems], fs[kScanItems];
    if (first + kScanItems <= a.n) {
        const uint4* pp = reinterpret_cast<const uint4*>(a.psize + first);
        const uint4* fp = reinterpret_cast<const uint4*>(a.fsize + first);
        const uint4 p0 = pp[0], p1 = pp[1], f0 = fp[0], f1 = fp[1];
        ps[0] = p0.x; ps[1] = p0.y; ps[2] = p0.z; ps[3] = p0.w;
        ps[4] = p1.x; ps[5] = p1.y; ps[6] = p1.z; ps[7] = p1.w;
        fs[0] = f0.x; fs[1] = f0.y; fs[2] = f0.z; fs[3] = f0.w;
        fs[4] = f1.x; fs[5] = f1.y; fs[6] = f1.z; fs[7] = f1.w;
    } else {
#pragma unroll
        for (int i = 0; i < kScanItems; ++i) {
            const bool in = first + i < a.n;
            ps[i] = in ? a.psize[first + i] : 0u;
            fs[i] = in ? a.fsize[first + i] : 0u;
        }
    }
    Pair own{0, 0};
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        own.p += ps[i];
        own.f += fs[i];
    }

    // ---- CTA-wide exclusive scan of the per-thread sums
    const Pair incl = warp_incl_scan(own, lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        Pair w = lane < kScanThreads / 32 ? s_warp[lane] : Pair{0, 0};
        const Pair wi = warp_incl_scan(w, lane);
        if (lane < kScanThreads / 32) s_warp[lane] = Pair{wi.p - w.p, wi.f - w.f};  // exclusive
        const Pair total{__shfl_sync(0xffffffffu, wi.p, kScanThreads / 32 - 1),
                         __shfl_sync(0xffffffffu, wi.f, kScanThreads / 32 - 1)};

        // ---- decoupled look-back (warp 0)
        Pair prefix{0, 0};
        if (tile == 0) {
            if (lane == 0) {
                __stcg(&a.incl[0], make_ulonglong2(total.p, total.f));
                st_release(&a.status[0], 2u);
            }
        } else {
            if (lane == 0) {
                __stcg(&a.agg[tile], make_ulonglong2(total.p, total.f));
                st_release(&a.status[tile], 1u);
            }
            int64_t j = int64_t(tile) - 1 - int64_t(lane);  // this lane's predecessor
            for (;;) {
                uint32_t st = j >= 0 ? ld_acquire(&a.status[j]) : 2u;
                // wait until every lane's predecessor has at least an aggregate
                while (!__all_sync(0xffffffffu, st != 0u)) {
                    __nanosleep(32);
                    if (st == 0u) st = ld_acquire(&a.status[j]);
                }
                const uint32_t incl_mask = __ballot_sync(0xffffffffu, st == 2u);
                // lanes up to and including the nearest inclusive predecessor contribute
                const uint32_t stop = incl_mask ? uint32_t(__ffs(incl_mask) - 1) : 31u;
                Pair c{0, 0};
                if (lane <= stop && j >= 0) {
                    const ulonglong2 v = st == 2u ? __ldcg(&a.incl[j]) : __ldcg(&a.agg[j]);
                    c = Pair{v.x, v.y};
                }
#pragma unroll
                for (int d = 16; d >= 1; d >>= 1) {
                    c.p += __shfl_xor_sync(0xffffffffu, c.p, d);
                    c.f += __shfl_xor_sync(0xffffffffu, c.f, d);
                }
                prefix.p += c.p;
                prefix.f += c.f;
                if (incl_mask) break;
                j -= 32;
            }
            if (lane == 0) {
                __stcg(&a.incl[tile], make_ulonglong2(prefix.p + total.p, prefix.f + total.f));
                st_release(&a.status[tile], 2u);
            }
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();

    // ---- write this thread's 8 exclusive prefixes (+ the carry of earlier
    // containers when the scan covers one container of a pipelined compress)
    Pair pre = s_prefix;
    if (a.carry_p) {
        pre.p += *a.carry_p;
        pre.f += *a.carry_f;
    }
    const Pair wex = s_warp[warp];
    unsigned long long rp = pre.p + wex.p + (incl.p - own.p);
    unsigned long long rf = pre.f + wex.f + (incl.f - own.f);
#pragma unroll
    for (int i = 0; i < kScanItems; ++i) {
        if (first + i < a.n) {
            a.P64[first + i] = rp;
            a.F64[first + i] = rf;
        }
        rp += ps[i];
        rf += fs[i];
        if (first + i + 1 == a.n) {  // the owner of the last chunk writes the totals
            a.P64[a.n] = rp;
            a.F64[a.n] = rf;
        }
    }
}

}  // namespace

void launch_scan(const ScanArgs& a, cudaStream_t st) {
    const uint64_t tiles = (a.n + kScanTile - 1) / kScanTile;
    if (tiles == 0) return;
    plz_scan_kernel<<<unsigned(tiles), kScanThreads, 0, st>>>(a);
}

void preload_scan_kernels() { preload_kernel(reinterpret_cast<const void*>(plz_scan_kernel)); }

}  // namespace plzgpu
