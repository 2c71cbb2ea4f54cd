// encode.cu — Kernel I: match + greedy token walk + encode, one warp per chunk.
//
// Reference contract:
//   matcher.cpp:71-111   longest match over w in [max(0,p-W), p), length capped
//                        at min(p-w, 255, n-p), ties to the largest offset;
//   matcher.cpp:113-131  positions with p % I != 0 are forced literals;
//   encoder.cpp:18-73    greedy walk from 0: pointer iff off != 0 and
//                        len >= min_match, MSB-first flag bits, pointer wire
//                        order [len][off], literal = the S raw bytes.
//
// B200 design.  A warp owns a chunk (dynamic scheduling over a persistent
// grid).  The chunk's bytes arrive in shared memory by one TMA bulk copy
// (cp.async.bulk + mbarrier).  A right-to-left ballot pass turns them into
// packed (symbol, equal-run) cells so a single shared load per side advances
// an lcp by a whole run (the run-skipping of matcher.cpp:42-59, exact with
// runs capped at 255 because no match exceeds 255).  The walk then only
// searches the positions it visits: the 32 lanes split the <= W window
// candidates, prune against the warp's best with REDUX max, and the packed key
// (len << 8 | off) makes max() reproduce the largest-offset tie-break.  Output
// tokens are staged in shared memory and flushed with 128-bit stores into a
// per-chunk slot; Kernel II/III compact them.
#include "common.cuh"

namespace plzgpu {
namespace {

// Continuation of an lcp once both positions sit at the same (symbol, run)
// cell: both runs end together, so compare again at relative position k.
template <int S>
__device__ __forceinline__ int lcp_continue(const typename Sym<S>::Cell* __restrict__ cells, int w,
                                         int p, int k, int ub) {
    while (k < ub) {
        const auto a = cells[w + k];
        const auto b = cells[p + k];
        if (a == b) {  // same symbol, same run: both runs end together
            k += static_cast<int>(cell_run<S>(a));
            continue;
        }
        if (cell_sym<S>(a) == cell_sym<S>(b)) {  // runs differ: mismatch at the shorter end
            const uint32_t ra = cell_run<S>(a), rb = cell_run<S>(b);
            k += static_cast<int>(ra < rb ? ra : rb);
        }
        break;
    }
    return k < ub ? k : ub;
}

// Warp-cooperative find_match at position p (p > 0).  Returns the packed key
// (len << 8) | off of the winning candidate (len may be 0 = no match).
//
// Lane l evaluates offsets o = lim - l - 32r, r = 0..7, in branch-free
// rounds: one shared load of the candidate's (symbol, run) cell settles it
// unless the cell is identical to p's (same symbol, same remaining run) — a
// different symbol gives 0, the same symbol with a different run length gives
// min(run_w, run_p).  Identical cells (~15 of ~230 candidates on quant codes)
// are only flagged in a per-lane bitmask and continued afterwards, so the
// divergent continuation runs once per search instead of once per round.
// One window candidate at offset o.  kCap: positions within 255 symbols of
// the chunk end also cap the length at n - p; elsewhere min(len, o) <= 255
// already.  Identical cells are flagged in `pending` for the continuation.
template <int S, bool kCap>
__device__ __forceinline__ void eval_candidate(typename Sym<S>::Cell cw, typename Sym<S>::Cell cp,
                                               uint32_t rp, uint32_t o, uint32_t cap,
                                               uint32_t bit, uint32_t& best, uint32_t& pending) {
    using Cell = typename Sym<S>::Cell;
    constexpr Cell kSymMask = (Cell(1) << (8 * S)) - 1;
    const uint32_t rw = cell_run<S>(cw);
    const uint32_t ub = kCap ? (o < cap ? o : cap) : o;
    uint32_t k = rw < rp ? rw : rp;  // same symbol: the shorter run ends first
    k = k < ub ? k : ub;
    const uint32_t key = ((cw ^ cp) & kSymMask) == 0 ? (k << 8) | o : o;
    best = key > best ? key : best;
    if (cw == cp) pending |= bit;
}

// All candidates of one search: rounds 0..full-1 have every lane valid, the
// tail round only lanes with offset >= 1.  The switch enters a straight-line
// unrolled sequence (no per-round branches).
template <int S, bool kCap>
__device__ __forceinline__ void eval_window(const typename Sym<S>::Cell* __restrict__ cw,
                                            typename Sym<S>::Cell cp, uint32_t rp, int o0,
                                            int full, uint32_t cap, uint32_t& best,
                                            uint32_t& pending) {
#define PLZ_ROUND(R) \
    eval_candidate<S, kCap>(cw[32 * (R)], cp, rp, uint32_t(o0 - 32 * (R)), cap, 1u << (R), best, pending)
    switch (full) {
        case 8: PLZ_ROUND(7); [[fallthrough]];
        case 7: PLZ_ROUND(6); [[fallthrough]];
        case 6: PLZ_ROUND(5); [[fallthrough]];
        case 5: PLZ_ROUND(4); [[fallthrough]];
        case 4: PLZ_ROUND(3); [[fallthrough]];
        case 3: PLZ_ROUND(2); [[fallthrough]];
        case 2: PLZ_ROUND(1); [[fallthrough]];
        case 1: PLZ_ROUND(0); [[fallthrough]];
        default: break;
    }
#undef PLZ_ROUND
    if (full < 8 && o0 - 32 * full >= 1)
        eval_candidate<S, kCap>(cw[32 * full], cp, rp, uint32_t(o0 - 32 * full), cap, 1u << full,
                                best, pending);
}

// ---- S in {1, 2}: two adjacent candidates per lane-instruction ------------
// Candidates are taken in aligned pairs (w, w+1), w even, so one shared load
// fetches both cells; symbols and runs are split into 16-bit halves with PRMT
// and evaluated with native 16x2 SIMD min/max (VIMNMX.U16x2).  Keys are the
// same (len << 8 | off) as the scalar path, one per half.
__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) { return __vminu2(a, b); }
__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b) { return __vmaxu2(a, b); }

template <int S>
__device__ __forceinline__ void load_pair(const typename Sym<S>::Cell* cells, int w,
                                          uint32_t& sym2, uint32_t& run2) {
    if constexpr (S == 1) {  // cell = sym8 | run8 << 8; a pair is one u32
        const uint32_t c = *reinterpret_cast<const uint32_t*>(cells + w);
        sym2 = __byte_perm(c, 0u, 0x4240);
        run2 = __byte_perm(c, 0u, 0x4341);
    } else {  // cell = sym16 | run8 << 16; a pair is one u64
        const uint2 c = *reinterpret_cast<const uint2*>(cells + w);
        sym2 = __byte_perm(c.x, c.y, 0x5410);
        run2 = __byte_perm(c.x, c.y, 0x7632);  // bytes 3/7 of a cell are zero
    }
}

template <int S, bool kCap, bool kMask>
__device__ __forceinline__ void eval_pair(const typename Sym<S>::Cell* cells, int w, int oa,
                                          int lim, uint32_t s2, uint32_t rp2, uint32_t cap2,
                                          uint32_t bit, uint32_t& best2, uint32_t& pending) {
    uint32_t sym2, run2;
    load_pair<S>(cells, w, sym2, run2);
    uint32_t o2 = (uint32_t(oa) & 0xffffu) | (uint32_t(oa - 1) << 16);
    // halves outside the window may hold offsets >= 256 (or wrapped negatives):
    // clamp so len * 256 + off cannot carry into the neighbouring half
    if constexpr (kMask) o2 = vmin2(o2, 0x00ff00ffu);
    const uint32_t ub2 = kCap ? vmin2(o2, cap2) : o2;
    const uint32_t d = sym2 ^ s2;
    const uint32_t differ = vmin2(d, 0x00010001u);                 // 1 where symbols differ
    const uint32_t keep = (differ ^ 0x00010001u) * 0xffffu;        // 0xffff where equal
    const uint32_t k2 = vmin2(vmin2(run2, rp2), ub2) & keep;       // same symbol: shorter run
    uint32_t key2 = k2 * 256u + o2;
    uint32_t ident = vmin2(d | (run2 ^ rp2), 0x00010001u) ^ 0x00010001u;  // identical cells
    if constexpr (kMask) {  // halves with offset outside [1, lim]
        const uint32_t m = ((oa >= 1 && oa <= lim) ? 0x0000ffffu : 0u) |
                           ((oa - 1 >= 1 && oa - 1 <= lim) ? 0xffff0000u : 0u);
        key2 &= m;
        ident &= m;
    }
    best2 = vmax2(best2, key2);
    pending += ident * bit;  // bits r (half a) and 16 + r (half b)
}

template <int S, bool kCap>
__device__ __forceinline__ uint32_t pair_window(const typename Sym<S>::Cell* __restrict__ cells,
                                                int p, int lim, uint32_t cap, uint32_t s2,
                                                uint32_t rp2, uint32_t lane, uint32_t& pending,
                                                int& w0_out) {
    const int w0 = (p - lim) & ~1;                 // pairs cover [w0, w0 + 2*npairs) >= window
    const int npairs = (p - w0 + 1) >> 1;
    const uint32_t cap2 = cap * 0x00010001u;
    const int wl = w0 + 2 * static_cast<int>(lane);
    const int oa0 = p - wl;
    uint32_t best2 = 0;
    if (npairs == 128) {  // W = 255 steady state: 4 rounds, edges only in rounds 0 and 3
        eval_pair<S, kCap, true>(cells, wl, oa0, lim, s2, rp2, cap2, 1u, best2, pending);
        eval_pair<S, kCap, false>(cells, wl + 64, oa0 - 64, lim, s2, rp2, cap2, 2u, best2, pending);
        eval_pair<S, kCap, false>(cells, wl + 128, oa0 - 128, lim, s2, rp2, cap2, 4u, best2, pending);
        eval_pair<S, kCap, true>(cells, wl + 192, oa0 - 192, lim, s2, rp2, cap2, 8u, best2, pending);
    } else {
        const int rounds = (npairs + 31) >> 5;
        for (int r = 0; r < rounds; ++r)
            eval_pair<S, kCap, true>(cells, wl + 64 * r, oa0 - 64 * r, lim, s2, rp2, cap2, 1u << r,
                                     best2, pending);
    }
    w0_out = w0;
    const uint32_t lo = best2 & 0xffffu, hi = best2 >> 16;
    return lo > hi ? lo : hi;
}

// Identical-cell candidates (both runs end together) continue past the run.
// Each lane holds a bitmask of its own; the warp compacts them into a list in
// shared memory so every lane continues at most a few, instead of a
// divergent per-lane loop.  offset_of(bit) maps a pending bit to its offset.
template <int S, typename OffsetOf>
__device__ __forceinline__ uint32_t continue_pending(const typename Sym<S>::Cell* __restrict__ cells,
                                                     int p, uint32_t cap, uint32_t rp,
                                                     uint8_t* list, uint32_t lane,
                                                     uint32_t pending, uint32_t best,
                                                     OffsetOf offset_of) {
    const uint32_t cnt = __popc(pending);
    if (!__any_sync(0xffffffffu, cnt != 0)) return best;
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= uint32_t(d)) incl += x;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t at = incl - cnt;
    while (pending) {
        const int b = __ffs(pending) - 1;
        pending &= pending - 1;
        list[at++] = uint8_t(offset_of(b));
    }
    __syncwarp();
    for (uint32_t i = lane; i < total; i += 32) {
        const int o = list[i];
        const int ub = o < int(cap) ? o : int(cap);
        if (int(rp) >= ub) continue;
        const uint32_t k = uint32_t(lcp_continue<S>(cells, p - o, p, static_cast<int>(rp), ub));
        const uint32_t key = (k << 8) | uint32_t(o);
        best = key > best ? key : best;
    }
    __syncwarp();
    return best;
}

template <int S>
__device__ __forceinline__ uint32_t find_match_warp(const typename Sym<S>::Cell* __restrict__ cells,
                                                    int p, int n, int W, uint32_t lane,
                                                    uint8_t* list) {
    using Cell = typename Sym<S>::Cell;
    const int lim = p < W ? p : W;  // offsets 1..lim are in the window
    const uint32_t cap = uint32_t((n - p) < 255 ? (n - p) : 255);
    const Cell cp = cells[p];
    const uint32_t rp = cell_run<S>(cp);
    const int o0 = lim - static_cast<int>(lane);  // round r: offset o0 - 32r
    const Cell* cw = cells + (p - o0);              // round r: cw[32r]
    const int full = lim >> 5;                      // rounds where every lane is valid
    uint32_t best = 0, pending = 0;
    if constexpr (S <= 2) {
        int w0 = 0;
        const uint32_t s2 = uint32_t(cell_sym<S>(cp)) * 0x00010001u, rp2 = rp * 0x00010001u;
        best = cap == 255 ? pair_window<S, false>(cells, p, lim, cap, s2, rp2, lane, pending, w0)
                          : pair_window<S, true>(cells, p, lim, cap, s2, rp2, lane, pending, w0);
        const int wl = w0 + 2 * static_cast<int>(lane);
        best = continue_pending<S>(cells, p, cap, rp, list, lane, pending, best,
                                   [&](int b) { return p - (wl + 64 * (b & 15) + (b >> 4)); });
        return __reduce_max_sync(0xffffffffu, best);
    }
    if (cap == 255 && full == 7) {  // steady state of W = 255: straight-line 7 rounds + tail
#pragma unroll
        for (int r = 0; r < 7; ++r)
            eval_candidate<S, false>(cw[32 * r], cp, rp, uint32_t(o0 - 32 * r), cap, 1u << r, best,
                                     pending);
        if (o0 - 224 >= 1)
            eval_candidate<S, false>(cw[224], cp, rp, uint32_t(o0 - 224), cap, 1u << 7, best,
                                     pending);
    } else if (cap == 255) {
        eval_window<S, false>(cw, cp, rp, o0, full, cap, best, pending);
    } else {
        eval_window<S, true>(cw, cp, rp, o0, full, cap, best, pending);
    }
    // identical cells: both runs end together, continue at relative rp
    best = continue_pending<S>(cells, p, cap, rp, list, lane, pending, best,
                               [&](int b) { return o0 - 32 * b; });
    return __reduce_max_sync(0xffffffffu, best);
}

// Kernel I, wide-cell pass: chunks the bitmap passes (bitmatch.cu) left
// because their alphabet exceeds kBmMaxSymsWide (src_list), or every chunk.
// Cells keep (symbol, run) in 2S bytes, so any alphabet works; tokens leave
// in 32-token batches as in the bitmap passes.
template <int S>
__global__ void __launch_bounds__(512) plz_encode_kernel(EncodeArgs a) {
    using T = typename Sym<S>::T;
    using Cell = typename Sym<S>::Cell;
    extern __shared__ __align__(16) uint8_t smem[];

    const uint32_t lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    const int C = a.C;
    constexpr size_t kHead = size_t(kEncodeHeadPerS) * S;
    uint8_t* base = smem + encode_warp_smem(C, S) * warp;
    // [head: kHead B][cells: C x sizeof(Cell)][flags: C/8 B][list][mbarrier]
    // (the head and flag areas are the layout plz_match_table_kernel shares;
    // this kernel writes its tokens straight to the slots)
    Cell* cells = reinterpret_cast<Cell*>(base + kHead);
    uint8_t* raw8 = base + kHead + size_t(C) * S;  // raw stage: the upper half of the cells
    uint8_t* flg = base + kHead + size_t(C) * sizeof(Cell);      // C/8 bytes
    uint8_t* list = flg + C / 8;                                  // 256 B continuation list
    uint64_t* mbar = reinterpret_cast<uint64_t*>(list + 256);     // 8B aligned

    if (lane == 0) mbar_init(mbar, 1);
    __syncwarp();
    uint32_t phase = 0;
    unsigned long long warp_ptr = 0, warp_tok = 0;  // stats, flushed once per warp

    for (;;) {
        uint64_t g = 0;
        if (lane == 0) {
            const uint32_t idx = atomicAdd(a.work, 1u);
            if (!a.src_list) g = idx;
            else g = idx < *a.src_count ? a.src_list[idx] : a.n_chunks;
        }
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= a.n_chunks) break;

        const int n = (g + 1 == a.n_chunks) ? static_cast<int>(a.last_len) : C;
        const uint32_t nbytes = uint32_t(n) * S;
        const uint8_t* src = a.in + g * uint64_t(C) * S;

        // H2D pipeline: wait (bounded, ~4 s) until this chunk's segment landed
        if (a.ready) {
            uint32_t ok = 1;
            if (lane == 0) {
                const uint32_t* f = a.ready + g / a.seg_chunks;
                const long long t0 = clock64();
                while (ld_acquire_sys(f) != a.epoch) {
                    __nanosleep(256);
                    if (clock64() - t0 > (1ll << 33)) {
                        atomicExch(a.stalled, 1u);
                        ok = 0;
                        break;
                    }
                }
                asm volatile("fence.proxy.async.global;" ::: "memory");
            }
            if (!__shfl_sync(0xffffffffu, ok, 0)) break;
        }

        // ---- stage the chunk's bytes
        if (a.bulk_ok && (nbytes & 15u) == 0) {
            fence_proxy_async_smem();  // prior generic accesses before the TMA write
            __syncwarp();
            if (lane == 0) bulk_g2s(raw8, src, nbytes, mbar);
            mbar_wait(mbar, phase);
            phase ^= 1u;
        } else {
            for (uint32_t i = lane; i < nbytes; i += 32) raw8[i] = src[i];
            __syncwarp();
        }

        {
            // ---- symbols into cells, in place, left to right (a word's writes
            // only clobber raw symbols that are already read)
            const T* raw = reinterpret_cast<const T*>(raw8);
            for (int w = 0; w <= (n - 1) >> 5; ++w) {
                const int i = (w << 5) + static_cast<int>(lane);
                const T v = i < n ? raw[i] : T(0);
                __syncwarp();
                if (i < n) cells[i] = Cell(v);
                __syncwarp();
            }
            // ---- equal-run lengths, right to left in 32-position words
            uint32_t carry = 0;
            for (int w = (n - 1) >> 5; w >= 0; --w) {
                const int i = (w << 5) + static_cast<int>(lane);
                const T v = i < n ? cell_sym<S>(cells[i]) : T(0);
                const bool eq = (i + 1 < n) && cell_sym<S>(cells[i + 1]) == v;
                const uint32_t m = __ballot_sync(0xffffffffu, eq);
                const uint32_t sh = m >> lane;
                uint32_t r;
                if (sh == (0xffffffffu >> lane))
                    r = (32u - lane) + carry;  // run continues into the next word
                else
                    r = static_cast<uint32_t>(__ffs(~sh));  // (#equal successors) + 1
                r = r < 255u ? r : 255u;
                carry = __shfl_sync(0xffffffffu, r, 0);
                __syncwarp();
                if (i < n) cells[i] = make_cell<S>(v, r);
            }
            __syncwarp();
        }

        // ---- greedy walk (encoder.cpp:25-41) with on-demand matching; lane
        // t % 32 holds token t until the batch of 32 is flushed straight into
        // the chunk's slots (literal symbols read back from the cells).
        // Position 0 and the unaligned positions up to the next multiple of
        // I are literals recorded up to 32 at a time.
        const int I = a.I, W = a.W, min_match = a.min_match;
        uint8_t* pay = a.pay_slots + g * uint64_t(C) * S;
        uint32_t* fl32 = reinterpret_cast<uint32_t*>(a.flag_slots + g * uint64_t(C / 8));
        uint32_t slot = 0, tb = 0, pl = 0, tokv = 0, nptr = 0;
        auto flush = [&](uint32_t cnt) {
            const bool valid = lane < cnt;
            const bool isptr = valid && (tokv >> 31);
            const uint32_t pm = __ballot_sync(0xffffffffu, isptr);
            const uint32_t vm = cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u);
            const uint32_t lm = (1u << lane) - 1u;
            const uint32_t at = pl + 2u * __popc(pm & lm) + uint32_t(S) * __popc(vm & ~pm & lm);
            if (valid) {
                if (isptr) {
                    if constexpr (S == 1) {
                        pay[at] = uint8_t(tokv);
                        pay[at + 1] = uint8_t(tokv >> 8);
                    } else {
                        *reinterpret_cast<uint16_t*>(pay + at) = uint16_t(tokv);
                    }
                    if (a.hist) atomicAdd(&a.hist[tokv & 0xffu], 1ull);
                } else {
                    const uint32_t v = uint32_t(cell_sym<S>(cells[tokv]));
                    if constexpr (S == 1) {
                        pay[at] = uint8_t(v);
                    } else {
                        *reinterpret_cast<uint16_t*>(pay + at) = uint16_t(v);
                        if constexpr (S == 4) *reinterpret_cast<uint16_t*>(pay + at + 2) = uint16_t(v >> 16);
                    }
                }
            }
            if (lane == 0) fl32[tb >> 5] = __byte_perm(__brev(pm), 0u, 0x0123);
            pl += 2u * __popc(pm) + uint32_t(S) * __popc(vm & ~pm);
            nptr += __popc(pm);
        };
        auto push = [&](uint32_t v) {
            if (lane == slot) tokv = v;
            if (++slot == 32u) {
                flush(32u);
                slot = 0;
                tb += 32u;
            }
        };
        auto literals = [&](int from, int to) {
            while (from < to) {
                const uint32_t m = min(uint32_t(to - from), 32u - slot);
                if (lane >= slot && lane < slot + m) tokv = uint32_t(from) + (lane - slot);
                slot += m;
                from += int(m);
                if (slot == 32u) {
                    flush(32u);
                    slot = 0;
                    tb += 32u;
                }
            }
        };
        int p = min(I, n);
        literals(0, p);
        while (p < n) {  // p is a multiple of I here
            const uint32_t key = find_match_warp<S>(cells, p, n, W, lane, list);
            const uint32_t k = key >> 8, o = key & 255u;
            const bool ptr = (o != 0) && (static_cast<int>(k) >= min_match);
            push(ptr ? (0x80000000u | k | (o << 8)) : uint32_t(p));
            p += ptr ? static_cast<int>(k) : 1;
            if (p & (I - 1)) {
                const int q = min((p + I - 1) & ~(I - 1), n);
                literals(p, q);
                p = q;
            }
        }
        if (slot) flush(slot);
        const uint32_t t = tb + slot;
        if (lane == 0) {
            a.psize[g] = pl;
            a.fsize[g] = (t + 7u) >> 3;
        }
        warp_ptr += nptr;
        warp_tok += t;
        __syncwarp();
    }
    if (lane == 0 && warp_tok) {
        atomicAdd(&a.stats[0], warp_ptr);
        atomicAdd(&a.stats[1], warp_tok - warp_ptr);
    }
}

// Full per-position match table of every chunk (matcher.cpp:113-131: aligned
// positions searched, others the forced literal {1, 0}) — the statistics /
// verification path (match_length_histogram raw mode), not the codec.  Same
// staging and find_match_warp as Kernel I; one warp per chunk.
template <int S>
__global__ void __launch_bounds__(512) plz_match_table_kernel(EncodeArgs a, uint8_t* len_out,
                                                              uint8_t* off_out,
                                                              unsigned long long* raw_hist) {
    using T = typename Sym<S>::T;
    using Cell = typename Sym<S>::Cell;
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t lane = lane_id();
    const int C = a.C;
    constexpr uint32_t kHead = kEncodeHeadPerS * S;
    uint8_t* base = smem + encode_warp_smem(C, S) * (threadIdx.x >> 5);
    Cell* cells = reinterpret_cast<Cell*>(base + kHead);
    uint8_t* raw8 = base + kHead + size_t(C) * S;
    uint8_t* list = base + kHead + size_t(C) * sizeof(Cell) + C / 8;
    for (;;) {
        uint64_t g = 0;
        if (lane == 0) g = atomicAdd(a.work, 1u);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= a.n_chunks) break;
        const int n = (g + 1 == a.n_chunks) ? static_cast<int>(a.last_len) : C;
        const uint8_t* src = a.in + g * uint64_t(C) * S;
        for (uint32_t i = lane; i < uint32_t(n) * S; i += 32) raw8[i] = src[i];
        __syncwarp();
        const T* raw = reinterpret_cast<const T*>(raw8);
        for (int w = 0; w <= (n - 1) >> 5; ++w) {
            const int i = (w << 5) + static_cast<int>(lane);
            const T v = i < n ? raw[i] : T(0);
            __syncwarp();
            if (i < n) cells[i] = Cell(v);
            __syncwarp();
        }
        uint32_t carry = 0;
        for (int w = (n - 1) >> 5; w >= 0; --w) {
            const int i = (w << 5) + static_cast<int>(lane);
            const T v = i < n ? cell_sym<S>(cells[i]) : T(0);
            const bool eq = (i + 1 < n) && cell_sym<S>(cells[i + 1]) == v;
            const uint32_t m = __ballot_sync(0xffffffffu, eq);
            const uint32_t sh = m >> lane;
            uint32_t r = sh == (0xffffffffu >> lane) ? (32u - lane) + carry
                                                     : static_cast<uint32_t>(__ffs(~sh));
            r = r < 255u ? r : 255u;
            carry = __shfl_sync(0xffffffffu, r, 0);
            __syncwarp();
            if (i < n) cells[i] = make_cell<S>(v, r);
        }
        __syncwarp();
        const uint64_t out0 = g * uint64_t(C);
        for (int p = 0; p < n; ++p) {
            uint32_t k = 1, o = 0;  // forced literal (matcher.cpp:121-123)
            if ((p & (a.I - 1)) == 0) {
                const uint32_t key = p > 0 ? find_match_warp<S>(cells, p, n, a.W, lane, list) : 0u;
                k = key >> 8;
                o = key & 255u;
                if (k == 0) o = 0;  // {0, 0}: no match (matcher.cpp:109)
            }
            if (lane == 0) {
                len_out[out0 + p] = uint8_t(k);
                off_out[out0 + p] = uint8_t(o);
                if (raw_hist && o != 0 && k > 0) atomicAdd(&raw_hist[k], 1ull);
            }
        }
        __syncwarp();
    }
}

}  // namespace

void launch_match_table(int S, const EncodeArgs& a, int grid, uint8_t* len_out, uint8_t* off_out,
                        unsigned long long* raw_hist, cudaStream_t st) {
    const size_t smem = encode_warp_smem(a.C, S) * a.warps_per_cta;
    const dim3 block(a.warps_per_cta * 32);
    switch (S) {
        case 1:
            plz_match_table_kernel<1><<<grid, block, smem, st>>>(a, len_out, off_out, raw_hist);
            break;
        case 2:
            plz_match_table_kernel<2><<<grid, block, smem, st>>>(a, len_out, off_out, raw_hist);
            break;
        default:
            plz_match_table_kernel<4><<<grid, block, smem, st>>>(a, len_out, off_out, raw_hist);
            break;
    }
}

const void* encode_kernel_for(int S) {
    if (S == 1) return reinterpret_cast<const void*>(plz_encode_kernel<1>);
    if (S == 2) return reinterpret_cast<const void*>(plz_encode_kernel<2>);
    return reinterpret_cast<const void*>(plz_encode_kernel<4>);
}

int encode_ctas_per_sm(int S, int C, int warps_per_cta) {
    int blocks = 0;
    const size_t smem = encode_warp_smem(C, S) * warps_per_cta;
    const void* fn = encode_kernel_for(S);
    if (!smem_fits(fn, smem)) return 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, warps_per_cta * 32, smem);
    return blocks;
}

cudaError_t launch_encode(int S, const EncodeArgs& a, int grid, cudaStream_t st) {
    const size_t smem = encode_warp_smem(a.C, S) * a.warps_per_cta;
    const void* fn = encode_kernel_for(S);
    void* args[] = {const_cast<EncodeArgs*>(&a)};
    return cudaLaunchKernel(fn, dim3(grid), dim3(a.warps_per_cta * 32), args, smem, st);
}

void preload_encode_kernels() {
    for (int S : {1, 2, 4}) preload_kernel(encode_kernel_for(S));
    preload_kernel(reinterpret_cast<const void*>(plz_match_table_kernel<1>));
    preload_kernel(reinterpret_cast<const void*>(plz_match_table_kernel<2>));
    preload_kernel(reinterpret_cast<const void*>(plz_match_table_kernel<4>));
}

}  // namespace plzgpu
