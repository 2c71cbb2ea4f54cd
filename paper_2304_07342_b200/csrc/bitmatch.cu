// bitmatch.cu — Kernel I, bitmap pass: match + greedy token walk + encode,
// one warp per chunk, bit-parallel (shift-and) longest-match search.
//
// Reference contract, identical to encode.cu:
//   matcher.cpp:71-111   longest match over w in [max(0,p-W), p), length
//                        k(w) = min(lcp(w,p), p-w, 255, n-p), ties to the
//                        largest offset (smallest w, strict '>' scanning up);
//   matcher.cpp:113-131  positions with p % I != 0 are forced literals;
//   encoder.cpp:18-73    greedy walk from 0: pointer iff off != 0 and
//                        len >= min_match, MSB-first flag bits, pointer wire
//                        order [len][off], literal = the S raw bytes.
//
// Search as set intersection.  For the position p being searched, number the
// window candidates by bit b = w - (p - W), b in [0, W).  With
//   A_0     = { b : w >= 0 }
//   A_{j+1} = A_j  ∩  { b : x[w + j] == x[p + j] }  ∩  { b : p - w >= j + 1 }
// candidate w has k(w) >= j iff b ∈ A_j, so the match length is the last j
// with A_j non-empty and the reference's tie-break (largest offset) is the
// LOWEST set bit of that A_K.  The middle set is a 256-bit window of the
// occurrence bitmap of symbol x[p+j] — one funnel shift of two shared words
// per 32 candidates — so a step costs O(W/32) word operations whatever the
// data, and the steps of one search sum to the match length: a chunk costs
// O(C * W / 32) word operations in total.
//
// Warp mapping: NW = ceil(W/32) (rounded to 1/2/4/8) lanes hold the NW words
// of a candidate set; the warp's G = 32/NW lane groups evaluate G consecutive
// steps j..j+G-1 at once and an AND prefix over the groups (shfl_up) gives
// A_{j+1..j+G}; one ballot tells how many of them are non-empty.
//
// Occurrence bitmaps need one row per distinct symbol of the chunk (quant
// codes: 3-9 per 2048-symbol chunk).  The chunk's symbols are renamed to
// ids 0..D-1 (first occurrence order).  The first pass keeps 12 rows per
// warp (36 warps/SM at c5, register-bound; 16 rows fitted 30: 2.5 % slower); a chunk with more distinct symbols is listed for
// a second bitmap pass with 32 rows, then a third with 64, and one with more
// than 64 for the wide-cell pass (encode.cu), which handles any alphabet.
#include "common.cuh"

namespace plzgpu {
namespace {

constexpr uint32_t kFull = 0xffffffffu;

// x >> s and x << s with PTX clamping (s >= 32 gives 0).
__device__ __forceinline__ uint32_t shr_clamp(uint32_t x, uint32_t s) {
    uint32_t r;
    asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
    return r;
}
__device__ __forceinline__ uint32_t shl_clamp(uint32_t x, uint32_t s) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(s));
    return r;
}
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}
// Shared-memory loads by 32-bit shared-window address (the search keeps its
// cursors as plain integers; volatile keeps them ordered with the warp's
// other shared-memory traffic).
__device__ __forceinline__ uint32_t lds_u8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// Issue the staging of chunk ck's bytes into raw: one TMA bulk copy (async,
// completes on mbar) when the chunk is 16-byte granular, else a warp copy.
// Waits first (bounded, ~4 s) for the chunk's H2D segment when the
// pipelined host path is active; returns false if it never arrives.
__device__ __forceinline__ bool stage_chunk(const EncodeArgs& a, uint64_t ck, int C, int S,
                                            uint8_t* raw, uint64_t* mbar, uint32_t lane,
                                            bool& async) {
    const int n = (ck + 1 == a.n_chunks) ? static_cast<int>(a.last_len) : C;
    const uint32_t nbytes = uint32_t(n) * S;
    const uint8_t* src = a.in + ck * uint64_t(C) * S;
    if (a.ready) {
        uint32_t ok = 1;
        if (lane == 0) {
            const uint32_t* f = a.ready + ck / a.seg_chunks;
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
        if (!__shfl_sync(kFull, ok, 0)) return false;
    }
    async = a.bulk_ok && (nbytes & 15u) == 0;
    if (async) {
        fence_proxy_async_smem();  // earlier generic reads of raw before the TMA write
        __syncwarp();
        if (lane == 0) bulk_g2s(raw, src, nbytes, mbar);
    } else {
        __syncwarp();
        for (uint32_t i = lane; i < nbytes; i += 32) raw[i] = src[i];
        __syncwarp();
    }
    return true;
}

// Write 32 (or the final cnt) tokens held one per lane: lane l holds token
// t0 + l as 0x80000000 | len | off << 8 (pointer) or its position (literal).
// Payload offsets follow from popcounts (pointer 2 B, literal S B); literal
// symbols come from the id table (lane d of `tab` holds id d's symbol).  The
// flag word is the ballot of pointer lanes, bit-reversed within each byte
// (MSB-first, encoder.cpp:33).
template <int S, int NT>
__device__ __noinline__ void flush_tokens(uint32_t tokv, uint32_t cnt, uint32_t t0,
                                             uint32_t& pl, uint32_t& nptr, const uint32_t (&tab)[NT],
                                             uint32_t s_ids,
                                             uint8_t* pay, uint32_t* fl32, uint32_t lane,
                                             unsigned long long* hist) {
    const bool valid = lane < cnt;
    const bool isptr = valid && (tokv >> 31);
    const uint32_t pm = __ballot_sync(kFull, isptr);
    const uint32_t vm = cnt >= 32 ? kFull : ((1u << cnt) - 1u);
    const uint32_t lm = lanemask_lt();
    const uint32_t at = pl + 2u * __popc(pm & lm) + uint32_t(S) * __popc(vm & ~pm & lm);
    const uint32_t id = (valid && !isptr) ? lds_u8(s_ids + tokv) : 0u;
    uint32_t sym = __shfl_sync(kFull, tab[0], id & 31u);
#pragma unroll
    for (int r = 1; r < NT; ++r) {
        const uint32_t v = __shfl_sync(kFull, tab[r], id & 31u);
        sym = (id >> 5) == uint32_t(r) ? v : sym;
    }
    if (valid) {
        if (isptr) {
            if constexpr (S == 1) {
                pay[at] = uint8_t(tokv);
                pay[at + 1] = uint8_t(tokv >> 8);
            } else {
                *reinterpret_cast<uint16_t*>(pay + at) = uint16_t(tokv);
            }
            if (hist) atomicAdd(&hist[tokv & 0xffu], 1ull);
        } else {
            if constexpr (S == 1) {
                pay[at] = uint8_t(sym);
            } else {
                *reinterpret_cast<uint16_t*>(pay + at) = uint16_t(sym);
                if constexpr (S == 4) *reinterpret_cast<uint16_t*>(pay + at + 2) = uint16_t(sym >> 16);
            }
        }
    }
    if (lane == 0) fl32[t0 >> 5] = __byte_perm(__brev(pm), 0u, 0x0123);
    pl += 2u * __popc(pm) + uint32_t(S) * __popc(vm & ~pm);
    nptr += __popc(pm);
}

// Pass 1: rename the chunk's symbols to ids 0..D-1 (first-occurrence order)
// in place (id i lands on byte i <= S*i, after word i/32 is read), through a
// small open-addressing table; lane d % 32 of the warp keeps id d's symbol in
// tab[d / 32].  New symbols (at most MAXS per chunk, so rare) are inserted
// one distinct value at a time.  Returns false when the chunk has more than
// MAXS distinct symbols.
template <int S, int MAXS>
__device__ __forceinline__ bool rename_symbols(uint8_t* raw, int n, uint2* tbl, uint32_t lane,
                                               int& D, uint32_t (&tab)[(MAXS + 31) / 32]) {
    using T = typename Sym<S>::T;
    constexpr uint32_t kEmpty = 0xffffffffu;
    constexpr int H = bm_hash_slots(MAXS);  // table slots: load factor <= 1/2
    constexpr int HB = H == 8 ? 3 : H == 16 ? 4 : H == 32 ? 5 : H == 64 ? 6 : 7;
    static_assert((1 << HB) == H, "hash size");
#pragma unroll
    for (int i = 0; i < (H + 31) / 32; ++i)
        if (H >= 32 || static_cast<int>(lane) < H) tbl[i * 32 + lane] = make_uint2(0u, kEmpty);
    __syncwarp();
    const T* rs = reinterpret_cast<const T*>(raw);
    D = 0;
#pragma unroll
    for (int r = 0; r < (MAXS + 31) / 32; ++r) tab[r] = 0;
    for (int wi = 0; wi * 32 < n; ++wi) {
        const int i = wi * 32 + static_cast<int>(lane);
        const bool valid = i < n;
        const uint32_t v = valid ? uint32_t(rs[i]) : 0u;
        uint32_t h = (v * 0x9E3779B1u) >> (32 - HB), id = kEmpty;
        if (valid) {
            for (;;) {
                const uint2 e = tbl[h];
                if (e.y == kEmpty) break;
                if (e.x == v) {
                    id = e.y;
                    break;
                }
                h = (h + 1u) & (H - 1);
            }
        }
        const bool missing = valid && id == kEmpty;
        if (__any_sync(kFull, missing)) {
            const uint32_t same = __match_any_sync(kFull, v) & __ballot_sync(kFull, missing);
            uint32_t lead = __ballot_sync(kFull, missing && __ffs(same) - 1 == static_cast<int>(lane));
            while (lead) {
                const int l = __ffs(lead) - 1;
                lead &= lead - 1;
                const uint32_t vl = __shfl_sync(kFull, v, l);
                if (D == MAXS) return false;
                if (lane == 0) {
                    uint32_t hh = (vl * 0x9E3779B1u) >> (32 - HB);
                    while (tbl[hh].y != kEmpty) hh = (hh + 1u) & (H - 1);
                    tbl[hh] = make_uint2(vl, uint32_t(D));
                }
#pragma unroll
                for (int r = 0; r < (MAXS + 31) / 32; ++r)
                    if (static_cast<int>(lane) + 32 * r == D) tab[r] = vl;
                if (missing && v == vl) id = uint32_t(D);
                ++D;
                __syncwarp();
            }
        }
        __syncwarp();  // every lane has read word wi before the in-place stores
        if (valid) raw[i] = uint8_t(id);
    }
    __syncwarp();
    return true;
}

// The chunk's number of distinct symbols, counted exactly up to
// kBmMaxSymsWide + 1, from the input in global memory (the first pass has
// overwritten part of its staged copy with ids).  Lane d % 32 keeps distinct
// symbol d in tab[d / 32]; each word's new values are appended one distinct
// value at a time.
template <int S>
__device__ __noinline__ int count_alphabet(const uint8_t* src, int n, uint32_t lane) {
    uint32_t tab[2] = {0u, 0u};
    int D = 0;
    for (int wi = 0; wi * 32 < n && D <= kBmMaxSymsWide; ++wi) {
        const int i = wi * 32 + static_cast<int>(lane);
        const bool valid = i < n;
        uint32_t v = 0;
        if (valid) {
            if constexpr (S == 1) v = src[i];
            else if constexpr (S == 2) v = uint32_t(src[2 * i]) | uint32_t(src[2 * i + 1]) << 8;
            else v = ld_le32(src + 4 * i);
        }
        const uint32_t same = __match_any_sync(kFull, v) & __ballot_sync(kFull, valid);
        uint32_t lead = __ballot_sync(kFull, valid && __ffs(same) - 1 == static_cast<int>(lane));
        while (lead && D <= kBmMaxSymsWide) {
            const int l = __ffs(lead) - 1;
            lead &= lead - 1;
            const uint32_t vl = __shfl_sync(kFull, v, l);
            const bool hit = __any_sync(kFull, (static_cast<int>(lane) < D && tab[0] == vl) ||
                                                   (static_cast<int>(lane) + 32 < D && tab[1] == vl));
            if (!hit) {
                if (D < 32) {
                    if (static_cast<int>(lane) == D) tab[0] = vl;
                } else if (D < 64) {
                    if (static_cast<int>(lane) == D - 32) tab[1] = vl;
                }
                ++D;
            }
        }
    }
    return D;
}

// Pass 2: occurrence rows from the ids.  Lanes holding equal ids form one
// __match_any_sync group, whose mask IS that id's bitmap word.  Rows 0..D
// are cleared first, with row D's whole reach (the all-zero row of
// position n).
template <int NW>
__device__ __forceinline__ void build_rows(uint8_t* ids, int n, int D, uint32_t* rows, int RW,
                                           uint32_t lane) {
    const int words = (D + 1) * RW + NW + 3;  // bm_rows_words
    for (int x = static_cast<int>(lane); x < words; x += 32) rows[x] = 0u;
    __syncwarp();
    for (int wi = 0; wi * 32 < n; ++wi) {
        const int i = wi * 32 + static_cast<int>(lane);
        const bool valid = i < n;
        const uint32_t id = valid ? uint32_t(ids[i]) : 0xffu;
        const uint32_t same = __match_any_sync(kFull, id);
        if (valid && __ffs(same) - 1 == static_cast<int>(lane)) rows[id * RW + NW + wi] = same;
    }
    // positions n .. n + 127 read the all-zero row D (steps past the chunk end
    // fail; the search's look-ahead reaches at most 3G - 1 <= 95 past n)
    for (int i = static_cast<int>(lane); i < kBmIdPad; i += 32) ids[n + i] = uint8_t(D);
    __syncwarp();
}

template <int S, int NW, int MAXS>
__global__ void __launch_bounds__(kBmMaxThreads) plz_bitmatch_kernel(EncodeArgs a) {
    constexpr int G = 32 / NW;
    constexpr int LNW = NW == 1 ? 0 : NW == 2 ? 1 : NW == 4 ? 2 : 3;
    extern __shared__ __align__(16) uint8_t smem[];

    const uint32_t lane = lane_id();
    const uint32_t warp = threadIdx.x >> 5;
    const int C = a.C, W = a.W;
    const int RW = bm_row_words(C, W);
    // [mbarrier 16][hash table][region: raw chunk -> ids [0, C) + rows at C]
    uint8_t* base = smem + bm_warp_smem(C, S, W, MAXS) * warp;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(base);
    uint2* tbl = reinterpret_cast<uint2*>(base + 16);
    uint8_t* raw = base + 16 + bm_hash_slots(MAXS) * 8;
    uint8_t* ids = raw;
    uint32_t* rows = reinterpret_cast<uint32_t*>(raw + C + kBmIdPad);

    if (lane == 0) mbar_init(mbar, 1);
    __syncwarp();
    uint32_t phase = 0;
    unsigned long long warp_ptr = 0, warp_tok = 0;

    const int grp = static_cast<int>(lane) >> LNW;  // step group
    const int jw = static_cast<int>(lane) & (NW - 1);  // word of the candidate set
    const int clg = 32 * (jw + 1) - W + grp;       // step-(k+grp) mask: ~0 >> max(clg + k, 0)
    const int qc = 32 * NW - W + 32 * jw + grp;    // row bit of candidate word jw at step grp: p + qc + k
    const int lbc = W - 32 * jw;                   // w >= 0  <=>  bit >= lbc - p
    const int Im1 = a.I - 1;
    const uint32_t min_match = uint32_t(a.min_match);

    for (;;) {
        uint64_t ck = 0;
        if (lane == 0) {
            const uint32_t idx = atomicAdd(a.work, 1u);
            if (!a.src_list) ck = idx;
            else ck = idx < *a.src_count ? a.src_list[idx] : a.n_chunks;
        }
        ck = __shfl_sync(kFull, ck, 0);
        if (ck >= a.n_chunks) break;
        const int n = (ck + 1 == a.n_chunks) ? static_cast<int>(a.last_len) : C;
        bool async = false;
        if (!stage_chunk(a, ck, C, S, raw, mbar, lane, async)) break;
        if (async) {
            mbar_wait(mbar, phase);
            phase ^= 1u;
        }

        int D;
        uint32_t tab[(MAXS + 31) / 32];
        if (!rename_symbols<S, MAXS>(raw, n, tbl, lane, D, tab)) {
            // too many distinct symbols: the wide-cell pass takes this chunk
            int cls = 0;
            if (MAXS == kBmMaxSyms && a.classify) {
                const int D2 = count_alphabet<S>(a.in + ck * uint64_t(C) * S, n, lane);
                cls = D2 <= kBmMaxSymsMid ? 0 : D2 <= kBmMaxSymsWide ? 1 : 2;
            }
            if (lane == 0) a.fb_list[cls][atomicAdd(a.fb_count[cls], 1u)] = uint32_t(ck);
            __syncwarp();
            continue;
        }
        build_rows<NW>(ids, n, D, rows, RW, lane);

        // ---- greedy walk (encoder.cpp:25-41); lane t % 32 holds token t
        // until the batch of 32 is flushed straight into the chunk's slots.
        // Runs of literals the walk cannot avoid — position 0 (empty window)
        // and the unaligned positions up to the next multiple of I (forced
        // literals, matcher.cpp:121-123) — are recorded up to 32 at a time.
        uint8_t* pay = a.pay_slots + ck * uint64_t(C) * S;
        uint32_t* fl32 = reinterpret_cast<uint32_t*>(a.flag_slots + ck * uint64_t(C / 8));
        const uint32_t s_ids = static_cast<uint32_t>(__cvta_generic_to_shared(ids));
        const uint32_t s_rows = static_cast<uint32_t>(__cvta_generic_to_shared(rows));
        uint32_t slot = 0, tb = 0, pl = 0, tokv = 0, nptr = 0;
        auto literals = [&](int from, int to) {  // positions [from, to) as literal tokens
            while (from < to) {
                const uint32_t m = min(uint32_t(to - from), 32u - slot);
                if (lane >= slot && lane < slot + m) tokv = uint32_t(from) + (lane - slot);
                slot += m;
                from += int(m);
                if (slot == 32u) {
                    flush_tokens<S, (MAXS + 31) / 32>(tokv, 32u, tb, pl, nptr, tab, s_ids, pay,
                                                      fl32, lane, a.hist);
                    slot = 0;
                    tb += 32u;
                }
            }
        };
        int p = min(Im1 + 1, n);
        literals(0, p);
        while (p < n) {  // p is a multiple of I here
            uint32_t K = 0, off = 0;
            {
                // bit b of word jw <-> candidate w = p - W + 32*jw + b.
                // Step k + grp reads the id of position p + k + grp (the ids
                // past n are D: the zero row) and the row bits from
                // p + qc + k; the next round's ids are loaded a round ahead.
                uint32_t A = shl_clamp(kFull, uint32_t(max(lbc - p, 0)));
                uint32_t x, nz;
                int q = p + qc;               // row bit cursor (advances G per round)
                const int mk = clg - q;       // mask shift of the round: max(mk + q, 0)
                const uint32_t ib = s_ids + uint32_t(p + grp) - uint32_t(q);  // + q: step's id
                const int q0 = q;
                uint32_t id = lds_u8(ib + uint32_t(q));
                uint32_t idn = lds_u8(ib + uint32_t(q + G));
#pragma unroll 2
                for (;;) {
                    const uint32_t ra = s_rows + id * uint32_t(RW * 4) + uint32_t((q >> 5) << 2);
                    const uint32_t lo = lds_u32(ra), hi = lds_u32(ra + 4);
                    id = idn;
                    idn = lds_u8(ib + uint32_t(q + 2 * G));
                    const uint32_t f = __funnelshift_r(lo, hi, uint32_t(q));
                    x = f & shr_clamp(kFull, uint32_t(max(mk + q, 0))) & A;
#pragma unroll
                    for (int d = 1; d < G; d <<= 1) x &= __shfl_up_sync(kFull, x, d * NW);
                    nz = __ballot_sync(kFull, x != 0u);
                    const uint32_t An = __shfl_sync(kFull, x, (G - 1) * NW + jw);
                    if ((nz >> (32 - NW)) == 0u) break;  // the search ends in this round
                    A = An;
                    q += G;
                }
                // steps matched in the last round: groups with non-empty sets
                const int e = (static_cast<int>(31 - __clz(nz)) + NW) >> LNW;  // nz == 0 -> 0
                K = uint32_t(q - q0 + e);
                if (K >= min_match) {
                    // winner: lowest set bit of A_K (group e-1 of x, or A)
                    const uint32_t val = e > 0 ? x : A;
                    const int gsel = e > 0 ? e - 1 : 0;
                    const uint32_t c = (grp == gsel && val != 0u)
                                           ? uint32_t(32 * jw + __ffs(val) - 1) : kFull;
                    off = uint32_t(W) - __reduce_min_sync(kFull, c);
                }
            }
            const bool ptr = K >= min_match;
            if (lane == slot) tokv = ptr ? (0x80000000u | K | (off << 8)) : uint32_t(p);
            p += ptr ? static_cast<int>(K) : 1;
            if (++slot == 32u) {
                flush_tokens<S, (MAXS + 31) / 32>(tokv, 32u, tb, pl, nptr, tab, s_ids, pay, fl32, lane, a.hist);
                slot = 0;
                tb += 32u;
            }
            if (p & Im1) {  // forced literals up to the next aligned position
                if ((p & Im1) == Im1 && p < n) {  // exactly one (always, for I = 2)
                    if (lane == slot) tokv = uint32_t(p);
                    ++p;
                    if (++slot == 32u) {
                        flush_tokens<S, (MAXS + 31) / 32>(tokv, 32u, tb, pl, nptr, tab, s_ids, pay,
                                                          fl32, lane, a.hist);
                        slot = 0;
                        tb += 32u;
                    }
                } else {
                    const int q = min((p + Im1) & ~Im1, n);
                    literals(p, q);
                    p = q;
                }
            }
        }
        if (slot) flush_tokens<S, (MAXS + 31) / 32>(tokv, slot, tb, pl, nptr, tab, s_ids, pay, fl32, lane, a.hist);
        const uint32_t t = tb + slot;
        if (lane == 0) {
            a.psize[ck] = pl;
            a.fsize[ck] = (t + 7u) >> 3;
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

template <int S, int MAXS>
const void* bitmatch_fn_s(int nw) {
    switch (nw) {
        case 1: return reinterpret_cast<const void*>(plz_bitmatch_kernel<S, 1, MAXS>);
        case 2: return reinterpret_cast<const void*>(plz_bitmatch_kernel<S, 2, MAXS>);
        case 4: return reinterpret_cast<const void*>(plz_bitmatch_kernel<S, 4, MAXS>);
        default: return reinterpret_cast<const void*>(plz_bitmatch_kernel<S, 8, MAXS>);
    }
}

template <int MAXS>
const void* bitmatch_fn_m(int S, int nw) {
    if (S == 1) return bitmatch_fn_s<1, MAXS>(nw);
    if (S == 2) return bitmatch_fn_s<2, MAXS>(nw);
    return bitmatch_fn_s<4, MAXS>(nw);
}

// Latency mode's classification: one warp per chunk (grid-stride).  Bytes
// (S = 1) are counted with a 256-bit presence bitmap in shared memory; wider
// symbols with count_alphabet.
template <int S>
__global__ void __launch_bounds__(128) plz_classify_kernel(EncodeArgs a, uint32_t* lists,
                                                           uint64_t stride, uint32_t* counts) {
    __shared__ uint32_t seen[4][8];
    __shared__ uint32_t lane_seen[4][8 * 32];  // per lane: 256-bit presence set, word w at [w * 32 + lane]
    const uint32_t lane = lane_id();
    uint32_t* bm = seen[threadIdx.x >> 5];
    const uint32_t s_ls = static_cast<uint32_t>(__cvta_generic_to_shared(lane_seen[threadIdx.x >> 5])) + 4u * lane;
    const uint64_t warps = uint64_t(gridDim.x) * (blockDim.x >> 5);
    for (uint64_t ck = uint64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
         ck < a.n_chunks; ck += warps) {
        const int n = (ck + 1 == a.n_chunks) ? static_cast<int>(a.last_len) : a.C;
        int D;
        if constexpr (S == 1) {
            if (lane < 8) bm[lane] = 0u;
            __syncwarp();
            const uint8_t* src = a.in + ck * uint64_t(a.C);
            if (n == a.C && n <= 4096 && a.bulk_ok) {
                // whole chunk of at most 4 KiB, 16-byte aligned: every lane's
                // 16-byte words loaded up front (one memory round trip per
                // chunk), each lane's bytes into its own 256-bit set in shared
                // memory (conflict-free: word w of lane l at w * 32 + l; no
                // warp-wide match per byte), the 32 sets OR-reduced at the end
#pragma unroll
                for (int w = 0; w < 8; ++w)
                    asm volatile("st.shared.u32 [%0], %1;" ::"r"(s_ls + 128u * w), "r"(0u) : "memory");
                uint4 v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (512 * k < n) v[k] = *reinterpret_cast<const uint4*>(src + 512 * k + 16 * lane);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (512 * k >= n) break;
                    const uint32_t w4[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
                    for (int b = 0; b < 16; ++b) {
                        const uint32_t x = (w4[b >> 2] >> (8 * (b & 3))) & 0xffu;
                        const uint32_t ad = s_ls + 128u * (x >> 5);
                        uint32_t m;
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(m) : "r"(ad) : "memory");
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(ad), "r"(m | (1u << (x & 31u))) : "memory");
                    }
                }
                uint32_t tot = 0;
#pragma unroll
                for (int w = 0; w < 8; ++w) {
                    uint32_t m;
                    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(m) : "r"(s_ls + 128u * w) : "memory");
                    tot += __popc(__reduce_or_sync(0xffffffffu, m));
                }
                D = int(tot);
            } else {
                for (int base = 0; base < n; base += 128) {  // uniform trip count (match_any)
                    const int i = base + 4 * static_cast<int>(lane);
                    uint32_t v;
                    if (i + 4 <= n && a.bulk_ok) {  // the input base is 16-byte aligned
                        v = *reinterpret_cast<const uint32_t*>(src + i);
                    } else {  // past the chunk: repeat its first byte, a no-op for the set
                        v = 0;
                        for (int b = 0; b < 4; ++b) v |= uint32_t(i + b < n ? src[i + b] : src[0]) << (8 * b);
                    }
#pragma unroll
                    for (int b = 0; b < 4; ++b) {  // one atomic per distinct value of the warp
                        const uint32_t x = (v >> (8 * b)) & 0xffu;
                        const uint32_t same = __match_any_sync(0xffffffffu, x);
                        if (__ffs(same) - 1 == static_cast<int>(lane)) atomicOr(&bm[x >> 5], 1u << (x & 31u));
                    }
                }
                __syncwarp();
                D = int(__reduce_add_sync(0xffffffffu, lane < 8 ? __popc(bm[lane]) : 0u));
            }
            __syncwarp();
        } else {
            D = count_alphabet<S>(a.in + ck * uint64_t(a.C) * S, n, lane);
        }
        const int k = D <= kBmMaxSymsTiny ? 0 : D <= kBmMaxSyms ? 1 : D <= kBmMaxSymsMid ? 2
                    : D <= kBmMaxSymsWide ? 3 : 4;
        if (lane == 0) lists[uint64_t(k) * stride + atomicAdd(&counts[k], 1u)] = uint32_t(ck);
    }
}

const void* bitmatch_fn(int S, int W, int maxsyms) {
    const int nw = bm_nw(W);
    if (maxsyms == kBmMaxSymsTiny) return bitmatch_fn_m<kBmMaxSymsTiny>(S, nw);
    return maxsyms == kBmMaxSyms      ? bitmatch_fn_m<kBmMaxSyms>(S, nw)
           : maxsyms == kBmMaxSymsMid ? bitmatch_fn_m<kBmMaxSymsMid>(S, nw)
                                      : bitmatch_fn_m<kBmMaxSymsWide>(S, nw);
}

}  // namespace

int bitmatch_ctas_per_sm(int S, int C, int W, int maxsyms, int warps_per_cta) {
    int blocks = 0;
    const size_t smem = bm_warp_smem(C, S, W, maxsyms) * warps_per_cta;
    const void* fn = bitmatch_fn(S, W, maxsyms);
    if (!smem_fits(fn, smem)) return 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, warps_per_cta * 32, smem);
    return blocks;
}

cudaError_t launch_bitmatch(int S, int maxsyms, const EncodeArgs& a, int grid, cudaStream_t st) {
    const size_t smem = bm_warp_smem(a.C, S, a.W, maxsyms) * a.warps_per_cta;
    const void* fn = bitmatch_fn(S, a.W, maxsyms);
    void* args[] = {const_cast<EncodeArgs*>(&a)};
    return cudaLaunchKernel(fn, dim3(grid), dim3(a.warps_per_cta * 32), args, smem, st);
}

void launch_classify(int S, const EncodeArgs& a, uint32_t* lists, uint64_t stride, uint32_t* counts,
                     int grid, cudaStream_t st) {
    if (S == 1) plz_classify_kernel<1><<<grid, 128, 0, st>>>(a, lists, stride, counts);
    else if (S == 2) plz_classify_kernel<2><<<grid, 128, 0, st>>>(a, lists, stride, counts);
    else plz_classify_kernel<4><<<grid, 128, 0, st>>>(a, lists, stride, counts);
}

void preload_bitmatch_kernels() {
    for (int S : {1, 2, 4})
        for (int W : {16, 48, 96, 255})
            for (int m : {kBmMaxSymsTiny, kBmMaxSyms, kBmMaxSymsMid, kBmMaxSymsWide})
                preload_kernel(bitmatch_fn(S, W, m));
    preload_kernel(reinterpret_cast<const void*>(plz_classify_kernel<1>));
    preload_kernel(reinterpret_cast<const void*>(plz_classify_kernel<2>));
    preload_kernel(reinterpret_cast<const void*>(plz_classify_kernel<4>));
}

}  // namespace plzgpu
