// decode.cu — container parse + block-parallel chunk decode.
//
// Reference: format.cpp:112-185 (read_container: every structural check, in
// order, with byte offsets relative to the container), decoder.cpp:22-90
// (walk_tokens / decompress_chunk: MSB-first flags, [len][off] pointers,
// forward overlapping copies, typed errors in walk order) and
// decoder.cpp:102-141 (containers back to back, chunk k written at k*C*S,
// tail appended).
//
// plz_parse_kernel: one CTA walks the container chain on the device (header
// fields by one thread, table monotonicity by the whole CTA with a min-reduce
// that keeps the reference's "first failing entry, payload before flag"
// order) and emits one descriptor per container.  No host round trip.
//
// plz_decode_kernel: persistent grid, one warp per chunk.  A chunk is decoded
// 32 tokens at a time: each lane takes one token's flag bit, warp scans turn
// token kinds into payload offsets and token lengths into output positions,
// the first failing token is found with a ballot, literals are scattered in
// parallel and pointers replayed in token order (lanes copy one pointer's
// symbols together; a malformed len > off replicates with period off, the
// forward-copy semantics of decoder.cpp:80-84).  Chunks up to 8 KiB decode in
// shared memory and leave with 128-bit stores.
#include "common.cuh"

namespace plzgpu {
namespace {

constexpr int kDecodeWarps = 4;
constexpr uint32_t kDecodeSmem = 4096;  // bytes of output staging per warp (4 KiB chunks;
                                        // larger chunks decode in global memory)
// + pad (a wave writes up to 31 positions past its batch's span) + token
// table (128 B) + start bitmap of a batch's span (one bit per output
// position: kDecodeSmem / 32 words cover any chunk that decodes in shared
// memory)
constexpr uint32_t kDecodePad = 128;
constexpr uint32_t kDecodeWarpSmem = kDecodeSmem + kDecodePad + 144 + kDecodeSmem / 8;
// The decode kernel's per-warp region (decode_chunk_fast): output stage
// (kDecodeSmem bytes), token table (one byte per token: a pointer's offset,
// 0 for a literal; fast_tokens<S>() entries — a chunk with more flag bits
// than that takes decode_chunk_smem), wave table (per 32 output positions:
// token-start bitmap + address of the token before the wave; read two
// entries at a time, so one spare entry).
constexpr uint32_t kFastTokens = 1024;  // S = 1 (c5 chunks carry at most ~600 tokens); the
                                        // region for 1024 and 9 CTAs/SM measured +2.9 % on c5
                                        // against 2048 and 8
constexpr uint32_t kFastPtab = kDecodeSmem;
constexpr uint32_t kFastMeta = kFastPtab + kFastTokens;
// the fast path serves chunks of at most kDecodeSmem bytes: up to 4096 output
// positions (S = 1), 128 waves
constexpr uint32_t kFastWaves = kDecodeSmem / 32;  // S = 1: 4096 positions
constexpr uint32_t kFastWarpSmem = kFastMeta + 8 * kFastWaves + 16;  // + the spare table pair
// Per width, the wave table needs only kDecodeSmem / (32 S) entries; the
// token table takes the rest of the region (S = 2: 1536 tokens, so chunks of
// up to 75 % literals — I = 16 streams — stay on the fast path; S = 1: 1024).
// The spare pair after a width's last wave also takes phase A's dump bits.
template <int S>
__host__ __device__ constexpr uint32_t fast_waves() { return kDecodeSmem / (32u * S); }
template <int S>
__host__ __device__ constexpr uint32_t fast_tokens() {
    return kFastWarpSmem - 16u - 8u * fast_waves<S>() - kFastPtab;
}
static_assert(fast_tokens<1>() == kFastTokens && fast_tokens<2>() == 1536u, "fast layout");
static_assert((kFastPtab + fast_tokens<2>()) % 16u == 0 && (kFastPtab + fast_tokens<4>()) % 16u == 0,
              "wave table alignment (read as uint4 pairs)");
static_assert(kFastWarpSmem >= kDecodeWarpSmem, "the exact path shares the warp's region");
constexpr bool kUseFast = true;
constexpr uint32_t kMainWarpSmem = kUseFast ? kFastWarpSmem : kDecodeWarpSmem;

__device__ __forceinline__ uint32_t warp_incl_scan_u32(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= uint32_t(d)) v += x;
    }
    return v;
}

// Output symbols of a chunk: aligned T elements, or byte-wise when the
// destination is not S-aligned (containers after a tailed one in a
// concatenated image).
template <int S, bool kBytes>
struct SymOut {
    using T = typename Sym<S>::T;
    uint8_t* p;
    __device__ __forceinline__ T load(uint64_t i) const {
        if constexpr (kBytes) {
            T v = 0;
#pragma unroll
            for (int b = 0; b < S; ++b) v |= T(p[i * S + b]) << (8 * b);
            return v;
        } else {
            return reinterpret_cast<const T*>(p)[i];
        }
    }
    __device__ __forceinline__ void store(uint64_t i, T v) const {
        if constexpr (kBytes) {
#pragma unroll
            for (int b = 0; b < S; ++b) p[i * S + b] = uint8_t(v >> (8 * b));
        } else {
            reinterpret_cast<T*>(p)[i] = v;
        }
    }
};

// Source position (relative) of position rel inside pointer entry e:
// relpos - off + ((rel - relpos) mod off), i.e. rel - off for well-formed
// pointers and LZ77-style replication when len > off (decoder.cpp:80-84).
__device__ __forceinline__ int source_of(uint32_t e, uint32_t rel) {
    const uint32_t rp = e >> 16, off = e & 0xffu;
    uint32_t d = rel - rp;
    if (d >= off) d %= off;  // only malformed pointers (len > off) replicate
    return int(rp) - int(off) + int(d);
}

// Token walk of one chunk by one warp; decoded symbols go to out[0, L).
// Returns a TokenErr and the failing token index (decoder.cpp:22-66 order).
//
// 32 tokens per batch: lane j takes token t+j's flag bit; warp scans turn
// token kinds into payload offsets and token lengths into output positions;
// the first failing token is found with a ballot.  Literals are written, then
// the batch's output positions are filled in 32-wide waves: a pointer
// position copies from its source, chasing back through pointers of the same
// wave (earlier waves and literals are already final).  `tab` is the warp's
// 33-entry token table in shared memory: relpos << 16 | is_ptr << 8 | off.
template <int S, bool kBytes>
__device__ uint32_t decode_chunk_warp(const uint8_t* __restrict__ flags, uint64_t nf,
                                      const uint8_t* __restrict__ pay, uint64_t np, uint64_t L,
                                      SymOut<S, kBytes> out, uint32_t* tab, uint32_t lane,
                                      uint64_t* err_tok) {
    using T = typename Sym<S>::T;
    uint64_t written = 0, in = 0, t = 0;
    while (written < L) {
        const uint64_t tt = t + lane;
        const bool hf = (tt >> 3) < nf;
        const uint32_t bit = hf ? (uint32_t(flags[tt >> 3]) >> (7u - uint32_t(tt & 7u))) & 1u : 0u;
        const uint32_t sz = bit ? 2u : uint32_t(S);
        // payload offset = 2 * (pointers before) + S * (literals before)
        const uint32_t below = (1u << lane) - 1u;
        const uint32_t nptr = __popc(__ballot_sync(0xffffffffu, bit) & below);
        const uint64_t pin = in + 2u * nptr + uint32_t(S) * (lane - nptr);
        const bool has = pin + sz <= np;
        uint32_t len = 0, off = 0;
        if (bit && has) {
            len = pay[pin];
            off = pay[pin + 1];
        }
        const uint32_t adv = bit ? len : 1u;
        const uint32_t rel = warp_incl_scan_u32(adv, lane) - adv;  // < 32*255
        const uint64_t pos = written + rel;
        const bool reached = pos < L;
        uint32_t e = TE_OK;
        if (!hf) e = TE_FLAGS_EXHAUSTED;
        else if (!has) e = TE_PAYLOAD_EXHAUSTED;
        else if (bit) {
            if (len == 0 || off == 0) e = TE_ZERO_FIELD;
            else if (off > pos) e = TE_OFFSET_BEFORE_START;
            else if (pos + len > L) e = TE_OVERRUN;
        }
        const uint32_t m_end = __ballot_sync(0xffffffffu, !reached);
        const uint32_t m_err = __ballot_sync(0xffffffffu, e != TE_OK && reached);
        const uint32_t first_end = m_end ? uint32_t(__ffs(m_end) - 1) : 32u;
        const uint32_t first_err = m_err ? uint32_t(__ffs(m_err) - 1) : 32u;
        if (first_err < first_end) {
            *err_tok = t + first_err;
            return __shfl_sync(0xffffffffu, e, first_err);
        }
        const bool act = lane < first_end;
        if (act && !bit) {
            T v = 0;
#pragma unroll
            for (int b = 0; b < S; ++b) v |= T(pay[pin + b]) << (8 * b);
            out.store(pos, v);
        }
        const uint32_t la = first_end - 1;
        const uint32_t span = __shfl_sync(0xffffffffu, rel + adv, la);
        const uint32_t pm = __ballot_sync(0xffffffffu, act && bit);
        if (pm) {
            tab[lane] = (rel << 16) | (bit << 8) | off;
            __syncwarp();
            for (uint32_t wbase = 0; wbase < span; wbase += 32) {
                // covering token of wave position i: (tokens starting before the
                // wave) + (token starts at <= i inside it) - 1
                const uint32_t before =
                    __popc(__ballot_sync(0xffffffffu, act && rel < wbase));
                const uint32_t starts = __reduce_or_sync(
                    0xffffffffu, (act && rel >= wbase && rel - wbase < 32u) ? 1u << (rel - wbase) : 0u);
                const uint32_t q = wbase + lane;
                if (q < span) {
                    const uint32_t ent = tab[before + __popc(starts & ((2u << lane) - 1u)) - 1u];
                    if (ent & 0x100u) {
                        int src = source_of(ent, q);
                        while (src >= int(wbase)) {  // source in this wave: chase it back
                            const uint32_t i = uint32_t(src) - wbase;
                            const uint32_t e2 = tab[before + __popc(starts & ((2u << i) - 1u)) - 1u];
                            if (!(e2 & 0x100u)) break;  // a literal: already written
                            src = source_of(e2, uint32_t(src));
                        }
                        out.store(written + q, out.load(uint64_t(int64_t(written) + src)));
                    }
                }
                __syncwarp();
            }
        } else {
            __syncwarp();
        }
        written += span;
        in = __shfl_sync(0xffffffffu, pin + sz, la);
        t += first_end;
    }
    if (in != np) {
        *err_tok = t;
        return TE_TRAILING_PAYLOAD;
    }
    // padding bits after the last token must be zero (decoder.cpp:61-63)
    const uint64_t b0 = t >> 3;
    for (uint64_t base = b0; base < nf; base += 32) {
        const uint64_t bi = base + lane;
        uint32_t v = bi < nf ? flags[bi] : 0u;
        if (bi == b0) v &= 0xffu >> uint32_t(t & 7u);
        const uint32_t m = __ballot_sync(0xffffffffu, v != 0u);
        if (m) {
            const int l = __ffs(m) - 1;
            const uint32_t vv = __shfl_sync(0xffffffffu, v, l);
            *err_tok = 8 * (base + uint64_t(l)) + uint64_t(__clz(vv) - 24);
            return TE_NONZERO_PADDING;
        }
    }
    if (nf != ((t + 7) >> 3)) {
        *err_tok = t;
        return TE_FLAG_COUNT;
    }
    return TE_OK;
}

// Shared-memory symbol access by 32-bit shared-window address.
template <int S>
__device__ __forceinline__ uint32_t lds_sym(uint32_t a) {
    uint32_t v;
    if constexpr (S == 1) asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    else if constexpr (S == 2) asm volatile("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(a));
    else asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
template <int S>
__device__ __forceinline__ void sts_sym(uint32_t a, uint32_t v) {
    if constexpr (S == 1) asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v));
    else if constexpr (S == 2) asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "r"(v));
    else asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// One aligned payload word per lane: the window [base, base + 128) with
// base = (pay + in) rounded down to 4.  A word is read only if it starts
// inside the stream (an aligned word holding a stream byte never leaves the
// allocation).
__device__ __forceinline__ uint32_t load_window(const uint8_t* pay, uint32_t np, uint32_t in,
                                                uint32_t lane) {
    const uintptr_t a = (reinterpret_cast<uintptr_t>(pay + in) & ~uintptr_t(3)) + 4u * lane;
    return a < reinterpret_cast<uintptr_t>(pay + np) ? *reinterpret_cast<const uint32_t*>(a) : 0u;
}

// decode_chunk_warp for the common case — the chunk's output fits the warp's
// shared-memory stage — with chunk-local 32-bit positions and shared-window
// addresses.  Same token semantics and error order.  Per batch of 32 tokens:
// literals are stored straight away; token starts are OR-ed into a bitmap of
// the batch's span (one bit per output position), so in each 32-position wave
// a lane finds its covering token with one popcount.  A pointer position q
// copies from q - off (the forward byte copy of decoder.cpp:80-84: for a
// malformed len > off the source lies inside the same token and the chase
// follows it back), chasing sources in the same wave back to a literal or an
// earlier wave.
template <int S>
__device__ uint32_t decode_chunk_smem(const uint8_t* __restrict__ flags, uint32_t nf,
                                      const uint8_t* __restrict__ pay, uint32_t np, uint32_t L,
                                      uint32_t s_out, uint32_t s_tab, uint32_t* bm,
                                      uint32_t lane, uint64_t* err_tok) {
    uint32_t written = 0, in = 0, t = 0;
    const uint32_t below = (1u << lane) - 1u, upto = (2u << lane) - 1u;
    const uint32_t s_bm = static_cast<uint32_t>(__cvta_generic_to_shared(bm));
    // Each batch's flag byte and a 128-byte payload window (one aligned word
    // per lane) are loaded one batch ahead, before the previous batch's
    // waves, so their latency overlaps the copies.  A batch consumes at most
    // 32 * max(S, 2) <= 128 payload bytes; a token that falls off the window
    // (S = 4, almost all literals) reads global memory directly.
    uint32_t fbyte = (lane >> 3) < nf ? flags[lane >> 3] : 0u;
    uint32_t win = load_window(pay, np, 0, lane);
    while (written < L) {
        const uint32_t tt = t + lane;
        const bool hf = (tt >> 3) < nf;
        const uint32_t bit = hf ? (fbyte >> (7u - (tt & 7u))) & 1u : 0u;
        const uint32_t pmask = __ballot_sync(0xffffffffu, bit);
        const uint32_t nptr = __popc(pmask & below);
        const uint32_t pin = in + 2u * nptr + uint32_t(S) * (lane - nptr);
        const uint32_t sz = bit ? 2u : uint32_t(S);
        const bool has = pin + sz <= np;
        const uint32_t o = pin - in + uint32_t(reinterpret_cast<uintptr_t>(pay + in) & 3u);
        const uint32_t wa = __shfl_sync(0xffffffffu, win, (o >> 2) & 31u);
        const uint32_t wb = __shfl_sync(0xffffffffu, win, ((o >> 2) + 1u) & 31u);
        uint32_t v = __funnelshift_r(wa, wb, 8u * (o & 3u));
        uint32_t len = 0, off = 0, lit = 0;
        if (has) {
            if (o + sz > 128u) {
                v = 0;
#pragma unroll
                for (int b = 0; b < (S > 2 ? S : 2); ++b)
                    if (uint32_t(b) < sz) v |= uint32_t(pay[pin + b]) << (8 * b);
            }
            if (bit) {
                len = v & 0xffu;
                off = (v >> 8) & 0xffu;
            } else {
                lit = S == 4 ? v : v & ((1u << (8 * S)) - 1u);
            }
        }
        const uint32_t adv = bit ? len : 1u;
        const uint32_t incl = warp_incl_scan_u32(adv, lane);
        const uint32_t rel = incl - adv;  // < 32*255
        const uint32_t pos = written + rel;
        const bool reached = pos < L;
        const bool bad = !hf || !has || (bit && (len == 0 || off == 0 || off > pos || pos + len > L));
        const uint32_t m_end = __ballot_sync(0xffffffffu, !reached);
        const uint32_t first_end = m_end ? uint32_t(__ffs(m_end) - 1) : 32u;
        const uint32_t m_err = __ballot_sync(0xffffffffu, bad && reached);
        if (m_err && uint32_t(__ffs(m_err) - 1) < first_end) {
            // the first failing token, classified in decoder.cpp:22-66 order
            uint32_t e = TE_OK;
            if (!hf) e = TE_FLAGS_EXHAUSTED;
            else if (!has) e = TE_PAYLOAD_EXHAUSTED;
            else if (bit) {
                if (len == 0 || off == 0) e = TE_ZERO_FIELD;
                else if (off > pos) e = TE_OFFSET_BEFORE_START;
                else if (pos + len > L) e = TE_OVERRUN;
            }
            const uint32_t first_err = uint32_t(__ffs(m_err) - 1);
            *err_tok = uint64_t(t) + first_err;
            return __shfl_sync(0xffffffffu, e, first_err);
        }
        const bool act = lane < first_end;
        if (act && !bit) sts_sym<S>(s_out + pos * S, lit);
        const uint32_t la = first_end - 1;
        const uint32_t span = __shfl_sync(0xffffffffu, incl, la);
        in = __shfl_sync(0xffffffffu, pin + sz, la);
        t += first_end;
        if (written + span < L) {  // the next batch's loads
            const uint32_t fi = (t + lane) >> 3;
            fbyte = fi < nf ? flags[fi] : 0u;
            win = load_window(pay, np, in, lane);
        }
        if (pmask & (first_end >= 32u ? 0xffffffffu : (1u << first_end) - 1u)) {
            // token table: -off for a pointer, 0 for a literal (its positions
            // then copy onto themselves)
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(s_tab + 4u * lane),
                         "r"(bit ? 0u - off : 0u));
            const uint32_t nw = (span + 31u) >> 5;
#pragma unroll 1
            for (uint32_t w = lane; w < nw; w += 32) bm[w] = 0u;
            __syncwarp();
            if (act) atomicOr(&bm[rel >> 5], 1u << (rel & 31u));
            __syncwarp();
            // Waves: every lane copies out[q] = out[src].  Positions past the
            // span (at most 31) land in the stage's pad or in positions a
            // later batch rewrites.
            const uint32_t s_w = s_out + written * S;
            const uint32_t s_tb = s_tab - 4u;  // index before + popc - 1
            uint32_t before = 0;  // batch tokens starting before the wave
            uint32_t a_bm = s_bm;                       // start-bitmap word of the wave
            uint32_t a_q = s_w + lane * uint32_t(S);    // this lane's output slot
#pragma unroll 1
            for (uint32_t w = 0; w < nw; ++w) {
                const uint32_t starts = lds32(a_bm);
                const int tv = int(lds32(s_tb + 4u * (before + __popc(starts & upto))));
                // in-wave index of the source (< 0: an earlier wave, final).  A
                // source inside the wave (0 < off <= lane) on a pointer position
                // is not final yet: the lane follows the chain itself through
                // the same lookups until a literal or an earlier wave
                int src = int(lane) + tv;
                if (tv != 0 && src >= 0) {
                    for (;;) {
                        const int t2 = int(lds32(s_tb + 4u * (before + __popc(starts & ((2u << src) - 1u)))));
                        if (t2 == 0) break;  // a literal: written above
                        src += t2;
                        if (src < 0) break;
                    }
                }
                sts_sym<S>(a_q, lds_sym<S>(uint32_t(int(a_q) + (src - int(lane)) * S)));
                before += __popc(starts);
                a_bm += 4u;
                a_q += 32u * S;
                __syncwarp();
            }
        }
        written += span;
    }
    if (in != np) {
        *err_tok = t;
        return TE_TRAILING_PAYLOAD;
    }
    // padding bits after the last token must be zero (decoder.cpp:61-63)
    const uint32_t b0 = t >> 3;
    for (uint32_t base = b0; base < nf; base += 32) {
        const uint32_t bi = base + lane;
        uint32_t v = bi < nf ? flags[bi] : 0u;
        if (bi == b0) v &= 0xffu >> (t & 7u);
        const uint32_t m = __ballot_sync(0xffffffffu, v != 0u);
        if (m) {
            const int l = __ffs(m) - 1;
            const uint32_t vv = __shfl_sync(0xffffffffu, v, l);
            *err_tok = 8 * (uint64_t(base) + uint64_t(l)) + uint64_t(__clz(vv) - 24);
            return TE_NONZERO_PADDING;
        }
    }
    if (nf != ((t + 7) >> 3)) {
        *err_tok = t;
        return TE_FLAG_COUNT;
    }
    return TE_OK;
}

// ------------------------------------------------------- fast chunk decode
// decode_chunk_fast: the decode kernel's chunk routine for chunks whose
// output fits the warp's stage.  Same token semantics as decode_chunk_smem
// (decoder.cpp:22-90), but it only answers "does the reference walk accept
// this chunk" — on any failure the chunk is reported and plz_chunk_detail_kernel
// re-walks it with decode_chunk_smem for the exact error and token — so it
// runs in two lean phases:
//
//  A. tokens, 256 per step: lane l owns flag byte l of the step and walks its
//     8 tokens itself (S = 2: their 16 payload bytes as 5 aligned words; the
//     8 lengths and offsets as two byte-permuted words each, literals masked
//     to length 1 / offset 0 by the flag byte spread to a byte mask, the
//     length sum by two 4-byte dot products), so one warp scan per 256 tokens
//     places them.  The 8 offsets land in the token table as one 8-byte
//     store; per token, the literal goes to the stage and the token start
//     into its wave's start bitmap.  Steps before the last need no
//     reached-token bookkeeping (zero pointer fields by a zero-byte test of
//     the packed words).
//  B. waves of 32 output positions in order, two per step: one 16-byte
//     shared load of both waves' bitmap + token base, a popcount gives each
//     lane its covering token, one byte load its offset, and the lane copies
//     out[q - off] (a literal position copies onto itself).  A lane whose
//     source is an in-wave pointer position (not final yet) follows the
//     chain itself through the same lookups — no shuffles or votes — and the
//     next pair's sources are resolved before this pair's copies.
//
// The chunk leaves the stage as one TMA bulk store (decode_one_chunk).

// Predicated shared-memory stores (no branch around them).
__device__ __forceinline__ void st_u16_if(bool p, uint32_t a, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u16 [%0], %1;\n\t}"
                 ::"r"(a), "r"(v), "r"(uint32_t(p)) : "memory");
}

__device__ __forceinline__ uint32_t warp_excl_scan_u32(uint32_t v, uint32_t lane) {
    return warp_incl_scan_u32(v, lane) - v;
}

template <int S>
__device__ bool decode_chunk_fast(const uint8_t* __restrict__ flags, uint32_t nf,
                                  const uint8_t* __restrict__ pay, uint32_t np, uint32_t L,
                                  uint8_t* wsm, uint32_t lane) {
    constexpr uint32_t FULL = 0xffffffffu;
    uint32_t* meta = reinterpret_cast<uint32_t*>(wsm + kFastPtab + fast_tokens<S>());  // pairs {starts, base}
    constexpr uint32_t kDump = 2u * fast_waves<S>();  // the spare pair: bits of unreached tokens
    const uint32_t s_stage = static_cast<uint32_t>(__cvta_generic_to_shared(wsm));
    const uint32_t s_ptab = s_stage + kFastPtab;
    const uint32_t nwv = (L + 31u) >> 5;
    for (uint32_t w = lane; w < nwv; w += 32) meta[2 * w] = 0u;
    __syncwarp();
    // ---- phase A
    uint32_t written = 0, in = 0, tbase = 0, T = 0, in_end = 0;
    for (uint32_t fb0 = 0;; fb0 += 32) {
        const uint32_t fidx = fb0 + lane;
        const bool hf = fidx < nf;
        const uint32_t fb = hf ? uint32_t(flags[fidx]) : 0u;
        if constexpr (S == 2) {
            // The lane's 8 tokens are its 16 payload bytes (every token is 2
            // bytes): 5 aligned words, funnel-shifted; token 2k is the low
            // half of wv[k], [len][off].  Lengths and offsets of 4 tokens per
            // word (byte permutes), pointer tokens as a byte mask from the
            // flag byte, the step's length sum by two 4-byte dot products.
            uint32_t wv[4];
            {
                const uintptr_t a = reinterpret_cast<uintptr_t>(pay) + in + 16u * lane;
                const uint32_t* wp = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
                const uintptr_t lim = reinterpret_cast<uintptr_t>(pay) + np;
                uint32_t x[5];
#pragma unroll
                for (int k = 0; k < 5; ++k)
                    x[k] = reinterpret_cast<uintptr_t>(wp + k) < lim ? wp[k] : 0u;
                const uint32_t sh = 8u * uint32_t(a & 3u);
#pragma unroll
                for (int k = 0; k < 4; ++k) wv[k] = __funnelshift_r(x[k], x[k + 1], sh);
            }
            const uint32_t r = __brev(fb) >> 24;  // bit i: token i is a pointer (MSB-first flags)
            const uint32_t pm0 = (((r & 15u) * 0x204081u) & 0x01010101u) * 255u;
            const uint32_t pm1 = ((((r >> 4) & 15u) * 0x204081u) & 0x01010101u) * 255u;
            // lengths (a literal: 1) and offsets (a literal: 0), tokens 0-3 / 4-7
            const uint32_t lm0 = (__byte_perm(wv[0], wv[1], 0x6420) & pm0) | (~pm0 & 0x01010101u);
            const uint32_t lm1 = (__byte_perm(wv[2], wv[3], 0x6420) & pm1) | (~pm1 & 0x01010101u);
            const uint32_t om0 = __byte_perm(wv[0], wv[1], 0x7531) & pm0;
            const uint32_t om1 = __byte_perm(wv[2], wv[3], 0x7531) & pm1;
            const uint32_t adv = __dp4a(lm0, 0x01010101u, 0u) + __dp4a(lm1, 0x01010101u, 0u);
            uint32_t pos = written + warp_excl_scan_u32(adv, lane);
            const uint32_t end = __shfl_sync(FULL, pos + adv, 31);
            // token table: the 8 offsets at once (tokens past the flag bytes
            // are never stored: that bounds the table, 8 * nf <= fast_tokens<S>())
            if (hf)
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(s_ptab + tbase + 8u * lane),
                             "r"(om0), "r"(om1) : "memory");
            bool bad = false;
            if (end < L) {
                // every token of the step is reached: zero pointer fields by a
                // zero-byte test of the packed words, per token only the
                // offset-before-start check, the literal store and the start bit
                auto zero_byte = [](uint32_t v) { return ((v - 0x01010101u) & ~v & 0x80808080u) != 0u; };
                bad = zero_byte(lm0) | zero_byte(lm1) | zero_byte(om0 | ~pm0) | zero_byte(om1 | ~pm1);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t len = ((i < 4 ? lm0 : lm1) >> (8 * (i & 3))) & 0xffu;
                    const uint32_t off = ((i < 4 ? om0 : om1) >> (8 * (i & 3))) & 0xffu;
                    const uint32_t fld = (i & 1) ? (wv[i >> 1] >> 16) : (wv[i >> 1] & 0xffffu);
                    bad |= off > pos;
                    st_u16_if(((r >> i) & 1u) == 0u, s_stage + 2u * pos, fld);
                    atomicOr(&meta[2u * (pos >> 5)], 1u << (pos & 31u));
                    pos += len;
                }
                if (__any_sync(FULL, bad)) return false;
                written = end;
                in += 512u;  // 256 two-byte tokens
                tbase += 256u;
                continue;
            }
            // the walk ends in this step: tokens from position L on are not
            // read.  Per token only the pointer fields; overrun (the last
            // reached token must end at L), missing payload and missing flag
            // bits (2T == np, nf == ceil(T/8) for T reached tokens) once.
            uint32_t nreach = 0, lend = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t len = ((i < 4 ? lm0 : lm1) >> (8 * (i & 3))) & 0xffu;
                const uint32_t off = ((i < 4 ? om0 : om1) >> (8 * (i & 3))) & 0xffu;
                const uint32_t fld = (i & 1) ? (wv[i >> 1] >> 16) : (wv[i >> 1] & 0xffffu);
                const uint32_t bit = (r >> i) & 1u;
                const bool reached = pos < L;
                bad |= reached & ((len == 0u) | ((bit != 0u) & (off == 0u)) | (off > pos));
                const bool ok = reached & hf;
                st_u16_if(ok & !bit, s_stage + 2u * pos, fld);
                atomicOr(&meta[ok ? 2u * (pos >> 5) : kDump], 1u << (pos & 31u));
                nreach += reached ? 1u : 0u;
                pos += len;
                lend = reached ? pos : lend;
            }
            if (__any_sync(FULL, bad)) return false;
            T = tbase + __reduce_add_sync(FULL, nreach);
            if (__reduce_max_sync(FULL, lend) != L) return false;  // overrun
            in_end = 2u * T;
            break;
        }
        if constexpr (S == 4 || S == 1) {
            // A pointer is 2 payload bytes, a literal S: the lane's 8 tokens
            // take 8S + (2 - S)p bytes (p pointers), placed by a warp scan;
            // token i starts Si + (2 - S) * (pointers before it) bytes in.  Each
            // field is read as two aligned words (only words that hold a
            // stream byte) and funnel-shifted.
            const uint32_t p = __popc(fb);
            const uint32_t pin = in + warp_excl_scan_u32(uint32_t(8 * S + (2 - S) * int(p)), lane);
            const uintptr_t pay0 = reinterpret_cast<uintptr_t>(pay);
            const uintptr_t lim = pay0 + np;
            uint32_t f[8];
            uint32_t adv = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t o = pin + uint32_t(S * i + (2 - S) * __popc(i ? fb >> (8 - i) : 0u));
                const uintptr_t a = pay0 + o;
                const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
                const uint32_t w0 = reinterpret_cast<uintptr_t>(w) < lim ? w[0] : 0u;
                const uint32_t w1 = reinterpret_cast<uintptr_t>(w + 1) < lim ? w[1] : 0u;
                f[i] = __funnelshift_r(w0, w1, 8u * uint32_t(a & 3u));
                adv += ((fb >> (7 - i)) & 1u) ? (f[i] & 0xffu) : 1u;
            }
            uint32_t pos = written + warp_excl_scan_u32(adv, lane);
            const uint32_t end = __shfl_sync(FULL, pos + adv, 31);
            // tokens from position L on are not read: per token the payload
            // bytes and the pointer fields are checked, overrun (the last
            // reached token must end at L) and missing flag bits once
            bool bad = false;
            uint32_t nreach = 0, lend = 0, o_reach = 0, om0 = 0, om1 = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const uint32_t bit = (fb >> (7 - i)) & 1u;
                const uint32_t o = uint32_t(S * i + (2 - S) * __popc(i ? fb >> (8 - i) : 0u));
                const uint32_t sz = bit ? 2u : uint32_t(S);
                const uint32_t len = bit ? (f[i] & 0xffu) : 1u;
                const uint32_t off = bit ? ((f[i] >> 8) & 0xffu) : 0u;
                const bool reached = pos < L;
                const bool has = pin + o + sz <= np;
                bad |= reached & (!has | ((bit != 0u) & ((len == 0u) | (off == 0u) | (off > pos))));
                const bool ok = reached & hf;
                if (ok & !bit) sts_sym<S>(s_stage + uint32_t(S) * pos, S == 4 ? f[i] : f[i] & 0xffu);
                atomicOr(&meta[ok ? 2u * (pos >> 5) : kDump], 1u << (pos & 31u));
                (i < 4 ? om0 : om1) |= off << (8 * (i & 3));
                nreach += reached ? 1u : 0u;
                o_reach = reached ? o + sz : o_reach;
                pos += len;
                lend = reached ? pos : lend;
            }
            if (hf)
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(s_ptab + tbase + 8u * lane),
                             "r"(om0), "r"(om1) : "memory");
            if (__any_sync(FULL, bad)) return false;
            if (end >= L) {  // the walk ends in this step
                T = tbase + __reduce_add_sync(FULL, nreach);
                if (__reduce_max_sync(FULL, lend) != L) return false;  // overrun
                const uint32_t m = __ballot_sync(FULL, nreach != 0u);
                in_end = __shfl_sync(FULL, pin + o_reach, 31 - __clz(m));
                break;
            }
            written = end;
            in = __shfl_sync(FULL, pin + uint32_t(8 * S + (2 - S) * __popc(fb)), 31);
            tbase += 256u;
            continue;
        }
        // other widths (not dispatched here; kept generic): payload offsets
        // by a warp scan, fields byte by byte
        const uint32_t pin = in + warp_excl_scan_u32(2u * __popc(fb) + uint32_t(S) * (8u - __popc(fb)), lane);
        // pass 1: token fields and lengths
        uint32_t lpk[2] = {0u, 0u}, opk[2] = {0u, 0u};  // lengths / offsets, 4 per word
        uint32_t adv = 0, o = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t bit = (fb >> (7 - i)) & 1u;
            uint32_t f = 0;
            {
                const uint32_t sz = bit ? 2u : uint32_t(S);
#pragma unroll
                for (int b = 0; b < (S > 2 ? S : 2); ++b)
                    if (uint32_t(b) < sz && pin + o + uint32_t(b) < np)
                        f |= uint32_t(pay[pin + o + uint32_t(b)]) << (8 * b);
                o += sz;
            }
            const uint32_t len = bit ? (f & 0xffu) : 1u;
            lpk[i >> 2] |= len << (8 * (i & 3));
            opk[i >> 2] |= (bit ? ((f >> 8) & 0xffu) : 0u) << (8 * (i & 3));
            adv += len;
        }
        uint32_t pos = written + warp_excl_scan_u32(adv, lane);
        // pass 2: checks and writes (tokens from position L on are not read)
        bool bad = false;
        uint32_t nreach = 0, o_reach = 0;
        o = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t bit = (fb >> (7 - i)) & 1u;
            const uint32_t sz = bit ? 2u : uint32_t(S);
            const uint32_t len = (lpk[i >> 2] >> (8 * (i & 3))) & 0xffu;
            const uint32_t off = (opk[i >> 2] >> (8 * (i & 3))) & 0xffu;
            uint32_t fld = 0;
            if (!bit)  // a literal's S bytes, read again
#pragma unroll
                for (int b = 0; b < S; ++b)
                    if (pin + o + uint32_t(b) < np) fld |= uint32_t(pay[pin + o + uint32_t(b)]) << (8 * b);
            const bool reached = pos < L;
            const bool b = !hf || pin + o + sz > np ||
                           (bit && (len == 0u || off == 0u || off > pos || pos + len > L));
            bad |= reached && b;
            if (reached && !b) {
                const uint32_t t = tbase + 8u * lane + uint32_t(i);
                if (!bit) sts_sym<S>(s_stage + pos * S, S == 4 ? fld : fld & ((1u << (8 * S)) - 1u));
                atomicOr(&meta[2 * (pos >> 5)], 1u << (pos & 31u));
                asm volatile("st.shared.u8 [%0], %1;" ::"r"(s_ptab + t), "r"(off));
                ++nreach;
                o_reach = o + sz;
            }
            pos += len;
            o += sz;
        }
        if (__any_sync(FULL, bad)) return false;
        const uint32_t end = __shfl_sync(FULL, pos, 31);
        if (end >= L) {  // the walk ends in this step: tokens read, payload consumed
            T = tbase + __reduce_add_sync(FULL, nreach);
            const uint32_t m = __ballot_sync(FULL, nreach != 0u);
            in_end = __shfl_sync(FULL, pin + o_reach, 31 - __clz(m));
            break;
        }
        written = end;
        in = __shfl_sync(FULL, pin + o, 31);
        tbase += 256u;
    }
    // the walk's end checks (decoder.cpp:58-65)
    if (in_end != np || nf != ((T + 7u) >> 3)) return false;
    if ((T & 7u) && (flags[T >> 3] & (0xffu >> (T & 7u)))) return false;
    __syncwarp();
    // ---- wave table: tokens before each wave (scan of the bitmaps' popcounts)
    uint32_t carry = 0;
    for (uint32_t w0 = 0; w0 < nwv; w0 += 32) {
        const uint32_t w = w0 + lane;
        const uint32_t c = w < nwv ? __popc(meta[2 * w]) : 0u;
        const uint32_t inc = warp_incl_scan_u32(c, lane);
        if (w < nwv) meta[2 * w + 1] = carry + inc - c - 1u;  // token before the wave
        carry += __shfl_sync(FULL, inc, 31);
    }
    __syncwarp();
    // ---- phase B: waves of 32 positions, two per step (one 16-byte load of
    // both table entries).  A lane's source q - off is final unless it lies
    // in the lane's own wave (off <= lane) on a pointer position: then the
    // lane alone follows the chain through the wave's token lookups (the
    // covering token of in-wave position s: popcount of the starts up to s)
    // until it reaches a literal or an earlier wave.  No votes: the chase is
    // a divergent branch that ~1 wave in 5 takes.
    const uint32_t upto = (2u << lane) - 1u;
    uint32_t a_q = s_stage + lane * uint32_t(S);
    // The token table and the wave table are read-only here: plain loads the
    // compiler may schedule ahead of the stage copies (each pair's lookups
    // are issued before the previous pair's copies).
    const uint4* meta4 = reinterpret_cast<const uint4*>(meta);
    // (not volatile: the address depends on a wave-table load, which is
    // ordered after the table writes)
    auto ptab = [&](uint32_t i) {
        uint32_t v;
        asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(s_ptab + i));
        return v;
    };
    // Source of the lane's position in a wave: in-wave index (< 0: an
    // earlier wave, final).  Reads only the token and wave tables, so the
    // next pair's sources are resolved before this pair's copies.
    auto source = [&](uint32_t st, uint32_t tb, uint32_t off) {
        int s = int(lane) - int(off);
        if (off != 0u && s >= 0) {
            for (;;) {
                const uint32_t o2 = ptab(tb + __popc(st & ((2u << s) - 1u)));
                if (o2 == 0u) break;  // a literal: written in phase A
                s -= int(o2);
                if (s < 0) break;
            }
        }
        return s;
    };
    auto sources = [&](const uint4& m, int& s0, int& s1) {
        const uint32_t off0 = ptab(m.y + __popc(m.x & upto)), off1 = ptab(m.w + __popc(m.z & upto));
        s0 = int(lane) - int(off0);
        s1 = int(lane) - int(off1);
        // one divergent region per pair, entered by ~1 pair in 3
        // (off - 1 < lane, unsigned: 0 < off <= lane — a source in the wave)
        if ((off0 - 1u < lane) | (off1 - 1u < lane)) {
            s0 = source(m.x, m.y, off0);
            s1 = source(m.z, m.w, off1);
        }
    };
    // A wave's copy reads what the previous wave's copy stored.  The warp is
    // converged from the __syncwarp that follows each group's sources()
    // (where the chase may diverge) through the group's copies — straight-line
    // code — so the stores of one warp-wide st.shared are visible to the next
    // warp-wide ld.shared without a barrier per wave; only the compiler is
    // kept from reordering them (volatile asm + memory clobber).  A
    // __syncwarp() per wave (a divergence check, UMOV + BRA.DIV, each) cost
    // 3.9 % of c5's decompress; one per pair 1.7 %, one per four waves ~1.2 %.
    auto copy = [&](int s) {
        sts_sym<S>(a_q, lds_sym<S>(uint32_t(int(a_q) + (s - int(lane)) * S)));
        a_q += 32u * S;
        asm volatile("" ::: "memory");
    };
    uint32_t w = 0;
    // S = 2: groups of four waves, one warp barrier per group (the S = 1 and
    // S = 4 instances spill with four sources live and take pairs)
    if (S == 2 && nwv >= 4u) {
        int s0, s1, s2, s3;
        sources(meta4[0], s0, s1);
        sources(meta4[1], s2, s3);
        __syncwarp();
        for (; w + 8u <= nwv; w += 4u) {
            int n0, n1, n2, n3;
            sources(meta4[(w >> 1) + 2u], n0, n1);
            sources(meta4[(w >> 1) + 3u], n2, n3);
            __syncwarp();  // converged, and the previous group's stores visible
            copy(s0);
            copy(s1);
            copy(s2);
            copy(s3);
            s0 = n0;
            s1 = n1;
            s2 = n2;
            s3 = n3;
        }
        copy(s0);
        copy(s1);
        copy(s2);
        copy(s3);
        w += 4u;
    }
    if (w + 2u <= nwv) {
        int s0, s1;
        sources(meta4[w >> 1], s0, s1);
        __syncwarp();  // converged, and the previous pair's stores visible
#pragma unroll 2
        for (; w + 4u <= nwv; w += 2u) {
            int n0, n1;
            sources(meta4[(w >> 1) + 1u], n0, n1);
            __syncwarp();
            copy(s0);
            copy(s1);
            s0 = n0;
            s1 = n1;
        }
        copy(s0);
        copy(s1);
        w += 2u;
    }
    if (w < nwv) {
        const uint32_t st = meta[2u * w], tb = meta[2u * w + 1u];
        const int s = source(st, tb, ptab(tb + __popc(st & upto)));
        __syncwarp();
        copy(s);
    }
    return true;
}

// ------------------------------------------------------------------ parse
enum ParseErr : uint32_t {
    PE_OK = 0,
    PE_TRUNC_HEADER = 1,
    PE_MAGIC = 2,
    PE_VERSION = 3,
    PE_RESERVED = 4,
    PE_PARAMS = 5,
    PE_TAIL = 6,
    PE_TRUNC_TABLES = 7,
    PE_PAYLOAD_MONO = 8,
    PE_FLAG_MONO = 9,
    PE_PAYLOAD_START = 10,
    PE_FLAG_START = 11,
    PE_TRUNC_STREAMS = 12,
    PE_ORIG_SMALL = 13,
    PE_ORIG_ALIGN = 14,
    PE_NUM_CHUNKS = 15,
    PE_CAPACITY = 16,
    PE_DESC_FULL = 17,
};

__device__ __forceinline__ bool header_params_ok(uint32_t S, uint32_t W, uint32_t I, uint32_t C) {
    if (S != 1 && S != 2 && S != 4) return false;
    if (W < 4 || W > 255) return false;
    if (C != 1024 && C != 2048 && C != 4096 && C != 8192 && C != 16384) return false;
    if (C <= W) return false;
    if (I != 1 && I != 2 && I != 4 && I != 8 && I != 16) return false;
    return true;  // C % I == 0 and the default block_bytes follow from the sets
}

__global__ void __launch_bounds__(256) plz_parse_kernel(DecodeArgs a) {
    __shared__ uint64_t s_at, s_out, s_chunks, s_j, s_n, s_maxcb;
    __shared__ unsigned long long s_bad;
    __shared__ uint32_t s_stop, s_err, s_kinds;
    __shared__ uint64_t s_eoff;
    const uint32_t tid = threadIdx.x;
    ParseResult* res = a.result;
    if (tid == 0) {
        s_stop = 0;
        res->err_kind = PE_OK;
        // Fast chain (thread 0, no barriers): every container that passes all
        // of read_container's checks gets its descriptor here with one round
        // of loads — the header and, at the chunk count predicted from the
        // previous container (every container but the last has the same),
        // the four table words the checks and the next container's offset
        // need.  At the first container with anything unusual (a failed
        // check, a mispredicted count, the descriptor table full) it stops,
        // and the exact loop below takes over from that container.
        uint64_t at = 0, out = 0, chunks = 0, j = 0, maxcb = 0, n_pred = 0;
        uint32_t kinds = 0;
        while (at < a.img_len && j < a.desc_cap) {
            const uint8_t* b = a.img + at;
            const uint64_t size = a.img_len - at;
            if (j == 0) n_pred = size >= 26 ? ld_le32(b + 21) : 0u;  // the first: read first
            if (size < 26 + 8 * (n_pred + 1)) break;
            const uint8_t* pt = b + 26;
            const uint8_t* ftp = pt + 4 * (n_pred + 1);
            const uint32_t p0 = ld_le32(pt), f0 = ld_le32(ftp);
            const uint64_t ptot = ld_le32(pt + 4 * n_pred), ftot = ld_le32(ftp + 4 * n_pred);
            const uint32_t S = b[5], W = b[6], I = b[7], C = ld_le32(b + 9), tail = b[25];
            const uint64_t orig = ld_le64(b + 13), n = ld_le32(b + 21);
            if (b[0] != 'P' || b[1] != 'L' || b[2] != 'Z' || b[3] != '1' || b[4] != 1 || b[8] != 0 ||
                !header_params_ok(S, W, I, C) || tail >= S || n != n_pred || p0 != 0 || f0 != 0)
                break;
            const uint64_t need = 26 + 8 * (n + 1) + ftot + ptot + tail;
            if (size < need || orig < tail || (orig - tail) % S != 0 ||
                ((orig - tail) / S + C - 1) / C != n || out + orig > a.out_cap)
                break;
            ContainerDesc d;
            d.img_off = at;
            d.out_off = out;
            d.chunk_base = chunks;
            d.flags_off = at + 26 + 8 * (n + 1);
            d.payload_off = d.flags_off + ftot;
            d.payload_len = ptot;
            d.original_len = orig;
            d.num_chunks = uint32_t(n);
            d.chunk_size = C;
            d.last_len = n ? uint32_t((orig - tail) / S - (n - 1) * C) : 0u;
            d.S = uint8_t(S);
            d.W = uint8_t(W);
            d.I = uint8_t(I);
            d.tail_len = uint8_t(tail);
            a.desc[j] = d;
            if (a.out)
                for (uint64_t i = 0; i < tail; ++i) a.out[out + orig - tail + i] = b[need - tail + i];
            if (uint64_t(C) * S > maxcb) maxcb = uint64_t(C) * S;
            if (n) kinds |= S == 2 ? 2u : S == 4 ? 4u : 1u;
            at += need;
            out += orig;
            chunks += n;
            ++j;
            n_pred = n;  // the next container's chunk count (a mispredict ends the chain)
        }
        s_at = at;
        s_out = out;
        s_chunks = chunks;
        s_j = j;
        s_maxcb = maxcb;
        s_kinds = kinds;
    }
    __syncthreads();
    for (;;) {
        if (tid == 0) {
            s_bad = ~0ull;
            const uint64_t at = s_at;
            if (at >= a.img_len) {
                s_stop = 1;
            } else if (s_j >= a.desc_cap) {
                res->err_kind = PE_DESC_FULL;
                s_stop = 1;
            } else {
                const uint8_t* b = a.img + at;
                const uint64_t size = a.img_len - at;
                uint32_t err = PE_OK, aux = 0;
                uint64_t eoff = 0;
                if (size < 26) {
                    err = PE_TRUNC_HEADER;
                    eoff = size;
                } else if (b[0] != 'P' || b[1] != 'L' || b[2] != 'Z' || b[3] != '1') {
                    err = PE_MAGIC;
                } else if (b[4] != 1) {
                    err = PE_VERSION;
                    aux = b[4];
                } else if (b[8] != 0) {
                    err = PE_RESERVED;
                    eoff = 8;
                } else if (!header_params_ok(b[5], b[6], b[7], ld_le32(b + 9))) {
                    err = PE_PARAMS;
                    eoff = 5;
                } else if (b[25] >= b[5]) {
                    err = PE_TAIL;
                    eoff = 25;
                } else {
                    const uint64_t n = ld_le32(b + 21);
                    if (size < 26 + 8 * (n + 1)) {
                        err = PE_TRUNC_TABLES;
                        eoff = size;
                    } else {
                        s_n = n;
                    }
                }
                if (err != PE_OK) {
                    res->err_kind = err;
                    res->err_aux = aux;
                    res->err_container = s_j;
                    res->err_offset = eoff;
                    res->hdr_S = b[5];
                    res->hdr_W = b[6];
                    res->hdr_I = b[7];
                    res->hdr_C = size >= 13 ? ld_le32(b + 9) : 0;
                    s_stop = 1;
                }
            }
        }
        __syncthreads();
        if (s_stop) break;
        if (tid == 0) {
            const uint64_t at = s_at, n = s_n;
            const uint8_t* b = a.img + at;
            const uint64_t size = a.img_len - at;
            const uint8_t* ptab = b + 26;
            const uint8_t* ftab = ptab + 4 * (n + 1);
            uint32_t err = PE_OK;
            uint64_t eoff = 0;
            const uint64_t S = b[5], C = ld_le32(b + 9), tail = b[25];
            const uint64_t orig = ld_le64(b + 13);
            const uint64_t ftot = ld_le32(ftab + 4 * n), ptot = ld_le32(ptab + 4 * n);
            const uint64_t need = 26 + 8 * (n + 1) + ftot + ptot + tail;
            if (ld_le32(ptab) != 0) {
                err = PE_PAYLOAD_START;
                eoff = 26;
            } else if (ld_le32(ftab) != 0) {
                err = PE_FLAG_START;
                eoff = 26 + 4 * (n + 1);
            } else if (size < need) {
                err = PE_TRUNC_STREAMS;
                eoff = size;
            } else if (orig < tail) {
                err = PE_ORIG_SMALL;
                eoff = 13;
            } else if ((orig - tail) % S != 0) {
                err = PE_ORIG_ALIGN;
                eoff = 13;
            } else if (((orig - tail) / S + C - 1) / C != n) {
                err = PE_NUM_CHUNKS;
                eoff = 21;
            } else if (s_out + orig > a.out_cap) {
                err = PE_CAPACITY;
            }
            s_err = err;
            s_eoff = eoff;
        }
        __syncthreads();
        if (s_err != PE_OK) {
            // the reference checks table monotonicity before these (format.cpp
            // order); a container that passes them has its monotonicity
            // checked by the decode kernel from the entries each chunk reads
            const uint8_t* ptab = a.img + s_at + 26;
            const uint64_t n = s_n;
            const uint8_t* ftab = ptab + 4 * (n + 1);
            for (uint64_t i = tid; i < n; i += blockDim.x) {
                if (ld_le32(ptab + 4 * (i + 1)) < ld_le32(ptab + 4 * i)) {
                    atomicMin(&s_bad, 2 * i);
                } else if (ld_le32(ftab + 4 * (i + 1)) < ld_le32(ftab + 4 * i)) {
                    atomicMin(&s_bad, 2 * i + 1);
                }
            }
            __syncthreads();
        }
        if (tid == 0) {
            const uint64_t at = s_at, n = s_n;
            const uint8_t* b = a.img + at;
            const uint64_t S = b[5], C = ld_le32(b + 9), tail = b[25];
            const uint64_t orig = ld_le64(b + 13);
            const uint8_t* ptab = b + 26;
            const uint8_t* ftab = ptab + 4 * (n + 1);
            const uint64_t ftot = ld_le32(ftab + 4 * n), ptot = ld_le32(ptab + 4 * n);
            const uint64_t need = 26 + 8 * (n + 1) + ftot + ptot + tail;
            uint32_t err = s_err;
            uint64_t eoff = s_eoff;
            if (s_bad != ~0ull) {
                const uint64_t i = s_bad >> 1;
                err = (s_bad & 1) ? PE_FLAG_MONO : PE_PAYLOAD_MONO;
                eoff = (s_bad & 1) ? 26 + 4 * (n + 1) + 4 * (i + 1) : 26 + 4 * (i + 1);
            }
            if (err != PE_OK) {
                res->err_kind = err;
                res->err_container = s_j;
                res->err_offset = eoff;
                s_stop = 1;
            } else {
                const uint64_t symbols = (orig - tail) / S;
                ContainerDesc d;
                d.img_off = at;
                d.out_off = s_out;
                d.chunk_base = s_chunks;
                d.flags_off = at + 26 + 8 * (n + 1);
                d.payload_off = d.flags_off + ftot;
                d.payload_len = ptot;
                d.original_len = orig;
                d.num_chunks = uint32_t(n);
                d.chunk_size = uint32_t(C);
                d.last_len = n ? uint32_t(symbols - (n - 1) * C) : 0u;
                d.S = uint8_t(S);
                d.W = b[6];
                d.I = b[7];
                d.tail_len = uint8_t(tail);
                a.desc[s_j] = d;
                // raw tail straight to the output (decoder.cpp:123-125)
                const uint8_t* ts = a.img + d.payload_off + ptot;
                if (a.out)
                    for (uint64_t i = 0; i < tail; ++i) a.out[s_out + orig - tail + i] = ts[i];
                if (C * S > s_maxcb) s_maxcb = C * S;
                if (n) s_kinds |= S == 2 ? 2u : S == 4 ? 4u : 1u;
                s_at = at + need;
                s_out += orig;
                s_chunks += n;
                s_j += 1;
            }
        }
        __syncthreads();
        if (s_stop) break;
        __syncthreads();  // every thread has read s_stop before thread 0 rewrites it
    }
    if (tid == 0) {
        res->n_containers = s_j;
        res->total_chunks = s_chunks;
        res->total_out = s_out;
        res->max_chunk_bytes = s_maxcb;
        res->absent_kinds = ~s_kinds & 7u;
        if (a.out_len) *a.out_len = s_out;
    }
}

// ----------------------------------------------------------------- decode
// Pipelined host image: waits (lane 0, bounded ~4 s) until the H2D segment
// holding image byte `b` has landed; all earlier segments land before it.
// bar.warp.sync in the broadcast orders the other lanes' later loads.
__device__ __forceinline__ bool wait_image(const DecodePipe& a, uint64_t b, uint32_t lane) {
    uint32_t ok = 1;
    if (lane == 0) {
        const uint32_t* f = a.in_ready + b / a.in_seg;
        const long long t0 = clock64();
        while (ld_acquire_sys(f) != a.epoch) {
            __nanosleep(256);
            if (clock64() - t0 > (1ll << 33)) {
                atomicExch(a.stalled, 1u);
                ok = 0;
                break;
            }
        }
    }
    return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// kExact: the error detail path (exact TokenErr and token index); otherwise
// chunks that fit the stage take decode_chunk_fast and a failure is reported
// as TE_FLAGS_EXHAUSTED, a placeholder the detail kernel replaces.
template <int S, bool kPipe, bool kExact>
__device__ __forceinline__ uint32_t decode_one_chunk(const DecodeArgs& a, const ContainerDesc& d,
                                                     uint64_t k, uint8_t* stage, uint32_t lane,
                                                     uint64_t* err_tok, const DecodePipe& pp) {
    // table entries k, k+1 of both tables: lanes 0-7 payload, 8-15 flags
    const uint8_t* ptab = a.img + d.img_off + 26;
    const uint8_t* ftab = ptab + 4 * (uint64_t(d.num_chunks) + 1);
    if (kPipe && !wait_image(pp, uint64_t(ftab - a.img) + 4 * k + 7, lane)) {
        *err_tok = 0;
        return TE_OK;  // stalled: the host reports it
    }
    uint32_t byte = 0;
    if (lane < 8) byte = ptab[4 * k + lane];
    else if (lane < 16) byte = ftab[4 * k + (lane - 8)];
    uint32_t v = byte << (8 * (lane & 3u));
    v |= __shfl_xor_sync(0xffffffffu, v, 1);
    v |= __shfl_xor_sync(0xffffffffu, v, 2);
    const uint32_t p0 = __shfl_sync(0xffffffffu, v, 0), p1 = __shfl_sync(0xffffffffu, v, 4);
    const uint32_t f0 = __shfl_sync(0xffffffffu, v, 8), f1 = __shfl_sync(0xffffffffu, v, 12);
    // table monotonicity (format.cpp order: payload entry before flag entry);
    // a violating chunk is not decoded — the whole container is corrupt
    if (p1 < p0 || f1 < f0) {
        if (lane == 0 && a.mono_key)
            atomicMin(a.mono_key, (unsigned long long)((d.chunk_base + k) << 1) | (p1 < p0 ? 0ull : 1ull));
        *err_tok = 0;
        return TE_OK;
    }
    // an entry past its stream's end implies a decrease further on (the last
    // entry is the stream size): skip, the violating chunk reports it
    if (p1 > d.payload_len || f1 > d.payload_off - d.flags_off) {
        *err_tok = 0;
        return TE_OK;
    }
    // the chunk's streams plus the decoder's read-ahead slack
    if (kPipe && !wait_image(pp, min(d.payload_off + p1 + 127, a.img_len - 1), lane)) {
        *err_tok = 0;
        return TE_OK;
    }
    const uint64_t C = d.chunk_size;
    const uint64_t L = (k + 1 == d.num_chunks) ? d.last_len : C;
    uint8_t* dst = a.out + d.out_off + k * C * S;
    const bool in_smem = C * S <= kDecodeSmem;
    const uint8_t* fl = a.img + d.flags_off + f0;
    const uint8_t* py = a.img + d.payload_off + p0;
    uint64_t tok = 0;
    uint32_t e;
    uint32_t* tab = reinterpret_cast<uint32_t*>(stage + kDecodeSmem + kDecodePad);
    bulk_store_drain(lane);  // the previous chunk's stage has left
    if (kUseFast && !kExact && in_smem && 8u * uint64_t(f1 - f0) <= fast_tokens<S>())
        e = decode_chunk_fast<S>(fl, f1 - f0, py, p1 - p0, uint32_t(L), stage, lane)
                ? TE_OK : TE_FLAGS_EXHAUSTED;
    else if (in_smem)
        e = decode_chunk_smem<S>(fl, f1 - f0, py, p1 - p0, uint32_t(L),
                                 static_cast<uint32_t>(__cvta_generic_to_shared(stage)),
                                 static_cast<uint32_t>(__cvta_generic_to_shared(tab)),
                                 reinterpret_cast<uint32_t*>(stage + kDecodeSmem + kDecodePad + 144),
                                 lane,
                                 &tok);
    else if ((reinterpret_cast<uintptr_t>(dst) & (S - 1)) == 0)
        e = decode_chunk_warp<S, false>(fl, f1 - f0, py, p1 - p0, L, SymOut<S, false>{dst}, tab,
                                        lane, &tok);
    else
        e = decode_chunk_warp<S, true>(fl, f1 - f0, py, p1 - p0, L, SymOut<S, true>{dst}, tab,
                                       lane, &tok);
    if (e == TE_OK && in_smem) {
        __syncwarp();
        const uint64_t bytes = L * S;
        if (!kPipe && ((reinterpret_cast<uintptr_t>(dst) | bytes) & 15u) == 0) {
            // one TMA bulk store of the whole stage (the next chunk's
            // bulk_store_drain waits until it has been read)
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) bulk_s2g(dst, stage, uint32_t(bytes));
        } else if ((reinterpret_cast<uintptr_t>(dst) & 15u) == 0) {
            uint4* d16 = reinterpret_cast<uint4*>(dst);
            const uint4* s16 = reinterpret_cast<const uint4*>(stage);
            for (uint64_t i = lane; i < (bytes >> 4); i += 32) d16[i] = s16[i];
            for (uint64_t i = ((bytes >> 4) << 4) + lane; i < bytes; i += 32) dst[i] = stage[i];
        } else {
            for (uint64_t i = lane; i < bytes; i += 32) dst[i] = stage[i];
        }
    }
    __syncwarp();
    *err_tok = tok;
    return e;
}

__device__ __forceinline__ uint64_t find_container(const ContainerDesc* desc, uint64_t nc,
                                                   uint64_t g) {
    uint64_t lo = 0, hi = nc - 1;  // last descriptor with chunk_base <= g
    while (lo < hi) {
        const uint64_t mid = (lo + hi + 1) >> 1;
        if (desc[mid].chunk_base <= g) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// kKind: which containers a decode kernel takes — kKindS2 the S = 2 ones
// (decode_chunk_fast), kKindOther the rest (decode_chunk_smem), kKindAll
// every one (the exact detail path).  Two specialised kernels keep the hot
// S = 2 instance's registers at 56 instead of the 80 the union of all widths
// needs (which would cost a fifth of the resident warps).
constexpr int kKindOther = 0, kKindS2 = 1, kKindS4 = 2, kKindAll = 3;

template <bool kPipe, bool kExact, int kKind>
__device__ __forceinline__ uint32_t decode_desc_chunk(const DecodeArgs& a, const ContainerDesc& d,
                                                      uint64_t k, uint8_t* stage, uint32_t lane,
                                                      uint64_t* tok, const DecodePipe& pp) {
    if constexpr (kKind == kKindS2) {
        return decode_one_chunk<2, kPipe, kExact>(a, d, k, stage, lane, tok, pp);
    } else if constexpr (kKind == kKindS4) {
        return decode_one_chunk<4, kPipe, kExact>(a, d, k, stage, lane, tok, pp);
    } else {
        switch (d.S) {
            case 1: return decode_one_chunk<1, kPipe, kExact || kKind == kKindAll>(a, d, k, stage, lane, tok, pp);
            case 2:
                if constexpr (kKind == kKindAll)
                    return decode_one_chunk<2, kPipe, true>(a, d, k, stage, lane, tok, pp);
                else
                    return TE_OK;  // not this kernel's container
            default:
                if constexpr (kKind == kKindAll)
                    return decode_one_chunk<4, kPipe, true>(a, d, k, stage, lane, tok, pp);
                else
                    return TE_OK;  // not this kernel's container
        }
    }
}

template <bool kPipe = false, bool kExact = false>
__device__ __forceinline__ uint32_t decode_global_chunk(const DecodeArgs& a, uint64_t g,
                                                        uint8_t* stage, uint32_t lane,
                                                        uint64_t* k, uint64_t* tok,
                                                        const DecodePipe& pp = DecodePipe{}) {
    const ContainerDesc d = a.desc[find_container(a.desc, a.result->n_containers, g)];
    *k = g - d.chunk_base;
    return decode_desc_chunk<kPipe, kExact, kKindAll>(a, d, *k, stage, lane, tok, pp);
}

// kPipe: the pipelined host path (per-chunk segment waits, output counts).
// Each kind has its own work counter (a.work[kind]); a warp that draws a
// chunk of a container the kernel does not take moves the counter past that
// container, so the other kernel's containers cost one draw each.
template <bool kPipe, int kKind>
__global__ void __launch_bounds__(kDecodeWarps * 32, 9) plz_decode_kernel(DecodeArgs a, DecodePipe pp) {
    extern __shared__ __align__(16) uint8_t smem[];
    constexpr uint32_t kWarpSmem = kMainWarpSmem;
    const uint32_t lane = lane_id();
    uint8_t* stage = smem + size_t(threadIdx.x >> 5) * kWarpSmem;
    uint32_t* work = a.work + kKind;
    // no container of this kernel's kind (the parse found none): nothing to
    // draw — without this the idle instance's warps contend on its counter
    // for ~0.12 ms at c5
    if ((a.result->absent_kinds >> kKind) & 1u) return;
    const uint64_t total = a.result->total_chunks;
    // the container of the warp's last chunk: consecutive draws almost always
    // fall into it, so the binary search over the descriptors (a chain of
    // dependent global loads) runs about once per container
    // (32-bit: the work counter is; fewer live registers across the decode)
    uint32_t cj = 0, c_lo = 1, c_hi = 0;
    for (;;) {
        uint32_t g = 0;
        if (lane == 0) g = atomicAdd(work, 1u);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= total) break;
        if (g < c_lo || g >= c_hi) {
            cj = uint32_t(find_container(a.desc, a.result->n_containers, g));
            c_lo = uint32_t(a.desc[cj].chunk_base);
            c_hi = c_lo + a.desc[cj].num_chunks;
        }
        const ContainerDesc d = a.desc[cj];
        if ((d.S == 2 ? kKindS2 : d.S == 4 ? kKindS4 : kKindOther) != kKind) {
            if (lane == 0) atomicMax(work, uint32_t(min(total, d.chunk_base + d.num_chunks)));
            continue;
        }
        const uint64_t k = g - d.chunk_base;
        uint64_t tok;
        const uint32_t e = decode_desc_chunk<kPipe, false, kKind>(a, d, k, stage, lane, &tok, pp);
        if (e != TE_OK && lane == 0) atomicMin(a.err_chunk, (unsigned long long)g);
        if (kPipe) {
            // counted whatever the outcome (the D2H stream must never wait
            // forever); a failed call is re-run on the resident path
            __threadfence_system();
            __syncwarp();
            if (lane == 0) {
                const uint64_t CS = uint64_t(d.chunk_size) * d.S;
                const uint64_t o0 = d.out_off + k * CS;
                const uint64_t o1 = o0 + (k + 1 == d.num_chunks ? uint64_t(d.last_len) * d.S : CS);
                for (uint64_t sg = o0 / pp.out_seg; sg * pp.out_seg < o1; ++sg) {
                    const uint64_t lo = max(o0, sg * pp.out_seg);
                    const uint64_t hi = min(o1, (sg + 1) * pp.out_seg);
                    atomicAdd(pp.out_done + sg, uint32_t(hi - lo));
                }
            }
        }
    }
    bulk_store_complete(lane);
}

// Chunk-range decode (plzgpu_decompress_range): the output bytes of global
// chunks [cb, ce) are [start(cb), start(ce)) with start(0) = 0, start(total)
// = total_out and otherwise the chunk's own output offset, so consecutive
// ranges partition the output (container tails, and containers without
// chunks, fall into the range that holds their bytes).  One warp: range
// bounds into res[0..1], the true chunk count into res[2], and every tail
// byte inside the range copied to out[byte - start(cb)].
__device__ __forceinline__ uint64_t chunk_start(const DecodeArgs& a, uint64_t g) {
    const ParseResult* r = a.result;
    if (g == 0) return 0;
    if (g >= r->total_chunks) return r->total_out;
    const ContainerDesc& d = a.desc[find_container(a.desc, r->n_containers, g)];
    return d.out_off + (g - d.chunk_base) * uint64_t(d.chunk_size) * d.S;
}

__global__ void plz_range_kernel(DecodeArgs a, uint64_t cb, uint64_t ce, uint8_t* out,
                                 uint64_t* res) {
    const uint64_t lo = chunk_start(a, cb), hi = chunk_start(a, ce);
    const uint64_t nc = out ? a.result->n_containers : 0;
    for (uint64_t j = threadIdx.x; j < nc; j += blockDim.x) {
        const ContainerDesc d = a.desc[j];
        const uint64_t t1 = d.out_off + d.original_len, t0 = t1 - d.tail_len;
        for (uint64_t t = max(t0, lo); t < min(t1, hi); ++t)
            out[t - lo] = a.img[d.payload_off + d.payload_len + (t - t0)];
    }
    if (threadIdx.x == 0) {
        res[0] = lo;
        res[1] = hi;
        res[2] = a.result->total_chunks;
    }
}

// Error details of the lowest failing chunk (re-decoded by one warp).
__global__ void plz_chunk_detail_kernel(DecodeArgs a, uint32_t* code, uint64_t* chunk,
                                        uint64_t* token) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint64_t g = *a.err_chunk;
    uint64_t k = 0, tok = 0;
    const uint32_t e = decode_global_chunk<false, true>(a, g, smem, lane_id(), &k, &tok);
    bulk_store_complete(lane_id());
    if (lane_id() == 0) {
        *code = e;
        *chunk = k;
        *token = tok;
    }
}

// The first monotonicity violation the decode kernel found: the container,
// its first chunk (errors of lower chunks belong to earlier containers and
// win), and the reference's byte offset of the offending entry.
__global__ void plz_mono_detail_kernel(DecodeArgs a, unsigned long long key, uint64_t* base) {
    const uint64_t g = key >> 1;
    const uint64_t j = find_container(a.desc, a.result->n_containers, g);
    const ContainerDesc d = a.desc[j];
    const uint64_t i = g - d.chunk_base, n = d.num_chunks;
    ParseResult* r = a.result;
    r->err_kind = (key & 1) ? PE_FLAG_MONO : PE_PAYLOAD_MONO;
    r->err_container = j;
    r->err_offset = (key & 1) ? 26 + 4 * (n + 1) + 4 * (i + 1) : 26 + 4 * (i + 1);
    *base = d.chunk_base;
}

__global__ void plz_decode_one_kernel(DecodeOneArgs a) {
    __shared__ uint32_t tab[33];
    const uint32_t lane = lane_id();
    uint64_t tok = 0;
    uint32_t e;
    switch (a.S) {
        case 1:
            e = decode_chunk_warp<1, true>(a.flags, a.n_flags, a.payload, a.n_payload, a.logical,
                                           SymOut<1, true>{a.out}, tab, lane, &tok);
            break;
        case 2:
            e = decode_chunk_warp<2, true>(a.flags, a.n_flags, a.payload, a.n_payload, a.logical,
                                           SymOut<2, true>{a.out}, tab, lane, &tok);
            break;
        default:
            e = decode_chunk_warp<4, true>(a.flags, a.n_flags, a.payload, a.n_payload, a.logical,
                                           SymOut<4, true>{a.out}, tab, lane, &tok);
            break;
    }
    if (lane == 0) {
        *a.err_code = e;
        *a.err_token = tok;
    }
}

}  // namespace

namespace {
template <bool kPipe, int kKind>
void launch_kind(const DecodeArgs& a, const DecodePipe& pp, int sms, cudaStream_t st) {
    constexpr uint32_t kWarpSmem = kMainWarpSmem;
    const size_t smem = size_t(kDecodeWarps) * kWarpSmem;
    static int per_sm = -1;  // same answer on every B200; computed once
    if (per_sm < 0) {
        int blocks = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, plz_decode_kernel<kPipe, kKind>,
                                                      kDecodeWarps * 32, smem);
        per_sm = blocks > 0 ? blocks : 1;
    }
    plz_decode_kernel<kPipe, kKind><<<sms * per_sm, kDecodeWarps * 32, smem, st>>>(a, pp);
}
}  // namespace

void launch_parse(const DecodeArgs& a, cudaStream_t st) {
    plz_parse_kernel<<<1, 256, 0, st>>>(a);
}

// the other widths first: in a one-width image (the usual case) that kernel
// only skips containers, then the S = 2 kernel does the work
void launch_decode(const DecodeArgs& a, int sms, cudaStream_t st) {
    launch_kind<false, kKindOther>(a, DecodePipe{}, sms, st);
    launch_kind<false, kKindS4>(a, DecodePipe{}, sms, st);
    launch_kind<false, kKindS2>(a, DecodePipe{}, sms, st);
}

void launch_range(const DecodeArgs& a, uint64_t cb, uint64_t ce, uint8_t* out, uint64_t* res,
                  cudaStream_t st) {
    plz_range_kernel<<<1, 32, 0, st>>>(a, cb, ce, out, res);
}

void launch_decode_pipelined(const DecodeArgs& a, const DecodePipe& pp, int sms, cudaStream_t st) {
    launch_kind<true, kKindOther>(a, pp, sms, st);
    launch_kind<true, kKindS4>(a, pp, sms, st);
    launch_kind<true, kKindS2>(a, pp, sms, st);
}

void launch_chunk_detail(const DecodeArgs& a, uint32_t* code, uint64_t* chunk, uint64_t* token,
                         cudaStream_t st) {
    plz_chunk_detail_kernel<<<1, 32, kDecodeWarpSmem, st>>>(a, code, chunk, token);
}

void launch_mono_detail(const DecodeArgs& a, unsigned long long key, uint64_t* base,
                        cudaStream_t st) {
    plz_mono_detail_kernel<<<1, 1, 0, st>>>(a, key, base);
}

void launch_decode_one(const DecodeOneArgs& a, cudaStream_t st) {
    plz_decode_one_kernel<<<1, 32, 0, st>>>(a);
}

void preload_decode_kernels() {
    for (const void* f : {reinterpret_cast<const void*>(plz_parse_kernel),
                          reinterpret_cast<const void*>(plz_decode_kernel<false, kKindOther>),
                          reinterpret_cast<const void*>(plz_decode_kernel<false, kKindS2>),
                          reinterpret_cast<const void*>(plz_decode_kernel<false, kKindS4>),
                          reinterpret_cast<const void*>(plz_decode_kernel<true, kKindS4>),

                          reinterpret_cast<const void*>(plz_decode_kernel<true, kKindOther>),
                          reinterpret_cast<const void*>(plz_decode_kernel<true, kKindS2>),
                          reinterpret_cast<const void*>(plz_chunk_detail_kernel),
                          reinterpret_cast<const void*>(plz_mono_detail_kernel),
                          reinterpret_cast<const void*>(plz_range_kernel),
                          reinterpret_cast<const void*>(plz_decode_one_kernel)})
        preload_kernel(f);
}

}  // namespace plzgpu
