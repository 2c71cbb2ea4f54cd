/*
 * plz_oracle.c — TEST INFRASTRUCTURE ONLY (see plz_oracle.h).
 *
 * Plain-C restatement of the reference CPU path, written from its behavioural
 * contract.  Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/).  Single-threaded and
 * deliberately simple: it is the checker, never the thing measured or shipped.
 */
#include "plz_oracle.h"

#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NO_INDEX UINT64_MAX

static int set_err(plzo_error* e, int code, uint64_t off, uint64_t chunk, uint64_t tok,
                   const char* fmt, ...) {
    if (e) {
        va_list ap;
        e->code = code;
        e->byte_offset = off;
        e->chunk_index = chunk;
        e->token_index = tok;
        va_start(ap, fmt);
        vsnprintf(e->message, sizeof e->message, fmt, ap);
        va_end(ap);
    }
    return code;
}

static void clear_err(plzo_error* e) {
    if (e) {
        memset(e, 0, sizeof *e);
        e->chunk_index = NO_INDEX;
        e->token_index = NO_INDEX;
    }
}

/* ---------------------------------------------------------------- params */

static int bad_param(plzo_error* e, const char* field, const char* legal) {
    return set_err(e, PLZO_VALIDATION, 0, NO_INDEX, NO_INDEX,
                   "invalid %s: legal range is %s", field, legal);
}

/* params.cpp:19-45 — same checks in the same order, min_match = 2/S + 1. */
int plzo_validate(const plzo_params* raw, plzo_params* out, plzo_error* err) {
    plzo_params p = *raw;
    clear_err(err);
    if (p.symbol_width != 1 && p.symbol_width != 2 && p.symbol_width != 4)
        return bad_param(err, "symbol_width", "{1,2,4}");
    if (p.window < 4 || p.window > 255)
        return bad_param(err, "window", "[4,255] (0 is reserved for no-match)");
    if (p.chunk_size != 1024 && p.chunk_size != 2048 && p.chunk_size != 4096 &&
        p.chunk_size != 8192 && p.chunk_size != 16384)
        return bad_param(err, "chunk_size", "{1024,2048,4096,8192,16384}");
    if (p.chunk_size <= p.window) return bad_param(err, "chunk_size", "greater than window");
    if (p.interval != 1 && p.interval != 2 && p.interval != 4 && p.interval != 8 &&
        p.interval != 16)
        return bad_param(err, "interval", "{1,2,4,8,16}");
    if (p.chunk_size % p.interval != 0)
        return bad_param(err, "interval", "a divisor of chunk_size");
    {
        uint64_t chunk_bytes = (uint64_t)p.chunk_size * (uint64_t)p.symbol_width;
        if (p.block_bytes == 0 || p.block_bytes % chunk_bytes != 0)
            return bad_param(err, "block_bytes",
                             "a positive multiple of chunk_size*symbol_width");
    }
    /* (power-of-two check at params.cpp:40-41 is implied by the set above) */
    p.min_match = 2 / p.symbol_width + 1;
    if (out) *out = p;
    return PLZO_OK;
}

/* params.cpp:47-55 */
int plzo_level_to_window(int level) {
    switch (level) {
        case 1: return 32;
        case 2: return 64;
        case 3: return 128;
        case 4: return 255;
        default: return -1;
    }
}

/* ------------------------------------------------------------- partition */

typedef struct {
    uint64_t byte_start, byte_len;
    uint32_t num_chunks, last_chunk_len;
    uint8_t tail_len;
} block_plan;

/* partition.cpp:5-25 for the block starting at `pos`. */
static block_plan plan_block(uint64_t pos, uint64_t total, const plzo_params* p) {
    block_plan b;
    uint64_t s = (uint64_t)p->symbol_width, c = (uint64_t)p->chunk_size, symbols;
    b.byte_start = pos;
    b.byte_len = total - pos < p->block_bytes ? total - pos : p->block_bytes;
    symbols = b.byte_len / s;
    b.tail_len = (uint8_t)(b.byte_len % s);
    b.num_chunks = 0;
    b.last_chunk_len = 0;
    if (symbols > 0) {
        b.num_chunks = (uint32_t)((symbols + c - 1) / c);
        b.last_chunk_len = (uint32_t)(symbols - (uint64_t)(b.num_chunks - 1) * c);
    }
    return b;
}

uint64_t plzo_compress_bound(uint64_t n, const plzo_params* p) {
    uint64_t pos = 0, total = 0;
    while (pos < n) {
        block_plan b = plan_block(pos, n, p);
        uint64_t symbols = b.byte_len / (uint64_t)p->symbol_width;
        /* all-literal chunks: S bytes/symbol + ceil(len/8) flag bytes per chunk */
        total += 26 + 8 * ((uint64_t)b.num_chunks + 1) + symbols * (uint64_t)p->symbol_width +
                 symbols / 8 + b.num_chunks + b.tail_len;
        pos += b.byte_len;
    }
    return total;
}

/* --------------------------------------------------------------- matcher */

/* matcher.cpp:9-34: little-endian S-byte symbols widened to u32. */
static uint32_t symbol_at(const uint8_t* bytes, uint64_t i, int s) {
    const uint8_t* q = bytes + i * (uint64_t)s;
    uint32_t v = 0;
    int b;
    for (b = 0; b < s; ++b) v |= (uint32_t)q[b] << (8 * b);
    return v;
}

/* The matcher's result contract (matcher.hpp:28-31, matcher.cpp:71-111,
 * test_matcher.cpp:26-42): over window starts w in [max(0,p-W), p), the
 * candidate length is the count of consecutive equal symbols capped at
 * min(p-w, 255, n-p); the longest wins and ties go to the smallest w (largest
 * offset).  Returns {len, off} with {0,0} for no match.  Restated as the plain
 * exhaustive scan; the reference's run-skipping and early exits do not change
 * the result (test_matcher.cpp:74-89). */
static void find_match(const uint32_t* sym, uint64_t n, uint64_t pos, int window,
                       uint8_t* len, uint8_t* off) {
    uint64_t lo = pos > (uint64_t)window ? pos - (uint64_t)window : 0, w;
    uint64_t best_len = 0, best_w = 0;
    for (w = lo; w < pos; ++w) {
        uint64_t cap = pos - w, k = 0;
        if (cap > 255) cap = 255;
        if (cap > n - pos) cap = n - pos;
        while (k < cap && sym[w + k] == sym[pos + k]) ++k;
        if (k > best_len) {
            best_len = k;
            best_w = w;
        }
    }
    if (best_len == 0) {
        *len = 0;
        *off = 0;
    } else {
        *len = (uint8_t)best_len;
        *off = (uint8_t)(pos - best_w);
    }
}

/* matcher.cpp:113-131: interval-aligned (chunk-relative) positions are
 * searched, every other position is the forced literal {1,0}. */
int plzo_match_chunk(const uint8_t* chunk_bytes, uint64_t n, const plzo_params* p,
                     uint8_t* len, uint8_t* off) {
    uint32_t* sym = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
    uint64_t i;
    if (!sym) return PLZO_CONTRACT;
    for (i = 0; i < n; ++i) sym[i] = symbol_at(chunk_bytes, i, p->symbol_width);
    for (i = 0; i < n; ++i) {
        if (i % (uint64_t)p->interval != 0) {
            len[i] = 1;
            off[i] = 0;
        } else {
            find_match(sym, n, i, p->window, &len[i], &off[i]);
        }
    }
    free(sym);
    return PLZO_OK;
}

/* --------------------------------------------------------------- encoder */

/* encoder.cpp:18-73 fused: the greedy walk from position 0 (pointer iff
 * offset != 0 and length >= min_match, encoder.cpp:12-14), MSB-first flag
 * bits (encoder.cpp:27,33), pointer wire order [length][offset]
 * (encoder.cpp:64-65), literal = the S raw input bytes (encoder.cpp:68).
 * Only records at positions the walk visits can influence the output, so the
 * match is computed exactly there (the same values match_chunk would hold).
 * Returns payload bytes; *n_flags / *n_tokens / *n_ptr receive the rest. */
static uint64_t encode_chunk(const uint8_t* bytes, uint64_t n, const plzo_params* p,
                             uint32_t* sym, uint8_t* payload, uint8_t* flags,
                             uint64_t* n_flags, uint64_t* n_tokens, uint64_t* n_ptr) {
    const int s = p->symbol_width;
    uint64_t i = 0, t = 0, pay = 0, ptr = 0;
    for (i = 0; i < n; ++i) sym[i] = symbol_at(bytes, i, s);
    i = 0;
    while (i < n) {
        uint8_t len = 1, off = 0;
        if (t % 8 == 0) flags[t / 8] = 0;
        if (i % (uint64_t)p->interval == 0) find_match(sym, n, i, p->window, &len, &off);
        if (off != 0 && (int)len >= p->min_match) {
            flags[t / 8] |= (uint8_t)(0x80u >> (t % 8));
            payload[pay++] = len;
            payload[pay++] = off;
            i += len;
            ++ptr;
        } else {
            memcpy(payload + pay, bytes + i * (uint64_t)s, (size_t)s);
            pay += (uint64_t)s;
            i += 1;
        }
        ++t;
    }
    *n_flags = (t + 7) / 8;
    *n_tokens = t;
    *n_ptr = ptr;
    return pay;
}

static void put_u32(uint8_t* o, uint32_t v) {
    o[0] = (uint8_t)v;
    o[1] = (uint8_t)(v >> 8);
    o[2] = (uint8_t)(v >> 16);
    o[3] = (uint8_t)(v >> 24);
}

static void put_u64(uint8_t* o, uint64_t v) {
    int i;
    for (i = 0; i < 8; ++i) o[i] = (uint8_t)(v >> (8 * i));
}

static uint32_t get_u32(const uint8_t* q) {
    return (uint32_t)q[0] | ((uint32_t)q[1] << 8) | ((uint32_t)q[2] << 16) |
           ((uint32_t)q[3] << 24);
}

static uint64_t get_u64(const uint8_t* q) {
    uint64_t v = 0;
    int i;
    for (i = 0; i < 8; ++i) v |= (uint64_t)q[i] << (8 * i);
    return v;
}

/* pipeline.cpp:26-99 + deflate.cpp:10-47 + scan.cpp:38-47 + format.cpp:75-104:
 * blocks in order; per block every chunk is encoded, sizes are prefix-summed
 * into u32 tables (overflow -> validation_error, scan.cpp:43-44), and the
 * container is serialised as header | payload_offsets | flag_offsets |
 * flag_stream | payload_stream | tail. */
int plzo_compress(const uint8_t* in, uint64_t n, const plzo_params* p, uint8_t* out,
                  uint64_t cap, uint64_t* out_len, uint64_t* stats, plzo_error* err) {
    plzo_params v;
    uint64_t pos = 0, at = 0, ptr_total = 0, lit_total = 0;
    const uint64_t s = (uint64_t)p->symbol_width, c = (uint64_t)p->chunk_size;
    uint32_t* sym = NULL;
    uint8_t *pay = NULL, *flg = NULL;
    uint64_t *psz = NULL, *fsz = NULL;
    int rc;

    clear_err(err);
    rc = plzo_validate(p, &v, err);
    if (rc) return rc;
    *out_len = 0;
    if (n == 0) return PLZO_OK;
    sym = (uint32_t*)malloc(c * sizeof(uint32_t));
    while (pos < n && rc == PLZO_OK) {
        block_plan b = plan_block(pos, n, p);
        uint64_t k, ptot = 0, ftot = 0, hdr, size;
        const uint8_t* blk = in + b.byte_start;
        pay = (uint8_t*)realloc(pay, b.byte_len + 16);
        flg = (uint8_t*)realloc(flg, b.byte_len / 8 + b.num_chunks + 16);
        psz = (uint64_t*)realloc(psz, ((uint64_t)b.num_chunks + 1) * sizeof(uint64_t));
        fsz = (uint64_t*)realloc(fsz, ((uint64_t)b.num_chunks + 1) * sizeof(uint64_t));
        for (k = 0; k < b.num_chunks; ++k) {
            uint64_t logical = k + 1 == b.num_chunks ? b.last_chunk_len : c;
            uint64_t nf, nt, np;
            psz[k] = encode_chunk(blk + k * c * s, logical, p, sym, pay + ptot, flg + ftot,
                                  &nf, &nt, &np);
            fsz[k] = nf;
            ptot += psz[k];
            ftot += nf;
            ptr_total += np;
            lit_total += nt - np;
            if (ptot > UINT32_MAX || ftot > UINT32_MAX) {
                rc = set_err(err, PLZO_VALIDATION, 0, NO_INDEX, NO_INDEX,
                             "block too large: offsets exceed 4-byte table range");
                break;
            }
        }
        if (rc) break;
        hdr = 26 + 8 * ((uint64_t)b.num_chunks + 1);
        size = hdr + ftot + ptot + b.tail_len;
        if (at + size > cap) {
            rc = set_err(err, PLZO_CAPACITY, 0, NO_INDEX, NO_INDEX, "output buffer too small");
            break;
        }
        {
            uint8_t* o = out + at;
            uint64_t acc;
            memcpy(o, "PLZ1", 4);
            o[4] = 1;
            o[5] = (uint8_t)p->symbol_width;
            o[6] = (uint8_t)p->window;
            o[7] = (uint8_t)p->interval;
            o[8] = 0;
            put_u32(o + 9, (uint32_t)p->chunk_size);
            put_u64(o + 13, b.byte_len);
            put_u32(o + 21, b.num_chunks);
            o[25] = b.tail_len;
            acc = 0;
            for (k = 0; k <= b.num_chunks; ++k) {
                put_u32(o + 26 + 4 * k, (uint32_t)acc);
                if (k < b.num_chunks) acc += psz[k];
            }
            acc = 0;
            for (k = 0; k <= b.num_chunks; ++k) {
                put_u32(o + 26 + 4 * ((uint64_t)b.num_chunks + 1) + 4 * k, (uint32_t)acc);
                if (k < b.num_chunks) acc += fsz[k];
            }
            memcpy(o + hdr, flg, ftot);
            memcpy(o + hdr + ftot, pay, ptot);
            memcpy(o + hdr + ftot + ptot, blk + b.byte_len - b.tail_len, b.tail_len);
        }
        at += size;
        pos += b.byte_len;
    }
    free(sym);
    free(pay);
    free(flg);
    free(psz);
    free(fsz);
    if (rc) return rc;
    *out_len = at;
    if (stats) {
        stats[0] = 0; /* max_cmp_per_pos: CPU-matcher instrumentation, n/a */
        stats[1] = ptr_total;
        stats[2] = lit_total;
    }
    return PLZO_OK;
}

/* --------------------------------------------------------------- decoder */

static int bad_token(plzo_error* e, const char* what, uint64_t chunk, uint64_t token) {
    return set_err(e, PLZO_CORRUPTION, 0, chunk, token, "corrupt chunk %llu, token %llu: %s",
                   (unsigned long long)chunk, (unsigned long long)token, what);
}

/* decoder.cpp:22-90 — token walk with the reference's checks in its order;
 * pointer copies run forward symbol-byte by byte so malformed overlapping
 * pointers replicate (decoder.cpp:80-84). */
int plzo_decompress_chunk(const uint8_t* flags, uint64_t nf, const uint8_t* payload,
                          uint64_t np, uint64_t logical, const plzo_params* p,
                          uint64_t chunk, uint8_t* out, plzo_error* err) {
    const uint64_t s = (uint64_t)p->symbol_width;
    uint64_t written = 0, in = 0, token = 0, b;
    clear_err(err);
    while (written < logical) {
        int pointer;
        if (token / 8 >= nf) return bad_token(err, "flag bits exhausted", chunk, token);
        pointer = (flags[token / 8] >> (7 - token % 8)) & 1;
        if (pointer) {
            uint8_t length, offset;
            uint64_t k;
            if (in + 2 > np) return bad_token(err, "payload exhausted", chunk, token);
            length = payload[in];
            offset = payload[in + 1];
            in += 2;
            if (length == 0 || offset == 0)
                return bad_token(err, "zero pointer field", chunk, token);
            if (offset > written) return bad_token(err, "offset before chunk start", chunk, token);
            if (written + length > logical)
                return bad_token(err, "pointer overruns chunk", chunk, token);
            for (k = 0; k < (uint64_t)length * s; ++k)
                out[written * s + k] = out[written * s - (uint64_t)offset * s + k];
            written += length;
        } else {
            if (in + s > np) return bad_token(err, "payload exhausted", chunk, token);
            memcpy(out + written * s, payload + in, (size_t)s);
            in += s;
            written += 1;
        }
        ++token;
    }
    if (in != np) return bad_token(err, "trailing payload bytes", chunk, token);
    for (b = token; b < nf * 8; ++b)
        if ((flags[b / 8] >> (7 - b % 8)) & 1)
            return bad_token(err, "nonzero flag padding", chunk, b);
    if (nf != (token + 7) / 8)
        return bad_token(err, "flag bytes inconsistent with token count", chunk, token);
    return PLZO_OK;
}

typedef struct {
    plzo_params p;
    uint64_t original_len;
    uint32_t chunk_size, num_chunks;
    uint8_t tail_len;
    const uint8_t *ptab, *ftab, *flags, *payload, *tail;
    uint64_t consumed;
} parsed_container;

static int corrupt(plzo_error* e, const char* what, uint64_t off) {
    return set_err(e, PLZO_CORRUPTION, off, NO_INDEX, NO_INDEX,
                   "corrupt container: %s (byte %llu)", what, (unsigned long long)off);
}

/* format.cpp:112-185 — every check in the reference's order, byte offsets
 * relative to the container start. */
static int read_container(const uint8_t* bytes, uint64_t size, parsed_container* c,
                          plzo_error* err) {
    uint64_t n, at, i, flag_total, payload_total, need, s, cs, symbol_bytes, symbols;
    plzo_params raw;
    plzo_error verr;
    if (size < 26) return corrupt(err, "truncated header", size);
    if (memcmp(bytes, "PLZ1", 4) != 0)
        return set_err(err, PLZO_UNSUPPORTED_FORMAT, 0, NO_INDEX, NO_INDEX,
                       "not a PLZ1 container (bad magic)");
    if (bytes[4] != 1)
        return set_err(err, PLZO_UNSUPPORTED_FORMAT, 0, NO_INDEX, NO_INDEX,
                       "unsupported container version %d", (int)bytes[4]);
    if (bytes[8] != 0) return corrupt(err, "nonzero reserved byte", 8);
    c->chunk_size = get_u32(bytes + 9);
    c->original_len = get_u64(bytes + 13);
    c->num_chunks = get_u32(bytes + 21);
    c->tail_len = bytes[25];
    /* params_from_header (format.cpp:60-67): default block_bytes */
    raw.symbol_width = bytes[5];
    raw.window = bytes[6];
    raw.interval = bytes[7];
    raw.chunk_size = (int32_t)c->chunk_size;
    raw.block_bytes = (uint64_t)256 << 20;
    raw.min_match = 2;
    raw.reserved = 0;
    if (plzo_validate(&raw, &c->p, &verr) != PLZO_OK) return corrupt(err, verr.message, 5);
    if (c->tail_len >= bytes[5]) return corrupt(err, "tail_len >= symbol_width", 25);
    n = c->num_chunks;
    at = 26;
    if (size < at + 8 * (n + 1)) return corrupt(err, "truncated offset tables", size);
    c->ptab = bytes + at;
    c->ftab = bytes + at + 4 * (n + 1);
    for (i = 0; i < n; ++i) {
        if (get_u32(c->ptab + 4 * (i + 1)) < get_u32(c->ptab + 4 * i))
            return corrupt(err, "payload offsets not monotone", 26 + 4 * (i + 1));
        if (get_u32(c->ftab + 4 * (i + 1)) < get_u32(c->ftab + 4 * i))
            return corrupt(err, "flag offsets not monotone", 26 + 4 * (n + 1) + 4 * (i + 1));
    }
    if (get_u32(c->ptab) != 0) return corrupt(err, "payload offsets must start at 0", 26);
    if (get_u32(c->ftab) != 0)
        return corrupt(err, "flag offsets must start at 0", 26 + 4 * (n + 1));
    flag_total = get_u32(c->ftab + 4 * n);
    payload_total = get_u32(c->ptab + 4 * n);
    need = 26 + 8 * (n + 1) + flag_total + payload_total + c->tail_len;
    if (size < need) return corrupt(err, "truncated streams", size);
    s = bytes[5];
    cs = c->chunk_size;
    if (c->original_len < c->tail_len) return corrupt(err, "original_len too small", 13);
    symbol_bytes = c->original_len - c->tail_len;
    if (symbol_bytes % s != 0) return corrupt(err, "original_len not aligned to symbols", 13);
    symbols = symbol_bytes / s;
    if ((symbols + cs - 1) / cs != n)
        return corrupt(err, "num_chunks inconsistent with original_len", 21);
    c->flags = bytes + 26 + 8 * (n + 1);
    c->payload = c->flags + flag_total;
    c->tail = c->payload + payload_total;
    c->consumed = need;
    return PLZO_OK;
}

/* decoder.cpp:102-141: containers in order; inside one, chunks in index
 * order (the threads=1 schedule, so the lowest failing chunk reports). */
int plzo_decompress(const uint8_t* img, uint64_t len, uint8_t* out, uint64_t cap,
                    uint64_t* out_len, plzo_error* err) {
    uint64_t at = 0, produced = 0;
    clear_err(err);
    *out_len = 0;
    while (at < len) {
        parsed_container c;
        int rc = read_container(img + at, len - at, &c, err);
        if (rc) {
            if (!out) {  /* size query: the parseable prefix; errors come from decoding */
                clear_err(err);
                break;
            }
            return rc;
        }
        if (out) {
            uint64_t k, s = (uint64_t)c.p.symbol_width, cs = c.chunk_size;
            uint64_t symbols = (c.original_len - c.tail_len) / s;
            if (produced + c.original_len > cap)
                return set_err(err, PLZO_CAPACITY, 0, NO_INDEX, NO_INDEX,
                               "output buffer too small");
            for (k = 0; k < c.num_chunks; ++k) {
                uint64_t logical = k + 1 == c.num_chunks ? symbols - k * cs : cs;
                uint32_t f0 = get_u32(c.ftab + 4 * k), f1 = get_u32(c.ftab + 4 * (k + 1));
                uint32_t p0 = get_u32(c.ptab + 4 * k), p1 = get_u32(c.ptab + 4 * (k + 1));
                rc = plzo_decompress_chunk(c.flags + f0, f1 - f0, c.payload + p0, p1 - p0,
                                           logical, &c.p, k, out + produced + k * cs * s, err);
                if (rc) return rc;
            }
            memcpy(out + produced + c.original_len - c.tail_len, c.tail, c.tail_len);
        }
        produced += c.original_len;
        at += c.consumed;
    }
    *out_len = produced;
    return PLZO_OK;
}
