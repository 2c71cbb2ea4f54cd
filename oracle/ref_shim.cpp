// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" face of the UNMODIFIED reference library, compiled from its own
// sources under /root/reference/proj/src with -Dplz=plzref (oracle/Makefile),
// so ctypes-based tests and bench.py's reference arm can call
// plzref::compress / plzref::decompress_bytes directly.  The reference's C++
// exceptions are mapped onto the same error codes the B200 C-ABI uses
// (include/plzgpu.h).  Output is allocated with malloc; free it with
// plzref_free.
#include <cstdlib>
#include <cstring>
#include <exception>
#include <span>
#include <vector>

#include "plz/decoder.hpp"
#include "plz/errors.hpp"
#include "plz/format.hpp"
#include "plz/matcher.hpp"
#include "plz/params.hpp"
#include "plz/partition.hpp"
#include "plz/pipeline.hpp"
#include "plz_oracle.h"

namespace {

void fill(plzo_error* e, int code, const char* msg, std::size_t off = 0,
          std::size_t chunk = SIZE_MAX, std::size_t token = SIZE_MAX) {
    if (!e) return;
    std::memset(e, 0, sizeof *e);
    e->code = code;
    e->byte_offset = off;
    e->chunk_index = chunk == SIZE_MAX ? UINT64_MAX : chunk;
    e->token_index = token == SIZE_MAX ? UINT64_MAX : token;
    std::strncpy(e->message, msg, sizeof e->message - 1);
}

template <typename F>
int guarded(plzo_error* err, F&& body) {
    fill(err, PLZO_OK, "");
    try {
        body();
        return PLZO_OK;
    } catch (const plz::corruption_error& e) {
        fill(err, PLZO_CORRUPTION, e.what(), e.byte_offset, e.chunk_index, e.token_index);
        return PLZO_CORRUPTION;
    } catch (const plz::unsupported_format_error& e) {
        fill(err, PLZO_UNSUPPORTED_FORMAT, e.what());
        return PLZO_UNSUPPORTED_FORMAT;
    } catch (const plz::validation_error& e) {
        fill(err, PLZO_VALIDATION, e.what());
        return PLZO_VALIDATION;
    } catch (const plz::contract_error& e) {
        fill(err, PLZO_CONTRACT, e.what());
        return PLZO_CONTRACT;
    } catch (const std::exception& e) {
        fill(err, 99, e.what());
        return 99;
    }
}

plz::Params to_params(const plzo_params* p) {
    plz::Params q;
    q.symbol_width = p->symbol_width;
    q.window = p->window;
    q.chunk_size = p->chunk_size;
    q.interval = p->interval;
    q.block_bytes = p->block_bytes;
    q.min_match = p->min_match;
    return q;
}

unsigned char* dup(const std::vector<std::uint8_t>& v) {
    auto* out = static_cast<unsigned char*>(std::malloc(v.size() ? v.size() : 1));
    if (!v.empty()) std::memcpy(out, v.data(), v.size());
    return out;
}

}  // namespace

extern "C" {

void plzref_free(void* p) { std::free(p); }

int plzref_validate(const plzo_params* raw, plzo_params* out, plzo_error* err) {
    return guarded(err, [&] {
        const plz::Params v = plz::validate(to_params(raw));
        *out = *raw;
        out->min_match = v.min_match;
    });
}

int plzref_compress(const unsigned char* in, std::uint64_t n, const plzo_params* p,
                    int threads, unsigned char** out, std::uint64_t* out_len,
                    std::uint64_t* stats, plzo_error* err) {
    *out = nullptr;
    *out_len = 0;
    return guarded(err, [&] {
        plz::PipelineStats st;
        const auto img =
            plz::compress(std::span<const std::uint8_t>(in, n), to_params(p), threads, &st);
        *out = dup(img);
        *out_len = img.size();
        if (stats) {
            stats[0] = st.max_cmp_per_pos;
            stats[1] = st.pointer_tokens;
            stats[2] = st.literal_tokens;
        }
    });
}

// plzref::compress_block (pipeline.cpp:26-86) for one block of a plan,
// serialised with plzref::write_container (format.cpp:75-104).
int plzref_compress_block(const unsigned char* block, std::uint64_t n, std::uint64_t byte_start,
                          std::uint64_t byte_len, std::uint32_t num_chunks,
                          std::uint32_t last_chunk_len, std::uint8_t tail_len,
                          const plzo_params* p, int threads, unsigned char** out,
                          std::uint64_t* out_len, std::uint64_t* stats, plzo_error* err) {
    *out = nullptr;
    *out_len = 0;
    return guarded(err, [&] {
        plz::BlockPlan bp;
        bp.byte_start = byte_start;
        bp.byte_len = byte_len;
        bp.num_chunks = num_chunks;
        bp.last_chunk_len = last_chunk_len;
        bp.tail_len = tail_len;
        plz::PipelineStats st;
        const plz::Container c = plz::compress_block(std::span<const std::uint8_t>(block, n), bp,
                                                     to_params(p), threads, &st);
        const auto img = plz::write_container(c);
        *out = dup(img);
        *out_len = img.size();
        if (stats) {
            stats[0] = st.max_cmp_per_pos;
            stats[1] = st.pointer_tokens;
            stats[2] = st.literal_tokens;
        }
    });
}

int plzref_decompress(const unsigned char* img, std::uint64_t len, int threads,
                      unsigned char** out, std::uint64_t* out_len, plzo_error* err) {
    *out = nullptr;
    *out_len = 0;
    return guarded(err, [&] {
        const auto data =
            plz::decompress_bytes(std::span<const std::uint8_t>(img, len), threads);
        *out = dup(data);
        *out_len = data.size();
    });
}

int plzref_decompress_chunk(const unsigned char* flags, std::uint64_t nf,
                            const unsigned char* payload, std::uint64_t np,
                            std::uint64_t logical, const plzo_params* p,
                            std::uint64_t chunk_index, unsigned char* out, plzo_error* err) {
    return guarded(err, [&] {
        const auto v = plz::decompress_chunk(std::span<const std::uint8_t>(flags, nf),
                                             std::span<const std::uint8_t>(payload, np),
                                             logical, to_params(p), chunk_index);
        if (!v.empty()) std::memcpy(out, v.data(), v.size());
    });
}

int plzref_match_chunk(const unsigned char* bytes, std::uint64_t n_symbols,
                       const plzo_params* p, unsigned char* len, unsigned char* off) {
    plzo_error err;
    return guarded(&err, [&] {
        std::vector<std::uint32_t> sym;
        plz::load_symbols(std::span<const std::uint8_t>(bytes, n_symbols * p->symbol_width),
                          p->symbol_width, sym);
        const plz::MatchTable t = plz::match_chunk(sym, to_params(p));
        for (std::size_t i = 0; i < t.records.size(); ++i) {
            len[i] = t.records[i].length;
            off[i] = t.records[i].offset;
        }
    });
}

}  // extern "C"
