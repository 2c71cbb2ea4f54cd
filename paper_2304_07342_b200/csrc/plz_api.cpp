// plz_api.cpp — the reference's public C++ API (include/plz/*.hpp) as a thin
// layer over the C-ABI.  compress / compress_block / decompress /
// decompress_bytes / decompress_chunk run on the GPU; the container
// (de)serialisers and parse_token_stream are host-side format helpers, as in
// the reference (format.cpp, decoder.cpp:92-100).
#include <cstring>
#include <memory>
#include <string>

#include "../../include/plz/decoder.hpp"
#include "../../include/plz/errors.hpp"
#include "../../include/plz/format.hpp"
#include "../../include/plz/params.hpp"
#include "../../include/plz/partition.hpp"
#include "../../include/plz/pipeline.hpp"
#include "../../include/plzgpu.h"

namespace plz {
namespace detail {

[[noreturn]] void raise(const plzgpu_error& e) {
    const std::string msg(e.message);
    switch (e.code) {
        case PLZGPU_VALIDATION: throw validation_error(msg);
        case PLZGPU_UNSUPPORTED_FORMAT: throw unsupported_format_error(msg);
        case PLZGPU_CORRUPTION:
            if (e.chunk_index != UINT64_MAX)
                throw corruption_error(msg, std::size_t(e.chunk_index), std::size_t(e.token_index));
            throw corruption_error(msg, std::size_t(e.byte_offset));
        case PLZGPU_CONTRACT: throw contract_error(msg);
        default: throw error(msg);
    }
}

void check(int rc, const plzgpu_error& e) {
    if (rc != PLZGPU_OK) raise(e);
}

struct CtxDeleter {
    void operator()(plzgpu_ctx* c) const { plzgpu_ctx_destroy(c); }
};

// One GPU context per host thread (plzgpu.h threading rule), on device 0
// unless PLZGPU_DEVICE says otherwise.
plzgpu_ctx* ctx() {
    thread_local std::unique_ptr<plzgpu_ctx, CtxDeleter> c;
    if (!c) {
        int dev = 0;
        if (const char* s = std::getenv("PLZGPU_DEVICE")) dev = std::atoi(s);
        plzgpu_ctx* raw = nullptr;
        plzgpu_error e;
        check(plzgpu_ctx_create(dev, &raw, &e), e);
        c.reset(raw);
    }
    return c.get();
}

plzgpu_params to_c(const Params& p) {
    plzgpu_params q{};
    q.symbol_width = p.symbol_width;
    q.window = p.window;
    q.chunk_size = p.chunk_size;
    q.interval = p.interval;
    q.block_bytes = p.block_bytes;
    q.min_match = p.min_match;
    return q;
}

void put_u32(std::vector<std::uint8_t>& o, std::uint32_t v) {
    for (int i = 0; i < 4; ++i) o.push_back(std::uint8_t(v >> (8 * i)));
}

std::uint32_t get_u32(const std::uint8_t* p) {
    return std::uint32_t(p[0]) | std::uint32_t(p[1]) << 8 | std::uint32_t(p[2]) << 16 |
           std::uint32_t(p[3]) << 24;
}

[[noreturn]] void corrupt(const std::string& what, std::size_t off) {
    throw corruption_error("corrupt container: " + what + " (byte " + std::to_string(off) + ")",
                           off);
}

[[noreturn]] void bad_token(const char* what, std::size_t chunk, std::size_t token) {
    throw corruption_error("corrupt chunk " + std::to_string(chunk) + ", token " +
                               std::to_string(token) + ": " + what,
                           chunk, token);
}

}  // namespace detail

using detail::check;

Params validate(Params raw) {
    plzgpu_params in = detail::to_c(raw), out{};
    plzgpu_error e;
    check(plzgpu_validate(&in, &out, &e), e);
    raw.min_match = out.min_match;
    return raw;
}

int level_to_window(int level) {
    std::int32_t w = 0;
    plzgpu_error e;
    check(plzgpu_level_to_window(level, &w, &e), e);
    return w;
}

PartitionPlan plan(std::uint64_t total_bytes, const Params& params) {
    const plzgpu_params p = detail::to_c(params);
    const std::uint64_t n = plzgpu_plan(total_bytes, &p, nullptr, 0);
    std::vector<plzgpu_block_plan> raw(n);
    plzgpu_plan(total_bytes, &p, raw.data(), n);
    PartitionPlan out;
    for (const auto& b : raw)
        out.blocks.push_back(BlockPlan{b.byte_start, b.byte_len, b.num_chunks, b.last_chunk_len,
                                       b.tail_len});
    return out;
}

std::size_t container_size(std::uint32_t num_chunks, std::size_t flag_total,
                           std::size_t payload_total, std::uint8_t tail_len) {
    return plzgpu_container_size(num_chunks, flag_total, payload_total, tail_len);
}

Params params_from_header(const ContainerHeader& h) {
    Params p;
    p.symbol_width = h.symbol_width;
    p.window = h.window;
    p.interval = h.interval;
    p.chunk_size = int(h.chunk_size);
    return validate(p);
}

// format.cpp:75-104 contract: tables consistent with streams before writing.
void append_container(std::vector<std::uint8_t>& out, const Container& c) {
    const std::size_t n = c.header.num_chunks;
    if (c.payload_offsets.size() != n + 1 || c.flag_offsets.size() != n + 1)
        throw contract_error("offset tables must have num_chunks+1 entries");
    for (std::size_t i = 0; i < n; ++i)
        if (c.payload_offsets[i + 1] < c.payload_offsets[i] ||
            c.flag_offsets[i + 1] < c.flag_offsets[i])
            throw contract_error("offset tables must be non-decreasing");
    if (c.payload_offsets[0] != 0 || c.flag_offsets[0] != 0)
        throw contract_error("offset tables must start at 0");
    if (c.payload_offsets[n] != c.payload_stream.size() ||
        c.flag_offsets[n] != c.flag_stream.size())
        throw contract_error("stream lengths must match final table entries");
    if (c.tail.size() != c.header.tail_len) throw contract_error("tail length mismatch");
    params_from_header(c.header);
    if (c.header.original_len < c.header.tail_len)
        throw contract_error("original_len smaller than tail");
    const std::uint64_t sym_bytes = c.header.original_len - c.header.tail_len;
    if (sym_bytes % c.header.symbol_width != 0)
        throw contract_error("original_len not aligned to symbols");
    const std::uint64_t syms = sym_bytes / c.header.symbol_width;
    if ((syms + c.header.chunk_size - 1) / c.header.chunk_size != c.header.num_chunks)
        throw contract_error("num_chunks inconsistent with original_len");

    out.reserve(out.size() + container_size(c.header.num_chunks, c.flag_stream.size(),
                                            c.payload_stream.size(), c.header.tail_len));
    out.insert(out.end(), kMagic.begin(), kMagic.end());
    out.push_back(kFormatVersion);
    out.push_back(c.header.symbol_width);
    out.push_back(c.header.window);
    out.push_back(c.header.interval);
    out.push_back(0);
    detail::put_u32(out, c.header.chunk_size);
    detail::put_u32(out, std::uint32_t(c.header.original_len));
    detail::put_u32(out, std::uint32_t(c.header.original_len >> 32));
    detail::put_u32(out, c.header.num_chunks);
    out.push_back(c.header.tail_len);
    for (const std::uint32_t v : c.payload_offsets) detail::put_u32(out, v);
    for (const std::uint32_t v : c.flag_offsets) detail::put_u32(out, v);
    out.insert(out.end(), c.flag_stream.begin(), c.flag_stream.end());
    out.insert(out.end(), c.payload_stream.begin(), c.payload_stream.end());
    out.insert(out.end(), c.tail.begin(), c.tail.end());
}

std::vector<std::uint8_t> write_container(const Container& c) {
    std::vector<std::uint8_t> out;
    append_container(out, c);
    return out;
}

// format.cpp:112-185: the same checks, order and byte offsets as the device
// parse kernel (decode.cu).
Container read_container(std::span<const std::uint8_t> b, std::size_t& consumed) {
    using detail::corrupt;
    using detail::get_u32;
    if (b.size() < kHeaderSize) corrupt("truncated header", b.size());
    if (std::memcmp(b.data(), kMagic.data(), 4) != 0)
        throw unsupported_format_error("not a PLZ1 container (bad magic)");
    if (b[4] != kFormatVersion)
        throw unsupported_format_error("unsupported container version " + std::to_string(int(b[4])));
    if (b[8] != 0) corrupt("nonzero reserved byte", 8);
    Container c;
    c.header.symbol_width = b[5];
    c.header.window = b[6];
    c.header.interval = b[7];
    c.header.chunk_size = get_u32(b.data() + 9);
    c.header.original_len = std::uint64_t(get_u32(b.data() + 13)) |
                            std::uint64_t(get_u32(b.data() + 17)) << 32;
    c.header.num_chunks = get_u32(b.data() + 21);
    c.header.tail_len = b[25];
    try {
        params_from_header(c.header);
    } catch (const validation_error& e) {
        corrupt(e.what(), 5);
    }
    if (c.header.tail_len >= c.header.symbol_width) corrupt("tail_len >= symbol_width", 25);
    const std::size_t n = c.header.num_chunks;
    std::size_t at = kHeaderSize;
    if (b.size() < at + 8 * (n + 1)) corrupt("truncated offset tables", b.size());
    c.payload_offsets.resize(n + 1);
    c.flag_offsets.resize(n + 1);
    for (std::size_t i = 0; i <= n; ++i, at += 4) c.payload_offsets[i] = get_u32(b.data() + at);
    for (std::size_t i = 0; i <= n; ++i, at += 4) c.flag_offsets[i] = get_u32(b.data() + at);
    for (std::size_t i = 0; i < n; ++i) {
        if (c.payload_offsets[i + 1] < c.payload_offsets[i])
            corrupt("payload offsets not monotone", kHeaderSize + 4 * (i + 1));
        if (c.flag_offsets[i + 1] < c.flag_offsets[i])
            corrupt("flag offsets not monotone", kHeaderSize + 4 * (n + 1) + 4 * (i + 1));
    }
    if (c.payload_offsets[0] != 0) corrupt("payload offsets must start at 0", kHeaderSize);
    if (c.flag_offsets[0] != 0) corrupt("flag offsets must start at 0", kHeaderSize + 4 * (n + 1));
    const std::size_t ftot = c.flag_offsets[n], ptot = c.payload_offsets[n];
    const std::size_t need = container_size(c.header.num_chunks, ftot, ptot, c.header.tail_len);
    if (b.size() < need) corrupt("truncated streams", b.size());
    const std::uint64_t S = c.header.symbol_width, C = c.header.chunk_size;
    if (c.header.original_len < c.header.tail_len) corrupt("original_len too small", 13);
    const std::uint64_t sym_bytes = c.header.original_len - c.header.tail_len;
    if (sym_bytes % S != 0) corrupt("original_len not aligned to symbols", 13);
    if ((sym_bytes / S + C - 1) / C != n) corrupt("num_chunks inconsistent with original_len", 21);
    c.flag_stream.assign(b.begin() + long(at), b.begin() + long(at + ftot));
    at += ftot;
    c.payload_stream.assign(b.begin() + long(at), b.begin() + long(at + ptot));
    at += ptot;
    c.tail.assign(b.begin() + long(at), b.begin() + long(at + c.header.tail_len));
    at += c.header.tail_len;
    consumed = at;
    return c;
}

std::vector<std::uint8_t> compress(std::span<const std::uint8_t> data, const Params& params,
                                   int /*threads*/, PipelineStats* stats) {
    const plzgpu_params p = detail::to_c(params);
    plzgpu_error e;
    {
        plzgpu_params v{};
        check(plzgpu_validate(&p, &v, &e), e);
    }
    std::vector<std::uint8_t> out(plzgpu_compress_bound(data.size(), &p));
    std::uint64_t len = 0;
    plzgpu_stats st{};
    plzgpu_ctx* c = detail::ctx();
    check(plzgpu_compress(c, &p, data.data(), data.size(), out.data(), out.size(), &len, &st,
                          plzgpu_ctx_stream(c), &e),
          e);
    out.resize(len);
    if (stats) {
        stats->pointer_tokens += st.pointer_tokens;
        stats->literal_tokens += st.literal_tokens;
    }
    return out;
}

Container compress_block(std::span<const std::uint8_t> block, const BlockPlan& bp,
                         const Params& params, int threads, PipelineStats* stats) {
    if (block.size() != bp.byte_len) throw contract_error("block span does not match plan");
    Params one = params;
    const std::size_t cb = std::size_t(params.chunk_size) * std::size_t(params.symbol_width);
    if (cb && one.block_bytes < block.size())  // keep the block in one container
        one.block_bytes = (block.size() + cb - 1) / cb * cb;
    const std::vector<std::uint8_t> img = compress(block, one, threads, stats);
    if (img.empty()) {
        Container c;
        c.header.symbol_width = std::uint8_t(params.symbol_width);
        c.header.window = std::uint8_t(params.window);
        c.header.interval = std::uint8_t(params.interval);
        c.header.chunk_size = std::uint32_t(params.chunk_size);
        c.payload_offsets = {0};
        c.flag_offsets = {0};
        return c;
    }
    std::size_t consumed = 0;
    return read_container(img, consumed);
}

std::vector<std::uint8_t> decompress_bytes(std::span<const std::uint8_t> bytes, int /*threads*/) {
    std::vector<std::uint8_t> out(plzgpu_decompressed_bound(bytes.data(), bytes.size()));
    std::uint64_t len = 0;
    plzgpu_error e;
    plzgpu_ctx* c = detail::ctx();
    check(plzgpu_decompress(c, bytes.data(), bytes.size(), out.data(), out.size(), &len,
                            plzgpu_ctx_stream(c), &e),
          e);
    out.resize(len);
    return out;
}

std::vector<std::uint8_t> decompress(const Container& container, int threads) {
    return decompress_bytes(write_container(container), threads);
}

std::vector<std::uint8_t> decompress_chunk(std::span<const std::uint8_t> flags,
                                           std::span<const std::uint8_t> payload,
                                           std::size_t logical_len, const Params& params,
                                           std::size_t chunk_index) {
    std::vector<std::uint8_t> out(logical_len * std::size_t(params.symbol_width));
    const plzgpu_params p = detail::to_c(params);
    plzgpu_error e;
    check(plzgpu_decompress_chunk(detail::ctx(), flags.data(), flags.size(), payload.data(),
                                  payload.size(), logical_len, &p, chunk_index, out.data(), &e),
          e);
    return out;
}

// decoder.cpp:22-66 token walk on the host — a verification/statistics API
// (the reference uses it from tests and tooling, never on the codec path).
std::vector<PlacedToken> parse_token_stream(std::span<const std::uint8_t> flags,
                                            std::span<const std::uint8_t> payload,
                                            std::size_t logical_len, const Params& params,
                                            std::size_t chunk_index) {
    using detail::bad_token;
    const std::size_t s = std::size_t(params.symbol_width);
    std::vector<PlacedToken> tokens;
    std::size_t written = 0, in = 0, t = 0;
    while (written < logical_len) {
        if (t / 8 >= flags.size()) bad_token("flag bits exhausted", chunk_index, t);
        const bool ptr = (flags[t / 8] >> (7 - t % 8)) & 1;
        PlacedToken tok;
        tok.pos = written;
        if (ptr) {
            if (in + 2 > payload.size()) bad_token("payload exhausted", chunk_index, t);
            tok.is_pointer = true;
            tok.length = payload[in];
            tok.offset = payload[in + 1];
            in += 2;
            if (tok.length == 0 || tok.offset == 0) bad_token("zero pointer field", chunk_index, t);
            if (tok.offset > written) bad_token("offset before chunk start", chunk_index, t);
            if (written + tok.length > logical_len)
                bad_token("pointer overruns chunk", chunk_index, t);
            written += tok.length;
        } else {
            if (in + s > payload.size()) bad_token("payload exhausted", chunk_index, t);
            std::memcpy(tok.literal.data(), payload.data() + in, s);
            in += s;
            written += 1;
        }
        tokens.push_back(tok);
        ++t;
    }
    if (in != payload.size()) bad_token("trailing payload bytes", chunk_index, t);
    for (std::size_t b = t; b < flags.size() * 8; ++b)
        if ((flags[b / 8] >> (7 - b % 8)) & 1) bad_token("nonzero flag padding", chunk_index, b);
    if (flags.size() != (t + 7) / 8)
        bad_token("flag bytes inconsistent with token count", chunk_index, t);
    return tokens;
}

}  // namespace plz
