// host_common.cpp — errors, parameter checks, geometry, the pipeline config
// and the driver entry points shared by every C-ABI unit (host_internal.h).
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "host_internal.h"

namespace plzhost {

int set_err(plzgpu_error* e, int code, uint64_t off, uint64_t chunk, uint64_t tok, const char* fmt,
            ...) {
    if (e) {
        e->code = code;
        e->reserved = 0;
        e->byte_offset = off;
        e->chunk_index = chunk;
        e->token_index = tok;
        va_list ap;
        va_start(ap, fmt);
        std::vsnprintf(e->message, sizeof e->message, fmt, ap);
        va_end(ap);
    }
    return code;
}

void clear_err(plzgpu_error* e) {
    if (e) {
        std::memset(e, 0, sizeof *e);
        e->chunk_index = kNoIndex;
        e->token_index = kNoIndex;
    }
}

int cuda_fail(plzgpu_error* e, cudaError_t c, const char* where) {
    return set_err(e, PLZGPU_CUDA, 0, kNoIndex, kNoIndex, "CUDA error in %s: %s", where,
                   cudaGetErrorString(c));
}

int bad_field(plzgpu_error* e, const char* field, const char* legal) {
    return set_err(e, PLZGPU_VALIDATION, 0, kNoIndex, kNoIndex, "invalid %s: legal range is %s",
                   field, legal);
}

int validate_fields(const plzgpu_params& p, plzgpu_error* e) {
    if (p.symbol_width != 1 && p.symbol_width != 2 && p.symbol_width != 4)
        return bad_field(e, "symbol_width", "{1,2,4}");
    if (p.window < 4 || p.window > 255)
        return bad_field(e, "window", "[4,255] (0 is reserved for no-match)");
    switch (p.chunk_size) {
        case 1024: case 2048: case 4096: case 8192: case 16384: break;
        default: return bad_field(e, "chunk_size", "{1024,2048,4096,8192,16384}");
    }
    if (p.chunk_size <= p.window) return bad_field(e, "chunk_size", "greater than window");
    switch (p.interval) {
        case 1: case 2: case 4: case 8: case 16: break;
        default: return bad_field(e, "interval", "{1,2,4,8,16}");
    }
    if (p.chunk_size % p.interval != 0) return bad_field(e, "interval", "a divisor of chunk_size");
    const uint64_t cb = uint64_t(p.chunk_size) * uint64_t(p.symbol_width);
    if (p.block_bytes == 0 || p.block_bytes % cb != 0)
        return bad_field(e, "block_bytes", "a positive multiple of chunk_size*symbol_width");
    return PLZGPU_OK;
}

Geometry geometry(uint64_t n, const plzgpu_params& p) {
    Geometry g;
    const uint64_t S = uint64_t(p.symbol_width), C = uint64_t(p.chunk_size);
    g.n_bytes = n;
    if (n == 0) return g;
    g.n_blocks = (n + p.block_bytes - 1) / p.block_bytes;
    g.cpb = p.block_bytes / (C * S);
    const uint64_t last_bytes = n - (g.n_blocks - 1) * p.block_bytes;
    const uint64_t last_syms = last_bytes / S;
    const uint64_t last_chunks = (last_syms + C - 1) / C;
    g.n_chunks = (g.n_blocks - 1) * g.cpb + last_chunks;
    g.last_len = last_chunks ? uint32_t(last_syms - (last_chunks - 1) * C) : uint32_t(C);
    return g;
}

int overflow_error(plzgpu_error* err) {
    return set_err(err, PLZGPU_VALIDATION, 0, kNoIndex, kNoIndex,
                   "block too large: offsets exceed 4-byte table range");
}

int corrupt(plzgpu_error* e, const std::string& what, uint64_t off) {
    return set_err(e, PLZGPU_CORRUPTION, off, kNoIndex, kNoIndex,
                   "corrupt container: %s (byte %llu)", what.c_str(), (unsigned long long)off);
}

// Map a ParseResult error onto the reference's exception (format.cpp:112-185).
int parse_error(const ParseResult& r, plzgpu_error* err) {
    const uint64_t off = r.err_offset;
    switch (r.err_kind) {
        case 1: return corrupt(err, "truncated header", off);
        case 2:
            return set_err(err, PLZGPU_UNSUPPORTED_FORMAT, 0, kNoIndex, kNoIndex,
                           "not a PLZ1 container (bad magic)");
        case 3:
            return set_err(err, PLZGPU_UNSUPPORTED_FORMAT, 0, kNoIndex, kNoIndex,
                           "unsupported container version %u", r.err_aux);
        case 4: return corrupt(err, "nonzero reserved byte", off);
        case 5: {
            plzgpu_params p{};
            p.symbol_width = r.hdr_S;
            p.window = r.hdr_W;
            p.interval = r.hdr_I;
            p.chunk_size = int32_t(r.hdr_C);
            p.block_bytes = uint64_t(256) << 20;
            plzgpu_error v;
            clear_err(&v);
            validate_fields(p, &v);
            return corrupt(err, v.message, off);
        }
        case 6: return corrupt(err, "tail_len >= symbol_width", off);
        case 7: return corrupt(err, "truncated offset tables", off);
        case 8: return corrupt(err, "payload offsets not monotone", off);
        case 9: return corrupt(err, "flag offsets not monotone", off);
        case 10: return corrupt(err, "payload offsets must start at 0", off);
        case 11: return corrupt(err, "flag offsets must start at 0", off);
        case 12: return corrupt(err, "truncated streams", off);
        case 13: return corrupt(err, "original_len too small", off);
        case 14: return corrupt(err, "original_len not aligned to symbols", off);
        case 15: return corrupt(err, "num_chunks inconsistent with original_len", off);
        case 16:
            return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                           "output buffer too small for the decoded image");
        default:
            return set_err(err, PLZGPU_CONTRACT, 0, kNoIndex, kNoIndex, "parse failure %u",
                           r.err_kind);
    }
}

namespace {
const char* token_what(uint32_t code) {
    switch (code) {
        case TE_FLAGS_EXHAUSTED: return "flag bits exhausted";
        case TE_PAYLOAD_EXHAUSTED: return "payload exhausted";
        case TE_ZERO_FIELD: return "zero pointer field";
        case TE_OFFSET_BEFORE_START: return "offset before chunk start";
        case TE_OVERRUN: return "pointer overruns chunk";
        case TE_TRAILING_PAYLOAD: return "trailing payload bytes";
        case TE_NONZERO_PADDING: return "nonzero flag padding";
        case TE_FLAG_COUNT: return "flag bytes inconsistent with token count";
        default: return "unknown";
    }
}

bool env_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && *v && *v != '0';
}

uint64_t env_u64(const char* name, uint64_t dflt, uint64_t unit, uint64_t min) {
    const char* v = std::getenv(name);
    if (!v || !*v) return dflt;
    const long long x = std::atoll(v);
    return std::max<uint64_t>(min, uint64_t(x < 0 ? 0 : x) * unit);
}

StreamValue32Fn entry_point(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
        (void)cudaGetLastError();
        p = nullptr;
    }
    return reinterpret_cast<StreamValue32Fn>(p);
}
}  // namespace

int token_error(uint32_t code, uint64_t chunk, uint64_t token, plzgpu_error* err) {
    return set_err(err, PLZGPU_CORRUPTION, 0, chunk, token, "corrupt chunk %llu, token %llu: %s",
                   (unsigned long long)chunk, (unsigned long long)token, token_what(code));
}

const PipelineConfig& pipeline_config() {
    static const PipelineConfig cfg = [] {
        PipelineConfig c;
        constexpr uint64_t MB = 1u << 20;
        c.no_pipe = env_flag("PLZGPU_NO_PIPE");
        c.no_pipe_asm = env_flag("PLZGPU_NO_PIPE_ASM");
        c.no_pipe_dec = env_flag("PLZGPU_NO_PIPE_DEC");
        c.asm_mapped = env_flag("PLZGPU_ASM_MAPPED");
        c.seg_bytes = env_u64("PLZGPU_SEG_MB", c.seg_bytes, MB, 1);
        c.copy_bytes = env_u64("PLZGPU_COPY_MB", c.copy_bytes, MB, 0);
        c.tail_bytes = env_u64("PLZGPU_TAIL_MB", c.tail_bytes, MB, 0);
        c.dseg_in = env_u64("PLZGPU_DSEG_IN_MB", c.dseg_in, MB, MB);
        c.dseg_out = env_u64("PLZGPU_DSEG_OUT_MB", c.dseg_out, MB, MB);
        c.dseg_lead = env_u64("PLZGPU_DSEG_LEAD", c.dseg_lead, 1, 1);
        c.dseg_group = env_u64("PLZGPU_DSEG_GROUP", c.dseg_group, 1, 1);
        c.dseg_group_out = env_u64("PLZGPU_DSEG_GROUP_OUT", c.dseg_group, 1, 1);
        c.pageable_stage = env_u64("PLZGPU_PAGEABLE_MB", c.pageable_stage, MB, MB);
        c.pageable_min = env_u64("PLZGPU_PAGEABLE_MIN_MB", c.pageable_min, MB, 0);
        c.copy_threads = int(env_u64("PLZGPU_COPY_THREADS", 0, 1, 0));
        c.asm_mode = int(env_u64("PLZGPU_ASM_MODE", 2, 1, 0));
        return c;
    }();
    return cfg;
}

StreamValue32Fn stream_write_value32() {
    static const StreamValue32Fn fn = entry_point("cuStreamWriteValue32");
    return fn;
}

StreamValue32Fn stream_wait_value32() {
    static const StreamValue32Fn fn = entry_point("cuStreamWaitValue32");
    return fn;
}

bool is_pinned_host(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

uint32_t next_epoch() {
    static std::atomic<uint32_t> counter{0};
    uint32_t e;
    do {
        e = counter.fetch_add(1, std::memory_order_relaxed) + 1;
    } while (e == 0);  // 0 is what a freshly cleared flag holds
    return e;
}

}  // namespace plzhost

namespace plzgpu {
int assemble_mode() { return plzhost::pipeline_config().asm_mode; }
}  // namespace plzgpu
