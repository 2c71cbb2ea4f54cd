// host.cpp — C-ABI implementation (include/plzgpu.h): parameter checks,
// partition geometry, device scratch, kernel orchestration and the mapping of
// device outcomes onto the reference's error types and messages.
//
// Reference behaviour mirrored here (paths under /root/reference/proj):
//   params.cpp:19-55     validation order and messages, min_match = 2/S + 1
//   partition.cpp:5-25   blocks of block_bytes, C-symbol chunks, raw tail
//   pipeline.cpp:88-99   image = containers back to back; empty input -> empty
//   scan.cpp:43-44       4-byte table overflow -> validation_error
//   format.cpp:112-185   read_container messages / byte offsets
//   decoder.cpp:13-18    "corrupt chunk K, token T: what"
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <thread>
#include <new>
#include <string>
#include <vector>

#include "../../include/plzgpu.h"
#include "kernels.h"

using namespace plzgpu;

namespace {

constexpr uint64_t kNoIndex = UINT64_MAX;

int set_err(plzgpu_error* e, int code, uint64_t off, uint64_t chunk, uint64_t tok,
            const char* fmt, ...) {
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

#define CK(call)                                                     \
    do {                                                             \
        const cudaError_t ck_ = (call);                              \
        if (ck_ != cudaSuccess) return cuda_fail(err, ck_, #call);   \
    } while (0)

// ------------------------------------------------------------ validation
int bad_field(plzgpu_error* e, const char* field, const char* legal) {
    return set_err(e, PLZGPU_VALIDATION, 0, kNoIndex, kNoIndex, "invalid %s: legal range is %s",
                   field, legal);
}

// params.cpp:19-45, same order, same messages
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

// Whole-input chunk geometry (partition.cpp:5-25 folded over all blocks).
struct Geometry {
    uint64_t n_bytes = 0, n_blocks = 0, cpb = 0, n_chunks = 0;
    uint32_t last_len = 0;
};

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

// cuStreamWriteValue32 through the runtime's driver entry point (no link-time
// libcuda dependency: the library must also load on GPU-less hosts).
typedef int (*StreamWriteValue32Fn)(void* stream, unsigned long long addr, uint32_t value,
                                    unsigned int flags);
StreamWriteValue32Fn stream_write_value32() {
    static StreamWriteValue32Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<StreamWriteValue32Fn>(p);
    }();
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

// --------------------------------------------------------------- scratch
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max(bytes, cap + cap / 2);
        want = (want + 255) & ~size_t(255);
        const cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// Small device words written by the kernels, read back in one copy.
struct Meta {
    uint64_t img_len;
    unsigned long long stats[2];
    uint32_t overflow;
    uint32_t detail_code;
    uint64_t detail_chunk;
    uint64_t detail_token;
    unsigned long long err_chunk;
    unsigned long long mono_key;  // first table-monotonicity violation, ~0 if none
    uint64_t mono_base;           // first chunk of its container
    uint32_t work[12];  // [0] first bitmap pass, [1] scan tiles, [2] assemble/decode,
                        // [4]/[6]/[8] overflow counts of the bitmap passes, [5]/[9]
                        // second/third bitmap pass, [7] wide pass
    uint32_t stalled;  // H2D pipeline: a segment never arrived
    uint32_t pad;
    uint64_t range[3];  // plzgpu_decompress_range: output range, total chunks
    ParseResult parse;
};

enum LastOp { OP_NONE, OP_COMPRESS, OP_DECOMPRESS };

}  // namespace

struct plzgpu_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    DevBuf in, img, out, pay_slots, flag_slots, psize, fsize, p64, f64, status, agg, incl, desc;
    DevBuf meta;
    Meta* host_meta = nullptr;  // pinned
    int last_launches = 0;
    LastOp last_op = OP_NONE;
    DecodeArgs last_decode{};
    int enc_wpc[2240] = {};  // launch shape cache per (pass, S, C)
    int enc_ctas[2240] = {};
    DevBuf fb;               // overflow lists of the bitmap passes (3 x G chunk indices)
    DevBuf shard_desc;        // ShardCont / HeaderDesc upload area
    // H2D pipeline of host inputs (plzgpu_compress): segment ready flags
    cudaStream_t copy_stream = nullptr;
    cudaStream_t asm_stream = nullptr;  // pipelined compress: per-container Kernel III
    cudaStream_t side_stream = nullptr;  // Kernel I: the 64-row pass beside the 32-row one
    cudaEvent_t side_ev[2] = {nullptr, nullptr};
    cudaEvent_t asm_ev[2] = {nullptr, nullptr};
    // pipelined compress into pinned host memory: per container, its scan
    // and its assembly done; the image goes down on d2h_stream, the
    // container sizes that place it come back on size_stream
    std::vector<cudaEvent_t> cont_ev;
    cudaStream_t d2h_stream = nullptr, size_stream = nullptr;
    uint64_t* host_scratch = nullptr;  // pinned, 4 words
    DevBuf ready, done;
    uint32_t epoch = 0;
    const uint32_t* pipe_ready = nullptr;  // set while enqueueing a pipelined encode
    uint32_t pipe_seg_chunks = 0;
    unsigned long long* enc_hist = nullptr;  // set while enqueueing a histogram encode
    DevBuf hist, table;
    DevBuf qtiles, qoff, qdelta;  // cuSZ quantizer scratch
    // last plzgpu_shard_encode: the range and its per-container local totals
    uint64_t sh_begin = 0, sh_end = 0, sh_n = 0;
    plzgpu_params sh_params{};
    std::vector<uint64_t> sh_touch;  // per touched container: {j, lo, hi, P, F}
};

namespace {

// NULL selects the legacy default stream (the CUDA convention, so callers
// passing torch's default stream handle 0 stay ordered with it).
cudaStream_t pick(plzgpu_ctx*, void* s) { return static_cast<cudaStream_t>(s); }

Meta* dmeta(plzgpu_ctx* c) { return c->meta.as<Meta>(); }

// A/B switch for measurements (PLZGPU_NO_PIPE_ASM=1: the whole-image path
// for host compresses); unset in normal use.
bool getenv_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && *v && *v != '0';
}

// Launch shape of Kernel I for (pass, S, C, W), cached per context: warps
// per CTA that maximise resident warps per SM (shared-memory limited).
// maxsyms: the bitmap pass's row budget (kBmMaxSyms / kBmMaxSymsWide), 0 for
// the wide-cell pass.  per_sm = 0: the pass does not fit.
void encode_shape(plzgpu_ctx* c, const plzgpu_params& p, int maxsyms, int* wpc_out,
                  int* per_sm_out) {
    const int pass = maxsyms == 0 ? 0 : (maxsyms == kBmMaxSyms ? 1 : maxsyms == kBmMaxSymsMid ? 5 : 9) +
                                             __builtin_ctz(unsigned(bm_nw(p.window)));  // 0..12
    const int key = pass * 160 + p.symbol_width * 32 + (__builtin_ctz(unsigned(p.chunk_size)) - 10);
    int& wpc = c->enc_wpc[key];
    int& per_sm = c->enc_ctas[key];
    if (wpc == 0) {
        int best_warps = 0;
        for (int cand = 1; cand <= (maxsyms ? kBmMaxThreads / 32 : 16); ++cand) {
            const int ctas = maxsyms ? bitmatch_ctas_per_sm(p.symbol_width, p.chunk_size, p.window,
                                                            maxsyms, cand)
                                     : encode_ctas_per_sm(p.symbol_width, p.chunk_size, cand);
            if (ctas * cand > best_warps) {
                best_warps = ctas * cand;
                wpc = cand;
                per_sm = ctas;
            }
        }
        if (best_warps == 0) {  // does not fit (huge chunks): one warp, one CTA
            wpc = 1;
            per_sm = 0;
        }
    }
    *wpc_out = wpc;
    *per_sm_out = per_sm;
}

// Enqueue Kernels I-III for a device-resident input.  img must hold
// compress_bound bytes; img_len receives the image length on the device.
// Kernels I and II over G chunks starting at d_in (chunk g at g*C*S); the
// last of them has logical length last_len.  Leaves psize/fsize, staging
// slots and exclusive prefixes P64/F64[0..G] in the context.
// g0/g1 (a pipelined compress, one container at a time): only chunks
// [g0, g1) of the G; their prefixes continue from P64/F64[g0].
int enqueue_encode_scan(plzgpu_ctx* c, const plzgpu_params& p, const uint8_t* d_in, uint64_t G,
                        uint32_t last_len, cudaStream_t st, plzgpu_error* err, int* launches,
                        bool scan = true, uint64_t g0 = 0, uint64_t g1 = UINT64_MAX,
                        bool side_passes = true) {
    const uint64_t S = uint64_t(p.symbol_width), C = uint64_t(p.chunk_size);
    if (g1 > G) g1 = G;
    const uint64_t Gr = g1 - g0;  // chunks of this call
    const uint64_t tiles = (G + kScanTile - 1) / kScanTile;
    CK(c->pay_slots.ensure(G * C * S + 64));
    CK(c->flag_slots.ensure(G * (C / 8) + 64));
    CK(c->psize.ensure(G * 4 + 64));
    CK(c->fsize.ensure(G * 4 + 64));
    CK(c->p64.ensure((G + 1) * 8));
    CK(c->f64.ensure((G + 1) * 8));
    CK(c->status.ensure(tiles * 4 + 4));
    CK(c->agg.ensure(tiles * 16 + 16));
    CK(c->incl.ensure(tiles * 16 + 16));
    Meta* m = dmeta(c);
    if (g0 == 0) {  // once per call: a later container must not clear an earlier stall
        CK(cudaMemsetAsync(&m->stats, 0, sizeof m->stats + sizeof m->overflow, st));
        CK(cudaMemsetAsync(&m->stalled, 0, sizeof m->stalled, st));
    }
    CK(cudaMemsetAsync(m->work, 0, sizeof m->work, st));
    if (G == 0) {
        CK(cudaMemsetAsync(c->p64.p, 0, 8, st));
        CK(cudaMemsetAsync(c->f64.p, 0, 8, st));
        return PLZGPU_OK;
    }
    const uint64_t rtiles = (Gr + kScanTile - 1) / kScanTile;
    CK(cudaMemsetAsync(c->status.p, 0, rtiles * 4, st));
    // ---- Kernel I
    const uint8_t* in0 = d_in + g0 * C * S;
    EncodeArgs e{};
    e.in = in0;
    e.pay_slots = c->pay_slots.as<uint8_t>() + g0 * C * S;
    e.flag_slots = c->flag_slots.as<uint8_t>() + g0 * (C / 8);
    e.psize = c->psize.as<uint32_t>() + g0;
    e.fsize = c->fsize.as<uint32_t>() + g0;
    e.stats = m->stats;
    e.work = &m->work[0];
    e.n_chunks = Gr;
    e.last_len = g1 == G ? last_len : uint32_t(C);
    e.C = p.chunk_size;
    e.W = p.window;
    e.I = p.interval;
    e.min_match = std::max(1, p.min_match);
    e.bulk_ok = (reinterpret_cast<uintptr_t>(in0) & 15u) == 0;
    e.ready = c->pipe_ready ? c->pipe_ready + g0 / c->pipe_seg_chunks : nullptr;
    e.epoch = c->epoch;
    e.seg_chunks = c->pipe_seg_chunks;
    e.stalled = &m->stalled;
    e.hist = c->enc_hist;
    // bitmap pass (16 rows) over every chunk, then the 32-row and 64-row
    // passes over what overflowed, then the wide-cell pass.  With few chunks
    // per resident warp the later passes' tails would add up, so the first
    // pass then sorts its overflow by exact alphabet size and the 32- and
    // 64-row passes run concurrently (two streams); otherwise they run one
    // after the other, each taking the previous one's overflow.
    CK(c->fb.ensure(3 * G * 4 + 16));
    uint32_t* lists[3] = {c->fb.as<uint32_t>(), c->fb.as<uint32_t>() + G,
                          c->fb.as<uint32_t>() + 2 * G};
    uint32_t* counts[3] = {&m->work[4], &m->work[6], &m->work[8]};
    uint32_t* works[4] = {&m->work[0], &m->work[5], &m->work[9], &m->work[7]};
    int wpc1 = 1, per_sm1 = 0;
    encode_shape(c, p, kBmMaxSyms, &wpc1, &per_sm1);
    const bool classify = side_passes && Gr < uint64_t(4) * c->sms * per_sm1 * wpc1;
    e.classify = classify ? 1 : 0;
    cudaError_t launch_err = cudaSuccess;  // first failed bitmap-pass launch
    auto bitmap_pass = [&](int maxsyms, int pass, const uint32_t* src, const uint32_t* src_n,
                           uint32_t* ovf, uint32_t* ovf_n, cudaStream_t s) -> bool {
        int wpc = 1, per_sm = 0;
        encode_shape(c, p, maxsyms, &wpc, &per_sm);
        if (per_sm == 0) return false;
        EncodeArgs b = e;
        b.work = works[pass];
        b.src_list = src;
        b.src_count = src_n;
        if (src) {
            b.ready = nullptr;  // every segment has landed after the first pass
            b.classify = 0;
            for (int i = 0; i < 2; ++i) {
                b.fb_list[i] = ovf;
                b.fb_count[i] = ovf_n;
            }
        }
        b.warps_per_cta = wpc;
        // a pipelined compress leaves one CTA slot per SM for the previous
        // container's Kernel III on the assembly stream
        const int resident = side_passes ? per_sm : std::max(1, per_sm - 1);
        const uint64_t ctas = std::min<uint64_t>(uint64_t(c->sms) * resident, (Gr + wpc - 1) / wpc);
        const cudaError_t le = launch_bitmatch(p.symbol_width, maxsyms, b, int(ctas), s);
        if (le != cudaSuccess && launch_err == cudaSuccess) launch_err = le;
        ++*launches;
        return true;
    };
    for (int i = 0; i < 3; ++i) {
        e.fb_list[i] = lists[i];
        e.fb_count[i] = counts[i];
    }
    const uint32_t* wide_src = nullptr;
    const uint32_t* wide_n = nullptr;
    if (bitmap_pass(kBmMaxSyms, 0, nullptr, nullptr, nullptr, nullptr, st)) {
        bool mid, wide;
        if (classify) {
            if (!c->side_stream) CK(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
            for (cudaEvent_t& ev : c->side_ev)
                if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(c->side_ev[0], st));
            CK(cudaStreamWaitEvent(c->side_stream, c->side_ev[0], 0));
            mid = bitmap_pass(kBmMaxSymsMid, 1, lists[0], counts[0], lists[2], counts[2], st);
            wide = bitmap_pass(kBmMaxSymsWide, 2, lists[1], counts[1], lists[2], counts[2],
                               c->side_stream);
            CK(cudaEventRecord(c->side_ev[1], c->side_stream));
            CK(cudaStreamWaitEvent(st, c->side_ev[1], 0));
        } else {
            mid = bitmap_pass(kBmMaxSymsMid, 1, lists[0], counts[0], lists[1], counts[1], st);
            wide = bitmap_pass(kBmMaxSymsWide, 2, lists[1], counts[1], lists[2], counts[2], st);
        }
        if (!mid || !wide)
            return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                           "chunk too large for the bitmap passes' shared memory");
        wide_src = lists[2];
        wide_n = counts[2];
    }
    {
        int wpc = 1, per_sm = 1;
        encode_shape(c, p, 0, &wpc, &per_sm);
        EncodeArgs f = e;
        f.work = works[3];
        f.src_list = wide_src;
        f.src_count = wide_n;
        if (wide_src) f.ready = nullptr;
        f.warps_per_cta = wpc;
        CK(launch_encode(p.symbol_width, f,
                         int(std::min<uint64_t>(uint64_t(c->sms) * std::max(per_sm, 1),
                                                (Gr + wpc - 1) / wpc)),
                         st));
        ++*launches;
    }
    CK(launch_err);
    if (!scan) return PLZGPU_OK;
    // ---- Kernel II
    ScanArgs sa{};
    sa.psize = e.psize;
    sa.fsize = e.fsize;
    sa.n = Gr;
    sa.P64 = c->p64.as<uint64_t>() + g0;
    sa.F64 = c->f64.as<uint64_t>() + g0;
    if (g0) {  // continue the earlier containers' totals
        sa.carry_p = c->p64.as<uint64_t>() + g0;
        sa.carry_f = c->f64.as<uint64_t>() + g0;
    }
    sa.status = c->status.as<uint32_t>();
    sa.agg = c->agg.as<ulonglong2>();
    sa.incl = c->incl.as<ulonglong2>();
    sa.tile_counter = &m->work[1];
    launch_scan(sa, st);
    ++*launches;
    return PLZGPU_OK;
}

// Enqueue Kernels I-III for a device-resident input.  img must hold
// compress_bound bytes; img_len receives the image length on the device.
int enqueue_compress(plzgpu_ctx* c, const plzgpu_params& p, const uint8_t* d_in, uint64_t n,
                     uint8_t* img, uint64_t* d_img_len, cudaStream_t st, plzgpu_error* err,
                     int last_stage = 3) {
    const Geometry g = geometry(n, p);
    const uint64_t G = g.n_chunks;
    int launches = 0;
    int rc = enqueue_encode_scan(c, p, d_in, G, g.last_len, st, err, &launches, last_stage > 1);
    if (rc) return rc;
    if (last_stage == 1) {
        CK(cudaGetLastError());
        c->last_launches = launches;
        c->last_op = OP_NONE;
        return PLZGPU_OK;
    }
    Meta* m = dmeta(c);
    // ---- Kernel III + headers
    AssembleArgs a{};
    a.in = d_in;
    a.pay_slots = c->pay_slots.as<uint8_t>();
    a.flag_slots = c->flag_slots.as<uint8_t>();
    a.psize = c->psize.as<uint32_t>();
    a.fsize = c->fsize.as<uint32_t>();
    a.P64 = c->p64.as<uint64_t>();
    a.F64 = c->f64.as<uint64_t>();
    a.img = img;
    a.img_len = d_img_len;
    a.overflow = &m->overflow;
    a.n_bytes = n;
    a.n_chunks = G;
    a.cpb = g.cpb;
    a.block_bytes = p.block_bytes;
    a.n_blocks = g.n_blocks;
    a.S = p.symbol_width;
    a.W = p.window;
    a.I = p.interval;
    a.C = p.chunk_size;
    if (G > 0) {
        launch_assemble(a, st);
        ++launches;
    }
    launch_headers(a, st);
    ++launches;
    CK(cudaGetLastError());
    c->last_launches = launches;
    c->last_op = OP_COMPRESS;
    return PLZGPU_OK;
}

// A pipelined compress of a host input (plzgpu_compress): one container at a
// time on `st` — its Kernel I passes (waiting on the container's H2D
// segments) and its scan, continuing the earlier containers' prefixes — and
// its Kernel III + header on c->asm_stream, writing into `img` (the caller's
// pinned host image, mapped) while `st` goes on with the next container.
int enqueue_compress_by_container(plzgpu_ctx* c, const plzgpu_params& p, const uint8_t* d_in,
                                  uint64_t n, uint8_t* img, cudaStream_t st, plzgpu_error* err) {
    const Geometry g = geometry(n, p);
    if (!c->asm_stream) CK(cudaStreamCreateWithFlags(&c->asm_stream, cudaStreamNonBlocking));
    for (cudaEvent_t& ev : c->asm_ev)
        if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    Meta* m = dmeta(c);
    while (c->cont_ev.size() < 2 * g.n_blocks) {
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        c->cont_ev.push_back(ev);
    }
    int launches = 0;
    for (uint64_t j = 0; j < g.n_blocks; ++j) {
        const uint64_t g0 = j * g.cpb, g1 = std::min(g.n_chunks, g0 + g.cpb);
        // (no side-stream passes here: Kernel III of the previous container
        // is running on the assembly stream)
        int rc = enqueue_encode_scan(c, p, d_in, g.n_chunks, g.last_len, st, err, &launches, true,
                                     g0, g1, false);
        if (rc) return rc;
        CK(cudaEventRecord(c->cont_ev[2 * j], st));
        CK(cudaEventRecord(c->asm_ev[0], st));
        CK(cudaStreamWaitEvent(c->asm_stream, c->asm_ev[0], 0));
        AssembleArgs a{};
        a.in = d_in;
        a.pay_slots = c->pay_slots.as<uint8_t>();
        a.flag_slots = c->flag_slots.as<uint8_t>();
        a.psize = c->psize.as<uint32_t>();
        a.fsize = c->fsize.as<uint32_t>();
        a.P64 = c->p64.as<uint64_t>();
        a.F64 = c->f64.as<uint64_t>();
        a.img = img;
        a.img_len = &m->img_len;
        a.overflow = &m->overflow;
        a.n_bytes = n;
        a.n_chunks = g.n_chunks;
        a.cpb = g.cpb;
        a.block_bytes = p.block_bytes;
        a.n_blocks = g.n_blocks;
        a.S = p.symbol_width;
        a.W = p.window;
        a.I = p.interval;
        a.C = p.chunk_size;
        a.j_lo = j;
        a.j_hi = j + 1;
        launch_assemble(a, c->asm_stream);
        launch_headers(a, c->asm_stream);
        CK(cudaEventRecord(c->cont_ev[2 * j + 1], c->asm_stream));
        launches += 2;
    }
    CK(cudaEventRecord(c->asm_ev[1], c->asm_stream));
    CK(cudaStreamWaitEvent(st, c->asm_ev[1], 0));
    CK(cudaGetLastError());
    c->last_launches = launches;
    c->last_op = OP_COMPRESS;
    return PLZGPU_OK;
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

int token_error(uint32_t code, uint64_t chunk, uint64_t token, plzgpu_error* err) {
    return set_err(err, PLZGPU_CORRUPTION, 0, chunk, token, "corrupt chunk %llu, token %llu: %s",
                   (unsigned long long)chunk, (unsigned long long)token, token_what(code));
}

int enqueue_decompress(plzgpu_ctx* c, const uint8_t* d_img, uint64_t len, uint8_t* d_out,
                       uint64_t cap, uint64_t* d_out_len, cudaStream_t st, plzgpu_error* err) {
    Meta* m = dmeta(c);
    if (c->desc.cap < 64 * sizeof(ContainerDesc)) CK(c->desc.ensure(64 * sizeof(ContainerDesc)));
    CK(cudaMemsetAsync(&m->parse, 0, sizeof m->parse, st));
    CK(cudaMemsetAsync(&m->err_chunk, 0xff, sizeof m->err_chunk + sizeof m->mono_key, st));
    CK(cudaMemsetAsync(m->work, 0, sizeof m->work, st));
    DecodeArgs a{};
    a.img = d_img;
    a.img_len = len;
    a.out = d_out;
    a.out_cap = cap;
    a.desc = c->desc.as<ContainerDesc>();
    a.desc_cap = c->desc.cap / sizeof(ContainerDesc);
    a.result = &m->parse;
    a.out_len = d_out_len;
    a.err_chunk = &m->err_chunk;
    a.mono_key = &m->mono_key;
    a.work = &m->work[2];
    launch_parse(a, st);
    int per_sm = decode_ctas_per_sm();
    if (per_sm < 1) per_sm = 1;
    launch_decode(a, c->sms * per_sm, st);
    CK(cudaGetLastError());
    c->last_launches = 2;
    c->last_op = OP_DECOMPRESS;
    c->last_decode = a;
    return PLZGPU_OK;
}

// After a decompress has completed: report its error, if any, in the
// reference's order (chunk errors of earlier containers before the parse
// error of a later one).  Sets *grow when the descriptor table overflowed.
int finish_decompress(plzgpu_ctx* c, cudaStream_t st, bool* grow, plzgpu_error* err) {
    Meta h;
    CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *grow = false;
    if (h.mono_key != ~0ull) {
        // a table-monotonicity violation in container j: chunk errors of
        // earlier containers come first (decoder order), then this one
        Meta* m = dmeta(c);
        launch_mono_detail(c->last_decode, h.mono_key, &m->mono_base, st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h.err_chunk == ~0ull || h.err_chunk >= h.mono_base) return parse_error(h.parse, err);
    }
    if (h.err_chunk != ~0ull) {
        Meta* m = dmeta(c);
        launch_chunk_detail(c->last_decode, &m->detail_code, &m->detail_chunk, &m->detail_token, st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return token_error(h.detail_code, h.detail_chunk, h.detail_token, err);
    }
    if (h.parse.err_kind == 17) {
        *grow = true;
        return PLZGPU_OK;
    }
    if (h.parse.err_kind != 0) return parse_error(h.parse, err);
    return PLZGPU_OK;
}

// Every kernel loaded once per device (see preload_kernel in kernels.h).
void preload_kernels(int device) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(done.begin(), done.end(), device) != done.end()) return;
    preload_bitmatch_kernels();
    preload_encode_kernels();
    preload_scan_kernels();
    preload_assemble_kernels();
    preload_decode_kernels();
    preload_cusz_kernels();
    done.push_back(device);
}

// cuStreamWaitValue32 (CU_STREAM_WAIT_VALUE_GEQ = 0) through the entry point.
typedef int (*StreamWaitValue32Fn)(void* stream, unsigned long long addr, uint32_t value,
                                   unsigned int flags);
StreamWaitValue32Fn stream_wait_value32() {
    static StreamWaitValue32Fn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<StreamWaitValue32Fn>(p);
    }();
    return fn;
}

uint32_t host_le32(const uint8_t* b) {
    return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
}

// Host image -> pinned host output, all three legs overlapped: the image
// goes up in segments (copy_stream, ready flags as in plzgpu_compress), the
// decode kernel waits per chunk for the segment its streams end in, and
// each decoded output segment goes down (asm_stream) as soon as the kernel
// has counted all of its bytes.  The container walk runs on the host over
// the caller's image; anything it does not accept as well-formed — and any
// error the kernel sees — falls back to the resident path, which reports
// the reference's exact error.  Returns 1 when it produced the output.
int try_decompress_pipelined(plzgpu_ctx* c, const uint8_t* img, uint64_t len, uint8_t* out,
                             uint64_t cap, uint64_t* out_len, cudaStream_t st,
                             plzgpu_error* err) {
    // Ready flags every seg_in bytes of image, output counters every seg_out
    // bytes; the first kLead transfers each way move one segment, later ones
    // kGroup segments at a time.  Env overrides for A/B (2/4 MiB segments
    // with 4 single and then 8-segment transfers measured no faster).
    auto env_int = [](const char* name, int dflt) {
        const char* v = std::getenv(name);
        return v ? std::max(1, std::atoi(v)) : dflt;
    };
    const uint64_t seg_in = uint64_t(env_int("PLZGPU_DSEG_IN_MB", 16)) << 20;
    const uint64_t seg_out = uint64_t(env_int("PLZGPU_DSEG_OUT_MB", 32)) << 20;
    const uint64_t kLead = uint64_t(env_int("PLZGPU_DSEG_LEAD", 1));
    const uint64_t kGroup = uint64_t(env_int("PLZGPU_DSEG_GROUP", 1));
    const uint64_t kGroupOut = uint64_t(env_int("PLZGPU_DSEG_GROUP_OUT", int(kGroup)));
    StreamWriteValue32Fn write_value = stream_write_value32();
    StreamWaitValue32Fn wait_value = stream_wait_value32();
    if (!write_value || !wait_value || getenv_flag("PLZGPU_NO_PIPE_DEC") || getenv_flag("PLZGPU_NO_PIPE"))
        return 0;
    // the container walk (format.cpp:112-185 on a well-formed image)
    std::vector<ContainerDesc> descs;
    uint64_t at = 0, total_out = 0, total_chunks = 0;
    while (at < len) {
        const uint8_t* b = img + at;
        const uint64_t size = len - at;
        if (size < 26 || b[0] != 'P' || b[1] != 'L' || b[2] != 'Z' || b[3] != '1' || b[4] != 1 ||
            b[8] != 0)
            return 0;
        const uint32_t S = b[5], W = b[6], I = b[7], C = host_le32(b + 9);
        if ((S != 1 && S != 2 && S != 4) || W < 4 || W > 255 || C <= W ||
            (C != 1024 && C != 2048 && C != 4096 && C != 8192 && C != 16384) ||
            (I != 1 && I != 2 && I != 4 && I != 8 && I != 16) || b[25] >= S)
            return 0;
        const uint64_t n = host_le32(b + 21), tail = b[25];
        if (size < 26 + 8 * (n + 1)) return 0;
        const uint8_t* ptab = b + 26;
        const uint8_t* ftab = ptab + 4 * (n + 1);
        const uint64_t ptot = host_le32(ptab + 4 * n), ftot = host_le32(ftab + 4 * n);
        const uint64_t orig = uint64_t(host_le32(b + 13)) | uint64_t(host_le32(b + 17)) << 32;
        const uint64_t need = 26 + 8 * (n + 1) + ftot + ptot + tail;
        if (host_le32(ptab) != 0 || host_le32(ftab) != 0 || size < need || orig < tail ||
            (orig - tail) % S != 0 || ((orig - tail) / S + C - 1) / C != n ||
            total_out + orig > cap)
            return 0;
        ContainerDesc d{};
        d.img_off = at;
        d.out_off = total_out;
        d.chunk_base = total_chunks;
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
        descs.push_back(d);
        at += need;
        total_out += orig;
        total_chunks += n;
    }
    if (descs.empty() || total_chunks == 0) return 0;
    const uint64_t nseg_in = (len + seg_in - 1) / seg_in;
    const uint64_t nseg_out = (total_out + seg_out - 1) / seg_out;
    if (nseg_in < 2 && nseg_out < 2) return 0;  // nothing to overlap
    // decoded bytes each output segment receives from chunks (tails excluded)
    std::vector<uint32_t> expect(nseg_out, 0);
    for (const ContainerDesc& d : descs) {
        const uint64_t o0 = d.out_off, o1 = d.out_off + d.original_len - d.tail_len;
        for (uint64_t sg = o0 / seg_out; sg * seg_out < o1; ++sg)
            expect[sg] += uint32_t(std::min(o1, (sg + 1) * seg_out) - std::max(o0, sg * seg_out));
    }
    if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    if (!c->asm_stream) CK(cudaStreamCreateWithFlags(&c->asm_stream, cudaStreamNonBlocking));
    if (!c->asm_ev[0]) {
        CK(cudaEventCreateWithFlags(&c->asm_ev[0], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->asm_ev[1], cudaEventDisableTiming));
    }
    CK(c->img.ensure(len + 16));
    CK(c->out.ensure(total_out + 16));
    CK(c->ready.ensure(nseg_in * 4));
    CK(c->done.ensure(nseg_out * 4));
    CK(c->desc.ensure(std::max<uint64_t>(descs.size(), 64) * sizeof(ContainerDesc)));
    Meta* m = dmeta(c);
    ++c->epoch;
    if (c->epoch == 0) {  // never reuse the initial 0 flags
        CK(cudaMemsetAsync(c->ready.p, 0, nseg_in * 4, st));
        ++c->epoch;
    }
    ParseResult pr{};
    pr.n_containers = descs.size();
    pr.total_chunks = total_chunks;
    pr.total_out = total_out;
    CK(cudaMemcpyAsync(c->desc.p, descs.data(), descs.size() * sizeof(ContainerDesc),
                       cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(&m->parse, &pr, sizeof pr, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(&m->err_chunk, 0xff, sizeof m->err_chunk + sizeof m->mono_key, st));
    CK(cudaMemsetAsync(m->work, 0, sizeof m->work + sizeof m->stalled, st));
    CK(cudaMemsetAsync(c->done.p, 0, nseg_out * 4, st));
    CK(cudaEventRecord(c->asm_ev[0], st));
    DecodeArgs a{};
    a.img = c->img.as<uint8_t>();
    a.img_len = len;
    a.out = c->out.as<uint8_t>();
    a.out_cap = cap;
    a.desc = c->desc.as<ContainerDesc>();
    a.desc_cap = c->desc.cap / sizeof(ContainerDesc);
    a.result = &m->parse;
    a.err_chunk = &m->err_chunk;
    a.mono_key = &m->mono_key;
    a.work = &m->work[2];
    DecodePipe pp{};
    pp.in_ready = c->ready.as<uint32_t>();
    pp.epoch = c->epoch;
    pp.stalled = &m->stalled;
    pp.in_seg = seg_in;
    pp.out_done = c->done.as<uint32_t>();
    pp.out_seg = seg_out;
    // the image up, segment by segment, after the flags' reset above
    CK(cudaStreamWaitEvent(c->copy_stream, c->asm_ev[0], 0));
    for (uint64_t sg = 0; sg < nseg_in;) {
        const uint64_t s_end = std::min(nseg_in, sg + (sg < kLead ? 1 : kGroup));
        const uint64_t lo = sg * seg_in, hi = std::min(len, s_end * seg_in);
        CK(cudaMemcpyAsync(c->img.as<uint8_t>() + lo, img + lo, hi - lo, cudaMemcpyHostToDevice,
                           c->copy_stream));
        for (; sg < s_end; ++sg)
            if (write_value(c->copy_stream, reinterpret_cast<unsigned long long>(pp.in_ready + sg),
                            c->epoch, 0) != 0)
                return 0;
    }
    int per_sm = decode_ctas_per_sm();
    if (per_sm < 1) per_sm = 1;
    launch_decode_pipelined(a, pp, c->sms * per_sm, st);
    CK(cudaGetLastError());
    // the output down, each segment once its decoded bytes are counted
    CK(cudaStreamWaitEvent(c->asm_stream, c->asm_ev[0], 0));
    for (uint64_t sg = 0; sg < nseg_out;) {
        const uint64_t s_end = std::min(nseg_out, sg + (sg < kLead ? 1 : kGroupOut));
        const uint64_t lo = sg * seg_out, hi = std::min(total_out, s_end * seg_out);
        for (; sg < s_end; ++sg)
            if (wait_value(c->asm_stream, reinterpret_cast<unsigned long long>(pp.out_done + sg),
                           expect[sg], 0) != 0)
                return 0;
        CK(cudaMemcpyAsync(out + lo, a.out + lo, hi - lo, cudaMemcpyDeviceToHost, c->asm_stream));
    }
    CK(cudaEventRecord(c->asm_ev[1], c->asm_stream));
    CK(cudaStreamWaitEvent(st, c->asm_ev[1], 0));
    Meta* h = c->host_meta;
    CK(cudaMemcpyAsync(h, m, sizeof(Meta), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaStreamSynchronize(c->copy_stream));
    c->last_launches = 1;
    c->last_op = OP_DECOMPRESS;
    c->last_decode = a;
    if (h->stalled || h->err_chunk != ~0ull || h->mono_key != ~0ull) return 0;
    // raw tails straight from the image (decoder.cpp:123-125)
    for (const ContainerDesc& d : descs)
        if (d.tail_len)
            std::memcpy(out + d.out_off + d.original_len - d.tail_len,
                        img + d.payload_off + d.payload_len, d.tail_len);
    *out_len = total_out;
    return 1;
}

}  // namespace

// =================================================================== C-ABI
extern "C" {

int plzgpu_abi_version(void) { return PLZGPU_ABI_VERSION; }

int plzgpu_validate(const plzgpu_params* raw, plzgpu_params* out, plzgpu_error* err) {
    clear_err(err);
    const int rc = validate_fields(*raw, err);
    if (rc) return rc;
    if (out) {
        *out = *raw;
        out->min_match = 2 / raw->symbol_width + 1;  // params.cpp:43
    }
    return PLZGPU_OK;
}

int plzgpu_level_to_window(int level, int32_t* window, plzgpu_error* err) {
    clear_err(err);
    static const int32_t w[] = {32, 64, 128, 255};  // params.cpp:47-55
    if (level < 1 || level > 4) return bad_field(err, "level", "[1,4]");
    *window = w[level - 1];
    return PLZGPU_OK;
}

uint64_t plzgpu_plan(uint64_t total, const plzgpu_params* p, plzgpu_block_plan* blocks,
                     uint64_t max_blocks) {
    const uint64_t S = uint64_t(p->symbol_width), C = uint64_t(p->chunk_size);
    uint64_t pos = 0, count = 0;
    while (pos < total) {
        plzgpu_block_plan b{};
        b.byte_start = pos;
        b.byte_len = std::min<uint64_t>(p->block_bytes, total - pos);
        const uint64_t syms = b.byte_len / S;
        b.tail_len = uint8_t(b.byte_len % S);
        if (syms > 0) {
            b.num_chunks = uint32_t((syms + C - 1) / C);
            b.last_chunk_len = uint32_t(syms - uint64_t(b.num_chunks - 1) * C);
        }
        if (count < max_blocks && blocks) blocks[count] = b;
        ++count;
        pos += b.byte_len;
        if (p->block_bytes == 0) break;
    }
    return count;
}

uint64_t plzgpu_container_size(uint32_t num_chunks, uint64_t flag_total, uint64_t payload_total,
                               uint8_t tail_len) {
    return 26 + 8 * (uint64_t(num_chunks) + 1) + flag_total + payload_total + tail_len;
}

uint64_t plzgpu_compress_bound(uint64_t n, const plzgpu_params* p) {
    if (n == 0 || p->block_bytes == 0) return 0;
    const uint64_t S = uint64_t(p->symbol_width);
    const uint64_t nb = (n + p->block_bytes - 1) / p->block_bytes;
    const Geometry g = geometry(n, *p);
    // all-literal payload (< n) + ceil(len/8) flags per chunk + headers/tables + tails
    return n + (n / S) / 8 + g.n_chunks + nb * 26 + 8 * (g.n_chunks + nb) + 16;
}

uint64_t plzgpu_decompressed_bound(const void* host_img, uint64_t len) {
    // format.cpp:112-185 checks on the host bytes; stops at the first
    // container that read_container would reject
    const uint8_t* b = static_cast<const uint8_t*>(host_img);
    uint64_t at = 0, total = 0;
    auto u32 = [](const uint8_t* q) {
        return uint64_t(q[0]) | (uint64_t(q[1]) << 8) | (uint64_t(q[2]) << 16) |
               (uint64_t(q[3]) << 24);
    };
    while (at < len) {
        const uint64_t size = len - at;
        const uint8_t* h = b + at;
        if (size < 26 || std::memcmp(h, "PLZ1", 4) != 0 || h[4] != 1 || h[8] != 0) break;
        plzgpu_params p{};
        p.symbol_width = h[5];
        p.window = h[6];
        p.interval = h[7];
        p.chunk_size = int32_t(u32(h + 9));
        p.block_bytes = uint64_t(256) << 20;
        if (validate_fields(p, nullptr) != PLZGPU_OK || h[25] >= h[5]) break;
        const uint64_t n = u32(h + 21);
        if (size < 26 + 8 * (n + 1)) break;
        const uint8_t* pt = h + 26;
        const uint8_t* ft = pt + 4 * (n + 1);
        bool mono = u32(pt) == 0 && u32(ft) == 0;
        for (uint64_t i = 0; mono && i < n; ++i)
            mono = u32(pt + 4 * (i + 1)) >= u32(pt + 4 * i) && u32(ft + 4 * (i + 1)) >= u32(ft + 4 * i);
        if (!mono) break;
        const uint64_t ptot = u32(pt + 4 * n), ftot = u32(ft + 4 * n);
        const uint64_t need = 26 + 8 * (n + 1) + ftot + ptot + h[25];
        if (size < need) break;
        uint64_t orig = 0;
        for (int i = 0; i < 8; ++i) orig |= uint64_t(h[13 + i]) << (8 * i);
        const uint64_t S = h[5], C = uint64_t(p.chunk_size);
        if (orig < h[25] || (orig - h[25]) % S != 0 || ((orig - h[25]) / S + C - 1) / C != n) break;
        total += orig;
        at += need;
    }
    return total;
}

int plzgpu_decompressed_size(plzgpu_ctx* c, const void* img, uint64_t len, uint64_t* out_len,
                             void* stream, plzgpu_error* err) {
    clear_err(err);
    *out_len = 0;
    if (len == 0) return PLZGPU_OK;
    if (!is_device_ptr(img)) {
        *out_len = plzgpu_decompressed_bound(img, len);
        return PLZGPU_OK;
    }
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    for (;;) {
        if (c->desc.cap < 64 * sizeof(ContainerDesc)) CK(c->desc.ensure(64 * sizeof(ContainerDesc)));
        Meta* m = dmeta(c);
        CK(cudaMemsetAsync(&m->parse, 0, sizeof m->parse, st));
        DecodeArgs a{};
        a.img = static_cast<const uint8_t*>(img);
        a.img_len = len;
        a.out = nullptr;  // size-only walk: no tails copied
        a.out_cap = UINT64_MAX;
        a.desc = c->desc.as<ContainerDesc>();
        a.desc_cap = c->desc.cap / sizeof(ContainerDesc);
        a.result = &m->parse;
        launch_parse(a, st);
        CK(cudaGetLastError());
        Meta h;
        CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h.parse.err_kind == 17) {
            CK(c->desc.ensure(c->desc.cap * 4));
            continue;
        }
        *out_len = h.parse.total_out;
        return PLZGPU_OK;
    }
}

int plzgpu_ctx_create(int device, plzgpu_ctx** out, plzgpu_error* err) {
    clear_err(err);
    *out = nullptr;
    plzgpu_ctx* c = new (std::nothrow) plzgpu_ctx();
    if (!c) return set_err(err, PLZGPU_CUDA, 0, kNoIndex, kNoIndex, "out of host memory");
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = c->meta.ensure(sizeof(Meta));
    if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&c->host_meta), sizeof(Meta));
    if (e == cudaSuccess) preload_kernels(device);
    if (e != cudaSuccess) {
        plzgpu_ctx_destroy(c);
        return cuda_fail(err, e, "plzgpu_ctx_create");
    }
    *out = c;
    return PLZGPU_OK;
}

void plzgpu_ctx_destroy(plzgpu_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (DevBuf* b : {&c->in, &c->img, &c->out, &c->pay_slots, &c->flag_slots, &c->psize,
                      &c->fsize, &c->p64, &c->f64, &c->status, &c->agg, &c->incl, &c->desc,
                      &c->meta})
        b->release();
    if (c->host_meta) cudaFreeHost(c->host_meta);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->asm_stream) {
        cudaStreamSynchronize(c->asm_stream);
        cudaStreamDestroy(c->asm_stream);
    }
    if (c->side_stream) {
        cudaStreamSynchronize(c->side_stream);
        cudaStreamDestroy(c->side_stream);
    }
    for (cudaEvent_t& ev : c->side_ev)
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t& ev : c->asm_ev)
        if (ev) cudaEventDestroy(ev);
    for (cudaStream_t sx : {c->d2h_stream, c->size_stream})
        if (sx) {
            cudaStreamSynchronize(sx);
            cudaStreamDestroy(sx);
        }
    for (cudaEvent_t ev : c->cont_ev)
        if (ev) cudaEventDestroy(ev);
    if (c->host_scratch) cudaFreeHost(c->host_scratch);
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamDestroy(c->copy_stream);
    }
    c->ready.release();
    c->done.release();
    c->shard_desc.release();
    delete c;
}

void* plzgpu_ctx_stream(plzgpu_ctx* c) { return c->stream; }

int plzgpu_ctx_last_launches(plzgpu_ctx* c) { return c->last_launches; }

int plzgpu_compress(plzgpu_ctx* c, const plzgpu_params* params, const void* in, uint64_t n,
                    void* out, uint64_t cap, uint64_t* out_len, plzgpu_stats* stats, void* stream,
                    plzgpu_error* err) {
    clear_err(err);
    *out_len = 0;
    if (stats) std::memset(stats, 0, sizeof *stats);
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    if (n == 0) return PLZGPU_OK;  // empty input -> empty image (test_decoder.cpp:76-80)
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const uint8_t* d_in = static_cast<const uint8_t*>(in);
    const bool host_in = !is_device_ptr(in);
    const uint64_t bound = plzgpu_compress_bound(n, params);
    const Geometry geo = geometry(n, *params);
    // H2D pipeline geometry (env overrides for A/B): ready flags every
    // PLZGPU_SEG_MB, copies of PLZGPU_COPY_MB except over the input's last
    // PLZGPU_TAIL_MB, sent flag segment by flag segment so the matching
    // that can only start after the last byte lands is short
    auto env_mb = [](const char* name, int dflt) {
        const char* v = std::getenv(name);
        return uint64_t(v ? std::max(0, std::atoi(v)) : dflt) << 20;
    };
    const uint64_t seg_bytes_target = std::max<uint64_t>(env_mb("PLZGPU_SEG_MB", 32), 1);
    const uint64_t copy_bytes = env_mb("PLZGPU_COPY_MB", 32);
    const uint64_t tail_bytes = env_mb("PLZGPU_TAIL_MB", 0);
    const uint64_t chunk_bytes = uint64_t(params->chunk_size) * params->symbol_width;
    const uint64_t seg_chunks = std::max<uint64_t>(1, seg_bytes_target / chunk_bytes);
    const uint64_t nseg = (geo.n_chunks + seg_chunks - 1) / seg_chunks;
    // Host input into a pinned host image of several containers: container
    // by container, Kernel III writing each one straight into the host
    // buffer (mapped) while the next container's segments still arrive.
    void* mapped = nullptr;
    const bool per_container =
        host_in && nseg > 1 && geo.n_blocks > 1 && cap >= bound && is_pinned_host(out) &&
        geo.cpb % 4 == 0 && geo.cpb % seg_chunks == 0 && !getenv_flag("PLZGPU_NO_PIPE_ASM") &&
        !getenv_flag("PLZGPU_NO_PIPE") &&
        (cudaHostGetDevicePointer(&mapped, out, 0) == cudaSuccess || (cudaGetLastError(), false));
    const bool direct = (is_device_ptr(out) || per_container) && cap >= bound;
    // per container: Kernel III into HBM and each finished container down on
    // the copy engine (default), or Kernel III writing the mapped host image
    const bool asm_mapped = getenv_flag("PLZGPU_ASM_MAPPED");
    uint8_t* img = static_cast<uint8_t*>(out);
    if (per_container && asm_mapped) {
        img = static_cast<uint8_t*>(mapped);
    } else if (per_container || !direct) {
        CK(c->img.ensure(bound));
        img = c->img.as<uint8_t>();
    }
    Meta* m = dmeta(c);
    StreamWriteValue32Fn write_value = stream_write_value32();
    // PLZGPU_NO_PIPE: no overlapped host paths (profilers serialise the
    // copies the waiting kernels depend on)
    if (host_in && write_value && nseg > 1 && !getenv_flag("PLZGPU_NO_PIPE")) {
        // H2D pipeline: Kernel I starts at once and each warp waits for its
        // chunk's segment; segments land on the copy stream, each followed by
        // a stream memory write of its ready flag.
        CK(c->in.ensure(n));
        CK(c->ready.ensure(nseg * 4));
        if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
        d_in = c->in.as<uint8_t>();
        ++c->epoch;
        if (c->epoch == 0) {  // never reuse the initial 0 flags
            CK(cudaMemsetAsync(c->ready.p, 0, nseg * 4, st));
            CK(cudaStreamSynchronize(st));
            ++c->epoch;
        }
        // the copies first: the H2D stream starts before the launches below
        // are enqueued (each warp of Kernel I waits for its own segment)
        const uint64_t seg_bytes = seg_chunks * chunk_bytes;
        const uint64_t per_copy = std::max<uint64_t>(1, copy_bytes / seg_bytes);
        const uint64_t tail_from = n > tail_bytes ? n - tail_bytes : 0;
        for (uint64_t sgi = 0; sgi < nseg;) {
            const uint64_t lo = sgi * seg_bytes;
            const uint64_t s_end = lo >= tail_from ? sgi + 1 : std::min(nseg, sgi + per_copy);
            const uint64_t hi = s_end == nseg ? n : std::min(n, s_end * seg_bytes);
            CK(cudaMemcpyAsync(c->in.as<uint8_t>() + lo, static_cast<const uint8_t*>(in) + lo,
                               hi - lo, cudaMemcpyHostToDevice, c->copy_stream));
            for (; sgi < s_end; ++sgi)
                if (write_value(c->copy_stream,
                                reinterpret_cast<unsigned long long>(c->ready.as<uint32_t>() + sgi),
                                c->epoch, 0) != 0)
                    return set_err(err, PLZGPU_CUDA, 0, kNoIndex, kNoIndex,
                                   "cuStreamWriteValue32 failed");
        }
        c->pipe_ready = c->ready.as<uint32_t>();
        c->pipe_seg_chunks = uint32_t(seg_chunks);
        if (per_container) {
            rc = enqueue_compress_by_container(c, *params, d_in, n, img, st, err);
        } else {
            rc = enqueue_compress(c, *params, d_in, n, img, &m->img_len, st, err);
        }
        c->pipe_ready = nullptr;
        if (rc) return rc;
        if (per_container && !asm_mapped) {
            // each container's image range is known once its scan is done
            // (global stream prefixes P64 / F64 at its first and last chunk):
            // read the four words, then send the range down after assembly
            for (cudaStream_t* sx : {&c->d2h_stream, &c->size_stream})
                if (!*sx) CK(cudaStreamCreateWithFlags(sx, cudaStreamNonBlocking));
            if (!c->host_scratch)
                CK(cudaMallocHost(reinterpret_cast<void**>(&c->host_scratch), 4 * sizeof(uint64_t)));
            uint64_t off = 0;
            for (uint64_t j = 0; j < geo.n_blocks; ++j) {
                const uint64_t g0 = j * geo.cpb, g1 = std::min(geo.n_chunks, g0 + geo.cpb);
                CK(cudaStreamWaitEvent(c->size_stream, c->cont_ev[2 * j], 0));
                const uint64_t* src[4] = {c->p64.as<uint64_t>() + g0, c->p64.as<uint64_t>() + g1,
                                          c->f64.as<uint64_t>() + g0, c->f64.as<uint64_t>() + g1};
                for (int k = 0; k < 4; ++k)
                    CK(cudaMemcpyAsync(c->host_scratch + k, src[k], 8, cudaMemcpyDeviceToHost,
                                       c->size_stream));
                CK(cudaStreamSynchronize(c->size_stream));
                const uint64_t* v = c->host_scratch;
                const uint64_t tail = j + 1 == geo.n_blocks ? n % uint64_t(params->symbol_width) : 0;
                const uint64_t size = 26 + 8 * (g1 - g0 + 1) + (v[3] - v[2]) + (v[1] - v[0]) + tail;
                if (off + size > cap) break;  // an offset overflow: reported below
                CK(cudaStreamWaitEvent(c->d2h_stream, c->cont_ev[2 * j + 1], 0));
                CK(cudaMemcpyAsync(static_cast<uint8_t*>(out) + off, img + off, size,
                                   cudaMemcpyDeviceToHost, c->d2h_stream));
                off += size;
            }
            CK(cudaStreamSynchronize(c->d2h_stream));
        }
    } else {
        if (host_in) {
            CK(c->in.ensure(n));
            CK(cudaMemcpyAsync(c->in.p, in, n, cudaMemcpyHostToDevice, st));
            d_in = c->in.as<uint8_t>();
        }
        rc = enqueue_compress(c, *params, d_in, n, img, &m->img_len, st, err);
        if (rc) return rc;
    }
    Meta* h = c->host_meta;
    CK(cudaMemcpyAsync(h, m, sizeof(Meta), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h->stalled)
        return set_err(err, PLZGPU_CUDA, 0, kNoIndex, kNoIndex,
                       "H2D pipeline stalled: an input segment never arrived");
    if (h->overflow) return overflow_error(err);
    if (h->img_len > cap)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                       "output buffer too small: need %llu bytes", (unsigned long long)h->img_len);
    if (!direct) {
        CK(cudaMemcpyAsync(out, img, h->img_len,
                           is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           st));
        CK(cudaStreamSynchronize(st));
    }
    *out_len = h->img_len;
    if (stats) {
        stats->max_cmp_per_pos = 0;
        stats->pointer_tokens = h->stats[0];
        stats->literal_tokens = h->stats[1];
    }
    return PLZGPU_OK;
}

int plzgpu_compress_async(plzgpu_ctx* c, const plzgpu_params* params, const void* d_in,
                          uint64_t n, void* d_out, uint64_t cap, uint64_t* d_out_len, void* stream,
                          plzgpu_error* err) {
    clear_err(err);
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    if (cap < plzgpu_compress_bound(n, params))
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                       "async compress needs cap >= plzgpu_compress_bound");
    if (n == 0) {
        CK(cudaMemsetAsync(d_out_len, 0, 8, st));
        Meta* m = dmeta(c);
        CK(cudaMemsetAsync(&m->stats, 0, sizeof m->stats + sizeof m->overflow, st));
        c->last_launches = 0;
        c->last_op = OP_COMPRESS;
        return PLZGPU_OK;
    }
    return enqueue_compress(c, *params, static_cast<const uint8_t*>(d_in), n,
                            static_cast<uint8_t*>(d_out), d_out_len, st, err);
}

int plzgpu_profile_encode(plzgpu_ctx* c, const plzgpu_params* params, const void* d_in,
                          uint64_t n, void* stream, plzgpu_error* err) {
    clear_err(err);
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    if (n == 0) return PLZGPU_OK;
    CK(cudaSetDevice(c->device));
    return enqueue_compress(c, *params, static_cast<const uint8_t*>(d_in), n, nullptr, nullptr,
                            pick(c, stream), err, 1);
}

int plzgpu_decompress(plzgpu_ctx* c, const void* img, uint64_t len, void* out, uint64_t cap,
                      uint64_t* out_len, void* stream, plzgpu_error* err) {
    clear_err(err);
    *out_len = 0;
    if (len == 0) return PLZGPU_OK;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const uint8_t* d_img = static_cast<const uint8_t*>(img);
    if (!is_device_ptr(img) && is_pinned_host(out) &&
        try_decompress_pipelined(c, static_cast<const uint8_t*>(img), len,
                                 static_cast<uint8_t*>(out), cap, out_len, st, err) == 1)
        return PLZGPU_OK;
    clear_err(err);  // the resident path below reports any error
    if (!is_device_ptr(img)) {
        CK(c->img.ensure(len));
        CK(cudaMemcpyAsync(c->img.p, img, len, cudaMemcpyHostToDevice, st));
        d_img = c->img.as<uint8_t>();
    }
    const bool direct = is_device_ptr(out) && (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    uint8_t* d_out = static_cast<uint8_t*>(out);
    if (!direct) {
        CK(c->out.ensure(cap + 16));
        d_out = c->out.as<uint8_t>();
    }
    for (;;) {
        int rc = enqueue_decompress(c, d_img, len, d_out, cap, nullptr, st, err);
        if (rc) return rc;
        bool grow = false;
        rc = finish_decompress(c, st, &grow, err);
        if (rc) return rc;
        if (!grow) break;
        CK(c->desc.ensure(c->desc.cap * 4));
    }
    Meta h;
    CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint64_t total = h.parse.total_out;
    if (!direct && total) {
        CK(cudaMemcpyAsync(out, d_out, total,
                           is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           st));
        CK(cudaStreamSynchronize(st));
    }
    *out_len = total;
    return PLZGPU_OK;
}

int plzgpu_decompress_range(plzgpu_ctx* c, const void* img, uint64_t len, uint64_t chunk_begin,
                            uint64_t chunk_end, void* out, uint64_t cap, uint64_t* out_begin,
                            uint64_t* out_len, uint64_t* total_chunks, void* stream,
                            plzgpu_error* err) {
    clear_err(err);
    *out_begin = 0;
    *out_len = 0;
    *total_chunks = 0;
    if (len == 0) return PLZGPU_OK;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const uint8_t* d_img = static_cast<const uint8_t*>(img);
    if (!is_device_ptr(img)) {
        CK(c->img.ensure(len));
        CK(cudaMemcpyAsync(c->img.p, img, len, cudaMemcpyHostToDevice, st));
        d_img = c->img.as<uint8_t>();
    }
    const bool query = out == nullptr;  // sizes only
    const bool direct = query || is_device_ptr(out);
    Meta* m = dmeta(c);
    // the header walk over the whole image (every container's checks), no
    // capacity check and no tails: the range kernel places those
    DecodeArgs a{};
    Meta h;
    for (;;) {
        if (c->desc.cap < 64 * sizeof(ContainerDesc)) CK(c->desc.ensure(64 * sizeof(ContainerDesc)));
        CK(cudaMemsetAsync(&m->parse, 0, sizeof m->parse, st));
        CK(cudaMemsetAsync(&m->err_chunk, 0xff, sizeof m->err_chunk + sizeof m->mono_key, st));
        CK(cudaMemsetAsync(m->work, 0, sizeof m->work, st));
        a = DecodeArgs{};
        a.img = d_img;
        a.img_len = len;
        a.out = nullptr;
        a.out_cap = UINT64_MAX;
        a.desc = c->desc.as<ContainerDesc>();
        a.desc_cap = c->desc.cap / sizeof(ContainerDesc);
        a.result = &m->parse;
        a.err_chunk = &m->err_chunk;
        a.mono_key = &m->mono_key;
        a.work = &m->work[2];
        launch_parse(a, st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h.parse.err_kind == 17) {
            CK(c->desc.ensure(c->desc.cap * 4));
            continue;
        }
        break;
    }
    if (h.parse.err_kind != 0) return parse_error(h.parse, err);
    const uint64_t total = h.parse.total_chunks;
    const uint64_t ce = std::min(chunk_end, total), cb = std::min(chunk_begin, ce);
    // output range and tails: into the caller's buffer when it is device
    // memory, else into the staging buffer (copied back below)
    uint8_t* d_out = static_cast<uint8_t*>(out);
    if (!direct) {
        CK(c->out.ensure(cap + 16));
        d_out = c->out.as<uint8_t>();
    }
    launch_range(a, cb, ce, d_out, m->range, st);  // d_out null: bounds only
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint64_t lo = h.range[0], hi = h.range[1];
    *total_chunks = total;
    if (query) {
        *out_begin = lo;
        *out_len = hi - lo;
        return PLZGPU_OK;
    }
    if (hi - lo > cap)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                       "output buffer too small: need %llu bytes", (unsigned long long)(hi - lo));
    if (ce > cb) {
        // the decode kernel over [cb, ce): work counter from cb, bound ce,
        // output addressed relative to the range's first byte
        const uint32_t w0 = uint32_t(cb);
        CK(cudaMemcpyAsync(&m->work[2], &w0, 4, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(&m->parse.total_chunks, &ce, 8, cudaMemcpyHostToDevice, st));
        a.out = reinterpret_cast<uint8_t*>(reinterpret_cast<uintptr_t>(d_out) - lo);
        a.out_cap = hi;
        int per_sm = decode_ctas_per_sm();
        if (per_sm < 1) per_sm = 1;
        launch_decode(a, c->sms * per_sm, st);
        CK(cudaGetLastError());
        c->last_launches = 3;
        c->last_op = OP_DECOMPRESS;
        c->last_decode = a;
        bool grow = false;
        const int rc = finish_decompress(c, st, &grow, err);
        if (rc) return rc;
    }
    if (!direct && hi > lo) {
        CK(cudaMemcpyAsync(out, d_out, hi - lo, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    *out_begin = lo;
    *out_len = hi - lo;
    return PLZGPU_OK;
}

int plzgpu_decompress_async(plzgpu_ctx* c, const void* d_img, uint64_t len, void* d_out,
                            uint64_t cap, uint64_t* d_out_len, void* stream, plzgpu_error* err) {
    clear_err(err);
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    if (reinterpret_cast<uintptr_t>(d_out) & 15u)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                       "async decompress needs a 16-byte aligned device output");
    if (len == 0) {
        CK(cudaMemsetAsync(d_out_len, 0, 8, st));
        Meta* m = dmeta(c);
        CK(cudaMemsetAsync(&m->parse, 0, sizeof m->parse, st));
        CK(cudaMemsetAsync(&m->err_chunk, 0xff, sizeof m->err_chunk + sizeof m->mono_key, st));
        c->last_launches = 0;
        c->last_op = OP_NONE;
        return PLZGPU_OK;
    }
    return enqueue_decompress(c, static_cast<const uint8_t*>(d_img), len,
                              static_cast<uint8_t*>(d_out), cap, d_out_len, st, err);
}

int plzgpu_ctx_finish(plzgpu_ctx* c, void* stream, plzgpu_stats* stats, plzgpu_error* err) {
    clear_err(err);
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    if (c->last_op == OP_DECOMPRESS) {
        bool grow = false;
        const int rc = finish_decompress(c, st, &grow, err);
        if (rc) return rc;
        if (grow)
            return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                           "too many containers for the async descriptor table; use "
                           "plzgpu_decompress once to size it");
        return PLZGPU_OK;
    }
    Meta* h = c->host_meta;
    CK(cudaMemcpyAsync(h, c->meta.p, sizeof(Meta), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (c->last_op == OP_COMPRESS) {
        if (h->overflow) return overflow_error(err);
        if (stats) {
            stats->max_cmp_per_pos = 0;
            stats->pointer_tokens = h->stats[0];
            stats->literal_tokens = h->stats[1];
        }
    }
    return PLZGPU_OK;
}

int plzgpu_decompress_chunk(plzgpu_ctx* c, const void* flags, uint64_t n_flags,
                            const void* payload, uint64_t n_payload, uint64_t logical,
                            const plzgpu_params* params, uint64_t chunk_index, void* out,
                            plzgpu_error* err) {
    clear_err(err);
    if (params->symbol_width != 1 && params->symbol_width != 2 && params->symbol_width != 4)
        return bad_field(err, "symbol_width", "{1,2,4}");
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = c->stream;  // private: synchronous call
    const uint64_t S = uint64_t(params->symbol_width);
    const uint64_t out_bytes = logical * S;
    // stage everything in one device scratch: flags | payload | out
    const uint64_t fo = 0, po = (n_flags + 15) & ~uint64_t(15);
    const uint64_t oo = po + ((n_payload + 15) & ~uint64_t(15));
    CK(c->in.ensure(oo + out_bytes + 16));
    uint8_t* base = c->in.as<uint8_t>();
    const bool dev_f = is_device_ptr(flags), dev_p = is_device_ptr(payload);
    if (n_flags)
        CK(cudaMemcpyAsync(base + fo, flags, n_flags,
                           dev_f ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    if (n_payload)
        CK(cudaMemcpyAsync(base + po, payload, n_payload,
                           dev_p ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    Meta* m = dmeta(c);
    DecodeOneArgs a{};
    a.flags = base + fo;
    a.n_flags = n_flags;
    a.payload = base + po;
    a.n_payload = n_payload;
    a.logical = logical;
    a.S = params->symbol_width;
    a.out = base + oo;
    a.err_code = &m->detail_code;
    a.err_token = &m->detail_token;
    launch_decode_one(a, st);
    CK(cudaGetLastError());
    c->last_launches = 1;
    Meta h;
    CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h.detail_code != TE_OK) return token_error(h.detail_code, chunk_index, h.detail_token, err);
    if (out_bytes)
        CK(cudaMemcpyAsync(out, base + oo, out_bytes,
                           is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           st));
    CK(cudaStreamSynchronize(st));
    return PLZGPU_OK;
}

// ------------------------------------------------------------ shards

// Segments of the final image a shard owns in one container:
// its slice of each offset table and of both streams.  Pure host arithmetic.
static uint64_t shard_segments_impl(const plzgpu_params& p, uint64_t n_total, uint64_t begin,
                                    uint64_t end, const uint64_t* totals, const uint64_t* bases,
                                    uint64_t n_touched, uint64_t* segs, uint64_t max_segs) {
    const Geometry g = geometry(n_total, p);
    uint64_t count = 0, local = 0;
    for (uint64_t i = 0; i < n_touched; ++i) {
        const uint64_t j = totals[3 * i];
        const uint64_t g0 = j * g.cpb;
        const uint64_t nj = (j + 1 == g.n_blocks) ? g.n_chunks - g0 : g.cpb;
        const uint64_t lo = std::max(begin, g0), hi = std::min(end, g0 + nj);
        const uint64_t k_lo = lo - g0, cnt = hi - lo;
        const uint64_t lp = totals[3 * i + 1], lf = totals[3 * i + 2];
        const uint64_t p_base = bases[4 * i], f_base = bases[4 * i + 1];
        const uint64_t img_off = bases[4 * i + 2], f_total = bases[4 * i + 3];
        const uint64_t tabs = img_off + 26, streams = tabs + 8 * (nj + 1);
        const uint64_t seg[4][2] = {{tabs + 4 * k_lo, 4 * cnt},
                                    {tabs + 4 * (nj + 1) + 4 * k_lo, 4 * cnt},
                                    {streams + f_base, lf},
                                    {streams + f_total + p_base, lp}};
        for (const auto& sg : seg) {
            if (count < max_segs && segs) {
                segs[3 * count] = sg[0];
                segs[3 * count + 1] = local;
                segs[3 * count + 2] = sg[1];
            }
            local += sg[1];
            ++count;
        }
    }
    return count;
}

uint64_t plzgpu_num_chunks(uint64_t n, const plzgpu_params* p) { return geometry(n, *p).n_chunks; }

uint64_t plzgpu_num_containers(uint64_t n, const plzgpu_params* p) {
    return geometry(n, *p).n_blocks;
}

uint64_t plzgpu_shard_segments(const plzgpu_params* p, uint64_t n_total, uint64_t chunk_begin,
                               uint64_t chunk_end, const uint64_t* totals, const uint64_t* bases,
                               uint64_t n_touched, uint64_t* segs, uint64_t max_segs) {
    return shard_segments_impl(*p, n_total, chunk_begin, chunk_end, totals, bases, n_touched, segs,
                               max_segs);
}

int plzgpu_shard_encode(plzgpu_ctx* c, const plzgpu_params* params, const void* in,
                        uint64_t n_total, uint64_t chunk_begin, uint64_t chunk_end,
                        uint64_t* totals, uint64_t max_touched, uint64_t* n_touched, void* stream,
                        plzgpu_error* err) {
    clear_err(err);
    *n_touched = 0;
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    const plzgpu_params& p = *params;
    const Geometry g = geometry(n_total, p);
    if (chunk_begin > chunk_end || chunk_end > g.n_chunks)
        return set_err(err, PLZGPU_CONTRACT, 0, kNoIndex, kNoIndex, "shard range outside the input");
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const uint64_t S = uint64_t(p.symbol_width), C = uint64_t(p.chunk_size);
    const uint64_t L = chunk_end - chunk_begin;
    const uint32_t last_len = chunk_end == g.n_chunks ? g.last_len : uint32_t(C);
    uint64_t local_bytes = L * C * S;
    if (chunk_end == g.n_chunks && L) local_bytes = n_total - chunk_begin * C * S;
    const uint8_t* d_in = static_cast<const uint8_t*>(in);
    if (L && !is_device_ptr(in)) {
        CK(c->in.ensure(local_bytes + 16));
        CK(cudaMemcpyAsync(c->in.p, in, local_bytes, cudaMemcpyHostToDevice, st));
        d_in = c->in.as<uint8_t>();
    }
    int launches = 0;
    rc = enqueue_encode_scan(c, p, d_in, L, last_len, st, err, &launches);
    if (rc) return rc;
    CK(cudaGetLastError());
    c->last_launches = launches;
    // per touched container: local prefix values at its range ends
    c->sh_touch.clear();
    const uint64_t j_first = L ? chunk_begin / g.cpb : 0, j_last = L ? (chunk_end - 1) / g.cpb : 0;
    std::vector<uint64_t> idx;
    for (uint64_t j = j_first; L && j <= j_last; ++j) {
        const uint64_t lo = std::max(chunk_begin, j * g.cpb);
        const uint64_t hi = std::min(chunk_end, std::min((j + 1) * g.cpb, g.n_chunks));
        c->sh_touch.insert(c->sh_touch.end(), {j, lo, hi, 0, 0});
        idx.push_back(lo - chunk_begin);
        idx.push_back(hi - chunk_begin);
    }
    std::vector<uint64_t> pv(idx.size()), fv(idx.size());
    for (size_t i = 0; i < idx.size(); ++i) {
        CK(cudaMemcpyAsync(&pv[i], c->p64.as<uint64_t>() + idx[i], 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&fv[i], c->f64.as<uint64_t>() + idx[i], 8, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    const uint64_t nt = c->sh_touch.size() / 5;
    for (uint64_t i = 0; i < nt; ++i) {
        c->sh_touch[5 * i + 3] = pv[2 * i + 1] - pv[2 * i];
        c->sh_touch[5 * i + 4] = fv[2 * i + 1] - fv[2 * i];
        if (i < max_touched && totals) {
            totals[3 * i] = c->sh_touch[5 * i];
            totals[3 * i + 1] = c->sh_touch[5 * i + 3];
            totals[3 * i + 2] = c->sh_touch[5 * i + 4];
        }
    }
    c->sh_begin = chunk_begin;
    c->sh_end = chunk_end;
    c->sh_n = n_total;
    c->sh_params = p;
    *n_touched = nt;
    return PLZGPU_OK;
}

int plzgpu_shard_assemble(plzgpu_ctx* c, const uint64_t* bases, void* d_out, uint64_t cap,
                          uint64_t* segs, uint64_t max_segs, uint64_t* n_segs, uint64_t* out_len,
                          void* stream, plzgpu_error* err) {
    clear_err(err);
    *n_segs = 0;
    *out_len = 0;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const plzgpu_params& p = c->sh_params;
    const uint64_t nt = c->sh_touch.size() / 5;
    std::vector<uint64_t> totals(3 * nt);
    for (uint64_t i = 0; i < nt; ++i) {
        totals[3 * i] = c->sh_touch[5 * i];
        totals[3 * i + 1] = c->sh_touch[5 * i + 3];
        totals[3 * i + 2] = c->sh_touch[5 * i + 4];
    }
    std::vector<uint64_t> sg(12 * nt + 3);
    const uint64_t ns = shard_segments_impl(p, c->sh_n, c->sh_begin, c->sh_end, totals.data(), bases,
                                            nt, sg.data(), 4 * nt);
    uint64_t total = 0;
    for (uint64_t i = 0; i < ns; ++i) total += sg[3 * i + 2];
    if (total > cap)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex, "shard buffer too small");
    std::vector<ShardCont> conts(nt);
    for (uint64_t i = 0; i < nt; ++i) {
        const Geometry g = geometry(c->sh_n, p);
        ShardCont& d = conts[i];
        const uint64_t j = c->sh_touch[5 * i], lo = c->sh_touch[5 * i + 1];
        d.g_lo = lo - c->sh_begin;
        d.g_hi = c->sh_touch[5 * i + 2] - c->sh_begin;
        d.k_lo = lo - j * g.cpb;
        d.p_base = bases[4 * i];
        d.f_base = bases[4 * i + 1];
        d.seg_ptab = sg[3 * (4 * i) + 1];
        d.seg_ftab = sg[3 * (4 * i + 1) + 1];
        d.seg_flags = sg[3 * (4 * i + 2) + 1];
        d.seg_pay = sg[3 * (4 * i + 3) + 1];
    }
    if (nt) {
        CK(c->shard_desc.ensure(nt * sizeof(ShardCont)));
        CK(cudaMemcpyAsync(c->shard_desc.p, conts.data(), nt * sizeof(ShardCont),
                           cudaMemcpyHostToDevice, st));
        Meta* m = dmeta(c);
        CK(cudaMemsetAsync(&m->overflow, 0, sizeof m->overflow, st));
        ShardAssembleArgs a{};
        a.pay_slots = c->pay_slots.as<uint8_t>();
        a.flag_slots = c->flag_slots.as<uint8_t>();
        a.psize = c->psize.as<uint32_t>();
        a.fsize = c->fsize.as<uint32_t>();
        a.P64 = c->p64.as<uint64_t>();
        a.F64 = c->f64.as<uint64_t>();
        a.conts = c->shard_desc.as<ShardCont>();
        a.n_conts = nt;
        a.out = static_cast<uint8_t*>(d_out);
        a.overflow = &m->overflow;
        a.n_chunks = c->sh_end - c->sh_begin;
        a.S = p.symbol_width;
        a.C = p.chunk_size;
        launch_shard_assemble(a, st);
        CK(cudaGetLastError());
        c->last_launches = 1;
        Meta h;
        CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h.overflow) return overflow_error(err);
    }
    for (uint64_t i = 0; i < ns && i < max_segs && segs; ++i)
        for (int q = 0; q < 3; ++q) segs[3 * i + q] = sg[3 * i + q];
    *n_segs = ns;
    *out_len = total;
    return PLZGPU_OK;
}

int plzgpu_shard_headers(plzgpu_ctx* c, const plzgpu_params* params, uint64_t n_total,
                         const uint64_t* totals, const void* tail, void* d_img, uint64_t cap,
                         uint64_t* img_len, void* stream, plzgpu_error* err) {
    clear_err(err);
    *img_len = 0;
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    const plzgpu_params& p = *params;
    const Geometry g = geometry(n_total, p);
    std::vector<HeaderDesc> hd(g.n_blocks);
    uint64_t at = 0;
    for (uint64_t j = 0; j < g.n_blocks; ++j) {
        HeaderDesc& d = hd[j];
        const uint64_t g0 = j * g.cpb;
        d.n = uint32_t((j + 1 == g.n_blocks) ? g.n_chunks - g0 : g.cpb);
        d.byte_len = (j + 1 == g.n_blocks) ? n_total - j * p.block_bytes : p.block_bytes;
        d.tail_len = uint8_t(d.byte_len % uint64_t(p.symbol_width));
        for (int i = 0; i < d.tail_len; ++i) d.tail[i] = static_cast<const uint8_t*>(tail)[i];
        d.ptot = totals[2 * j];
        d.ftot = totals[2 * j + 1];
        if (d.ptot > 0xffffffffull || d.ftot > 0xffffffffull) return overflow_error(err);
        d.img_off = at;
        at += 26 + 8 * (uint64_t(d.n) + 1) + d.ptot + d.ftot + d.tail_len;
    }
    if (at > cap)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex, "image buffer too small");
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    if (g.n_blocks) {
        CK(c->shard_desc.ensure(g.n_blocks * sizeof(HeaderDesc)));
        CK(cudaMemcpyAsync(c->shard_desc.p, hd.data(), g.n_blocks * sizeof(HeaderDesc),
                           cudaMemcpyHostToDevice, st));
        launch_shard_headers(c->shard_desc.as<HeaderDesc>(), g.n_blocks,
                             static_cast<uint8_t*>(d_img), p.symbol_width, p.window, p.interval,
                             p.chunk_size, st);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
    }
    *img_len = at;
    return PLZGPU_OK;
}

// --------------------------------------------------- statistics / matcher

int plzgpu_match_table(plzgpu_ctx* c, const plzgpu_params* params, const void* in, uint64_t n,
                       void* len_out, void* off_out, uint64_t* raw_hist, void* stream,
                       plzgpu_error* err) {
    clear_err(err);
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    const plzgpu_params& p = *params;
    const Geometry g = geometry(n, p);
    const uint64_t S = uint64_t(p.symbol_width), C = uint64_t(p.chunk_size);
    const uint64_t nsym = n / S;
    if (raw_hist) std::memset(raw_hist, 0, 256 * sizeof(uint64_t));
    if (g.n_chunks == 0) return PLZGPU_OK;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const uint8_t* d_in = static_cast<const uint8_t*>(in);
    if (!is_device_ptr(in)) {
        CK(c->in.ensure(n + 16));
        CK(cudaMemcpyAsync(c->in.p, in, n, cudaMemcpyHostToDevice, st));
        d_in = c->in.as<uint8_t>();
    }
    const uint64_t tab_bytes = g.n_chunks * C;  // chunk g's records at g*C
    CK(c->table.ensure(2 * tab_bytes + 16));
    CK(c->hist.ensure(256 * 8));
    uint8_t* dl = c->table.as<uint8_t>();
    uint8_t* dof = dl + tab_bytes;
    Meta* m = dmeta(c);
    CK(cudaMemsetAsync(m->work, 0, sizeof m->work, st));
    CK(cudaMemsetAsync(c->hist.p, 0, 256 * 8, st));
    EncodeArgs e{};
    e.in = d_in;
    e.work = &m->work[0];
    e.n_chunks = g.n_chunks;
    e.last_len = g.last_len;
    e.C = p.chunk_size;
    e.W = p.window;
    e.I = p.interval;
    e.min_match = std::max(1, p.min_match);
    int wpc = 1, per_sm = 1;
    encode_shape(c, p, 0, &wpc, &per_sm);
    e.warps_per_cta = wpc;
    uint64_t grid = std::min<uint64_t>(uint64_t(c->sms) * per_sm, (g.n_chunks + wpc - 1) / wpc);
    launch_match_table(p.symbol_width, e, int(grid), dl, dof,
                       reinterpret_cast<unsigned long long*>(c->hist.p), st);
    CK(cudaGetLastError());
    c->last_launches = 1;
    // gather the chunk-strided tables into symbol order
    const bool dev_out = is_device_ptr(len_out);
    const cudaMemcpyKind kind = dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (len_out && off_out) {
        CK(cudaMemcpyAsync(len_out, dl, nsym, kind, st));
        CK(cudaMemcpyAsync(off_out, dof, nsym, kind, st));
    }
    if (raw_hist) CK(cudaMemcpyAsync(raw_hist, c->hist.p, 256 * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return PLZGPU_OK;
}

// ----------------------------------------------------------- cuSZ use case
namespace {
int lorenzo_args(const void* a, const void* b, uint64_t nx, uint64_t ny, uint64_t nz, double eb,
                 int32_t radius, plzgpu_error* err) {
    if (!(eb > 0.0) || !(eb < 1e30))
        return set_err(err, PLZGPU_VALIDATION, 0, kNoIndex, kNoIndex, "eb must be positive");
    if (radius < 1 || radius > 32768)
        return set_err(err, PLZGPU_VALIDATION, 0, kNoIndex, kNoIndex, "radius must be in [1,32768]");
    if (nx == 0 || ny == 0 || nz == 0)
        return set_err(err, PLZGPU_VALIDATION, 0, kNoIndex, kNoIndex, "dimensions must be >= 1");
    if (!is_device_ptr(a) || !is_device_ptr(b))
        return set_err(err, PLZGPU_VALIDATION, 0, kNoIndex, kNoIndex,
                       "the quantizer takes device buffers");
    return PLZGPU_OK;
}
}  // namespace

int plzgpu_lorenzo_quantize(plzgpu_ctx* c, const float* d_field, uint64_t nx, uint64_t ny,
                            uint64_t nz, double eb, int32_t radius, uint16_t* d_codes,
                            uint64_t* d_outlier_idx, int32_t* d_outlier_val, uint64_t outlier_cap,
                            uint64_t* n_outliers, void* stream, plzgpu_error* err) {
    clear_err(err);
    CK(cudaSetDevice(c->device));
    if (int rc = lorenzo_args(d_field, d_codes, nx, ny, nz, eb, radius, err)) return rc;
    const cudaStream_t st = pick(c, stream);
    const uint64_t n = nx * ny * nz, tiles = lorenzo_tiles(n);
    CK(c->qtiles.ensure(tiles * 4 + 64));
    CK(c->qoff.ensure(2 * (tiles + 1) * 8 + 16));  // exclusive prefixes + a scratch twin
    const uint64_t stiles = (tiles + kScanTile - 1) / kScanTile;
    CK(c->status.ensure(stiles * 4 + 4));
    CK(c->agg.ensure(stiles * 16 + 16));
    CK(c->incl.ensure(stiles * 16 + 16));
    const float s = float(1.0 / (2.0 * eb));
    launch_lorenzo_quantize(d_field, nx, ny, nz, s, radius, d_codes, c->qtiles.as<uint32_t>(), st);
    // exclusive scan of the per-tile counts: Kernel II (the flag half of its
    // pair scan runs on the same counts into a scratch twin)
    Meta* m = dmeta(c);
    CK(cudaMemsetAsync(c->status.p, 0, stiles * 4, st));
    CK(cudaMemsetAsync(&m->work[1], 0, 4, st));
    ScanArgs sa{};
    sa.psize = c->qtiles.as<uint32_t>();
    sa.fsize = c->qtiles.as<uint32_t>();
    sa.n = tiles;
    sa.P64 = c->qoff.as<uint64_t>();
    sa.F64 = c->qoff.as<uint64_t>() + tiles + 1;
    sa.status = c->status.as<uint32_t>();
    sa.agg = c->agg.as<ulonglong2>();
    sa.incl = c->incl.as<ulonglong2>();
    sa.tile_counter = &m->work[1];
    launch_scan(sa, st);
    launch_outlier_write(d_field, nx, ny, nz, s, d_codes, c->qtiles.as<uint32_t>(),
                         c->qoff.as<uint64_t>(), d_outlier_idx, d_outlier_val, outlier_cap, st);
    CK(cudaGetLastError());
    uint64_t total = 0;
    CK(cudaMemcpyAsync(&total, c->qoff.as<uint64_t>() + tiles, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    c->last_launches = 3;
    if (n_outliers) *n_outliers = total;
    if (total > outlier_cap)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                       "%llu outliers exceed the outlier buffer (%llu)",
                       (unsigned long long)total, (unsigned long long)outlier_cap);
    return PLZGPU_OK;
}

int plzgpu_lorenzo_reconstruct(plzgpu_ctx* c, const uint16_t* d_codes,
                               const uint64_t* d_outlier_idx, const int32_t* d_outlier_val,
                               uint64_t n_outliers, uint64_t nx, uint64_t ny, uint64_t nz,
                               double eb, int32_t radius, float* d_field, void* stream,
                               plzgpu_error* err) {
    clear_err(err);
    CK(cudaSetDevice(c->device));
    if (int rc = lorenzo_args(d_codes, d_field, nx, ny, nz, eb, radius, err)) return rc;
    const cudaStream_t st = pick(c, stream);
    const uint64_t n = nx * ny * nz;
    CK(c->qdelta.ensure(n * 4 + 16));
    launch_lorenzo_reconstruct(d_codes, d_outlier_idx, d_outlier_val, n_outliers, nx, ny, nz,
                               radius, float(2.0 * eb), c->qdelta.as<int32_t>(), d_field, c->sms,
                               st);
    CK(cudaGetLastError());
    c->last_launches = 5;
    return PLZGPU_OK;
}

int plzgpu_pointer_histogram(plzgpu_ctx* c, const plzgpu_params* params, const void* in,
                             uint64_t n, uint64_t* hist, void* stream, plzgpu_error* err) {
    clear_err(err);
    std::memset(hist, 0, 256 * sizeof(uint64_t));
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    const Geometry g = geometry(n, *params);
    if (g.n_chunks == 0) return PLZGPU_OK;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const uint8_t* d_in = static_cast<const uint8_t*>(in);
    if (!is_device_ptr(in)) {
        CK(c->in.ensure(n + 16));
        CK(cudaMemcpyAsync(c->in.p, in, n, cudaMemcpyHostToDevice, st));
        d_in = c->in.as<uint8_t>();
    }
    CK(c->hist.ensure(256 * 8));
    CK(cudaMemsetAsync(c->hist.p, 0, 256 * 8, st));
    c->enc_hist = reinterpret_cast<unsigned long long*>(c->hist.p);
    int launches = 0;
    rc = enqueue_encode_scan(c, *params, d_in, g.n_chunks, g.last_len, st, err, &launches, false);
    c->enc_hist = nullptr;
    if (rc) return rc;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(hist, c->hist.p, 256 * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return PLZGPU_OK;
}


// One stream compressed by several GPUs of this process:
// the shard protocol of dist.py with host threads for ranks — chunk ranges
// encoded concurrently (one context and host thread per listed device), the
// offset plan from the per-container totals, every rank's segments copied
// into one image on the first device (peer copies), headers there, then the
// image to `out`.  The image equals plzgpu_compress's byte for byte.
int plzgpu_compress_multi(const int* devices, int n_devices, const plzgpu_params* params,
                          const void* in, uint64_t n, void* out, uint64_t cap, uint64_t* out_len,
                          plzgpu_stats* stats, plzgpu_error* err) {
    clear_err(err);
    *out_len = 0;
    if (stats) std::memset(stats, 0, sizeof *stats);
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    if (n_devices < 1 || !devices)
        return set_err(err, PLZGPU_CONTRACT, 0, kNoIndex, kNoIndex, "empty device list");
    if (n == 0) return PLZGPU_OK;
    const plzgpu_params& p = *params;
    const Geometry g = geometry(n, p);
    const uint64_t S = uint64_t(p.symbol_width), C = uint64_t(p.chunk_size), N = uint64_t(n_devices);
    const bool dev_in = is_device_ptr(in);
    std::vector<plzgpu_ctx*> ctx(N, nullptr);
    std::vector<void*> allocs;  // (device, pointer) pairs freed at the end
    std::vector<int> alloc_dev;
    auto cleanup = [&](int code) {
        for (size_t i = 0; i < allocs.size(); ++i) {
            cudaSetDevice(alloc_dev[i]);
            cudaFree(allocs[i]);
        }
        for (plzgpu_ctx* c : ctx)
            if (c) plzgpu_ctx_destroy(c);
        return code;
    };
    auto dev_alloc = [&](int dev, uint64_t bytes, uint8_t** ptr) -> cudaError_t {
        cudaError_t e = cudaSetDevice(dev);
        if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(ptr), bytes);
        if (e == cudaSuccess) {
            allocs.push_back(*ptr);
            alloc_dev.push_back(dev);
        }
        return e;
    };
    for (uint64_t r = 0; r < N; ++r) {
        rc = plzgpu_ctx_create(devices[r], &ctx[r], err);
        if (rc) return cleanup(rc);
    }
    // ---- ranks encode their chunk ranges concurrently
    uint64_t max_touched = 1;
    std::vector<uint64_t> rb(N), re(N);
    for (uint64_t r = 0; r < N; ++r) {
        rb[r] = g.n_chunks * r / N;
        re[r] = g.n_chunks * (r + 1) / N;
        max_touched = std::max(max_touched, (re[r] - rb[r] + g.cpb - 1) / g.cpb + 1);
    }
    std::vector<uint8_t*> slice(N, nullptr);
    for (uint64_t r = 0; r < N; ++r) {  // a device input: each rank's slice onto its own GPU
        const uint64_t lo = rb[r] * C * S, hi = re[r] == g.n_chunks ? n : re[r] * C * S;
        if (!dev_in || hi <= lo) continue;
        cudaError_t e = dev_alloc(devices[r], hi - lo, &slice[r]);
        if (e == cudaSuccess)
            e = cudaMemcpy(slice[r], static_cast<const uint8_t*>(in) + lo, hi - lo, cudaMemcpyDefault);
        if (e != cudaSuccess) return cleanup(cuda_fail(err, e, "plzgpu_compress_multi input"));
    }
    std::vector<std::vector<uint64_t>> tot(N);
    std::vector<int> rcs(N, PLZGPU_OK);
    std::vector<plzgpu_error> errs(N);
    {
        std::vector<std::thread> th;
        for (uint64_t r = 0; r < N; ++r)
            th.emplace_back([&, r] {
                const void* src = slice[r] ? static_cast<const void*>(slice[r])
                                           : static_cast<const uint8_t*>(in) + rb[r] * C * S;
                tot[r].assign(3 * max_touched, 0);
                uint64_t nt = 0;
                rcs[r] = plzgpu_shard_encode(ctx[r], &p, src, n, rb[r], re[r], tot[r].data(),
                                             max_touched, &nt, nullptr, &errs[r]);
                tot[r].resize(3 * nt);
            });
        for (std::thread& t : th) t.join();
    }
    for (uint64_t r = 0; r < N; ++r)
        if (rcs[r]) {
            if (err) *err = errs[r];
            return cleanup(rcs[r]);
        }
    // ---- the offset plan (dist.plan_offsets)
    std::vector<uint64_t> ptot(g.n_blocks, 0), ftot(g.n_blocks, 0), img_off(g.n_blocks, 0);
    std::vector<std::vector<uint64_t>> bases(N);
    for (uint64_t r = 0; r < N; ++r)
        for (size_t i = 0; 3 * i < tot[r].size(); ++i) {
            const uint64_t j = tot[r][3 * i];
            bases[r].insert(bases[r].end(), {ptot[j], ftot[j], 0, 0});
            ptot[j] += tot[r][3 * i + 1];
            ftot[j] += tot[r][3 * i + 2];
        }
    uint64_t image_len = 0;
    for (uint64_t j = 0; j < g.n_blocks; ++j) {
        const uint64_t nj = (j + 1 == g.n_blocks) ? g.n_chunks - j * g.cpb : g.cpb;
        const uint64_t bytes = (j + 1 == g.n_blocks) ? n - j * p.block_bytes : p.block_bytes;
        img_off[j] = image_len;
        image_len += 26 + 8 * (nj + 1) + ptot[j] + ftot[j] + bytes % S;
    }
    for (uint64_t r = 0; r < N; ++r)
        for (size_t i = 0; 3 * i < tot[r].size(); ++i) {
            const uint64_t j = tot[r][3 * i];
            bases[r][4 * i + 2] = img_off[j];
            bases[r][4 * i + 3] = ftot[j];
        }
    if (image_len > cap)
        return cleanup(set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                               "output buffer too small: need %llu bytes",
                               (unsigned long long)image_len));
    // ---- every rank's segments into one image on the first device
    uint8_t* d_img = nullptr;
    cudaError_t e = dev_alloc(devices[0], image_len + 16, &d_img);
    if (e != cudaSuccess) return cleanup(cuda_fail(err, e, "plzgpu_compress_multi image"));
    for (uint64_t r = 0; r < N; ++r) {
        const uint64_t nt = tot[r].size() / 3;
        if (nt == 0) continue;
        uint64_t local = 8 * (re[r] - rb[r]) + 16;
        for (uint64_t i = 0; i < nt; ++i) local += tot[r][3 * i + 1] + tot[r][3 * i + 2];
        uint8_t* d_local = nullptr;
        e = dev_alloc(devices[r], local, &d_local);
        if (e != cudaSuccess) return cleanup(cuda_fail(err, e, "plzgpu_compress_multi segments"));
        std::vector<uint64_t> segs(12 * nt);
        uint64_t ns = 0, ln = 0;
        rc = plzgpu_shard_assemble(ctx[r], bases[r].data(), d_local, local, segs.data(), 4 * nt,
                                   &ns, &ln, nullptr, err);
        if (rc) return cleanup(rc);
        for (uint64_t k = 0; k < ns; ++k)
            if (segs[3 * k + 2]) {
                e = cudaMemcpy(d_img + segs[3 * k], d_local + segs[3 * k + 1], segs[3 * k + 2],
                               cudaMemcpyDefault);
                if (e != cudaSuccess) return cleanup(cuda_fail(err, e, "plzgpu_compress_multi gather"));
            }
    }
    // ---- headers, final table entries and the tail on the root, then out
    std::vector<uint64_t> totals(2 * g.n_blocks);
    for (uint64_t j = 0; j < g.n_blocks; ++j) {
        totals[2 * j] = ptot[j];
        totals[2 * j + 1] = ftot[j];
    }
    uint8_t tail[4] = {0, 0, 0, 0};
    const uint64_t tl = n % S;
    if (tl) {
        e = cudaMemcpy(tail, static_cast<const uint8_t*>(in) + (n - tl), tl, cudaMemcpyDefault);
        if (e != cudaSuccess) return cleanup(cuda_fail(err, e, "plzgpu_compress_multi tail"));
    }
    uint64_t img_len = 0;
    rc = plzgpu_shard_headers(ctx[0], &p, n, totals.data(), tail, d_img, image_len + 16, &img_len,
                              nullptr, err);
    if (rc) return cleanup(rc);
    e = cudaMemcpy(out, d_img, img_len, cudaMemcpyDefault);
    if (e != cudaSuccess) return cleanup(cuda_fail(err, e, "plzgpu_compress_multi output"));
    if (stats) {
        for (uint64_t r = 0; r < N; ++r) {
            unsigned long long st2[2] = {0, 0};
            cudaSetDevice(devices[r]);
            if (cudaMemcpy(st2, dmeta(ctx[r])->stats, sizeof st2, cudaMemcpyDeviceToHost) == cudaSuccess) {
                stats->pointer_tokens += st2[0];
                stats->literal_tokens += st2[1];
            }
        }
    }
    *out_len = img_len;
    return cleanup(PLZGPU_OK);
}


// One image decompressed by several GPUs of this process: rank r decodes the
// global chunk range r (plzgpu_decompress_range) on its own device, from a
// copy of the image there when the image is another device's memory, and
// its slice is copied to its offset in `out`.  The first failing rank's
// error is the single call's (ranks are in chunk order; header errors are
// every rank's).
int plzgpu_decompress_multi(const int* devices, int n_devices, const void* img, uint64_t len,
                            void* out, uint64_t cap, uint64_t* out_len, plzgpu_error* err) {
    clear_err(err);
    *out_len = 0;
    if (n_devices < 1 || !devices)
        return set_err(err, PLZGPU_CONTRACT, 0, kNoIndex, kNoIndex, "empty device list");
    if (len == 0) return PLZGPU_OK;
    const uint64_t N = uint64_t(n_devices);
    int img_dev = -1;
    {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, img) == cudaSuccess && at.type == cudaMemoryTypeDevice)
            img_dev = at.device;
        else
            cudaGetLastError();
    }
    std::vector<plzgpu_ctx*> ctx(N, nullptr);
    std::vector<void*> allocs;
    std::vector<int> alloc_dev;
    auto cleanup = [&](int code) {
        for (size_t i = 0; i < allocs.size(); ++i) {
            cudaSetDevice(alloc_dev[i]);
            cudaFree(allocs[i]);
        }
        for (plzgpu_ctx* c : ctx)
            if (c) plzgpu_ctx_destroy(c);
        return code;
    };
    for (uint64_t r = 0; r < N; ++r) {
        const int rc = plzgpu_ctx_create(devices[r], &ctx[r], err);
        if (rc) return cleanup(rc);
    }
    // the image each rank reads: the caller's (host, or on the rank's device)
    // or a copy on the rank's device
    std::vector<const void*> src(N, img);
    for (uint64_t r = 0; r < N; ++r) {
        if (img_dev < 0 || img_dev == devices[r]) continue;
        void* p = nullptr;
        cudaError_t e = cudaSetDevice(devices[r]);
        if (e == cudaSuccess) e = cudaMalloc(&p, len);
        if (e == cudaSuccess) {
            allocs.push_back(p);
            alloc_dev.push_back(devices[r]);
            e = cudaMemcpy(p, img, len, cudaMemcpyDefault);
        }
        if (e != cudaSuccess) return cleanup(cuda_fail(err, e, "plzgpu_decompress_multi image"));
        src[r] = p;
    }
    uint64_t b0 = 0, l0 = 0, total = 0;
    int rc = plzgpu_decompress_range(ctx[0], src[0], len, 0, 0, nullptr, 0, &b0, &l0, &total,
                                     nullptr, err);
    if (rc) return cleanup(rc);
    std::vector<int> rcs(N, PLZGPU_OK);
    std::vector<plzgpu_error> errs(N);
    std::vector<uint64_t> begin(N, 0), size(N, 0);
    std::vector<uint8_t*> slice(N, nullptr);
    std::mutex mu;  // allocation bookkeeping
    {
        std::vector<std::thread> th;
        for (uint64_t r = 0; r < N; ++r)
            th.emplace_back([&, r] {
                const uint64_t cb = total * r / N, ce = total * (r + 1) / N;
                uint64_t tc = 0;
                rcs[r] = plzgpu_decompress_range(ctx[r], src[r], len, cb, ce, nullptr, 0, &begin[r],
                                                 &size[r], &tc, nullptr, &errs[r]);
                if (rcs[r] || size[r] == 0) return;
                void* p = nullptr;
                cudaError_t e = cudaSetDevice(devices[r]);
                if (e == cudaSuccess) e = cudaMalloc(&p, size[r] + 16);
                if (e != cudaSuccess) {
                    rcs[r] = cuda_fail(&errs[r], e, "plzgpu_decompress_multi slice");
                    return;
                }
                {
                    std::lock_guard<std::mutex> lock(mu);
                    allocs.push_back(p);
                    alloc_dev.push_back(devices[r]);
                }
                slice[r] = static_cast<uint8_t*>(p);
                uint64_t b2 = 0, l2 = 0;
                rcs[r] = plzgpu_decompress_range(ctx[r], src[r], len, cb, ce, p, size[r] + 16, &b2,
                                                 &l2, &tc, nullptr, &errs[r]);
            });
        for (std::thread& t : th) t.join();
    }
    for (uint64_t r = 0; r < N; ++r)
        if (rcs[r]) {
            if (err) *err = errs[r];
            return cleanup(rcs[r]);
        }
    const uint64_t total_out = begin[N - 1] + size[N - 1];
    if (total_out > cap)
        return cleanup(set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                               "output buffer too small: need %llu bytes",
                               (unsigned long long)total_out));
    for (uint64_t r = 0; r < N; ++r)
        if (size[r]) {
            const cudaError_t e = cudaMemcpy(static_cast<uint8_t*>(out) + begin[r], slice[r], size[r],
                                             cudaMemcpyDefault);
            if (e != cudaSuccess) return cleanup(cuda_fail(err, e, "plzgpu_decompress_multi output"));
        }
    *out_len = total_out;
    return cleanup(PLZGPU_OK);
}

}  // extern "C"
