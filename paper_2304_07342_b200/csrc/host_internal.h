// host_internal.h — shared pieces of the C-ABI implementation (include/plzgpu.h).
//
// The host side is split by concern:
//   host_common.cpp    errors, parameter checks, geometry, pipeline config, driver entry points
//   context.cpp        plzgpu_ctx lifetime, kernel preload, ctx_finish
//   api_params.cpp     validate / level_to_window / plan / bounds (pure host arithmetic)
//   compress.cpp       Kernels I-III enqueue, plzgpu_compress[_async], profiling hook
//   decompress.cpp     parse + decode enqueue, plzgpu_decompress[_range|_async|_chunk]
//   host_pipeline.cpp  host-buffer paths: H2D segments with ready flags, per-container
//                      assembly + D2H, pipelined host-image decode
//   shards.cpp         chunk-range shard protocol (plzgpu_shard_*)
//   multi.cpp          one stream over a device list (plzgpu_compress_multi / _decompress_multi)
//   stats.cpp          match table / pointer histogram
//   cusz_host.cpp      cuSZ dual-quantization entry points
//
// Reference behaviour mirrored (paths under /root/reference/proj):
//   params.cpp:19-55     validation order and messages, min_match = 2/S + 1
//   partition.cpp:5-25   blocks of block_bytes, C-symbol chunks, raw tail
//   pipeline.cpp:88-99   image = containers back to back; empty input -> empty
//   scan.cpp:43-44       4-byte table overflow -> validation_error
//   format.cpp:112-185   read_container messages / byte offsets
//   decoder.cpp:13-18    "corrupt chunk K, token T: what"
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/plzgpu.h"
#include "kernels.h"

namespace plzhost {

using namespace plzgpu;

constexpr uint64_t kNoIndex = UINT64_MAX;

// ------------------------------------------------------------------ errors
int set_err(plzgpu_error* e, int code, uint64_t off, uint64_t chunk, uint64_t tok, const char* fmt,
            ...);
void clear_err(plzgpu_error* e);
int cuda_fail(plzgpu_error* e, cudaError_t c, const char* where);
int bad_field(plzgpu_error* e, const char* field, const char* legal);
int overflow_error(plzgpu_error* err);
int corrupt(plzgpu_error* e, const std::string& what, uint64_t off);
int parse_error(const ParseResult& r, plzgpu_error* err);
int token_error(uint32_t code, uint64_t chunk, uint64_t token, plzgpu_error* err);

#define CK(call)                                                     \
    do {                                                             \
        const cudaError_t ck_ = (call);                              \
        if (ck_ != cudaSuccess) return cuda_fail(err, ck_, #call);   \
    } while (0)

// params.cpp:19-45, same order, same messages
int validate_fields(const plzgpu_params& p, plzgpu_error* e);

// Whole-input chunk geometry (partition.cpp:5-25 folded over all blocks).
struct Geometry {
    uint64_t n_bytes = 0, n_blocks = 0, cpb = 0, n_chunks = 0;
    uint32_t last_len = 0;
};
Geometry geometry(uint64_t n, const plzgpu_params& p);

// ------------------------------------------------------- pipeline config
// Every tuning knob of the host-buffer paths, read from the environment
// once per process (PLZGPU_*; unset in normal use — they exist for A/B
// measurements and for profilers, which serialise the copies the
// overlapped paths' kernels wait on).
struct PipelineConfig {
    bool no_pipe = false;         // PLZGPU_NO_PIPE: no overlapped host paths at all
    bool no_pipe_asm = false;     // PLZGPU_NO_PIPE_ASM: host compress assembles the whole image
    bool no_pipe_dec = false;     // PLZGPU_NO_PIPE_DEC: host decompress via the resident path
    bool asm_mapped = false;      // PLZGPU_ASM_MAPPED: Kernel III writes the mapped host image
    uint64_t seg_bytes = 32u << 20;   // PLZGPU_SEG_MB: compress ready-flag granularity
    uint64_t copy_bytes = 32u << 20;  // PLZGPU_COPY_MB: compress H2D copy size
    uint64_t tail_bytes = 0;          // PLZGPU_TAIL_MB: last stretch sent flag segment by segment
    uint64_t dseg_in = 16u << 20;     // PLZGPU_DSEG_IN_MB: decompress image segment
    uint64_t dseg_out = 32u << 20;    // PLZGPU_DSEG_OUT_MB: decompress output segment
    uint64_t dseg_lead = 1;           // PLZGPU_DSEG_LEAD: single-segment transfers first
    uint64_t dseg_group = 1;          // PLZGPU_DSEG_GROUP: segments per later H2D transfer
    uint64_t dseg_group_out = 1;      // PLZGPU_DSEG_GROUP_OUT: segments per later D2H transfer
    uint64_t pageable_stage = 64u << 20;  // PLZGPU_PAGEABLE_MB: one pinned bounce slot
    uint64_t pageable_min = 64u << 20;    // PLZGPU_PAGEABLE_MIN_MB: staged copies from this size on
    int copy_threads = 0;                 // PLZGPU_COPY_THREADS: host copy workers (0: cores - 1, <= 15)
    int asm_mode = 2;                     // PLZGPU_ASM_MODE: Kernel III 0 register-staged, 1 TMA ring, 2 batched runs
};
const PipelineConfig& pipeline_config();

// ------------------------------------------------------- driver entry points
// cuStreamWriteValue32 / cuStreamWaitValue32 through the runtime's driver
// entry point (no link-time libcuda dependency: the library must also load on
// GPU-less hosts).
typedef int (*StreamValue32Fn)(void* stream, unsigned long long addr, uint32_t value,
                               unsigned int flags);
StreamValue32Fn stream_write_value32();
StreamValue32Fn stream_wait_value32();  // flags 0 = CU_STREAM_WAIT_VALUE_GEQ

bool is_pinned_host(const void* p);
bool is_device_ptr(const void* p);
inline uint32_t host_le32(const uint8_t* b) {
    return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
}
// Ready-flag epochs are drawn from one process-wide counter, so flags left in
// a recycled allocation by another context can never equal a live epoch.
uint32_t next_epoch();

// Restores the calling thread's current device on scope exit (entry points
// switch to their context's device; the caller's device must not change).
struct DeviceGuard {
    int saved = -1;
    DeviceGuard() {
        if (cudaGetDevice(&saved) != cudaSuccess) {
            (void)cudaGetLastError();
            saved = -1;
        }
    }
    ~DeviceGuard() {
        if (saved >= 0) cudaSetDevice(saved);
    }
};

// --------------------------------------------------------------- scratch
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    // grows (never shrinks); *fresh tells the caller the bytes are new
    cudaError_t ensure(size_t bytes, bool* fresh = nullptr) {
        if (fresh) *fresh = false;
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        size_t want = std::max(bytes, cap + cap / 2);
        want = (want + 255) & ~size_t(255);
        const cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) {
            cap = want;
            if (fresh) *fresh = true;
        }
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
    uint32_t work[12];  // [0] first bitmap pass, [1] scan tiles, [2]/[3]/[4] the decode kernels,
                        // [4]/[6]/[8] overflow counts of the bitmap passes, [5]/[9]
                        // second/third bitmap pass, [7] wide pass
    uint32_t stalled;  // H2D pipeline: a segment never arrived
    uint32_t pad;
    uint32_t lat_count[8];  // latency mode: chunks per tier list (tiny, 16, 32, 64, wide, spill)
    uint32_t lat_work[8];   // latency mode: the tier kernels' work counters
    uint64_t range[3];  // plzgpu_decompress_range: output range, total chunks
    ParseResult parse;
};

enum LastOp { OP_NONE, OP_COMPRESS, OP_DECOMPRESS };

}  // namespace plzhost

struct plzgpu_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    plzhost::DevBuf in, img, out, pay_slots, flag_slots, psize, fsize, p64, f64, status, agg, incl,
        desc;
    plzhost::DevBuf meta;
    plzhost::Meta* host_meta = nullptr;  // pinned
    int last_launches = 0;
    plzhost::LastOp last_op = plzhost::OP_NONE;
    plzgpu::DecodeArgs last_decode{};
    int enc_wpc[4096] = {};  // launch shape cache per (pass, S, C)
    int enc_ctas[4096] = {};
    plzhost::DevBuf fb;          // overflow lists of the bitmap passes (3 x G chunk indices)
    plzhost::DevBuf shard_desc;  // ShardCont / HeaderDesc upload area
    // H2D pipeline of host inputs (plzgpu_compress): segment ready flags
    cudaStream_t copy_stream = nullptr;
    cudaStream_t asm_stream = nullptr;   // pipelined compress: per-container Kernel III
    cudaStream_t side_stream = nullptr;  // Kernel I: the 64-row pass beside the 32-row one
    cudaEvent_t side_ev[2] = {nullptr, nullptr};
    cudaStream_t lat_stream[4] = {nullptr, nullptr, nullptr, nullptr};  // latency-mode tiers
    cudaEvent_t lat_ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t asm_ev[2] = {nullptr, nullptr};
    // pipelined compress into pinned host memory: per container, its scan
    // and its assembly done; the image goes down on d2h_stream, the
    // container sizes that place it come back on size_stream
    std::vector<cudaEvent_t> cont_ev;
    cudaStream_t d2h_stream = nullptr, size_stream = nullptr;
    uint64_t* host_scratch = nullptr;  // pinned, 4 words
    plzhost::DevBuf ready, done;
    uint32_t epoch = 0;
    const uint32_t* pipe_ready = nullptr;  // set while enqueueing a pipelined encode
    uint32_t pipe_seg_chunks = 0;
    unsigned long long* enc_hist = nullptr;  // set while enqueueing a histogram encode
    plzhost::DevBuf hist, table;
    plzhost::DevBuf qtiles, qoff, qdelta;  // cuSZ quantizer scratch
    // pageable host buffers: pinned bounce slots (staged copies)
    uint8_t* bounce[3] = {nullptr, nullptr, nullptr};
    size_t bounce_cap = 0;
    cudaEvent_t bounce_ev[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t order_ev = nullptr;
    // last plzgpu_shard_encode: the range and its per-container local totals
    uint64_t sh_begin = 0, sh_end = 0, sh_n = 0;
    plzgpu_params sh_params{};
    std::vector<uint64_t> sh_touch;  // per touched container: {j, lo, hi, P, F}
};

namespace plzhost {

// NULL selects the legacy default stream (the CUDA convention, so callers
// passing torch's default stream handle 0 stay ordered with it).
inline cudaStream_t pick(plzgpu_ctx*, void* s) { return static_cast<cudaStream_t>(s); }
inline Meta* dmeta(plzgpu_ctx* c) { return c->meta.as<Meta>(); }

void preload_kernels(int device);

// compress.cpp
int enqueue_encode_scan(plzgpu_ctx* c, const plzgpu_params& p, const uint8_t* d_in, uint64_t G,
                        uint32_t last_len, cudaStream_t st, plzgpu_error* err, int* launches,
                        bool scan = true, uint64_t g0 = 0, uint64_t g1 = UINT64_MAX,
                        bool side_passes = true);
void fill_assemble_args(plzgpu_ctx* c, const plzgpu_params& p, const Geometry& g,
                        const uint8_t* d_in, uint8_t* img, uint64_t* d_img_len, AssembleArgs* a);
int enqueue_compress(plzgpu_ctx* c, const plzgpu_params& p, const uint8_t* d_in, uint64_t n,
                     uint8_t* img, uint64_t* d_img_len, cudaStream_t st, plzgpu_error* err,
                     int last_stage = 3);
// host_pipeline.cpp
int compress_host_input(plzgpu_ctx* c, const plzgpu_params& p, const uint8_t* in, uint64_t n,
                        uint8_t* out, uint64_t cap, uint8_t** img_out, bool* direct_out,
                        cudaStream_t st, plzgpu_error* err);
int try_decompress_pipelined(plzgpu_ctx* c, const uint8_t* img, uint64_t len, uint8_t* out,
                             uint64_t cap, uint64_t* out_len, cudaStream_t st, plzgpu_error* err);
// Pageable host memory <-> device through the context's pinned bounce slots
// (staging.cpp): a process-wide pool of host threads copies between the
// caller's pages and one slot while the copy engine moves another (a plain
// cudaMemcpy of pageable memory goes through the driver's own
// single-threaded staging, ~10 GB/s).  The DMAs run on c->copy_stream.
//  h2d: after_st orders the copies after the work already on st.  With
//       `ready`, each slot's DMA is followed by the ready flags (= epoch) of
//       the seg_bytes segments it completes, for kernels already waiting on
//       them; without, st waits for the copies.  Returns once every DMA is
//       enqueued.
//  d2h: after the work on st; returns once h_dst holds the bytes.
bool use_staged(const void* host_ptr, uint64_t n);  // pageable and large enough
int h2d_pageable(plzgpu_ctx* c, uint8_t* d_dst, const uint8_t* h_src, uint64_t n,
                 cudaStream_t st, bool after_st, const uint32_t* ready, uint64_t seg_bytes,
                 uint32_t epoch, plzgpu_error* err);
int d2h_pageable(plzgpu_ctx* c, uint8_t* h_dst, const uint8_t* d_src, uint64_t n, cudaStream_t st,
                 plzgpu_error* err);
// memcpy between host buffers split over the copy pool's threads
void pool_memcpy(void* dst, const void* src, size_t n);
// decompress.cpp
int enqueue_decompress(plzgpu_ctx* c, const uint8_t* d_img, uint64_t len, uint8_t* d_out,
                       uint64_t cap, uint64_t* d_out_len, cudaStream_t st, plzgpu_error* err);
int finish_decompress(plzgpu_ctx* c, cudaStream_t st, bool* grow, plzgpu_error* err);

}  // namespace plzhost
