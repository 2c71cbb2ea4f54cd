/*
 * plzgpu.h — C-ABI drop-in boundary of the B200-native GPULZ path.
 *
 * The reference (`plz`, /root/reference/proj) exposes its compress /
 * decompress path as a C++ API.  This header is the
 * language-neutral boundary underneath the B200 re-implementation of that API
 * (include/plz/ headers): plain pointers and sizes, no torch or C++ types.
 * Each entry point names the reference interface it replaces.
 *
 * Buffers: every `in` / `img` / `out` pointer may be HOST memory (pageable or
 * pinned) or DEVICE memory on the context's GPU (cudaMalloc / torch CUDA
 * tensors).  Host buffers are staged through the context; device buffers are
 * used in place.  Streams are `cudaStream_t` passed as `void*`; NULL is the
 * legacy default stream (CUDA convention); plzgpu_ctx_stream() returns the
 * context's private non-blocking stream.
 *
 * Errors: functions return a plzgpu_status and, when `err` is non-NULL, fill
 * it.  Codes 1-4 correspond one-to-one to the reference's exception types
 * (errors.hpp:10-41); byte_offset / chunk_index / token_index carry the same
 * values the reference stores in plz::corruption_error.
 *
 * Threading: a context owns device scratch and one stream; use one context per
 * host thread.  Calls on distinct contexts may run concurrently.
 */
#ifndef PLZGPU_H
#define PLZGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLZGPU_ABI_VERSION 1

typedef enum plzgpu_status {
    PLZGPU_OK = 0,
    PLZGPU_VALIDATION = 1,          /* plz::validation_error        (errors.hpp:15) */
    PLZGPU_UNSUPPORTED_FORMAT = 2,  /* plz::unsupported_format_error (errors.hpp:20) */
    PLZGPU_CORRUPTION = 3,          /* plz::corruption_error         (errors.hpp:27) */
    PLZGPU_CONTRACT = 4,            /* plz::contract_error           (errors.hpp:39) */
    PLZGPU_CUDA = 5,                /* CUDA runtime failure (no reference equivalent) */
    PLZGPU_CAPACITY = 6             /* caller's output buffer too small */
} plzgpu_status;

/* plz::Params (params.hpp:18-25).  min_match is derived by plzgpu_validate. */
typedef struct plzgpu_params {
    int32_t symbol_width; /* S: 1, 2 or 4 */
    int32_t window;       /* W: 4..255 */
    int32_t chunk_size;   /* C: 1024..16384 symbols, power of two, > W */
    int32_t interval;     /* I: 1, 2, 4, 8, 16; divides C */
    uint64_t block_bytes; /* bytes per container; multiple of C*S */
    int32_t min_match;    /* derived: 2/S + 1 */
    int32_t reserved;
} plzgpu_params;

/* plz::PipelineStats (pipeline.hpp:14-18).  max_cmp_per_pos is an
 * instrumentation counter of the reference's CPU matcher; the GPU matcher
 * reports 0. */
typedef struct plzgpu_stats {
    uint64_t max_cmp_per_pos;
    uint64_t pointer_tokens;
    uint64_t literal_tokens;
} plzgpu_stats;

typedef struct plzgpu_error {
    int32_t code;
    int32_t reserved;
    uint64_t byte_offset; /* corruption_error::byte_offset (relative to the container) */
    uint64_t chunk_index; /* UINT64_MAX when not applicable */
    uint64_t token_index; /* UINT64_MAX when not applicable */
    char message[240];    /* the reference's what() text */
} plzgpu_error;

/* plz::BlockPlan (partition.hpp:14-20) */
typedef struct plzgpu_block_plan {
    uint64_t byte_start;
    uint64_t byte_len;
    uint32_t num_chunks;
    uint32_t last_chunk_len;
    uint8_t tail_len;
    uint8_t pad[7];
} plzgpu_block_plan;

typedef struct plzgpu_ctx plzgpu_ctx;

/* ------------------------------------------------------------ host-side */

int plzgpu_abi_version(void);

/* replaces plz::validate (params.hpp:30, params.cpp:19-45) */
int plzgpu_validate(const plzgpu_params* raw, plzgpu_params* out, plzgpu_error* err);

/* replaces plz::level_to_window (params.hpp:33, params.cpp:47-55) */
int plzgpu_level_to_window(int level, int32_t* window, plzgpu_error* err);

/* replaces plz::plan (partition.hpp:28, partition.cpp:5-25).  Writes up to
 * max_blocks entries and returns the total block count. */
uint64_t plzgpu_plan(uint64_t total_bytes, const plzgpu_params* params,
                     plzgpu_block_plan* blocks, uint64_t max_blocks);

/* replaces plz::container_size (format.hpp:53-54, format.cpp:69-73) */
uint64_t plzgpu_container_size(uint32_t num_chunks, uint64_t flag_total,
                               uint64_t payload_total, uint8_t tail_len);

/* Worst-case image size for n input bytes (every chunk all-literal).  An
 * output buffer of this size never overflows. */
uint64_t plzgpu_compress_bound(uint64_t n, const plzgpu_params* params);

/* Host walk of a HOST image with read_container's checks (format.cpp:112-185):
 * the decoded size of the longest prefix of containers that parse.  Sizes the
 * output of plzgpu_decompress; the errors themselves come from decompress. */
uint64_t plzgpu_decompressed_bound(const void* host_img, uint64_t len);

/* -------------------------------------------------------------- device */

int plzgpu_ctx_create(int device, plzgpu_ctx** out, plzgpu_error* err);
void plzgpu_ctx_destroy(plzgpu_ctx* ctx);
/* the context's stream as cudaStream_t */
void* plzgpu_ctx_stream(plzgpu_ctx* ctx);
/* number of kernels the last compress / decompress enqueued */
int plzgpu_ctx_last_launches(plzgpu_ctx* ctx);

/* Same quantity for a host OR device image (device: the parse kernel runs
 * and one small result is read back). */
int plzgpu_decompressed_size(plzgpu_ctx* ctx, const void* img, uint64_t len, uint64_t* out_len,
                             void* stream, plzgpu_error* err);

/* replaces plz::compress (pipeline.hpp:28-30, pipeline.cpp:88-99).
 * Writes the bit-exact .plz image to out[0..*out_len).  Synchronous. */
int plzgpu_compress(plzgpu_ctx* ctx, const plzgpu_params* params, const void* in,
                    uint64_t n, void* out, uint64_t cap, uint64_t* out_len,
                    plzgpu_stats* stats, void* stream, plzgpu_error* err);

/* Stream-ordered variant for device-resident data: d_in and d_out are device
 * pointers, cap >= plzgpu_compress_bound(n); the image length lands in the
 * device word *d_out_len.  Returns after enqueueing; device-detected errors
 * (4-byte table overflow) are reported by plzgpu_ctx_finish. */
int plzgpu_compress_async(plzgpu_ctx* ctx, const plzgpu_params* params, const void* d_in,
                          uint64_t n, void* d_out, uint64_t cap, uint64_t* d_out_len,
                          void* stream, plzgpu_error* err);

/* replaces plz::decompress_bytes (decoder.hpp:42-43, decoder.cpp:129-141).
 * Synchronous. */
int plzgpu_decompress(plzgpu_ctx* ctx, const void* img, uint64_t len, void* out,
                      uint64_t cap, uint64_t* out_len, void* stream, plzgpu_error* err);

/* Decodes the global chunks [chunk_begin, chunk_end) of an image (chunk
 * index space of the whole container chain, as plzgpu_num_chunks counts it
 * for the input) — one rank's share of a sharded decompress (SURVEY.md §8e:
 * "decompress shards the same way ... by chunk range using the tables").
 * `out` receives decompressed bytes [*out_begin, *out_begin + *out_len):
 * start(chunk_begin) to start(chunk_end), where start(g) is chunk g's output
 * offset, start(0) = 0 and start(total) = the decompressed size, so
 * consecutive ranges partition the output (tails included where their bytes
 * fall).  *total_chunks reports the image's chunk count (call with an empty
 * range to learn it).  Every container header is checked (decoder order);
 * token errors are those of the range's chunks.  Ranges past the end are
 * clamped.  out = NULL: only the three sizes, nothing decoded.  Replaces nothing in the reference (its decoder is one process);
 * the per-rank entry point of dist.decompress_sharded. */
int plzgpu_decompress_range(plzgpu_ctx* ctx, const void* img, uint64_t len, uint64_t chunk_begin,
                            uint64_t chunk_end, void* out, uint64_t cap, uint64_t* out_begin,
                            uint64_t* out_len, uint64_t* total_chunks, void* stream,
                            plzgpu_error* err);

/* One stream compressed by several GPUs of this process (SURVEY.md §8b item
 * 4: "a multi-GPU variant taking a device list"): chunk ranges encoded
 * concurrently (one pooled context and host thread per entry of `devices`;
 * an entry may repeat a device), each rank's Kernel III writing its segments
 * straight into the image on devices[0] through peer access (NVLink), the
 * headers written there, then the image to `out` (host or device; a device
 * `out` on devices[0] is written in place).  The image equals
 * plzgpu_compress's.  Contexts and scratch persist across calls (per device,
 * process-wide pool); the caller's current device is preserved.  A device
 * `in` must be complete when the call starts (the ranks run on their own
 * streams): synchronize the stream that wrote it first.  Replaces
 * plz::compress (pipeline.hpp:28-30) for a device list; the
 * one-process-per-GPU form is dist.compress_sharded. */
int plzgpu_compress_multi(const int* devices, int n_devices, const plzgpu_params* params,
                          const void* in, uint64_t n, void* out, uint64_t cap, uint64_t* out_len,
                          plzgpu_stats* stats, plzgpu_error* err);

/* One image decompressed by several GPUs of this process: rank r decodes the
 * global chunk range r (plzgpu_decompress_range) on devices[r]; with a
 * device `out` its slice is decoded straight into `out` at its offset
 * (peer stores), with a host `out` it is copied there from rank r's GPU.
 * Output and errors equal plzgpu_decompress's.  Same pooling, device and
 * ordering rules as plzgpu_compress_multi. */
int plzgpu_decompress_multi(const int* devices, int n_devices, const void* img, uint64_t len,
                            void* out, uint64_t cap, uint64_t* out_len, plzgpu_error* err);

/* Stream-ordered variant: device image and output; the decoded length lands
 * in *d_out_len.  Errors are reported by plzgpu_ctx_finish. */
int plzgpu_decompress_async(plzgpu_ctx* ctx, const void* d_img, uint64_t len, void* d_out,
                            uint64_t cap, uint64_t* d_out_len, void* stream,
                            plzgpu_error* err);

/* Waits for the context's last async operation on `stream` and reports its
 * device-side errors (and, after a compress, its stats). */
int plzgpu_ctx_finish(plzgpu_ctx* ctx, void* stream, plzgpu_stats* stats, plzgpu_error* err);

/* replaces plz::decompress_chunk (decoder.hpp:25-28, decoder.cpp:70-90):
 * decodes one chunk's flag/payload slices (host or device memory) into
 * out[0 .. logical_len*S). */
int plzgpu_decompress_chunk(plzgpu_ctx* ctx, const void* flags, uint64_t n_flags,
                            const void* payload, uint64_t n_payload, uint64_t logical_len,
                            const plzgpu_params* params, uint64_t chunk_index, void* out,
                            plzgpu_error* err);

/* ---------------------------------------------------- multi-GPU shards */
/* SURVEY.md §8e.  Chunks are independent, so any contiguous chunk range of
 * the input's partition compresses on its own GPU; ranks then agree on
 * per-container stream totals (a few u64 over NCCL), each writes the table
 * and stream slices it owns as image segments, and the root gathers them and
 * writes the container headers.  The gathered image equals plzgpu_compress of
 * the whole input, byte for byte. */

/* chunk / container counts of the partition of n input bytes */
uint64_t plzgpu_num_chunks(uint64_t n, const plzgpu_params* params);
uint64_t plzgpu_num_containers(uint64_t n, const plzgpu_params* params);

/* Kernels I+II over chunks [chunk_begin, chunk_end) of an n_total-byte input.
 * `in` (host or device) points at byte chunk_begin*C*S of the input and
 * holds the range's bytes (for the final range: through the end of the
 * input, tail included).  totals receives, per container the range touches
 * (in order), {container index, payload bytes, flag bytes}.  The context keeps
 * the encoded range for plzgpu_shard_assemble. */
int plzgpu_shard_encode(plzgpu_ctx* ctx, const plzgpu_params* params, const void* in,
                        uint64_t n_total, uint64_t chunk_begin, uint64_t chunk_end,
                        uint64_t* totals, uint64_t max_touched, uint64_t* n_touched, void* stream,
                        plzgpu_error* err);

/* Host arithmetic: the image segments {image_offset, local_offset, length}
 * (4 per touched container: payload-table slice, flag-table slice, flag
 * bytes, payload bytes) of a shard, given its totals and, per touched
 * container, bases = {payload_base, flag_base, container image offset,
 * container flag total}.  Returns the segment count. */
uint64_t plzgpu_shard_segments(const plzgpu_params* params, uint64_t n_total, uint64_t chunk_begin,
                               uint64_t chunk_end, const uint64_t* totals, const uint64_t* bases,
                               uint64_t n_touched, uint64_t* segs, uint64_t max_segs);

/* Write the last plzgpu_shard_encode's segments into d_out (device), laid
 * out back to back in segment order; segs as plzgpu_shard_segments. */
int plzgpu_shard_assemble(plzgpu_ctx* ctx, const uint64_t* bases, void* d_out, uint64_t cap,
                          uint64_t* segs, uint64_t max_segs, uint64_t* n_segs, uint64_t* out_len,
                          void* stream, plzgpu_error* err);

/* The same segments written straight to their offsets in the final image
 * d_img (img_cap bytes; device memory of this context's GPU or, with peer
 * access enabled, of another GPU: Kernel III then stores over NVLink and
 * nothing is gathered afterwards). */
int plzgpu_shard_assemble_into(plzgpu_ctx* ctx, const uint64_t* bases, void* d_img,
                               uint64_t img_cap, void* stream, plzgpu_error* err);

/* Root: write every container's header, final table entries and tail into
 * d_img given per-container {payload total, flag total} for ALL containers and
 * the input's last tail_len (< S) bytes (host).  *img_len = image length. */
int plzgpu_shard_headers(plzgpu_ctx* ctx, const plzgpu_params* params, uint64_t n_total,
                         const uint64_t* totals, const void* tail, void* d_img, uint64_t cap,
                         uint64_t* img_len, void* stream, plzgpu_error* err);

/* ------------------------------------------------ statistics / matcher */

/* replaces plz::match_chunk (matcher.hpp:49-50, matcher.cpp:113-131) over a
 * whole input: len_out/off_out (host or device, n/S entries) receive the
 * record of every symbol of every chunk (chunk g's symbol i at g*C + i):
 * interval-aligned positions hold the longest match (ties to the largest
 * offset, {0,0} for none), others the forced literal {1,0}.  raw_hist (host,
 * 256 u64, may be NULL) tallies the lengths of records with offset != 0
 * (match_length_histogram raw mode, corpus.cpp:199-204). */
int plzgpu_match_table(plzgpu_ctx* ctx, const plzgpu_params* params, const void* in, uint64_t n,
                       void* len_out, void* off_out, uint64_t* raw_hist, void* stream,
                       plzgpu_error* err);

/* Lengths of the pointer tokens compress would emit (corpus.cpp:205-217,
 * match_length_histogram encoded mode): hist[len] counts, 256 u64 (host). */
int plzgpu_pointer_histogram(plzgpu_ctx* ctx, const plzgpu_params* params, const void* in,
                             uint64_t n, uint64_t* hist, void* stream, plzgpu_error* err);

/* ------------------------------------------------------ profiling hook */

/* Enqueue Kernel I (match + encode) alone on a device input, so its share of
 * a compress can be timed with CUDA events (bench.py roofline).  No image is
 * produced. */
int plzgpu_profile_encode(plzgpu_ctx* ctx, const plzgpu_params* params, const void* d_in,
                          uint64_t n, void* stream, plzgpu_error* err);

/* Per-stage CUDA-event times of a device-resident compress (bench.py's
 * per-kernel rooflines): ms[0] Kernel I (match + encode), ms[1] Kernel II
 * (global scan), ms[2] Kernel III + headers (deflate / container assembly),
 * each the mean over `steps` compresses of `d_in` into `d_img` (capacity
 * `cap` >= plzgpu_compress_bound).  The image is complete after the call. */
int plzgpu_profile_stages(plzgpu_ctx* ctx, const plzgpu_params* params, const void* d_in,
                          uint64_t n, void* d_img, uint64_t cap, int steps, double* ms,
                          void* stream, plzgpu_error* err);

/* Measured int32 lane-op throughput of `device` (lane operations per
 * second): op 0 = LOP3, 1 = IADD, 2 = SHF (funnel shift), 3 = POPC + IADD.
 * The denominator of the matching kernel's integer roofline (SURVEY.md
 * §8d); runs two short launches on the device's legacy stream. */
int plzgpu_int_peak(int device, int op, double* lane_ops_per_s, plzgpu_error* err);

/* ---------------------------------- cuSZ dual quantization (use case) */

/* The producer of the quantization codes GPULZ compresses in the paper's
 * improved cuSZ (PAPER.md "Use-case of gpuLZ", Table 3; no counterpart in
 * the reference library).  Device buffers only; enqueued on `stream`.
 *   q    = rint(f * s), s = float32(1 / (2 eb))        (round half to even)
 *   d    = Lorenzo residual Δx Δy Δz q, q = 0 outside  (x fastest; ny/nz = 1
 *          give 2-D / 1-D)
 *   code = d + radius if |d| < radius, else 0          (u16; radius <= 32768)
 * Outliers (code 0) are listed as (index, d) in index order; *n_outliers (a
 * host word) receives their count — the call synchronises on `stream` for
 * it.  More than outlier_cap outliers -> PLZGPU_CAPACITY (the list is
 * truncated; *n_outliers still holds the full count). */
int plzgpu_lorenzo_quantize(plzgpu_ctx* ctx, const float* d_field, uint64_t nx, uint64_t ny,
                            uint64_t nz, double eb, int32_t radius, uint16_t* d_codes,
                            uint64_t* d_outlier_idx, int32_t* d_outlier_val, uint64_t outlier_cap,
                            uint64_t* n_outliers, void* stream, plzgpu_error* err);

/* Inverse: codes + outliers -> f' = float32(Σx Σy Σz d) * float32(2 eb),
 * |f - f'| <= eb up to float32 rounding.  Enqueued on `stream`. */
int plzgpu_lorenzo_reconstruct(plzgpu_ctx* ctx, const uint16_t* d_codes,
                               const uint64_t* d_outlier_idx, const int32_t* d_outlier_val,
                               uint64_t n_outliers, uint64_t nx, uint64_t ny, uint64_t nz,
                               double eb, int32_t radius, float* d_field, void* stream,
                               plzgpu_error* err);

#ifdef __cplusplus
}
#endif
#endif /* PLZGPU_H */
