// kernels.h — host-visible launchers and argument blocks of the sm_100a kernels.
//
//   Kernel I   plz_bitmatch_kernel<S,NW> match + greedy token walk + encode, one warp per chunk
//              plz_encode_kernel<S>     the same for chunks with a large alphabet (wide cells)
//   Kernel II  plz_scan_kernel          decoupled look-back exclusive scan of (payload, flag) sizes
//   Kernel III plz_assemble_kernel      tables + flag/payload streams into the image (128-bit stores)
//              plz_headers_kernel       container headers, last table entries, tails, image length
//   Decode     plz_parse_kernel         container-chain walk with the reference's checks
//              plz_decode_kernel        block-parallel chunk decode, one warp per chunk
//              plz_decode_one_kernel    single-chunk decode (decompress_chunk / error details)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace plzgpu {

// Device-side error codes of token walks (decoder.cpp:22-66 order).
enum TokenErr : uint32_t {
    TE_OK = 0,
    TE_FLAGS_EXHAUSTED = 1,
    TE_PAYLOAD_EXHAUSTED = 2,
    TE_ZERO_FIELD = 3,
    TE_OFFSET_BEFORE_START = 4,
    TE_OVERRUN = 5,
    TE_TRAILING_PAYLOAD = 6,
    TE_NONZERO_PADDING = 7,
    TE_FLAG_COUNT = 8,
};

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;  // chunks per look-back tile

// Per-warp shared-memory bytes of the encode kernel for chunk size C, width S:
// C (symbol, run) cells of 2S bytes (the raw chunk is staged in their upper
// half), a kEncodeHeadPerS*S-byte payload head (the rest of the payload
// spills into dead cells), C/8 flag bytes, a 256-byte continuation list and
// an mbarrier.
constexpr uint32_t kEncodeHeadPerS = 512;  // >= 2*W + 1 for W <= 255
__host__ __device__ inline size_t encode_warp_smem(int C, int S) {
    // + 64 cells of slack: the last partial round of pair candidates may read
    // (and discard) up to 62 cells past the chunk end
    size_t b = size_t(C) * 2 * S + size_t(kEncodeHeadPerS) * S + size_t(C) / 8 + 256 + 16 + 128 * S;
    return (b + 15) & ~size_t(15);
}

// Bitmap passes of Kernel I (bitmatch.cu): chunks with at most kBmMaxSyms
// (then kBmMaxSymsWide) distinct symbols.  Per warp:
//   [mbarrier 16][id hash table: 2*maxsyms x {key, id} u32 pairs]
//   [region: max(C*S, C + rows) + 16 bytes]
// The region first holds the raw chunk (TMA target); pass 1 renames the
// symbols to ids in place (bytes [0, C), then D up to byte n + 127); pass 2
// builds the occurrence rows at byte C + 128, over the raw bytes pass 1 has
// consumed.  Rows are strided by
// C/32 + NW words: row r's word w (w counts NW front words, then the C-bit
// bitmap) is rows[r * stride + w], so a row's front words are the previous
// row's tail.  Those reads only ever feed candidate bits the search masks
// out (w < 0 is cleared from A, bits past position n-1 fail the o >= j+1
// mask), so their content is irrelevant — except for row D, the all-zero
// row standing for position n, which is zeroed over its whole reach (front
// NW words, bitmap, NW + 3 words behind: the search's one-round look-ahead).
constexpr int kBmMaxSymsTiny = 4;   // latency mode: chunks with at most 4 symbols
constexpr int kBmMaxSyms = 12;      // first bitmap pass: all chunks (12 rows: 36 warps/SM at c5)
constexpr int kBmMaxSymsMid = 32;   // second bitmap pass: the first pass's overflow
constexpr int kBmMaxSymsWide = 64;  // third bitmap pass: the second pass's overflow
constexpr int kBmMaxThreads = 128;   // CTA size bound (registers: up to 255 per thread)
__host__ __device__ inline int bm_nw(int W) { return W <= 32 ? 1 : W <= 64 ? 2 : W <= 128 ? 4 : 8; }
__host__ __device__ inline int bm_row_words(int C, int W) { return C / 32 + bm_nw(W); }  // stride
__host__ __device__ inline int bm_rows_words(int C, int W, int D) {  // rows 0..D, row D's reach
    return (D + 1) * bm_row_words(C, W) + bm_nw(W) + 3;
}
constexpr int kBmIdPad = 128;  // ids[n .. n+127] = D: the search reads ids unclamped
__host__ __device__ inline size_t bm_region(int C, int S, int W, int maxsyms) {
    const size_t raw = size_t(C) * S;
    const size_t rows = size_t(C) + kBmIdPad + size_t(bm_rows_words(C, W, maxsyms)) * 4;
    return (raw > rows ? raw : rows) + 16;
}
// renaming hash table: a power of two >= 2 * maxsyms slots (load factor <= 1/2)
__host__ __device__ constexpr int bm_hash_slots(int maxsyms) {
    return maxsyms <= 4 ? 8 : maxsyms <= 8 ? 16 : maxsyms <= 16 ? 32 : maxsyms <= 32 ? 64 : 128;
}
__host__ __device__ inline size_t bm_warp_smem(int C, int S, int W, int maxsyms) {
    const size_t b = 16 + size_t(bm_hash_slots(maxsyms)) * 8 + bm_region(C, S, W, maxsyms);
    return (b + 15) & ~size_t(15);
}

struct EncodeArgs {
    const uint8_t* in;           // byte 0 of global chunk 0
    uint8_t* pay_slots;          // chunk g payload staged at g * C * S
    uint8_t* flag_slots;         // chunk g flags staged at g * C / 8
    uint32_t* psize;             // per-chunk payload bytes
    uint32_t* fsize;             // per-chunk flag bytes
    unsigned long long* stats;   // [0] pointer tokens, [1] literal tokens
    uint32_t* work;              // dynamic chunk counter (zeroed before launch)
    uint64_t n_chunks;           // global chunk count
    uint32_t last_len;           // logical symbols of global chunk n_chunks-1
    int C, W, I, min_match;
    int bulk_ok;                 // input base 16B-aligned: TMA bulk loads allowed
    int warps_per_cta;
    // optional H2D pipeline: chunk g may be read once ready[g / seg_chunks]
    // == epoch (written by a stream memory operation after its segment's copy)
    const uint32_t* ready;
    uint32_t epoch;
    uint32_t seg_chunks;
    uint32_t* stalled;           // set if a segment never arrives (bounded wait)
    unsigned long long* hist;    // optional: selected pointer lengths [256]
    // chunk source: src_list[0..*src_count) when src_list is set (the passes
    // after the first), else chunks 0..n_chunks-1
    const uint32_t* src_list;
    const uint32_t* src_count;
    // bitmap passes: chunks whose alphabet does not fit are appended to
    // fb_list[c]: c = 0 (<= kBmMaxSymsMid symbols), 1 (<= kBmMaxSymsWide),
    // 2 (more).  The first pass classifies its overflow exactly; the later
    // passes only ever use fb_list[2].
    uint32_t* fb_list[3];
    uint32_t* fb_count[3];
    int classify;                // first pass: sort its overflow by alphabet size (else list 0)
};
// the wide-cell kernel (any alphabet)
cudaError_t launch_encode(int S, const EncodeArgs& a, int grid, cudaStream_t st);
// the bitmap kernel (bitmatch.cu): chunks with <= maxsyms distinct symbols
// (maxsyms = kBmMaxSyms, kBmMaxSymsMid or kBmMaxSymsWide)
cudaError_t launch_bitmatch(int S, int maxsyms, const EncodeArgs& a, int grid, cudaStream_t st);
int bitmatch_ctas_per_sm(int S, int C, int W, int maxsyms, int warps_per_cta);
// Latency mode (inputs of a few waves of chunks): every chunk's alphabet is
// counted first and the chunk listed for the smallest tier that holds it —
// lists[k * stride + i], k = 0 (<= kBmMaxSymsTiny symbols), 1 (<= kBmMaxSyms),
// 2 (<= kBmMaxSymsMid), 3 (<= kBmMaxSymsWide), 4 (more: the wide-cell pass),
// counts[k] — so all tiers can run at once instead of one after the other.
void launch_classify(int S, const EncodeArgs& a, uint32_t* lists, uint64_t stride, uint32_t* counts,
                     int grid, cudaStream_t st);
// full per-position match table (I-aligned searched, else {1,0}); optional raw histogram
void launch_match_table(int S, const EncodeArgs& a, int grid, uint8_t* len_out, uint8_t* off_out,
                        unsigned long long* raw_hist, cudaStream_t st);
int encode_ctas_per_sm(int S, int C, int warps_per_cta);

struct ScanArgs {
    const uint32_t* psize;
    const uint32_t* fsize;
    uint64_t n;                  // chunk count
    uint64_t* P64;               // n+1 exclusive prefixes of payload sizes
    uint64_t* F64;               // n+1 exclusive prefixes of flag sizes
    uint32_t* status;            // per tile: 0 empty, 1 aggregate, 2 inclusive
    ulonglong2* agg;             // per tile (payload, flag) aggregate
    ulonglong2* incl;            // per tile inclusive prefix
    uint32_t* tile_counter;      // zeroed before launch
    // optional: prefixes start at *carry_p / *carry_f (a container scanned
    // on its own, continuing the earlier containers' totals)
    const uint64_t* carry_p;
    const uint64_t* carry_f;
};
void launch_scan(const ScanArgs& a, cudaStream_t st);

// Geometry shared by Kernel III and the header kernel.  Containers 0..nb-2
// hold cpb full chunks; the last holds n_chunks - (nb-1)*cpb.
struct AssembleArgs {
    const uint8_t* in;           // input byte 0 (tails)
    const uint8_t* pay_slots;
    const uint8_t* flag_slots;
    const uint32_t* psize;
    const uint32_t* fsize;
    const uint64_t* P64;
    const uint64_t* F64;
    uint8_t* img;                // output image
    uint64_t* img_len;           // device word: total image bytes
    uint32_t* overflow;          // device word: 1 if a 4-byte table entry overflows
    uint64_t n_bytes;            // input bytes
    uint64_t n_chunks;
    uint64_t cpb;                // chunks per full container
    uint64_t block_bytes;
    uint64_t n_blocks;
    int S, W, I, C;
    // containers [j_lo, j_hi) only (their chunks): one container of a
    // pipelined compress; the defaults (0, 0) mean every container
    uint64_t j_lo, j_hi;
};
void launch_assemble(const AssembleArgs& a, cudaStream_t st);
// Kernel III variant (PipelineConfig::asm_mode; host_common.cpp): 0 register-staged,
// 1 TMA ring, 2 batched runs (default)
int assemble_mode();
void launch_headers(const AssembleArgs& a, cudaStream_t st);

// ---------------------------------------------------- multi-GPU shards
// One container touched by a shard's chunk range [g_lo, g_hi) (local
// chunk indices).  The shard writes four segments of the final image into a
// local buffer: its payload-table entries, flag-table entries, flag bytes and
// payload bytes, rebased by the bytes earlier shards contribute (p_base,
// f_base) to the container's streams.
struct ShardCont {
    uint64_t g_lo, g_hi;         // local chunk range
    uint64_t k_lo;               // container-relative index of local chunk g_lo
    uint64_t p_base, f_base;     // shard's first byte in the container's streams
    uint64_t seg_ptab, seg_ftab, seg_flags, seg_pay;  // local buffer offsets
};
struct ShardAssembleArgs {
    const uint8_t* pay_slots;
    const uint8_t* flag_slots;
    const uint32_t* psize;
    const uint32_t* fsize;
    const uint64_t* P64;         // local exclusive prefixes (n_chunks + 1)
    const uint64_t* F64;
    const ShardCont* conts;
    uint64_t n_conts;
    uint8_t* out;
    uint32_t* overflow;
    uint64_t n_chunks;           // local chunk count
    int S, C;
};
void launch_shard_assemble(const ShardAssembleArgs& a, cudaStream_t st);

// Root side: header, final table entries and tail of every container.
struct HeaderDesc {
    uint64_t img_off, byte_len, ptot, ftot;
    uint32_t n;
    uint8_t tail_len;
    uint8_t tail[3];
};
void launch_shard_headers(const HeaderDesc* d, uint64_t n_conts, uint8_t* img, int S, int W, int I,
                          int C, cudaStream_t st);

// ------------------------------------------------------------- decode side
struct ContainerDesc {
    uint64_t img_off;            // container byte 0 in the image
    uint64_t out_off;            // decoded byte 0 in the output
    uint64_t chunk_base;         // global index of the container's chunk 0
    uint64_t flags_off;          // absolute image offset of the flag stream
    uint64_t payload_off;        // absolute image offset of the payload stream
    uint64_t payload_len;        // payload stream bytes (the last payload-table entry)
    uint64_t original_len;
    uint32_t num_chunks;
    uint32_t chunk_size;
    uint32_t last_len;
    uint8_t S, W, I, tail_len;
};

// Parse outcome (written by plz_parse_kernel).  err_kind values are listed in
// host.cpp (format.cpp:112-185 order); err_* describe the first failing
// container.
struct ParseResult {
    uint64_t n_containers;
    uint64_t total_chunks;
    uint64_t total_out;
    uint32_t err_kind;
    uint32_t err_aux;            // version byte for the version error
    uint64_t err_container;
    uint64_t err_offset;         // byte offset relative to that container
    uint8_t hdr_S, hdr_W, hdr_I, pad0;
    uint32_t hdr_C;              // raw header fields for the validation message
    uint32_t absent_kinds;       // bit k: no container for decode kernel kind k (0: S = 1, 1: S = 2, 2: S = 4)
    uint32_t pad1;
    uint64_t max_chunk_bytes;
};

struct DecodeArgs {
    const uint8_t* img;
    uint64_t img_len;
    uint8_t* out;
    uint64_t out_cap;
    ContainerDesc* desc;
    uint64_t desc_cap;
    ParseResult* result;
    uint64_t* out_len;           // device word (async API)
    unsigned long long* err_chunk;  // min failing global chunk (atomicMin), ~0 if none
    uint32_t* work;
    // first table-monotonicity violation (global chunk << 1 | flag table),
    // ~0 if none; null: not checked (size-only walks)
    unsigned long long* mono_key;
};
// H2D/D2H pipeline of host buffers (plzgpu_decompress): image byte b may be
// read once in_ready[b / in_seg] == epoch; each chunk adds its decoded bytes
// to out_done[o / out_seg] for every output segment it covers once they are
// written (the D2H stream waits on those counts)
struct DecodePipe {
    const uint32_t* in_ready;
    uint32_t epoch;
    uint32_t* stalled;
    uint64_t in_seg;
    uint32_t* out_done;
    uint64_t out_seg;
};
void launch_parse(const DecodeArgs& a, cudaStream_t st);
// two launches (the S = 2 containers and the rest), each a persistent grid
// sized for `sms` SMs; work counters a.work[0] and a.work[1]
void launch_decode(const DecodeArgs& a, int sms, cudaStream_t st);
void launch_decode_pipelined(const DecodeArgs& a, const DecodePipe& pp, int sms, cudaStream_t st);
// chunk-range decode: res[0..2] = output range of chunks [cb, ce), total chunks;
// writes the tails inside the range to out (relative to res[0])
void launch_range(const DecodeArgs& a, uint64_t cb, uint64_t ce, uint8_t* out, uint64_t* res,
                  cudaStream_t st);
// re-decodes chunk *a.err_chunk and reports (TokenErr, chunk within container, token)
void launch_chunk_detail(const DecodeArgs& a, uint32_t* code, uint64_t* chunk, uint64_t* token,
                         cudaStream_t st);

// Lazy module loading (the CUDA 12 default) loads a kernel at its first
// launch, and that load waits for the device's running work: a launch queued
// behind a kernel that spins on H2D segments the host has not enqueued yet
// would stall the pipeline.  Each file's kernels are loaded up front instead
// (cudaFuncGetAttributes forces the load).
// The same pass raises each kernel's dynamic shared-memory limit to the
// device's opt-in maximum once; launches never set it again (a limit set per
// launch races between host threads: one thread's occupancy probe could
// lower it between another's set and launch, failing that launch).
inline void preload_kernel(const void* f) {
    cudaFuncAttributes at;
    if (cudaFuncGetAttributes(&at, f) != cudaSuccess) {
        (void)cudaGetLastError();
        return;
    }
    int dev = 0, optin = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - int(at.sharedSizeBytes)) != cudaSuccess)
        (void)cudaGetLastError();
}
// whether `smem` dynamic bytes fit the kernel's (preloaded) limit
inline bool smem_fits(const void* f, size_t smem) {
    cudaFuncAttributes at;
    if (cudaFuncGetAttributes(&at, f) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return smem <= size_t(at.maxDynamicSharedSizeBytes);
}
void preload_assemble_kernels();
void preload_scan_kernels();
void preload_cusz_kernels();
void preload_decode_kernels();
void preload_encode_kernels();
void preload_bitmatch_kernels();

struct DecodeOneArgs {
    const uint8_t* flags;
    uint64_t n_flags;
    const uint8_t* payload;
    uint64_t n_payload;
    uint64_t logical;
    int S;
    uint8_t* out;                // logical*S bytes (may be null for error-only runs)
    uint32_t* err_code;          // TokenErr
    uint64_t* err_token;
};
void launch_decode_one(const DecodeOneArgs& a, cudaStream_t st);
// ParseResult error fields for a monotonicity key; *base = the container's first chunk
void launch_mono_detail(const DecodeArgs& a, unsigned long long key, uint64_t* base,
                        cudaStream_t st);

// ------------------------------------------------ cuSZ dual quantization
uint64_t lorenzo_tiles(uint64_t n);
// codes + per-tile (1024 elements) outlier counts; the host scans the counts
// with Kernel II (launch_scan) before launch_outlier_write
void launch_lorenzo_quantize(const float* f, uint64_t nx, uint64_t ny, uint64_t nz, float s,
                             int32_t radius, uint16_t* codes, uint32_t* tile_count,
                             cudaStream_t st);
void launch_outlier_write(const float* f, uint64_t nx, uint64_t ny, uint64_t nz, float s,
                          const uint16_t* codes, const uint32_t* tile_count,
                          const uint64_t* tile_off, uint64_t* out_idx, int32_t* out_val,
                          uint64_t cap, cudaStream_t st);
// d: n int32 scratch
void launch_lorenzo_reconstruct(const uint16_t* codes, const uint64_t* out_idx,
                                const int32_t* out_val, uint64_t n_out, uint64_t nx, uint64_t ny,
                                uint64_t nz, int32_t radius, float two_eb, int32_t* d, float* f,
                                int sms, cudaStream_t st);

}  // namespace plzgpu
