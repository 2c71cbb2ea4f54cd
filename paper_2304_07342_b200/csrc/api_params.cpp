// api_params.cpp — the C-ABI's pure host arithmetic: parameter validation
// (params.cpp:19-55), the block plan (partition.cpp:5-25), container sizes
// (format.cpp:69-73) and the image / output bounds.
#include <cstring>

#include "host_internal.h"

using namespace plzhost;

extern "C" {

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
    while (at < len) {
        const uint64_t size = len - at;
        const uint8_t* h = b + at;
        if (size < 26 || std::memcmp(h, "PLZ1", 4) != 0 || h[4] != 1 || h[8] != 0) break;
        plzgpu_params p{};
        p.symbol_width = h[5];
        p.window = h[6];
        p.interval = h[7];
        p.chunk_size = int32_t(host_le32(h + 9));
        p.block_bytes = uint64_t(256) << 20;
        if (validate_fields(p, nullptr) != PLZGPU_OK || h[25] >= h[5]) break;
        const uint64_t n = host_le32(h + 21);
        if (size < 26 + 8 * (n + 1)) break;
        const uint8_t* pt = h + 26;
        const uint8_t* ft = pt + 4 * (n + 1);
        bool mono = host_le32(pt) == 0 && host_le32(ft) == 0;
        for (uint64_t i = 0; mono && i < n; ++i)
            mono = host_le32(pt + 4 * (i + 1)) >= host_le32(pt + 4 * i) &&
                   host_le32(ft + 4 * (i + 1)) >= host_le32(ft + 4 * i);
        if (!mono) break;
        const uint64_t ptot = host_le32(pt + 4 * n), ftot = host_le32(ft + 4 * n);
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

uint64_t plzgpu_num_chunks(uint64_t n, const plzgpu_params* p) { return geometry(n, *p).n_chunks; }

uint64_t plzgpu_num_containers(uint64_t n, const plzgpu_params* p) {
    return geometry(n, *p).n_blocks;
}

}  // extern "C"
