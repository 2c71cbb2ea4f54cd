// compress_block_parity.cpp — GPU test program (tests/test_gpu_dropin.py).
//
// plz::compress_block of the B200 drop-in (include/plz/pipeline.hpp,
// libplzgpu.so) against the reference's own plzref::compress_block
// (/root/reference/proj/src/pipeline.cpp:26-86, compiled unmodified into
// oracle/_ref/libplzref.so and reached through oracle/ref_shim.cpp): every
// block of plz::plan for a grid of parameters and input sizes — full and
// partial final chunks, final blocks with a raw tail, non-final blocks, a
// tail-only block — serialised with plz::write_container must equal the
// reference's container byte for byte, with equal pointer / literal counts;
// a span that does not match its plan raises contract_error, as in
// pipeline.cpp:28-29.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <span>
#include <vector>

#include "plz/errors.hpp"
#include "plz/format.hpp"
#include "plz/partition.hpp"
#include "plz/pipeline.hpp"
#include "plz_oracle.h"

extern "C" int plzref_compress_block(const unsigned char* block, std::uint64_t n,
                                     std::uint64_t byte_start, std::uint64_t byte_len,
                                     std::uint32_t num_chunks, std::uint32_t last_chunk_len,
                                     std::uint8_t tail_len, const plzo_params* p, int threads,
                                     unsigned char** out, std::uint64_t* out_len,
                                     std::uint64_t* stats, plzo_error* err);
extern "C" void plzref_free(void* p);

namespace {

std::uint64_t splitmix(std::uint64_t& s) {
    std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// quant-code-like symbols: a dominant centre with small excursions and runs
std::vector<std::uint8_t> make_input(std::size_t n, int S, std::uint64_t seed) {
    std::vector<std::uint8_t> v(n);
    std::uint64_t s = seed;
    std::uint32_t sym = 512;
    for (std::size_t i = 0; i < n; i += std::size_t(S)) {
        const std::uint64_t r = splitmix(s);
        if (r % 8 == 0) sym = 512 + std::uint32_t(r >> 8) % 9 - 4;
        else if (r % 31 == 0) sym = std::uint32_t(r >> 16);
        for (int b = 0; b < S && i + std::size_t(b) < n; ++b) v[i + std::size_t(b)] = std::uint8_t(sym >> (8 * b));
    }
    return v;
}

}  // namespace

int main() {
    struct Case { int S, W, C, I; std::uint64_t block_bytes; std::size_t n; };
    const Case cases[] = {
        {2, 255, 2048, 2, 3 * 4096, 5 * 4096 + 1001},      // 2 blocks, partial last chunk, tail 1
        {2, 128, 2048, 1, 2 * 4096, 4 * 4096},             // exact blocks, no tail
        {1, 128, 4096, 1, 4096, 3 * 4096 + 77},            // u8, partial last block
        {4, 255, 1024, 4, 2 * 4096, 3 * 4096 + 3},         // u32, tail 3
        {4, 64, 1024, 8, 4096, 4096 + 2},                  // final block: a 2-byte tail alone
        {2, 32, 1024, 16, 2048, 2048 * 3 + 1},             // final block: a 1-byte tail alone
        {1, 255, 16384, 1, 16384, 16384 + 5000},           // large chunks
        {2, 255, 2048, 2, 256ull << 20, 300000 + 1},       // one container (default block size)
    };
    int blocks = 0, failures = 0;
    for (const Case& k : cases) {
        plz::Params p;
        p.symbol_width = k.S;
        p.window = k.W;
        p.chunk_size = k.C;
        p.interval = k.I;
        p.block_bytes = k.block_bytes;
        p = plz::validate(p);
        const std::vector<std::uint8_t> data = make_input(k.n, k.S, 1234 + k.n);
        const plz::PartitionPlan plan = plz::plan(data.size(), p);
        plzo_params q{};
        q.symbol_width = p.symbol_width;
        q.window = p.window;
        q.chunk_size = p.chunk_size;
        q.interval = p.interval;
        q.block_bytes = p.block_bytes;
        q.min_match = p.min_match;
        for (const plz::BlockPlan& b : plan.blocks) {
            const std::span<const std::uint8_t> blk(data.data() + b.byte_start, b.byte_len);
            plz::PipelineStats st;
            const plz::Container c = plz::compress_block(blk, b, p, 0, &st);
            const std::vector<std::uint8_t> got = plz::write_container(c);
            unsigned char* ref = nullptr;
            std::uint64_t ref_len = 0, rs[3] = {0, 0, 0};
            plzo_error e{};
            if (plzref_compress_block(blk.data(), blk.size(), b.byte_start, b.byte_len, b.num_chunks,
                                      b.last_chunk_len, b.tail_len, &q, 0, &ref, &ref_len, rs,
                                      &e) != 0) {
                std::printf("reference failed: %s\n", e.message);
                return 2;
            }
            const bool same = got.size() == ref_len && std::memcmp(got.data(), ref, ref_len) == 0;
            const bool same_stats = st.pointer_tokens == rs[1] && st.literal_tokens == rs[2];
            plzref_free(ref);
            ++blocks;
            if (!same || !same_stats) {
                ++failures;
                std::printf("MISMATCH S=%d W=%d C=%d I=%d block@%llu len=%llu tail=%u: image %s, "
                            "stats %s\n", k.S, k.W, k.C, k.I, (unsigned long long)b.byte_start,
                            (unsigned long long)b.byte_len, unsigned(b.tail_len),
                            same ? "equal" : "differs", same_stats ? "equal" : "differ");
            }
        }
        // a span that does not match its plan (pipeline.cpp:28-29)
        try {
            plz::compress_block(std::span<const std::uint8_t>(data.data(), plan.blocks[0].byte_len - 1),
                                plan.blocks[0], p);
            ++failures;
            std::printf("MISMATCH: no contract_error for a short span\n");
        } catch (const plz::contract_error& ex) {
            if (std::strcmp(ex.what(), "block span does not match plan") != 0) {
                ++failures;
                std::printf("MISMATCH: contract_error text '%s'\n", ex.what());
            }
        }
    }
    std::printf("compress_block parity: %d blocks, %d failures\n", blocks, failures);
    return failures ? 1 : 0;
}
