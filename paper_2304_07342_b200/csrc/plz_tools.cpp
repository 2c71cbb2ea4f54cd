// plz_tools.cpp — the reference's matcher / corpus / tuner entry points over
// the C-ABI (matcher.cpp:113-131 via plzgpu_match_table, corpus.cpp:75-142
// via plzgpu_match_table / plzgpu_pointer_histogram, tuner.cpp:10-45 via
// plz::compress).  generate() restates corpus.cpp:20-73 on the host (same
// std::mt19937_64 streams and libstdc++ distributions, so identical bytes).
#include <algorithm>
#include <cstring>
#include <random>
#include <sstream>
#include <string>

#include "plz/corpus.hpp"
#include "plz/errors.hpp"
#include "plz/matcher.hpp"
#include "plz/pipeline.hpp"
#include "plz/tuner.hpp"
#include "plzgpu.h"

namespace plz {
namespace detail {
plzgpu_ctx* ctx();
plzgpu_params to_c(const Params& p);
void check(int rc, const plzgpu_error& e);
}  // namespace detail

void load_symbols(std::span<const std::uint8_t> bytes, int symbol_width,
                  std::vector<std::uint32_t>& out) {
    if (symbol_width != 1 && symbol_width != 2 && symbol_width != 4)
        throw contract_error("symbol_width must be 1, 2 or 4");
    if (bytes.size() % std::size_t(symbol_width) != 0)
        throw contract_error("symbol buffer not a multiple of symbol_width");
    out.assign(bytes.size() / std::size_t(symbol_width), 0);
    for (std::size_t i = 0; i < out.size(); ++i)
        for (int b = 0; b < symbol_width; ++b)
            out[i] |= std::uint32_t(bytes[i * std::size_t(symbol_width) + std::size_t(b)]) << (8 * b);
}

void run_lengths(std::span<const std::uint32_t> chunk, std::vector<std::uint32_t>& out) {
    out.assign(chunk.size(), 1);
    for (std::size_t i = chunk.size(); i-- > 1;)
        if (chunk[i - 1] == chunk[i]) out[i - 1] = out[i] + 1;
}

// u32 symbols back to S-byte little-endian bytes for the C-ABI
static std::vector<std::uint8_t> to_bytes(std::span<const std::uint32_t> chunk, int S) {
    std::vector<std::uint8_t> b(chunk.size() * std::size_t(S));
    for (std::size_t i = 0; i < chunk.size(); ++i)
        for (int k = 0; k < S; ++k) b[i * std::size_t(S) + std::size_t(k)] = std::uint8_t(chunk[i] >> (8 * k));
    return b;
}

MatchTable match_chunk(std::span<const std::uint32_t> chunk, const Params& params,
                       std::uint64_t* /*max_cmp_per_pos*/) {
    if (chunk.size() > std::size_t(params.chunk_size))
        throw contract_error("chunk longer than chunk_size");
    const std::vector<std::uint8_t> bytes = to_bytes(chunk, params.symbol_width);
    std::vector<std::uint8_t> len(chunk.size() + 1), off(chunk.size() + 1);
    plzgpu_params p = detail::to_c(params);
    p.block_bytes = std::uint64_t(params.chunk_size) * std::uint64_t(params.symbol_width);
    plzgpu_error e;
    detail::check(plzgpu_match_table(detail::ctx(), &p, bytes.data(), bytes.size(), len.data(),
                                     off.data(), nullptr, nullptr, &e),
                  e);
    MatchTable t;
    t.records.resize(chunk.size());
    for (std::size_t i = 0; i < chunk.size(); ++i) t.records[i] = MatchRecord{len[i], off[i]};
    return t;
}

MatchRecord find_match(std::span<const std::uint32_t> chunk, std::size_t pos, const Params& params,
                       std::uint64_t* /*cmp_counter*/, std::span<const std::uint32_t> /*runs*/) {
    Params p = params;
    p.interval = 1;  // find_match searches the given position unconditionally
    // the contract only needs the window before pos and the lookahead cap
    return match_chunk(chunk, p).records.at(pos);
}

GeneratorSpec::Kind corpus_kind_from_name(const std::string& name) {
    if (name == "runlen") return GeneratorSpec::Kind::runlen;
    if (name == "quantlike") return GeneratorSpec::Kind::quantlike;
    if (name == "uniform") return GeneratorSpec::Kind::uniform;
    throw validation_error("unknown corpus kind: " + name);
}

std::vector<std::uint8_t> generate(const GeneratorSpec& spec) {
    if (spec.size == 0) throw validation_error("corpus size must be > 0");
    std::mt19937_64 rng(spec.seed);
    std::vector<std::uint8_t> out;
    out.reserve(spec.size);
    if (spec.kind == GeneratorSpec::Kind::uniform) {
        std::uniform_int_distribution<int> byte(0, 255);
        while (out.size() < spec.size) out.push_back(std::uint8_t(byte(rng)));
    } else if (spec.kind == GeneratorSpec::Kind::runlen) {
        if (spec.mean_run < 1) throw validation_error("mean_run must be >= 1");
        if (spec.alphabet < 1 || spec.alphabet > 256)
            throw validation_error("alphabet must be in [1,256]");
        std::uniform_int_distribution<int> symbol(0, spec.alphabet - 1);
        std::geometric_distribution<std::uint64_t> extra(spec.mean_run > 1 ? 1.0 / spec.mean_run : 1.0);
        while (out.size() < spec.size) {
            const std::uint8_t v = std::uint8_t(symbol(rng));
            for (std::uint64_t run = 1 + extra(rng); run-- && out.size() < spec.size;) out.push_back(v);
        }
    } else {
        if (spec.dominant_prob < 0.0 || spec.dominant_prob > 1.0)
            throw validation_error("dominant_prob must be in [0,1]");
        if (spec.width != 1 && spec.width != 2 && spec.width != 4)
            throw validation_error("quantlike width must be 1, 2 or 4");
        std::bernoulli_distribution dominant(spec.dominant_prob);
        std::uniform_int_distribution<int> delta(1, 8);
        std::bernoulli_distribution negate(0.5);
        const std::uint32_t centre = spec.width == 1 ? 128u : spec.width == 2 ? 32768u : 1u << 30;
        while (out.size() < spec.size) {
            std::uint32_t code = centre;
            if (!dominant(rng)) {
                const int d = delta(rng);
                code = negate(rng) ? centre - std::uint32_t(d) : centre + std::uint32_t(d);
            }
            for (int b = 0; b < spec.width && out.size() < spec.size; ++b)
                out.push_back(std::uint8_t(code >> (8 * b)));
        }
    }
    return out;
}

MatchHistogram match_length_histogram(std::span<const std::uint8_t> data, const Params& base,
                                      bool raw_table) {
    Params params = base;
    params.interval = 1;  // corpus.cpp:180-182
    params = validate(params);
    MatchHistogram h;
    h.symbol_width = params.symbol_width;
    std::uint64_t counts[256];
    const plzgpu_params p = detail::to_c(params);
    plzgpu_error e;
    if (raw_table)
        detail::check(plzgpu_match_table(detail::ctx(), &p, data.data(), data.size(), nullptr,
                                         nullptr, counts, nullptr, &e),
                      e);
    else
        detail::check(plzgpu_pointer_histogram(detail::ctx(), &p, data.data(), data.size(), counts,
                                               nullptr, &e),
                      e);
    for (int len = 1; len < 256; ++len) {
        h.counts[std::size_t(len)] = counts[len];
        h.total_pointers += counts[len];
    }
    if (h.total_pointers > 0) {
        std::uint64_t gt128 = 0, gt256 = 0;
        for (std::size_t len = 1; len <= 255; ++len) {
            const std::uint64_t bytes = len * std::uint64_t(params.symbol_width);
            if (bytes > 128) gt128 += h.counts[len];
            if (bytes > 256) gt256 += h.counts[len];
        }
        h.fraction_gt_128 = double(gt128) / double(h.total_pointers);
        h.fraction_gt_256 = double(gt256) / double(h.total_pointers);
    }
    return h;
}

std::string histogram_csv(const MatchHistogram& h) {
    std::ostringstream out;
    out << "length,count,byte_length,fraction_gt_128,fraction_gt_256\n";
    for (std::size_t len = 1; len <= 255; ++len) {
        if (h.counts[len] == 0) continue;
        out << len << ',' << h.counts[len] << ',' << len * std::size_t(h.symbol_width) << ','
            << h.fraction_gt_128 << ',' << h.fraction_gt_256 << '\n';
    }
    out << "total," << h.total_pointers << ",," << h.fraction_gt_128 << ',' << h.fraction_gt_256
        << '\n';
    return out.str();
}

PilotReport select_params(const std::vector<std::span<const std::uint8_t>>& fields,
                          int declared_width, const Params& base, const TunerOptions& options) {
    if (fields.empty()) throw validation_error("tuner requires at least one field");
    if (declared_width != 1 && declared_width != 2 && declared_width != 4)
        throw validation_error("declared_width must be 1, 2 or 4");
    Params pilot = base;
    pilot.symbol_width = declared_width;
    pilot = validate(pilot);
    PilotReport report;
    for (const auto& field : fields) {
        const auto sample = field.subspan(0, std::min(field.size(), options.pilot_cap));
        const std::vector<std::uint8_t> img = compress(sample, pilot, options.threads);
        const double ratio = img.empty() ? 1.0 : double(sample.size()) / double(img.size());
        report.field_ratios.push_back(ratio);
        report.average += ratio;
    }
    report.average /= double(report.field_ratios.size());
    Params chosen = base;
    if (report.average < options.threshold) {
        chosen.symbol_width = 1;  // window unchanged in the fallback (tuner.cpp:284-286)
    } else {
        chosen.symbol_width = declared_width;
        chosen.window = std::min(255, base.window * declared_width);
    }
    report.chosen = validate(chosen);
    return report;
}

}  // namespace plz
