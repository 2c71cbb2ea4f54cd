// cli.cpp — `plz_b200`, the reference's command-line front end
// (tools/plz.cpp:149-355) on the B200 path: compress / decompress / tune /
// stats / bench with the same flags, key:value reports, CSV rows and exit
// codes (0 ok, 1 other error, 2 usage / validation, 3 corrupt input).
// Argument parsing is hand-rolled (the reference's CLI11 is not vendored).
#include <chrono>
#include <cstdint>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "plz/corpus.hpp"
#include "plz/decoder.hpp"
#include "plz/errors.hpp"
#include "plz/params.hpp"
#include "plz/pipeline.hpp"
#include "plz/tuner.hpp"
#include "plzgpu.h"

namespace {

constexpr const char* kCsvHeader =
    "corpus,S,W,C,I,threads,in_bytes,out_bytes,ratio,seconds,throughput_bps\n";

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::vector<std::uint8_t> read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw plz::error("cannot open for reading: " + path);
    return std::vector<std::uint8_t>((std::istreambuf_iterator<char>(in)),
                                     std::istreambuf_iterator<char>());
}

void write_file(const std::string& path, const std::vector<std::uint8_t>& data) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw plz::error("cannot open for writing: " + path);
    out.write(reinterpret_cast<const char*>(data.data()), std::streamsize(data.size()));
    if (!out) throw plz::error("write failed: " + path);
}

// --name value / -X value options, bare flags, positionals
struct Args {
    std::map<std::string, std::string> opt;
    std::vector<std::string> pos;
    std::vector<std::string> flags;

    Args(int argc, char** argv, int from, const std::vector<std::string>& with_value,
         const std::vector<std::string>& bare) {
        for (int i = from; i < argc; ++i) {
            const std::string a = argv[i];
            bool matched = false;
            for (const auto& f : bare)
                if (a == f) {
                    flags.push_back(a);
                    matched = true;
                }
            if (matched) continue;
            for (const auto& n : with_value) {
                if (a == n) {
                    if (i + 1 >= argc) throw UsageError(n + " needs a value");
                    opt[n] = argv[++i];
                    matched = true;
                    break;
                }
                if (a.rfind(n + "=", 0) == 0) {
                    opt[n] = a.substr(n.size() + 1);
                    matched = true;
                    break;
                }
            }
            if (matched) continue;
            if (a.size() > 1 && a[0] == '-') throw UsageError("unknown option " + a);
            pos.push_back(a);
        }
    }
    bool has(const std::string& n) const { return opt.count(n) != 0; }
    std::string get(const std::string& a, const std::string& b, const std::string& dflt) const {
        if (opt.count(a)) return opt.at(a);
        if (opt.count(b)) return opt.at(b);
        return dflt;
    }
};

long long to_int(const std::string& s, const std::string& what) {
    try {
        std::size_t used = 0;
        const long long v = std::stoll(s, &used);
        if (used != s.size()) throw 0;
        return v;
    } catch (...) {
        throw UsageError(what + ": bad number '" + s + "'");
    }
}

const std::vector<std::string> kParamOpts = {"-S", "--symbol-width", "-W", "--window", "-C",
                                             "--chunk", "-I", "--interval", "--level",
                                             "--block-bytes"};

plz::Params params_from(const Args& a) {
    if ((a.has("-W") || a.has("--window")) && a.has("--level"))
        throw UsageError("--level and -W are mutually exclusive");
    plz::Params p;
    p.symbol_width = int(to_int(a.get("-S", "--symbol-width", "2"), "-S"));
    p.window = a.has("--level") ? plz::level_to_window(int(to_int(a.opt.at("--level"), "--level")))
                                : int(to_int(a.get("-W", "--window", "128"), "-W"));
    p.chunk_size = int(to_int(a.get("-C", "--chunk", "2048"), "-C"));
    p.interval = int(to_int(a.get("-I", "--interval", "1"), "-I"));
    p.block_bytes = std::size_t(to_int(a.get("--block-bytes", "--block-bytes",
                                             std::to_string(std::size_t{256} << 20)),
                                       "--block-bytes"));
    return plz::validate(p);
}

struct RunReport {
    std::string corpus;
    plz::Params params;
    int threads = 0;
    std::uint64_t in_bytes = 0, out_bytes = 0;
    double seconds = 0;
    double ratio() const { return out_bytes ? double(in_bytes) / double(out_bytes) : 0.0; }
    double throughput() const { return seconds > 0 ? double(in_bytes) / seconds : 0.0; }
    void print_kv(std::ostream& os) const {
        os << "input_bytes: " << in_bytes << "\noutput_bytes: " << out_bytes
           << "\nratio: " << ratio() << "\nseconds: " << seconds
           << "\nthroughput_bps: " << throughput() << "\nthreads: " << threads
           << "\nS: " << params.symbol_width << "\nW: " << params.window
           << "\nC: " << params.chunk_size << "\nI: " << params.interval << '\n';
    }
    std::string csv_row() const {
        std::ostringstream os;
        os << corpus << ',' << params.symbol_width << ',' << params.window << ','
           << params.chunk_size << ',' << params.interval << ',' << threads << ',' << in_bytes
           << ',' << out_bytes << ',' << ratio() << ',' << seconds << ',' << throughput() << '\n';
        return os.str();
    }
};

void append_csv(const std::string& path, const std::string& rows) {
    const bool fresh = !std::ifstream(path).good();
    std::ofstream out(path, std::ios::app);
    if (!out) throw plz::error("cannot open for writing: " + path);
    if (fresh) out << kCsvHeader;
    out << rows;
}

// --gpus 0,1,...: one stream over a device list (plzgpu_compress_multi /
// plzgpu_decompress_multi); errors mapped like the C++ API's
void throw_gpu_error(int rc, const plzgpu_error& e) {
    const std::string msg = e.message;
    switch (rc) {
        case PLZGPU_VALIDATION: throw plz::validation_error(msg);
        case PLZGPU_UNSUPPORTED_FORMAT: throw plz::unsupported_format_error(msg);
        case PLZGPU_CORRUPTION: throw plz::corruption_error(msg, e.byte_offset);
        default: throw plz::error(msg);
    }
}

std::vector<int> g_devices;  // set by --gpus

std::vector<std::uint8_t> compress_on(const std::vector<std::uint8_t>& data, const plz::Params& p,
                                      int threads) {
    if (g_devices.empty()) return plz::compress(data, p, threads);
    plzgpu_params cp{p.symbol_width, p.window, p.chunk_size, p.interval,
                     uint64_t(p.block_bytes), p.min_match, 0};
    std::vector<std::uint8_t> out(plzgpu_compress_bound(data.size(), &cp) + 16);
    uint64_t n = 0;
    plzgpu_error e{};
    const int rc = plzgpu_compress_multi(g_devices.data(), int(g_devices.size()), &cp, data.data(),
                                         data.size(), out.data(), out.size(), &n, nullptr, &e);
    if (rc) throw_gpu_error(rc, e);
    out.resize(n);
    return out;
}

std::vector<std::uint8_t> decompress_on(const std::vector<std::uint8_t>& img) {
    if (g_devices.empty()) return plz::decompress_bytes(img);
    std::vector<std::uint8_t> out(plzgpu_decompressed_bound(img.data(), img.size()) + 16);
    uint64_t n = 0;
    plzgpu_error e{};
    const int rc = plzgpu_decompress_multi(g_devices.data(), int(g_devices.size()), img.data(),
                                           img.size(), out.data(), out.size(), &n, &e);
    if (rc) throw_gpu_error(rc, e);
    out.resize(n);
    return out;
}

// wall time around plz::compress only (tools/plz.cpp:115-131)
RunReport timed_compress(const std::string& name, const std::vector<std::uint8_t>& data,
                         const plz::Params& p, int threads, std::vector<std::uint8_t>* out) {
    RunReport r{name, p, threads, data.size(), 0, 0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::uint8_t> img = compress_on(data, p, threads);
    r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r.out_bytes = img.size();
    if (out) *out = std::move(img);
    return r;
}

template <typename T>
std::vector<T> parse_list(const std::string& csv, const char* what) {
    std::vector<T> out;
    std::stringstream ss(csv);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(T(to_int(item, what)));
    if (out.empty()) throw UsageError(std::string(what) + ": empty list");
    return out;
}

void emit(const std::string& text, const std::string& path) {
    if (path.empty()) {
        std::cout << text;
        return;
    }
    std::ofstream out(path);
    if (!out) throw plz::error("cannot open for writing: " + path);
    out << text;
}

int run(int argc, char** argv) {
    if (argc < 2) throw UsageError("usage: plz_b200 {compress|decompress|tune|stats|bench} ...");
    const std::string cmd = argv[1];
    if (cmd == "compress") {
        std::vector<std::string> opts = kParamOpts;
        opts.insert(opts.end(), {"--threads", "--csv", "--gpus"});
        const Args a(argc, argv, 2, opts, {});
        if (a.pos.size() != 2) throw UsageError("compress needs input and output paths");
        if (a.has("--gpus")) g_devices = parse_list<int>(a.opt.at("--gpus"), "--gpus");
        const plz::Params p = params_from(a);
        const int threads = int(to_int(a.get("--threads", "--threads", "0"), "--threads"));
        const std::vector<std::uint8_t> data = read_file(a.pos[0]);
        std::vector<std::uint8_t> out;
        const RunReport r = timed_compress(a.pos[0], data, p, threads, &out);
        write_file(a.pos[1], out);
        r.print_kv(std::cout);
        if (a.has("--csv")) append_csv(a.opt.at("--csv"), r.csv_row());
        return 0;
    }
    if (cmd == "decompress") {
        const Args a(argc, argv, 2, {"--threads", "--gpus"}, {});
        if (a.pos.size() != 2) throw UsageError("decompress needs input and output paths");
        if (a.has("--gpus")) g_devices = parse_list<int>(a.opt.at("--gpus"), "--gpus");
        const std::vector<std::uint8_t> data = read_file(a.pos[0]);
        try {
            write_file(a.pos[1], decompress_on(data));
        } catch (const plz::corruption_error& e) {
            std::cerr << "error: " << e.what() << '\n';
            return 3;
        } catch (const plz::unsupported_format_error& e) {
            std::cerr << "error: " << e.what() << '\n';
            return 3;
        }
        return 0;
    }
    if (cmd == "tune") {
        std::vector<std::string> opts = kParamOpts;
        opts.insert(opts.end(), {"--declared-width", "--threshold", "--pilot-cap", "--out"});
        const Args a(argc, argv, 2, opts, {});
        if (!a.has("--declared-width")) throw UsageError("--declared-width is required");
        if (a.pos.empty()) throw UsageError("tune needs field files");
        std::vector<std::vector<std::uint8_t>> data;
        std::vector<std::span<const std::uint8_t>> fields;
        for (const auto& path : a.pos) data.push_back(read_file(path));
        for (const auto& d : data) fields.emplace_back(d);
        plz::TunerOptions o;
        if (a.has("--threshold")) o.threshold = std::stod(a.opt.at("--threshold"));
        if (a.has("--pilot-cap")) o.pilot_cap = std::size_t(to_int(a.opt.at("--pilot-cap"), "--pilot-cap"));
        const plz::PilotReport rep = plz::select_params(
            fields, int(to_int(a.opt.at("--declared-width"), "--declared-width")), params_from(a), o);
        std::ostringstream os;
        for (std::size_t i = 0; i < rep.field_ratios.size(); ++i)
            os << "field_" << i << "_ratio: " << rep.field_ratios[i] << '\n';
        os << "average_ratio: " << rep.average << "\nthreshold: " << o.threshold
           << "\nchosen_S: " << rep.chosen.symbol_width << "\nchosen_W: " << rep.chosen.window
           << "\nchosen_C: " << rep.chosen.chunk_size << "\nchosen_I: " << rep.chosen.interval
           << "\nchosen_flags: -S " << rep.chosen.symbol_width << " -W " << rep.chosen.window
           << " -C " << rep.chosen.chunk_size << " -I " << rep.chosen.interval << '\n';
        emit(os.str(), a.get("--out", "--out", ""));
        return 0;
    }
    if (cmd == "stats") {
        std::vector<std::string> opts = kParamOpts;
        opts.push_back("--out");
        const Args a(argc, argv, 2, opts, {"--raw"});
        if (a.pos.size() != 1) throw UsageError("stats needs one input path");
        const bool raw = !a.flags.empty();
        emit(plz::histogram_csv(plz::match_length_histogram(read_file(a.pos[0]), params_from(a), raw)),
             a.get("--out", "--out", ""));
        return 0;
    }
    if (cmd == "bench") {
        const Args a(argc, argv, 2,
                     {"--kind", "--size", "--seed", "--mean-run", "--alphabet", "--dominant-prob",
                      "--width", "-S", "--symbol-width", "-W", "--window", "-C", "--chunk", "-I",
                      "--interval", "--threads", "--csv"},
                     {});
        const auto s_vals = parse_list<int>(a.get("-S", "--symbol-width", "2"), "-S");
        const auto w_vals = parse_list<int>(a.get("-W", "--window", "128"), "-W");
        const auto c_vals = parse_list<int>(a.get("-C", "--chunk", "2048"), "-C");
        const auto i_vals = parse_list<int>(a.get("-I", "--interval", "1"), "-I");
        const auto t_vals = parse_list<int>(a.get("--threads", "--threads", "0"), "--threads");
        std::ostringstream rows;
        std::stringstream kinds(a.get("--kind", "--kind", "runlen"));
        std::string kind;
        while (std::getline(kinds, kind, ',')) {
            plz::GeneratorSpec spec;
            spec.kind = plz::corpus_kind_from_name(kind);
            spec.size = std::size_t(to_int(a.get("--size", "--size", std::to_string(16u << 20)), "--size"));
            spec.seed = std::uint64_t(to_int(a.get("--seed", "--seed", "42"), "--seed"));
            spec.mean_run = std::stod(a.get("--mean-run", "--mean-run", "64"));
            spec.alphabet = int(to_int(a.get("--alphabet", "--alphabet", "4"), "--alphabet"));
            spec.dominant_prob = std::stod(a.get("--dominant-prob", "--dominant-prob", "0.9"));
            spec.width = int(to_int(a.get("--width", "--width", "2"), "--width"));
            const std::vector<std::uint8_t> data = plz::generate(spec);
            for (int s : s_vals)
                for (int w : w_vals)
                    for (int c : c_vals)
                        for (int i : i_vals)
                            for (int t : t_vals) {
                                plz::Params p;
                                p.symbol_width = s;
                                p.window = w;
                                p.chunk_size = c;
                                p.interval = i;
                                rows << timed_compress(kind, data, plz::validate(p), t, nullptr).csv_row();
                            }
        }
        if (a.has("--csv"))
            append_csv(a.opt.at("--csv"), rows.str());
        else
            std::cout << kCsvHeader << rows.str();
        return 0;
    }
    throw UsageError("unknown subcommand " + cmd);
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    } catch (const plz::validation_error& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    } catch (const plz::error& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
