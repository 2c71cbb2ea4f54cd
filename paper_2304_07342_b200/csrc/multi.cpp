// multi.cpp — one stream over a device list in one process (SURVEY.md §8b
// item 4, §8e): the shard protocol of dist.py with host threads for ranks.
//
// Contexts come from a process-wide pool (one per device entry, reused by
// later calls: no per-call context creation, kernel preload or scratch
// allocation once warm).  Peer access between the root (devices[0]) and
// every other listed GPU is enabled once; with it, each rank's Kernel III
// stores its table and stream segments straight into the root's image over
// NVLink (plzgpu_shard_assemble_into) and a rank's decode writes its output
// slice straight into a device `out`.  Without peer access the segments are
// assembled locally and moved with cudaMemcpyPeerAsync on the rank's stream.
// The caller's current device is restored on return.
#include <cstring>
#include <mutex>
#include <set>
#include <thread>
#include <utility>

#include "host_internal.h"

using namespace plzhost;

namespace {

struct Pool {
    std::mutex mu;
    std::vector<plzgpu_ctx*> idle;
};
Pool& pool() {
    static Pool* p = new Pool;  // never destroyed: contexts outlive static teardown
    return *p;
}

int acquire(int device, plzgpu_ctx** out, plzgpu_error* err) {
    {
        std::lock_guard<std::mutex> lock(pool().mu);
        auto& v = pool().idle;
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i]->device == device) {
                *out = v[i];
                v.erase(v.begin() + long(i));
                return PLZGPU_OK;
            }
    }
    return plzgpu_ctx_create(device, out, err);
}

void release(plzgpu_ctx* c) {
    if (!c) return;
    std::lock_guard<std::mutex> lock(pool().mu);
    pool().idle.push_back(c);
}

struct Lease {  // the call's contexts, returned to the pool on scope exit
    std::vector<plzgpu_ctx*> ctx;
    ~Lease() {
        for (plzgpu_ctx* c : ctx) release(c);
    }
};

// Whether device `from` can store to / load from device `to` memory.
bool peer_ok(int from, int to) {
    if (from == to) return true;
    static std::mutex mu;
    static std::set<std::pair<int, int>> ok, bad;
    std::lock_guard<std::mutex> lock(mu);
    if (ok.count({from, to})) return true;
    if (bad.count({from, to})) return false;
    int can = 0;
    bool good = cudaDeviceCanAccessPeer(&can, from, to) == cudaSuccess && can;
    if (good) {
        DeviceGuard keep;
        cudaSetDevice(from);
        const cudaError_t e = cudaDeviceEnablePeerAccess(to, 0);
        good = e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled;
    }
    (void)cudaGetLastError();
    (good ? ok : bad).insert({from, to});
    return good;
}

int device_of(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) == cudaSuccess &&
        (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged))
        return at.device;
    (void)cudaGetLastError();
    return -1;
}

template <typename F>
void run_ranks(uint64_t N, F&& body) {
    std::vector<std::thread> th;
    for (uint64_t r = 0; r < N; ++r) th.emplace_back([&, r] { body(r); });
    for (std::thread& t : th) t.join();
}

}  // namespace

extern "C" {

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
    DeviceGuard keep;
    const plzgpu_params& p = *params;
    const Geometry g = geometry(n, p);
    const uint64_t S = uint64_t(p.symbol_width), C = uint64_t(p.chunk_size), N = uint64_t(n_devices);
    const int root = devices[0];
    const int in_dev = device_of(in);
    Lease lease;
    lease.ctx.assign(N, nullptr);
    for (uint64_t r = 0; r < N; ++r)
        if ((rc = acquire(devices[r], &lease.ctx[r], err))) return rc;
    std::vector<plzgpu_ctx*>& ctx = lease.ctx;
    // ---- ranks encode their chunk ranges concurrently (a device input on
    // another GPU is first brought to the rank's GPU, peer to peer)
    uint64_t max_touched = 1;
    std::vector<uint64_t> rb(N), re(N);
    for (uint64_t r = 0; r < N; ++r) {
        rb[r] = g.n_chunks * r / N;
        re[r] = g.n_chunks * (r + 1) / N;
        max_touched = std::max(max_touched, (re[r] - rb[r] + g.cpb - 1) / g.cpb + 1);
    }
    std::vector<std::vector<uint64_t>> tot(N);
    std::vector<int> rcs(N, PLZGPU_OK);
    std::vector<plzgpu_error> errs(N);
    run_ranks(N, [&](uint64_t r) {
        plzgpu_ctx* c = ctx[r];
        plzgpu_error* err = &errs[r];
        rcs[r] = [&]() -> int {
            CK(cudaSetDevice(c->device));
            const uint64_t lo = rb[r] * C * S, hi = re[r] == g.n_chunks ? n : re[r] * C * S;
            const void* src = static_cast<const uint8_t*>(in) + lo;
            if (in_dev >= 0 && in_dev != c->device && hi > lo) {
                CK(c->in.ensure(hi - lo + 16));
                CK(cudaMemcpyPeerAsync(c->in.p, c->device, src, in_dev, hi - lo, c->stream));
                src = c->in.p;
            }
            tot[r].assign(3 * max_touched, 0);
            uint64_t nt = 0;
            const int rc2 = plzgpu_shard_encode(c, &p, src, n, rb[r], re[r], tot[r].data(),
                                                max_touched, &nt, c->stream, err);
            tot[r].resize(3 * nt);
            return rc2;
        }();
    });
    for (uint64_t r = 0; r < N; ++r)
        if (rcs[r]) {
            if (err) *err = errs[r];
            return rcs[r];
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
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                       "output buffer too small: need %llu bytes", (unsigned long long)image_len);
    // ---- the image on the root: the caller's buffer when it is the root's
    // device memory, else the root context's scratch
    const bool in_place = device_of(out) == root;
    uint8_t* d_img = static_cast<uint8_t*>(out);
    if (!in_place) {
        CK(cudaSetDevice(root));
        CK(ctx[0]->img.ensure(image_len + 16));
        d_img = ctx[0]->img.as<uint8_t>();
    }
    const uint64_t img_cap = in_place ? cap : image_len + 16;
    // ---- every rank's segments into the image
    run_ranks(N, [&](uint64_t r) {
        plzgpu_ctx* c = ctx[r];
        plzgpu_error* err = &errs[r];
        rcs[r] = [&]() -> int {
            if (tot[r].empty()) return PLZGPU_OK;
            CK(cudaSetDevice(c->device));
            if (peer_ok(c->device, root))
                return plzgpu_shard_assemble_into(c, bases[r].data(), d_img, img_cap, c->stream,
                                                  err);
            const uint64_t nt = tot[r].size() / 3;
            uint64_t local = 8 * (re[r] - rb[r]) + 16;
            for (uint64_t i = 0; i < nt; ++i) local += tot[r][3 * i + 1] + tot[r][3 * i + 2];
            CK(c->out.ensure(local));
            std::vector<uint64_t> segs(12 * nt);
            uint64_t ns = 0, ln = 0;
            int rc2 = plzgpu_shard_assemble(c, bases[r].data(), c->out.p, local, segs.data(),
                                            4 * nt, &ns, &ln, c->stream, err);
            if (rc2) return rc2;
            for (uint64_t k = 0; k < ns; ++k)
                if (segs[3 * k + 2])
                    CK(cudaMemcpyPeerAsync(d_img + segs[3 * k], root,
                                           c->out.as<uint8_t>() + segs[3 * k + 1], c->device,
                                           segs[3 * k + 2], c->stream));
            CK(cudaStreamSynchronize(c->stream));
            return PLZGPU_OK;
        }();
    });
    for (uint64_t r = 0; r < N; ++r)
        if (rcs[r]) {
            if (err) *err = errs[r];
            return rcs[r];
        }
    // ---- headers, final table entries and the tail on the root, then out
    std::vector<uint64_t> totals(2 * g.n_blocks);
    for (uint64_t j = 0; j < g.n_blocks; ++j) {
        totals[2 * j] = ptot[j];
        totals[2 * j + 1] = ftot[j];
    }
    uint8_t tail[4] = {0, 0, 0, 0};
    const uint64_t tl = n % S;
    CK(cudaSetDevice(root));
    if (tl) CK(cudaMemcpy(tail, static_cast<const uint8_t*>(in) + (n - tl), tl, cudaMemcpyDefault));
    uint64_t img_len = 0;
    rc = plzgpu_shard_headers(ctx[0], &p, n, totals.data(), tail, d_img, img_cap, &img_len,
                              ctx[0]->stream, err);
    if (rc) return rc;
    if (!in_place) {
        CK(cudaMemcpyAsync(out, d_img, img_len, cudaMemcpyDefault, ctx[0]->stream));
        CK(cudaStreamSynchronize(ctx[0]->stream));
    }
    if (stats) {
        for (uint64_t r = 0; r < N; ++r) {
            unsigned long long st2[2] = {0, 0};
            CK(cudaSetDevice(ctx[r]->device));
            CK(cudaMemcpy(st2, dmeta(ctx[r])->stats, sizeof st2, cudaMemcpyDeviceToHost));
            stats->pointer_tokens += st2[0];
            stats->literal_tokens += st2[1];
        }
    }
    *out_len = img_len;
    return PLZGPU_OK;
}

int plzgpu_decompress_multi(const int* devices, int n_devices, const void* img, uint64_t len,
                            void* out, uint64_t cap, uint64_t* out_len, plzgpu_error* err) {
    clear_err(err);
    *out_len = 0;
    if (n_devices < 1 || !devices)
        return set_err(err, PLZGPU_CONTRACT, 0, kNoIndex, kNoIndex, "empty device list");
    if (len == 0) return PLZGPU_OK;
    DeviceGuard keep;
    const uint64_t N = uint64_t(n_devices);
    const int img_dev = device_of(img);
    const int out_dev = device_of(out);
    Lease lease;
    lease.ctx.assign(N, nullptr);
    int rc = PLZGPU_OK;
    for (uint64_t r = 0; r < N; ++r)
        if ((rc = acquire(devices[r], &lease.ctx[r], err))) return rc;
    std::vector<plzgpu_ctx*>& ctx = lease.ctx;
    // the image each rank reads: the caller's when it is on the rank's GPU,
    // else a copy there (one H2D or peer copy per rank and call)
    std::vector<const void*> src(N, img);
    std::vector<int> rcs(N, PLZGPU_OK);
    std::vector<plzgpu_error> errs(N);
    std::vector<uint64_t> begin(N, 0), size(N, 0), total(N, 0);
    run_ranks(N, [&](uint64_t r) {
        plzgpu_ctx* c = ctx[r];
        plzgpu_error* err = &errs[r];
        rcs[r] = [&]() -> int {
            CK(cudaSetDevice(c->device));
            if (img_dev != c->device) {
                CK(c->img.ensure(len + 16));
                if (img_dev >= 0)
                    CK(cudaMemcpyPeerAsync(c->img.p, c->device, img, img_dev, len, c->stream));
                else
                    CK(cudaMemcpyAsync(c->img.p, img, len, cudaMemcpyHostToDevice, c->stream));
                src[r] = c->img.p;
            }
            // the chunk count (and every header's checks)
            uint64_t b0 = 0, l0 = 0;
            return plzgpu_decompress_range(c, src[r], len, 0, 0, nullptr, 0, &b0, &l0, &total[r],
                                           c->stream, err);
        }();
    });
    // Any failure: the single-context decode reports it, in the reference's
    // order (a header error of a later container only after the token
    // errors of earlier containers' chunks, decoder.cpp:129-141).
    auto report = [&](uint64_t r) {
        uint64_t ol = 0;
        CK(cudaSetDevice(ctx[0]->device));
        const int rc2 = plzgpu_decompress(ctx[0], img, len, out, cap, &ol, ctx[0]->stream, err);
        if (rc2) return rc2;
        if (err) *err = errs[r];
        return rcs[r];
    };
    for (uint64_t r = 0; r < N; ++r)
        if (rcs[r]) return report(r);
    const uint64_t T = total[0];
    run_ranks(N, [&](uint64_t r) {
        plzgpu_ctx* c = ctx[r];
        plzgpu_error* err = &errs[r];
        rcs[r] = [&]() -> int {
            CK(cudaSetDevice(c->device));
            const uint64_t cb = T * r / N, ce = T * (r + 1) / N;
            uint64_t tc = 0;
            int rc2 = plzgpu_decompress_range(c, src[r], len, cb, ce, nullptr, 0, &begin[r],
                                              &size[r], &tc, c->stream, err);
            if (rc2 || size[r] == 0) return rc2;
            if (begin[r] + size[r] > cap)
                return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                               "output buffer too small: need %llu bytes",
                               (unsigned long long)(begin[r] + size[r]));
            uint64_t b2 = 0, l2 = 0;
            if (out_dev >= 0 && peer_ok(c->device, out_dev))  // straight into `out`
                return plzgpu_decompress_range(c, src[r], len, cb, ce,
                                               static_cast<uint8_t*>(out) + begin[r], size[r],
                                               &b2, &l2, &tc, c->stream, err);
            CK(c->out.ensure(size[r] + 16));
            rc2 = plzgpu_decompress_range(c, src[r], len, cb, ce, c->out.p, size[r] + 16, &b2, &l2,
                                          &tc, c->stream, err);
            if (rc2) return rc2;
            if (out_dev >= 0)
                CK(cudaMemcpyPeerAsync(static_cast<uint8_t*>(out) + begin[r], out_dev, c->out.p,
                                       c->device, size[r], c->stream));
            else
                CK(cudaMemcpyAsync(static_cast<uint8_t*>(out) + begin[r], c->out.p, size[r],
                                   cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            return PLZGPU_OK;
        }();
    });
    for (uint64_t r = 0; r < N; ++r)
        if (rcs[r]) return report(r);
    *out_len = begin[N - 1] + size[N - 1];
    return PLZGPU_OK;
}

}  // extern "C"
