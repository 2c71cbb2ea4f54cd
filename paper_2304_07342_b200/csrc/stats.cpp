// stats.cpp — the matcher-side statistics of SURVEY.md §8f on the GPU:
// the full per-position match table (matcher.cpp:113-131) with its raw
// length histogram, and the histogram of the pointers the greedy encoder
// selects (corpus.cpp:75-129).
#include <cstring>

#include "host_internal.h"

using namespace plzhost;

namespace {
// the launch shape of the wide-cell pass (the match table runs in it)
void wide_shape(plzgpu_ctx* c, const plzgpu_params& p, int* wpc, int* per_sm) {
    int best = 0;
    *wpc = 1;
    *per_sm = 1;
    for (int cand = 1; cand <= 16; ++cand) {
        const int ctas = encode_ctas_per_sm(p.symbol_width, p.chunk_size, cand);
        if (ctas * cand > best) {
            best = ctas * cand;
            *wpc = cand;
            *per_sm = ctas;
        }
    }
    (void)c;
}
}  // namespace

extern "C" {

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
    DeviceGuard keep;
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
    wide_shape(c, p, &wpc, &per_sm);
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

int plzgpu_pointer_histogram(plzgpu_ctx* c, const plzgpu_params* params, const void* in,
                             uint64_t n, uint64_t* hist, void* stream, plzgpu_error* err) {
    clear_err(err);
    std::memset(hist, 0, 256 * sizeof(uint64_t));
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    const Geometry g = geometry(n, *params);
    if (g.n_chunks == 0) return PLZGPU_OK;
    DeviceGuard keep;
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

}  // extern "C"
