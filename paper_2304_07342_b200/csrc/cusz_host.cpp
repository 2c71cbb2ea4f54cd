// cusz_host.cpp — the cuSZ dual-quantization entry points (SURVEY.md §8f
// rank 4): Lorenzo quantizer with outlier list, and its
// inverse, keeping field -> codes -> GPULZ image -> field in HBM.
#include <cstring>

#include "host_internal.h"

using namespace plzhost;

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

extern "C" {

int plzgpu_lorenzo_quantize(plzgpu_ctx* c, const float* d_field, uint64_t nx, uint64_t ny,
                            uint64_t nz, double eb, int32_t radius, uint16_t* d_codes,
                            uint64_t* d_outlier_idx, int32_t* d_outlier_val, uint64_t outlier_cap,
                            uint64_t* n_outliers, void* stream, plzgpu_error* err) {
    clear_err(err);
    DeviceGuard keep;
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
    DeviceGuard keep;
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

}  // extern "C"
