// context.cpp — plzgpu_ctx lifetime (scratch, streams, pinned words), the
// once-per-device kernel preload and plzgpu_ctx_finish.
#include <cstring>
#include <mutex>
#include <new>

#include "host_internal.h"

using namespace plzhost;

namespace plzhost {

// Every kernel loaded once per device (see preload_kernel in kernels.h).
void preload_kernels(int device) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(done.begin(), done.end(), device) != done.end()) return;
    preload_bitmatch_kernels();
    preload_encode_kernels();
    preload_scan_kernels();
    preload_assemble_kernels();
    preload_decode_kernels();
    preload_cusz_kernels();
    done.push_back(device);
}

}  // namespace plzhost

extern "C" {

int plzgpu_abi_version(void) { return PLZGPU_ABI_VERSION; }

int plzgpu_ctx_create(int device, plzgpu_ctx** out, plzgpu_error* err) {
    clear_err(err);
    *out = nullptr;
    DeviceGuard keep;
    plzgpu_ctx* c = new (std::nothrow) plzgpu_ctx();
    if (!c) return set_err(err, PLZGPU_CUDA, 0, kNoIndex, kNoIndex, "out of host memory");
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = c->meta.ensure(sizeof(Meta));
    if (e == cudaSuccess) e = cudaMemset(c->meta.p, 0, sizeof(Meta));
    if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&c->host_meta), sizeof(Meta));
    if (e == cudaSuccess) preload_kernels(device);
    if (e != cudaSuccess) {
        plzgpu_ctx_destroy(c);
        return cuda_fail(err, e, "plzgpu_ctx_create");
    }
    *out = c;
    return PLZGPU_OK;
}

void plzgpu_ctx_destroy(plzgpu_ctx* c) {
    if (!c) return;
    DeviceGuard keep;
    cudaSetDevice(c->device);
    for (cudaStream_t sx : {c->stream, c->asm_stream, c->side_stream, c->d2h_stream, c->size_stream,
                            c->copy_stream, c->lat_stream[0], c->lat_stream[1], c->lat_stream[2],
                            c->lat_stream[3]})
        if (sx) cudaStreamSynchronize(sx);
    for (DevBuf* b : {&c->in, &c->img, &c->out, &c->pay_slots, &c->flag_slots, &c->psize,
                      &c->fsize, &c->p64, &c->f64, &c->status, &c->agg, &c->incl, &c->desc,
                      &c->meta, &c->fb, &c->shard_desc, &c->ready, &c->done, &c->hist, &c->table,
                      &c->qtiles, &c->qoff, &c->qdelta})
        b->release();
    if (c->host_meta) cudaFreeHost(c->host_meta);
    if (c->host_scratch) cudaFreeHost(c->host_scratch);
    for (uint8_t* b : c->bounce)
        if (b) cudaFreeHost(b);
    for (cudaStream_t sx : {c->stream, c->asm_stream, c->side_stream, c->d2h_stream, c->size_stream,
                            c->copy_stream, c->lat_stream[0], c->lat_stream[1], c->lat_stream[2],
                            c->lat_stream[3]})
        if (sx) cudaStreamDestroy(sx);
    for (cudaEvent_t ev : {c->side_ev[0], c->side_ev[1], c->asm_ev[0], c->asm_ev[1],
                           c->bounce_ev[0], c->bounce_ev[1], c->bounce_ev[2], c->order_ev,
                           c->lat_ev[0], c->lat_ev[1], c->lat_ev[2], c->lat_ev[3], c->lat_ev[4]})
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t ev : c->cont_ev)
        if (ev) cudaEventDestroy(ev);
    delete c;
}

void* plzgpu_ctx_stream(plzgpu_ctx* c) { return c->stream; }

int plzgpu_ctx_last_launches(plzgpu_ctx* c) { return c->last_launches; }

int plzgpu_ctx_finish(plzgpu_ctx* c, void* stream, plzgpu_stats* stats, plzgpu_error* err) {
    clear_err(err);
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    if (c->last_op == OP_DECOMPRESS) {
        bool grow = false;
        const int rc = finish_decompress(c, st, &grow, err);
        if (rc) return rc;
        if (grow)
            return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                           "too many containers for the async descriptor table; use "
                           "plzgpu_decompress once to size it");
        return PLZGPU_OK;
    }
    Meta* h = c->host_meta;
    CK(cudaMemcpyAsync(h, c->meta.p, sizeof(Meta), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (c->last_op == OP_COMPRESS) {
        if (h->overflow) return overflow_error(err);
        if (stats) {
            stats->max_cmp_per_pos = 0;
            stats->pointer_tokens = h->stats[0];
            stats->literal_tokens = h->stats[1];
        }
    }
    return PLZGPU_OK;
}

}  // extern "C"
