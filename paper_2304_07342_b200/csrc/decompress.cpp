// decompress.cpp — the decode side of the C-ABI: the container walk
// (format.cpp:112-185, plz_parse_kernel), the block-parallel chunk decode
// (decoder.cpp:22-141, plz_decode_kernel) and the mapping of the first
// failure onto the reference's exception, in the reference's order.
#include <cstring>

#include "host_internal.h"

using namespace plzhost;

namespace plzhost {

int enqueue_decompress(plzgpu_ctx* c, const uint8_t* d_img, uint64_t len, uint8_t* d_out,
                       uint64_t cap, uint64_t* d_out_len, cudaStream_t st, plzgpu_error* err) {
    Meta* m = dmeta(c);
    if (c->desc.cap < 64 * sizeof(ContainerDesc)) CK(c->desc.ensure(64 * sizeof(ContainerDesc)));
    CK(cudaMemsetAsync(&m->parse, 0, sizeof m->parse, st));
    CK(cudaMemsetAsync(&m->err_chunk, 0xff, sizeof m->err_chunk + sizeof m->mono_key, st));
    CK(cudaMemsetAsync(m->work, 0, sizeof m->work, st));
    DecodeArgs a{};
    a.img = d_img;
    a.img_len = len;
    a.out = d_out;
    a.out_cap = cap;
    a.desc = c->desc.as<ContainerDesc>();
    a.desc_cap = c->desc.cap / sizeof(ContainerDesc);
    a.result = &m->parse;
    a.out_len = d_out_len;
    a.err_chunk = &m->err_chunk;
    a.mono_key = &m->mono_key;
    a.work = &m->work[2];
    launch_parse(a, st);
    launch_decode(a, c->sms, st);
    CK(cudaGetLastError());
    c->last_launches = 4;  // parse + the three decode kernels
    c->last_op = OP_DECOMPRESS;
    c->last_decode = a;
    return PLZGPU_OK;
}

// After a decompress has completed: report its error, if any, in the
// reference's order (chunk errors of earlier containers before the parse
// error of a later one).  Sets *grow when the descriptor table overflowed.
int finish_decompress(plzgpu_ctx* c, cudaStream_t st, bool* grow, plzgpu_error* err) {
    Meta h;
    CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *grow = false;
    if (h.mono_key != ~0ull) {
        // a table-monotonicity violation in container j: chunk errors of
        // earlier containers come first (decoder order), then this one
        Meta* m = dmeta(c);
        launch_mono_detail(c->last_decode, h.mono_key, &m->mono_base, st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h.err_chunk == ~0ull || h.err_chunk >= h.mono_base) return parse_error(h.parse, err);
    }
    if (h.err_chunk != ~0ull) {
        Meta* m = dmeta(c);
        launch_chunk_detail(c->last_decode, &m->detail_code, &m->detail_chunk, &m->detail_token, st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return token_error(h.detail_code, h.detail_chunk, h.detail_token, err);
    }
    if (h.parse.err_kind == 17) {
        *grow = true;
        return PLZGPU_OK;
    }
    if (h.parse.err_kind != 0) return parse_error(h.parse, err);
    return PLZGPU_OK;
}

}  // namespace plzhost

extern "C" {

int plzgpu_decompressed_size(plzgpu_ctx* c, const void* img, uint64_t len, uint64_t* out_len,
                             void* stream, plzgpu_error* err) {
    clear_err(err);
    *out_len = 0;
    if (len == 0) return PLZGPU_OK;
    if (!is_device_ptr(img)) {
        *out_len = plzgpu_decompressed_bound(img, len);
        return PLZGPU_OK;
    }
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    for (;;) {
        if (c->desc.cap < 64 * sizeof(ContainerDesc)) CK(c->desc.ensure(64 * sizeof(ContainerDesc)));
        Meta* m = dmeta(c);
        CK(cudaMemsetAsync(&m->parse, 0, sizeof m->parse, st));
        DecodeArgs a{};
        a.img = static_cast<const uint8_t*>(img);
        a.img_len = len;
        a.out = nullptr;  // size-only walk: no tails copied
        a.out_cap = UINT64_MAX;
        a.desc = c->desc.as<ContainerDesc>();
        a.desc_cap = c->desc.cap / sizeof(ContainerDesc);
        a.result = &m->parse;
        launch_parse(a, st);
        CK(cudaGetLastError());
        Meta h;
        CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h.parse.err_kind == 17) {
            CK(c->desc.ensure(c->desc.cap * 4));
            continue;
        }
        *out_len = h.parse.total_out;
        return PLZGPU_OK;
    }
}

int plzgpu_decompress(plzgpu_ctx* c, const void* img, uint64_t len, void* out, uint64_t cap,
                      uint64_t* out_len, void* stream, plzgpu_error* err) {
    clear_err(err);
    *out_len = 0;
    if (len == 0) return PLZGPU_OK;
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const uint8_t* d_img = static_cast<const uint8_t*>(img);
    if (!is_device_ptr(img) && is_pinned_host(out) &&
        try_decompress_pipelined(c, static_cast<const uint8_t*>(img), len,
                                 static_cast<uint8_t*>(out), cap, out_len, st, err) == 1)
        return PLZGPU_OK;
    clear_err(err);  // the resident path below reports any error
    if (!is_device_ptr(img)) {
        CK(c->img.ensure(len));
        if (use_staged(img, len)) {
            const int rc = h2d_pageable(c, c->img.as<uint8_t>(), static_cast<const uint8_t*>(img),
                                        len, st, true, nullptr, 0, 0, err);
            if (rc) return rc;
        } else {
            CK(cudaMemcpyAsync(c->img.p, img, len, cudaMemcpyHostToDevice, st));
        }
        d_img = c->img.as<uint8_t>();
    }
    const bool direct = is_device_ptr(out) && (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    uint8_t* d_out = static_cast<uint8_t*>(out);
    if (!direct) {
        CK(c->out.ensure(cap + 16));
        d_out = c->out.as<uint8_t>();
    }
    for (;;) {
        int rc = enqueue_decompress(c, d_img, len, d_out, cap, nullptr, st, err);
        if (rc) return rc;
        bool grow = false;
        rc = finish_decompress(c, st, &grow, err);
        if (rc) return rc;
        if (!grow) break;
        CK(c->desc.ensure(c->desc.cap * 4));
    }
    Meta h;
    CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint64_t total = h.parse.total_out;
    if (!direct && total) {
        if (use_staged(out, total)) {
            const int rc = d2h_pageable(c, static_cast<uint8_t*>(out), d_out, total, st, err);
            if (rc) return rc;
        } else {
            CK(cudaMemcpyAsync(out, d_out, total,
                               is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                               st));
            CK(cudaStreamSynchronize(st));
        }
    }
    *out_len = total;
    return PLZGPU_OK;
}

int plzgpu_decompress_range(plzgpu_ctx* c, const void* img, uint64_t len, uint64_t chunk_begin,
                            uint64_t chunk_end, void* out, uint64_t cap, uint64_t* out_begin,
                            uint64_t* out_len, uint64_t* total_chunks, void* stream,
                            plzgpu_error* err) {
    clear_err(err);
    *out_begin = 0;
    *out_len = 0;
    *total_chunks = 0;
    if (len == 0) return PLZGPU_OK;
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const uint8_t* d_img = static_cast<const uint8_t*>(img);
    if (!is_device_ptr(img)) {
        CK(c->img.ensure(len));
        CK(cudaMemcpyAsync(c->img.p, img, len, cudaMemcpyHostToDevice, st));
        d_img = c->img.as<uint8_t>();
    }
    const bool query = out == nullptr;  // sizes only
    const bool direct = query || is_device_ptr(out);
    Meta* m = dmeta(c);
    // the header walk over the whole image (every container's checks), no
    // capacity check and no tails: the range kernel places those
    DecodeArgs a{};
    Meta h;
    for (;;) {
        if (c->desc.cap < 64 * sizeof(ContainerDesc)) CK(c->desc.ensure(64 * sizeof(ContainerDesc)));
        CK(cudaMemsetAsync(&m->parse, 0, sizeof m->parse, st));
        CK(cudaMemsetAsync(&m->err_chunk, 0xff, sizeof m->err_chunk + sizeof m->mono_key, st));
        CK(cudaMemsetAsync(m->work, 0, sizeof m->work, st));
        a = DecodeArgs{};
        a.img = d_img;
        a.img_len = len;
        a.out = nullptr;
        a.out_cap = UINT64_MAX;
        a.desc = c->desc.as<ContainerDesc>();
        a.desc_cap = c->desc.cap / sizeof(ContainerDesc);
        a.result = &m->parse;
        a.err_chunk = &m->err_chunk;
        a.mono_key = &m->mono_key;
        a.work = &m->work[2];
        launch_parse(a, st);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h.parse.err_kind == 17) {
            CK(c->desc.ensure(c->desc.cap * 4));
            continue;
        }
        break;
    }
    if (h.parse.err_kind != 0) return parse_error(h.parse, err);
    const uint64_t total = h.parse.total_chunks;
    const uint64_t ce = std::min(chunk_end, total), cb = std::min(chunk_begin, ce);
    // output range and tails: into the caller's buffer when it is device
    // memory, else into the staging buffer (copied back below)
    uint8_t* d_out = static_cast<uint8_t*>(out);
    if (!direct) {
        CK(c->out.ensure(cap + 16));
        d_out = c->out.as<uint8_t>();
    }
    launch_range(a, cb, ce, d_out, m->range, st);  // d_out null: bounds only
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint64_t lo = h.range[0], hi = h.range[1];
    *total_chunks = total;
    if (query) {
        *out_begin = lo;
        *out_len = hi - lo;
        return PLZGPU_OK;
    }
    if (hi - lo > cap)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                       "output buffer too small: need %llu bytes", (unsigned long long)(hi - lo));
    if (ce > cb) {
        // the decode kernel over [cb, ce): work counter from cb, bound ce,
        // output addressed relative to the range's first byte
        const uint32_t w0[3] = {uint32_t(cb), uint32_t(cb), uint32_t(cb)};  // the decode kernels' counters
        CK(cudaMemcpyAsync(&m->work[2], w0, sizeof w0, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(&m->parse.total_chunks, &ce, 8, cudaMemcpyHostToDevice, st));
        a.out = reinterpret_cast<uint8_t*>(reinterpret_cast<uintptr_t>(d_out) - lo);
        a.out_cap = hi;
        launch_decode(a, c->sms, st);
        CK(cudaGetLastError());
        c->last_launches = 5;
        c->last_op = OP_DECOMPRESS;
        c->last_decode = a;
        bool grow = false;
        const int rc = finish_decompress(c, st, &grow, err);
        if (rc) return rc;
    }
    if (!direct && hi > lo) {
        CK(cudaMemcpyAsync(out, d_out, hi - lo, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    *out_begin = lo;
    *out_len = hi - lo;
    return PLZGPU_OK;
}

int plzgpu_decompress_async(plzgpu_ctx* c, const void* d_img, uint64_t len, void* d_out,
                            uint64_t cap, uint64_t* d_out_len, void* stream, plzgpu_error* err) {
    clear_err(err);
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    if (reinterpret_cast<uintptr_t>(d_out) & 15u)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                       "async decompress needs a 16-byte aligned device output");
    if (len == 0) {
        CK(cudaMemsetAsync(d_out_len, 0, 8, st));
        Meta* m = dmeta(c);
        CK(cudaMemsetAsync(&m->parse, 0, sizeof m->parse, st));
        CK(cudaMemsetAsync(&m->err_chunk, 0xff, sizeof m->err_chunk + sizeof m->mono_key, st));
        c->last_launches = 0;
        c->last_op = OP_NONE;
        return PLZGPU_OK;
    }
    return enqueue_decompress(c, static_cast<const uint8_t*>(d_img), len,
                              static_cast<uint8_t*>(d_out), cap, d_out_len, st, err);
}

int plzgpu_decompress_chunk(plzgpu_ctx* c, const void* flags, uint64_t n_flags,
                            const void* payload, uint64_t n_payload, uint64_t logical,
                            const plzgpu_params* params, uint64_t chunk_index, void* out,
                            plzgpu_error* err) {
    clear_err(err);
    if (params->symbol_width != 1 && params->symbol_width != 2 && params->symbol_width != 4)
        return bad_field(err, "symbol_width", "{1,2,4}");
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = c->stream;  // private: synchronous call
    const uint64_t S = uint64_t(params->symbol_width);
    const uint64_t out_bytes = logical * S;
    // stage everything in one device scratch: flags | payload | out
    const uint64_t fo = 0, po = (n_flags + 15) & ~uint64_t(15);
    const uint64_t oo = po + ((n_payload + 15) & ~uint64_t(15));
    CK(c->in.ensure(oo + out_bytes + 16));
    uint8_t* base = c->in.as<uint8_t>();
    const bool dev_f = is_device_ptr(flags), dev_p = is_device_ptr(payload);
    if (n_flags)
        CK(cudaMemcpyAsync(base + fo, flags, n_flags,
                           dev_f ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    if (n_payload)
        CK(cudaMemcpyAsync(base + po, payload, n_payload,
                           dev_p ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    Meta* m = dmeta(c);
    DecodeOneArgs a{};
    a.flags = base + fo;
    a.n_flags = n_flags;
    a.payload = base + po;
    a.n_payload = n_payload;
    a.logical = logical;
    a.S = params->symbol_width;
    a.out = base + oo;
    a.err_code = &m->detail_code;
    a.err_token = &m->detail_token;
    launch_decode_one(a, st);
    CK(cudaGetLastError());
    c->last_launches = 1;
    Meta h;
    CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h.detail_code != TE_OK) return token_error(h.detail_code, chunk_index, h.detail_token, err);
    if (out_bytes)
        CK(cudaMemcpyAsync(out, base + oo, out_bytes,
                           is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                           st));
    CK(cudaStreamSynchronize(st));
    return PLZGPU_OK;
}

}  // extern "C"
