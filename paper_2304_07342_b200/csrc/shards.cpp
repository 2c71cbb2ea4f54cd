// shards.cpp — the chunk-range shard protocol of SURVEY.md §8e on the
// C-ABI side (plzgpu_shard_*): a rank encodes a contiguous chunk range
// (Kernels I+II), reports per-container stream totals, writes its rebased
// table and stream segments of the final image, and the root writes the
// container headers, last table entries and the tail.
#include <cstring>

#include "host_internal.h"

using namespace plzhost;

extern "C" {

// Segments of the final image a shard owns in one container:
// its slice of each offset table and of both streams.  Pure host arithmetic.
static uint64_t shard_segments_impl(const plzgpu_params& p, uint64_t n_total, uint64_t begin,
                                    uint64_t end, const uint64_t* totals, const uint64_t* bases,
                                    uint64_t n_touched, uint64_t* segs, uint64_t max_segs) {
    const Geometry g = geometry(n_total, p);
    uint64_t count = 0, local = 0;
    for (uint64_t i = 0; i < n_touched; ++i) {
        const uint64_t j = totals[3 * i];
        const uint64_t g0 = j * g.cpb;
        const uint64_t nj = (j + 1 == g.n_blocks) ? g.n_chunks - g0 : g.cpb;
        const uint64_t lo = std::max(begin, g0), hi = std::min(end, g0 + nj);
        const uint64_t k_lo = lo - g0, cnt = hi - lo;
        const uint64_t lp = totals[3 * i + 1], lf = totals[3 * i + 2];
        const uint64_t p_base = bases[4 * i], f_base = bases[4 * i + 1];
        const uint64_t img_off = bases[4 * i + 2], f_total = bases[4 * i + 3];
        const uint64_t tabs = img_off + 26, streams = tabs + 8 * (nj + 1);
        const uint64_t seg[4][2] = {{tabs + 4 * k_lo, 4 * cnt},
                                    {tabs + 4 * (nj + 1) + 4 * k_lo, 4 * cnt},
                                    {streams + f_base, lf},
                                    {streams + f_total + p_base, lp}};
        for (const auto& sg : seg) {
            if (count < max_segs && segs) {
                segs[3 * count] = sg[0];
                segs[3 * count + 1] = local;
                segs[3 * count + 2] = sg[1];
            }
            local += sg[1];
            ++count;
        }
    }
    return count;
}

uint64_t plzgpu_shard_segments(const plzgpu_params* p, uint64_t n_total, uint64_t chunk_begin,
                               uint64_t chunk_end, const uint64_t* totals, const uint64_t* bases,
                               uint64_t n_touched, uint64_t* segs, uint64_t max_segs) {
    return shard_segments_impl(*p, n_total, chunk_begin, chunk_end, totals, bases, n_touched, segs,
                               max_segs);
}

int plzgpu_shard_encode(plzgpu_ctx* c, const plzgpu_params* params, const void* in,
                        uint64_t n_total, uint64_t chunk_begin, uint64_t chunk_end,
                        uint64_t* totals, uint64_t max_touched, uint64_t* n_touched, void* stream,
                        plzgpu_error* err) {
    clear_err(err);
    *n_touched = 0;
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    const plzgpu_params& p = *params;
    const Geometry g = geometry(n_total, p);
    if (chunk_begin > chunk_end || chunk_end > g.n_chunks)
        return set_err(err, PLZGPU_CONTRACT, 0, kNoIndex, kNoIndex, "shard range outside the input");
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const uint64_t S = uint64_t(p.symbol_width), C = uint64_t(p.chunk_size);
    const uint64_t L = chunk_end - chunk_begin;
    const uint32_t last_len = chunk_end == g.n_chunks ? g.last_len : uint32_t(C);
    uint64_t local_bytes = L * C * S;
    if (chunk_end == g.n_chunks && L) local_bytes = n_total - chunk_begin * C * S;
    const uint8_t* d_in = static_cast<const uint8_t*>(in);
    if (L && !is_device_ptr(in)) {
        CK(c->in.ensure(local_bytes + 16));
        CK(cudaMemcpyAsync(c->in.p, in, local_bytes, cudaMemcpyHostToDevice, st));
        d_in = c->in.as<uint8_t>();
    }
    int launches = 0;
    rc = enqueue_encode_scan(c, p, d_in, L, last_len, st, err, &launches);
    if (rc) return rc;
    CK(cudaGetLastError());
    c->last_launches = launches;
    c->last_op = OP_COMPRESS;  // plzgpu_ctx_finish reports the shard's token counts
    // per touched container: local prefix values at its range ends
    c->sh_touch.clear();
    const uint64_t j_first = L ? chunk_begin / g.cpb : 0, j_last = L ? (chunk_end - 1) / g.cpb : 0;
    std::vector<uint64_t> idx;
    for (uint64_t j = j_first; L && j <= j_last; ++j) {
        const uint64_t lo = std::max(chunk_begin, j * g.cpb);
        const uint64_t hi = std::min(chunk_end, std::min((j + 1) * g.cpb, g.n_chunks));
        c->sh_touch.insert(c->sh_touch.end(), {j, lo, hi, 0, 0});
        idx.push_back(lo - chunk_begin);
        idx.push_back(hi - chunk_begin);
    }
    std::vector<uint64_t> pv(idx.size()), fv(idx.size());
    for (size_t i = 0; i < idx.size(); ++i) {
        CK(cudaMemcpyAsync(&pv[i], c->p64.as<uint64_t>() + idx[i], 8, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&fv[i], c->f64.as<uint64_t>() + idx[i], 8, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    const uint64_t nt = c->sh_touch.size() / 5;
    for (uint64_t i = 0; i < nt; ++i) {
        c->sh_touch[5 * i + 3] = pv[2 * i + 1] - pv[2 * i];
        c->sh_touch[5 * i + 4] = fv[2 * i + 1] - fv[2 * i];
        if (i < max_touched && totals) {
            totals[3 * i] = c->sh_touch[5 * i];
            totals[3 * i + 1] = c->sh_touch[5 * i + 3];
            totals[3 * i + 2] = c->sh_touch[5 * i + 4];
        }
    }
    c->sh_begin = chunk_begin;
    c->sh_end = chunk_end;
    c->sh_n = n_total;
    c->sh_params = p;
    *n_touched = nt;
    return PLZGPU_OK;
}

}  // extern "C"

namespace {
// Kernel III of a shard.  direct = false: the segments land back to back in
// d_out (local buffer, cap bytes); direct = true: d_out is the final image
// (possibly another GPU's memory, written over NVLink through peer access)
// and every segment lands at its image offset.
int shard_assemble_impl(plzgpu_ctx* c, const uint64_t* bases, void* d_out, uint64_t cap,
                        bool direct, uint64_t* segs, uint64_t max_segs, uint64_t* n_segs,
                        uint64_t* out_len, void* stream, plzgpu_error* err) {
    clear_err(err);
    *n_segs = 0;
    *out_len = 0;
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const plzgpu_params& p = c->sh_params;
    const uint64_t nt = c->sh_touch.size() / 5;
    std::vector<uint64_t> totals(3 * nt);
    for (uint64_t i = 0; i < nt; ++i) {
        totals[3 * i] = c->sh_touch[5 * i];
        totals[3 * i + 1] = c->sh_touch[5 * i + 3];
        totals[3 * i + 2] = c->sh_touch[5 * i + 4];
    }
    std::vector<uint64_t> sg(12 * nt + 3);
    const uint64_t ns = shard_segments_impl(p, c->sh_n, c->sh_begin, c->sh_end, totals.data(), bases,
                                            nt, sg.data(), 4 * nt);
    uint64_t total = 0, reach = 0;
    for (uint64_t i = 0; i < ns; ++i) {
        total += sg[3 * i + 2];
        reach = std::max(reach, sg[3 * i] + sg[3 * i + 2]);
    }
    if ((direct ? reach : total) > cap)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex, "shard buffer too small");
    const int at = direct ? 0 : 1;  // which offset of a segment the kernel writes at
    std::vector<ShardCont> conts(nt);
    for (uint64_t i = 0; i < nt; ++i) {
        const Geometry g = geometry(c->sh_n, p);
        ShardCont& d = conts[i];
        const uint64_t j = c->sh_touch[5 * i], lo = c->sh_touch[5 * i + 1];
        d.g_lo = lo - c->sh_begin;
        d.g_hi = c->sh_touch[5 * i + 2] - c->sh_begin;
        d.k_lo = lo - j * g.cpb;
        d.p_base = bases[4 * i];
        d.f_base = bases[4 * i + 1];
        d.seg_ptab = sg[3 * (4 * i) + at];
        d.seg_ftab = sg[3 * (4 * i + 1) + at];
        d.seg_flags = sg[3 * (4 * i + 2) + at];
        d.seg_pay = sg[3 * (4 * i + 3) + at];
    }
    if (nt) {
        CK(c->shard_desc.ensure(nt * sizeof(ShardCont)));
        CK(cudaMemcpyAsync(c->shard_desc.p, conts.data(), nt * sizeof(ShardCont),
                           cudaMemcpyHostToDevice, st));
        Meta* m = dmeta(c);
        CK(cudaMemsetAsync(&m->overflow, 0, sizeof m->overflow, st));
        ShardAssembleArgs a{};
        a.pay_slots = c->pay_slots.as<uint8_t>();
        a.flag_slots = c->flag_slots.as<uint8_t>();
        a.psize = c->psize.as<uint32_t>();
        a.fsize = c->fsize.as<uint32_t>();
        a.P64 = c->p64.as<uint64_t>();
        a.F64 = c->f64.as<uint64_t>();
        a.conts = c->shard_desc.as<ShardCont>();
        a.n_conts = nt;
        a.out = static_cast<uint8_t*>(d_out);
        a.overflow = &m->overflow;
        a.n_chunks = c->sh_end - c->sh_begin;
        a.S = p.symbol_width;
        a.C = p.chunk_size;
        launch_shard_assemble(a, st);
        CK(cudaGetLastError());
        c->last_launches = 1;
        Meta h;
        CK(cudaMemcpyAsync(&h, c->meta.p, sizeof h, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h.overflow) return overflow_error(err);
    }
    for (uint64_t i = 0; i < ns && i < max_segs && segs; ++i)
        for (int q = 0; q < 3; ++q) segs[3 * i + q] = sg[3 * i + q];
    *n_segs = ns;
    *out_len = total;
    return PLZGPU_OK;
}
}  // namespace

extern "C" {

int plzgpu_shard_assemble(plzgpu_ctx* c, const uint64_t* bases, void* d_out, uint64_t cap,
                          uint64_t* segs, uint64_t max_segs, uint64_t* n_segs, uint64_t* out_len,
                          void* stream, plzgpu_error* err) {
    return shard_assemble_impl(c, bases, d_out, cap, false, segs, max_segs, n_segs, out_len,
                               stream, err);
}

int plzgpu_shard_assemble_into(plzgpu_ctx* c, const uint64_t* bases, void* d_img,
                               uint64_t img_cap, void* stream, plzgpu_error* err) {
    uint64_t ns = 0, ln = 0;
    return shard_assemble_impl(c, bases, d_img, img_cap, true, nullptr, 0, &ns, &ln, stream, err);
}

int plzgpu_shard_headers(plzgpu_ctx* c, const plzgpu_params* params, uint64_t n_total,
                         const uint64_t* totals, const void* tail, void* d_img, uint64_t cap,
                         uint64_t* img_len, void* stream, plzgpu_error* err) {
    clear_err(err);
    *img_len = 0;
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    const plzgpu_params& p = *params;
    const Geometry g = geometry(n_total, p);
    std::vector<HeaderDesc> hd(g.n_blocks);
    uint64_t at = 0;
    for (uint64_t j = 0; j < g.n_blocks; ++j) {
        HeaderDesc& d = hd[j];
        const uint64_t g0 = j * g.cpb;
        d.n = uint32_t((j + 1 == g.n_blocks) ? g.n_chunks - g0 : g.cpb);
        d.byte_len = (j + 1 == g.n_blocks) ? n_total - j * p.block_bytes : p.block_bytes;
        d.tail_len = uint8_t(d.byte_len % uint64_t(p.symbol_width));
        for (int i = 0; i < d.tail_len; ++i) d.tail[i] = static_cast<const uint8_t*>(tail)[i];
        d.ptot = totals[2 * j];
        d.ftot = totals[2 * j + 1];
        if (d.ptot > 0xffffffffull || d.ftot > 0xffffffffull) return overflow_error(err);
        d.img_off = at;
        at += 26 + 8 * (uint64_t(d.n) + 1) + d.ptot + d.ftot + d.tail_len;
    }
    if (at > cap)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex, "image buffer too small");
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    if (g.n_blocks) {
        CK(c->shard_desc.ensure(g.n_blocks * sizeof(HeaderDesc)));
        CK(cudaMemcpyAsync(c->shard_desc.p, hd.data(), g.n_blocks * sizeof(HeaderDesc),
                           cudaMemcpyHostToDevice, st));
        launch_shard_headers(c->shard_desc.as<HeaderDesc>(), g.n_blocks,
                             static_cast<uint8_t*>(d_img), p.symbol_width, p.window, p.interval,
                             p.chunk_size, st);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));
    }
    *img_len = at;
    return PLZGPU_OK;
}

}  // extern "C"
