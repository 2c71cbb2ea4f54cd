// host_pipeline.cpp — the host-buffer paths of plzgpu_compress /
// plzgpu_decompress: the input streams to the device in segments while the
// kernels run (ready flags written by stream memory operations after each
// segment's copy, waited on per chunk by the kernels), and results stream
// back while later work is still running.  Tuning knobs: PipelineConfig.
#include <cstring>

#include "host_internal.h"

namespace plzhost {

namespace {

// A pipelined compress of a host input: one container at a time on `st` —
// its Kernel I passes (waiting on the container's H2D segments) and its
// scan, continuing the earlier containers' prefixes — and its Kernel III +
// header on c->asm_stream, writing into `img` while `st` goes on with the
// next container.
int enqueue_compress_by_container(plzgpu_ctx* c, const plzgpu_params& p, const uint8_t* d_in,
                                  uint64_t n, uint8_t* img, cudaStream_t st, plzgpu_error* err) {
    const Geometry g = geometry(n, p);
    if (!c->asm_stream) CK(cudaStreamCreateWithFlags(&c->asm_stream, cudaStreamNonBlocking));
    for (cudaEvent_t& ev : c->asm_ev)
        if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    Meta* m = dmeta(c);
    while (c->cont_ev.size() < 2 * g.n_blocks) {
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        c->cont_ev.push_back(ev);
    }
    int launches = 0;
    for (uint64_t j = 0; j < g.n_blocks; ++j) {
        const uint64_t g0 = j * g.cpb, g1 = std::min(g.n_chunks, g0 + g.cpb);
        // (no side-stream passes here: Kernel III of the previous container
        // is running on the assembly stream)
        int rc = enqueue_encode_scan(c, p, d_in, g.n_chunks, g.last_len, st, err, &launches, true,
                                     g0, g1, false);
        if (rc) return rc;
        CK(cudaEventRecord(c->cont_ev[2 * j], st));
        CK(cudaEventRecord(c->asm_ev[0], st));
        CK(cudaStreamWaitEvent(c->asm_stream, c->asm_ev[0], 0));
        AssembleArgs a{};
        fill_assemble_args(c, p, g, d_in, img, &m->img_len, &a);
        a.j_lo = j;
        a.j_hi = j + 1;
        launch_assemble(a, c->asm_stream);
        launch_headers(a, c->asm_stream);
        CK(cudaEventRecord(c->cont_ev[2 * j + 1], c->asm_stream));
        launches += 2;
    }
    CK(cudaEventRecord(c->asm_ev[1], c->asm_stream));
    CK(cudaStreamWaitEvent(st, c->asm_ev[1], 0));
    CK(cudaGetLastError());
    c->last_launches = launches;
    c->last_op = OP_COMPRESS;
    return PLZGPU_OK;
}

}  // namespace

// Compress of a host input.  With several flag segments the input goes up on
// the copy stream while Kernel I runs (each warp waits for its chunk's
// segment); into a pinned host image of several containers the compress
// runs container by container and each finished container goes down on its
// own stream.  *img_out: where the image is on the device (unless
// *direct_out: already in `out`).
int compress_host_input(plzgpu_ctx* c, const plzgpu_params& p, const uint8_t* in, uint64_t n,
                        uint8_t* out, uint64_t cap, uint8_t** img_out, bool* direct_out,
                        cudaStream_t st, plzgpu_error* err) {
    const PipelineConfig& cfg = pipeline_config();
    const uint64_t bound = plzgpu_compress_bound(n, &p);
    const Geometry geo = geometry(n, p);
    const uint64_t chunk_bytes = uint64_t(p.chunk_size) * p.symbol_width;
    const uint64_t seg_chunks = std::max<uint64_t>(1, cfg.seg_bytes / chunk_bytes);
    const uint64_t nseg = (geo.n_chunks + seg_chunks - 1) / seg_chunks;
    void* mapped = nullptr;
    const bool per_container =
        nseg > 1 && geo.n_blocks > 1 && cap >= bound && is_pinned_host(out) &&
        geo.cpb % 4 == 0 && geo.cpb % seg_chunks == 0 && !cfg.no_pipe_asm && !cfg.no_pipe &&
        (cudaHostGetDevicePointer(&mapped, out, 0) == cudaSuccess || (cudaGetLastError(), false));
    const bool direct = (is_device_ptr(out) || per_container) && cap >= bound;
    uint8_t* img = out;
    if (per_container && cfg.asm_mapped) {
        img = static_cast<uint8_t*>(mapped);
    } else if (per_container || !direct) {
        CK(c->img.ensure(bound));
        img = c->img.as<uint8_t>();
    }
    *img_out = img;
    *direct_out = direct;
    Meta* m = dmeta(c);
    CK(c->in.ensure(n));
    const uint8_t* d_in = c->in.as<uint8_t>();
    const StreamValue32Fn write_value = stream_write_value32();
    if (!write_value || nseg < 2 || cfg.no_pipe) {
        CK(cudaMemcpyAsync(c->in.p, in, n, cudaMemcpyHostToDevice, st));
        return enqueue_compress(c, p, d_in, n, img, &m->img_len, st, err);
    }
    // H2D pipeline: Kernel I starts at once and each warp waits for its
    // chunk's segment; segments land on the copy stream, each followed by a
    // stream memory write of its ready flag.
    bool fresh = false;
    CK(c->ready.ensure(nseg * 4, &fresh));
    if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    if (fresh) {  // a recycled allocation may hold any value
        CK(cudaMemsetAsync(c->ready.p, 0, c->ready.cap, st));
        CK(cudaStreamSynchronize(st));
    }
    c->epoch = next_epoch();
    auto enqueue_copies = [&]() -> int {
        const uint64_t seg_bytes = seg_chunks * chunk_bytes;
        const uint64_t per_copy = std::max<uint64_t>(1, cfg.copy_bytes / seg_bytes);
        const uint64_t tail_from = n > cfg.tail_bytes ? n - cfg.tail_bytes : 0;
        for (uint64_t sgi = 0; sgi < nseg;) {
            const uint64_t lo = sgi * seg_bytes;
            const uint64_t s_end = lo >= tail_from ? sgi + 1 : std::min(nseg, sgi + per_copy);
            const uint64_t hi = s_end == nseg ? n : std::min(n, s_end * seg_bytes);
            CK(cudaMemcpyAsync(c->in.as<uint8_t>() + lo, in + lo, hi - lo, cudaMemcpyHostToDevice,
                               c->copy_stream));
            for (; sgi < s_end; ++sgi)
                if (write_value(c->copy_stream,
                                reinterpret_cast<unsigned long long>(c->ready.as<uint32_t>() + sgi),
                                c->epoch, 0) != 0)
                    return set_err(err, PLZGPU_CUDA, 0, kNoIndex, kNoIndex,
                                   "cuStreamWriteValue32 failed");
        }
        return PLZGPU_OK;
    };
    // A pinned input: the copies first, so the H2D stream starts before the
    // launches are enqueued.  A pageable input: each copy returns only once
    // the driver has staged its bytes, so the kernels go first (they wait
    // for the flags) and the staging overlaps the matching.
    const bool pinned_in = is_pinned_host(in);
    int rc = PLZGPU_OK;
    if (pinned_in && (rc = enqueue_copies())) return rc;
    c->pipe_ready = c->ready.as<uint32_t>();
    c->pipe_seg_chunks = uint32_t(seg_chunks);
    rc = per_container ? enqueue_compress_by_container(c, p, d_in, n, img, st, err)
                       : enqueue_compress(c, p, d_in, n, img, &m->img_len, st, err);
    c->pipe_ready = nullptr;
    if (rc) return rc;
    if (!pinned_in) {  // pageable: staged by the copy pool when large
        rc = use_staged(in, n) ? h2d_pageable(c, c->in.as<uint8_t>(), in, n, st, false,
                                              c->ready.as<uint32_t>(), seg_chunks * chunk_bytes,
                                              c->epoch, err)
                               : enqueue_copies();
        if (rc) return rc;
    }
    if (!per_container || cfg.asm_mapped) return PLZGPU_OK;
    // each container's image range is known once its scan is done (global
    // stream prefixes P64 / F64 at its first and last chunk): read the four
    // words, then send the range down after assembly
    for (cudaStream_t* sx : {&c->d2h_stream, &c->size_stream})
        if (!*sx) CK(cudaStreamCreateWithFlags(sx, cudaStreamNonBlocking));
    if (!c->host_scratch)
        CK(cudaMallocHost(reinterpret_cast<void**>(&c->host_scratch), 4 * sizeof(uint64_t)));
    uint64_t off = 0;
    for (uint64_t j = 0; j < geo.n_blocks; ++j) {
        const uint64_t g0 = j * geo.cpb, g1 = std::min(geo.n_chunks, g0 + geo.cpb);
        CK(cudaStreamWaitEvent(c->size_stream, c->cont_ev[2 * j], 0));
        const uint64_t* src[4] = {c->p64.as<uint64_t>() + g0, c->p64.as<uint64_t>() + g1,
                                  c->f64.as<uint64_t>() + g0, c->f64.as<uint64_t>() + g1};
        for (int k = 0; k < 4; ++k)
            CK(cudaMemcpyAsync(c->host_scratch + k, src[k], 8, cudaMemcpyDeviceToHost,
                               c->size_stream));
        CK(cudaStreamSynchronize(c->size_stream));
        const uint64_t* v = c->host_scratch;
        const uint64_t tail = j + 1 == geo.n_blocks ? n % uint64_t(p.symbol_width) : 0;
        const uint64_t size = 26 + 8 * (g1 - g0 + 1) + (v[3] - v[2]) + (v[1] - v[0]) + tail;
        if (off + size > cap) break;  // an offset overflow: reported by the caller
        CK(cudaStreamWaitEvent(c->d2h_stream, c->cont_ev[2 * j + 1], 0));
        CK(cudaMemcpyAsync(out + off, img + off, size, cudaMemcpyDeviceToHost, c->d2h_stream));
        off += size;
    }
    CK(cudaStreamSynchronize(c->d2h_stream));
    return PLZGPU_OK;
}

// Host image -> pinned host output, all three legs overlapped: the image
// goes up in segments (copy_stream, ready flags as in plzgpu_compress), the
// decode kernel waits per chunk for the segment its streams end in, and
// each decoded output segment goes down (asm_stream) as soon as the kernel
// has counted all of its bytes.  The container walk runs on the host over
// the caller's image; anything it does not accept as well-formed — and any
// error the kernel sees — falls back to the resident path, which reports
// the reference's exact error.  Returns 1 when it produced the output.
int try_decompress_pipelined(plzgpu_ctx* c, const uint8_t* img, uint64_t len, uint8_t* out,
                             uint64_t cap, uint64_t* out_len, cudaStream_t st,
                             plzgpu_error* err) {
    // Ready flags every seg_in bytes of image, output counters every seg_out
    // bytes; the first kLead transfers each way move one segment, later ones
    // kGroup segments at a time.  Env overrides for A/B (2/4 MiB segments
    // with 4 single and then 8-segment transfers measured no faster).
    const PipelineConfig& cfg = pipeline_config();
    const uint64_t seg_in = cfg.dseg_in, seg_out = cfg.dseg_out;
    const uint64_t kLead = cfg.dseg_lead, kGroup = cfg.dseg_group, kGroupOut = cfg.dseg_group_out;
    const StreamValue32Fn write_value = stream_write_value32();
    const StreamValue32Fn wait_value = stream_wait_value32();
    if (!write_value || !wait_value || cfg.no_pipe_dec || cfg.no_pipe) return 0;
    // the container walk (format.cpp:112-185 on a well-formed image)
    std::vector<ContainerDesc> descs;
    uint64_t at = 0, total_out = 0, total_chunks = 0;
    while (at < len) {
        const uint8_t* b = img + at;
        const uint64_t size = len - at;
        if (size < 26 || b[0] != 'P' || b[1] != 'L' || b[2] != 'Z' || b[3] != '1' || b[4] != 1 ||
            b[8] != 0)
            return 0;
        const uint32_t S = b[5], W = b[6], I = b[7], C = host_le32(b + 9);
        if ((S != 1 && S != 2 && S != 4) || W < 4 || W > 255 || C <= W ||
            (C != 1024 && C != 2048 && C != 4096 && C != 8192 && C != 16384) ||
            (I != 1 && I != 2 && I != 4 && I != 8 && I != 16) || b[25] >= S)
            return 0;
        const uint64_t n = host_le32(b + 21), tail = b[25];
        if (size < 26 + 8 * (n + 1)) return 0;
        const uint8_t* ptab = b + 26;
        const uint8_t* ftab = ptab + 4 * (n + 1);
        const uint64_t ptot = host_le32(ptab + 4 * n), ftot = host_le32(ftab + 4 * n);
        const uint64_t orig = uint64_t(host_le32(b + 13)) | uint64_t(host_le32(b + 17)) << 32;
        const uint64_t need = 26 + 8 * (n + 1) + ftot + ptot + tail;
        if (host_le32(ptab) != 0 || host_le32(ftab) != 0 || size < need || orig < tail ||
            (orig - tail) % S != 0 || ((orig - tail) / S + C - 1) / C != n ||
            total_out + orig > cap)
            return 0;
        ContainerDesc d{};
        d.img_off = at;
        d.out_off = total_out;
        d.chunk_base = total_chunks;
        d.flags_off = at + 26 + 8 * (n + 1);
        d.payload_off = d.flags_off + ftot;
        d.payload_len = ptot;
        d.original_len = orig;
        d.num_chunks = uint32_t(n);
        d.chunk_size = C;
        d.last_len = n ? uint32_t((orig - tail) / S - (n - 1) * C) : 0u;
        d.S = uint8_t(S);
        d.W = uint8_t(W);
        d.I = uint8_t(I);
        d.tail_len = uint8_t(tail);
        descs.push_back(d);
        at += need;
        total_out += orig;
        total_chunks += n;
    }
    if (descs.empty() || total_chunks == 0) return 0;
    const uint64_t nseg_in = (len + seg_in - 1) / seg_in;
    const uint64_t nseg_out = (total_out + seg_out - 1) / seg_out;
    if (nseg_in < 2 && nseg_out < 2) return 0;  // nothing to overlap
    // decoded bytes each output segment receives from chunks (tails excluded)
    std::vector<uint32_t> expect(nseg_out, 0);
    for (const ContainerDesc& d : descs) {
        const uint64_t o0 = d.out_off, o1 = d.out_off + d.original_len - d.tail_len;
        for (uint64_t sg = o0 / seg_out; sg * seg_out < o1; ++sg)
            expect[sg] += uint32_t(std::min(o1, (sg + 1) * seg_out) - std::max(o0, sg * seg_out));
    }
    if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    if (!c->asm_stream) CK(cudaStreamCreateWithFlags(&c->asm_stream, cudaStreamNonBlocking));
    if (!c->asm_ev[0]) {
        CK(cudaEventCreateWithFlags(&c->asm_ev[0], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->asm_ev[1], cudaEventDisableTiming));
    }
    CK(c->img.ensure(len + 16));
    CK(c->out.ensure(total_out + 16));
    bool fresh = false;
    CK(c->ready.ensure(nseg_in * 4, &fresh));
    if (fresh) CK(cudaMemsetAsync(c->ready.p, 0, c->ready.cap, st));  // recycled bytes
    CK(c->done.ensure(nseg_out * 4));
    CK(c->desc.ensure(std::max<uint64_t>(descs.size(), 64) * sizeof(ContainerDesc)));
    Meta* m = dmeta(c);
    c->epoch = next_epoch();
    ParseResult pr{};
    pr.n_containers = descs.size();
    pr.total_chunks = total_chunks;
    pr.total_out = total_out;
    uint32_t kinds = 0;
    for (const ContainerDesc& d : descs)
        if (d.num_chunks) kinds |= d.S == 2 ? 2u : d.S == 4 ? 4u : 1u;
    pr.absent_kinds = ~kinds & 7u;
    CK(cudaMemcpyAsync(c->desc.p, descs.data(), descs.size() * sizeof(ContainerDesc),
                       cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(&m->parse, &pr, sizeof pr, cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(&m->err_chunk, 0xff, sizeof m->err_chunk + sizeof m->mono_key, st));
    CK(cudaMemsetAsync(m->work, 0, sizeof m->work + sizeof m->stalled, st));
    CK(cudaMemsetAsync(c->done.p, 0, nseg_out * 4, st));
    CK(cudaEventRecord(c->asm_ev[0], st));
    DecodeArgs a{};
    a.img = c->img.as<uint8_t>();
    a.img_len = len;
    a.out = c->out.as<uint8_t>();
    a.out_cap = cap;
    a.desc = c->desc.as<ContainerDesc>();
    a.desc_cap = c->desc.cap / sizeof(ContainerDesc);
    a.result = &m->parse;
    a.err_chunk = &m->err_chunk;
    a.mono_key = &m->mono_key;
    a.work = &m->work[2];
    DecodePipe pp{};
    pp.in_ready = c->ready.as<uint32_t>();
    pp.epoch = c->epoch;
    pp.stalled = &m->stalled;
    pp.in_seg = seg_in;
    pp.out_done = c->done.as<uint32_t>();
    pp.out_seg = seg_out;
    // the image up, segment by segment, after the flags' reset above (a
    // large pageable image: staged by the copy pool, after the launch below)
    const bool staged = use_staged(img, len);
    CK(cudaStreamWaitEvent(c->copy_stream, c->asm_ev[0], 0));
    for (uint64_t sg = staged ? nseg_in : 0; sg < nseg_in;) {
        const uint64_t s_end = std::min(nseg_in, sg + (sg < kLead ? 1 : kGroup));
        const uint64_t lo = sg * seg_in, hi = std::min(len, s_end * seg_in);
        CK(cudaMemcpyAsync(c->img.as<uint8_t>() + lo, img + lo, hi - lo, cudaMemcpyHostToDevice,
                           c->copy_stream));
        for (; sg < s_end; ++sg)
            if (write_value(c->copy_stream, reinterpret_cast<unsigned long long>(pp.in_ready + sg),
                            c->epoch, 0) != 0)
                return 0;
    }
    launch_decode_pipelined(a, pp, c->sms, st);
    CK(cudaGetLastError());
    if (staged) {
        const int rc = h2d_pageable(c, c->img.as<uint8_t>(), img, len, st, false, pp.in_ready, seg_in,
                                    c->epoch, err);
        if (rc) return rc;
    }
    // the output down, each segment once its decoded bytes are counted
    CK(cudaStreamWaitEvent(c->asm_stream, c->asm_ev[0], 0));
    for (uint64_t sg = 0; sg < nseg_out;) {
        const uint64_t s_end = std::min(nseg_out, sg + (sg < kLead ? 1 : kGroupOut));
        const uint64_t lo = sg * seg_out, hi = std::min(total_out, s_end * seg_out);
        for (; sg < s_end; ++sg)
            if (wait_value(c->asm_stream, reinterpret_cast<unsigned long long>(pp.out_done + sg),
                           expect[sg], 0) != 0)
                return 0;
        CK(cudaMemcpyAsync(out + lo, a.out + lo, hi - lo, cudaMemcpyDeviceToHost, c->asm_stream));
    }
    CK(cudaEventRecord(c->asm_ev[1], c->asm_stream));
    CK(cudaStreamWaitEvent(st, c->asm_ev[1], 0));
    Meta* h = c->host_meta;
    CK(cudaMemcpyAsync(h, m, sizeof(Meta), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaStreamSynchronize(c->copy_stream));
    c->last_launches = 3;
    c->last_op = OP_DECOMPRESS;
    c->last_decode = a;
    if (h->stalled || h->err_chunk != ~0ull || h->mono_key != ~0ull) return 0;
    // raw tails straight from the image (decoder.cpp:123-125)
    for (const ContainerDesc& d : descs)
        if (d.tail_len)
            std::memcpy(out + d.out_off + d.original_len - d.tail_len,
                        img + d.payload_off + d.payload_len, d.tail_len);
    *out_len = total_out;
    return 1;
}

}  // namespace plzhost
