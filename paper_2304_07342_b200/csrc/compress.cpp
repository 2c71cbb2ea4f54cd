// compress.cpp — Kernels I-III enqueue for one compress call
// (pipeline.cpp:26-99: every container's chunks matched and encoded, the
// two global scans, deflate + container serialisation) and the C-ABI
// compress entry points.  Host-buffer inputs go through host_pipeline.cpp.
#include <cstring>

#include "host_internal.h"

using namespace plzhost;

namespace plzhost {

// Kernel III / header arguments over the whole input (every container).
void fill_assemble_args(plzgpu_ctx* c, const plzgpu_params& p, const Geometry& g,
                        const uint8_t* d_in, uint8_t* img, uint64_t* d_img_len, AssembleArgs* a) {
    *a = AssembleArgs{};
    a->in = d_in;
    a->pay_slots = c->pay_slots.as<uint8_t>();
    a->flag_slots = c->flag_slots.as<uint8_t>();
    a->psize = c->psize.as<uint32_t>();
    a->fsize = c->fsize.as<uint32_t>();
    a->P64 = c->p64.as<uint64_t>();
    a->F64 = c->f64.as<uint64_t>();
    a->img = img;
    a->img_len = d_img_len;
    a->overflow = &dmeta(c)->overflow;
    a->n_bytes = g.n_bytes;
    a->n_chunks = g.n_chunks;
    a->cpb = g.cpb;
    a->block_bytes = p.block_bytes;
    a->n_blocks = g.n_blocks;
    a->S = p.symbol_width;
    a->W = p.window;
    a->I = p.interval;
    a->C = p.chunk_size;
}

// Launch shape of Kernel I for (pass, S, C, W), cached per context: warps
// per CTA that maximise resident warps per SM (shared-memory limited).
// maxsyms: the bitmap pass's row budget (kBmMaxSyms / kBmMaxSymsWide), 0 for
// the wide-cell pass.  per_sm = 0: the pass does not fit.
static void encode_shape(plzgpu_ctx* c, const plzgpu_params& p, int maxsyms, int* wpc_out,
                  int* per_sm_out) {
    const int pass = maxsyms == 0 ? 0
                                  : (maxsyms == kBmMaxSyms ? 1 : maxsyms == kBmMaxSymsMid ? 5
                                                           : maxsyms == kBmMaxSymsWide ? 9 : 13) +
                                        __builtin_ctz(unsigned(bm_nw(p.window)));  // 0..16
    const int key = pass * 160 + p.symbol_width * 32 + (__builtin_ctz(unsigned(p.chunk_size)) - 10);
    int& wpc = c->enc_wpc[key];
    int& per_sm = c->enc_ctas[key];
    if (wpc == 0) {
        int best_warps = 0;
        for (int cand = 1; cand <= (maxsyms ? kBmMaxThreads / 32 : 16); ++cand) {
            const int ctas = maxsyms ? bitmatch_ctas_per_sm(p.symbol_width, p.chunk_size, p.window,
                                                            maxsyms, cand)
                                     : encode_ctas_per_sm(p.symbol_width, p.chunk_size, cand);
            if (ctas * cand > best_warps) {
                best_warps = ctas * cand;
                wpc = cand;
                per_sm = ctas;
            }
        }
        if (best_warps == 0) {  // does not fit (huge chunks): one warp, one CTA
            wpc = 1;
            per_sm = 0;
        }
    }
    *wpc_out = wpc;
    *per_sm_out = per_sm;
}

// Latency mode of Kernel I (inputs of at most a few waves of chunks, where a
// chunk's serial greedy walk — ~0.2 ms at c1 — is the time, not the
// throughput): every chunk's alphabet is counted first (plz_classify_kernel)
// and all tiers run at once on their own streams — the 64/32/12-row bitmap
// passes and the wide-cell pass over their short lists, then the 4-row pass,
// small enough in shared memory for a whole 16 MiB input in one wave, over
// the rest — instead of each tier starting when the previous one has found
// its overflow.  Returns -1 when a tier does not fit (huge chunks): the
// caller takes the sequential passes.
static int enqueue_tiers(plzgpu_ctx* c, const plzgpu_params& p, const EncodeArgs& e, uint64_t Gr,
                         cudaStream_t st, plzgpu_error* err, int* launches) {
    const int tiers[4] = {kBmMaxSymsTiny, kBmMaxSyms, kBmMaxSymsMid, kBmMaxSymsWide};
    int wpc[5], per_sm[5];
    for (int k = 0; k < 4; ++k) {
        encode_shape(c, p, tiers[k], &wpc[k], &per_sm[k]);
        if (per_sm[k] == 0) return -1;
    }
    encode_shape(c, p, 0, &wpc[4], &per_sm[4]);
    Meta* m = dmeta(c);
    CK(c->fb.ensure(6 * Gr * 4 + 16));
    uint32_t* L = c->fb.as<uint32_t>();  // list k at L + k * Gr; list 5: spills (none expected)
    CK(cudaMemsetAsync(m->lat_count, 0, sizeof m->lat_count + sizeof m->lat_work, st));
    launch_classify(p.symbol_width, e, L, Gr, m->lat_count,
                    int(std::min<uint64_t>(uint64_t(c->sms) * 16, (Gr + 3) / 4)), st);
    ++*launches;
    for (int i = 0; i < 4; ++i)
        if (!c->lat_stream[i]) CK(cudaStreamCreateWithFlags(&c->lat_stream[i], cudaStreamNonBlocking));
    for (cudaEvent_t& ev : c->lat_ev)
        if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(c->lat_ev[0], st));
    for (int i = 0; i < 4; ++i) CK(cudaStreamWaitEvent(c->lat_stream[i], c->lat_ev[0], 0));
    auto tier_args = [&](int k) {
        EncodeArgs b = e;
        b.work = &m->lat_work[k];
        b.src_list = L + uint64_t(k) * Gr;
        b.src_count = &m->lat_count[k];
        b.classify = 0;
        for (int i = 0; i < 3; ++i) {
            b.fb_list[i] = L + 5 * Gr;
            b.fb_count[i] = &m->lat_count[5];
        }
        b.warps_per_cta = wpc[k];
        return b;
    };
    // the short lists first, so their CTAs are placed before the 4-row
    // pass's fill the SMs (idle CTAs of an empty list exit at once)
    CK(launch_encode(p.symbol_width, tier_args(4), c->sms * std::max(per_sm[4], 1), c->lat_stream[3]));
    for (int k = 3; k >= 1; --k)
        CK(launch_bitmatch(p.symbol_width, tiers[k], tier_args(k), c->sms * per_sm[k],
                           c->lat_stream[k - 1]));
    CK(launch_bitmatch(p.symbol_width, tiers[0], tier_args(0), c->sms * per_sm[0], st));
    *launches += 5;
    for (int i = 0; i < 4; ++i) {
        CK(cudaEventRecord(c->lat_ev[1 + i], c->lat_stream[i]));
        CK(cudaStreamWaitEvent(st, c->lat_ev[1 + i], 0));
    }
    // chunks a tier could not hold after all (an exact count makes this list
    // empty): the wide-cell pass
    EncodeArgs f = tier_args(4);
    f.work = &m->lat_work[5];
    f.src_list = L + 5 * Gr;
    f.src_count = &m->lat_count[5];
    CK(launch_encode(p.symbol_width, f, c->sms, st));
    ++*launches;
    return PLZGPU_OK;
}

// Enqueue Kernels I-III for a device-resident input.  img must hold
// compress_bound bytes; img_len receives the image length on the device.
// Kernels I and II over G chunks starting at d_in (chunk g at g*C*S); the
// last of them has logical length last_len.  Leaves psize/fsize, staging
// slots and exclusive prefixes P64/F64[0..G] in the context.
// g0/g1 (a pipelined compress, one container at a time): only chunks
// [g0, g1) of the G; their prefixes continue from P64/F64[g0].
// Kernel II over chunks [g0, g0 + Gr) of the context's size arrays (status
// words and the tile counter cleared by the Kernel I enqueue).
static void enqueue_scan(plzgpu_ctx* c, uint64_t g0, uint64_t Gr, cudaStream_t st) {
    Meta* m = dmeta(c);
    ScanArgs sa{};
    sa.psize = c->psize.as<uint32_t>() + g0;
    sa.fsize = c->fsize.as<uint32_t>() + g0;
    sa.n = Gr;
    sa.P64 = c->p64.as<uint64_t>() + g0;
    sa.F64 = c->f64.as<uint64_t>() + g0;
    if (g0) {  // continue the earlier containers' totals
        sa.carry_p = c->p64.as<uint64_t>() + g0;
        sa.carry_f = c->f64.as<uint64_t>() + g0;
    }
    sa.status = c->status.as<uint32_t>();
    sa.agg = c->agg.as<ulonglong2>();
    sa.incl = c->incl.as<ulonglong2>();
    sa.tile_counter = &m->work[1];
    launch_scan(sa, st);
}

int enqueue_encode_scan(plzgpu_ctx* c, const plzgpu_params& p, const uint8_t* d_in, uint64_t G,
                        uint32_t last_len, cudaStream_t st, plzgpu_error* err, int* launches,
                        bool scan, uint64_t g0, uint64_t g1, bool side_passes) {
    const uint64_t S = uint64_t(p.symbol_width), C = uint64_t(p.chunk_size);
    if (g1 > G) g1 = G;
    const uint64_t Gr = g1 - g0;  // chunks of this call
    const uint64_t tiles = (G + kScanTile - 1) / kScanTile;
    CK(c->pay_slots.ensure(G * C * S + 64));
    CK(c->flag_slots.ensure(G * (C / 8) + 64));
    CK(c->psize.ensure(G * 4 + 64));
    CK(c->fsize.ensure(G * 4 + 64));
    CK(c->p64.ensure((G + 1) * 8));
    CK(c->f64.ensure((G + 1) * 8));
    CK(c->status.ensure(tiles * 4 + 4));
    CK(c->agg.ensure(tiles * 16 + 16));
    CK(c->incl.ensure(tiles * 16 + 16));
    Meta* m = dmeta(c);
    if (g0 == 0) {  // once per call: a later container must not clear an earlier stall
        CK(cudaMemsetAsync(&m->stats, 0, sizeof m->stats + sizeof m->overflow, st));
        CK(cudaMemsetAsync(&m->stalled, 0, sizeof m->stalled, st));
    }
    CK(cudaMemsetAsync(m->work, 0, sizeof m->work, st));
    if (G == 0) {
        CK(cudaMemsetAsync(c->p64.p, 0, 8, st));
        CK(cudaMemsetAsync(c->f64.p, 0, 8, st));
        return PLZGPU_OK;
    }
    const uint64_t rtiles = (Gr + kScanTile - 1) / kScanTile;
    CK(cudaMemsetAsync(c->status.p, 0, rtiles * 4, st));
    // ---- Kernel I
    const uint8_t* in0 = d_in + g0 * C * S;
    EncodeArgs e{};
    e.in = in0;
    e.pay_slots = c->pay_slots.as<uint8_t>() + g0 * C * S;
    e.flag_slots = c->flag_slots.as<uint8_t>() + g0 * (C / 8);
    e.psize = c->psize.as<uint32_t>() + g0;
    e.fsize = c->fsize.as<uint32_t>() + g0;
    e.stats = m->stats;
    e.work = &m->work[0];
    e.n_chunks = Gr;
    e.last_len = g1 == G ? last_len : uint32_t(C);
    e.C = p.chunk_size;
    e.W = p.window;
    e.I = p.interval;
    e.min_match = std::max(1, p.min_match);
    e.bulk_ok = (reinterpret_cast<uintptr_t>(in0) & 15u) == 0;
    e.ready = c->pipe_ready ? c->pipe_ready + g0 / c->pipe_seg_chunks : nullptr;
    e.epoch = c->epoch;
    e.seg_chunks = c->pipe_seg_chunks;
    e.stalled = &m->stalled;
    e.hist = c->enc_hist;
    // bitmap pass (12 rows) over every chunk, then the 32-row and 64-row
    // passes over what overflowed, then the wide-cell pass.  With few chunks
    // per resident warp the later passes' tails would add up, so the first
    // pass then sorts its overflow by exact alphabet size and the 32- and
    // 64-row passes run concurrently (two streams); otherwise they run one
    // after the other, each taking the previous one's overflow.
    CK(c->fb.ensure(3 * G * 4 + 16));
    uint32_t* lists[3] = {c->fb.as<uint32_t>(), c->fb.as<uint32_t>() + G,
                          c->fb.as<uint32_t>() + 2 * G};
    uint32_t* counts[3] = {&m->work[4], &m->work[6], &m->work[8]};
    uint32_t* works[4] = {&m->work[0], &m->work[5], &m->work[9], &m->work[7]};
    int wpc1 = 1, per_sm1 = 0;
    encode_shape(c, p, kBmMaxSyms, &wpc1, &per_sm1);
    const bool few = Gr < uint64_t(4) * c->sms * per_sm1 * wpc1;
    if (few && side_passes && !c->pipe_ready) {
        const int rc = enqueue_tiers(c, p, e, Gr, st, err, launches);
        if (rc != -1) {
            if (rc) return rc;
            goto scan;
        }
    }
    {
    const bool classify = side_passes && few;
    e.classify = classify ? 1 : 0;
    cudaError_t launch_err = cudaSuccess;  // first failed bitmap-pass launch
    auto bitmap_pass = [&](int maxsyms, int pass, const uint32_t* src, const uint32_t* src_n,
                           uint32_t* ovf, uint32_t* ovf_n, cudaStream_t s) -> bool {
        int wpc = 1, per_sm = 0;
        encode_shape(c, p, maxsyms, &wpc, &per_sm);
        if (per_sm == 0) return false;
        EncodeArgs b = e;
        b.work = works[pass];
        b.src_list = src;
        b.src_count = src_n;
        if (src) {
            b.ready = nullptr;  // every segment has landed after the first pass
            b.classify = 0;
            for (int i = 0; i < 2; ++i) {
                b.fb_list[i] = ovf;
                b.fb_count[i] = ovf_n;
            }
        }
        b.warps_per_cta = wpc;
        // a pipelined compress leaves one CTA slot per SM for the previous
        // container's Kernel III on the assembly stream
        const int resident = side_passes ? per_sm : std::max(1, per_sm - 1);
        const uint64_t ctas = std::min<uint64_t>(uint64_t(c->sms) * resident, (Gr + wpc - 1) / wpc);
        const cudaError_t le = launch_bitmatch(p.symbol_width, maxsyms, b, int(ctas), s);
        if (le != cudaSuccess && launch_err == cudaSuccess) launch_err = le;
        ++*launches;
        return true;
    };
    for (int i = 0; i < 3; ++i) {
        e.fb_list[i] = lists[i];
        e.fb_count[i] = counts[i];
    }
    const uint32_t* wide_src = nullptr;
    const uint32_t* wide_n = nullptr;
    if (bitmap_pass(kBmMaxSyms, 0, nullptr, nullptr, nullptr, nullptr, st)) {
        bool mid, wide;
        if (classify) {
            if (!c->side_stream) CK(cudaStreamCreateWithFlags(&c->side_stream, cudaStreamNonBlocking));
            for (cudaEvent_t& ev : c->side_ev)
                if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            CK(cudaEventRecord(c->side_ev[0], st));
            CK(cudaStreamWaitEvent(c->side_stream, c->side_ev[0], 0));
            mid = bitmap_pass(kBmMaxSymsMid, 1, lists[0], counts[0], lists[2], counts[2], st);
            wide = bitmap_pass(kBmMaxSymsWide, 2, lists[1], counts[1], lists[2], counts[2],
                               c->side_stream);
            CK(cudaEventRecord(c->side_ev[1], c->side_stream));
            CK(cudaStreamWaitEvent(st, c->side_ev[1], 0));
        } else {
            mid = bitmap_pass(kBmMaxSymsMid, 1, lists[0], counts[0], lists[1], counts[1], st);
            wide = bitmap_pass(kBmMaxSymsWide, 2, lists[1], counts[1], lists[2], counts[2], st);
        }
        if (!mid || !wide)
            return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                           "chunk too large for the bitmap passes' shared memory");
        wide_src = lists[2];
        wide_n = counts[2];
    }
    {
        int wpc = 1, per_sm = 1;
        encode_shape(c, p, 0, &wpc, &per_sm);
        EncodeArgs f = e;
        f.work = works[3];
        f.src_list = wide_src;
        f.src_count = wide_n;
        if (wide_src) f.ready = nullptr;
        f.warps_per_cta = wpc;
        CK(launch_encode(p.symbol_width, f,
                         int(std::min<uint64_t>(uint64_t(c->sms) * std::max(per_sm, 1),
                                                (Gr + wpc - 1) / wpc)),
                         st));
        ++*launches;
    }
    CK(launch_err);
    }
scan:
    if (!scan) return PLZGPU_OK;
    // ---- Kernel II
    enqueue_scan(c, g0, Gr, st);
    ++*launches;
    return PLZGPU_OK;
}

// Enqueue Kernels I-III for a device-resident input.  img must hold
// compress_bound bytes; img_len receives the image length on the device.
int enqueue_compress(plzgpu_ctx* c, const plzgpu_params& p, const uint8_t* d_in, uint64_t n,
                     uint8_t* img, uint64_t* d_img_len, cudaStream_t st, plzgpu_error* err,
                     int last_stage) {
    const Geometry g = geometry(n, p);
    const uint64_t G = g.n_chunks;
    int launches = 0;
    int rc = enqueue_encode_scan(c, p, d_in, G, g.last_len, st, err, &launches, last_stage > 1);
    if (rc) return rc;
    if (last_stage == 1) {
        CK(cudaGetLastError());
        c->last_launches = launches;
        c->last_op = OP_NONE;
        return PLZGPU_OK;
    }
    // ---- Kernel III + headers
    AssembleArgs a{};
    fill_assemble_args(c, p, g, d_in, img, d_img_len, &a);
    if (G > 0) {
        launch_assemble(a, st);
        ++launches;
    }
    launch_headers(a, st);
    ++launches;
    CK(cudaGetLastError());
    c->last_launches = launches;
    c->last_op = OP_COMPRESS;
    return PLZGPU_OK;
}
}  // namespace plzhost

extern "C" {

int plzgpu_compress(plzgpu_ctx* c, const plzgpu_params* params, const void* in, uint64_t n,
                    void* out, uint64_t cap, uint64_t* out_len, plzgpu_stats* stats, void* stream,
                    plzgpu_error* err) {
    clear_err(err);
    *out_len = 0;
    if (stats) std::memset(stats, 0, sizeof *stats);
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    if (n == 0) return PLZGPU_OK;  // empty input -> empty image (test_decoder.cpp:76-80)
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    Meta* m = dmeta(c);
    uint8_t* img = nullptr;
    bool direct = false;  // the image already sits in `out`
    if (!is_device_ptr(in)) {
        rc = compress_host_input(c, *params, static_cast<const uint8_t*>(in), n,
                                 static_cast<uint8_t*>(out), cap, &img, &direct, st, err);
    } else {
        const uint64_t bound = plzgpu_compress_bound(n, params);
        direct = is_device_ptr(out) && cap >= bound;
        img = static_cast<uint8_t*>(out);
        if (!direct) {
            CK(c->img.ensure(bound));
            img = c->img.as<uint8_t>();
        }
        rc = enqueue_compress(c, *params, static_cast<const uint8_t*>(in), n, img, &m->img_len, st,
                              err);
    }
    if (rc) return rc;
    Meta* h = c->host_meta;
    CK(cudaMemcpyAsync(h, m, sizeof(Meta), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h->stalled)
        return set_err(err, PLZGPU_CUDA, 0, kNoIndex, kNoIndex,
                       "H2D pipeline stalled: an input segment never arrived");
    if (h->overflow) return overflow_error(err);
    if (h->img_len > cap)
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                       "output buffer too small: need %llu bytes", (unsigned long long)h->img_len);
    if (!direct) {
        if (use_staged(out, h->img_len)) {
            rc = d2h_pageable(c, static_cast<uint8_t*>(out), img, h->img_len, st, err);
            if (rc) return rc;
        } else {
            CK(cudaMemcpyAsync(out, img, h->img_len,
                               is_device_ptr(out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                               st));
            CK(cudaStreamSynchronize(st));
        }
    }
    *out_len = h->img_len;
    if (stats) {
        stats->max_cmp_per_pos = 0;
        stats->pointer_tokens = h->stats[0];
        stats->literal_tokens = h->stats[1];
    }
    return PLZGPU_OK;
}

int plzgpu_compress_async(plzgpu_ctx* c, const plzgpu_params* params, const void* d_in,
                          uint64_t n, void* d_out, uint64_t cap, uint64_t* d_out_len, void* stream,
                          plzgpu_error* err) {
    clear_err(err);
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    if (cap < plzgpu_compress_bound(n, params))
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex,
                       "async compress needs cap >= plzgpu_compress_bound");
    if (n == 0) {
        CK(cudaMemsetAsync(d_out_len, 0, 8, st));
        Meta* m = dmeta(c);
        CK(cudaMemsetAsync(&m->stats, 0, sizeof m->stats + sizeof m->overflow, st));
        c->last_launches = 0;
        c->last_op = OP_COMPRESS;
        return PLZGPU_OK;
    }
    return enqueue_compress(c, *params, static_cast<const uint8_t*>(d_in), n,
                            static_cast<uint8_t*>(d_out), d_out_len, st, err);
}

int plzgpu_profile_encode(plzgpu_ctx* c, const plzgpu_params* params, const void* d_in,
                          uint64_t n, void* stream, plzgpu_error* err) {
    clear_err(err);
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    if (n == 0) return PLZGPU_OK;
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    return enqueue_compress(c, *params, static_cast<const uint8_t*>(d_in), n, nullptr, nullptr,
                            pick(c, stream), err, 1);
}


int plzgpu_profile_stages(plzgpu_ctx* c, const plzgpu_params* params, const void* d_in,
                          uint64_t n, void* d_img, uint64_t cap, int steps, double* ms,
                          void* stream, plzgpu_error* err) {
    clear_err(err);
    int rc = validate_fields(*params, err);
    if (rc) return rc;
    ms[0] = ms[1] = ms[2] = 0.0;
    if (n == 0 || steps <= 0) return PLZGPU_OK;
    if (cap < plzgpu_compress_bound(n, params))
        return set_err(err, PLZGPU_CAPACITY, 0, kNoIndex, kNoIndex, "image buffer below compress_bound");
    DeviceGuard keep;
    CK(cudaSetDevice(c->device));
    const cudaStream_t st = pick(c, stream);
    const plzgpu_params& p = *params;
    const Geometry g = geometry(n, p);
    cudaEvent_t ev[4];
    for (cudaEvent_t& e : ev) CK(cudaEventCreate(&e));
    int launches = 0;
    for (int s = 0; s < steps && rc == PLZGPU_OK; ++s) {
        CK(cudaEventRecord(ev[0], st));
        rc = enqueue_encode_scan(c, p, static_cast<const uint8_t*>(d_in), g.n_chunks, g.last_len,
                                 st, err, &launches, false);
        if (rc) break;
        CK(cudaEventRecord(ev[1], st));
        if (g.n_chunks) enqueue_scan(c, 0, g.n_chunks, st);
        CK(cudaEventRecord(ev[2], st));
        AssembleArgs a{};
        fill_assemble_args(c, p, g, static_cast<const uint8_t*>(d_in), static_cast<uint8_t*>(d_img),
                           &dmeta(c)->img_len, &a);
        if (g.n_chunks) launch_assemble(a, st);
        launch_headers(a, st);
        CK(cudaEventRecord(ev[3], st));
        CK(cudaEventSynchronize(ev[3]));
        for (int k = 0; k < 3; ++k) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, ev[k], ev[k + 1]));
            ms[k] += t / steps;
        }
    }
    for (cudaEvent_t& e : ev) cudaEventDestroy(e);
    CK(cudaGetLastError());
    c->last_op = OP_NONE;
    return rc;
}

}  // extern "C"
