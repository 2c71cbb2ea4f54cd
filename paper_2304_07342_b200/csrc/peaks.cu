// peaks.cu — measured int32 lane-op throughput of the device (the
// denominator of Kernel I's integer roofline: SURVEY.md §8d asks for the
// int32 peak measured on the box, which MEASURED_PEAKS.json does not hold).
//
// Each thread runs 8 independent dependency chains of one SASS integer op
// (LOP3, IADD3, SHF funnel shift, POPC — the ops the bitmap matcher's inner
// loop issues), so the ALU pipe, not latency, is the limit; a persistent
// grid of 4 x 512-thread CTAs per SM.  Lane-ops/s = threads x iterations x 8
// / CUDA-event time of the launch (after a warm-up launch).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../../include/plzgpu.h"

namespace {

constexpr int kChains = 8;
constexpr int kThreads = 512;
constexpr int kUnroll = 16;

template <int OP>
__global__ void __launch_bounds__(kThreads) plz_int_peak_kernel(uint32_t* sink, int iters,
                                                                uint32_t seed) {
    uint32_t a[kChains];
    const uint32_t b = seed ^ (threadIdx.x * 0x9E3779B9u), c = blockIdx.x * 0x85EBCA6Bu + 7u;
#pragma unroll
    for (int j = 0; j < kChains; ++j) a[j] = threadIdx.x + 0x1000193u * uint32_t(j) + seed;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
            for (int j = 0; j < kChains; ++j) {
                if constexpr (OP == 0) {
                    asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[j]) : "r"(b), "r"(c));
                } else if constexpr (OP == 1) {
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(b));
                } else if constexpr (OP == 2) {
                    asm volatile("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(b), "r"(c));
                } else {
                    uint32_t t;
                    asm volatile("popc.b32 %0, %1;" : "=r"(t) : "r"(a[j]));
                    a[j] += t;  // IADD3 beside every POPC: counts two ops
                }
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < kChains; ++j) s ^= a[j];
    if (s == 0x2545F491u) sink[blockIdx.x * blockDim.x + threadIdx.x] = s;  // never taken, not dead
}

template <int OP>
cudaError_t run(int sms, int iters, uint32_t* sink, float* ms) {
    cudaEvent_t e0, e1;
    cudaError_t e = cudaEventCreate(&e0);
    if (e == cudaSuccess) e = cudaEventCreate(&e1);
    if (e != cudaSuccess) return e;
    const int grid = sms * 4;
    plz_int_peak_kernel<OP><<<grid, kThreads>>>(sink, iters / 8 + 1, 1u);  // warm-up
    cudaEventRecord(e0);
    plz_int_peak_kernel<OP><<<grid, kThreads>>>(sink, iters, 3u);
    cudaEventRecord(e1);
    e = cudaEventSynchronize(e1);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaEventElapsedTime(ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return e;
}

}  // namespace

extern "C" int plzgpu_int_peak(int device, int op, double* lane_ops_per_s, plzgpu_error* err) {
    *lane_ops_per_s = 0;
    auto fail = [&](cudaError_t c) {
        if (err) {
            err->code = PLZGPU_CUDA;
            err->byte_offset = 0;
            err->chunk_index = err->token_index = UINT64_MAX;
            snprintf(err->message, sizeof err->message, "plzgpu_int_peak: %s", cudaGetErrorString(c));
        }
        return PLZGPU_CUDA;
    };
    if (err) {
        err->code = PLZGPU_OK;
        err->message[0] = 0;
    }
    int saved = 0;
    cudaGetDevice(&saved);
    cudaError_t e = cudaSetDevice(device);
    int sms = 148;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    uint32_t* sink = nullptr;
    if (e == cudaSuccess) e = cudaMalloc(&sink, size_t(sms) * 4 * kThreads * 4);
    const int iters = 4096;
    float ms = 0;
    if (e == cudaSuccess) {
        switch (op) {
            case 0: e = run<0>(sms, iters, sink, &ms); break;
            case 1: e = run<1>(sms, iters, sink, &ms); break;
            case 2: e = run<2>(sms, iters, sink, &ms); break;
            default: e = run<3>(sms, iters, sink, &ms); break;
        }
    }
    if (sink) cudaFree(sink);
    cudaSetDevice(saved);
    if (e != cudaSuccess) return fail(e);
    // SASS lane-ops: ptxas pairs the chained adds of op 1 into one IADD3 each
    const double per = op == 1 ? 0.5 : op == 3 ? 2.0 : 1.0;
    const double ops = double(sms) * 4 * kThreads * double(iters) * kUnroll * kChains * per;
    *lane_ops_per_s = ops / (double(ms) * 1e-3);
    return PLZGPU_OK;
}
