// peak.cu — FP64 roofline denominators measured on the box (MEASURED_PEAKS.json carries
// only HBM and bf16): a register-resident DFMA loop and a register-resident DMMA loop.
#include <cuda_profiler_api.h>

#include <algorithm>

#include "../../include/fastkf_b200.h"
#include "common.cuh"

namespace fkb {

__global__ void __launch_bounds__(256) k_peak_dfma(double* out, int iters, double seed) {
    double a[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = seed + threadIdx.x * 1e-9 + c;
    const double m = 0.999999, b = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) a[c] = fma(a[c], m, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += a[c];
    if (s == 12345.678) out[0] = s;  // keep the loop alive
}

__global__ void __launch_bounds__(256) k_peak_dmma(double* out, int iters, double seed) {
    double c[8][2];
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
    const double a = seed + threadIdx.x * 1e-9, b = 1.0 - seed;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[q][0]), "+d"(c[q][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
    if (s == 12345.678) out[0] = s;
}

}  // namespace fkb

extern "C" int fkb_set_device(int dev) { return cudaSetDevice(dev) == cudaSuccess ? 0 : 3; }
extern "C" int fkb_profiler(int on) {
    return (on ? cudaProfilerStart() : cudaProfilerStop()) == cudaSuccess ? 0 : 3;
}

extern "C" int fkb_fp64_peak(int mode, double* tflops) {
    // mode 0: DFMA, mode 1: DMMA.  Best of 3 timed launches (CUDA events).
    try {
        int dev = 0, sms = 0;
        FKB_CUDA(cudaGetDevice(&dev));
        FKB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        fkb::DBuf<double> out(1);
        cudaEvent_t e0, e1;
        FKB_CUDA(cudaEventCreate(&e0));
        FKB_CUDA(cudaEventCreate(&e1));
        const int blocks = sms * 8, threads = 256, iters = 4096;
        double best = 0.0;
        for (int rep = 0; rep < 4; ++rep) {
            FKB_CUDA(cudaEventRecord(e0));
            if (mode == 0) fkb::k_peak_dfma<<<blocks, threads>>>(out.p, iters, 0.5);
            else fkb::k_peak_dmma<<<blocks, threads>>>(out.p, iters, 0.5);
            FKB_CUDA(cudaEventRecord(e1));
            FKB_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            FKB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            const double flops = mode == 0 ? 2.0 * 8 * iters * double(blocks) * threads
                                           : 512.0 * 8 * iters * double(blocks) * (threads / 32);
            if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *tflops = best;
        return 0;
    } catch (const std::exception&) {
        return 3;
    }
}
