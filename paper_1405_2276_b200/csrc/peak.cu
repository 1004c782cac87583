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

// L2→SM read bandwidth: every CTA sweeps an L2-resident buffer with 16-byte L1-bypassing
// loads (a warp reads 512 contiguous bytes per load), 8 loads in flight per thread.
__global__ void __launch_bounds__(256) k_peak_l2(const double2* __restrict__ a, long long n2, int passes,
                                                 double* out) {
    double acc = 0.0;
    for (int p = 0; p < passes; ++p) {
        const long long start = (blockIdx.x * 2654435761LL + p * 40503LL) % (n2 / 2048) * 2048;
        for (long long b = 0; b < n2; b += 8 * 256) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                long long i = start + b + u * 256 + threadIdx.x;
                i = i >= n2 ? i - n2 : i;
                v[u] = __ldcg(a + i);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
        }
    }
    if (acc == 12345.678) out[0] = acc;
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

// L2→SM read bandwidth in GB/s (best of 3 timed launches after a warm-up) over an L2-resident
// buffer of `mbytes` MB: the denominator for kernels whose traffic is served from L2 (the
// offline SpMM's X-row gathers).
extern "C" int fkb_l2_peak(int mbytes, double* gbs) {
    try {
        int dev = 0, sms = 0;
        FKB_CUDA(cudaGetDevice(&dev));
        FKB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const long long n2 = (long long)std::max(mbytes, 1) * (1 << 20) / 16 / 2048 * 2048;
        fkb::DBuf<double2> buf{static_cast<size_t>(n2)};
        fkb::DBuf<double> out(1);
        FKB_CUDA(cudaMemset(buf.p, 0, buf.bytes()));
        cudaEvent_t e0, e1;
        FKB_CUDA(cudaEventCreate(&e0));
        FKB_CUDA(cudaEventCreate(&e1));
        const int blocks = sms * 4, passes = 1;
        double best = 0.0;
        for (int rep = 0; rep < 4; ++rep) {
            FKB_CUDA(cudaEventRecord(e0));
            fkb::k_peak_l2<<<blocks, 256>>>(buf.p, n2, passes, out.p);
            FKB_CUDA(cudaEventRecord(e1));
            FKB_CUDA(cudaEventSynchronize(e1));
            float ms = 0;
            FKB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            const double bytes = 16.0 * double(n2) * blocks * passes;
            if (rep > 0) best = std::max(best, bytes / (ms * 1e-3) / 1e9);
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        *gbs = best;
        return 0;
    } catch (const std::exception&) {
        return 3;
    }
}
