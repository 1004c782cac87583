// Microbenchmark: does the 32 MB eigenvector matrix P stay L2-resident between the step's two
// rotations (r̃ = Pᵀr, then z = P·s̃)?  Times k_gemv_cm / k_coldot cold (after a 256 MB flush)
// and warm (right after a coldot over the same P).  Build (from repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1405_2276_b200/csrc \
//        scripts/microbench/l2reuse.cu -o scripts/microbench/l2reuse
#include <cstdio>

#include "gemv.cuh"

namespace fkb {
unsigned long long g_launches = 0;
int g_sync_check = 0;
void sync_check(const char*) {}
}  // namespace fkb

using namespace fkb;

struct EpiSt {
    double* y;
    __device__ __forceinline__ void operator()(long long i, double v) const { y[i] = v; }
};

template <int UNROLL>
__global__ void __launch_bounds__(256) k_read(const double2* __restrict__ a, long long n2, double* out) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    double acc = 0.0;
    for (; i + (UNROLL - 1) * stride < n2; i += UNROLL * stride) {
        double2 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc += v[u].x + v[u].y;
    }
    for (; i < n2; i += stride) acc += a[i].x + a[i].y;
    if (acc == 12345.678) out[0] = acc;
}

template <class F>
float time_ms(F&& f, int reps, cudaStream_t s) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps * 1e3f;  // us
}

int main() {
    cudaStream_t s;
    cudaStreamCreate(&s);
    const int m = 2048;
    double *P, *Pt, *x, *y, *flush;
    cudaMalloc(&P, sizeof(double) * m * m);
    cudaMalloc(&Pt, sizeof(double) * m * m);
    cudaMalloc(&x, sizeof(double) * m);
    cudaMalloc(&y, sizeof(double) * m);
    cudaMalloc(&flush, 256 << 20);
    cudaMemset(P, 0, sizeof(double) * m * m);
    cudaMemset(Pt, 0, sizeof(double) * m * m);
    cudaMemset(x, 0, sizeof(double) * m);
    const int reps = 20;
    auto fl = [&] {
        cudaMemsetAsync(flush, 0, 256 << 20, s);
        launch_gemv_rowmajor((256LL << 20) / 8 / 256, 256, flush, 256, XPlain{x}, EpiSt{y}, s);
    };
    const float tf = time_ms(fl, reps, s);
    const float t_in = time_ms([&] { fl(); launch_coldot(m, m, P, m, XPlain{x}, EpiSt{y}, s); }, reps, s) - tf;
    const float t_in2 = time_ms([&] { fl(); launch_coldot(m, m, P, m, XPlain{x}, EpiSt{y}, s);
                                      launch_coldot(m, m, P, m, XPlain{x}, EpiSt{y}, s); }, reps, s) - tf;
    const float t_pt = time_ms([&] { fl(); launch_coldot(m, m, P, m, XPlain{x}, EpiSt{y}, s);
                                     launch_coldot(m, m, Pt, m, XPlain{x}, EpiSt{y}, s); }, reps, s) - tf;
    const float t_cmw = time_ms([&] { fl(); launch_coldot(m, m, P, m, XPlain{x}, EpiSt{y}, s);
                                      launch_gemv_cm(m, m, P, m, x, EpiSt{y}, s); }, reps, s) - tf;
    const float t_cmc = time_ms([&] { fl(); launch_gemv_cm(m, m, P, m, x, EpiSt{y}, s); }, reps, s) - tf;
    auto cd = [&](int cpc) {
        if (cpc == 1) k_coldot<XPlain, EpiSt, 1><<<m, 256, 0, s>>>(m, m, P, m, XPlain{x}, EpiSt{y});
        if (cpc == 2) k_coldot<XPlain, EpiSt, 2><<<m / 2, 256, 0, s>>>(m, m, P, m, XPlain{x}, EpiSt{y});
        if (cpc == 4) k_coldot<XPlain, EpiSt, 4><<<m / 4, 256, 0, s>>>(m, m, P, m, XPlain{x}, EpiSt{y});
        if (cpc == 8) k_coldot<XPlain, EpiSt, 8><<<m / 8, 256, 0, s>>>(m, m, P, m, XPlain{x}, EpiSt{y});
    };
    for (int cpc : {1, 2, 4, 8}) {
        const float c = time_ms([&] { fl(); cd(cpc); }, reps, s) - tf;
        const float w = time_ms([&] { fl(); cd(cpc); cd(cpc); }, reps, s) - tf - c;
        printf("coldot<%d>: cold %.2f us, warm %.2f us\n", cpc, c, w);
    }
    for (int blocks : {148, 296, 592, 1184, 2368}) {
        const float c = time_ms([&] { fl(); k_read<4><<<blocks, 256, 0, s>>>((const double2*)P, (long long)m * m / 2, y); }, reps, s) - tf;
        const float c8 = time_ms([&] { fl(); k_read<8><<<blocks, 256, 0, s>>>((const double2*)P, (long long)m * m / 2, y); }, reps, s) - tf;
        printf("plain read 32 MB, %d CTAs: unroll4 %.2f us, unroll8 %.2f us\n", blocks, c, c8);
    }
    printf("coldot(P) cold            %.2f us  (%.0f GB/s)\n", t_in, 8.0 * m * m / (t_in * 1e-6) / 1e9);
    printf("coldot(P) after coldot(P) %.2f us\n", t_in2 - t_in);
    printf("coldot(Pt) after coldot(P) %.2f us\n", t_pt - t_in);
    printf("gemv_cm(P) after coldot(P) %.2f us\n", t_cmw - t_in);
    printf("gemv_cm(P) cold           %.2f us\n", t_cmc);
    return 0;
}
