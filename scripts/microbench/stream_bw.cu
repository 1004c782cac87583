// Microbenchmark: streaming dot products over a row-major 65536×300 FP64 matrix (the mean
// update's U pass) and a 2048×2048 column-major P (rotations): TMA-bulk k_stream_dot vs the
// load/store kernels.  Build (from repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I paper_1405_2276_b200/csrc \
//        -I scripts/microbench scripts/microbench/stream_bw.cu -o scripts/microbench/stream_bw
// Result on B200 (round 1): the TMA-bulk variant peaked at 3.8 TB/s (U) / 2.6 TB/s (P) vs
// 4.5 / 3.1 TB/s for the LDG kernels, so the product keeps the LDG kernels.
#include <cstdio>
#include <vector>
#include <type_traits>
#include <algorithm>

#include "gemv.cuh"
#include "stream.cuh"

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

// U pass variant: RPW rows per warp, 16-byte loads, every load of the warp's rows in flight
template <int RPW>
__global__ void __launch_bounds__(256) k_upass_v2(long long m, int k, const double* __restrict__ A,
                                                 const double* __restrict__ x, double* __restrict__ y) {
    extern __shared__ double xs[];
    for (int c = threadIdx.x; c < k; c += blockDim.x) xs[c] = x[c];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
    const int k2 = k / 2;  // k even
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w * RPW < m; w += nw) {
        const long long r0 = w * RPW;
        double s[RPW];
        double2 v[RPW][5];
#pragma unroll
        for (int q = 0; q < RPW; ++q)
#pragma unroll
            for (int u = 0; u < 5; ++u) {
                const int c2 = lane + 32 * u;
                v[q][u] = (c2 < k2 && r0 + q < m) ? __ldcs(reinterpret_cast<const double2*>(A + (r0 + q) * k) + c2)
                                                  : make_double2(0.0, 0.0);
            }
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
            s[q] = 0.0;
#pragma unroll
            for (int u = 0; u < 5; ++u) {
                const int c2 = lane + 32 * u;
                if (c2 < k2) s[q] = fma(v[q][u].x, xs[2 * c2], fma(v[q][u].y, xs[2 * c2 + 1], s[q]));
            }
        }
#pragma unroll
        for (int q = 0; q < RPW; ++q)
            for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
        if (lane < RPW && r0 + lane < m) {
            double v0 = s[0];
#pragma unroll
            for (int q = 1; q < RPW; ++q)
                if (lane == q) v0 = s[q];
            y[r0 + lane] = v0;
        }
    }
}

// column dots with 16-byte loads: CTA owns CPC columns, thread t covers row pairs
template <int CPC, int EP>
__global__ void __launch_bounds__(256) k_coldot2(int m, int n, const double* __restrict__ A, long long lda,
                                                const double* __restrict__ x, double* __restrict__ y) {
    const int j0 = blockIdx.x * CPC;
    double acc[CPC];
#pragma unroll
    for (int c = 0; c < CPC; ++c) acc[c] = 0.0;
    const int m2 = m / 2;
    for (int i0 = 0; i0 < m2; i0 += 256 * EP) {
        double2 xv[EP], e[CPC][EP];
#pragma unroll
        for (int q = 0; q < EP; ++q) {
            const int i = i0 + threadIdx.x + 256 * q;
            xv[q] = i < m2 ? reinterpret_cast<const double2*>(x)[i] : make_double2(0.0, 0.0);
#pragma unroll
            for (int c = 0; c < CPC; ++c)
                e[c][q] = (i < m2 && j0 + c < n) ? __ldcs(reinterpret_cast<const double2*>(A + (long long)(j0 + c) * lda) + i)
                                                 : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int c = 0; c < CPC; ++c)
#pragma unroll
            for (int q = 0; q < EP; ++q) acc[c] = fma(e[c][q].x, xv[q].x, fma(e[c][q].y, xv[q].y, acc[c]));
    }
    __shared__ double red[8][CPC];
#pragma unroll
    for (int c = 0; c < CPC; ++c) {
        double v = acc[c];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = v;
    }
    __syncthreads();
    if (threadIdx.x < CPC && j0 + threadIdx.x < n) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
        y[j0 + threadIdx.x] = v;
    }
}

// plain streaming read: every thread sums 16-byte loads (grid-stride), UNROLL in flight
template <int UNROLL>
__global__ void __launch_bounds__(256) k_read(const double2* __restrict__ a, long long n2, double* out) {
    double acc = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
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
    return ms / reps;
}

int main() {
    cudaStream_t s;
    cudaStreamCreate(&s);
    const long long n = 65536;
    const int r = 300, m = 2048;
    double *U, *x, *y, *P, *flush;
    cudaMalloc(&U, sizeof(double) * n * r);
    cudaMalloc(&P, sizeof(double) * m * m);
    cudaMalloc(&x, sizeof(double) * 4096);
    cudaMalloc(&y, sizeof(double) * n);
    cudaMalloc(&flush, 256 << 20);
    cudaMemset(U, 0, sizeof(double) * n * r);
    cudaMemset(P, 0, sizeof(double) * m * m);
    cudaMemset(x, 0, sizeof(double) * 4096);
    const int reps = 20;
    double* rd;
    cudaMalloc(&rd, sizeof(double) * 4);
    // write flush, then a read sweep of the same size so no dirty line is written back inside
    // the measured kernel
    auto fl = [&] {
        cudaMemsetAsync(flush, 0, 256 << 20, s);
        launch_coldot(1 << 21, 4, flush, 1 << 21, XPlain{flush}, EpiSt{rd}, s);  // reads 4×16 MB... (sweep below)
        launch_gemv_rowmajor((256LL << 20) / 8 / 256, 256, flush, 256, XPlain{x}, EpiSt{y}, s);
    };
    float tf = time_ms(fl, reps, s);
    for (int blocks : {148 * 4, 148 * 8, 148 * 16, 148 * 32}) {
        float t = time_ms([&] { fl(); k_read<4><<<blocks, 256, 0, s>>>(reinterpret_cast<const double2*>(U), n * r / 2, y); }, reps, s) - tf;
        printf("plain read U (157 MB) blocks %5d unroll 4: %.2f us  %.0f GB/s\n", blocks, t * 1e3, 8.0 * n * r / (t * 1e-3) / 1e9);
        t = time_ms([&] { fl(); k_read<8><<<blocks, 256, 0, s>>>(reinterpret_cast<const double2*>(U), n * r / 2, y); }, reps, s) - tf;
        printf("plain read U (157 MB) blocks %5d unroll 8: %.2f us  %.0f GB/s\n", blocks, t * 1e3, 8.0 * n * r / (t * 1e-3) / 1e9);
    }
    for (long long tb : {64 << 10}) {
        float t = time_ms([&] { fl(); launch_stream_dot(n, r, r, U, XPlain{x}, EpiSt{y}, s, tb); }, reps, s) - tf;
        printf("U pass stream_dot tile %3lld KB: %.2f us  %.0f GB/s\n", tb >> 10, t * 1e3, 8.0 * n * r / (t * 1e-3) / 1e9);
    }
    for (long long mc : {0LL, 592LL, 1184LL, 1776LL, 4096LL}) {
        float t = time_ms([&] { fl(); launch_gemv_rowmajor(n, r, U, r, XPlain{x}, EpiSt{y}, s, mc); }, reps, s) - tf;
        printf("U pass gemv_rowmajor max_ctas %5lld: %.2f us  %.0f GB/s\n", mc, t * 1e3, 8.0 * n * r / (t * 1e-3) / 1e9);
    }
    for (int ctas : {0}) {
        auto run = [&](auto rpw) {
            constexpr int RPW = decltype(rpw)::value;
            long long need = (n / RPW + 7) / 8;
            long long g = ctas ? std::min<long long>(need, ctas) : need;
            float t = time_ms([&] { fl(); k_upass_v2<RPW><<<g, 256, r * 8, s>>>(n, r, U, x, y); }, reps, s) - tf;
            printf("U pass v2 RPW %d ctas %5lld: %.2f us  %.0f GB/s\n", RPW, g, t * 1e3, 8.0 * n * r / (t * 1e-3) / 1e9);
        };
        run(std::integral_constant<int, 2>{});
        run(std::integral_constant<int, 4>{});
        run(std::integral_constant<int, 8>{});
    }
    for (long long tb : {64 << 10}) {
        float t = time_ms([&] { fl(); launch_stream_dot(m, m, m, P, XPlain{x}, EpiSt{y}, s, tb); }, reps, s) - tf;
        printf("P pass stream_dot tile %3lld KB: %.2f us  %.0f GB/s\n", tb >> 10, t * 1e3, 8.0 * m * m / (t * 1e-3) / 1e9);
    }
    {
        float t = time_ms([&] { fl(); launch_coldot(m, m, P, m, XPlain{x}, EpiSt{y}, s); }, reps, s) - tf;
        printf("P pass coldot (auto CPC):      %.2f us  %.0f GB/s\n", t * 1e3, 8.0 * m * m / (t * 1e-3) / 1e9);
        t = time_ms([&] { fl(); k_coldot<XPlain, EpiSt, 1><<<m, 256, 0, s>>>(m, m, P, m, XPlain{x}, EpiSt{y}); }, reps, s) - tf;
        printf("P pass coldot CPC1:            %.2f us  %.0f GB/s\n", t * 1e3, 8.0 * m * m / (t * 1e-3) / 1e9);
        t = time_ms([&] { fl(); k_coldot<XPlain, EpiSt, 2><<<m / 2, 256, 0, s>>>(m, m, P, m, XPlain{x}, EpiSt{y}); }, reps, s) - tf;
        printf("P pass coldot CPC2:            %.2f us  %.0f GB/s\n", t * 1e3, 8.0 * m * m / (t * 1e-3) / 1e9);
        t = time_ms([&] { fl(); k_coldot<XPlain, EpiSt, 8><<<m / 8, 256, 0, s>>>(m, m, P, m, XPlain{x}, EpiSt{y}); }, reps, s) - tf;
        printf("P pass coldot CPC8:            %.2f us  %.0f GB/s\n", t * 1e3, 8.0 * m * m / (t * 1e-3) / 1e9);
        auto run2 = [&](auto cpc, auto ep) {
            constexpr int CPC = decltype(cpc)::value, EP = decltype(ep)::value;
            float t2 = time_ms([&] { fl(); k_coldot2<CPC, EP><<<m / CPC, 256, 0, s>>>(m, m, P, m, x, y); }, reps, s) - tf;
            printf("P pass coldot2 CPC %d EP %d:    %.2f us  %.0f GB/s\n", CPC, EP, t2 * 1e3, 8.0 * m * m / (t2 * 1e-3) / 1e9);
        };
        run2(std::integral_constant<int, 1>{}, std::integral_constant<int, 4>{});
        run2(std::integral_constant<int, 2>{}, std::integral_constant<int, 4>{});
        run2(std::integral_constant<int, 4>{}, std::integral_constant<int, 4>{});
        run2(std::integral_constant<int, 8>{}, std::integral_constant<int, 4>{});
        run2(std::integral_constant<int, 2>{}, std::integral_constant<int, 2>{});
        run2(std::integral_constant<int, 4>{}, std::integral_constant<int, 2>{});
    }
    printf("flush %.2f us; %s\n", tf * 1e3, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
