// gemv.cuh — HBM-bound FP64 matrix–vector kernels with fused prologue/epilogue functors.
//
// k_gemv_rows: y = A·x for column-major A (m×k).  A CTA owns 32 rows; its 8 warps split the
//   columns (stride 8) so each warp load is one coalesced 256-B row segment, four
//   independent accumulators per lane keep loads in flight, and a fixed-order shared-memory
//   reduction keeps results deterministic.  Grid = ⌈m/32⌉ CTAs (m = 2048 → 64 CTAs,
//   N = 65536 → 2048 CTAs).
// k_gemv_cols: y = Aᵀ·x, one warp per column, lanes stride the rows, 4 accumulators.
#pragma once

#include "common.cuh"

namespace fkb {

struct XPlain {
    const double* x;
    __device__ __forceinline__ double operator()(long long c) const { return __ldg(x + c); }
};
struct XProd {  // x_c = a_c · b_c
    const double* a;
    const double* b;
    __device__ __forceinline__ double operator()(long long c) const { return __ldg(a + c) * __ldg(b + c); }
};
struct EpiAxpby {  // y_i = α·v + β·y_i
    double* y;
    double alpha, beta;
    __device__ __forceinline__ void operator()(long long i, double v) const {
        y[i] = beta == 0.0 ? alpha * v : alpha * v + beta * y[i];
    }
};

template <class XL, class Epi>
__global__ void __launch_bounds__(256) k_gemv_rows(long long m, int k, const double* __restrict__ A, long long lda,
                                                  XL xl, Epi epi) {
    __shared__ double red[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long row = blockIdx.x * 32LL + lane;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (row < m) {
        const double* Ar = A + row;
        int c = w;
        for (; c + 24 < k; c += 32) {
            a0 = fma(Ar[(long long)c * lda], xl(c), a0);
            a1 = fma(Ar[(long long)(c + 8) * lda], xl(c + 8), a1);
            a2 = fma(Ar[(long long)(c + 16) * lda], xl(c + 16), a2);
            a3 = fma(Ar[(long long)(c + 24) * lda], xl(c + 24), a3);
        }
        for (; c < k; c += 8) a0 = fma(Ar[(long long)c * lda], xl(c), a0);
    }
    red[w][lane] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (w == 0 && row < m) {
        double v = red[0][lane];
#pragma unroll
        for (int q = 1; q < 8; ++q) v += red[q][lane];
        epi(row, v);
    }
}

template <class XL, class Epi>
__global__ void __launch_bounds__(256) k_gemv_cols(long long n, int k, const double* __restrict__ A, long long lda,
                                                  XL xl, Epi epi) {
    const int lane = threadIdx.x & 31;
    const long long col = blockIdx.x * 8LL + (threadIdx.x >> 5);
    if (col >= k) return;
    const double* a = A + col * lda;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    long long i = lane;
    for (; i + 96 < n; i += 128) {
        s0 = fma(a[i], xl(i), s0);
        s1 = fma(a[i + 32], xl(i + 32), s1);
        s2 = fma(a[i + 64], xl(i + 64), s2);
        s3 = fma(a[i + 96], xl(i + 96), s3);
    }
    for (; i < n; i += 32) s0 = fma(a[i], xl(i), s0);
    double s = (s0 + s1) + (s2 + s3);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) epi(col, s);
}

template <class XL, class Epi>
inline void launch_gemv_rows(long long m, int k, const double* A, long long lda, XL xl, Epi epi, cudaStream_t s) {
    if (m <= 0) return;
    k_gemv_rows<XL, Epi><<<(unsigned)((m + 31) / 32), 256, 0, s>>>(m, k, A, lda, xl, epi);
    FKB_LAUNCH_CHECK();
    count_launch();
}
template <class XL, class Epi>
inline void launch_gemv_cols(long long n, int k, const double* A, long long lda, XL xl, Epi epi, cudaStream_t s) {
    if (k <= 0) return;
    k_gemv_cols<XL, Epi><<<(unsigned)((k + 7) / 8), 256, 0, s>>>(n, k, A, lda, xl, epi);
    FKB_LAUNCH_CHECK();
    count_launch();
}

}  // namespace fkb
