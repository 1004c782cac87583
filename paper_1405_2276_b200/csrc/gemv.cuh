// gemv.cuh — HBM-bound FP64 matrix–vector kernels with fused prologue/epilogue functors:
// k_gemv_rowmajor (row-major A, the step's U pass) and k_coldot (column dots of a
// column-major A: the P/Pᵀ rotations, the capacitance RHS, Bᵀz).
#pragma once

#include <cstdint>
#include <cstdlib>

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

// y_i = epi(i, Σ_j A_ij·x_j) for ROW-MAJOR A (m×k, ld ≥ k): each warp owns 4 rows and reads
// each row as contiguous 256-B chunks, so the matrix streams linearly from HBM (the
// step's U-pass; U is stored once more row-major for this).
template <class XL, class Epi>
__global__ void __launch_bounds__(256) k_gemv_rowmajor(long long m, int k, const double* __restrict__ A,
                                                      long long ld, XL xl, Epi epi) {
    extern __shared__ double xs[];
    for (int c = threadIdx.x; c < k; c += blockDim.x) xs[c] = xl(c);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;  // grid-stride over 4-row groups
    for (long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; w * 4 < m; w += nw) {
    const long long r0 = w * 4;
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    const int nq = (int)min(4LL, m - r0);
    int c = lane;
    for (; c + 96 < k; c += 128) {  // 16 independent loads in flight per lane
        double v[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int u = 0; u < 4; ++u) v[q][u] = q < nq ? __ldcs(A + (r0 + q) * ld + c + 32 * u) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double xv = xs[c + 32 * u];
#pragma unroll
            for (int q = 0; q < 4; ++q) s[q] = fma(v[q][u], xv, s[q]);
        }
    }
    for (; c < k; c += 32) {
        const double xv = xs[c];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < nq) s[q] = fma(__ldcs(A + (r0 + q) * ld + c), xv, s[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
    if (lane < 4 && r0 + lane < m) {
        const double v = lane == 0 ? s[0] : lane == 1 ? s[1] : lane == 2 ? s[2] : s[3];
        epi(r0 + lane, v);
    }
    }
}

template <class XL, class Epi>
inline void launch_gemv_rowmajor(long long m, int k, const double* A, long long ld, XL xl, Epi epi, cudaStream_t s,
                                 long long max_ctas = 0) {
    if (m <= 0) return;
    const long long warps = (m + 3) / 4;
    long long ctas = (warps + 7) / 8;
    if (max_ctas > 0) ctas = std::min(ctas, max_ctas);
    k_gemv_rowmajor<XL, Epi><<<(unsigned)ctas, 256, sizeof(double) * size_t(std::max(k, 1)), s>>>(m, k, A, ld, xl,
                                                                                                 epi);
    FKB_LAUNCH_CHECK();
    count_launch();
}

// ---- single-launch column dots: out_j = epi(j, Σ_i A_ij·x_i) for column-major A (m×n).
// A CTA owns CPC consecutive columns; each thread keeps its x values in registers (reused
// over the CPC columns) and issues every load of a 2048-row chunk × CPC columns before the
// first FMA, so a chunk costs one memory latency.  Fixed-order reductions (deterministic),
// no split partials and no second kernel.
template <class XL, class Epi, int CPC>
__global__ void __launch_bounds__(256) k_coldot(int m, int n, const double* __restrict__ A, long long lda, XL xl,
                                               Epi epi) {
    constexpr int EPT = 8;
    const int j0 = blockIdx.x * CPC;
    double acc[CPC];
#pragma unroll
    for (int c = 0; c < CPC; ++c) acc[c] = 0.0;
    for (int i0 = 0; i0 < m; i0 += 256 * EPT) {
        double xv[EPT], e[CPC][EPT];
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
            const int i = i0 + threadIdx.x + 256 * q;
            xv[q] = i < m ? xl(i) : 0.0;
#pragma unroll
            for (int c = 0; c < CPC; ++c) e[c][q] = (i < m && j0 + c < n) ? A[i + (long long)(j0 + c) * lda] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < CPC; ++c)
#pragma unroll
            for (int q = 0; q < EPT; ++q) acc[c] = fma(e[c][q], xv[q], acc[c]);
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
        epi(j0 + threadIdx.x, v);
    }
}

template <class XL, class Epi>
inline void launch_coldot(int m, int n, const double* A, long long lda, XL xl, Epi epi, cudaStream_t s) {
    if (n <= 0) return;
    if (n >= 8 * 296) {
        k_coldot<XL, Epi, 8><<<(unsigned)((n + 7) / 8), 256, 0, s>>>(m, n, A, lda, xl, epi);
    } else if (n >= 4 * 296) {
        k_coldot<XL, Epi, 4><<<(unsigned)((n + 3) / 4), 256, 0, s>>>(m, n, A, lda, xl, epi);
    } else if (n >= 2 * 296) {
        k_coldot<XL, Epi, 2><<<(unsigned)((n + 1) / 2), 256, 0, s>>>(m, n, A, lda, xl, epi);
    } else {
        k_coldot<XL, Epi, 1><<<(unsigned)n, 256, 0, s>>>(m, n, A, lda, xl, epi);
    }
    FKB_LAUNCH_CHECK();
    count_launch();
}

}  // namespace fkb
