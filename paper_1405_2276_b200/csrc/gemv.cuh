// gemv.cuh — HBM-bound FP64 matrix–vector kernels with fused prologue/epilogue functors.
//
// k_gemv_rows: y = A·x for column-major A (m×k).  A CTA owns 32 rows and a chunk of
//   columns; its 8 warps split the chunk (stride 8) so each warp load is one coalesced
//   256-B row segment, and 8 independent accumulators per lane keep 8 loads in flight.
//   When ⌈m/32⌉ CTAs cannot fill the GPU (m×m rotations with m = 2048 → 64 CTAs) the
//   columns are split over S CTAs and a second kernel reduces the partials in a fixed
//   order (deterministic), then applies the epilogue.
// k_gemv_cols: y = Aᵀ·x, one warp per column, lanes stride the rows, 8 loads in flight.
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
struct EpiStore {  // partial sums
    double* p;
    __device__ __forceinline__ void operator()(long long i, double v) const { p[i] = v; }
};

// RG row groups of 32 rows per CTA (RG = 4 for very tall A: 1 KB contiguous per column
// per CTA, better DRAM page locality); the 8/RG warps of a row group split the columns.
template <class XL, class Epi, int RG = 1>
__global__ void __launch_bounds__(256) k_gemv_rows(long long m, int k, const double* __restrict__ A, long long lda,
                                                  XL xl, Epi epi, int kchunk, long long pstride) {
    constexpr int NCP = 8 / RG;  // column phases per row group
    __shared__ double red[8][33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int rg = w % RG, cph = w / RG;
    const long long row = blockIdx.x * (32LL * RG) + rg * 32 + lane;
    const int c0 = blockIdx.y * kchunk, c1 = min(k, c0 + kchunk);
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = 0.0;
    if (row < m) {
        const double* Ar = A + row;
        int c = c0 + cph;
        for (; c + 7 * NCP < c1; c += 8 * NCP) {
#pragma unroll
            for (int q = 0; q < 8; ++q) a[q] = fma(Ar[(long long)(c + NCP * q) * lda], xl(c + NCP * q), a[q]);
        }
        for (; c < c1; c += NCP) a[0] = fma(Ar[(long long)c * lda], xl(c), a[0]);
    }
    red[w][lane] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
    __syncthreads();
    if (w < RG && row < m) {
        double v = red[w][lane];
#pragma unroll
        for (int q = 1; q < NCP; ++q) v += red[w + q * RG][lane];
        epi(row + blockIdx.y * pstride, v);
    }
}

template <class Epi>
__global__ void k_gemv_rows_reduce(long long m, int S, const double* __restrict__ part, Epi epi) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int s = 0; s < S; ++s) v += part[i + s * m];
        epi(i, v);
    }
}

template <class XL, class Epi>
__global__ void __launch_bounds__(256) k_gemv_cols(long long n, int k, const double* __restrict__ A, long long lda,
                                                  XL xl, Epi epi) {
    const int lane = threadIdx.x & 31;
    const long long col = blockIdx.x * 8LL + (threadIdx.x >> 5);
    if (col >= k) return;
    const double* a = A + col * lda;
    double s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = 0.0;
    long long i = lane;
    for (; i + 224 < n; i += 256) {
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] = fma(a[i + 32 * q], xl(i + 32 * q), s[q]);
    }
    for (; i < n; i += 32) s[0] = fma(a[i], xl(i), s[0]);
    double t = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (lane == 0) epi(col, t);
}

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

// Column splits so that the launch covers ≥ ~4 CTAs per SM; part needs S·m doubles.
inline int gemv_rows_splits(long long m, int k) {
    const long long tiles = (m + 31) / 32;
    if (tiles >= 592 || k < 256) return 1;
    return int(std::max<long long>(1, std::min<long long>((592 + tiles - 1) / tiles, k / 128)));
}

template <class XL, class Epi>
inline void launch_gemv_rows(long long m, int k, const double* A, long long lda, XL xl, Epi epi, cudaStream_t s,
                             double* part = nullptr) {
    if (m <= 0) return;
    const unsigned tiles = (unsigned)((m + 31) / 32);
    const int S = part ? gemv_rows_splits(m, k) : 1;
    if (S == 1 && m >= 148 * 128 * 4) {  // very tall (U: N×r): 128-row CTAs
        k_gemv_rows<XL, Epi, 4><<<(unsigned)((m + 127) / 128), 256, 0, s>>>(m, k, A, lda, xl, epi, std::max(k, 1), 0);
        FKB_LAUNCH_CHECK();
        count_launch();
        return;
    }
    if (S == 1) {
        k_gemv_rows<XL, Epi><<<tiles, 256, 0, s>>>(m, k, A, lda, xl, epi, std::max(k, 1), 0);
        FKB_LAUNCH_CHECK();
        count_launch();
        return;
    }
    const int kchunk = ((k + S - 1) / S + 7) / 8 * 8;
    const int Sx = (k + kchunk - 1) / kchunk;
    k_gemv_rows<XL, EpiStore><<<dim3(tiles, Sx), 256, 0, s>>>(m, k, A, lda, xl, EpiStore{part}, kchunk, m);
    FKB_LAUNCH_CHECK();
    k_gemv_rows_reduce<Epi><<<(unsigned)std::min<long long>((m + 255) / 256, 1184), 256, 0, s>>>(m, Sx, part, epi);
    FKB_LAUNCH_CHECK();
    count_launch(2);
}
// Row-split variant of k_gemv_cols: CTA (x, s) sums rows [s·rchunk, (s+1)·rchunk) of 8 columns.
template <class XL>
__global__ void __launch_bounds__(256) k_gemv_cols_part(long long n, int k, const double* __restrict__ A,
                                                       long long lda, XL xl, long long rchunk,
                                                       double* __restrict__ part) {
    const int lane = threadIdx.x & 31;
    const long long col = blockIdx.x * 8LL + (threadIdx.x >> 5);
    if (col >= k) return;
    const long long i0 = blockIdx.y * rchunk, i1 = min(n, i0 + rchunk);
    const double* a = A + col * lda;
    double s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = 0.0;
    long long i = i0 + lane;
    for (; i + 224 < i1; i += 256) {
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] = fma(a[i + 32 * q], xl(i + 32 * q), s[q]);
    }
    for (; i < i1; i += 32) s[0] = fma(a[i], xl(i), s[0]);
    double t = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (lane == 0) part[blockIdx.y * (long long)k + col] = t;
}

template <class Epi>
__global__ void k_gemv_cols_reduce(int k, int S, const double* __restrict__ part, Epi epi) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int s = 0; s < S; ++s) v += part[(long long)s * k + c];
        epi(c, v);
    }
}

template <class XL, class Epi>
inline void launch_gemv_cols(long long n, int k, const double* A, long long lda, XL xl, Epi epi, cudaStream_t s,
                             double* part = nullptr) {
    if (k <= 0) return;
    const long long ctas = (k + 7) / 8;
    int S = 1;
    if (part && ctas < 592) S = int(std::max<long long>(1, std::min<long long>((592 + ctas - 1) / ctas, n / 256)));
    if (S == 1) {
        k_gemv_cols<XL, Epi><<<(unsigned)ctas, 256, 0, s>>>(n, k, A, lda, xl, epi);
        FKB_LAUNCH_CHECK();
        count_launch();
        return;
    }
    const long long rchunk = ((n + S - 1) / S + 31) / 32 * 32;
    const int Sx = int((n + rchunk - 1) / rchunk);
    k_gemv_cols_part<XL><<<dim3((unsigned)ctas, Sx), 256, 0, s>>>(n, k, A, lda, xl, rchunk, part);
    FKB_LAUNCH_CHECK();
    k_gemv_cols_reduce<Epi><<<(k + 255) / 256, 256, 0, s>>>(k, Sx, part, epi);
    FKB_LAUNCH_CHECK();
    count_launch(2);
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
