// sparse.cu — K2: CSR SpMM for the ray operator H and its explicit transpose; K3: Ω.
//
// Reference products: fast_filter.hpp:63-66 (Hᵀ(Hv)/σ²), :71 (H·ΓHᵀ), :73 (H·U),
// :108 (H·mean); Eigen sparse × dense.  H rows are rays (≈ 2.5·n nonzeros each),
// Hᵀ rows are cells (≈ m·nnz/N ≈ 5–10 nonzeros each), so two kernels:
//   k_spmm_warp   — one warp per row, lanes stride the row's nonzeros, 4 columns per
//                   pass with warp-shuffle reductions (long rows: H);
//   k_spmm_thread — one thread per (row, column), sequential over the short row
//                   (Hᵀ), consecutive threads write consecutive rows (coalesced).

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "rng_device.cuh"
#include "sparse.cuh"

namespace fkb {

__global__ void __launch_bounds__(256) k_spmm_warp(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                                                  const double* __restrict__ v, const double* __restrict__ X,
                                                  long long ldx, int ncols, double* __restrict__ Y, long long ldy,
                                                  double alpha, double beta, const double* __restrict__ Yin) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int b0 = blockIdx.y * 4;
    if (warp >= rows) return;
    const int e0 = rp[warp], e1 = rp[warp + 1];
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    const int nb = min(4, ncols - b0);
    for (int e = e0 + lane; e < e1; e += 32) {
        const long long c = ci[e];
        const double w = v[e];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < nb) s[q] = fma(w, __ldg(X + c + (long long)(b0 + q) * ldx), s[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_down_sync(0xffffffffu, s[q], o);
    // lane 0 holds the four reduced sums; broadcast and let lanes 0..nb-1 write
    double t0 = __shfl_sync(0xffffffffu, s[0], 0);
    double t1 = __shfl_sync(0xffffffffu, s[1], 0);
    double t2 = __shfl_sync(0xffffffffu, s[2], 0);
    double t3 = __shfl_sync(0xffffffffu, s[3], 0);
    if (lane < nb) {
        const double r = lane == 0 ? t0 : lane == 1 ? t1 : lane == 2 ? t2 : t3;
        double* y = Y + warp + (long long)(b0 + lane) * ldy;
        *y = beta == 0.0 ? alpha * r : alpha * r + beta * Yin[warp + (long long)(b0 + lane) * ldy];
    }
}

__global__ void __launch_bounds__(256) k_spmm_thread(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                                                    const double* __restrict__ v, const double* __restrict__ X,
                                                    long long ldx, double* __restrict__ Y, long long ldy,
                                                    double alpha, double beta, const double* __restrict__ Yin) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (r >= rows) return;
    const double* x = X + (long long)b * ldx;
    double s = 0.0;
    for (int e = rp[r]; e < rp[r + 1]; ++e) s = fma(v[e], __ldg(x + ci[e]), s);
    double* y = Y + r + (long long)b * ldy;
    *y = beta == 0.0 ? alpha * s : alpha * s + beta * Yin[r + (long long)b * ldy];
}

// Single-vector SpMV for short rows (Hᵀ: ≈ 10 nonzeros per cell): 8 lanes per row, each
// lane prefetches 4 (col, val) pairs then gathers 4 x values (two memory latencies per 32
// nonzeros instead of two per nonzero), 3-level shuffle reduction.
__global__ void __launch_bounds__(256) k_spmv_sub8(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                                                  const double* __restrict__ v, const double* __restrict__ x,
                                                  double* __restrict__ y, double alpha) {
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 3, sub = threadIdx.x & 7;
    const bool live = row < rows;
    const int e0 = live ? rp[row] : 0, e1 = live ? rp[row + 1] : 0;
    double s = 0.0;
    for (int eb = e0; eb < e1; eb += 32) {
        int c[4];
        double w[4], xv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = eb + sub + 8 * q;
            c[q] = e < e1 ? ci[e] : 0;
            w[q] = e < e1 ? v[e] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) xv[q] = __ldg(x + c[q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) s = fma(w[q], xv[q], s);
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (live && sub == 0) y[row] = alpha * s;
}

void spmv_short(const DevCsr& A, const double* x, double* y, double alpha, cudaStream_t s) {
    if (A.rows <= 0) return;
    k_spmv_sub8<<<ceil_div((long long)A.rows * 8, 256), 256, 0, s>>>(A.rows, A.rowptr.p, A.col.p, A.val.p, x, y, alpha);
    FKB_LAUNCH_CHECK();
    count_launch();
}

// SpMM on ROW-major blocks (X: cols(A) × ncols with row stride ldx, Y: rows(A) × ncols with
// row stride ldy): one warp per row of A, lanes over 32·Q consecutive columns.  The row's
// (col, val) pairs are fetched 32 at a time with one coalesced load and broadcast by shuffles;
// 4 nonzeros × Q columns of X (each nonzero a contiguous 8·ncols-byte row) are in flight per
// lane.  X rows are shared by the ~10 rays through a cell, so they are served from L2.
template <int Q, int U>
__global__ void __launch_bounds__(256) k_spmm_rm(int rows, const int* __restrict__ rp, const int* __restrict__ ci,
                                                const double* __restrict__ v, const double* __restrict__ X,
                                                long long ldx, int ncols, double* __restrict__ Y, long long ldy,
                                                double alpha) {
    const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (row >= rows) return;
    const int col0 = blockIdx.y * 32 * Q;
    double acc[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = 0.0;
    const int e0 = rp[row], e1 = rp[row + 1];
    for (int eb = e0; eb < e1; eb += 32) {
        const int cnt = min(32, e1 - eb);
        const int myc = lane < cnt ? ci[eb + lane] : 0;
        const double myv = lane < cnt ? v[eb + lane] : 0.0;
        for (int u0 = 0; u0 < cnt; u0 += U) {
            int c[U];
            double w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                c[u] = __shfl_sync(0xffffffffu, myc, (u0 + u) & 31);
                w[u] = __shfl_sync(0xffffffffu, myv, (u0 + u) & 31);
                if (u0 + u >= cnt) w[u] = 0.0;
            }
            double x[U][Q];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    const int col = col0 + lane + 32 * q;
                    x[u][q] = col < ncols ? __ldg(X + (long long)c[u] * ldx + col) : 0.0;
                }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int q = 0; q < Q; ++q) acc[q] = fma(w[u], x[u][q], acc[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const int col = col0 + lane + 32 * q;
        if (col < ncols) Y[(long long)row * ldy + col] = alpha * acc[q];
    }
}

void spmm_rm(const DevCsr& A, const double* X, long long ldx, int ncols, double* Y, long long ldy, double alpha,
             cudaStream_t s) {
    if (A.rows <= 0 || ncols <= 0) return;
    // Every nonzero streams a full X row from L2 (X is shared by the ~10 rays through a cell):
    // 8·nnz·l bytes of L2→SM traffic, which this kernel moves at 0.58 of the measured L2→SM
    // read peak (fkb_l2_peak, 20.4 TB/s).  Measured at c2 (l = 320): long rows (rays, ~320
    // nonzeros) 128 columns per warp with 16 nonzeros per batch (64 / 160-column slabs,
    // 16-byte lane loads, 4–32 nonzeros per batch and cp.async.bulk row staging through shared
    // memory all measured 0.23–0.59); short rows (cells, ~10) 256 columns with 4.
    const bool longrows = double(A.nnz) / A.rows > 64.0;
    const int Q = ncols <= 32 ? 1 : longrows ? 4 : 8;
    const dim3 grid(ceil_div((long long)A.rows * 32, 256), ceil_div(ncols, 32 * Q));
    if (Q == 1)
        k_spmm_rm<1, 8><<<grid, 256, 0, s>>>(A.rows, A.rowptr.p, A.col.p, A.val.p, X, ldx, ncols, Y, ldy, alpha);
    else if (Q == 4)
        k_spmm_rm<4, 16><<<grid, 256, 0, s>>>(A.rows, A.rowptr.p, A.col.p, A.val.p, X, ldx, ncols, Y, ldy, alpha);
    else
        k_spmm_rm<8, 4><<<grid, 256, 0, s>>>(A.rows, A.rowptr.p, A.col.p, A.val.p, X, ldx, ncols, Y, ldy, alpha);
    FKB_LAUNCH_CHECK();
    count_launch();
}

void spmm(const DevCsr& A, const double* X, long long ldx, int ncols, double* Y, long long ldy, double alpha,
          double beta, cudaStream_t s, const double* Yin) {
    if (!Yin) Yin = Y;
    if (A.rows <= 0 || ncols <= 0) return;
    const double avg = A.rows ? double(A.nnz) / A.rows : 0.0;
    if (avg > 24.0) {
        for (int c0 = 0; c0 < ncols; c0 += 4 * 65535) {
            const int nc = std::min(ncols - c0, 4 * 65535);
            dim3 grid(ceil_div((long long)A.rows * 32, 256), ceil_div(nc, 4));
            k_spmm_warp<<<grid, 256, 0, s>>>(A.rows, A.rowptr.p, A.col.p, A.val.p, X + (long long)c0 * ldx, ldx, nc,
                                             Y + (long long)c0 * ldy, ldy, alpha, beta, Yin + (long long)c0 * ldy);
            FKB_LAUNCH_CHECK();
            count_launch();
        }
    } else {
        for (int c0 = 0; c0 < ncols; c0 += 65535) {
            const int nc = std::min(ncols - c0, 65535);
            dim3 grid(ceil_div(A.rows, 256), nc);
            k_spmm_thread<<<grid, 256, 0, s>>>(A.rows, A.rowptr.p, A.col.p, A.val.p, X + (long long)c0 * ldx, ldx,
                                               Y + (long long)c0 * ldy, ldy, alpha, beta, Yin + (long long)c0 * ldy);
            FKB_LAUNCH_CHECK();
            count_launch();
        }
    }
}

void upload_csr_pair(int rows, int cols, const int* rowptr, const int* col, const double* val, DevCsr& A,
                     DevCsr& AT) {
    const long long nnz = rowptr[rows];
    std::vector<int> trp(static_cast<size_t>(cols) + 1, 0), tci(static_cast<size_t>(nnz));
    std::vector<double> tv(static_cast<size_t>(nnz));
    for (long long e = 0; e < nnz; ++e) {
        if (col[e] < 0 || col[e] >= cols) throw std::invalid_argument("csr: column index out of range");
        ++trp[size_t(col[e]) + 1];
    }
    for (int c = 0; c < cols; ++c) trp[size_t(c) + 1] += trp[size_t(c)];
    std::vector<int> fill(trp.begin(), trp.end() - 1);
    for (int r = 0; r < rows; ++r)
        for (int e = rowptr[r]; e < rowptr[r + 1]; ++e) {
            const int p = fill[size_t(col[e])]++;
            tci[size_t(p)] = r;
            tv[size_t(p)] = val[e];
        }
    A.rows = rows; A.cols = cols; A.nnz = nnz;
    AT.rows = cols; AT.cols = rows; AT.nnz = nnz;
    A.rowptr.alloc(size_t(rows) + 1);
    A.col.alloc(size_t(std::max<long long>(nnz, 1)));
    A.val.alloc(size_t(std::max<long long>(nnz, 1)));
    AT.rowptr.alloc(size_t(cols) + 1);
    AT.col.alloc(size_t(std::max<long long>(nnz, 1)));
    AT.val.alloc(size_t(std::max<long long>(nnz, 1)));
    FKB_CUDA(cudaMemcpy(A.rowptr.p, rowptr, sizeof(int) * (size_t(rows) + 1), cudaMemcpyHostToDevice));
    FKB_CUDA(cudaMemcpy(AT.rowptr.p, trp.data(), sizeof(int) * trp.size(), cudaMemcpyHostToDevice));
    if (nnz) {
        FKB_CUDA(cudaMemcpy(A.col.p, col, sizeof(int) * size_t(nnz), cudaMemcpyHostToDevice));
        FKB_CUDA(cudaMemcpy(A.val.p, val, sizeof(double) * size_t(nnz), cudaMemcpyHostToDevice));
        FKB_CUDA(cudaMemcpy(AT.col.p, tci.data(), sizeof(int) * size_t(nnz), cudaMemcpyHostToDevice));
        FKB_CUDA(cudaMemcpy(AT.val.p, tv.data(), sizeof(double) * size_t(nnz), cudaMemcpyHostToDevice));
    }
}

// --------------------------------------------------------------------------- K3: Ω
__global__ void k_gaussian_matrix(long long rows, int cols, uint64_t seed, uint64_t base, double* __restrict__ out,
                                  long long ld) {
    const long long pairs = (rows + 1) / 2;
    const int j = blockIdx.y;
    const uint64_t st0 = splitmix64(seed ^ splitmix64(base + (uint64_t)j));  // derive_seed(seed, stream)
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < pairs; p += (long long)gridDim.x * blockDim.x) {
        double c, s;
        rng_normal_pair(st0, (uint64_t)p, c, s);
        double* o = out + (long long)j * ld + 2 * p;
        o[0] = c;
        if (2 * p + 1 < rows) o[1] = s;
    }
}

void gaussian_matrix(long long rows, int cols, uint64_t seed, uint64_t base_stream, double* out, long long ld,
                     cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return;
    for (int c0 = 0; c0 < cols; c0 += 65535) {
        const int nc = std::min(cols - c0, 65535);
        dim3 grid(std::min(ceil_div((rows + 1) / 2, 256), 1024), nc);
        k_gaussian_matrix<<<grid, 256, 0, s>>>(rows, nc, seed, base_stream + uint64_t(c0), out + (long long)c0 * ld, ld);
        FKB_LAUNCH_CHECK();
        count_launch();
    }
}

__global__ void k_sumsq_partial(const double* __restrict__ x, long long n, double* __restrict__ part) {
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        s = fma(x[i], x[i], s);
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
    }
}

double sumsq(const double* x, long long n, double* ws, cudaStream_t s) {
    const int blocks = 256;
    k_sumsq_partial<<<blocks, 256, 0, s>>>(x, n, ws);
    FKB_LAUNCH_CHECK();
    count_launch();
    std::vector<double> h(blocks);
    FKB_CUDA(cudaMemcpyAsync(h.data(), ws, sizeof(double) * blocks, cudaMemcpyDeviceToHost, s));
    FKB_CUDA(cudaStreamSynchronize(s));
    double t = 0.0;
    for (double v : h) t += v;
    return t;
}

}  // namespace fkb
