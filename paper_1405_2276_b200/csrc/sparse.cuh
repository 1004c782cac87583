// sparse.cuh — K2 (CSR SpMM over ray paths) and K3 (Ω generator).
#pragma once

#include "common.cuh"

namespace fkb {

struct DevCsr {  // SparseRowMatrix (grid.hpp:15) on the device: int32 indices, FP64 values
    int rows = 0, cols = 0;
    long long nnz = 0;
    DBuf<int> rowptr, col;
    DBuf<double> val;
};

// Y[:, b] = alpha · A X[:, b] + beta · Yin[:, b] for b < ncols (Yin defaults to Y);
// X, Y, Yin column-major device blocks (Yin shares Y's leading dimension).
void spmm(const DevCsr& A, const double* X, long long ldx, int ncols, double* Y, long long ldy, double alpha,
          double beta, cudaStream_t s, const double* Yin = nullptr);
// Y = alpha · A X on row-major blocks (row strides ldx, ldy; ncols columns), warp per row of A
void spmm_rm(const DevCsr& A, const double* X, long long ldx, int ncols, double* Y, long long ldy, double alpha,
             cudaStream_t s);
// y = alpha · A x for one vector, rows of ≲ 32 nonzeros (8 lanes per row)
void spmv_short(const DevCsr& A, const double* x, double* y, double alpha, cudaStream_t s);
// Upload host CSR and build the explicit transposed CSR (rows ascending inside each column).
void upload_csr_pair(int rows, int cols, const int* rowptr, const int* col, const double* val, DevCsr& A,
                     DevCsr& AT);
// Ω: N×l column-major, column j = normals of Rng(seed, j) (rng.hpp:79-86)
void gaussian_matrix(long long rows, int cols, uint64_t seed, uint64_t base_stream, double* out, long long ld,
                     cudaStream_t s);
// sum of squares of a device vector (deterministic two-stage reduction), result on host
double sumsq(const double* x, long long n, double* ws, cudaStream_t s);

}  // namespace fkb
