// dense.cuh — FP64 dense kernels on sm_100a (K4/K5/K6 building blocks).
#pragma once

#include "common.cuh"

namespace fkb {

// Column-major FP64 GEMM on the DMMA tensor path (mma.sync m8n8k4 f64 → SASS DMMA):
//   C[i,j] = alpha·Σ_k opA(i,k)·dA[k]·opB(k,j) + beta·Cin[i,j] + (i==j ? diag_add : 0)
// opA = A (transA=0, M×K, lda) or Aᵀ (transA=1, A stored K×M); same for B.
// dA (optional) scales column k of opA.  lower_only computes tiles on/below the diagonal
// only (SYRK-style; entries above the diagonal inside diagonal tiles are also written).
// Split-K uses a deterministic two-stage reduction through `ws` (sized by gemm_ws_elems).
struct GemmArgs {
    int M = 0, N = 0, K = 0;
    const double* A = nullptr;
    long long lda = 0;
    int transA = 0;
    const double* B = nullptr;
    long long ldb = 0;
    int transB = 0;
    const double* dA = nullptr;
    double alpha = 1.0;
    double beta = 0.0;
    const double* beta_ptr = nullptr;  // device scalar overriding beta (graph-captured steps)
    const double* Cin = nullptr;       // defaults to C when beta != 0
    long long ldcin = 0;
    double* C = nullptr;
    long long ldc = 0;
    double diag_add = 0.0;
    const double* rs = nullptr;  // optional epilogue row scale:    acc_ij · rs_i
    const double* cs = nullptr;  // optional epilogue column scale: acc_ij · cs_j
    int lower_only = 0;
    int splitk = 1;
};
size_t gemm_ws_elems(const GemmArgs& g);
// Gram-shaped product (transA = 1, transB = 0, k contiguous in both operands): 16-byte
// cp.async DMMA kernel; falls back to gemm() for odd K/ld.
void gram(const GemmArgs& g, double* ws, cudaStream_t s);
size_t gram_ws_elems(int M, int N, int K);
// Symmetric Gram C = epi(Aᵀ·diag(dA)·A) (rs = cs, beta = 0): lower tiles, cluster split-K
// reduced through DSMEM, both triangles written; one launch, no workspace.
void gram_sym(const GemmArgs& g, cudaStream_t s);
void gemm(const GemmArgs& g, double* ws, cudaStream_t s);
int gemm_pick_splitk(int M, int N, int K);


// In-place lower Cholesky of the n×n SPD matrix A (column-major, lda).  Sets *info
// (device int) to j+1 at the first non-positive pivot, leaves it 0 on success.  A workspace
// of potrf_ws_elems(n) selects the DMMA panel path and leaves the 64×64 diagonal-block
// inverses at ws (block b at ws + b·64·64) for potrs_lower_multi.
void potrf_lower(int n, double* A, long long lda, int* info, double* ws, size_t ws_elems, cudaStream_t s);
size_t potrf_ws_elems(int n);
// Solves L Lᵀ x = b in place (x on entry holds b).  flags: device int[2·ceil(n/64)].
void potrs_lower(int n, const double* L, long long lda, double* x, int* flags, cudaStream_t s);
// The same for nrhs right-hand sides B (n×nrhs, ldb), blocked: 64×64 diagonal solves plus
// DMMA trailing updates.
// dinv (the inverses left by potrf_lower's workspace) and tmp (64·nrhs) make every block a
// DMMA product; without them the 64×64 blocks are solved by substitution.
void potrs_lower_multi(int n, const double* L, long long lda, double* B, long long ldb, int nrhs, cudaStream_t s,
                       const double* dinv = nullptr, double* tmp = nullptr);

}  // namespace fkb
