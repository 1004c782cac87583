// eig.cuh — device symmetric eigensolver (block Jacobi) for the offline G = PΘPᵀ.
#pragma once

#include "common.cuh"

namespace fkb {

// Overwrites A (m×m symmetric, column-major) with its diagonalized form; theta receives the
// eigenvalues (unsorted), V the orthogonal eigenvectors (m×m, ld = m).  Returns the number
// of sweeps performed.  tol bounds max |a_ij|/√(a_ii a_jj) measured before each pair solve.
int sym_eig_device(int m, double* A, long long lda, double* theta, double* V, cudaStream_t s, double tol = 1e-15,
                   int max_sweeps = 40);

// The same, then eigenpairs sorted by ascending eigenvalue (θ, V reordered in place; A is
// left diagonalized but unsorted).
int sym_eig_sorted_device(int m, double* A, long long lda, double* theta, double* V, cudaStream_t s,
                          double tol = 1e-15, int max_sweeps = 40);

// Householder tridiagonalization + QL with the O(n³) parts on the GPU (tdeig.cu): A (device,
// n×n column-major symmetric, overwritten) → eigenvalues ascending (host w) and eigenvector
// columns (device Z, n×n column-major).  For the GHEP core and the add_low_rank core.
void sym_eig_tridiag_device(int n, double* A, double* w_host, double* Z, cudaStream_t s);

}  // namespace fkb
