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

}  // namespace fkb
