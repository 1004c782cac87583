// cappcg.cuh — cluster Jacobi-PCG for the per-step capacitance system (n ≤ 1024).
#pragma once

#include "common.cuh"

namespace fkb {

// Solves K x = u (K full symmetric, column-major) in place in u.  work: ≥ n+1 doubles.
// If maxit iterations do not reach ‖r‖ ≤ tol·‖u‖, u is left unchanged and *fallback = 1.
void cap_pcg(int n, const double* K, long long ld, double* u, double* work, int* fallback, cudaStream_t s,
             int maxit = 200, double tol = 1e-14, unsigned long long* ts = nullptr);

}  // namespace fkb
