// cappcg.cuh — cluster Jacobi-PCG for the per-step capacitance system (n ≤ 1024).
#pragma once

#include "common.cuh"

namespace fkb {

// Solves K x = u (K full symmetric, column-major) in place in u.  work: ≥ n+2 doubles.
// If maxit iterations do not reach ‖r‖ ≤ tol·‖u‖ (recursive residual), or — with vtol > 0 —
// the recomputed true residual ‖u − Kx‖ exceeds vtol·‖u‖, u is left unchanged and
// *fallback = 1 (work[n] = iterations, work[n+1] = 1 when the true-residual check failed).
// Optional fused right-hand side (the Woodbury capacitance RHS of the filter step): with
// rhs.E set, u_j = sqd_j · Σ_i E_ij·wsq_i·rt_i (E column-major m×n) is formed inside the
// kernel by the CTA owning row j (and stored to u for the Cholesky fallback) instead of
// being read from u.
struct PcgRhs {
    const double* E = nullptr;
    long long lde = 0;
    int m = 0;
    const double* wsq = nullptr;
    const double* rt = nullptr;
    const double* sqd = nullptr;
};
void cap_pcg(int n, const double* K, long long ld, double* u, double* work, int* fallback, cudaStream_t s,
             int maxit = 200, double tol = 1e-14, unsigned long long* ts = nullptr, double vtol = 0.0,
             PcgRhs rhs = PcgRhs{});

}  // namespace fkb
