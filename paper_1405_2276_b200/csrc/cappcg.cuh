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
// Partial-sum mode (parts set): u_j = sqd_j · Σ_{b<nparts} parts[b·n + j], the per-CTA partials
// of Eᵀ(Λ_M⁻¹r̃) that the rotate-in kernel leaves (each of its CTAs owns a few rows of E).
struct PcgRhs {
    const double* E = nullptr;
    long long lde = 0;
    int m = 0;
    const double* wsq = nullptr;
    const double* rt = nullptr;
    const double* sqd = nullptr;
    const double* parts = nullptr;
    int nparts = 0;
    const int* cert = nullptr;  // == 3: K is not certified SPD — give up at once (exact path decides)
    // parts written by a kernel that may still be running (the pipelined batch launches this
    // cluster first so it owns its 16 SMs): wait until *ready == alpha_dev[0] + 1, the epoch the
    // producer's last CTA publishes (gemv.cuh CtaParts), at most ready_timeout_ns — a timeout
    // (a profiler serializing kernels) makes the solve give up, i.e. the step is rerun exactly
    const double* ready = nullptr;
    const double* alpha_dev = nullptr;
    unsigned long long ready_timeout_ns = 2000000ull;
};
// Optional tail (st set; needs vtol > 0): after a verified solve the cluster finishes the
// filter step's Woodbury back-substitution and commit instead of a separate kernel:
//   s̃_i = wsq_i·(rt_i + Σ_j Erow_ij·sqd_j·x_j)  (Erow m×n row-major; rows split over the CTAs)
//   dc_j = sqd_j·x_j;  d_j ← (d_j + αλ_j(α − d_j)) / (1 + λ_j(α − d_j));  α_dev[0] = α_dev[1]
// (fast_filter.hpp:114-123), all skipped while *info ≠ 0 (sticky failure of an earlier step).
// A solve that does not verify sets *info = kInfoRetry (when it was 0): the step's state
// epilogues are gated off and the host reruns the step on the exact Cholesky path.
constexpr int kInfoRetry = -1;
struct PcgTail {
    const double* Erow = nullptr;
    int m = 0;
    const double* wsq = nullptr;
    const double* rt = nullptr;
    const double* sqd = nullptr;
    double* st = nullptr;
    double* dc = nullptr;
    double* d = nullptr;
    const double* lam = nullptr;
    double* alpha_dev = nullptr;
    int* info = nullptr;
    const unsigned long long* hout = nullptr;  // [1]: mapped pinned host d (0 = none)
    // parity snapshots written with the commit (filter.cu EpiCtzD): the step's α, gate = 0, new d
    double* alpha_q = nullptr;
    int* gate_q = nullptr;
    double* d_q = nullptr;
    bool retry_only = false;  // no tail; only raise kInfoRetry (a dependent kernel finishes the step)
};
void cap_pcg(int n, const double* K, long long ld, double* u, double* work, int* fallback, cudaStream_t s,
             int maxit = 200, double tol = 1e-14, unsigned long long* ts = nullptr, double vtol = 0.0,
             PcgRhs rhs = PcgRhs{}, PcgTail tail = PcgTail{});

}  // namespace fkb
