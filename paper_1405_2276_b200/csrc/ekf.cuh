// ekf.cuh — the fast extended filter (fekf_step, fast_filter.hpp:127-224) on the device.
#pragma once

#include <deque>
#include <string>
#include <vector>

#include "filter.cuh"

namespace fkb {

struct EkfOptions {  // FekfOptions fast_filter.hpp:127-134
    long long k_rank = -1;  // -1: n_m
    long long oversampling = 20;
    double trunc_tol = 1e-5;
    int relinearizations = 1;
    uint64_t seed = 0;
};

// std::domain_error of the Box–Cox maps (boxcox.hpp:58-75) crosses the C ABI as status 4.
struct DomainError : std::domain_error {
    using std::domain_error::domain_error;
};

// LowRankState driven by fekf_step, device resident.  Besides W the state carries
// W̄ = Γ⁻¹W: the reference applies Γ⁻¹ by CG on the fast operator (covariance.hpp:145-152,
// the B-metric of add_low_rank), which stalls beyond desk scale; here every Γ⁻¹ product
// the step needs is a linear combination of W̄ and the GHEP's Ū = Γ⁻¹U = Q̄S.
struct Ekf {
    Cov* cov = nullptr;
    cudaStream_t s = nullptr;
    long long n = 0;
    int m = 0;
    DevCsr H, HT, Hk, HkT;  // base ray operator and its linearization H·diag(∂s/∂ŝ)
    DBuf<int> ht_cell;      // cell (row of Hᵀ) of every Hᵀ entry

    double alpha = 0.0;
    int step_no = 0;
    int r = 0;
    std::vector<double> d_h;
    DBuf<double> mean, W, Wbar, d;
    int last_gep_rank = 0, last_relin = 0;

    DBuf<double> eta, eta2, jac, sinv, heta, G, S, HW, z, tv, gt, dc, ybuf, ws, pws;
    // persistent temporaries of the per-step GHEP and add_low_rank (no per-step cudaMalloc/Free)
    GepDev gep;
    DBuf<double> Wn, Wbn, Vh, Vhb, hgh_ws;
    std::deque<DBuf<double>> scratch;  // deque: growing keeps references to earlier slots valid
    DBuf<double>& tmp(size_t slot, size_t count) {
        if (scratch.size() <= slot) scratch.resize(slot + 1);
        scratch[slot].ensure(std::max<size_t>(count, 1));
        return scratch[slot];
    }
    DBuf<int> info, flags, bad;

    Ekf(Cov* c, int m, int h_cols, const int* rowptr, const int* col, const double* val);
    void reset(const double* mean0_host);
    void step(const double* y_host, double sigma2, double bc_alpha, const EkfOptions& o);
    void uq_scalars(double& trace, double& entropy);  // trace_criterion / relative_entropy
    // diag Σ (var) and `count` realizations (draws first…first+count−1) into device buffers
    void uq(uint64_t seed, uint64_t first, int count, double* X, double* var);

  private:
    void linearize(double bc_alpha);
    void add_low_rank(const std::vector<double>& d_bar, GepDev& g, double trunc_tol, double a);
};

}  // namespace fkb
