// shim_fekf_demo.cpp — reference-style caller of the extended filter, compiled against
// include/fastkf_b200.hpp only.  Mirrors the ekf branch of cmd_run (driver.hpp:304-333):
// state = zero_start with mean = forward(init_slowness), then fekf_step per observation with
// opts.seed = derived per step.  Reads n_steps rows of m observations and one seed per row
// from stdin; prints alpha, rank and the mean per step.
#include <cmath>
#include <cstdio>
#include <iostream>

#include "fastkf_b200.hpp"

int main(int argc, char** argv) {
    using namespace fastkf;
    const int n_steps = argc > 1 ? std::atoi(argv[1]) : 3;
    const Grid grid(8, 8);
    KernelSpec spec;
    spec.family = KernelFamily::powered_exponential;
    spec.theta = 1e-4;
    spec.length = 0.2;
    spec.power = 0.5;
    const CovarianceOperator cov(grid, spec, CovMode::fft);
    const SparseRowMatrix h = build_H(grid, SourceReceiverLayout::cross_well(grid, 2, 4));
    const BoxCox transform{2.0};
    FekfOptions opts;
    opts.k_rank = h.rows();
    opts.trunc_tol = 0.0;
    LowRankState state = LowRankState::zero_start(grid.size());
    const double s0 = transform.alpha * (std::pow(1e-4, 1.0 / transform.alpha) - 1.0);  // forward(init_slowness)
    state.mean = Vector::Constant(grid.size(), s0);
    try {  // relinearizations outside [1, 5] must raise std::invalid_argument (fast_filter.hpp:149-150)
        FekfOptions bad = opts;
        bad.relinearizations = 9;
        fekf_step(state, cov, h, Vector(h.rows()), 2e-4, transform, bad);
        std::printf("ERROR no exception\n");
        return 1;
    } catch (const std::invalid_argument&) {
    }
    try {  // Box–Cox domain violation → std::domain_error naming the index (boxcox.hpp:58-75)
        LowRankState neg = LowRankState::zero_start(grid.size());
        neg.mean = Vector::Constant(grid.size(), -5.0);
        fekf_step(neg, cov, h, Vector(h.rows()), 2e-4, transform, opts);
        std::printf("ERROR no domain error\n");
        return 1;
    } catch (const std::domain_error&) {
    }
    for (int k = 0; k < n_steps; ++k) {
        Vector y(h.rows());
        for (Index i = 0; i < y.size(); ++i) std::cin >> y[i];
        unsigned long long seed = 0;
        std::cin >> seed;
        opts.seed = seed;
        state = fekf_step(state, cov, h, y, 2e-4, transform, opts);
        const Matrix w = state.w;
        std::printf("step %d alpha %.17g rank %lld wcols %lld\n", state.step, state.alpha, state.rank(), w.cols());
        for (Index i = 0; i < state.mean.size(); ++i) std::printf("%.17g\n", state.mean[i]);
    }
    return 0;
}
