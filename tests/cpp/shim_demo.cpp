// shim_demo.cpp — reference-style caller compiled against include/fastkf_b200.hpp only.
// Mirrors the fkf branch of cmd_run (driver.hpp:278-303): build H, CovarianceOperator,
// fkf_init, then fkf_step per observation with UQ.  Reads observations from stdin
// (n_steps rows of m values), prints alpha, trace, entropy, and the mean per step.
#include <cstdio>
#include <iostream>

#include "fastkf_b200.hpp"

int main(int argc, char** argv) {
    using namespace fastkf;
    const int nx = 12, ny = 12, n_steps = argc > 1 ? std::atoi(argv[1]) : 3;
    const Grid grid(nx, ny);
    KernelSpec spec;
    spec.family = KernelFamily::powered_exponential;
    spec.theta = 1e-4;
    spec.length = 0.2;
    spec.power = 0.5;
    const CovarianceOperator cov(grid, spec, CovMode::fft);
    const SparseRowMatrix h = build_H(grid, SourceReceiverLayout::cross_well(grid, 3, 8));
    FkfContext ctx = fkf_init(cov, h, 2e-4, 16, 20, 11);
    LowRankState state = LowRankState::zero_start(grid.size());
    try {  // mismatched observation length must raise std::invalid_argument
        fkf_step(state, ctx, Vector(h.rows() + 1));
        std::printf("ERROR no exception\n");
        return 1;
    } catch (const std::invalid_argument&) {
    }
    for (int k = 0; k < n_steps; ++k) {
        Vector y(h.rows());
        for (Index i = 0; i < y.size(); ++i) std::cin >> y[i];
        state = fkf_step(state, ctx, y);
        std::printf("step %d alpha %.17g trace %.17g entropy %.17g\n", state.step, state.alpha,
                    trace_criterion(state, ctx), relative_entropy(state, ctx));
        for (Index i = 0; i < state.mean.size(); ++i) std::printf("%.17g\n", state.mean[i]);
    }
    return 0;
}
