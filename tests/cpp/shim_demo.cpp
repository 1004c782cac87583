// shim_demo.cpp — reference-style caller compiled against include/fastkf_b200.hpp only.
// Mirrors the fkf branch of cmd_run (driver.hpp:278-303): build H, CovarianceOperator,
// fkf_init, then fkf_step per observation with UQ.  Reads observations from stdin
// (n_steps rows of m values), prints alpha, trace, entropy, and the mean per step.
#include <cmath>
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
    const FkfContext ctx = fkf_init(cov, h, 2e-4, 16, 20, 11);
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
                    trace_criterion(state, cov), relative_entropy(state));
        for (Index i = 0; i < state.mean.size(); ++i) std::printf("%.17g\n", state.mean[i]);
    }
    // value semantics (fast_filter.hpp:84-125): an edited copy, then the unedited state again
    Vector y(h.rows());
    for (Index i = 0; i < y.size(); ++i) y[i] = 1e-3 * double(i % 7);
    const LowRankState s1 = fkf_step(state, ctx, y);
    LowRankState edited = state;
    edited.mean[0] += 1.0;
    edited.alpha += 0.5;
    const LowRankState s2 = fkf_step(edited, ctx, y);
    const LowRankState s3 = fkf_step(state, ctx, y);
    // s1 continued the device chain (which carries H·mean = y − σ²z), s3 re-uploaded the state
    // (H·mean recomputed): the same function of (state, y) up to rounding, d and α exactly
    auto close = [](const Vector& a, const Vector& b) {
        double num = 0.0, den = 0.0;
        for (size_t i = 0; i < a.v.size(); ++i) {
            num += (a.v[i] - b.v[i]) * (a.v[i] - b.v[i]);
            den += b.v[i] * b.v[i];
        }
        return a.v.size() == b.v.size() && num <= 1e-24 * den;
    };
    if (!close(s3.mean, s1.mean) || s3.d.v != s1.d.v || s3.alpha != s1.alpha) return 7;
    if (s2.mean.v == s1.mean.v || s2.alpha != state.alpha + 1.5) return 8;
    const FkfContext& cctx = ctx;  // const context, reference signatures
    if (std::abs(trace_criterion(s3, cov) - trace_criterion(s3, cctx)) > 1e-12 * std::abs(trace_criterion(s3, cctx)))
        return 9;
    std::printf("edit ok\n");
    // the driver's loop as one call (extension fkf_run) ≡ fkf_step step by step
    Matrix ys(h.rows(), 2);
    for (Index i = 0; i < h.rows(); ++i) {
        ys(i, 0) = y[i];
        ys(i, 1) = 0.5 * y[i];
    }
    Vector y2(h.rows());
    for (Index i = 0; i < h.rows(); ++i) y2[i] = 0.5 * y[i];
    const LowRankState r1 = fkf_step(s3, ctx, y), r2 = fkf_step(r1, ctx, y2);
    const std::vector<LowRankState> run = fkf_run(s3, ctx, ys);
    if (run.size() != 2 || !close(run[1].mean, r2.mean) || run[1].d.v != r2.d.v || run[1].alpha != r2.alpha ||
        !close(run[0].mean, r1.mean) || run[1].step != r2.step)
        return 10;
    const LowRankState r3 = fkf_step(run[1], ctx, y);  // continues from the mirrored state
    const LowRankState r4 = fkf_step(r2, ctx, y);
    if (!close(r3.mean, r4.mean)) return 11;
    std::printf("run ok\n");
    return 0;
}
