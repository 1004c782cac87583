// driver_verbatim.cpp — the reference driver's fkf code, written as the reference writes it
// (cmd_run's fkf branch, driver.hpp:278-303, and cmd_uq's per-step loop, :394-406), compiled
// against include/fastkf_b200.hpp only: const FkfContext, fkf_step(state, ctx, y),
// trace_criterion(state, cov), relative_entropy(state), write_state(path, state),
// read_state + variance/trace/entropy of the file states.  Plus the standalone
// randomized_ghep (lowrank.hpp:208-213) and RealizationPropagator::at in FFT mode.
//
// The harness around the bodies stands in for what the driver gets from ExperimentConfig
// (config.hpp) — the problem is read from <in>/problem.txt, H from <in>/h.txt and the
// observations from <in>/obs.txt (written by tests/test_gpu_driver_verbatim.py).
//   driver_verbatim <in_dir> <out_dir>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <filesystem>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <limits>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "fastkf_b200.hpp"

namespace fs = std::filesystem;

namespace fastkf {
namespace detail {  // the driver's helpers (driver.hpp:43-87), restated for the harness
inline std::string step_file(const std::string& prefix, int step, const std::string& ext) {
    std::ostringstream name;
    name << prefix << std::setw(3) << std::setfill('0') << step << ext;
    return name.str();
}
template <class Fn>
double time_call(Fn&& fn) {
    const auto t0 = std::chrono::steady_clock::now();
    fn();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
inline std::uint64_t splitmix64(std::uint64_t x) {  // rng.hpp:12-18
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag) { return splitmix64(seed ^ splitmix64(tag)); }
inline std::uint64_t ghep_seed(std::uint64_t seed) { return derive_seed(seed, 3000); }
inline std::uint64_t sample_seed(std::uint64_t seed) { return derive_seed(seed, 5000); }
inline double rel_l2_vs(const Vector&, const std::optional<std::vector<Vector>>&, int) {
    return std::numeric_limits<double>::quiet_NaN();  // no reference run in this harness
}
}  // namespace detail

struct MetricsRow {  // driver.hpp:155-163
    int step = 0;
    double wall_s = 0.0, rel_l2 = 0.0, effective_rank = 0.0, trace = 0.0, entropy = 0.0;
};
struct RunResult {
    std::vector<MetricsRow> metrics;
};
struct Cfg {  // the ExperimentConfig fields the bodies read
    Grid grid;
    KernelSpec kernel;
    double sigma2 = 0.0;
    std::uint64_t seed = 0;
    int rank = 0;
    struct { Index oversampling = 20; } filter;
    struct { int n_steps = 0; } time;
    Index ghep_rank() const { return rank; }
};
inline CovarianceOperator build_operator(const Grid& g, const KernelSpec& k, CovMode mode) { return {g, k, mode}; }
enum class UqWhat { variance, trace, entropy };
}  // namespace fastkf

using namespace fastkf;

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    const fs::path in_dir = argv[1], out_dir = argv[2];
    fs::create_directories(out_dir);
    Cfg cfg;
    {
        std::ifstream pf(in_dir / "problem.txt");
        int nx = 0, ny = 0, fam = 0;
        pf >> nx >> ny >> fam >> cfg.kernel.theta >> cfg.kernel.length >> cfg.kernel.nu >> cfg.sigma2 >> cfg.seed >>
            cfg.rank >> cfg.filter.oversampling >> cfg.time.n_steps;
        cfg.grid = Grid(nx, ny);
        cfg.kernel.family = fam ? KernelFamily::matern : KernelFamily::powered_exponential;
    }
    SparseRowMatrix h;
    {
        std::ifstream hf(in_dir / "h.txt");
        long long nnz = 0;
        hf >> h.m >> h.n >> nnz;
        h.rowptr.resize(size_t(h.m) + 1);
        h.col.resize(size_t(nnz));
        h.val.resize(size_t(nnz));
        for (auto& v : h.rowptr) hf >> v;
        for (auto& v : h.col) hf >> v;
        for (auto& v : h.val) hf >> v;
    }
    std::vector<Vector> obs(size_t(cfg.time.n_steps), Vector(h.m));
    {
        std::ifstream of(in_dir / "obs.txt");
        for (auto& y : obs)
            for (Index i = 0; i < y.size(); ++i) of >> y[i];
    }
    const int n_steps = cfg.time.n_steps;
    const Index n = cfg.grid.size();
    std::optional<std::vector<Vector>> refs;
    RunResult result;
    auto write_mean = [&](int step, const Vector& mean) {
        write_field(out_dir / detail::step_file("mean_step", step, ".fkf"), cfg.grid.nx, cfg.grid.ny, mean);
    };

    {  // ---- cmd_run, FilterKind::fkf (driver.hpp:278-303)
        const CovarianceOperator cov = build_operator(cfg.grid, cfg.kernel, CovMode::fft);
        const Index l_max = std::min<Index>(cfg.ghep_rank() + cfg.filter.oversampling, n);
        const Index k_rank = std::min<Index>(cfg.ghep_rank(), l_max);
        const FkfContext ctx = fkf_init(cov, h, cfg.sigma2, k_rank, l_max - k_rank, detail::ghep_seed(cfg.seed));
        LowRankState state = LowRankState::zero_start(n);
        write_mean(0, state.mean);
        for (int k = 1; k <= n_steps; ++k) {
            MetricsRow row;
            row.step = k;
            row.wall_s = detail::time_call([&] { state = fkf_step(state, ctx, obs[static_cast<std::size_t>(k - 1)]); });
            row.rel_l2 = detail::rel_l2_vs(state.mean, refs, k);
            row.effective_rank = static_cast<double>(state.rank());
            row.trace = trace_criterion(state, cov);
            row.entropy = relative_entropy(state);
            result.metrics.push_back(row);
            write_mean(k, state.mean);
            write_state(out_dir / detail::step_file("state_step", k, ".fks"), state);
        }
        std::ofstream mf(out_dir / "metrics.csv");
        mf << "step,trace_criterion,relative_entropy,effective_rank\n" << std::setprecision(17);
        for (const auto& r : result.metrics) mf << r.step << "," << r.trace << "," << r.entropy << "," << r.effective_rank << "\n";

        // RealizationPropagator in FFT mode on the final state (draws 0..2 of sample_seed)
        for (std::uint64_t j = 0; j < 3; ++j) {
            const RealizationPropagator prop(cov, detail::sample_seed(cfg.seed), j);
            write_field(out_dir / detail::step_file("sample_r", int(j), ".fkf"), cfg.grid.nx, cfg.grid.ny,
                        prop.at(state));
        }
        // the dense-root signature refuses FFT mode as the reference does (covariance.hpp:156-159)
        bool refused = false;
        try {
            RealizationPropagator bad(cov, Vector(n));
        } catch (const std::runtime_error& e) {
            refused = std::string(e.what()).find("dense") != std::string::npos;
        }
        if (!refused) return 5;
        // standalone randomized_ghep (lowrank.hpp:208-213) with a_apply = HᵀH/σ²
        const GepResult g = randomized_ghep(normal_operator(h, cfg.sigma2), cov, k_rank, l_max - k_rank,
                                            detail::ghep_seed(cfg.seed));
        std::ofstream lf(out_dir / "ghep_lambda.txt");
        lf << std::setprecision(17);
        for (Index i = 0; i < g.lambda.size(); ++i) lf << g.lambda[i] << "\n";
        if (g.u.cols() != g.rank() || g.u.rows() != n) return 6;
    }

    {  // ---- cmd_uq (driver.hpp:394-406) over the saved states, all three measures
        const fs::path run_dir = out_dir;
        const fs::path uq_dir = out_dir / "uq";
        fs::create_directories(uq_dir);
        const CovarianceOperator cov = build_operator(cfg.grid, cfg.kernel, CovMode::fft);
        for (UqWhat what : {UqWhat::variance, UqWhat::trace, UqWhat::entropy}) {
            std::optional<std::ofstream> csv;
            if (what == UqWhat::trace) {
                csv.emplace(uq_dir / "uq_trace.csv");
                *csv << std::setprecision(17) << "step,trace_criterion\n";
            } else if (what == UqWhat::entropy) {
                csv.emplace(uq_dir / "uq_entropy.csv");
                *csv << std::setprecision(17) << "step,relative_entropy\n";
            }
            for (int k = 1; k <= n_steps; ++k) {
                const LowRankState state = read_state(run_dir / detail::step_file("state_step", k, ".fks"));
                switch (what) {
                    case UqWhat::variance:
                        write_field(uq_dir / detail::step_file("variance_step", k, ".fkf"), cfg.grid.nx, cfg.grid.ny,
                                    variance(state, cov));
                        break;
                    case UqWhat::trace:
                        *csv << k << "," << trace_criterion(state, cov) << "\n";
                        break;
                    case UqWhat::entropy:
                        *csv << k << "," << relative_entropy(state) << "\n";
                        break;
                }
            }
        }
    }
    std::printf("driver ok\n");
    return 0;
}
