// fkb_run.cpp — reference-style driver over the drop-in shim (include/fastkf_b200.hpp), the
// commands of driver.hpp that sit on the filter hot path:
//
//   fkb_run <data_dir> <out_dir> fkf|ekf|enkf [--members N] [--boxcox A] [--init S] [--states W]
//       cmd_run (driver.hpp:203-340) on an experiment directory written by
//       paper_1405_2276_b200/experiment.py (truth_stepNNN.fkf, observations.csv, layout.csv,
//       experiment.txt — the reference keeps the parameters in config.json, whose JSON parser is
//       not part of this build).  Writes mean_stepNNN.fkf per step, FKS1 states (--states
//       final|all|none; a constant-H state fetches W = U from the device only here), metrics.csv
//       (driver.hpp:155-171, rel_l2 against the truth fields) and the run's parameters
//       (experiment.txt + layout.csv [+ ray_std.csv], the cfg.save of :338).
//   fkb_run uq <run_dir> <out_dir> variance|trace|entropy [--steps 1,2,...]
//       cmd_uq (driver.hpp:368-406) over the FKS1 states of an fkf/ekf run.
//   fkb_run sample <run_dir> <out_dir> <count> [--seed S] [--steps 1,2,...]
//       cmd_sample (driver.hpp:411-460) in FFT mode: realization j
//       propagates the torus draw j of sample_seed through every selected state of an fkf run
//       (W = U of the rebuilt context, whose Γ⁻¹U the GHEP provides).  ekf runs are refused:
//       their files carry W but not Γ⁻¹W.
//   fkb_run bench <data_dir> <out_csv> <grids WxH,...> [fkf|ekf|enkf] [--members N]
//       cmd_bench (driver.hpp:489-616): per grid, the offline time (operator + fkf_init), one
//       warm step, then the median/min/max of 5 timed steps from the warm state, on a cross-well
//       layout with the experiment's sources/receivers per side and y = gaussian_vector(m,
//       derive_seed(seed, 7000)); CSV "grid,nx,ny,n_s,kind,offline_s,step_median_s,...".
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "fastkf_b200.hpp"

using namespace fastkf;
namespace fs = std::filesystem;

namespace {
std::string step_file(const std::string& dir, const char* prefix, int k, const char* ext) {  // driver.hpp:43-47
    char b[64];
    std::snprintf(b, sizeof b, "%s%03d%s", prefix, k, ext);
    return dir + "/" + b;
}
std::map<std::string, std::string> read_params(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open " + path);
    std::map<std::string, std::string> kv;
    std::string k, v;
    while (in >> k >> v) kv[k] = v;
    return kv;
}
std::vector<Vector> read_observations(const std::string& path, int n_steps, Index m) {  // driver.hpp:100-130
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open observations: " + path);
    std::string line;
    if (!std::getline(in, line) || line.rfind("step,measurement,value", 0) != 0)
        throw std::runtime_error("unexpected observations header in " + path);
    std::vector<Vector> out(static_cast<size_t>(n_steps), Vector{m});
    while (std::getline(in, line)) {
        int k = 0;
        long long i = 0;
        double v = 0.0;
        if (std::sscanf(line.c_str(), "%d,%lld,%lf", &k, &i, &v) != 3) continue;
        if (k >= 1 && k <= n_steps && i >= 0 && i < m) out[size_t(k - 1)][i] = v;
    }
    return out;
}
double rel_l2(const Vector& a, const Vector& ref) {
    double num = 0.0, den = 0.0;
    for (Index i = 0; i < a.size(); ++i) {
        num += (a[i] - ref[i]) * (a[i] - ref[i]);
        den += ref[i] * ref[i];
    }
    return den > 0.0 ? std::sqrt(num / den) : std::numeric_limits<double>::quiet_NaN();
}
template <class Fn>
double timed(Fn&& fn) {  // detail::time_call (driver.hpp:63-69)
    const auto t0 = std::chrono::steady_clock::now();
    fn();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}
std::vector<int> parse_steps(const std::string& text, int n_steps) {
    std::vector<int> steps;
    std::istringstream in(text);
    std::string item;
    while (std::getline(in, item, ','))
        if (!item.empty()) steps.push_back(std::stoi(item));
    if (steps.empty())
        for (int k = 1; k <= n_steps; ++k) steps.push_back(k);
    return steps;
}
struct Row {
    int step;
    double wall, rel, rank, trace, entropy;
};

// The experiment (the parts of ExperimentConfig the filter path reads): grid, kernel, noise,
// GHEP sizes, seed, and H built per layout block with the rows stacked (tomography.hpp:130-146);
// per-ray noise (ray_std.csv) is whitened exactly (σ² = 1).
struct Experiment {
    std::map<std::string, std::string> P;
    Grid grid;
    KernelSpec spec;
    double sigma2 = 0.0;
    Index k_rank = 0, p_over = 20;
    std::uint64_t seed = 0;
    int n_steps = 0;
    SparseRowMatrix h;
    std::vector<double> ray_sd;  // empty: scalar noise
    std::map<int, SourceReceiverLayout> blocks;
};
Experiment load_experiment(const std::string& dir) {
    Experiment e;
    e.P = read_params(dir + "/experiment.txt");
    auto& P = e.P;
    e.grid = Grid(std::stoi(P["nx"]), std::stoi(P["ny"]));
    e.spec.family = std::stoi(P["family"]) ? KernelFamily::matern : KernelFamily::powered_exponential;
    e.spec.theta = std::stod(P["theta"]);
    e.spec.length = std::stod(P["length"]);
    e.spec.nu = std::stod(P["nu"]);
    e.sigma2 = std::stod(P["sigma2"]);
    e.k_rank = std::stoll(P["rank"]);
    e.p_over = std::stoll(P["oversampling"]);
    e.seed = std::stoull(P["seed"]);
    e.n_steps = std::stoi(P["n_steps"]);
    std::ifstream lay(dir + "/layout.csv");
    if (!lay) throw std::runtime_error("cannot open " + dir + "/layout.csv");
    std::string line;
    std::getline(lay, line);
    while (std::getline(lay, line)) {
        int b = 0;
        char role[8] = {0};
        double x = 0.0, y = 0.0;
        if (std::sscanf(line.c_str(), "%d,%3[a-z],%lf,%lf", &b, role, &x, &y) != 4) continue;
        (std::string(role) == "src" ? e.blocks[b].sources : e.blocks[b].receivers).push_back({x, y});
    }
    e.h.n = int(e.grid.size());
    for (auto& [b, L] : e.blocks) {
        const SparseRowMatrix hb = build_H(e.grid, L);
        for (int r = 0; r < hb.m; ++r) {
            for (int k = hb.rowptr[size_t(r)]; k < hb.rowptr[size_t(r) + 1]; ++k) {
                e.h.col.push_back(hb.col[size_t(k)]);
                e.h.val.push_back(hb.val[size_t(k)]);
            }
            e.h.rowptr.push_back(int(e.h.col.size()));
        }
        e.h.m += hb.m;
    }
    std::ifstream rs(dir + "/ray_std.csv");
    if (rs) {
        e.ray_sd.resize(size_t(e.h.m));
        for (auto& v : e.ray_sd) rs >> v;
        for (int r = 0; r < e.h.m; ++r)
            for (int k = e.h.rowptr[size_t(r)]; k < e.h.rowptr[size_t(r) + 1]; ++k) e.h.val[size_t(k)] /= e.ray_sd[size_t(r)];
        e.sigma2 = 1.0;
    }
    return e;
}
void save_experiment(const std::string& data, const std::string& out, const std::string& kind) {  // cfg.save (:338)
    fs::copy_file(data + "/experiment.txt", out + "/experiment.txt", fs::copy_options::overwrite_existing);
    fs::copy_file(data + "/layout.csv", out + "/layout.csv", fs::copy_options::overwrite_existing);
    if (fs::exists(data + "/ray_std.csv"))
        fs::copy_file(data + "/ray_std.csv", out + "/ray_std.csv", fs::copy_options::overwrite_existing);
    std::ofstream(out + "/experiment.txt", std::ios::app) << "kind " << kind << "\n";
}

// ------------------------------------------------------------------------- cmd_run
int cmd_run(int argc, char** argv) {
    const std::string data = argv[1], out = argv[2], kind = argv[3];
    Index members = 1000;
    double bc = 1.0, init = 0.0;
    std::string states = "final";
    for (int a = 4; a + 1 < argc; a += 2) {
        const std::string f = argv[a], v = argv[a + 1];
        if (f == "--members") members = std::stoll(v);
        else if (f == "--boxcox") bc = std::stod(v);
        else if (f == "--init") init = std::stod(v);
        else if (f == "--states") states = v;
    }
    fs::create_directories(out);
    Experiment e = load_experiment(data);
    const int nx = e.grid.nx, ny = e.grid.ny, n_steps = e.n_steps;
    const SparseRowMatrix& h = e.h;
    std::vector<Vector> obs = read_observations(data + "/observations.csv", n_steps, h.m);
    if (!e.ray_sd.empty())
        for (auto& y : obs)
            for (Index r = 0; r < y.size(); ++r) y[r] /= e.ray_sd[size_t(r)];
    const CovarianceOperator cov(e.grid, e.spec, CovMode::fft);
    std::vector<Row> rows;
    const double nan = std::numeric_limits<double>::quiet_NaN();
    if (kind == "fkf") {  // driver.hpp:278-303
        const FkfContext ctx = fkf_init(cov, h, e.sigma2, e.k_rank, e.p_over, derive_seed(e.seed, 3000));  // ghep_seed (:83)
        LowRankState st = LowRankState::zero_start(e.grid.size());
        write_field(step_file(out, "mean_step", 0, ".fkf"), nx, ny, st.mean);
        for (int k = 1; k <= n_steps; ++k) {
            Row r{k, 0, 0, 0, 0, 0};
            r.wall = timed([&] { st = fkf_step(st, ctx, obs[size_t(k - 1)]); });
            r.rel = rel_l2(st.mean, read_field(step_file(data, "truth_step", k, ".fkf")).data);
            r.rank = double(st.rank());
            r.trace = trace_criterion(st, cov);
            r.entropy = relative_entropy(st);
            rows.push_back(r);
            write_field(step_file(out, "mean_step", k, ".fkf"), nx, ny, st.mean);
            if (states == "all" || (states == "final" && k == n_steps))
                write_state(step_file(out, "state_step", k, ".fks"), st);
        }
    } else if (kind == "ekf") {  // driver.hpp:304-333
        const BoxCox t{bc};
        FekfOptions opts;
        opts.k_rank = e.k_rank;
        opts.oversampling = e.p_over;
        opts.trunc_tol = 1e-5;
        LowRankState st = LowRankState::zero_start(e.grid.size());
        const double s0 = bc == 1.0 ? init - 1.0 : bc * (std::pow(init, 1.0 / bc) - 1.0);  // forward(init)
        st.mean = Vector::Constant(e.grid.size(), s0);
        auto physical = [&](const Vector& m) {
            Vector o(m.size());
            for (Index i = 0; i < m.size(); ++i) o[i] = bc == 1.0 ? m[i] + 1.0 : std::pow((m[i] + bc) / bc, bc);
            return o;
        };
        write_field(step_file(out, "mean_step", 0, ".fkf"), nx, ny, physical(st.mean));
        for (int k = 1; k <= n_steps; ++k) {
            opts.seed = derive_seed(e.seed, 4000 + std::uint64_t(k));  // ekf_seed (driver.hpp:84-86)
            Row r{k, 0, 0, 0, 0, 0};
            r.wall = timed([&] { st = fekf_step(st, cov, h, obs[size_t(k - 1)], e.sigma2, t, opts); });
            const Vector phys = physical(st.mean);
            r.rel = rel_l2(phys, read_field(step_file(data, "truth_step", k, ".fkf")).data);
            r.rank = double(st.rank());
            r.trace = trace_criterion(st, cov);  // driver.hpp:328-329
            r.entropy = relative_entropy(st);
            rows.push_back(r);
            write_field(step_file(out, "mean_step", k, ".fkf"), nx, ny, phys);
            if (states == "all" || (states == "final" && k == n_steps))
                write_state(step_file(out, "state_step", k, ".fks"), st);
        }
    } else if (kind == "enkf") {  // driver.hpp (enkf branch)
        Ensemble ens = enkf_init(cov, h, members);
        for (int k = 1; k <= n_steps; ++k) {
            const std::uint64_t es = derive_seed(e.seed, 2000 + std::uint64_t(k));  // enkf_seed (driver.hpp:80-82)
            Row r{k, 0, 0, double(members), nan, nan};
            r.wall = timed([&] { enkf_step(ens, h, obs[size_t(k - 1)], cov, e.sigma2, es); });
            const Vector m = ens.mean();
            r.rel = rel_l2(m, read_field(step_file(data, "truth_step", k, ".fkf")).data);
            rows.push_back(r);
            write_field(step_file(out, "mean_step", k, ".fkf"), nx, ny, m);
        }
    } else {
        throw std::invalid_argument("unknown filter kind: " + kind);
    }
    std::ofstream mf(out + "/metrics.csv");  // write_metrics (driver.hpp:163-171)
    mf.precision(17);
    mf << "step,wall_time_s,rel_l2_error,effective_rank,trace_criterion,relative_entropy\n";
    for (const Row& r : rows)
        mf << r.step << "," << r.wall << "," << r.rel << "," << r.rank << "," << r.trace << "," << r.entropy << "\n";
    save_experiment(data, out, kind);
    std::printf("%s: %d steps, last rel_l2 %.6g\n", kind.c_str(), n_steps, rows.empty() ? nan : rows.back().rel);
    return 0;
}

// ------------------------------------------------------------------------- cmd_uq
int cmd_uq(int argc, char** argv) {  // driver.hpp:368-406
    const std::string run = argv[2], out = argv[3], what = argv[4];
    std::string steps_arg;
    for (int a = 5; a + 1 < argc; a += 2)
        if (std::string(argv[a]) == "--steps") steps_arg = argv[a + 1];
    Experiment e = load_experiment(run);
    const std::string kind = e.P["kind"];
    if (kind != "fkf" && kind != "ekf")
        throw std::runtime_error("cmd_uq: measures need low-rank covariance snapshots, which '" + kind +
                                 "' runs do not save");
    if (what != "variance" && what != "trace" && what != "entropy")
        throw std::invalid_argument("cmd_uq: unknown measure '" + what + "'");
    const std::vector<int> steps = parse_steps(steps_arg, e.n_steps);
    fs::create_directories(out);
    const CovarianceOperator cov(e.grid, e.spec, CovMode::fft);
    std::optional<std::ofstream> csv;
    if (what == "trace") {
        csv.emplace(out + "/uq_trace.csv");
        *csv << "step,trace_criterion\n";
    } else if (what == "entropy") {
        csv.emplace(out + "/uq_entropy.csv");
        *csv << "step,relative_entropy\n";
    }
    if (csv) csv->precision(17);
    for (int k : steps) {
        if (k < 1 || k > e.n_steps)
            throw std::runtime_error("cmd_uq: step " + std::to_string(k) + " outside 1.." + std::to_string(e.n_steps));
        const LowRankState state = read_state(step_file(run, "state_step", k, ".fks"));
        if (what == "variance")
            write_field(step_file(out, "variance_step", k, ".fkf"), e.grid.nx, e.grid.ny, variance(state, cov));
        else if (what == "trace")
            *csv << k << "," << trace_criterion(state, cov) << "\n";
        else
            *csv << k << "," << relative_entropy(state) << "\n";
    }
    return 0;
}

// ------------------------------------------------------------------------- cmd_sample
int cmd_sample(int argc, char** argv) {  // driver.hpp:411-460, FFT mode
    const std::string run = argv[2], out = argv[3];
    const int count = std::stoi(argv[4]);
    std::string steps_arg;
    std::optional<std::uint64_t> seed_override;
    for (int a = 5; a + 1 < argc; a += 2) {
        const std::string f = argv[a];
        if (f == "--steps") steps_arg = argv[a + 1];
        else if (f == "--seed") seed_override = std::stoull(argv[a + 1]);
    }
    Experiment e = load_experiment(run);
    const std::string kind = e.P["kind"];
    if (kind != "fkf" && kind != "ekf")
        throw std::runtime_error("cmd_sample: sampling needs low-rank covariance snapshots, which '" + kind +
                                 "' runs do not save");
    if (kind == "ekf")
        throw std::runtime_error("cmd_sample: FFT-mode sampling of saved ekf states needs Γ⁻¹W, which FKS1 files "
                                 "do not carry (sample from a live fekf filter instead)");
    if (count < 1) throw std::invalid_argument("cmd_sample: count must be positive");
    const std::vector<int> steps = parse_steps(steps_arg, e.n_steps);
    std::vector<LowRankState> states;
    for (int k : steps) {
        if (k < 1 || k > e.n_steps)
            throw std::runtime_error("cmd_sample: step " + std::to_string(k) + " outside 1.." + std::to_string(e.n_steps));
        states.push_back(read_state(step_file(run, "state_step", k, ".fks")));
    }
    fs::create_directories(out);
    const CovarianceOperator cov(e.grid, e.spec, CovMode::fft);
    // W = U of the run's context: rebuild it (deterministic in the GHEP seed) and check the
    // saved W against it, then bind the saved (α, d, mean) to it — W̄ = Γ⁻¹U comes with it
    const FkfContext ctx = fkf_init(cov, e.h, e.sigma2, e.k_rank, e.p_over, derive_seed(e.seed, 3000));
    const Matrix& U = ctx.gep.u.get();
    for (size_t si = 0; si < states.size(); ++si) {
        LowRankState& s = states[si];
        if (s.rank() && (s.w.cols() != U.cols() || s.w.get().a != U.a))
            throw std::runtime_error("cmd_sample: the saved W of step " + std::to_string(steps[si]) +
                                     " is not the context's U (different configuration or build)");
        s.fkf = ctx.dev;
    }
    const std::uint64_t seed = derive_seed(seed_override.value_or(e.seed), 5000);  // sample_seed (:87)
    for (int j = 0; j < count; ++j) {
        const RealizationPropagator prop(cov, seed, std::uint64_t(j));
        for (size_t si = 0; si < steps.size(); ++si) {
            char name[64];
            std::snprintf(name, sizeof name, "/sample_step%03d_r%03d.fkf", steps[si], j);
            write_field(out + name, e.grid.nx, e.grid.ny, prop.at(states[si]));
        }
    }
    return 0;
}

// ------------------------------------------------------------------------- cmd_bench
int cmd_bench(int argc, char** argv) {  // driver.hpp:489-616
    const std::string data = argv[2], out_csv = argv[3], grid_list = argv[4];
    std::string kind = argc > 5 && argv[5][0] != '-' ? argv[5] : "fkf";
    Index members = 1000;
    for (int a = 5; a + 1 < argc; ++a)
        if (std::string(argv[a]) == "--members") members = std::stoll(argv[a + 1]);
    Experiment e = load_experiment(data);
    if (e.blocks.empty()) throw std::invalid_argument("bench: the experiment has no ray layout");
    const int n_sou = int(e.blocks.begin()->second.sources.size());
    const int n_rec = int(e.blocks.begin()->second.receivers.size());
    std::vector<Grid> grids;
    {
        std::istringstream in(grid_list);
        std::string item;
        while (std::getline(in, item, ',')) {
            const auto sep = item.find('x');
            if (sep == std::string::npos) throw std::invalid_argument("bench: grid '" + item + "' is not WxH");
            grids.emplace_back(std::stoi(item.substr(0, sep)), std::stoi(item.substr(sep + 1)));
        }
        if (grids.empty()) throw std::invalid_argument("bench: empty grid list");
    }
    constexpr int kReps = 5;
    std::ofstream out(out_csv);
    if (!out) throw std::runtime_error("cannot open for writing: " + out_csv);
    out << "grid,nx,ny,n_s,kind,offline_s,step_median_s,step_min_s,step_max_s\n";
    for (const Grid& grid : grids) {
        const SparseRowMatrix h = build_H(grid, SourceReceiverLayout::cross_well(grid, n_sou, n_rec));
        const Vector y = gaussian_vector(h.rows(), derive_seed(e.seed, 7000));
        const Index n = grid.size();
        double offline = 0.0;
        std::vector<double> times;
        if (kind == "fkf") {
            std::optional<CovarianceOperator> cov;
            std::optional<FkfContext> ctx;
            offline = timed([&] {
                cov.emplace(grid, e.spec, CovMode::fft);
                const Index l_max = std::min<Index>(e.k_rank + e.p_over, n);
                const Index k_rank = std::min<Index>(e.k_rank, l_max);
                ctx = fkf_init(*cov, h, e.sigma2, k_rank, l_max - k_rank, derive_seed(e.seed, 3000));
            });
            const LowRankState warm = fkf_step(LowRankState::zero_start(n), *ctx, y);
            for (int rep = 0; rep < kReps; ++rep) {
                LowRankState state = warm;
                times.push_back(timed([&] { state = fkf_step(state, *ctx, y); }));
            }
        } else if (kind == "ekf") {
            std::optional<CovarianceOperator> cov;
            offline = timed([&] { cov.emplace(grid, e.spec, CovMode::fft); });
            FekfOptions opts;
            opts.k_rank = std::min<Index>(e.k_rank, n - e.p_over);
            opts.oversampling = e.p_over;
            opts.seed = derive_seed(e.seed, 4001);
            LowRankState start = LowRankState::zero_start(n);
            start.mean = Vector::Constant(n, -1.0);  // Box–Cox 1, init_slowness 0
            LowRankState state = fekf_step(start, *cov, h, y, e.sigma2, BoxCox{1.0}, opts);
            // a device fekf filter holds only its latest state: the reps continue the chain
            for (int rep = 0; rep < kReps; ++rep) {
                opts.seed = derive_seed(e.seed, 4000 + std::uint64_t(2 + rep));
                times.push_back(timed([&] { state = fekf_step(state, *cov, h, y, e.sigma2, BoxCox{1.0}, opts); }));
            }
        } else if (kind == "enkf") {
            std::optional<CovarianceOperator> cov;
            offline = timed([&] { cov.emplace(grid, e.spec, CovMode::fft); });
            Ensemble ens = enkf_init(*cov, h, members);
            enkf_step(ens, h, y, *cov, e.sigma2, derive_seed(e.seed, 2001));
            for (int rep = 0; rep < kReps; ++rep)
                times.push_back(timed([&] { enkf_step(ens, h, y, *cov, e.sigma2, derive_seed(e.seed, 2000 + 2 + rep)); }));
        } else {
            throw std::invalid_argument("bench: unknown filter kind '" + kind + "'");
        }
        out.precision(9);
        out << grid.nx << "x" << grid.ny << "," << grid.nx << "," << grid.ny << "," << n << "," << kind << "," << offline
            << "," << median(times) << "," << *std::min_element(times.begin(), times.end()) << ","
            << *std::max_element(times.begin(), times.end()) << "\n";
    }
    if (!out) throw std::runtime_error("write failed: " + out_csv);
    return 0;
}
}  // namespace

int main(int argc, char** argv) {
    const std::string cmd = argc > 1 ? argv[1] : "";
    try {
        if (cmd == "uq" && argc >= 5) return cmd_uq(argc, argv);
        if (cmd == "sample" && argc >= 5) return cmd_sample(argc, argv);
        if (cmd == "bench" && argc >= 5) return cmd_bench(argc, argv);
        if (argc >= 4 && cmd != "uq" && cmd != "sample" && cmd != "bench") return cmd_run(argc, argv);
        std::fprintf(stderr,
                     "usage: fkb_run <data_dir> <out_dir> fkf|ekf|enkf [--members N] [--boxcox A] [--init S] "
                     "[--states final|all|none]\n"
                     "       fkb_run uq <run_dir> <out_dir> variance|trace|entropy [--steps 1,2,...]\n"
                     "       fkb_run sample <run_dir> <out_dir> <count> [--seed S] [--steps 1,2,...]\n"
                     "       fkb_run bench <data_dir> <out_csv> <WxH,...> [fkf|ekf|enkf] [--members N]\n");
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "fkb_run: %s\n", e.what());
        return 1;
    }
}
