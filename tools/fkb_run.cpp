// fkb_run.cpp — reference-style driver over the drop-in shim (include/fastkf_b200.hpp):
// the fkf / ekf / enkf branches of cmd_run (driver.hpp:203-340) on an experiment directory
// written by paper_1405_2276_b200/experiment.py (truth_stepNNN.fkf, observations.csv,
// layout.csv, experiment.txt; the reference keeps the parameters in config.json, whose JSON
// parser is not part of this build).  Writes mean_stepNNN.fkf per step, FKS1 states
// (--states final|all|none; a constant-H state fetches W = U from the device only here) and
// metrics.csv (driver.hpp:155-171), with rel_l2 against the truth fields.
//
//   fkb_run <data_dir> <out_dir> fkf|ekf|enkf [--members N] [--boxcox A] [--init S] [--states W]
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <limits>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "fastkf_b200.hpp"

using namespace fastkf;

namespace {
std::uint64_t splitmix64(std::uint64_t z) {  // rng.hpp:12-18
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t tag) { return splitmix64(seed ^ splitmix64(tag)); }  // :22-24
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
struct Row {
    int step;
    double wall, rel, rank, trace, entropy;
};
}  // namespace

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: fkb_run <data_dir> <out_dir> fkf|ekf|enkf [--members N] [--boxcox A] "
                             "[--init S] [--states final|all|none]\n");
        return 2;
    }
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
    try {
        std::filesystem::create_directories(out);
        auto P = read_params(data + "/experiment.txt");
        const int nx = std::stoi(P["nx"]), ny = std::stoi(P["ny"]), n_steps = std::stoi(P["n_steps"]);
        const Grid grid(nx, ny);
        KernelSpec spec;
        spec.family = std::stoi(P["family"]) ? KernelFamily::matern : KernelFamily::powered_exponential;
        spec.theta = std::stod(P["theta"]);
        spec.length = std::stod(P["length"]);
        spec.nu = std::stod(P["nu"]);
        double sigma2 = std::stod(P["sigma2"]);
        const Index k_rank = std::stoll(P["rank"]), p_over = std::stoll(P["oversampling"]);
        const std::uint64_t seed = std::stoull(P["seed"]);
        // H: build_H per layout block, rows stacked (tomography.hpp:130-146)
        std::ifstream lay(data + "/layout.csv");
        std::string line;
        std::getline(lay, line);
        std::map<int, SourceReceiverLayout> blocks;
        while (std::getline(lay, line)) {
            int b = 0;
            char role[8] = {0};
            double x = 0.0, y = 0.0;
            if (std::sscanf(line.c_str(), "%d,%3[a-z],%lf,%lf", &b, role, &x, &y) != 4) continue;
            (std::string(role) == "src" ? blocks[b].sources : blocks[b].receivers).push_back({x, y});
        }
        SparseRowMatrix h;
        h.n = int(grid.size());
        for (auto& [b, L] : blocks) {
            const SparseRowMatrix hb = build_H(grid, L);
            for (int r = 0; r < hb.m; ++r) {
                for (int e = hb.rowptr[size_t(r)]; e < hb.rowptr[size_t(r) + 1]; ++e) {
                    h.col.push_back(hb.col[size_t(e)]);
                    h.val.push_back(hb.val[size_t(e)]);
                }
                h.rowptr.push_back(int(h.col.size()));
            }
            h.m += hb.m;
        }
        std::vector<Vector> obs = read_observations(data + "/observations.csv", n_steps, h.m);
        std::ifstream rs(data + "/ray_std.csv");
        if (rs) {  // per-ray noise: exact whitening, σ² = 1
            std::vector<double> sd(size_t(h.m));
            for (auto& v : sd) rs >> v;
            for (int r = 0; r < h.m; ++r)
                for (int e = h.rowptr[size_t(r)]; e < h.rowptr[size_t(r) + 1]; ++e) h.val[size_t(e)] /= sd[size_t(r)];
            for (auto& y : obs)
                for (Index r = 0; r < y.size(); ++r) y[r] /= sd[size_t(r)];
            sigma2 = 1.0;
        }
        const CovarianceOperator cov(grid, spec, CovMode::fft);
        std::vector<Row> rows;
        auto timed = [](auto&& fn) {
            const auto t0 = std::chrono::steady_clock::now();
            fn();
            return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        };
        const double nan = std::numeric_limits<double>::quiet_NaN();
        if (kind == "fkf") {  // driver.hpp:278-303
            FkfContext c2 = fkf_init(cov, h, sigma2, k_rank, p_over, derive_seed(seed, 3000));  // ghep_seed (:83)
            LowRankState st = LowRankState::zero_start(grid.size());
            write_field(step_file(out, "mean_step", 0, ".fkf"), nx, ny, st.mean);
            for (int k = 1; k <= n_steps; ++k) {
                Row r{k, 0, 0, 0, 0, 0};
                r.wall = timed([&] { st = fkf_step(st, c2, obs[size_t(k - 1)]); });
                r.rel = rel_l2(st.mean, read_field(step_file(data, "truth_step", k, ".fkf")).data);
                r.rank = double(st.rank());
                r.trace = trace_criterion(st, c2);
                r.entropy = relative_entropy(st, c2);
                rows.push_back(r);
                write_field(step_file(out, "mean_step", k, ".fkf"), nx, ny, st.mean);
                if (states == "all" || (states == "final" && k == n_steps))
                    write_state(step_file(out, "state_step", k, ".fks"), st, c2);
            }
        } else if (kind == "ekf") {  // driver.hpp:304-333
            const BoxCox t{bc};
            FekfOptions opts;
            opts.k_rank = k_rank;
            opts.oversampling = p_over;
            opts.trunc_tol = 1e-5;
            LowRankState st = LowRankState::zero_start(grid.size());
            const double s0 = bc == 1.0 ? init - 1.0 : bc * (std::pow(init, 1.0 / bc) - 1.0);  // forward(init)
            st.mean = Vector::Constant(grid.size(), s0);
            auto physical = [&](const Vector& m) {
                Vector o(m.size());
                for (Index i = 0; i < m.size(); ++i) o[i] = bc == 1.0 ? m[i] + 1.0 : std::pow((m[i] + bc) / bc, bc);
                return o;
            };
            write_field(step_file(out, "mean_step", 0, ".fkf"), nx, ny, physical(st.mean));
            for (int k = 1; k <= n_steps; ++k) {
                opts.seed = derive_seed(seed, 4000 + std::uint64_t(k));  // ekf_seed (driver.hpp:84-86)
                Row r{k, 0, 0, 0, 0, 0};
                r.wall = timed([&] { st = fekf_step(st, cov, h, obs[size_t(k - 1)], sigma2, t, opts); });
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
                const std::uint64_t es = derive_seed(seed, 2000 + std::uint64_t(k));  // enkf_seed (driver.hpp:80-82)
                Row r{k, 0, 0, double(members), nan, nan};
                r.wall = timed([&] { enkf_step(ens, h, obs[size_t(k - 1)], cov, sigma2, es); });
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
        std::printf("%s: %d steps, last rel_l2 %.6g\n", kind.c_str(), n_steps, rows.empty() ? nan : rows.back().rel);
        return 0;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "fkb_run: %s\n", e.what());
        return 1;
    }
}
