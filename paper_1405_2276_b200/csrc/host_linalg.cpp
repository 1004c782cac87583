// host_linalg.cpp — host-side setup pieces of the product library.
//
//  * build_H: straight-ray travel-time operator (tomography.hpp:29-146).  The survey
//    keeps H construction on the host: it runs once, and the
//    exact floating-point order of the reference decides cells on grid lines.
//  * sym_eig_small: symmetric eigensolver for the Gram/core matrices of
//    the randomized GHEP (lowrank.hpp:193 uses Eigen::SelfAdjointEigenSolver on the
//    host too).  Householder tridiagonalization + implicit-shift QL, eigenvalues
//    ascending with matching eigenvector columns.
//
// Compiled with -ffp-contract=off so trace_ray rounds exactly like the reference.

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <cstdlib>
#include <vector>

#include "host_linalg.h"

namespace fkb {

// --------------------------------------------------------------------------- tomography.hpp
struct Seg {
    long long cell;
    double length;
};

static std::vector<Seg> trace_ray(int nx, int ny, double lx, double ly, double sx, double sy, double rx,
                                  double ry) {  // tomography.hpp:29-86
    const double tol_x = 1e-12 * lx, tol_y = 1e-12 * ly;
    const double pts[2][2] = {{sx, sy}, {rx, ry}};
    for (const auto& p : pts)
        if (p[0] < -tol_x || p[0] > lx + tol_x || p[1] < -tol_y || p[1] > ly + tol_y)
            throw std::invalid_argument("trace_ray: endpoint (" + std::to_string(p[0]) + ", " + std::to_string(p[1]) +
                                        ") lies outside the domain");
    const double ddx = rx - sx, ddy = ry - sy;
    const double len = std::sqrt(ddx * ddx + ddy * ddy);
    if (len == 0.0) throw std::invalid_argument("trace_ray: degenerate zero-length ray");
    const double gdx = lx / nx, gdy = ly / ny;
    std::vector<double> ts;
    ts.reserve(size_t(nx + ny + 2));
    ts.push_back(0.0);
    ts.push_back(1.0);
    if (ddx != 0.0)
        for (int i = 1; i < nx; ++i) {
            const double t = (i * gdx - sx) / ddx;
            if (t > 0.0 && t < 1.0) ts.push_back(t);
        }
    if (ddy != 0.0)
        for (int j = 1; j < ny; ++j) {
            const double t = (j * gdy - sy) / ddy;
            if (t > 0.0 && t < 1.0) ts.push_back(t);
        }
    std::sort(ts.begin(), ts.end());
    std::vector<Seg> segs;
    double tp = ts.front();
    for (size_t i = 1; i < ts.size(); ++i) {
        const double t = ts[i];
        if (t - tp <= 1e-12) continue;  // corner sliver folds into the next interval
        const double h = 0.5 * (tp + t);
        const double mxp = sx + h * ddx, myp = sy + h * ddy;
        const int ix = std::clamp(int(std::floor(mxp / gdx)), 0, nx - 1);
        const int iy = std::clamp(int(std::floor(myp / gdy)), 0, ny - 1);
        const long long cell = (long long)ix * ny + iy;
        const double sl = (t - tp) * len;
        if (!segs.empty() && segs.back().cell == cell) segs.back().length += sl;
        else segs.push_back({cell, sl});
        tp = t;
    }
    return segs;
}

int trace_ray_into(int nx, int ny, double lx, double ly, double sx, double sy, double rx, double ry, int cap,
                   long long* cells, double* lengths) {
    auto segs = trace_ray(nx, ny, lx, ly, sx, sy, rx, ry);
    for (int i = 0; i < std::min<int>(cap, int(segs.size())); ++i) {
        cells[i] = segs[size_t(i)].cell;
        lengths[i] = segs[size_t(i)].length;
    }
    return int(segs.size());
}

void build_H(int nx, int ny, double lx, double ly, int ns, const double* src, int nr, const double* rec,
             std::vector<int>& rowptr, std::vector<int>& col, std::vector<double>& val) {  // :130-146
    if (nx < 1 || ny < 1) throw std::invalid_argument("grid: nx and ny must be positive");
    if (ns < 1 || nr < 1) throw std::invalid_argument("layout: sources and receivers must be nonempty");
    for (int e = 0; e < ns + nr; ++e) {  // SourceReceiverLayout::validate :115-125
        const double* p = e < ns ? src + 2 * e : rec + 2 * (e - ns);
        if (!(p[0] >= 0.0 && p[0] <= lx && p[1] >= 0.0 && p[1] <= ly))
            throw std::invalid_argument(e < ns ? "layout: source outside domain" : "layout: receiver outside domain");
    }
    rowptr.assign(1, 0);
    col.clear();
    val.clear();
    for (int s = 0; s < ns; ++s)
        for (int r = 0; r < nr; ++r) {
            auto segs = trace_ray(nx, ny, lx, ly, src[2 * s], src[2 * s + 1], rec[2 * r], rec[2 * r + 1]);
            // setFromTriplets: ascending column order, duplicate entries summed in input order
            std::stable_sort(segs.begin(), segs.end(), [](const Seg& a, const Seg& b) { return a.cell < b.cell; });
            long long last = -1;
            for (const Seg& g : segs) {
                if (g.cell == last) {
                    val.back() += g.length;
                    continue;
                }
                col.push_back(int(g.cell));
                val.push_back(g.length);
                last = g.cell;
            }
            rowptr.push_back(int(col.size()));
        }
}

// --------------------------------------------------------------------------- small symmetric eig
// A (n×n column-major, symmetric) → w ascending, Z eigenvectors (column j ↔ w[j]).
// Householder tridiagonalization (unblocked, column-oriented: every inner loop runs down a
// contiguous column; OpenMP over columns), explicit Q by backward accumulation, then
// implicit-shift QL whose rotations are recorded per sweep and applied to Q by row chunks in
// parallel.  The splitting test is relative to the neighbouring diagonal or to ‖T‖ (the
// reduction is backward stable to ε‖A‖ only, so a graded tridiagonal can hold off-diagonals
// at ε‖T‖ that never fall below ε(|d_m| + |d_m+1|)).
void sym_eig_small(int n, const double* A, double* w, double* Z) {
    if (n <= 0) return;
    const size_t N = size_t(n);
    std::vector<double> a(A, A + N * N);
    std::vector<double> d(N, 0.0), e(N, 0.0), tau(N, 0.0);
    auto at = [&](int i, int j) -> double& { return a[size_t(i) + size_t(j) * N]; };
    for (int j = 0; j < n; ++j)  // symmetrize into full storage from the lower triangle
        for (int i = j + 1; i < n; ++i) at(j, i) = at(i, j);
    static const int par_min = std::getenv("FKB_EIG_PAR") ? std::atoi(std::getenv("FKB_EIG_PAR")) : 400;
    const bool par = n >= par_min;  // below this the OpenMP fork/join costs more than it saves
    std::vector<double> p(N), wv(N);
    for (int k = 0; k + 2 < n; ++k) {
        // Householder v (v₀ = 1) with (I − τvvᵀ)x = βe₁ for x = A[k+1:, k]
        double* x = &at(k + 1, k);
        const int len = n - k - 1;
        double sig = 0.0;
        for (int i = 1; i < len; ++i) sig += x[i] * x[i];
        const double x0 = x[0];
        double t = 0.0, beta = x0;
        if (sig != 0.0) {
            const double mu = std::sqrt(x0 * x0 + sig);
            beta = x0 <= 0.0 ? mu : -mu;
            const double v0 = x0 - beta;
            t = -v0 / beta;  // τ = (β − x₀)/β
            for (int i = 1; i < len; ++i) x[i] /= v0;
        }
        d[size_t(k)] = at(k, k);
        e[size_t(k)] = beta;
        tau[size_t(k)] = t;
        x[0] = 1.0;  // v stored in place (v₀ = 1 explicitly during the update)
        if (t != 0.0) {
            // p = τ·A22·v (A22 symmetric, full storage: column sweeps)
            const int o = k + 1;
#pragma omp parallel for schedule(static) if (par)
            for (int i = 0; i < len; ++i) {
                const double* col = &at(o, o + i);  // A22[:, i] = A22[i, :]
                double acc = 0.0;
                for (int q = 0; q < len; ++q) acc += col[q] * x[q];
                p[size_t(i)] = t * acc;
            }
            double pv = 0.0;
            for (int i = 0; i < len; ++i) pv += p[size_t(i)] * x[i];
            const double h = 0.5 * t * pv;
            for (int i = 0; i < len; ++i) wv[size_t(i)] = p[size_t(i)] - h * x[i];
            // A22 −= v wᵀ + w vᵀ
#pragma omp parallel for schedule(static) if (par)
            for (int j = 0; j < len; ++j) {
                double* col = &at(o, o + j);
                const double vj = x[j], wj = wv[size_t(j)];
                for (int i = 0; i < len; ++i) col[i] -= x[i] * wj + wv[size_t(i)] * vj;
            }
        }
    }
    if (n >= 2) {
        d[N - 2] = at(n - 2, n - 2);
        e[N - 2] = at(n - 1, n - 2);
    }
    d[N - 1] = at(n - 1, n - 1);
    // Q = H₀H₁…H_{n−3} by backward accumulation into q (column-major)
    std::vector<double> q(N * N, 0.0);
    auto qt = [&](int i, int j) -> double& { return q[size_t(i) + size_t(j) * N]; };
    for (int i = 0; i < n; ++i) qt(i, i) = 1.0;
    for (int k = n - 3; k >= 0; --k) {
        const double t = tau[size_t(k)];
        if (t == 0.0) continue;
        const double* v = &at(k + 1, k);
        const int o = k + 1, len = n - o;
#pragma omp parallel for schedule(static) if (par)
        for (int j = o; j < n; ++j) {
            double* col = &qt(o, j);
            double acc = 0.0;
            for (int i = 0; i < len; ++i) acc += v[i] * col[i];
            acc *= t;
            for (int i = 0; i < len; ++i) col[i] -= acc * v[i];
        }
    }
    // implicit-shift QL on (d, e); e[i] couples d[i] and d[i+1]
    double tnorm = 0.0;
    for (int i = 0; i < n; ++i) tnorm = std::max(tnorm, std::fabs(d[size_t(i)]) + std::fabs(e[size_t(i)]));
    e[N - 1] = 0.0;
    const double eps = 2.220446049250313e-16;
    std::vector<double> rc(N), rs(N);
    for (int l = 0; l < n; ++l) {
        int iter = 0;
        int m;
        do {
            for (m = l; m < n - 1; ++m) {
                const double dd = std::fabs(d[size_t(m)]) + std::fabs(d[size_t(m + 1)]);
                const double em = std::fabs(e[size_t(m)]);
                if (em <= 1e-300 + eps * dd || em <= 0.5 * eps * tnorm) break;
            }
            if (m != l) {
                if (++iter > 60) throw std::runtime_error("sym_eig_small: QL iteration did not converge");
                double g = (d[size_t(l + 1)] - d[size_t(l)]) / (2.0 * e[size_t(l)]);
                double r = std::hypot(g, 1.0);
                g = d[size_t(m)] - d[size_t(l)] + e[size_t(l)] / (g + (g >= 0.0 ? std::fabs(r) : -std::fabs(r)));
                double sn = 1.0, c = 1.0, pp = 0.0;
                int i;
                int nrot = 0;
                bool early = false;
                for (i = m - 1; i >= l; --i) {
                    double f = sn * e[size_t(i)];
                    const double b = c * e[size_t(i)];
                    e[size_t(i + 1)] = r = std::hypot(f, g);
                    if (r == 0.0) {
                        d[size_t(i + 1)] -= pp;
                        e[size_t(m)] = 0.0;
                        early = true;
                        break;
                    }
                    sn = f / r;
                    c = g / r;
                    g = d[size_t(i + 1)] - pp;
                    r = (d[size_t(i)] - g) * sn + 2.0 * c * b;
                    d[size_t(i + 1)] = g + (pp = sn * r);
                    g = c * r - b;
                    rc[size_t(nrot)] = c;
                    rs[size_t(nrot)] = sn;
                    ++nrot;
                }
                // rotations (i = m−1 … l) on columns (i, i+1) of Q, row chunks in parallel
                const int i_first = m - 1;
#pragma omp parallel for schedule(static) if (par && nrot > 16)
                for (int k0 = 0; k0 < n; k0 += 64) {
                    const int k1 = std::min(n, k0 + 64);
                    for (int t2 = 0; t2 < nrot; ++t2) {
                        const int ii = i_first - t2;
                        const double cc = rc[size_t(t2)], ss = rs[size_t(t2)];
                        double* c0 = &qt(0, ii);
                        double* c1 = &qt(0, ii + 1);
                        for (int k = k0; k < k1; ++k) {
                            const double f = c1[k];
                            c1[k] = ss * c0[k] + cc * f;
                            c0[k] = cc * c0[k] - ss * f;
                        }
                    }
                }
                if (early) continue;
                d[size_t(l)] -= pp;
                e[size_t(l)] = g;
                e[size_t(m)] = 0.0;
            }
        } while (m != l);
    }
    std::vector<int> order(N);
    for (int i = 0; i < n; ++i) order[size_t(i)] = i;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return d[size_t(x)] < d[size_t(y)]; });
    for (int j = 0; j < n; ++j) {
        w[j] = d[size_t(order[size_t(j)])];
        std::copy(&qt(0, order[size_t(j)]), &qt(0, order[size_t(j)]) + n, Z + size_t(j) * N);
    }
}

}  // namespace fkb
