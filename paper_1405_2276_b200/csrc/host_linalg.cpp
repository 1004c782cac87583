// host_linalg.cpp — host-side setup pieces of the product library.
//
//  * build_H: straight-ray travel-time operator (tomography.hpp:29-146).  The survey
//    keeps H construction on the host: it runs once, and the
//    exact floating-point order of the reference decides cells on grid lines.
//  * sym_eig_small: symmetric eigensolver for the ≤ 540×540 Gram/core matrices of
//    the randomized GHEP (lowrank.hpp:193 uses Eigen::SelfAdjointEigenSolver on the
//    host too).  Householder tridiagonalization + implicit-shift QL, eigenvalues
//    ascending with matching eigenvector columns.
//
// Compiled with -ffp-contract=off so trace_ray rounds exactly like the reference.

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
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
void sym_eig_small(int n, const double* A, double* w, double* Z) {
    std::vector<double> a(A, A + size_t(n) * n);  // working copy, becomes Q
    std::vector<double> d(static_cast<size_t>(n)), e(static_cast<size_t>(n));
    auto at = [&](int i, int j) -> double& { return a[size_t(i) + size_t(j) * n]; };
    // Householder reduction to tridiagonal form, accumulating the orthogonal transform.
    for (int i = n - 1; i > 0; --i) {
        const int l = i - 1;
        double h = 0.0, scale = 0.0;
        if (l > 0) {
            for (int k = 0; k <= l; ++k) scale += std::fabs(at(i, k));
            if (scale == 0.0) {
                e[size_t(i)] = at(i, l);
            } else {
                for (int k = 0; k <= l; ++k) {
                    at(i, k) /= scale;
                    h += at(i, k) * at(i, k);
                }
                double f = at(i, l);
                double g = f >= 0.0 ? -std::sqrt(h) : std::sqrt(h);
                e[size_t(i)] = scale * g;
                h -= f * g;
                at(i, l) = f - g;
                f = 0.0;
                for (int j = 0; j <= l; ++j) {
                    at(j, i) = at(i, j) / h;
                    g = 0.0;
                    for (int k = 0; k <= j; ++k) g += at(j, k) * at(i, k);
                    for (int k = j + 1; k <= l; ++k) g += at(k, j) * at(i, k);
                    e[size_t(j)] = g / h;
                    f += e[size_t(j)] * at(i, j);
                }
                const double hh = f / (h + h);
                for (int j = 0; j <= l; ++j) {
                    f = at(i, j);
                    e[size_t(j)] = g = e[size_t(j)] - hh * f;
                    for (int k = 0; k <= j; ++k) at(j, k) -= (f * e[size_t(k)] + g * at(i, k));
                }
            }
        } else {
            e[size_t(i)] = at(i, l);
        }
        d[size_t(i)] = h;
    }
    d[0] = 0.0;
    e[0] = 0.0;
    for (int i = 0; i < n; ++i) {
        const int l = i - 1;
        if (d[size_t(i)] != 0.0) {
            for (int j = 0; j <= l; ++j) {
                double g = 0.0;
                for (int k = 0; k <= l; ++k) g += at(i, k) * at(k, j);
                for (int k = 0; k <= l; ++k) at(k, j) -= g * at(k, i);
            }
        }
        d[size_t(i)] = at(i, i);
        at(i, i) = 1.0;
        for (int j = 0; j <= l; ++j) at(j, i) = at(i, j) = 0.0;
    }
    // Implicit-shift QL on the tridiagonal (d, e), rotating the columns of `a`.
    for (int i = 1; i < n; ++i) e[size_t(i - 1)] = e[size_t(i)];
    if (n > 0) e[size_t(n - 1)] = 0.0;
    for (int l = 0; l < n; ++l) {
        int iter = 0;
        int m;
        do {
            for (m = l; m < n - 1; ++m) {
                const double dd = std::fabs(d[size_t(m)]) + std::fabs(d[size_t(m + 1)]);
                if (std::fabs(e[size_t(m)]) <= 1e-300 + 2.220446049250313e-16 * dd) break;
            }
            if (m != l) {
                if (++iter > 60) throw std::runtime_error("sym_eig_small: QL iteration did not converge");
                double g = (d[size_t(l + 1)] - d[size_t(l)]) / (2.0 * e[size_t(l)]);
                double r = std::hypot(g, 1.0);
                g = d[size_t(m)] - d[size_t(l)] + e[size_t(l)] / (g + (g >= 0.0 ? std::fabs(r) : -std::fabs(r)));
                double s = 1.0, c = 1.0, p = 0.0;
                int i;
                for (i = m - 1; i >= l; --i) {
                    double f = s * e[size_t(i)];
                    const double b = c * e[size_t(i)];
                    e[size_t(i + 1)] = r = std::hypot(f, g);
                    if (r == 0.0) {
                        d[size_t(i + 1)] -= p;
                        e[size_t(m)] = 0.0;
                        break;
                    }
                    s = f / r;
                    c = g / r;
                    g = d[size_t(i + 1)] - p;
                    r = (d[size_t(i)] - g) * s + 2.0 * c * b;
                    d[size_t(i + 1)] = g + (p = s * r);
                    g = c * r - b;
                    for (int k = 0; k < n; ++k) {
                        f = at(k, i + 1);
                        at(k, i + 1) = s * at(k, i) + c * f;
                        at(k, i) = c * at(k, i) - s * f;
                    }
                }
                if (r == 0.0 && i >= l) continue;
                d[size_t(l)] -= p;
                e[size_t(l)] = g;
                e[size_t(m)] = 0.0;
            }
        } while (m != l);
    }
    std::vector<int> order(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) order[size_t(i)] = i;
    std::sort(order.begin(), order.end(), [&](int x, int y) { return d[size_t(x)] < d[size_t(y)]; });
    for (int j = 0; j < n; ++j) {
        w[j] = d[size_t(order[size_t(j)])];
        for (int i = 0; i < n; ++i) Z[size_t(i) + size_t(j) * n] = at(i, order[size_t(j)]);
    }
}

}  // namespace fkb
