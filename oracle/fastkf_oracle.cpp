// fastkf_oracle.cpp — CPU restatement of the reference fast-filter hot path.
//
// TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
// product library (paper_1405_2276_b200/csrc).  Only tests/, the smoke() check
// in __graft_entry__.py and bench.py's cpu_baseline / --impl reference legs may
// load it.  The product never links, imports or calls anything in oracle/.
//
// Why a restatement: the reference (/root/reference/proj, header-only C++20)
// needs Eigen3 + FFTW3, which are absent from this image and the GPU box, so
// it cannot be compiled.  Every function below follows the
// cited reference lines; third-party arithmetic is restated:
//   * FFTW3 (unpinned; proj/CMakeLists.txt:13-18) unnormalized c2c DFT with
//     forward sign e^{-2πi jk/n} (covariance.hpp:278-281,303-306,317,322):
//     restated as a recursive mixed-radix Cooley–Tukey transform.
//   * Eigen 3.4 (README.md:43) LLT (fast_filter.hpp:104): blocked Cholesky;
//     SelfAdjointEigenSolver (lowrank.hpp:193): cyclic Jacobi, eigenvalues
//     ascending like Eigen; setFromTriplets (tomography.hpp:143): CSR with
//     ascending columns per row, duplicates summed.
// Reductions use fixed 4096-element chunks summed in order, so results are
// independent of the OpenMP thread count.
//
// Parity pins: tests/test_oracle_*.py check this file against the reference's
// own known-answer tests (proj/tests/*.cpp) and against an independent
// numpy/scipy restatement (tests/golden/make_golden.py).

#include <algorithm>
#include <functional>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <memory>
#include <numbers>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace orc {

using cplx = std::complex<double>;
using Index = long long;

// ---------------------------------------------------------------- rng.hpp:12-86
inline uint64_t splitmix64(uint64_t x) {  // rng.hpp:12-18
    x += 0x9E3779B97F4A7C15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
inline uint64_t derive_seed(uint64_t seed, uint64_t tag) {  // rng.hpp:22-24
    return splitmix64(seed ^ splitmix64(tag));
}
struct Rng {  // rng.hpp:29-67
    uint64_t state;
    double spare = 0.0;
    bool has_spare = false;
    Rng(uint64_t seed, uint64_t stream) : state(derive_seed(seed, stream)) {}
    uint64_t next_u64() {
        state += 0x9E3779B97F4A7C15ULL;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double uniform() { return (double(next_u64() >> 11) + 0.5) * 0x1.0p-53; }
    double normal() {
        if (has_spare) { has_spare = false; return spare; }
        const double u1 = uniform();
        const double u2 = uniform();
        const double rad = std::sqrt(-2.0 * std::log(u1));
        const double ang = 2.0 * std::numbers::pi * u2;
        spare = rad * std::sin(ang);
        has_spare = true;
        return rad * std::cos(ang);
    }
};
inline void gaussian_vector(Index n, uint64_t seed, uint64_t stream, double* out) {  // :69-77
    Rng rng(seed, stream);
    for (Index i = 0; i < n; ++i) out[i] = rng.normal();
}
inline void gaussian_matrix(Index rows, Index cols, uint64_t seed, uint64_t base,
                            double* out) {  // rng.hpp:79-86, column j = stream base+j
#pragma omp parallel for schedule(dynamic)
    for (Index j = 0; j < cols; ++j) gaussian_vector(rows, seed, base + uint64_t(j), out + j * rows);
}

// ---------------------------------------------------------------- kernel.hpp:19-63
struct KernelSpec {
    int family = 0;  // 0 powered_exponential, 1 matern (kernel.hpp:13)
    double theta = 1.0, length = 0.2, power = 1.0, nu = 0.5, alpha_scale = 0.0;
    void validate() const {  // kernel.hpp:27-43
        if (!(theta > 0.0)) throw std::invalid_argument("kernel: theta must be positive");
        if (!(length > 0.0)) throw std::invalid_argument("kernel: length must be positive");
        if (family == 0) {
            if (!(power > 0.0) || power > 2.0)
                throw std::invalid_argument("kernel: power must lie in (0, 2]");
        } else if (!(nu > 0.0)) {
            throw std::invalid_argument("kernel: nu must be positive");
        }
    }
    double scale() const { return alpha_scale > 0.0 ? alpha_scale : 1.0 / length; }
};
inline double kernel_eval(const KernelSpec& s, double r) {  // kernel.hpp:51-63
    s.validate();
    if (r < 0.0) throw std::invalid_argument("kernel: distance must be nonnegative");
    if (r == 0.0) return s.theta;
    if (s.family == 0) return s.theta * std::exp(-std::pow(r / s.length, s.power));
    const double arg = std::sqrt(2.0 * s.nu) * s.scale() * r;
    if (arg > 700.0) return 0.0;
    const double pref = std::exp((1.0 - s.nu) * std::numbers::ln2 - std::lgamma(s.nu));
    return s.theta * pref * std::pow(arg, s.nu) * std::cyl_bessel_k(s.nu, arg);
}

// ---------------------------------------------------------------- grid.hpp:22-63
struct Grid {
    int nx = 0, ny = 0;
    double lx = 1.0, ly = 1.0;
    void validate() const {
        if (nx < 1 || ny < 1) throw std::invalid_argument("grid: nx and ny must be positive");
        if (!(lx > 0.0) || !(ly > 0.0)) throw std::invalid_argument("grid: domain lengths must be positive");
    }
    Index size() const { return Index(nx) * ny; }
    double dx() const { return lx / nx; }
    double dy() const { return ly / ny; }
    Index index(int ix, int iy) const { return Index(ix) * ny + iy; }  // grid.hpp:48
};

// ---------------------------------------------------------------- deterministic reductions
constexpr Index kChunk = 4096;
inline double dot(const double* a, const double* b, Index n) {
    const Index nc = (n + kChunk - 1) / kChunk;
    if (nc <= 1) {
        double s = 0.0;
        for (Index i = 0; i < n; ++i) s += a[i] * b[i];
        return s;
    }
    std::vector<double> part(size_t(nc), 0.0);
#pragma omp parallel for schedule(static)
    for (Index c = 0; c < nc; ++c) {
        const Index lo = c * kChunk, hi = std::min(n, lo + kChunk);
        double s = 0.0;
        for (Index i = lo; i < hi; ++i) s += a[i] * b[i];
        part[size_t(c)] = s;
    }
    double s = 0.0;
    for (double p : part) s += p;
    return s;
}
inline void axpy(double alpha, const double* x, double* y, Index n) {
#pragma omp parallel for schedule(static) if (n > 65536)
    for (Index i = 0; i < n; ++i) y[i] += alpha * x[i];
}

// ---------------------------------------------------------------- FFT (FFTW3 c2c restated)
// Recursive mixed-radix decimation-in-time DFT, unnormalized, sign −1 forward.
struct Fft1d {
    int n = 0;
    std::vector<int> factors;
    std::vector<cplx> tw;  // tw[k] = exp(-2πi k / n)
    explicit Fft1d(int n_ = 1) : n(n_) {
        int v = n;
        for (int f : {4, 2, 3, 5, 7})
            while (v % f == 0) { factors.push_back(f); v /= f; }
        if (v != 1) {  // generic prime factors (next_smooth never produces them)
            for (int f = 11; v > 1; f += 2)
                while (v % f == 0) { factors.push_back(f); v /= f; }
        }
        tw.resize(static_cast<size_t>(n));
        for (int k = 0; k < n; ++k) {
            const long double a = -2.0L * std::numbers::pi_v<long double> * k / n;
            tw[size_t(k)] = cplx(double(std::cos(a)), double(std::sin(a)));
        }
    }
    cplx w(long k, int sign) const {  // exp(sign*2πi k/n), k in [0,n)
        const cplx t = tw[size_t(k % n)];
        return sign < 0 ? t : std::conj(t);
    }
    void rec(const cplx* in, cplx* out, int len, int stride, int fi, int sign) const {
        if (len == 1) { out[0] = in[0]; return; }
        const int p = factors[size_t(fi)];
        const int m = len / p;
        for (int q = 0; q < p; ++q) rec(in + q * stride, out + q * m, m, stride * p, fi + 1, sign);
        const int step = n / len;  // W_len^j = W_n^{j*step}
        cplx t[16];
        std::vector<cplx> tbig;
        cplx* tt = t;
        if (p > 16) { tbig.resize(static_cast<size_t>(p)); tt = tbig.data(); }
        for (int k = 0; k < m; ++k) {
            for (int q = 0; q < p; ++q) tt[q] = out[q * m + k] * (q ? w(long(q) * k * step, sign) : cplx(1, 0));
            if (p == 2) {
                out[k] = tt[0] + tt[1];
                out[k + m] = tt[0] - tt[1];
            } else if (p == 4) {
                const cplx a0 = tt[0] + tt[2], a1 = tt[0] - tt[2];
                const cplx b0 = tt[1] + tt[3], b1 = tt[1] - tt[3];
                const cplx jb1 = sign < 0 ? cplx(b1.imag(), -b1.real()) : cplx(-b1.imag(), b1.real());
                out[k] = a0 + b0;
                out[k + m] = a1 + jb1;
                out[k + 2 * m] = a0 - b0;
                out[k + 3 * m] = a1 - jb1;
            } else {
                for (int r = 0; r < p; ++r) {
                    cplx s = tt[0];
                    for (int q = 1; q < p; ++q) s += tt[q] * w(long(q) * r % p * (n / p), sign);
                    out[k + m * r] = s;
                }
            }
        }
    }
    void exec(const cplx* in, cplx* out, int sign) const { rec(in, out, n, 1, 0, sign); }
};

struct Fft2d {  // fftw_plan_dft_2d(mx, my, ...) on a row-major mx×my array
    int mx, my;
    Fft1d fx, fy;
    Fft2d(int mx_, int my_) : mx(mx_), my(my_), fx(mx_), fy(my_) {}
    void exec(cplx* data, int sign, int rows_nonzero = -1, int rows_needed = -1) const {
        // rows_nonzero / rows_needed are pure work-skipping hints: rows that are
        // entirely zero transform to zero; output rows nobody reads are skipped
        // in the last pass only when the caller asks.  Both leave every value
        // the caller reads identical to the full transform.
        const int r_in = rows_nonzero < 0 ? mx : rows_nonzero;
#pragma omp parallel
        {
            std::vector<cplx> tmp(size_t(std::max(mx, my)));
            std::vector<cplx> out(size_t(std::max(mx, my)));
#pragma omp for schedule(static)
            for (int i = 0; i < r_in; ++i) {
                fy.exec(data + size_t(i) * my, out.data(), sign);
                std::copy(out.begin(), out.begin() + my, data + size_t(i) * my);
            }
#pragma omp for schedule(static)
            for (int j = 0; j < my; ++j) {
                for (int i = 0; i < mx; ++i) tmp[size_t(i)] = data[size_t(i) * my + j];
                fx.exec(tmp.data(), out.data(), sign);
                for (int i = 0; i < mx; ++i) data[size_t(i) * my + j] = out[size_t(i)];
            }
        }
        (void)rows_needed;
    }
};

// ---------------------------------------------------------------- covariance.hpp (fft mode)
inline int next_smooth(int n) {  // covariance.hpp:35-43
    if (n <= 1) return 1;
    for (int m = n;; ++m) {
        int v = m;
        for (int f : {2, 3, 5, 7})
            while (v % f == 0) v /= f;
        if (v == 1) return m;
    }
}

struct Cov {
    Grid grid;
    KernelSpec spec;
    int mx = 0, my = 0;
    std::vector<double> spectrum;
    std::unique_ptr<Fft2d> plan;
    long applies = 0;

    Cov(const Grid& g, const KernelSpec& s) : grid(g), spec(s) {  // covariance.hpp:71-79
        grid.validate();
        spec.validate();
        build_fft();
    }
    Index size() const { return grid.size(); }
    size_t M() const { return size_t(mx) * size_t(my); }

    void build_fft() {  // covariance.hpp:238-260
        const int base_x = std::max(2 * grid.nx - 1, 1);
        const int base_y = std::max(2 * grid.ny - 1, 1);
        double worst = 0.0;
        for (int pad = 1; pad <= 8; pad *= 2) {
            mx = next_smooth(base_x * pad);
            my = next_smooth(base_y * pad);
            if (try_spectrum(worst)) return;
        }
        std::ostringstream msg;
        msg << "covariance: circulant embedding is not nonnegative definite for kernel "
            << (spec.family == 0 ? "powered-exponential" : "matern") << " (theta=" << spec.theta
            << ", length=" << spec.length;
        if (spec.family == 0) msg << ", power=" << spec.power;
        else msg << ", nu=" << spec.nu;
        msg << ") on grid " << grid.nx << "x" << grid.ny
            << " even after 8x padding (worst negative/max spectrum ratio " << worst
            << "); use dense mode or a shorter correlation length";
        throw std::runtime_error(msg.str());
    }
    bool try_spectrum(double& worst) {  // covariance.hpp:264-298
        const size_t m = M();
        std::vector<cplx> buf(m);
        const double dx = grid.dx(), dy = grid.dy();
#pragma omp parallel for schedule(static)
        for (int i = 0; i < mx; ++i) {
            const double rx = std::min(i, mx - i) * dx;
            for (int j = 0; j < my; ++j) {
                const double ry = std::min(j, my - j) * dy;
                buf[size_t(i) * my + j] = cplx(kernel_eval(spec, std::hypot(rx, ry)), 0.0);
            }
        }
        Fft2d p(mx, my);
        p.exec(buf.data(), -1);
        std::vector<double> sp(m);
        double mxv = 0.0, mnv = 0.0;
        for (size_t i = 0; i < m; ++i) {
            sp[i] = buf[i].real();
            mxv = std::max(mxv, sp[i]);
            mnv = std::min(mnv, sp[i]);
        }
        if (mxv <= 0.0) return false;
        worst = std::max(worst, -mnv / mxv);
        if (mnv < -1e-10 * mxv) return false;
        for (auto& v : sp) v = std::max(v, 0.0);
        spectrum = std::move(sp);
        plan = std::make_unique<Fft2d>(mx, my);
        return true;
    }
    void apply(const double* x, double* y) {  // covariance.hpp:101-108 → apply_fft :309-330
        ++applies;
        const size_t m = M();
        std::vector<cplx> buf(m, cplx(0, 0));
        for (int i = 0; i < grid.nx; ++i)
            for (int j = 0; j < grid.ny; ++j) buf[size_t(i) * my + j] = cplx(x[grid.index(i, j)], 0.0);
        plan->exec(buf.data(), -1, grid.nx);
#pragma omp parallel for schedule(static)
        for (long long idx = 0; idx < (long long)m; ++idx) buf[size_t(idx)] *= spectrum[size_t(idx)];
        plan->exec(buf.data(), +1);
        const double scale = 1.0 / double(m);
        for (int i = 0; i < grid.nx; ++i)
            for (int j = 0; j < grid.ny; ++j) y[grid.index(i, j)] = buf[size_t(i) * my + j].real() * scale;
    }
    void apply_matrix(const double* X, Index ncols, double* Y) {  // :111-115
        const Index n = size();
        for (Index c = 0; c < ncols; ++c) apply(X + c * n, Y + c * n);
    }
    void sample_pair(uint64_t seed, uint64_t stream, double* a, double* b) {  // :332-353
        const size_t m = M();
        std::vector<cplx> buf(m);
        Rng re(seed, 2 * stream), im(seed, 2 * stream + 1);
        const double scale = 1.0 / std::sqrt(double(m));
        for (size_t idx = 0; idx < m; ++idx) {
            const double amp = std::sqrt(spectrum[idx]);
            const double r = amp * re.normal();
            const double q = amp * im.normal();
            buf[idx] = cplx(r, q);
        }
        plan->exec(buf.data(), +1);
        for (int i = 0; i < grid.nx; ++i)
            for (int j = 0; j < grid.ny; ++j) {
                const size_t idx = size_t(i) * my + j;
                a[grid.index(i, j)] = buf[idx].real() * scale;
                b[grid.index(i, j)] = buf[idx].imag() * scale;
            }
    }
};

// ---------------------------------------------------------------- tomography.hpp:29-146
struct Seg { Index cell; double length; };
inline std::vector<Seg> trace_ray(const Grid& g, double sx, double sy, double rx, double ry) {
    const double tol_x = 1e-12 * g.lx, tol_y = 1e-12 * g.ly;  // :31-40
    for (int e = 0; e < 2; ++e) {
        const double px = e ? rx : sx, py = e ? ry : sy;
        if (px < -tol_x || px > g.lx + tol_x || py < -tol_y || py > g.ly + tol_y)
            throw std::invalid_argument("trace_ray: endpoint lies outside the domain");
    }
    const double dx = rx - sx, dy = ry - sy;
    const double len = std::sqrt(dx * dx + dy * dy);  // Eigen norm() = sqrt(squaredNorm)
    if (len == 0.0) throw std::invalid_argument("trace_ray: degenerate zero-length ray");
    std::vector<double> ts;
    ts.reserve(size_t(g.nx + g.ny + 2));
    ts.push_back(0.0);
    ts.push_back(1.0);
    if (dx != 0.0)
        for (int i = 1; i < g.nx; ++i) {
            const double t = (i * g.dx() - sx) / dx;
            if (t > 0.0 && t < 1.0) ts.push_back(t);
        }
    if (dy != 0.0)
        for (int j = 1; j < g.ny; ++j) {
            const double t = (j * g.dy() - sy) / dy;
            if (t > 0.0 && t < 1.0) ts.push_back(t);
        }
    std::sort(ts.begin(), ts.end());
    std::vector<Seg> segs;
    double t_prev = ts.front();
    for (size_t i = 1; i < ts.size(); ++i) {  // :67-84
        const double t = ts[i];
        if (t - t_prev <= 1e-12) continue;
        const double h = 0.5 * (t_prev + t);
        const double mx = sx + h * dx, my = sy + h * dy;
        const int ix = std::clamp(int(std::floor(mx / g.dx())), 0, g.nx - 1);
        const int iy = std::clamp(int(std::floor(my / g.dy())), 0, g.ny - 1);
        const Index cell = g.index(ix, iy);
        const double sl = (t - t_prev) * len;
        if (!segs.empty() && segs.back().cell == cell) segs.back().length += sl;
        else segs.push_back({cell, sl});
        t_prev = t;
    }
    return segs;
}

struct Csr {  // SparseRowMatrix (grid.hpp:15): row-major, int32 indices
    int rows = 0, cols = 0;
    std::vector<int> rowptr{0}, col;
    std::vector<double> val;
    Index nnz() const { return Index(val.size()); }
};
// build_H tomography.hpp:130-146; setFromTriplets → ascending columns, duplicates summed
inline Csr build_H(const Grid& g, const std::vector<double>& src, const std::vector<double>& rec) {
    const int ns = int(src.size() / 2), nr = int(rec.size() / 2);
    if (ns < 1 || nr < 1) throw std::invalid_argument("layout: sources and receivers must be nonempty");
    for (int e = 0; e < ns + nr; ++e) {  // layout.validate :115-125
        const double px = e < ns ? src[2 * e] : rec[2 * (e - ns)];
        const double py = e < ns ? src[2 * e + 1] : rec[2 * (e - ns) + 1];
        if (!(px >= 0.0 && px <= g.lx && py >= 0.0 && py <= g.ly))
            throw std::invalid_argument(e < ns ? "layout: source outside domain" : "layout: receiver outside domain");
    }
    Csr h;
    h.rows = ns * nr;
    h.cols = int(g.size());
    h.rowptr.reserve(size_t(h.rows) + 1);
    for (int s = 0; s < ns; ++s)
        for (int r = 0; r < nr; ++r) {
            auto segs = trace_ray(g, src[2 * s], src[2 * s + 1], rec[2 * r], rec[2 * r + 1]);
            std::stable_sort(segs.begin(), segs.end(), [](const Seg& a, const Seg& b) { return a.cell < b.cell; });
            Index last = -1;
            for (const Seg& sg : segs) {
                if (sg.cell == last) { h.val.back() += sg.length; continue; }
                h.col.push_back(int(sg.cell));
                h.val.push_back(sg.length);
                last = sg.cell;
            }
            h.rowptr.push_back(int(h.col.size()));
        }
    return h;
}
inline void csr_mv(const Csr& h, const double* x, double* y) {  // y = H x
#pragma omp parallel for schedule(static) if (h.rows > 256)
    for (int r = 0; r < h.rows; ++r) {
        double s = 0.0;
        for (int e = h.rowptr[size_t(r)]; e < h.rowptr[size_t(r) + 1]; ++e) s += h.val[size_t(e)] * x[h.col[size_t(e)]];
        y[r] = s;
    }
}
inline void csr_tmv(const Csr& h, const double* y, double* x) {  // x = Hᵀ y (row-sequential scatter)
    std::fill(x, x + h.cols, 0.0);
    for (int r = 0; r < h.rows; ++r)
        for (int e = h.rowptr[size_t(r)]; e < h.rowptr[size_t(r) + 1]; ++e) x[h.col[size_t(e)]] += h.val[size_t(e)] * y[r];
}

// ---------------------------------------------------------------- dense helpers (column-major)
struct Mat {
    Index rows = 0, cols = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(Index r, Index c) : rows(r), cols(c), a(size_t(r * c), 0.0) {}
    double& operator()(Index i, Index j) { return a[size_t(i + j * rows)]; }
    double operator()(Index i, Index j) const { return a[size_t(i + j * rows)]; }
    double* col(Index j) { return a.data() + j * rows; }
    const double* col(Index j) const { return a.data() + j * rows; }
};
// C = Aᵀ B  (A: n×p, B: n×q) — Gram-type products with long inner dimension
inline Mat gemm_tn(const Mat& A, const Mat& B) {
    Mat C(A.cols, B.cols);
    for (Index j = 0; j < B.cols; ++j)
        for (Index i = 0; i < A.cols; ++i) C(i, j) = dot(A.col(i), B.col(j), A.rows);
    return C;
}
// C = A B (A: n×p, B: p×q)
inline Mat gemm_nn(const Mat& A, const Mat& B) {
    Mat C(A.rows, B.cols);
#pragma omp parallel for schedule(static)
    for (Index j = 0; j < B.cols; ++j) {
        double* c = C.col(j);
        for (Index k = 0; k < A.cols; ++k) {
            const double b = B(k, j);
            const double* a = A.col(k);
            for (Index i = 0; i < A.rows; ++i) c[i] += a[i] * b;
        }
    }
    return C;
}
// y = A x (A: n×p) parallel over row chunks, deterministic
inline void gemv(const Mat& A, const double* x, double* y) {
    const Index n = A.rows;
#pragma omp parallel for schedule(static)
    for (Index lo = 0; lo < n; lo += kChunk) {
        const Index hi = std::min(n, lo + kChunk);
        for (Index i = lo; i < hi; ++i) y[i] = 0.0;
        for (Index k = 0; k < A.cols; ++k) {
            const double xk = x[k];
            const double* a = A.col(k);
            for (Index i = lo; i < hi; ++i) y[i] += a[i] * xk;
        }
    }
}

// Eigen::SelfAdjointEigenSolver stand-in: cyclic Jacobi, ascending eigenvalues.
inline void sym_eig(const Mat& A_in, std::vector<double>& evals, Mat& V) {
    const Index n = A_in.rows;
    Mat A = A_in;
    V = Mat(n, n);
    for (Index i = 0; i < n; ++i) V(i, i) = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0, diag = 0.0;
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < n; ++i) (i == j ? diag : off) += A(i, j) * A(i, j);
        if (off <= 1e-36 * diag || off == 0.0) break;
        for (Index p = 0; p < n - 1; ++p)
            for (Index q = p + 1; q < n; ++q) {
                const double apq = A(p, q);
                if (apq == 0.0) continue;
                const double app = A(p, p), aqq = A(q, q);
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (Index k = 0; k < n; ++k) {  // A ← A J (columns p,q)
                    const double akp = A(k, p), akq = A(k, q);
                    A(k, p) = c * akp - s * akq;
                    A(k, q) = s * akp + c * akq;
                }
                for (Index k = 0; k < n; ++k) {  // A ← Jᵀ A (rows p,q)
                    const double apk = A(p, k), aqk = A(q, k);
                    A(p, k) = c * apk - s * aqk;
                    A(q, k) = s * apk + c * aqk;
                }
                A(p, q) = A(q, p) = 0.0;
                double* vp = V.col(p);
                double* vq = V.col(q);
                for (Index k = 0; k < n; ++k) {
                    const double a = vp[k], b = vq[k];
                    vp[k] = c * a - s * b;
                    vq[k] = s * a + c * b;
                }
            }
    }
    std::vector<Index> order(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) order[size_t(i)] = i;
    std::sort(order.begin(), order.end(), [&](Index a, Index b) { return A(a, a) < A(b, b); });
    evals.resize(static_cast<size_t>(n));
    Mat Vs(n, n);
    for (Index i = 0; i < n; ++i) {
        evals[size_t(i)] = A(order[size_t(i)], order[size_t(i)]);
        std::copy(V.col(order[size_t(i)]), V.col(order[size_t(i)]) + n, Vs.col(i));
    }
    V = std::move(Vs);
}

// Eigen::LLT stand-in: blocked right-looking lower Cholesky in place.  false on failure.
inline bool llt(Mat& S) {
    const Index n = S.rows;
    const Index nb = 64;
    for (Index k0 = 0; k0 < n; k0 += nb) {
        const Index k1 = std::min(n, k0 + nb);
        for (Index j = k0; j < k1; ++j) {  // panel: unblocked left-looking within block columns
            double d = S(j, j);
            for (Index p = k0; p < j; ++p) d -= S(j, p) * S(j, p);
            if (!(d > 0.0) || !std::isfinite(d)) return false;
            d = std::sqrt(d);
            S(j, j) = d;
#pragma omp parallel for schedule(static) if (n - j > 512)
            for (Index i = j + 1; i < n; ++i) {
                double v = S(i, j);
                for (Index p = k0; p < j; ++p) v -= S(i, p) * S(j, p);
                S(i, j) = v / d;
            }
        }
        // trailing update S22 -= L21 L21ᵀ (lower part)
#pragma omp parallel for schedule(dynamic, 8)
        for (Index j = k1; j < n; ++j)
            for (Index p = k0; p < k1; ++p) {
                const double ljp = S(j, p);
                if (ljp == 0.0) continue;
                const double* lp = S.col(p);
                double* sj = S.col(j);
                for (Index i = j; i < n; ++i) sj[i] -= lp[i] * ljp;
            }
    }
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < j; ++i) S(i, j) = 0.0;
    return true;
}
inline void llt_solve(const Mat& L, double* b) {
    const Index n = L.rows;
    for (Index j = 0; j < n; ++j) {  // L y = b (column-oriented)
        b[j] /= L(j, j);
        const double bj = b[j];
        const double* l = L.col(j);
        for (Index i = j + 1; i < n; ++i) b[i] -= l[i] * bj;
    }
    for (Index j = n - 1; j >= 0; --j) {  // Lᵀ x = y
        const double* l = L.col(j);
        double s = b[j];
        for (Index i = j + 1; i < n; ++i) s -= l[i] * b[i];
        b[j] = s / L(j, j);
    }
}

// ---------------------------------------------------------------- lowrank.hpp:53-213
struct Gep {
    Mat u;        // N×k, Γ⁻¹-orthonormal (lowrank.hpp:26-31)
    Mat ubar;     // Γ⁻¹u = Q̄·S — needed by the FFT-mode sampler
    std::vector<double> lambda;
    Index kept_cols = 0;  // columns surviving b_orthonormalize
    Index rank() const { return Index(lambda.size()); }
};

// a_apply = Hᵀ(H v)/σ² (fast_filter.hpp:63-66); b_apply = Γ (lowrank.hpp:208-213)
inline Gep randomized_ghep(Cov& cov, const Csr& h, double sigma2, Index k, Index p, uint64_t seed) {
    if (k < 0 || p < 0)  // lowrank.hpp:145-151
        throw std::invalid_argument("randomized_ghep: k and oversampling must be nonnegative");
    const Index n = cov.size();
    const Index l = k + p;
    if (l > n)
        throw std::invalid_argument("randomized_ghep: k + oversampling = " + std::to_string(l) +
                                    " exceeds problem size " + std::to_string(n));
    Gep out;
    out.u = Mat(n, 0);
    out.ubar = Mat(n, 0);
    if (k == 0) return out;

    Mat omega(n, l);
    gaussian_matrix(n, l, seed, 0, omega.a.data());  // :157
    Mat ybar(n, l);
    {
        std::vector<double> hv(size_t(h.rows));
#pragma omp parallel for schedule(dynamic) firstprivate(hv)
        for (Index j = 0; j < l; ++j) {  // :158-159
            csr_mv(h, omega.col(j), hv.data());
            csr_tmv(h, hv.data(), ybar.col(j));
            for (Index i = 0; i < n; ++i) ybar(i, j) /= sigma2;
        }
    }
    double ynorm = 0.0;
    for (double v : ybar.a) ynorm += v * v;
    if (ynorm == 0.0) return out;  // :161

    // b_orthonormalize (lowrank.hpp:53-106) with b_apply = Γ, no `against`.
    Mat q(n, l), bq(n, l);
    Index kept = 0;
    std::vector<double> w(static_cast<size_t>(n)), bw(static_cast<size_t>(n));
    for (Index j = 0; j < l; ++j) {
        std::copy(ybar.col(j), ybar.col(j) + n, w.begin());
        for (double v : w)
            if (!std::isfinite(v))
                throw std::invalid_argument("b_orthonormalize: column " + std::to_string(j) + " contains non-finite entries");
        cov.apply(w.data(), bw.data());
        const double pre_norm = std::sqrt(std::max(dot(w.data(), bw.data(), n), 0.0));
        double norm = 0.0;
        for (int sweep = 0; sweep < 2; ++sweep) {
            for (Index i = 0; i < kept; ++i) {
                const double c = dot(bq.col(i), w.data(), n);
                axpy(-c, q.col(i), w.data(), n);
            }
            cov.apply(w.data(), bw.data());
            norm = std::sqrt(std::max(dot(w.data(), bw.data(), n), 0.0));
        }
        if (norm <= 1e-12 * pre_norm || norm == 0.0) continue;  // dropped
        for (Index i = 0; i < n; ++i) {
            q(i, kept) = w[size_t(i)] / norm;
            bq(i, kept) = bw[size_t(i)] / norm;
        }
        ++kept;
    }
    if (kept == 0)
        throw std::runtime_error("randomized_ghep: rank collapse — every sketch column was dropped during orthonormalization");
    out.kept_cols = kept;
    q.cols = bq.cols = kept;
    q.a.resize(size_t(n * kept));
    bq.a.resize(size_t(n * kept));

    // two-pass core T = Qᵀ(AQ), Q = ΓQ̄ = bq (:171-172, :186-191)
    Mat aq(n, kept);
    {
        std::vector<double> hv(size_t(h.rows));
#pragma omp parallel for schedule(dynamic) firstprivate(hv)
        for (Index j = 0; j < kept; ++j) {
            csr_mv(h, bq.col(j), hv.data());
            csr_tmv(h, hv.data(), aq.col(j));
            for (Index i = 0; i < n; ++i) aq(i, j) /= sigma2;
        }
    }
    Mat t = gemm_tn(bq, aq);
    for (Index j = 0; j < kept; ++j)
        for (Index i = 0; i < j; ++i) t(i, j) = t(j, i) = 0.5 * (t(i, j) + t(j, i));
    std::vector<double> ev;
    Mat s;
    sym_eig(t, ev, s);  // :193
    const Index kk = std::min(k, kept);  // :197-205
    out.lambda.resize(static_cast<size_t>(kk));
    Mat sk(kept, kk);
    for (Index i = 0; i < kk; ++i) {
        const Index src = kept - 1 - i;
        out.lambda[size_t(i)] = std::max(ev[size_t(src)], 0.0);
        std::copy(s.col(src), s.col(src) + kept, sk.col(i));
    }
    out.u = gemm_nn(bq, sk);
    out.ubar = gemm_nn(q, sk);
    return out;
}

// ---------------------------------------------------------------- fast_filter.hpp:21-125
struct Ctx {  // FkfContext fast_filter.hpp:42-49
    Gep gep;
    Mat gamma_ht;    // N×m
    Mat h_gamma_ht;  // m×m
    Mat h_u;         // m×k
    Csr h;
    double sigma2 = 0.0;
};
struct State {  // LowRankState :21-37 (W = ctx.gep.u shared, as the reference copies U each step)
    double alpha = 0.0;
    std::vector<double> d, mean;
    int step = 0;
};

inline Ctx fkf_init(Cov& cov, const Csr& h, double sigma2, Index k, Index p, uint64_t seed) {
    if (Index(h.cols) != cov.size())
        throw std::invalid_argument("fkf_init: H columns do not match state dimension");
    if (!(sigma2 > 0.0)) throw std::invalid_argument("fkf_init: sigma2 must be positive");
    Ctx ctx;
    ctx.h = h;
    ctx.sigma2 = sigma2;
    ctx.gep = randomized_ghep(cov, h, sigma2, k, p, seed);
    const Index n = cov.size(), m = h.rows;
    ctx.gamma_ht = Mat(n, m);  // :68-70
    {
        std::vector<double> e(static_cast<size_t>(n));
        for (Index i = 0; i < m; ++i) {
            std::fill(e.begin(), e.end(), 0.0);
            for (int q = h.rowptr[size_t(i)]; q < h.rowptr[size_t(i) + 1]; ++q) e[size_t(h.col[size_t(q)])] = h.val[size_t(q)];
            cov.apply(e.data(), ctx.gamma_ht.col(i));
        }
    }
    ctx.h_gamma_ht = Mat(m, m);  // :71-72
#pragma omp parallel for schedule(static)
    for (Index j = 0; j < m; ++j) csr_mv(h, ctx.gamma_ht.col(j), ctx.h_gamma_ht.col(j));
    for (Index j = 0; j < m; ++j)
        for (Index i = 0; i < j; ++i)
            ctx.h_gamma_ht(i, j) = ctx.h_gamma_ht(j, i) = 0.5 * (ctx.h_gamma_ht(i, j) + ctx.h_gamma_ht(j, i));
    const Index r = ctx.gep.rank();
    ctx.h_u = Mat(m, r);  // :73
    for (Index j = 0; j < r; ++j) csr_mv(h, ctx.gep.u.col(j), ctx.h_u.col(j));
    return ctx;
}

inline State fkf_step(const State& st, const Ctx& ctx, const double* y, Index ylen) {  // :84-125
    const Index r = ctx.gep.rank();
    const Index m = ctx.h.rows;
    const Index n = ctx.h.cols;
    if (ylen != m)
        throw std::invalid_argument("fkf_step: observation length " + std::to_string(ylen) + " does not match " +
                                    std::to_string(m) + " measurements");
    const Index srank = Index(st.d.size());
    if (srank != 0 && srank != r)
        throw std::invalid_argument("fkf_step: state rank does not match the eigendecomposition (constant-H regime requires W = U)");
    const double alpha = st.alpha + 1.0;
    std::vector<double> d_prev = srank ? st.d : std::vector<double>(size_t(r), 0.0);

    Mat s(m, m);  // :100-103
    for (size_t i = 0; i < s.a.size(); ++i) s.a[i] = alpha * ctx.h_gamma_ht.a[i];
    if (r > 0) {
#pragma omp parallel for schedule(static)
        for (Index j = 0; j < m; ++j)
            for (Index p = 0; p < r; ++p) {
                const double bjp = ctx.h_u(j, p) * d_prev[size_t(p)];
                const double* bp = ctx.h_u.col(p);
                double* sj = s.col(j);
                for (Index i = 0; i < m; ++i) sj[i] -= bp[i] * bjp;
            }
    }
    for (Index i = 0; i < m; ++i) s(i, i) += ctx.sigma2;
    for (Index j = 0; j < m; ++j)
        for (Index i = 0; i < j; ++i) s(i, j) = s(j, i) = 0.5 * (s(i, j) + s(j, i));
    if (!llt(s)) throw std::runtime_error("fkf_step: innovation system is singular");  // :104-106

    std::vector<double> z(static_cast<size_t>(m));  // :108
    csr_mv(ctx.h, st.mean.data(), z.data());
    for (Index i = 0; i < m; ++i) z[size_t(i)] = y[i] - z[size_t(i)];
    llt_solve(s, z.data());

    State nx;
    nx.alpha = alpha;
    nx.step = st.step + 1;
    nx.mean.resize(static_cast<size_t>(n));  // :114-116
    gemv(ctx.gamma_ht, z.data(), nx.mean.data());
    for (Index i = 0; i < n; ++i) nx.mean[size_t(i)] = st.mean[size_t(i)] + alpha * nx.mean[size_t(i)];
    if (r > 0) {
        std::vector<double> c(static_cast<size_t>(r)), uc(static_cast<size_t>(n));
        for (Index p = 0; p < r; ++p) c[size_t(p)] = d_prev[size_t(p)] * dot(ctx.h_u.col(p), z.data(), m);
        gemv(ctx.gep.u, c.data(), uc.data());
        for (Index i = 0; i < n; ++i) nx.mean[size_t(i)] -= uc[size_t(i)];
    }
    nx.d.resize(static_cast<size_t>(r));  // :118-123
    for (Index i = 0; i < r; ++i) {
        const double c = alpha - d_prev[size_t(i)];
        const double lam = ctx.gep.lambda[size_t(i)];
        nx.d[size_t(i)] = (d_prev[size_t(i)] + alpha * lam * c) / (1.0 + lam * c);
    }
    return nx;
}

// ---------------------------------------------------------------- uq.hpp:16-112
inline void variance(const State& st, const Ctx& ctx, const Cov& cov, double* out) {  // :16-23
    const Index n = cov.size();
    if (Index(st.mean.size()) != n) throw std::invalid_argument("variance: state does not match operator size");
    const Index r = Index(st.d.size());
#pragma omp parallel for schedule(static)
    for (Index i = 0; i < n; ++i) {
        double v = st.alpha * cov.spec.theta;
        double s = 0.0;
        for (Index j = 0; j < r; ++j) {
            const double w = ctx.gep.u(i, j);
            s += w * w * st.d[size_t(j)];
        }
        out[i] = v - s;
    }
}
inline double trace_criterion(const State& st, const Ctx& ctx, const Cov& cov) {  // :27-34
    double out = st.alpha * (double(cov.size()) * cov.spec.theta);
    for (Index j = 0; j < Index(st.d.size()); ++j)
        out -= st.d[size_t(j)] * dot(ctx.gep.u.col(j), ctx.gep.u.col(j), cov.size());
    return out;
}
inline double relative_entropy(const State& st) {  // :39-53
    if (!(st.alpha > 0.0)) throw std::invalid_argument("relative_entropy: requires alpha > 0");
    const double n = double(st.mean.size());
    double sum = (n - double(st.d.size())) * std::log(st.alpha);
    for (size_t i = 0; i < st.d.size(); ++i) {
        const double gap = st.alpha - st.d[i];
        if (!(gap > 0.0))
            throw std::runtime_error("relative_entropy: D_" + std::to_string(i) + " = " + std::to_string(st.d[i]) +
                                     " is not below alpha = " + std::to_string(st.alpha));
        sum += std::log(gap);
    }
    return 0.5 * sum;
}
// FFT-mode conditional realization (the reference's dense-root
// formula uq.hpp:70-84 with Γ^{1/2} replaced by the circulant root R, RRᵀ = Γ):
//   x = mean + √α (z − U(Σ₋ ⊙ (Ūᵀ z))),  Σ₋ = 1 − √(1 − d/α)  (uq.hpp:59-64)
inline void realization(const State& st, const Ctx& ctx, const double* z, double* out) {
    const Index n = Index(st.mean.size());
    if (st.alpha == 0.0) {  // uq.hpp:73
        std::copy(st.mean.begin(), st.mean.end(), out);
        return;
    }
    const double ra = std::sqrt(st.alpha);
    const Index r = Index(st.d.size());
    std::vector<double> proj(static_cast<size_t>(r)), up(size_t(n), 0.0);
    for (Index j = 0; j < r; ++j) {
        const double sm = 1.0 - std::sqrt(std::max(1.0 - st.d[size_t(j)] / st.alpha, 0.0));
        proj[size_t(j)] = sm * dot(ctx.gep.ubar.col(j), z, n);
    }
    if (r > 0) gemv(ctx.gep.u, proj.data(), up.data());
    for (Index i = 0; i < n; ++i) out[i] = st.mean[size_t(i)] + (ra * z[i] - ra * up[size_t(i)]);
}


// ---------------------------------------------------------------- boxcox.hpp:14-90
struct BoxCox {
    double alpha = 1.0;
    void validate() const {  // :19-23
        if (!(alpha > 0.0)) throw std::invalid_argument("boxcox: alpha must be positive, got " + std::to_string(alpha));
    }
    double forward(double s) const {  // :25-31
        validate();
        if (alpha == 1.0) return s - 1.0;
        if (s < 0.0) throw std::domain_error("boxcox: forward transform requires s >= 0");
        return alpha * (std::pow(s, 1.0 / alpha) - 1.0);
    }
    double inverse(double shat) const {  // :33-40
        validate();
        if (alpha == 1.0) return shat + 1.0;
        const double base = (shat + alpha) / alpha;
        if (base < 0.0) throw std::domain_error("boxcox: inverse transform requires (shat + alpha)/alpha >= 0");
        return std::pow(base, alpha);
    }
    double derivative(double shat) const {  // :43-50
        validate();
        if (alpha == 1.0) return 1.0;
        const double base = (shat + alpha) / alpha;
        if (base < 0.0) throw std::domain_error("boxcox: derivative requires (shat + alpha)/alpha >= 0");
        return std::pow(base, alpha - 1.0);
    }
    // vector map with the component index in the message (:58-75); which: 0 fwd, 1 inv, 2 der
    void map(const double* x, double* out, Index n, int which) const {
        static const char* what[3] = {"forward", "inverse", "derivative"};
        for (Index i = 0; i < n; ++i) {
            try {
                out[i] = which == 0 ? forward(x[i]) : which == 1 ? inverse(x[i]) : derivative(x[i]);
            } catch (const std::domain_error&) {
                throw std::domain_error("boxcox: " + std::string(what[which]) + " domain violation at index " +
                                        std::to_string(i) + " (value " + std::to_string(x[i]) + ")");
            }
            if (!std::isfinite(out[i]))
                throw std::domain_error("boxcox: " + std::string(what[which]) +
                                        " produced a non-finite value at index " + std::to_string(i));
        }
    }
};

// ekf_linearize boxcox.hpp:81-90: H_k = H·diag(∂s/∂ŝ), h(ŝ) = H·s(ŝ), same sparsity
inline void ekf_linearize(const Csr& h, const double* mean, const BoxCox& t, Csr& hk, std::vector<double>& h_of_mean) {
    const Index n = h.cols;
    std::vector<double> jac(static_cast<size_t>(n)), s(static_cast<size_t>(n));
    t.map(mean, jac.data(), n, 2);
    hk = h;
    for (size_t e = 0; e < hk.val.size(); ++e) hk.val[e] = h.val[e] * jac[size_t(h.col[e])];
    t.map(mean, s.data(), n, 1);
    h_of_mean.assign(size_t(h.rows), 0.0);
    csr_mv(h, s.data(), h_of_mean.data());
}

// CovarianceOperator::inverse_apply in fft mode (covariance.hpp:145-152): CG on the fast
// matvec (cg.hpp:20-50), tol 1e-12, max 10·√n + 10 iterations (:125), throwing on failure (:130-139)
inline void cov_solve(Cov& cov, const double* b, double* x, double tol = 1e-12) {
    const Index n = cov.size();
    const int max_iter = static_cast<int>(10.0 * std::sqrt(double(n))) + 10;
    std::fill(x, x + n, 0.0);
    const double bnorm = std::sqrt(dot(b, b, n));
    if (bnorm == 0.0) return;
    std::vector<double> r(b, b + n), p(b, b + n), ap(static_cast<size_t>(n));
    double rs = dot(r.data(), r.data(), n);
    int it = 0;
    double res = 0.0;
    for (; it < max_iter; ++it) {
        cov.apply(p.data(), ap.data());
        const double a = rs / dot(p.data(), ap.data(), n);
        axpy(a, p.data(), x, n);
        axpy(-a, ap.data(), r.data(), n);
        const double rs_next = dot(r.data(), r.data(), n);
        if (std::sqrt(rs_next) <= tol * bnorm) return;
        for (Index i = 0; i < n; ++i) p[size_t(i)] = r[size_t(i)] + (rs_next / rs) * p[size_t(i)];
        rs = rs_next;
        res = std::sqrt(rs) / bnorm;
    }
    std::ostringstream msg;
    msg << "cov_solve: CG did not converge within " << it << " iterations; achieved relative residual " << res
        << " (requested " << tol << ")";
    throw std::runtime_error(msg.str());
}

using BApply = std::function<void(const double*, double*)>;

// b_orthonormalize lowrank.hpp:53-106 with `against` and cached B·against
struct BOrtho { Mat q, bq; };
inline BOrtho b_orthonormalize_against(const Mat& v, const BApply& b_apply, const Mat& ag, const Mat& b_ag) {
    const Index n = v.rows, m = v.cols;
    BOrtho out;
    out.q = Mat(n, m);
    out.bq = Mat(n, m);
    Index kept = 0;
    std::vector<double> w(static_cast<size_t>(n)), bw(static_cast<size_t>(n));
    for (Index j = 0; j < m; ++j) {
        std::copy(v.col(j), v.col(j) + n, w.begin());
        for (double x : w)
            if (!std::isfinite(x))
                throw std::invalid_argument("b_orthonormalize: column " + std::to_string(j) + " contains non-finite entries");
        b_apply(w.data(), bw.data());
        const double pre_norm = std::sqrt(std::max(dot(w.data(), bw.data(), n), 0.0));
        double norm = 0.0;
        for (int sweep = 0; sweep < 2; ++sweep) {
            for (Index i = 0; i < ag.cols; ++i) axpy(-dot(b_ag.col(i), w.data(), n), ag.col(i), w.data(), n);
            for (Index i = 0; i < kept; ++i) axpy(-dot(out.bq.col(i), w.data(), n), out.q.col(i), w.data(), n);
            b_apply(w.data(), bw.data());
            norm = std::sqrt(std::max(dot(w.data(), bw.data(), n), 0.0));
        }
        if (norm <= 1e-12 * pre_norm || norm == 0.0) continue;
        for (Index i = 0; i < n; ++i) {
            out.q(i, kept) = w[size_t(i)] / norm;
            out.bq(i, kept) = bw[size_t(i)] / norm;
        }
        ++kept;
    }
    out.q.cols = out.bq.cols = kept;
    out.q.a.resize(size_t(n * kept));
    out.bq.a.resize(size_t(n * kept));
    return out;
}

// add_low_rank lowrank.hpp:238-294: U D_U Uᵀ + V D_V Vᵀ in one B-orthonormal factorization
struct LowRankSym { Mat w; std::vector<double> d; };
inline LowRankSym add_low_rank(const Mat& u, const std::vector<double>& d_u, const Mat& v,
                               const std::vector<double>& d_v, const BApply& b_apply, double tol) {
    if (u.cols != Index(d_u.size()) || v.cols != Index(d_v.size()))
        throw std::invalid_argument("add_low_rank: basis/diagonal size mismatch");
    if (tol < 0.0) throw std::invalid_argument("add_low_rank: tol must be nonnegative");
    if (v.cols == 0) return {u, d_u};
    if (u.cols == 0) return {v, d_v};
    const Index n = u.rows, ru = u.cols;
    Mat bu(n, ru);
    for (Index j = 0; j < ru; ++j) b_apply(u.col(j), bu.col(j));
    BOrtho orth = b_orthonormalize_against(v, b_apply, u, bu);
    const Index rv = orth.q.cols;
    const Mat c = gemm_tn(bu, v);           // ru × kv
    const Mat rh = gemm_tn(orth.bq, v);     // rv × kv
    const Index nm = ru + rv, kv = v.cols;
    Mat m(nm, nm);
    auto zrow = [&](Index i, Index k) { return i < ru ? c(i, k) : rh(i - ru, k); };
    for (Index j = 0; j < nm; ++j)
        for (Index i = 0; i < nm; ++i) {
            double sacc = 0.0;
            for (Index k = 0; k < kv; ++k) sacc += zrow(i, k) * d_v[size_t(k)] * zrow(j, k);
            m(i, j) = sacc + (i == j && i < ru ? d_u[size_t(i)] : 0.0);
        }
    for (Index j = 0; j < nm; ++j)
        for (Index i = 0; i < j; ++i) m(i, j) = m(j, i) = 0.5 * (m(i, j) + m(j, i));
    std::vector<double> ev;
    Mat vec;
    sym_eig(m, ev, vec);
    double max_abs = 0.0;
    for (double e : ev) max_abs = std::max(max_abs, std::fabs(e));
    std::vector<Index> keep;
    for (Index i = 0; i < nm; ++i)
        if (std::fabs(ev[size_t(i)]) >= tol * max_abs && ev[size_t(i)] != 0.0) keep.push_back(i);
    std::stable_sort(keep.begin(), keep.end(), [&](Index a, Index b) { return std::fabs(ev[size_t(a)]) > std::fabs(ev[size_t(b)]); });
    LowRankSym out;
    out.w = Mat(n, Index(keep.size()));
    out.d.resize(keep.size());
    for (size_t i = 0; i < keep.size(); ++i) {
        out.d[i] = ev[size_t(keep[i])];
        const double* e = vec.col(keep[i]);
        double* o = out.w.col(Index(i));
        for (Index k = 0; k < ru; ++k) axpy(e[k], u.col(k), o, n);
        for (Index k = 0; k < rv; ++k) axpy(e[ru + k], orth.q.col(k), o, n);
    }
    return out;
}

// ---------------------------------------------------------------- fast_filter.hpp:127-224 (extended filter)
struct FekfOptions {  // :127-134
    Index k_rank = -1;
    Index oversampling = 20;
    double trunc_tol = 1e-5;
    int relinearizations = 1;
    uint64_t seed = 0;
};
struct EState {  // LowRankState with its own W (fast_filter.hpp:21-37)
    double alpha = 0.0;
    int step = 0;
    std::vector<double> mean, d;
    Mat w;
};
inline EState fekf_step(const EState& st, Cov& cov, const Csr& h, const double* y, Index ylen, double sigma2,
                        const BoxCox& t, const FekfOptions& opts) {
    const Index n = cov.size();
    if (h.cols != n || Index(st.mean.size()) != n || ylen != h.rows)
        throw std::invalid_argument("fekf_step: dimension mismatch");
    if (!(sigma2 > 0.0)) throw std::invalid_argument("fekf_step: sigma2 must be positive");
    if (opts.relinearizations < 1 || opts.relinearizations > 5)
        throw std::invalid_argument("fekf_step: relinearizations must lie in [1, 5]");
    const double alpha = st.alpha + 1.0;
    const Index r = Index(st.d.size());
    std::vector<double> d_bar(static_cast<size_t>(r));
    for (Index i = 0; i < r; ++i) {
        if (!(st.d[size_t(i)] < alpha)) throw std::runtime_error("fekf_step: state diagonal exceeds alpha");
        d_bar[size_t(i)] = st.d[size_t(i)] / (alpha * (alpha - st.d[size_t(i)]));
    }
    const Index m = h.rows;
    std::vector<double> eta = st.mean;
    Csr h_last;
    for (int it = 0; it < opts.relinearizations; ++it) {  // :167-196
        Csr hk;
        std::vector<double> h_eta;
        ekf_linearize(h, eta.data(), t, hk, h_eta);
        Mat ght(n, m);  // ΓH_kᵀ column by column (:171-172)
        {
            std::vector<double> row(static_cast<size_t>(n));
            for (Index i = 0; i < m; ++i) {
                std::fill(row.begin(), row.end(), 0.0);
                for (int e = hk.rowptr[size_t(i)]; e < hk.rowptr[size_t(i) + 1]; ++e) row[size_t(hk.col[size_t(e)])] = hk.val[size_t(e)];
                cov.apply(row.data(), ght.col(i));
            }
        }
        Mat hw(m, r);  // H_k W
        for (Index j = 0; j < r; ++j) csr_mv(hk, st.w.col(j), hw.col(j));
        Mat s(m, m);
        for (Index j = 0; j < m; ++j) csr_mv(hk, ght.col(j), s.col(j));  // H_k ΓH_kᵀ
        for (Index j = 0; j < m; ++j)
            for (Index i = 0; i < m; ++i) {
                double acc = alpha * s(i, j);
                for (Index q = 0; q < r; ++q) acc -= hw(i, q) * st.d[size_t(q)] * hw(j, q);
                s(i, j) = acc + (i == j ? sigma2 : 0.0);
            }
        for (Index j = 0; j < m; ++j)
            for (Index i = 0; i < j; ++i) s(i, j) = s(j, i) = 0.5 * (s(i, j) + s(j, i));
        if (!llt(s)) throw std::runtime_error("fekf_step: innovation system is singular");
        std::vector<double> dm(static_cast<size_t>(n)), hdm(static_cast<size_t>(m)), z(static_cast<size_t>(m));
        for (Index i = 0; i < n; ++i) dm[size_t(i)] = st.mean[size_t(i)] - eta[size_t(i)];
        csr_mv(hk, dm.data(), hdm.data());
        for (Index i = 0; i < m; ++i) z[size_t(i)] = y[i] - h_eta[size_t(i)] - hdm[size_t(i)];
        llt_solve(s, z.data());
        std::vector<double> eta_next(st.mean);
        std::vector<double> gz(static_cast<size_t>(n));
        gemv(ght, z.data(), gz.data());
        axpy(alpha, gz.data(), eta_next.data(), n);
        if (r > 0) {
            std::vector<double> dc(static_cast<size_t>(r)), wdc(static_cast<size_t>(n));
            for (Index q = 0; q < r; ++q) dc[size_t(q)] = st.d[size_t(q)] * dot(hw.col(q), z.data(), m);
            gemv(st.w, dc.data(), wdc.data());
            axpy(-1.0, wdc.data(), eta_next.data(), n);
        }
        std::vector<double> diff(static_cast<size_t>(n));
        for (Index i = 0; i < n; ++i) diff[size_t(i)] = eta_next[size_t(i)] - eta[size_t(i)];
        const double change = std::sqrt(dot(diff.data(), diff.data(), n));
        h_last = std::move(hk);
        eta = std::move(eta_next);
        if (change <= 1e-6 * std::sqrt(dot(eta.data(), eta.data(), n))) break;
    }
    const Index k_rank = opts.k_rank < 0 ? m : opts.k_rank;  // :198-203
    Gep gep = randomized_ghep(cov, h_last, sigma2, k_rank, opts.oversampling, opts.seed);
    const BApply b_apply = [&cov](const double* x, double* out) { cov_solve(cov, x, out); };
    LowRankSym sum = add_low_rank(st.w, d_bar, gep.u, gep.lambda, b_apply, opts.trunc_tol);
    EState next;  // :210-222
    next.alpha = alpha;
    next.step = st.step + 1;
    next.mean = std::move(eta);
    std::vector<Index> keep;
    for (Index i = 0; i < Index(sum.d.size()); ++i)
        if (sum.d[size_t(i)] > 1e-14) keep.push_back(i);
    next.w = Mat(n, Index(keep.size()));
    next.d.resize(keep.size());
    for (size_t i = 0; i < keep.size(); ++i) {
        const double dhat = sum.d[size_t(keep[i])];
        next.d[i] = alpha * alpha * dhat / (1.0 + alpha * dhat);
        std::copy(sum.w.col(keep[i]), sum.w.col(keep[i]) + n, next.w.col(Index(i)));
    }
    return next;
}


// ---------------------------------------------------------------- enkf.hpp:43-94 (perturbed-observation EnKF)
inline void enkf_step(Mat& members, const Csr& h, const double* y, Index ylen, Cov& cov, double sigma2,
                      uint64_t seed) {
    const Index n = members.rows, ne = members.cols;
    if (ne < 2) throw std::invalid_argument("enkf_step: ensemble size must be at least 2");
    if (h.cols != n || ylen != h.rows) throw std::invalid_argument("enkf_step: dimension mismatch");
    if (sigma2 < 0.0) throw std::invalid_argument("enkf_step: sigma2 must be nonnegative");
    const uint64_t seed_forecast = derive_seed(seed, 1), seed_perturb = derive_seed(seed, 2);  // :61-62
    const Index m = h.rows;
    {  // forecast increments (:64-70), pairs in parallel (independent streams)
        const Index np = (ne + 1) / 2;
#pragma omp parallel for schedule(dynamic)
        for (Index j2 = 0; j2 < np; ++j2) {
            std::vector<double> a(static_cast<size_t>(n)), b(static_cast<size_t>(n));
            cov.sample_pair(seed_forecast, uint64_t(j2), a.data(), b.data());
            axpy(1.0, a.data(), members.col(2 * j2), n);
            if (2 * j2 + 1 < ne) axpy(1.0, b.data(), members.col(2 * j2 + 1), n);
        }
    }
    Mat hm(m, ne);
#pragma omp parallel for schedule(static)
    for (Index j = 0; j < ne; ++j) csr_mv(h, members.col(j), hm.col(j));  // :72
    std::vector<double> mmean(static_cast<size_t>(n), 0.0), hmean(static_cast<size_t>(m), 0.0);  // :73-74
    for (Index j = 0; j < ne; ++j) {
        axpy(1.0, members.col(j), mmean.data(), n);
        axpy(1.0, hm.col(j), hmean.data(), m);
    }
    for (auto& v : mmean) v /= double(ne);
    for (auto& v : hmean) v /= double(ne);
    Mat dev(n, ne), hdev(m, ne);  // :75-76
    for (Index j = 0; j < ne; ++j) {
        for (Index i = 0; i < n; ++i) dev(i, j) = members(i, j) - mmean[size_t(i)];
        for (Index i = 0; i < m; ++i) hdev(i, j) = hm(i, j) - hmean[size_t(i)];
    }
    Mat cyy(m, m);  // :78-80
    {
        Mat hdt(ne, m);
        for (Index j = 0; j < ne; ++j)
            for (Index i = 0; i < m; ++i) hdt(j, i) = hdev(i, j);
#pragma omp parallel for schedule(static)
        for (Index b = 0; b < m; ++b)
            for (Index a = 0; a < m; ++a) cyy(a, b) = dot(hdt.col(a), hdt.col(b), ne) / double(ne - 1);
    }
    for (Index i = 0; i < m; ++i) cyy(i, i) += sigma2;
    for (Index b = 0; b < m; ++b)
        for (Index a = 0; a < b; ++a) cyy(a, b) = cyy(b, a) = 0.5 * (cyy(a, b) + cyy(b, a));
    if (!llt(cyy))  // :81-85
        throw std::runtime_error("enkf_step: sample innovation covariance is singular even with observation noise added");
    // innovations (:89-96) solved in place: Z = C_yy⁻¹ (y + σ v_j − Hm_j)
    Mat z(m, ne);
    const double sigma = std::sqrt(sigma2);
#pragma omp parallel for schedule(static)
    for (Index j = 0; j < ne; ++j) {
        double* c = z.col(j);
        if (sigma2 > 0.0) {
            gaussian_vector(m, seed_perturb, uint64_t(j), c);
            for (Index i = 0; i < m; ++i) c[i] = y[i] + sigma * c[i] - hm(i, j);
        } else {
            for (Index i = 0; i < m; ++i) c[i] = y[i] - hm(i, j);
        }
        llt_solve(cyy, c);
    }
    // members += C_sy Z, C_sy = dev·hdevᵀ/(ne − 1) (:87, :97)
    Mat csy(n, m);
#pragma omp parallel for schedule(static)
    for (Index b = 0; b < m; ++b) {
        double* c = csy.col(b);
        for (Index j = 0; j < ne; ++j) {
            const double w = hdev(b, j) / double(ne - 1);
            const double* d = dev.col(j);
            for (Index i = 0; i < n; ++i) c[i] += d[i] * w;
        }
    }
#pragma omp parallel for schedule(static)
    for (Index j = 0; j < ne; ++j) {
        double* x = members.col(j);
        for (Index b = 0; b < m; ++b) {
            const double w = z(b, j);
            const double* c = csy.col(b);
            for (Index i = 0; i < n; ++i) x[i] += c[i] * w;
        }
    }
}

}  // namespace orc

// =================================================================== C API (ctypes)
namespace {
thread_local std::string g_err;
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}
orc::KernelSpec mk_kernel(int family, double theta, double length, double power, double nu, double alpha_scale) {
    orc::KernelSpec s;
    s.family = family;
    s.theta = theta;
    s.length = length;
    s.power = power;
    s.nu = nu;
    s.alpha_scale = alpha_scale;
    return s;
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
int orc_max_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

uint64_t orc_splitmix64(uint64_t x) { return orc::splitmix64(x); }
uint64_t orc_derive_seed(uint64_t s, uint64_t t) { return orc::derive_seed(s, t); }
void orc_gaussian_vector(long long n, uint64_t seed, uint64_t stream, double* out) { orc::gaussian_vector(n, seed, stream, out); }
void orc_gaussian_matrix(long long r, long long c, uint64_t seed, uint64_t base, double* out) { orc::gaussian_matrix(r, c, seed, base, out); }
void orc_uniforms(long long n, uint64_t seed, uint64_t stream, double* out) {
    orc::Rng rng(seed, stream);
    for (long long i = 0; i < n; ++i) out[i] = rng.uniform();
}

int orc_kernel_eval(int family, double theta, double length, double power, double nu, double alpha_scale, double r, double* out) {
    return guarded([&] { *out = orc::kernel_eval(mk_kernel(family, theta, length, power, nu, alpha_scale), r); });
}
int orc_next_smooth(int n) { return orc::next_smooth(n); }

// 2-D unnormalized c2c DFT, interleaved complex, row-major mx×my; sign −1 forward.
void orc_fft2d(int mx, int my, double* data, int sign) {
    orc::Fft2d p(mx, my);
    p.exec(reinterpret_cast<orc::cplx*>(data), sign);
}

void* orc_cov_create(int nx, int ny, double lx, double ly, int family, double theta, double length, double power,
                     double nu, double alpha_scale) {
    orc::Cov* c = nullptr;
    const int rc = guarded([&] {
        orc::Grid g{nx, ny, lx, ly};
        c = new orc::Cov(g, mk_kernel(family, theta, length, power, nu, alpha_scale));
    });
    return rc ? nullptr : c;
}
void orc_cov_destroy(void* c) { delete static_cast<orc::Cov*>(c); }
void orc_cov_dims(void* c, int* mx, int* my) {
    *mx = static_cast<orc::Cov*>(c)->mx;
    *my = static_cast<orc::Cov*>(c)->my;
}
void orc_cov_spectrum(void* c, double* out) {
    auto* cv = static_cast<orc::Cov*>(c);
    std::copy(cv->spectrum.begin(), cv->spectrum.end(), out);
}
long orc_cov_apply_count(void* c) { return static_cast<orc::Cov*>(c)->applies; }
int orc_cov_apply(void* c, const double* x, long long ncols, double* y) {
    return guarded([&] { static_cast<orc::Cov*>(c)->apply_matrix(x, ncols, y); });
}
int orc_cov_sample_pair(void* c, uint64_t seed, uint64_t stream, double* a, double* b) {
    return guarded([&] { static_cast<orc::Cov*>(c)->sample_pair(seed, stream, a, b); });
}

// trace_ray: returns number of segments (≤ cap) or −1 with error
int orc_trace_ray(int nx, int ny, double lx, double ly, double sx, double sy, double rx, double ry, int cap,
                  long long* cells, double* lengths) {
    int n = -1;
    const int rc = guarded([&] {
        orc::Grid g{nx, ny, lx, ly};
        g.validate();
        auto segs = orc::trace_ray(g, sx, sy, rx, ry);
        n = int(segs.size());
        for (int i = 0; i < std::min(n, cap); ++i) {
            cells[i] = segs[size_t(i)].cell;
            lengths[i] = segs[size_t(i)].length;
        }
    });
    return rc ? -1 : n;
}

void* orc_build_H(int nx, int ny, double lx, double ly, int ns, const double* src, int nr, const double* rec) {
    orc::Csr* h = nullptr;
    const int rc = guarded([&] {
        orc::Grid g{nx, ny, lx, ly};
        g.validate();
        h = new orc::Csr(orc::build_H(g, std::vector<double>(src, src + 2 * ns), std::vector<double>(rec, rec + 2 * nr)));
    });
    return rc ? nullptr : h;
}
void* orc_csr_create(int rows, int cols, const int* rowptr, const int* col, const double* val) {
    auto* h = new orc::Csr;
    h->rows = rows;
    h->cols = cols;
    h->rowptr.assign(rowptr, rowptr + rows + 1);
    h->col.assign(col, col + rowptr[rows]);
    h->val.assign(val, val + rowptr[rows]);
    return h;
}
void orc_csr_destroy(void* h) { delete static_cast<orc::Csr*>(h); }
void orc_csr_dims(void* h, int* rows, int* cols, long long* nnz) {
    auto* c = static_cast<orc::Csr*>(h);
    *rows = c->rows;
    *cols = c->cols;
    *nnz = c->nnz();
}
void orc_csr_get(void* h, int* rowptr, int* col, double* val) {
    auto* c = static_cast<orc::Csr*>(h);
    std::copy(c->rowptr.begin(), c->rowptr.end(), rowptr);
    std::copy(c->col.begin(), c->col.end(), col);
    std::copy(c->val.begin(), c->val.end(), val);
}

// GHEP alone (lowrank.hpp:208-213 with a_apply = HᵀH/σ²).  Output into a Ctx-less holder.
void* orc_ghep(void* cov, void* h, double sigma2, long long k, long long p, uint64_t seed) {
    orc::Gep* g = nullptr;
    const int rc = guarded([&] {
        g = new orc::Gep(orc::randomized_ghep(*static_cast<orc::Cov*>(cov), *static_cast<orc::Csr*>(h), sigma2, k, p, seed));
    });
    return rc ? nullptr : g;
}
void orc_ghep_destroy(void* g) { delete static_cast<orc::Gep*>(g); }
long long orc_ghep_rank(void* g) { return static_cast<orc::Gep*>(g)->rank(); }
long long orc_ghep_kept_cols(void* g) { return static_cast<orc::Gep*>(g)->kept_cols; }
void orc_ghep_get(void* g, double* lambda, double* u, double* ubar) {
    auto* G = static_cast<orc::Gep*>(g);
    std::copy(G->lambda.begin(), G->lambda.end(), lambda);
    if (u) std::copy(G->u.a.begin(), G->u.a.end(), u);
    if (ubar) std::copy(G->ubar.a.begin(), G->ubar.a.end(), ubar);
}

struct OrcFilter {
    orc::Cov* cov;
    orc::Ctx ctx;
    orc::State st;
};
void* orc_fkf_init(void* cov, void* h, double sigma2, long long k, long long p, uint64_t seed) {
    OrcFilter* f = nullptr;
    const int rc = guarded([&] {
        auto* c = static_cast<orc::Cov*>(cov);
        f = new OrcFilter{c, orc::fkf_init(*c, *static_cast<orc::Csr*>(h), sigma2, k, p, seed), {}};
        f->st.mean.assign(size_t(c->size()), 0.0);  // zero_start fast_filter.hpp:30-36
    });
    return rc ? nullptr : f;
}
void orc_fkf_destroy(void* f) { delete static_cast<OrcFilter*>(f); }
long long orc_fkf_rank(void* f) { return static_cast<OrcFilter*>(f)->ctx.gep.rank(); }
void orc_fkf_ctx_get(void* f, double* lambda, double* u, double* ubar, double* g, double* b, double* gamma_ht) {
    auto* F = static_cast<OrcFilter*>(f);
    const auto& c = F->ctx;
    if (lambda) std::copy(c.gep.lambda.begin(), c.gep.lambda.end(), lambda);
    if (u) std::copy(c.gep.u.a.begin(), c.gep.u.a.end(), u);
    if (ubar) std::copy(c.gep.ubar.a.begin(), c.gep.ubar.a.end(), ubar);
    if (g) std::copy(c.h_gamma_ht.a.begin(), c.h_gamma_ht.a.end(), g);
    if (b) std::copy(c.h_u.a.begin(), c.h_u.a.end(), b);
    if (gamma_ht) std::copy(c.gamma_ht.a.begin(), c.gamma_ht.a.end(), gamma_ht);
}
int orc_fkf_step(void* f, const double* y, long long ylen) {
    return guarded([&] {
        auto* F = static_cast<OrcFilter*>(f);
        F->st = orc::fkf_step(F->st, F->ctx, y, ylen);
    });
}
void orc_fkf_state(void* f, double* alpha, double* d, double* mean, int* step) {
    auto* F = static_cast<OrcFilter*>(f);
    if (alpha) *alpha = F->st.alpha;
    if (d) std::copy(F->st.d.begin(), F->st.d.end(), d);
    if (mean) std::copy(F->st.mean.begin(), F->st.mean.end(), mean);
    if (step) *step = F->st.step;
}
long long orc_fkf_state_rank(void* f) { return (long long)static_cast<OrcFilter*>(f)->st.d.size(); }
void orc_fkf_set_state(void* f, double alpha, const double* d, long long r, const double* mean, int step) {
    auto* F = static_cast<OrcFilter*>(f);
    F->st.alpha = alpha;
    F->st.d.assign(d, d + r);
    F->st.mean.assign(mean, mean + F->cov->size());
    F->st.step = step;
}
int orc_variance(void* f, double* out) {
    return guarded([&] {
        auto* F = static_cast<OrcFilter*>(f);
        orc::variance(F->st, F->ctx, *F->cov, out);
    });
}
int orc_trace_criterion(void* f, double* out) {
    return guarded([&] {
        auto* F = static_cast<OrcFilter*>(f);
        *out = orc::trace_criterion(F->st, F->ctx, *F->cov);
    });
}
int orc_relative_entropy(void* f, double* out) {
    return guarded([&] { *out = orc::relative_entropy(static_cast<OrcFilter*>(f)->st); });
}
// `count` realizations: draw s uses sample_pair stream s/2, Re for even s, Im for odd.
int orc_realizations(void* f, uint64_t seed, int count, double* out) {
    return guarded([&] {
        auto* F = static_cast<OrcFilter*>(f);
        const long long n = F->cov->size();
        std::vector<double> a(static_cast<size_t>(n)), b(static_cast<size_t>(n));
        for (int s = 0; s < count; s += 2) {
            F->cov->sample_pair(seed, uint64_t(s / 2), a.data(), b.data());
            orc::realization(F->st, F->ctx, a.data(), out + (long long)s * n);
            if (s + 1 < count) orc::realization(F->st, F->ctx, b.data(), out + (long long)(s + 1) * n);
        }
    });
}

}  // extern "C"

// ---- extended filter (fast_filter.hpp:127-224), Box–Cox (boxcox.hpp), CG Γ⁻¹ (covariance.hpp:118-152)
extern "C" {
int orc_boxcox_map(double alpha, int which, const double* x, long long n, double* out) {
    return guarded([&] { orc::BoxCox{alpha}.map(x, out, n, which); });
}
int orc_cov_solve(void* c, const double* b, double tol, double* x) {
    return guarded([&] { orc::cov_solve(*static_cast<orc::Cov*>(c), b, x, tol); });
}
void* orc_fekf_create(long long n, const double* mean0) {
    auto* st = new orc::EState;
    st->mean.assign(mean0, mean0 + n);
    st->w = orc::Mat(n, 0);
    return st;
}
void orc_fekf_destroy(void* st) { delete static_cast<orc::EState*>(st); }
int orc_fekf_step(void* st, void* cov, void* h, const double* y, long long ylen, double sigma2, double bc_alpha,
                  long long k_rank, long long p, double trunc_tol, int relin, uint64_t seed) {
    return guarded([&] {
        orc::FekfOptions o;
        o.k_rank = k_rank;
        o.oversampling = p;
        o.trunc_tol = trunc_tol;
        o.relinearizations = relin;
        o.seed = seed;
        auto* s = static_cast<orc::EState*>(st);
        *s = orc::fekf_step(*s, *static_cast<orc::Cov*>(cov), *static_cast<orc::Csr*>(h), y, ylen, sigma2,
                            orc::BoxCox{bc_alpha}, o);
    });
}
void orc_fekf_dims(void* st, double* alpha, int* step, long long* rank) {
    auto* s = static_cast<orc::EState*>(st);
    *alpha = s->alpha;
    *step = s->step;
    *rank = (long long)s->d.size();
}
void orc_fekf_read(void* st, double* mean, double* d, double* w) {
    auto* s = static_cast<orc::EState*>(st);
    std::copy(s->mean.begin(), s->mean.end(), mean);
    std::copy(s->d.begin(), s->d.end(), d);
    std::copy(s->w.a.begin(), s->w.a.end(), w);
}
}  // extern "C"

extern "C" {
// enkf_step (enkf.hpp:43-94) on a column-major n×ne member block, in place
int orc_enkf_step(double* members, long long n, long long ne, void* h, const double* y, long long ylen, void* cov,
                  double sigma2, uint64_t seed) {
    return guarded([&] {
        orc::Mat x(n, ne);
        std::copy(members, members + n * ne, x.a.begin());
        orc::enkf_step(x, *static_cast<orc::Csr*>(h), y, ylen, *static_cast<orc::Cov*>(cov), sigma2, seed);
        std::copy(x.a.begin(), x.a.end(), members);
    });
}
}  // extern "C"
