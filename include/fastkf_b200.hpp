// fastkf_b200.hpp — drop-in C++ shim restoring the reference's `namespace fastkf` hot-path
// API (/root/reference/proj/include/fastkf/*.hpp) on top of the C ABI in fastkf_b200.h.
//
// Same class/function names, argument meaning and exception types as the reference:
//   Grid (grid.hpp:22-63), KernelSpec/KernelFamily (kernel.hpp:19-48), kernel_eval (:51-63),
//   CovarianceOperator FFT mode (covariance.hpp:69-353), SourceReceiverLayout (tomography.hpp:
//   90-126), build_H (:130-146), GepResult (lowrank.hpp:26-31), randomized_ghep specialised to
//   A = HᵀH/σ² (lowrank.hpp:208-213 with fast_filter.hpp:63-66), FkfContext/fkf_init
//   (fast_filter.hpp:42-75), LowRankState/fkf_step (:21-37, :84-125), variance /
//   trace_criterion / relative_entropy (uq.hpp:16-53), BoxCox/FekfOptions/fekf_step
//   (boxcox.hpp:14-17, fast_filter.hpp:127-224), Field/write_field/read_field/write_state/
//   read_state (field_io.hpp:18-135), Ensemble/enkf_init/enkf_step (enkf.hpp:15-94).
// Eigen is not required: Vector/Matrix/SparseRowMatrix are thin column-major stand-ins with
// the subset of API callers use (SURVEY.md §8b caveat 2).  Error codes map back to
// std::invalid_argument (1) and std::runtime_error (2, 3).
//
// Value semantics are kept: fkf_step returns a new LowRankState.  The filter state lives on
// the GPU; a state whose token matches the context's device state is stepped without any
// upload, otherwise it is uploaded first (so arbitrary user-constructed states still work).
#pragma once

#include <bit>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fastkf_b200.h"

namespace fastkf {

using Index = long long;

namespace detail {
inline void check(int rc) {
    if (rc == FKB_OK) return;
    const std::string msg = fkb_last_error();
    if (rc == FKB_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == FKB_DOMAIN_ERROR) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}
}  // namespace detail

struct Vector {
    std::vector<double> v;
    Vector() = default;
    explicit Vector(Index n, double x = 0.0) : v(size_t(n), x) {}
    static Vector Zero(Index n) { return Vector(n); }
    static Vector Constant(Index n, double x) { return Vector(n, x); }
    Index size() const { return Index(v.size()); }
    double& operator[](Index i) { return v[size_t(i)]; }
    double operator[](Index i) const { return v[size_t(i)]; }
    double* data() { return v.data(); }
    const double* data() const { return v.data(); }
};

struct Matrix {  // column-major (Eigen::MatrixXd default)
    Index r = 0, c = 0;
    std::vector<double> a;
    Matrix() = default;
    Matrix(Index rows, Index cols) : r(rows), c(cols), a(size_t(rows * cols), 0.0) {}
    Index rows() const { return r; }
    Index cols() const { return c; }
    double& operator()(Index i, Index j) { return a[size_t(i + j * r)]; }
    double operator()(Index i, Index j) const { return a[size_t(i + j * r)]; }
    double* data() { return a.data(); }
    const double* data() const { return a.data(); }
};

struct SparseRowMatrix {  // CSR, int32 indices (grid.hpp:15)
    int m = 0, n = 0;
    std::vector<int> rowptr{0}, col;
    std::vector<double> val;
    Index rows() const { return m; }
    Index cols() const { return n; }
    Index nonZeros() const { return Index(val.size()); }
};

struct Grid {  // grid.hpp:22-63
    int nx = 0, ny = 0;
    double lx = 1.0, ly = 1.0;
    Grid() = default;
    Grid(int nx_, int ny_, double lx_ = 1.0, double ly_ = 1.0) : nx(nx_), ny(ny_), lx(lx_), ly(ly_) { validate(); }
    void validate() const {
        if (nx < 1 || ny < 1)
            throw std::invalid_argument("grid: nx and ny must be positive, got " + std::to_string(nx) + "x" +
                                        std::to_string(ny));
        if (!(lx > 0.0) || !(ly > 0.0)) throw std::invalid_argument("grid: domain lengths must be positive");
    }
    Index size() const { return Index(nx) * ny; }
    double dx() const { return lx / nx; }
    double dy() const { return ly / ny; }
    Index index(int ix, int iy) const { return Index(ix) * ny + iy; }
};

enum class KernelFamily { powered_exponential, matern };
enum class CovMode { fft, dense };

struct KernelSpec {  // kernel.hpp:19-48
    KernelFamily family = KernelFamily::powered_exponential;
    double theta = 1.0, length = 0.2, power = 1.0, nu = 0.5, alpha_scale = 0.0;
};

inline double kernel_eval(const KernelSpec& s, double r) {  // kernel.hpp:51-63
    double out = 0.0;
    detail::check(fkb_kernel_eval(int(s.family), s.theta, s.length, s.power, s.nu, s.alpha_scale, r, &out));
    return out;
}

class CovarianceOperator {  // covariance.hpp:69-353 (FFT mode on the GPU)
public:
    CovarianceOperator(const Grid& g, const KernelSpec& s, CovMode mode = CovMode::fft) : grid_(g), spec_(s) {
        if (mode != CovMode::fft)
            throw std::runtime_error("covariance: the B200 path implements the circulant-fft mode only");
        fkb_cov* h = nullptr;
        detail::check(fkb_cov_create(g.nx, g.ny, g.lx, g.ly, int(s.family), s.theta, s.length, s.power, s.nu,
                                     s.alpha_scale, &h));
        h_.reset(h);
    }
    CovarianceOperator(const CovarianceOperator&) = delete;
    CovarianceOperator& operator=(const CovarianceOperator&) = delete;
    const Grid& grid() const { return grid_; }
    const KernelSpec& spec() const { return spec_; }
    Index size() const { return grid_.size(); }
    Vector apply(const Vector& x) const {
        if (x.size() != size())
            throw std::invalid_argument("cov_apply: expected vector of length " + std::to_string(size()) + ", got " +
                                        std::to_string(x.size()));
        Vector y(size());
        detail::check(fkb_cov_apply(h_.get(), x.data(), size(), 1, y.data(), size()));
        return y;
    }
    Matrix apply_matrix(const Matrix& xs) const {
        if (xs.rows() != size()) throw std::invalid_argument("cov_apply: dimension mismatch");
        Matrix out(xs.rows(), xs.cols());
        detail::check(fkb_cov_apply(h_.get(), xs.data(), size(), int(xs.cols()), out.data(), size()));
        return out;
    }
    Vector diagonal() const { return Vector::Constant(size(), spec_.theta); }
    double trace() const { return double(size()) * spec_.theta; }
    std::pair<Vector, Vector> sample_pair(std::uint64_t seed, std::uint64_t stream = 0) const {
        Vector a(size()), b(size());
        detail::check(fkb_cov_sample_pair(h_.get(), seed, stream, a.data(), b.data()));
        return {std::move(a), std::move(b)};
    }
    Vector spectrum() const {
        int mx = 0, my = 0;
        detail::check(fkb_cov_dims(h_.get(), &mx, &my));
        Vector s(Index(mx) * my);
        detail::check(fkb_cov_spectrum(h_.get(), s.data()));
        return s;
    }
    long apply_count() const { return long(fkb_cov_apply_count(h_.get())); }
    fkb_cov* handle() const { return h_.get(); }

private:
    struct Del {
        void operator()(fkb_cov* p) const { fkb_cov_destroy(p); }
    };
    Grid grid_;
    KernelSpec spec_;
    std::unique_ptr<fkb_cov, Del> h_;
};

struct SourceReceiverLayout {  // tomography.hpp:90-126
    std::vector<std::pair<double, double>> sources, receivers;
    Index n_m() const { return Index(sources.size()) * Index(receivers.size()); }
    static SourceReceiverLayout cross_well(const Grid& g, int n_sou, int n_rec, double source_x = 0.0,
                                           double receiver_x = -1.0) {
        if (n_sou < 1 || n_rec < 1) throw std::invalid_argument("layout: n_sou and n_rec must be positive");
        if (receiver_x < 0.0) receiver_x = g.lx;
        SourceReceiverLayout L;
        for (int i = 0; i < n_sou; ++i) L.sources.push_back({source_x, (i + 0.5) * g.ly / n_sou});
        for (int j = 0; j < n_rec; ++j) L.receivers.push_back({receiver_x, (j + 0.5) * g.ly / n_rec});
        return L;
    }
};

inline SparseRowMatrix build_H(const Grid& g, const SourceReceiverLayout& L) {  // tomography.hpp:130-146
    std::vector<double> s, r;
    for (auto& p : L.sources) { s.push_back(p.first); s.push_back(p.second); }
    for (auto& p : L.receivers) { r.push_back(p.first); r.push_back(p.second); }
    int rows = 0;
    long long nnz = 0;
    detail::check(fkb_build_H(g.nx, g.ny, g.lx, g.ly, int(L.sources.size()), s.data(), int(L.receivers.size()),
                              r.data(), &rows, &nnz, nullptr, nullptr, nullptr, 0));
    SparseRowMatrix h;
    h.m = rows;
    h.n = int(g.size());
    h.rowptr.resize(size_t(rows) + 1);
    h.col.resize(size_t(nnz));
    h.val.resize(size_t(nnz));
    detail::check(fkb_build_H(g.nx, g.ny, g.lx, g.ly, int(L.sources.size()), s.data(), int(L.receivers.size()),
                              r.data(), &rows, &nnz, h.rowptr.data(), h.col.data(), h.val.data(), nnz));
    return h;
}

struct GepResult {  // lowrank.hpp:26-31
    Matrix u;
    Vector lambda;
    Index rank() const { return lambda.size(); }
};

namespace detail {
struct EkfDevice {  // device-resident extended-filter state (W, W̄ = Γ⁻¹W) behind fekf_step
    fkb_ekf* e = nullptr;
    const void* cov = nullptr;
    const void* h = nullptr;
    long long generation = 0;
    ~EkfDevice() {
        if (e) fkb_ekf_destroy(e);
    }
};
}  // namespace detail

struct LowRankState {  // fast_filter.hpp:21-37 (W ≡ U lives on the device)
    double alpha = 0.0;
    Vector d;
    Vector mean;
    int step = 0;
    const void* token = nullptr;  // context whose device state this mirrors ...
    long long generation = -1;    // ... at this generation of that context
    // extended filter (fekf_step): W and Γ⁻¹W stay on the device; w() downloads W
    std::shared_ptr<detail::EkfDevice> ekf;
    long long ekf_generation = -1;
    Matrix w_host;  // W of a state read from a FKS1 file (read_state)
    Index rank() const { return d.size(); }
    Matrix w() const {
        if (w_host.cols() == rank() && w_host.rows() == mean.size() && (rank() || !ekf)) return w_host;
        if (!ekf) throw std::invalid_argument("LowRankState::w: W is held by the filter context (W = U)");
        Matrix W(mean.size(), rank());
        if (rank()) detail::check(fkb_ekf_read(ekf->e, nullptr, nullptr, W.data(), nullptr));
        return W;
    }
    static LowRankState zero_start(Index n) {
        LowRankState s;
        s.mean = Vector::Zero(n);
        return s;
    }
};

class FkfContext {  // fast_filter.hpp:42-49 + device-resident state
public:
    FkfContext(const CovarianceOperator& cov, const SparseRowMatrix& h, double sigma2, Index k_rank,
               Index p_oversample, std::uint64_t seed)
        : n_(cov.size()), m_(h.m), sigma2_(sigma2) {
        fkb_filter* f = nullptr;
        detail::check(fkb_fkf_init(cov.handle(), h.m, h.n, h.rowptr.data(), h.col.empty() ? nullptr : h.col.data(),
                                   h.val.empty() ? nullptr : h.val.data(), sigma2, k_rank, p_oversample, seed, &f));
        f_.reset(f);
        detail::check(fkb_filter_rank(f_.get(), &r_, nullptr));
        gep_.lambda = Vector(r_);
        if (r_) detail::check(fkb_filter_lambda(f_.get(), gep_.lambda.data()));
    }
    const GepResult& gep() const { return gep_; }
    Matrix u() const {  // GepResult::u on demand (N×r)
        Matrix U(n_, r_);
        if (r_) detail::check(fkb_filter_get(f_.get(), 0, U.data()));
        return U;
    }
    Index rank() const { return r_; }
    Index n_m() const { return m_; }
    double sigma2() const { return sigma2_; }
    fkb_filter* handle() const { return f_.get(); }
    long long generation = 0;  // bumped on every device-state change; tokens must match it

private:
    struct Del {
        void operator()(fkb_filter* p) const { fkb_filter_destroy(p); }
    };
    Index n_ = 0, m_ = 0;
    int r_ = 0;
    double sigma2_ = 0.0;
    GepResult gep_;
    std::unique_ptr<fkb_filter, Del> f_;
};

inline FkfContext fkf_init(const CovarianceOperator& cov, const SparseRowMatrix& h, double sigma2, Index k_rank,
                           Index p_oversample, std::uint64_t seed) {  // fast_filter.hpp:51-75
    if (h.cols() != cov.size()) throw std::invalid_argument("fkf_init: H columns do not match state dimension");
    if (!(sigma2 > 0.0)) throw std::invalid_argument("fkf_init: sigma2 must be positive");
    return FkfContext(cov, h, sigma2, k_rank, p_oversample, seed);
}

namespace detail {
inline void sync_state(const LowRankState& s, FkfContext& ctx) {
    if (s.token == ctx.handle() && s.generation == ctx.generation) return;
    detail::check(fkb_filter_set_state(ctx.handle(), s.alpha, s.step, int(s.rank()), s.rank() ? s.d.data() : nullptr,
                                       s.mean.data()));
    ++ctx.generation;
}
}  // namespace detail

// fast_filter.hpp:84-125
inline LowRankState fkf_step(const LowRankState& state, FkfContext& ctx, const Vector& y) {
    if (y.size() != ctx.n_m())
        throw std::invalid_argument("fkf_step: observation length " + std::to_string(y.size()) + " does not match " +
                                    std::to_string(ctx.n_m()) + " measurements");
    if (state.rank() != 0 && state.rank() != ctx.rank())
        throw std::invalid_argument(
            "fkf_step: state rank does not match the eigendecomposition (constant-H regime requires W = U)");
    detail::sync_state(state, ctx);
    LowRankState next;
    next.d = Vector(ctx.rank());
    next.mean = Vector(state.mean.size());
    // step + new state in one round trip (value semantics of fast_filter.hpp:84-125)
    detail::check(fkb_fkf_step_state(ctx.handle(), y.data(), y.size(), &next.alpha, next.d.data(), next.mean.data()));
    int rank = 0;
    detail::check(fkb_filter_state(ctx.handle(), nullptr, &next.step, &rank, nullptr, nullptr));
    next.d.v.resize(size_t(rank));
    next.token = ctx.handle();
    next.generation = ++ctx.generation;
    return next;
}

// uq.hpp:16-53 (evaluated on the context's device state after syncing `state`)
inline Vector variance(const LowRankState& state, FkfContext& ctx) {
    detail::sync_state(state, ctx);
    Vector out(state.mean.size());
    detail::check(fkb_variance(ctx.handle(), out.data()));
    return out;
}
inline double trace_criterion(const LowRankState& state, FkfContext& ctx) {
    detail::sync_state(state, ctx);
    double v = 0.0;
    detail::check(fkb_trace_criterion(ctx.handle(), &v));
    return v;
}
inline double relative_entropy(const LowRankState& state, FkfContext& ctx) {
    detail::sync_state(state, ctx);
    double v = 0.0;
    detail::check(fkb_relative_entropy(ctx.handle(), &v));
    return v;
}

// ---- extended fast filter (fast_filter.hpp:127-224, boxcox.hpp:14-17)
struct BoxCox {
    double alpha = 1.0;
};
enum class GhepMode { two_pass, single_pass };
struct FekfOptions {  // fast_filter.hpp:127-134
    Index k_rank = -1;
    Index oversampling = 20;
    double trunc_tol = 1e-5;
    int relinearizations = 1;
    GhepMode mode = GhepMode::two_pass;
    std::uint64_t seed = 0;
};

// fekf_step (fast_filter.hpp:142-224).  Value semantics as the reference: a new state is
// returned.  States produced by this function keep W and Γ⁻¹W on the device (shared handle);
// a rank-0 state (zero_start with any mean) starts a new device filter.  A state is stepped in
// place when it is the latest one of its device filter, otherwise it is rejected (W̄ = Γ⁻¹W of an
// older state is no longer held).
inline LowRankState fekf_step(const LowRankState& state, const CovarianceOperator& cov, const SparseRowMatrix& h,
                              const Vector& y, double sigma2, const BoxCox& transform, const FekfOptions& opts) {
    if (h.cols() != cov.size() || state.mean.size() != cov.size() || y.size() != h.rows())
        throw std::invalid_argument("fekf_step: dimension mismatch");
    if (opts.mode != GhepMode::two_pass)
        throw std::invalid_argument("fekf_step: only the two-pass GHEP is provided on the GPU");
    std::shared_ptr<detail::EkfDevice> dev = state.ekf;
    const bool live = dev && dev->cov == cov.handle() && dev->h == &h && state.ekf_generation == dev->generation;
    if (!live) {
        if (state.rank() != 0)
            throw std::invalid_argument("fekf_step: a state with W must be the latest state of its device filter");
        if (state.alpha != 0.0 || state.step != 0)
            throw std::invalid_argument("fekf_step: a fresh device filter starts from zero_start (alpha = 0)");
        dev = std::make_shared<detail::EkfDevice>();
        detail::check(fkb_ekf_create(cov.handle(), h.m, h.n, h.rowptr.data(), h.col.empty() ? nullptr : h.col.data(),
                                     h.val.empty() ? nullptr : h.val.data(), &dev->e));
        dev->cov = cov.handle();
        dev->h = &h;
        detail::check(fkb_ekf_reset(dev->e, state.mean.data()));
    }
    detail::check(fkb_ekf_step(dev->e, y.data(), y.size(), sigma2, transform.alpha, opts.k_rank, opts.oversampling,
                               opts.trunc_tol, opts.relinearizations, opts.seed));
    LowRankState next;
    int rank = 0;
    detail::check(fkb_ekf_state(dev->e, &next.alpha, &next.step, &rank));
    next.d = Vector(rank);
    next.mean = Vector(state.mean.size());
    detail::check(fkb_ekf_read(dev->e, next.mean.data(), rank ? next.d.data() : nullptr, nullptr, nullptr));
    next.ekf = dev;
    next.ekf_generation = ++dev->generation;
    return next;
}

// ---- enkf.hpp:15-94 — the ensemble lives on the device, bound to Γ and H at enkf_init
class Ensemble {
public:
    Ensemble(const CovarianceOperator& cov, const SparseRowMatrix& h, Index n_members) : n_(cov.size()) {
        fkb_enkf* e = nullptr;
        detail::check(fkb_enkf_init(cov.handle(), h.m, h.n, h.rowptr.data(), h.col.empty() ? nullptr : h.col.data(),
                                    h.val.empty() ? nullptr : h.val.data(), int(n_members), &e));
        e_.reset(e);
        ne_ = n_members;
        cov_ = cov.handle();
        h_ = &h;
    }
    Index size() const { return ne_; }
    Vector mean() const {  // Ensemble::mean (:20)
        Vector m(n_);
        detail::check(fkb_enkf_mean(e_.get(), m.data()));
        return m;
    }
    Matrix members() const {  // n × N_e
        Matrix x(n_, ne_);
        detail::check(fkb_enkf_members(e_.get(), x.data()));
        return x;
    }
    fkb_enkf* handle() const { return e_.get(); }
    const void* cov_ = nullptr;
    const SparseRowMatrix* h_ = nullptr;

private:
    struct Del {
        void operator()(fkb_enkf* p) const { fkb_enkf_destroy(p); }
    };
    Index n_ = 0, ne_ = 0;
    std::unique_ptr<fkb_enkf, Del> e_;
};
// enkf_init (:30-34) — takes Γ and H so the members can stay on the device
inline Ensemble enkf_init(const CovarianceOperator& cov, const SparseRowMatrix& h, Index n_members) {
    return Ensemble(cov, h, n_members);
}
// enkf_step (:49-94), advancing the device ensemble in place and returning it
inline Ensemble& enkf_step(Ensemble& ens, const SparseRowMatrix& h, const Vector& y, const CovarianceOperator& cov,
                           double sigma2, std::uint64_t seed) {
    if (ens.cov_ != cov.handle() || ens.h_ != &h)
        throw std::invalid_argument("enkf_step: the ensemble is bound to another operator pair");
    detail::check(fkb_enkf_step(ens.handle(), y.data(), y.size(), sigma2, seed));
    return ens;
}

// ---- field_io.hpp: FKF1 field and FKS1 state snapshots (little-endian, host I/O)
static_assert(std::endian::native == std::endian::little,
              "field formats are little-endian; big-endian hosts are unsupported");  // field_io.hpp:15-16
struct Field {
    int nx = 0;
    int ny = 0;
    Vector data;
};

namespace detail {
inline std::FILE* open_file(const std::string& path, const char* mode) {
    std::FILE* f = std::fopen(path.c_str(), mode);
    if (!f) throw std::runtime_error(std::string(mode[0] == 'w' ? "cannot open for writing: " : "cannot open for reading: ") + path);
    return f;
}
struct FileCloser {
    std::FILE* f;
    ~FileCloser() {
        if (f) std::fclose(f);
    }
};
inline void write_bytes(std::FILE* f, const void* p, size_t n, const std::string& path) {
    if (n && std::fwrite(p, 1, n, f) != n) throw std::runtime_error("write failed: " + path);
}
inline void read_bytes(std::FILE* f, void* p, size_t n, const std::string& path) {
    if (n && std::fread(p, 1, n, f) != n) throw std::runtime_error("truncated file: " + path);
}
}  // namespace detail

// write_field field_io.hpp:66-79: "FKF1", uint32 nx, uint32 ny, nx·ny float64 (x-major)
inline void write_field(const std::string& path, int nx, int ny, const Vector& data) {
    if (data.size() != static_cast<Index>(nx) * ny)
        throw std::invalid_argument("write_field: data length does not match " + std::to_string(nx) + "x" +
                                    std::to_string(ny));
    detail::FileCloser c{detail::open_file(path, "wb")};
    const std::uint32_t dims[2] = {std::uint32_t(nx), std::uint32_t(ny)};
    detail::write_bytes(c.f, "FKF1", 4, path);
    detail::write_bytes(c.f, dims, sizeof dims, path);
    detail::write_bytes(c.f, data.data(), sizeof(double) * size_t(data.size()), path);
}

// read_field field_io.hpp:81-95
inline Field read_field(const std::string& path) {
    detail::FileCloser c{detail::open_file(path, "rb")};
    char magic[4] = {0, 0, 0, 0};
    if (std::fread(magic, 1, 4, c.f) != 4 || std::string(magic, 4) != "FKF1")
        throw std::runtime_error("not a FKF1 field file: " + path);
    std::uint32_t dims[2];
    detail::read_bytes(c.f, dims, sizeof dims, path);
    Field f;
    f.nx = int(dims[0]);
    f.ny = int(dims[1]);
    if (f.nx < 1 || f.ny < 1 || static_cast<long long>(f.nx) * f.ny > (1LL << 31))
        throw std::runtime_error("implausible field dimensions in " + path);
    f.data = Vector(Index(f.nx) * f.ny);
    detail::read_bytes(c.f, f.data.data(), sizeof(double) * size_t(f.data.size()), path);
    return f;
}

// write_state field_io.hpp:100-113: "FKS1", uint32 n, uint32 r, uint32 step, float64 α,
// mean (n), D (r), W (n·r column-major).  W is fetched from the device only here.
inline void write_state(const std::string& path, const LowRankState& state, const Matrix& w) {
    if (w.rows() != state.mean.size() || w.cols() != state.rank())
        throw std::invalid_argument("write_state: W does not match the state");
    detail::FileCloser c{detail::open_file(path, "wb")};
    const std::uint32_t hdr[3] = {std::uint32_t(state.mean.size()), std::uint32_t(state.rank()),
                                  std::uint32_t(state.step)};
    detail::write_bytes(c.f, "FKS1", 4, path);
    detail::write_bytes(c.f, hdr, sizeof hdr, path);
    detail::write_bytes(c.f, &state.alpha, sizeof(double), path);
    detail::write_bytes(c.f, state.mean.data(), sizeof(double) * size_t(state.mean.size()), path);
    detail::write_bytes(c.f, state.d.data(), sizeof(double) * size_t(state.d.size()), path);
    detail::write_bytes(c.f, w.data(), sizeof(double) * w.a.size(), path);
}
// extended-filter states (and states read from disk) carry their own W
inline void write_state(const std::string& path, const LowRankState& state) { write_state(path, state, state.w()); }
// constant-H states: W = U of the context (fast_filter.hpp:113); a rank-0 state has no W
inline void write_state(const std::string& path, const LowRankState& state, const FkfContext& ctx) {
    write_state(path, state, state.rank() ? ctx.u() : Matrix(state.mean.size(), 0));
}

// read_state field_io.hpp:115-135
inline LowRankState read_state(const std::string& path) {
    detail::FileCloser c{detail::open_file(path, "rb")};
    char magic[4] = {0, 0, 0, 0};
    if (std::fread(magic, 1, 4, c.f) != 4 || std::string(magic, 4) != "FKS1")
        throw std::runtime_error("not a FKS1 state file: " + path);
    std::uint32_t hdr[3];
    detail::read_bytes(c.f, hdr, sizeof hdr, path);
    LowRankState s;
    s.step = int(hdr[2]);
    detail::read_bytes(c.f, &s.alpha, sizeof(double), path);
    s.mean = Vector(Index(hdr[0]));
    s.d = Vector(Index(hdr[1]));
    s.w_host = Matrix(Index(hdr[0]), Index(hdr[1]));
    detail::read_bytes(c.f, s.mean.data(), sizeof(double) * size_t(hdr[0]), path);
    detail::read_bytes(c.f, s.d.data(), sizeof(double) * size_t(hdr[1]), path);
    detail::read_bytes(c.f, s.w_host.data(), sizeof(double) * s.w_host.a.size(), path);
    return s;
}

// trace_criterion / relative_entropy of an extended-filter state (uq.hpp:25-53), W on the device
inline double trace_criterion(const LowRankState& state, const CovarianceOperator&) {
    if (!state.ekf) throw std::invalid_argument("trace_criterion: use the FkfContext overload for constant-H states");
    double t = 0.0;
    detail::check(fkb_ekf_uq(state.ekf->e, &t, nullptr));
    return t;
}
inline double relative_entropy(const LowRankState& state) {
    if (!state.ekf) throw std::invalid_argument("relative_entropy: use the FkfContext overload for constant-H states");
    double h = 0.0;
    detail::check(fkb_ekf_uq(state.ekf->e, nullptr, &h));
    return h;
}

}  // namespace fastkf
