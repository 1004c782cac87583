// capi.cu — extern "C" boundary (include/fastkf_b200.h) over the device runtime.
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>

#include "../../include/fastkf_b200.h"
#include "eig.cuh"
#include "ekf.cuh"
#include "enkf.cuh"
#include "filter.cuh"
#include "host_linalg.h"

namespace fkb {
unsigned long long g_launches = 0;
int g_sync_check = std::getenv("FKB_SYNC_CHECK") ? std::atoi(std::getenv("FKB_SYNC_CHECK")) : 0;

__attribute__((noinline)) void sync_check(const char*) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        Dl_info info{};
        void* ra = __builtin_return_address(0);
        dladdr(ra, &info);
        const long off = long((char*)ra - (char*)info.dli_fbase);
        throw CudaError(std::string("CUDA error ") + cudaGetErrorString(e) + " after launch #" +
                        std::to_string(g_launches) + " caller offset 0x" + [&] {
                            char b[32];
                            std::snprintf(b, sizeof b, "%lx", off);
                            return std::string(b);
                        }());
    }
}
}  // namespace fkb

// The operator is reference counted: every filter / ensemble / GHEP result built on it holds
// a reference, so fkb_cov_destroy before them only drops the caller's reference (the device
// objects run on the operator's stream and Γ-apply).
struct fkb_cov {
    int refs = 1;
    cudaStream_t stream = nullptr;
    std::unique_ptr<fkb::Cov> cov;
    ~fkb_cov() {
        if (stream) cudaStreamSynchronize(stream);
        cov.reset();
        if (stream) cudaStreamDestroy(stream);
    }
};
namespace {
void cov_release(fkb_cov* c) {
    if (c && --c->refs == 0) delete c;
}
// a reference to the operator held by a device object (released after the object's members)
struct CovRef {
    fkb_cov* c = nullptr;
    CovRef() = default;
    CovRef(const CovRef&) = delete;
    CovRef& operator=(fkb_cov* p) {
        cov_release(c);
        c = p;
        if (c) ++c->refs;
        return *this;
    }
    ~CovRef() { cov_release(c); }
    fkb_cov* operator->() const { return c; }
    explicit operator bool() const { return c != nullptr; }
};
}  // namespace
struct fkb_filter {
    CovRef owner;  // declared first: released after f
    std::unique_ptr<fkb::Filter> f;
};
struct fkb_ekf {
    CovRef owner;
    std::unique_ptr<fkb::Ekf> e;
};
struct fkb_enkf {
    CovRef owner;
    std::unique_ptr<fkb::Enkf> e;
};
struct fkb_ghep {  // a standalone randomized_ghep result (lowrank.hpp:132-213), device resident
    CovRef owner;
    fkb::DevCsr H, HT;
    fkb::GepDev g;
    double sigma2 = 0.0;
};

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& fn) {
    try {
        fn();
        return FKB_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return FKB_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return FKB_DOMAIN_ERROR;
    } catch (const fkb::CudaError& e) {
        g_err = e.what();
        return FKB_CUDA_ERROR;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FKB_RUNTIME_ERROR;
    }
}
void need(const void* p, const char* what) {
    if (!p) throw std::invalid_argument(std::string("null pointer: ") + what);
}
}  // namespace

extern "C" {

const char* fkb_last_error(void) { return g_err.c_str(); }
unsigned long long fkb_launch_count(void) { return fkb::g_launches; }
int fkb_version(void) { return 1; }
int fkb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int fkb_kernel_eval(int family, double theta, double length, double power, double nu, double alpha_scale, double r,
                    double* out) {
    return guarded([&] {
        fkb::KernelSpec s;
        s.family = family; s.theta = theta; s.length = length; s.power = power; s.nu = nu; s.alpha_scale = alpha_scale;
        *out = fkb::kernel_eval(s, r);
    });
}
int fkb_next_smooth(int n) { return fkb::next_smooth(n); }

int fkb_trace_ray(int nx, int ny, double lx, double ly, double sx, double sy, double rx, double ry, int cap,
                  long long* cells, double* lengths, int* count) {
    return guarded([&] {
        if (nx < 1 || ny < 1) throw std::invalid_argument("grid: nx and ny must be positive");
        *count = fkb::trace_ray_into(nx, ny, lx, ly, sx, sy, rx, ry, cap, cells, lengths);
    });
}

int fkb_build_H(int nx, int ny, double lx, double ly, int n_src, const double* src_xy, int n_rec,
                const double* rec_xy, int* rows, long long* nnz, int* rowptr, int* col, double* val, long long cap) {
    return guarded([&] {
        std::vector<int> rp, ci;
        std::vector<double> v;
        fkb::build_H(nx, ny, lx, ly, n_src, src_xy, n_rec, rec_xy, rp, ci, v);
        *rows = n_src * n_rec;
        *nnz = (long long)v.size();
        if (cap >= (long long)v.size()) {
            std::memcpy(rowptr, rp.data(), rp.size() * sizeof(int));
            std::memcpy(col, ci.data(), ci.size() * sizeof(int));
            std::memcpy(val, v.data(), v.size() * sizeof(double));
        }
    });
}

int fkb_sym_eig(int n, const double* A, double* w, double* Z) {
    return guarded([&] { fkb::sym_eig_small(n, A, w, Z); });
}
int fkb_sym_eig_device(int n, const double* A, double* w, double* Z, int* sweeps) {
    return guarded([&] {
        if (n < 0) throw std::invalid_argument("sym_eig: negative size");
        if (n == 0) return;
        cudaStream_t s = nullptr;
        FKB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        struct Guard { cudaStream_t s; ~Guard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } g{s};
        fkb::DBuf<double> Ad(size_t(n) * n), th{size_t(n)}, V(size_t(n) * n);
        FKB_CUDA(cudaMemcpyAsync(Ad.p, A, sizeof(double) * size_t(n) * n, cudaMemcpyHostToDevice, s));
        const int sw = fkb::sym_eig_sorted_device(n, Ad.p, n, th.p, V.p, s);
        if (sweeps) *sweeps = sw;
        FKB_CUDA(cudaMemcpyAsync(w, th.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaMemcpyAsync(Z, V.p, sizeof(double) * size_t(n) * n, cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaStreamSynchronize(s));
    });
}

int fkb_cov_create(int nx, int ny, double lx, double ly, int family, double theta, double length, double power,
                   double nu, double alpha_scale, fkb_cov** out) {
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        auto h = std::make_unique<fkb_cov>();
        // the operator's stream carries the filter step's main chain: highest priority, so its
        // CTAs are dispatched ahead of the step's low-priority side branch (the U pass)
        int lo = 0, hi = 0;
        FKB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        FKB_CUDA(cudaStreamCreateWithPriority(&h->stream, cudaStreamNonBlocking, hi));
        fkb::KernelSpec s;
        s.family = family; s.theta = theta; s.length = length; s.power = power; s.nu = nu; s.alpha_scale = alpha_scale;
        h->cov = std::make_unique<fkb::Cov>(nx, ny, lx, ly, s, h->stream);
        *out = h.release();
    });
}
void fkb_cov_destroy(fkb_cov* c) { cov_release(c); }
int fkb_cov_dims(const fkb_cov* c, int* mx, int* my) {
    return guarded([&] {
        need(c, "cov");
        *mx = c->cov->mx;
        *my = c->cov->my;
    });
}
int fkb_cov_spectrum(fkb_cov* c, double* out) {
    return guarded([&] {
        need(c, "cov");
        auto v = c->cov->spectrum_host();
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}
int fkb_cov_apply_device(fkb_cov* c, const double* dX, long long ldx, int ncols, double* dY, long long ldy) {
    return guarded([&] {
        need(c, "cov");
        if (ncols < 0 || ldx < c->cov->size() || ldy < c->cov->size())
            throw std::invalid_argument("cov_apply: expected vector of length " + std::to_string(c->cov->size()));
        c->cov->apply(dX, ldx, ncols, dY, ldy);
    });
}
int fkb_cov_apply(fkb_cov* c, const double* X, long long ldx, int ncols, double* Y, long long ldy) {
    return guarded([&] {
        need(c, "cov");
        const long long n = c->cov->size();
        if (ncols < 0 || ldx < n || ldy < n)
            throw std::invalid_argument("cov_apply: expected vector of length " + std::to_string(n));
        if (ncols == 0) return;
        fkb::DBuf<double> d(size_t(n) * ncols);
        cudaStream_t s = c->stream;
        for (int j = 0; j < ncols; ++j)
            FKB_CUDA(cudaMemcpyAsync(d.p + (long long)j * n, X + (long long)j * ldx, n * sizeof(double),
                                     cudaMemcpyHostToDevice, s));
        c->cov->apply(d.p, n, ncols, d.p, n);
        for (int j = 0; j < ncols; ++j)
            FKB_CUDA(cudaMemcpyAsync(Y + (long long)j * ldy, d.p + (long long)j * n, n * sizeof(double),
                                     cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaStreamSynchronize(s));
    });
}
int fkb_cov_sample_pair(fkb_cov* c, uint64_t seed, uint64_t stream, double* a, double* b) {
    return guarded([&] {
        need(c, "cov");
        const long long n = c->cov->size();
        fkb::DBuf<double> d(size_t(2 * n));
        c->cov->sample_pair(seed, stream, d.p, d.p + n);
        FKB_CUDA(cudaMemcpyAsync(a, d.p, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        FKB_CUDA(cudaMemcpyAsync(b, d.p + n, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        FKB_CUDA(cudaStreamSynchronize(c->stream));
    });
}
long long fkb_cov_apply_count(const fkb_cov* c) { return c ? c->cov->applies : 0; }
void* fkb_cov_stream(fkb_cov* c) { return c ? (void*)c->stream : nullptr; }

int fkb_gaussian_matrix(long long rows, int cols, uint64_t seed, uint64_t base_stream, double* out) {
    return guarded([&] {
        if (rows < 0 || cols < 0) throw std::invalid_argument("gaussian_matrix: negative size");
        fkb::DBuf<double> d(size_t(rows) * cols);
        fkb::gaussian_matrix(rows, cols, seed, base_stream, d.p, rows, nullptr);
        FKB_CUDA(cudaMemcpy(out, d.p, d.bytes(), cudaMemcpyDeviceToHost));
    });
}

int fkb_fkf_init(fkb_cov* c, int m, int h_cols, const int* rowptr, const int* col, const double* val, double sigma2,
                 long long k_rank, long long p_oversample, uint64_t seed, fkb_filter** out) {
    return guarded([&] {
        need(c, "cov");
        need(out, "out");
        need(rowptr, "rowptr");
        *out = nullptr;
        auto h = std::make_unique<fkb_filter>();
        h->owner = c;
        h->f = std::make_unique<fkb::Filter>(c->cov.get(), m, h_cols, rowptr, col, val, sigma2, k_rank, p_oversample,
                                             seed);
        *out = h.release();
    });
}
void fkb_filter_destroy(fkb_filter* f) { delete f; }
int fkb_filter_rank(const fkb_filter* f, int* rank, int* kept_cols) {
    return guarded([&] {
        need(f, "filter");
        if (rank) *rank = f->f->r;
        if (kept_cols) *kept_cols = f->f->kept_cols;
    });
}
int fkb_filter_ghep_residual(fkb_filter* f, double* out) {
    return guarded([&] {
        need(f, "filter");
        const auto res = f->f->ghep_residual();
        if (!res.empty()) std::memcpy(out, res.data(), res.size() * sizeof(double));
    });
}
int fkb_filter_lambda(fkb_filter* f, double* out) {
    return guarded([&] {
        need(f, "filter");
        std::memcpy(out, f->f->lambda_h.data(), f->f->lambda_h.size() * sizeof(double));
    });
}
int fkb_filter_get(fkb_filter* f, int which, double* out) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        const double* src = nullptr;
        size_t count = 0;
        switch (which) {
            case 0: src = F.U.p; count = size_t(F.n) * F.r; break;
            case 1: src = F.Ubar.p; count = size_t(F.n) * F.r; break;
            case 2: src = F.G.p; count = size_t(F.m) * F.m; break;
            case 3: src = F.B.p; count = size_t(F.m) * F.r; break;
            case 4: src = F.colsq.p; count = size_t(F.r); break;
            default: throw std::invalid_argument("filter_get: unknown product");
        }
        if (count) {
            FKB_CUDA(cudaMemcpyAsync(out, src, count * sizeof(double), cudaMemcpyDeviceToHost, F.s));
            FKB_CUDA(cudaStreamSynchronize(F.s));
        }
    });
}
int fkb_fkf_step(fkb_filter* f, const double* y, long long ylen) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (ylen != F.m)
            throw std::invalid_argument("fkf_step: observation length " + std::to_string(ylen) + " does not match " +
                                        std::to_string(F.m) + " measurements");
        F.set_step_uq(false);
        F.step_host(y);
    });
}
int fkb_fkf_step_state(fkb_filter* f, const double* y, long long ylen, double* alpha, double* d, double* mean) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (ylen != F.m)
            throw std::invalid_argument("fkf_step: observation length " + std::to_string(ylen) + " does not match " +
                                        std::to_string(F.m) + " measurements");
        F.set_step_uq(false);
        F.step_host_state(y, d, mean);
        if (alpha) *alpha = F.alpha;
    });
}
int fkb_fkf_run(fkb_filter* f, const double* ys, int nsteps, long long ldy, double* alphas, double* d, long long ldd,
                double* mean, long long ldm) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (nsteps < 0) throw std::invalid_argument("fkf_run: negative step count");
        if (nsteps > 0) need(ys, "ys");
        if (ldy < F.m || (d && ldd < F.r) || (mean && ldm < F.n))
            throw std::invalid_argument("fkf_run: leading dimension smaller than the vector length");
        F.run_host(ys, nsteps, ldy, alphas, d, ldd, mean, ldm);
    });
}
int fkb_fkf_run_uq(fkb_filter* f, const double* ys, int nsteps, long long ldy, uint64_t seed, int count, double* x,
                   double* var, double* alphas, double* d, long long ldd, double* mean, long long ldm) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (nsteps < 0) throw std::invalid_argument("fkf_run: negative step count");
        if (count < 0 || count > 8) throw std::invalid_argument("fkf_run: realization count must be in [0, 8]");
        if (nsteps > 0) need(ys, "ys");
        if (ldy < F.m || (d && ldd < F.r) || (mean && ldm < F.n))
            throw std::invalid_argument("fkf_run: leading dimension smaller than the vector length");
        if (F.r == 0) throw std::invalid_argument("fkf_run: the fused UQ batch needs a rank > 0 state");
        F.run_host(ys, nsteps, ldy, alphas, d, ldd, mean, ldm, count, seed, x, var);
    });
}
int fkb_fkf_step_device(fkb_filter* f, const double* d_y) {
    return guarded([&] {
        need(f, "filter");
        f->f->set_step_uq(false);
        f->f->step(d_y);
    });
}
int fkb_fkf_steps_async(fkb_filter* f, const double* d_ys, int nsteps, long long ldy) {
    return guarded([&] {
        need(f, "filter");
        f->f->set_step_uq(false);
        f->f->steps_async(d_ys, nsteps, ldy);
    });
}
int fkb_fkf_step_uq_device(fkb_filter* f, const double* d_y, uint64_t seed, int count, double* d_x, double* d_var) {
    return guarded([&] {
        need(f, "filter");
        f->f->step_uq(d_y, seed, count, d_x, d_var);
    });
}
int fkb_fkf_step_uq(fkb_filter* f, const double* y, long long ylen, uint64_t seed, int count, double* x, double* var,
                    double* alpha, double* d, double* mean) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (ylen != F.m)
            throw std::invalid_argument("fkf_step: observation length " + std::to_string(ylen) + " does not match " +
                                        std::to_string(F.m) + " measurements");
        F.step_uq_host(y, seed, count, x, var, d, mean);
        if (alpha) *alpha = F.alpha;
    });
}
int fkb_fkf_sync(fkb_filter* f, int nsteps) {
    return guarded([&] {
        need(f, "filter");
        f->f->finish_async(nsteps);
    });
}
int fkb_filter_state(fkb_filter* f, double* alpha, int* step, int* rank, double* d, double* mean) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (alpha) *alpha = F.alpha;
        if (step) *step = F.step_no;
        if (rank) *rank = F.state_rank;
        if (d && F.state_rank) FKB_CUDA(cudaMemcpyAsync(d, F.d.p, sizeof(double) * F.r, cudaMemcpyDeviceToHost, F.s));
        if (mean) FKB_CUDA(cudaMemcpyAsync(mean, F.mean.p, sizeof(double) * F.n, cudaMemcpyDeviceToHost, F.s));
        FKB_CUDA(cudaStreamSynchronize(F.s));
    });
}
int fkb_filter_set_state(fkb_filter* f, double alpha, int step, int rank, const double* d, const double* mean) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (rank != 0 && rank != F.r)  // fast_filter.hpp:92-95
            throw std::invalid_argument(
                "fkf_step: state rank does not match the eigendecomposition (constant-H regime requires W = U)");
        const double a2[2] = {alpha, alpha};
        FKB_CUDA(cudaMemsetAsync(F.info.p, 0, sizeof(int), F.s));  // a new state starts unflagged
        FKB_CUDA(cudaMemsetAsync(F.ready.p, 0, sizeof(double), F.s));  // no stale epoch for the new α
        FKB_CUDA(cudaMemcpyAsync(F.alpha_dev.p, a2, sizeof(a2), cudaMemcpyHostToDevice, F.s));
        if (rank) FKB_CUDA(cudaMemcpyAsync(F.d.p, d, sizeof(double) * F.r, cudaMemcpyHostToDevice, F.s));
        else FKB_CUDA(cudaMemsetAsync(F.d.p, 0, F.d.bytes(), F.s));
        if (mean) FKB_CUDA(cudaMemcpyAsync(F.mean.p, mean, sizeof(double) * F.n, cudaMemcpyHostToDevice, F.s));
        FKB_CUDA(cudaStreamSynchronize(F.s));
        F.alpha = alpha;
        F.step_no = step;
        F.state_rank = rank;
        F.k_valid = false;  // the precomputed capacitance belongs to the old (α, d)
        if (mean) F.hm_valid = false;  // the carried image H·mean too
    });
}
int fkb_filter_reset(fkb_filter* f) {
    return guarded([&] {
        need(f, "filter");
        f->f->reset();
    });
}
int fkb_filter_mean_device(fkb_filter* f, const double** d_mean) {
    return guarded([&] {
        need(f, "filter");
        *d_mean = f->f->mean.p;
    });
}

int fkb_variance_device(fkb_filter* f, double* d_out) {
    return guarded([&] {
        need(f, "filter");
        f->f->variance(d_out);
    });
}
int fkb_variance(fkb_filter* f, double* out) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        F.host_out.ensure(static_cast<size_t>(F.n));  // persistent staging (no per-call allocation)
        F.variance(F.host_out.p);
        FKB_CUDA(cudaMemcpyAsync(out, F.host_out.p, sizeof(double) * size_t(F.n), cudaMemcpyDeviceToHost, F.s));
        FKB_CUDA(cudaStreamSynchronize(F.s));
    });
}
int fkb_trace_criterion(fkb_filter* f, double* out) {
    return guarded([&] {
        need(f, "filter");
        *out = f->f->trace_criterion();
    });
}
int fkb_relative_entropy(fkb_filter* f, double* out) {
    return guarded([&] {
        need(f, "filter");
        *out = f->f->relative_entropy();
    });
}
int fkb_realizations_device(fkb_filter* f, uint64_t seed, int count, double* d_out, double* d_var) {
    return guarded([&] {
        need(f, "filter");
        f->f->realizations(seed, count, d_out, d_var);
    });
}
int fkb_realizations(fkb_filter* f, uint64_t seed, int count, double* out) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (count < 0 || count > 8) throw std::invalid_argument("realizations: count must lie in [0, 8]");
        if (count == 0) return;
        F.host_out.ensure(size_t(F.n) * count);
        F.realizations(seed, count, F.host_out.p, nullptr);
        FKB_CUDA(cudaMemcpyAsync(out, F.host_out.p, sizeof(double) * size_t(F.n) * count, cudaMemcpyDeviceToHost, F.s));
        FKB_CUDA(cudaStreamSynchronize(F.s));
    });
}
int fkb_realization_at(fkb_filter* f, uint64_t seed, uint64_t draw, double* out) {
    return guarded([&] {
        need(f, "filter");
        need(out, "out");
        auto& F = *f->f;
        F.host_out.ensure(size_t(F.n));
        F.realization_at(seed, draw, F.host_out.p);
        FKB_CUDA(cudaMemcpyAsync(out, F.host_out.p, sizeof(double) * size_t(F.n), cudaMemcpyDeviceToHost, F.s));
        FKB_CUDA(cudaStreamSynchronize(F.s));
    });
}
int fkb_lowrank_uq(fkb_cov* c, long long n, int r, double alpha, const double* d, const double* w, long long ldw,
                   double* var, double* colsq) {
    return guarded([&] {
        need(c, "cov");
        auto& C = *c->cov;
        if (n != C.size()) throw std::invalid_argument("variance: state does not match operator size");  // uq.hpp:17-18
        if (r < 0 || ldw < n) throw std::invalid_argument("lowrank_uq: bad W dimensions");
        if (r) { need(d, "d"); need(w, "w"); }
        cudaStream_t s = C.stream;
        fkb::DBuf<double> dW{size_t(n) * std::max(r, 1)}, dd{size_t(std::max(r, 1))}, da{1}, dv{size_t(n)},
            dc{size_t(std::max(r, 1))}, scratch;
        if (r) {
            FKB_CUDA(cudaMemcpy2DAsync(dW.p, sizeof(double) * size_t(n), w, sizeof(double) * size_t(ldw),
                                       sizeof(double) * size_t(n), size_t(r), cudaMemcpyHostToDevice, s));
            FKB_CUDA(cudaMemcpyAsync(dd.p, d, sizeof(double) * size_t(r), cudaMemcpyHostToDevice, s));
        }
        FKB_CUDA(cudaMemcpyAsync(da.p, &alpha, sizeof(double), cudaMemcpyHostToDevice, s));
        fkb::lowrank_uq(&C, n, r, da.p, dd.p, dW.p, nullptr, nullptr, 0, 0, 0, nullptr, var ? dv.p : nullptr,
                        (colsq && r) ? dc.p : nullptr, scratch);
        if (var) FKB_CUDA(cudaMemcpyAsync(var, dv.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
        if (colsq && r) FKB_CUDA(cudaMemcpyAsync(colsq, dc.p, sizeof(double) * size_t(r), cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaStreamSynchronize(s));
    });
}
int fkb_dense_product(int which, long long n, int p, int q, const double* dA, const double* dB, double* dC,
                      void* stream) {
    return guarded([&] {
        if (n < 0 || p < 0 || q < 0) throw std::invalid_argument("dense_product: negative size");
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        static fkb::DBuf<double> ws;
        if (which == 0) fkb::gram_tn(n, p, q, dA, dB, dC, ws, s);
        else if (which == 1) fkb::tall_times_small(n, p, q, dA, dB, dC, s);
        else if (which == 2) {  // symmetric Gram AᵀA (n×p A, both triangles): the capacitance kernel
            if (q != p) throw std::invalid_argument("dense_product: the symmetric Gram needs q == p");
            fkb::GemmArgs g;
            g.M = p; g.N = p; g.K = int(n);
            g.A = dA; g.lda = n; g.transA = 1;
            g.B = dA; g.ldb = n;
            g.C = dC; g.ldc = p;
            fkb::gram_sym(g, s);
        } else throw std::invalid_argument("dense_product: which must be 0 (AᵀB), 1 (A·B) or 2 (AᵀA)");
    });
}
int fkb_ghep_run(fkb_cov* c, int m, int h_cols, const int* rowptr, const int* col, const double* val, double sigma2,
                 long long k, long long p, uint64_t seed, fkb_ghep** out) {
    return guarded([&] {
        need(c, "cov");
        need(out, "out");
        need(rowptr, "rowptr");
        *out = nullptr;
        auto& C = *c->cov;
        if ((long long)h_cols != C.size()) throw std::invalid_argument("randomized_ghep: H columns do not match state dimension");
        if (!(sigma2 > 0.0)) throw std::invalid_argument("randomized_ghep: sigma2 must be positive");
        for (int i = 0; i < m; ++i)
            for (int e = rowptr[i]; e < rowptr[i + 1]; ++e)
                if (col[e] < 0 || col[e] >= h_cols) throw std::invalid_argument("randomized_ghep: H column index out of range");
        auto g = std::make_unique<fkb_ghep>();
        g->owner = c;
        g->sigma2 = sigma2;
        fkb::upload_csr_pair(m, h_cols, rowptr, col, val, g->H, g->HT);
        fkb::DBuf<double> ws;
        fkb::randomized_ghep_device(&C, g->H, g->HT, sigma2, k, p, seed, ws, C.stream, g->g);
        g->g.scratch.clear();  // the sketch temporaries are not needed after the call
        *out = g.release();
    });
}
void fkb_ghep_destroy(fkb_ghep* g) {
    if (!g) return;
    if (g->owner && g->owner->stream) cudaStreamSynchronize(g->owner->stream);
    delete g;
}
int fkb_ghep_info(const fkb_ghep* g, int* rank, int* kept_cols) {
    return guarded([&] {
        need(g, "ghep");
        if (rank) *rank = g->g.r;
        if (kept_cols) *kept_cols = g->g.kept_cols;
    });
}
int fkb_ghep_get(fkb_ghep* g, int which, double* out) {
    return guarded([&] {
        need(g, "ghep");
        need(out, "out");
        const long long n = g->owner->cov->size();
        const int r = g->g.r;
        cudaStream_t s = g->owner->stream;
        if (which == 0) {
            std::copy(g->g.lambda_h.begin(), g->g.lambda_h.end(), out);
            return;
        }
        const double* src = which == 1 ? g->g.U.p : which == 2 ? g->g.Ubar.p : nullptr;
        if (!src && r) throw std::invalid_argument("ghep_get: unknown product");
        if (r) FKB_CUDA(cudaMemcpyAsync(out, src, sizeof(double) * size_t(n) * r, cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaStreamSynchronize(s));
    });
}
int fkb_realizations_with_variance(fkb_filter* f, uint64_t seed, int count, double* out, double* var) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (count < 0 || count > 8) throw std::invalid_argument("realizations: count must lie in [0, 8]");
        F.host_out.ensure(size_t(F.n) * (count + 1));
        double* xo = F.host_out.p + F.n;
        F.realizations(seed, count, xo, F.host_out.p);  // one pass over U for both
        if (var) FKB_CUDA(cudaMemcpyAsync(var, F.host_out.p, sizeof(double) * size_t(F.n), cudaMemcpyDeviceToHost, F.s));
        if (count && out)
            FKB_CUDA(cudaMemcpyAsync(out, xo, sizeof(double) * size_t(F.n) * count, cudaMemcpyDeviceToHost, F.s));
        FKB_CUDA(cudaStreamSynchronize(F.s));
    });
}

int fkb_filter_spmm(fkb_filter* f, int trans, const double* dX, long long ldx, int ncols, double* dY, long long ldy) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        fkb::spmm(trans ? F.HT : F.H, dX, ldx, ncols, dY, ldy, 1.0, 0.0, F.s);
    });
}
int fkb_filter_spmm_rm(fkb_filter* f, int trans, const double* dX, int ncols, double* dY) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (ncols < 0) throw std::invalid_argument("spmm: negative column count");
        fkb::spmm_rm(trans ? F.HT : F.H, dX, ncols, ncols, dY, ncols, 1.0, F.s);
    });
}
void* fkb_filter_stream(fkb_filter* f) { return f ? (void*)f->f->s : nullptr; }
int fkb_filter_set_solver(fkb_filter* f, int mode) {
    return guarded([&] {
        need(f, "filter");
        f->f->set_solver(mode);
    });
}
int fkb_filter_eig_sweeps(fkb_filter* f) { return f ? f->f->eig_sweeps : 0; }
int fkb_filter_set_pcg_maxit(fkb_filter* f, int maxit) {
    return guarded([&] {
        need(f, "filter");
        if (maxit < 0) throw std::invalid_argument("pcg: maxit must be nonnegative");
        auto& F = *f->f;
        F.pcg_maxit = maxit;
        F.drop_graphs();  // the cap is baked into the captured step
    });
}
int fkb_filter_pcg_stamps(fkb_filter* f, unsigned long long* out) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (!F.pcg_ts.p) throw std::invalid_argument("PCG stamps need FKB_PCG_STAMPS=1 at fkf_init");
        FKB_CUDA(cudaMemcpyAsync(out, F.pcg_ts.p, 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, F.s));
        FKB_CUDA(cudaStreamSynchronize(F.s));
    });
}

int fkb_filter_cap_stats(fkb_filter* f, int* iterations, int* fallback) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        double it = 0.0;
        int fb = 0;
        if (F.r > 0 && F.solver == 1) {
            FKB_CUDA(cudaMemcpyAsync(&it, F.pcgwork.p + F.r, sizeof(double), cudaMemcpyDeviceToHost, F.s));
            FKB_CUDA(cudaMemcpyAsync(&fb, F.pcgflag.p, sizeof(int), cudaMemcpyDeviceToHost, F.s));
            FKB_CUDA(cudaStreamSynchronize(F.s));
        }
        if (iterations) *iterations = int(it);
        if (fallback) *fallback = fb;
    });
}
int fkb_filter_phase_times(fkb_filter* f, int reps, double* ms, char* names, int names_len, int* nphases) {
    return guarded([&] {
        need(f, "filter");
        auto v = f->f->phase_times(reps);
        std::string joined;
        for (size_t i = 0; i < v.size(); ++i) {
            if (ms) ms[i] = v[i].second;
            if (i) joined += ",";
            joined += v[i].first;
        }
        if (names && names_len > 0) {
            std::strncpy(names, joined.c_str(), size_t(names_len) - 1);
            names[names_len - 1] = 0;
        }
        *nphases = int(v.size());
    });
}
int fkb_filter_graph_timing(fkb_filter* f, int on) {
    return guarded([&] {
        need(f, "filter");
        f->f->set_graph_timing(on != 0);
    });
}
int fkb_filter_graph_phase_times(fkb_filter* f, double* ms, char* names, int names_len, int* nphases) {
    return guarded([&] {
        need(f, "filter");
        auto v = f->f->graph_phase_times();
        std::string joined;
        for (size_t i = 0; i < v.size(); ++i) {
            if (ms) ms[i] = v[i].second;
            if (i) joined += ",";
            joined += v[i].first;
        }
        if (names && names_len > 0) {
            std::strncpy(names, joined.c_str(), size_t(names_len) - 1);
            names[names_len - 1] = 0;
        }
        *nphases = int(v.size());
    });
}
int fkb_filter_get_eig(fkb_filter* f, double* theta, double* P) {
    return guarded([&] {
        need(f, "filter");
        auto& F = *f->f;
        if (theta) FKB_CUDA(cudaMemcpyAsync(theta, F.theta.p, sizeof(double) * F.m, cudaMemcpyDeviceToHost, F.s));
        if (P) FKB_CUDA(cudaMemcpyAsync(P, F.P.p, sizeof(double) * size_t(F.m) * F.m, cudaMemcpyDeviceToHost, F.s));
        FKB_CUDA(cudaStreamSynchronize(F.s));
    });
}
int fkb_filter_launches_per_step(fkb_filter* f) { return f ? f->f->launches_per_step : 0; }

int fkb_dmalloc(void** p, size_t bytes) { return guarded([&] { FKB_CUDA(cudaMalloc(p, bytes)); }); }
int fkb_dfree(void* p) { return guarded([&] { FKB_CUDA(cudaFree(p)); }); }
// The library's streams are non-blocking (they do not order against the legacy default
// stream), so these plumbing copies synchronize the device first: a copy never races a kernel
// still writing or reading the buffer on a context stream.
int fkb_h2d(void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        FKB_CUDA(cudaDeviceSynchronize());
        FKB_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
        // a pageable-source cudaMemcpy may return before its DMA lands; kernels on the
        // library's non-blocking streams are not ordered after it, so wait here
        FKB_CUDA(cudaDeviceSynchronize());
    });
}
int fkb_d2h(void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        FKB_CUDA(cudaDeviceSynchronize());
        FKB_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    });
}
int fkb_dsync(void) { return guarded([&] { FKB_CUDA(cudaDeviceSynchronize()); }); }


int fkb_ekf_create(fkb_cov* c, int m, int h_cols, const int* rowptr, const int* col, const double* val,
                   fkb_ekf** out) {
    return guarded([&] {
        need(c, "cov");
        need(out, "out");
        need(rowptr, "rowptr");
        *out = nullptr;
        auto h = std::make_unique<fkb_ekf>();
        h->owner = c;
        h->e = std::make_unique<fkb::Ekf>(c->cov.get(), m, h_cols, rowptr, col, val);
        *out = h.release();
    });
}
void fkb_ekf_destroy(fkb_ekf* e) {
    if (e && e->e && e->e->s) cudaStreamSynchronize(e->e->s);
    delete e;
}
int fkb_ekf_reset(fkb_ekf* e, const double* mean0) {
    return guarded([&] {
        need(e, "ekf");
        need(mean0, "mean0");
        e->e->reset(mean0);
    });
}
int fkb_ekf_step(fkb_ekf* e, const double* y, long long ylen, double sigma2, double boxcox_alpha, long long k_rank,
                 long long oversampling, double trunc_tol, int relinearizations, uint64_t seed) {
    return guarded([&] {
        need(e, "ekf");
        if (ylen != e->e->m) throw std::invalid_argument("fekf_step: dimension mismatch");  // :145-147
        if (ylen) need(y, "y");
        fkb::EkfOptions o;
        o.k_rank = k_rank;
        o.oversampling = oversampling;
        o.trunc_tol = trunc_tol;
        o.relinearizations = relinearizations;
        o.seed = seed;
        e->e->step(y, sigma2, boxcox_alpha, o);
    });
}
int fkb_ekf_state(fkb_ekf* e, double* alpha, int* step, int* rank) {
    return guarded([&] {
        need(e, "ekf");
        if (alpha) *alpha = e->e->alpha;
        if (step) *step = e->e->step_no;
        if (rank) *rank = e->e->r;
    });
}
int fkb_ekf_read(fkb_ekf* e, double* mean, double* d, double* w, double* wbar) {
    return guarded([&] {
        need(e, "ekf");
        auto& E = *e->e;
        const size_t n = size_t(E.n), r = size_t(E.r);
        if (mean) FKB_CUDA(cudaMemcpyAsync(mean, E.mean.p, sizeof(double) * n, cudaMemcpyDeviceToHost, E.s));
        if (d && r) std::memcpy(d, E.d_h.data(), sizeof(double) * r);
        if (w && r) FKB_CUDA(cudaMemcpyAsync(w, E.W.p, sizeof(double) * n * r, cudaMemcpyDeviceToHost, E.s));
        if (wbar && r) FKB_CUDA(cudaMemcpyAsync(wbar, E.Wbar.p, sizeof(double) * n * r, cudaMemcpyDeviceToHost, E.s));
        FKB_CUDA(cudaStreamSynchronize(E.s));
    });
}
int fkb_ekf_uq(fkb_ekf* e, double* trace, double* entropy) {
    return guarded([&] {
        need(e, "ekf");
        double t = 0.0, h = 0.0;
        e->e->uq_scalars(t, h);
        if (trace) *trace = t;
        if (entropy) *entropy = h;
    });
}
int fkb_ekf_realizations(fkb_ekf* e, uint64_t seed, uint64_t first_draw, int count, double* out, double* var) {
    return guarded([&] {
        need(e, "ekf");
        auto& E = *e->e;
        if (count < 0 || count > 8) throw std::invalid_argument("realizations: count must lie in [0, 8]");
        fkb::DBuf<double> buf(size_t(E.n) * (count + 1));
        E.uq(seed, first_draw, count, buf.p + E.n, var ? buf.p : nullptr);
        if (var) FKB_CUDA(cudaMemcpyAsync(var, buf.p, sizeof(double) * size_t(E.n), cudaMemcpyDeviceToHost, E.s));
        if (count && out)
            FKB_CUDA(cudaMemcpyAsync(out, buf.p + E.n, sizeof(double) * size_t(E.n) * count, cudaMemcpyDeviceToHost, E.s));
        FKB_CUDA(cudaStreamSynchronize(E.s));
    });
}
int fkb_ekf_last(fkb_ekf* e, int* gep_rank, int* sweeps) {
    return guarded([&] {
        need(e, "ekf");
        if (gep_rank) *gep_rank = e->e->last_gep_rank;
        if (sweeps) *sweeps = e->e->last_relin;
    });
}


int fkb_enkf_init(fkb_cov* c, int m, int h_cols, const int* rowptr, const int* col, const double* val,
                  int n_members, fkb_enkf** out) {
    return guarded([&] {
        need(c, "cov");
        need(out, "out");
        need(rowptr, "rowptr");
        *out = nullptr;
        auto h = std::make_unique<fkb_enkf>();
        h->owner = c;
        h->e = std::make_unique<fkb::Enkf>(c->cov.get(), m, h_cols, rowptr, col, val, n_members);
        *out = h.release();
    });
}
void fkb_enkf_destroy(fkb_enkf* e) {
    if (e && e->e && e->e->s) cudaStreamSynchronize(e->e->s);
    delete e;
}
int fkb_enkf_step(fkb_enkf* e, const double* y, long long ylen, double sigma2, uint64_t seed) {
    return guarded([&] {
        need(e, "enkf");
        if (ylen != e->e->m) throw std::invalid_argument("enkf_step: dimension mismatch");  // enkf.hpp:53-54
        if (ylen) need(y, "y");
        e->e->step(y, sigma2, seed);
    });
}
int fkb_enkf_members(fkb_enkf* e, double* out) {
    return guarded([&] {
        need(e, "enkf");
        need(out, "out");
        auto& E = *e->e;
        FKB_CUDA(cudaMemcpyAsync(out, E.X.p, E.X.bytes(), cudaMemcpyDeviceToHost, E.s));
        FKB_CUDA(cudaStreamSynchronize(E.s));
    });
}
int fkb_enkf_set_members(fkb_enkf* e, const double* in) {
    return guarded([&] {
        need(e, "enkf");
        need(in, "in");
        auto& E = *e->e;
        FKB_CUDA(cudaMemcpyAsync(E.X.p, in, E.X.bytes(), cudaMemcpyHostToDevice, E.s));
        FKB_CUDA(cudaStreamSynchronize(E.s));
    });
}
int fkb_enkf_mean(fkb_enkf* e, double* out) {
    return guarded([&] {
        need(e, "enkf");
        need(out, "out");
        auto& E = *e->e;
        E.member_mean(E.mean.p);
        FKB_CUDA(cudaMemcpyAsync(out, E.mean.p, sizeof(double) * size_t(E.n), cudaMemcpyDeviceToHost, E.s));
        FKB_CUDA(cudaStreamSynchronize(E.s));
    });
}

}  // extern "C"
