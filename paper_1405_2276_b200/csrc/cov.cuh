// cov.cuh — Γ_sys on the device: FFT circulant embedding (reference covariance.hpp FFT mode).
#pragma once

#include "common.cuh"
#include "fft.cuh"

namespace fkb {

struct KernelSpec {  // kernel.hpp:19-48
    int family = 0;  // 0 powered_exponential, 1 matern
    double theta = 1.0, length = 0.2, power = 1.0, nu = 0.5, alpha_scale = 0.0;
    void validate() const;
    double scale() const { return alpha_scale > 0.0 ? alpha_scale : 1.0 / length; }
};
double kernel_eval(const KernelSpec& s, double r);  // kernel.hpp:51-63
int next_smooth(int n);                             // covariance.hpp:35-43

// Epilogue of the single-vector inverse pass when it carries the filter step's mean update
// (fast_filter.hpp:114-116): y ← (y + (*coef)·Γx) − sub, gated on *gate; hout (device copy
// of the mapped host pointers, Filter::hostout): [0] new mean, [2] failure flag.
struct MeanUpd {
    const double* coef = nullptr;
    const int* gate = nullptr;
    const double* sub = nullptr;
    const unsigned long long* hout = nullptr;
    long long* ycnt = nullptr;  // incremented once per step (the host batch's observation row)
};

struct Cov {
    int nx = 0, ny = 0;
    double lx = 1.0, ly = 1.0;
    KernelSpec spec;
    int mx = 0, my = 0, nky = 0;  // nky = my/2 + 1 (Hermitian half along y)
    cudaStream_t stream = nullptr;
    FftLen fx, fy;
    FftLen fx8, fy8;  // radix ≤ 8 schedules (single-vector kernels), same twiddle tables
    DBuf<double2> twx, twy;
    DBuf<double2> twpx, twpy;  // per-pass twiddles of the compile-time schedules (FftLen::twp)
    DBuf<double> spec_half;  // [ky][kx], clipped ≥ 0 (covariance.hpp:295)
    DBuf<double> amp_full;   // √spectrum on the full torus, row-major mx×my (sampler :339)
    DBuf<double2> work;      // intermediate [col][ky][ix]
    DBuf<double2> swork;     // batched sampler intermediate [pair][ky][ix]
    int batch_cap = 0;
    long long applies = 0;

    Cov(int nx, int ny, double lx, double ly, const KernelSpec& spec, cudaStream_t s);
    long long size() const { return (long long)nx * ny; }
    long long M() const { return (long long)mx * my; }

    // Y = Γ X, X/Y column-major device blocks (covariance.hpp:101-115); Y may alias X.
    void apply(const double* dX, long long ldx, int ncols, double* dY, long long ldy);
    void apply1(const double* dx, double* dy);  // single vector (CTA-per-transform kernels)
    // the single-vector apply split at its last pass: forward rows + column pass into the work
    // buffer, then the inverse rows pass storing Γx into dy, or (upd.coef ≠ null) the filter's
    // mean update dy ← (dy + (*upd.coef)·Γx) − upd.sub unless *upd.gate (see MeanUpd)
    void apply1_fwd(const double* dx, int ncols = 1, long long ldx = 0);
    void apply1_inv(double* dy, const MeanUpd& upd, int ncols = 1, long long ldy = 0);
    // Two N(0,Γ) draws (covariance.hpp:332-353) into device vectors.
    void sample_pair(uint64_t seed, uint64_t stream_id, double* da, double* db);
    // X[:, j] += draw j of the pairs (seed, sid0 + j/2) (Re → even j, Im → odd j), j < ncols
    // (the EnKF forecast, enkf.hpp:67-72), batched over pairs.
    void sample_pairs_add(uint64_t seed, uint64_t sid0, double* X, long long ldx, int ncols);
    // Host copy of the full clipped spectrum (covariance.hpp:207-211), row-major mx×my.
    std::vector<double> spectrum_host() const;

  private:
    bool try_spectrum(double& worst);
    void setup_len(FftLen& L, DBuf<double2>& tw, int n);
    void setup_static_tw(FftLen& L, DBuf<double2>& tw, int n);
    void ensure_work(int ncols);
};

}  // namespace fkb
