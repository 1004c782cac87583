// cov.cu — K1: batched FP64 FFT circulant-embedding Γ·X on sm_100a.
//
// Reference: CovarianceOperator FFT mode, /root/reference/proj/include/fastkf/
// covariance.hpp:238-353.  The reference applies Γ one column at a time with
// two full mx×my complex FFTs (apply_fft :309-330).  Here a block of columns is
// transformed at once, and the zero padding is exploited:
//   pass A  rows:    real length-my rows ix < nx → Hermitian half (two rows per
//                    complex transform), stored transposed as W[col][ky][ix];
//   pass B  columns: per ky, zero-pad ix to mx, forward FFT, × spectrum,
//                    inverse FFT, keep ix < nx (in place in W);
//   pass C  rows:    Hermitian half → real rows, ×1/M, crop iy < ny.
// The intermediate W for a batch is sized to stay L2-resident.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <sstream>
#include <type_traits>

#include "cov.cuh"
#include "fft_device.cuh"
#include "rng_device.cuh"

namespace fkb {

static bool g_odd_ready = false;

static void init_odd_tables() {
    if (g_odd_ready) return;
    OddRadixTables t;
    for (int j = 0; j < 3; ++j) { t.c3[j] = double(cosl(2.0L * std::numbers::pi_v<long double> * j / 3)); t.s3[j] = double(sinl(2.0L * std::numbers::pi_v<long double> * j / 3)); }
    for (int j = 0; j < 5; ++j) { t.c5[j] = double(cosl(2.0L * std::numbers::pi_v<long double> * j / 5)); t.s5[j] = double(sinl(2.0L * std::numbers::pi_v<long double> * j / 5)); }
    for (int j = 0; j < 7; ++j) { t.c7[j] = double(cosl(2.0L * std::numbers::pi_v<long double> * j / 7)); t.s7[j] = double(sinl(2.0L * std::numbers::pi_v<long double> * j / 7)); }
    FKB_CUDA(cudaMemcpyToSymbol(c_odd, &t, sizeof(t)));
    g_odd_ready = true;
}

// --------------------------------------------------------------------------- host math
void KernelSpec::validate() const {  // kernel.hpp:27-43
    if (!(theta > 0.0)) throw std::invalid_argument("kernel: theta must be positive, got " + std::to_string(theta));
    if (!(length > 0.0)) throw std::invalid_argument("kernel: length must be positive, got " + std::to_string(length));
    if (family == 0) {
        if (!(power > 0.0) || power > 2.0)
            throw std::invalid_argument("kernel: power must lie in (0, 2], got " + std::to_string(power));
    } else if (!(nu > 0.0)) {
        throw std::invalid_argument("kernel: nu must be positive, got " + std::to_string(nu));
    }
}

double kernel_eval(const KernelSpec& s, double r) {  // kernel.hpp:51-63 (host: symbol only)
    s.validate();
    if (r < 0.0) throw std::invalid_argument("kernel: distance must be nonnegative");
    if (r == 0.0) return s.theta;
    if (s.family == 0) return s.theta * std::exp(-std::pow(r / s.length, s.power));
    const double arg = std::sqrt(2.0 * s.nu) * s.scale() * r;
    if (arg > 700.0) return 0.0;
    const double pref = std::exp((1.0 - s.nu) * std::numbers::ln2 - std::lgamma(s.nu));
    return s.theta * pref * std::pow(arg, s.nu) * std::cyl_bessel_k(s.nu, arg);
}

int next_smooth(int n) {  // covariance.hpp:35-43
    if (n <= 1) return 1;
    for (int m = n;; ++m) {
        int v = m;
        for (int f : {2, 3, 5, 7})
            while (v % f == 0) v /= f;
        if (v == 1) return m;
    }
}

// --------------------------------------------------------------------------- kernels
constexpr int kThreads = 256;

// Pass A: rows → Hermitian half along y.  Block = (row group, column).
// Each complex transform packs two real rows (two-for-one).  Rows ≥ nx_in are zero.
// Output W[col][ky][ix] for ix < nx_out (ld_w per column, ld_ky = nx_out).
__global__ void __launch_bounds__(kThreads) k_rows_fwd(const double* __restrict__ X, long long ldx, int nx_in,
                                                      int ny, int nx_out, FftLen fy, double2* __restrict__ W,
                                                      long long ldw, int pairs) {
    extern __shared__ double2 sm[];
    const int my = fy.n, nky = my / 2 + 1;
    double2* a = sm;
    double2* b = sm + pairs * my;
    const int ix0 = blockIdx.x * pairs * 2;
    const double* x = X + (long long)blockIdx.y * ldx;
    for (int e = threadIdx.x; e < pairs * my; e += blockDim.x) {
        const int t = e / my, iy = e - t * my;
        const int r0 = ix0 + 2 * t, r1 = r0 + 1;
        double v0 = 0.0, v1 = 0.0;
        if (iy < ny) {
            if (r0 < nx_in) v0 = x[(long long)r0 * ny + iy];
            if (r1 < nx_in) v1 = x[(long long)r1 * ny + iy];
        }
        a[e] = make_double2(v0, v1);
    }
    __syncthreads();
    const double2* z = fft_smem<-1>(a, b, fy, pairs);
    double2* w = W + (long long)blockIdx.y * ldw;
    const int rows = pairs * 2;
    for (int e = threadIdx.x; e < rows * nky; e += blockDim.x) {
        const int ky = e / rows, rl = e - ky * rows;
        const int ix = ix0 + rl;
        if (ix >= nx_out) continue;
        const int t = rl >> 1;
        const double2 p = z[t * my + ky];
        const double2 q = cconj(z[t * my + (ky == 0 ? 0 : my - ky)]);
        double2 o;
        if ((rl & 1) == 0) o = make_double2(0.5 * (p.x + q.x), 0.5 * (p.y + q.y));  // (Z + conj Z−)/2
        else o = make_double2(0.5 * (p.y - q.y), -0.5 * (p.x - q.x));              // (Z − conj Z−)/(2i)
        w[(long long)ky * nx_out + ix] = o;
    }
}

// Pass B: along x per ky column.  mode 0: zero-pad nx→mx, FFT, × spectrum, iFFT, keep nx.
// mode 1 (spectrum build): forward only over the full mx, write mx entries.
__global__ void __launch_bounds__(kThreads) k_cols(double2* __restrict__ W, long long ldw, int nx, FftLen fx,
                                                  int nky, const double* __restrict__ spec_half, int kt,
                                                  int mode) {
    extern __shared__ double2 sm[];
    const int mx = fx.n;
    double2* a = sm;
    double2* b = sm + kt * mx;
    const int ky0 = blockIdx.x * kt;
    double2* w = W + (long long)blockIdx.y * ldw;
    const int ld = (mode == 0) ? nx : mx;
    for (int e = threadIdx.x; e < kt * mx; e += blockDim.x) {
        const int t = e / mx, ix = e - t * mx;
        const int ky = ky0 + t;
        double2 v = make_double2(0.0, 0.0);
        if (ky < nky && ix < ld) v = w[(long long)ky * ld + ix];
        a[e] = v;
    }
    __syncthreads();
    double2* f = fft_smem<-1>(a, b, fx, kt);
    double2* g = (f == a) ? b : a;
    if (mode == 0) {
        for (int e = threadIdx.x; e < kt * mx; e += blockDim.x) {
            const int t = e / mx, kx = e - t * mx;
            const int ky = min(ky0 + t, nky - 1);
            f[e] = cscale(f[e], __ldg(spec_half + (long long)ky * mx + kx));
        }
        __syncthreads();
        f = fft_smem<+1>(f, g, fx, kt);
    }
    const int keep = (mode == 0) ? nx : mx;
    for (int e = threadIdx.x; e < kt * keep; e += blockDim.x) {
        const int t = e / keep, ix = e - t * keep;
        const int ky = ky0 + t;
        if (ky < nky) w[(long long)ky * ld + ix] = f[t * mx + ix];
    }
}

// Pass C: Hermitian half → real rows (two rows per complex transform), ×scale, crop.
__global__ void __launch_bounds__(kThreads) k_rows_inv(const double2* __restrict__ W, long long ldw, int nx,
                                                      int ny, FftLen fy, double* __restrict__ Y, long long ldy,
                                                      int pairs, double scale) {
    extern __shared__ double2 sm[];
    const int my = fy.n;
    double2* a = sm;
    double2* b = sm + pairs * my;
    const int ix0 = blockIdx.x * pairs * 2;
    const double2* w = W + (long long)blockIdx.y * ldw;
    for (int e = threadIdx.x; e < pairs * my; e += blockDim.x) {
        const int t = e / my, ky = e - t * my;
        const int r0 = ix0 + 2 * t, r1 = r0 + 1;
        const bool hi = ky > my / 2;
        const int kk = hi ? my - ky : ky;
        double2 x1 = make_double2(0.0, 0.0), x2 = make_double2(0.0, 0.0);
        if (r0 < nx) x1 = w[(long long)kk * nx + r0];
        if (r1 < nx) x2 = w[(long long)kk * nx + r1];
        if (hi) { x1 = cconj(x1); x2 = cconj(x2); }
        a[e] = make_double2(x1.x - x2.y, x1.y + x2.x);  // X1 + i·X2
    }
    __syncthreads();
    const double2* z = fft_smem<+1>(a, b, fy, pairs);
    double* y = Y + (long long)blockIdx.y * ldy;
    for (int e = threadIdx.x; e < pairs * 2 * ny; e += blockDim.x) {
        const int rl = e / ny, iy = e - rl * ny;
        const int ix = ix0 + rl;
        if (ix >= nx) continue;
        const double2 v = z[(rl >> 1) * my + iy];
        y[(long long)ix * ny + iy] = ((rl & 1) ? v.y : v.x) * scale;
    }
}

// ---- single-vector path (the per-step Γ(Hᵀz)).  One transform per CTA with a radix-≤8
// schedule and n/8 threads, so each thread's serial chain is a few radix-8 butterflies (the
// batched radix-16 kernels keep one butterfly per thread busy for ~4× longer); twiddles are
// staged in shared memory alongside the data.

// Every global load of a kernel is issued before the first shared-memory store (≤ 8 elements
// per thread since blockDim ≥ n/8), so the load phase costs one memory latency, not eight.
constexpr int kEpt = 8;
constexpr int kRowPairs = 4;   // batched: 8 consecutive rows per CTA (128-byte W segments)
constexpr int kRowPairs1 = 2;  // single vector: fewer, still-coalesced CTAs (measured best)  // transforms per CTA in the batched register-resident rows passes

// Per-transform buffer stride of the register-resident rows passes with RP transforms per CTA:
// the inverse pass maps lane t to (transform t % RP, index t / RP), so a quarter-warp's 16-byte
// exchange accesses hit banks (p·stride + index) mod 8 — a stride ≡ 8/RP (mod 8) makes them
// distinct (the bare NT + NT/8 + 1 ≡ 1 had 2-way conflicts for RP = 4: half of the pass's
// shared-memory wavefronts).  The forward pass (one transform per warp) is unaffected.
__host__ __device__ __forceinline__ int rows_bl(int n, int rp) {
    const int b = n + n / 8 + 1;
    if (rp <= 1 || rp >= 8) return b;
    const int want = 8 / rp;
    return b + ((want - b % 8) % 8 + 8) % 8;
}

// Shared layout of the single-transform kernels: twiddles | a | b.  NT > 0 (compile-time
// power-of-two length): per-pass twiddle table and padded buffers (fft_block_p); NT = 0:
// base table tw[0..n) and plain buffers (runtime schedule, fft_block).
template <int NT>
struct Lay1 {
    static constexpr bool ST = NT > 0;
    __device__ __forceinline__ static int tlen(int n) { return ST ? static_tw_len(NT) : n; }
    __device__ __forceinline__ static int blen(int n) { return ST ? NT + NT / 8 + 1 : n; }
    __device__ __forceinline__ static int ix(int e) { return ST ? fpad(e) : e; }
    __device__ __forceinline__ static double2 twv(const FftLen& L, int i) { return ST ? L.twp[i] : L.tw[i]; }
    template <int SIGN>
    __device__ __forceinline__ static double2* fft(double2* a, double2* b, const FftLen& L, const double2* tw) {
        if constexpr (ST) return fft_block_p<SIGN, NT>(a, b, tw);
        else return fft_block<SIGN>(a, b, L, tw);
    }
};

// Pass A: CTA = real rows 2b, 2b+1 (two-for-one) → W[ky][ix].
template <int NT>
__global__ void __launch_bounds__(256) k_rows_fwd_1(const double* __restrict__ x, int nx, int ny, FftLen fy,
                                                   double2* __restrict__ W, long long ldx, long long ldw) {
    using L = Lay1<NT>;
    extern __shared__ double2 sm[];
    x += blockIdx.y * ldx;  // column blockIdx.y of a batch
    W += blockIdx.y * ldw;
    const int my = fy.n, nky = my / 2 + 1, T = blockDim.x;
    const int tl = L::tlen(my);
    double2* tw = sm;
    double2* a = sm + tl;
    double2* b = a + L::blen(my);
    const int r0 = 2 * blockIdx.x, r1 = r0 + 1;
    if constexpr (reg_fft_len<NT>()) {
        // register-resident transforms, kRowPairs per CTA (rows ix0 … ix0 + 2·kRowPairs − 1):
        // thread (pair p, index j) loads 32 consecutive y of two rows per warp, and the W tile
        // is written 2·kRowPairs consecutive ix (128 B) per ky
        constexpr int TPT = (reg_fft_len<NT>() ? NT : 512) / 8;  // threads per transform
        const int RP = blockDim.x / TPT;                          // transforms (row pairs) per CTA
        const int t = threadIdx.x, p = t / TPT, j = t % TPT;
        const int ix0 = blockIdx.x * 2 * RP;
        const int q0 = ix0 + 2 * p, q1 = q0 + 1;
        const int bl = rows_bl(my, RP);
        double2* ap = sm + p * bl;  // twiddles come from the global per-pass table (fft_reg)
        double2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int iy = j + q * TPT;
            v[q] = make_double2((iy < ny && q0 < nx) ? x[(long long)q0 * ny + iy] : 0.0,
                                (iy < ny && q1 < nx) ? x[(long long)q1 * ny + iy] : 0.0);
        }
        fft_reg<-1, (reg_fft_len<NT>() ? NT : 512)>(v, ap, RP == 1 ? ap + bl : nullptr, fy.twp, j, fy.tw);  // ping-pong if alone
        __syncthreads();  // last exchange loads done before the result overwrites the buffer
#pragma unroll
        for (int q = 0; q < 8; ++q) ap[fpad(j + q * TPT)] = v[q];
        __syncthreads();
        const int rows = 2 * RP;
        for (int e = t; e < rows * nky; e += blockDim.x) {
            const int ky = e / rows, rl = e - ky * rows;
            const int ix = ix0 + rl;
            if (ix >= nx) continue;
            const double2* zt = sm + (rl >> 1) * bl;
            const double2 pp = zt[fpad(ky)];
            const double2 qq = cconj(zt[fpad(ky == 0 ? 0 : my - ky)]);
            W[(long long)ky * nx + ix] = (rl & 1) == 0 ? make_double2(0.5 * (pp.x + qq.x), 0.5 * (pp.y + qq.y))
                                                       : make_double2(0.5 * (pp.y - qq.y), -0.5 * (pp.x - qq.x));
        }
        return;
    }
    double2 tv[kEpt];
    double v0[kEpt], v1[kEpt];
#pragma unroll
    for (int q = 0; q < kEpt; ++q) {
        const int iy = threadIdx.x + q * T;
        tv[q] = iy < tl ? L::twv(fy, iy) : make_double2(0.0, 0.0);
        v0[q] = iy < ny ? x[(long long)r0 * ny + iy] : 0.0;
        v1[q] = (iy < ny && r1 < nx) ? x[(long long)r1 * ny + iy] : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kEpt; ++q) {
        const int iy = threadIdx.x + q * T;
        if (iy < tl) tw[iy] = tv[q];
        if (iy < my) a[L::ix(iy)] = make_double2(v0[q], v1[q]);
    }
    __syncthreads();
    const double2* z = L::template fft<-1>(a, b, fy, tw);
    for (int ky = threadIdx.x; ky < nky; ky += T) {
        const double2 p = z[L::ix(ky)];
        const double2 q = cconj(z[L::ix(ky == 0 ? 0 : my - ky)]);
        W[(long long)ky * nx + r0] = make_double2(0.5 * (p.x + q.x), 0.5 * (p.y + q.y));      // (Z + conj Z−)/2
        if (r1 < nx) W[(long long)ky * nx + r1] = make_double2(0.5 * (p.y - q.y), -0.5 * (p.x - q.x));  // /(2i)
    }
}

// Pass B: CTA = column ky: zero-pad, FFT, × spectrum, iFFT, keep ix < nx.
template <int NT>
__global__ void __launch_bounds__(256) k_cols_1(double2* __restrict__ W, int nx, FftLen fx,
                                               const double* __restrict__ spec_half, long long ldw) {
    using L = Lay1<NT>;
    extern __shared__ double2 sm[];
    W += blockIdx.y * ldw;
    const int mx = fx.n, T = blockDim.x;
    const int tl = L::tlen(mx);
    double2* tw = sm;
    double2* a = sm + tl;
    double2* b = a + L::blen(mx);
    double2* w = W + (long long)blockIdx.x * nx;
    const double* sp = spec_half + (long long)blockIdx.x * mx;
    if constexpr (reg_fft_len<NT>()) {  // forward → × spectrum → inverse, all in registers
        const int j = threadIdx.x;
        double2* ra = sm;  // no shared twiddle table on this path
        double2* rb = sm + L::blen(mx);
        double2 v[8];
        double spv[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int ix = j + q * T;
            v[q] = ix < nx ? w[ix] : make_double2(0.0, 0.0);
            spv[q] = __ldg(sp + ix);
        }
        fft_reg<-1, (reg_fft_len<NT>() ? NT : 512)>(v, ra, rb, fx.twp, j, fx.tw);
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = cscale(v[q], spv[q]);
        fft_reg<+1, (reg_fft_len<NT>() ? NT : 512)>(v, ra, rb, fx.twp, j, fx.tw);
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (j + q * T < nx) w[j + q * T] = v[q];
        return;
    }
    double2 tv[kEpt], dv[kEpt];
    double spv[kEpt];
#pragma unroll
    for (int q = 0; q < kEpt; ++q) {
        const int ix = threadIdx.x + q * T;
        tv[q] = ix < tl ? L::twv(fx, ix) : make_double2(0.0, 0.0);
        dv[q] = ix < nx ? w[ix] : make_double2(0.0, 0.0);
        spv[q] = ix < mx ? __ldg(sp + ix) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kEpt; ++q) {
        const int ix = threadIdx.x + q * T;
        if (ix < tl) tw[ix] = tv[q];
        if (ix < mx) a[L::ix(ix)] = dv[q];
    }
    __syncthreads();
    double2* f = L::template fft<-1>(a, b, fx, tw);
    double2* g = (f == a) ? b : a;
#pragma unroll
    for (int q = 0; q < kEpt; ++q) {
        const int kx = threadIdx.x + q * T;
        if (kx < mx) f[L::ix(kx)] = cscale(f[L::ix(kx)], spv[q]);
    }
    __syncthreads();
    f = L::template fft<+1>(f, g, fx, tw);
    for (int ix = threadIdx.x; ix < nx; ix += T) w[ix] = f[L::ix(ix)];
}

// Pass C: CTA = rows 2b, 2b+1 rebuilt from the Hermitian half, ×scale, crop.  With
// upd.coef set the pass is the filter step's mean update instead of a plain store:
// y_i ← (y_i + c·(Γx)_i) − sub_i (fast_filter.hpp:114-116, sub = U·dc from the concurrent U
// pass), skipped when *upd.gate (failed step); the new value also goes to the mapped host
// buffer upd.hout[0] and the failure flag to upd.hout[2] when set.
template <int NT, bool UPD>
__global__ void __launch_bounds__(256) k_rows_inv_1(const double2* __restrict__ W, int nx, int ny, FftLen fy,
                                                   double* __restrict__ y, double scale, MeanUpd upd,
                                                   long long ldw, long long ldy) {
    const double* __restrict__ acc_coef = UPD ? upd.coef : nullptr;
    const int* __restrict__ gate = upd.gate;
    const double* __restrict__ sub = upd.sub;
    if (UPD && upd.ycnt && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *upd.ycnt += 1;  // next batch row
    double* hm = nullptr;
    if (acc_coef && upd.hout) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && upd.hout[2])
            *reinterpret_cast<volatile int*>(upd.hout[2]) = gate ? *gate : 0;
        hm = reinterpret_cast<double*>(upd.hout[0]);
    }
    using L = Lay1<NT>;
    extern __shared__ double2 sm[];
    W += blockIdx.y * ldw;
    y += blockIdx.y * ldy;
    const int my = fy.n, T = blockDim.x;
    const int tl = L::tlen(my);
    double2* tw = sm;
    double2* a = sm + tl;
    double2* b = a + L::blen(my);
    const int r0 = 2 * blockIdx.x, r1 = r0 + 1;
    if constexpr (reg_fft_len<NT>()) {
        // kRowPairs transforms per CTA; thread (p = t % kRowPairs, j = t / kRowPairs) so the
        // 2·kRowPairs consecutive W entries of a ky (128 B) are read by consecutive lanes
        constexpr int TPT = (reg_fft_len<NT>() ? NT : 512) / 8;
        const int RP = blockDim.x / TPT;
        const int t = threadIdx.x, p = t % RP, j = t / RP;
        const int ix0 = blockIdx.x * 2 * RP;
        const int q0 = ix0 + 2 * p, q1 = q0 + 1;
        const int bl = rows_bl(my, RP);
        double2* ap = sm + p * bl;  // twiddles come from the global per-pass table (fft_reg)
        // mean-update operands loaded up front (independent of the transform, their latency
        // hides under it; loaded after the stores below they would serialize on aliasing)
        double2 ym[8], ys[8];
        if (acc_coef) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int iy = j + q * TPT;
                const bool in = iy < ny;
                const long long i0 = (long long)q0 * ny + iy, i1 = (long long)q1 * ny + iy;
                ym[q] = make_double2(in && q0 < nx ? y[i0] : 0.0, in && q1 < nx ? y[i1] : 0.0);
                ys[q] = make_double2(in && q0 < nx && sub ? sub[i0] : 0.0, in && q1 < nx && sub ? sub[i1] : 0.0);
            }
        }
        double2 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int ky = j + q * TPT;
            const bool hi = ky > my / 2;
            const int kk = hi ? my - ky : ky;
            double2 u1 = q0 < nx ? W[(long long)kk * nx + q0] : make_double2(0.0, 0.0);
            double2 u2 = q1 < nx ? W[(long long)kk * nx + q1] : make_double2(0.0, 0.0);
            if (hi) { u1 = cconj(u1); u2 = cconj(u2); }
            v[q] = make_double2(u1.x - u2.y, u1.y + u2.x);  // X1 + i·X2
        }
        fft_reg<+1, (reg_fft_len<NT>() ? NT : 512)>(v, ap, RP == 1 ? ap + bl : nullptr, fy.twp, j, fy.tw);
        if (acc_coef && gate && *gate) return;
        const double c = acc_coef ? *acc_coef : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int iy = j + q * TPT;
            if (iy >= ny) continue;
            if (q0 < nx) {
                const long long i0 = (long long)q0 * ny + iy;
                double nv = acc_coef ? ym[q].x + c * (v[q].x * scale) : v[q].x * scale;
                if (sub) nv -= ys[q].x;
                y[i0] = nv;
                if (hm) hm[i0] = nv;
            }
            if (q1 < nx) {
                const long long i1 = (long long)q1 * ny + iy;
                double nv = acc_coef ? ym[q].y + c * (v[q].y * scale) : v[q].y * scale;
                if (sub) nv -= ys[q].y;
                y[i1] = nv;
                if (hm) hm[i1] = nv;
            }
        }
        return;
    }
    double2 tv[kEpt], x1[kEpt], x2[kEpt];
#pragma unroll
    for (int q = 0; q < kEpt; ++q) {
        const int ky = threadIdx.x + q * T;
        const int kk = ky > my / 2 ? my - ky : ky;
        tv[q] = ky < tl ? L::twv(fy, ky) : make_double2(0.0, 0.0);
        x1[q] = ky < my ? W[(long long)kk * nx + r0] : make_double2(0.0, 0.0);
        x2[q] = (ky < my && r1 < nx) ? W[(long long)kk * nx + r1] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int q = 0; q < kEpt; ++q) {
        const int ky = threadIdx.x + q * T;
        if (ky < tl) tw[ky] = tv[q];
        if (ky < my) {
            double2 u1 = x1[q], u2 = x2[q];
            if (ky > my / 2) { u1 = cconj(u1); u2 = cconj(u2); }
            a[L::ix(ky)] = make_double2(u1.x - u2.y, u1.y + u2.x);  // X1 + i·X2
        }
    }
    __syncthreads();
    const double2* z = L::template fft<+1>(a, b, fy, tw);
    if (acc_coef) {  // y = (y + c·Γx) − sub (the mean update), skipped when *gate
        if (gate && *gate) return;
        const double c = *acc_coef;
        for (int iy = threadIdx.x; iy < ny; iy += T) {
            const double2 v = z[L::ix(iy)];
            const long long i0 = (long long)r0 * ny + iy;
            double nv = y[i0] + c * (v.x * scale);
            if (sub) nv -= sub[i0];
            y[i0] = nv;
            if (hm) hm[i0] = nv;
            if (r1 < nx) {
                const long long i1 = (long long)r1 * ny + iy;
                double nw = y[i1] + c * (v.y * scale);
                if (sub) nw -= sub[i1];
                y[i1] = nw;
                if (hm) hm[i1] = nw;
            }
        }
        return;
    }
    for (int iy = threadIdx.x; iy < ny; iy += T) {
        const double2 v = z[L::ix(iy)];
        y[(long long)r0 * ny + iy] = v.x * scale;
        if (r1 < nx) y[(long long)r1 * ny + iy] = v.y * scale;
    }
}

// Sampler pass 1: draw amp·(n_re + i n_im) on the torus for a tile of ky columns,
// inverse FFT along x, keep ix < nx → T[ky][ix] (full ky range).
// blockIdx.y = pair p of a batch: streams (seed, 2(sid0+p)) and (seed, 2(sid0+p)+1), T offset by p·my·nx
__global__ void __launch_bounds__(kThreads) k_sampler_cols(const double* __restrict__ amp, int my, int nx,
                                                          FftLen fx, uint64_t seed, uint64_t sid0,
                                                          double2* __restrict__ T, int kt) {
    extern __shared__ double2 sm[];
    const int mx = fx.n;
    const uint64_t sid = sid0 + blockIdx.y;
    const uint64_t st_re = splitmix64(seed ^ splitmix64(2 * sid)), st_im = splitmix64(seed ^ splitmix64(2 * sid + 1));
    T += (long long)blockIdx.y * my * nx;
    double2* a = sm;
    double2* b = sm + kt * mx;
    const int ky0 = blockIdx.x * kt;
    for (int e = threadIdx.x; e < kt * mx; e += blockDim.x) {
        const int t = e / mx, kx = e - t * mx;
        const int ky = ky0 + t;
        double2 v = make_double2(0.0, 0.0);
        if (ky < my) {
            const unsigned long long idx = (unsigned long long)kx * my + ky;  // covariance.hpp:338-342
            const double am = __ldg(amp + idx);
            v = make_double2(am * rng_normal_at(st_re, idx), am * rng_normal_at(st_im, idx));
        }
        a[e] = v;
    }
    __syncthreads();
    const double2* f = fft_smem<+1>(a, b, fx, kt);
    for (int e = threadIdx.x; e < kt * nx; e += blockDim.x) {
        const int t = e / nx, ix = e - t * nx;
        const int ky = ky0 + t;
        if (ky < my) T[(long long)ky * nx + ix] = f[t * mx + ix];
    }
}

// Sampler pass 2: per row ix, inverse c2c FFT along y, crop, Re → a, Im → b (×1/√M).
// blockIdx.y = pair p: outputs da + p·ld_pair, db + p·ld_pair (db skipped when 2p+1 ≥ ncols);
// accumulate: add into the outputs instead of storing
__global__ void __launch_bounds__(kThreads) k_sampler_rows(const double2* __restrict__ T, int nx, int ny,
                                                          FftLen fy, double* __restrict__ da,
                                                          double* __restrict__ db, int rows, double scale,
                                                          long long ld_pair, int ncols, int accumulate) {
    extern __shared__ double2 sm[];
    const int my = fy.n;
    const int p = blockIdx.y;
    T += (long long)p * my * nx;
    da += p * ld_pair;
    db = 2 * p + 1 < ncols ? db + p * ld_pair : nullptr;
    double2* a = sm;
    double2* b = sm + rows * my;
    const int ix0 = blockIdx.x * rows;
    for (int e = threadIdx.x; e < rows * my; e += blockDim.x) {
        const int t = e / my, ky = e - t * my;
        const int ix = ix0 + t;
        a[e] = ix < nx ? T[(long long)ky * nx + ix] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const double2* f = fft_smem<+1>(a, b, fy, rows);
    for (int e = threadIdx.x; e < rows * ny; e += blockDim.x) {
        const int t = e / ny, iy = e - t * ny;
        const int ix = ix0 + t;
        if (ix < nx) {
            const double2 v = f[t * my + iy];
            const long long o = (long long)ix * ny + iy;
            if (accumulate) {
                da[o] += v.x * scale;
                if (db) db[o] += v.y * scale;
            } else {
                da[o] = v.x * scale;
                if (db) db[o] = v.y * scale;
            }
        }
    }
}

// ---- fast sampler path for 512×512 tori (register-resident radix-8 transforms).
// Pass 1: a CTA owns 4 consecutive ky columns (ky0 ≡ 0 mod 4): the 4×512 torus inputs
// amp·(n_re + i·n_im) are generated into shared memory with one Box–Muller evaluation per
// two normals (idx = kx·my + ky: ky0+2q and ky0+2q+1 share the pair idx/2), then each
// 64-thread group runs an inverse 512-point transform along x in registers; rows ix < nx are
// stored ix-major, T[ix][ky] (64-byte segments of the 4 columns).
__global__ void __launch_bounds__(256) k_samp_cols512(const double* __restrict__ amp, int my, int nx,
                                                      const double2* __restrict__ twp, uint64_t seed, uint64_t sid0,
                                                      double2* __restrict__ T) {
    constexpr int N = 512, BL = N + N / 8 + 1;
    extern __shared__ double2 sm[];
    double2* g = sm;                 // [4][512] generated inputs, reused as the output stage
    double2* fb = sm + 4 * N;        // 4 transforms × 2 ping-pong buffers
    const uint64_t sid = sid0 + blockIdx.y;
    const uint64_t st_re = splitmix64(seed ^ splitmix64(2 * sid)), st_im = splitmix64(seed ^ splitmix64(2 * sid + 1));
    T += (long long)blockIdx.y * nx * my;
    const int ky0 = blockIdx.x * 4;
    for (int e = threadIdx.x; e < N * 2; e += blockDim.x) {  // (kx, q): pair of columns ky0+2q, +1
        const int kx = e >> 1, q = e & 1;
        const unsigned long long idx = (unsigned long long)kx * my + ky0 + 2 * q;  // even
        double r0, r1, i0, i1;
        rng_normal_pair(st_re, idx >> 1, r0, r1);
        rng_normal_pair(st_im, idx >> 1, i0, i1);
        const double a0 = __ldg(amp + idx), a1 = __ldg(amp + idx + 1);
        g[(2 * q) * N + kx] = make_double2(a0 * r0, a0 * i0);
        g[(2 * q + 1) * N + kx] = make_double2(a1 * r1, a1 * i1);
    }
    __syncthreads();
    const int t = threadIdx.x >> 6, j = threadIdx.x & 63;
    double2 v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = g[t * N + j + 64 * r];
    double2* ba = fb + t * 2 * BL;
    fft_reg<+1, N>(v, ba, ba + BL, twp, j);
    __syncthreads();  // every transform has consumed g
#pragma unroll
    for (int r = 0; r < 8; ++r) g[t * N + j + 64 * r] = v[r];
    __syncthreads();
    for (int e = threadIdx.x; e < nx * 4; e += blockDim.x) {
        const int ix = e >> 2, c = e & 3;
        T[(long long)ix * my + ky0 + c] = g[c * N + ix];
    }
}

// Pass 2: a CTA owns 4 rows ix; each 64-thread group loads T[ix][0..512) coalesced, runs the
// inverse transform along y in registers and adds Re → a, Im → b (×1/√M) for iy < ny.
__global__ void __launch_bounds__(256) k_samp_rows512(const double2* __restrict__ T, int nx, int ny,
                                                      const double2* __restrict__ twp, double* __restrict__ da,
                                                      double* __restrict__ db, double scale, long long ld_pair,
                                                      int ncols) {
    constexpr int N = 512, BL = N + N / 8 + 1;
    extern __shared__ double2 sm[];
    const int p = blockIdx.y;
    T += (long long)p * nx * N;
    da += p * ld_pair;
    db = 2 * p + 1 < ncols ? db + p * ld_pair : nullptr;
    const int t = threadIdx.x >> 6, j = threadIdx.x & 63;
    const int ix = blockIdx.x * 4 + t;
    double2 v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = ix < nx ? T[(long long)ix * N + j + 64 * r] : make_double2(0.0, 0.0);
    double2* ba = sm + t * 2 * BL;
    fft_reg<+1, N>(v, ba, ba + BL, twp, j);
    if (ix >= nx) return;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int iy = j + 64 * r;
        if (iy < ny) {
            const long long o = (long long)ix * ny + iy;
            da[o] += v[r].x * scale;
            if (db) db[o] += v[r].y * scale;
        }
    }
}

// --------------------------------------------------------------------------- host orchestration
// lengths with a compile-time single-transform schedule (see with_len)
static bool static_len(int n) { return n == 64 || n == 128 || n == 256 || n == 512 || n == 1024 || n == 2048; }

static void plan_radices(FftLen& L, int n, bool max8 = false) {
    L.n = n;
    L.npass = 0;
    int v = n;
    auto push = [&](int r) {
        if (L.npass >= kMaxPasses) throw std::runtime_error("fft: too many passes");
        L.radix[L.npass++] = r;
    };
    if (max8)
        while (v % 8 == 0) { push(8); v /= 8; }
    while (v % 16 == 0) { push(16); v /= 16; }
    if (v % 8 == 0) { push(8); v /= 8; }
    if (v % 4 == 0) { push(4); v /= 4; }
    if (v % 2 == 0) { push(2); v /= 2; }
    for (int f : {3, 5, 7})
        while (v % f == 0) { push(f); v /= f; }
    if (v != 1) throw std::invalid_argument("fft: length " + std::to_string(n) + " is not {2,3,5,7}-smooth");
}

// per-pass twiddle table of the compile-time schedule (FftLen::twp), same angles as the
// base table: exp(−2πi·r·k·(n/(NS·R))/n)
void Cov::setup_static_tw(FftLen& L, DBuf<double2>& tw, int n) {
    L.twp = nullptr;
    if (!static_len(n)) return;
    std::vector<double2> h;
    for (int ns = 1; ns < n;) {
        const int R = (n / ns) % 8 == 0 ? 8 : n / ns;
        if (ns > 1)
            for (int r = 1; r < R; ++r)
                for (int k = 0; k < ns; ++k) {
                    const long long e = (long long)r * k * (n / (ns * R));
                    const long double ang = -2.0L * std::numbers::pi_v<long double> * (long double)e / n;
                    h.push_back(make_double2(double(cosl(ang)), double(sinl(ang))));
                }
        ns *= R;
    }
    if (int(h.size()) != static_tw_len(n)) throw std::logic_error("fft: static twiddle table size");
    tw.alloc(std::max<size_t>(h.size(), 1));
    if (!h.empty()) FKB_CUDA(cudaMemcpy(tw.p, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice));
    L.twp = tw.p;
}

void Cov::setup_len(FftLen& L, DBuf<double2>& tw, int n) {
    plan_radices(L, n);
    std::vector<double2> h(static_cast<size_t>(n));
    for (int k = 0; k < n; ++k) {
        const long double ang = -2.0L * std::numbers::pi_v<long double> * k / n;
        h[size_t(k)] = make_double2(double(cosl(ang)), double(sinl(ang)));
    }
    tw.alloc(size_t(n));
    FKB_CUDA(cudaMemcpy(tw.p, h.data(), sizeof(double2) * size_t(n), cudaMemcpyHostToDevice));
    L.tw = tw.p;
}

static int pairs_for(int my) { return my >= 1024 ? 2 : (my >= 512 ? 4 : std::max(4, 2048 / std::max(my, 1) / 2)); }
static int kt_for(int mx) { return mx >= 1024 ? 2 : (mx >= 512 ? 4 : std::max(4, 2048 / std::max(mx, 1))); }
static size_t smem_bytes(int batch, int n) { return 2 * size_t(batch) * size_t(n) * sizeof(double2); }

static void set_smem(const void* fn, size_t bytes) {
    if (bytes > 227 * 1024) throw std::invalid_argument("fft: transform too large for shared memory");
    FKB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
}

Cov::Cov(int nx_, int ny_, double lx_, double ly_, const KernelSpec& s, cudaStream_t st)
    : nx(nx_), ny(ny_), lx(lx_), ly(ly_), spec(s), stream(st) {
    if (nx < 1 || ny < 1)
        throw std::invalid_argument("grid: nx and ny must be positive, got " + std::to_string(nx) + "x" + std::to_string(ny));
    if (!(lx > 0.0) || !(ly > 0.0)) throw std::invalid_argument("grid: domain lengths must be positive");
    spec.validate();
    init_odd_tables();
    const int base_x = std::max(2 * nx - 1, 1), base_y = std::max(2 * ny - 1, 1);
    double worst = 0.0;
    for (int pad = 1; pad <= 8; pad *= 2) {  // covariance.hpp:238-260
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
    msg << ") on grid " << nx << "x" << ny << " even after 8x padding (worst negative/max spectrum ratio " << worst
        << "); use dense mode or a shorter correlation length";
    throw std::runtime_error(msg.str());
}

void Cov::ensure_work(int ncols) {
    const size_t need = size_t(ncols) * size_t(nky) * size_t(std::max(nx, mx));
    if (work.n < need) work.alloc(need);
}

bool Cov::try_spectrum(double& worst) {  // covariance.hpp:264-298
    nky = my / 2 + 1;
    setup_len(fx, twx, mx);
    setup_len(fy, twy, my);
    fx8 = fx;  // same twiddle tables, radix ≤ 8 schedules for the single-vector kernels
    fy8 = fy;
    plan_radices(fx8, mx, true);
    plan_radices(fy8, my, true);
    setup_static_tw(fx8, twpx, mx);
    setup_static_tw(fy8, twpy, my);
    // Symbol on the torus at wrapped distances (:269-277), evaluated on the host with the
    // reference formula (std::cyl_bessel_k); only the unique quarter is evaluated.
    const double dx = lx / nx, dy = ly / ny;
    const int hx = mx / 2 + 1, hy = my / 2 + 1;
    std::vector<double> quarter(static_cast<size_t>(hx) * hy);
    for (int i = 0; i < hx; ++i)
        for (int j = 0; j < hy; ++j)
            quarter[size_t(i) * hy + j] = kernel_eval(spec, std::hypot(std::min(i, mx - i) * dx, std::min(j, my - j) * dy));
    std::vector<double> sym(static_cast<size_t>(M()));
    for (int i = 0; i < mx; ++i)
        for (int j = 0; j < my; ++j) sym[size_t(i) * my + j] = quarter[size_t(std::min(i, mx - i)) * hy + std::min(j, my - j)];
    DBuf<double> dsym(sym.size());
    FKB_CUDA(cudaMemcpyAsync(dsym.p, sym.data(), sym.size() * sizeof(double), cudaMemcpyHostToDevice, stream));
    // Forward 2-D DFT of the real symbol: rows (R2C) then full columns, on the GPU.
    ensure_work(1);
    const int pairs = pairs_for(my), kt = kt_for(mx);
    set_smem((const void*)k_rows_fwd, smem_bytes(pairs, my));
    set_smem((const void*)k_cols, smem_bytes(kt, mx));
    set_smem((const void*)k_rows_inv, smem_bytes(pairs, my));
    k_rows_fwd<<<dim3(ceil_div(mx, 2 * pairs), 1), kThreads, smem_bytes(pairs, my), stream>>>(
        dsym.p, 0, mx, my, mx, fy, work.p, 0, pairs);
    FKB_LAUNCH_CHECK();
    k_cols<<<dim3(ceil_div(nky, kt), 1), kThreads, smem_bytes(kt, mx), stream>>>(work.p, 0, mx, fx, nky, nullptr, kt, 1);
    FKB_LAUNCH_CHECK();
    count_launch(2);
    std::vector<double2> half(static_cast<size_t>(nky) * mx);
    FKB_CUDA(cudaMemcpyAsync(half.data(), work.p, half.size() * sizeof(double2), cudaMemcpyDeviceToHost, stream));
    FKB_CUDA(cudaStreamSynchronize(stream));
    // Full-torus real spectrum: S[kx][ky] = Re(half[ky][kx]) for ky ≤ my/2 and the even
    // mirror S[kx][ky] = S[−kx][−ky] above (exact for the DFT of a real even symbol).
    std::vector<double> full(static_cast<size_t>(M()));
    double mxv = 0.0, mnv = 0.0;
    for (int kx = 0; kx < mx; ++kx)
        for (int ky = 0; ky < my; ++ky) {
            double v;
            if (ky < nky) v = half[size_t(ky) * mx + kx].x;
            else v = half[size_t(my - ky) * mx + (kx == 0 ? 0 : mx - kx)].x;
            full[size_t(kx) * my + ky] = v;
            mxv = std::max(mxv, v);
            mnv = std::min(mnv, v);
        }
    if (mxv <= 0.0) return false;
    worst = std::max(worst, -mnv / mxv);
    if (mnv < -1e-10 * mxv) return false;
    std::vector<double> sh(static_cast<size_t>(nky) * mx), amp(static_cast<size_t>(M()));
    for (int ky = 0; ky < nky; ++ky)
        for (int kx = 0; kx < mx; ++kx) sh[size_t(ky) * mx + kx] = std::max(half[size_t(ky) * mx + kx].x, 0.0);
    for (size_t i = 0; i < full.size(); ++i) {
        full[i] = std::max(full[i], 0.0);
        amp[i] = std::sqrt(full[i]);
    }
    spec_half.alloc(sh.size());
    amp_full.alloc(amp.size());
    FKB_CUDA(cudaMemcpyAsync(spec_half.p, sh.data(), sh.size() * sizeof(double), cudaMemcpyHostToDevice, stream));
    FKB_CUDA(cudaMemcpyAsync(amp_full.p, amp.data(), amp.size() * sizeof(double), cudaMemcpyHostToDevice, stream));
    FKB_CUDA(cudaStreamSynchronize(stream));
    // Column batches of the blocked Γ·X: larger batches shorten the per-launch wave tails of
    // the three passes, and that outweighs keeping the intermediate L2-resident (measured at
    // c2: 45 columns (48 MB) 9.9 TF/s, 128 10.6, 256 11.2, 592 11.6).  Budget 640 MB, ≤ 1024.
    const size_t per_col = size_t(nky) * size_t(nx) * sizeof(double2);
    batch_cap = int(std::max<size_t>(1, std::min<size_t>(1024, (size_t(640) << 20) / per_col)));
    if (const char* e = std::getenv("FKB_GX_BATCH")) batch_cap = std::max(1, std::atoi(e));  // tuning aid
    // One workspace for the whole lifetime (graph-captured steps hold its address):
    // batched Γ-apply intermediate or the sampler's my×nx column pass.
    work.release();
    work.alloc(std::max(size_t(batch_cap) * nky * nx, size_t(my) * nx));
    return true;
}

std::vector<double> Cov::spectrum_host() const {
    std::vector<double> amp(static_cast<size_t>(M()));
    FKB_CUDA(cudaMemcpy(amp.data(), amp_full.p, amp.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (auto& v : amp) v = v * v;
    return amp;
}

// threads per transform of the single-vector kernels: n/8 (one radix-8 butterfly each per
// pass), a multiple of 32 in [32, 256]
static int threads_1(int n) { return std::max(32, ((n / kEpt + 31) / 32) * 32); }
// shared bytes of a single-transform kernel of length n (see Lay1)
static size_t smem_1(int n) {
    if (n == 512 || n == 1024) return 2 * size_t(n + n / 8 + 1) * sizeof(double2);  // register-resident: buffers only
    if (static_len(n)) return (size_t(static_tw_len(n)) + 2 * size_t(n + n / 8 + 1)) * sizeof(double2);
    return 3 * size_t(n) * sizeof(double2);
}
// rows passes: register-resident lengths hold kRowPairs single buffers
static size_t smem_rows(int n, int rp) {
    if (n == 512 || n == 1024) return size_t(std::max(rp, 2)) * rows_bl(n, rp) * sizeof(double2);
    return smem_1(n);
}

// transforms (row pairs) per CTA of the register-resident rows passes: ≤ 256 threads per CTA
template <int NT>
static int rows_rp(int ncols) {
    if (!reg_fft_len<NT>()) return 1;
    const int cap = 256 / (NT / 8);
    return std::min(ncols >= 8 ? kRowPairs : kRowPairs1, std::max(cap, 1));
}

template <int NT>
static void set_smem_1() {
    set_smem((const void*)k_rows_fwd_1<NT>, 0);
    set_smem((const void*)k_cols_1<NT>, 0);
    set_smem((const void*)k_rows_inv_1<NT, false>, 0);
    set_smem((const void*)k_rows_inv_1<NT, true>, 0);
}

// launch one of the three single-vector passes with a compile-time length when n is a
// supported power of two (radix-8 schedule folded to constants), else the runtime plan
template <class F>
static void with_len(int n, F&& f) {
    switch (n) {
        case 64: f(std::integral_constant<int, 64>{}); break;
        case 128: f(std::integral_constant<int, 128>{}); break;
        case 256: f(std::integral_constant<int, 256>{}); break;
        case 512: f(std::integral_constant<int, 512>{}); break;
        case 1024: f(std::integral_constant<int, 1024>{}); break;
        case 2048: f(std::integral_constant<int, 2048>{}); break;
        default: f(std::integral_constant<int, 0>{}); break;
    }
}

void Cov::apply1(const double* dx, double* dy) {
    apply1_fwd(dx);
    apply1_inv(dy, MeanUpd{});
}

void Cov::apply1_fwd(const double* dx, int ncols, long long ldx) {
    static bool attr = false;
    if (!attr) {
        for (int n : {64, 128, 256, 512, 1024, 2048, 0}) with_len(n, [](auto c) { set_smem_1<decltype(c)::value>(); });
        attr = true;
    }
    const size_t sy = smem_1(my), sx = smem_1(mx);
    if (sy > 227 * 1024 || sx > 227 * 1024 || threads_1(mx) > 256 || threads_1(my) > 256)
        throw std::invalid_argument("fft: transform too large for the single-vector kernels");
    const long long ldw = (long long)nky * nx;
    with_len(my, [&](auto c) {
        constexpr int NT = decltype(c)::value;
        const int rp = rows_rp<NT>(ncols);  // coalescing vs CTA count
        k_rows_fwd_1<NT><<<dim3(ceil_div(nx, 2 * rp), ncols), threads_1(my) * rp, smem_rows(my, rp), stream>>>(
            dx, nx, ny, fy8, work.p, ldx, ldw);
    });
    FKB_LAUNCH_CHECK();
    with_len(mx, [&](auto c) {
        k_cols_1<decltype(c)::value><<<dim3(nky, ncols), threads_1(mx), sx, stream>>>(work.p, nx, fx8, spec_half.p,
                                                                                     ldw);
    });
    FKB_LAUNCH_CHECK();
    count_launch(2);
}

void Cov::apply1_inv(double* dy, const MeanUpd& upd, int ncols, long long ldy) {
    const size_t sy = smem_1(my);
    const long long ldw = (long long)nky * nx;
    with_len(my, [&](auto c) {
        constexpr int NT = decltype(c)::value;
        const int rp = rows_rp<NT>(ncols);
        if (upd.coef)
            k_rows_inv_1<NT, true><<<dim3(ceil_div(nx, 2 * rp), ncols), threads_1(my) * rp, smem_rows(my, rp), stream>>>(
                work.p, nx, ny, fy8, dy, 1.0 / double(M()), upd, ldw, ldy);
        else
            k_rows_inv_1<NT, false><<<dim3(ceil_div(nx, 2 * rp), ncols), threads_1(my) * rp, smem_rows(my, rp), stream>>>(
                work.p, nx, ny, fy8, dy, 1.0 / double(M()), upd, ldw, ldy);
    });
    FKB_LAUNCH_CHECK();
    count_launch();
}

void Cov::apply(const double* dX, long long ldx, int ncols, double* dY, long long ldy) {
    if (ncols <= 0) return;
    ++applies;
    if (ncols == 1) {
        apply1(dX, dY);
        return;
    }
    // Blocks of columns: the CTA-per-transform kernels with blockIdx.y = column, in batches
    // whose intermediate stays L2-resident (the generic batched kernels below remain for
    // lengths the single-transform kernels cannot hold).
    if (smem_1(mx) <= 227 * 1024 && smem_1(my) <= 227 * 1024 && threads_1(mx) <= 256 && threads_1(my) <= 256) {
        for (int c0 = 0; c0 < ncols; c0 += batch_cap) {
            const int bc = std::min(batch_cap, ncols - c0);
            apply1_fwd(dX + (long long)c0 * ldx, bc, ldx);
            apply1_inv(dY + (long long)c0 * ldy, MeanUpd{}, bc, ldy);
        }
        return;
    }
    const bool narrow = ncols < 8;
    const int pairs = narrow ? 1 : pairs_for(my), kt = narrow ? 1 : kt_for(mx);
    const int tA = narrow ? std::max(64, std::min(kThreads, my / 4)) : kThreads;
    const int tB = narrow ? std::max(64, std::min(kThreads, mx / 4)) : kThreads;
    const long long ldw = (long long)nky * nx;
    const double scale = 1.0 / double(M());
    for (int c0 = 0; c0 < ncols; c0 += batch_cap) {
        const int bc = std::min(batch_cap, ncols - c0);
        k_rows_fwd<<<dim3(ceil_div(nx, 2 * pairs), bc), tA, smem_bytes(pairs, my), stream>>>(
            dX + (long long)c0 * ldx, ldx, nx, ny, nx, fy, work.p, ldw, pairs);
        FKB_LAUNCH_CHECK();
        k_cols<<<dim3(ceil_div(nky, kt), bc), tB, smem_bytes(kt, mx), stream>>>(work.p, ldw, nx, fx, nky,
                                                                               spec_half.p, kt, 0);
        FKB_LAUNCH_CHECK();
        k_rows_inv<<<dim3(ceil_div(nx, 2 * pairs), bc), tA, smem_bytes(pairs, my), stream>>>(
            work.p, ldw, nx, ny, fy, dY + (long long)c0 * ldy, ldy, pairs, scale);
        FKB_LAUNCH_CHECK();
        count_launch(3);
    }
}

void Cov::sample_pair(uint64_t seed, uint64_t sid, double* da, double* db) {
    const int kt = kt_for(mx);
    const int rows = std::max(1, std::min(4, 4096 / my));
    set_smem((const void*)k_sampler_cols, smem_bytes(kt, mx));
    set_smem((const void*)k_sampler_rows, smem_bytes(rows, my));
    k_sampler_cols<<<ceil_div(my, kt), kThreads, smem_bytes(kt, mx), stream>>>(amp_full.p, my, nx, fx, seed, sid,
                                                                             work.p, kt);
    FKB_LAUNCH_CHECK();
    k_sampler_rows<<<ceil_div(nx, rows), kThreads, smem_bytes(rows, my), stream>>>(
        work.p, nx, ny, fy, da, db, rows, 1.0 / std::sqrt(double(M())), 0, 2, 0);
    FKB_LAUNCH_CHECK();
    count_launch(2);
}

void Cov::sample_pairs_add(uint64_t seed, uint64_t sid0, double* X, long long ldx, int ncols) {
    if (ncols <= 0) return;
    const int kt = kt_for(mx);
    const int rows = std::max(1, std::min(4, 4096 / my));
    set_smem((const void*)k_sampler_cols, smem_bytes(kt, mx));
    set_smem((const void*)k_sampler_rows, smem_bytes(rows, my));
    const int npairs = (ncols + 1) / 2;
    const size_t per = size_t(my) * size_t(nx);
    if (mx == 512 && my == 512 && fx8.twp && fy8.twp) {  // register-resident fast path
        constexpr int N = 512, BL = N + N / 8 + 1;
        const size_t sm1 = (4 * N + 4 * 2 * BL) * sizeof(double2), sm2 = 4 * 2 * BL * sizeof(double2);
        FKB_CUDA(cudaFuncSetAttribute(k_samp_cols512, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm1)));
        FKB_CUDA(cudaFuncSetAttribute(k_samp_rows512, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm2)));
        const int bp = int(std::max<size_t>(1, std::min<size_t>(npairs, (size_t(1) << 26) / per)));
        if (swork.n < per * size_t(bp)) swork.alloc(per * size_t(bp));
        for (int p0 = 0; p0 < npairs; p0 += bp) {
            const int np = std::min(bp, npairs - p0);
            k_samp_cols512<<<dim3(my / 4, np), 256, sm1, stream>>>(amp_full.p, my, nx, fx8.twp, seed,
                                                                  sid0 + uint64_t(p0), swork.p);
            FKB_LAUNCH_CHECK();
            double* xa = X + (long long)(2 * p0) * ldx;
            k_samp_rows512<<<dim3(ceil_div(nx, 4), np), 256, sm2, stream>>>(
                swork.p, nx, ny, fy8.twp, xa, xa + ldx, 1.0 / std::sqrt(double(M())), 2 * ldx, ncols - 2 * p0);
            FKB_LAUNCH_CHECK();
            count_launch(2);
        }
        return;
    }
    const int bp = int(std::max<size_t>(1, std::min<size_t>(npairs, (size_t(1) << 26) / per)));  // ≤ 1 GiB
    if (swork.n < per * size_t(bp)) swork.alloc(per * size_t(bp));
    for (int p0 = 0; p0 < npairs; p0 += bp) {
        const int np = std::min(bp, npairs - p0);
        k_sampler_cols<<<dim3(ceil_div(my, kt), np), kThreads, smem_bytes(kt, mx), stream>>>(
            amp_full.p, my, nx, fx, seed, sid0 + uint64_t(p0), swork.p, kt);
        FKB_LAUNCH_CHECK();
        double* xa = X + (long long)(2 * p0) * ldx;
        k_sampler_rows<<<dim3(ceil_div(nx, rows), np), kThreads, smem_bytes(rows, my), stream>>>(
            swork.p, nx, ny, fy, xa, xa + ldx, rows, 1.0 / std::sqrt(double(M())), 2 * ldx, ncols - 2 * p0, 1);
        FKB_LAUNCH_CHECK();
        count_launch(2);
    }
}

}  // namespace fkb
