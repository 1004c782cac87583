// filter.cu — randomized GHEP, fkf_init, fkf_step and the UQ kernels on sm_100a.
//
// Reference: lowrank.hpp:141-213 (randomized_ghep, two-pass), fast_filter.hpp:51-125
// (fkf_init / fkf_step), uq.hpp:16-112 (variance, trace, entropy, realizations).
//
// Γ-metric orthonormalization.  The reference orthonormalizes Ȳ = AΩ column by column
// (modified Gram–Schmidt, 3 Γ-applies per column, lowrank.hpp:53-106).  Its outputs
// (λ, U·f(D)·Uᵀ) depend only on span(AΩ), so the device path uses a
// span-equivalent block method: one batched Γ-apply Z = ΓȲ, then two Gram passes
// (G₁ = ȲᵀZ, G₂ = Q̄₁ᵀZ₁ on DMMA) each followed by a small host eigensolve, dropping
// Gram directions below 1e-13·max (the rank-revealing counterpart of the reference's
// 1e-12 norm-ratio drop).  The second pass needs no new Γ-apply because ΓQ̄₁ = Z·W₁.
// Two-pass core T = Qᵀ(AQ) = (HQ)ᵀ(HQ)/σ².

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <string>

#include "eig.cuh"
#include "filter.cuh"
#include "gemv.cuh"
#include "host_linalg.h"
#include "smallchol.cuh"
#include "cappcg.cuh"

namespace fkb {

// --------------------------------------------------------------------------- small kernels
__global__ void k_densify_rows(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                               int row0, int nrows, double* __restrict__ out, long long ld) {
    const int r = blockIdx.y;
    if (r >= nrows) return;
    const int e0 = rp[row0 + r], e1 = rp[row0 + r + 1];
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) out[ci[e] + (long long)r * ld] = v[e];
}

__global__ void k_symmetrize(double* A, int n, long long lda) {  // A = ½(A + Aᵀ)
    const long long total = (long long)n * n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int i = int(e % n), j = int(e / n);
        if (i <= j) continue;
        const double v = 0.5 * (A[i + (long long)j * lda] + A[j + (long long)i * lda]);
        A[i + (long long)j * lda] = v;
        A[j + (long long)i * lda] = v;
    }
}

// out[:, i] = in[:, ncol − 1 − i] (n rows, ld n; blockIdx.y = i; ncol = n here)
__global__ void k_reverse_cols(int n, const double* __restrict__ in, int ncol, double* __restrict__ out) {
    const int i = blockIdx.y, r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) out[r + (long long)i * n] = in[r + (long long)(ncol - 1 - i) * n];
}

__global__ void k_colsq(long long n, const double* __restrict__ U, double* __restrict__ out) {
    const double* u = U + (long long)blockIdx.x * n;
    double s = 0.0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) s = fma(u[i], u[i], s);
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) out[blockIdx.x] = s;
    }
}

// out (cols×rows... row-major copy): out[i·r + j] = in[i + j·n]  (32×32 tiles through smem)
__global__ void k_transpose(long long n, int r, const double* __restrict__ in, double* __restrict__ out) {
    __shared__ double t[32][33];
    const long long i0 = blockIdx.x * 32LL;
    const int j0 = blockIdx.y * 32;
    for (int q = threadIdx.y; q < 32; q += blockDim.y) {
        const long long i = i0 + threadIdx.x;
        const int j = j0 + q;
        t[q][threadIdx.x] = (i < n && j < r) ? in[i + (long long)j * n] : 0.0;
    }
    __syncthreads();
    for (int q = threadIdx.y; q < 32; q += blockDim.y) {
        const long long i = i0 + q;
        const int j = j0 + threadIdx.x;
        if (i < n && j < r) out[i * r + j] = t[threadIdx.x][q];
    }
}

// Step prologue (fast_filter.hpp:97, :108): α ← α + 1, the PCG fallback flag cleared, Woodbury
// scalars wsq_i = 1/(α θ_i + σ²) (Λ_M⁻¹) and sqd_j = √d_j (when wsq ≠ null), a snapshot of the
// committed d for the side branch that forms the next step's capacitance (dsnap ≠ null; the
// step's own epilogue overwrites d concurrently), and the residual z = y − H·mean.
// The failure flag *info is sticky: a failed step leaves it set, so every later step of an
// asynchronous batch is a no-op (its epilogues are gated on it) until the host clears it.
// The observation: y, or (ysrc set) row ysrc[2] of the block at ysrc[0] with ld ysrc[1] — the
// host batch (Filter::run_host) uploads all its observations once.
//
// The residual is taken from the carried image of the mean, hm = H·mean: z = y − hm, no pass
// over H.  The step keeps hm current without H either: S z = y − H·mean
// with S = H·Σ_pred·Hᵀ + σ²I, so H·mean_new = H·mean + H·Σ_pred·Hᵀz = y − σ²z exactly (the
// rotate-out epilogue EpiZHm stores it; rounding as the reference's own H·mean, plus the
// solve's residual).  The next step's chain therefore does not wait for
// this step's N-space mean update.  Also: the observation copied to ycur (EpiZHm reads it
// after the batch row has advanced), the parity's commit gate closed (gate = 1 until the
// step's epilogue commits), and the host batch's observation row ysrc[2] advanced by the last
// CTA to finish (every CTA has read the row by then).
__global__ void __launch_bounds__(256) k_step_prologue(int m, int r, const double* y, const double* __restrict__ hm,
                                                      double* __restrict__ z, double* __restrict__ ycur,
                                                      double* alpha_dev, const double* __restrict__ theta,
                                                      const double* __restrict__ d, double sigma2,
                                                      double* __restrict__ wsq, double* __restrict__ sqd,
                                                      double* __restrict__ dsnap, int* __restrict__ pcgflag,
                                                      long long* ysrc, int* __restrict__ gate, unsigned* ticket) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // rotate_in may stage P now
    const int gid = blockIdx.x * blockDim.x + threadIdx.x, nthreads = gridDim.x * blockDim.x;
    const double alpha = alpha_dev[0] + 1.0;
    if (gid == 0) {
        alpha_dev[1] = alpha;
        if (pcgflag) *pcgflag = 0;
        *gate = 1;
    }
    if (dsnap)
        for (int j = gid; j < r; j += nthreads) dsnap[j] = d[j];
    if (wsq) {
        for (int i = gid; i < m; i += nthreads) wsq[i] = 1.0 / (alpha * theta[i] + sigma2);
        for (int j = gid; j < r; j += nthreads) sqd[j] = sqrt(d[j]);
    }
    if (ysrc) y = reinterpret_cast<const double*>(ysrc[0]) + ysrc[2] * ysrc[1];
    for (int i = gid; i < m; i += nthreads) {
        const double yi = y[i];
        ycur[i] = yi;
        z[i] = yi - hm[i];
    }
    if (ysrc) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
                *ticket = 0;
                ysrc[2] += 1;
            }
        }
    }
}

// rotate-out epilogue: z_i = (P·s̃)_i and, unless the step failed, the image of the new mean
// hm_i = y_i − σ²z_i (see k_step_prologue)
struct EpiZHm {
    double* z;
    double* hm;
    const double* ycur;
    double sigma2;
    const int* info;
    __device__ __forceinline__ void operator()(long long i, double v) const {
        z[i] = v;
        if (!*info) hm[i] = ycur[i] - sigma2 * v;
    }
};
__global__ void k_image_update(int m, const double* __restrict__ z, double* __restrict__ hm,
                               const double* __restrict__ ycur, double sigma2, const int* __restrict__ info) {
    if (*info) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        hm[i] = ycur[i] - sigma2 * z[i];
}

// Woodbury scalars wsq_i = 1/(α θ_i + σ²) (Λ_M⁻¹) and sqd_j = √d_j for a step that has not
// run yet.  mode 0: α = α_dev[0] + 1 with the committed d; mode 1 (side branch of step t): the
// step after t, α = α_dev[1] + 1 and d_j advanced by the same SMW update the step commits
// (fast_filter.hpp:118-123; d does not depend on the observation).
__global__ void k_woodbury_scalars(int m, int r, int mode, const double* __restrict__ alpha_dev,
                                   const double* __restrict__ theta, const double* __restrict__ d,
                                   const double* __restrict__ lam, double sigma2, double* __restrict__ wsq,
                                   double* __restrict__ sqd, int* __restrict__ cert) {
    if (cert && blockIdx.x == 0 && threadIdx.x == 0) *cert = 0;  // k_cap_certificate ORs into it
    const double a_step = mode == 0 ? alpha_dev[0] + 1.0 : alpha_dev[1];
    const double alpha = mode == 0 ? a_step : a_step + 1.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
        wsq[i] = 1.0 / (alpha * theta[i] + sigma2);
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < r; j += gridDim.x * blockDim.x) {
        double dj = d[j];
        if (mode == 1) {
            const double c = a_step - dj, l = lam[j];
            dj = (dj + a_step * l * c) / (1.0 + l * c);
        }
        sqd[j] = sqrt(dj);
    }
}

// Positive-definiteness certificate of the capacitance K (side branch, next to its Gram): by
// Gershgorin, K is SPD if every row is strictly diagonally dominant — either as it stands or
// after the symmetric Jacobi scaling D^{-½}KD^{-½} (unit diagonal).  *cert = 0 when either
// test holds for every row, else 1; the step's PCG then gives up at once and the step is rerun
// on the exact Cholesky path, so a K the Krylov space would not expose as indefinite still
// gets the reference LLT's verdict (fast_filter.hpp:104-106).  A warp per row, failures
// OR-ed into the flag (zeroed by k_woodbury_scalars earlier on the same branch); bit 0: the
// unscaled test failed somewhere, bit 1: the scaled one — certified iff not both.
__global__ void __launch_bounds__(256) k_cap_certificate(int r, const double* __restrict__ K, int* __restrict__ cert,
                                                        int force_fail) {
    extern __shared__ double rdiag[];  // 1/√K_jj
    for (int j = threadIdx.x; j < r; j += blockDim.x) {
        const double kjj = K[j + (long long)j * r];
        rdiag[j] = kjj > 0.0 ? rsqrt(kjj) : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= r) return;
    const double* col = K + (long long)i * r;  // column i = row i (symmetric)
    double sa = 0.0, sb = 0.0;
    for (int j = lane; j < r; j += 32) {
        const double a = j == i ? 0.0 : fabs(col[j]);
        sa += a;
        sb = fma(a, rdiag[j], sb);
    }
    for (int o = 16; o > 0; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    if (lane == 0) {
        const double kii = col[i];
        const int f = (!(kii - sa > 0.0) ? 1 : 0) | ((!(rdiag[i] > 0.0) || !(1.0 - sb * rdiag[i] > 0.0)) ? 2 : 0);
        if (f || (force_fail && i == 0)) atomicOr(cert, force_fail ? 3 : f);
    }
}

// Second-chance certificate: a K that fails both Gershgorin tests (c1 has such steps) is
// factored — a copy, the PCG needs K intact — by the cluster Cholesky on the side branch; a
// clean factorization certifies it.  Idle (early exit) whenever Gershgorin succeeded.
__global__ void k_cert_prepare(int r, const double* __restrict__ K, double* __restrict__ Kc, const int* __restrict__ cert,
                               int* __restrict__ gate, int* __restrict__ cinfo) {
    const bool run = *cert == 3;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *gate = run ? 1 : 0;
        *cinfo = 0;
    }
    if (!run) return;
    const long long total = (long long)r * r;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
        Kc[e] = K[e];
}
__global__ void k_cert_finish(int* __restrict__ cert, const int* __restrict__ gate, const int* __restrict__ cinfo) {
    if (*gate && *cinfo == 0) *cert = 0;
}

// u_j = sqd_j · v  (capacitance right-hand side from the column dot Eᵀ(Λ_M⁻¹ r̃); Λ_M⁻¹ and D^½
// of this step were formed by the previous step's side branch)
struct EpiScaleOut {
    double* u;
    const double* sc;
    __device__ __forceinline__ void operator()(long long j, double v) const { u[j] = sc[j] * v; }
};
// (Bᵀz)_j → dc_j = d_j·(Bᵀz)_j for the mean update, then d_j ← (d_j + αλ_j(α − d_j)) /
// (1 + λ_j(α − d_j)) (fast_filter.hpp:114-123); column 0 commits α.  Skipped when the step
// failed (*info).
struct EpiCtzD {
    double* dc;
    double* d;
    const double* lam;
    double* alpha_dev;
    const int* info;
    const unsigned long long* hout;  // [1]: mapped pinned host d (0 = none), see Filter::hostout
    // the parity's snapshots for a deferred mean side (Filter::enqueue_mean_side): the step's α,
    // the commit gate (0 = committed) and, for the fused UQ pass, the new d
    double* alpha_q;
    int* gate_q;
    double* d_q;
    __device__ __forceinline__ void commit(long long j, double alpha, double dn) const {
        d[j] = dn;
        if (d_q) d_q[j] = dn;
        if (hout[1]) reinterpret_cast<double*>(hout[1])[j] = dn;
        if (j == 0) {
            alpha_dev[0] = alpha;
            *alpha_q = alpha;
            *gate_q = 0;
        }
    }
    __device__ __forceinline__ void operator()(long long j, double v) const {
        if (*info) return;
        const double alpha = alpha_dev[1];
        const double dj = d[j], l = lam[j], c = alpha - dj;
        dc[j] = dj * v;
        commit(j, alpha, (dj + alpha * l * c) / (1.0 + l * c));
    }
    // dc_j = sqd_j·x_j given directly (Woodbury path), then the same d/α commit
    __device__ __forceinline__ void operator()(long long j, double xj, double sqdj) const {
        if (*info) return;
        const double alpha = alpha_dev[1];
        const double dj = d[j], l = lam[j], c = alpha - dj;
        dc[j] = sqdj * xj;
        commit(j, alpha, (dj + alpha * l * c) / (1.0 + l * c));
    }
};

// s̃_i = wsq_i · (r̃_i + Σ_j E_ij · (sqd_j · x_j))   ([Λ_M − EDEᵀ]⁻¹ r̃ via Woodbury); warp per
// row of the row-major E copy, every load of the row in flight.
// The extra last CTA forms the mean update's coefficients and commits d and α: with
// u = D^½EᵀΛ_M⁻¹r̃ and K = I − D^½EᵀΛ_M⁻¹ED^½, D^½Eᵀs̃ = u + (I − K)x = x, so
// d ⊙ Bᵀz = d ⊙ EᵀPᵀP s̃ = D^½x — no pass over B or E (fast_filter.hpp:114-123)
__global__ void __launch_bounds__(256) k_woodbury_st(int m, int r, const double* __restrict__ Erow,
                                                    const double* __restrict__ sqd, const double* __restrict__ x,
                                                    const double* __restrict__ wsq, const double* __restrict__ rt,
                                                    double* __restrict__ st, EpiCtzD upd) {
    if (blockIdx.x == gridDim.x - 1) {
        for (int j = threadIdx.x; j < r; j += blockDim.x) upd(j, x[j], sqd[j]);
        return;
    }
    const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (i >= m) return;
    const double* er = Erow + (long long)i * r;
    double acc = 0.0;
    for (int j0 = 0; j0 < r; j0 += 32 * 16) {
        double e[16], y[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int j = j0 + lane + 32 * q;
            e[q] = j < r ? er[j] : 0.0;
            y[q] = j < r ? sqd[j] * x[j] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) acc = fma(e[q], y[q], acc);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) st[i] = wsq[i] * (rt[i] + acc);
}

// The same product launched as a programmatic dependent of the PCG cluster: its CTAs become
// resident while the 16-SM PCG runs and load their rows of E, Λ_M⁻¹ and r̃ (none depend on the
// solve), then wait for the PCG grid (griddepcontrol.wait) and read only x.
__global__ void __launch_bounds__(256) k_woodbury_st_pdl(int m, int r, const double* __restrict__ Erow,
                                                        const double* __restrict__ sqd, const double* __restrict__ x,
                                                        const double* __restrict__ wsq, const double* rt,
                                                        double* __restrict__ st, EpiCtzD upd, int rt_late) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // rotate_out may stage Pᵀ now
    if (blockIdx.x == gridDim.x - 1) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int j = threadIdx.x; j < r; j += blockDim.x) upd(j, x[j], sqd[j]);
        return;
    }
    const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    const bool on = i < m;
    const double* er = Erow + (long long)(on ? i : 0) * r;
    constexpr int NQ = 16;  // r ≤ 512 held in registers across the wait
    double e[NQ], sq[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int j = lane + 32 * q;
        e[q] = (on && j < r) ? er[j] : 0.0;
        sq[q] = j < r ? __ldg(sqd + j) : 0.0;
    }
    // rt_late: r̃ comes from a rotate_in that runs beside the PCG (early-PCG graphs) — read it
    // only once the PCG, which waited for it, has completed
    const double wi = on ? wsq[i] : 0.0;
    double ri = (on && !rt_late) ? rt[i] : 0.0;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (on && rt_late) ri = *reinterpret_cast<const volatile double*>(rt + i);
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const int j = lane + 32 * q;
        acc = fma(e[q], j < r ? sq[q] * x[j] : 0.0, acc);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (on && lane == 0) st[i] = wi * (ri + acc);
}

// d'_i = (d_i + αλ_i(α − d_i)) / (1 + λ_i(α − d_i))  (fast_filter.hpp:118-123); commits α
__global__ void k_d_update(int r, double* __restrict__ d, const double* __restrict__ lam, double* alpha_dev,
                           const int* __restrict__ info, double* alpha_q, int* gate_q) {
    if (*info) return;
    const double alpha = alpha_dev[1];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < r; i += gridDim.x * blockDim.x) {
        const double c = alpha - d[i];
        const double l = lam[i];
        d[i] = (d[i] + alpha * l * c) / (1.0 + l * c);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        alpha_dev[0] = alpha;
        *alpha_q = alpha;
        *gate_q = 0;
    }
}

// diag Σ and conditional realizations from one pass over U (uq.hpp:16-23, App. A.4):
//   var_i = αθ − Σ_j d_j U_ij²;  x_s,i = mean_i + (√α z_s,i − √α Σ_j U_ij Σ₋_j (Ūᵀz_s)_j)
__global__ void __launch_bounds__(256) k_uq(long long n, int r, const double* __restrict__ U,
                                           const double* __restrict__ d, const double* __restrict__ alpha_dev,
                                           double theta, const double* __restrict__ mean, int count,
                                           const double* __restrict__ Z, const double* __restrict__ proj,
                                           double* __restrict__ X, double* __restrict__ var) {
    extern __shared__ double sh[];
    double* ds = sh;          // r
    double* P = sh + r;       // r × count
    const double alpha = alpha_dev[0];
    for (int j = threadIdx.x; j < r; j += blockDim.x) {
        ds[j] = d[j];
        const double sm = alpha == 0.0 ? 0.0 : 1.0 - sqrt(fmax(1.0 - d[j] / alpha, 0.0));  // uq.hpp:59-64
        for (int s = 0; s < count; ++s) P[j * count + s] = sm * proj[j + (long long)s * r];
    }
    __syncthreads();
    const double ra = sqrt(alpha);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double vs = 0.0;
        double acc[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) acc[s] = 0.0;
        int j0 = 0;
        for (; j0 + 8 <= r; j0 += 8) {  // 8 coalesced column loads in flight per thread
            double u[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) u[q] = __ldcs(U + i + (long long)(j0 + q) * n);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int j = j0 + q;
                vs = fma(u[q] * u[q], ds[j], vs);
#pragma unroll
                for (int s = 0; s < 8; ++s)
                    if (s < count) acc[s] = fma(u[q], P[j * count + s], acc[s]);
            }
        }
        for (int j = j0; j < r; ++j) {
            const double u = U[i + (long long)j * n];
            vs = fma(u * u, ds[j], vs);
#pragma unroll
            for (int s = 0; s < 8; ++s)
                if (s < count) acc[s] = fma(u, P[j * count + s], acc[s]);
        }
        if (var) var[i] = alpha * theta - vs;
        if (count == 0) continue;  // variance only (mean may be null)
        const double mi = mean[i];
#pragma unroll
        for (int s = 0; s < 8; ++s)
            if (s < count) {
                const double z = Z[i + (long long)s * n];
                X[i + (long long)s * n] = alpha == 0.0 ? mi : mi + (ra * z - ra * acc[s]);
            }
    }
}

// The step's U pass fused with the UQ of the new state (c3-style workloads: diag Σ and
// `count` conditional realizations after every step): per row i of the column-major U,
//   mean_i ← (mean_i + α·t_i) − Σ_j U_ij dc_j                      (fast_filter.hpp:114-116)
//   var_i = αθ − Σ_j d_j U_ij²,  x_s,i = mean_i + √α(z_s,i − Σ_j U_ij Σ₋_j (Ūᵀz_s)_j)
// with α, d already updated for this step (α_dev[1]; d by the Woodbury epilogue), one thread
// per row and 16 coalesced column loads in flight (the default shape; k_mean_uq below holds
// the shared-memory-record variants).  The failure flag gates every write, as EpiMean, and is
// published to the mapped host slot.
__global__ void __launch_bounds__(128, 3) k_mean_uq1(long long n, int r, const double* __restrict__ U,
                                                   const double* __restrict__ dc, const double* __restrict__ d,
                                                   const double* __restrict__ alpha_dev, double theta,
                                                   const double* __restrict__ t, double* __restrict__ mean, int count,
                                                   const double* __restrict__ Z, const double* __restrict__ proj,
                                                   double* __restrict__ X, double* __restrict__ var,
                                                   const int* __restrict__ info,
                                                   const unsigned long long* __restrict__ hout,
                                                   long long* __restrict__ ycnt) {
    extern __shared__ double sh[];
    double* cs = sh;           // dc (r)
    double* ds = sh + r;       // d  (r)
    double* P = sh + 2 * r;    // Σ₋ ⊙ Ūᵀz_s (r × count)
    const int bad = *info;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (hout[2]) *reinterpret_cast<volatile int*>(hout[2]) = bad;
        if (ycnt) *ycnt += 1;  // the host batch's next observation row (see k_step_prologue)
    }
    if (bad) return;
    const double alpha = alpha_dev[1];
    for (int j = threadIdx.x; j < r; j += blockDim.x) {
        cs[j] = dc[j];
        ds[j] = d[j];
        const double sm = 1.0 - sqrt(fmax(1.0 - d[j] / alpha, 0.0));  // uq.hpp:59-64
        for (int s = 0; s < count; ++s) P[j * count + s] = sm * proj[j + (long long)s * r];
    }
    __syncthreads();
    const double ra = sqrt(alpha);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double vm = 0.0, vs = 0.0;
        double acc[8];
#pragma unroll
        for (int s = 0; s < 8; ++s) acc[s] = 0.0;
        int j0 = 0;
        for (; j0 + 16 <= r; j0 += 16) {  // 16 coalesced column loads in flight per thread
            double u[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) u[q] = __ldcs(U + i + (long long)(j0 + q) * n);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int j = j0 + q;
                vm = fma(u[q], cs[j], vm);
                vs = fma(u[q] * u[q], ds[j], vs);
#pragma unroll
                for (int s = 0; s < 8; ++s)
                    if (s < count) acc[s] = fma(u[q], P[j * count + s], acc[s]);
            }
        }
        for (int j = j0; j < r; ++j) {
            const double u = U[i + (long long)j * n];
            vm = fma(u, cs[j], vm);
            vs = fma(u * u, ds[j], vs);
#pragma unroll
            for (int s = 0; s < 8; ++s)
                if (s < count) acc[s] = fma(u, P[j * count + s], acc[s]);
        }
        const double mi = (mean[i] + alpha * t[i]) - vm;
        mean[i] = mi;
        if (hout[0]) reinterpret_cast<double*>(hout[0])[i] = mi;
        double* vo = hout[4] ? reinterpret_cast<double*>(hout[4]) : var;  // mapped host or device
        double* xo = hout[3] ? reinterpret_cast<double*>(hout[3]) : X;
        if (vo) vo[i] = alpha * theta - vs;
#pragma unroll
        for (int s = 0; s < 8; ++s)
            if (s < count) {
                const double z = Z[i + (long long)s * n];
                xo[i + (long long)s * n] = mi + (ra * z - ra * acc[s]);
            }
    }
}

// The step's U pass fused with the UQ of the new state (c3-style workloads: diag Σ and
// `count` conditional realizations after every step): per row i of the column-major U,
//   mean_i ← (mean_i + α·t_i) − Σ_j U_ij dc_j                      (fast_filter.hpp:114-116)
//   var_i = αθ − Σ_j d_j U_ij²,  x_s,i = mean_i + √α(z_s,i − Σ_j U_ij Σ₋_j (Ūᵀz_s)_j)
// with α, d already updated for this step (α_dev[1]; d by the Woodbury epilogue).  Each thread
// owns R rows 128 apart (a warp reads 256 B of a column per load, 8·R loads in flight); the
// per-column constants (dc_j, d_j and the CNT projections) sit in shared memory as one record
// per column, read with 16-byte broadcasts and reused over the R rows — the shared-memory
// issue rate, not HBM, bounded the one-row version.  The failure flag gates every write, as
// EpiMean, and is published to the mapped host slot.
template <int CNT, int R, int JB>
__global__ void __launch_bounds__(128, 3) k_mean_uq(long long n, int r, const double* __restrict__ U,
                                                   const double* __restrict__ dc, const double* __restrict__ d,
                                                   const double* __restrict__ alpha_dev, double theta,
                                                   const double* __restrict__ t, double* __restrict__ mean,
                                                   const double* __restrict__ Z, const double* __restrict__ proj,
                                                   double* __restrict__ X, double* __restrict__ var,
                                                   const int* __restrict__ info,
                                                   const unsigned long long* __restrict__ hout,
                                                   long long* __restrict__ ycnt) {
    constexpr int SW = (2 + CNT + 1) & ~1;  // record: dc, d, Σ₋⊙Ūᵀz_s (s < CNT), pad
    extern __shared__ double2 rec2[];
    double* rec = reinterpret_cast<double*>(rec2);
    const int bad = *info;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (hout[2]) *reinterpret_cast<volatile int*>(hout[2]) = bad;
        if (ycnt) *ycnt += 1;  // the host batch's next observation row (see k_step_prologue)
    }
    if (bad) return;
    const double alpha = alpha_dev[1];
    const int rp = (r + 15) / 16 * 16;
    for (int j = threadIdx.x; j < rp; j += blockDim.x) {
        double* q = rec + (long long)j * SW;
        const bool in = j < r;
        const double dj = in ? d[j] : 0.0;
        q[0] = in ? dc[j] : 0.0;
        q[1] = dj;
        const double sm = in ? 1.0 - sqrt(fmax(1.0 - dj / alpha, 0.0)) : 0.0;  // uq.hpp:59-64
#pragma unroll
        for (int s = 0; s < CNT; ++s) q[2 + s] = in ? sm * proj[j + (long long)s * r] : 0.0;
        if (SW > 2 + CNT) q[SW - 1] = 0.0;
    }
    __syncthreads();
    const double ra = sqrt(alpha);
    double* vo = hout[4] ? reinterpret_cast<double*>(hout[4]) : var;  // mapped host or device
    double* xo = hout[3] ? reinterpret_cast<double*>(hout[3]) : X;
    const long long span = (long long)blockDim.x * R;
    for (long long i0 = blockIdx.x * span + threadIdx.x; i0 < n; i0 += (long long)gridDim.x * span) {
        double vm[R], vs[R], acc[R][CNT > 0 ? CNT : 1];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            vm[q] = vs[q] = 0.0;
#pragma unroll
            for (int s = 0; s < CNT; ++s) acc[q][s] = 0.0;
        }
        for (int j0 = 0; j0 < r; j0 += JB) {
            double u[R][JB];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const long long i = i0 + q * (long long)blockDim.x;
#pragma unroll
                for (int c = 0; c < JB; ++c)
                    u[q][c] = (i < n && j0 + c < r) ? __ldcs(U + i + (long long)(j0 + c) * n) : 0.0;
            }
#pragma unroll
            for (int c = 0; c < JB; ++c) {
                const double2* p = rec2 + (long long)(j0 + c) * (SW / 2);
                const double2 cd = p[0];
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    vm[q] = fma(u[q][c], cd.x, vm[q]);
                    vs[q] = fma(u[q][c] * u[q][c], cd.y, vs[q]);
                }
#pragma unroll
                for (int s = 0; s + 1 < CNT; s += 2) {
                    const double2 pp = p[1 + s / 2];
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        acc[q][s] = fma(u[q][c], pp.x, acc[q][s]);
                        acc[q][s + 1] = fma(u[q][c], pp.y, acc[q][s + 1]);
                    }
                }
                if constexpr (CNT & 1) {
                    const double pl = p[1 + CNT / 2].x;
#pragma unroll
                    for (int q = 0; q < R; ++q) acc[q][CNT - 1] = fma(u[q][c], pl, acc[q][CNT - 1]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const long long i = i0 + q * (long long)blockDim.x;
            if (i >= n) continue;
            const double mi = (mean[i] + alpha * t[i]) - vm[q];
            mean[i] = mi;
            if (hout[0]) reinterpret_cast<double*>(hout[0])[i] = mi;
            if (vo) vo[i] = alpha * theta - vs[q];
#pragma unroll
            for (int s = 0; s < CNT; ++s) {
                const double z = Z[i + (long long)s * n];
                xo[i + (long long)s * n] = mi + (ra * z - ra * acc[q][s]);
            }
        }
    }
}

// The fused U pass + UQ on the FP64 tensor path: the per-row products with the count
// projections, acc_s = Σ_j U_ij·(Σ₋⊙Ūᵀz_s)_j (s < 8), are an N×r by r×8 product — one DMMA
// m8n8k4 per 8 rows × 4 columns of U — while U·dc and Σ_j d_j U_ij² ride along on the same
// A-fragment registers (DFMA).  A warp owns 32 rows (four m-tiles); lane (g = lane/4,
// q = lane%4) holds U[row 8t+g, col j0+q], i.e. 4 × 64-byte column segments per load
// instruction; 4 k-steps (16 loads) in flight.  The B fragment (P[j0+q][g]), dc and d come
// from shared memory (one LDS each per k-step).  Removes the per-element shared-memory
// broadcasts that bounded k_mean_uq1.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__global__ void __launch_bounds__(256, 2) k_mean_uq_mma(long long n, int r, const double* __restrict__ U,
                                                       const double* __restrict__ dc, const double* __restrict__ d,
                                                       const double* __restrict__ alpha_dev, double theta,
                                                       const double* __restrict__ t, double* __restrict__ mean,
                                                       int count, const double* __restrict__ Z,
                                                       const double* __restrict__ proj, double* __restrict__ X,
                                                       double* __restrict__ var, const int* __restrict__ info,
                                                       const unsigned long long* __restrict__ hout,
                                                       long long* __restrict__ ycnt) {
    extern __shared__ double msm[];
    const int r4 = (r + 15) & ~15;  // k-steps of 4, unrolled by 4
    double* Bt = msm;               // [r4][8]
    double* dcs = Bt + (size_t)r4 * 8;
    double* ds = dcs + r4;
    const int bad = *info;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (hout[2]) *reinterpret_cast<volatile int*>(hout[2]) = bad;
        if (ycnt) *ycnt += 1;
    }
    if (bad) return;
    const double alpha = alpha_dev[1];
    for (int j = threadIdx.x; j < r4; j += blockDim.x) {
        const bool in = j < r;
        const double dj = in ? d[j] : 0.0;
        dcs[j] = in ? dc[j] : 0.0;
        ds[j] = dj;
        const double sm = in ? 1.0 - sqrt(fmax(1.0 - dj / alpha, 0.0)) : 0.0;  // uq.hpp:59-64
        for (int s2 = 0; s2 < 8; ++s2) Bt[j * 8 + s2] = (in && s2 < count) ? sm * proj[j + (long long)s2 * r] : 0.0;
    }
    __syncthreads();
    const double ra = sqrt(alpha);
    double* vo = hout[4] ? reinterpret_cast<double*>(hout[4]) : var;
    double* xo = hout[3] ? reinterpret_cast<double*>(hout[3]) : X;
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    const long long wstride = (long long)gridDim.x * (blockDim.x >> 5) * 32;
    for (long long i0 = ((long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; i0 < n; i0 += wstride) {
        double acc[4][2], vm[4], vs[4];
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) acc[tt][0] = acc[tt][1] = vm[tt] = vs[tt] = 0.0;
        bool rin[4];
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) rin[tt] = i0 + 8 * tt + g < n;
        for (int j0 = 0; j0 < r4; j0 += 16) {
            double a[4][4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int j = j0 + 4 * kk + q;
#pragma unroll
                for (int tt = 0; tt < 4; ++tt)
                    a[kk][tt] = (j < r && rin[tt]) ? __ldcs(U + (long long)j * n + i0 + 8 * tt + g) : 0.0;
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int j = j0 + 4 * kk + q;
                const double b = Bt[(j0 + 4 * kk + q) * 8 + g];
                const double cj = dcs[j], dj = ds[j];
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) {
                    dmma884(acc[tt][0], acc[tt][1], a[kk][tt], b);
                    vm[tt] = fma(a[kk][tt], cj, vm[tt]);
                    vs[tt] = fma(a[kk][tt] * a[kk][tt], dj, vs[tt]);
                }
            }
        }
#pragma unroll
        for (int tt = 0; tt < 4; ++tt) {
            // the row's four column classes q: fixed butterfly (same sum in all four lanes)
            vm[tt] += __shfl_xor_sync(0xffffffffu, vm[tt], 1);
            vm[tt] += __shfl_xor_sync(0xffffffffu, vm[tt], 2);
            vs[tt] += __shfl_xor_sync(0xffffffffu, vs[tt], 1);
            vs[tt] += __shfl_xor_sync(0xffffffffu, vs[tt], 2);
            if (!rin[tt]) continue;
            const long long i = i0 + 8 * tt + g;
            const double mi = (mean[i] + alpha * t[i]) - vm[tt];
            if (q == 0) {
                mean[i] = mi;
                if (hout[0]) reinterpret_cast<double*>(hout[0])[i] = mi;
                if (vo) vo[i] = alpha * theta - vs[tt];
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int s2 = 2 * q + h;
                if (s2 < count) {
                    const double z = Z[i + (long long)s2 * n];
                    xo[i + (long long)s2 * n] = mi + (ra * z - ra * acc[tt][h]);
                }
            }
        }
    }
}

void launch_mean_uq(int count, long long n, int r, const double* U, const double* dc, const double* d,
                    const double* alpha_dev, double theta, const double* t, double* mean, const double* Z,
                    const double* proj, double* X, double* var, const int* info, const unsigned long long* hout,
                    long long* ycnt, cudaStream_t s) {
    // FKB_UQ_SHAPE: 9 (default) k_mean_uq_mma — the projections on DMMA; 0 k_mean_uq1 — one
    // row per thread, separate constant arrays; 116 / 208 — shared-memory records, 1 row × 16
    // or 2 rows × 8 columns per batch (c3, in graph: 53 / 64 / 80 / 68 µs)
    static const int shape = [] {
        const char* e = std::getenv("FKB_UQ_SHAPE");
        return e ? std::atoi(e) : 9;
    }();
    auto go = [&](auto c) {
        constexpr int CNT = decltype(c)::value;
        constexpr int SW = (2 + CNT + 1) & ~1;
        const size_t shm = sizeof(double) * size_t((r + 15) / 16 * 16) * SW;
        auto launch = [&](auto kern, int R) {  // (one lambda type per CNT: the attribute is set per call)
            FKB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            kern<<<ceil_div(n, 128 * R), 128, shm, s>>>(n, r, U, dc, d, alpha_dev, theta, t, mean, Z, proj, X, var,
                                                       info, hout, ycnt);
        };
        if (shape == 9) {  // the DMMA pass (k_mean_uq_mma)
            const int r16 = (r + 15) & ~15;
            const size_t shm9 = sizeof(double) * size_t(r16) * 10;
            FKB_CUDA(cudaFuncSetAttribute(k_mean_uq_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            int dev = 0, sms = 0;
            FKB_CUDA(cudaGetDevice(&dev));
            FKB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            const long long warps = (n + 31) / 32;
            const int grid = int(std::min<long long>((warps + 7) / 8, 2LL * sms));
            k_mean_uq_mma<<<grid, 256, shm9, s>>>(n, r, U, dc, d, alpha_dev, theta, t, mean, count, Z, proj, X, var,
                                                  info, hout, ycnt);
        } else if (shape == 208) launch(k_mean_uq<CNT, 2, 8>, 2);
        else if (shape == 116) launch(k_mean_uq<CNT, 1, 16>, 1);
        else {
            const size_t shm1 = sizeof(double) * size_t(r) * (2 + std::max(count, 1));
            k_mean_uq1<<<ceil_div(n, 128), 128, shm1, s>>>(n, r, U, dc, d, alpha_dev, theta, t, mean, count, Z, proj,
                                                           X, var, info, hout, ycnt);
        }
    };
    switch (count) {
        case 0: go(std::integral_constant<int, 0>{}); break;
        case 1: go(std::integral_constant<int, 1>{}); break;
        case 2: go(std::integral_constant<int, 2>{}); break;
        case 3: go(std::integral_constant<int, 3>{}); break;
        case 4: go(std::integral_constant<int, 4>{}); break;
        case 5: go(std::integral_constant<int, 5>{}); break;
        case 6: go(std::integral_constant<int, 6>{}); break;
        case 7: go(std::integral_constant<int, 7>{}); break;
        default: go(std::integral_constant<int, 8>{}); break;
    }
    FKB_LAUNCH_CHECK();
    count_launch();
}

// ghep_residual (lowrank.hpp:215-228) per pair j: ‖A u_j − λ_j Γ⁻¹u_j‖ / max(λ_j‖Γ⁻¹u_j‖, ε)
// with A u_j = Hᵀ(H u_j)/σ² (= Hᵀ B_j/σ², B = HU) and Γ⁻¹u_j = Ū_j exactly (no CG solve)
__global__ void k_gep_resid(long long n, const double* __restrict__ AU, const double* __restrict__ Ub,
                            const double* __restrict__ lam, double* __restrict__ out) {
    const int j = blockIdx.x;
    const double l = lam[j];
    const double* a = AU + (long long)j * n;
    const double* u = Ub + (long long)j * n;
    double sr = 0.0, su = 0.0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = a[i] - l * u[i];
        sr = fma(v, v, sr);
        su = fma(u[i], u[i], su);
    }
    __shared__ double red[2][32];
    for (int o = 16; o > 0; o >>= 1) {
        sr += __shfl_down_sync(0xffffffffu, sr, o);
        su += __shfl_down_sync(0xffffffffu, su, o);
    }
    if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = sr; red[1][threadIdx.x >> 5] = su; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a2 = 0.0, u2 = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a2 += red[0][w]; u2 += red[1][w]; }
        out[j] = sqrt(a2) / fmax(l * sqrt(u2), 2.220446049250313e-16);
    }
}

// --------------------------------------------------------------------------- host side
void check_nonneg_args(long long k, long long p, long long n) {  // lowrank.hpp:145-151
    if (k < 0 || p < 0) throw std::invalid_argument("randomized_ghep: k and oversampling must be nonnegative");
    if (k + p > n)
        throw std::invalid_argument("randomized_ghep: k + oversampling = " + std::to_string(k + p) +
                                    " exceeds problem size " + std::to_string(n));
}

std::vector<double> download(const double* p, size_t count, cudaStream_t s) {
    std::vector<double> h(count);
    if (count) {
        FKB_CUDA(cudaMemcpyAsync(h.data(), p, count * sizeof(double), cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaStreamSynchronize(s));
    }
    return h;
}
void upload(double* p, const std::vector<double>& h, cudaStream_t s) {
    if (!h.empty()) FKB_CUDA(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, s));
}

// Gram C = Aᵀ B for tall-skinny A (n×p), B (n×q) on DMMA with split-K
void gram_tn(long long n, int p, int q, const double* A, const double* B, double* C, DBuf<double>& ws,
                    cudaStream_t s) {
    GemmArgs g;
    g.M = p; g.N = q; g.K = int(n);
    g.A = A; g.lda = n; g.transA = 1;
    g.B = B; g.ldb = n; g.transB = 0;
    g.C = C; g.ldc = p;
    g.splitk = gemm_pick_splitk(p, q, int(n));
    ws.ensure(std::max(gemm_ws_elems(g), gram_ws_elems(p, q, int(n))));
    gram(g, ws.p, s);
}
// C (n×q) = A (n×p) · W (p×q), W on the device
void tall_times_small(long long n, int p, int q, const double* A, const double* W, double* C, cudaStream_t s) {
    GemmArgs g;
    g.M = int(n); g.N = q; g.K = p;
    g.A = A; g.lda = n;
    g.B = W; g.ldb = p;
    g.C = C; g.ldc = n;
    gemm(g, nullptr, s);
}

// Orthonormalizing transform of a small Gram G (p×p): returns W (p×kept) with WᵀGW = I.
// Well-conditioned G (every Cholesky pivot² ≥ 1e-10·max G_jj, i.e. far from the tol·max
// eigenvalue drop): W = L⁻ᵀ from G = LLᵀ (CholQR; ~p³/1.5 flops).  Otherwise the symmetric
// eigendecomposition: W = V·diag(w^{-1/2}) over eigenvalues above tol·max (rank-revealing
// drop), ordered by ascending eigenvalue.  Both span the same columns when nothing is dropped.
std::vector<double> gram_inv_sqrt(int p, const std::vector<double>& Gh, double tol, int& kept) {
    if (p > 0) {
        // L held row-major (Lr[i·p + k] = L_ik) so every dot product below runs over contiguous
        // memory; the rows of a column and the columns of the inverse are independent and run
        // on the host threads (the arithmetic order per entry is fixed: bit-identical results)
        std::vector<double> Lr(static_cast<size_t>(p) * p, 0.0);
        for (int i = 0; i < p; ++i)
            for (int j = 0; j <= i; ++j) Lr[size_t(i) * p + j] = Gh[size_t(i) + size_t(j) * p];
        double dmax = 0.0;
        for (int j = 0; j < p; ++j) dmax = std::max(dmax, Gh[size_t(j) + size_t(j) * p]);
        bool ok = dmax > 0.0;
        // left-looking Cholesky on the lower triangle; one parallel region (a fork/join per
        // column cost more than the column's work): the pivot in `single`, the rows in `for`
#pragma omp parallel if (p > 64)
        for (int j = 0; j < p; ++j) {
#pragma omp single
            {
                const double* lj = Lr.data() + size_t(j) * p;
                double dj = ok ? lj[j] : 0.0;
                for (int k = 0; k < j; ++k) dj -= lj[k] * lj[k];
                if (!(dj >= 1e-10 * dmax)) ok = false;
                else Lr[size_t(j) * p + j] = std::sqrt(dj);
            }  // implicit barrier: every thread sees ok and L_jj
            if (!ok) break;
            const double* lj = Lr.data() + size_t(j) * p;
            const double ljj = lj[j];
#pragma omp for schedule(static)
            for (int i = j + 1; i < p; ++i) {
                double* li = Lr.data() + size_t(i) * p;
                double v = 0.5 * (li[j] + Gh[size_t(j) + size_t(i) * p]);  // symmetrized entry
                for (int k = 0; k < j; ++k) v -= li[k] * lj[k];
                li[j] = v / ljj;
            }
        }
        if (ok) {
            // W = L⁻ᵀ (upper triangular): solve Lᵀ W = I column by column; Lc = L column-major
            std::vector<double> Lc(static_cast<size_t>(p) * p);
            for (int i = 0; i < p; ++i)
                for (int k = 0; k <= i; ++k) Lc[size_t(i) + size_t(k) * p] = Lr[size_t(i) * p + k];
            std::vector<double> W(static_cast<size_t>(p) * p, 0.0);
#pragma omp parallel for schedule(dynamic, 8)
            for (int c = 0; c < p; ++c) {
                double* w = W.data() + size_t(c) * p;
                for (int i = c; i >= 0; --i) {
                    const double* li = Lc.data() + size_t(i) * p;  // column i of L
                    double v = i == c ? 1.0 : 0.0;
                    for (int k = i + 1; k <= c; ++k) v -= li[k] * w[k];
                    w[i] = v / li[i];
                }
            }
            kept = p;
            return W;
        }
    }
    std::vector<double> G = Gh;
    for (int j = 0; j < p; ++j)
        for (int i = 0; i < j; ++i) G[size_t(i) + size_t(j) * p] = G[size_t(j) + size_t(i) * p] =
                                        0.5 * (G[size_t(i) + size_t(j) * p] + G[size_t(j) + size_t(i) * p]);
    std::vector<double> w(static_cast<size_t>(p)), V(static_cast<size_t>(p) * p);
    sym_eig_small(p, G.data(), w.data(), V.data());
    const double wmax = p ? w[size_t(p - 1)] : 0.0;
    std::vector<int> keep;
    if (wmax > 0.0)
        for (int j = 0; j < p; ++j)
            if (w[size_t(j)] > tol * wmax) keep.push_back(j);
    kept = int(keep.size());
    std::vector<double> W(static_cast<size_t>(p) * std::max(kept, 1));
    for (int c = 0; c < kept; ++c) {
        const double sc = 1.0 / std::sqrt(w[size_t(keep[size_t(c)])]);
        for (int i = 0; i < p; ++i) W[size_t(i) + size_t(c) * p] = V[size_t(i) + size_t(keep[size_t(c)]) * p] * sc;
    }
    return W;
}

// FKB_EKF_TRACE=1: phase times of the GHEP on stderr (stream-synchronized)
struct GhepClock {
    cudaStream_t s;
    bool on = std::getenv("FKB_EKF_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void lap(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[ekf]   %-22s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

void randomized_ghep_device(Cov* cov, const DevCsr& H, const DevCsr& HT, double sigma2, long long k, long long p,
                            uint64_t seed, DBuf<double>& ws, cudaStream_t s, GepDev& out) {
    const long long n = cov->size();
    const int m = H.rows;
    check_nonneg_args(k, p, n);
    GhepClock gclk{s};
    int& r = out.r;
    int& kept_cols = out.kept_cols;
    std::vector<double>& lambda_h = out.lambda_h;
    DBuf<double>& lambda = out.lambda;
    DBuf<double>& U = out.U;
    DBuf<double>& Ubar = out.Ubar;
    r = 0;
    kept_cols = 0;
    lambda_h.clear();
    if (k == 0) return;
    const int l = int(k + p);
    DBuf<double>& A = out.tmp(0, size_t(n) * l);
    DBuf<double>& Y = out.tmp(1, size_t(n) * l);
    DBuf<double>& HO = out.tmp(2, size_t(std::max(m, 1)) * l);
    gaussian_matrix(n, l, seed, 0, A.p, n, s);                    // Ω (lowrank.hpp:157)
    {
        // Ȳ = Hᵀ(HΩ)/σ² (:158-159) on row-major blocks: every nonzero then streams one
        // contiguous 8·l-byte row of its operand (the column-major kernel gathers 8-byte
        // pieces); Ω is transposed in, Ȳ transposed back for the column-major stages.
        k_transpose<<<dim3(ceil_div(n, 32), ceil_div(l, 32)), dim3(32, 8), 0, s>>>(n, l, A.p, Y.p);  // Ω row-major
        FKB_LAUNCH_CHECK();
        count_launch();
        spmm_rm(H, Y.p, l, l, HO.p, l, 1.0, s);                     // HΩ (row-major m×l)
        spmm_rm(HT, HO.p, l, l, A.p, l, 1.0 / sigma2, s);           // Ȳ (row-major N×l)
        k_transpose<<<dim3(ceil_div(l, 32), ceil_div(n, 32)), dim3(32, 8), 0, s>>>(l, int(n), A.p, Y.p);
        FKB_LAUNCH_CHECK();
        count_launch();
    }
    ws.ensure(4096);
    if (sumsq(Y.p, (long long)n * l, ws.p, s) == 0.0) return;     // A = 0 (:161)
    gclk.lap("ghep: sketch");
    DBuf<double>& Z = A;                                           // Ω no longer needed
    cov->apply(Y.p, n, l, Z.p, n);                                 // Z = ΓȲ
    DBuf<double>& Gd = out.tmp(3, size_t(l) * l);
    gram_tn(n, l, l, Y.p, Z.p, Gd.p, ws, s);                       // G₁ = ȲᵀΓȲ
    gclk.lap("ghep: gamma_x + gram1");
    int k1 = 0;
    std::vector<double> W1 = gram_inv_sqrt(l, download(Gd.p, size_t(l) * l, s), 1e-13, k1);
    gclk.lap("ghep: orth1 (host)");
    if (k1 == 0)
        throw std::runtime_error("randomized_ghep: rank collapse — every sketch column was dropped during orthonormalization");
    DBuf<double>& Wd = out.tmp(4, W1.size());
    upload(Wd.p, W1, s);
    DBuf<double>& Q1 = out.tmp(5, size_t(n) * k1);
    DBuf<double>& Z1 = out.tmp(6, size_t(n) * k1);
    tall_times_small(n, l, k1, Y.p, Wd.p, Q1.p, s);                // Q̄₁ = Ȳ W₁
    tall_times_small(n, l, k1, Z.p, Wd.p, Z1.p, s);                // ΓQ̄₁ = Z W₁
    gram_tn(n, k1, k1, Q1.p, Z1.p, Gd.p, ws, s);                   // G₂ = Q̄₁ᵀ Γ Q̄₁
    int k2 = 0;
    std::vector<double> W2 = gram_inv_sqrt(k1, download(Gd.p, size_t(k1) * k1, s), 1e-13, k2);
    gclk.lap("ghep: orth2 (host)");
    if (k2 == 0)
        throw std::runtime_error("randomized_ghep: rank collapse — every sketch column was dropped during orthonormalization");
    kept_cols = k2;
    upload(Wd.p, W2, s);
    // Q̄ = Q̄₁W₂ (into Y), Q = ΓQ̄ = Z₁W₂ (into Z)
    tall_times_small(n, k1, k2, Q1.p, Wd.p, Y.p, s);
    tall_times_small(n, k1, k2, Z1.p, Wd.p, Z.p, s);
    // T = Qᵀ(AQ) = (HQ)ᵀ(HQ)/σ², symmetrized (:186-191)
    // HQ on row-major blocks (Q transposed into the free Q̄₁ buffer, streaming ray SpMM); the
    // m×k₂ row-major result is (HQ)ᵀ column-major, so T = XXᵀ/σ² with X = (HQ)ᵀ
    transpose_cm(n, k2, Z.p, Q1.p, s);
    spmm_rm(H, Q1.p, k2, k2, HO.p, k2, 1.0, s);
    DBuf<double>& Td = out.tmp(7, size_t(k2) * k2);
    {
        GemmArgs g;
        g.M = k2; g.N = k2; g.K = m;
        g.A = HO.p; g.lda = k2; g.transA = 0;
        g.B = HO.p; g.ldb = k2; g.transB = 1;
        g.alpha = 1.0 / sigma2;
        g.C = Td.p; g.ldc = k2;
        g.splitk = gemm_pick_splitk(k2, k2, m);
        ws.ensure(gemm_ws_elems(g));
        gemm(g, ws.p, s);
    }
    symmetrize(k2, Td.p, k2, s);
    std::vector<double> ev(static_cast<size_t>(k2));
    DBuf<double>& Svd = out.tmp(8, size_t(k2) * k2);
    sym_eig_tridiag_device(k2, Td.p, ev.data(), Svd.p, s);         // (:193)
    gclk.lap("ghep: T eig");
    const int kk = int(std::min<long long>(k, k2));                // (:197-205)
    r = kk;
    lambda_h.resize(size_t(kk));
    for (int i = 0; i < kk; ++i) lambda_h[size_t(i)] = std::max(ev[size_t(k2 - 1 - i)], 0.0);
    Wd.ensure(size_t(k2) * std::max(kk, 1));
    if (kk > 0)  // S = eigenvectors in descending order: columns k2−1 … k2−kk
        k_reverse_cols<<<dim3(ceil_div(k2, 256), kk), 256, 0, s>>>(k2, Svd.p, k2, Wd.p);
    FKB_LAUNCH_CHECK();
    count_launch();
    lambda.ensure(size_t(std::max(kk, 1)));
    upload(lambda.p, lambda_h, s);
    U.ensure(size_t(n) * std::max(kk, 1));
    Ubar.ensure(size_t(n) * std::max(kk, 1));
    tall_times_small(n, k2, kk, Z.p, Wd.p, U.p, s);                // U = Q S
    tall_times_small(n, k2, kk, Y.p, Wd.p, Ubar.p, s);             // Ū = Q̄ S = Γ⁻¹U
    FKB_CUDA(cudaStreamSynchronize(s));
}

void Filter::ghep(long long k, long long p, uint64_t seed) {
    GepDev g;
    randomized_ghep_device(cov, H, HT, sigma2, k, p, seed, ws, s, g);
    r = g.r;
    kept_cols = g.kept_cols;
    lambda_h = std::move(g.lambda_h);
    lambda = std::move(g.lambda);
    U = std::move(g.U);
    Ubar = std::move(g.Ubar);
}

// G = H·ΓHᵀ, symmetrized (fast_filter.hpp:68-72): ΓHᵀ streamed in column batches of ≤ 2²⁷/N
// densified rows of H, never stored.
void build_hgh(Cov* cov, const DevCsr& H, double* G, cudaStream_t s, DBuf<double>* scratch) {
    const long long n = cov->size();
    const int m = H.rows;
    if (m <= 0) return;
    const int bc = int(std::max<long long>(1, std::min<long long>(m, (1LL << 27) / std::max<long long>(n, 1))));
    DBuf<double> own;
    DBuf<double>& Ec = scratch ? *scratch : own;
    Ec.ensure(2 * size_t(n) * bc);  // ΓHᵀ batch (column-major) and its row-major copy
    double* Er = Ec.p + size_t(n) * bc;
    for (int c0 = 0; c0 < m; c0 += bc) {
        const int nb = std::min(bc, m - c0);
        FKB_CUDA(cudaMemsetAsync(Ec.p, 0, sizeof(double) * size_t(n) * nb, s));
        k_densify_rows<<<dim3(1, nb), 128, 0, s>>>(H.rowptr.p, H.col.p, H.val.p, c0, nb, Ec.p, n);
        FKB_LAUNCH_CHECK();
        count_launch();
        cov->apply(Ec.p, n, nb, Ec.p, n);
        // H·(ΓHᵀ) on row-major blocks: every nonzero streams one contiguous 8·nb-byte row (the
        // column-major SpMM would gather 8-byte pieces); the m×nb result lands transposed in
        // rows c0… of G, which is symmetric (averaged below)
        transpose_cm(n, nb, Ec.p, Er, s);
        spmm_rm(H, Er, nb, nb, G + c0, m, 1.0, s);
    }
    symmetrize(m, G, m, s);
}

void column_sumsq(long long n, int r, const double* A, double* out, cudaStream_t s) {
    if (r <= 0) return;
    k_colsq<<<r, 256, 0, s>>>(n, A, out);
    FKB_LAUNCH_CHECK();
    count_launch();
}

void transpose_cm(long long n, int r, const double* in, double* out, cudaStream_t s) {
    if (n <= 0 || r <= 0) return;
    k_transpose<<<dim3(ceil_div(n, 32), ceil_div(r, 32)), dim3(32, 8), 0, s>>>(n, r, in, out);
    FKB_LAUNCH_CHECK();
    count_launch();
}

void symmetrize(int n, double* A, long long lda, cudaStream_t s) {
    if (n <= 1) return;
    k_symmetrize<<<std::min(ceil_div((long long)n * n, 256), 4096), 256, 0, s>>>(A, n, lda);
    FKB_LAUNCH_CHECK();
    count_launch();
}

Filter::Filter(Cov* c, int m_, int h_cols, const int* rowptr, const int* col, const double* val, double sig2,
               long long k, long long p, uint64_t seed)
    : cov(c), s(c->stream), n(c->size()), m(m_), sigma2(sig2) {
    {  // side branches at the lowest priority (the main chain is on the operator's high-priority stream)
        int lo = 0, hi = 0;
        FKB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        FKB_CUDA(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, lo));
    }
    FKB_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    FKB_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    FKB_CUDA(cudaEventCreateWithFlags(&ev_join2, cudaEventDisableTiming));
    FKB_CUDA(cudaEventCreateWithFlags(&ev_ctz, cudaEventDisableTiming));
    FKB_CUDA(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
    FKB_CUDA(cudaStreamCreateWithFlags(&s4, cudaStreamNonBlocking));  // a deferred mean side (launch_step_piped)
    {
        int lo = 0, hi = 0;
        FKB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        FKB_CUDA(cudaStreamCreateWithPriority(&s5, cudaStreamNonBlocking, hi));  // the chain's head (early-PCG graphs)
        int dev = 0;
        FKB_CUDA(cudaGetDevice(&dev));
        FKB_CUDA(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));
    }
    FKB_CUDA(cudaEventCreateWithFlags(&ev_rfork, cudaEventDisableTiming));
    FKB_CUDA(cudaEventCreateWithFlags(&ev_rjoin, cudaEventDisableTiming));
    FKB_CUDA(cudaEventCreateWithFlags(&ev_mfork, cudaEventDisableTiming));
    FKB_CUDA(cudaEventCreateWithFlags(&ev_mjoin, cudaEventDisableTiming));
    if (m < 0) throw std::invalid_argument("fkf_init: negative measurement count");
    if ((long long)h_cols != n) throw std::invalid_argument("fkf_init: H columns do not match state dimension");
    for (int i = 0; i < m; ++i)
        for (int e = rowptr[i]; e < rowptr[i + 1]; ++e)
            if (col[e] < 0 || col[e] >= n) throw std::invalid_argument("fkf_init: H column index out of range");
    if (!(sigma2 > 0.0)) throw std::invalid_argument("fkf_init: sigma2 must be positive");  // :54-57
    upload_csr_pair(m, int(n), rowptr, col, val, H, HT);
    ghep(k, p, seed);                                                                    // :63-66
    // G = H·ΓHᵀ, symmetrized (:68-72): ΓHᵀ streamed in column batches, never stored.
    G.alloc(size_t(std::max(m, 1)) * std::max(m, 1));
    build_hgh(cov, H, G.p, s);
    B.alloc(size_t(std::max(m, 1)) * std::max(r, 1));  // HU (:73)
    spmm(H, U.p, n, r, B.p, m, 1.0, 0.0, s);
    colsq.alloc(size_t(std::max(r, 1)));
    Urow.alloc(size_t(n) * std::max(r, 1));
    if (r > 0) {
        k_colsq<<<r, 256, 0, s>>>(n, U.p, colsq.p);
        FKB_LAUNCH_CHECK();
        k_transpose<<<dim3(ceil_div(n, 32), ceil_div(r, 32)), dim3(32, 8), 0, s>>>(n, r, U.p, Urow.p);
        FKB_LAUNCH_CHECK();
        count_launch(2);
    }
    // Offline diagonalization of the α-dependence: G = P·diag(θ)·Pᵀ (block Jacobi), E = PᵀB.
    P.alloc(size_t(std::max(m, 1)) * std::max(m, 1));
    theta.alloc(size_t(std::max(m, 1)));
    E.alloc(size_t(std::max(m, 1)) * std::max(r, 1));
    if (m > 0) {
        S.alloc(size_t(m) * m);
        FKB_CUDA(cudaMemcpyAsync(S.p, G.p, sizeof(double) * size_t(m) * m, cudaMemcpyDeviceToDevice, s));
        eig_sweeps = sym_eig_device(m, S.p, m, theta.p, P.p, s);
        Pt.alloc(size_t(m) * m);  // Pᵀ (row-major P) for the per-step z = P·s̃ column dots
        k_transpose<<<dim3(ceil_div(m, 32), ceil_div(m, 32)), dim3(32, 8), 0, s>>>(m, m, P.p, Pt.p);
        FKB_LAUNCH_CHECK();
        count_launch();
        if (r > 0) {
            GemmArgs g;
            g.M = m; g.N = r; g.K = m;
            g.A = P.p; g.lda = m; g.transA = 1;
            g.B = B.p; g.ldb = m;
            g.C = E.p; g.ldc = m;
            gemm(g, nullptr, s);
            Erow.alloc(size_t(m) * r);  // row-major copy for the per-step s̃ rows
            k_transpose<<<dim3(ceil_div(m, 32), ceil_div(r, 32)), dim3(32, 8), 0, s>>>(m, r, E.p, Erow.p);
            FKB_LAUNCH_CHECK();
            count_launch();
        }
        S.release();
    }
    // state + workspaces
    alpha_dev.alloc(2);
    d.alloc(size_t(std::max(r, 1)));
    mean.alloc(size_t(n));
    for (int q = 0; q < 2; ++q) {
        wsqb[q].alloc(size_t(std::max(m, 1)));
        sqdb[q].alloc(size_t(std::max(r, 1)));
        Kb[q].alloc(size_t(std::max(r, 1)) * std::max(r, 1));
    }
    select_parity(0);
    rt.alloc(size_t(std::max(m, 1)));
    st.alloc(size_t(std::max(m, 1)));
    ucap.alloc(size_t(std::max(r, 1)));
    rdg.alloc(std::max<size_t>(chol_solve_scratch(r), 1));
    pcgwork.alloc(size_t(std::max(r, 1)) + 2);
    dsnap.alloc(size_t(std::max(r, 1)));
    pcgflag.alloc(1);
    parts.alloc(size_t(std::max(coldot_grid(m), 1)) * std::max(r, 1));
    for (int q = 0; q < 2; ++q) {
        certb[q].alloc(1);
        FKB_CUDA(cudaMemset(certb[q].p, 0, sizeof(int)));
    }
    if (r > 0 && r <= 640) {
        Kchk.alloc(size_t(r) * r);
        bchk.alloc(size_t(r));
        FKB_CUDA(cudaMemset(bchk.p, 0, bchk.bytes()));
        rdg2.alloc(std::max<size_t>(chol_solve_scratch(r), 1));
        cgate.alloc(2);
        FKB_CUDA(cudaMemset(cgate.p, 0, cgate.bytes()));
    }
    if (const char* e = std::getenv("FKB_CAP_CERT")) cert_force_fail = std::string(e) == "fail";
    if (std::getenv("FKB_PCG_STAMPS")) pcg_ts.alloc(64);
    {
        GemmArgs g;  // split-K workspace of the capacitance Gram
        g.M = r; g.N = r; g.K = m;
        g.splitk = gemm_pick_splitk(r, r, m);
        ws_step.alloc(std::max<size_t>(std::max(gemm_ws_elems(g), gram_ws_elems(r, r, m)), 1));  // graph-captured
    }
    for (int q = 0; q < 2; ++q) {
        zb[q].alloc(size_t(std::max(m, 1)));
        cvb[q].alloc(size_t(std::max(r, 1)));
        dq[q].alloc(size_t(std::max(r, 1)));
    }
    hm.alloc(size_t(std::max(m, 1)));
    ycur.alloc(size_t(std::max(m, 1)));
    alphaq.alloc(2);
    gateq.alloc(2);
    ticket.alloc(2);
    FKB_CUDA(cudaMemset(ticket.p, 0, 2 * sizeof(unsigned)));
    ready.alloc(1);
    FKB_CUDA(cudaMemset(ready.p, 0, sizeof(double)));
    // opt-in: on B200 the whole-GPU kernels of the two overlapped steps crowd each other out of
    // the SMs (c2: 96 µs per step against 80 µs for the full graphs back to back)
    piped_ok = false;
    if (const char* e = std::getenv("FKB_PIPED")) piped_ok = std::atoi(e) != 0;
    if (const char* e = std::getenv("FKB_EARLY_PCG")) early_pcg = std::atoi(e) != 0;
    t.alloc(size_t(n));
    vsub.alloc(size_t(n));
    if (const char* e = std::getenv("FKB_UPASS_CTAS")) upass_per_sm = std::atoi(e);
    if (const char* e = std::getenv("FKB_UPASS_THREADS")) upass_threads = std::atoi(e) == 128 ? 128 : 256;
    // the next-K Gram forks at the step's start when it is short (rank ≤ 320: ≈ 40 µs, hidden
    // beside the early main chain); at larger rank (c3/c4: 50–100 µs) beside the 16-SM PCG
    kfork = r <= 320 ? 1 : 0;
    if (const char* e = std::getenv("FKB_KFORK")) kfork = std::atoi(e);
    if (const char* e = std::getenv("FKB_UFORK")) ufork = std::atoi(e);
    if (const char* e = std::getenv("FKB_FUSE_RHS")) fuse_rhs = std::atoi(e) != 0;
    // the PDL-launched s̃ kernel wins when the U pass runs beside the chain (rank ≤ 320, c2); at
    // larger rank its early-resident CTAs crowd the next-K Gram, so the PCG cluster's tail does it
    fused_chain = r <= 320 ? 2 : 1;
    if (const char* e = std::getenv("FKB_FUSED_CHAIN")) fused_chain = std::atoi(e);
    pdl_mask = 3;  // rotate_in / rotate_out stage their first chunk of P / Pᵀ before the wait
    if (const char* e = std::getenv("FKB_PDL")) pdl_mask = std::atoi(e);
    if (const char* e = std::getenv("FKB_UPASS_GRID")) upass_per_sm = -std::atoi(e);  // total CTAs
    if (const char* e = std::getenv("FKB_UPASS_SIDE")) upass_side_mode = std::atoi(e);
    ybuf.alloc(size_t(std::max(m, 1)));
    ysrc.alloc(3);
    set_ysrc(ybuf.p, 0);
    info.alloc(1);
    hostout.alloc(10);  // [5q .. 5q+4]: the slots the parity-q step graph reads
    FKB_CUDA(cudaMemset(hostout.p, 0, hostout.bytes()));
    select_parity(0);
    flags.alloc(size_t(2 * ceil_div(std::max(m, 1), 64) + 2));
    reset();
}

Filter::~Filter() {
    // outstanding steps (asynchronous replays on s, s2, s3) must finish before buffers go back
    // to the allocator, or a later allocation could be overwritten
    if (s) cudaStreamSynchronize(s);
    if (s2) cudaStreamSynchronize(s2);
    if (s3) cudaStreamSynchronize(s3);
    if (s4) cudaStreamSynchronize(s4);
    if (s5) cudaStreamSynchronize(s5);
    if (cs) cudaStreamSynchronize(cs);
    drop_graphs();
    for (int q = 0; q < 2; ++q) {
        if (ev_done[q]) cudaEventDestroy(ev_done[q]);
        if (ev_copied[q]) cudaEventDestroy(ev_copied[q]);
    }
    if (cs) cudaStreamDestroy(cs);
    if (h_info) cudaFreeHost(h_info);
    if (h_hostout) cudaFreeHost(h_hostout);
    if (h_ysrc) cudaFreeHost(h_ysrc);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_join2) cudaEventDestroy(ev_join2);
    if (ev_ctz) cudaEventDestroy(ev_ctz);
    if (ev_rfork) cudaEventDestroy(ev_rfork);
    if (ev_rjoin) cudaEventDestroy(ev_rjoin);
    if (s5) cudaStreamDestroy(s5);
    if (ev_mfork) cudaEventDestroy(ev_mfork);
    if (ev_mjoin) cudaEventDestroy(ev_mjoin);
    if (s4) cudaStreamDestroy(s4);
    if (s3) cudaStreamDestroy(s3);
    if (s2) cudaStreamDestroy(s2);
}

void Filter::reset() {  // LowRankState::zero_start (fast_filter.hpp:30-36)
    FKB_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), s));
    FKB_CUDA(cudaMemsetAsync(alpha_dev.p, 0, 2 * sizeof(double), s));
    FKB_CUDA(cudaMemsetAsync(d.p, 0, d.bytes(), s));
    FKB_CUDA(cudaMemsetAsync(mean.p, 0, mean.bytes(), s));
    FKB_CUDA(cudaMemsetAsync(hm.p, 0, hm.bytes(), s));  // H·0
    FKB_CUDA(cudaMemsetAsync(ready.p, 0, sizeof(double), s));
    FKB_CUDA(cudaStreamSynchronize(s));
    hm_valid = true;
    alpha = 0.0;
    step_no = 0;
    state_rank = 0;
    k_valid = false;
}

void Filter::mark_on(cudaStream_t st, const char* name) {
    if (phase_events) {  // un-graphed serial phase timing: everything runs on s
        cudaEvent_t e;
        FKB_CUDA(cudaEventCreate(&e));
        FKB_CUDA(cudaEventRecord(e, s));
        phase_events->push_back(e);
        phase_names.emplace_back(name);
        return;
    }
    if (!(capturing && gtime)) return;
    cudaEvent_t e;
    FKB_CUDA(cudaEventCreate(&e));
    FKB_CUDA(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    const int q = par_next;  // the graph being captured
    int prev = -1;
    bool seen = false;
    for (auto& pl : gt_last)
        if (pl.first == st) {
            prev = pl.second;
            pl.second = int(gt_ev[q].size());
            seen = true;
        }
    if (!seen) gt_last.emplace_back(st, int(gt_ev[q].size()));
    gt_ev[q].push_back(e);
    gt_name[q].emplace_back(name);
    gt_prev[q].push_back(prev);
}

void Filter::drop_graphs() {
    for (int q = 0; q < 2; ++q) {
        for (int v = 0; v < 3; ++v) {
            if (graphv[v][q]) cudaGraphExecDestroy(graphv[v][q]);
            graphv[v][q] = nullptr;
        }
        if (graph[q]) cudaGraphExecDestroy(graph[q]);
        graph[q] = nullptr;
        graph_ready[q] = false;
        for (auto e : gt_ev[q]) cudaEventDestroy(e);
        gt_ev[q].clear();
        gt_name[q].clear();
        gt_prev[q].clear();
    }
}

void Filter::set_graph_timing(bool on) {
    if (on == gtime) return;
    gtime = on;
    drop_graphs();
}

std::vector<std::pair<std::string, double>> Filter::graph_phase_times() {
    std::vector<std::pair<std::string, double>> out;
    const int q = gt_last_par;
    if (!gtime || !graph_ready[q]) return out;
    FKB_CUDA(cudaStreamSynchronize(s));
    for (size_t i = 0; i < gt_ev[q].size(); ++i) {
        if (gt_prev[q][i] < 0) continue;
        float ms = 0.f;
        FKB_CUDA(cudaEventElapsedTime(&ms, gt_ev[q][size_t(gt_prev[q][i])], gt_ev[q][i]));
        out.emplace_back(gt_name[q][i], double(ms));
    }
    return out;
}

std::vector<std::pair<std::string, double>> Filter::phase_times(int reps) {
    std::vector<std::pair<std::string, double>> acc;
    set_hostout(0, 0, 0);  // the diagnostic steps must not write through a caller's stale mapped buffers
    for (int rep = 0; rep < reps; ++rep) {
        std::vector<cudaEvent_t> ev;
        phase_events = &ev;
        phase_names.clear();
        prime_capacitance();
        select_parity(par_next);
        mark("begin");
        try {
            enqueue_step(ybuf.p);
        } catch (...) {
            phase_events = nullptr;
            throw;
        }
        phase_events = nullptr;
        FKB_CUDA(cudaStreamSynchronize(s));
        if (acc.empty())
            for (size_t i = 1; i < ev.size(); ++i) acc.emplace_back(phase_names[i], 0.0);
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0.f;
            FKB_CUDA(cudaEventElapsedTime(&ms, ev[i - 1], ev[i]));
            acc[i - 1].second += ms / reps;
        }
        for (auto e : ev) cudaEventDestroy(e);
        gt_last_par = par_next;  // the parity a rerun of this step would use
        par_next ^= 1;
        check_info();
        alpha += 1.0;
        ++step_no;
        state_rank = r;
    }
    return acc;
}

void Filter::set_solver(int mode) {
    if (mode != 0 && mode != 1) throw std::invalid_argument("fkf: solver must be 0 (dense LLT) or 1 (Woodbury)");
    if (mode == solver) return;
    solver = mode;
    k_valid = false;
    if (mode == 0 && S.n < size_t(m) * m) S.alloc(size_t(std::max(m, 1)) * std::max(m, 1));  // before any capture
    if (mode == 0) potrf_ws.ensure(potrf_ws_elems(m));  // DMMA panel path inside the captured graph
    drop_graphs();
}

void Filter::fork() {
    if (side() == s) return;
    FKB_CUDA(cudaEventRecord(ev_fork, s));
    FKB_CUDA(cudaStreamWaitEvent(s2, ev_fork, 0));
    mark_on(s2, "fork");
}
void Filter::join(cudaEvent_t ev) {
    if (side() == s) return;
    FKB_CUDA(cudaEventRecord(ev, s2));
    FKB_CUDA(cudaStreamWaitEvent(s, ev, 0));
}

void Filter::enqueue_capacitance(cudaStream_t b, int mode, double* wsq_o, double* sqd_o, double* K_o) {
    if (solver != 1 || r <= 0) return;
    // mode 1 (inside the step graph) reads the snapshot of the committed d taken by the step's
    // first kernel: the step's own epilogue commits the new d concurrently with this branch
    k_woodbury_scalars<<<std::max(1, std::min(ceil_div(std::max(m, r), 256), 148)), 256, 0, b>>>(
        m, r, mode, alpha_dev.p, theta.p, mode == 1 ? dsnap.p : d.p, lambda.p, sigma2, wsq_o, sqd_o,
        K_o == Kb[0].p ? certb[0].p : certb[1].p);
    FKB_LAUNCH_CHECK();
    count_launch();
    GemmArgs g;  // K = I − D^½·Eᵀ·Λ_M⁻¹·E·D^½
    g.M = r; g.N = r; g.K = m;
    g.A = E.p; g.lda = m; g.transA = 1;
    g.B = E.p; g.ldb = m;
    g.dA = wsq_o;
    g.rs = sqd_o; g.cs = sqd_o;
    g.alpha = -1.0;
    g.C = K_o; g.ldc = r;
    g.diag_add = 1.0;
    gram_sym(g, b);  // full symmetric K (the PCG reads columns)
    int* cert_o = K_o == Kb[0].p ? certb[0].p : certb[1].p;
    k_cap_certificate<<<ceil_div(r, 8), 256, sizeof(double) * size_t(r), b>>>(r, K_o, cert_o, cert_force_fail ? 1 : 0);
    FKB_LAUNCH_CHECK();
    count_launch();
    if (r <= 640 && !cert_force_fail) {  // the cluster Cholesky's staging limit
        k_cert_prepare<<<std::min(ceil_div((long long)r * r, 256), 296), 256, 0, b>>>(r, K_o, Kchk.p, cert_o, cgate.p,
                                                                                      cgate.p + 1);
        FKB_LAUNCH_CHECK();
        chol_solve_small(r, Kchk.p, r, bchk.p, rdg2.p, cgate.p + 1, b, nullptr, cgate.p);
        k_cert_finish<<<1, 1, 0, b>>>(cert_o, cgate.p, cgate.p + 1);
        FKB_LAUNCH_CHECK();
        count_launch(2);
    }
}

// hm = H·mean after the mean was set from outside (set_state); the steps keep it current
void Filter::prime_image() {
    if (hm_valid) return;
    if (m > 0) spmm(H, mean.p, n, 1, hm.p, m, 1.0, 0.0, s);
    hm_valid = true;
}

void Filter::prime_capacitance() {  // K, wsq, sqd of the next step (parity par_next), eagerly
    prime_image();
    if (k_valid || solver != 1 || r <= 0) return;
    enqueue_capacitance(s, 0, wsqb[par_next].p, sqdb[par_next].p, Kb[par_next].p);
    k_valid = true;
}

// The commit epilogue of the step being enqueued (parity buffers selected by select_parity)
EpiCtzD Filter::commit_epi() {
    return EpiCtzD{cv_c, d.p, lambda.p, alpha_dev.p, info.p, hout_c, aq_c, gate_c, uq_count >= 0 ? dq_c : nullptr};
}

// One step = the m-space chain (enqueue_chain: everything the NEXT step depends on — α, d, the
// image hm of the mean) followed by the N-space mean side (enqueue_mean_side: Γ(Hᵀz), the U
// pass, the mean update and the fused UQ).  The chain does not read the mean (k_step_prologue),
// so a batch can run step t's mean side beside step t+1's chain (launch_step_piped).
void Filter::enqueue_step(const double* d_y) {
    enqueue_chain(d_y, false);
    MeanSide ms;
    ms.z = z_c; ms.cv = cv_c; ms.alpha1 = alpha_dev.p; ms.gate = info.p; ms.d = d.p; ms.hout = hout_c;
    ms.sqd = sqd_c;
    enqueue_mean_side(ms, s, false);
}

void Filter::enqueue_chain(const double* d_y, bool deferred, const std::function<void()>& after_prologue) {
    (void)d_y;  // the observation is read through ysrc (per-call: ybuf)
    // Pipelined batch graphs launch the PCG cluster FIRST (a root of the graph, on the main
    // stream): it needs 16 empty SMs of one GPC, which it would wait for behind the previous
    // step's mean side; resident from the start it stages K and spins until rotate_in's last
    // CTA publishes the partials (PcgRhs::ready).  The prologue and rotate_in then run on the
    // head stream s5 beside it.
    hs = s;
    if (deferred && solver == 1 && r > 0 && fused_chain && side() != s && early_pcg) {
        hs = s5;
        FKB_CUDA(cudaEventRecord(ev_rfork, s));
        FKB_CUDA(cudaStreamWaitEvent(s5, ev_rfork, 0));
    }
    // α ← α + 1, flags, z = y − hm (:97, :108): one kernel
    {
        const int blocks = std::max(1, std::min(ceil_div(std::max(m, 1), 256), 148));
        k_step_prologue<<<blocks, 256, 0, hs>>>(m, r, ybuf.p, hm.p, z_c, ycur.p, alpha_dev.p, theta.p, d.p, sigma2,
                                                (solver == 1 && r == 0) ? wsq_c : nullptr, sqd_c,
                                                (solver == 1 && r > 0) ? dsnap.p : nullptr,
                                                (solver == 1 && !exact) ? pcgflag.p : nullptr, ysrc.p, gate_c,
                                                ticket.p);
        FKB_LAUNCH_CHECK();
        count_launch();
    }
    if (after_prologue) after_prologue();
    mark_on(hs, "residual");
    chain_deferred = deferred;
    if (solver == 0) {
        enqueue_solve_dense();
        k_image_update<<<std::max(1, ceil_div(m, 256)), 256, 0, s>>>(m, z_c, hm.p, ycur.p, sigma2, info.p);
        FKB_LAUNCH_CHECK();
        count_launch();
    } else {
        enqueue_solve_woodbury();
    }
    // dc = d ⊙ Bᵀz with d and α updated in the same pass (solver 0: a side-branch pass over B;
    // solver 1: D^½x inside k_woodbury_st)
    if (r > 0 && solver == 0) {
        if (!deferred) fork();
        launch_coldot(m, r, B.p, m, XPlain{z_c}, commit_epi(), deferred ? s : side());
        mark_on(deferred ? s : side(), "ctz_d_update");
        if (!deferred) {
            if (upass_side()) {
                launch_u_pass(XPlain{cv_c}, side(), true);
                mark_on(side(), "u_pass");
            }
            if (side() != s) FKB_CUDA(cudaEventRecord(ev_join, s2));
        }
    } else if (r == 0) {
        k_d_update<<<1, 32, 0, s>>>(0, d.p, lambda.p, alpha_dev.p, info.p, aq_c, gate_c);  // commits α
        FKB_LAUNCH_CHECK();
        count_launch();
    }
    chain_deferred = false;
    hs = s;
}

// The N-space side of a step whose chain has committed: t = Γ(Hᵀz); v = U·dc; the last FFT
// pass applies mean ← (mean + α·t) − v (:114-116), or the fused pass k_mean_uq does it with
// diag Σ and the realizations.  ms names the step's buffers: the step just enqueued on this
// stream (deferred = false: the U pass may already run on the side branch, forked inside the
// chain), or the previous step's parity snapshots (deferred = true: everything is launched
// here, on sm and the U-pass branch s2).
void Filter::enqueue_mean_side(const MeanSide& ms, cudaStream_t sm, bool deferred) {
    const bool par = side() != s;
    const bool fused_uq = uq_count >= 0 && r > 0;
    cudaStream_t cov_stream = cov->stream;
    cov->stream = sm;
    struct Restore {
        Cov* c;
        cudaStream_t st;
        ~Restore() { c->stream = st; }
    } restore{cov, cov_stream};
    const bool u_beside = r > 0 && upass_side() && par;
    // beside a chain whose PCG cluster owns 16 SMs the persistent U pass takes the others
    upass_leave = deferred && sm != s ? 16 : 0;
    struct Leave {
        int& v;
        ~Leave() { v = 0; }
    } leave{upass_leave};
    if (deferred && u_beside) {  // the U pass beside Γ(Hᵀz)
        FKB_CUDA(cudaEventRecord(ev_fork, sm));
        FKB_CUDA(cudaStreamWaitEvent(s2, ev_fork, 0));
        mark_on(s2, "fork");
        launch_u_pass(XPlain{ms.cv}, s2, true);
        mark_on(s2, "u_pass");
        FKB_CUDA(cudaEventRecord(ev_join, s2));
    }
    spmv_short(HT, ms.z, t.p, 1.0, sm);
    mark_on(sm, "ht_z");
    if (!deferred && ufork == 3 && solver == 1) fork_upass();
    if (fused_uq) {  // U pass + diag Σ + realizations of the new state in one pass (needs t)
        cov->apply1(t.p, t.p);
        mark_on(sm, "gamma_apply");
        if (!deferred && par && solver == 0) FKB_CUDA(cudaStreamWaitEvent(sm, ev_join, 0));  // dc ready
        launch_mean_uq(uq_count, n, r, U.p, ms.cv, ms.d, ms.alpha1, cov->spec.theta, t.p, mean.p,
                       uq_count ? draws.p : nullptr, uq_count ? draw_proj.p : nullptr, uq_x.p, uq_var.p, ms.gate,
                       ms.hout, nullptr, sm);
        if (!deferred && solver == 1 && par) FKB_CUDA(cudaStreamWaitEvent(sm, ev_join2, 0));  // next K ready
        mark_on(sm, "mean_update");
        return;
    }
    cov->apply1_fwd(t.p);
    mark_on(sm, "gamma_fwd");
    const bool u_joined = r > 0 && par && (deferred ? u_beside : (upass_side() || solver == 0));
    if (u_joined) FKB_CUDA(cudaStreamWaitEvent(sm, ev_join, 0));  // v = U·dc (or solver 0's dc) ready
    if (r > 0 && !(upass_side() && (par || !deferred)) ) {
        // the long U pass (rank > 320) on the whole GPU, or the serial phase-timing order
        if (deferred || solver == 0) launch_u_pass(XPlain{ms.cv}, sm, false);
        else launch_u_pass(XProd{ms.sqd, ucap.p}, sm, false);
        mark_on(sm, "u_pass");
    }
    cov->apply1_inv(mean.p, MeanUpd{ms.alpha1 + 1, ms.gate, r > 0 ? vsub.p : nullptr, ms.hout, nullptr});
    if (!deferred && solver == 1 && r > 0 && par) FKB_CUDA(cudaStreamWaitEvent(sm, ev_join2, 0));  // next K ready
    mark_on(sm, "mean_update");
}

// v = U·dc (the mean update's low-rank term) streaming the row-major U: beside the main chain
// at upass_per_sm CTAs per SM (so the latency-bound chain it overlaps keeps room), or on the
// main stream with the whole GPU
template <class XL>
void Filter::launch_u_pass(XL xl, cudaStream_t st, bool beside) {
    int cap = beside ? upass_per_sm : 0;
    if (upass_leave > 0 && cap >= 0 && sm_count > upass_leave)
        cap = -(sm_count - upass_leave) * (beside ? std::max(upass_per_sm, 1) : 2);
    launch_gemv_rowmajor(n, r, Urow.p, std::max(r, 1), xl, EpiStore{vsub.p}, st, cap, upass_threads);
}

// z ← S⁻¹z with S = P[Λ_M − E·D·Eᵀ]Pᵀ (Woodbury with the k×k capacitance K).
// Fused chain (default): rotate_in also leaves per-CTA partials of u = D^½Eᵀ(Λ_M⁻¹r̃); the PCG
// cluster sums them, solves K x = u, verifies the true residual and, in its tail, forms
// s̃ = Λ_M⁻¹(r̃ + E·D^½x) and commits d and α — three dependent launches instead of five.  A
// solve that does not verify raises kInfoRetry: the step's state epilogues are gated off and
// the host reruns it on the exact path (exact = true: column-dot RHS, cluster Cholesky,
// k_woodbury_st), which also reproduces the reference's "singular" error.
void Filter::enqueue_solve_woodbury() {
    // side branch: the NEXT step's Woodbury scalars and K into the other parity's buffers (they
    // depend on α and d only); forked at kfork: 0 before the capacitance solve (beside the
    // 16-SM PCG cluster), 1 at the start of the step, 2 after the capacitance solve
    auto fork_next_k = [&](cudaStream_t at) {
        if (r <= 0) return;
        if (side() != s) {
            FKB_CUDA(cudaEventRecord(ev_ctz, at));
            FKB_CUDA(cudaStreamWaitEvent(s3, ev_ctz, 0));
            mark_on(s3, "fork_k");
        }
        enqueue_capacitance(side() != s ? s3 : s, 1, wsq_n, sqd_n, K_n);
        mark_on(side() != s ? s3 : s, "capacitance");
        if (side() != s) FKB_CUDA(cudaEventRecord(ev_join2, s3));
    };
    auto fork_u = [&] {
        if (!chain_deferred) fork_upass();  // a deferred mean side launches its own U pass
    };
    if (kfork == 1) fork_next_k(hs);
    const bool fused = fused_chain && !exact && r > 0;
    if (fused) {
        // r̃ = Pᵀ(y − H·mean) and the partials of Eᵀ(Λ_M⁻¹r̃) in one pass
        auto rotate_in = [&] {
            launch_coldot(m, m, P.p, m, XPlain{z_c}, EpiAxpby{rt.p, 1.0, 0.0}, hs,
                          CtaParts{Erow.p, r, wsq_c, parts.p, ready.p, ticket.p + 1, alpha_dev.p}, (pdl_mask & 1) != 0);
            mark_on(hs, "rotate_in");
            if (kfork == 0) fork_next_k(hs);
        };
        auto solve = [&] {
            PcgRhs rhs;
            rhs.parts = parts.p; rhs.nparts = coldot_grid(m); rhs.sqd = sqd_c; rhs.cert = cert_c;
            rhs.ready = ready.p; rhs.alpha_dev = alpha_dev.p;
            PcgTail tl;
            const bool pdl = fused_chain == 2 && r <= 512;
            tl.info = info.p;
            tl.retry_only = pdl;
            if (!pdl) {
                tl.Erow = Erow.p; tl.m = m; tl.wsq = wsq_c; tl.rt = rt.p; tl.sqd = sqd_c; tl.st = st.p; tl.dc = cv_c;
                tl.d = d.p; tl.lam = lambda.p; tl.alpha_dev = alpha_dev.p; tl.hout = hout_c;
                tl.alpha_q = aq_c; tl.gate_q = gate_c; tl.d_q = uq_count >= 0 ? dq_c : nullptr;
            }
            cap_pcg(r, K_c, r, ucap.p, pcgwork.p, pcgflag.p, s, pcg_maxit, 1e-12, pcg_ts.p, 1e-11, rhs, tl);
            if (pdl) {  // s̃ and the d/α commit by a programmatic dependent (gated on the flag the PCG raises)
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(std::max(1, ceil_div(m, 8)) + 1, 1, 1);
                cfg.blockDim = dim3(256, 1, 1);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                FKB_CUDA(cudaLaunchKernelEx(&cfg, k_woodbury_st_pdl, m, r, (const double*)Erow.p, (const double*)sqd_c,
                                            (const double*)ucap.p, (const double*)wsq_c, (const double*)rt.p, st.p,
                                            commit_epi(), hs != s ? 1 : 0));
                count_launch();
            }
        };
        if (hs != s) {  // early PCG: the cluster is captured (and dispatched) ahead of rotate_in
            solve();
            rotate_in();
        } else {
            rotate_in();
            solve();
        }
        mark("cap_solve");
        if (kfork == 2) fork_next_k(s);
        if (ufork <= 1) fork_u();
    } else {
        launch_coldot(m, m, P.p, m, XPlain{z_c}, EpiAxpby{rt.p, 1.0, 0.0}, s);  // r̃ = Pᵀ(y − H·mean)
        mark("rotate_in");
        if (r > 0) {
            // u = D^½·Eᵀ·Λ_M⁻¹·r̃: formed by the PCG kernel itself (fuse_rhs) or as column dots
            PcgRhs rhs;
            rhs.cert = cert_c;
            if (fuse_rhs && !exact) {
                rhs.E = E.p; rhs.lde = m; rhs.m = m; rhs.wsq = wsq_c; rhs.rt = rt.p; rhs.sqd = sqd_c;
            } else {
                launch_coldot(m, r, E.p, m, XProd{wsq_c, rt.p}, EpiScaleOut{ucap.p, sqd_c}, s);
                mark("cap_rhs");
            }
            if (kfork == 0) fork_next_k(s);
            // x = K⁻¹u: Jacobi-PCG in one cluster; exact Cholesky only if PCG hits its cap.
            // ‖Kx − u‖ ≤ 1e-12‖u‖: the solve's error reaches the mean through U·D^½x at ~1e-12
            // relative, three orders below the 1e-9 parity bar.  A converged x is re-checked
            // against the true residual ‖u − Kx‖ ≤ 1e-11‖u‖ inside the kernel (the pipelined
            // recursion can drift); a miss routes to the Cholesky.  The exact rerun of a step
            // goes to the Cholesky directly.
            if (!exact) cap_pcg(r, K_c, r, ucap.p, pcgwork.p, pcgflag.p, s, pcg_maxit, 1e-12, pcg_ts.p, 1e-11, rhs);
            chol_solve_small(r, K_c, r, ucap.p, rdg.p, info.p, s, nullptr, exact ? nullptr : pcgflag.p);
            mark("cap_solve");
            if (kfork == 2) fork_next_k(s);
            if (ufork == 0) fork_u();
        }
        // s̃ = Λ_M⁻¹(r̃ + E·D^½·x): one warp per row of the row-major copy of E
        k_woodbury_st<<<std::max(1, ceil_div(m, 8)) + 1, 256, 0, s>>>(
            m, r, Erow.p, sqd_c, ucap.p, wsq_c, rt.p, st.p, commit_epi());
        FKB_LAUNCH_CHECK();
        count_launch();
        mark("woodbury_st");
        if (ufork == 1) fork_u();
    }
    launch_coldot(m, m, Pt.p, m, XPlain{st.p}, EpiZHm{z_c, hm.p, ycur.p, sigma2, info.p}, s, NoCta{},  // z = P·s̃ (rows of P); hm = y − σ²z
                  fused && fused_chain == 2 && r <= 512 && (pdl_mask & 2));
    mark("rotate_out");
    if (hs != s) {  // the head stream (prologue, rotate_in) rejoins
        FKB_CUDA(cudaEventRecord(ev_rjoin, hs));
        FKB_CUDA(cudaStreamWaitEvent(s, ev_rjoin, 0));
    }
    if (ufork == 2) fork_u();
}

// the U pass v = U·(D^½x) beside the rest of the chain (x from the capacitance solve)
void Filter::fork_upass() {
    if (r <= 0 || !upass_side()) return;
    fork();
    launch_u_pass(XProd{sqd_c, ucap.p}, side(), true);
    mark_on(side(), "u_pass");
    if (side() != s) FKB_CUDA(cudaEventRecord(ev_join, s2));
}

// z ← S⁻¹z forming S = α·G − B·diag(d)·Bᵀ + σ²I and its LLT, as fast_filter.hpp:100-108.
void Filter::enqueue_solve_dense() {
    GemmArgs g;
    g.M = m; g.N = m; g.K = r;
    g.A = B.p; g.lda = m; g.transA = 0;
    g.B = B.p; g.ldb = m; g.transB = 1;
    g.dA = d.p;
    g.alpha = -1.0;
    g.beta_ptr = alpha_dev.p + 1;
    g.beta = 1.0;
    g.Cin = G.p; g.ldcin = m;
    g.C = S.p; g.ldc = m;
    g.diag_add = sigma2;
    g.lower_only = 1;
    gemm(g, nullptr, s);
    mark("innovation_build");
    potrf_lower(m, S.p, m, info.p, potrf_ws.p, potrf_ws.n, s);  // LLT (:104-106)
    mark("llt");
    potrs_lower(m, S.p, m, z_c, flags.p, s);         // z = S⁻¹(y − H·mean) (:108)
    mark("llt_solve");
}

void Filter::check_info() {
    int h = 0;
    FKB_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    FKB_CUDA(cudaStreamSynchronize(s));
    if (h == kInfoRetry) {
        rerun_exact(gt_last_par);
        FKB_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaStreamSynchronize(s));
    }
    if (h) fail_step("fkf_step: innovation system is singular");
}

// The step replayed with parity q left the state untouched because its capacitance PCG did not
// verify (kInfoRetry): clear the flag and run the same step (observation in ybuf, the same
// parity's K, wsq and sqd) eagerly on the exact path — cluster Cholesky, which reports a
// non-positive-definite system exactly like the reference LLT (fast_filter.hpp:104-106).  The
// side branch recomputes the next step's K as usual.
void Filter::rerun_exact(int q) {
    FKB_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), s));
    FKB_CUDA(cudaMemsetAsync(ready.p, 0, sizeof(double), s));  // the failed step's epoch must not satisfy a later wait
    // this step's K, Λ_M⁻¹ and D^½ afresh from the committed α and d: inside an asynchronous
    // batch the no-op steps behind the sticky flag have overwritten the parity buffers
    if (solver == 1 && r > 0) enqueue_capacitance(s, 0, wsqb[q].p, sqdb[q].p, Kb[q].p);
    select_parity(q);
    exact = true;
    try {
        enqueue_step(ybuf.p);
    } catch (...) {
        exact = false;
        throw;
    }
    exact = false;
}

// A failed step: clear the sticky device flag (so the next step can run), invalidate the
// precomputed capacitance (the side branch assumed the step would commit its d update) and
// raise the reference's error (fast_filter.hpp:104-106).
void Filter::fail_step(const std::string& msg) {
    FKB_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), s));
    FKB_CUDA(cudaMemsetAsync(ready.p, 0, sizeof(double), s));
    FKB_CUDA(cudaStreamSynchronize(s));
    k_valid = false;
    throw std::runtime_error(msg);
}

void Filter::launch_step() {
    prime_capacitance();
    const int q = par_next;
    if (!graph_ready[q]) {
        // Capture the step once per parity (it reads y from ybuf and α from alpha_dev);
        // replays remove the per-kernel launch latency.
        const unsigned long long before = g_launches;
        for (auto e : gt_ev[q]) cudaEventDestroy(e);
        gt_ev[q].clear();
        gt_name[q].clear();
        gt_prev[q].clear();
        gt_last.clear();
        select_parity(q);
        cudaGraph_t gr;
        FKB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        capturing = true;
        try {
            mark("begin");
            enqueue_step(ybuf.p);
        } catch (...) {
            capturing = false;
            cudaStreamEndCapture(s, &gr);
            throw;
        }
        capturing = false;
        FKB_CUDA(cudaStreamEndCapture(s, &gr));
        // per-node priorities as captured: the main chain's CTAs go ahead of the U pass's
        FKB_CUDA(cudaGraphInstantiate(&graph[q], gr, cudaGraphInstantiateFlagUseNodePriority));
        cudaGraphDestroy(gr);
        launches_per_step = int(g_launches - before);
        g_launches = before;
        graph_ready[q] = true;
    }
    FKB_CUDA(cudaGraphLaunch(graph[q], s));
    count_launch(launches_per_step);
    gt_last_par = q;
    par_next ^= 1;
}

Filter::MeanSide Filter::snapshot_side(int q) {
    MeanSide ms;
    ms.z = zb[q].p; ms.cv = cvb[q].p; ms.alpha1 = alphaq.p + q - 1; ms.gate = gateq.p + q; ms.d = dq[q].p;
    ms.hout = hostout.p + 5 * q;
    return ms;
}

// Pipelined batch graphs (see graphv): variant v for the step of parity q.
void Filter::launch_piped(int v, int q) {
    if (v != 2) prime_capacitance();
    if (!graphv[v][q]) {
        const unsigned long long before = g_launches;
        select_parity(q);
        cudaGraph_t gr;
        FKB_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        capturing = true;
        try {
            const bool par = side() != s;
            if (v == 0) {
                enqueue_chain(ybuf.p, true);
                if (par) FKB_CUDA(cudaStreamWaitEvent(s, ev_join2, 0));  // next K ready
            } else if (v == 1) {
                // the previous step's mean side forks after this step's prologue: by then the
                // PCG cluster (a root of the graph) owns its SMs
                enqueue_chain(ybuf.p, true, [&] {
                    FKB_CUDA(cudaEventRecord(ev_mfork, hs));
                    FKB_CUDA(cudaStreamWaitEvent(s4, ev_mfork, 0));
                    enqueue_mean_side(snapshot_side(q ^ 1), s4, true);
                    FKB_CUDA(cudaEventRecord(ev_mjoin, s4));
                });
                if (par) FKB_CUDA(cudaStreamWaitEvent(s, ev_join2, 0));
                FKB_CUDA(cudaStreamWaitEvent(s, ev_mjoin, 0));
            } else {
                enqueue_mean_side(snapshot_side(q), s, true);
            }
        } catch (...) {
            capturing = false;
            cudaStreamEndCapture(s, &gr);
            throw;
        }
        capturing = false;
        FKB_CUDA(cudaStreamEndCapture(s, &gr));
        FKB_CUDA(cudaGraphInstantiate(&graphv[v][q], gr, cudaGraphInstantiateFlagUseNodePriority));
        cudaGraphDestroy(gr);
        launches_v[v] = int(g_launches - before);
        g_launches = before;
    }
    FKB_CUDA(cudaGraphLaunch(graphv[v][q], s));
    count_launch(launches_v[v]);
    if (v != 2) {
        gt_last_par = q;
        par_next = q ^ 1;
    }
}

// Step t of a pipelined batch: the head graph (chain only), then the steady graph (the chain
// beside step t−1's mean side); the caller flushes the last mean side with launch_piped(2, ·).
void Filter::run_piped(int t) { launch_piped(t == 0 ? 0 : 1, par_next); }

void Filter::step(const double* d_y) {
    set_hostout(0, 0, 0);
    if (d_y != ybuf.p)
        FKB_CUDA(cudaMemcpyAsync(ybuf.p, d_y, sizeof(double) * size_t(m), cudaMemcpyDeviceToDevice, s));
    launch_step();
    check_info();
    alpha += 1.0;
    ++step_no;
    state_rank = r;
}

// One step from a host observation with the new state downloaded in the same round trip
// (the reference's fkf_step returns the new LowRankState by value): H2D y, graph replay, D2H of
// the failure flag, d and mean, ONE stream synchronization.
// device address of a page-locked (mapped) host buffer, 0 for pageable memory
static unsigned long long mapped_host(const void* p) {
    if (!p) return 0;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return a.type == cudaMemoryTypeHost && a.devicePointer ? reinterpret_cast<unsigned long long>(a.devicePointer) : 0;
}

// Stream-ordered: the values come from a page-locked staging slot per (base, ld) pair that is
// only rewritten after a stream synchronization.
void Filter::set_ysrc(const double* base, long long ld) {
    if (!h_ysrc) FKB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_ysrc), 6 * sizeof(long long), cudaHostAllocDefault));
    const long long b = static_cast<long long>(reinterpret_cast<uintptr_t>(base));
    const int slot = ld == 0 ? 0 : 1;  // 0: the per-call buffer, 1: the host batch's block
    long long* v = h_ysrc + 3 * slot;
    if (v[0] != b || v[1] != ld) {
        FKB_CUDA(cudaStreamSynchronize(s));  // an earlier copy may still read the slot
        v[0] = b;
        v[1] = ld;
        v[2] = 0;
    }
    FKB_CUDA(cudaMemcpyAsync(ysrc.p, v, 3 * sizeof(long long), cudaMemcpyHostToDevice, s));
}

void Filter::set_hostout(unsigned long long hm, unsigned long long hd, unsigned long long hi, unsigned long long hx,
                         unsigned long long hv) {
    const unsigned long long want[10] = {hm, hd, hi, hx, hv, hm, hd, hi, hx, hv};  // both parities
    set_hostout_all(want);
}
void Filter::set_hostout_all(const unsigned long long (&want)[10]) {
    if (std::equal(want, want + 10, hostout_cache)) return;
    if (!h_hostout)
        FKB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_hostout), 10 * sizeof(unsigned long long),
                               cudaHostAllocDefault));
    FKB_CUDA(cudaStreamSynchronize(s));  // the staging slots may still feed an earlier copy
    for (int i = 0; i < 10; ++i) h_hostout[i] = hostout_cache[i] = want[i];
    FKB_CUDA(cudaMemcpyAsync(hostout.p, h_hostout, 10 * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
}

// nsteps steps from host observations with every step's new state (and, count ≥ 0, its diag Σ
// and `count` realizations) returned in host arrays — the reference driver's loop
// (driver.hpp:283-300) as one call.  Each step's graph writes its outputs into per-parity
// device snapshots (the hostout slots of that parity); a copy stream moves them to the host
// while the next step runs, and step t+2 (same parity) waits only for step t's copies.  The
// observation of step t is copied host → ybuf on the main stream right before its graph.
// Failures as finish_async (kInfoRetry steps rerun exactly, "singular" names the step).
void Filter::run_host(const double* h_ys, int nsteps, long long ldy, double* h_alpha, double* h_d, long long ldd,
                      double* h_mean, long long ldm, int count, uint64_t seed, double* h_x, double* h_var) {
    if (nsteps <= 0) return;
    const bool uq = count >= 0 && r > 0;
    set_step_uq(uq, seed, uq ? count : 0);
    if (!cs) {
        FKB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (int q = 0; q < 2; ++q) {
            FKB_CUDA(cudaEventCreateWithFlags(&ev_done[q], cudaEventDisableTiming));
            FKB_CUDA(cudaEventCreateWithFlags(&ev_copied[q], cudaEventDisableTiming));
        }
    }
    const int cnt = uq ? count : 0;
    for (int q = 0; q < 2; ++q) {
        snap_mean[q].ensure(size_t(n));
        snap_d[q].ensure(size_t(std::max(r, 1)));
        if (uq) {
            snap_x[q].ensure(size_t(n) * std::max(cnt, 1));
            snap_v[q].ensure(size_t(n));
        }
    }
    auto u = [](const void* p) { return reinterpret_cast<unsigned long long>(p); };
    unsigned long long want[10];
    for (int q = 0; q < 2; ++q) {
        want[5 * q + 0] = u(snap_mean[q].p);
        want[5 * q + 1] = r > 0 ? u(snap_d[q].p) : 0;
        want[5 * q + 2] = 0;
        want[5 * q + 3] = uq && cnt ? u(snap_x[q].p) : 0;
        want[5 * q + 4] = uq ? u(snap_v[q].p) : 0;
    }
    set_hostout_all(want);
    // every step's observation uploaded once; the graphs read row ysrc[2] of the block
    if (ys_dev.n < size_t(std::max(m, 1)) * nsteps)  // grown geometrically: repeated batches do not reallocate
        ys_dev.ensure(std::max(size_t(std::max(m, 1)) * nsteps, 2 * ys_dev.n));
    set_ysrc(ys_dev.p, m);
    if (m > 0)
        FKB_CUDA(cudaMemcpy2DAsync(ys_dev.p, sizeof(double) * size_t(m), h_ys, sizeof(double) * size_t(ldy),
                                   sizeof(double) * size_t(m), size_t(nsteps), cudaMemcpyHostToDevice, s));
    const double alpha0 = alpha;
    const int par0 = par_next;
    // step t's snapshot (parity q) → host rows; what: 1 = d (the chain's), 2 = mean, diag Σ and
    // realizations (the mean side's)
    auto copy_out = [&](int q, int t, cudaStream_t st, int what) {
        if ((what & 1) && h_d && r > 0)
            FKB_CUDA(cudaMemcpyAsync(h_d + t * ldd, snap_d[q].p, sizeof(double) * size_t(r), cudaMemcpyDeviceToHost, st));
        if (!(what & 2)) return;
        if (h_mean) FKB_CUDA(cudaMemcpyAsync(h_mean + t * ldm, snap_mean[q].p, sizeof(double) * size_t(n),
                                             cudaMemcpyDeviceToHost, st));
        if (uq && h_var) FKB_CUDA(cudaMemcpyAsync(h_var + (long long)t * n, snap_v[q].p, sizeof(double) * size_t(n),
                                                  cudaMemcpyDeviceToHost, st));
        if (uq && cnt && h_x)
            FKB_CUDA(cudaMemcpyAsync(h_x + (long long)t * n * cnt, snap_x[q].p, sizeof(double) * size_t(n) * cnt,
                                     cudaMemcpyDeviceToHost, st));
    };
    // FKB_RUN_TRACE=1: per-step timing events (main stream before the input copy, after the
    // graph; copy stream after the outputs), printed after the batch (diagnostics)
    static const bool trace = std::getenv("FKB_RUN_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto tmark = [&](cudaStream_t st) {
        if (!trace) return;
        cudaEvent_t e;
        FKB_CUDA(cudaEventCreate(&e));
        FKB_CUDA(cudaEventRecord(e, st));
        tev.push_back(e);
    };
    // Pipelined: graph t runs step t's chain beside step t−1's mean side, so after graph t the
    // copy stream takes d of step t and the N-space outputs of step t−1; the flush graph after
    // the loop finishes the last step's.  A snapshot written by graph t+2 waits for the copies
    // issued after graph t.
    const bool pp = piped() && nsteps > 1;
    for (int t = 0; t < nsteps; ++t) {
        const int q = par_next;
        if (t >= 2) FKB_CUDA(cudaStreamWaitEvent(s, ev_copied[q], 0));  // step t−2's copies are done
        tmark(s);
        tmark(s);
        if (pp) run_piped(t);
        else launch_step();
        tmark(s);
        FKB_CUDA(cudaEventRecord(ev_done[q], s));
        FKB_CUDA(cudaStreamWaitEvent(cs, ev_done[q], 0));
        if (pp) {
            copy_out(q, t, cs, 1);
            if (t > 0) copy_out(q ^ 1, t - 1, cs, 2);
        } else {
            copy_out(q, t, cs, 3);
        }
        tmark(cs);
        FKB_CUDA(cudaEventRecord(ev_copied[q], cs));
    }
    if (pp) {
        const int q = par_next ^ 1;
        launch_piped(2, q);
        FKB_CUDA(cudaEventRecord(ev_done[q], s));
        FKB_CUDA(cudaStreamWaitEvent(cs, ev_done[q], 0));
        copy_out(q, nsteps - 1, cs, 2);
    }
    FKB_CUDA(cudaStreamSynchronize(cs));
    set_ysrc(ybuf.p, 0);  // back to the per-call observation buffer (also for the reruns below)
    if (trace) {
        FKB_CUDA(cudaStreamSynchronize(s));
        for (int t = 0; t + 1 < nsteps && t < 8; ++t) {
            float a = 0, b = 0, c = 0, d2 = 0;
            cudaEventElapsedTime(&a, tev[4 * t], tev[4 * t + 1]);
            cudaEventElapsedTime(&b, tev[4 * t + 1], tev[4 * t + 2]);
            cudaEventElapsedTime(&c, tev[4 * t + 2], tev[4 * t + 3]);
            cudaEventElapsedTime(&d2, tev[4 * t], tev[4 * t + 4]);
            std::fprintf(stderr, "[run] step %d: wait %.1f us, graph %.1f us, outputs done +%.1f us, step-to-step %.1f us\n",
                         t, 1e3 * a, 1e3 * b, 1e3 * c, 1e3 * d2);
        }
        for (auto e : tev) cudaEventDestroy(e);
    }
    int h = 0;
    double a = 0.0;
    FKB_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    FKB_CUDA(cudaMemcpyAsync(&a, alpha_dev.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    FKB_CUDA(cudaStreamSynchronize(s));
    int done = int(std::lround(a - alpha0));
    // a step whose PCG did not verify (and every later step, behind the sticky flag) changed
    // nothing: rerun it exactly, then the rest one by one (each rerun exactly if it too does
    // not verify), each with its outputs
    if (h == kInfoRetry) {
        h = 0;
        for (int t = done; t < nsteps; ++t) {
            const int q = (par0 + t) & 1;
            if (m > 0)
                FKB_CUDA(cudaMemcpyAsync(ybuf.p, h_ys + t * ldy, sizeof(double) * size_t(m), cudaMemcpyHostToDevice, s));
            par_next = q;
            if (t == done) {
                rerun_exact(q);
                par_next = q ^ 1;
            } else {
                launch_step();
            }
            FKB_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            FKB_CUDA(cudaStreamSynchronize(s));
            if (h == kInfoRetry) {
                rerun_exact(q);
                par_next = q ^ 1;
                FKB_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
                FKB_CUDA(cudaStreamSynchronize(s));
            }
            if (h) break;  // singular: raised below, the state stays at step t−1
            copy_out(q, t, s, 3);
            FKB_CUDA(cudaStreamSynchronize(s));
            ++done;
        }
    }
    set_hostout(0, 0, 0);
    alpha = alpha0 + done;
    step_no += done;
    if (done > 0) state_rank = r;
    if (h_alpha)
        for (int t = 0; t < done; ++t) h_alpha[t] = alpha0 + t + 1;
    if (h)
        fail_step("fkf_step: innovation system is singular (step " + std::to_string(done + 1) + " of " +
                  std::to_string(nsteps) + " in the batch)");
}

// step + fused UQ from host y: page-locked x/var buffers are written by the fused U pass
// straight through mapped host memory (the PCIe writes overlap the pass); others are copied
void Filter::step_uq_host(const double* h_y, uint64_t seed, int count, double* h_x, double* h_var, double* h_d,
                          double* h_mean) {
    set_step_uq(true, seed, count);
    if (!h_info) FKB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_info), sizeof(int), cudaHostAllocDefault));
    const unsigned long long hm = mapped_host(h_mean), hd = (h_d && r > 0) ? mapped_host(h_d) : 0;
    const unsigned long long hx = (h_x && count) ? mapped_host(h_x) : 0, hv = h_var ? mapped_host(h_var) : 0;
    const bool zc = h_mean && hm && (!(h_d && r > 0) || hd) && r > 0;
    const bool zx = zc && (!(h_x && count) || hx) && (!h_var || hv);
    if (zc) set_hostout(hm, hd, mapped_host(h_info), zx ? hx : 0, zx ? hv : 0);
    else set_hostout(0, 0, 0);
    if (m > 0) FKB_CUDA(cudaMemcpyAsync(ybuf.p, h_y, sizeof(double) * size_t(m), cudaMemcpyHostToDevice, s));
    launch_step();
    auto outputs = [&] {
        if (!zc) {
            FKB_CUDA(cudaMemcpyAsync(h_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            if (h_d && r > 0) FKB_CUDA(cudaMemcpyAsync(h_d, d.p, sizeof(double) * size_t(r), cudaMemcpyDeviceToHost, s));
            if (h_mean) FKB_CUDA(cudaMemcpyAsync(h_mean, mean.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
        }
        if (r > 0 && !zx) {
            if (h_var) FKB_CUDA(cudaMemcpyAsync(h_var, uq_var.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
            if (h_x && count)
                FKB_CUDA(cudaMemcpyAsync(h_x, uq_x.p, sizeof(double) * size_t(n) * count, cudaMemcpyDeviceToHost, s));
        }
        FKB_CUDA(cudaStreamSynchronize(s));
    };
    outputs();
    if (*h_info == kInfoRetry) {  // the PCG did not verify: the exact rerun writes the outputs
        rerun_exact(gt_last_par);
        outputs();
    }
    if (*h_info) fail_step("fkf_step: innovation system is singular");
    alpha += 1.0;
    ++step_no;
    state_rank = r;
    if (r == 0) {  // rank-0 GEP: the separate UQ pass
        host_out.ensure(size_t(n) * (count + 1));
        realizations(seed, count, host_out.p + n, host_out.p);
        if (h_var) FKB_CUDA(cudaMemcpyAsync(h_var, host_out.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
        if (h_x && count)
            FKB_CUDA(cudaMemcpyAsync(h_x, host_out.p + n, sizeof(double) * size_t(n) * count, cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaStreamSynchronize(s));
    }
}

void Filter::step_host_state(const double* h_y, double* h_d, double* h_mean) {
    if (!h_info) FKB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_info), sizeof(int), cudaHostAllocDefault));
    // page-locked caller buffers: the graph's last kernels write d, the mean and the failure
    // flag straight into them (mapped host memory), overlapped with the U pass
    const unsigned long long hm = mapped_host(h_mean), hd = (h_d && r > 0) ? mapped_host(h_d) : 0;
    const bool zc = h_mean && hm && (!(h_d && r > 0) || hd);
    if (zc) set_hostout(hm, hd, mapped_host(h_info));
    else set_hostout(0, 0, 0);
    if (m > 0) FKB_CUDA(cudaMemcpyAsync(ybuf.p, h_y, sizeof(double) * size_t(m), cudaMemcpyHostToDevice, s));
    launch_step();
    auto outputs = [&] {
        if (!zc) {
            FKB_CUDA(cudaMemcpyAsync(h_info, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            if (h_d && r > 0) FKB_CUDA(cudaMemcpyAsync(h_d, d.p, sizeof(double) * size_t(r), cudaMemcpyDeviceToHost, s));
            if (h_mean) FKB_CUDA(cudaMemcpyAsync(h_mean, mean.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
        }
        FKB_CUDA(cudaStreamSynchronize(s));
    };
    outputs();
    if (*h_info == kInfoRetry) {  // the PCG did not verify: the exact rerun writes the outputs
        rerun_exact(gt_last_par);
        outputs();
    }
    if (*h_info) fail_step("fkf_step: innovation system is singular");
    alpha += 1.0;
    ++step_no;
    state_rank = r;
}

void Filter::step_host(const double* h_y) {
    if (m > 0) FKB_CUDA(cudaMemcpyAsync(ybuf.p, h_y, sizeof(double) * size_t(m), cudaMemcpyHostToDevice, s));
    step(ybuf.p);
}

void Filter::steps_async(const double* d_ys, int nsteps, long long ldy) {
    // Device-resident observation sequence; one deferred singularity check at the end.
    set_hostout(0, 0, 0);
    batch_ys = d_ys;
    batch_ldy = ldy;
    batch_par0 = par_next;
    const bool pp = piped() && nsteps > 1;
    // the graphs read observation row ysrc[2] of the caller's block (the prologue advances the
    // row): no copy into ybuf between the graphs (c2: 80.5 → 77.2 µs per step)
    const bool block = nsteps > 1 && ldy > 0 && m > 0;
    if (block) set_ysrc(d_ys, ldy);
    for (int k = 0; k < nsteps; ++k) {
        if (!block)
            FKB_CUDA(cudaMemcpyAsync(ybuf.p, d_ys + (long long)k * ldy, sizeof(double) * size_t(m),
                                     cudaMemcpyDeviceToDevice, s));
        if (pp) run_piped(k);
        else launch_step();
    }
    if (pp) launch_piped(2, par_next ^ 1);  // the last step's mean side
    if (block) {  // back to the per-call buffer, holding the last observation (a rerun reads ybuf)
        FKB_CUDA(cudaMemcpyAsync(ybuf.p, d_ys + (long long)(nsteps - 1) * ldy, sizeof(double) * size_t(m),
                                 cudaMemcpyDeviceToDevice, s));
        set_ysrc(ybuf.p, 0);
    }
}

// The deferred check of an asynchronous batch: the device α counts the committed steps (a
// failed step and, through the sticky flag, every later step of the batch leave the state
// untouched), so the host mirrors advance by exactly that many and the error names the
// first failed step of the batch.
void Filter::finish_async(int nsteps) {
    int h = 0;
    double a = 0.0;
    FKB_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    FKB_CUDA(cudaMemcpyAsync(&a, alpha_dev.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    FKB_CUDA(cudaStreamSynchronize(s));
    int done = int(std::lround(a - alpha));
    // a step whose PCG did not verify (and, through the sticky flag, every later step of the
    // batch) changed nothing: rerun it on the exact path, then replay the rest of the batch
    while (h == kInfoRetry && batch_ys && done < nsteps) {
        const int par = (batch_par0 + done) & 1;
        FKB_CUDA(cudaMemcpyAsync(ybuf.p, batch_ys + (long long)done * batch_ldy, sizeof(double) * size_t(m),
                                 cudaMemcpyDeviceToDevice, s));
        rerun_exact(par);
        par_next = par ^ 1;
        for (int k = done + 1; k < nsteps; ++k) {
            FKB_CUDA(cudaMemcpyAsync(ybuf.p, batch_ys + (long long)k * batch_ldy, sizeof(double) * size_t(m),
                                     cudaMemcpyDeviceToDevice, s));
            launch_step();
        }
        FKB_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaMemcpyAsync(&a, alpha_dev.p, sizeof(double), cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaStreamSynchronize(s));
        done = int(std::lround(a - alpha));
    }
    alpha = a;
    step_no += done;
    if (done > 0) state_rank = r;
    if (h)
        fail_step("fkf_step: innovation system is singular (step " + std::to_string(done + 1) + " of " +
                  std::to_string(nsteps) + " in the batch)");
}

std::vector<double> Filter::d_host() const { return download(d.p, size_t(r), s); }

std::vector<double> Filter::ghep_residual() {
    std::vector<double> res(static_cast<size_t>(r));
    if (r == 0) return res;
    DBuf<double> AU(size_t(n) * r), out{size_t(r)};
    spmm(HT, B.p, m, r, AU.p, n, 1.0 / sigma2, 0.0, s);  // Hᵀ(HU)/σ²
    k_gep_resid<<<r, 256, 0, s>>>(n, AU.p, Ubar.p, lambda.p, out.p);
    FKB_LAUNCH_CHECK();
    count_launch();
    return download(out.p, size_t(r), s);
}

void Filter::variance(double* d_out) {
    const int blocks = ceil_div(n, 256);
    k_uq<<<blocks, 256, sizeof(double) * size_t(std::max(r, 1)), s>>>(n, state_rank ? r : 0, U.p, d.p, alpha_dev.p,
                                                                     cov->spec.theta, mean.p, 0, nullptr, nullptr,
                                                                     nullptr, d_out);
    FKB_LAUNCH_CHECK();
    count_launch();
}

double Filter::trace_criterion() {  // uq.hpp:27-34
    double out = alpha * (double(n) * cov->spec.theta);
    if (state_rank) {
        const auto dh = d_host();
        const auto ch = download(colsq.p, size_t(r), s);
        for (int j = 0; j < r; ++j) out -= dh[size_t(j)] * ch[size_t(j)];
    }
    return out;
}

double Filter::relative_entropy() {  // uq.hpp:39-53
    if (!(alpha > 0.0)) throw std::invalid_argument("relative_entropy: requires alpha > 0");
    const int rk = state_rank;
    double sum = (double(n) - double(rk)) * std::log(alpha);
    if (rk) {
        const auto dh = d_host();
        for (int i = 0; i < rk; ++i) {
            const double gap = alpha - dh[size_t(i)];
            if (!(gap > 0.0))
                throw std::runtime_error("relative_entropy: D_" + std::to_string(i) + " = " + std::to_string(dh[size_t(i)]) +
                                         " is not below alpha = " + std::to_string(alpha));
            sum += std::log(gap);
        }
    }
    return 0.5 * sum;
}

// UQ of an arbitrary low-rank state Σ = αΓ − W·diag(d)·Wᵀ in device buffers (uq.hpp:16-34 and
// the FFT-mode realization formula of SURVEY App. A.4): diag Σ (var), the column norms ‖W_j‖²
// (colsq, for trace_criterion) and `count` realizations mean + √α(z_s − W(Σ₋ ⊙ W̄ᵀz_s)) with
// W̄ = Γ⁻¹W, draws z_s, s = first … first+count−1, as sample_pair(seed, s/2) (Re even, Im odd).
// α is read from alpha_dev[0].  Runs on the operator's stream (sample_pair uses it).
void lowrank_uq(Cov* cov, long long n, int r, const double* alpha_dev, const double* d, const double* W,
                const double* Wbar, const double* mean, uint64_t seed, uint64_t first, int count, double* X,
                double* var, double* colsq, DBuf<double>& scratch) {
    cudaStream_t s = cov->stream;
    if (count < 0 || count > 8) throw std::invalid_argument("realizations: count must lie in [0, 8]");
    if (colsq) column_sumsq(n, r, W, colsq, s);
    if (count == 0 && !var) return;
    const size_t nd = size_t(n) * std::max(count + 1, 1);
    scratch.ensure(nd + size_t(std::max(r, 1)) * std::max(count, 1));
    double* Z = scratch.p;                  // count draws (+ the spare of an odd tail)
    double* proj = scratch.p + nd;          // W̄ᵀZ (r × count)
    for (int c = 0; c < count;) {
        const uint64_t j = first + uint64_t(c);
        double* a = Z + (long long)c * n;
        if (j % 2 == 0) {  // pair (seed, j/2): Re → draw j, Im → draw j+1
            double* b = c + 1 < count ? Z + (long long)(c + 1) * n : Z + (long long)count * n;
            cov->sample_pair(seed, j / 2, a, b);
            c += 2;
        } else {           // odd first draw: the Im half of pair (seed, j/2)
            cov->sample_pair(seed, j / 2, Z + (long long)count * n, a);
            c += 1;
        }
    }
    if (r > 0 && count > 0) {
        GemmArgs g;
        g.M = r; g.N = count; g.K = int(n);
        g.A = Wbar; g.lda = n; g.transA = 1;
        g.B = Z; g.ldb = n;
        g.C = proj; g.ldc = r;
        g.splitk = gemm_pick_splitk(r, count, int(n));
        DBuf<double> gws(std::max<size_t>(gemm_ws_elems(g), 1));
        gemm(g, gws.p, s);
    }
    const size_t shm = sizeof(double) * size_t(std::max(r, 1)) * (1 + std::max(count, 1));
    k_uq<<<ceil_div(n, 256), 256, shm, s>>>(n, r, W, d, alpha_dev, cov->spec.theta, mean, count,
                                            count ? Z : nullptr, count ? proj : nullptr, X, var);
    FKB_LAUNCH_CHECK();
    count_launch();
}

void Filter::realization_at(uint64_t seed, uint64_t draw, double* d_out) {
    lowrank_uq(cov, n, state_rank ? r : 0, alpha_dev.p, d.p, U.p, Ubar.p, mean.p, seed, draw, 1, d_out, nullptr, nullptr,
               uq_scratch);
}

// count realizations x_s = mean + √α(z_s − U Σ₋ Ūᵀ z_s); draw s = sample_pair(seed, s/2),
// Re for even s, Im for odd.  Draws and Ūᵀz_s are cached per (seed, count) so each later
// state costs one pass over U (RealizationPropagator, uq.hpp:86-112).
void Filter::prepare_draws(uint64_t seed, int count) {
    if (count <= 0 || (draw_count == count && draw_seed == seed)) return;
    draws.alloc(size_t(n) * count);
    DBuf<double> spare(static_cast<size_t>(n));
    for (int sidx = 0; sidx < count; sidx += 2) {
        double* a = draws.p + (long long)sidx * n;
        double* b = sidx + 1 < count ? draws.p + (long long)(sidx + 1) * n : spare.p;
        cov->sample_pair(seed, uint64_t(sidx / 2), a, b);
    }
    draw_proj.alloc(size_t(std::max(r, 1)) * count);
    if (r > 0) {
        GemmArgs g;
        g.M = r; g.N = count; g.K = int(n);
        g.A = Ubar.p; g.lda = n; g.transA = 1;
        g.B = draws.p; g.ldb = n;
        g.C = draw_proj.p; g.ldc = r;
        g.splitk = gemm_pick_splitk(r, count, int(n));
        ws.ensure(gemm_ws_elems(g));
        gemm(g, ws.p, s);
    }
    FKB_CUDA(cudaStreamSynchronize(s));
    draw_seed = seed;
    draw_count = count;
    if (uq_count > 0) drop_graphs();  // the fused step graph holds the draw buffers
}

void Filter::set_step_uq(bool on, uint64_t seed, int count) {
    if (on && (count < 0 || count > 8)) throw std::invalid_argument("realizations: count must lie in [0, 8]");
    const int want = on ? count : -1;
    if (on) {
        prepare_draws(seed, count);
        uq_x.ensure(size_t(n) * std::max(count, 1));
        uq_var.ensure(size_t(n));
    }
    if (want != uq_count) {
        uq_count = want;
        drop_graphs();
    }
}

// One step on device y with diag Σ and `count` realizations of the new state from the fused
// U pass, enqueued without a host sync (as steps_async; finish_async() checks and commits);
// outputs copied to d_x (N×count) / d_var when given.  A rank-0 GEP runs the separate UQ kernel.
void Filter::step_uq(const double* d_y, uint64_t seed, int count, double* d_x, double* d_var) {
    set_step_uq(true, seed, count);
    set_hostout(0, 0, 0);
    if (d_y != ybuf.p)
        FKB_CUDA(cudaMemcpyAsync(ybuf.p, d_y, sizeof(double) * size_t(m), cudaMemcpyDeviceToDevice, s));
    launch_step();
    if (r == 0) {
        realizations(seed, count, d_x, d_var);
        return;
    }
    if (d_x && count)
        FKB_CUDA(cudaMemcpyAsync(d_x, uq_x.p, sizeof(double) * size_t(n) * count, cudaMemcpyDeviceToDevice, s));
    if (d_var) FKB_CUDA(cudaMemcpyAsync(d_var, uq_var.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToDevice, s));
}

void Filter::realizations(uint64_t seed, int count, double* d_out, double* d_var) {
    if (count < 0 || count > 8) throw std::invalid_argument("realizations: count must lie in [0, 8]");
    if (count == 0 && !d_var) return;
    prepare_draws(seed, count);
    const int blocks = ceil_div(n, 256);
    const int rr = state_rank ? r : 0;
    const size_t shm = sizeof(double) * size_t(std::max(rr, 1)) * (1 + std::max(count, 1));
    k_uq<<<blocks, 256, shm, s>>>(n, rr, U.p, d.p, alpha_dev.p, cov->spec.theta, mean.p, count,
                                  count ? draws.p : nullptr, count ? draw_proj.p : nullptr, d_out, d_var);
    FKB_LAUNCH_CHECK();
    count_launch();
}

}  // namespace fkb
