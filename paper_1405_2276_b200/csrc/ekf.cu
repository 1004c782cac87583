// ekf.cu — fekf_step (fast_filter.hpp:127-224): the extended fast filter for a linearized,
// time-varying H_k = H·diag(∂s/∂ŝ) with a per-step GHEP merged into the state by
// add_low_rank (lowrank.hpp:238-294) under the Γ⁻¹ metric.
//
// One step:
//   1. D̄ = α⁻¹(αI − D)⁻¹D (:152-158).
//   2. ≤ 5 relinearizations (:163-196): Box–Cox Jacobian and inverse at η (boxcox.hpp:81-90),
//      H_k values rescaled in place (same sparsity), G_k = H_kΓH_kᵀ streamed in column
//      batches (build_hgh), S = αG_k − (H_kW)D(H_kW)ᵀ + σ²I on DMMA, blocked LLT,
//      z = S⁻¹(y − h(η) − H_k(mean − η)), η' = mean + αΓ(H_kᵀz) − W(d ⊙ (H_kW)ᵀz).
//   3. GHEP of H_lastᵀH_last/σ² against Γ (randomized_ghep_device, shared with fkf_init).
//   4. add_low_rank(W, D̄, U, λ, Γ⁻¹): the reference runs column MGS in the Γ⁻¹ metric with
//      CG solves (lowrank.hpp:53-106); here V = U is projected out of span(W) by two block
//      classical Gram–Schmidt passes whose Γ⁻¹ products come from W̄ = Γ⁻¹W and Ū = Γ⁻¹U,
//      then orthonormalized by two Gram passes on DMMA with small eigensolves (the same
//      span-equivalent scheme as the GHEP, drop rule 1e-12 on the projected norms).  The core
//      matrix M = diag(D̄, 0) + [C; R̂]Λ[C; R̂]ᵀ is formed on DMMA and diagonalized on the host
//      (≤ 1024) or by the device block Jacobi; truncation, ordering and D = α²D̂(I + αD̂)⁻¹
//      follow :205-222.  W̄' = [W̄, V̂̄]·E is carried with W' = [W, V̂]·E.

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <numeric>
#include <sstream>

#include "eig.cuh"
#include "ekf.cuh"
#include "host_linalg.h"

namespace fkb {

// ∂s/∂ŝ and s(ŝ) at η (boxcox.hpp:33-50); bad[0]/bad[1] = first failing index of the
// derivative / inverse map (domain violation or non-finite value)
__global__ void k_boxcox_lin(long long n, const double* __restrict__ eta, double a, double* __restrict__ jac,
                             double* __restrict__ sinv, int* bad) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double x = eta[i];
        double j, v;
        bool dom = false;
        if (a == 1.0) {
            j = 1.0;
            v = x + 1.0;
        } else {
            const double base = (x + a) / a;
            dom = base < 0.0;
            j = pow(base, a - 1.0);
            v = pow(base, a);
        }
        jac[i] = j;
        sinv[i] = v;
        if (dom || !isfinite(j)) atomicMin(bad, int(i));
        if (dom || !isfinite(v)) atomicMin(bad + 1, int(i));
    }
}

// H_k = H·diag(jac) on both stored orientations (rows of Hᵀ are cells)
__global__ void k_scale_cols(long long nnz, const int* __restrict__ col, const double* __restrict__ v,
                             const double* __restrict__ jac, double* __restrict__ out) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nnz; e += (long long)gridDim.x * blockDim.x)
        out[e] = v[e] * jac[col[e]];
}

__global__ void k_rows_of(int rows, const int* __restrict__ rp, int* __restrict__ row_of) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    for (int e = rp[r]; e < rp[r + 1]; ++e) row_of[e] = r;
}

// out = a − b (n)
__global__ void k_sub(long long n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = a[i] - b[i];
}
// z = y − h(η) − z   (z holds H_k(mean − η) on entry)
__global__ void k_innovation(int m, const double* __restrict__ y, const double* __restrict__ heta, double* z) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) z[i] = y[i] - heta[i] - z[i];
}
// out = mean + a·g
__global__ void k_axpy_to(long long n, const double* __restrict__ mean, double a, const double* __restrict__ g,
                          double* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = fma(a, g[i], mean[i]);
}
// A[i,i] += v[i], i < k
__global__ void k_add_diag(int k, const double* __restrict__ v, double* A, long long lda) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) A[i + (long long)i * lda] += v[i];
}
// columns j of A (n×p): A[:, j] *= sc[j]
__global__ void k_scale_columns(long long n, int p, double* A, const double* __restrict__ sc) {
    const int j = blockIdx.y;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        A[i + (long long)j * n] *= sc[j];
}

// FKB_EKF_TRACE=1: per-phase wall times of each step on stderr (stream-synchronized)
static bool ekf_trace() {
    static const bool on = std::getenv("FKB_EKF_TRACE") != nullptr;
    return on;
}
struct PhaseClock {
    cudaStream_t s;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void lap(const char* what) {
        if (!ekf_trace()) return;
        cudaStreamSynchronize(s);
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[ekf] %-18s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

static int grid_for(long long n) { return int(std::max<long long>(1, std::min<long long>((n + 255) / 256, 2048))); }

// C (n×q) = beta·Cin + alpha·A (n×p) · B (p×q, ld ldb), all column-major on the device
static void gemm_nn(long long n, int q, int p, double alpha, const double* A, const double* B, long long ldb,
                    double beta, const double* Cin, double* C, cudaStream_t s) {
    GemmArgs g;
    g.M = int(n); g.N = q; g.K = p;
    g.A = A; g.lda = n;
    g.B = B; g.ldb = ldb;
    g.alpha = alpha;
    g.beta = beta;
    g.Cin = Cin; g.ldcin = n;
    g.C = C; g.ldc = n;
    gemm(g, nullptr, s);
}

Ekf::Ekf(Cov* c, int m_, int h_cols, const int* rowptr, const int* col, const double* val)
    : cov(c), s(c->stream), n(c->size()), m(m_) {
    if (m < 0) throw std::invalid_argument("fekf_step: negative measurement count");
    if ((long long)h_cols != n) throw std::invalid_argument("fekf_step: dimension mismatch");
    for (int i = 0; i < m; ++i)
        for (int e = rowptr[i]; e < rowptr[i + 1]; ++e)
            if (col[e] < 0 || col[e] >= n) throw std::invalid_argument("fekf_step: H column index out of range");
    upload_csr_pair(m, int(n), rowptr, col, val, H, HT);
    upload_csr_pair(m, int(n), rowptr, col, val, Hk, HkT);
    ht_cell.alloc(size_t(std::max<long long>(HT.nnz, 1)));
    if (HT.nnz) {
        k_rows_of<<<ceil_div(HT.rows, 256), 256, 0, s>>>(HT.rows, HT.rowptr.p, ht_cell.p);
        FKB_LAUNCH_CHECK();
        count_launch();
    }
    mean.alloc(size_t(n));
    for (DBuf<double>* b : {&eta, &eta2, &jac, &sinv, &tv, &gt}) b->alloc(size_t(n));
    for (DBuf<double>* b : {&heta, &z, &ybuf}) b->alloc(size_t(std::max(m, 1)));
    G.alloc(size_t(std::max(m, 1)) * std::max(m, 1));
    S.alloc(size_t(std::max(m, 1)) * std::max(m, 1));
    info.alloc(1);
    flags.alloc(size_t(2 * ceil_div(std::max(m, 1), 64) + 2));
    bad.alloc(2);
    std::vector<double> zero(static_cast<size_t>(n), 0.0);
    reset(zero.data());
}

void Ekf::reset(const double* mean0) {  // LowRankState::zero_start + initial mean (driver.hpp:315-316)
    FKB_CUDA(cudaMemcpyAsync(mean.p, mean0, sizeof(double) * size_t(n), cudaMemcpyHostToDevice, s));
    FKB_CUDA(cudaStreamSynchronize(s));
    alpha = 0.0;
    step_no = 0;
    r = 0;
    d_h.clear();
    W.release();
    Wbar.release();
    d.release();
}

void Ekf::linearize(double a) {  // ekf_linearize (boxcox.hpp:81-90)
    FKB_CUDA(cudaMemsetAsync(bad.p, 0x7f, 2 * sizeof(int), s));
    k_boxcox_lin<<<grid_for(n), 256, 0, s>>>(n, eta.p, a, jac.p, sinv.p, bad.p);
    FKB_LAUNCH_CHECK();
    count_launch();
    int b[2];
    FKB_CUDA(cudaMemcpyAsync(b, bad.p, sizeof b, cudaMemcpyDeviceToHost, s));
    FKB_CUDA(cudaStreamSynchronize(s));
    for (int which = 0; which < 2; ++which) {  // derivative first, then inverse (boxcox.hpp:86-88)
        if (b[which] == 0x7f7f7f7f) continue;
        const int i = b[which];
        double x = 0.0;
        FKB_CUDA(cudaMemcpy(&x, eta.p + i, sizeof(double), cudaMemcpyDeviceToHost));
        const char* what = which ? "inverse" : "derivative";
        const double base = (x + a) / a;
        if (a != 1.0 && base < 0.0)
            throw DomainError(std::string("boxcox: ") + what + " domain violation at index " + std::to_string(i) +
                              " (value " + std::to_string(x) + ")");
        throw DomainError(std::string("boxcox: ") + what + " produced a non-finite value at index " +
                          std::to_string(i));
    }
    if (H.nnz) {
        k_scale_cols<<<grid_for(H.nnz), 256, 0, s>>>(H.nnz, H.col.p, H.val.p, jac.p, Hk.val.p);
        FKB_LAUNCH_CHECK();
        k_scale_cols<<<grid_for(HT.nnz), 256, 0, s>>>(HT.nnz, ht_cell.p, HT.val.p, jac.p, HkT.val.p);
        FKB_LAUNCH_CHECK();
        count_launch(2);
    }
    spmm(H, sinv.p, n, 1, heta.p, std::max(m, 1), 1.0, 0.0, s);  // h(η) = H·s(η)
}

void Ekf::step(const double* y_h, double sigma2, double a_bc, const EkfOptions& o) {
    if (!(sigma2 > 0.0)) throw std::invalid_argument("fekf_step: sigma2 must be positive");  // :145-150
    if (o.relinearizations < 1 || o.relinearizations > 5)
        throw std::invalid_argument("fekf_step: relinearizations must lie in [1, 5]");
    const double a = alpha + 1.0;  // :152
    std::vector<double> d_bar(static_cast<size_t>(r));
    for (int i = 0; i < r; ++i) {  // :155-159
        if (!(d_h[size_t(i)] < a)) throw std::runtime_error("fekf_step: state diagonal exceeds alpha");
        d_bar[size_t(i)] = d_h[size_t(i)] / (a * (a - d_h[size_t(i)]));
    }
    if (!(a_bc > 0.0)) throw std::invalid_argument("boxcox: alpha must be positive, got " + std::to_string(a_bc));
    if (m > 0) FKB_CUDA(cudaMemcpyAsync(ybuf.p, y_h, sizeof(double) * size_t(m), cudaMemcpyHostToDevice, s));
    FKB_CUDA(cudaMemcpyAsync(eta.p, mean.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToDevice, s));
    if (r > 0) HW.ensure(size_t(std::max(m, 1)) * r);
    last_relin = 0;
    PhaseClock clk{s};
    for (int it = 0; it < o.relinearizations; ++it) {  // :163-196
        ++last_relin;
        linearize(a_bc);
        clk.lap("linearize");
        if (m > 0) {
            build_hgh(cov, Hk, G.p, s, &hgh_ws);  // H_k Γ H_kᵀ (:171-176)
            clk.lap("HkGHkT");
            if (r > 0) spmm(Hk, W.p, n, r, HW.p, m, 1.0, 0.0, s);  // H_k W (:173)
            GemmArgs g;  // S = αG_k − (H_kW) D (H_kW)ᵀ + σ²I (:175-178)
            g.M = m; g.N = m; g.K = r;
            g.A = HW.p; g.lda = m;
            g.B = HW.p; g.ldb = m; g.transB = 1;
            g.dA = r ? d.p : nullptr;
            g.alpha = -1.0;
            g.beta = a;
            g.Cin = G.p; g.ldcin = m;
            g.C = S.p; g.ldc = m;
            g.diag_add = sigma2;
            gemm(g, nullptr, s);
            symmetrize(m, S.p, m, s);
            FKB_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), s));
            pws.ensure(potrf_ws_elems(m));
            potrf_lower(m, S.p, m, info.p, pws.p, potrf_ws_elems(m), s);  // LLT (:179-181)
            int h = 0;
            FKB_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
            FKB_CUDA(cudaStreamSynchronize(s));
            if (h) throw std::runtime_error("fekf_step: innovation system is singular");
            clk.lap("S build + LLT");
            // z = S⁻¹(y − h(η) − H_k(mean − η)) (:183-184)
            k_sub<<<grid_for(n), 256, 0, s>>>(n, mean.p, eta.p, tv.p);
            FKB_LAUNCH_CHECK();
            count_launch();
            spmm(Hk, tv.p, n, 1, z.p, m, 1.0, 0.0, s);
            k_innovation<<<ceil_div(m, 256), 256, 0, s>>>(m, ybuf.p, heta.p, z.p);
            FKB_LAUNCH_CHECK();
            count_launch();
            potrs_lower(m, S.p, m, z.p, flags.p, s);
            // η' = mean + α·Γ(H_kᵀz) − W(d ⊙ (H_kW)ᵀz) (:185-187)
            spmm(HkT, z.p, m, 1, tv.p, n, 1.0, 0.0, s);
            cov->apply(tv.p, n, 1, gt.p, n);
            k_axpy_to<<<grid_for(n), 256, 0, s>>>(n, mean.p, a, gt.p, eta2.p);
            FKB_LAUNCH_CHECK();
            count_launch();
            if (r > 0) {
                dc.ensure(size_t(r));
                GemmArgs u;  // dc = d ⊙ (H_kW)ᵀz
                u.M = r; u.N = 1; u.K = m;
                u.A = HW.p; u.lda = m; u.transA = 1;
                u.B = z.p; u.ldb = m;
                u.rs = d.p;
                u.C = dc.p; u.ldc = r;
                gemm(u, nullptr, s);
                gemm_nn(n, 1, r, -1.0, W.p, dc.p, r, 1.0, eta2.p, eta2.p, s);
            }
        } else {
            FKB_CUDA(cudaMemcpyAsync(eta2.p, mean.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToDevice, s));
        }
        // change = ‖η' − η‖ ≤ 1e-6‖η'‖ ends the sweeps (:189-195)
        k_sub<<<grid_for(n), 256, 0, s>>>(n, eta2.p, eta.p, tv.p);
        FKB_LAUNCH_CHECK();
        count_launch();
        ws.ensure(4096);
        const double change = std::sqrt(sumsq(tv.p, n, ws.p, s));
        std::swap(eta, eta2);
        const double enorm = std::sqrt(sumsq(eta.p, n, ws.p, s));
        clk.lap("mean update");
        if (change <= 1e-6 * enorm) break;
    }
    // GHEP of H_lastᵀH_last/σ² (:198-203); H_k holds the last linearization
    const long long k_rank = o.k_rank < 0 ? m : o.k_rank;
    GepDev& g = gep;  // device temporaries persist across steps
    randomized_ghep_device(cov, Hk, HkT, sigma2, k_rank, o.oversampling, o.seed, ws, s, g);
    last_gep_rank = g.r;
    clk.lap("ghep");
    add_low_rank(d_bar, g, o.trunc_tol, a);
    clk.lap("add_low_rank");
    std::swap(mean, eta);  // :212
    alpha = a;
    ++step_no;
}

void Ekf::add_low_rank(const std::vector<double>& d_bar, GepDev& g, double tol, double a) {
    if (tol < 0.0) throw std::invalid_argument("add_low_rank: tol must be nonnegative");
    PhaseClock ck{s};
    const int kv = g.r;
    std::vector<double> dsum;  // D̂ before the d̂ > 1e-14 filter (lowrank.hpp:248-249)
    std::vector<int> keep;
    std::vector<double> Ek;  // (r + kh) × |keep| combination of [W, V̂], column-major
    int nm = 0, kh = 0;
    if (kv == 0 || r == 0) {
        if (kv == 0) dsum = d_bar;
        else dsum = g.lambda_h;
        for (int i = 0; i < int(dsum.size()); ++i)
            if (dsum[size_t(i)] > 1e-14) keep.push_back(i);  // fast_filter.hpp:207-209
        const int rk = int(keep.size());
        const int src_r = kv == 0 ? r : kv;
        const double* src = kv == 0 ? W.p : g.U.p;
        const double* srcb = kv == 0 ? Wbar.p : g.Ubar.p;
        Wn.ensure(size_t(n) * std::max(rk, 1));
        Wbn.ensure(size_t(n) * std::max(rk, 1));
        for (int i = 0; i < rk; ++i) {
            FKB_CUDA(cudaMemcpyAsync(Wn.p + (long long)i * n, src + (long long)keep[size_t(i)] * n, sizeof(double) * n,
                                     cudaMemcpyDeviceToDevice, s));
            FKB_CUDA(cudaMemcpyAsync(Wbn.p + (long long)i * n, srcb + (long long)keep[size_t(i)] * n,
                                     sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        }
        (void)src_r;
    } else {
        // ---- b_orthonormalize(V = U, Γ⁻¹, against = W) by block CGS2 (lowrank.hpp:53-106, :254)
        DBuf<double>& C = tmp(0, size_t(r) * kv);
        DBuf<double>& C2 = tmp(1, size_t(r) * kv);
        DBuf<double>& V = tmp(2, size_t(n) * kv);
        DBuf<double>& Vb = tmp(3, size_t(n) * kv);
        gram_tn(n, r, kv, Wbar.p, g.U.p, C.p, ws, s);                                // C = W̄ᵀV (:258)
        gemm_nn(n, kv, r, -1.0, W.p, C.p, r, 1.0, g.U.p, V.p, s);                    // V₁ = V − WC
        gemm_nn(n, kv, r, -1.0, Wbar.p, C.p, r, 1.0, g.Ubar.p, Vb.p, s);             // V̄₁ = V̄ − W̄C
        gram_tn(n, r, kv, Wbar.p, V.p, C2.p, ws, s);                                 // second pass
        gemm_nn(n, kv, r, -1.0, W.p, C2.p, r, 1.0, V.p, V.p, s);
        gemm_nn(n, kv, r, -1.0, Wbar.p, C2.p, r, 1.0, Vb.p, Vb.p, s);
        DBuf<double>& Gd = tmp(4, size_t(kv) * kv);
        gram_tn(n, kv, kv, V.p, Vb.p, Gd.p, ws, s);
        std::vector<double> Gh = download(Gd.p, size_t(kv) * kv, s);
        // projected Γ⁻¹-norms (pre-norms are 1: U is Γ⁻¹-orthonormal); MGS drops ≤ 1e-12 (:92-95)
        std::vector<int> live;
        std::vector<double> sc(static_cast<size_t>(kv), 0.0);
        for (int j = 0; j < kv; ++j) {
            const double nj = std::sqrt(std::max(Gh[size_t(j) + size_t(j) * kv], 0.0));
            if (nj > 1e-12) {
                live.push_back(j);
                sc[size_t(j)] = 1.0 / nj;
            }
        }
        const int kl = int(live.size());
        if (kl > 0) {
            // first Gram pass on the unit-scaled live columns
            std::vector<double> Gs(static_cast<size_t>(kl) * kl);
            for (int q = 0; q < kl; ++q)
                for (int p = 0; p < kl; ++p)
                    Gs[size_t(p) + size_t(q) * kl] = Gh[size_t(live[size_t(p)]) + size_t(live[size_t(q)]) * kv] *
                                                     sc[size_t(live[size_t(p)])] * sc[size_t(live[size_t(q)])];
            int k1 = 0;
            std::vector<double> W1 = gram_inv_sqrt(kl, Gs, 1e-13, k1);
            if (k1 > 0) {
                std::vector<double> T1(static_cast<size_t>(kv) * k1, 0.0);  // kv × k1 with the column scaling
                for (int c = 0; c < k1; ++c)
                    for (int p = 0; p < kl; ++p)
                        T1[size_t(live[size_t(p)]) + size_t(c) * kv] = W1[size_t(p) + size_t(c) * kl] * sc[size_t(live[size_t(p)])];
                DBuf<double>& Td = tmp(5, T1.size());
                upload(Td.p, T1, s);
                DBuf<double>& Q = tmp(6, size_t(n) * k1);
                DBuf<double>& Qb = tmp(7, size_t(n) * k1);
                DBuf<double>& C3 = tmp(8, size_t(r) * k1);
                tall_times_small(n, kv, k1, V.p, Td.p, Q.p, s);
                tall_times_small(n, kv, k1, Vb.p, Td.p, Qb.p, s);
                gram_tn(n, r, k1, Wbar.p, Q.p, C3.p, ws, s);  // third projection after normalization
                gemm_nn(n, k1, r, -1.0, W.p, C3.p, r, 1.0, Q.p, Q.p, s);
                gemm_nn(n, k1, r, -1.0, Wbar.p, C3.p, r, 1.0, Qb.p, Qb.p, s);
                DBuf<double>& G2 = tmp(9, size_t(k1) * k1);
                gram_tn(n, k1, k1, Q.p, Qb.p, G2.p, ws, s);
                std::vector<double> W2 = gram_inv_sqrt(k1, download(G2.p, size_t(k1) * k1, s), 1e-13, kh);
                if (kh > 0) {
                    DBuf<double>& T2 = tmp(10, W2.size());
                    upload(T2.p, W2, s);
                    Vh.ensure(size_t(n) * kh);
                    Vhb.ensure(size_t(n) * kh);
                    tall_times_small(n, k1, kh, Q.p, T2.p, Vh.p, s);   // V̂
                    tall_times_small(n, k1, kh, Qb.p, T2.p, Vhb.p, s); // Γ⁻¹V̂
                }
            }
        }
        // ---- core matrix M = diag(D̄, 0) + [C; R̂] Λ [C; R̂]ᵀ (:257-265)
        nm = r + kh;
        DBuf<double>& Z = tmp(11, size_t(nm) * kv);
        DBuf<double>& Md = tmp(12, size_t(nm) * nm);
        DBuf<double>& lam = tmp(13, size_t(kv));
        {
            GemmArgs gc;  // rows 0..r-1: C = W̄ᵀV (recomputed into Z's rows)
            gc.M = r; gc.N = kv; gc.K = int(n);
            gc.A = Wbar.p; gc.lda = n; gc.transA = 1;
            gc.B = g.U.p; gc.ldb = n;
            gc.C = Z.p; gc.ldc = nm;
            gc.splitk = gemm_pick_splitk(r, kv, int(n));
            ws.ensure(gemm_ws_elems(gc));
            gemm(gc, ws.p, s);
            if (kh > 0) {  // rows r..: R̂ = (Γ⁻¹V̂)ᵀV (:259)
                GemmArgs gr = gc;
                gr.M = kh;
                gr.A = Vhb.p;
                gr.C = Z.p + r;
                gr.splitk = gemm_pick_splitk(kh, kv, int(n));
                ws.ensure(gemm_ws_elems(gr));
                gemm(gr, ws.p, s);
            }
        }
        upload(lam.p, g.lambda_h, s);
        {
            GemmArgs gm;
            gm.M = nm; gm.N = nm; gm.K = kv;
            gm.A = Z.p; gm.lda = nm;
            gm.B = Z.p; gm.ldb = nm; gm.transB = 1;
            gm.dA = lam.p;
            gm.C = Md.p; gm.ldc = nm;
            gemm(gm, nullptr, s);
            DBuf<double>& db = tmp(14, size_t(r));
            upload(db.p, d_bar, s);
            k_add_diag<<<ceil_div(r, 256), 256, 0, s>>>(r, db.p, Md.p, nm);
            FKB_LAUNCH_CHECK();
            count_launch();
            symmetrize(nm, Md.p, nm, s);
            FKB_CUDA(cudaStreamSynchronize(s));
        }
        ck.lap("alr: project+core");
        std::vector<double> ev(static_cast<size_t>(nm)), vec(static_cast<size_t>(nm) * nm);
        if (nm <= 2048) {  // Householder + QL, O(n³) on the GPU (tdeig.cu); block Jacobi beyond
            DBuf<double>& Vd = tmp(16, size_t(nm) * nm);
            sym_eig_tridiag_device(nm, Md.p, ev.data(), Vd.p, s);
            vec = download(Vd.p, size_t(nm) * nm, s);
        } else {
            DBuf<double>& th = tmp(15, size_t(nm));
            DBuf<double>& Vd = tmp(16, size_t(nm) * nm);
            sym_eig_device(nm, Md.p, nm, th.p, Vd.p, s);
            ev = download(th.p, size_t(nm), s);
            vec = download(Vd.p, size_t(nm) * nm, s);
        }
        ck.lap("alr: core eig");
        double max_abs = 0.0;
        for (double e : ev) max_abs = std::max(max_abs, std::fabs(e));
        std::vector<int> order;
        for (int i = 0; i < nm; ++i)
            if (std::fabs(ev[size_t(i)]) >= tol * max_abs && ev[size_t(i)] != 0.0) order.push_back(i);
        std::stable_sort(order.begin(), order.end(),
                         [&](int x, int y) { return std::fabs(ev[size_t(x)]) > std::fabs(ev[size_t(y)]); });
        for (int i : order) dsum.push_back(ev[size_t(i)]);
        for (int i = 0; i < int(dsum.size()); ++i)
            if (dsum[size_t(i)] > 1e-14) keep.push_back(i);
        const int rk = int(keep.size());
        Ek.assign(size_t(nm) * std::max(rk, 1), 0.0);
        for (int c = 0; c < rk; ++c) {
            const int src = order[size_t(keep[size_t(c)])];
            std::copy(vec.begin() + size_t(src) * nm, vec.begin() + size_t(src + 1) * nm, Ek.begin() + size_t(c) * nm);
        }
        Wn.ensure(size_t(n) * std::max(rk, 1));
        Wbn.ensure(size_t(n) * std::max(rk, 1));
        if (rk > 0) {
            DBuf<double>& Ed = tmp(17, Ek.size());
            upload(Ed.p, Ek, s);
            gemm_nn(n, rk, r, 1.0, W.p, Ed.p, nm, 0.0, nullptr, Wn.p, s);      // W' = [W, V̂]·E (:272-277)
            gemm_nn(n, rk, r, 1.0, Wbar.p, Ed.p, nm, 0.0, nullptr, Wbn.p, s);
            if (kh > 0) {
                gemm_nn(n, rk, kh, 1.0, Vh.p, Ed.p + r, nm, 1.0, Wn.p, Wn.p, s);
                gemm_nn(n, rk, kh, 1.0, Vhb.p, Ed.p + r, nm, 1.0, Wbn.p, Wbn.p, s);
            }
        }
    }
    // D = α²D̂(I + αD̂)⁻¹ on the kept modes (fast_filter.hpp:214-221)
    const int rk = int(keep.size());
    std::vector<double> dn(static_cast<size_t>(rk));
    for (int i = 0; i < rk; ++i) {
        const double dh = dsum[size_t(keep[size_t(i)])];
        dn[size_t(i)] = a * a * dh / (1.0 + a * dh);
    }
    FKB_CUDA(cudaStreamSynchronize(s));
    std::swap(W, Wn);  // the previous W/W̄ buffers become the next step's output buffers
    std::swap(Wbar, Wbn);
    d.ensure(size_t(std::max(rk, 1)));
    upload(d.p, dn, s);
    d_h = std::move(dn);
    r = rk;
    FKB_CUDA(cudaStreamSynchronize(s));
}

// diag Σ and realizations of the extended state (uq.hpp:16-23, :86-112 in FFT mode, SURVEY
// App. A.4): the carried W̄ = Γ⁻¹W plays Γ^{−1/2}-projected draws, no solve is needed
void Ekf::uq(uint64_t seed, uint64_t first, int count, double* X, double* var) {
    DBuf<double>& ad = tmp(19, 1);
    upload(ad.p, std::vector<double>{alpha}, s);
    lowrank_uq(cov, n, r, ad.p, d.p, W.p, Wbar.p, mean.p, seed, first, count, X, var, nullptr, tmp(20, 1));
}

// trace_criterion (uq.hpp:25-34) and relative_entropy (uq.hpp:36-53) of the extended state:
// φ = αNθ − Σ_j d_j‖W_j‖² (column norms on the device), ½[(N − r)ln α + Σ ln(α − d_j)]
void Ekf::uq_scalars(double& trace, double& entropy) {
    trace = alpha * double(n) * cov->spec.theta;
    if (r > 0) {
        DBuf<double>& cs = tmp(18, size_t(r));
        column_sumsq(n, r, W.p, cs.p, s);
        const std::vector<double> c = download(cs.p, size_t(r), s);
        for (int j = 0; j < r; ++j) trace -= d_h[size_t(j)] * c[size_t(j)];
    }
    if (!(alpha > 0.0)) throw std::invalid_argument("relative_entropy: requires alpha > 0");
    double sum = (double(n) - double(r)) * std::log(alpha);
    for (int i = 0; i < r; ++i) {
        const double gap = alpha - d_h[size_t(i)];
        if (!(gap > 0.0))
            throw std::runtime_error("relative_entropy: D_" + std::to_string(i) + " = " + std::to_string(d_h[size_t(i)]) +
                                     " is not below alpha = " + std::to_string(alpha));
        sum += std::log(gap);
    }
    entropy = 0.5 * sum;
}

}  // namespace fkb
