// enkf.cu — enkf_step (enkf.hpp:49-94), the perturbed-observation EnKF for the random-walk
// model, with the members resident in HBM (n×N_e column-major).
//
//   forecast   X[:, j] += circulant draw (seed_f, j/2) — Re for even j, Im for odd j
//              (covariance.hpp:332-353), all pairs batched through the two sampler passes;
//   HX         X transposed to row-major so the ray SpMM streams contiguous member rows
//              (k_spmm_rm), transposed back;
//   anomalies  D = X − x̄, HD = HX − Hx̄;
//   C_yy       HD·HDᵀ/(N_e − 1) + σ²I on DMMA, symmetrized, blocked LLT;
//   Z          C_yy⁻¹(y + σ·v_j − HX_j) with v_j = gaussian_vector(m, seed_p, j) (the K3
//              generator), all N_e right-hand sides by blocked TRSM on DMMA;
//   update     X += C_sy·Z with C_sy = D·HDᵀ/(N_e − 1): evaluated as D·(HDᵀZ)/(N_e − 1) when
//              N_e ≤ m (2nN_e² flops instead of 4nmN_e), else in the reference order.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "enkf.cuh"
#include "rng_device.cuh"

namespace fkb {

// out[i] = (1/ne)·Σ_j A[i + j·lda] (row means of a column-major block)
__global__ void k_row_mean(long long n, int ne, const double* __restrict__ A, long long lda, double* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < ne; ++j) acc += A[i + (long long)j * lda];
        out[i] = acc / double(ne);
    }
}
// out[:, j] = A[:, j] − mu (column-major n×ne)
__global__ void k_sub_rowvec(long long n, int ne, const double* __restrict__ A, const double* __restrict__ mu,
                             double* __restrict__ out) {
    const long long total = n * ne;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x)
        out[e] = A[e] - mu[e % n];
}
// Z[:, j] = y + σ·Z[:, j] − HX[:, j]   (Z holds the standard normals on entry; σ = 0: y − HX)
__global__ void k_perturbed_innov(int m, int ne, const double* __restrict__ y, double sigma, const double* __restrict__ HX,
                                  double* __restrict__ Z) {
    const long long total = (long long)m * ne;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int i = int(e % m);
        Z[e] = sigma > 0.0 ? y[i] + sigma * Z[e] - HX[e] : y[i] - HX[e];
    }
}

// FKB_ENKF_TRACE=1: per-phase wall times of each step on stderr (stream-synchronized)
struct EnkfClock {
    cudaStream_t s;
    bool on = std::getenv("FKB_ENKF_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void lap(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(s);
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[enkf] %-14s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    }
};

static int grid_of(long long n) { return int(std::max<long long>(1, std::min<long long>((n + 255) / 256, 4096))); }

Enkf::Enkf(Cov* c, int m_, int h_cols, const int* rowptr, const int* col, const double* val, int n_members)
    : cov(c), s(c->stream), n(c->size()), m(m_), ne(n_members) {
    if (ne < 2) throw std::invalid_argument("enkf_init: ensemble size must be at least 2");  // enkf.hpp:31-32
    if (m < 0) throw std::invalid_argument("enkf_step: dimension mismatch");
    if ((long long)h_cols != n) throw std::invalid_argument("enkf_step: dimension mismatch");
    for (int i = 0; i < m; ++i)
        for (int e = rowptr[i]; e < rowptr[i + 1]; ++e)
            if (col[e] < 0 || col[e] >= n) throw std::invalid_argument("enkf_step: H column index out of range");
    upload_csr_pair(m, int(n), rowptr, col, val, H, HT);
    X.alloc(size_t(n) * ne);
    FKB_CUDA(cudaMemsetAsync(X.p, 0, X.bytes(), s));  // enkf_init: Σ_{0|0} = 0 (:30-34)
    Xr.alloc(size_t(n) * ne);
    const size_t me = size_t(std::max(m, 1)) * ne;
    HXr.alloc(me);
    HX.alloc(me);
    Z.alloc(me);
    mean.alloc(size_t(n));
    hmean.alloc(size_t(std::max(m, 1)));
    Cyy.alloc(size_t(std::max(m, 1)) * std::max(m, 1));
    ybuf.alloc(size_t(std::max(m, 1)));
    info.alloc(1);
    FKB_CUDA(cudaStreamSynchronize(s));
}

void Enkf::member_mean(double* out) {
    k_row_mean<<<grid_of(n), 256, 0, s>>>(n, ne, X.p, n, out);
    FKB_LAUNCH_CHECK();
    count_launch();
}

void Enkf::step(const double* y_h, double sigma2, uint64_t seed) {
    if (sigma2 < 0.0) throw std::invalid_argument("enkf_step: sigma2 must be nonnegative");  // :55-56
    const uint64_t seed_f = derive_seed_host(seed, 1), seed_p = derive_seed_host(seed, 2);  // :58-59
    if (m > 0) FKB_CUDA(cudaMemcpyAsync(ybuf.p, y_h, sizeof(double) * size_t(m), cudaMemcpyHostToDevice, s));
    // the new members are formed in Xr (D, then X + update) so a singular C_yy leaves X untouched
    DBuf<double>& D = Xr;
    EnkfClock clk{s};
    Xf.ensure(size_t(n) * ne);  // forecast members
    FKB_CUDA(cudaMemcpyAsync(Xf.p, X.p, X.bytes(), cudaMemcpyDeviceToDevice, s));
    cov->sample_pairs_add(seed_f, 0, Xf.p, n, ne);  // (:61-67)
    clk.lap("forecast");
    if (m == 0) {
        FKB_CUDA(cudaMemcpyAsync(X.p, Xf.p, X.bytes(), cudaMemcpyDeviceToDevice, s));
        FKB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    // HX (:69): row-major members through the streaming ray SpMM
    transpose_cm(n, ne, Xf.p, D.p, s);
    spmm_rm(H, D.p, ne, ne, HXr.p, ne, 1.0, s);
    transpose_cm(ne, m, HXr.p, HX.p, s);
    clk.lap("HX");
    // anomalies (:70-73)
    k_row_mean<<<grid_of(n), 256, 0, s>>>(n, ne, Xf.p, n, mean.p);
    FKB_LAUNCH_CHECK();
    k_row_mean<<<grid_of(m), 256, 0, s>>>(m, ne, HX.p, m, hmean.p);
    FKB_LAUNCH_CHECK();
    k_sub_rowvec<<<grid_of((long long)n * ne), 256, 0, s>>>(n, ne, Xf.p, mean.p, D.p);
    FKB_LAUNCH_CHECK();
    k_sub_rowvec<<<grid_of((long long)m * ne), 256, 0, s>>>(m, ne, HX.p, hmean.p, HXr.p);  // HD into HXr
    FKB_LAUNCH_CHECK();
    count_launch(4);
    double* HD = HXr.p;
    clk.lap("anomalies");
    const double inv = 1.0 / double(ne - 1);
    {  // C_yy = HD·HDᵀ/(N_e − 1) + σ²I (:75-77)
        GemmArgs g;
        g.M = m; g.N = m; g.K = ne;
        g.A = HD; g.lda = m;
        g.B = HD; g.ldb = m; g.transB = 1;
        g.alpha = inv;
        g.diag_add = sigma2;
        g.C = Cyy.p; g.ldc = m;
        g.lower_only = 1;  // the LLT reads the lower triangle only; symmetric by construction
        g.splitk = gemm_pick_splitk(m, m, ne);
        ws.ensure(std::max<size_t>(gemm_ws_elems(g), 1));
        gemm(g, ws.p, s);
    }
    FKB_CUDA(cudaMemsetAsync(info.p, 0, sizeof(int), s));
    pws.ensure(potrf_ws_elems(m) + size_t(64) * ne);
    potrf_lower(m, Cyy.p, m, info.p, pws.p, potrf_ws_elems(m), s);  // (:78-82)
    int h = 0;
    FKB_CUDA(cudaMemcpyAsync(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    FKB_CUDA(cudaStreamSynchronize(s));
    if (h)
        throw std::runtime_error(
            "enkf_step: sample innovation covariance is singular even with observation noise added");
    clk.lap("Cyy + LLT");
    // perturbed innovations (:86-92) and Z = C_yy⁻¹·innovations
    if (sigma2 > 0.0) gaussian_matrix(m, ne, seed_p, 0, Z.p, m, s);
    k_perturbed_innov<<<grid_of((long long)m * ne), 256, 0, s>>>(m, ne, ybuf.p, std::sqrt(sigma2), HX.p, Z.p);
    FKB_LAUNCH_CHECK();
    count_launch();
    potrs_lower_multi(m, Cyy.p, m, Z.p, m, ne, s, pws.p, pws.p + potrf_ws_elems(m));
    clk.lap("innov + TRSM");
    // X = X_f + C_sy·Z (:93)
    if (ne <= m) {
        T.ensure(size_t(ne) * ne);
        GemmArgs g;  // T = HDᵀ·Z (N_e × N_e)
        g.M = ne; g.N = ne; g.K = m;
        g.A = HD; g.lda = m; g.transA = 1;
        g.B = Z.p; g.ldb = m;
        g.C = T.p; g.ldc = ne;
        g.splitk = gemm_pick_splitk(ne, ne, m);
        ws.ensure(std::max<size_t>(gemm_ws_elems(g), 1));
        gemm(g, ws.p, s);
        GemmArgs u;  // X = X_f + D·T/(N_e − 1)
        u.M = int(n); u.N = ne; u.K = ne;
        u.A = D.p; u.lda = n;
        u.B = T.p; u.ldb = ne;
        u.alpha = inv;
        u.beta = 1.0;
        u.Cin = Xf.p; u.ldcin = n;
        u.C = X.p; u.ldc = n;
        gemm(u, nullptr, s);
    } else {
        T.ensure(size_t(n) * m);
        GemmArgs g;  // C_sy = D·HDᵀ/(N_e − 1) (N × m)
        g.M = int(n); g.N = m; g.K = ne;
        g.A = D.p; g.lda = n;
        g.B = HD; g.ldb = m; g.transB = 1;
        g.alpha = inv;
        g.C = T.p; g.ldc = n;
        gemm(g, nullptr, s);
        GemmArgs u;  // X = X_f + C_sy·Z
        u.M = int(n); u.N = ne; u.K = m;
        u.A = T.p; u.lda = n;
        u.B = Z.p; u.ldb = m;
        u.beta = 1.0;
        u.Cin = Xf.p; u.ldcin = n;
        u.C = X.p; u.ldc = n;
        gemm(u, nullptr, s);
    }
    clk.lap("update");
    FKB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace fkb
