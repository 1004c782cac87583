// cappcg.cu — per-step capacitance solve K x = u by Jacobi-preconditioned conjugate
// gradients inside ONE thread-block cluster (16 CTAs, distributed-shared-memory reductions).
//
// K = I − D^½EᵀΛ_M⁻¹ED^½ is the Woodbury capacitance matrix of the innovation system
// S(α,d) = αG + σ²I − B·diag(d)·Bᵀ (fast_filter.hpp:100-108) in G's eigenbasis.  Because
// the GHEP modes nearly diagonalize G, K is close to diagonal: after Jacobi scaling its
// condition number is 1.008 at c2 (≈1.7 at c1), so PCG reaches ‖r‖ ≤ 1e-14‖u‖ in a few
// iterations — far less latency than any dense factorization of a 300–500 row matrix.
// Convergence is tested on the device; if the iteration cap is hit the kernel leaves u in
// place and raises *fallback so the cluster Cholesky (smallchol.cu) solves exactly.
//
// Layout: CTA c of the cluster owns rows [c·rb, (c+1)·rb); K (full, column-major, L2
// resident) is read row-block-wise each iteration; p is exchanged through DSMEM; scalar
// reductions are done with per-CTA partials read back through DSMEM in a fixed order
// (deterministic).

#include <cooperative_groups.h>

#include <algorithm>

#include "cappcg.cuh"
#include "common.cuh"

namespace cg = cooperative_groups;

namespace fkb {

constexpr int PC_CL = 16;   // CTAs per cluster (non-portable size, opt-in attribute)
constexpr int PC_T = 256;   // threads per CTA
constexpr int PC_MAXN = 1024;

struct PcgShared {
    double p[PC_MAXN];      // full search direction (gathered)
    double q[PC_MAXN / PC_CL];
    double part[4];         // this CTA's partial sums
    double red[PC_T / 32][4];
};

__device__ __forceinline__ double cluster_sum(cg::cluster_group& cl, PcgShared& sh, int slot) {
    // every CTA has written sh.part[slot]; sum them in rank order (deterministic)
    double v[PC_CL];
#pragma unroll
    for (int c = 0; c < PC_CL; ++c) v[c] = cl.map_shared_rank(&sh, c)->part[slot];  // all loads in flight
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < PC_CL; ++c) s += v[c];
    return s;
}

// three block partials with one __syncthreads → sh.part[0..2]
__device__ __forceinline__ void block_partial3(PcgShared& sh, double a, double b, double c) {
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, o);
        b += __shfl_down_sync(0xffffffffu, b, o);
        c += __shfl_down_sync(0xffffffffu, c, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sh.red[threadIdx.x >> 5][0] = a;
        sh.red[threadIdx.x >> 5][1] = b;
        sh.red[threadIdx.x >> 5][2] = c;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double s = 0.0;
        for (int w = 0; w < PC_T / 32; ++w) s += sh.red[w][threadIdx.x];
        sh.part[threadIdx.x] = s;
    }
}

__device__ __forceinline__ void cluster_sum3(cg::cluster_group& cl, PcgShared& sh, double* out) {
    double v[PC_CL][3];
#pragma unroll
    for (int c = 0; c < PC_CL; ++c) {
        PcgShared* rs = cl.map_shared_rank(&sh, c);
#pragma unroll
        for (int q = 0; q < 3; ++q) v[c][q] = rs->part[q];
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < PC_CL; ++c) s += v[c][q];
        out[q] = s;
    }
}

__device__ __forceinline__ void block_partial(PcgShared& sh, double v, int slot) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh.red[threadIdx.x >> 5][slot] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < PC_T / 32; ++w) s += sh.red[w][slot];
        sh.part[slot] = s;
    }
}

__global__ void __launch_bounds__(PC_T) k_cap_pcg(const double* __restrict__ K, long long ld, int n,
                                                 double* __restrict__ u, double* __restrict__ work,
                                                 int* __restrict__ fallback, int maxit, double tol, int kstage) {
    __shared__ PcgShared sh;
    extern __shared__ double Ks[];  // this CTA's columns of K (rb × n) when kstage
    cg::cluster_group cl = cg::this_cluster();
    const int crank = int(cl.block_rank());
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rb = (n + PC_CL - 1) / PC_CL;
    const int r0 = crank * rb, r1 = min(n, r0 + rb);
    if (kstage) {
        const int cnt = (r1 - r0) * n;
        for (int e0 = 0; e0 < cnt; e0 += 4 * PC_T) {
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = e0 + tid + q * PC_T;
                v[q] = e < cnt ? K[(long long)(r0 + e / n) * ld + e % n] : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = e0 + tid + q * PC_T;
                if (e < cnt) Ks[e] = v[q];
            }
        }
        __syncthreads();
    }
    // per-row state lives in registers of the owning thread (rows r0 + tid, r0 + tid + 256, …)
    // rb ≤ 64 for n ≤ 1024 → one row per thread among the first rb threads
    const int row = r0 + tid;
    const bool own = tid < rb && row < r1;
    double dinv = 0.0, b = 0.0, x = 0.0, r = 0.0;
    if (own) {
        dinv = 1.0 / K[row + (long long)row * ld];
        b = u[row];
        r = b;
    }
    // w = K·z for the owned rows: gather the full z through DSMEM (every remote load in
    // flight at once), then one warp per row over this CTA's staged columns of K.
    // Chronopoulos–Gear PCG (one fused reduction per iteration): with z = M⁻¹r, w = Kz,
    // γ = rᵀz, δ = zᵀw: β = γ/γ_prev, α = γ/(δ − βγ/α_prev), p = z + βp, s = w + βs,
    // x += αp, r −= αs.  Two cluster barriers per iteration: z published (inside matvec) and
    // the partials of (γ, δ, rᵀr) published.  Every CTA sees identical sums (rank-ordered),
    // so all leave the loop together.
    double p = 0.0, sv = 0.0, gamma_prev = 1.0, alpha_prev = 1.0;
    int it = 0;
    bool done = false;
    double stop = 0.0;
    while (true) {
        const double z = dinv * r;
        double w = 0.0;
        {  // w = K·z for the owned rows (z gathered through DSMEM)
            if (own) sh.p[row] = z;
            cl.sync();  // all z blocks published
            {
                double v[PC_MAXN / PC_T];
#pragma unroll
                for (int q = 0; q < PC_MAXN / PC_T; ++q) {
                    const int i = tid + q * PC_T;
                    const int owner = min(i / rb, PC_CL - 1);  // never form an out-of-cluster address
                    v[q] = 0.0;
                    if (i < n && owner != crank) v[q] = cl.map_shared_rank(&sh, owner)->p[i];
                }
#pragma unroll
                for (int q = 0; q < PC_MAXN / PC_T; ++q) {
                    const int i = tid + q * PC_T;
                    if (i < n && i / rb != crank) sh.p[i] = v[q];
                }
            }
            __syncthreads();
            for (int i = r0 + warp; i < r1; i += PC_T / 32) {
                const double* Kc = kstage ? Ks + (long long)(i - r0) * n : K + (long long)i * ld;
                double s0 = 0.0, s1 = 0.0;
                int j = lane;
                for (; j + 32 < n; j += 64) {
                    s0 = fma(Kc[j], sh.p[j], s0);
                    s1 = fma(Kc[j + 32], sh.p[j + 32], s1);
                }
                if (j < n) s0 = fma(Kc[j], sh.p[j], s0);
                double s = s0 + s1;
                for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
                if (lane == 0) sh.q[i - r0] = s;
            }
            __syncthreads();
            w = own ? sh.q[tid] : 0.0;
        }
        block_partial3(sh, own ? r * z : 0.0, own ? z * w : 0.0, own ? r * r : 0.0);
        cl.sync();
        double g3[3];
        cluster_sum3(cl, sh, g3);
        const double gamma = g3[0], delta = g3[1], rr = g3[2];
        if (it == 0) stop = tol * tol * rr;  // r₀ = b
        if (rr <= stop || rr == 0.0) {
            done = true;
            break;
        }
        if (it >= maxit) break;
        const double beta = it == 0 ? 0.0 : gamma / gamma_prev;
        const double alpha = it == 0 ? gamma / delta : gamma / (delta - beta * gamma / alpha_prev);
        if (own) {
            p = fma(beta, p, z);
            sv = fma(beta, sv, w);
            x = fma(alpha, p, x);
            r = fma(-alpha, sv, r);
        }
        gamma_prev = gamma;
        alpha_prev = alpha;
        ++it;
    }
    cl.sync();  // no CTA may exit while a peer still reads its partials through DSMEM
    if (done) {
        if (own) u[row] = x;
    } else if (crank == 0 && tid == 0) {
        *fallback = 1;
    }
    if (crank == 0 && tid == 0) work[n] = double(it);  // iteration count (diagnostics)
}

static bool g_pcg_attr = false;

void cap_pcg(int n, const double* K, long long ld, double* u, double* work, int* fallback, cudaStream_t s, int maxit,
             double tol) {
    if (n <= 0) return;
    if (n > PC_MAXN) throw std::invalid_argument("cap_pcg: n exceeds 1024");
    const int rb = (n + PC_CL - 1) / PC_CL;
    const size_t stage = sizeof(double) * size_t(rb) * n;
    const int kstage = stage <= 190 * 1024 ? 1 : 0;  // K columns resident in shared memory
    if (!g_pcg_attr) {
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_cap_pcg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_cap_pcg, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      190 * 1024));
        g_pcg_attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(PC_CL, 1, 1);
    cfg.blockDim = dim3(PC_T, 1, 1);
    cfg.dynamicSmemBytes = kstage ? stage : 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = PC_CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FKB_CUDA(cudaLaunchKernelEx(&cfg, k_cap_pcg, K, ld, n, u, work, fallback, maxit, tol, kstage));
    count_launch();
}

}  // namespace fkb
