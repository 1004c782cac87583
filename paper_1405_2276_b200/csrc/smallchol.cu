// smallchol.cu — SPD factor-and-solve K x = b for the k×k capacitance matrix of the
// per-step Woodbury solve (k ≤ 640), in ONE thread-block cluster.
//
// The reference factors the m×m innovation system every step (Eigen LLT,
// fast_filter.hpp:104).  With G = PΘPᵀ precomputed (eig.cu), S(α,d) = P(Λ_M − E D Eᵀ)Pᵀ
// and only K = I − D^½EᵀΛ_M⁻¹ED^½ (k×k, κ(K) = O(α)) must be factored per step.  The
// factorization is right-looking over 32×32 tiles; the cluster's CTAs share work through
// L2-resident global memory and synchronize with hardware cluster barriers.  Per panel j:
//   A  (CTA 0, 256 threads)  unscaled LDLᵀ elimination of the diagonal tile in shared memory
//                            (one __syncthreads per column, element-parallel updates), the
//                            same eliminations applied to I (L̃⁻¹) and to the RHS block; then
//                            L_jj = L̃·D^½, Linv_jj = D^-½·L̃⁻¹, y_j = D^-½·w_j
//   B  (all warps)           L_ij = K_ij·Linv_jjᵀ on DMMA (no substitution chains) and the
//                            RHS update b_i −= L_ij·y_j
//   C  (all warps)           trailing update K_il −= L_ij·L_ljᵀ on DMMA (i ≥ l > j)
// Backward substitution (CTA 0): x_j = Linv_jjᵀ·(y_j − Σ_{l>j} L_ljᵀ x_l), right-looking,
// with every L load issued before the wait on x_j.

#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "smallchol.cuh"

namespace cg = cooperative_groups;

namespace fkb {

constexpr int SC_CL = 8;      // CTAs per cluster
constexpr int SC_T = 256;     // threads per CTA
constexpr int SC_WARPS = SC_T / 32;
constexpr int SC_MAXT = 20;   // max tiles per dimension (k ≤ 640)
constexpr int TLD = 33;       // padded tile leading dimension in shared memory

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// K: n×n (lower used; overwritten by L).  b: RHS → solution.  LinvG: T·1024 doubles scratch
// (diagonal-tile inverses, row-major 32×32 each).  rdg unused scratch kept for ABI stability.
__global__ void __cluster_dims__(SC_CL, 1, 1) __launch_bounds__(SC_T)
    k_chol_solve(double* __restrict__ K, long long ld, int n, double* __restrict__ b, double* __restrict__ LinvG,
                 int* __restrict__ info, unsigned long long* __restrict__ tdbg) {
#define SC_STAMP(slot)                                                          \
    do {                                                                        \
        if (tdbg && blockIdx.x == 0 && threadIdx.x == 0) tdbg[slot] = gtimer(); \
    } while (0)
    extern __shared__ double sc_sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int crank = int(cl.block_rank());
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gwarp = crank * SC_WARPS + warp, nwarps = SC_CL * SC_WARPS;
    const int g = lane >> 2, t4 = lane & 3;
    const int T = (n + 31) / 32;
    double* At = sc_sm;                // 32×33  working tile (phase A) / Linv stage (phase B)
    double* Iv = sc_sm + 32 * TLD;     // 32×33  L̃⁻¹ accumulation (phase A)
    double* bb = Iv + 32 * TLD;        // 32     RHS block / y_j
    double* dd = bb + 32;              // 32     pivots
    __shared__ int failed;
    if (tdbg && blockIdx.x == 0 && threadIdx.x == 0) tdbg[158] = clock64();

    for (int j = 0; j < T; ++j) {
        const int j0 = j * 32, nj = min(32, n - j0);
        SC_STAMP(6 * j);
        // ---- A: diagonal tile
        if (crank == 0) {
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = tid + q * SC_T, r = e & 31, c = e >> 5;
                v[q] = (r < nj && c < nj) ? K[(j0 + r) + (long long)(j0 + c) * ld] : (r == c ? 1.0 : 0.0);
            }
            const double bv = tid < 32 ? (tid < nj ? b[j0 + tid] : 0.0) : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = tid + q * SC_T, r = e & 31, c = e >> 5;
                At[r * TLD + c] = v[q];
                Iv[r * TLD + c] = (r == c) ? 1.0 : 0.0;
            }
            if (tid < 32) bb[tid] = bv;
            const int er = tid & 31, ec0 = tid >> 5;  // this thread's elements: (er, ec0 + 8q)
            for (int c = 0; c < 32; ++c) {
                __syncthreads();
                // all shared-memory reads of the column step first (no store→load chains)
                const double d = At[c * TLD + c];
                const double arc = At[er * TLD + c];
                double ac2c[4], arc2[4], ivc[4], ivr[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int c2 = ec0 + 8 * q;
                    ac2c[q] = At[c2 * TLD + c];
                    arc2[q] = At[er * TLD + c2];
                    ivc[q] = Iv[c * TLD + c2];
                    ivr[q] = Iv[er * TLD + c2];
                }
                const double bc = bb[c], bt = tid < 32 ? bb[tid] : 0.0;
                const double invd = 1.0 / d;
                const double lrc = arc * invd;  // L̃_{er,c}
                if (er > c) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int c2 = ec0 + 8 * q;
                        if (c2 > c && c2 <= er) At[er * TLD + c2] = fma(-lrc, ac2c[q], arc2[q]);
                        if (c2 <= c) Iv[er * TLD + c2] = fma(-lrc, ivc[q], ivr[q]);
                    }
                }
                if (tid > c && tid < 32) bb[tid] = fma(-lrc, bc, bt);
                if (tid == c) {
                    dd[c] = d;
                    if (!(d > 0.0) && c < nj) atomicCAS(info, 0, j0 + c + 1);
                }
            }
            __syncthreads();
            // scale: L = L̃·D^½ (column scale), Linv = D^-½·L̃⁻¹ (row scale), y = D^-½ w
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = tid + q * SC_T, r = e & 31, c = e >> 5;
                if (r < nj && c < nj) {
                    const double rc = rsqrt(dd[c]);
                    if (r > c) K[(j0 + r) + (long long)(j0 + c) * ld] = At[r * TLD + c] * rc;
                    else if (r == c) K[(j0 + r) + (long long)(j0 + c) * ld] = dd[c] * rc;
                }
                LinvG[(long long)j * 1024 + r * 32 + c] = (c <= r) ? Iv[r * TLD + c] * rsqrt(dd[r]) : 0.0;
            }
            if (tid < nj) b[j0 + tid] = bb[tid] * rsqrt(dd[tid]);
        }
        SC_STAMP(6 * j + 1);
        cl.sync();
        SC_STAMP(6 * j + 2);
        if (tid == 0) failed = *((volatile int*)info);
        // stage Linv_jj (row-major) and y_j
        {
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = LinvG[(long long)j * 1024 + tid + q * SC_T];
            const double yv = tid < 32 ? (tid < nj ? b[j0 + tid] : 0.0) : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = tid + q * SC_T;
                At[(e >> 5) * TLD + (e & 31)] = v[q];
            }
            if (tid < 32) bb[tid] = yv;
        }
        __syncthreads();
        if (failed) return;
        // ---- B: L_ij = K_ij · Linvᵀ (DMMA), b_i −= L_ij·y_j; one warp per row tile
        for (int i = j + 1 + gwarp; i < T; i += nwarps) {
            const int i0 = i * 32;
            double af[8][4];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) {
                    const int r = i0 + mi * 8 + g, c = kk * 4 + t4;
                    af[kk][mi] = (r < n && c < nj) ? K[r + (long long)(j0 + c) * ld] : 0.0;
                }
            double acc[4][4][2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                double bf[4];
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) bf[ni] = At[(ni * 8 + g) * TLD + kk * 4 + t4];  // Linv(n, k)
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[kk][mi], bf[ni]);
            }
            // store L_ij and fold the RHS update (row = mi*8+g, cols = ni*8+2t4+q)
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                const int r = i0 + mi * 8 + g;
                double part = 0.0;
#pragma unroll
                for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int c = ni * 8 + t4 * 2 + q;
                        if (r < n && c < nj) K[r + (long long)(j0 + c) * ld] = acc[mi][ni][q];
                        part = fma(acc[mi][ni][q], bb[c], part);
                    }
                part += __shfl_xor_sync(0xffffffffu, part, 1);
                part += __shfl_xor_sync(0xffffffffu, part, 2);
                if (t4 == 0 && r < n) b[r] -= part;
            }
        }
        SC_STAMP(6 * j + 3);
        cl.sync();
        SC_STAMP(6 * j + 4);
        // ---- C: trailing update of lower tiles (i ≥ l > j) on DMMA, one warp per tile
        const int rem = T - j - 1;
        const int ntiles = rem * (rem + 1) / 2;
        for (int tt = gwarp; tt < ntiles; tt += nwarps) {
            int ii = int((sqrt(8.0 * tt + 1.0) - 1.0) * 0.5);
            while ((ii + 1) * (ii + 2) / 2 <= tt) ++ii;
            while (ii * (ii + 1) / 2 > tt) --ii;
            const int ll = tt - ii * (ii + 1) / 2;
            const int i0 = (j + 1 + ii) * 32, l0 = (j + 1 + ll) * 32;
            double af[8][4], bfr[8][4], cv[4][4][2];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int kc = j0 + kk * 4 + t4;
                const bool kv = kk * 4 + t4 < nj;
#pragma unroll
                for (int mi = 0; mi < 4; ++mi) {
                    const int r = i0 + mi * 8 + g;
                    af[kk][mi] = (kv && r < n) ? K[r + (long long)kc * ld] : 0.0;
                    const int rl = l0 + mi * 8 + g;
                    bfr[kk][mi] = (kv && rl < n) ? K[rl + (long long)kc * ld] : 0.0;
                }
            }
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int r = i0 + mi * 8 + g, c = l0 + ni * 8 + t4 * 2 + q;
                        cv[mi][ni][q] = (r < n && c < n) ? K[r + (long long)c * ld] : 0.0;
                    }
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni) dmma(cv[mi][ni][0], cv[mi][ni][1], -af[kk][mi], bfr[kk][ni]);
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const int r = i0 + mi * 8 + g, c = l0 + ni * 8 + t4 * 2 + q;
                        if (r < n && c < n && c <= r) K[r + (long long)c * ld] = cv[mi][ni][q];
                    }
        }
        cl.sync();
        SC_STAMP(6 * j + 5);
    }
    // ---- backward substitution Lᵀ x = y in CTA 0
    if (crank != 0) return;
    SC_STAMP(6 * SC_MAXT);
    double* D = sc_sm;           // T Linv tiles, row-major 32×33
    double* xs = D + T * 32 * TLD;
    for (int e0 = 0; e0 < T * 1024; e0 += 4 * SC_T) {
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = e0 + tid + q * SC_T;
            v[q] = e < T * 1024 ? LinvG[e] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = e0 + tid + q * SC_T;
            if (e < T * 1024) D[(e >> 10) * 32 * TLD + ((e >> 5) & 31) * TLD + (e & 31)] = v[q];
        }
    }
    __syncthreads();
    constexpr int RPT = 3;  // rows per thread in the update (T·32 ≤ 640 ≤ 3·256)
    for (int j = T - 1; j >= 0; --j) {
        const int j0 = j * 32, nj = min(32, n - j0);
        // prefetch L_jl entries for the rows this thread updates (rows < j0), independent of x_j
        double pv[RPT][32];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int r = tid + q * SC_T;
#pragma unroll
            for (int c = 0; c < 32; ++c) pv[q][c] = (r < j0 && c < nj) ? K[(j0 + c) + (long long)r * ld] : 0.0;
        }
        if (warp == 0) {  // x_j = Linv_jjᵀ·y_j : lane c → Σ_i Linv(i, c)·y_i
            const double y = lane < nj ? b[j0 + lane] : 0.0;
            const double* Dj = D + j * 32 * TLD;
            double x = 0.0;
#pragma unroll
            for (int i = 0; i < 32; ++i) x = fma(Dj[i * TLD + lane], __shfl_sync(0xffffffffu, y, i), x);
            xs[lane] = lane < nj ? x : 0.0;
            if (lane < nj) b[j0 + lane] = x;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int r = tid + q * SC_T;
            if (r < j0) {
                double a0 = 0.0, a1 = 0.0;
#pragma unroll
                for (int c = 0; c < 32; c += 2) {
                    a0 = fma(pv[q][c], xs[c], a0);
                    a1 = fma(pv[q][c + 1], xs[c + 1], a1);
                }
                b[r] -= a0 + a1;
            }
        }
        __syncthreads();
        SC_STAMP(6 * SC_MAXT + 1 + (T - 1 - j));
    }
    if (tdbg && blockIdx.x == 0 && threadIdx.x == 0) tdbg[159] = clock64();
#undef SC_STAMP
}

size_t chol_solve_smem(int n) {
    const int T = (n + 31) / 32;
    const size_t loop = 2 * 32 * TLD + 64;
    const size_t back = size_t(T) * 32 * TLD + 32;
    return sizeof(double) * std::max(loop, back);
}

void chol_solve_small(int n, double* K, long long ld, double* b, double* LinvG, int* info, cudaStream_t s,
                      unsigned long long* tdbg) {
    if (n <= 0) return;
    if (n > SC_MAXT * 32) throw std::invalid_argument("chol_solve_small: n exceeds 640 (shared-memory staging limit)");
    const size_t sm = chol_solve_smem(n);
    static size_t attr = 0;
    if (sm > attr) {
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_chol_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        attr = sm;
    }
    k_chol_solve<<<SC_CL, SC_T, sm, s>>>(K, ld, n, b, LinvG, info, tdbg);
    FKB_LAUNCH_CHECK();
    count_launch();
}

size_t chol_solve_scratch(int n) { return size_t((n + 31) / 32) * 1024; }

}  // namespace fkb

// test hook: factor+solve a host SPD matrix; L (lower) and x returned, per-phase
// %globaltimer stamps (ns) in stamps[0 .. 160) when non-null.
extern "C" int fkb_chol_solve_small(int n, const double* K, const double* b, double* L, double* x,
                                    unsigned long long* stamps) {
    try {
        fkb::DBuf<double> dK(static_cast<size_t>(n) * n), db(static_cast<size_t>(n)),
            sc(fkb::chol_solve_scratch(n));
        fkb::DBuf<int> info(1);
        fkb::DBuf<unsigned long long> ts(160);
        FKB_CUDA(cudaMemcpy(dK.p, K, sizeof(double) * size_t(n) * n, cudaMemcpyHostToDevice));
        FKB_CUDA(cudaMemcpy(db.p, b, sizeof(double) * size_t(n), cudaMemcpyHostToDevice));
        FKB_CUDA(cudaMemset(info.p, 0, sizeof(int)));
        FKB_CUDA(cudaMemset(ts.p, 0, ts.bytes()));
        fkb::chol_solve_small(n, dK.p, n, db.p, sc.p, info.p, nullptr, stamps ? ts.p : nullptr);
        FKB_CUDA(cudaDeviceSynchronize());
        int h = 0;
        FKB_CUDA(cudaMemcpy(&h, info.p, sizeof(int), cudaMemcpyDeviceToHost));
        if (L) FKB_CUDA(cudaMemcpy(L, dK.p, sizeof(double) * size_t(n) * n, cudaMemcpyDeviceToHost));
        if (x) FKB_CUDA(cudaMemcpy(x, db.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost));
        if (stamps) FKB_CUDA(cudaMemcpy(stamps, ts.p, ts.bytes(), cudaMemcpyDeviceToHost));
        return h ? 2 : 0;
    } catch (const std::exception&) {
        return 3;
    }
}
