// smallchol.cu — SPD factor-and-solve K x = b for the k×k capacitance matrix of the
// per-step Woodbury solve (k ≤ 640), in ONE thread-block cluster.
//
// The reference factors the m×m innovation system every step (Eigen LLT,
// fast_filter.hpp:104).  With G = PΘPᵀ precomputed (eig.cu), S(α,d) = P(Λ_M − E D Eᵀ)Pᵀ
// and only K = I − D^½EᵀΛ_M⁻¹ED^½ (k×k, κ(K) = O(α)) must be factored per step.
//
// Right-looking Cholesky over 32×32 tiles; the cluster's CTAs share the L2-resident matrix
// and synchronize with hardware cluster barriers.  Every triangular recurrence is written
// right-looking (after x_c is known, the remaining entries are updated by independent
// FMAs), so the serial dependency per column is one FMA + one multiply instead of a dot
// product.  Per panel j:
//   A (one warp, registers, lane = row)  factor tile (j,j): pivots, column scale, rank-1
//       updates broadcast by warp shuffles; forward-solve the RHS block y_j.
//       Look-ahead: the warp that updates tile (j+1, j+1) in phase C(j) factors it
//       immediately, overlapping A(j+1) with the rest of C(j).
//   B (all warps, lane = row)  L_ij = K_ij·L_jj⁻ᵀ right-looking with L_jj staged in
//       shared memory; RHS update b_i −= L_ij·y_j.
//   C (all warps)  trailing update K_il −= L_ij·L_ljᵀ on DMMA (i ≥ l > j).
// Backward substitution Lᵀx = y runs in CTA 0 (right-looking inside each diagonal tile,
// prefetched off-diagonal loads for the cross-tile updates).

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
constexpr int TLD = 33;

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

// Phase A: factor diagonal tile j in one warp.  Writes L_jj (lower) into K, 1/L_cc into
// rdg[j0+c], y_j into b.  Flags the first non-positive pivot in *info.
// Compact loops over a lane-private shared-memory row (T[lane·TLD + c]): a fully unrolled
// register version is ~25k straight-line instructions that one warp runs once, which is
// instruction-fetch bound; broadcasts go through shared memory (64-bit shuffles cost two
// SHFL issues each).
__device__ __noinline__ void diag_factor_warp(double* __restrict__ K, long long ld, int n, int j,
                                              double* __restrict__ b, double* __restrict__ rdg,
                                              int* __restrict__ info, double* T, volatile double* colbuf) {
    const int lane = threadIdx.x & 31;
    const int j0 = j * 32, nj = min(32, n - j0);
    const int row = j0 + lane;
    (void)T;
    double a[32];  // lane's row, compile-time indexed only
#pragma unroll
    for (int c = 0; c < 32; ++c)
        a[c] = (lane < nj && c < nj) ? K[row + (long long)(j0 + c) * ld] : (c == lane ? 1.0 : 0.0);
    double rhs = lane < nj ? b[row] : 0.0;
    double rmine = 1.0;
    int bad = 0;
#pragma unroll 1
    for (int c = 0; c < 32; ++c) {  // runtime loop: compact code
        double ac = 0.0;
#pragma unroll
        for (int q = 0; q < 32; ++q) ac = (q == c) ? a[q] : ac;  // a[c] without local memory
        if (lane == c) {
            colbuf[32] = ac;  // pivot (updated by all earlier columns)
            colbuf[33] = rhs;
        }
        __syncwarp();
        const double d = colbuf[32];
        const double rinv = rsqrt(d);
        const double yc = colbuf[33] * rinv;
        if (!(d > 0.0) && !bad) bad = c + 1;
        const double lc = lane > c ? ac * rinv : (lane == c ? d * rinv : 0.0);
        if (lane == c) {
            rmine = rinv;
            rhs = yc;
        } else if (lane > c) {
            rhs = fma(-lc, yc, rhs);
        }
        colbuf[lane] = lc;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 32; ++q) {
            const double l2 = colbuf[q];
            a[q] = (q == c && lane >= c) ? lc : ((q > c && q <= lane) ? fma(-lc, l2, a[q]) : a[q]);
        }
        __syncwarp();
    }
    if (bad && bad <= nj && lane == 0) atomicCAS(info, 0, j0 + bad);
    if (lane < nj) {
#pragma unroll
        for (int c = 0; c < 32; ++c)
            if (c <= lane) K[row + (long long)(j0 + c) * ld] = a[c];
        b[row] = rhs;
        rdg[row] = rmine;
    }
}

template <int RPT>  // rows per thread in the backward cross-tile update (T·32 ≤ RPT·256)
__global__ void __cluster_dims__(SC_CL, 1, 1) __launch_bounds__(SC_T)
    k_chol_solve(double* __restrict__ K, long long ld, int n, double* __restrict__ b, double* __restrict__ rdg,
                 int* __restrict__ info, unsigned long long* __restrict__ tdbg, const int* __restrict__ gate) {
    if (gate && *gate == 0) return;  // used as the exact fallback of the PCG solve (cappcg.cu)
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
    double* Lj = sc_sm;            // 32×33 L_jj (row-major)
    double* rj = Lj + 32 * TLD;    // 32 reciprocal pivots
    double* yj = rj + 32;          // 32 y_j
    double* colbuf = yj + 32;      // 34: phase-A column/pivot broadcast (warp 0 of CTA 0)
    double* Tw = colbuf + 34;      // SC_WARPS × 32×33 lane-private row tiles (phases A and B)
    __shared__ int failed;
    if (tdbg && blockIdx.x == 0 && threadIdx.x == 0) tdbg[158] = clock64();

    SC_STAMP(150);
    if (crank == 0 && warp == 0) diag_factor_warp(K, ld, n, 0, b, rdg, info, Tw, colbuf);
    SC_STAMP(151);
    for (int j = 0; j < T; ++j) {
        const int j0 = j * 32, nj = min(32, n - j0);
        SC_STAMP(6 * j);
        cl.sync();
        SC_STAMP(6 * j + 1);
        if (tid == 0) failed = *((volatile int*)info);
        {
            double v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = tid + q * SC_T, r = e & 31, c = e >> 5;
                v[q] = (r < nj && c < nj && c <= r) ? K[(j0 + r) + (long long)(j0 + c) * ld] : 0.0;
            }
            const double rv = tid < 32 ? (tid < nj ? rdg[j0 + tid] : 1.0) : 0.0;
            const double yv = tid < 32 ? (tid < nj ? b[j0 + tid] : 0.0) : 0.0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = tid + q * SC_T;
                Lj[(e & 31) * TLD + (e >> 5)] = v[q];
            }
            if (tid < 32) {
                rj[tid] = rv;
                yj[tid] = yv;
            }
        }
        __syncthreads();
        if (failed) return;
        SC_STAMP(6 * j + 2);
        // ---- B: L_ij = K_ij·L_jj⁻ᵀ (right-looking, lane = row), b_i −= L_ij·y_j
        for (int i = j + 1 + gwarp; i < T; i += nwarps) {
            const int row = i * 32 + lane;
            const bool live = row < n;
            double x[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) x[c] = (live && c < nj) ? K[row + (long long)(j0 + c) * ld] : 0.0;
            double acc = 0.0;
#pragma unroll 1
            for (int c = 0; c < 32; ++c) {  // runtime loop, register row: x_c then the right-looking update
                double xc = 0.0;
#pragma unroll
                for (int q = 0; q < 32; ++q) xc = (q == c) ? x[q] : xc;
                xc *= rj[c];
                acc = fma(xc, yj[c], acc);
                const double* Lc = Lj + c;  // column c of L_jj: Lj[q·TLD + c]
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const double l = Lc[q * TLD];
                    x[q] = (q == c) ? xc : ((q > c) ? fma(-xc, l, x[q]) : x[q]);
                }
            }
            if (live) {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                    if (c < nj) K[row + (long long)(j0 + c) * ld] = x[c];
                b[row] -= acc;
            }
        }
        SC_STAMP(6 * j + 3);
        cl.sync();
        SC_STAMP(6 * j + 4);
        // ---- C: trailing update (i ≥ l > j); tile 0 = (j+1, j+1) goes to warp 0 of CTA 0,
        // which then factors it right away (look-ahead A(j+1)).
        const int rem = T - j - 1;
        const int ntiles = rem * (rem + 1) / 2;
        const int stride = gwarp == 0 ? ntiles + 1 : nwarps - 1;
        for (int tt = (gwarp == 0 ? 0 : gwarp); tt < ntiles; tt += stride) {
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
            if (tt == 0) {
                __syncwarp();
                __threadfence_block();
                diag_factor_warp(K, ld, n, j + 1, b, rdg, info, Tw, colbuf);  // look-ahead A(j+1)
            }
        }
        SC_STAMP(6 * j + 5);
    }
    // ---- backward substitution Lᵀ x = y in CTA 0
    cl.sync();
    if (crank != 0) return;
    SC_STAMP(6 * SC_MAXT);
    double* D = sc_sm;                  // T diagonal tiles, row-major 32×33 (D[r][c] = L(r,c))
    double* ra = D + T * 32 * TLD;      // T·32 reciprocal pivots
    double* xs = ra + T * 32;           // 32
    for (int e0 = 0; e0 < T * 1024; e0 += 4 * SC_T) {
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = e0 + tid + q * SC_T;
            const int jt = e >> 10, r = e & 31, c = (e >> 5) & 31;
            const int jj0 = jt * 32, njt = min(32, n - jj0);
            v[q] = (e < T * 1024 && r < njt && c < njt && c <= r) ? K[(jj0 + r) + (long long)(jj0 + c) * ld] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = e0 + tid + q * SC_T;
            if (e < T * 1024) D[(e >> 10) * 32 * TLD + (e & 31) * TLD + ((e >> 5) & 31)] = v[q];
        }
    }
    for (int e = tid; e < T * 32; e += SC_T) ra[e] = e < n ? rdg[e] : 1.0;
    __syncthreads();
    for (int j = T - 1; j >= 0; --j) {
        const int j0 = j * 32, nj = min(32, n - j0);
        double pv[RPT][32];  // L_jl entries for this thread's rows (independent of x_j)
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int r = tid + q * SC_T;
#pragma unroll
            for (int c = 0; c < 32; ++c) pv[q][c] = (r < j0 && c < nj) ? K[(j0 + c) + (long long)r * ld] : 0.0;
        }
        if (warp == 0) {  // Lᵀ_jj x = y_j, right-looking from the last row: lane = row
            double y = lane < nj ? b[j0 + lane] : 0.0;
            const double* Dj = D + j * 32 * TLD;
            const double* rr = ra + j0;
#pragma unroll
            for (int c = 31; c >= 0; --c) {
                const double xc = __shfl_sync(0xffffffffu, y, c) * rr[c];
                if (lane == c) y = xc;
                else if (lane < c) y = fma(-Dj[c * TLD + lane], xc, y);
            }
            xs[lane] = lane < nj ? y : 0.0;
            if (lane < nj) b[j0 + lane] = y;
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
    const size_t loop = 32 * TLD + 64 + 34 + size_t(SC_WARPS) * 32 * TLD;
    const size_t back = size_t(T) * 32 * TLD + size_t(T) * 32 + 32;
    return sizeof(double) * std::max(loop, back);
}

void chol_solve_small(int n, double* K, long long ld, double* b, double* rdg, int* info, cudaStream_t s,
                      unsigned long long* tdbg, const int* gate) {
    if (n <= 0) return;
    if (n > SC_MAXT * 32) throw std::invalid_argument("chol_solve_small: n exceeds 640 (shared-memory staging limit)");
    const size_t sm = chol_solve_smem(n);
    static size_t attr = 0;
    if (sm > attr) {
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_chol_solve<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_chol_solve<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm)));
        attr = sm;
    }
    if (n <= 2 * SC_T) k_chol_solve<2><<<SC_CL, SC_T, sm, s>>>(K, ld, n, b, rdg, info, tdbg, gate);
    else k_chol_solve<3><<<SC_CL, SC_T, sm, s>>>(K, ld, n, b, rdg, info, tdbg, gate);
    FKB_LAUNCH_CHECK();
    count_launch();
}

size_t chol_solve_scratch(int n) { return size_t(std::max(n, 1)); }

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
