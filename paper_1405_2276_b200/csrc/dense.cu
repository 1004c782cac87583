// dense.cu — FP64 dense kernels for sm_100a: DMMA GEMM (K4/K5/K6), blocked Cholesky (K6),
// flag-chained triangular solves, tall-skinny GEMV (K7/K8).
//
// FP64 has no tcgen05 kind; the FP64 tensor path on B200 is mma.sync .f64 (SASS DMMA).
// Replaces the reference's Eigen products and LLT (fast_filter.hpp:100-108,
// lowrank.hpp:186-205).

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "dense.cuh"

namespace fkb {

// --------------------------------------------------------------------------- DMMA GEMM
constexpr int GBM = 64, GBN = 64, GBK = 16, GLD = GBM + 4, GTHREADS = 128;

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, const double* safe, bool valid) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int sz = valid ? 8 : 0;  // src-size 0 → zero fill, nothing read
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(valid ? src : safe), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__global__ void __launch_bounds__(GTHREADS) k_gemm(GemmArgs g, int kchunk, double* __restrict__ partial) {
    __shared__ __align__(16) double As[2][GBK][GLD];
    __shared__ __align__(16) double Bs[2][GBK][GLD];
    const int i0 = blockIdx.x * GBM, j0 = blockIdx.y * GBN;
    if (g.lower_only && j0 > i0 + GBM - 1) return;
    const int kbeg = blockIdx.z * kchunk;
    const int kend = min(g.K, kbeg + kchunk);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;

    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    auto load = [&](int st, int k0) {
#pragma unroll
        for (int r = 0; r < (GBK * GBM) / GTHREADS; ++r) {
            const int e = tid + r * GTHREADS;
            int ii, kk;
            if (g.transA == 0) { kk = e / GBM; ii = e - kk * GBM; }
            else { ii = e / GBK; kk = e - ii * GBK; }
            const int gi = i0 + ii, gk = k0 + kk;
            const bool v = gi < g.M && gk < kend;
            const double* src = g.transA == 0 ? g.A + gi + (long long)gk * g.lda : g.A + gk + (long long)gi * g.lda;
            cp_async8(&As[st][kk][ii], src, g.A, v);
        }
#pragma unroll
        for (int r = 0; r < (GBK * GBN) / GTHREADS; ++r) {
            const int e = tid + r * GTHREADS;
            int jj, kk;
            if (g.transB == 0) { jj = e / GBK; kk = e - jj * GBK; }
            else { kk = e / GBN; jj = e - kk * GBN; }
            const int gj = j0 + jj, gk = k0 + kk;
            const bool v = gj < g.N && gk < kend;
            const double* src = g.transB == 0 ? g.B + gk + (long long)gj * g.ldb : g.B + gj + (long long)gk * g.ldb;
            cp_async8(&Bs[st][kk][jj], src, g.B, v);
        }
        cp_async_commit();
    };

    const int nk = (kend - kbeg + GBK - 1) / GBK;
    if (nk > 0) load(0, kbeg);
    for (int it = 0; it < nk; ++it) {
        const int st = it & 1;
        if (it + 1 < nk) {
            load(st ^ 1, kbeg + (it + 1) * GBK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GBK; kk += 4) {
            double a[4], b[4];
            double sc = 1.0;
            if (g.dA) {
                const int gk = kbeg + it * GBK + kk + tq;
                sc = gk < kend ? __ldg(g.dA + gk) : 0.0;
            }
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = As[st][kk + tq][wm + mi * 8 + gq] * sc;
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) b[ni] = Bs[st][kk + tq][wn + ni * 8 + gq];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
        __syncthreads();
    }

    const double beta = g.beta_ptr ? *g.beta_ptr : g.beta;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int i = i0 + wm + mi * 8 + gq;
                const int j = j0 + wn + ni * 8 + tq * 2 + q;
                if (i >= g.M || j >= g.N) continue;
                if (partial) {
                    partial[(long long)blockIdx.z * g.M * g.N + i + (long long)j * g.M] = acc[mi][ni][q];
                } else {
                    double a = acc[mi][ni][q];
                    if (g.rs) a *= g.rs[i];
                    if (g.cs) a *= g.cs[j];
                    double out = g.alpha * a;
                    if (beta != 0.0) out += beta * g.Cin[i + (long long)j * g.ldcin];
                    if (i == j) out += g.diag_add;
                    g.C[i + (long long)j * g.ldc] = out;
                }
            }
}

__global__ void k_splitk_reduce(GemmArgs g, const double* __restrict__ partial) {
    const long long total = (long long)g.M * g.N;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int i = int(e % g.M), j = int(e / g.M);
        if (g.lower_only && (j / GBN) * GBN > (i / GBM) * GBM + GBM - 1) continue;
        double s = 0.0;
        for (int z = 0; z < g.splitk; ++z) s += partial[(long long)z * total + e];
        if (g.rs) s *= g.rs[i];
        if (g.cs) s *= g.cs[j];
        double out = g.alpha * s;
        const double beta = g.beta_ptr ? *g.beta_ptr : g.beta;
        if (beta != 0.0) out += beta * g.Cin[i + (long long)j * g.ldcin];
        if (i == j) out += g.diag_add;
        g.C[i + (long long)j * g.ldc] = out;
    }
}

int gemm_pick_splitk(int M, int N, int K) {
    const long long tiles = (long long)ceil_div(M, GBM) * ceil_div(N, GBN);
    if (tiles <= 0 || tiles >= 296 || K < 256) return 1;
    const long long want = (296 + tiles - 1) / tiles;
    return int(std::max<long long>(1, std::min<long long>(want, K / 128)));
}

size_t gemm_ws_elems(const GemmArgs& g) { return g.splitk > 1 ? size_t(g.splitk) * g.M * g.N : 0; }

void gemm(const GemmArgs& g_in, double* ws, cudaStream_t s) {
    GemmArgs g = g_in;
    if (g.M <= 0 || g.N <= 0) return;
    if (!g.Cin) { g.Cin = g.C; g.ldcin = g.ldc; }
    if (g.splitk < 1) g.splitk = 1;
    int kchunk = g.K;
    if (g.splitk > 1) {
        kchunk = ((ceil_div(g.K, g.splitk) + GBK - 1) / GBK) * GBK;
        g.splitk = ceil_div(g.K, kchunk);
    }
    dim3 grid(ceil_div(g.M, GBM), ceil_div(g.N, GBN), g.splitk);
    if (g.K <= 0) {  // pure epilogue
        g.splitk = 1;
        grid.z = 1;
    }
    k_gemm<<<grid, GTHREADS, 0, s>>>(g, std::max(kchunk, 1), g.splitk > 1 ? ws : nullptr);
    FKB_LAUNCH_CHECK();
    count_launch();
    if (g.splitk > 1) {
        const long long total = (long long)g.M * g.N;
        k_splitk_reduce<<<std::min<long long>(4096, (total + 255) / 256), 256, 0, s>>>(g, ws);
        FKB_LAUNCH_CHECK();
        count_launch();
    }
}

// --------------------------------------------------------------------------- Gram C = Aᵀ·diag(w)·B
// A (K×M) and B (K×N) column-major with k contiguous (Gram/capacitance shapes).  64×64 tiles,
// BK = 32, 256 threads (2×4 warps, warp tile 32×16 = 4×2 DMMA 8×8), 16-byte cp.async into
// k-contiguous shared rows (ld 36 doubles: conflict-free fragment loads), double buffered.
// Split-K partials go to `partial` (reduced by k_splitk_reduce with the same epilogue).
constexpr int QB = 64, QK = 32, QLD = 36, QT = 256;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid, const void* safe) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(valid ? src : safe), "r"(sz));
}

__global__ void __launch_bounds__(QT) k_gram(GemmArgs g, int kchunk, double* __restrict__ partial) {
    extern __shared__ __align__(16) double qsm[];
    double* As = qsm;                       // [2][QB][QLD]
    double* Bs = qsm + 2 * QB * QLD;        // [2][QB][QLD]
    double* Ws = qsm + 4 * QB * QLD;        // [2][QK] diagonal weights dA
    const int i0 = blockIdx.x * QB, j0 = blockIdx.y * QB;
    if (g.lower_only && j0 > i0 + QB - 1) return;
    const int kbeg = blockIdx.z * kchunk, kend = min(g.K, kbeg + kchunk);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    auto load = [&](int st, int k0) {
#pragma unroll
        for (int q = 0; q < (QB * QK / 2) / QT; ++q) {  // 4 chunks of 2 doubles per operand
            const int e = tid + q * QT;
            const int row = e / (QK / 2), kc = (e % (QK / 2)) * 2;
            const int gk = k0 + kc;
            const int ga = i0 + row, gb = j0 + row;
            const bool kv = gk + 1 < kend;  // K chunk edges are even (kchunk % QK == 0, K even checked)
            cp_async16(As + (st * QB + row) * QLD + kc, g.A + gk + (long long)ga * g.lda, kv && ga < g.M, g.A);
            cp_async16(Bs + (st * QB + row) * QLD + kc, g.B + gk + (long long)gb * g.ldb, kv && gb < g.N, g.B);
        }
        if (g.dA && tid < QK / 2) {  // the chunk's diagonal weights ride along with the tiles
            const int gk = k0 + 2 * tid;
            cp_async16(Ws + st * QK + 2 * tid, g.dA + gk, gk + 1 < kend, g.dA);
        }
        cp_async_commit();
    };
    const int nk = (kend - kbeg + QK - 1) / QK;
    if (nk > 0) load(0, kbeg);
    for (int it = 0; it < nk; ++it) {
        const int st = it & 1;
        if (it + 1 < nk) {
            load(st ^ 1, kbeg + (it + 1) * QK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* Ab = As + st * QB * QLD;
        const double* Bb = Bs + st * QB * QLD;
#pragma unroll
        for (int kk = 0; kk < QK; kk += 4) {
            const int gk = kbeg + it * QK + kk + tq;
            const double wk = g.dA ? (gk < kend ? Ws[st * QK + kk + tq] : 0.0) : 1.0;
            double a[4], b[2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = Ab[(wm + mi * 8 + gq) * QLD + kk + tq];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) b[ni] = Bb[(wn + ni * 8 + gq) * QLD + kk + tq] * wk;
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
        __syncthreads();
    }
    const double beta = g.beta_ptr ? *g.beta_ptr : g.beta;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int i = i0 + wm + mi * 8 + gq;
                const int j = j0 + wn + ni * 8 + tq * 2 + q;
                if (i >= g.M || j >= g.N) continue;
                if (partial) {
                    partial[(long long)blockIdx.z * g.M * g.N + i + (long long)j * g.M] = acc[mi][ni][q];
                } else {
                    double v = acc[mi][ni][q];
                    if (g.rs) v *= g.rs[i];
                    if (g.cs) v *= g.cs[j];
                    double out = g.alpha * v;
                    if (beta != 0.0) out += beta * g.Cin[i + (long long)j * g.ldcin];
                    if (i == j) out += g.diag_add;
                    g.C[i + (long long)j * g.ldc] = out;
                }
            }
}

// C = epilogue(Aᵀ·diag(dA)·B) for k-contiguous A (K×M) and B (K×N); same GemmArgs semantics
// as gemm() with transA = 1, transB = 0.  Requires K, lda, ldb even (16-byte chunks).
// Split-K factor of the Gram: all tiles·s CTAs are resident at once (3 per SM: 74 KB of shared
// memory each), so the launch takes as long as the busiest SM — ceil(tiles·s / SMs) CTAs of
// K/s each.  Pick the s that minimizes that (ties: the larger s — l = 420 ties at 1, 2 and 3
// CTAs per SM, and one CTA per SM leaves the DMMA pipe waiting on shared-memory loads):
// l = 320 gives 25 tiles, where ceil(296/25) = 12 put three CTAs on four SMs and two on the
// rest (SMs busy 66 % of the launch, profiles/round2_ncu_wprod_c2_v3.txt); s = 17 keeps every
// SM within 4 % of the even split.
static int gram_pick_splitk(long long tiles, int K) {
    static const int sms = [] {
        int dev = 0, n = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return std::max(n, 1);
    }();
    const long long smax = std::min<long long>(3LL * sms / std::max<long long>(tiles, 1), K / 128);
    int best = 1;
    double best_cost = 1e300;
    for (long long sk = 1; sk <= std::max<long long>(smax, 1); ++sk) {
        const double cost = double((tiles * sk + sms - 1) / sms) / double(sk);
        if (cost <= best_cost * (1.0 + 1e-9)) {  // ties: more CTAs per SM hide the DMMA latency better
            best_cost = cost;
            best = int(sk);
        }
    }
    return best;
}

void gram(const GemmArgs& g_in, double* ws, cudaStream_t s) {
    GemmArgs g = g_in;
    if (g.M <= 0 || g.N <= 0) return;
    if (g.K <= 0 || (g.K & 1) || (g.lda & 1) || (g.ldb & 1) || g.transA != 1 || g.transB != 0) {
        gemm(g, ws, s);  // shapes the 16-byte path cannot take: the general DMMA kernel
        return;
    }
    if (!g.Cin) { g.Cin = g.C; g.ldcin = g.ldc; }
    const long long tiles = (long long)ceil_div(g.M, QB) * ceil_div(g.N, QB);
    int splitk = 1;
    if (ws && tiles < 296) splitk = gram_pick_splitk(tiles, g.K);
    int kchunk = ((ceil_div(g.K, splitk) + QK - 1) / QK) * QK;
    splitk = ceil_div(g.K, kchunk);
    g.splitk = splitk;
    const size_t smem = sizeof(double) * (4 * QB * QLD + 2 * QK);
    static bool attr = false;
    if (!attr) {
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        attr = true;
    }
    k_gram<<<dim3(ceil_div(g.M, QB), ceil_div(g.N, QB), splitk), QT, smem, s>>>(g, kchunk, splitk > 1 ? ws : nullptr);
    FKB_LAUNCH_CHECK();
    count_launch();
    if (splitk > 1) {
        const long long total = (long long)g.M * g.N;
        k_splitk_reduce<<<std::min<long long>(4096, (total + 255) / 256), 256, 0, s>>>(g, ws);
        FKB_LAUNCH_CHECK();
        count_launch();
    }
}

// ---- symmetric Gram with cluster split-K: C = epi(Aᵀ·diag(dA)·A) for the per-step
// capacitance K = I − D^½EᵀΛ_M⁻¹ED^½.  Only lower 64×64 tiles are computed (half the
// DMMA work of the full product); the S CTAs of a cluster split K, park their partial tile
// in shared memory and reduce it through DSMEM in rank order (deterministic, no workspace,
// no second kernel); each CTA finalizes 64/S rows of the tile and writes them and their
// mirror, so K is exactly symmetric.
__global__ void __launch_bounds__(QT) k_gram_sym(GemmArgs g, int kchunk) {
    namespace cg = cooperative_groups;
    extern __shared__ __align__(16) double qsm[];
    double* As = qsm;
    double* Bs = qsm + 2 * QB * QLD;
    double* Ws = qsm + 4 * QB * QLD;
    cg::cluster_group cl = cg::this_cluster();
    const int S = int(cl.num_blocks()), z = int(cl.block_rank());
    int ti = int((std::sqrt(8.0 * blockIdx.x + 1.0) - 1.0) * 0.5);
    while ((ti + 1) * (ti + 2) / 2 <= int(blockIdx.x)) ++ti;
    while (ti * (ti + 1) / 2 > int(blockIdx.x)) --ti;
    const int tj = int(blockIdx.x) - ti * (ti + 1) / 2;
    const int i0 = ti * QB, j0 = tj * QB;
    const int kbeg = z * kchunk, kend = min(g.K, kbeg + kchunk);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gq = lane >> 2, tq = lane & 3;
    const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    auto load = [&](int st, int k0) {
#pragma unroll
        for (int q = 0; q < (QB * QK / 2) / QT; ++q) {
            const int e = tid + q * QT;
            const int row = e / (QK / 2), kc = (e % (QK / 2)) * 2;
            const int gk = k0 + kc;
            const int ga = i0 + row, gb = j0 + row;
            const bool kv = gk + 1 < kend;
            cp_async16(As + (st * QB + row) * QLD + kc, g.A + gk + (long long)ga * g.lda, kv && ga < g.M, g.A);
            cp_async16(Bs + (st * QB + row) * QLD + kc, g.B + gk + (long long)gb * g.ldb, kv && gb < g.N, g.B);
        }
        if (g.dA && tid < QK / 2) {  // the chunk's diagonal weights ride along with the tiles
            const int gk = k0 + 2 * tid;
            cp_async16(Ws + st * QK + 2 * tid, g.dA + gk, gk + 1 < kend, g.dA);
        }
        cp_async_commit();
    };
    const int nk = kend > kbeg ? (kend - kbeg + QK - 1) / QK : 0;
    if (nk > 0) load(0, kbeg);
    for (int it = 0; it < nk; ++it) {
        const int st = it & 1;
        if (it + 1 < nk) {
            load(st ^ 1, kbeg + (it + 1) * QK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* Ab = As + st * QB * QLD;
        const double* Bb = Bs + st * QB * QLD;
#pragma unroll
        for (int kk = 0; kk < QK; kk += 4) {
            const int gk = kbeg + it * QK + kk + tq;
            const double wk = g.dA ? (gk < kend ? Ws[st * QK + kk + tq] : 0.0) : 1.0;
            double a[4], b[2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) a[mi] = Ab[(wm + mi * 8 + gq) * QLD + kk + tq];
#pragma unroll
            for (int ni = 0; ni < 2; ++ni) b[ni] = Bb[(wn + ni * 8 + gq) * QLD + kk + tq] * wk;
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 2; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
        __syncthreads();
    }
    // partial tile → this CTA's shared memory (row-major, ld 65), then cluster-wide reduction
    constexpr int PLD = QB + 1;
    double* part = qsm;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni)
#pragma unroll
            for (int q = 0; q < 2; ++q)
                part[(wm + mi * 8 + gq) * PLD + wn + ni * 8 + tq * 2 + q] = acc[mi][ni][q];
    cl.sync();
    const int rows_per = QB / S;
    for (int e = tid; e < rows_per * QB; e += QT) {
        const int il = z * rows_per + e / QB, jl = e % QB;
        double v = 0.0;
        for (int c = 0; c < S; ++c) v += cl.map_shared_rank(part, c)[il * PLD + jl];
        const int i = i0 + il, j = j0 + jl;
        if (i >= g.M || j >= g.N || (ti == tj && i < j)) continue;
        if (g.rs) v *= g.rs[i];
        if (g.cs) v *= g.cs[j];
        double out = g.alpha * v;
        if (i == j) out += g.diag_add;
        g.C[i + (long long)j * g.ldc] = out;
        if (i != j) g.C[j + (long long)i * g.ldc] = out;
    }
    cl.sync();  // peers may still be reading this CTA's partial tile
}

void gram_sym(const GemmArgs& g_in, cudaStream_t s) {
    GemmArgs g = g_in;
    if (g.M <= 0) return;
    if (g.M != g.N || g.A != g.B || g.lda != g.ldb || g.K <= 0 || (g.K & 1) || (g.lda & 1) || g.transA != 1 ||
        g.transB != 0 || g.rs != g.cs || g.beta != 0.0 || g.beta_ptr) {
        g.lower_only = 0;
        gram(g, nullptr, s);  // general path (not expected on the step)
        return;
    }
    const int nt = ceil_div(g.M, QB), tiles = nt * (nt + 1) / 2;
    int S = 8;  // portable cluster; measured faster than 16 (a 16-CTA cluster needs a whole GPC)
    while (S > 1 && (tiles * S > 2 * 148 || g.K / S < 2 * QK)) S >>= 1;
    const int kchunk = ((ceil_div(g.K, S) + QK - 1) / QK) * QK;
    const size_t smem = sizeof(double) * (4 * QB * QLD + 2 * QK);
    static bool attr = false;
    if (!attr) {
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_gram_sym, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_gram_sym, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tiles, 1, S);
    cfg.blockDim = dim3(QT, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr_[1];
    attr_[0].id = cudaLaunchAttributeClusterDimension;
    attr_[0].val.clusterDim.x = 1;
    attr_[0].val.clusterDim.y = 1;
    attr_[0].val.clusterDim.z = S;
    cfg.attrs = attr_;
    cfg.numAttrs = 1;
    FKB_CUDA(cudaLaunchKernelEx(&cfg, k_gram_sym, g, kchunk));
    count_launch();
}

size_t gram_ws_elems(int M, int N, int K) {
    const long long tiles = (long long)ceil_div(M, QB) * ceil_div(N, QB);
    if (tiles <= 0 || tiles >= 296) return 0;
    const long long s = gram_pick_splitk(tiles, K);
    return size_t(s + 1) * M * N;
}

// --------------------------------------------------------------------------- GEMV

// --------------------------------------------------------------------------- Cholesky
constexpr int CNB = 64;

// Factor the kb×kb diagonal block at (k0, k0) in shared memory (right-looking, 256 threads as a
// 16×16 grid that sweeps only the shrinking trailing triangle; every thread derives the pivot
// itself, so a step costs two barriers); write L11 back, and when dinv ≠ null also L11⁻¹ (kb×kb,
// ld CNB) to dinv + k0·CNB by the same row-operation sweep on the identity.
__global__ void __launch_bounds__(256) k_potrf_diag(double* A, long long lda, int kb, int k0, int* info,
                                                   double* __restrict__ dinv) {
    extern __shared__ double potrf_sm[];
    double (*s)[CNB + 1] = reinterpret_cast<double (*)[CNB + 1]>(potrf_sm);
    double (*x)[CNB + 1] = reinterpret_cast<double (*)[CNB + 1]>(potrf_sm + CNB * (CNB + 1));
    __shared__ double ld[CNB];
    if (*info) return;
    double* a = A + k0 + (long long)k0 * lda;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    for (int e = tid; e < CNB * CNB; e += 256) {
        const int i = e & (CNB - 1), j = e >> 6;
        s[i][j] = (i < kb && j < kb && i >= j) ? a[i + (long long)j * lda] : 0.0;
        x[i][j] = i == j ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int j = 0; j < kb; ++j) {
        const double djj = s[j][j];  // final: updated by step j−1 before the last barrier
        if (!(djj > 0.0)) {
            if (tid == 0) atomicCAS(info, 0, k0 + j + 1);
            return;  // uniform: every thread read the same pivot
        }
        const double ljj = sqrt(djj), rinv = 1.0 / ljj;
        if (tid == 0) ld[j] = ljj;
        if (tid > j && tid < kb) s[tid][j] *= rinv;
        __syncthreads();
        // trailing triangle rows/cols j+1..kb−1: s[i][c] −= L_ij·L_cj (i ≥ c)
        for (int c = j + 1 + tx; c < kb; c += 16) {
            const double lc = s[c][j];
            for (int i = c + ty; i < kb; i += 16) s[i][c] = fma(-s[i][j], lc, s[i][c]);
        }
        __syncthreads();
    }
    for (int e = tid; e < kb * kb; e += 256) {
        const int i = e % kb, j = e / kb;
        if (i > j) a[i + (long long)j * lda] = s[i][j];
        else if (i == j) a[i + (long long)j * lda] = ld[j];
    }
    if (!dinv) return;
    if (tid < kb) s[tid][tid] = ld[tid];
    __syncthreads();
    // L X = I by row sweeps: row j ← row j / L_jj, then rows i > j −= L_ij · row j (cols ≤ j)
    for (int j = 0; j < kb; ++j) {
        const double rinv = 1.0 / s[j][j];
        if (tid <= j) x[j][tid] *= rinv;
        __syncthreads();
        for (int c = tx; c <= j; c += 16) {
            const double xj = x[j][c];
            for (int i = j + 1 + ty; i < kb; i += 16) x[i][c] = fma(-s[i][j], xj, x[i][c]);
        }
        __syncthreads();
    }
    double* di = dinv + (long long)k0 * CNB;  // block b at dinv + b·CNB·CNB (k0 = b·CNB)
    for (int e = tid; e < CNB * CNB; e += 256) {
        const int i = e & (CNB - 1), j = e >> 6;
        di[i + j * CNB] = (i < kb && j < kb) ? x[i][j] : 0.0;
    }
}

// L21 = A21 · L11⁻ᵀ for a 64-row block below the diagonal block at k0.
__global__ void __launch_bounds__(CNB) k_trsm_panel(double* A, long long lda, int n, int k0, int kb, const int* info) {
    extern __shared__ double trsm_sm[];
    double (*L)[CNB + 1] = reinterpret_cast<double (*)[CNB + 1]>(trsm_sm);
    double (*X)[CNB + 1] = reinterpret_cast<double (*)[CNB + 1]>(trsm_sm + CNB * (CNB + 1));
    if (*info) return;
    const int r0 = k0 + kb + blockIdx.x * CNB;
    const int rb = min(CNB, n - r0);
    for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
        const int i = e % kb, j = e / kb;
        L[i][j] = i >= j ? A[(k0 + i) + (long long)(k0 + j) * lda] : 0.0;
    }
    for (int e = threadIdx.x; e < rb * kb; e += blockDim.x) {
        const int i = e % rb, j = e / rb;
        X[i][j] = A[(r0 + i) + (long long)(k0 + j) * lda];
    }
    __syncthreads();
    const int r = threadIdx.x;
    if (r < rb) {
        for (int j = 0; j < kb; ++j) {
            double v = X[r][j];
            for (int p = 0; p < j; ++p) v -= X[r][p] * L[j][p];
            X[r][j] = v / L[j][j];
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rb * kb; e += blockDim.x) {
        const int i = e % rb, j = e / rb;
        A[(r0 + i) + (long long)(k0 + j) * lda] = X[i][j];
    }
}

static size_t potrf_inv_elems(int n) { return size_t(std::max(ceil_div(n, CNB), 1)) * CNB * CNB; }
size_t potrf_ws_elems(int n) {
    // full 64×64 diagonal-block inverses (ceil(n/64)·64·64) + the panel product L21 (n·64)
    return potrf_inv_elems(n) + size_t(std::max(n, 1)) * CNB;
}

// With a workspace (ws_elems ≥ potrf_ws_elems(n)) every panel is one DMMA product
// L21 = A21·L11⁻ᵀ with the diagonal inverse formed beside L11, and the inverses stay in ws
// for potrs_lower_multi; without one (graph-captured solver 0) the substitution panel kernel.
void potrf_lower(int n, double* A, long long lda, int* info, double* ws, size_t ws_elems, cudaStream_t s) {
    const size_t trsm_smem = 2 * sizeof(double) * CNB * (CNB + 1);
    static bool attr = false;
    if (!attr) {
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_trsm_panel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(trsm_smem)));
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_potrf_diag, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(trsm_smem)));
        attr = true;
    }
    const bool inv = ws && ws_elems >= potrf_ws_elems(n);
    double* dinv = inv ? ws : nullptr;
    double* pan = inv ? ws + potrf_inv_elems(n) : nullptr;
    for (int k0 = 0; k0 < n; k0 += CNB) {
        const int kb = std::min(CNB, n - k0);
        k_potrf_diag<<<1, 256, trsm_smem, s>>>(A, lda, kb, k0, info, dinv);
        FKB_LAUNCH_CHECK();
        count_launch();
        const int rest = n - k0 - kb;
        if (rest <= 0) break;
        double* a21 = A + (k0 + kb) + (long long)k0 * lda;
        if (inv) {
            GemmArgs p;  // L21 = A21 · L11⁻ᵀ into the panel scratch (ld rest)
            p.M = rest; p.N = kb; p.K = kb;
            p.A = a21; p.lda = lda;
            p.B = dinv + (long long)k0 * CNB; p.ldb = CNB; p.transB = 1;
            p.C = pan; p.ldc = rest;
            gemm(p, nullptr, s);
            FKB_CUDA(cudaMemcpy2DAsync(a21, sizeof(double) * size_t(lda), pan, sizeof(double) * size_t(rest),
                                       sizeof(double) * size_t(rest), size_t(kb), cudaMemcpyDeviceToDevice, s));
        } else {
            k_trsm_panel<<<ceil_div(rest, CNB), CNB, trsm_smem, s>>>(A, lda, n, k0, kb, info);
            FKB_LAUNCH_CHECK();
            count_launch();
        }
        GemmArgs g;  // A22 −= L21 L21ᵀ (lower tiles)
        g.M = rest; g.N = rest; g.K = kb;
        g.A = inv ? pan : a21; g.lda = inv ? rest : lda; g.transA = 0;
        g.B = g.A; g.ldb = g.lda; g.transB = 1;
        g.alpha = -1.0; g.beta = 1.0;
        g.C = A + (k0 + kb) + (long long)(k0 + kb) * lda; g.ldc = lda;
        g.lower_only = 1;
        gemm(g, nullptr, s);
    }
}

// --------------------------------------------------------------------------- triangular solves
// Flag-chained block substitution: CTA b owns rows [64b, 64b+64); it folds in finished
// blocks as their flags appear, then solves its diagonal block and publishes.  All CTAs
// are co-resident (≤ 64 CTAs of 256 threads), and CTAs only wait on lower blockIdx.
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

template <bool TRANS>
__global__ void __launch_bounds__(256) k_trsv(const double* __restrict__ L, long long lda, int n,
                                             double* x, int* flags) {
    const int nblk = (n + CNB - 1) / CNB;
    const int b = TRANS ? nblk - 1 - blockIdx.x : blockIdx.x;
    const int r0 = b * CNB, rb = min(CNB, n - r0);
    __shared__ double part[4][CNB];
    __shared__ double ysh[CNB];
    __shared__ double D[CNB][CNB + 1];
    const int tid = threadIdx.x;
    // diagonal block
    for (int e = tid; e < rb * rb; e += blockDim.x) {
        const int i = e % rb, j = e / rb;
        D[i][j] = L[(r0 + i) + (long long)(r0 + j) * lda];
    }
    double acc = 0.0;
    const int r = TRANS ? (tid >> 2) : (tid & 63);
    const int q = TRANS ? (tid & 3) : (tid >> 6);
    const int jlo = TRANS ? b + 1 : 0, jhi = TRANS ? nblk : b;
    for (int jj = jlo; jj < jhi; ++jj) {
        const int j = TRANS ? (nblk - 1 - (jj - jlo)) : jj;  // consume in publication order
        if (tid == 0)
            while (ld_acquire(flags + j) == 0) {
            }
        __syncthreads();
        const int c0 = j * CNB, cb = min(CNB, n - c0);
        if (tid < cb) ysh[tid] = __ldcg(x + c0 + tid);
        __syncthreads();
        if (r < rb) {
            for (int cc = 0; cc < 16; ++cc) {
                const int c = q * 16 + cc;
                if (c < cb) {
                    const double l = TRANS ? L[(c0 + c) + (long long)(r0 + r) * lda] : L[(r0 + r) + (long long)(c0 + c) * lda];
                    acc = fma(l, ysh[c], acc);
                }
            }
        }
        __syncthreads();
    }
    if (r < CNB) part[q][r] = acc;
    __syncthreads();
    if (tid < 32) {
        // rhs for the two rows this lane owns
        double v0 = 0.0, v1 = 0.0;
        const int i0 = tid, i1 = tid + 32;
        if (i0 < rb) v0 = x[r0 + i0] - (part[0][i0] + part[1][i0] + part[2][i0] + part[3][i0]);
        if (i1 < rb) v1 = x[r0 + i1] - (part[0][i1] + part[1][i1] + part[2][i1] + part[3][i1]);
        if (!TRANS) {
            for (int k = 0; k < rb; ++k) {
                const double vk = __shfl_sync(0xffffffffu, k < 32 ? v0 : v1, k & 31);
                const double yk = vk / D[k][k];
                if (i0 == k) v0 = yk;
                if (i1 == k) v1 = yk;
                if (i0 > k && i0 < rb) v0 -= D[i0][k] * yk;
                if (i1 > k && i1 < rb) v1 -= D[i1][k] * yk;
            }
        } else {
            for (int k = rb - 1; k >= 0; --k) {
                const double vk = __shfl_sync(0xffffffffu, k < 32 ? v0 : v1, k & 31);
                const double yk = vk / D[k][k];
                if (i0 == k) v0 = yk;
                if (i1 == k) v1 = yk;
                if (i0 < k) v0 -= D[k][i0] * yk;
                if (i1 < k) v1 -= D[k][i1] * yk;
            }
        }
        if (i0 < rb) x[r0 + i0] = v0;
        if (i1 < rb) x[r0 + i1] = v1;
        __threadfence();
        __syncwarp();
        if (tid == 0) st_release(flags + b, 1);
    }
}

void potrs_lower(int n, const double* L, long long lda, double* x, int* flags, cudaStream_t s) {
    const int nblk = ceil_div(n, CNB);
    FKB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * 2 * size_t(nblk), s));
    k_trsv<false><<<nblk, 256, 0, s>>>(L, lda, n, x, flags);
    FKB_LAUNCH_CHECK();
    k_trsv<true><<<nblk, 256, 0, s>>>(L, lda, n, x, flags + nblk);
    FKB_LAUNCH_CHECK();
    count_launch(2);
}

// --------------------------------------------------------------------------- multi-RHS potrs
// Diagonal-block solve for nrhs right-hand sides: the kb×kb block of L at (k0, k0) in shared
// memory, 32 RHS columns per CTA staged transposed; one thread per column substitutes
// sequentially (forward L·y = b, or backward Lᵀ·x = y when TRANS).
constexpr int TRC = 16;  // right-hand sides per CTA of the multi-RHS diagonal solve
template <bool TRANS>
__global__ void __launch_bounds__(256) k_trsm_diag(const double* __restrict__ L, long long lda, int k0, int kb,
                                                  double* __restrict__ B, long long ldb, int nrhs) {
    __shared__ double D[CNB][CNB + 1];
    __shared__ double Y[TRC][CNB + 1];
    const int c0 = blockIdx.x * TRC;
    for (int e = threadIdx.x; e < kb * kb; e += blockDim.x) {
        const int i = e % kb, j = e / kb;
        D[i][j] = L[(k0 + i) + (long long)(k0 + j) * lda];
    }
    for (int e = threadIdx.x; e < TRC * kb; e += blockDim.x) {
        const int i = e % kb, c = e / kb;
        Y[c][i] = c0 + c < nrhs ? B[(k0 + i) + (long long)(c0 + c) * ldb] : 0.0;
    }
    __syncthreads();
    if (threadIdx.x < TRC) {
        double* y = Y[threadIdx.x];
        if (!TRANS) {
            for (int i = 0; i < kb; ++i) {
                double v = y[i];
                for (int k = 0; k < i; ++k) v = fma(-D[i][k], y[k], v);
                y[i] = v / D[i][i];
            }
        } else {
            for (int i = kb - 1; i >= 0; --i) {
                double v = y[i];
                for (int k = i + 1; k < kb; ++k) v = fma(-D[k][i], y[k], v);
                y[i] = v / D[i][i];
            }
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < TRC * kb; e += blockDim.x) {
        const int i = e % kb, c = e / kb;
        if (c0 + c < nrhs) B[(k0 + i) + (long long)(c0 + c) * ldb] = Y[c][i];
    }
}

void potrs_lower_multi(int n, const double* L, long long lda, double* B, long long ldb, int nrhs, cudaStream_t s,
                       const double* dinv, double* tmp) {
    if (n <= 0 || nrhs <= 0) return;
    const int nblk = ceil_div(n, CNB);
    const bool inv = dinv && tmp;
    for (int b = 0; b < nblk; ++b) {  // L·Y = B, trailing updates on DMMA
        const int k0 = b * CNB, kb = std::min(CNB, n - k0), k1 = k0 + kb;
        if (inv) {
            GemmArgs d;  // Y_b = L_bb⁻¹ · B_b
            d.M = kb; d.N = nrhs; d.K = kb;
            d.A = dinv + (long long)k0 * CNB; d.lda = CNB;
            d.B = B + k0; d.ldb = ldb;
            d.C = tmp; d.ldc = CNB;
            gemm(d, nullptr, s);
            FKB_CUDA(cudaMemcpy2DAsync(B + k0, sizeof(double) * size_t(ldb), tmp, sizeof(double) * CNB,
                                       sizeof(double) * size_t(kb), size_t(nrhs), cudaMemcpyDeviceToDevice, s));
        } else {
            k_trsm_diag<false><<<ceil_div(nrhs, TRC), 256, 0, s>>>(L, lda, k0, kb, B, ldb, nrhs);
            FKB_LAUNCH_CHECK();
            count_launch();
        }
        if (k1 < n) {
            GemmArgs g;
            g.M = n - k1; g.N = nrhs; g.K = kb;
            g.A = L + k1 + (long long)k0 * lda; g.lda = lda;
            g.B = B + k0; g.ldb = ldb;
            g.alpha = -1.0; g.beta = 1.0;
            g.C = B + k1; g.ldc = ldb;
            gemm(g, nullptr, s);
        }
    }
    for (int b = nblk - 1; b >= 0; --b) {  // Lᵀ·X = Y
        const int k0 = b * CNB, kb = std::min(CNB, n - k0);
        if (inv) {
            GemmArgs d;  // X_b = L_bb⁻ᵀ · Y_b
            d.M = kb; d.N = nrhs; d.K = kb;
            d.A = dinv + (long long)k0 * CNB; d.lda = CNB; d.transA = 1;
            d.B = B + k0; d.ldb = ldb;
            d.C = tmp; d.ldc = CNB;
            gemm(d, nullptr, s);
            FKB_CUDA(cudaMemcpy2DAsync(B + k0, sizeof(double) * size_t(ldb), tmp, sizeof(double) * CNB,
                                       sizeof(double) * size_t(kb), size_t(nrhs), cudaMemcpyDeviceToDevice, s));
        } else {
            k_trsm_diag<true><<<ceil_div(nrhs, TRC), 256, 0, s>>>(L, lda, k0, kb, B, ldb, nrhs);
            FKB_LAUNCH_CHECK();
            count_launch();
        }
        if (k0 > 0) {
            GemmArgs g;  // X[0:k0] −= L[k0:k1, 0:k0]ᵀ · X[k0:k1]
            g.M = k0; g.N = nrhs; g.K = kb;
            g.A = L + k0; g.lda = lda; g.transA = 1;
            g.B = B + k0; g.ldb = ldb;
            g.alpha = -1.0; g.beta = 1.0;
            g.C = B; g.ldc = ldb;
            gemm(g, nullptr, s);
        }
    }
}

}  // namespace fkb
