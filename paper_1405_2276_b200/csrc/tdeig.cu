// tdeig.cu — symmetric eigendecomposition A = Z·diag(w)·Zᵀ for the GHEP core T and the
// add_low_rank core M (n ≈ 300–1,000), the Eigen SelfAdjointEigenSolver calls of the
// reference (lowrank.hpp:193, :265-270), with the O(n³) work on the GPU:
//
//   1. Householder tridiagonalization A = Q·T·Qᵀ in ONE cooperative kernel (all SMs): per
//      column k, the warp that owns the next column forms its reflector right after the
//      rank-2 update, so a step costs two grid barriers (reflector → p = τ·A₂₂·v → update);
//      the matrix stays in L2.
//   2. Q = H₀·H₁·…·H_{n−3} by backward accumulation: every column of Q is independent, one
//      warp per column walks all reflectors — no barrier.
//   3. Implicit-shift QL on the tridiagonal (d, e) on the host — O(n²) scalar recurrences,
//      the same iteration and splitting test as host_linalg.cpp's sym_eig_small — recording
//      every Givens rotation (c, s) of every sweep.
//   4. The recorded rotations applied to the rows of Q on the GPU: row k of Q sees the same
//      rotation sequence, so one thread per row streams it (the sweep's carried element in a
//      register, one load and one store per rotation).
//   5. Eigenvalues ascending, eigenvector columns gathered in that order.
// Backward stable like the host path (Householder + QL): ‖AZ − ZΛ‖ ≈ ε‖A‖, ‖ZᵀZ − I‖ ≈ ε·n.

#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "eig.cuh"

namespace cg = cooperative_groups;

namespace fkb {

// √(a² + b²) without std::hypot's cost when the squares cannot overflow or underflow
static inline double fast_hypot(double a, double b) {
    const double m = std::max(std::fabs(a), std::fabs(b));
    if (m > 1e-140 && m < 1e140) return std::sqrt(a * a + b * b);
    return std::hypot(a, b);
}

constexpr int TD_T = 256;  // threads per CTA of the tridiagonalization

// Householder reflector of x = col[0..len) (column k below the diagonal, in place):
// (I − τvvᵀ)x = βe₁ with v₀ = 1; v[1..) overwrites x[1..), x[0] ← 1.  One warp.
__device__ __forceinline__ void warp_reflector(double* __restrict__ x, int len, double* __restrict__ dk_out,
                                               double dk, double* __restrict__ e_out, double* __restrict__ tau_out) {
    const int lane = threadIdx.x & 31;
    double sig = 0.0;
    for (int i = 1 + lane; i < len; i += 32) sig = fma(x[i], x[i], sig);
    for (int o = 16; o > 0; o >>= 1) sig += __shfl_xor_sync(0xffffffffu, sig, o);
    const double x0 = x[0];
    double t = 0.0, beta = x0, v0 = 1.0;
    if (sig != 0.0) {
        const double mu = sqrt(x0 * x0 + sig);
        beta = x0 <= 0.0 ? mu : -mu;
        v0 = x0 - beta;
        t = -v0 / beta;
        for (int i = 1 + lane; i < len; i += 32) x[i] /= v0;
    }
    __syncwarp();
    if (lane == 0) {
        *dk_out = dk;
        *e_out = beta;
        *tau_out = t;
        x[0] = 1.0;
    }
}

// A (n×n, column-major, full symmetric storage) → tridiagonal (d, e) with the reflectors'
// v stored below the subdiagonal of A (v₀ = 1 at A[k+1, k]) and τ in tau.  Cooperative
// launch; p (n) and part (gridDim.x) are scratch.
__global__ void __launch_bounds__(TD_T) k_tridiag(int n, double* __restrict__ A, double* __restrict__ d,
                                                  double* __restrict__ e, double* __restrict__ tau,
                                                  double* __restrict__ p, double* __restrict__ part) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int wpb = TD_T / 32, nw = gridDim.x * wpb, gw = blockIdx.x * wpb + wib;
    __shared__ double red[TD_T / 32];
    auto at = [&](int i, int j) -> double& { return A[(long long)i + (long long)j * n]; };
    // column 0's reflector (global warp 0)
    if (n > 2 && gw == 0) warp_reflector(&at(1, 0), n - 1, d, at(0, 0), e, tau);
    grid.sync();
    for (int k = 0; k + 2 < n; ++k) {
        const int o = k + 1, len = n - o;
        const double t = tau[k];
        const double* v = &at(o, k);
        // p = τ·A₂₂·v, one warp per column of A₂₂ (= row by symmetry); per-CTA partial of pᵀv
        double pv = 0.0;
        if (t != 0.0) {
            for (int i = gw; i < len; i += nw) {
                const double* col = &at(o, o + i);
                double acc = 0.0, acc1 = 0.0;
                int q = lane;
                for (; q + 32 < len; q += 64) {  // two independent chains, loads pipelined
                    acc = fma(col[q], v[q], acc);
                    acc1 = fma(col[q + 32], v[q + 32], acc1);
                }
                if (q < len) acc = fma(col[q], v[q], acc);
                acc += acc1;
                for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
                acc *= t;
                if (lane == 0) p[i] = acc;
                pv = fma(acc, v[i], pv);
            }
        }
        if (lane == 0) red[wib] = pv;
        __syncthreads();
        if (threadIdx.x == 0) {
            double sacc = 0.0;
            for (int w = 0; w < wpb; ++w) sacc += red[w];
            part[blockIdx.x] = sacc;
        }
        grid.sync();
        // A₂₂ −= v·wᵀ + w·vᵀ with w = p − ½τ(pᵀv)·v; the owner of column o (A₂₂ column 0)
        // then forms step k+1's reflector from its updated column
        if (t != 0.0) {
            double ptv = 0.0;
            for (int c = 0; c < (int)gridDim.x; ++c) ptv += part[c];  // same order in every CTA
            const double h = 0.5 * t * ptv;
            for (int j = gw; j < len; j += nw) {
                double* col = &at(o, o + j);
                const double vj = v[j], wj = p[j] - h * vj;
#pragma unroll 4
                for (int i = lane; i < len; i += 32) col[i] -= v[i] * wj + (p[i] - h * v[i]) * vj;
            }
        }
        if (k + 3 < n && gw == 0) {
            __syncwarp();
            warp_reflector(&at(o + 1, o), len - 1, d + o, at(o, o), e + o, tau + o);
        }
        grid.sync();
    }
    if (gw == 0 && lane == 0) {
        if (n >= 2) {
            d[n - 2] = at(n - 2, n - 2);
            e[n - 2] = at(n - 1, n - 2);
        }
        d[n - 1] = at(n - 1, n - 1);
        e[n - 1] = 0.0;
        if (n == 1) d[0] = at(0, 0);
    }
}

// Cluster-resident tridiagonalization for n ≤ ~660: the 16 CTAs of one cluster hold A in shared
// memory, column j in CTA j mod 16 (cyclic, so the shrinking trailing matrix stays balanced).
// Step k: the owner of column k forms the reflector from its (already updated) column and
// stores v into every CTA (DSMEM), cluster barrier; each CTA forms p_j = τ·(A₂₂v)_j for its
// columns plus its partial of pᵀv and stores them into every CTA, cluster barrier; each CTA
// applies A₂₂ −= v·wᵀ + w·vᵀ to its columns (w = p − ½τ(pᵀv)v, partials summed in CTA order:
// bit-identical everywhere).  v/p buffers alternate by step parity.  Two cluster barriers per
// step instead of two grid barriers and L2 round trips; A (with the v's below the subdiagonal,
// as k_tridiag leaves it) is written back at the end.
constexpr int TDC = 16;      // CTAs per cluster
constexpr int TDC_T = 1024;  // threads per CTA
__device__ __forceinline__ void dsmem_st(double* local, int rank, double v) {
    unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(local)), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
__global__ void __cluster_dims__(TDC, 1, 1) __launch_bounds__(TDC_T) k_tridiag_cluster(
    int n, double* __restrict__ A, double* __restrict__ d, double* __restrict__ e, double* __restrict__ tau) {
    extern __shared__ double tsm[];
    cg::cluster_group cl = cg::this_cluster();
    const int crank = int(cl.block_rank());
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = TDC_T / 32;
    const int ncl = (n - crank + TDC - 1) / TDC;  // columns owned: crank, crank + 16, …
    const int ldc = n;
    double* cols = tsm;                               // [ncl][n]
    double* vb = cols + (size_t)((n + TDC - 1) / TDC) * ldc;  // [2][n]
    double* pb = vb + 2 * n;                          // [2][n]
    double* part = pb + 2 * n;                        // [2][TDC]
    double* sc = part + 2 * TDC;                      // [4] τ of the step, per parity (+ pad)
    for (long long q = tid; q < (long long)ncl * n; q += TDC_T) {
        const int lc = int(q / n), i = int(q % n);
        cols[(size_t)lc * ldc + i] = A[(long long)i + (long long)(crank + TDC * lc) * n];
    }
    __syncthreads();
    // reflector of column k by warp 0 of its owner; v (len values) and τ to every CTA
    auto reflector = [&](int k) {
        const int o = k + 1, len = n - o, par = k & 1;
        double* x = cols + (size_t)(k / TDC) * ldc + o;
        if (warp == 0) {
            double sig = 0.0;
            for (int i = 1 + lane; i < len; i += 32) sig = fma(x[i], x[i], sig);
            for (int s = 16; s > 0; s >>= 1) sig += __shfl_xor_sync(0xffffffffu, sig, s);
            const double x0 = x[0];
            double t = 0.0, beta = x0, v0 = 1.0;
            if (sig != 0.0) {
                const double mu = sqrt(x0 * x0 + sig);
                beta = x0 <= 0.0 ? mu : -mu;
                v0 = x0 - beta;
                t = -v0 / beta;
                for (int i = 1 + lane; i < len; i += 32) x[i] /= v0;
            }
            __syncwarp();
            if (lane == 0) {
                d[k] = cols[(size_t)(k / TDC) * ldc + k];
                e[k] = beta;
                tau[k] = t;
                x[0] = 1.0;
                for (int c = 0; c < TDC; ++c) dsmem_st(&sc[par], c, t);
            }
        }
        __syncthreads();
        for (int q = tid; q < len * TDC; q += TDC_T) {  // v to every CTA (consecutive threads: one CTA, consecutive i)
            const int c = q / len, i = q % len;
            dsmem_st(&vb[par * n + o + i], c, x[i]);
        }
    };
    if (n > 2 && crank == 0) reflector(0);
    cl.sync();
    for (int k = 0; k + 2 < n; ++k) {
        const int o = k + 1, len = n - o, par = k & 1;
        const double t = sc[par];
        const double* v = vb + par * n;  // v_i at index i ≥ o
        // p_j for owned columns j ≥ o, warp per column; partial pᵀv in CTA order
        const int lc0 = (o - crank + TDC - 1) / TDC;  // first owned column ≥ o
        double pv = 0.0;
        if (t != 0.0) {
            for (int lc = lc0 + warp; lc < ncl; lc += nw) {
                const int j = crank + TDC * lc;
                const double* col = cols + (size_t)lc * ldc;
                double acc = 0.0, acc1 = 0.0;
                int i = o + lane;
                for (; i + 32 < n; i += 64) {
                    acc = fma(col[i], v[i], acc);
                    acc1 = fma(col[i + 32], v[i + 32], acc1);
                }
                if (i < n) acc = fma(col[i], v[i], acc);
                acc += acc1;
                for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
                acc *= t;
                if (lane < TDC) dsmem_st(&pb[par * n + j], lane, acc);
                pv = fma(acc, v[j], pv);
            }
        }
        __shared__ double red[TDC_T / 32];
        if (lane == 0) red[warp] = pv;
        __syncthreads();
        if (tid < TDC) {
            double sacc = 0.0;
            for (int w = 0; w < nw; ++w) sacc += red[w];
            dsmem_st(&part[par * TDC + crank], tid, sacc);
        }
        cl.sync();  // p and the pᵀv partials everywhere
        if (t != 0.0) {
            double ptv = 0.0;
            for (int c = 0; c < TDC; ++c) ptv += part[par * TDC + c];
            const double h = 0.5 * t * ptv;
            const double* p = pb + par * n;
            for (int lc = lc0 + warp; lc < ncl; lc += nw) {
                const int j = crank + TDC * lc;
                double* col = cols + (size_t)lc * ldc;
                const double vj = v[j], wj = p[j] - h * vj;
                for (int i = o + lane; i < n; i += 32) col[i] -= v[i] * wj + (p[i] - h * v[i]) * vj;
            }
        }
        __syncthreads();
        if (k + 3 < n && (o % TDC) == crank) reflector(o);
        cl.sync();  // the next reflector everywhere
    }
    if (crank == (n - 2 + TDC) % TDC && tid == 0 && n >= 2) {
        d[n - 2] = cols[(size_t)((n - 2) / TDC) * ldc + n - 2];
        e[n - 2] = cols[(size_t)((n - 2) / TDC) * ldc + n - 1];
    }
    if (crank == (n - 1) % TDC && tid == 0) {
        d[n - 1] = cols[(size_t)((n - 1) / TDC) * ldc + n - 1];
        e[n - 1] = 0.0;
    }
    for (long long q = tid; q < (long long)ncl * n; q += TDC_T) {
        const int lc = int(q / n), i = int(q % n);
        A[(long long)i + (long long)(crank + TDC * lc) * n] = cols[(size_t)lc * ldc + i];
    }
}
static size_t tridiag_cluster_smem(int n) {
    return sizeof(double) * (size_t((n + TDC - 1) / TDC) * n + 4 * size_t(n) + 2 * TDC + 4);
}

// Q = H₀H₁…H_{n−3} (column-major n×n), one warp per column held in registers (lane l owns
// rows l, l+32, …): column j starts as e_j and meets the reflectors k = n−3 … 0 (only
// k ≤ j−1 touch it); per reflector one pipelined read of v, a warp reduction, an axpy.
template <int K>
__global__ void __launch_bounds__(256) k_form_q(int n, const double* __restrict__ A, const double* __restrict__ tau,
                                               double* __restrict__ Q) {
    const int lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (j >= n) return;
    double q[K];
#pragma unroll
    for (int c = 0; c < K; ++c) q[c] = lane + 32 * c == j ? 1.0 : 0.0;
    for (int k = min(n - 3, j - 1); k >= 0; --k) {
        const double t = tau[k];
        if (t == 0.0) continue;
        const int o = k + 1;
        const double* v = A + (long long)k * n;  // v_i at row i ≥ o (v stored below the diagonal)
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < K; ++c) {
            const int i = lane + 32 * c;
            acc = fma((i >= o && i < n) ? __ldg(v + i) : 0.0, q[c], acc);
        }
        for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
        acc *= t;
#pragma unroll
        for (int c = 0; c < K; ++c) {  // v again, from L1
            const int i = lane + 32 * c;
            q[c] = fma(-acc, (i >= o && i < n) ? __ldg(v + i) : 0.0, q[c]);
        }
    }
    double* out = Q + (long long)j * n;
#pragma unroll
    for (int c = 0; c < K; ++c)
        if (lane + 32 * c < n) out[lane + 32 * c] = q[c];
}

// The QL sweeps' rotations on the rows of Q: sweep s covers columns (i, i+1) for
// i = first[s], first[s]−1, …, first[s]−cnt[s]+1 with (c, s) = rot[off[s] + t].  One thread
// per row; the element carried down a sweep stays in a register.
__global__ void __launch_bounds__(128) k_apply_rotations(int n, double* __restrict__ Q, int nsweep,
                                                        const int* __restrict__ first, const int* __restrict__ cnt,
                                                        const int* __restrict__ off, const double2* __restrict__ rot) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double* q = Q + k;  // element (k, c) at q[c·n]
    for (int sw = 0; sw < nsweep; ++sw) {
        const int i0 = first[sw], c = cnt[sw];
        const double2* rs = rot + off[sw];
        double carry = q[(long long)(i0 + 1) * n];
        int t = 0;
        // the sweep reads columns i0, i0−1, … and writes i0+1, i0, … behind them: chunks of
        // 8 loads are issued before the chunk's stores (no load waits on a store)
        for (; t + 8 <= c; t += 8) {
            double qi[8];
            double2 cs[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                qi[u] = q[(long long)(i0 - t - u) * n];
                cs[u] = __ldg(rs + t + u);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                q[(long long)(i0 - t - u + 1) * n] = cs[u].y * qi[u] + cs[u].x * carry;
                carry = cs[u].x * qi[u] - cs[u].y * carry;
            }
        }
        for (; t < c; ++t) {
            const int ii = i0 - t;
            const double2 cs = __ldg(rs + t);  // (c, s)
            const double qi = q[(long long)ii * n];
            q[(long long)(ii + 1) * n] = cs.y * qi + cs.x * carry;
            carry = cs.x * qi - cs.y * carry;
        }
        q[(long long)(i0 - c + 1) * n] = carry;
    }
}

// The same rotations with each thread's row of Q resident in shared memory (stride n + 1:
// conflict-free column access across the rows of a warp) and the rotation stream staged
// through shared memory a chunk of whole sweeps at a time (≤ RCH rotations; a sweep has at
// most n − 1 ≤ 2047): the chunk's (c, s) are one coalesced load, and within a sweep a row's
// next 8 elements are loaded before the 8 rotations that consume them (the carried DFMA chain
// is then the only serial dependency) — one shared load and store per rotation.
constexpr int RCH = 2048;
__global__ void __launch_bounds__(64) k_apply_rotations_smem(int n, int rows, double* __restrict__ Q,
                                                            const int* __restrict__ first, const int* __restrict__ cnt,
                                                            const int* __restrict__ off, const double2* __restrict__ rot,
                                                            int nchunk, const int* __restrict__ chunk_sw) {
    extern __shared__ double qs[];  // qs[lr·(n+1) + c], then the staged chunk
    const int k0 = blockIdx.x * rows, nr = min(rows, n - k0);
    const int ld = n + 1;
    double2* rc = reinterpret_cast<double2*>(qs + ((size_t(rows) * ld + 1) & ~size_t(1)));
    for (long long e = threadIdx.x; e < (long long)nr * n; e += blockDim.x) {
        const int lr = int(e % nr), c = int(e / nr);
        qs[lr * ld + c] = Q[k0 + lr + (long long)c * n];
    }
    const int lr = threadIdx.x;
    double* q = qs + lr * ld;
    for (int ch = 0; ch < nchunk; ++ch) {
        const int s0 = __ldg(chunk_sw + ch), s1 = __ldg(chunk_sw + ch + 1);
        const int r0 = __ldg(off + s0), r1 = __ldg(off + s1 - 1) + __ldg(cnt + s1 - 1);
        __syncthreads();  // the previous chunk is consumed (and, first time, Q is staged)
        for (int e = threadIdx.x; e < r1 - r0; e += blockDim.x) rc[e] = __ldg(rot + r0 + e);
        __syncthreads();
        if (lr >= nr) continue;
        for (int sw = s0; sw < s1; ++sw) {
            const int i0 = __ldg(first + sw), c = __ldg(cnt + sw);
            const double2* rs = rc + (__ldg(off + sw) - r0);
            double carry = q[i0 + 1];
            int t = 0;
            for (; t + 8 <= c; t += 8) {
                double qi[8];
                double2 cs[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    qi[u] = q[i0 - t - u];
                    cs[u] = rs[t + u];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    q[i0 - t - u + 1] = cs[u].y * qi[u] + cs[u].x * carry;
                    carry = cs[u].x * qi[u] - cs[u].y * carry;
                }
            }
            for (; t < c; ++t) {
                const double2 cs = rs[t];
                const double qi = q[i0 - t];
                q[i0 - t + 1] = cs.y * qi + cs.x * carry;
                carry = cs.x * qi - cs.y * carry;
            }
            q[i0 - c + 1] = carry;
        }
    }
    __syncthreads();
    for (long long e = threadIdx.x; e < (long long)nr * n; e += blockDim.x) {
        const int r2 = int(e % nr), c = int(e / nr);
        Q[k0 + r2 + (long long)c * n] = qs[r2 * ld + c];
    }
}

__global__ void k_gather_cols(int n, const double* __restrict__ Q, const int* __restrict__ perm, double* __restrict__ Z) {
    const long long total = (long long)n * n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int i = int(e % n), j = int(e / n);
        Z[e] = Q[i + (long long)perm[j] * n];
    }
}

void sym_eig_tridiag_device(int n, double* A, double* w_host, double* Z, cudaStream_t s) {
    // FKB_CORE_EIG=jacobi: the device block-Jacobi solver (eig.cu) for the same contract
    static const bool jac = [] {
        const char* e = std::getenv("FKB_CORE_EIG");
        return e && std::string(e) == "jacobi";
    }();
    if (jac && n > 0) {
        DBuf<double> th{size_t(n)};
        sym_eig_sorted_device(n, A, n, th.p, Z, s);
        FKB_CUDA(cudaMemcpyAsync(w_host, th.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
        FKB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    if (n <= 0) return;
    static const bool trace = std::getenv("FKB_TDEIG_TRACE") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(s);
        const auto t1 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[tdeig n=%d] %-12s %8.3f ms\n", n, what, std::chrono::duration<double, std::milli>(t1 - t0).count());
        t0 = t1;
    };
    DBuf<double> d{size_t(n)}, e{size_t(n)}, tau{size_t(std::max(n, 1))}, p{size_t(n)}, Q{size_t(n) * n};
    int dev = 0, sms = 0, per = 0;
    FKB_CUDA(cudaGetDevice(&dev));
    FKB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_tridiag, TD_T, 0));
    // enough CTAs for one warp per column of A₂₂, never more than can be co-resident
    const int want = std::max(1, ceil_div(n, TD_T / 32));
    const int grid = std::max(1, std::min(want, sms * std::max(per, 1)));
    DBuf<double> part{size_t(grid)};
    FKB_CUDA(cudaMemsetAsync(tau.p, 0, tau.bytes(), s));
    static const bool cl_ok = std::getenv("FKB_TDEIG_GRID") == nullptr;
    if (cl_ok && n >= 3 && tridiag_cluster_smem(n) <= 225 * 1024) {  // A resident in one 16-CTA cluster
        static bool attr = false;
        if (!attr) {
            FKB_CUDA(cudaFuncSetAttribute((const void*)k_tridiag_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            FKB_CUDA(cudaFuncSetAttribute((const void*)k_tridiag_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          225 * 1024));
            attr = true;
        }
        k_tridiag_cluster<<<TDC, TDC_T, tridiag_cluster_smem(n), s>>>(n, A, d.p, e.p, tau.p);
        FKB_LAUNCH_CHECK();
        count_launch();
    } else {
        void* args[] = {&n, &A, &d.p, &e.p, &tau.p, &p.p, &part.p};
        FKB_CUDA(cudaLaunchCooperativeKernel((const void*)k_tridiag, dim3(grid), dim3(TD_T), args, 0, s));
        count_launch();
    }
    lap("tridiag");
    if (n <= 256) k_form_q<8><<<ceil_div(n, 8), 256, 0, s>>>(n, A, tau.p, Q.p);
    else if (n <= 512) k_form_q<16><<<ceil_div(n, 8), 256, 0, s>>>(n, A, tau.p, Q.p);
    else if (n <= 1024) k_form_q<32><<<ceil_div(n, 8), 256, 0, s>>>(n, A, tau.p, Q.p);
    else if (n <= 2048) k_form_q<64><<<ceil_div(n, 8), 256, 0, s>>>(n, A, tau.p, Q.p);
    else throw std::invalid_argument("sym_eig_tridiag: n exceeds 2048");
    FKB_LAUNCH_CHECK();
    count_launch();
    lap("form Q");
    std::vector<double> dh(static_cast<size_t>(n)), eh(static_cast<size_t>(n));
    FKB_CUDA(cudaMemcpyAsync(dh.data(), d.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
    FKB_CUDA(cudaMemcpyAsync(eh.data(), e.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, s));
    FKB_CUDA(cudaStreamSynchronize(s));
    // implicit-shift QL on (d, e), e[i] coupling d[i] and d[i+1]; rotations recorded per sweep
    double tnorm = 0.0;
    for (int i = 0; i < n; ++i) tnorm = std::max(tnorm, std::fabs(dh[size_t(i)]) + std::fabs(eh[size_t(i)]));
    eh[size_t(n - 1)] = 0.0;
    const double eps = 2.220446049250313e-16;
    std::vector<int> first, cnt, off;
    std::vector<double2> rot;
    rot.reserve(size_t(n) * 4);
    for (int l = 0; l < n; ++l) {
        int iter = 0, m;
        do {
            for (m = l; m < n - 1; ++m) {
                const double dd = std::fabs(dh[size_t(m)]) + std::fabs(dh[size_t(m + 1)]);
                const double em = std::fabs(eh[size_t(m)]);
                if (em <= 1e-300 + eps * dd || em <= 0.5 * eps * tnorm) break;
            }
            if (m != l) {
                if (++iter > 60) throw std::runtime_error("sym_eig: QL iteration did not converge");
                double g = (dh[size_t(l + 1)] - dh[size_t(l)]) / (2.0 * eh[size_t(l)]);
                double r = fast_hypot(g, 1.0);
                g = dh[size_t(m)] - dh[size_t(l)] + eh[size_t(l)] / (g + (g >= 0.0 ? std::fabs(r) : -std::fabs(r)));
                double sn = 1.0, c = 1.0, pp = 0.0;
                bool early = false;
                const int start = int(rot.size());
                for (int i = m - 1; i >= l; --i) {
                    const double f = sn * eh[size_t(i)];
                    const double b = c * eh[size_t(i)];
                    eh[size_t(i + 1)] = r = fast_hypot(f, g);
                    if (r == 0.0) {
                        dh[size_t(i + 1)] -= pp;
                        eh[size_t(m)] = 0.0;
                        early = true;
                        break;
                    }
                    sn = f / r;
                    c = g / r;
                    g = dh[size_t(i + 1)] - pp;
                    r = (dh[size_t(i)] - g) * sn + 2.0 * c * b;
                    dh[size_t(i + 1)] = g + (pp = sn * r);
                    g = c * r - b;
                    rot.push_back(make_double2(c, sn));
                }
                const int nrot = int(rot.size()) - start;
                if (nrot > 0) {
                    first.push_back(m - 1);
                    cnt.push_back(nrot);
                    off.push_back(start);
                }
                if (early) continue;
                dh[size_t(l)] -= pp;
                eh[size_t(l)] = g;
                eh[size_t(m)] = 0.0;
            }
        } while (m != l);
    }
    const int nsweep = int(first.size());
    lap("host QL");
    if (nsweep > 0) {
        DBuf<int> df{size_t(nsweep)}, dc{size_t(nsweep)}, doff{size_t(nsweep)};
        DBuf<double2> drot(rot.size());
        FKB_CUDA(cudaMemcpyAsync(df.p, first.data(), sizeof(int) * size_t(nsweep), cudaMemcpyHostToDevice, s));
        FKB_CUDA(cudaMemcpyAsync(dc.p, cnt.data(), sizeof(int) * size_t(nsweep), cudaMemcpyHostToDevice, s));
        FKB_CUDA(cudaMemcpyAsync(doff.p, off.data(), sizeof(int) * size_t(nsweep), cudaMemcpyHostToDevice, s));
        FKB_CUDA(cudaMemcpyAsync(drot.p, rot.data(), sizeof(double2) * rot.size(), cudaMemcpyHostToDevice, s));
        // rows of Q resident in shared memory next to a staged chunk of whole sweeps (≤ 200 KB
        // per CTA) unless n is too large for it
        const size_t chunk_bytes = size_t(RCH) * sizeof(double2) + 16;
        const int rows = int(std::min<long long>(64, (200LL * 1024 - (long long)chunk_bytes) / (8LL * (n + 1))));
        static const bool smem_rot = std::getenv("FKB_TDEIG_L2ROT") == nullptr;
        if (smem_rot && rows >= 4) {
            std::vector<int> csw{0};  // chunk boundaries (sweep indices), ≤ RCH rotations each
            int acc = 0;
            for (int sw = 0; sw < nsweep; ++sw) {
                if (acc + cnt[size_t(sw)] > RCH) {
                    csw.push_back(sw);
                    acc = 0;
                }
                acc += cnt[size_t(sw)];
            }
            csw.push_back(nsweep);
            DBuf<int> dcsw(csw.size());
            FKB_CUDA(cudaMemcpyAsync(dcsw.p, csw.data(), sizeof(int) * csw.size(), cudaMemcpyHostToDevice, s));
            const size_t shm = sizeof(double) * ((size_t(rows) * (n + 1) + 1) & ~size_t(1)) + chunk_bytes;
            static bool attr = false;
            if (!attr) {
                FKB_CUDA(cudaFuncSetAttribute(k_apply_rotations_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              210 * 1024));
                attr = true;
            }
            k_apply_rotations_smem<<<ceil_div(n, rows), 64, shm, s>>>(n, rows, Q.p, df.p, dc.p, doff.p, drot.p,
                                                                      int(csw.size()) - 1, dcsw.p);
            FKB_LAUNCH_CHECK();
            FKB_CUDA(cudaStreamSynchronize(s));  // dcsw goes out of scope
        } else {
            k_apply_rotations<<<ceil_div(n, 128), 128, 0, s>>>(n, Q.p, nsweep, df.p, dc.p, doff.p, drot.p);
        }
        FKB_LAUNCH_CHECK();
        count_launch();
        FKB_CUDA(cudaStreamSynchronize(s));  // the rotation buffers go out of scope
    }
    lap("rotations");
    std::vector<int> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int x, int y) { return dh[size_t(x)] < dh[size_t(y)]; });
    for (int j = 0; j < n; ++j) w_host[j] = dh[size_t(order[size_t(j)])];
    DBuf<int> perm{size_t(n)};
    FKB_CUDA(cudaMemcpyAsync(perm.p, order.data(), sizeof(int) * size_t(n), cudaMemcpyHostToDevice, s));
    k_gather_cols<<<std::min(ceil_div((long long)n * n, 256), 4096), 256, 0, s>>>(n, Q.p, perm.p, Z);
    FKB_LAUNCH_CHECK();
    count_launch();
    FKB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace fkb

// test hook: host A (n×n column-major symmetric) → w ascending, Z (column-major) on the host
extern "C" int fkb_sym_eig_tridiag(int n, const double* A, double* w, double* Z) {
    try {
        if (n < 0) return 1;
        if (n == 0) return 0;
        fkb::DBuf<double> dA(size_t(n) * n), dZ(size_t(n) * n);
        FKB_CUDA(cudaMemcpy(dA.p, A, sizeof(double) * size_t(n) * n, cudaMemcpyHostToDevice));
        fkb::sym_eig_tridiag_device(n, dA.p, w, dZ.p, nullptr);
        FKB_CUDA(cudaMemcpy(Z, dZ.p, sizeof(double) * size_t(n) * n, cudaMemcpyDeviceToHost));
        return 0;
    } catch (const std::exception&) {
        return 3;
    }
}
