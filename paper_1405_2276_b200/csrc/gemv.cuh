// gemv.cuh — HBM-bound FP64 matrix–vector kernels with fused prologue/epilogue functors:
// k_gemv_rowmajor (row-major A, the step's U pass) and k_coldot (column dots of a
// column-major A: the P/Pᵀ rotations, the capacitance RHS, Bᵀz).
#pragma once

#include <cstdint>
#include <cstdlib>

#include "common.cuh"

namespace fkb {

// preferred shared-memory carveout (%) of the kernels that run beside the step's FFT passes
// (FKB_CARVEOUT, default 50: ~100 KB shared memory, the rest L1 for the in-flight loads)
inline int carveout_pct() {
    static const int v = [] {
        const char* e = std::getenv("FKB_CARVEOUT");
        return e ? std::atoi(e) : 50;
    }();
    return v;
}

struct XPlain {
    const double* x;
    __device__ __forceinline__ double operator()(long long c) const { return __ldg(x + c); }
};
struct XProd {  // x_c = a_c · b_c
    const double* a;
    const double* b;
    __device__ __forceinline__ double operator()(long long c) const { return __ldg(a + c) * __ldg(b + c); }
};
struct EpiStore {  // y_i = v
    double* y;
    __device__ __forceinline__ void operator()(long long i, double v) const { y[i] = v; }
};
struct EpiAxpby {  // y_i = α·v + β·y_i
    double* y;
    double alpha, beta;
    __device__ __forceinline__ void operator()(long long i, double v) const {
        y[i] = beta == 0.0 ? alpha * v : alpha * v + beta * y[i];
    }
};

// y_i = epi(i, Σ_j A_ij·x_j) for ROW-MAJOR A (m×k, ld ≥ k): each warp reads rows as contiguous
// 256-B chunks, 4 rows at a time, so the matrix streams linearly from HBM (the step's U-pass;
// U is stored once more row-major for this).  The grid is persistent (one wave
// of resident CTAs) and each warp owns a contiguous, balanced slice of rows — no second
// partial wave, every warp finishes within one 4-row group of the others.
template <class XL, class Epi>
__global__ void __launch_bounds__(256) k_gemv_rowmajor(long long m, int k, const double* __restrict__ A,
                                                      long long ld, XL xl, Epi epi) {
    extern __shared__ double xs[];
    for (int c = threadIdx.x; c < k; c += blockDim.x) xs[c] = xl(c);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long lo = m * w / nw, hi = m * (w + 1) / nw;  // this warp's contiguous rows
    for (long long r0 = lo; r0 < hi; r0 += 4) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    const int nq = (int)min(4LL, hi - r0);
    int c = lane;
    for (; c + 96 < k; c += 128) {  // 16 independent loads in flight per lane
        double v[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int u = 0; u < 4; ++u) v[q][u] = q < nq ? __ldcs(A + (r0 + q) * ld + c + 32 * u) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double xv = xs[c + 32 * u];
#pragma unroll
            for (int q = 0; q < 4; ++q) s[q] = fma(v[q][u], xv, s[q]);
        }
    }
    for (; c < k; c += 32) {
        const double xv = xs[c];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < nq) s[q] = fma(__ldcs(A + (r0 + q) * ld + c), xv, s[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
    if (lane < nq) {
        const double v = lane == 0 ? s[0] : lane == 1 ? s[1] : lane == 2 ? s[2] : s[3];
        epi(r0 + lane, v);
    }
    }
}

// Short-row variant (k ≤ 32·KC): a lane holds its KC row chunks of 4 rows in registers, so a
// whole 4-row group (4·k doubles per warp) is one round trip to HBM instead of one per
// 128-column slice plus the 32-wide tail; x lives in registers too.
template <int KC, class XL, class Epi>
__global__ void __launch_bounds__(256, 2) k_gemv_rowmajor_reg(long long m, int k, const double* __restrict__ A,
                                                             long long ld, XL xl, Epi epi) {
    const int lane = threadIdx.x & 31;
    double xv[KC];
#pragma unroll
    for (int u = 0; u < KC; ++u) xv[u] = lane + 32 * u < k ? xl(lane + 32 * u) : 0.0;
    const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long lo = m * w / nw, hi = m * (w + 1) / nw;
    for (long long r0 = lo; r0 < hi; r0 += 4) {
        const int nq = (int)min(4LL, hi - r0);
        double v[4][KC];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int u = 0; u < KC; ++u)
                v[q][u] = (q < nq && lane + 32 * u < k) ? __ldcs(A + (r0 + q) * ld + lane + 32 * u) : 0.0;
        double s[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            s[q] = 0.0;
#pragma unroll
            for (int u = 0; u < KC; ++u) s[q] = fma(v[q][u], xv[u], s[q]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
        if (lane < nq) epi(r0 + lane, lane == 0 ? s[0] : lane == 1 ? s[1] : lane == 2 ? s[2] : s[3]);
    }
}

template <int KC, class XL, class Epi>
inline void launch_gemv_rowmajor_reg(long long m, int k, const double* A, long long ld, XL xl, Epi epi,
                                     cudaStream_t s, int per_sm_cap, int threads) {
    int dev = 0, sms = 0, per_sm = 0;
    FKB_CUDA(cudaGetDevice(&dev));
    FKB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    FKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gemv_rowmajor_reg<KC, XL, Epi>, threads, 0));
    long long cap = (long long)std::max(sms, 1) * std::max(per_sm, 1);
    if (per_sm_cap >= 1000) cap = 1LL << 40;  // non-persistent: one CTA per row block
    else if (per_sm_cap > 0) cap = std::min(cap, (long long)std::max(sms, 1) * per_sm_cap);
    if (per_sm_cap < 0) cap = std::min(cap, (long long)-per_sm_cap);  // negative: a total CTA count
    const long long ctas = std::min((m + threads / 8 - 1) / (threads / 8), cap);
    k_gemv_rowmajor_reg<KC, XL, Epi><<<(unsigned)ctas, threads, 0, s>>>(m, k, A, ld, xl, epi);
}

// per_sm_cap > 0 limits the resident CTAs per SM (the step runs the U pass beside the
// latency-bound main chain, which needs room on every SM)
template <class XL, class Epi>
inline void launch_gemv_rowmajor(long long m, int k, const double* A, long long ld, XL xl, Epi epi, cudaStream_t s,
                                 int per_sm_cap = 0, int threads = 256) {
    if (m <= 0) return;
    if (k >= 1 && k <= 320) {  // the step's U pass: rank ≤ 320 held in registers
        const int c = per_sm_cap, t = threads;
        switch ((k + 31) / 32) {
            case 1: launch_gemv_rowmajor_reg<1>(m, k, A, ld, xl, epi, s, c, t); break;
            case 2: launch_gemv_rowmajor_reg<2>(m, k, A, ld, xl, epi, s, c, t); break;
            case 3: launch_gemv_rowmajor_reg<3>(m, k, A, ld, xl, epi, s, c, t); break;
            case 4: launch_gemv_rowmajor_reg<4>(m, k, A, ld, xl, epi, s, c, t); break;
            case 5: launch_gemv_rowmajor_reg<5>(m, k, A, ld, xl, epi, s, c, t); break;
            case 6: launch_gemv_rowmajor_reg<6>(m, k, A, ld, xl, epi, s, c, t); break;
            case 7: launch_gemv_rowmajor_reg<7>(m, k, A, ld, xl, epi, s, c, t); break;
            case 8: launch_gemv_rowmajor_reg<8>(m, k, A, ld, xl, epi, s, c, t); break;
            case 9: launch_gemv_rowmajor_reg<9>(m, k, A, ld, xl, epi, s, c, t); break;
            default: launch_gemv_rowmajor_reg<10>(m, k, A, ld, xl, epi, s, c, t); break;
        }
        FKB_LAUNCH_CHECK();
        count_launch();
        return;
    }
    const size_t shm = sizeof(double) * size_t(std::max(k, 1));
    int dev = 0, sms = 0, per_sm = 0;
    FKB_CUDA(cudaGetDevice(&dev));
    FKB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    static bool carve = false;  // beside the step's FFT kernels: room for their CTAs, L1 kept
    if (!carve) {
        FKB_CUDA(cudaFuncSetAttribute(k_gemv_rowmajor<XL, Epi>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_pct()));
        carve = true;
    }
    FKB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gemv_rowmajor<XL, Epi>, 256, shm));
    if (per_sm_cap > 0 && per_sm_cap < 1000) per_sm = std::min(per_sm, per_sm_cap);
    const long long warps = (m + 3) / 4;  // at least one 4-row group per warp
    long long ctas = per_sm_cap >= 1000 ? (warps + 7) / 8  // non-persistent
                                        : std::min((warps + 7) / 8, (long long)std::max(sms, 1) * std::max(per_sm, 1));
    if (per_sm_cap < 0) ctas = std::min(ctas, (long long)-per_sm_cap);  // negative: a total CTA count
    k_gemv_rowmajor<XL, Epi><<<(unsigned)ctas, 256, shm, s>>>(m, k, A, ld, xl, epi);
    FKB_LAUNCH_CHECK();
    count_launch();
}

// Optional CTA epilogue of k_coldot, run by the whole CTA once its CPC column values are known
// (vals in shared memory): NoCta does nothing; CtaParts leaves this CTA's partial of the
// capacitance right-hand side, parts[b·r + l] = Σ_c Erow[j0+c, l]·wsq_{j0+c}·vals_c, so the
// rotate-in r̃ = Pᵀz and Eᵀ(Λ_M⁻¹r̃) share one pass (the PCG kernel sums the partials).
struct NoCta {
    static constexpr bool active = false;
    __device__ __forceinline__ void operator()(int, int, const double*) const {}
};
struct CtaParts {
    static constexpr bool active = true;
    const double* Erow;  // m×r row-major
    int r;
    const double* wsq;
    double* parts;  // gridDim.x × r
    // Completion signal for a consumer that is already resident (the pipelined batch launches
    // the PCG cluster first, cappcg.cuh PcgRhs::ready): the last CTA to leave its partials
    // publishes the step's α (alpha_dev[1], set by the step prologue) as the epoch.
    double* ready = nullptr;
    unsigned* ticket = nullptr;
    const double* alpha_dev = nullptr;
    __device__ __forceinline__ void operator()(int j0, int nc, const double* vals) const {
        partials(j0, nc, vals);
        if (!ready) return;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
                *ticket = 0;
                __threadfence();
                *reinterpret_cast<volatile double*>(ready) = alpha_dev[1];
            }
        }
    }
    __device__ __forceinline__ void partials(int j0, int nc, const double* vals) const {
        double w[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) w[c] = c < nc ? __ldg(wsq + j0 + c) * vals[c] : 0.0;
        for (int l = threadIdx.x; l < r; l += blockDim.x) {
            double acc = 0.0;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c < nc) acc = fma(__ldg(Erow + (long long)(j0 + c) * r + l), w[c], acc);
            parts[(long long)blockIdx.x * r + l] = acc;
        }
    }
};

// ---- single-launch column dots: out_j = epi(j, Σ_i A_ij·x_i) for column-major A (m×n).
// A CTA owns CPC consecutive columns; each thread keeps its x values in registers (reused
// over the CPC columns) and issues every load of a 2048-row chunk × CPC columns before the
// first FMA, so a chunk costs one memory latency.  Fixed-order reductions (deterministic),
// no split partials and no second kernel.
template <class XL, class Epi, int CPC, class CE = NoCta, bool PDL = false>
__global__ void __launch_bounds__(256, CPC == 4 ? 4 : 1) k_coldot(int m, int n, const double* __restrict__ A, long long lda, XL xl,
                                               Epi epi, CE cepi = CE{}) {
    constexpr int EPT = CPC == 4 ? 4 : 8;  // CPC 4: ≤ 64 regs, 4 CTAs/SM, n = 2048 in one wave
    const int j0 = blockIdx.x * CPC;
    double acc[CPC];
#pragma unroll
    for (int c = 0; c < CPC; ++c) acc[c] = 0.0;
    auto chunk = [&](int i0, const double (&e)[CPC][EPT]) {
        double xv[EPT];
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
            const int i = i0 + threadIdx.x + 256 * q;
            xv[q] = i < m ? xl(i) : 0.0;
        }
#pragma unroll
        for (int c = 0; c < CPC; ++c)
#pragma unroll
            for (int q = 0; q < EPT; ++q) acc[c] = fma(e[c][q], xv[q], acc[c]);
    };
    auto load = [&](int i0, double (&e)[CPC][EPT]) {
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
            const int i = i0 + threadIdx.x + 256 * q;
#pragma unroll
            for (int c = 0; c < CPC; ++c) e[c][q] = (i < m && j0 + c < n) ? A[i + (long long)(j0 + c) * lda] : 0.0;
        }
    };
    int istart = 0;
    if constexpr (PDL) {
        // programmatic dependent launch: the first chunk of A does not depend on the producer
        // kernel, so it is in flight before waiting for that kernel's x
        double e[CPC][EPT];
        load(0, e);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        chunk(0, e);
        istart = 256 * EPT;
    }
    for (int i0 = istart; i0 < m; i0 += 256 * EPT) {
        double e[CPC][EPT];
        load(i0, e);  // every load of the chunk (and x's) before the first FMA
        chunk(i0, e);
    }
    __shared__ double red[8][CPC];
#pragma unroll
    for (int c = 0; c < CPC; ++c) {
        double v = acc[c];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = v;
    }
    __syncthreads();
    __shared__ double colv[CPC];
    if (threadIdx.x < CPC && j0 + threadIdx.x < n) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
        epi(j0 + threadIdx.x, v);
        colv[threadIdx.x] = v;
    }
    if constexpr (CE::active) {
        __syncthreads();
        cepi(j0, min(CPC, n - j0), colv);
    }
}

inline int coldot_cpc(int n) {
    static const int forced = [] {  // FKB_COLDOT_CPC: columns per CTA for every size (measurement)
        const char* e = std::getenv("FKB_COLDOT_CPC");
        const int v = e ? std::atoi(e) : 0;
        return (v == 1 || v == 2 || v == 4 || v == 8) ? v : 0;
    }();
    if (forced) return forced;
    // 8 columns per CTA (≈ 180 registers, one CTA per SM, 3.5 waves at n = 4096) measured slower
    // than 4 (≤ 64 registers, 4 CTAs per SM) at every size: c4 rotate_in 45 → 33 µs, rotate_out
    // 33 → 27 µs (5.0 TB/s), step 351 → 332 µs
    return n >= 4 * 296 ? 4 : n >= 2 * 296 ? 2 : 1;
}
inline int coldot_grid(int n) { return n <= 0 ? 0 : (n + coldot_cpc(n) - 1) / coldot_cpc(n); }

template <class XL, class Epi, class CE = NoCta>
inline void launch_coldot(int m, int n, const double* A, long long lda, XL xl, Epi epi, cudaStream_t s,
                          CE cepi = CE{}, bool pdl = false) {
    if (n <= 0) return;
    const unsigned g = (unsigned)coldot_grid(n);
    auto go = [&](auto kplain, auto kpdl) {
        if (!pdl) {
            kplain<<<g, 256, 0, s>>>(m, n, A, lda, xl, epi, cepi);
            return;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(g, 1, 1);
        cfg.blockDim = dim3(256, 1, 1);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        FKB_CUDA(cudaLaunchKernelEx(&cfg, kpdl, m, n, A, lda, xl, epi, cepi));
    };
    switch (coldot_cpc(n)) {
        case 8: go(k_coldot<XL, Epi, 8, CE, false>, k_coldot<XL, Epi, 8, CE, true>); break;
        case 4: go(k_coldot<XL, Epi, 4, CE, false>, k_coldot<XL, Epi, 4, CE, true>); break;
        case 2: go(k_coldot<XL, Epi, 2, CE, false>, k_coldot<XL, Epi, 2, CE, true>); break;
        default: go(k_coldot<XL, Epi, 1, CE, false>, k_coldot<XL, Epi, 1, CE, true>); break;
    }
    FKB_LAUNCH_CHECK();
    count_launch();
}

}  // namespace fkb
