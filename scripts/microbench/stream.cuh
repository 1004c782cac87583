// stream.cuh — TMA-bulk streaming dot products for the HBM-bound passes of a step.
//
// out_v = epi(v, Σ_c A[v·ld + c]·x_c) for nvec contiguous vectors of length len (A row-major
// with rows = vectors: the row-major U of the mean update, the columns of P / Pᵀ of the
// rotations).  A persistent grid (one CTA per SM) walks tiles of `vt` consecutive vectors;
// each tile is ONE cp.async.bulk global→shared copy completed on an mbarrier, `stages`
// tiles in flight per SM, so the SM issues a handful of instructions per 20–64 KB instead of
// one load per 8 bytes and HBM sees long sequential bursts.  x lives in shared memory.
#pragma once

#include <algorithm>
#include <cstdint>

#include "common.cuh"

namespace fkb {

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    unsigned ok = 0;
    while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(smem))),
                 "l"(gmem), "r"(bytes), "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
                 : "memory");
}

constexpr int kStreamThreads = 256;
constexpr int kStreamMaxStages = 4;

template <class XL, class Epi>
__global__ void __launch_bounds__(kStreamThreads) k_stream_dot(long long nvec, int len, long long ld,
                                                              const double* __restrict__ A, XL xl, Epi epi, int vt,
                                                              int stages) {
    extern __shared__ __align__(16) double smem[];
    __shared__ __align__(8) unsigned long long full[kStreamMaxStages];
    __shared__ double red[kStreamThreads / 32];
    double* xs = smem;                                            // len (padded to 2)
    double* buf = smem + ((len + 1) & ~1);                        // stages × vt·ld
    const long long tile_elems = (long long)vt * ld;
    const long long ntiles = (nvec + vt - 1) / vt;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int c = tid; c < len; c += kStreamThreads) xs[c] = xl(c);
    __syncthreads();
    auto issue = [&](long long t, int s) {
        const long long v0 = t * vt;
        const long long nv = min((long long)vt, nvec - v0);
        const unsigned bytes = unsigned(nv * ld * 8);
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(buf + s * tile_elems, A + v0 * ld, bytes, &full[s]);
    };
    long long t = blockIdx.x;
    if (tid == 0)
        for (int s = 0; s < stages; ++s)
            if (t + (long long)s * gridDim.x < ntiles) issue(t + (long long)s * gridDim.x, s);
    // warp ↦ (vector, segment): wpv warps per vector when vt < 8, else vectors strided by 8
    const int nw = kStreamThreads / 32;
    const int wpv = vt >= nw ? 1 : nw / vt;
    const int seg = (len + wpv - 1) / wpv;
    for (int it = 0; t < ntiles; ++it, t += gridDim.x) {
        const int s = it % stages;
        const unsigned parity = unsigned((it / stages) & 1);
        mbar_wait(&full[s], parity);
        const double* tb = buf + s * tile_elems;
        const long long v0 = t * vt;
        const int nv = int(min((long long)vt, nvec - v0));
        if (vt >= nw) {
            for (int v = warp; v < nv; v += nw) {
                const double* a = tb + (long long)v * ld;
                double acc0 = 0.0, acc1 = 0.0;
                int c = lane;
                for (; c + 32 < len; c += 64) {
                    acc0 = fma(a[c], xs[c], acc0);
                    acc1 = fma(a[c + 32], xs[c + 32], acc1);
                }
                if (c < len) acc0 = fma(a[c], xs[c], acc0);
                double acc = acc0 + acc1;
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (lane == 0) epi(v0 + v, acc);
            }
            __syncthreads();  // stage s fully consumed
        } else {
            const int v = warp / wpv, sg = warp % wpv;
            double acc = 0.0;
            if (v < nv) {
                const double* a = tb + (long long)v * ld;
                const int c0 = sg * seg, c1 = min(len, c0 + seg);
                double acc1 = 0.0;
                int c = c0 + lane;
                for (; c + 32 < c1; c += 64) {
                    acc = fma(a[c], xs[c], acc);
                    acc1 = fma(a[c + 32], xs[c + 32], acc1);
                }
                if (c < c1) acc = fma(a[c], xs[c], acc);
                acc += acc1;
            }
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (lane == 0) red[warp] = acc;
            __syncthreads();  // partials visible; stage s fully consumed
            if (tid < nv) {
                double sum = 0.0;
                for (int q = 0; q < wpv; ++q) sum += red[tid * wpv + q];
                epi(v0 + tid, sum);
            }
            __syncthreads();  // red reusable
        }
        if (tid == 0 && t + (long long)stages * gridDim.x < ntiles) issue(t + (long long)stages * gridDim.x, s);
    }
}

inline int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        FKB_CUDA(cudaGetDevice(&dev));
        FKB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    }
    return sms;
}

// vt vectors per tile chosen so a tile is ~tile_bytes; stages so the ring fits in shared
// memory.  Returns false (nothing launched) when the rows are not 16-byte aligned or too long;
// the caller then uses its load/store kernel.
template <class XL, class Epi>
inline bool launch_stream_dot(long long nvec, int len, long long ld, const double* A, XL xl, Epi epi, cudaStream_t s,
                              long long tile_bytes = 40 * 1024) {
    if (nvec <= 0) return true;
    if ((ld * 8) % 16 != 0 || (reinterpret_cast<uintptr_t>(A) & 15) != 0 || len <= 0) return false;
    int vt = int(std::max<long long>(1, tile_bytes / (ld * 8)));
    if (vt > 8) vt = (vt / 8) * 8;
    else vt = vt >= 8 ? 8 : vt >= 4 ? 4 : vt >= 2 ? 2 : 1;
    const size_t xs_bytes = sizeof(double) * size_t((len + 1) & ~1);
    const size_t tile = sizeof(double) * size_t(vt) * size_t(ld);
    int stages = kStreamMaxStages;
    while (stages > 2 && xs_bytes + stages * tile > 200 * 1024) --stages;
    if (xs_bytes + stages * tile > 200 * 1024) return false;
    const size_t smem = xs_bytes + stages * tile;
    static bool attr = false;  // per template instance
    if (!attr) {
        FKB_CUDA(cudaFuncSetAttribute((const void*)k_stream_dot<XL, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
        attr = true;
    }
    const long long ntiles = (nvec + vt - 1) / vt;
    const int grid = int(std::min<long long>(ntiles, sm_count()));
    k_stream_dot<XL, Epi><<<grid, kStreamThreads, smem, s>>>(nvec, len, ld, A, xl, epi, vt, stages);
    FKB_LAUNCH_CHECK();
    count_launch();
    return true;
}

}  // namespace fkb
