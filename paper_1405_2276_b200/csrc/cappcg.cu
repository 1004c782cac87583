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

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int PC_CL = 16;   // CTAs per cluster (non-portable size, opt-in attribute)
constexpr int PC_T = 512;   // threads per CTA
constexpr int PC_MAXN = 1024;

struct PcgShared {
    double v[2][PC_MAXN];      // vector being multiplied by K, double-buffered by iteration parity
    double part[2][PC_CL][4];  // (γ, δ, rᵀr) partials, slot c written by CTA c
    double q[PC_MAXN / PC_CL];
    double red[PC_T / 32][4];
};

__device__ __forceinline__ void st_cluster(double* local_addr, int rank, double v) {
    // remote shared-memory store into CTA `rank` of this cluster (fire and forget; made
    // visible by the next barrier.cluster arrive.release / wait.acquire pair)
    unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(local_addr)), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

// remote store into CTA `rank` that also signals `bytes` on that CTA's mbarrier (the mbarrier
// is at the same shared offset in every CTA): no cluster barrier needed on the receive side
__device__ __forceinline__ void st_async_cluster(double* local_addr, unsigned long long* local_bar, int rank, double v) {
    unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(local_addr)), ra;
    unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(local_bar)), rb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(b), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(ra), "d"(v), "r"(rb)
                 : "memory");
}

__device__ __forceinline__ void cp_async8(double* smem, const double* g) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(a), "l"(g) : "memory");
}

// sh.q[i − r0] = (K·v)_i for this CTA's rows, v = sh.v[buf]: 16 lanes per row (two rows
// per warp, PC_T/16 rows per pass) over the staged K block, 4-level shuffle reduction
__device__ __forceinline__ void block_matvec(PcgShared& sh, const double* Ks, const double* K, long long ld, int n,
                                             int r0, int r1, int buf, int kstage) {
    const int sub = threadIdx.x & 15, slot = threadIdx.x >> 4;
    const double* v = sh.v[buf];
    for (int i0 = r0; i0 < r1; i0 += PC_T / 16) {  // uniform trip count across the CTA
        const int i = i0 + slot;
        double s0 = 0.0, s1 = 0.0;
        if (i < r1) {
            const double* Kc = kstage ? Ks + (long long)(i - r0) * n : K + (long long)i * ld;
            // four independent FMA chains (FP64 latency dominates this short dot)
            double s2 = 0.0, s3 = 0.0;
            int j = sub;
            for (; j + 48 < n; j += 64) {
                s0 = fma(Kc[j], v[j], s0);
                s1 = fma(Kc[j + 16], v[j + 16], s1);
                s2 = fma(Kc[j + 32], v[j + 32], s2);
                s3 = fma(Kc[j + 48], v[j + 48], s3);
            }
            for (; j < n; j += 16) s0 = fma(Kc[j], v[j], s0);
            s0 += s2;
            s1 += s3;
        }
        double s = s0 + s1;
        for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (sub == 0 && i < r1) sh.q[i - r0] = s;
    }
    __syncthreads();
}

// Same product with this thread's K entries held in registers (KR > 0: n ≤ 16·KR, one row
// per 16-lane group, entries j = sub + 16k): per iteration only the exchanged vector is read
// from shared memory (one broadcast wavefront per load) — the K block is read once per solve.
template <int KR>
__device__ __forceinline__ void block_matvec_reg(PcgShared& sh, const double (&kr)[KR], int r0, int r1, int buf) {
    const int sub = threadIdx.x & 15, slot = threadIdx.x >> 4;
    const double* v = sh.v[buf] + sub;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int k = 0; k < KR; ++k) a[k & 3] = fma(kr[k], v[16 * k], a[k & 3]);
    double s = (a[0] + a[1]) + (a[2] + a[3]);
    for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (sub == 0 && r0 + slot < r1) sh.q[slot] = s;
    __syncthreads();
}

// sh.q[c] = sqd_j · Σ_i E_ij·wsq_i·rt_i for this CTA's rows j = r0 + c (the fused capacitance
// RHS): the CTA's threads split the m rows of E, every column's loads in flight together,
// warp shuffles then one pass over per-warp partials in fixed order (deterministic)
__device__ __forceinline__ void fused_rhs(PcgShared& sh, const PcgRhs& ra, int r0, int r1) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ double part[PC_T / 32][8];
    for (int c0 = r0; c0 < r1; c0 += 8) {
        const int nc = min(8, r1 - c0);
        double acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = 0.0;
        int i = tid;
        for (; i + 3 * PC_T < ra.m; i += 4 * PC_T) {  // 4 rows × 8 columns of loads in flight
            double w[4], e[4][8];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int iq = i + q * PC_T;
                w[q] = __ldg(ra.wsq + iq) * __ldg(ra.rt + iq);
#pragma unroll
                for (int c = 0; c < 8; ++c) e[q][c] = c < nc ? __ldg(ra.E + iq + (long long)(c0 + c) * ra.lde) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[c] = fma(e[q][c], w[q], acc[c]);
        }
        for (; i < ra.m; i += PC_T) {
            const double w = __ldg(ra.wsq + i) * __ldg(ra.rt + i);
#pragma unroll
            for (int c = 0; c < 8; ++c)
                if (c < nc) acc[c] = fma(__ldg(ra.E + i + (long long)(c0 + c) * ra.lde), w, acc[c]);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            double v = acc[c];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) part[warp][c] = v;
        }
        __syncthreads();
        if (tid < nc) {
            double v = 0.0;
            for (int w = 0; w < PC_T / 32; ++w) v += part[w][tid];
            sh.q[c0 - r0 + tid] = __ldg(ra.sqd + c0 + tid) * v;
        }
        __syncthreads();
    }
}

// sh.q[c] = sqd_j · Σ_b parts[b·n + j] for this CTA's rows j = r0 + c (the rotate-in kernel's
// per-CTA partials of Eᵀ(Λ_M⁻¹r̃)): warp w sums parts b ≡ w (mod 16), lane l column r0 + l
// (+32), 16 loads in flight per lane; the 16 warp sums are then added in warp order
// (deterministic).
__device__ __forceinline__ void parts_rhs(PcgShared& sh, const PcgRhs& ra, int n, int r0, int r1) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = PC_T / 32;
    __shared__ double part[NW][32];
    for (int c0 = 0; c0 < r1 - r0; c0 += 32) {
        const int c = c0 + lane;
        const bool on = r0 + c < r1;
        double acc = 0.0;
        for (int b0 = warp; b0 < ra.nparts; b0 += NW * 16) {
            double v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                const int b = b0 + q * NW;
                v[q] = (on && b < ra.nparts) ? __ldcg(ra.parts + (long long)b * n + r0 + c) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) acc += v[q];
        }
        part[warp][lane] = acc;
        __syncthreads();
        if (tid < 32 && on) {
            double v = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) v += part[w][lane];
            sh.q[c] = __ldg(ra.sqd + r0 + c) * v;
        }
        __syncthreads();
    }
}

// The filter step's Woodbury tail (PcgTail): x (all n entries) is in xs on every CTA.
// s̃ rows split over the cluster, a warp per 4 rows with 32 loads in flight per lane; then each
// CTA commits d for the capacitance rows it owns and CTA 0 commits α.
__device__ __forceinline__ void woodbury_tail(const PcgTail& tl, const double* xs, double* ys, int n, int crank,
                                              bool own, int row, double x, bool zero) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int j = tid; j < n; j += PC_T) ys[j] = zero ? 0.0 : __ldg(tl.sqd + j) * xs[j];
    __syncthreads();
    const int mb = (tl.m + PC_CL - 1) / PC_CL;
    const int i0 = min(tl.m, crank * mb), i1 = min(tl.m, i0 + mb);
    for (int ib = i0 + warp * 4; ib < i1; ib += (PC_T / 32) * 4) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int jb = 0; jb < n; jb += 32 * 8) {
            double e[4][8];
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int j = jb + lane + 32 * c;
                    e[q][c] = (ib + q < i1 && j < n) ? __ldcg(tl.Erow + (long long)(ib + q) * n + j) : 0.0;
                }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int j = jb + lane + 32 * c;
                const double yv = j < n ? ys[j] : 0.0;
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q] = fma(e[q][c], yv, acc[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            for (int o = 16; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
        if (lane < 4 && ib + lane < i1) {
            const int i = ib + lane;
            const double a = lane == 0 ? acc[0] : lane == 1 ? acc[1] : lane == 2 ? acc[2] : acc[3];
            tl.st[i] = __ldg(tl.wsq + i) * (__ldg(tl.rt + i) + a);
        }
    }
    const double alpha = tl.alpha_dev[1];
    if (own) {
        const double dj = tl.d[row], l = tl.lam[row], c = alpha - dj;
        tl.dc[row] = zero ? 0.0 : __ldg(tl.sqd + row) * x;
        const double dn = (dj + alpha * l * c) / (1.0 + l * c);
        tl.d[row] = dn;
        if (tl.d_q) tl.d_q[row] = dn;
        if (tl.hout[1]) reinterpret_cast<double*>(tl.hout[1])[row] = dn;
    }
    if (crank == 0 && tid == 0) {
        tl.alpha_dev[0] = alpha;
        if (tl.alpha_q) *tl.alpha_q = alpha;
        if (tl.gate_q) *tl.gate_q = 0;
    }
}

template <int KR>
__global__ void __launch_bounds__(PC_T) k_cap_pcg(const double* __restrict__ K, long long ld, int n,
                                                 double* __restrict__ u, double* __restrict__ work,
                                                 int* __restrict__ fallback, int maxit, double tol, int kstage,
                                                 unsigned long long* __restrict__ ts, double vtol, PcgRhs ra,
                                                 PcgTail tl) {
    __shared__ PcgShared sh;
    extern __shared__ double Ks[];  // this CTA's columns of K (rb × n) when kstage
    // a programmatic dependent (the step's k_woodbury_st_pdl) may start staging its operands now;
    // it waits for this grid's completion before reading x
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const bool stamp = ts && blockIdx.x == 0 && threadIdx.x == 0;
    if (stamp) ts[0] = gtimer();
    cg::cluster_group cl = cg::this_cluster();
    const int crank = int(cl.block_rank());
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rb = (n + PC_CL - 1) / PC_CL;  // ≤ 64: owned rows live in warps 0–1
    const int r0 = min(n, crank * rb), r1 = min(n, r0 + rb);
    // Stage this CTA's K block (columns r0..r1, contiguous when ld == n): one TMA bulk copy
    // tracked by an mbarrier when 16-byte aligned, else 8-byte cp.async; it lands while the
    // initial residual is exchanged.
    __shared__ alignas(8) unsigned long long kbar;
    __shared__ alignas(8) unsigned long long xbar[2];  // per-parity exchange barriers
    const int cnt = kstage ? (r1 - r0) * n : 0;
    const unsigned bytes = unsigned(cnt) * 8u;
    const bool bulk = kstage && ld == n && ((long long)r0 * n) % 2 == 0 && bytes % 16 == 0 && bytes > 0;
    const unsigned kbar_a = static_cast<unsigned>(__cvta_generic_to_shared(&kbar));
    if (tid == 0) {
        for (int q = 0; q < 2; ++q) {
            const unsigned xa = static_cast<unsigned>(__cvta_generic_to_shared(&xbar[q]));
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(xa) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (bulk) {
        if (tid == 0) {
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(kbar_a) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(kbar_a), "r"(bytes) : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    static_cast<unsigned>(__cvta_generic_to_shared(Ks))),
                "l"(K + (long long)r0 * n), "r"(bytes), "r"(kbar_a)
                : "memory");
        }
    } else if (kstage) {
        for (int e = tid; e < cnt; e += PC_T) cp_async8(Ks + e, K + (long long)(r0 + e / n) * ld + e % n);
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    if constexpr (KR > 0)  // entries n..16·KR−1 of both exchange buffers multiply zero K entries
        for (int e = n + tid; e < 16 * KR; e += PC_T) sh.v[0][e] = sh.v[1][e] = 0.0;
    __syncthreads();  // mbarrier initialized before anyone waits on it
    __shared__ int spin_fail;
    if (ra.ready) {  // the producer of parts may still be running (K is staging meanwhile)
        if (tid == 0) {
            const double want = ra.alpha_dev[0] + 1.0;
            const unsigned long long t0 = gtimer();
            int fail = 0;
            while (*reinterpret_cast<const volatile double*>(ra.ready) != want) {
                if (gtimer() - t0 > ra.ready_timeout_ns) {
                    fail = 1;
                    break;
                }
                __nanosleep(64);
            }
            __threadfence();
            spin_fail = fail;
        }
        __syncthreads();
    }
    if (ra.E) fused_rhs(sh, ra, r0, r1);  // overlaps the K staging copy
    else if (ra.parts) parts_rhs(sh, ra, n, r0, r1);
    // Pipelined Jacobi-PCG (Ghysels–Vanroose): the matvec n = K·m and the reductions
    // γ = rᵀu, δ = wᵀu of the same iteration are independent, so one cluster exchange per
    // iteration carries both: owners push m into every CTA and every CTA pushes its
    // partials into every CTA (DSMEM stores), one cluster barrier, then each CTA sums the 16
    // slots in rank order (identical values everywhere → all CTAs branch alike) and
    // multiplies its own K rows locally.  Buffers alternate by parity, so a CTA that runs
    // ahead never overwrites data a peer is still reading.
    const int row = r0 + tid;
    const bool own = row < r1;
    double dinv = 0.0, x = 0.0, r = 0.0, uu = 0.0, w = 0.0, u0 = 0.0;
    double zv = 0.0, qv = 0.0, sv = 0.0, pv = 0.0;
    double nonpos = 0.0;  // K_ii ≤ 0: K (hence S) is not positive definite
    if (own) {
        const double kii = K[row + (long long)row * ld];
        nonpos = (kii > 0.0 && !(ra.cert && *ra.cert == 3)) ? 0.0 : 1.0;  // both Gershgorin tests failed
        if (ra.ready && spin_fail) nonpos = 1.0;  // the partials never arrived: give up (exact rerun)
        dinv = 1.0 / kii;
        if (ra.E || ra.parts) {
            r = sh.q[tid];
            u[row] = r;  // the Cholesky fallback's right-hand side
        } else {
            r = u[row];
        }
        u0 = r;
        uu = dinv * r;
#pragma unroll
        for (int c = 0; c < PC_CL; ++c) st_cluster(&sh.v[1][row], c, uu);
    }
    if (bulk) {
        unsigned ok = 0;
        while (!ok)
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(ok)
                : "r"(kbar_a)
                : "memory");
    } else if (kstage) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    cl.sync();  // u₀ exchanged; also orders every thread's staged K before the first matvec
    double kr[KR > 0 ? KR : 1];
    if constexpr (KR > 0) {
        const int sub = tid & 15, i = r0 + (tid >> 4);
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int j = sub + 16 * k;
            kr[k] = (i < r1 && j < n) ? Ks[(long long)(i - r0) * n + j] : 0.0;
        }
        block_matvec_reg<KR>(sh, kr, r0, r1, 1);  // w₀ = K u₀
    } else {
        block_matvec(sh, Ks, K, ld, n, r0, r1, 1, kstage);  // w₀ = K u₀
    }
    if (own) w = sh.q[tid];
    if (stamp) ts[1] = gtimer();
    double inv_gamma_prev = 1.0, inv_alpha_prev = 1.0, stop = 0.0;
    int it = 0;
    bool done = false;
    // exchange bytes every CTA receives per iteration: all n entries of m + 16×3 partials
    const unsigned xbytes = unsigned(n) * 8u + unsigned(PC_CL) * 32u;
    // Roles: the owner warp(s) (rows r0..r1 live in threads 0..rb−1) push m and the partials,
    // reduce the 16 slots and run the scalar recurrence; meanwhile every warp multiplies its
    // rows of K by m.  The owners' verdict (continue / converged / give up) reaches the other
    // warps through a per-parity shared flag published before the matvec's CTA barrier.
    const bool scal = warp < ((rb + 31) >> 5);
    __shared__ int xflag[2];
    double mv = 0.0, gamma = 0.0, alpha = 0.0, beta = 0.0;
    while (true) {
        const int buf = it & 1;
        const unsigned parity = unsigned((it >> 1) & 1);
        const unsigned xa = static_cast<unsigned>(__cvta_generic_to_shared(&xbar[buf]));
        if (stamp && it == 3) ts[39] = clock64();
        if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(xa), "r"(xbytes) : "memory");
        if (scal) {
            mv = dinv * w;
            if (own)  // the vector first: its stores overlap the partial-sum shuffles below
#pragma unroll
                for (int cc = 0; cc < PC_CL; ++cc) st_async_cluster(&sh.v[buf][row], &xbar[buf], cc, mv);
            double a = own ? r * uu : 0.0, bq = own ? w * uu : 0.0, c = own ? r * r : 0.0;
            double e = it == 0 ? nonpos : 0.0;
            for (int o = 16; o > 0; o >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, o);
                bq += __shfl_xor_sync(0xffffffffu, bq, o);
                c += __shfl_xor_sync(0xffffffffu, c, o);
                e += __shfl_xor_sync(0xffffffffu, e, o);
            }
            if (rb > 32) {  // two owner warps: combine through shared memory (named barrier)
                if (lane == 0) {
                    sh.red[warp][0] = a;
                    sh.red[warp][1] = bq;
                    sh.red[warp][2] = c;
                    sh.red[warp][3] = e;
                }
                asm volatile("bar.sync 1, 64;" ::: "memory");
                a = sh.red[0][0] + sh.red[1][0];
                bq = sh.red[0][1] + sh.red[1][1];
                c = sh.red[0][2] + sh.red[1][2];
                e = sh.red[0][3] + sh.red[1][3];
            }
            if (warp == 0 && lane < PC_CL) {  // lanes 0..15 push the sums to CTA `lane`
                st_async_cluster(&sh.part[buf][crank][0], &xbar[buf], lane, a);
                st_async_cluster(&sh.part[buf][crank][1], &xbar[buf], lane, bq);
                st_async_cluster(&sh.part[buf][crank][2], &xbar[buf], lane, c);
                st_async_cluster(&sh.part[buf][crank][3], &xbar[buf], lane, e);
            }
        }
        if (stamp && it == 3) ts[40] = clock64();
        {  // m and all partials delivered (this CTA's barrier of this parity)
            unsigned ok = 0;
            while (!ok)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                    : "=r"(ok)
                    : "r"(xa), "r"(parity)
                    : "memory");
        }
        if (stamp && it == 3) ts[41] = clock64();
        if (scal) {
            // lane-parallel sum of the 16 CTA slots (lane l reads slot l & 15, xor butterfly):
            // each add pairs the same two operands in every lane, warp and CTA (a + b = b + a
            // exactly), so all CTAs hold bit-identical scalars and decide alike
            const double* ps = sh.part[buf][lane & 15];
            double g = ps[0], dl = ps[1], rr = ps[2], bad = ps[3];
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) {
                g += __shfl_xor_sync(0xffffffffu, g, o);
                dl += __shfl_xor_sync(0xffffffffu, dl, o);
                rr += __shfl_xor_sync(0xffffffffu, rr, o);
                bad += __shfl_xor_sync(0xffffffffu, bad, o);
            }
            if (stamp && it == 3) ts[45] = clock64();
            int fl = 0;
            // a non-positive pivot means K (hence S) is not SPD: leave it to the Cholesky,
            // which reports "singular" exactly like the reference LLT (fast_filter.hpp:104-106)
            if (bad > 0.0) {
                fl = 2;
            } else {
                if (it == 0) stop = tol * tol * rr;  // r₀ = u
                if (rr <= stop || rr == 0.0) fl = 1;
                else if (it >= maxit) fl = 2;
            }
            if (fl == 0) {
                // 1/γ_prev and 1/α_prev were formed last iteration: one division here
                gamma = g;
                beta = it == 0 ? 0.0 : g * inv_gamma_prev;
                const double eta = it == 0 ? dl : dl - beta * g * inv_alpha_prev;  // = pᵀKp
                if (!(eta > 0.0)) fl = 2;  // non-positive curvature: not SPD (or breakdown)
                else alpha = g / eta;
            }
            if (stamp && it == 3) ts[46] = clock64();
            if (tid == 0) xflag[buf] = fl;
        }
        if (stamp && it == 3) ts[42] = clock64();
        if constexpr (KR > 0) block_matvec_reg<KR>(sh, kr, r0, r1, buf);  // n = K m (ends in a CTA barrier)
        else block_matvec(sh, Ks, K, ld, n, r0, r1, buf, kstage);
        if (stamp && it == 3) ts[43] = clock64();
        const int fl = xflag[buf];
        if (fl) {
            done = fl == 1;
            break;
        }
        if (scal) {
            if (own) {
                const double nv = sh.q[tid];
                zv = fma(beta, zv, nv);
                qv = fma(beta, qv, mv);
                sv = fma(beta, sv, w);
                pv = fma(beta, pv, uu);
                x = fma(alpha, pv, x);
                r = fma(-alpha, sv, r);
                uu = fma(-alpha, qv, uu);
                w = fma(-alpha, zv, w);
            }
            inv_gamma_prev = 1.0 / gamma;
            inv_alpha_prev = 1.0 / alpha;
        }
        ++it;
        if (stamp && it < 60) ts[1 + it] = gtimer();
        if (stamp && it == 4) ts[44] = clock64();
    }
    // True-residual check: the pipelined recursion for r can drift from u − Kx, so a converged
    // x is exchanged once more, multiplied by this CTA's K rows, and ‖u − Kx‖² and ‖u‖² are
    // summed in rank order (two more exchanges on the same parity sequence: iterations it+1 and
    // it+2).  A miss beyond vtol·‖u‖ hands the solve to the exact Cholesky.
    if (done && it > 0 && vtol > 0.0) {
        {
            const int b1 = (it + 1) & 1;
            const unsigned par1 = unsigned(((it + 1) >> 1) & 1);
            const unsigned xa = static_cast<unsigned>(__cvta_generic_to_shared(&xbar[b1]));
            if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(xa), "r"(unsigned(n) * 8u) : "memory");
            if (own)
#pragma unroll
                for (int cc = 0; cc < PC_CL; ++cc) st_async_cluster(&sh.v[b1][row], &xbar[b1], cc, x);
            unsigned ok = 0;
            while (!ok)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                    : "=r"(ok)
                    : "r"(xa), "r"(par1)
                    : "memory");
            if constexpr (KR > 0) block_matvec_reg<KR>(sh, kr, r0, r1, b1);  // q = K x (CTA barrier)
            else block_matvec(sh, Ks, K, ld, n, r0, r1, b1, kstage);
        }
        const int b2 = (it + 2) & 1;
        const unsigned par2 = unsigned(((it + 2) >> 1) & 1);
        const unsigned xa = static_cast<unsigned>(__cvta_generic_to_shared(&xbar[b2]));
        if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(xa), "r"(unsigned(PC_CL) * 16u) : "memory");
        if (scal) {
            const double e = own ? u0 - sh.q[tid] : 0.0;
            double a = e * e, c = own ? u0 * u0 : 0.0;
            for (int o = 16; o > 0; o >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, o);
                c += __shfl_xor_sync(0xffffffffu, c, o);
            }
            if (rb > 32) {
                if (lane == 0) {
                    sh.red[warp][0] = a;
                    sh.red[warp][2] = c;
                }
                asm volatile("bar.sync 1, 64;" ::: "memory");
                a = sh.red[0][0] + sh.red[1][0];
                c = sh.red[0][2] + sh.red[1][2];
            }
            if (warp == 0 && lane < PC_CL) {
                st_async_cluster(&sh.part[b2][crank][0], &xbar[b2], lane, a);
                st_async_cluster(&sh.part[b2][crank][2], &xbar[b2], lane, c);
            }
        }
        {
            unsigned ok = 0;
            while (!ok)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                    : "=r"(ok)
                    : "r"(xa), "r"(par2)
                    : "memory");
        }
        if (scal) {
            const double* ps = sh.part[b2][lane & 15];
            double e2 = ps[0], u2 = ps[2];
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) {
                e2 += __shfl_xor_sync(0xffffffffu, e2, o);
                u2 += __shfl_xor_sync(0xffffffffu, u2, o);
            }
            if (tid == 0) xflag[b2] = (e2 <= vtol * vtol * u2) ? 1 : 2;
        }
        __syncthreads();
        done = xflag[b2] == 1;
        if (crank == 0 && tid == 0 && !done) work[n + 1] = 1.0;  // diagnostics: the check failed
    }
    cl.sync();  // no CTA exits while a peer's asynchronous stores may still target it
    if (done) {
        if (own) u[row] = x;
    } else if (crank == 0 && tid == 0) {
        *fallback = 1;
        if (tl.st || tl.retry_only) atomicCAS(tl.info, 0, kInfoRetry);
    }
    // Woodbury tail: the residual check left x (all n entries) in sh.v[(it + 1) & 1] of every
    // CTA; it == 0 means u = 0, x = 0.  *info is uniform here (set only by earlier kernels).
    if (tl.st && done && *reinterpret_cast<volatile int*>(tl.info) == 0) {
        const int xb = (it + 1) & 1;
        woodbury_tail(tl, sh.v[xb], sh.v[xb ^ 1], n, crank, own, row, x, it == 0);
    }
    if (crank == 0 && tid == 0) work[n] = double(it);  // iteration count (diagnostics)
    if (stamp) ts[63] = gtimer();
}

static bool g_pcg_attr = false;

void cap_pcg(int n, const double* K, long long ld, double* u, double* work, int* fallback, cudaStream_t s, int maxit,
             double tol, unsigned long long* ts, double vtol, PcgRhs rhs, PcgTail tail) {
    if (n <= 0) return;
    if (n > PC_MAXN) throw std::invalid_argument("cap_pcg: n exceeds 1024");
    if (tail.st && !(vtol > 0.0)) throw std::invalid_argument("cap_pcg: the Woodbury tail needs the residual check");
    const int rb = (n + PC_CL - 1) / PC_CL;
    const size_t stage = sizeof(double) * size_t(rb) * n;
    const int kstage = stage <= 190 * 1024 ? 1 : 0;  // K columns resident in shared memory
    if (!g_pcg_attr) {
        for (const void* fn : {(const void*)k_cap_pcg<0>, (const void*)k_cap_pcg<20>, (const void*)k_cap_pcg<32>}) {
            FKB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            FKB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 190 * 1024));
        }
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
    if (kstage && n <= 16 * 20)
        FKB_CUDA(cudaLaunchKernelEx(&cfg, k_cap_pcg<20>, K, ld, n, u, work, fallback, maxit, tol, kstage, ts, vtol, rhs, tail));
    else if (kstage && n <= 16 * 32)
        FKB_CUDA(cudaLaunchKernelEx(&cfg, k_cap_pcg<32>, K, ld, n, u, work, fallback, maxit, tol, kstage, ts, vtol, rhs, tail));
    else
        FKB_CUDA(cudaLaunchKernelEx(&cfg, k_cap_pcg<0>, K, ld, n, u, work, fallback, maxit, tol, kstage, ts, vtol, rhs, tail));
    count_launch();
}

}  // namespace fkb

// test hook: solve K x = b (host K column-major, n ≤ 1024); iteration count and %globaltimer
// stamps (ns; [0] start, [1] K staged, [1+it] per iteration, [63] end) returned.
extern "C" int fkb_cap_pcg_test(int n, const double* K, const double* b, double* x, int* iters,
                                unsigned long long* stamps) {
    try {
        fkb::DBuf<double> dK(static_cast<size_t>(n) * n), du(static_cast<size_t>(n)), w(static_cast<size_t>(n) + 2);
        fkb::DBuf<int> fb(1);
        fkb::DBuf<unsigned long long> ts(64);
        FKB_CUDA(cudaMemcpy(dK.p, K, sizeof(double) * size_t(n) * n, cudaMemcpyHostToDevice));
        FKB_CUDA(cudaMemcpy(du.p, b, sizeof(double) * size_t(n), cudaMemcpyHostToDevice));
        FKB_CUDA(cudaMemset(fb.p, 0, sizeof(int)));
        FKB_CUDA(cudaMemset(ts.p, 0, ts.bytes()));
        fkb::cap_pcg(n, dK.p, n, du.p, w.p, fb.p, nullptr, 200, 1e-14, stamps ? ts.p : nullptr, 1e-13);
        FKB_CUDA(cudaDeviceSynchronize());
        int h = 0;
        double itd = 0.0;
        FKB_CUDA(cudaMemcpy(&h, fb.p, sizeof(int), cudaMemcpyDeviceToHost));
        FKB_CUDA(cudaMemcpy(&itd, w.p + n, sizeof(double), cudaMemcpyDeviceToHost));
        if (iters) *iters = int(itd);
        if (x) FKB_CUDA(cudaMemcpy(x, du.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost));
        if (stamps) FKB_CUDA(cudaMemcpy(stamps, ts.p, ts.bytes(), cudaMemcpyDeviceToHost));
        return h ? 2 : 0;
    } catch (const std::exception&) {
        return 3;
    }
}
