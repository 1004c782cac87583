// fft_device.cuh — device-side FP64 Stockham FFT in shared memory (K1 core).
//
// Mixed-radix {16, 8, 4, 2, 3, 5, 7} self-sorting Stockham passes; each thread
// performs whole radix-R butterflies from registers, twiddles come from a
// per-length table tw[k] = exp(−2πi k/n) read through the read-only path.
#pragma once

#include "fft.cuh"

namespace fkb {

// defined here: this header is included by exactly one translation unit (cov.cu)
__constant__ OddRadixTables c_odd;

// W16^q for q in 0..7 (forward sign): cos(2πq/16), −sin(2πq/16)
__device__ __forceinline__ constexpr double w16c(int q) {
    return q == 0 ? 1.0
         : q == 1 ? 0.92387953251128674
         : q == 2 ? 0.70710678118654757
         : q == 3 ? 0.38268343236508978
         : q == 4 ? 0.0
         : q == 5 ? -0.38268343236508978
         : q == 6 ? -0.70710678118654757
                  : -0.92387953251128674;
}
__device__ __forceinline__ constexpr double w16s(int q) {
    return q == 0 ? 0.0
         : q == 1 ? 0.38268343236508978
         : q == 2 ? 0.70710678118654757
         : q == 3 ? 0.92387953251128674
         : q == 4 ? 1.0
         : q == 5 ? 0.92387953251128674
         : q == 6 ? 0.70710678118654757
                  : 0.38268343236508978;
}

// b · exp(SIGN·2πi q/16), q compile-time after unrolling
template <int SIGN>
__device__ __forceinline__ double2 tw16(double2 b, int q) {
    if (q == 0) return b;
    if (q == 4) return cmul_i<SIGN>(b);
    const double c = w16c(q), s = SIGN < 0 ? -w16s(q) : w16s(q);
    if (q == 2 || q == 6) {  // |c| = |s| = √2/2
        const double h = 0.70710678118654757;
        const double sc = (q == 2) ? 1.0 : -1.0;  // sign of c
        const double ss = s > 0 ? 1.0 : -1.0;
        // (bx + i by)(sc·h + i ss·h) = h·(sc·bx − ss·by) + i h·(ss·bx + sc·by)
        return make_double2(h * (sc * b.x - ss * b.y), h * (ss * b.x + sc * b.y));
    }
    return make_double2(fma(b.x, c, -b.y * s), fma(b.x, s, b.y * c));
}

template <int R>
__device__ __forceinline__ constexpr int brev(int i) {
    int r = 0;
    for (int b = 1; b < R; b <<= 1) {
        r = (r << 1) | (i & 1);
        i >>= 1;
    }
    return r;
}

template <int R, int SIGN>
__device__ __forceinline__ void dft_pow2(double2* v) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
        const int j = brev<R>(i);
        if (j > i) {
            const double2 t = v[i];
            v[i] = v[j];
            v[j] = t;
        }
    }
#pragma unroll
    for (int len = 2; len <= R; len <<= 1) {
#pragma unroll
        for (int i = 0; i < R; i += len) {
#pragma unroll
            for (int k = 0; k < len / 2; ++k) {
                const double2 a = v[i + k];
                const double2 b = tw16<SIGN>(v[i + k + len / 2], k * (16 / len));
                v[i + k] = cadd(a, b);
                v[i + k + len / 2] = csub(a, b);
            }
        }
    }
}

template <int R, int SIGN>
__device__ __forceinline__ void dft_odd(double2* v) {
    const double* cs = R == 3 ? c_odd.c3 : (R == 5 ? c_odd.c5 : c_odd.c7);
    const double* sn = R == 3 ? c_odd.s3 : (R == 5 ? c_odd.s5 : c_odd.s7);
    double2 out[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
        double2 acc = v[0];
#pragma unroll
        for (int r = 1; r < R; ++r) {
            const int idx = (r * q) % R;
            const double2 w = make_double2(cs[idx], SIGN < 0 ? -sn[idx] : sn[idx]);
            acc = cadd(acc, cmul(v[r], w));
        }
        out[q] = acc;
    }
#pragma unroll
    for (int q = 0; q < R; ++q) v[q] = out[q];
}

template <int R, int SIGN>
__device__ __forceinline__ void dft(double2* v) {
    if constexpr (R == 2 || R == 4 || R == 8 || R == 16)
        dft_pow2<R, SIGN>(v);
    else
        dft_odd<R, SIGN>(v);
}

// One Stockham pass over `batch` contiguous transforms of length L.n.
template <int R, int SIGN>
__device__ __forceinline__ void stockham_pass(const double2* __restrict__ in, double2* __restrict__ out,
                                              const FftLen& L, int batch, int Ns) {
    const int n = L.n, nb = n / R, total = nb * batch;
    const int tws = n / (Ns * R);
    for (int w = threadIdx.x; w < total; w += blockDim.x) {
        const int t = w / nb, j = w - t * nb;
        const double2* src = in + t * n;
        double2* dst = out + t * n;
        const int k = j % Ns;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = src[j + r * nb];
        if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                double2 tw = __ldg(L.tw + r * k * tws);
                if (SIGN > 0) tw.y = -tw.y;
                v[r] = cmul(v[r], tw);
            }
        }
        dft<R, SIGN>(v);
        const int d = (j / Ns) * Ns * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[d + r * Ns] = v[r];
    }
}

// Transforms `batch` contiguous length-L.n sequences held in `a` (scratch `b`).
// Returns the buffer holding the result.  Caller must __syncthreads() before.
template <int SIGN>
__device__ double2* fft_smem(double2* a, double2* b, const FftLen& L, int batch) {
    double2* in = a;
    double2* out = b;
    int Ns = 1;
    for (int p = 0; p < L.npass; ++p) {
        const int R = L.radix[p];
        switch (R) {
            case 16: stockham_pass<16, SIGN>(in, out, L, batch, Ns); break;
            case 8: stockham_pass<8, SIGN>(in, out, L, batch, Ns); break;
            case 4: stockham_pass<4, SIGN>(in, out, L, batch, Ns); break;
            case 2: stockham_pass<2, SIGN>(in, out, L, batch, Ns); break;
            case 3: stockham_pass<3, SIGN>(in, out, L, batch, Ns); break;
            case 5: stockham_pass<5, SIGN>(in, out, L, batch, Ns); break;
            default: stockham_pass<7, SIGN>(in, out, L, batch, Ns); break;
        }
        __syncthreads();
        double2* t = in;
        in = out;
        out = t;
        Ns *= R;
    }
    return in;
}

// Generic-thread-range Stockham pass (same arithmetic as stockham_pass): threads t0, t0+nt, …
// of the caller cover the butterflies of ONE transform; twiddles from `tw` (shared memory).
template <int R, int SIGN>
__device__ __forceinline__ void stockham_pass_r(const double2* __restrict__ in, double2* __restrict__ out, int n,
                                                const double2* __restrict__ tw, int Ns, int t0, int nt) {
    const int nb = n / R;
    const int tws = n / (Ns * R);
    for (int j = t0; j < nb; j += nt) {
        const int k = j % Ns;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = in[j + r * nb];
        if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                double2 w = tw[r * k * tws];
                if (SIGN > 0) w.y = -w.y;
                v[r] = cmul(v[r], w);
            }
        }
        dft<R, SIGN>(v);
        const int d = (j / Ns) * Ns * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) out[d + r * Ns] = v[r];
    }
}

// One transform of length L.n per CTA (all blockDim.x threads), twiddle table in shared
// memory.  Returns the result buffer.  Caller must __syncthreads() after filling a and tw.
template <int SIGN>
__device__ double2* fft_block(double2* a, double2* b, const FftLen& L, const double2* tw) {
    double2* in = a;
    double2* out = b;
    int Ns = 1;
    for (int p = 0; p < L.npass; ++p) {
        const int R = L.radix[p];
        switch (R) {
            case 16: stockham_pass_r<16, SIGN>(in, out, L.n, tw, Ns, threadIdx.x, blockDim.x); break;
            case 8: stockham_pass_r<8, SIGN>(in, out, L.n, tw, Ns, threadIdx.x, blockDim.x); break;
            case 4: stockham_pass_r<4, SIGN>(in, out, L.n, tw, Ns, threadIdx.x, blockDim.x); break;
            case 2: stockham_pass_r<2, SIGN>(in, out, L.n, tw, Ns, threadIdx.x, blockDim.x); break;
            case 3: stockham_pass_r<3, SIGN>(in, out, L.n, tw, Ns, threadIdx.x, blockDim.x); break;
            case 5: stockham_pass_r<5, SIGN>(in, out, L.n, tw, Ns, threadIdx.x, blockDim.x); break;
            default: stockham_pass_r<7, SIGN>(in, out, L.n, tw, Ns, threadIdx.x, blockDim.x); break;
        }
        __syncthreads();
        double2* t = in;
        in = out;
        out = t;
        Ns *= R;
    }
    return in;
}

// ---- compile-time schedules for power-of-two lengths (single-vector kernels): radix-8
// passes then one radix-2/4 pass; Ns, strides and index math fold to constants.
template <int R, int SIGN, int N, int NS>
__device__ __forceinline__ void stockham_pass_c(const double2* __restrict__ in, double2* __restrict__ out,
                                                const double2* __restrict__ tw) {
    constexpr int nb = N / R, tws = N / (NS * R);
    for (int j = threadIdx.x; j < nb; j += blockDim.x) {
        const int k = j % NS;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = in[j + r * nb];
        if constexpr (NS > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                double2 w = tw[r * k * tws];
                if (SIGN > 0) w.y = -w.y;
                v[r] = cmul(v[r], w);
            }
        }
        dft<R, SIGN>(v);
        const int d = (j / NS) * NS * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) out[d + r * NS] = v[r];
    }
}

template <int N>
constexpr int static_radix(int ns) {  // radix of the pass that starts at stride ns
    return (N / ns) % 8 == 0 ? 8 : N / ns;
}

// Returns the result buffer (a or b); caller __syncthreads() after filling a and tw.
template <int SIGN, int N, int NS = 1>
__device__ __forceinline__ double2* fft_block_c(double2* a, double2* b, const double2* tw) {
    if constexpr (NS >= N) {
        return a;
    } else {
        constexpr int R = static_radix<N>(NS);
        stockham_pass_c<R, SIGN, N, NS>(a, b, tw);
        __syncthreads();
        return fft_block_c<SIGN, N, NS * R>(b, a, tw);
    }
}

// ---- compile-time schedules on a PADDED shared layout (slot(e) = e + e/8): every radix-8
// pass's strided stores (stride 8·16 B at NS = 1) and loads become ≤ 4-way bank-conflict-free
// (the 16-byte minimum), and each pass reads its own r-major twiddle sub-table (consecutive
// k → consecutive banks).  Padded buffers hold n + n/8 + 1 entries.
__device__ __forceinline__ int fpad(int e) { return e + (e >> 3); }

template <int R, int SIGN, int N, int NS>
__device__ __forceinline__ void stockham_pass_p(const double2* __restrict__ in, double2* __restrict__ out,
                                                const double2* __restrict__ tp) {
    constexpr int nb = N / R;
    for (int j = threadIdx.x; j < nb; j += blockDim.x) {
        const int k = j % NS;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = in[fpad(j + r * nb)];
        if constexpr (NS > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                double2 w = tp[(r - 1) * NS + k];
                if (SIGN > 0) w.y = -w.y;
                v[r] = cmul(v[r], w);
            }
        }
        dft<R, SIGN>(v);
        const int d = (j / NS) * NS * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) out[fpad(d + r * NS)] = v[r];
    }
}

template <int SIGN, int N, int NS = 1, int OFF = 0>
__device__ __forceinline__ double2* fft_block_p(double2* a, double2* b, const double2* tp) {
    if constexpr (NS >= N) {
        return a;
    } else {
        constexpr int R = static_radix<N>(NS);
        stockham_pass_p<R, SIGN, N, NS>(a, b, tp + OFF);
        __syncthreads();
        return fft_block_p<SIGN, N, NS * R, OFF + (NS > 1 ? (R - 1) * NS : 0)>(b, a, tp);
    }
}

// ---- register-resident radix-8 FFT for N = 8^a with N/8 threads: thread j holds
// v[r] = x[j + r·N/8] on entry and X[j + r·N/8] on exit (the Stockham input and output
// orderings coincide for this mapping), so the first pass needs no shared-memory load and the
// last pass no store — a forward and an inverse transform chain through registers.  Passes
// exchange through two padded ping-pong buffers (one barrier each); twiddles as fft_block_p.
template <int N>
constexpr bool reg_fft_len() { return N == 512 || N == 1024 || N == 4096; }  // N/8 threads: ≥ 64

// N = 1024 = 2·8·8·8 with 128 threads, thread j holding v[r] = x[j + 128r]: a register
// radix-2 pass (its pairs (x[j'], x[j'+512]) are (v[q], v[q+4]) for j' = j + 128q), then three
// radix-8 Stockham passes with one exchange before each; the last pass leaves X[j + 128r] in
// v[r] like the 8^a kernel.  One twiddle per radix-8 pass from the base table
// tw[q] = exp(−2πi·q/1024) (k = j mod ns, angle k/(8·ns)), its powers by products.
template <int SIGN>
__device__ __forceinline__ void fft_reg1024(double2 (&v)[8], double2* bufA, double2* bufB, const double2* __restrict__ tw,
                                            int j) {
    constexpr int N = 1024, nb = N / 8;
    double2 w1s[3];
    w1s[0] = __ldg(tw + (j % 2) * (N / 16));
    w1s[1] = __ldg(tw + (j % 16) * (N / 128));
    w1s[2] = __ldg(tw + j % 128);
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // pass NS = 1, R = 2 (no twiddles)
        const double2 a = v[q], b = v[q + 4];
        v[q] = cadd(a, b);
        v[q + 4] = csub(a, b);
    }
    double2* buf = bufA;
    // three exchanges end on bufA, where a preceding transform of the same threads (the
    // column pass's forward before its inverse) made its last reads: wait for them
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // outputs y[2j' + t]
        const int jj = j + nb * q;
        buf[fpad(2 * jj)] = v[q];
        buf[fpad(2 * jj + 1)] = v[q + 4];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = buf[fpad(j + r * nb)];
    int ns = 2;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        {
            double2 w1 = w1s[p];
            if (SIGN > 0) w1.y = -w1.y;
            const double2 w2 = cmul(w1, w1), w3 = cmul(w2, w1), w4 = cmul(w2, w2);
            const double2 w5 = cmul(w4, w1), w6 = cmul(w3, w3), w7 = cmul(w6, w1);
            v[1] = cmul(v[1], w1);
            v[2] = cmul(v[2], w2);
            v[3] = cmul(v[3], w3);
            v[4] = cmul(v[4], w4);
            v[5] = cmul(v[5], w5);
            v[6] = cmul(v[6], w6);
            v[7] = cmul(v[7], w7);
        }
        dft<8, SIGN>(v);
        if (p < 2) {
            if (bufB) buf = (buf == bufA) ? bufB : bufA;
            else __syncthreads();  // single buffer: the previous loads are done
            const int k = j % ns, d = (j / ns) * ns * 8 + k;
#pragma unroll
            for (int r = 0; r < 8; ++r) buf[fpad(d + r * ns)] = v[r];
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 8; ++r) v[r] = buf[fpad(j + r * nb)];
            ns *= 8;
        }
    }
}

// j = index within the transform (0..N/8−1); several transforms may share a CTA (every
// thread of the CTA must call with the same N).  bufB == nullptr: one buffer per transform
// and a second barrier per exchange.
template <int SIGN, int N>
__device__ __forceinline__ void fft_reg(double2 (&v)[8], double2* bufA, double2* bufB, const double2* __restrict__ tp,
                                        int j, const double2* __restrict__ tw_base = nullptr) {
    static_assert(reg_fft_len<N>(), "fft_reg: N must be 1024 or a power of 8");
    if constexpr (N == 1024) {
        fft_reg1024<SIGN>(v, bufA, bufB, tw_base, j);
        return;
    }
    constexpr int nb = N / 8;
    constexpr int NX = N == 512 ? 2 : 3;  // exchanges (passes after the first)
    // each pass needs ONE twiddle per thread (w = ω^k₂, the rest are its powers): fetched from
    // the global per-pass table (L1-resident, 8 KB) before the first exchange — no shared-memory
    // staging or loads for twiddles
    double2 w1s[NX];
    {
        int off = 0, ns2 = 8;
#pragma unroll
        for (int p = 0; p < NX; ++p) {
            w1s[p] = __ldg(tp + off + j % ns2);
            off += 7 * ns2;
            ns2 *= 8;
        }
    }
    dft<8, SIGN>(v);  // pass NS = 1: no twiddles
    int pidx = 0;
    double2* buf = bufA;
#pragma unroll
    for (int ns = 1; ns < nb; ns *= 8) {
        if (!bufB && ns > 1) __syncthreads();  // single buffer: previous loads done
        {
            const int k = j % ns, d = (j / ns) * ns * 8 + k;
#pragma unroll
            for (int r = 0; r < 8; ++r) buf[fpad(d + r * ns)] = v[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = buf[fpad(j + r * nb)];
        {  // w^r from the pass's one twiddle: w² = w·w, w³ = w²·w, … (≤ 4 ulp)
            double2 w1 = w1s[pidx++];
            if (SIGN > 0) w1.y = -w1.y;
            const double2 w2 = cmul(w1, w1), w3 = cmul(w2, w1), w4 = cmul(w2, w2);
            const double2 w5 = cmul(w4, w1), w6 = cmul(w3, w3), w7 = cmul(w6, w1);
            v[1] = cmul(v[1], w1);
            v[2] = cmul(v[2], w2);
            v[3] = cmul(v[3], w3);
            v[4] = cmul(v[4], w4);
            v[5] = cmul(v[5], w5);
            v[6] = cmul(v[6], w6);
            v[7] = cmul(v[7], w7);
        }
        dft<8, SIGN>(v);
        if (bufB) buf = (buf == bufA) ? bufB : bufA;
    }
}

}  // namespace fkb
