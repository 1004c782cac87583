// fft.cuh — FP64 shared-memory Stockham FFT building blocks (K1).
//
// Replaces FFTW's c2c execute calls in the reference's covariance operator
// (covariance.hpp:278-281, 303-306, 317, 322).  Convention is FFTW's:
// unnormalized, forward = exp(−2πi jk/n), backward = exp(+2πi jk/n).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace fkb {

constexpr int kMaxPasses = 12;

// One 1-D transform length: radix schedule + device twiddle table tw[k] = exp(−2πi k/n).
struct FftLen {
    int n = 0;
    int npass = 0;
    int radix[kMaxPasses] = {0};
    const double2* tw = nullptr;
    // compile-time-schedule twiddles (radix-8 passes, then one radix-2/4): for each pass that
    // starts at stride NS > 1, entries [(r−1)·NS + k] = exp(−2πi·r·k/(NS·R)), r = 1..R−1
    const double2* twp = nullptr;
};

// host/device: length of that table for a power-of-two n (0 for n ≤ 8)
constexpr int static_tw_len(int n) {
    int tot = 0, ns = 1;
    while (ns < n) {
        const int R = (n / ns) % 8 == 0 ? 8 : n / ns;
        if (ns > 1) tot += (R - 1) * ns;
        ns *= R;
    }
    return tot;
}

// constants for the generic odd radices 3, 5, 7: cos/sin(2π j/R), filled at init
struct OddRadixTables {
    double c3[3], s3[3], c5[5], s5[5], c7[7], s7[7];
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by −i (SIGN<0) or +i (SIGN>0)
template <int SIGN>
__device__ __forceinline__ double2 cmul_i(double2 a) {
    return SIGN < 0 ? make_double2(a.y, -a.x) : make_double2(-a.y, a.x);
}

}  // namespace fkb
