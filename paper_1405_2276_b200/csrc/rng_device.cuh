// rng_device.cuh — counter-addressed restatement of the reference RNG (K3 core).
//
// Reference: rng.hpp:12-86.  Rng(seed, stream) starts at state0 = derive_seed(seed,
// stream); call t (1-based) returns mix(state0 + t·γ).  normal() is Box–Muller over
// calls (2p+1, 2p+2) and yields rad·cos for normal 2p, then the spare rad·sin for 2p+1.
// Integer parts are bit-exact; log/sqrt/sin/cos are CUDA libdevice (≤ 2 ulp).
#pragma once

#include <cstdint>

namespace fkb {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) { return mix64(x + kGolden); }
inline uint64_t derive_seed_host(uint64_t seed, uint64_t tag) { return splitmix64(seed ^ splitmix64(tag)); }

__device__ __forceinline__ double rng_uniform_call(uint64_t state0, uint64_t t) {
    return (double(mix64(state0 + t * kGolden) >> 11) + 0.5) * 0x1.0p-53;
}
// Both normals of Box–Muller pair p: (cos branch = normal 2p, sin branch = normal 2p+1).
__device__ __forceinline__ void rng_normal_pair(uint64_t state0, uint64_t p, double& c, double& s) {
    const double u1 = rng_uniform_call(state0, 2 * p + 1);
    const double u2 = rng_uniform_call(state0, 2 * p + 2);
    const double rad = sqrt(-2.0 * log(u1));
    const double ang = 6.283185307179586 * u2;  // 2.0 * std::numbers::pi, rounded once
    double sn, cs;
    sincos(ang, &sn, &cs);
    c = rad * cs;
    s = rad * sn;
}
__device__ __forceinline__ double rng_normal_at(uint64_t state0, uint64_t idx) {
    double c, s;
    rng_normal_pair(state0, idx >> 1, c, s);
    return (idx & 1) ? s : c;
}

}  // namespace fkb
