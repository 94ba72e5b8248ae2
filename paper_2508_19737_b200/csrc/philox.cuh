// philox.cuh — counter-based Philox4x32-10 + Box-Muller for the random input
// Theta ~ N(0, 1/d) (Alg. 1 l.2).  The paper names
// no generator; reading A11 fixes this one (cuRAND-compatible stream
// layout).  Product code: independent of oracle/ (which re-implements the same
// published algorithm from its definition).
#pragma once
#include <stdint.h>

namespace igp {

struct U4 {
    uint32_t x, y, z, w;
};

// Philox4x32 with 10 rounds; round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
// c <- (hi1^c1^k0, lo1, hi0^c3^k1, lo0); key bumped by the Weyl constants.
__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// draws of block b of the (seed, sub) stream
__device__ __forceinline__ U4 philox_block(uint64_t seed, uint64_t sub, uint64_t b) {
    return philox4x32_10(U4{(uint32_t)b, (uint32_t)(b >> 32), (uint32_t)sub, (uint32_t)(sub >> 32)},
                         (uint32_t)seed, (uint32_t)(seed >> 32));
}

// Box-Muller in fp64: u = (re + 1/2) 2^-32, v = (ro + 1/2) 2^-32;
// n_even = sqrt(-2 ln u) sin(2 pi v), n_odd = sqrt(-2 ln u) cos(2 pi v)
__device__ __forceinline__ void box_muller64(uint32_t re, uint32_t ro, double& ne, double& no) {
    const double u = ((double)re + 0.5) * 2.3283064365386962890625e-10;
    const double v = ((double)ro + 0.5) * 2.3283064365386962890625e-10;
    const double R = sqrt(-2.0 * log(u));
    double sn, cs;
    sincospi(2.0 * v, &sn, &cs);
    ne = R * sn;
    no = R * cs;
}

}  // namespace igp
