// Test-only library pin: cuRAND's own Philox4_32_10 device-API code, compiled
// for the HOST (QUALIFIERS redefined), so the CPU test suite can pin the
// oracle's Philox and Box-Muller against a library routine without a GPU.
// Shares nothing with oracle/ or the product path; only tests/ load it.
#define QUALIFIERS static inline __host__ __device__
#include <curand_kernel.h>
#include <stdint.h>

extern "C" {

// curand_init(seed, subsequence, offset) then n4 calls to curand4 -> out[4*n4]
void pin_curand4(uint64_t seed, uint64_t subsequence, uint64_t offset, int64_t n4, uint32_t* out) {
    curandStatePhilox4_32_10_t s;
    curand_init(seed, subsequence, offset, &s);
    for (int64_t k = 0; k < n4; ++k) {
        uint4 r = curand4(&s);
        out[4 * k + 0] = r.x; out[4 * k + 1] = r.y; out[4 * k + 2] = r.z; out[4 * k + 3] = r.w;
    }
}

// the raw block function curand_Philox4x32_10(counter, key)
void pin_philox_block(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
    uint4 c = make_uint4(ctr[0], ctr[1], ctr[2], ctr[3]);
    uint2 k = make_uint2(key[0], key[1]);
    uint4 r = curand_Philox4x32_10(c, k);
    out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
}

// curand_init(seed, subsequence, offset) then n4 calls to curand_normal4 (host: float libm)
void pin_curand_normal4(uint64_t seed, uint64_t subsequence, uint64_t offset, int64_t n4, float* out) {
    curandStatePhilox4_32_10_t s;
    curand_init(seed, subsequence, offset, &s);
    for (int64_t k = 0; k < n4; ++k) {
        float4 r = curand_normal4(&s);
        out[4 * k + 0] = r.x; out[4 * k + 1] = r.y; out[4 * k + 2] = r.z; out[4 * k + 3] = r.w;
    }
}

}
