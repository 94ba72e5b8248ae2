// philox.cu — standalone random-stream entry points (igp_philox_bits / igp_philox_normal),
// used by the parity tests to pin the generator bit-exactly; the embed path
// draws the same stream inside its input kernel (embed.cu).
#include "igp_internal.cuh"
#include "philox.cuh"

namespace igp {
namespace {

__global__ void philox_bits_kernel(uint64_t seed, uint64_t sub, int64_t count, uint32_t* __restrict__ out) {
    const int64_t nb = (count + 3) / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += stride) {
        const U4 r = philox_block(seed, sub, (uint64_t)b);
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (4 * b + q < count) out[4 * b + q] = w[q];
    }
}

__global__ void philox_normal_kernel(uint64_t seed, uint64_t sub, int64_t count, float4* __restrict__ out) {
    const int64_t nb = count / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += stride) {
        const U4 r = philox_block(seed, sub, (uint64_t)b);
        double n0, n1, n2, n3;
        box_muller64(r.x, r.y, n0, n1);
        box_muller64(r.z, r.w, n2, n3);
        out[b] = make_float4((float)n0, (float)n1, (float)n2, (float)n3);
    }
}

int blocks_for(int64_t items, int threads) {
    DeviceInfo di;
    device_info(&di);
    int64_t g = (items + threads - 1) / threads;
    int64_t cap = (int64_t)(di.num_sms > 0 ? di.num_sms : 148) * 8;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

igp_status launch_philox_bits(uint64_t seed, uint64_t sub, int64_t count, uint32_t* out, cudaStream_t s) {
    if (count <= 0) return IGP_OK;
    philox_bits_kernel<<<blocks_for((count + 3) / 4, 256), 256, 0, s>>>(seed, sub, count, out);
    return launch_status("philox_bits_kernel");
}

igp_status launch_philox_normal(uint64_t seed, uint64_t sub, int64_t count, float* out, cudaStream_t s) {
    if (count <= 0) return IGP_OK;
    philox_normal_kernel<<<blocks_for(count / 4, 256), 256, 0, s>>>(seed, sub, count, (float4*)out);
    return launch_status("philox_normal_kernel");
}

}  // namespace igp
