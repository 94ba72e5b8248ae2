// dsmem_lab.cu — go / no-go for community-tiled staging of the filter step's gathers in
// distributed shared memory (tooling, not product).
//
// The question: can random 128-byte row gathers be served from a thread-block cluster's
// distributed shared memory (ld.shared::cluster) faster than from L2?  If a cluster of C CTAs
// held a community's y-slice, the in-community gathers (~71% at Headline) would come from
// DSMEM.  Measured here with the gather pattern of the filter step (a row = 8 lanes x 16 B,
// 8 independent gathers in flight per lane, random rows), rows drawn uniformly from:
//   local   : the CTA's own shared memory (cluster size 1)
//   dsmem C : the C CTAs' shared memory of the cluster (C = 2, 4, 8, 16), via mapa
//   global  : a global array of the same total size (L2-resident) and of 128 MB (L2-sized)
// Each configuration reports gathered GB/s over the whole GPU (148 SMs, one CTA per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lab/dsmem_lab tools/lab/dsmem_lab.cu
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#include <cstdint>
#include <cstdio>

namespace cg = cooperative_groups;

constexpr int kThreads = 512;
constexpr int kRowBytes = 128;
constexpr int kSmemBytes = 192 * 1024;  // per CTA
constexpr int kRowsPerCta = kSmemBytes / kRowBytes;
constexpr int kDepth = 8;  // gathers in flight per lane

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

__device__ __forceinline__ uint4 ld_dsmem(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared::cluster.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t map_rank(uint32_t local_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
    return r;
}

// MODE 0: shared memory of this CTA (C = 1) or of the cluster (C > 1)
template <int C>
__global__ void __launch_bounds__(kThreads, 1) gather_dsmem(int iters, uint32_t* sink) {
    extern __shared__ __align__(16) unsigned char tile[];
    for (int i = threadIdx.x; i < kSmemBytes / 4; i += kThreads) reinterpret_cast<uint32_t*>(tile)[i] = i * 2654435761u;
    cg::this_cluster().sync();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(tile);
    const int lane8 = threadIdx.x & 7;  // 8 lanes x 16 B = one 128-B row
    const uint32_t seed = (blockIdx.x * kThreads + threadIdx.x) >> 3;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint4 v[kDepth];
#pragma unroll
        for (int k = 0; k < kDepth; ++k) {
            const uint32_t h = hash32(seed * 7919u + (uint32_t)(it * kDepth + k));
            const uint32_t row = h % (uint32_t)(kRowsPerCta * C);
            const uint32_t local = base + (row % kRowsPerCta) * kRowBytes + lane8 * 16;
            const uint32_t addr = C == 1 ? local : map_rank(local, row / kRowsPerCta);
            if (C == 1) {
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "r"(addr));
            } else {
                v[k] = ld_dsmem(addr);
            }
        }
#pragma unroll
        for (int k = 0; k < kDepth; ++k) acc += v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    cg::this_cluster().sync();  // no CTA exits while others read its shared memory
    if (acc == 0x12345678u) sink[0] = acc;
}

// the same gathers from a global array of `rows` rows (LDG.128, L1 bypassed like the product's
// cross-community traffic would be from L2)
__global__ void __launch_bounds__(kThreads, 1) gather_global(const uint4* __restrict__ src, uint32_t rows, int iters,
                                                            uint32_t* sink) {
    const int lane8 = threadIdx.x & 7;
    const uint32_t seed = (blockIdx.x * kThreads + threadIdx.x) >> 3;
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
        uint4 v[kDepth];
#pragma unroll
        for (int k = 0; k < kDepth; ++k) {
            const uint32_t h = hash32(seed * 7919u + (uint32_t)(it * kDepth + k));
            const uint32_t row = h % rows;
            const uint4* p = src + (size_t)row * (kRowBytes / 16) + lane8;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(p));
        }
#pragma unroll
        for (int k = 0; k < kDepth; ++k) acc += v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

template <int C>
float run_dsmem(int sms, int iters, uint32_t* sink) {
    auto k = gather_dsmem<C>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    if (C > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    const int grid = sms / C * C;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, k, &cfg) != cudaSuccess || ncl == 0) {
        cudaGetLastError();
        printf("dsmem C=%-2d: not launchable (max active clusters %d)\n", C, ncl);
        return -1.f;
    }
    cfg.gridDim = dim3((ncl < grid / C ? ncl : grid / C) * C);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaLaunchKernelEx(&cfg, k, iters, sink);  // warm
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k, iters, sink);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)cfg.gridDim.x * kThreads / 8 * iters * kDepth * kRowBytes;
    printf("dsmem C=%-2d (%3u CTAs, %2d clusters x %d): %8.3f ms  %8.0f GB/s gathered  %s\n", C, cfg.gridDim.x,
           cfg.gridDim.x / C, C, ms, bytes / ms / 1e6, e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    return (float)(bytes / ms / 1e6);
}

void run_global(int sms, uint32_t rows, int iters, uint32_t* sink, const char* what) {
    uint4* src = nullptr;
    cudaMalloc(&src, (size_t)rows * kRowBytes);
    cudaMemset(src, 1, (size_t)rows * kRowBytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather_global<<<sms, kThreads>>>(src, rows, iters, sink);
    cudaEventRecord(a);
    gather_global<<<sms, kThreads>>>(src, rows, iters, sink);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)sms * kThreads / 8 * iters * kDepth * kRowBytes;
    printf("global %-28s: %8.3f ms  %8.0f GB/s gathered  %s\n", what, ms, bytes / ms / 1e6,
           e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    cudaFree(src);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* sink = nullptr;
    cudaMalloc(&sink, 64);
    const int iters = 2000;
    printf("random 128-B row gathers, 8 lanes x 16 B per row, %d gathers in flight per lane, 512 threads/CTA, "
           "%d KB shared memory per CTA, %d SMs\n", kDepth, kSmemBytes / 1024, sms);
    run_dsmem<1>(sms, iters, sink);
    run_dsmem<2>(sms, iters, sink);
    run_dsmem<4>(sms, iters, sink);
    run_dsmem<8>(sms, iters, sink);
    run_dsmem<16>(sms, iters, sink);
    run_global(sms, (uint32_t)(16 * kRowsPerCta), iters, sink, "(3 MB: one 16-CTA cluster's tile)");
    run_global(sms, (uint32_t)(128u << 20) / kRowBytes, iters, sink, "(128 MB: an L2-sized slice)");
    run_global(sms, (uint32_t)(1024u << 20) / kRowBytes, iters, sink, "(1 GB: beyond L2)");
    return 0;
}
