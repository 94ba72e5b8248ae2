// gather_bench.cu — microbenchmark of random row-gather bandwidth on B200 (tooling, not product).
// For row size R (bytes) and footprint F (MB): M random row ids; each group of R/16
// lanes gathers one row with LDG.128 and accumulates. Reports gathered GB/s.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

template <int R, int MODE>
__global__ void __launch_bounds__(256) gather(const float4* __restrict__ y, const int* __restrict__ idx, long m,
                                              float* out) {
  constexpr int LPR = R / 16, G = 32 / LPR;
  const int lane = threadIdx.x & 31, q = lane % LPR, g = lane / LPR;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  uint64_t pol = 0;
  if (MODE == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  for (long e0 = warp * 32; e0 < m; e0 += nw * 32) {
    int jl = (e0 + lane < m) ? __ldg(idx + e0 + lane) : 0;
    float4 v[LPR];
#pragma unroll
    for (int t = 0; t < LPR; ++t) {
      int j = __shfl_sync(0xffffffffu, jl, t * G + g);
      const float4* p = y + (long)j * LPR + q;
      if (MODE == 0) v[t] = __ldg(p);
      else if (MODE == 1) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v[t].x), "=f"(v[t].y), "=f"(v[t].z), "=f"(v[t].w) : "l"(p));
      } else {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;" : "=f"(v[t].x), "=f"(v[t].y), "=f"(v[t].z), "=f"(v[t].w) : "l"(p), "l"(pol));
      }
    }
#pragma unroll
    for (int t = 0; t < LPR; ++t) { acc.x += v[t].x; acc.y += v[t].y; acc.z += v[t].z; acc.w += v[t].w; }
  }
  if (acc.x == 12345.f) out[0] = acc.y + acc.z + acc.w;
}

__global__ void fill_idx(int* idx, long m, long rows, unsigned seed) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < m; i += (long)gridDim.x * blockDim.x) {
    unsigned long x = (unsigned long)i * 0x9E3779B97F4A7C15ul + seed;
    x ^= x >> 33; x *= 0xff51afd7ed558ccdul; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ul; x ^= x >> 33;
    idx[i] = (int)(x % (unsigned long)rows);
  }
}

template <int R, int MODE>
float run(const float4* y, const int* idx, long m, float* out, int grid) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  gather<R, MODE><<<grid, 256>>>(y, idx, m, out);
  cudaEventRecord(a);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) gather<R, MODE><<<grid, 256>>>(y, idx, m, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char** argv) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("SMs %d L2 %d MB\n", sms, l2 >> 20);
  const long m = 40l << 20;  // 40M gathers
  int* idx; cudaMalloc(&idx, m * 4);
  float* out; cudaMalloc(&out, 4);
  const size_t maxF = 512ul << 20;
  float4* y; cudaMalloc(&y, maxF);
  cudaMemset(y, 0, maxF);
  const int fps[] = {8, 16, 32, 48, 64, 96, 128, 192, 256, 512};
  printf("mode R_bytes F_MB grid ms gatherGBps\n");
  for (int mode = 0; mode < 3; ++mode)
  for (int R : {16, 32, 64, 128, 256}) {
    for (int F : fps) {
      long rows = ((long)F << 20) / R;
      fill_idx<<<1024, 256>>>(idx, m, rows, 1u);
      for (int occ : {4, 8}) {
        int grid = sms * occ;
        float ms = 0;
#define CASE(RR) if (R == RR) { ms = mode == 0 ? run<RR, 0>(y, idx, m, out, grid) : mode == 1 ? run<RR, 1>(y, idx, m, out, grid) : run<RR, 2>(y, idx, m, out, grid); }
        CASE(16) CASE(32) CASE(64) CASE(128) CASE(256)
        printf("%d %d %d %d %.3f %.1f\n", mode, R, F, grid, ms, (double)m * R / ms / 1e6);
      }
    }
  }
  // streaming copy reference
  {
    size_t bytes = 256ul << 20; float4* a; float4* b; cudaMalloc(&a, bytes); cudaMalloc(&b, bytes);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaMemcpy(b, a, bytes, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0); for (int r = 0; r < 10; ++r) cudaMemcpy(b, a, bytes, cudaMemcpyDeviceToDevice); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 256MB: %.1f GB/s (r+w)\n", 2.0 * bytes * 10 / ms / 1e6);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
