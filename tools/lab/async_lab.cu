// async_lab.cu — does moving the gathers' in-flight buffer from registers to shared memory
// (cp.async 16-byte LDGSTS into a per-warp ring) raise the segment-free gather ceiling on the real
// headline CSR?  Tooling, not product ("rejected variants").
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/lab/async_lab tools/lab/async_lab.cu
//   tools/lab/async_lab /tmp/labd.rp /tmp/labd.ci N nnz
// Every variant gathers the nnz rows (128 B: one W = 32 slice) named by the column stream in
// order and sums them per lane; the sums are checked against each other (same edges per lane
// position are not guaranteed, so only the grand total is compared, in fp64).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void ldg256(const void* p, uint64_t (&v)[4]) {
  asm volatile("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float2 unpack2(uint64_t v) {
  float2 f;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(f.x), "=f"(f.y) : "l"(v));
  return f;
}

// register baseline: 4 lanes x 32 B per row, BATCH gathers per lane in flight
template <int BATCH, int MINB>
__global__ void __launch_bounds__(256, MINB) flat_reg(const int* __restrict__ ci, long nnz, const float* __restrict__ y,
                                                      double* __restrict__ total) {
  constexpr int LPR = 4, G = 8, PER = G * BATCH;
  const int lane = threadIdx.x & 31, q = lane % LPR, g = lane / LPR;
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(y);
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  uint64_t acc[4] = {};
  for (long e0 = warp * PER; e0 < nnz; e0 += nw * PER) {
    const int jl = (lane < PER && e0 + lane < nnz) ? __ldg(ci + e0 + lane) : -1;
    uint64_t v[BATCH][4];
#pragma unroll
    for (int t = 0; t < BATCH; ++t) {
      const int j = __shfl_sync(kFull, jl, (t * G + g) & 31);
      ldg256(Y + ((size_t)(j < 0 ? 0 : j) * LPR + q) * 4, v[t]);  // tail slots read row 0 (ceiling only)
    }
#pragma unroll
    for (int t = 0; t < BATCH; ++t)
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = fadd2(acc[k], v[t][k]);
  }
  double x = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 f = unpack2(acc[k]);
    x += (double)f.x + (double)f.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(total, x);  // one atomic per warp
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// shared-memory ring: 8 lanes x 16 B per row (4 rows per instruction), U instructions per stage
// (4U gathers), S stages per warp; each lane reads back only the slots it filled itself.
template <int U, int S>
__global__ void __launch_bounds__(256) flat_async(const int* __restrict__ ci, long nnz, const float* __restrict__ y,
                                                  double* __restrict__ total) {
  constexpr int LPR = 8, G = 4, PER = G * U;
  static_assert(PER <= 32, "one index per lane per stage");
  extern __shared__ uint4 ring[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane % LPR, g = lane / LPR;
  uint4* my = ring + (size_t)warp * S * U * 32 + lane;
  const uint4* Y = reinterpret_cast<const uint4*>(y);
  const long gw = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  const long first = gw * PER, stride = nw * PER;
  const long count = first < nnz ? (nnz - first + stride - 1) / stride : 0;  // stages of this warp
  auto load_j = [&](long k) -> int {
    const long e = first + k * stride + lane;
    return (k < count && lane < PER && e < nnz) ? __ldg(ci + e) : -1;
  };
  auto issue = [&](int jl, int slot) {
#pragma unroll
    for (int t = 0; t < U; ++t) {
      const int j = __shfl_sync(kFull, jl, t * G + g);
      cp_async16(my + (slot * U + t) * 32, Y + ((size_t)(j < 0 ? 0 : j) * LPR + q), j < 0 ? 0 : 16);
    }
  };
  int jn = load_j(0);
#pragma unroll
  for (int k = 0; k < S - 1; ++k) {
    if (k < count) issue(jn, k);
    cp_commit();
    jn = load_j(k + 1);
  }
  uint64_t acc[2] = {};
  for (long k = 0; k < count; ++k) {
    const long kn = k + S - 1;
    if (kn < count) issue(jn, (int)(kn % S));
    cp_commit();
    jn = load_j(kn + 1);
    cp_wait<S - 1>();
    const int slot = (int)(k % S);
#pragma unroll
    for (int t = 0; t < U; ++t) {
      const uint4 v = my[(slot * U + t) * 32];
      acc[0] = fadd2(acc[0], (uint64_t)v.x | ((uint64_t)v.y << 32));
      acc[1] = fadd2(acc[1], (uint64_t)v.z | ((uint64_t)v.w << 32));
    }
  }
  cp_wait<0>();
  double x = 0.0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float2 f = unpack2(acc[k]);
    x += (double)f.x + (double)f.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(total, x);  // one atomic per warp
}

template <typename K>
float timeit(K kern, int grid, size_t smem, const int* ci, long nnz, const float* y, double* tot, int reps,
             double* sum) {
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaMemset(tot, 0, 8);
  kern<<<grid, 256, smem>>>(ci, nnz, y, tot);
  cudaMemcpy(sum, tot, 8, cudaMemcpyDeviceToHost);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) kern<<<grid, 256, smem>>>(ci, nnz, y, tot);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: async_lab rp ci N nnz\n");
    return 2;
  }
  const int n = atoi(argv[3]);
  const long nnz = atol(argv[4]);
  std::vector<int> hci(nnz);
  FILE* f = fopen(argv[2], "rb");
  if (!f || fread(hci.data(), 4, nnz, f) != (size_t)nnz) return 3;
  fclose(f);
  int* ci;
  float* y;
  double* tot;
  cudaMalloc(&ci, 4 * nnz);
  cudaMalloc(&y, 128l * n);
  cudaMalloc(&tot, 8);
  cudaMemcpy(ci, hci.data(), 4 * nnz, cudaMemcpyHostToDevice);
  {
    std::vector<float> hy((size_t)n * 32);
    for (size_t k = 0; k < hy.size(); ++k) hy[k] = (float)((k * 2654435761u) % 1000) * 1e-3f;  // >= 0
    cudaMemcpy(y, hy.data(), 128l * n, cudaMemcpyHostToDevice);
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double gbytes = 128.0 * nnz / 1e9;
  const int reps = 20;
  double ref = 0.0;
#define RUN(NAME, KERN, SMEM)                                                                                  \
  {                                                                                                            \
    int occ = 0;                                                                                               \
    if ((SMEM) > 48 * 1024) cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(SMEM)); \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, KERN, 256, SMEM);                                       \
    cudaFuncAttributes fa;                                                                                     \
    cudaFuncGetAttributes(&fa, KERN);                                                                          \
    double sum = 0.0;                                                                                          \
    float ms = timeit(KERN, sms * occ, SMEM, ci, nnz, y, tot, reps, &sum);                                     \
    if (ref == 0.0) ref = sum;                                                                                 \
    printf("%-34s regs %3d smem %6d occ %d: %8.1f us  gather %7.0f GB/s  rel.diff %.1e  %s\n", NAME, fa.numRegs, \
           (int)(SMEM), occ, ms * 1e3, gbytes / ms * 1e3, (sum - ref) / ref,                                   \
           cudaGetErrorString(cudaGetLastError()));                                                            \
  }
  RUN("reg B4 occ4", (flat_reg<4, 4>), 0);
  RUN("reg B8 occ2", (flat_reg<8, 2>), 0);
  RUN("reg B8 occ3", (flat_reg<8, 3>), 0);
  RUN("reg B2 occ4", (flat_reg<2, 4>), 0);
  RUN("reg B4 occ2", (flat_reg<4, 2>), 0);
  RUN("async U8 S2", (flat_async<8, 2>), 8 * 2 * 8 * 512);
  RUN("async U8 S3", (flat_async<8, 3>), 8 * 3 * 8 * 512);
  RUN("async U8 S4", (flat_async<8, 4>), 8 * 4 * 8 * 512);
  RUN("async U4 S4", (flat_async<4, 4>), 8 * 4 * 4 * 512);
  RUN("async U4 S6", (flat_async<4, 6>), 8 * 6 * 4 * 512);
  RUN("async U4 S8", (flat_async<4, 8>), 8 * 8 * 4 * 512);
  RUN("async U2 S8", (flat_async<2, 8>), 8 * 8 * 2 * 512);
  RUN("async U2 S12", (flat_async<2, 12>), 8 * 12 * 2 * 512);
  return 0;
}
