// store_lab.cu — where does the filter step's own-row read + output store cost go? (tooling, not product)
// A flat (segment-free) 8-deep gather over the CSR column stream of the headline graph, W = 32
// (128-B rows, 4 lanes per row, 16 warps per SM as in layer_kernel), plus the epilogue's streaming
// traffic in variants that separate its two possible costs:
//   L2 pollution : the 128 MB output slice written through L2 beside the 128 MB gathered slice;
//   latency stall: the own-row load issued after the gathers, the warp then having none in flight.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/lab/store_lab tools/lab/store_lab.cu
//   tools/lab/store_lab /tmp/lab.rp /tmp/lab.ci N nnz
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int W = 32, LPR = 4, G = 8, NV = 4, BATCH = 8, PER = G * BATCH;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void ldg256(const void* p, uint64_t (&v)[4]) {
  asm volatile("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}
__device__ __forceinline__ void stg256(void* p, const uint64_t (&v)[4], uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.b64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "l"(v[0]), "l"(v[1]), "l"(v[2]),
               "l"(v[3]), "l"(pol)
               : "memory");
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// MODE: 0 gathers only; 1 + own read (after the gathers) + store, full N x W buffers;
// 2 + store only (full buffer); 3 + own read + store into a 4 MB wrap-around window (no pollution);
// 4 = 1 with the own read issued one event ahead (no stall); 5 = 1 with evict_first stores;
// 6 = 4 with evict_first stores.  One own/store row event per group every 5 warp iterations
// (~40 gathers per row, the headline's mean degree).
template <int MODE>
__global__ void __launch_bounds__(256, 2) flat_rw(const int* __restrict__ rp, const int* __restrict__ ci,
                                                   const float* __restrict__ yin, float* __restrict__ yout,
                                                   const float* __restrict__ own_src, int n) {
  const int lane = threadIdx.x & 31, q = lane % LPR, g = lane / LPR;
  const long nnz = rp[n];
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  const uint64_t* S = reinterpret_cast<const uint64_t*>(own_src);
  uint64_t* O = reinterpret_cast<uint64_t*>(yout);
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  uint64_t pol;
  if (MODE == 5 || MODE == 6)
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  uint64_t acc[NV] = {};
  uint64_t own[NV] = {};
  long ev = 0;  // own/store events of this warp
  auto row_of = [&](long k) -> long {
    long r = (warp + k * nw) * G + g;
    if (MODE == 3) r &= 32767;  // 32768 rows x 128 B = 4 MB window
    return r;
  };
  if (MODE == 4 || MODE == 6) {
    const long r = row_of(0);
    if (r < n) ldg256(S + ((size_t)r * LPR + q) * NV, own);
  }
  int it = 0;
  for (long e0 = warp * PER; e0 < nnz; e0 += nw * PER) {
    const int jl = (e0 + lane < nnz) ? __ldg(ci + e0 + lane) : 0;
    const int jh = (e0 + 32 + lane < nnz) ? __ldg(ci + e0 + 32 + lane) : 0;
    uint64_t v[BATCH][NV];
#pragma unroll
    for (int t = 0; t < BATCH; ++t) {
      const int src = t * G + g;
      const int j = __shfl_sync(kFull, src < 32 ? jl : jh, src & 31);
      ldg256(Y + ((size_t)j * LPR + q) * NV, v[t]);
    }
#pragma unroll
    for (int t = 0; t < BATCH; ++t)
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] = fadd2(acc[k], v[t][k]);
    if (MODE != 0 && ++it == 5) {
      it = 0;
      const long r = row_of(ev);
      if (r < n) {
        uint64_t o[NV];
        if (MODE == 1 || MODE == 3 || MODE == 5) ldg256(S + ((size_t)r * LPR + q) * NV, own);
#pragma unroll
        for (int k = 0; k < NV; ++k) o[k] = MODE == 2 ? acc[k] : fadd2(own[k], acc[k]);
        stg256(O + ((size_t)r * LPR + q) * NV, o, pol);
      }
      ++ev;
      if (MODE == 4 || MODE == 6) {
        const long r2 = row_of(ev);
        if (r2 < n) ldg256(S + ((size_t)r2 * LPR + q) * NV, own);
      }
    }
  }
  if (MODE == 0) {
    float x = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) x += __uint_as_float((uint32_t)acc[k]);
    if (x == 1234.5f) yout[0] = x;
  }
}

template <typename K>
float timeit(K kern, int grid, const int* rp, const int* ci, float* y0, float* y1, int n, int reps, int* regs) {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  *regs = fa.numRegs;
  kern<<<grid, 256>>>(rp, ci, y0, y1, y0, n);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  // ping-pong like the product: the buffer written by one launch is gathered (and own-read) by the next
  for (int r = 0; r < reps; ++r) {
    float* in = (r & 1) ? y1 : y0;
    float* out = (r & 1) ? y0 : y1;
    kern<<<grid, 256>>>(rp, ci, in, out, in, n);
  }
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: store_lab rp ci N nnz\n");
    return 2;
  }
  const int n = atoi(argv[3]);
  const long nnz = atol(argv[4]);
  std::vector<int> hrp(n + 1), hci(nnz + 64, 0);
  FILE* f = fopen(argv[1], "rb");
  if (!f || fread(hrp.data(), 4, n + 1, f) != (size_t)n + 1) return 3;
  fclose(f);
  f = fopen(argv[2], "rb");
  if (!f || fread(hci.data(), 4, nnz, f) != (size_t)nnz) return 3;
  fclose(f);
  int *rp, *ci;
  float *y0, *y1;
  cudaMalloc(&rp, 4 * (n + 1));
  cudaMalloc(&ci, 4 * (nnz + 64));
  cudaMalloc(&y0, 4l * n * W);
  cudaMalloc(&y1, 4l * n * W);
  cudaMemcpy(rp, hrp.data(), 4 * (n + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(ci, hci.data(), 4 * (nnz + 64), cudaMemcpyHostToDevice);
  {
    std::vector<float> hy((size_t)n * W);
    for (size_t k = 0; k < hy.size(); ++k) hy[k] = (float)((k * 2654435761u) % 1000) * 1e-6f;
    cudaMemcpy(y0, hy.data(), 4l * n * W, cudaMemcpyHostToDevice);
    cudaMemcpy(y1, hy.data(), 4l * n * W, cudaMemcpyHostToDevice);
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double gbytes = 4.0 * W * nnz / 1e9;
  const int reps = 20;
#define RUN(NAME, KERN)                                                                                       \
  {                                                                                                           \
    int regs = 0;                                                                                             \
    float ms = timeit(KERN, sms * 2, rp, ci, y0, y1, n, reps, &regs);                                         \
    printf("%-58s regs %3d: %8.1f us  gather %7.0f GB/s  %s\n", NAME, regs, ms * 1e3, gbytes / ms * 1e3,      \
           cudaGetErrorString(cudaGetLastError()));                                                           \
  }
  RUN("0 flat gathers only", flat_rw<0>);
  RUN("1 + own read after gathers + store (full buffers)", flat_rw<1>);
  RUN("2 + store only (full buffer)", flat_rw<2>);
  RUN("3 + own read + store in a 4 MB window (no pollution)", flat_rw<3>);
  RUN("4 + own read one event ahead + store (no stall)", flat_rw<4>);
  RUN("5 = 1 with evict_first stores", flat_rw<5>);
  RUN("6 = 4 with evict_first stores", flat_rw<6>);
  RUN("0 flat gathers only (again)", flat_rw<0>);
  return 0;
}
