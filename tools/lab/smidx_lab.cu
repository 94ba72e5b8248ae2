// smidx_lab.cu — can the filter step's gather core hold 8-deep gather batches at more warps per SM
// if the neighbour-index chunks live in shared memory (cp.async, double-buffered) instead of
// registers?  Tooling, not product.  Same arithmetic as layer_lab's lab_pre:
// out_i = s_i tanh(0.1 y_i + s_i sum_j y_j) on a W = 32 slice, row batches of 8 rows per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/lab/smidx_lab tools/lab/smidx_lab.cu
//   tools/lab/smidx_lab /tmp/labd.rp /tmp/labd.ci N nnz
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int W = 32;
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
__device__ __forceinline__ uint64_t pack2(float a, float b) {
  uint64_t v;
  asm("mov.b64 %0, {%1,%2};" : "=l"(v) : "f"(a), "f"(b));
  return v;
}
__device__ __forceinline__ int4 ld_idx4(const int* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void load_idx4(const int* ci, int e0, int end, int q, int (&jr)[4]) {
  const int e = e0 + q * 4;
  if (e >= end) {
    jr[0] = jr[1] = jr[2] = jr[3] = 0;
    return;
  }
  const int4 v = ld_idx4(ci + e);
  jr[0] = v.x, jr[1] = v.y, jr[2] = v.z, jr[3] = v.w;
}

// epilogue shared by both variants
__device__ __forceinline__ void finish_row(const uint64_t* Y, uint64_t* O, const float* s, int row, int q,
                                           const uint64_t (&acc)[4]) {
  const float si = s[row];
  const uint64_t* op = Y + ((size_t)row * 4 + q) * 4;
  uint64_t own[4], o[4];
  ldg256(op, own);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 y = unpack2(own[k]);
    const float2 a = unpack2(acc[k]);
    o[k] = pack2(si * tanhf(0.1f * y.x + si * a.x), si * tanhf(0.1f * y.y + si * a.y));
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) O[((size_t)row * 4 + q) * 4 + k] = o[k];
}

// reference: indices in registers (the product's structure: next chunk and next batch's first chunk
// prefetched into registers, broadcast by shuffles)
template <int NW, int MB>
__global__ void __launch_bounds__(NW * 32, MB) reg_idx(const int* __restrict__ rp, const int* __restrict__ ci,
                                                       const float* __restrict__ s, const float* __restrict__ yin,
                                                       float* __restrict__ yout, int n) {
  constexpr int LPR = 4, G = 8, IPL = 4, NG = NW * G, B = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane % LPR, g = lane / LPR;
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  uint64_t* O = reinterpret_cast<uint64_t*>(yout);
  const long step = (long)gridDim.x * NG;
  long base = (long)blockIdx.x * NG + warp * G;
  int nbeg = 0, nend = 0, jfirst[IPL];
  if (base + g < n) nbeg = __ldg(rp + base + g), nend = __ldg(rp + base + g + 1);
  load_idx4(ci, nbeg & ~3, nend, q, jfirst);
  for (; base < n; base += step) {
    const int row = (int)(base + g);
    const int beg = nbeg, end = nend, start = beg & ~3;
    int jr[IPL];
#pragma unroll
    for (int k = 0; k < IPL; ++k) jr[k] = jfirst[k];
    nbeg = nend = 0;
    if (base + step + g < n) nbeg = __ldg(rp + base + step + g), nend = __ldg(rp + base + step + g + 1);
    uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
    const int nch = end > beg ? (end - start + 15) / 16 : 0;
    const int max_nch = __reduce_max_sync(kFull, nch);
    if (max_nch == 0) load_idx4(ci, nbeg & ~3, nend, q, jfirst);
    for (int c = 0; c < max_nch; ++c) {
      const int e0 = start + c * 16;
      int jn[IPL];
      load_idx4(ci, e0 + 16, end, q, jn);
      if (c == 0) load_idx4(ci, nbeg & ~3, nend, q, jfirst);
      const int lo = beg > e0 ? beg - e0 : 0;
      int hi = end - e0;
      hi = hi < 0 ? 0 : (hi > 16 ? 16 : hi);
      const bool full = __all_sync(kFull, lo == 0 && hi == 16);
#pragma unroll
      for (int u0 = 0; u0 < 16; u0 += B) {
        uint64_t v[B][4];
#pragma unroll
        for (int t = 0; t < B; ++t) {
          const int u = u0 + t;
          const int j = __shfl_sync(kFull, jr[u % IPL], u / IPL, LPR);
          if (full || (u >= lo && u < hi)) ldg256(Y + ((size_t)j * LPR + q) * 4, v[t]);
          else v[t][0] = v[t][1] = v[t][2] = v[t][3] = 0ull;
        }
#pragma unroll
        for (int t = 0; t < B; ++t)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[k] = fadd2(acc[k], v[t][k]);
      }
#pragma unroll
      for (int k = 0; k < IPL; ++k) jr[k] = jn[k];
    }
    if (row < n) finish_row(Y, O, s, row, q, acc);
  }
}

// indices in shared memory: each lane cp.async-copies its 4 indices (16 B) of the next chunk into
// the other half of a per-warp double buffer; gathers read j with a broadcast LDS.  The chunk after
// a batch's last chunk is the next batch's first chunk, so one copy group is always in flight.
template <int NW, int MB>
__global__ void __launch_bounds__(NW * 32, MB) sm_idx(const int* __restrict__ rp, const int* __restrict__ ci,
                                                      const float* __restrict__ s, const float* __restrict__ yin,
                                                      float* __restrict__ yout, int n) {
  constexpr int LPR = 4, G = 8, NG = NW * G, B = 8;
  __shared__ __align__(16) int sidx[NW][2][G][16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, q = lane % LPR, g = lane / LPR;
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  uint64_t* O = reinterpret_cast<uint64_t*>(yout);
  const long step = (long)gridDim.x * NG;
  long base = (long)blockIdx.x * NG + warp * G;
  int nbeg = 0, nend = 0;
  if (base + g < n) nbeg = __ldg(rp + base + g), nend = __ldg(rp + base + g + 1);
  int buf = 0;
  {
    const int e = (nbeg & ~3) + q * 4;
    cp_async16(&sidx[warp][0][g][q * 4], ci + (e < nend ? e : 0), e < nend ? 16 : 0);
    cp_commit();
  }
  for (; base < n; base += step) {
    const int row = (int)(base + g);
    const int beg = nbeg, end = nend, start = beg & ~3;
    nbeg = nend = 0;
    if (base + step + g < n) nbeg = __ldg(rp + base + step + g), nend = __ldg(rp + base + step + g + 1);
    uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
    const int nch = end > beg ? (end - start + 15) / 16 : 0;
    const int max_nch = __reduce_max_sync(kFull, nch);
    if (max_nch == 0) {  // nothing to gather: queue the next batch's first chunk
      const int e = (nbeg & ~3) + q * 4;
      cp_async16(&sidx[warp][buf ^ 1][g][q * 4], ci + (e < nend ? e : 0), e < nend ? 16 : 0);
      cp_commit();
      buf ^= 1;
    }
    for (int c = 0; c < max_nch; ++c) {
      const int e0 = start + c * 16;
      {
        const bool last = c + 1 == max_nch;
        const int e = (last ? (nbeg & ~3) : e0 + 16) + q * 4, lim = last ? nend : end;
        cp_async16(&sidx[warp][buf ^ 1][g][q * 4], ci + (e < lim ? e : 0), e < lim ? 16 : 0);
        cp_commit();
      }
      cp_wait1();
      __syncwarp();
      const int* jr = sidx[warp][buf][g];
      const int lo = beg > e0 ? beg - e0 : 0;
      int hi = end - e0;
      hi = hi < 0 ? 0 : (hi > 16 ? 16 : hi);
      const bool full = __all_sync(kFull, lo == 0 && hi == 16);
#pragma unroll
      for (int u0 = 0; u0 < 16; u0 += B) {
        uint64_t v[B][4];
#pragma unroll
        for (int t = 0; t < B; ++t) {
          const int u = u0 + t;
          const int j = jr[u];
          if (full || (u >= lo && u < hi)) ldg256(Y + ((size_t)j * LPR + q) * 4, v[t]);
          else v[t][0] = v[t][1] = v[t][2] = v[t][3] = 0ull;
        }
#pragma unroll
        for (int t = 0; t < B; ++t)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[k] = fadd2(acc[k], v[t][k]);
      }
      __syncwarp();  // every lane has read this half before it is refilled
      buf ^= 1;
    }
    if (row < n) finish_row(Y, O, s, row, q, acc);
  }
  cp_wait0();
}

template <typename K>
float timeit(K kern, int grid, int block, const int* rp, const int* ci, const float* s, float* y0, float* y1, int n,
             int reps) {
  kern<<<grid, block>>>(rp, ci, s, y0, y1, n);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) kern<<<grid, block>>>(rp, ci, s, (r & 1) ? y1 : y0, (r & 1) ? y0 : y1, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: smidx_lab rp ci N nnz\n");
    return 2;
  }
  const int n = atoi(argv[3]);
  const long nnz = atol(argv[4]);
  std::vector<int> hrp(n + 1), hci(nnz + 16, 0);
  FILE* f = fopen(argv[1], "rb");
  if (!f || fread(hrp.data(), 4, n + 1, f) != (size_t)n + 1) return 3;
  fclose(f);
  f = fopen(argv[2], "rb");
  if (!f || fread(hci.data(), 4, nnz, f) != (size_t)nnz) return 3;
  fclose(f);
  int *rp, *ci;
  float *s, *y0, *y1, *yr, *yt, *yinit;
  cudaMalloc(&rp, 4 * (n + 1));
  cudaMalloc(&ci, 4 * (nnz + 16));
  cudaMalloc(&s, 4 * n);
  for (float** p : {&y0, &y1, &yr, &yt, &yinit}) cudaMalloc(p, 4l * n * W);
  cudaMemcpy(rp, hrp.data(), 4 * (n + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(ci, hci.data(), 4 * (nnz + 16), cudaMemcpyHostToDevice);
  {
    std::vector<float> hs(n), hy((size_t)n * W);
    for (int i = 0; i < n; ++i) {
      const int d = hrp[i + 1] - hrp[i];
      hs[i] = d > 0 ? 1.0f / sqrtf((float)d) : 1.0f;
    }
    for (size_t k = 0; k < hy.size(); ++k) hy[k] = (float)((k * 2654435761u) % 1000) * 1e-3f - 0.5f;
    cudaMemcpy(s, hs.data(), 4 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(y0, hy.data(), 4l * n * W, cudaMemcpyHostToDevice);
    cudaMemcpy(y1, hy.data(), 4l * n * W, cudaMemcpyHostToDevice);
    cudaMemcpy(yinit, hy.data(), 4l * n * W, cudaMemcpyHostToDevice);  // the timing loops ping-pong y0/y1
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double gbytes = 4.0 * W * nnz / 1e9;
  const int reps = 20;
  reg_idx<8, 2><<<sms * 2, 256>>>(rp, ci, s, yinit, yr, n);  // reference output
  std::vector<float> hr((size_t)n * W), ht((size_t)n * W);
  cudaMemcpy(hr.data(), yr, 4l * n * W, cudaMemcpyDeviceToHost);
#define RUN(NAME, KERN, NWV)                                                                                     \
  {                                                                                                              \
    int occ = 0;                                                                                                 \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, KERN, NWV * 32, 0);                                      \
    cudaFuncAttributes fa;                                                                                       \
    cudaFuncGetAttributes(&fa, KERN);                                                                            \
    const int grid = sms * occ;                                                                                  \
    float ms = timeit(KERN, grid, NWV * 32, rp, ci, s, y0, y1, n, reps);                                         \
    KERN<<<grid, NWV * 32>>>(rp, ci, s, yinit, yt, n);                                                              \
    cudaMemcpy(ht.data(), yt, 4l * n * W, cudaMemcpyDeviceToHost);                                              \
    double md = 0;                                                                                               \
    for (size_t k = 0; k < ht.size(); ++k) md = fmax(md, fabs((double)ht[k] - hr[k]));                           \
    printf("%-30s regs %3d warps/SM %2d: %8.1f us  gather %7.0f GB/s  max|diff| %.1e  %s\n", NAME, fa.numRegs,   \
           occ * NWV, ms * 1e3, gbytes / ms * 1e3, md, cudaGetErrorString(cudaGetLastError()));                  \
  }
  RUN("reg-idx 8x2", (reg_idx<8, 2>), 8);
  RUN("reg-idx 7x3", (reg_idx<7, 3>), 7);
  RUN("smem-idx 8x2", (sm_idx<8, 2>), 8);
  RUN("smem-idx 7x3", (sm_idx<7, 3>), 7);
  RUN("smem-idx 6x3", (sm_idx<6, 3>), 6);
  RUN("smem-idx 5x4", (sm_idx<5, 4>), 5);
  RUN("smem-idx 8x3", (sm_idx<8, 3>), 8);
  RUN("smem-idx 4x5", (sm_idx<4, 5>), 4);
  return 0;
}
