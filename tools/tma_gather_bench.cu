// tma_gather_bench.cu — random row-gather bandwidth with TMA tile::gather4 (tooling, not product).
// A producer warp streams 4-row gathers (cp.async.bulk.tensor.2d.tile::gather4) of a [rows][W]
// fp32 tensor into a shared-memory ring; consumer warps sum the landed rows.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
               : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
  return ok;
}

template <int W, int R, int S>
__global__ void __launch_bounds__(256) tma_gather(const __grid_constant__ CUtensorMap tm, const int* __restrict__ idx,
                                                  long m, float* out) {
  constexpr int STAGE_FLOATS = R * W;
  extern __shared__ __align__(1024) float ring[];  // [S][R][W]
  __shared__ __align__(8) uint64_t full[S], empty[S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int CW = 7;  // consumer warps
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(CW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const long nchunks = m / R;
  float acc = 0.f;
  if (warp == 0) {
    int it = 0;
    for (long c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
      const int s = it % S;
      const uint32_t ph = (it / S) & 1;
      if (it >= S) { long spin = 0; while (!try_wait(&empty[s], ph ^ 1)) if (++spin > (1l << 26)) __trap(); }
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(STAGE_FLOATS * 4));
      __syncwarp();
      for (int k = lane; k < R / 4; k += 32) {
        const int4 r = *reinterpret_cast<const int4*>(idx + c * R + 4 * k);
        float* dst = ring + s * STAGE_FLOATS + 4 * k * W;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            ::"r"(sa(dst)), "l"(&tm), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(sa(&full[s]))
            : "memory");
      }
    }
  } else {
    int it = 0;
    for (long c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
      const int s = it % S;
      const uint32_t ph = (it / S) & 1;
      { long spin = 0; while (!try_wait(&full[s], ph)) if (++spin > (1l << 26)) __trap(); }
      const float* src = ring + s * STAGE_FLOATS;
      for (int t = threadIdx.x - 32; t < STAGE_FLOATS; t += CW * 32) acc += src[t];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    }
  }
  if (acc == 12345.f) out[0] = acc;
}

__global__ void fill_idx(int* idx, long m, long rows, unsigned seed) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < m; i += (long)gridDim.x * blockDim.x) {
    unsigned long x = (unsigned long)i * 0x9E3779B97F4A7C15ul + seed;
    x ^= x >> 33; x *= 0xff51afd7ed558ccdul; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ul; x ^= x >> 33;
    idx[i] = (int)(x % (unsigned long)rows);
  }
}

template <int W, int R, int S>
void run(EncodeFn enc, float* y, long rows, const int* idx, long m, float* out, int sms, int bps) {
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {(cuuint32_t)W, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d (W=%d)\n", (int)r, W); return; }
  const size_t smem = (size_t)S * R * W * 4;
  cudaFuncSetAttribute(tma_gather<W, R, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = sms * bps;
  tma_gather<W, R, S><<<grid, 256, smem>>>(tm, idx, m, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  const int reps = 3;
  for (int i = 0; i < reps; ++i) tma_gather<W, R, S><<<grid, 256, smem>>>(tm, idx, m, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= reps;
  cudaError_t e = cudaGetLastError();
  printf("W=%3d R=%3d S=%2d smem=%6zu bps=%d footprint=%4ld MB: %.3f ms  %.0f GB/s  %s\n", W, R, S, smem, bps,
         (rows * W * 4) >> 20, ms, (double)m * W * 4 / ms / 1e6, cudaGetErrorString(e));
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (!fn) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
  EncodeFn enc = (EncodeFn)fn;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long m = 40l << 20;
  int* idx; cudaMalloc(&idx, m * 4);
  float* out; cudaMalloc(&out, 4);
  float* y; cudaMalloc(&y, 512ul << 20);
  cudaMemset(y, 0, 512ul << 20);
  for (int fmb : {16, 32, 64, 128, 256}) {
    long rows16 = ((long)fmb << 20) / 64, rows32 = ((long)fmb << 20) / 128, rows64 = ((long)fmb << 20) / 256;
    fill_idx<<<1024, 256>>>(idx, m, rows16, 1u);
    run<16, 128, 8>(enc, y, rows16, idx, m, out, sms, 2);
    run<16, 128, 8>(enc, y, rows16, idx, m, out, sms, 3);
    run<16, 64, 16>(enc, y, rows16, idx, m, out, sms, 3);
    fill_idx<<<1024, 256>>>(idx, m, rows32, 1u);
    run<32, 128, 4>(enc, y, rows32, idx, m, out, sms, 2);
    run<32, 64, 8>(enc, y, rows32, idx, m, out, sms, 3);
    fill_idx<<<1024, 256>>>(idx, m, rows64, 1u);
    run<64, 64, 4>(enc, y, rows64, idx, m, out, sms, 2);
    run<64, 32, 8>(enc, y, rows64, idx, m, out, sms, 3);
  }
  return 0;
}
