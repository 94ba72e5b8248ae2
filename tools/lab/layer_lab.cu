// layer_lab.cu — variants of the filter step's gather core on a real relabelled CSR (tooling, not product).
// Each variant computes, for a W=32 column slice, out_i = s_i tanh(0.1 y_i + s_i sum_j y_j) and is timed
// over repeated launches.  Used to choose the product kernel's gather pipeline.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/layer_lab tools/lab/layer_lab.cu
//   /tmp/layer_lab /tmp/lab.rp /tmp/lab.ci N nnz
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int W = 32;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void ldg256(const void* p, uint64_t (&v)[4]) {
  asm volatile("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ldg256na(const void* p, uint64_t (&v)[4]) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}
__device__ __forceinline__ void ldg128(const void* p, uint64_t (&v)[2]) {
  asm volatile("ld.global.nc.v2.b64 {%0,%1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "l"(p));
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
__device__ __forceinline__ int2 ld_idx2(const int* p) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ void pf_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

template <int IPL>
__device__ __forceinline__ void load_idx(const int* ci, int e0, int end, int q, int (&jr)[IPL]) {
  const int e = e0 + q * IPL;
  if (e >= end) {
#pragma unroll
    for (int k = 0; k < IPL; ++k) jr[k] = 0;
    return;
  }
  if constexpr (IPL == 4) {
    int4 v = ld_idx4(ci + e);
    jr[0] = v.x, jr[1] = v.y, jr[2] = v.z, jr[3] = v.w;
  } else if constexpr (IPL == 2) {
    int2 v = ld_idx2(ci + e);
    jr[0] = v.x, jr[1] = v.y;
  } else {
    jr[0] = ci[e];
  }
}

// VB: bytes per lane per gathered row (32: LDG.256, 16: LDG.128).  BATCH: gathers issued before consuming.
// PF: 1 = prefetch.global.L2 the next chunk's rows (each lane its own held indices).  NA: L1::no_allocate gathers.
template <int VB, int BATCH, int PF, int NA, int MINB>
__global__ void __launch_bounds__(256, MINB) lab(const int* __restrict__ rp, const int* __restrict__ ci,
                                                  const float* __restrict__ s, const float* __restrict__ yin,
                                                  float* __restrict__ yout, int n) {
  constexpr int LPR = W * 4 / VB, G = 32 / LPR, IPL = 16 / LPR, NV = VB / 8;  // NV u64 per lane per row
  constexpr int NG = 8 * G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % LPR, g = lane / LPR;
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  uint64_t* O = reinterpret_cast<uint64_t*>(yout);
  const long step = (long)gridDim.x * NG;
  for (long base = (long)blockIdx.x * NG + warp * G; base < n; base += step) {
    const int row = (int)(base + g);
    const bool valid = row < n;
    int beg = 0, end = 0;
    if (valid) {
      beg = __ldg(rp + row);
      end = __ldg(rp + row + 1);
    }
    uint64_t acc[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = 0ull;
    const int start = beg & ~3;
    const int nch = end > beg ? (end - start + 15) / 16 : 0;
    const int max_nch = __reduce_max_sync(kFull, nch);
    int jr[IPL];
    load_idx<IPL>(ci, start, end, q, jr);
    for (int c = 0; c < max_nch; ++c) {
      const int e0 = start + c * 16, e1 = e0 + 16;
      int jn[IPL];
      load_idx<IPL>(ci, e1, end, q, jn);
      if (PF == 1) {
#pragma unroll
        for (int k = 0; k < IPL; ++k)
          if (e1 + q * IPL + k < end) pf_l2(Y + (size_t)jn[k] * (W / 2));
      } else if (PF == 2) {
#pragma unroll
        for (int k = 0; k < IPL; ++k)
          if (e1 + q * IPL + k < end) pf_l1(Y + (size_t)jn[k] * (W / 2));
      }
      const int lo = beg > e0 ? beg - e0 : 0;
      int hi = end - e0;
      hi = hi < 0 ? 0 : (hi > 16 ? 16 : hi);
      const bool full = __all_sync(kFull, lo == 0 && hi == 16);
#pragma unroll
      for (int u0 = 0; u0 < 16; u0 += BATCH) {
        uint64_t v[BATCH][NV];
#pragma unroll
        for (int t = 0; t < BATCH; ++t) {
          const int u = u0 + t;
          const int j = __shfl_sync(kFull, jr[u % IPL], u / IPL, LPR);
          const uint64_t* p = Y + ((size_t)j * LPR + q) * NV;
          if (full || (u >= lo && u < hi)) {
            if constexpr (NV == 4) {
              if (NA) ldg256na(p, v[t]); else ldg256(p, v[t]);
            } else {
              ldg128(p, v[t]);
            }
          } else {
#pragma unroll
            for (int k = 0; k < NV; ++k) v[t][k] = 0ull;
          }
        }
#pragma unroll
        for (int t = 0; t < BATCH; ++t)
#pragma unroll
          for (int k = 0; k < NV; ++k) acc[k] = fadd2(acc[k], v[t][k]);
      }
#pragma unroll
      for (int k = 0; k < IPL; ++k) jr[k] = jn[k];
    }
    if (valid) {
      const float si = s[row];
      const uint64_t* own = Y + ((size_t)row * LPR + q) * NV;
      uint64_t o[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const float2 y = unpack2(own[k]);
        const float2 a = unpack2(acc[k]);
        o[k] = pack2(si * tanhf(0.1f * y.x + si * a.x), si * tanhf(0.1f * y.y + si * a.y));
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) O[((size_t)row * LPR + q) * NV + k] = o[k];
    }
  }
}

// Software-pipelined variant: batches of B4 gathers double-buffered across the whole row (always one
// batch in flight while the previous is consumed).  VB = 32.
template <int B4, int MINB>
__global__ void __launch_bounds__(256, MINB) lab_pipe(const int* __restrict__ rp, const int* __restrict__ ci,
                                                       const float* __restrict__ s, const float* __restrict__ yin,
                                                       float* __restrict__ yout, int n) {
  constexpr int LPR = 4, G = 8, IPL = 4, NV = 4, NG = 8 * G;
  constexpr int NB = 16 / B4;  // batches per chunk
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % LPR, g = lane / LPR;
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  uint64_t* O = reinterpret_cast<uint64_t*>(yout);
  const long step = (long)gridDim.x * NG;
  for (long base = (long)blockIdx.x * NG + warp * G; base < n; base += step) {
    const int row = (int)(base + g);
    const bool valid = row < n;
    int beg = 0, end = 0;
    if (valid) {
      beg = __ldg(rp + row);
      end = __ldg(rp + row + 1);
    }
    uint64_t acc[NV] = {0ull, 0ull, 0ull, 0ull};
    const int start = beg & ~3;
    const int nch = end > beg ? (end - start + 15) / 16 : 0;
    const int max_nch = __reduce_max_sync(kFull, nch);
    int jr[IPL], jn[IPL];
    load_idx<IPL>(ci, start, end, q, jr);
    load_idx<IPL>(ci, start + 16, end, q, jn);
    uint64_t va[B4][NV], vb[B4][NV];
    auto issue = [&](uint64_t (&v)[B4][NV], const int (&jj)[IPL], int e0, int u0) {
#pragma unroll
      for (int t = 0; t < B4; ++t) {
        const int u = u0 + t;
        const int j = __shfl_sync(kFull, jj[u % IPL], u / IPL, LPR);
        const int e = e0 + u;
        if (e >= beg && e < end) ldg256(Y + ((size_t)j * LPR + q) * NV, v[t]);
        else v[t][0] = v[t][1] = v[t][2] = v[t][3] = 0ull;
      }
    };
    auto consume = [&](uint64_t (&v)[B4][NV]) {
#pragma unroll
      for (int t = 0; t < B4; ++t)
#pragma unroll
        for (int k = 0; k < NV; ++k) acc[k] = fadd2(acc[k], v[t][k]);
    };
    if (max_nch > 0) issue(va, jr, start, 0);
    for (int c = 0; c < max_nch; ++c) {
      const int e0 = start + c * 16;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        // issue the next batch (possibly the next chunk's first), then consume the current one
        if (b + 1 < NB) {
          if (b % 2 == 0) issue(vb, jr, e0, (b + 1) * B4); else issue(va, jr, e0, (b + 1) * B4);
        } else if (c + 1 < max_nch) {
          if (b % 2 == 0) issue(vb, jn, e0 + 16, 0); else issue(va, jn, e0 + 16, 0);
        }
        if (b % 2 == 0) consume(va); else consume(vb);
      }
      // NB even: the next chunk's first batch is in va again
#pragma unroll
      for (int k = 0; k < IPL; ++k) jr[k] = jn[k];
      load_idx<IPL>(ci, e0 + 32, end, q, jn);
    }
    if (valid) {
      const float si = s[row];
      const uint64_t* own = Y + ((size_t)row * LPR + q) * NV;
      uint64_t o[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const float2 y = unpack2(own[k]);
        const float2 a = unpack2(acc[k]);
        o[k] = pack2(si * tanhf(0.1f * y.x + si * a.x), si * tanhf(0.1f * y.y + si * a.y));
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) O[((size_t)row * LPR + q) * NV + k] = o[k];
    }
  }
}

// Segment-free gather ceiling: the CSR column stream as a flat list of row gathers (no rows, no
// epilogue), LPR lanes per 128-byte row, BATCH rows per lane in flight.  Sums are discarded.
template <int VB, int BATCH, int MINB>
__global__ void __launch_bounds__(256, MINB) flat(const int* __restrict__ rp, const int* __restrict__ ci,
                                                   const float* __restrict__ s, const float* __restrict__ yin,
                                                   float* __restrict__ yout, int n) {
  constexpr int LPR = W * 4 / VB, G = 32 / LPR, NV = VB / 8;
  const int lane = threadIdx.x & 31, q = lane % LPR, g = lane / LPR;
  const long nnz = rp[n];
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  constexpr int PER = G * BATCH;  // gathers per warp iteration
  uint64_t acc[NV] = {};
  for (long e0 = warp * PER; e0 < nnz; e0 += nw * PER) {
    int jl = (lane < PER && e0 + lane < nnz) ? __ldg(ci + e0 + lane) : 0;
    uint64_t v[BATCH][NV];
#pragma unroll
    for (int t = 0; t < BATCH; ++t) {
      const int j = __shfl_sync(kFull, jl, (t * G + g) & 31);
      const uint64_t* p = Y + ((size_t)j * LPR + q) * NV;
      if constexpr (NV == 4) ldg256(p, v[t]); else ldg128(p, v[t]);
    }
#pragma unroll
    for (int t = 0; t < BATCH; ++t)
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] = fadd2(acc[k], v[t][k]);
  }
  float x = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) x += unpack2(acc[k]).x;
  if (x == 1234.5f) yout[0] = x;
}

// Edge-balanced "pieces" variant: a warp takes R consecutive rows, splits their contiguous edge range
// into 8 equal pieces (one per 4-lane group), each group streams its piece 4 edges at a time with no
// row-boundary masking, flushing finished rows to shared memory; partial rows at piece boundaries are
// combined in edge order (deterministic).  VB = 32.
template <int R, int MINB>
__global__ void __launch_bounds__(256, MINB) lab_pieces(const int* __restrict__ rp, const int* __restrict__ ci,
                                                         const float* __restrict__ s, const float* __restrict__ yin,
                                                         float* __restrict__ yout, int n) {
  constexpr int LPR = 4, G = 8, NV = 4;
  __shared__ __align__(16) uint64_t rowacc[8][R][16];
  __shared__ __align__(16) uint64_t headacc[8][G][16];
  __shared__ int headrow[8][G];
  __shared__ int srp[8][R + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % LPR, g = lane / LPR;
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  uint64_t* O = reinterpret_cast<uint64_t*>(yout);
  int* sr = srp[warp];
  for (long r0l = ((long)blockIdx.x * 8 + warp) * R; r0l < n; r0l += (long)gridDim.x * 8 * R) {
    const int r0 = (int)r0l;
    const int nr = min(R, n - r0);
    if (lane <= nr) sr[lane] = __ldg(rp + r0 + lane);
    if (lane < G) headrow[warp][lane] = -1;
    __syncwarp();
    const int E0 = sr[0], E1 = sr[nr];
    const int P = (((E1 - E0) + 7) / 8 + 3) & ~3;
    const int pb = min(E0 + g * P, E1), pe = min(pb + P, E1);
    // row of the piece's first edge: the last row r with sr[r] <= pb (skipping empty rows)
    int cur = 0;
    while (cur + 1 < nr && sr[cur + 1] <= pb) ++cur;
    int cend = sr[cur + 1];
    bool head = pb > sr[cur];
    uint64_t acc[NV] = {0ull, 0ull, 0ull, 0ull};
    auto flush = [&]() {
      uint64_t* dst = head ? headacc[warp][g] : rowacc[warp][cur];
      *reinterpret_cast<uint4*>(dst + q * 4) = make_uint4((uint32_t)acc[0], (uint32_t)(acc[0] >> 32), (uint32_t)acc[1], (uint32_t)(acc[1] >> 32));
      *reinterpret_cast<uint4*>(dst + q * 4 + 2) = make_uint4((uint32_t)acc[2], (uint32_t)(acc[2] >> 32), (uint32_t)acc[3], (uint32_t)(acc[3] >> 32));
      if (head && q == 0) headrow[warp][g] = cur;
      head = false;
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] = 0ull;
    };
    const int steps = __reduce_max_sync(kFull, (pe - pb + 3) / 4);
    int jn = (pb + q < pe) ? __ldg(ci + pb + q) : 0;
    for (int it = 0; it < steps; ++it) {
      const int e = pb + it * 4;
      const int jq = jn;
      jn = (e + 4 + q < pe) ? __ldg(ci + e + 4 + q) : 0;
      uint64_t v[4][NV];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int j = __shfl_sync(kFull, jq, t, LPR);
        if (e + t < pe) ldg256(Y + ((size_t)j * LPR + q) * NV, v[t]);
        else v[t][0] = v[t][1] = v[t][2] = v[t][3] = 0ull;
      }
      if (e + 3 < cend) {  // all four edges in the current row (or past the piece end: zeros)
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int k = 0; k < NV; ++k) acc[k] = fadd2(acc[k], v[t][k]);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (e + t < pe) {
            while (e + t >= cend) {
              flush();
              ++cur;
              cend = sr[cur + 1];
            }
#pragma unroll
            for (int k = 0; k < NV; ++k) acc[k] = fadd2(acc[k], v[t][k]);
          }
        }
      }
    }
    if (pb < pe) flush();
    __syncwarp();
    for (int rl = g; rl < nr; rl += G) {
      const int row = r0 + rl;
      uint64_t a[NV] = {0ull, 0ull, 0ull, 0ull};
      if (sr[rl + 1] > sr[rl]) {
        const uint4 x0 = *reinterpret_cast<const uint4*>(&rowacc[warp][rl][q * 4]);
        const uint4 x1 = *reinterpret_cast<const uint4*>(&rowacc[warp][rl][q * 4 + 2]);
        a[0] = ((uint64_t)x0.y << 32) | x0.x; a[1] = ((uint64_t)x0.w << 32) | x0.z;
        a[2] = ((uint64_t)x1.y << 32) | x1.x; a[3] = ((uint64_t)x1.w << 32) | x1.z;
        for (int gg = 0; gg < G; ++gg) {
          if (headrow[warp][gg] == rl) {
            const uint64_t* h = headacc[warp][gg] + q * 4;
#pragma unroll
            for (int k = 0; k < NV; ++k) a[k] = fadd2(a[k], h[k]);
          }
        }
      }
      const float si = s[row];
      const uint64_t* own = Y + ((size_t)row * LPR + q) * NV;
      uint64_t o[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const float2 y = unpack2(own[k]);
        const float2 aa = unpack2(a[k]);
        o[k] = pack2(si * tanhf(0.1f * y.x + si * aa.x), si * tanhf(0.1f * y.y + si * aa.y));
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) O[((size_t)row * LPR + q) * NV + k] = o[k];
    }
    __syncwarp();
  }
}

// Row-per-group variant with 4-gather batches that skip fully-masked batches, and the next row
// batch's row pointers loaded ahead.  VB = 32.
template <int MINB>
__global__ void __launch_bounds__(256, MINB) lab_row2(const int* __restrict__ rp, const int* __restrict__ ci,
                                                       const float* __restrict__ s, const float* __restrict__ yin,
                                                       float* __restrict__ yout, int n) {
  constexpr int LPR = 4, G = 8, IPL = 4, NV = 4, NG = 8 * G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % LPR, g = lane / LPR;
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  uint64_t* O = reinterpret_cast<uint64_t*>(yout);
  const long step = (long)gridDim.x * NG;
  long base = (long)blockIdx.x * NG + warp * G;
  int nbeg = 0, nend = 0;
  if (base + g < n) { nbeg = __ldg(rp + base + g); nend = __ldg(rp + base + g + 1); }
  for (; base < n; base += step) {
    const int row = (int)(base + g);
    const bool valid = row < n;
    const int beg = nbeg, end = nend;
    if (base + step + g < n) { nbeg = __ldg(rp + base + step + g); nend = __ldg(rp + base + step + g + 1); }
    uint64_t acc[NV] = {0ull, 0ull, 0ull, 0ull};
    const int start = beg & ~3;
    const int nch = end > beg ? (end - start + 15) / 16 : 0;
    const int max_nch = __reduce_max_sync(kFull, nch);
    int jr[IPL];
    load_idx<IPL>(ci, start, end, q, jr);
    for (int c = 0; c < max_nch; ++c) {
      const int e0 = start + c * 16, e1 = e0 + 16;
      int jn[IPL];
      load_idx<IPL>(ci, e1, end, q, jn);
      const int lo = beg > e0 ? beg - e0 : 0;
      int hi = end - e0;
      hi = hi < 0 ? 0 : (hi > 16 ? 16 : hi);
      const int maxhi = __reduce_max_sync(kFull, hi);
#pragma unroll
      for (int u0 = 0; u0 < 16; u0 += 4) {
        if (u0 >= maxhi) break;
        uint64_t v[4][NV];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int u = u0 + t;
          const int j = __shfl_sync(kFull, jr[u % IPL], u / IPL, LPR);
          if (u >= lo && u < hi) ldg256(Y + ((size_t)j * LPR + q) * NV, v[t]);
          else v[t][0] = v[t][1] = v[t][2] = v[t][3] = 0ull;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int k = 0; k < NV; ++k) acc[k] = fadd2(acc[k], v[t][k]);
      }
#pragma unroll
      for (int k = 0; k < IPL; ++k) jr[k] = jn[k];
    }
    if (valid) {
      const float si = s[row];
      const uint64_t* own = Y + ((size_t)row * LPR + q) * NV;
      uint64_t o[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const float2 y = unpack2(own[k]);
        const float2 a = unpack2(acc[k]);
        o[k] = pack2(si * tanhf(0.1f * y.x + si * a.x), si * tanhf(0.1f * y.y + si * a.y));
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) O[((size_t)row * LPR + q) * NV + k] = o[k];
    }
  }
}

// The product structure (full-chunk fast path, BATCH gathers per round) with the row-batch latency
// chain hidden: PRE >= 1 loads the next row batch's row pointers during the current batch; PRE >= 2
// also its first index chunk; PRE >= 3 issues the own-row load at the start of the batch.
template <int BATCH, int PRE, int MINB>
__global__ void __launch_bounds__(256, MINB) lab_pre(const int* __restrict__ rp, const int* __restrict__ ci,
                                                      const float* __restrict__ s, const float* __restrict__ yin,
                                                      float* __restrict__ yout, int n) {
  constexpr int LPR = 4, G = 8, IPL = 4, NV = 4, NG = 8 * G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % LPR, g = lane / LPR;
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  uint64_t* O = reinterpret_cast<uint64_t*>(yout);
  const long step = (long)gridDim.x * NG;
  long base = (long)blockIdx.x * NG + warp * G;
  int nbeg = 0, nend = 0;
  int jfirst[IPL] = {0, 0, 0, 0};
  if (PRE >= 1 && base + g < n) {
    nbeg = __ldg(rp + base + g);
    nend = __ldg(rp + base + g + 1);
    if (PRE >= 2) load_idx<IPL>(ci, nbeg & ~3, nend, q, jfirst);
  }
  for (; base < n; base += step) {
    const int row = (int)(base + g);
    const bool valid = row < n;
    int beg = 0, end = 0;
    int jr[IPL];
    if (PRE >= 1) {
      beg = nbeg, end = nend;
      if (PRE >= 2) {
#pragma unroll
        for (int k = 0; k < IPL; ++k) jr[k] = jfirst[k];
      }
    } else if (valid) {
      beg = __ldg(rp + row);
      end = __ldg(rp + row + 1);
    }
    uint64_t own[NV];
    if (PRE == 3 && valid) {
      const uint64_t* op = Y + ((size_t)row * LPR + q) * NV;
      ldg256(op, own);
    }
    const int start = beg & ~3;
    if (PRE < 2) load_idx<IPL>(ci, start, end, q, jr);
    if (PRE >= 1) {
      const long nb = base + step + g;
      nbeg = nend = 0;
      if (nb < n) {
        nbeg = __ldg(rp + nb);
        nend = __ldg(rp + nb + 1);
      }
    }
    uint64_t acc[NV] = {0ull, 0ull, 0ull, 0ull};
    const int nch = end > beg ? (end - start + 15) / 16 : 0;
    const int max_nch = __reduce_max_sync(kFull, nch);
    for (int c = 0; c < max_nch; ++c) {
      const int e0 = start + c * 16, e1 = e0 + 16;
      int jn[IPL];
      load_idx<IPL>(ci, e1, end, q, jn);
      if (PRE >= 2 && c == 0) load_idx<IPL>(ci, nbeg & ~3, nend, q, jfirst);
      const int lo = beg > e0 ? beg - e0 : 0;
      int hi = end - e0;
      hi = hi < 0 ? 0 : (hi > 16 ? 16 : hi);
      const bool full = __all_sync(kFull, lo == 0 && hi == 16);
#pragma unroll
      for (int u0 = 0; u0 < 16; u0 += BATCH) {
        uint64_t v[BATCH][NV];
#pragma unroll
        for (int t = 0; t < BATCH; ++t) {
          const int u = u0 + t;
          const int j = __shfl_sync(kFull, jr[u % IPL], u / IPL, LPR);
          if (full || (u >= lo && u < hi)) ldg256(Y + ((size_t)j * LPR + q) * NV, v[t]);
          else v[t][0] = v[t][1] = v[t][2] = v[t][3] = 0ull;
        }
#pragma unroll
        for (int t = 0; t < BATCH; ++t)
#pragma unroll
          for (int k = 0; k < NV; ++k) acc[k] = fadd2(acc[k], v[t][k]);
      }
#pragma unroll
      for (int k = 0; k < IPL; ++k) jr[k] = jn[k];
    }
    if (PRE >= 2 && max_nch == 0) load_idx<IPL>(ci, nbeg & ~3, nend, q, jfirst);
    if (PRE == 4 && valid) {  // gather-only: the raw neighbour sums, for a separate epilogue pass
#pragma unroll
      for (int k = 0; k < NV; ++k) O[((size_t)row * LPR + q) * NV + k] = acc[k];
    } else if (valid) {
      const float si = s[row];
      if (PRE != 3) {
        const uint64_t* op = Y + ((size_t)row * LPR + q) * NV;
#pragma unroll
        for (int k = 0; k < NV; ++k) own[k] = op[k];
      }
      uint64_t o[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const float2 y = unpack2(own[k]);
        const float2 a = unpack2(acc[k]);
        o[k] = pack2(si * tanhf(0.1f * y.x + si * a.x), si * tanhf(0.1f * y.y + si * a.y));
      }
#pragma unroll
      for (int k = 0; k < NV; ++k) O[((size_t)row * LPR + q) * NV + k] = o[k];
    }
  }
}

// flat + the epilogue's streaming traffic: every warp also reads and writes its share of a
// separate N x W buffer (own-row read + output store), optionally with an L2 evict_first store hint.
template <int EF>
__global__ void __launch_bounds__(256, 4) flat_rw(const int* __restrict__ rp, const int* __restrict__ ci,
                                                   const float* __restrict__ s, const float* __restrict__ yin,
                                                   float* __restrict__ yout, int n) {
  constexpr int LPR = 4, G = 8, NV = 4, BATCH = 4, PER = G * BATCH;
  const int lane = threadIdx.x & 31, q = lane % LPR, g = lane / LPR;
  const long nnz = rp[n];
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  uint64_t* O = reinterpret_cast<uint64_t*>(yout);
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
  uint64_t acc[NV] = {};
  long it = 0;
  for (long e0 = warp * PER; e0 < nnz; e0 += nw * PER, ++it) {
    int jl = (e0 + lane < nnz) ? __ldg(ci + e0 + lane) : 0;
    uint64_t v[BATCH][NV];
#pragma unroll
    for (int t = 0; t < BATCH; ++t) {
      const int j = __shfl_sync(kFull, jl, (t * G + g) & 31);
      ldg256(Y + ((size_t)j * LPR + q) * NV, v[t]);
    }
#pragma unroll
    for (int t = 0; t < BATCH; ++t)
#pragma unroll
      for (int k = 0; k < NV; ++k) acc[k] = fadd2(acc[k], v[t][k]);
    // one row of own-read + store per ~40 gathers per group: every 5th iteration (32 gathers/warp/iter)
    const long row = (warp + it * nw) % n;
    if ((it % 5) == 0) {
      const long r = ((e0 / PER) / 5 * G + g) % n;
      uint64_t own[NV];
      ldg256(Y + ((size_t)r * LPR + q) * NV, own);
#pragma unroll
      for (int k = 0; k < NV; ++k) own[k] = fadd2(own[k], acc[k]);
      uint64_t* dst = O + ((size_t)r * LPR + q) * NV;
      if (EF) asm volatile("st.global.L2::cache_hint.v4.b64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(dst), "l"(own[0]), "l"(own[1]), "l"(own[2]), "l"(own[3]), "l"(pol) : "memory");
      else asm volatile("st.global.v4.b64 [%0], {%1,%2,%3,%4};" ::"l"(dst), "l"(own[0]), "l"(own[1]), "l"(own[2]), "l"(own[3]) : "memory");
    }
    (void)row;
  }
}

// The product structure with chunked dynamic row scheduling: a block grabs K consecutive row
// batches (K x 64 rows) at a time from a global counter, so consecutive batches of a community
// run on one SM (L1 reuse of shared neighbours) while the grid stays balanced.
__device__ int g_chunk_counter;
template <int K>
__global__ void __launch_bounds__(256, 2) lab_chunk(const int* __restrict__ rp, const int* __restrict__ ci,
                                                     const float* __restrict__ s, const float* __restrict__ yin,
                                                     float* __restrict__ yout, int n) {
  constexpr int LPR = 4, G = 8, IPL = 4, NV = 4, NG = 8 * G, BATCH = 8;
  __shared__ int chunk;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane % LPR, g = lane / LPR;
  const uint64_t* Y = reinterpret_cast<const uint64_t*>(yin);
  uint64_t* O = reinterpret_cast<uint64_t*>(yout);
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) chunk = atomicAdd(&g_chunk_counter, 1);
    __syncthreads();
    const long c0 = (long)chunk * K * NG;
    if (c0 >= n) break;
    for (int k = 0; k < K; ++k) {
      const long base = c0 + (long)k * NG + warp * G;
      if (base >= n) break;
      const int row = (int)(base + g);
      const bool valid = row < n;
      int beg = 0, end = 0;
      if (valid) { beg = __ldg(rp + row); end = __ldg(rp + row + 1); }
      uint64_t acc[NV] = {0ull, 0ull, 0ull, 0ull};
      const int start = beg & ~3;
      const int nch = end > beg ? (end - start + 15) / 16 : 0;
      const int max_nch = __reduce_max_sync(kFull, nch);
      int jr[IPL];
      load_idx<IPL>(ci, start, end, q, jr);
      for (int c = 0; c < max_nch; ++c) {
        const int e0 = start + c * 16, e1 = e0 + 16;
        int jn[IPL];
        load_idx<IPL>(ci, e1, end, q, jn);
        const int lo = beg > e0 ? beg - e0 : 0;
        int hi = end - e0;
        hi = hi < 0 ? 0 : (hi > 16 ? 16 : hi);
        const bool full = __all_sync(kFull, lo == 0 && hi == 16);
#pragma unroll
        for (int u0 = 0; u0 < 16; u0 += BATCH) {
          uint64_t v[BATCH][NV];
#pragma unroll
          for (int t = 0; t < BATCH; ++t) {
            const int u = u0 + t;
            const int j = __shfl_sync(kFull, jr[u % IPL], u / IPL, LPR);
            if (full || (u >= lo && u < hi)) ldg256(Y + ((size_t)j * LPR + q) * NV, v[t]);
            else v[t][0] = v[t][1] = v[t][2] = v[t][3] = 0ull;
          }
#pragma unroll
          for (int t = 0; t < BATCH; ++t)
#pragma unroll
            for (int kk = 0; kk < NV; ++kk) acc[kk] = fadd2(acc[kk], v[t][kk]);
        }
#pragma unroll
        for (int kk = 0; kk < IPL; ++kk) jr[kk] = jn[kk];
      }
      if (valid) {
        const float si = s[row];
        const uint64_t* own = Y + ((size_t)row * LPR + q) * NV;
        uint64_t o[NV];
#pragma unroll
        for (int kk = 0; kk < NV; ++kk) {
          const float2 y = unpack2(own[kk]);
          const float2 a = unpack2(acc[kk]);
          o[kk] = pack2(si * tanhf(0.1f * y.x + si * a.x), si * tanhf(0.1f * y.y + si * a.y));
        }
#pragma unroll
        for (int kk = 0; kk < NV; ++kk) O[((size_t)row * LPR + q) * NV + kk] = o[kk];
      }
    }
  }
}

template <typename K>
float timeit(K kern, int grid, const int* rp, const int* ci, const float* s, float* y0, float* y1, int n, int reps,
             int* regs) {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  *regs = fa.numRegs;
  kern<<<grid, 256>>>(rp, ci, s, y0, y1, n);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) kern<<<grid, 256>>>(rp, ci, s, (r & 1) ? y1 : y0, (r & 1) ? y0 : y1, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: layer_lab rp ci N nnz\n");
    return 2;
  }
  const int n = atoi(argv[3]);
  const long nnz = atol(argv[4]);
  std::vector<int> hrp(n + 1), hci(nnz + 16, 0);
  FILE* f = fopen(argv[1], "rb");
  if (fread(hrp.data(), 4, n + 1, f) != (size_t)n + 1) return 3;
  fclose(f);
  f = fopen(argv[2], "rb");
  if (fread(hci.data(), 4, nnz, f) != (size_t)nnz) return 3;
  fclose(f);
  int *rp, *ci;
  float *s, *y0, *y1;
  cudaMalloc(&rp, 4 * (n + 1));
  cudaMalloc(&ci, 4 * (nnz + 16));
  cudaMalloc(&s, 4 * n);
  cudaMalloc(&y0, 4l * n * W);
  cudaMalloc(&y1, 4l * n * W);
  cudaMemcpy(rp, hrp.data(), 4 * (n + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(ci, hci.data(), 4 * (nnz + 16), cudaMemcpyHostToDevice);
  {
    std::vector<float> hs(n), hy((size_t)n * W);
    for (int i = 0; i < n; ++i) {
      int d = hrp[i + 1] - hrp[i];
      hs[i] = d > 0 ? 1.0f / sqrtf((float)d) : 1.0f;
    }
    for (size_t k = 0; k < hy.size(); ++k) hy[k] = (float)((k * 2654435761u) % 1000) * 1e-3f - 0.5f;
    cudaMemcpy(s, hs.data(), 4 * n, cudaMemcpyHostToDevice);
    cudaMemcpy(y0, hy.data(), 4l * n * W, cudaMemcpyHostToDevice);
    cudaMemcpy(y1, hy.data(), 4l * n * W, cudaMemcpyHostToDevice);
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double gbytes = 4.0 * W * nnz / 1e9;
  const int reps = 20;
#define RUN(NAME, KERN, OCC)                                                                                       \
  {                                                                                                                \
    int occ = 0, regs = 0;                                                                                         \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, KERN, 256, 0);                                             \
    int g = sms * (OCC > 0 ? OCC : occ);                                                                           \
    float ms = timeit(KERN, g, rp, ci, s, y0, y1, n, reps, &regs);                                                 \
    printf("%-44s regs %3d occ %d grid %5d: %8.1f us  gather %7.0f GB/s  %s\n", NAME, regs, occ, g, ms * 1e3,      \
           gbytes / ms * 1e3, cudaGetErrorString(cudaGetLastError()));                                             \
  }
  RUN("flat VB32 B4 occ4", (flat<32, 4, 4>), 4);
  RUN("base VB32 B8 + L1 prefetch of next chunk", (lab<32, 8, 2, 0, 2>), 0);
  RUN("base VB32 B4 + L1 prefetch of next chunk", (lab<32, 4, 2, 0, 2>), 0);
  RUN("base VB32 B4 occ4 + L1 prefetch", (lab<32, 4, 2, 0, 4>), 0);
#define RUNC(NAME, KK)                                                                                             \
  {                                                                                                                \
    cudaEvent_t a0, b0;                                                                                            \
    cudaEventCreate(&a0);                                                                                          \
    cudaEventCreate(&b0);                                                                                          \
    int zero = 0;                                                                                                  \
    float tot = 0;                                                                                                 \
    for (int r = 0; r < reps + 1; ++r) {                                                                           \
      cudaMemcpyToSymbol(g_chunk_counter, &zero, sizeof(int));                                                    \
      cudaEventRecord(a0);                                                                                         \
      lab_chunk<KK><<<sms * 2, 256>>>(rp, ci, s, (r & 1) ? y1 : y0, (r & 1) ? y0 : y1, n);                         \
      cudaEventRecord(b0);                                                                                         \
      cudaEventSynchronize(b0);                                                                                    \
      float ms;                                                                                                    \
      cudaEventElapsedTime(&ms, a0, b0);                                                                           \
      if (r) tot += ms;                                                                                            \
    }                                                                                                              \
    printf("%-44s                          : %8.1f us  gather %7.0f GB/s  %s\n", NAME, tot / reps * 1e3,            \
           gbytes / (tot / reps) * 1e3, cudaGetErrorString(cudaGetLastError()));                                   \
  }
  RUNC("chunk K=1 (dynamic)", 1);
  RUNC("chunk K=2", 2);
  RUNC("chunk K=4", 4);
  RUNC("chunk K=8", 8);
  RUNC("chunk K=16", 16);
  RUN("flat + own/store stream", (flat_rw<0>), 4);
  RUN("flat + own/store stream (store evict_first)", (flat_rw<1>), 4);
  RUN("base VB32 B8 (product structure)", (lab<32, 8, 0, 0, 2>), 0);
  RUN("pre0 B8 occ2", (lab_pre<8, 0, 2>), 0);
  RUN("pre1 B8 occ2 (next rp)", (lab_pre<8, 1, 2>), 0);
  RUN("pre2 B8 occ2 (+ next idx)", (lab_pre<8, 2, 2>), 0);
  RUN("pre3 B8 occ2 (+ own early)", (lab_pre<8, 3, 2>), 0);
  RUN("pre2 B4 occ4", (lab_pre<4, 2, 4>), 0);
  RUN("pre3 B4 occ4", (lab_pre<4, 3, 4>), 0);
  RUN("pre2 B4 occ3", (lab_pre<4, 2, 3>), 0);
  RUN("pre2 B8 occ3", (lab_pre<8, 2, 3>), 0);
  RUN("gather-only B8 occ2 (sums stored)", (lab_pre<8, 4, 2>), 0);
  RUN("gather-only B8 occ3 (sums stored)", (lab_pre<8, 4, 3>), 0);
  RUN("gather-only B4 occ4 (sums stored)", (lab_pre<4, 4, 4>), 0);
  // correctness: pieces vs base (same math, summation order differs)
  {
    int regs;
    float *ya, *yb;
    cudaMalloc(&ya, 4l * n * W);
    cudaMalloc(&yb, 4l * n * W);
    lab<32, 8, 0, 0, 2><<<sms * 2, 256>>>(rp, ci, s, y0, ya, n);
    lab_pre<8, 3, 2><<<sms * 2, 256>>>(rp, ci, s, y0, yb, n);
    std::vector<float> ha((size_t)n * W), hb((size_t)n * W);
    cudaMemcpy(ha.data(), ya, 4l * n * W, cudaMemcpyDeviceToHost);
    cudaMemcpy(hb.data(), yb, 4l * n * W, cudaMemcpyDeviceToHost);
    double md = 0;
    for (size_t k = 0; k < ha.size(); ++k) md = fmax(md, fabs((double)ha[k] - hb[k]));
    lab_pre<4, 2, 4><<<sms * 4, 256>>>(rp, ci, s, y0, yb, n);
    cudaMemcpy(hb.data(), yb, 4l * n * W, cudaMemcpyDeviceToHost);
    double md2 = 0;
    for (size_t k = 0; k < ha.size(); ++k) md2 = fmax(md2, fabs((double)ha[k] - hb[k]));
    printf("max |pre3 - base| = %.3e   max |pre2B4 - base| = %.3e  (%s)\n", md, md2, cudaGetErrorString(cudaGetLastError()));
    (void)regs;
  }
  return 0;
}
