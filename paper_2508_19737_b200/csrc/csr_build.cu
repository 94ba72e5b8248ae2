// csr_build.cu — device CSR builder (igp_build_graph), SURVEY.md §8(a) rows a1-a3.
//
// Problem statement (§II): G = (V, E) undirected, unweighted,
// A_ij = A_ji = 1 iff (v_i, v_j) in E — so the builder symmetrises, drops self
// loops and removes duplicates.  The result is the unique canonical CSR (rows
// ascending, columns strictly ascending), bit-exact by construction: no step's
// output depends on thread timing once the per-row sort has run.
//
// Pipeline (one radix-N counting-sort pass on the row digit + a per-row sort):
//   B1 count      validate 0 <= u,v < N (device error flag), skip u == v,
//                 histogram both orientations per row            (atomics, grid over edges)
//   B2 scan       exclusive scan of row counts -> bucket offsets (3-phase scan)
//   B3 scatter    both orientations into their row bucket        (order within a row arbitrary)
//   B4 row sort   per-row sort + in-row dedup -> unique counts:
//                   len <= 64:            one warp per row, bitonic network in registers (shuffles)
//                   64 < len <= 1024:     one warp per row, bitonic sort in shared memory
//                   1024 < len <= 16384:  one block per row, bitonic sort in shared memory
//                   len > 16384:          one block per row, N-bit bitmap in global scratch
//   B5 scan+compact  row_ptr = scan(unique counts); col_idx = compacted rows
//   B6 row order  degree-descending (counting sort by degree, ascending id within a degree)
//   B7 (optional) label-propagation communities, rows bucketed by label, degree order within
//   B6b relabel   the CSR the filter steps traverse: rows in that order, each row's
//                 neighbours relabelled and kept in canonical order
// No host synchronisation: the column arrays are sized by the 2E directed entries
// before deduplication; nnz = row_ptr[N] and the range-error flag stay on the device
// until the caller asks (igp_api.cu).
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "igp_internal.cuh"

namespace igp {
namespace {

constexpr int kWarpSortCap = 1024;
constexpr int kBlockSortCap = 16384;
constexpr int kGiantBlocks = 16;
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------- B1 / B3
__global__ void count_kernel(const int32_t* __restrict__ edges, int64_t E, int32_t n,
                             int32_t* __restrict__ cnt, int32_t* __restrict__ err) {  // err: CsrDevice::meta[0]
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += stride) {
        const int32_t u = __ldg(edges + 2 * e), v = __ldg(edges + 2 * e + 1);
        if ((unsigned)u >= (unsigned)n || (unsigned)v >= (unsigned)n) {
            atomicOr(err, 1);
            continue;
        }
        if (u == v) continue;
        atomicAdd(cnt + u, 1);
        atomicAdd(cnt + v, 1);
    }
}

__global__ void scatter_kernel(const int32_t* __restrict__ edges, int64_t E, int32_t n,
                               const int32_t* __restrict__ off, int32_t* __restrict__ fill,
                               int32_t* __restrict__ tmp) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += stride) {
        const int32_t u = __ldg(edges + 2 * e), v = __ldg(edges + 2 * e + 1);
        if ((unsigned)u >= (unsigned)n || (unsigned)v >= (unsigned)n || u == v) continue;
        const int32_t pu = off[u] + atomicAdd(fill + u, 1);
        IGP_DASSERT(pu >= off[u] && pu < off[u + 1]);
        tmp[pu] = v;
        tmp[off[v] + atomicAdd(fill + v, 1)] = u;
    }
}

// ---------------------------------------------------------------- B2 scan
__device__ __forceinline__ int32_t block_exclusive_scan(int32_t x, int32_t* warp_tot, int32_t* total) {
    // blockDim.x <= 1024, multiple of 32; returns exclusive prefix of x, *total = block sum
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int32_t w = lane < nw ? warp_tot[lane] : 0;
        int32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < nw) warp_tot[lane] = wi - w;  // exclusive warp offsets
        if (lane == nw - 1) *total = wi;
    }
    __syncthreads();
    int32_t r = warp_tot[warp] + inc - x;
    __syncthreads();  // warp_tot reusable by the caller afterwards
    return r;
}

__global__ void scan_reduce_kernel(const int32_t* __restrict__ in, int32_t n, int32_t* __restrict__ bsum) {
    __shared__ int32_t red[kScanThreads / 32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
    int32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = base + k * kScanThreads + threadIdx.x;
        if (i < n) s += in[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += red[w];
        bsum[blockIdx.x] = t;
    }
}

// single block: exclusive scan of nb block sums in place; out_total <- sum
__global__ void scan_blocksums_kernel(int32_t* __restrict__ bsum, int32_t nb, int32_t* __restrict__ out_total) {
    __shared__ int32_t wt[32];
    __shared__ int32_t tot;
    int32_t carry = 0;
    for (int32_t b0 = 0; b0 < nb; b0 += blockDim.x) {
        int32_t i = b0 + threadIdx.x;
        int32_t x = i < nb ? bsum[i] : 0;
        int32_t ex = block_exclusive_scan(x, wt, &tot);
        if (i < nb) bsum[i] = carry + ex;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) *out_total = carry;
}

__global__ void scan_apply_kernel(const int32_t* __restrict__ in, int32_t n, const int32_t* __restrict__ bsum,
                                  int32_t* __restrict__ out) {
    __shared__ int32_t tile[kScanTile];
    __shared__ int32_t wt[32];
    __shared__ int32_t tot;
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = base + k * kScanThreads + threadIdx.x;
        tile[k * kScanThreads + threadIdx.x] = i < n ? in[i] : 0;
    }
    __syncthreads();
    int32_t loc[kScanItems];
    int32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        loc[k] = s;
        s += tile[threadIdx.x * kScanItems + k];
    }
    int32_t ex = block_exclusive_scan(s, wt, &tot) + bsum[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) tile[threadIdx.x * kScanItems + k] = ex + loc[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = base + k * kScanThreads + threadIdx.x;
        if (i < n) out[i] = tile[k * kScanThreads + threadIdx.x];
    }
}

// scan_apply_kernel with the block's offset reduced from the raw block sums by the block itself
// (nb <= 4 kScanThreads), so the single-block scan of the block sums is not a launch of its own;
// the last block writes the total to out[n]
__global__ void scan_apply_prefix_kernel(const int32_t* __restrict__ in, int32_t n, const int32_t* __restrict__ bsum,
                                         int32_t nb, int32_t* __restrict__ out) {
    __shared__ int32_t tile[kScanTile];
    __shared__ int32_t wt[32];
    __shared__ int32_t tot;
    __shared__ int32_t pre;
    int32_t v = 0;
    for (int32_t i = threadIdx.x; i < (int32_t)blockIdx.x; i += kScanThreads) v += bsum[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) wt[threadIdx.x >> 5] = v;
    const int64_t base = (int64_t)blockIdx.x * kScanTile;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = base + k * kScanThreads + threadIdx.x;
        tile[k * kScanThreads + threadIdx.x] = i < n ? in[i] : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += wt[w];
        pre = t;
        if ((int32_t)blockIdx.x == nb - 1) out[n] = t + bsum[nb - 1];
    }
    __syncthreads();
    int32_t loc[kScanItems];
    int32_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        loc[k] = s;
        s += tile[threadIdx.x * kScanItems + k];
    }
    int32_t ex = block_exclusive_scan(s, wt, &tot) + pre;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) tile[threadIdx.x * kScanItems + k] = ex + loc[k];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        int64_t i = base + k * kScanThreads + threadIdx.x;
        if (i < n) out[i] = tile[k * kScanThreads + threadIdx.x];
    }
}

// ---------------------------------------------------------------- B4 row sort + dedup
__device__ __forceinline__ int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// warp-cooperative bitonic sort of buf[0..P) (P power of two) in shared memory
__device__ __forceinline__ void warp_bitonic(int32_t* buf, int P, int lane) {
    for (int k = 2; k <= P; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < P; i += 32) {
                int ixj = i ^ j;
                if (ixj > i) {
                    int32_t a = buf[i], b = buf[ixj];
                    bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        buf[i] = b;
                        buf[ixj] = a;
                    }
                }
            }
            __syncwarp();
        }
    }
}

// Sort + dedup seg[0..len) (len <= 32*E) in place with one warp; returns the unique count.
// Element i = h*32 + lane lives in a[h]; bitonic stages with partner distance j < 32 use
// shuffles, j >= 32 exchange registers within the lane.  All lanes must call it (converged).
template <int E>
__device__ __forceinline__ int warp_sort_dedup(int32_t* seg, int len, int lane) {
    int32_t a[E];
#pragma unroll
    for (int h = 0; h < E; ++h) a[h] = h * 32 + lane < len ? seg[h * 32 + lane] : INT_MAX;
    int P = 32;
    while (P < len) P <<= 1;
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
        if (k > P) continue;  // warp-uniform; `continue` keeps the loop fully unrolled (static indices)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int hj = j >> 5;
#pragma unroll
                for (int h = 0; h < E; ++h) {
                    if (h & hj) continue;  // (h, h | hj) pairs, handled from the lower index
                    const int i = h * 32 + lane;
                    const bool up = (i & k) == 0;
                    const int32_t x = a[h], y = a[h | hj];
                    a[h] = up ? min(x, y) : max(x, y);
                    a[h | hj] = up ? max(x, y) : min(x, y);
                }
            } else {
#pragma unroll
                for (int h = 0; h < E; ++h) {
                    const int i = h * 32 + lane;
                    const int32_t b = __shfl_xor_sync(0xffffffffu, a[h], j);
                    const bool up = (i & k) == 0, lower = (i & j) == 0;
                    a[h] = (lower == up) ? min(a[h], b) : max(a[h], b);
                }
            }
        }
    }
    // dedup: keep the first of each run of equal values, compact in order
    int base = 0;
    int32_t carry = 0;  // last element of the previous register row
#pragma unroll
    for (int h = 0; h < E; ++h) {
        const int i = h * 32 + lane;
        int32_t prev = __shfl_up_sync(0xffffffffu, a[h], 1);
        if (lane == 0) prev = carry;
        carry = __shfl_sync(0xffffffffu, a[h], 31);
        const bool keep = i < len && (i == 0 || a[h] != prev);
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) seg[base + __popc(m & lanemask_lt())] = a[h];
        base += __popc(m);
    }
    return base;
}

// rows of <= 16 entries are sorted by one thread each (a 16-input bitonic network in registers,
// INT_MAX padding), then deduplicated: a warp takes 32 rows at a time (streaming merges and
// sparse graphs are mostly such rows); the warp's longer rows follow one at a time
constexpr int kThreadSortCap = 16;

__device__ __forceinline__ void cas(int32_t& a, int32_t& b, bool up) {
    const int32_t lo = a < b ? a : b, hi = a < b ? b : a;
    a = up ? lo : hi;
    b = up ? hi : lo;
}

__device__ int thread_sort_dedup16(int32_t* row, int len) {
    int32_t v[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) v[k] = k < len ? row[k] : INT_MAX;
#pragma unroll
    for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int ixj = i ^ j;
                if (ixj > i) cas(v[i], v[ixj], (i & k) == 0);
            }
    int u = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k)
        if (k < len && (k == 0 || v[k] != v[k - 1])) row[u++] = v[k];
    return u;
}

__device__ void warp_sort_row(int32_t* __restrict__ tmp, int32_t* __restrict__ ucnt, int32_t* buf, int64_t r,
                              int32_t o, int len, int lane) {
    if (len <= 256) {  // registers: up to 8 elements per lane, bitonic network over shuffles
        const int u = len <= 64    ? warp_sort_dedup<2>(tmp + o, len, lane)
                      : len <= 128 ? warp_sort_dedup<4>(tmp + o, len, lane)
                                   : warp_sort_dedup<8>(tmp + o, len, lane);  // len is warp-uniform
        if (lane == 0) ucnt[r] = u;
        return;
    }
    const int P = next_pow2(len);
    for (int i = lane; i < P; i += 32) buf[i] = i < len ? tmp[o + i] : INT_MAX;
    __syncwarp();
    warp_bitonic(buf, P, lane);
    int base = 0;
    for (int i0 = 0; i0 < len; i0 += 32) {
        const int i = i0 + lane;
        bool keep = false;
        int32_t v = 0;
        if (i < len) {
            v = buf[i];
            keep = (i == 0) || (v != buf[i - 1]);
        }
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        if (keep) tmp[o + base + __popc(m & lanemask_lt())] = v;
        base += __popc(m);
    }
    if (lane == 0) ucnt[r] = base;
    __syncwarp();
}

__global__ void __launch_bounds__(256) sort_rows_warp_kernel(const int32_t* __restrict__ off, int32_t* __restrict__ tmp,
                                                             int32_t* __restrict__ ucnt, int32_t n,
                                                             int32_t* __restrict__ big_list, int32_t* __restrict__ big_count,
                                                             int32_t* __restrict__ giant_list,
                                                             int32_t* __restrict__ giant_count) {
    __shared__ int32_t sbuf[8][kWarpSortCap];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t* buf = sbuf[warp];
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    for (int64_t r0 = ((int64_t)blockIdx.x * 8 + warp) * 32; r0 < n; r0 += nwarps * 32) {
        // one row per lane: short rows sorted by their lane, the others collected
        const int64_t r = r0 + lane;
        int32_t o = 0;
        int len = 0;
        bool warp_row = false;
        if (r < n) {
            o = off[r];
            len = off[r + 1] - o;
            if (len > kWarpSortCap) {
                if (len <= kBlockSortCap) big_list[atomicAdd(big_count, 1)] = (int32_t)r;
                else giant_list[atomicAdd(giant_count, 1)] = (int32_t)r;
            } else if (len <= kThreadSortCap) {
                ucnt[r] = len <= 1 ? len : thread_sort_dedup16(tmp + o, len);
            } else {
                warp_row = true;
            }
        }
        unsigned pending = __ballot_sync(0xffffffffu, warp_row);
        while (pending) {
            const int src = __ffs(pending) - 1;
            pending &= pending - 1;
            const int32_t ro = __shfl_sync(0xffffffffu, o, src);
            const int rl = __shfl_sync(0xffffffffu, len, src);
            warp_sort_row(tmp, ucnt, buf, r0 + src, ro, rl, lane);
        }
    }
}

// one block (1024 threads) per row with kWarpSortCap < len <= kBlockSortCap
__global__ void __launch_bounds__(1024) sort_rows_block_kernel(const int32_t* __restrict__ off, int32_t* __restrict__ tmp,
                                                               int32_t* __restrict__ ucnt,
                                                               const int32_t* __restrict__ big_list,
                                                               const int32_t* __restrict__ big_count) {
    extern __shared__ int32_t buf[];  // kBlockSortCap
    __shared__ int32_t wt[32];
    __shared__ int32_t tot;
    const int32_t cnt = *big_count;
    for (int64_t b = blockIdx.x; b < cnt; b += gridDim.x) {
        const int32_t r = big_list[b];
        const int32_t o = off[r];
        const int len = off[r + 1] - o;
        const int P = next_pow2(len);
        for (int i = threadIdx.x; i < P; i += blockDim.x) buf[i] = i < len ? tmp[o + i] : INT_MAX;
        __syncthreads();
        for (int k = 2; k <= P; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < P; i += blockDim.x) {
                    int ixj = i ^ j;
                    if (ixj > i) {
                        int32_t a = buf[i], c = buf[ixj];
                        bool up = (i & k) == 0;
                        if ((a > c) == up) {
                            buf[i] = c;
                            buf[ixj] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
        int32_t base = 0;
        for (int i0 = 0; i0 < len; i0 += blockDim.x) {
            const int i = i0 + threadIdx.x;
            int32_t v = 0, keep = 0;
            if (i < len) {
                v = buf[i];
                keep = (i == 0) || (v != buf[i - 1]);
            }
            int32_t pos = block_exclusive_scan(keep, wt, &tot);
            if (keep) tmp[o + base + pos] = v;
            base += tot;
        }
        if (threadIdx.x == 0) ucnt[r] = base;
        __syncthreads();
    }
}

// one block (1024 threads) per row with len > kBlockSortCap: N-bit bitmap (sorted + unique by construction)
__global__ void __launch_bounds__(1024) sort_rows_giant_kernel(const int32_t* __restrict__ off, int32_t* __restrict__ tmp,
                                                               int32_t* __restrict__ ucnt,
                                                               const int32_t* __restrict__ giant_list,
                                                               const int32_t* __restrict__ giant_count,
                                                               uint32_t* __restrict__ bitmap, int32_t n) {
    __shared__ int32_t wt[32];
    __shared__ int32_t tot;
    const int32_t words = (int32_t)(((int64_t)n + 31) >> 5);
    uint32_t* bm = bitmap + (int64_t)blockIdx.x * words;
    const int32_t cnt = *giant_count;
    const int32_t per = (words + blockDim.x - 1) / blockDim.x;
    for (int64_t b = blockIdx.x; b < cnt; b += gridDim.x) {
        const int32_t r = giant_list[b];
        const int32_t o = off[r];
        const int32_t len = off[r + 1] - o;
        for (int32_t w = threadIdx.x; w < words; w += blockDim.x) bm[w] = 0u;
        __syncthreads();
        for (int32_t i = threadIdx.x; i < len; i += blockDim.x) {
            const int32_t v = tmp[o + i];
            atomicOr(bm + (v >> 5), 1u << (v & 31));
        }
        __syncthreads();
        const int32_t w0 = threadIdx.x * per, w1 = min(words, w0 + per);
        int32_t c = 0;
        for (int32_t w = w0; w < w1; ++w) c += __popc(bm[w]);
        int32_t pos = block_exclusive_scan(c, wt, &tot);
        for (int32_t w = w0; w < w1; ++w) {
            uint32_t bits = bm[w];
            while (bits) {
                const int t = __ffs(bits) - 1;
                tmp[o + pos++] = (w << 5) + t;
                bits &= bits - 1;
            }
        }
        if (threadIdx.x == 0) ucnt[r] = tot;
        __syncthreads();
    }
}

// ---------------------------------------------------------------- B5 compact
__global__ void compact_kernel(const int32_t* __restrict__ off, const int32_t* __restrict__ tmp,
                               const int32_t* __restrict__ row_ptr, int32_t* __restrict__ col_idx, int32_t n) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += nwarps) {
        const int32_t src = off[r], dst = row_ptr[r], len = row_ptr[r + 1] - dst;
        for (int32_t i = lane; i < len; i += 32) {
            IGP_DASSERT(tmp[src + i] >= 0 && tmp[src + i] < n);
            col_idx[dst + i] = tmp[src + i];
        }
    }
}

// ---------------------------------------------------------------- row schedule (degree-descending order)
// Bucket key = kDegBuckets-1-min(deg, kDegBuckets-1), sorted stably (ties by ascending id):
// the order is deterministic, so the per-row summation order and the output are too.
constexpr int kDegBuckets = 1024;

__device__ __forceinline__ int deg_key(const int32_t* rp, int32_t i) {
    const int32_t deg = rp[i + 1] - rp[i];
    return kDegBuckets - 1 - (deg < kDegBuckets - 1 ? deg : kDegBuckets - 1);
}

// ---------------------------------------------------------------- stable LSD counting-sort passes
// Sort (key, val) pairs by key, stably (equal keys keep their input order), one 2^kDigitBits
// digit per pass: per-tile digit histograms (key-major, so one exclusive scan gives every
// (digit, tile) its output offset), then one warp per tile walks its elements in order and
// ranks equal digits with __match_any_sync.  Used for the row orders (degree buckets; labels
// over the degree order), which must be deterministic.
constexpr int kDigitBits = 12;
constexpr int kDigits = 1 << kDigitBits;
constexpr int kSortTile = 2048;  // largest tile; graphs with few nodes use smaller tiles (more warps)

// tile of the stable sort passes for n elements: enough tiles to give every SM several warps
int sort_tile(int32_t n, int num_sms) {
    int t = 256;
    while (t < kSortTile && (int64_t)n / (2 * t) >= (int64_t)num_sms * 8) t *= 2;
    return t;
}

__global__ void degree_keys_kernel(const int32_t* __restrict__ rp, int32_t n, int32_t* __restrict__ keys,
                                   int32_t* __restrict__ vals) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        keys[i] = deg_key(rp, (int32_t)i);
        vals[i] = (int32_t)i;
    }
}

__global__ void label_keys_kernel(const int32_t* __restrict__ order, const int32_t* __restrict__ lab, int32_t n,
                                  int32_t* __restrict__ keys, int32_t* __restrict__ vals) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += stride) {
        const int32_t v = order[k];
        keys[k] = lab[v];
        vals[k] = v;
    }
}

// `nd` digits of the pass (a power of 2 <= kDigits), `tile` elements per tile
__global__ void __launch_bounds__(256) tile_digit_hist_kernel(const int32_t* __restrict__ keys, int32_t n, int shift,
                                                              int nd, int tile, int32_t ntiles, int32_t* __restrict__ H) {
    __shared__ int32_t h[kDigits];
    for (int b = threadIdx.x; b < nd; b += blockDim.x) h[b] = 0;
    __syncthreads();
    const int64_t t0 = (int64_t)blockIdx.x * tile;
    for (int i = threadIdx.x; i < tile; i += blockDim.x)
        if (t0 + i < n) atomicAdd(&h[(keys[t0 + i] >> shift) & (nd - 1)], 1);
    __syncthreads();
    for (int b = threadIdx.x; b < nd; b += blockDim.x) H[(int64_t)b * ntiles + blockIdx.x] = h[b];
}

__global__ void __launch_bounds__(32) tile_digit_scatter_kernel(const int32_t* __restrict__ keys,
                                                                const int32_t* __restrict__ vals, int32_t n,
                                                                int shift, int nd, int tile, int32_t ntiles,
                                                                const int32_t* __restrict__ Hs,
                                                                int32_t* __restrict__ okeys,
                                                                int32_t* __restrict__ ovals) {
    __shared__ int32_t cnt[kDigits];
    const int lane = threadIdx.x;
    for (int b = lane; b < nd; b += 32) cnt[b] = 0;
    __syncwarp();
    const int64_t t0 = (int64_t)blockIdx.x * tile;
    for (int c = 0; c < tile; c += 32) {
        const int64_t i = t0 + c + lane;
        const bool act = i < n;
        const unsigned am = __ballot_sync(0xffffffffu, act);
        if (am == 0u) break;
        int32_t key = 0, val = 0, dg = -1;
        if (act) {
            key = keys[i];
            val = vals[i];
            dg = (key >> shift) & (nd - 1);
        }
        if (act) {
            const unsigned peers = __match_any_sync(am, dg);
            const int leader = __ffs(peers) - 1;
            const int32_t base = cnt[dg];  // read by all peers before the leader updates it
            __syncwarp(am);
            if (lane == leader) cnt[dg] = base + __popc(peers);
            const int64_t pos = (int64_t)Hs[(int64_t)dg * ntiles + blockIdx.x] + base + __popc(peers & lanemask_lt());
            IGP_DASSERT(pos >= 0 && pos < n);
            okeys[pos] = key;
            ovals[pos] = val;
        }
        __syncwarp();
    }
}

int grid_for(int64_t work, int threads, int num_sms, int per_sm) {
    int64_t g = (work + threads - 1) / threads;
    int64_t cap = (int64_t)num_sms * per_sm;
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

namespace {
__global__ void degrees_kernel(const int32_t* __restrict__ rp, int32_t n, int32_t* __restrict__ deg) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) deg[i] = rp[i + 1] - rp[i];
}
}  // namespace

igp_status launch_degrees(const int32_t* rp, int32_t n, int32_t* deg, cudaStream_t s) {
    DeviceInfo di;
    if (!device_info(&di)) return IGP_ERR_CUDA;
    degrees_kernel<<<grid_for(n, 256, di.num_sms, 8), 256, 0, s>>>(rp, n, deg);
    return launch_status("degrees_kernel");
}

igp_status scan_exclusive(const int32_t* in, int32_t* out, int32_t n, cudaStream_t s) {
    const int32_t nb = (n + kScanTile - 1) / kScanTile;
    int32_t* bsum = nullptr;
    IGP_CUDA(alloc_async((void**)&bsum, sizeof(int32_t) * (size_t)(nb > 0 ? nb : 1), s), "scan alloc");
    if (nb > 0) {
        scan_reduce_kernel<<<nb, kScanThreads, 0, s>>>(in, n, bsum);
        IGP_TRY(launch_status("scan_reduce_kernel"));
    }
    if (nb > 0 && nb <= 4 * kScanThreads) {  // up to ~2M elements: two launches
        scan_apply_prefix_kernel<<<nb, kScanThreads, 0, s>>>(in, n, bsum, nb, out);
        IGP_TRY(launch_status("scan_apply_prefix_kernel"));
        free_async(bsum, s);
        return IGP_OK;
    }
    scan_blocksums_kernel<<<1, 1024, 0, s>>>(bsum, nb, out + n);
    IGP_TRY(launch_status("scan_blocksums_kernel"));
    if (nb > 0) {
        scan_apply_kernel<<<nb, kScanThreads, 0, s>>>(in, n, bsum, out);
        IGP_TRY(launch_status("scan_apply_kernel"));
    }
    free_async(bsum, s);
    return IGP_OK;
}

namespace {

// ---------------------------------------------------------------- B6 degree-sorted relabelling
// order[r] = original id of new row r (descending degree, ascending id within a degree
// bucket after the segmented sort: deterministic); inv[order[r]] = r.
__global__ void inverse_perm_kernel(const int32_t* __restrict__ order, int32_t n, int32_t* __restrict__ inv,
                                    const int32_t* __restrict__ rp, int32_t* __restrict__ degp) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += stride) {
        const int32_t o = order[r];
        inv[o] = (int32_t)r;
        degp[r] = rp[o + 1] - rp[o];
    }
}

// new row r takes original row order[r] with every neighbour id mapped through inv
__global__ void perm_scatter_kernel(const int32_t* __restrict__ order, const int32_t* __restrict__ inv,
                                    const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                    const int32_t* __restrict__ rpp, int32_t* __restrict__ cip, int32_t n) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += nw) {
        const int32_t o = order[r];
        const int32_t src = rp[o], len = rp[o + 1] - src, dst = rpp[r];
        for (int32_t k = lane; k < len; k += 32) {
            IGP_DASSERT(ci[src + k] >= 0 && ci[src + k] < n && inv[ci[src + k]] >= 0 && inv[ci[src + k]] < n);
            cip[dst + k] = inv[ci[src + k]];
        }
    }
}

struct SortScratch {
    int32_t* big_list;     // capacity >= number of segments
    int32_t* giant_list;   // capacity >= number of segments
    int32_t* counters;     // [2]
    uint32_t* bitmap;      // kGiantBlocks x ceil(value_range / 32) words
};

// sort (and dedup) every segment data[off[k] .. off[k+1]) ascending; ucnt[k] = unique count
igp_status segmented_sort(const int32_t* off, int32_t* data, int32_t* ucnt, int32_t nseg, int64_t max_len,
                          int32_t value_range, const SortScratch& sc, cudaStream_t s, const DeviceInfo& di) {
    IGP_CUDA(cudaMemsetAsync(sc.counters, 0, 2 * sizeof(int32_t), s), "memset");
    const int rg = grid_for((int64_t)nseg * 32, 256, di.num_sms, 8);
    sort_rows_warp_kernel<<<rg, 256, 0, s>>>(off, data, ucnt, nseg, sc.big_list, sc.counters, sc.giant_list,
                                             sc.counters + 1);
    IGP_TRY(launch_status("sort_rows_warp_kernel"));
    if (max_len > kWarpSortCap) {
        cudaFuncSetAttribute(sort_rows_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kBlockSortCap * (int)sizeof(int32_t));
        sort_rows_block_kernel<<<di.num_sms, 1024, kBlockSortCap * sizeof(int32_t), s>>>(off, data, ucnt, sc.big_list,
                                                                                         sc.counters);
        IGP_TRY(launch_status("sort_rows_block_kernel"));
        if (max_len > kBlockSortCap) {
            sort_rows_giant_kernel<<<kGiantBlocks, 1024, 0, s>>>(off, data, ucnt, sc.giant_list, sc.counters + 1,
                                                                 sc.bitmap, value_range);
            IGP_TRY(launch_status("sort_rows_giant_kernel"));
        }
    }
    return IGP_OK;
}

}  // namespace

namespace {

struct PairSortScratch {
    int32_t* keys[2];
    int32_t* vals[2];
    int32_t* H;   // kDigits x ntiles + 1
    int32_t* Hs;  // exclusive scan of H
};

// stable sort of (keys, vals) (n pairs, in scratch keys[0]/vals[0]) by the low `key_bits` bits of
// the key; the sorted values are written to `out` (which may be one of the scratch buffers)
igp_status stable_sort_pairs(int32_t n, int key_bits, const PairSortScratch& sc, int32_t* out, cudaStream_t s,
                             const DeviceInfo& di) {
    const int tile = sort_tile(n, di.num_sms);
    const int32_t ntiles = (n + tile - 1) / tile;
    int cur = 0;
    for (int shift = 0; shift < key_bits; shift += kDigitBits) {
        const bool last = shift + kDigitBits >= key_bits;
        const int bits = key_bits - shift < kDigitBits ? key_bits - shift : kDigitBits;
        const int nd = 1 << bits;
        tile_digit_hist_kernel<<<ntiles, 256, 0, s>>>(sc.keys[cur], n, shift, nd, tile, ntiles, sc.H);
        IGP_TRY(launch_status("tile_digit_hist_kernel"));
        IGP_TRY(scan_exclusive(sc.H, sc.Hs, nd * ntiles, s));
        int32_t* ov = last ? out : sc.vals[cur ^ 1];
        tile_digit_scatter_kernel<<<ntiles, 32, 0, s>>>(sc.keys[cur], sc.vals[cur], n, shift, nd, tile, ntiles, sc.Hs,
                                                        sc.keys[cur ^ 1], ov);
        IGP_TRY(launch_status("tile_digit_scatter_kernel"));
        cur ^= 1;
    }
    return IGP_OK;
}

}  // namespace

// Streaming merge (Alg. 2 l.1): row r of the union = the sorted, duplicate-free
// merge of the base graph's canonical row B (sorted, unique) and the new edges' row U (sorted and
// deduplicated on their own first).
//  - merge_count_kernel (one thread per row): drops the entries of U already in B (binary search),
//    compacting the rest U' in place; |row| = |B| + |U'|.
//  - merge_write_kernel (one warp per row): B[i] goes to position i + #{U' < B[i]}, U'[j] to
//    j + #{B < U'[j]}: both sides written straight into the final CSR, B read coalesced.
__device__ __forceinline__ int32_t lower_bound_i32(const int32_t* __restrict__ a, int32_t n, int32_t x) {
    int32_t lo = 0, hi = n;
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void merge_count_kernel(const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                                   const int32_t* __restrict__ noff, int32_t* __restrict__ ndata,
                                   int32_t* __restrict__ ncnt, int32_t n, int32_t* __restrict__ ucnt) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += stride) {
        const int32_t b0 = brp[r], nb = brp[r + 1] - b0;
        const int32_t u0 = noff[r], nu = ncnt[r];
        int32_t w = 0;
        for (int32_t j = 0; j < nu; ++j) {
            const int32_t u = ndata[u0 + j];
            const int32_t pos = lower_bound_i32(bci + b0, nb, u);
            if (pos == nb || bci[b0 + pos] != u) ndata[u0 + w++] = u;  // not in B: kept (in order)
        }
        ncnt[r] = w;
        ucnt[r] = nb + w;
    }
}

// PERM: the relabelled CSR is written in the same pass (row order computed from the merged
// degrees before this kernel): row r's entries also go, mapped through inv, to relabelled row
// inv[r] at the same positions (a relabelled row keeps the canonical neighbour order), so no
// separate relabelling pass re-reads the merged CSR
template <bool PERM>
__global__ void merge_write_kernel(const int32_t* __restrict__ brp, const int32_t* __restrict__ bci,
                                   const int32_t* __restrict__ noff, const int32_t* __restrict__ ndata,
                                   const int32_t* __restrict__ ncnt, int32_t n, const int32_t* __restrict__ row_ptr,
                                   int32_t* __restrict__ col_idx, const int32_t* __restrict__ inv,
                                   const int32_t* __restrict__ rpp, int32_t* __restrict__ cip) {
    const int lane = threadIdx.x & 31;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += nwarps) {
        const int32_t b0 = brp[r], nb = brp[r + 1] - b0;
        const int32_t* U = ndata + noff[r];
        const int32_t nu = ncnt[r];
        int32_t* out = col_idx + row_ptr[r];
        int32_t* outp = PERM ? cip + rpp[inv[r]] : nullptr;
        for (int32_t i = lane; i < nb; i += 32) {
            const int32_t x = bci[b0 + i];
            const int32_t pos = i + lower_bound_i32(U, nu, x);
            out[pos] = x;
            if (PERM) outp[pos] = inv[x];
        }
        for (int32_t j = lane; j < nu; j += 32) {
            const int32_t u = U[j];
            const int32_t pos = j + lower_bound_i32(bci + b0, nb, u);
            out[pos] = u;
            if (PERM) outp[pos] = inv[u];
        }
    }
}

__global__ void iota_kernel(int32_t* __restrict__ a, int32_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) a[i] = (int32_t)i;
}

// ---------------------------------------------------------------- B7 community row order (optional)
// Label propagation, one warp per row: the new label of row r is the most frequent label among
// its first (up to) 31 neighbours (canonical order) and r itself, ties to the smallest label.
// Synchronous sweeps (lin -> lout) make the result independent of scheduling.
__global__ void __launch_bounds__(256) label_prop_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                         int32_t n, const int32_t* __restrict__ lin,
                                                         int32_t* __restrict__ lout) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += nw) {
        const int32_t beg = rp[r];
        const int len = min(rp[r + 1] - beg, 31);
        const bool act = lane <= len;
        int32_t lab = INT_MAX;
        if (lane < len) {
            IGP_DASSERT(ci[beg + lane] >= 0 && ci[beg + lane] < n);
            lab = lin[ci[beg + lane]];
        }
        else if (lane == len) lab = lin[r];
        const unsigned am = __ballot_sync(0xffffffffu, act);
        int cnt = 0;
        if (act) cnt = __popc(__match_any_sync(am, lab));
        const int best = __reduce_max_sync(0xffffffffu, cnt);
        const int32_t l = __reduce_min_sync(0xffffffffu, (act && cnt == best) ? lab : INT_MAX);
        if (lane == 0) lout[r] = l;
    }
}

// label-propagation sweep 1 from lin[i] = i (all counts 1): the smallest id among the node and its
// first <= 31 neighbours; neighbours are in ascending order, so that is min(i, first neighbour)
__global__ void lp_first_sweep_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, int32_t n,
                                      int32_t* __restrict__ lout) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int32_t beg = rp[i];
        lout[i] = rp[i + 1] > beg ? min((int32_t)i, ci[beg]) : (int32_t)i;
    }
}

void free_csr(const CsrDevice& c, cudaStream_t s) {
    free_async(c.row_ptr, s);
    free_async(c.col_idx, s);
    free_async(c.order, s);
    free_async(c.meta, s);
    free_async(c.labels, s);
    if (!c.perm_alias) {
        free_async(c.rp_perm, s);
        free_async(c.col_perm, s);
    }
}

igp_status build_csr(const int32_t* d_edges, int64_t E, int32_t n, RowOrder row_order, cudaStream_t s,
                     CsrDevice* out, const CsrDevice* base) {
    const bool reorder = row_order != kOrderNone;
    const bool community = row_order == kOrderCommunity;
    DeviceInfo di;
    if (!device_info(&di)) return IGP_ERR_CUDA;
    // both orientations of the new edges (before dedup / self-loop removal), plus the base rows
    const int64_t raw = 2 * E + (base ? base->cap : 0);
    if (raw > kMaxEntries) {
        set_error("edge count exceeds the int32 CSR index range");
        return IGP_ERR_UNSUPPORTED;
    }
    const int32_t words = (int32_t)(((int64_t)n + 31) >> 5);
    const int32_t lists = n > kDegBuckets ? n : kDegBuckets;
    // temporaries in one stream-ordered block
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t o_cnt = 0;
    size_t o_off = al(o_cnt + sizeof(int32_t) * (size_t)n);
    size_t o_ucnt = al(o_off + sizeof(int32_t) * ((size_t)n + 1));
    size_t o_big = al(o_ucnt + sizeof(int32_t) * (size_t)lists);
    size_t o_giant = al(o_big + sizeof(int32_t) * (size_t)lists);
    size_t o_flags = al(o_giant + sizeof(int32_t) * (size_t)lists);  // err, sort counters
    size_t o_inv = al(o_flags + 4 * sizeof(int32_t));
    size_t o_degp = al(o_inv + sizeof(int32_t) * (size_t)n);
    size_t o_bitmap = al(o_degp + sizeof(int32_t) * (size_t)n);
    size_t o_tmp = al(o_bitmap + sizeof(uint32_t) * (size_t)words * kGiantBlocks);
    // stable pair sorts of the row orders: keys / vals double buffers and tile digit histograms
    const int32_t ntiles = (n + sort_tile(n, di.num_sms) - 1) / sort_tile(n, di.num_sms);
    const size_t hbytes = al(sizeof(int32_t) * ((size_t)kDigits * ntiles + 1));
    size_t o_psort = al(o_tmp + sizeof(int32_t) * (size_t)(raw > 0 ? raw : 1));
    size_t o_comm = o_psort + (reorder ? al(sizeof(int32_t) * (size_t)n) * 4 + 2 * hbytes : 0);
    // community order: two label buffers, label bucket offsets / fill, bucketed ranks, degree order
    const size_t comm_bytes = community ? al(sizeof(int32_t) * (size_t)n) * 2 : 0;  // two label buffers
    size_t total = o_comm + comm_bytes;
    char* ws = nullptr;
    IGP_CUDA(alloc_async((void**)&ws, total, s), "build workspace alloc");
    int32_t* cnt = (int32_t*)(ws + o_cnt);
    int32_t* off = (int32_t*)(ws + o_off);
    int32_t* ucnt = (int32_t*)(ws + o_ucnt);
    int32_t* flags = (int32_t*)(ws + o_flags);
    int32_t* inv = (int32_t*)(ws + o_inv);
    int32_t* degp = (int32_t*)(ws + o_degp);
    int32_t* tmp = (int32_t*)(ws + o_tmp);
    SortScratch sc{(int32_t*)(ws + o_big), (int32_t*)(ws + o_giant), flags, (uint32_t*)(ws + o_bitmap)};
    PairSortScratch psc{};
    if (reorder) {
        const size_t nb4 = al(sizeof(int32_t) * (size_t)n);
        psc.keys[0] = (int32_t*)(ws + o_psort);
        psc.vals[0] = (int32_t*)(ws + o_psort + nb4);
        psc.keys[1] = (int32_t*)(ws + o_psort + 2 * nb4);
        psc.vals[1] = (int32_t*)(ws + o_psort + 3 * nb4);
        psc.H = (int32_t*)(ws + o_psort + 4 * nb4);
        psc.Hs = (int32_t*)(ws + o_psort + 4 * nb4 + hbytes);
    }

    CsrDevice c;
    c.n = n;
    c.cap = raw;
    // the column arrays are sized by the entries before deduplication, so nothing on the
    // host waits for nnz; vector index loads may read up to kColPad entries past a row
    const size_t cbytes = sizeof(int32_t) * (size_t)(raw + kColPad);
    igp_status st =
        cuda_status(alloc_async((void**)&c.row_ptr, sizeof(int32_t) * ((size_t)n + 1 + kRpPad), s), "alloc");
    if (st == IGP_OK) st = cuda_status(alloc_async((void**)&c.order, sizeof(int32_t) * (size_t)n, s), "alloc");
    if (st == IGP_OK) st = cuda_status(alloc_async((void**)&c.meta, 4 * sizeof(int32_t), s), "alloc");
    if (st == IGP_OK) st = cuda_status(alloc_async((void**)&c.col_idx, cbytes, s), "col_idx alloc");
    // row-pointer arrays padded by kRpPad entries: 16-byte bulk copies of a slice may overrun the end
    if (st == IGP_OK && reorder)
        st = cuda_status(alloc_async((void**)&c.rp_perm, sizeof(int32_t) * ((size_t)n + 1 + kRpPad), s), "alloc");
    if (st == IGP_OK && reorder) st = cuda_status(alloc_async((void**)&c.col_perm, cbytes, s), "col_perm alloc");
    if (st == IGP_OK && community)
        st = cuda_status(alloc_async((void**)&c.labels, sizeof(int32_t) * (size_t)n, s), "labels alloc");
    if (!reorder) c.perm_alias = true;
    cudaEvent_t ev_csr = nullptr, ev_lp = nullptr;  // community order: side-stream fork / join
    auto fail = [&](igp_status e) {
        if (ev_lp) cudaStreamWaitEvent(s, ev_lp, 0);  // never free under the side stream's work
        if (ev_csr) cudaEventDestroy(ev_csr);
        if (ev_lp) cudaEventDestroy(ev_lp);
        free_async(ws, s);
        free_csr(c, s);
        return e;
    };
    if (st != IGP_OK) return fail(st);
#define IGP_STEP(expr)                                  \
    do {                                                \
        igp_status _s = (expr);                         \
        if (_s != IGP_OK) return fail(_s);              \
    } while (0)
    IGP_STEP(cuda_status(cudaMemsetAsync(flags, 0, 4 * sizeof(int32_t), s), "memset"));
    // range-error flag: a merge inherits the base graph's (asynchronous builds report it lazily)
    if (base)
        IGP_STEP(cuda_status(cudaMemcpyAsync(c.meta, base->meta, 4 * sizeof(int32_t), cudaMemcpyDeviceToDevice, s),
                             "meta copy"));
    else
        IGP_STEP(cuda_status(cudaMemsetAsync(c.meta, 0, 4 * sizeof(int32_t), s), "memset"));
    IGP_STEP(cuda_status(cudaMemsetAsync(c.col_idx + raw, 0, sizeof(int32_t) * kColPad, s), "pad memset"));
    if (reorder) IGP_STEP(cuda_status(cudaMemsetAsync(c.col_perm + raw, 0, sizeof(int32_t) * kColPad, s), "pad memset"));
    // B1-B3: count, scan, scatter both orientations of the NEW edges into row buckets
    IGP_STEP(cuda_status(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)n, s), "memset"));
    const int eg = grid_for(E, 256, di.num_sms, 16);
    if (E > 0) {
        count_kernel<<<eg, 256, 0, s>>>(d_edges, E, n, cnt, c.meta);
        IGP_STEP(launch_status("count_kernel"));
    }
    IGP_STEP(scan_exclusive(cnt, off, n, s));
    IGP_STEP(cuda_status(cudaMemsetAsync(c.row_ptr + n + 1, 0, kRpPad * sizeof(int32_t), s), "pad memset"));
    const int rg = grid_for((int64_t)n * 32, 256, di.num_sms, 8);
    // a streaming merge in degree order writes the relabelled CSR in the merge pass itself
    const bool fused = base != nullptr && reorder && !community;
    if (E > 0) {
        IGP_STEP(cuda_status(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (size_t)n, s), "memset"));
        scatter_kernel<<<eg, 256, 0, s>>>(d_edges, E, n, off, cnt, tmp);
        IGP_STEP(launch_status("scatter_kernel"));
    }
    // B4: per-row sort + dedup of the new entries
    IGP_STEP(segmented_sort(off, tmp, base ? cnt : ucnt, n, 2 * E, n, sc, s, di));
    if (base) {
        // streaming merge: the base rows are already canonical; merge each with its sorted new
        // run (no re-sort of the base): count (dropping new entries already present), then write
        // both sides at their merged positions
        const int tg = grid_for(n, 256, di.num_sms, 8);
        merge_count_kernel<<<tg, 256, 0, s>>>(base->row_ptr, base->col_idx, off, tmp, cnt, n, ucnt);
        IGP_STEP(launch_status("merge_count_kernel"));
        IGP_STEP(scan_exclusive(ucnt, c.row_ptr, n, s));
        if (fused) {
            // degree order from the merged row lengths, then one pass writes both CSRs
            const int ng = grid_for(n, 256, di.num_sms, 8);
            degree_keys_kernel<<<ng, 256, 0, s>>>(c.row_ptr, n, psc.keys[0], psc.vals[0]);
            IGP_STEP(launch_status("degree_keys_kernel"));
            IGP_STEP(stable_sort_pairs(n, 10, psc, c.order, s, di));
            inverse_perm_kernel<<<ng, 256, 0, s>>>(c.order, n, inv, c.row_ptr, degp);
            IGP_STEP(launch_status("inverse_perm_kernel"));
            IGP_STEP(scan_exclusive(degp, c.rp_perm, n, s));
            IGP_STEP(cuda_status(cudaMemsetAsync(c.rp_perm + n + 1, 0, kRpPad * sizeof(int32_t), s), "pad memset"));
            merge_write_kernel<true><<<rg, 256, 0, s>>>(base->row_ptr, base->col_idx, off, tmp, cnt, n, c.row_ptr,
                                                        c.col_idx, inv, c.rp_perm, c.col_perm);
            IGP_STEP(launch_status("merge_write_kernel<perm>"));
            free_async(ws, s);
            *out = c;
            return IGP_OK;
        }
        merge_write_kernel<false><<<rg, 256, 0, s>>>(base->row_ptr, base->col_idx, off, tmp, cnt, n, c.row_ptr,
                                                     c.col_idx, nullptr, nullptr, nullptr);
        IGP_STEP(launch_status("merge_write_kernel"));
    } else {
        // B5: row pointers, compaction
        IGP_STEP(scan_exclusive(ucnt, c.row_ptr, n, s));
        if (raw > 0) {
            compact_kernel<<<rg, 256, 0, s>>>(off, tmp, c.row_ptr, c.col_idx, n);
            IGP_STEP(launch_status("compact_kernel"));
        }
    }
    if (!reorder) {  // the filter steps run on the canonical CSR itself
        iota_kernel<<<grid_for(n, 256, di.num_sms, 8), 256, 0, s>>>(c.order, n);  // identity labelling
        IGP_STEP(launch_status("iota_kernel"));
        c.rp_perm = c.row_ptr;
        c.col_perm = c.col_idx;
        free_async(ws, s);
        *out = c;
        return IGP_OK;
    }
    // B7 label propagation (community order) depends only on the canonical CSR: it runs on a
    // side stream while B6a computes the degree order on `s` (LP is bound by the warp-match
    // pipe, the degree sort by loads and ALU, so the two overlap)
    const size_t nb = al(sizeof(int32_t) * (size_t)n);
    int32_t* lab0 = (int32_t*)(ws + o_comm);
    int32_t* lab1 = (int32_t*)(ws + o_comm + nb);
    if (community) {
        cudaStream_t ss = side_stream(di.device);
        IGP_STEP(cuda_status(ss ? cudaSuccess : cudaErrorInvalidResourceHandle, "side stream"));
        IGP_STEP(cuda_status(cudaEventCreateWithFlags(&ev_csr, cudaEventDisableTiming), "event"));
        cudaEvent_t lp = nullptr;
        IGP_STEP(cuda_status(cudaEventCreateWithFlags(&lp, cudaEventDisableTiming), "event"));
        IGP_STEP(cuda_status(cudaEventRecord(ev_csr, s), "event record"));
        IGP_STEP(cuda_status(cudaStreamWaitEvent(ss, ev_csr, 0), "stream wait"));
        const int ng = grid_for(n, 256, di.num_sms, 8);
        igp_status lst = IGP_OK;
        int sweeps = kLabelPropIters;
        if (base && base->labels) {
            // streaming merge: warm start from the previous graph's communities (the new edges
            // only move labels locally), a few sweeps instead of a full propagation
            lst = cuda_status(cudaMemcpyAsync(lab0, base->labels, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice,
                                              ss),
                              "labels copy");
            sweeps = kLabelPropWarmIters + 1;
        } else {
            // sweep 1 from the identity labels in closed form: every label counts once, so the tie rule
            // picks the smallest of {i} and the first <= 31 neighbours, i.e. min(i, first neighbour)
            lp_first_sweep_kernel<<<ng, 256, 0, ss>>>(c.row_ptr, c.col_idx, n, lab0);
            lst = launch_status("lp_first_sweep_kernel");
        }
        for (int it = 1; it < sweeps && lst == IGP_OK; ++it) {
            label_prop_kernel<<<grid_for((int64_t)n * 32, 256, di.num_sms, 8), 256, 0, ss>>>(c.row_ptr, c.col_idx, n,
                                                                                             lab0, lab1);
            lst = launch_status("label_prop_kernel");
            int32_t* t = lab0;
            lab0 = lab1;
            lab1 = t;
        }
        if (lst == IGP_OK)  // kept with the graph: the next merge's warm start
            lst = cuda_status(cudaMemcpyAsync(c.labels, lab0, sizeof(int32_t) * (size_t)n, cudaMemcpyDeviceToDevice, ss),
                              "labels copy");
        if (lst == IGP_OK) lst = cuda_status(cudaEventRecord(lp, ss), "event record");
        if (lst != IGP_OK) {  // drain what was enqueued on the side stream before freeing anything
            cudaStreamSynchronize(ss);
            cudaEventDestroy(lp);
            return fail(lst);
        }
        ev_lp = lp;
    }
    // B6a: degree-descending order, ties by ascending id: one stable counting-sort pass of the
    // ids by degree bucket (also after a streaming merge: measured, keeping the base graph's
    // order instead slows the later stages' filter steps by up to 20%, profiles/r02)
    const int ng = grid_for(n, 256, di.num_sms, 8);
    degree_keys_kernel<<<ng, 256, 0, s>>>(c.row_ptr, n, psc.keys[0], psc.vals[0]);
    IGP_STEP(launch_status("degree_keys_kernel"));
    IGP_STEP(stable_sort_pairs(n, 10, psc, c.order, s, di));  // kDegBuckets = 2^10 keys
    if (community) {
        // B7 (continued): rows grouped by label (descending degree within), after the side
        // stream's label propagation
        IGP_STEP(cuda_status(cudaStreamWaitEvent(s, ev_lp, 0), "stream wait"));
        cudaEventDestroy(ev_csr);  // released by the runtime once complete
        cudaEventDestroy(ev_lp);
        ev_csr = ev_lp = nullptr;
        // stable sort of the degree-ordered node sequence by label: communities in label order,
        // degree order (then id) inside each
        label_keys_kernel<<<ng, 256, 0, s>>>(c.order, lab0, n, psc.keys[0], psc.vals[0]);
        IGP_STEP(launch_status("label_keys_kernel"));
        int lbits = 1;
        while (lbits < 31 && ((int64_t)1 << lbits) < (int64_t)n) ++lbits;  // labels are node ids < n
        IGP_STEP(stable_sort_pairs(n, lbits, psc, c.order, s, di));
    }
    // B6b: the relabelled CSR the filter steps run on (rows by descending degree, or by community)
    inverse_perm_kernel<<<grid_for(n, 256, di.num_sms, 8), 256, 0, s>>>(c.order, n, inv, c.row_ptr, degp);
    IGP_STEP(launch_status("inverse_perm_kernel"));
    IGP_STEP(scan_exclusive(degp, c.rp_perm, n, s));
    IGP_STEP(cuda_status(cudaMemsetAsync(c.rp_perm + n + 1, 0, kRpPad * sizeof(int32_t), s), "pad memset"));
    if (raw > 0) {
        // each relabelled row keeps its canonical neighbour order (ascending original id), so a
        // row's summation order is the same under any permutation (up to where the 128-neighbour
        // fp64 folds of rows longer than 124 fall); no re-sort is needed
        perm_scatter_kernel<<<rg, 256, 0, s>>>(c.order, inv, c.row_ptr, c.col_idx, c.rp_perm, c.col_perm, n);
        IGP_STEP(launch_status("perm_scatter_kernel"));
    }
#undef IGP_STEP
    free_async(ws, s);
    *out = c;
    return IGP_OK;
}

}  // namespace igp
