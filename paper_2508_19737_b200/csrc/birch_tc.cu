// birch_tc.cu — BIRCH predict's nearest-centroid search on the 5th-generation tensor cores.
//
// Labels (Alg. 1 l.7; Alg. 2 l.11) are
//     label_i = argmin_j  d_ij,   d_ij = |c_j|^2 - 2 c_j . x_i      (first minimum, reading B5)
// with d_ij in fp64 in the oracle's operation order (oracle/birch_oracle.c).  Over all rows and
// clusters the scores c_j . x_i form a dense (m x d) . (d x K) contraction, so they run as
// tcgen05.mma (kind::tf32; operands in shared memory, accumulator in TMEM) instead of fp64 FMAs
// on the CUDA cores.  TF32 keeps 11 significant bits, so each operand is split v = hi + lo
// (hi = v rounded to TF32, lo = v - hi) and the three products lo.hi + hi.lo + hi.hi are
// accumulated ("3xTF32"): the result is within a few fp32 ulps of the product sum.
//
// The labels must still be the fp64 labels bit for bit.  The tensor-core pass therefore only
// certifies: a_ij = |c_j|^2 - 2 acc_ij is within a margin M of the fp64 d_ij (M bounds every
// rounding of the split, the products, the fp32 accumulation and the epilogue; DESIGN.md
// §5 "Predict" derives it, with a factor-2 safety).  Three passes:
//   1. every row: 8 (best, index, second) trackers per row; with thr = best + 2M, if every
//      tracker's second exceeds thr the fp64 minimum is among the trackers' bests within thr --
//      one: the label; several (near ties): their d_ij in fp64, in the oracle's order, in the
//      kernel.  Otherwise (M = inf when a magnitude leaves the safe fp32 range) the row is listed
//      with its thr;
//   2. the listed rows as their own row tiles (centroid tiles split over CTA columns when few):
//      every column with a <= thr (a superset of the fp64 minimisers) into a per-row list;
//   3. tc_recheck_kernel: fp64 over each list.  Rows without a usable list (none or > 32
//      candidates) are left listed for birch.cu's fp64 kernel over all clusters.
//
// Kernel layout (birch_tc_kernel<N, collect>: one CTA = 128 rows, warp-specialised, 192 threads):
//   warp 0      : producer -- cp.async.bulk of the row tile (once) and of each N-centroid tile
//                 (hi, lo) in stages of 32 K columns through a 2-stage shared-memory ring,
//                 completion on mbarriers
//   warp 1      : TMEM allocator + MMA issuer (one lane): 3 x d/8 tcgen05.mma (M = 128, N, K = 8)
//                 per tile into one of two N-column TMEM accumulators, tcgen05.commit -> ring
//                 stage / epilogue.  N = 256 for d >= 48 (half the row-tile operand re-reads per
//                 flop), 128 below (where a 256-column epilogue would outlast the MMAs)
//   warps 2..5  : epilogue -- tcgen05.ld of the accumulator (warp w reads TMEM lanes
//                 32(w%4)..+31 = its 32 rows), a = fma(-2, acc, |c|^2), the trackers (pass 1) or
//                 the threshold test (pass 2)
// Operands are pre-arranged in global memory in the UMMA canonical K-major no-swizzle layout
// (core matrices of 8 rows x 16 bytes; row groups SBO = 32 w bytes apart for a block w columns
// wide, K chunks LBO = 128 bytes apart), so every tile stage is ONE contiguous bulk copy.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "igp_internal.cuh"

namespace igp {
namespace {

constexpr int kTcM = 128;      // rows per CTA: MMA M, TMEM lanes
// centroids per tile (MMA N, TMEM columns per accumulator): a template parameter N -- 256 for
// d >= 48 (half the row-tile re-reads per flop: the operand reads share the shared-memory pipe with
// the ring fills), 128 below (there the 256-column epilogue would outlast the tile's MMAs)
constexpr int kTcKC = 32;      // K columns per ring stage (a centroid tile is ceil(d / 32) stages)
constexpr int kTcStages = 2;   // ring depth
constexpr int kTcThreads = 192;
// idesc (kind::tf32): c_format F32 (bits 4-5 = 1), a/b_format TF32 (bits 7-9, 10-12 = 2),
// both K-major (bits 15, 16 = 0), N >> 3 at bits 17-22, M >> 4 at bits 24-28
template <int N>
__host__ __device__ constexpr uint32_t idesc_tf32() {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kTcM >> 4) << 24);
}

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n\t"
        "DONE:\n\t}" ::"r"(sa(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
                 "l"(src), "r"(bytes), "r"(sa(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// shared-memory matrix descriptor: start >> 4 (bits 0-13), LBO >> 4 (16-29), SBO >> 4 (32-45),
// version 1 (46-47), base offset 0, no swizzle (61-63 = 0)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
template <int N>
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %4, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(accumulate), "r"(idesc_tf32<N>())
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(bar)) : "memory");
}
// 64 consecutive fp32 accumulator columns of this thread's TMEM lane: two loads and the wait in
// ONE asm statement, so no use of the registers can be scheduled before the wait
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float (&v)[64]) {
    uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%64];\n\t"
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%65];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr), "r"(taddr + 32u)
        : "memory");
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float to_tf32(float v) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
    return __uint_as_float(r);
}

// stats word: max_j |c_j|^2 as an fp32 bit pattern (non-negative: unsigned max == float max)
enum { S_SQMAX = 0, S_WORDS = 4 };

// Split rows [rows][d] (fp32 or fp64) into TF32 hi / fp32 lo, both written in the tiled
// canonical K-major layout: tile r >> 7, row group (r & 127) >> 3, K chunk k >> 2, row r & 7.
// One thread per row: for a fixed chunk the 32 lanes write 4 row groups x 128 contiguous bytes.
// Rows >= `rows` (padding up to a multiple of 128) are zero.  Rows (T = float): norm[r] = an
// upper bound of |x_r| (NaN / inf propagate).  Centroids (sqn given): sq32[r] = (float)sqn[r]
// (+inf for padding, so padded centroids never win) and stats[S_SQMAX] = max sqn.
// Tiles of TR rows; inside a tile, K chunks of KC columns (the last one d - KC floor(..) wide), each
// chunk a canonical block (row groups 32 w bytes apart for chunk width w) -- rows: TR = 128, KC = d
// (one block per tile); centroids: TR = 256, KC = 32 (one block per ring stage).
template <typename T>
__global__ void tc_split_kernel(const T* __restrict__ src, const int32_t* __restrict__ list, int64_t rows,
                                int64_t rows_pad, int d, int TR, int KC, float* __restrict__ hi, float* __restrict__ lo,
                                float* __restrict__ norm, const double* __restrict__ sqn, float* __restrict__ sq32,
                                unsigned* stats) {
    float smax = 0.f;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows_pad; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t tile = r / TR;
        const int rr = (int)(r - tile * TR);
        float n2 = 0.f;
        for (int c = 0; c < d / 4; ++c) {
            const int k0 = 4 * c, ck = k0 / KC, w = d - ck * KC < KC ? d - ck * KC : KC;
            const int64_t off = tile * (int64_t)TR * d + (int64_t)ck * TR * KC + (rr >> 3) * (int64_t)8 * w +
                                ((k0 - ck * KC) >> 2) * 32 + (rr & 7) * 4;
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (r < rows) {
                const T* p = src + (list ? (int64_t)list[r] : r) * d + 4 * c;
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = (float)p[u];
            }
            float4 vh, vl;
            vh.x = to_tf32(v[0]); vh.y = to_tf32(v[1]); vh.z = to_tf32(v[2]); vh.w = to_tf32(v[3]);
            vl.x = v[0] - vh.x; vl.y = v[1] - vh.y; vl.z = v[2] - vh.z; vl.w = v[3] - vh.w;  // exact in fp32
            *reinterpret_cast<float4*>(hi + off) = vh;
            *reinterpret_cast<float4*>(lo + off) = vl;
            n2 = fmaf(v[0], v[0], fmaf(v[1], v[1], fmaf(v[2], v[2], fmaf(v[3], v[3], n2))));
        }
        // fp32 sum of d squares: relative error below d 2^-24; inflate past it
        if (norm && r < rows) norm[r] = sqrtf(n2 * (1.f + (float)(d + 2) * 0x1p-23f)) * (1.f + 0x1p-20f);
        if (sqn) {
            const float sv = r < rows ? (float)sqn[r] : INFINITY;
            sq32[r] = sv;
            if (r < rows) smax = (sv == sv) ? fmaxf(smax, sv) : INFINITY;
        }
    }
    if (sqn) {
        unsigned u = __float_as_uint(smax);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) u = max(u, __shfl_xor_sync(0xffffffffu, u, o));
        if ((threadIdx.x & 31) == 0) atomicMax(stats + S_SQMAX, u);
    }
}

struct TcArgs {
    const float* xh;  // row tiles, canonical layout
    const float* xl;
    const float* ch;  // centroid tiles, canonical layout
    const float* cl;
    const float* sq;  // [n_tiles * N] |c_j|^2 (fp32), +inf padding
    const float* xnorm;  // [m] upper bounds of |x_i|
    const unsigned* stats;
    const float* X;      // the rows [m][d] and the clusters (fp64), for the exact re-check
    const double* cen;
    const double* sqn;
    int64_t m;     // rows of this launch (a chunk of the call's rows)
    int64_t row0;  // the chunk's first row in the call (amb_rows holds call-level indices)
    int n_tiles;
    int tiles_per_split;  // centroid tiles per CTA column: blockIdx.y takes [y tps, (y+1) tps)
    int d;
    int32_t* labels;
    int32_t* amb_rows;
    unsigned long long* amb_count;  // [0] rows left to the fp64 pass, [1] rows re-checked here in fp64
    float* amb_thr;                 // pass 1: each listed row's threshold best + 2M (beside amb_rows)
    // pass 2 (collect mode): the rows are the listed ones; each row's pass-1 threshold in, every
    // column with a <= threshold out (ccnt counts the appends; past kCandCap only the count grows)
    const float* row_thr;
    int32_t* cand;
    int32_t* ccnt;
};

constexpr int kCandCap = 32;

// d_ij in fp64 exactly as the oracle (and birch.cu's fp64 kernel) evaluates it: eight partial
// sums p[k mod 8] by fma, combined pairwise, then sqn_j + (-2 dot)
__device__ __forceinline__ double exact_dist(const float* __restrict__ x, const double* __restrict__ c, double sq, int d) {
    double p[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int k = 0; k < d; k += 8) {  // d is a multiple of 8 on this path
#pragma unroll
        for (int q = 0; q < 8; ++q) p[q] = __fma_rn(c[k + q], (double)x[k + q], p[q]);
    }
    const double dt = __dadd_rn(__dadd_rn(__dadd_rn(p[0], p[1]), __dadd_rn(p[2], p[3])),
                                __dadd_rn(__dadd_rn(p[4], p[5]), __dadd_rn(p[6], p[7])));
    return __dadd_rn(sq, -2.0 * dt);
}

template <int kTcN, bool kCollect>
__global__ void __launch_bounds__(kTcThreads, 1) birch_tc_kernel(TcArgs a) {
    constexpr int kTcTmemCols = 2 * kTcN;  // two accumulators
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    __shared__ __align__(8) uint64_t bar_full[kTcStages], bar_empty[kTcStages], bar_tfull[2], bar_tempty[2], bar_a;
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(16) float sq_stage[4 * 2 * kTcN];  // epilogue warps' |c_j|^2 tiles
    const int d = a.d;
    const int nc = (d + kTcKC - 1) / kTcKC;  // ring stages per centroid tile
    const uint32_t a_floats = (uint32_t)kTcM * d, a_bytes = 4u * a_floats;
    const uint32_t st_floats = (uint32_t)kTcN * (d < kTcKC ? d : kTcKC);  // one stage's hi (or lo) capacity
    float* sA_hi = reinterpret_cast<float*>(tc_smem);
    float* sA_lo = sA_hi + a_floats;
    float* sB = sA_lo + a_floats;  // stage q: hi at sB + 2 q st_floats, lo right after
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t mt = blockIdx.x;
    const int t0 = blockIdx.y * a.tiles_per_split;  // this CTA's centroid tiles: [t0, t0 + nT)
    const int nT = a.n_tiles - t0 < a.tiles_per_split ? a.n_tiles - t0 : a.tiles_per_split;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&bar_full[s], 1);
            mbar_init(&bar_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&bar_tfull[b], 1);
            mbar_init(&bar_tempty[b], 4);  // one arrival per epilogue warp
        }
        mbar_init(&bar_a, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tmem_slot)),
                     "n"(kTcTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(&bar_a, 2 * a_bytes);
            bulk_g2s(sA_hi, a.xh + mt * a_floats, a_bytes, &bar_a);
            bulk_g2s(sA_lo, a.xl + mt * a_floats, a_bytes, &bar_a);
            for (int t = 0; t < nT; ++t) {
                for (int c = 0; c < nc; ++c) {
                    const int u = t * nc + c, q = u % kTcStages;  // stage use u
                    const int w = d - c * kTcKC < kTcKC ? d - c * kTcKC : kTcKC;
                    const uint32_t bytes = 4u * kTcN * w;
                    if (u >= kTcStages) mbar_wait(&bar_empty[q], (uint32_t)((u / kTcStages - 1) & 1));
                    float* dst = sB + (size_t)2 * q * st_floats;
                    const size_t src = (size_t)(t0 + t) * kTcN * d + (size_t)c * kTcN * kTcKC;
                    mbar_expect_tx(&bar_full[q], 2 * bytes);
                    bulk_g2s(dst, a.ch + src, bytes, &bar_full[q]);
                    bulk_g2s(dst + st_floats, a.cl + src, bytes, &bar_full[q]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            mbar_wait(&bar_a, 0);
            tc_fence_after();
            const uint32_t a_hi = sa(sA_hi), a_lo = sa(sA_lo), sbo_a = 32u * d;
            for (int t = 0; t < nT; ++t) {
                const int b = t & 1;
                if (t >= 2) mbar_wait(&bar_tempty[b], (uint32_t)(((t >> 1) - 1) & 1));
                const uint32_t acc = tmem + (uint32_t)(b * kTcN);
                for (int c = 0; c < nc; ++c) {
                    const int u = t * nc + c, q = u % kTcStages;
                    const int w = d - c * kTcKC < kTcKC ? d - c * kTcKC : kTcKC;
                    mbar_wait(&bar_full[q], (uint32_t)((u / kTcStages) & 1));
                    tc_fence_after();
                    const uint32_t b_hi = sa(sB + (size_t)2 * q * st_floats), b_lo = sa(sB + (size_t)(2 * q + 1) * st_floats);
                    const uint32_t sbo_b = 32u * w;
                    for (int kk = 0; kk < w / 8; ++kk) {  // K = 8 tf32 = two 16-byte chunks per MMA
                        const uint32_t oa = 128u * (uint32_t)(c * kTcKC / 4 + 2 * kk), ob = 256u * kk;
                        mma_tf32<kTcN>(acc, umma_desc(a_lo + oa, 128, sbo_a), umma_desc(b_hi + ob, 128, sbo_b), c > 0 || kk > 0);
                        mma_tf32<kTcN>(acc, umma_desc(a_hi + oa, 128, sbo_a), umma_desc(b_lo + ob, 128, sbo_b), 1);
                        mma_tf32<kTcN>(acc, umma_desc(a_hi + oa, 128, sbo_a), umma_desc(b_hi + ob, 128, sbo_b), 1);
                    }
                    mma_commit(&bar_empty[q]);  // ring stage free once these MMAs have read it
                }
                mma_commit(&bar_tfull[b]);  // accumulator b complete
            }
        }
    } else {
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int row = q * 32 + lane;
        const int64_t gi = mt * kTcM + row;
        if constexpr (kCollect) {  // pass 2: every column within the row's pass-1 threshold
            const float thr = gi < a.m ? a.row_thr[gi] : -INFINITY;
            for (int t = 0; t < nT; ++t) {
                const int b = t & 1;
                mbar_wait(&bar_tfull[b], (uint32_t)((t >> 1) & 1));
                tc_fence_after();
                const float* sqt = a.sq + (size_t)(t0 + t) * kTcN;
#pragma unroll 1
                for (int c0 = 0; c0 < kTcN; c0 += 64) {
                    float v[64];
                    tmem_ld64(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * kTcN + c0), v);
#pragma unroll
                    for (int j = 0; j < 64; j += 4) {
                        const float4 s4 = __ldg(reinterpret_cast<const float4*>(sqt + c0 + j));
                        const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            if (fmaf(-2.f, v[j + u], sv[u]) <= thr) {  // rare: near ties only
                                const int slot = atomicAdd(a.ccnt + gi, 1);  // CTA columns append
                                if (slot < kCandCap) a.cand[gi * kCandCap + slot] = (t0 + t) * kTcN + c0 + j + u;
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&bar_tempty[b]);
            }
        } else {
        // the certified margin M_i: S_i = |x_i| max_j |c_j| bounds sum_k |x_ik c_jk|
        const float sqmax = __uint_as_float(a.stats[S_SQMAX]);
        const float cn = sqrtf(sqmax) * (1.f + 0x1p-20f);
        const float xn = gi < a.m ? a.xnorm[gi] : 0.f;
        float M = INFINITY;
        if (xn < 1e15f && cn < 1e15f && sqmax < 1e30f) {  // every fp32 partial sum stays far from overflow
            const float S = xn * cn;
            // + flushed subnormal operands / products (each below 2^-126 times a magnitude)
            M = (float)(6 * d + 24) * 0x1p-22f * S + 0x1p-22f * sqmax + (float)(8 * d) * 0x1p-118f * (xn + cn + 1.f);
        }
        // kTr independent (best, index, second) trackers, tracker u taking the columns j = u mod kTr:
        // the compare-select chains interleave instead of serialising 128 columns per tile
        constexpr int kTr = 8;
        float bb[kTr], ss[kTr];
        int jj[kTr];
#pragma unroll
        for (int u = 0; u < kTr; ++u) {
            bb[u] = ss[u] = INFINITY;
            jj[u] = 0;
        }
        // |c_j|^2 of the tile, staged per warp in shared memory (broadcast reads), the next tile's
        // values loaded into registers while this tile is processed
        float* sqw = sq_stage + q * 2 * kTcN;
        constexpr int kV = kTcN / 128;  // float4s per lane per tile
        float4 nxt[kV];
#pragma unroll
        for (int v = 0; v < kV; ++v)
            nxt[v] = __ldg(reinterpret_cast<const float4*>(a.sq + (size_t)t0 * kTcN) + 32 * v + lane);
        for (int t = 0; t < nT; ++t) {  // pass 1 runs with one CTA column: t0 = 0, nT = n_tiles
            const int b = t & 1;
#pragma unroll
            for (int v = 0; v < kV; ++v) reinterpret_cast<float4*>(sqw + b * kTcN)[32 * v + lane] = nxt[v];
            __syncwarp();
            if (t + 1 < nT) {
#pragma unroll
                for (int v = 0; v < kV; ++v)
                    nxt[v] = __ldg(reinterpret_cast<const float4*>(a.sq + (size_t)(t0 + t + 1) * kTcN) + 32 * v + lane);
            }
            mbar_wait(&bar_tfull[b], (uint32_t)((t >> 1) & 1));
            tc_fence_after();
            const float* sqt = sqw + b * kTcN;
#pragma unroll 1
            for (int c0 = 0; c0 < kTcN; c0 += 64) {
                float v[64];
                tmem_ld64(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * kTcN + c0), v);
#pragma unroll
                for (int j = 0; j < 64; j += kTr) {
                    const float4 s0 = *reinterpret_cast<const float4*>(sqt + c0 + j);
                    const float4 s1 = *reinterpret_cast<const float4*>(sqt + c0 + j + 4);
                    const float sv[kTr] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
                    for (int u = 0; u < kTr; ++u) {
                        const float av = fmaf(-2.f, v[j + u], sv[u]);
                        const bool nb = av < bb[u];
                        ss[u] = nb ? bb[u] : fminf(ss[u], av);
                        jj[u] = nb ? (t0 + t) * kTcN + c0 + j + u : jj[u];
                        bb[u] = nb ? av : bb[u];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_tempty[b]);
        }
        if (gi < a.m) {
            // Certification: every a_ij is within M of d_ij.  Let best = min a and
            // thr = best + 2M.  A column outside the trackers' bests has a >= its tracker's second;
            // if every second exceeds thr, such columns have d > best + M >= d_min: the exact
            // first minimum is among the trackers' bests with a <= thr.  One such candidate: it is
            // the label.  Several: their d_ij are evaluated here in fp64 (the oracle's order) and
            // the smallest (lowest index on ties) is the label.  Otherwise the fp64 pass decides.
            float best = bb[0];
#pragma unroll
            for (int u = 1; u < kTr; ++u) best = fminf(best, bb[u]);
            const float thr = best + 2.f * M;
            bool cert = true;
            int ncand = 0, cand = 0;
#pragma unroll
            for (int u = 0; u < kTr; ++u) {
                cert = cert && (ss[u] > thr);
                if (bb[u] <= thr) {
                    ++ncand;
                    cand = jj[u];
                }
            }
            cert = cert && ncand >= 1;  // NaN scores (M = inf rows excepted) never certify
            if (cert && ncand == 1) {
                a.labels[gi] = cand;
            } else if (cert) {
                const float* x = a.X + gi * d;
                double dbest = INFINITY;
                int lbest = INT32_MAX;
#pragma unroll
                for (int u = 0; u < kTr; ++u) {  // unrolled: the trackers stay in registers
                    if (!(bb[u] <= thr)) continue;
                    const int j = jj[u];
                    const double dj = exact_dist(x, a.cen + (int64_t)j * d, a.sqn[j], d);
                    if (dj < dbest || (dj == dbest && j < lbest)) {
                        dbest = dj;
                        lbest = j;
                    }
                }
                a.labels[gi] = lbest;
                atomicAdd(a.amb_count + 1, 1ull);
            } else {  // not certified alone: pass 2 collects the row's candidates
                a.labels[gi] = -1;
                const unsigned long long k = atomicAdd(a.amb_count, 1ull);
                a.amb_rows[k] = (int32_t)(a.row0 + gi);
                a.amb_thr[k] = thr;
            }
        }
        }  // pass 1
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcTmemCols) : "memory");
}

// pass 3: the listed rows' labels from their candidates in fp64 (the oracle's order; smallest
// distance, lowest index on ties); rows without a usable list (none, or more than kCandCap) go to
// `out` for the fp64 pass over every cluster
__global__ void tc_recheck_kernel(const int32_t* __restrict__ rows, int64_t n, const int32_t* __restrict__ cand,
                                  const int32_t* __restrict__ ccnt, const float* __restrict__ X,
                                  const double* __restrict__ cen, const double* __restrict__ sqn, int d,
                                  int32_t* __restrict__ labels, int32_t* __restrict__ out,
                                  unsigned long long* __restrict__ counts) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t row = rows[k];
        const int c = ccnt[k];
        if (c <= 0 || c > kCandCap) {
            out[atomicAdd(counts, 1ull)] = row;
            continue;
        }
        const float* x = X + (int64_t)row * d;
        double dbest = INFINITY;
        int lbest = INT32_MAX;
        for (int i = 0; i < c; ++i) {
            const int j = cand[k * kCandCap + i];
            const double dj = exact_dist(x, cen + (int64_t)j * d, sqn[j], d);
            if (dj < dbest || (dj == dbest && j < lbest)) {
                dbest = dj;
                lbest = j;
            }
        }
        labels[row] = lbest;
        atomicAdd(counts + 1, 1ull);
    }
}

int tc_tile_n(int d) { return d >= 48 ? 256 : 128; }

size_t tc_smem_bytes(int d) {
    const size_t kc = d < kTcKC ? d : kTcKC, n = tc_tile_n(d);
    const size_t need = sizeof(float) * ((size_t)2 * kTcM * d + (size_t)2 * kTcStages * n * kc);
    // at most 512 / (2 n) CTAs per SM, so their TMEM columns always fit: N = 256 needs the whole
    // TMEM (more than half an SM's shared memory), N = 128 half of it (over a third)
    const size_t floor_bytes = n == 256 ? 120 * 1024 : 80 * 1024;
    return need > floor_bytes ? need : floor_bytes;
}

}  // namespace

bool birch_tc_eligible(int d, int64_t K) {
    DeviceInfo di;
    if (!device_info(&di)) return false;
    return d >= 8 && d <= kBirchTcMaxD && d % 8 == 0 && K >= 1 && K < (int64_t)INT32_MAX - 256 &&
           tc_smem_bytes(d) <= (size_t)di.max_smem_optin;
}

igp_status launch_birch_tc(const double* cen, const double* sqn, int64_t K, int d, const float* X, int64_t m,
                           int32_t* labels, int32_t* amb_rows, unsigned long long* amb_count, cudaStream_t s) {
    // rows in chunks of at most kChunk (bounded workspace), the centroids split once
    constexpr int64_t kChunk = (int64_t)1 << 22;
    const int kTcN = tc_tile_n(d);
    const int64_t mc = m < kChunk ? m : kChunk;
    const int64_t mt = (mc + kTcM - 1) / kTcM, nt = (K + kTcN - 1) / kTcN;
    const size_t xf = (size_t)mt * kTcM * d, cf = (size_t)nt * kTcN * d;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t o_xl = al(4 * xf), o_ch = o_xl + al(4 * xf), o_cl = o_ch + al(4 * cf), o_sq = o_cl + al(4 * cf),
                 o_xn = o_sq + al(4 * (size_t)nt * kTcN), o_st = o_xn + al(4 * (size_t)mc),
                 o_thr = o_st + al(4 * S_WORDS), total = o_thr + al(4 * (size_t)m);
    char* ws = nullptr;
    IGP_CUDA(alloc_async_class((void**)&ws, total, s), "birch tc workspace");
    float* xh = (float*)ws;
    float* xl = (float*)(ws + o_xl);
    float* ch = (float*)(ws + o_ch);
    float* cl = (float*)(ws + o_cl);
    float* sq = (float*)(ws + o_sq);
    float* xn = (float*)(ws + o_xn);
    unsigned* st = (unsigned*)(ws + o_st);
    float* thr = (float*)(ws + o_thr);
    igp_status r = cuda_status(cudaMemsetAsync(st, 0, 4 * S_WORDS, s), "memset");
    if (r == IGP_OK) r = cuda_status(cudaMemsetAsync(amb_count, 0, 2 * sizeof(unsigned long long), s), "memset");
    if (r == IGP_OK) {
        tc_split_kernel<double><<<(unsigned)((nt * kTcN + 255) / 256), 256, 0, s>>>(cen, nullptr, K, nt * kTcN, d, kTcN,
                                                                                kTcKC, ch, cl, nullptr, sqn, sq, st);
        r = launch_status("tc_split_kernel<double>");
    }
    const size_t smem = tc_smem_bytes(d);
    auto kern = kTcN == 256 ? birch_tc_kernel<256, false> : birch_tc_kernel<128, false>;
    auto kcol = kTcN == 256 ? birch_tc_kernel<256, true> : birch_tc_kernel<128, true>;
    if (r == IGP_OK)
        r = cuda_status(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "birch tc smem attribute");
    if (r == IGP_OK)
        r = cuda_status(cudaFuncSetAttribute(kcol, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                        "birch tc smem attribute");
    // pass 1: every row; certified rows are labelled, the rest listed with their thresholds
    for (int64_t row0 = 0; row0 < m && r == IGP_OK; row0 += kChunk) {
        const int64_t rows = m - row0 < kChunk ? m - row0 : kChunk;
        const int64_t rt = (rows + kTcM - 1) / kTcM;
        const float* Xc = X + row0 * d;
        tc_split_kernel<float><<<(unsigned)((rt * kTcM + 255) / 256), 256, 0, s>>>(Xc, nullptr, rows, rt * kTcM, d, kTcM,
                                                                              d, xh, xl, xn, nullptr, nullptr, nullptr);
        r = launch_status("tc_split_kernel<float>");
        if (r == IGP_OK) {
            TcArgs ar{xh,  xl,   ch,      cl,      sq, xn,           st,       Xc,        cen, sqn,     rows,
                      row0, (int)nt, (int)nt, d, labels + row0, amb_rows, amb_count, thr, nullptr, nullptr, nullptr};
            kern<<<(unsigned)rt, kTcThreads, smem, s>>>(ar);
            r = launch_status("birch_tc_kernel");
        }
    }
    unsigned long long h[2] = {0, 0};
    if (r == IGP_OK) r = cuda_status(cudaMemcpyAsync(h, amb_count, sizeof(h), cudaMemcpyDeviceToHost, s), "readback");
    if (r == IGP_OK) r = cuda_status(cudaStreamSynchronize(s), "sync");
    const int64_t n1 = (int64_t)h[0];
    if (r == IGP_OK && n1 > 0) {
        // pass 2 (the listed rows, as tiles of their own): every column within the row's threshold;
        // pass 3: fp64 over those candidates.  Rows without a usable list stay listed (in place:
        // the list is rebuilt from the front) for the fp64 pass over every cluster.
        constexpr int64_t kChunk2 = (int64_t)1 << 20;
        const int64_t c2 = n1 < kChunk2 ? n1 : kChunk2;
        int32_t* cand = nullptr;
        r = cuda_status(
            alloc_async_class((void**)&cand, sizeof(int32_t) * ((size_t)c2 * (kCandCap + 1) + 2 * (size_t)n1 + 8), s),
            "alloc");
        if (r == IGP_OK) {
            int32_t* ccnt = cand + (size_t)c2 * kCandCap;
            int32_t* rows1 = ccnt + c2;        // the pass-1 list (a copy: amb_rows is rebuilt)
            const size_t o_cnt = ((size_t)c2 * (kCandCap + 1) + (size_t)n1 + 1) & ~(size_t)1;  // 8-byte aligned
            unsigned long long* cnt2 = reinterpret_cast<unsigned long long*>(cand + o_cnt);
            r = cuda_status(cudaMemcpyAsync(rows1, amb_rows, sizeof(int32_t) * (size_t)n1, cudaMemcpyDeviceToDevice, s),
                            "list copy");
            if (r == IGP_OK) r = cuda_status(cudaMemsetAsync(cnt2, 0, 2 * sizeof(unsigned long long), s), "memset");
            for (int64_t k0 = 0; k0 < n1 && r == IGP_OK; k0 += kChunk2) {
                const int64_t rows = n1 - k0 < kChunk2 ? n1 - k0 : kChunk2;
                const int64_t rt = (rows + kTcM - 1) / kTcM;
                tc_split_kernel<float><<<(unsigned)((rt * kTcM + 255) / 256), 256, 0, s>>>(
                    X, rows1 + k0, rows, rt * kTcM, d, kTcM, d, xh, xl, nullptr, nullptr, nullptr, nullptr);
                r = launch_status("tc_split_kernel<float>");
                // few rows: the centroid tiles are split over CTA columns to fill the GPU
                DeviceInfo di;
                const int sms = device_info(&di) ? di.num_sms : 148;
                const int64_t ys = std::max<int64_t>(1, std::min<int64_t>(nt, (2 * sms + rt - 1) / rt));
                const int tps = (int)((nt + ys - 1) / ys);
                const unsigned gy = (unsigned)((nt + tps - 1) / tps);
                if (r == IGP_OK) r = cuda_status(cudaMemsetAsync(ccnt, 0, sizeof(int32_t) * (size_t)rows, s), "memset");
                if (r == IGP_OK) {
                    TcArgs ar{xh,  xl,      ch,  cl, sq,      nullptr, st,      X,       cen,      sqn,  rows,
                              k0,  (int)nt, tps, d,  nullptr, nullptr, nullptr, nullptr, thr + k0, cand, ccnt};
                    kcol<<<dim3((unsigned)rt, gy), kTcThreads, smem, s>>>(ar);
                    r = launch_status("birch_tc_kernel<collect>");
                }
                if (r == IGP_OK) {
                    tc_recheck_kernel<<<(unsigned)std::min<int64_t>((rows + 127) / 128, 8192), 128, 0, s>>>(
                        rows1 + k0, rows, cand, ccnt, X, cen, sqn, d, labels, amb_rows, cnt2);
                    r = launch_status("tc_recheck_kernel");
                }
            }
            // amb_count: [0] = rows still listed, [1] += rows settled by the candidate re-check
            unsigned long long h2[2] = {0, 0};
            if (r == IGP_OK) r = cuda_status(cudaMemcpyAsync(h2, cnt2, sizeof(h2), cudaMemcpyDeviceToHost, s), "readback");
            if (r == IGP_OK) r = cuda_status(cudaStreamSynchronize(s), "sync");
            if (r == IGP_OK) {
                const unsigned long long hn[2] = {h2[0], h[1] + h2[1]};
                r = cuda_status(cudaMemcpyAsync(amb_count, hn, sizeof(hn), cudaMemcpyHostToDevice, s), "count");
                if (r == IGP_OK) r = cuda_status(cudaStreamSynchronize(s), "sync");  // hn is on this stack frame
            }
            free_async(cand, s);
        }
    }
    free_async(ws, s);
    return r;
}

}  // namespace igp
