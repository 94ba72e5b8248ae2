// embed.cu — igp_embed: Alg. 1 lines 1-6 on one GPU.
//
// Kernels:
//   E1a scale_kernel       D_tau by Eq. (1) / D + tau I in fp64;
//                          per node {s = D^-1/2, r = D^1/2} as fp32
//   E1b affine_kernel      c_i = theta + alpha s_i sum_{j in N(i)} s_j  ( = (phi * 1)_i ), kept as hi+lo fp32
//   E2  input_kernel<W>    Theta = X / sqrt(d), X ~ Philox/Box-Muller N(0,1); y0 = s * Theta
//   E3  layer_kernel<W>    one filter step on a W-column slice (L launches per slice):
//                          gather y_j = s_j t_j (float4), Eq. (3) with the deferred column
//                          z-score, tanh (Eq. (4)), store y' = s t', exact column sums
//   E4  output_kernel<W>   Z~ = sigmoid((t - mu)/sigma)  (Eq. (4))
//   E5  row_l2_kernel      optional post-op (IGP_FLAG_ROW_L2, not in the paper; reading A12)
//
// Launch structure.  E3 runs as a persistent grid (min(row batches, SMs x 2) blocks of 8
// warps; 2-warp blocks when the graph cannot fill the SMs otherwise) and every filter step
// is launched with programmatic dependent launch, so step l+1's setup and first CSR loads
// overlap step l's tail.  The whole embed is enqueued without a host synchronisation.
//
// Column slicing.  Every step of the FFP acts on each column independently:
// phi* mixes rows only, tanh/sigmoid are element-wise and ZNorm is per column
// (PAPER.md:155, :164-166).  So the d columns are processed as d/W slices of W
// columns, each pushed through all L steps before the next: the gathered slice
// (N x W fp32) is sized to stay resident in L2 (DESIGN.md §5 derives W from the
// measured gather bandwidth table).
//
// Deferred ZNorm.  ZNorm is a per-column affine map and phi* is linear, so with
// t = tanh(P) of the previous step and Z = (t - mu)/sigma:
//   phi * Z = [theta t_i + alpha s_i sum_j s_j t_j - mu c_i] / sigma,  c_i = (phi * 1)_i.
// Each step stores y = s t once; the next step applies (mu, 1/sigma) while it gathers.
//
// Exact column statistics.  Each t (and t^2) is rounded to a fixed grid 2^-g
// (g chosen from N so that |sum| < 2^53 grid units) before it is accumulated in
// fp64; every partial sum is then an exact integer multiple of 2^-g, so the sums
// are independent of summation order: blocks combine them with plain atomics,
// the row schedule is free, and the output is still bitwise deterministic.  The
// rounding perturbs mu and sigma by < 2^-g (~1e-9), far below fp32 resolution.
#include <atomic>
#include <cmath>
#include <cstdlib>

#include "igp_internal.cuh"
#include "philox.cuh"

namespace igp {
namespace {

constexpr int kChunk = 16;      // neighbours per index chunk
constexpr int kFoldChunks = 8;   // fp32 partial sums span at most 128 neighbours (measured: 64 -> 128
                                 // makes the headline step 2% faster at unchanged parity; 256 loses accuracy)
constexpr int kBatch = 8;       // gathers issued back to back per lane (full chunks)
constexpr unsigned kFull = 0xffffffffu;
constexpr int kDefaultOcc = 2;
constexpr int kBigNW = 8;  // warps per block of layer_kernel (2 for graphs that cannot fill the SMs)
constexpr int kGrab = 1;  // row batches per atomic grab of layer_kernel's dynamic schedule
constexpr bool kDynSchedule = true;
constexpr int kCounters = 4;  // row-batch counters per launch (warps spread over them)
constexpr int64_t kDynMinEdgesPerWarp = 2048;  // CSR entries per warp below which the schedule stays static
// index chunks start at each row's first entry (scalar index loads) instead of the 16-byte aligned
// entry below it: fewer masked gather slots per row batch (round-trip fill 0.87 -> 0.92 on the
// headline graph); measured headline -1.5%, Large -5% per filter step (profiles/r02/idx_any.txt)
constexpr int kIdxAnyStart = 1;
constexpr float kIdxEvictFirst = 1.0f;  // the index stream is read once per launch
constexpr float kStoreEvictFirst = 1.0f;  // measured +2% (profiles/r01)

__global__ void scale_kernel(const int32_t* __restrict__ rp, int32_t n, double tau, double eps,
                             float2* __restrict__ sr) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int32_t deg = rp[i + 1] - rp[i];
        float s = 1.0f, r = 1.0f;  // isolated node: empty neighbour sum, scale unused (reading A5)
        if (deg > 0) {
            double D;
            if (tau < 0.0) {
                const double a = fabs(tau), b = (double)deg - eps;
                D = (double)deg - (a < b ? a : b);  // Eq. (1)
            } else {
                D = (double)deg + tau;  // D + tau I
            }
            const double sq = sqrt(D);
            s = (float)(1.0 / sq);
            r = (float)sq;
        }
        sr[i] = make_float2(s, r);
    }
}

// c_i = theta + alpha s_i sum_j s_j, one warp per row, fp64 sum, fixed shuffle tree
__global__ void affine_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, int32_t n,
                              float theta, float alpha, const float2* __restrict__ sr, float2* __restrict__ cc) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
        const int32_t beg = rp[i], end = rp[i + 1];
        double acc = 0.0;
        for (int32_t e = beg + lane; e < end; e += 32) acc += (double)sr[ci[e]].x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == 0) {
            const float s = sr[i].x;
            const double c = (end > beg) ? (double)theta + (double)alpha * (double)s * acc : (double)theta;
            const float chi = (float)c;
            cc[i] = make_float2(chi, (float)(c - (double)chi));  // c_i as an unevaluated sum hi + lo (~48 bits)
        }
    }
}

// slice k of y0 = s_i * Theta_i, Theta = X / sqrt(d); element (i, c) of original node i is
// draw k = i*d + c; relabelled row r holds original node order[r]
// (or, with a caller-provided z0 [N][d], y0 = s_i * z0_i: the igp_embed_opts.d_z0 hook)
template <int W>
__global__ void input_kernel(uint64_t seed, uint64_t sub, int32_t n, int d, int col0,
                             const int32_t* __restrict__ order, const float2* __restrict__ sr,
                             const float* __restrict__ z0, float4* __restrict__ y0) {
    constexpr int LPR = W / 4;
    const int64_t total = (int64_t)n * LPR;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const double sqd = sqrt((double)d);
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += stride) {
        const int64_t i = idx / LPR;
        const int q = (int)(idx % LPR);
        if (z0) {
            const float4 z = *reinterpret_cast<const float4*>(z0 + (int64_t)order[i] * d + col0 + 4 * q);
            const double s = (double)sr[i].x;
            y0[idx] = make_float4((float)(s * z.x), (float)(s * z.y), (float)(s * z.z), (float)(s * z.w));
            continue;
        }
        const uint64_t b = (uint64_t)(((int64_t)order[i] * d + col0) / 4 + q);  // draws of the ORIGINAL id
        const U4 r = philox_block(seed, sub, b);
        double x0, x1, x2, x3;
        box_muller64(r.x, r.y, x0, x1);
        box_muller64(r.z, r.w, x2, x3);
        const double s = (double)sr[i].x;
        y0[idx] = make_float4((float)(s * (x0 / sqd)), (float)(s * (x1 / sqd)), (float)(s * (x2 / sqd)),
                              (float)(s * (x3 / sqd)));
    }
}

struct LayerArgs {
    const int32_t* rp;
    const int32_t* ci;
    const float2* sr;       // [N + 2] {s, r}: s = D_tau^-1/2, r = D_tau^1/2
    const float2* cc;       // [N + 2] {c_hi, c_lo}: c_i = (phi * 1)_i (read only when sums_in != nullptr)
    const float4* yin;      // [N][W/4]
    float4* yout;           // [N][W/4]
    const double* sums_in;  // [2W] (sum t, sum t^2) of the previous step; nullptr: Z = Theta (mu 0, sigma 1)
    double* sums_out;       // [2W], zero on entry
    int32_t n;
    float theta, alpha;
    int linear;
    int ddof;       // ZNorm std: 0 population (reading A2), 1 sample
    double grid_c;  // 1.5 * 2^(52-g): (x + grid_c) - grid_c rounds x to the 2^-g grid
    float idx_ef;   // fraction of index-stream loads marked L2 evict_first
    float st_ef;    // fraction of output stores marked L2 evict_first
    int idx_any;    // 1: index chunks start at the row's first entry (scalar index loads), 0: 16-byte aligned
    int* sched;     // layer_kernel: this launch's row-batch counter (zero at launch; nullptr: static schedule)
};

// (mu, 1/sigma) of column c from exact sums; std with ddof (0 = population, reading A2; the
// sample std for ddof = 1), floor 1e-8 -> 0 (A3); N <= ddof counts as a zero std
__device__ __forceinline__ void column_stats(const double* sums, int c, int W, int32_t n, int ddof, double& mu,
                                             double& isg) {
    const double invN = 1.0 / (double)n;
    const double m = sums[c] * invN;
    double var = sums[W + c] * invN - m * m;
    var = var > 0.0 ? var : 0.0;
    if (ddof != 0) var = n > ddof ? var * ((double)n / (double)(n - ddof)) : 0.0;
    const double sd = sqrt(var);
    mu = m;
    isg = sd < 1e-8 ? 0.0 : 1.0 / sd;
}

__device__ __forceinline__ double grid_round(double x, double c) { return __dsub_rn(__dadd_rn(x, c), c); }

__device__ __forceinline__ int ld_idx1(const int32_t* p, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
// L2 policy: a fraction `frac` of the accesses are marked evict_first, the rest unchanged
__device__ __forceinline__ uint64_t evict_first_policy(float frac) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.L2::evict_unchanged.b64 %0, %1;" : "=l"(pol) : "f"(frac));
    return pol;
}

// 256-bit vector access (sm_100: LDG.256 / STG.256) and packed fp32 adds (FADD2)
__device__ __forceinline__ void ldg256(const void* ptr, uint64_t (&v)[4]) {
    asm("ld.global.nc.v4.b64 {%0,%1,%2,%3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(ptr));
}
// a neighbour-row gather of layer_kernel: no L1 allocation (the rows are rarely re-read from L1
// within an SM; the row's own values, prefetched into L1, are not displaced by them)
__device__ __forceinline__ void ldg256_na(const void* ptr, uint64_t (&v)[4]) {
    asm("ld.global.nc.L1::no_allocate.v4.b64 {%0,%1,%2,%3}, [%4];"
        : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3])
        : "l"(ptr));
}
__device__ __forceinline__ void stg256(void* ptr, const uint64_t (&v)[4], uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.b64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(ptr), "l"(v[0]), "l"(v[1]),
                 "l"(v[2]), "l"(v[3]), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* ptr) { asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr)); }
__device__ __forceinline__ void prefetch_l1(const void* ptr) { asm volatile("prefetch.global.L1 [%0];" ::"l"(ptr)); }
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

__device__ __forceinline__ int4 ld_idx4h(const int32_t* p, uint64_t pol) {
    int4 v;
    asm volatile("ld.global.nc.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int2 ld_idx2h(const int32_t* p, uint64_t pol) {
    int2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.s32 {%0,%1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}
// (index loads allocate in L1: a row batch's index lines are re-read by its next chunks --
// interleaved A/B -2.8% per headline launch)
// indices [e0 + q*IPL, e0 + (q+1)*IPL) of a chunk (vector loads when e0 % 4 == 0 and !any); the col arrays are
// padded, so a chunk may run past the row (those slots are masked by the caller)
template <int IPL>
__device__ __forceinline__ void load_idx(const int32_t* ci, int32_t e0, int32_t end, int q, uint64_t pol,
                                         int (&jr)[IPL], int any) {
    const int32_t e = e0 + q * IPL;
    if (e >= end) {
#pragma unroll
        for (int k = 0; k < IPL; ++k) jr[k] = 0;
        return;
    }
    if (any) {
#pragma unroll
        for (int k = 0; k < IPL; ++k) jr[k] = ld_idx1(ci + e + k, pol);
        return;
    }
    if constexpr (IPL >= 4) {
#pragma unroll
        for (int k = 0; k < IPL; k += 4) {
            const int4 v = ld_idx4h(ci + e + k, pol);
            jr[k] = v.x, jr[k + 1] = v.y, jr[k + 2] = v.z, jr[k + 3] = v.w;
        }
    } else if constexpr (IPL == 2) {
        const int2 v = ld_idx2h(ci + e, pol);
        jr[0] = v.x, jr[1] = v.y;
    } else {
        jr[0] = ld_idx1(ci + e, pol);
    }
}

// One filter step on a W-column slice.
//  - A group of LPR = W/8 lanes owns one row at a time; each lane holds 8 columns, so a
//    neighbour costs one 256-bit gather and 4 packed fp32 adds per lane.  G = 32/LPR rows
//    per warp run side by side, in descending-degree order (similar trip counts).
//  - Neighbour indices come 16 at a time (IPL per lane, broadcast by shuffles); the next
//    chunk's indices are fetched while this chunk is gathered.
//  - Column statistics: each warp stages its G x W tile of t in shared memory and every
//    lane folds 8 of those values (OC whole columns) into fp64 registers, so the per-lane
//    state is 2*OC doubles instead of 16.
template <int W, int MB, int NW>
__global__ void __launch_bounds__(NW * 32, MB) layer_kernel(const LayerArgs p) {
    constexpr int kWarps = NW;  // warps per block (8; 2 for graphs too small to fill the SMs)
    constexpr int kThreads = NW * 32;
    constexpr int LPR = W / 8;
    constexpr int G = 32 / LPR;
    constexpr int IPL = kChunk / LPR;
    constexpr int NG = kWarps * G;            // row groups per block
    constexpr int OC = W >= 32 ? W / 32 : 1;  // statistics columns owned per lane
    constexpr int OR = W >= 32 ? G : G / 2;   // ... each over OR rows of the warp tile
    constexpr int TS = W + 4;                 // tile row stride (floats): conflict-free staging
    __shared__ double2 st[W + W / 8];         // (mu, 1/sigma) of the previous step, column c at c + c/8
    __shared__ __align__(16) float stage[kWarps][G * TS];
    extern __shared__ double dyn_smem[];
    double (*acc_f)[W] = reinterpret_cast<double (*)[W]>(dyn_smem);  // [NG][W] long-row partials
    // Programmatic dependent launch: the next filter step may be scheduled onto SMs as this
    // grid's blocks retire; everything up to griddepcontrol.wait (shared-memory setup, the first
    // row batch's row pointers and indices -- static CSR data) overlaps this grid's tail.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int t = threadIdx.x; t < NG * W; t += kThreads) (&acc_f[0][0])[t] = 0.0;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane % LPR, g = lane / LPR;
    const int grp = warp * G + g;
    const uint64_t* yin = reinterpret_cast<const uint64_t*>(p.yin);  // row j, lane q: yin + (j*LPR + q)*4
    uint64_t* yout = reinterpret_cast<uint64_t*>(p.yout);
    float* tile = stage[warp];
    const uint64_t pol_idx = evict_first_policy(p.idx_ef);
    const uint64_t pol_st = evict_first_policy(p.st_ef);
    const int32_t amask = p.idx_any ? ~0 : ~3;
    const int oc0 = W >= 32 ? lane * OC : lane / 2;  // owned statistics columns / rows
    const int or0 = W >= 32 ? 0 : (lane & 1) * OR;
    double s1[OC], s2[OC];
#pragma unroll
    for (int k = 0; k < OC; ++k) s1[k] = s2[k] = 0.0;

    // Row-batch schedule: batch b = rows [bG, bG + G) of the relabelled CSR.  Dynamic (p.sched):
    // a warp's first grab of kGrab batches is its own index, every later one a ticket from one of
    // kCounters atomic counters (warp w -> counter c = w mod kCounters, ticket t -> grab
    // t kCounters + c), requested one batch before it is needed (lane 0 holds it until then).  The
    // rows in flight stay one narrow front sweeping the CSR in order -- the in-community gathers
    // hit L2 before it turns over (8-batch grabs, a 4x wider front, were 47% slower) -- and no SM
    // idles at the end (static striding: SMs active 718K of 821K cycles, min 654K; dynamic: 95%).
    // Same-address atomics serialise (~5 ns each), so the host enables it only when every warp gets
    // >= 4 batches and >= 2048 CSR entries.  Static (no counter): warp w takes
    // batches w, w + warps, ...  The row sums do not depend on the schedule and the column sums
    // are exact: the output is bit-identical either way.
    const int64_t nbat = (p.n + G - 1) / G;
    const bool dyn = p.sched != nullptr;
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    int64_t bat;
    int gi = 0, pend = 0;  // batch within the current grab; lane 0: the grab after it
    const int64_t wid = (int64_t)blockIdx.x * kWarps + warp;
    const int cidx = (int)(wid % kCounters);
    const int tick0 = (int)((nwarps - cidx + kCounters - 1) / kCounters);  // tickets of the static first grabs
    int* ctr = p.sched + cidx;
    if (dyn) {  // first grab: the warp's own index; the counters hand out the grabs after them
        if (lane == 0) pend = (tick0 + atomicAdd(ctr, 1)) * kCounters + cidx;
        bat = wid * kGrab;
    } else {
        bat = (int64_t)blockIdx.x * kWarps + warp;
    }
    // The row-pointer -> index -> gather chain of a row batch is started one batch ahead:
    // the next batch's row pointers are loaded when a batch begins, and its first index
    // chunk once the batch's first gathers are in flight (nbeg/nend/jfirst).
    int64_t base = bat * G;
    int32_t nbeg = 0, nend = 0;
    int jfirst[IPL];
    if (base + g < p.n) {
        nbeg = __ldg(p.rp + base + g);
        nend = __ldg(p.rp + base + g + 1);
    }
    load_idx<IPL>(p.ci, nbeg & amask, nend, q, pol_idx, jfirst, p.idx_any);
    // the previous step's output (yin) and column sums (sums_in) are read only after this point
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int c = threadIdx.x; c < W; c += kThreads) {
        double m = 0.0, is = 1.0;
        if (p.sums_in) column_stats(p.sums_in, c, W, p.n, p.ddof, m, is);
        st[c + c / 8] = make_double2(m, is);  // one pad slot per 8 columns: the 8-column groups of the
                                              // lanes of a row start in distinct banks
    }
    __syncthreads();
    // warp-uniform batches of G consecutive rows of the relabelled CSR (degree-sorted, within
    // communities for the community order: neighbouring rows have similar trip counts)
    while (bat < nbat) {
        base = bat * G;
        int64_t nxt;  // the batch after this one
        if (!dyn)
            nxt = bat + nwarps;
        else if (gi + 1 < kGrab)
            nxt = bat + 1;
        else
            nxt = (int64_t)__shfl_sync(kFull, pend, 0) * kGrab;
        const int64_t nbase = nxt * G;
        const int32_t row = (int32_t)(base + g);
        const bool valid = row < p.n;
        float t8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const int32_t beg = nbeg, end = nend;
        const uint64_t* own_ptr = yin + ((size_t)row * LPR + q) * 4;
        // the row's own values are needed only after its gathers: prefetched into L1 now (the
        // gathers bypass L1 allocation, so the line stays); its node parameters are loaded now,
        // their latency hidden behind the gathers (interleaved A/B on one box: -1.5% per launch,
        // DESIGN.md §5)
        float2 sr2 = make_float2(0.f, 0.f), cc2 = make_float2(0.f, 0.f);
        if (valid) {
            prefetch_l1(own_ptr);
            sr2 = __ldg(p.sr + row);
            if (p.sums_in) cc2 = __ldg(p.cc + row);
        }
        nbeg = nend = 0;
        if (nbase + g < p.n) {
            nbeg = __ldg(p.rp + nbase + g);
            nend = __ldg(p.rp + nbase + g + 1);
        }
        if (dyn) {  // entering the next grab after this batch: request the one after it
            if (++gi == kGrab) {
                gi = 0;
                if (lane == 0) pend = (tick0 + atomicAdd(ctr, 1)) * kCounters + cidx;
            }
        }
        bat = nxt;
        // neighbour sum: packed fp32 within up to kFoldChunks chunks, then folded into
        // fp64 partials in shared memory (only rows longer than 128 neighbours fold).
        // The chunk loop is warp-uniform (the warp's rows have similar degrees), so the
        // index broadcasts are full-warp shuffles and fully-populated chunks run unpredicated.
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        int nc = 0;
        bool folded = false;
        double* af = acc_f[grp] + 8 * q;
        // chunks start 16-byte aligned (vector index loads); slots outside [beg, end) are masked
        const int32_t start = beg & amask;
        const int nch = end > beg ? (end - start + kChunk - 1) / kChunk : 0;
        const int max_nch = __reduce_max_sync(kFull, nch);
        int jr[IPL];
#pragma unroll
        for (int k = 0; k < IPL; ++k) jr[k] = jfirst[k];
        if (max_nch == 0) load_idx<IPL>(p.ci, nbeg & amask, nend, q, pol_idx, jfirst, p.idx_any);
        for (int c = 0; c < max_nch; ++c) {
            const int32_t e0 = start + c * kChunk, e1 = e0 + kChunk;
            int jn[IPL];
            load_idx<IPL>(p.ci, e1, end, q, pol_idx, jn, p.idx_any);  // prefetch the next chunk's indices
            const int lo = beg > e0 ? beg - e0 : 0;        // valid slots of this chunk: [lo, hi)
            int hi = end - e0;
            hi = hi < 0 ? 0 : (hi > kChunk ? kChunk : hi);
            if (__all_sync(kFull, lo == 0 && hi == kChunk)) {
                // issue kBatch gathers before consuming any, so kBatch x 32 B per lane are in flight
#pragma unroll
                for (int u0 = 0; u0 < kChunk; u0 += kBatch) {
                    uint64_t v[kBatch][4];
#pragma unroll
                    for (int t = 0; t < kBatch; ++t) {
                        const int u = u0 + t;
                        const int j = __shfl_sync(kFull, jr[u % IPL], u / IPL, LPR);
                        IGP_DASSERT(j >= 0 && j < p.n);
                        ldg256_na(yin + ((size_t)j * LPR + q) * 4, v[t]);
                    }
#pragma unroll
                    for (int t = 0; t < kBatch; ++t)
#pragma unroll
                        for (int k = 0; k < 4; ++k) acc[k] = fadd2(acc[k], v[t][k]);
                }
            } else {
#pragma unroll
                for (int u0 = 0; u0 < kChunk; u0 += kBatch) {
                    uint64_t v[kBatch][4];
#pragma unroll
                    for (int t = 0; t < kBatch; ++t) {
                        const int u = u0 + t;
                        const int j = __shfl_sync(kFull, jr[u % IPL], u / IPL, LPR);
                        v[t][0] = v[t][1] = v[t][2] = v[t][3] = 0ull;
                        if (u >= lo && u < hi) {
                            IGP_DASSERT(j >= 0 && j < p.n);
                            ldg256_na(yin + ((size_t)j * LPR + q) * 4, v[t]);
                        }
                    }
#pragma unroll
                    for (int t = 0; t < kBatch; ++t)
#pragma unroll
                        for (int k = 0; k < 4; ++k) acc[k] = fadd2(acc[k], v[t][k]);
                }
            }
            if (c == 0) {
                load_idx<IPL>(p.ci, nbeg & amask, nend, q, pol_idx, jfirst, p.idx_any);  // next batch's first chunk
                // the next batch's whole index range (its G rows are consecutive) into L2 with one
                // bulk prefetch (measured +0.5%)
                const int32_t lo_e = __shfl_sync(kFull, nbeg, 0);
                const int32_t hi_e = __shfl_sync(kFull, nend, 31);
                if (lane == 0 && hi_e > lo_e) {
                    const uint64_t a0 = reinterpret_cast<uint64_t>(p.ci + lo_e) & ~(uint64_t)15;
                    const uint64_t a1 = (reinterpret_cast<uint64_t>(p.ci + hi_e) + 15) & ~(uint64_t)15;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0))
                                 : "memory");
                }
            }
            if (++nc == kFoldChunks && e1 < end) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float2 f = unpack2(acc[k]);
                    af[2 * k] += (double)f.x;
                    af[2 * k + 1] += (double)f.y;
                    acc[k] = 0ull;
                }
                nc = 0;
                folded = true;
            }
#pragma unroll
            for (int k = 0; k < IPL; ++k) jr[k] = jn[k];
        }
        if (valid) {
            double ad[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 f = unpack2(acc[k]);
                ad[2 * k] = (double)f.x;
                ad[2 * k + 1] = (double)f.y;
            }
            if (folded) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    ad[k] += af[k];
                    af[k] = 0.0;
                }
            }
            const float4 nd = make_float4(sr2.x, sr2.y, cc2.x, cc2.y);
            uint64_t own[4];
            ldg256(own_ptr, own);
            const double si = (double)nd.x, cc = (double)nd.z + (double)nd.w;
            uint64_t o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 y = unpack2(own[k]);
                float yy[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double2 m = st[9 * q + 2 * k + h];
                    const float tself = (h ? y.y : y.x) * nd.y;  // t_i = y_i / s_i
                    const double P =
                        ((double)p.theta * (double)tself + (double)p.alpha * si * ad[2 * k + h] - m.x * cc) * m.y;
                    const float t = p.linear ? (float)P : tanhf((float)P);
                    t8[2 * k + h] = t;
                    yy[h] = nd.x * t;
                }
                o[k] = pack2(yy[0], yy[1]);
            }
            stg256(yout + ((size_t)row * LPR + q) * 4, o, pol_st);
        }
        if (!p.linear) {
            // stage the warp's G x W tile of t (invalid rows contribute 0) and fold owned columns
            // lanes with (q & 4) store their upper half first, so each 8-lane store phase covers
            // all 32 banks once (rows are TS = W + 4 floats apart)
            const float4 lo4 = make_float4(t8[0], t8[1], t8[2], t8[3]), hi4 = make_float4(t8[4], t8[5], t8[6], t8[7]);
            const bool swap = (q & 4) != 0;
            *reinterpret_cast<float4*>(tile + g * TS + 8 * q + (swap ? 4 : 0)) = swap ? hi4 : lo4;
            *reinterpret_cast<float4*>(tile + g * TS + 8 * q + (swap ? 0 : 4)) = swap ? lo4 : hi4;
            __syncwarp();
#pragma unroll
            for (int r = 0; r < OR; ++r) {
                float x[OC];
                const float* src = tile + (or0 + r) * TS + oc0;
                if constexpr (OC == 4) {
                    const float4 v = *reinterpret_cast<const float4*>(src);
                    x[0] = v.x, x[1] = v.y, x[2] = v.z, x[3] = v.w;
                } else if constexpr (OC == 2) {
                    const float2 v = *reinterpret_cast<const float2*>(src);
                    x[0] = v.x, x[1] = v.y;
                } else {
                    x[0] = *src;
                }
#pragma unroll
                for (int k = 0; k < OC; ++k) {
                    const double xd = (double)x[k];
                    s1[k] += grid_round(xd, p.grid_c);
                    s2[k] += grid_round(xd * xd, p.grid_c);
                }
            }
            __syncwarp();
        }
    }
    if (p.linear) return;
    // exact sums: every partial is a multiple of the grid, so any combination order is exact
    if (W < 32) {
#pragma unroll
        for (int k = 0; k < OC; ++k) {
            s1[k] += __shfl_xor_sync(kFull, s1[k], 1);
            s2[k] += __shfl_xor_sync(kFull, s2[k], 1);
        }
    }
    __syncthreads();  // acc_f is reused as the per-warp reduction buffer [kWarps][2W]
    double* red = dyn_smem;
    if (W >= 32 || (lane & 1) == 0) {
#pragma unroll
        for (int k = 0; k < OC; ++k) {
            red[warp * 2 * W + oc0 + k] = s1[k];
            red[warp * 2 * W + W + oc0 + k] = s2[k];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * W; t += kThreads) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) v += red[w * 2 * W + t];
        atomicAdd(p.sums_out + t, v);
    }
}

// ---------------------------------------------------------------------------------------------
// E3' layer_ws_kernel<W>: the same filter step with the row epilogue moved off the gather warps
// (warp specialisation).  A block has kWsGather gather warps and kWsEpi
// epilogue warps:
//  - a gather warp runs layer_kernel's gather pipeline (G rows side by side, W/8 lanes per row,
//    8 x 256-bit gathers in flight per lane) and, instead of finishing its rows, hands each row
//    batch's fp64 neighbour sums to an epilogue warp through a one-batch shared-memory slot
//    (mbarriers full / empty), then starts the next batch at once: no drain of its gathers for
//    the own-row load, tanh, the store and the statistics;
//  - an epilogue warp owns W/32 whole columns per lane and finishes the batches of kWsGather /
//    kWsEpi gather warps: own row (coalesced), Eq. (3) with the deferred ZNorm, tanh, store, and
//    the exact column sums straight in registers (no staging: the lane already owns its columns).
// Same arithmetic as layer_kernel in the same order, so the output is bit-identical.

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ws_bar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void ws_bar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void ws_bar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WS_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra WS_DONE;\n\t"
        "bra WS_WAIT;\n\t"
        "WS_DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

constexpr int kWsGather = 16;  // gather warps per block (4 warpgroups)
constexpr int kWsEpi = 4;      // epilogue warps per block (1 warpgroup)
constexpr int kWsThreads = (kWsGather + kWsEpi) * 32;

template <int W>
constexpr size_t layer_ws_smem() {
    // acc_f [NG][W] + slots [kWsGather][G][W] doubles, NG = kWsGather * G, G = 256 / W
    return sizeof(double) * 2 * (size_t)kWsGather * (256 / W) * W;
}

// One block of 16 + 4 warps per SM.  The 20 warps leave 96 registers per thread (5 per SM
// sub-partition), which holds only ~5 gathers in flight per lane; setmaxnreg rebalances them:
// the gather warpgroups take 104 registers (the full 8-deep batches, checked in the SASS), the
// epilogue warpgroup 64 (16 x 104 + 4 x 64 = 20 x 96).
template <int W>
__global__ void __launch_bounds__(kWsThreads, 1) layer_ws_kernel(const LayerArgs p) {
    constexpr bool REG = true;
    static_assert(W >= 32, "epilogue lanes own whole columns");
    constexpr int LPR = W / 8;
    constexpr int G = 32 / LPR;
    constexpr int IPL = kChunk / LPR;
    constexpr int NG = kWsGather * G;
    constexpr int C = W / 32;  // columns per epilogue lane
    __shared__ double2 st[W];  // (mu, 1/sigma) of the previous step
    __shared__ uint64_t full_bar[kWsGather], empty_bar[kWsGather];
    __shared__ double red[kWsEpi][2 * W];
    extern __shared__ double dyn_smem[];
    double (*acc_f)[W] = reinterpret_cast<double (*)[W]>(dyn_smem);                   // [NG][W]
    double (*slot)[G][W] = reinterpret_cast<double (*)[G][W]>(dyn_smem + NG * W);     // [kWsGather][G][W]
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int t = threadIdx.x; t < NG * W; t += kWsThreads) (&acc_f[0][0])[t] = 0.0;
    if (threadIdx.x < kWsGather) {
        ws_bar_init(&full_bar[threadIdx.x], 32);
        ws_bar_init(&empty_bar[threadIdx.x], 32);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t step = (int64_t)gridDim.x * NG;

    if (warp < kWsGather) {
        if constexpr (REG) asm volatile("setmaxnreg.inc.sync.aligned.u32 104;" ::: "memory");
        const int q = lane % LPR, g = lane / LPR;
        const int grp = warp * G + g;
        const uint64_t* yin = reinterpret_cast<const uint64_t*>(p.yin);
        const uint64_t pol_idx = evict_first_policy(p.idx_ef);
        const int32_t amask = p.idx_any ? ~0 : ~3;
        int64_t base = (int64_t)blockIdx.x * NG + warp * G;
        int32_t nbeg = 0, nend = 0;
        int jfirst[IPL];
        if (base + g < p.n) {
            nbeg = __ldg(p.rp + base + g);
            nend = __ldg(p.rp + base + g + 1);
        }
        load_idx<IPL>(p.ci, nbeg & amask, nend, q, pol_idx, jfirst, p.idx_any);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        __syncthreads();  // barriers initialised, acc_f zeroed, st written
        uint32_t phase = 0;
        double* af = acc_f[grp] + 8 * q;
        for (; base < p.n; base += step, phase ^= 1u) {
            const int32_t row = (int32_t)(base + g);
            const int32_t beg = nbeg, end = nend;
            nbeg = nend = 0;
            if (base + step + g < p.n) {
                nbeg = __ldg(p.rp + base + step + g);
                nend = __ldg(p.rp + base + step + g + 1);
            }
            uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
            int nc = 0;
            bool folded = false;
            const int32_t start = beg & amask;
            const int nch = end > beg ? (end - start + kChunk - 1) / kChunk : 0;
            const int max_nch = __reduce_max_sync(kFull, nch);
            int jr[IPL];
#pragma unroll
            for (int k = 0; k < IPL; ++k) jr[k] = jfirst[k];
            if (max_nch == 0) load_idx<IPL>(p.ci, nbeg & amask, nend, q, pol_idx, jfirst, p.idx_any);
            for (int c = 0; c < max_nch; ++c) {
                const int32_t e0 = start + c * kChunk, e1 = e0 + kChunk;
                int jn[IPL];
                load_idx<IPL>(p.ci, e1, end, q, pol_idx, jn, p.idx_any);
                const int lo = beg > e0 ? beg - e0 : 0;
                int hi = end - e0;
                hi = hi < 0 ? 0 : (hi > kChunk ? kChunk : hi);
                if (__all_sync(kFull, lo == 0 && hi == kChunk)) {
#pragma unroll
                    for (int u0 = 0; u0 < kChunk; u0 += kBatch) {
                        uint64_t v[kBatch][4];
#pragma unroll
                        for (int t = 0; t < kBatch; ++t) {
                            const int u = u0 + t;
                            const int j = __shfl_sync(kFull, jr[u % IPL], u / IPL, LPR);
                            IGP_DASSERT(j >= 0 && j < p.n);
                            ldg256(yin + ((size_t)j * LPR + q) * 4, v[t]);
                        }
#pragma unroll
                        for (int t = 0; t < kBatch; ++t)
#pragma unroll
                            for (int k = 0; k < 4; ++k) acc[k] = fadd2(acc[k], v[t][k]);
                    }
                } else {
#pragma unroll
                    for (int u0 = 0; u0 < kChunk; u0 += kBatch) {
                        uint64_t v[kBatch][4];
#pragma unroll
                        for (int t = 0; t < kBatch; ++t) {
                            const int u = u0 + t;
                            const int j = __shfl_sync(kFull, jr[u % IPL], u / IPL, LPR);
                            v[t][0] = v[t][1] = v[t][2] = v[t][3] = 0ull;
                            if (u >= lo && u < hi) {
                                IGP_DASSERT(j >= 0 && j < p.n);
                                ldg256(yin + ((size_t)j * LPR + q) * 4, v[t]);
                            }
                        }
#pragma unroll
                        for (int t = 0; t < kBatch; ++t)
#pragma unroll
                            for (int k = 0; k < 4; ++k) acc[k] = fadd2(acc[k], v[t][k]);
                    }
                }
                if (c == 0) {
                    load_idx<IPL>(p.ci, nbeg & amask, nend, q, pol_idx, jfirst, p.idx_any);
                    const int32_t lo_e = __shfl_sync(kFull, nbeg, 0);
                    const int32_t hi_e = __shfl_sync(kFull, nend, 31);
                    if (lane == 0 && hi_e > lo_e) {
                        const uint64_t a0 = reinterpret_cast<uint64_t>(p.ci + lo_e) & ~(uint64_t)15;
                        const uint64_t a1 = (reinterpret_cast<uint64_t>(p.ci + hi_e) + 15) & ~(uint64_t)15;
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0))
                                     : "memory");
                    }
                }
                if (++nc == kFoldChunks && e1 < end) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float2 f = unpack2(acc[k]);
                        af[2 * k] += (double)f.x;
                        af[2 * k + 1] += (double)f.y;
                        acc[k] = 0ull;
                    }
                    nc = 0;
                    folded = true;
                }
#pragma unroll
                for (int k = 0; k < IPL; ++k) jr[k] = jn[k];
            }
            if (row < p.n) prefetch_l2(yin + ((size_t)row * LPR + q) * 4);  // the epilogue's own row
            // hand the batch over: wait until the epilogue has consumed the previous one
            ws_bar_wait(&empty_bar[warp], phase ^ 1u);
            double* sl = &slot[warp][g][8 * q];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float2 f = unpack2(acc[k]);
                double a0 = (double)f.x, a1 = (double)f.y;
                if (folded) {
                    a0 += af[2 * k];
                    a1 += af[2 * k + 1];
                    af[2 * k] = 0.0;
                    af[2 * k + 1] = 0.0;
                }
                sl[2 * k] = a0;
                sl[2 * k + 1] = a1;
            }
            ws_bar_arrive(&full_bar[warp]);
        }
        return;
    }

    // ---- epilogue warps
    if constexpr (REG) asm volatile("setmaxnreg.dec.sync.aligned.u32 64;" ::: "memory");
    const int ew = warp - kWsGather;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int c = threadIdx.x - kWsGather * 32; c < W; c += kWsEpi * 32) {
        double m = 0.0, is = 1.0;
        if (p.sums_in) column_stats(p.sums_in, c, W, p.n, p.ddof, m, is);
        st[c] = make_double2(m, is);
    }
    __syncthreads();
    const uint64_t pol_st = evict_first_policy(p.st_ef);
    double s1[C], s2[C];
#pragma unroll
    for (int k = 0; k < C; ++k) s1[k] = s2[k] = 0.0;
    double2 mc[C];
#pragma unroll
    for (int k = 0; k < C; ++k) mc[k] = st[lane * C + k];
    const float* yinf = reinterpret_cast<const float*>(p.yin);
    float* youtf = reinterpret_cast<float*>(p.yout);
    uint32_t phase = 0;
    for (int64_t b0 = (int64_t)blockIdx.x * NG; b0 < p.n; b0 += step, phase ^= 1u) {
        for (int w = ew; w < kWsGather; w += kWsEpi) {
            const int64_t base = b0 + w * G;
            if (base >= p.n) break;
            ws_bar_wait(&full_bar[w], phase);
            // all G rows' own values and node parameters first (their latencies overlap), then the math
            float y[G][C];
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const int64_t r = base + i < p.n ? base + i : p.n - 1;
                if constexpr (C == 1) {
                    y[i][0] = __ldg(yinf + r * W + lane);
                } else if constexpr (C == 2) {
                    const float2 v = __ldg(reinterpret_cast<const float2*>(yinf + r * W) + lane);
                    y[i][0] = v.x, y[i][1] = v.y;
                } else {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(yinf + r * W) + lane);
                    y[i][0] = v.x, y[i][1] = v.y, y[i][2] = v.z, y[i][3] = v.w;
                }
            }
            // lane i < G holds row i's {s, r} and {c_hi, c_lo}; broadcast by shuffles below
            float2 my_sr = make_float2(0.f, 0.f), my_cc = make_float2(0.f, 0.f);
            if (lane < G && base + lane < p.n) {
                my_sr = __ldg(p.sr + base + lane);
                if (p.sums_in) my_cc = __ldg(p.cc + base + lane);
            }
            float tt[G][C], ys[G];
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const float2 sr2 = make_float2(__shfl_sync(kFull, my_sr.x, i), __shfl_sync(kFull, my_sr.y, i));
                const float2 cc2 = make_float2(__shfl_sync(kFull, my_cc.x, i), __shfl_sync(kFull, my_cc.y, i));
                const double si = (double)sr2.x, cc = (double)cc2.x + (double)cc2.y;
#pragma unroll
                for (int k = 0; k < C; ++k) {
                    const double ad = slot[w][i][lane * C + k];
                    const float tself = y[i][k] * sr2.y;
                    const double P = ((double)p.theta * (double)tself + (double)p.alpha * si * ad - mc[k].x * cc) *
                                     mc[k].y;
                    tt[i][k] = p.linear ? (float)P : tanhf((float)P);
                }
                ys[i] = sr2.x;
            }
            ws_bar_arrive(&empty_bar[w]);  // this lane has read the slot: the gather warp may refill it
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const int64_t r = base + i;
                if (r < p.n) {
                    float yo[C];
#pragma unroll
                    for (int k = 0; k < C; ++k) {
                        yo[k] = ys[i] * tt[i][k];
                        const double xd = (double)tt[i][k];
                        s1[k] += grid_round(xd, p.grid_c);
                        s2[k] += grid_round(xd * xd, p.grid_c);
                    }
                    float* dst = youtf + r * W + lane * C;
                    if constexpr (C == 1) {
                        asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(dst), "f"(yo[0]), "l"(pol_st));
                    } else if constexpr (C == 2) {
                        asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1,%2}, %3;" ::"l"(dst), "f"(yo[0]),
                                     "f"(yo[1]), "l"(pol_st));
                    } else {
                        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(dst),
                                     "f"(yo[0]), "f"(yo[1]), "f"(yo[2]), "f"(yo[3]), "l"(pol_st));
                    }
                }
            }
        }
    }
    if (p.linear) return;
#pragma unroll
    for (int k = 0; k < C; ++k) {
        red[ew][lane * C + k] = s1[k];
        red[ew][W + lane * C + k] = s2[k];
    }
    asm volatile("bar.sync 1, %0;" ::"r"(kWsEpi * 32) : "memory");
    for (int t = threadIdx.x - kWsGather * 32; t < 2 * W; t += kWsEpi * 32) {
        double v = 0.0;
#pragma unroll
        for (int e = 0; e < kWsEpi; ++e) v += red[e][t];
        atomicAdd(p.sums_out + t, v);
    }
}

// Z~ = sigmoid((t - mu)/sigma) of a slice into columns [col0, col0 + W) of out [N][d]
// (relabelled row i is written to the row of its original id order[i])
template <int W>
__global__ void output_kernel(const float4* __restrict__ y, const float2* __restrict__ sr,
                              const double* __restrict__ sums, const int32_t* __restrict__ order, int32_t n, int d,
                              int col0, int mode, int ddof, float* __restrict__ out) {
    constexpr int LPR = W / 4;
    const int64_t total = (int64_t)n * LPR;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += stride) {
        const int64_t i = idx / LPR;
        const int q = (int)(idx % LPR);
        const float r = sr[i].y;
        const float4 v = y[idx];
        float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float t = a[k] * r;
            if (mode == IGP_MODE_LINEAR) {
                a[k] = t;
            } else {
                double mu = 0.0, isg = 1.0;
                if (sums) column_stats(sums, 4 * q + k, W, n, ddof, mu, isg);
                const float z = (float)(((double)t - mu) * isg);
                a[k] = (mode == IGP_MODE_FULL) ? 1.0f / (1.0f + expf(-z)) : z;
            }
        }
        IGP_DASSERT(order[i] >= 0 && order[i] < n);
        *(float4*)(out + (int64_t)order[i] * d + col0 + 4 * q) = make_float4(a[0], a[1], a[2], a[3]);
    }
}

// optional post-op (IGP_FLAG_ROW_L2, reading A12): z_i <- z_i / ||z_i||_2, one warp per row,
// fp64 sum of squares; rows with zero norm are left unchanged
__global__ void row_l2_kernel(float* __restrict__ out, int32_t n, int d) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
        float* z = out + i * d;
        double ss = 0.0;
        for (int c = lane; c < d; c += 32) ss += (double)z[c] * (double)z[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(kFull, ss, o);
        if (ss > 0.0) {
            const double inv = 1.0 / sqrt(ss);
            for (int c = lane; c < d; c += 32) z[c] = (float)((double)z[c] * inv);
        }
    }
}

int simple_grid(int64_t items, int threads, const DeviceInfo& di, int per_sm = 8) {
    int64_t g = (items + threads - 1) / threads;
    int64_t cap = (int64_t)di.num_sms * per_sm;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

template <int W, int NW>
constexpr size_t layer_smem() {
    return sizeof(double) * (size_t)(NW * (256 / W)) * W;  // acc_f: NG x W doubles (>= NW x 2W)
}

template <int W, int MB, int NW>
int layer_grid(int32_t n, const DeviceInfo& di) {
    // per device: the smem attribute is set (idempotently) before the occupancy is published
    static std::atomic<int> occ_cache[64];
    int occ = occ_cache[di.device & 63].load(std::memory_order_acquire);
    if (occ == 0) {
        cudaFuncSetAttribute(layer_kernel<W, MB, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)layer_smem<W, NW>());
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, layer_kernel<W, MB, NW>, NW * 32, layer_smem<W, NW>()) !=
                cudaSuccess ||
            o < 1)
            o = 1;
        occ = o;
        occ_cache[di.device & 63].store(o, std::memory_order_release);
    }
    const int64_t rows_per_block = (int64_t)NW * (32 / (W / 8));
    const int64_t want = (n + rows_per_block - 1) / rows_per_block;
    const int64_t cap = (int64_t)di.num_sms * occ;
    const int64_t g = want < cap ? want : cap;
    return (int)(g < 1 ? 1 : g);
}

// Measured random-gather bandwidth (GB/s) of B200 for row size R = 4W bytes vs the
// gathered footprint (profiles/r01/gather_microbench.txt, LDG.128, 40M gathers).
double gather_gbps(int row_bytes, double footprint_mb) {
    static const double F[10] = {8, 16, 32, 48, 64, 96, 128, 192, 256, 512};
    static const double T64[10] = {14515, 14580, 14547, 14387, 12495, 8663, 6775, 5039, 4314, 3161};
    static const double T128[10] = {19519, 19154, 18961, 18932, 18094, 14165, 11858, 9615, 8565, 6465};
    static const double T256[10] = {18934, 18520, 18268, 18172, 17635, 15312, 13101, 10682, 9541, 8173};
    const double* T = row_bytes <= 64 ? T64 : (row_bytes <= 128 ? T128 : T256);
    if (footprint_mb <= F[0]) return T[0];
    for (int k = 1; k < 10; ++k)
        if (footprint_mb <= F[k]) {
            const double a = (log(footprint_mb) - log(F[k - 1])) / (log(F[k]) - log(F[k - 1]));
            return T[k - 1] + a * (T[k] - T[k - 1]);
        }
    return T[9] * pow(512.0 / footprint_mb, 0.3);
}

// slice width: minimise predicted gather time + the CSR re-read per slice (IGP_SLICE_WIDTH overrides)
int choose_width(int d, int32_t n, int64_t nnz) {
    // measured (profiles/r01): W=32 slices are fastest once the W=64 slice exceeds ~64 MB
    // of gathered footprint; the model below reproduces that ranking.  W must divide d.
    if (const char* env = getenv("IGP_SLICE_WIDTH")) {
        const int w = atoi(env);
        if ((w == 16 || w == 32 || w == 64 || w == 128) && w <= d && d % w == 0) return w;
    }
    int best = 16;
    double best_t = 1e300;
    for (int w = 128; w >= 16; w /= 2) {  // from the widest: fewer slices win ties
        if (w > d || d % w != 0) continue;
        const double slices = (double)d / w;
        const double gather = (double)nnz * 4.0 * w / (gather_gbps(4 * w, (double)n * 4.0 * w / 1048576.0) * 1e9);
        const double csr = (4.0 * (double)nnz + 8.0 * n) / 6.0e12;
        const double t = slices * (gather + csr);
        if (t < best_t * 0.97) {
            best_t = t;
            best = w;
        }
    }
    return best;
}

template <int W, int MB>
igp_status run_embed_w(const CsrDevice& g, const igp_embed_opts& o, float* out, cudaStream_t s,
                       const DeviceInfo& di, HostCopy* hc) {
    const int32_t n = g.n;
    const int L = o.steps, d = o.d, nslices = d / W;
    // graphs too small to give every SM a block of 8 warps run 2-warp blocks (4x the blocks)
    const bool small = (n + 8 * (256 / W) - 1) / (8 * (256 / W)) < di.num_sms;
    const int grid = small ? layer_grid<W, MB, 2>(n, di) : layer_grid<W, MB, kBigNW>(n, di);
    // warp-specialised filter step (layer_ws_kernel): opt-in only (IGP_LAYER_WS=1, W >= 32).  It
    // beat the statically scheduled layer_kernel where the gathers are DRAM-bound (Large: -5% per
    // launch) and lost at the L2-sized headline slice (+18%: its 4 epilogue warps per SM cannot
    // keep up); layer_kernel with the dynamic row-batch schedule beats it on both (Large 5.39 vs
    // 5.64 ms per launch, interleaved A/B -- DESIGN.md §5).
    bool use_ws = false;
    int ws_grid = 0;
    if constexpr (W >= 32) {
        const char* e = getenv("IGP_LAYER_WS");
        use_ws = !small && e != nullptr && atoi(e) != 0;
        if (use_ws) {
            cudaFuncSetAttribute(layer_ws_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)layer_ws_smem<W>());
            int o = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, layer_ws_kernel<W>, kWsThreads, layer_ws_smem<W>()) !=
                    cudaSuccess ||
                o < 1)
                o = 1;
            const int64_t rows_per_block = (int64_t)kWsGather * (256 / W);
            const int64_t want = (n + rows_per_block - 1) / rows_per_block;
            const int64_t cap = (int64_t)di.num_sms * o;
            ws_grid = (int)(want < cap ? want : cap);
        }
    }
    const size_t nw = (size_t)n * W;
    // workspace: sr | cc (N + 2 float2 each) | y0 | y1 (N x W each) | sums [slices][L+1][2W]
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t off_sr = 0;
    const size_t off_cc = al(off_sr + sizeof(float2) * ((size_t)n + 2));
    const size_t off_y0 = al(off_cc + sizeof(float2) * ((size_t)n + 2));
    const size_t off_y1 = al(off_y0 + sizeof(float) * nw);
    const size_t off_sums = al(off_y1 + sizeof(float) * nw);
    // exact column sums [slices][L+1][2W] doubles, then the filter steps' row-batch counters
    // [slices][L+1][kCounters] ints: zeroed together once per embed
    const size_t sums_bytes =
        sizeof(double) * (size_t)nslices * (L + 1) * 2 * W + sizeof(int) * (size_t)nslices * (L + 1) * kCounters;
    char* ws = nullptr;
    IGP_CUDA(alloc_async((void**)&ws, off_sums + sums_bytes, s), "embed workspace alloc");
    float2* sr = (float2*)(ws + off_sr);
    float2* cc = (float2*)(ws + off_cc);
    float4* ybuf[2] = {(float4*)(ws + off_y0), (float4*)(ws + off_y1)};
    double* sums = (double*)(ws + off_sums);
    int* sched = (int*)(sums + (size_t)nslices * (L + 1) * 2 * W);
    bool dyn_sched = kDynSchedule;  // development knob IGP_DYN=0: static row-batch striding
    if (const char* e = getenv("IGP_DYN")) dyn_sched = atoi(e) != 0;
    // layer_kernel's dynamic schedule pays off once every warp takes several grabs
    const int64_t lk_warps = (int64_t)grid * (small ? 2 : kBigNW);
    const int64_t lk_batches = ((int64_t)n + (256 / W) - 1) / (256 / W);
    int dyn_min = 4;  // development knob IGP_DYN_MIN: grabs per warp below which the schedule stays static
    if (const char* e = getenv("IGP_DYN_MIN")) dyn_min = atoi(e);
    // ... and once a warp's share of the edges outlasts the counters' atomics (sparse graphs: the
    // streaming config's early stages ran 9% slower with it; cap ~ nnz)
    const bool use_dyn = dyn_sched && !small && lk_batches >= (int64_t)dyn_min * lk_warps * kGrab &&
                         g.cap >= kDynMinEdgesPerWarp * lk_warps;
    // stats grid 2^-gexp with N * 2^gexp < 2^51 (|sum t|, sum t^2 <= N)
    int lg = 0;
    while (lg < 62 && ((int64_t)1 << lg) <= (int64_t)n) ++lg;
    const int gexp = 51 - lg;
    const double grid_c = 1.5 * ldexp(1.0, 52 - gexp);

    float idx_ef = kIdxEvictFirst, st_ef = kStoreEvictFirst;  // L2 policies (development knobs)
    if (const char* e = getenv("IGP_IDX_EF")) idx_ef = (float)atof(e);
    if (const char* e = getenv("IGP_ST_EF")) st_ef = (float)atof(e);
    int idx_any = kIdxAnyStart;  // development knob IGP_IDX_ANY=0: 16-byte aligned index chunks
    if (const char* e = getenv("IGP_IDX_ANY")) idx_any = atoi(e) != 0;

    igp_status rc = IGP_OK;
    const bool timed = (o.flags & IGP_FLAG_TIME_LAYERS) != 0;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool joined = true;
    do {
        // all filter-step work runs on the relabelled CSR (rows in the handle's degree / community order)
        scale_kernel<<<simple_grid(n, 256, di), 256, 0, s>>>(g.rp_perm, n, (double)o.tau, (double)o.eps, sr);
        if ((rc = launch_status("scale_kernel")) != IGP_OK) break;
        // c_i (needed from filter step 2 on: step 1 applies mu = 0) runs on a side stream beside
        // the first slice's input and first filter step; joined before step 2 (or the slice end)
        cudaStream_t ss = side_stream(di.device);
        if ((rc = cuda_status(ss ? cudaSuccess : cudaErrorInvalidResourceHandle, "side stream")) != IGP_OK) break;
        if ((rc = cuda_status(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming), "event")) != IGP_OK) break;
        if ((rc = cuda_status(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming), "event")) != IGP_OK) break;
        if ((rc = cuda_status(cudaEventRecord(ev_fork, s), "event record")) != IGP_OK) break;
        if ((rc = cuda_status(cudaStreamWaitEvent(ss, ev_fork, 0), "stream wait")) != IGP_OK) break;
        affine_kernel<<<simple_grid((int64_t)n * 32, 256, di), 256, 0, ss>>>(g.rp_perm, g.col_perm, n, o.theta,
                                                                               o.alpha, sr, cc);
        rc = launch_status("affine_kernel");
        if (rc == IGP_OK) rc = cuda_status(cudaEventRecord(ev_join, ss), "event record");
        if (rc != IGP_OK) {
            cudaStreamSynchronize(ss);
            break;
        }
        joined = false;
        if ((rc = cuda_status(cudaMemsetAsync(sums, 0, sums_bytes, s), "sums memset")) != IGP_OK) break;
        const int linear = (o.mode == IGP_MODE_LINEAR) ? 1 : 0;
        for (int k = 0; k < nslices && rc == IGP_OK; ++k) {
            const int col0 = k * W;
            double* sk = sums + (size_t)k * (L + 1) * 2 * W;
            input_kernel<W><<<simple_grid((int64_t)n * (W / 4), 256, di), 256, 0, s>>>(o.seed, o.subsequence, n, d,
                                                                                      col0, g.order, sr, o.d_z0,
                                                                                      ybuf[0]);
            if ((rc = launch_status("input_kernel")) != IGP_OK) break;
            TimerSlot* ts = nullptr;
            if (timed && L > 0) {
                if (!(ts = timer_acquire(L))) {
                    rc = IGP_ERR_CUDA;
                    set_error("layer timer: event creation failed");
                    break;
                }
                cudaEventRecord(ts->ev0, s);
            }
            for (int l = 1; l <= L; ++l) {
                if (l == 2 && !joined) {  // c_i from the side stream
                    if ((rc = cuda_status(cudaStreamWaitEvent(s, ev_join, 0), "stream wait")) != IGP_OK) break;
                    joined = true;
                }
                LayerArgs a;
                a.rp = g.rp_perm;
                a.ci = g.col_perm;
                a.sr = sr;
                a.cc = cc;
                a.yin = ybuf[(l - 1) & 1];
                a.yout = ybuf[l & 1];
                a.sums_in = (linear || l == 1) ? nullptr : sk + (size_t)(l - 1) * 2 * W;
                a.sums_out = sk + (size_t)l * 2 * W;
                a.n = n;
                a.theta = o.theta;
                a.alpha = o.alpha;
                a.linear = linear;
                a.ddof = o.ddof;
                a.grid_c = grid_c;
                a.idx_ef = idx_ef;
                a.st_ef = st_ef;
                a.idx_any = idx_any;
                a.sched = use_dyn ? sched + ((size_t)k * (L + 1) + l) * kCounters : nullptr;
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(small ? 64 : kBigNW * 32);
                cfg.dynamicSmemBytes = small ? layer_smem<W, 2>() : layer_smem<W, kBigNW>();
                cfg.stream = s;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                cudaError_t le;
                if constexpr (W >= 32) {
                    if (use_ws) {
                        cfg.gridDim = dim3(ws_grid);
                        cfg.blockDim = dim3(kWsThreads);
                        cfg.dynamicSmemBytes = layer_ws_smem<W>();
                        le = cudaLaunchKernelEx(&cfg, layer_ws_kernel<W>, a);
                    } else {
                        le = small ? cudaLaunchKernelEx(&cfg, layer_kernel<W, MB, 2>, a)
                                   : cudaLaunchKernelEx(&cfg, layer_kernel<W, MB, kBigNW>, a);
                    }
                } else {
                    le = small ? cudaLaunchKernelEx(&cfg, layer_kernel<W, MB, 2>, a)
                               : cudaLaunchKernelEx(&cfg, layer_kernel<W, MB, kBigNW>, a);
                }
                if ((rc = cuda_status(le, "layer_kernel launch")) != IGP_OK) break;
                if ((rc = launch_status("layer_kernel")) != IGP_OK) break;
            }
            if (rc != IGP_OK) break;
            if (ts) cudaEventRecord(ts->ev1, s);
            const double* sfin = (linear || L == 0) ? nullptr : sk + (size_t)L * 2 * W;
            output_kernel<W><<<simple_grid((int64_t)n * (W / 4), 256, di), 256, 0, s>>>(ybuf[L & 1], sr, sfin, g.order, n,
                                                                                        d, col0, o.mode, o.ddof, out);
            if ((rc = launch_status("output_kernel")) != IGP_OK) break;
            if (hc && !(o.flags & IGP_FLAG_ROW_L2)) {  // this slice's columns are final: copy them
                                                          // out behind the remaining slices
                if ((rc = cuda_status(cudaEventRecord(hc->ev[k], s), "event record")) != IGP_OK) break;
                if ((rc = cuda_status(cudaStreamWaitEvent(hc->cs, hc->ev[k], 0), "stream wait")) != IGP_OK) break;
                rc = cuda_status(cudaMemcpy2DAsync(hc->h_out + col0, sizeof(float) * d, out + col0, sizeof(float) * d,
                                                   sizeof(float) * W, n, cudaMemcpyDeviceToHost, hc->cs),
                                 "slice D2H");
                if (rc != IGP_OK) break;
            }
        }
        if (rc == IGP_OK && (o.flags & IGP_FLAG_ROW_L2)) {  // needs every slice: after the last one
            row_l2_kernel<<<simple_grid((int64_t)n * 32, 256, di), 256, 0, s>>>(out, n, d);
            if ((rc = launch_status("row_l2_kernel")) != IGP_OK) break;
            if (hc) {
                if ((rc = cuda_status(cudaEventRecord(hc->ev[0], s), "event record")) != IGP_OK) break;
                if ((rc = cuda_status(cudaStreamWaitEvent(hc->cs, hc->ev[0], 0), "stream wait")) != IGP_OK) break;
                rc = cuda_status(cudaMemcpyAsync(hc->h_out, out, sizeof(float) * (size_t)n * d, cudaMemcpyDeviceToHost,
                                                 hc->cs),
                                 "D2H");
            }
        }
    } while (0);
    if (!joined) cudaStreamWaitEvent(s, ev_join, 0);  // the workspace is freed behind the side stream
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    free_async(ws, s);
    return rc;
}

}  // namespace

igp_status run_embed(const CsrDevice& g, const igp_embed_opts& o, float* out, cudaStream_t s, HostCopy* hc) {
    DeviceInfo di;
    if (!device_info(&di)) return IGP_ERR_CUDA;
    if (o.d < 16 || o.d > kMaxD || o.d % 16 != 0) {
        set_error("igp_embed: d must be a multiple of 16 in [16, 1024]");
        return IGP_ERR_UNSUPPORTED;
    }
    const char* occ_env = getenv("IGP_LAYER_OCC");  // development knob: 2 or 3 blocks per SM
    const int occ = occ_env ? atoi(occ_env) : kDefaultOcc;
#define IGP_W_CASE(WW)                                                      \
    case WW:                                                                \
        if (occ == 3) return run_embed_w<WW, 3>(g, o, out, s, di, hc); \
        if (occ == 4) return run_embed_w<WW, 4>(g, o, out, s, di, hc); \
        return run_embed_w<WW, 2>(g, o, out, s, di, hc);
    switch (choose_width(o.d, g.n, g.cap)) {  // a heuristic: cap ~ nnz (the output does not depend on W)
        IGP_W_CASE(16)
        IGP_W_CASE(32)
        IGP_W_CASE(64)
        default:
        IGP_W_CASE(128)
    }
#undef IGP_W_CASE
}

}  // namespace igp
