// embed.cu — igp_embed: Alg. 1 lines 1-6 on one GPU.
//
// Kernels:
//   E1a scale_kernel     D_tau by Eq. (1) / D + tau I in fp64;
//                        per node {s = D^-1/2, r = D^1/2} as fp32
//   E1b affine_kernel    c_i = theta + alpha s_i sum_{j in N(i)} s_j   ( = (phi * 1)_i )
//   E2  input_kernel     Theta = X / sqrt(d), X ~ Philox/Box-Muller N(0,1);  y0 = s * Theta
//   E3  layer_kernel<D>  one filter step, L launches:  gather y_j = s_j t_j rows
//                        (float4, one warp per row, 32/(D/4) neighbour groups),
//                        Eq. (3) with the deferred column z-score, tanh (Eq. (4)),
//                        store y' = s t', per-column fp64 sum / sum-of-squares;
//                        the last block to finish reduces the block partials in a
//                        fixed order and publishes (mu, 1/sigma) for the next step
//   E4  output_kernel    Z~ = sigmoid((t - mu)/sigma)  (Eq. (4))
//
// Deferred ZNorm.  ZNorm is a per-column affine map and phi* is linear, so with
// t = tanh(P) of the previous step and Z = (t - mu)/sigma:
//   phi * Z = [theta t_i + alpha s_i sum_j s_j t_j - mu c_i] / sigma,  c_i = (phi * 1)_i.
// Hence the normalised matrix is never written: each step stores y = s t once
// and the next step applies (mu, 1/sigma) while it gathers.
#include <cmath>

#include "igp_internal.cuh"
#include "philox.cuh"

namespace igp {
namespace {

constexpr int kLayerThreads = 256;
constexpr unsigned kFull = 0xffffffffu;

__global__ void scale_kernel(const int32_t* __restrict__ rp, int32_t n, double tau, double eps,
                             float4* __restrict__ node, double2* __restrict__ st0, int d,
                             unsigned* __restrict__ counter) {
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
        node[i] = make_float4(s, r, 0.0f, 0.0f);
    }
    if (blockIdx.x == 0) {
        for (int c = threadIdx.x; c < d; c += blockDim.x) st0[c] = make_double2(0.0, 1.0);  // Z^(0) = Theta
        if (threadIdx.x == 0) *counter = 0u;
    }
}

// c_i = theta + alpha s_i sum_j s_j, one warp per row, fp64 sum, fixed shuffle tree
__global__ void affine_kernel(const int32_t* __restrict__ rp, const int32_t* __restrict__ ci, int32_t n,
                              float theta, float alpha, float4* __restrict__ node) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
        const int32_t beg = rp[i], end = rp[i + 1];
        double acc = 0.0;
        for (int32_t e = beg + lane; e < end; e += 32) acc += (double)node[ci[e]].x;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == 0) {
            const float s = node[i].x;
            const double c = (end > beg) ? (double)theta + (double)alpha * (double)s * acc : (double)theta;
            const float chi = (float)c;
            node[i].z = chi;  // c_i as an unevaluated sum hi + lo (~48 bits)
            node[i].w = (float)(c - (double)chi);
        }
    }
}

// y0 = s_i * Theta_i,  Theta = X / sqrt(d); element (i, c) is draw k = i*d + c (block k/4)
__global__ void input_kernel(uint64_t seed, uint64_t sub, int32_t n, int d, const float4* __restrict__ node,
                             float4* __restrict__ y0) {
    const int64_t nb = (int64_t)n * d / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const double sqd = sqrt((double)d);
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += stride) {
        const U4 r = philox_block(seed, sub, (uint64_t)b);
        double x0, x1, x2, x3;
        box_muller64(r.x, r.y, x0, x1);
        box_muller64(r.z, r.w, x2, x3);
        const double s = (double)node[(4 * b) / d].x;
        y0[b] = make_float4((float)(s * (x0 / sqd)), (float)(s * (x1 / sqd)), (float)(s * (x2 / sqd)),
                            (float)(s * (x3 / sqd)));
    }
}

struct LayerParams {
    const int32_t* rp;
    const int32_t* ci;
    const float4* node;
    const float4* yin;
    float4* yout;
    const double2* st_in;  // [D] (mu, 1/sigma) of the previous step
    double2* st_out;       // [D] (mu, 1/sigma) of this step
    double* st64_out;      // [2D] (mu, sigma) record
    double* partials;     // [gridDim.x][2D]
    unsigned* counter;
    int32_t n;
    float theta, alpha;
    int linear;
};

__device__ __forceinline__ float4 ldg4(const float4* p) { return __ldg(p); }

__device__ __forceinline__ void add4(float4& a, const float4& b) {
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
}

template <int D>
__global__ void __launch_bounds__(kLayerThreads) layer_kernel(const LayerParams p) {
    constexpr int LPR = D / 4;   // lanes per feature row (one float4 each)
    constexpr int G = 32 / LPR;  // neighbour groups per warp
    constexpr int NW = kLayerThreads / 32;
    constexpr int B = LPR < 8 ? LPR : 8;  // loads in flight per lane per batch
    __shared__ double red[NW][2 * D];
    __shared__ double fin[kLayerThreads];
    __shared__ int is_last;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = lane % LPR, g = lane / LPR;
    double mu[4], isg[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double2 m = p.st_in[4 * q + k];
        mu[k] = m.x;
        isg[k] = m.y;
    }
    double s1[4] = {0.0, 0.0, 0.0, 0.0}, s2[4] = {0.0, 0.0, 0.0, 0.0};

    for (int32_t row = blockIdx.x * NW + warp; row < p.n; row += gridDim.x * NW) {
        const int32_t beg = __ldg(p.rp + row), end = __ldg(p.rp + row + 1);
        // neighbour sum: fp32 within a 32-neighbour chunk, chunks folded in fp64
        double ad[4] = {0.0, 0.0, 0.0, 0.0};
        for (int32_t e0 = beg; e0 < end; e0 += 32) {
            const int cnt = min(32, end - e0);
            const int32_t jl = lane < cnt ? __ldg(p.ci + e0 + lane) : 0;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int t0 = 0; t0 < LPR; t0 += B) {
                if (t0 * G >= cnt) break;
                float4 v[B];
#pragma unroll
                for (int t = 0; t < B; ++t) {
                    const int k = (t0 + t) * G + g;
                    const int32_t j = __shfl_sync(kFull, jl, k);
                    v[t] = (k < cnt) ? ldg4(p.yin + (size_t)j * LPR + q) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int t = 0; t < B; ++t) add4(acc, v[t]);
            }
            ad[0] += (double)acc.x;
            ad[1] += (double)acc.y;
            ad[2] += (double)acc.z;
            ad[3] += (double)acc.w;
        }
#pragma unroll
        for (int o = LPR; o < 32; o <<= 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) ad[k] += __shfl_xor_sync(kFull, ad[k], o);
        }
        if (g == 0) {
            const float4 nd = __ldg(p.node + row);  // {s, r, c_hi, c_lo}
            const float4 own = ldg4(p.yin + (size_t)row * LPR + q);
            const double si = (double)nd.x, ci = (double)nd.z + (double)nd.w;
            const float y[4] = {own.x, own.y, own.z, own.w};
            float o4[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float tself = y[k] * nd.y;  // t_i = y_i / s_i
                const double P = ((double)p.theta * (double)tself + (double)p.alpha * si * ad[k] - mu[k] * ci) * isg[k];
                const float t = p.linear ? (float)P : tanhf((float)P);
                s1[k] += (double)t;
                s2[k] = fma((double)t, (double)t, s2[k]);
                o4[k] = nd.x * t;
            }
            p.yout[(size_t)row * LPR + q] = make_float4(o4[0], o4[1], o4[2], o4[3]);
        }
    }
    if (p.linear) return;

    // ---- block partials of (sum t, sum t^2) per column, fixed order
    if (g == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            red[warp][4 * q + k] = s1[k];
            red[warp][D + 4 * q + k] = s2[k];
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * D; t += kLayerThreads) {
        double v = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) v += red[w][t];
        p.partials[(size_t)blockIdx.x * (2 * D) + t] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(p.counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!is_last) return;
    __threadfence();

    // ---- last block: fixed-order reduction over blocks, then (mu, 1/sigma)
    constexpr int NS = 2 * D;
    constexpr int NG = kLayerThreads / NS > 0 ? kLayerThreads / NS : 1;
    double v = 0.0;
    if (threadIdx.x < NS * NG) {
        const int t = threadIdx.x % NS, grp = threadIdx.x / NS;
#pragma unroll 8
        for (int b = grp; b < (int)gridDim.x; b += NG) v += __ldcg(p.partials + (size_t)b * NS + t);
    }
    fin[threadIdx.x] = v;
    __syncthreads();
    if (threadIdx.x < NS) {
        double tot = 0.0;
        for (int grp = 0; grp < NG; ++grp) tot += fin[grp * NS + threadIdx.x];
        red[0][threadIdx.x] = tot;
    }
    __syncthreads();
    if (threadIdx.x < D) {
        const double S = red[0][threadIdx.x], Q = red[0][D + threadIdx.x];
        const double invN = 1.0 / (double)p.n;
        const double m = S * invN;
        double var = Q * invN - m * m;  // population variance (reading A2)
        var = var > 0.0 ? var : 0.0;
        const double sd = sqrt(var);
        const double inv = sd < 1e-8 ? 0.0 : 1.0 / sd;  // degenerate column -> 0 (reading A3)
        p.st_out[threadIdx.x] = make_double2(m, inv);
        p.st64_out[threadIdx.x] = m;
        p.st64_out[D + threadIdx.x] = sd;
    }
    if (threadIdx.x == 0) *p.counter = 0u;
}

template <int D>
__global__ void output_kernel(float4* __restrict__ y, const float4* __restrict__ node, const double2* __restrict__ st,
                              int32_t n, int mode) {
    constexpr int LPR = D / 4;
    const int64_t total = (int64_t)n * LPR;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += stride) {
        const int64_t i = idx / LPR;
        const int q = (int)(idx % LPR);
        const float r = node[i].y;
        float4 v = y[idx];
        float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float t = a[k] * r;
            if (mode == IGP_MODE_LINEAR) {
                a[k] = t;
            } else {
                const double2 m = st[4 * q + k];
                const float z = (float)(((double)t - m.x) * m.y);
                a[k] = (mode == IGP_MODE_FULL) ? 1.0f / (1.0f + expf(-z)) : z;
            }
        }
        y[idx] = make_float4(a[0], a[1], a[2], a[3]);
    }
}

template <int D>
int layer_grid(int32_t n, const DeviceInfo& di) {
    static int occ_cache[64] = {0};
    int& occ = occ_cache[di.device & 63];
    if (occ == 0) {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, layer_kernel<D>, kLayerThreads, 0) != cudaSuccess || o < 1)
            o = 1;
        occ = o;
    }
    const int64_t rows_per_block = kLayerThreads / 32;
    int64_t want = (n + rows_per_block - 1) / rows_per_block;
    int64_t cap = (int64_t)di.num_sms * occ;
    int64_t gsz = want < cap ? want : cap;
    return (int)(gsz < 1 ? 1 : gsz);
}

int simple_grid(int64_t items, int threads, const DeviceInfo& di, int per_sm = 8) {
    int64_t g = (items + threads - 1) / threads;
    int64_t cap = (int64_t)di.num_sms * per_sm;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

template <int D>
igp_status run_embed_d(const CsrDevice& g, const igp_embed_opts& o, float* out, cudaStream_t s, EmbedTiming* timing) {
    DeviceInfo di;
    if (!device_info(&di)) return IGP_ERR_CUDA;
    const int32_t n = g.n;
    const int L = o.steps;
    const int grid = layer_grid<D>(n, di);
    const size_t nd = (size_t)n * D;
    // workspace: node | y (N x D) | partials | st | st64 | counter
    size_t off_node = 0;
    size_t off_y = off_node + sizeof(float4) * (size_t)n;
    size_t off_part = off_y + sizeof(float) * nd;
    size_t off_st = off_part + sizeof(double) * (size_t)grid * 2 * D;
    size_t off_st64 = off_st + sizeof(double2) * (size_t)(L + 1) * D;
    size_t off_cnt = off_st64 + sizeof(double) * (size_t)(L + 1) * 2 * D;
    size_t total = off_cnt + 256;
    char* ws = nullptr;
    IGP_CUDA(alloc_async((void**)&ws, total, s), "embed workspace alloc");
    float4* node = (float4*)(ws + off_node);
    float* ybuf = (float*)(ws + off_y);
    double* partials = (double*)(ws + off_part);
    double2* st = (double2*)(ws + off_st);
    double* st64 = (double*)(ws + off_st64);
    unsigned* counter = (unsigned*)(ws + off_cnt);
    auto buf = [&](int l) -> float* { return ((L - l) % 2 == 0) ? out : ybuf; };

    igp_status rc = IGP_OK;
    do {
        scale_kernel<<<simple_grid(n, 256, di), 256, 0, s>>>(g.row_ptr, n, (double)o.tau, (double)o.eps, node, st, D,
                                                               counter);
        if ((rc = launch_status("scale_kernel")) != IGP_OK) break;
        // (an empty graph gives c_i = theta for every row)
        affine_kernel<<<simple_grid((int64_t)n * 32, 256, di), 256, 0, s>>>(g.row_ptr, g.col_idx, n, o.theta,
                                                                              o.alpha, node);
        if ((rc = launch_status("affine_kernel")) != IGP_OK) break;
        input_kernel<<<simple_grid((int64_t)nd / 4, 256, di), 256, 0, s>>>(o.seed, o.subsequence, n, D, node,
                                                                            (float4*)buf(0));
        if ((rc = launch_status("input_kernel")) != IGP_OK) break;
        const bool timed = (o.flags & IGP_FLAG_TIME_LAYERS) && timing;
        if (timed) {
            if (!timing->ev0) cudaEventCreate(&timing->ev0);
            if (!timing->ev1) cudaEventCreate(&timing->ev1);
            cudaEventRecord(timing->ev0, s);
        }
        const int linear = (o.mode == IGP_MODE_LINEAR) ? 1 : 0;
        for (int l = 1; l <= L; ++l) {
            LayerParams lp;
            lp.rp = g.row_ptr;
            lp.ci = g.col_idx;
            lp.node = node;
            lp.yin = (const float4*)buf(l - 1);
            lp.yout = (float4*)buf(l);
            lp.st_in = linear ? st : st + (size_t)(l - 1) * D;
            lp.st_out = st + (size_t)l * D;
            lp.st64_out = st64 + (size_t)l * 2 * D;
            lp.partials = partials;
            lp.counter = counter;
            lp.n = n;
            lp.theta = o.theta;
            lp.alpha = o.alpha;
            lp.linear = linear;
            layer_kernel<D><<<grid, kLayerThreads, 0, s>>>(lp);
            if ((rc = launch_status("layer_kernel")) != IGP_OK) break;
        }
        if (rc != IGP_OK) break;
        if (timed) {
            cudaEventRecord(timing->ev1, s);
            timing->launches = L;
            timing->valid = true;
        }
        const double2* st_final = linear ? st : st + (size_t)L * D;
        output_kernel<D><<<simple_grid((int64_t)nd / 4, 256, di), 256, 0, s>>>((float4*)out, node, st_final, n,
                                                                               o.mode);
        if ((rc = launch_status("output_kernel")) != IGP_OK) break;
    } while (0);
    free_async(ws, s);
    return rc;
}

}  // namespace

igp_status run_embed(const CsrDevice& g, const igp_embed_opts& o, float* out, cudaStream_t s, EmbedTiming* timing) {
    switch (o.d) {
        case 16: return run_embed_d<16>(g, o, out, s, timing);
        case 32: return run_embed_d<32>(g, o, out, s, timing);
        case 64: return run_embed_d<64>(g, o, out, s, timing);
        case 128: return run_embed_d<128>(g, o, out, s, timing);
        default:
            set_error("igp_embed: d must be one of 16, 32, 64, 128");
            return IGP_ERR_UNSUPPORTED;
    }
}

}  // namespace igp
