// birch.cu — BIRCH on the GPU: the downstream clustering of InfraredGP's embeddings
// (Alg. 1 l.7; streaming Alg. 2 l.9-11).
//
// The paper feeds Z~ to BIRCH (Zhang et al. 1996; scikit-learn's implementation with no
// cluster count): a single pass of CF-tree insertions in row order, the
// leaf entries being the K-agnostic clusters, then every row labelled by its nearest leaf
// centroid.  Insertion is inherently sequential (each point's path depends on every earlier
// point), so the fit runs as ONE persistent CTA that inserts the points one after another
// with all of its 128 threads on each insertion:
//   - the distances from x to a node's <= B + 1 entry centroids: one 2-lane group per entry,
//     the eight fma partials over k mod 8 split between the two lanes and combined in the
//     oracle's fixed order (reading B6), so every distance is bit-identical;
//   - first-minimum argmin over the entries (warp shuffles + one shared-memory round);
//   - the leaf's merge test (radius^2 <= T^2) and the CF updates of the path, parallel over
//     the d coordinates;
//   - node splits: all pairwise entry distances (upper triangle, 2 lanes per pair), the first
//     farthest pair, the two halves' CF sums in entry order.
// Everything is fp64 and follows oracle/birch_oracle.c step for step (same formulas, same
// operation order), so the tree -- and hence the clusters and labels -- are bit-identical to
// the oracle's.  The entry and node pools live in global memory (L1/L2-resident for the top
// levels); the fit stops cleanly before a point whose worst-case growth would overflow a pool,
// the host doubles the pools and relaunches from that point.
//
// Predict (Alg. 2 l.11) is data-parallel: label_i = argmin_j sqn_j - 2 c_j . x_i over the K
// leaf centroids (first minimum), one thread per point, cluster tiles staged in shared memory.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "igp_internal.cuh"

namespace igp {
namespace {

constexpr int kFitThreads = 128;  // 64 groups of 2 lanes: one node's <= B + 1 <= 64 entries at once
constexpr int kMaxDepth = 64;
constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kMaxBirchD = 1024;
constexpr int kMaxBirchBranching = 63;

// rows of X staged in shared memory ahead of the insertions (two chunks of ring_rows(d) rows, by
// cp.async): the next rows' loads overlap the current insertions instead of one DRAM round trip
// sitting on every insertion's critical path
__host__ __device__ constexpr int ring_rows(int d) { return 8192 / d < 2 ? 2 : (8192 / d > 64 ? 64 : 8192 / d); }

// tree header (device int64 words)
enum { H_NS = 0, H_NN, H_ROOT, H_FIRST_LEAF, H_NPOINTS, H_STOP, H_DEPTH, H_WORDS };

struct TreeDev {
    int d, B;
    double T2;
    // entries
    double* n;
    double* ls;   // [cap_s][d]
    double* ss;
    double* cen;  // [cap_s][ldc]
    int ldc;      // centroid row stride (doubles): d in global memory; d + 2 in the shared pool for even d
                  // (rows of consecutive entries then start in different bank groups)
    double* sqn;
    int32_t* child;
    int64_t cap_s;
    // nodes
    int32_t* is_leaf;
    int32_t* nsub;
    int32_t* sub;  // [cap_n][B + 1]
    int32_t* prev;
    int32_t* next;
    int64_t cap_n;
    long long* hdr;
};

// dot(a, b) in the oracle's order (reading B6: eight fma partials p_r over k = r (mod 8), k
// ascending, combined ((p0+p1)+(p2+p3))+((p4+p5)+(p6+p7))) on the 2 lanes of the calling group:
// lane h accumulates the partials r = 4h .. 4h+3 (contiguous k: 16-byte vector loads), forms its
// half of the tree locally, and one shuffle adds the two halves.  Both lanes return the full dot.
// `mask`: the calling lanes.
__device__ __forceinline__ double dot2(const double* a, const double* b, int d, int h, unsigned mask = kFullMask) {
    double p[4] = {0.0, 0.0, 0.0, 0.0};  // p[q] = partial r = 4h + q
    int k0 = 0;
    if ((d & 1) == 0) {  // rows start 16-byte aligned: two double2 loads per operand and block
        for (; k0 + 8 <= d; k0 += 8) {
            const double2 a0 = *reinterpret_cast<const double2*>(a + k0 + 4 * h);
            const double2 a1 = *reinterpret_cast<const double2*>(a + k0 + 4 * h + 2);
            const double2 b0 = *reinterpret_cast<const double2*>(b + k0 + 4 * h);
            const double2 b1 = *reinterpret_cast<const double2*>(b + k0 + 4 * h + 2);
            p[0] = __fma_rn(a0.x, b0.x, p[0]);
            p[1] = __fma_rn(a0.y, b0.y, p[1]);
            p[2] = __fma_rn(a1.x, b1.x, p[2]);
            p[3] = __fma_rn(a1.y, b1.y, p[3]);
        }
    } else {
        for (; k0 + 8 <= d; k0 += 8) {
#pragma unroll
            for (int q = 0; q < 4; ++q) p[q] = __fma_rn(a[k0 + 4 * h + q], b[k0 + 4 * h + q], p[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (k0 + 4 * h + q < d) p[q] = __fma_rn(a[k0 + 4 * h + q], b[k0 + 4 * h + q], p[q]);
    const double half = __dadd_rn(__dadd_rn(p[0], p[1]), __dadd_rn(p[2], p[3]));
    return __dadd_rn(half, __shfl_xor_sync(mask, half, 1));  // left + right on both lanes (commutative)
}

__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

struct FitShared {
    double best_d[kFitThreads / 32];
    int best_j[kFitThreads / 32 > 8 ? kFitThreads / 32 : 8];  // per-warp argmax (splits); split results
    double am_d[2][kFitThreads / 32];                           // per-warp argmin, two alternating slots
    int am_j[2][kFitThreads / 32];
    int path_node[kMaxDepth];
    int path_j[kMaxDepth];
    int ch[2][64];  // global trees: each entry's child, published by the argmin's barrier (alternating)
    int depth;
    int cur;      // broadcast slot
    int flag;
    double scal[4];
};

// argmin over groups g < cnt of dist (held by lane r == 0 of each group); first minimum.  One
// barrier: every thread reduces the per-warp results itself; the per-warp slots alternate between
// calls (`slot` toggles), and consecutive calls are separated by at least one other barrier.
__device__ int block_argmin(double dist, int g, int cnt, FitShared& sh, int& slot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double bd = (g < cnt && (threadIdx.x & 1) == 0) ? dist : INFINITY;
    int bj = (g < cnt && (threadIdx.x & 1) == 0) ? g : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(kFullMask, bd, o);
        const int oj = __shfl_xor_sync(kFullMask, bj, o);
        if (od < bd || (od == bd && oj < bj)) {
            bd = od;
            bj = oj;
        }
    }
    if (lane == 0) {
        sh.am_d[slot][warp] = bd;
        sh.am_j[slot][warp] = bj;
    }
    __syncthreads();
    double b = sh.am_d[slot][0];
    int j = sh.am_j[slot][0];
#pragma unroll
    for (int w = 1; w < kFitThreads / 32; ++w) {
        const double v = sh.am_d[slot][w];
        const int jw = sh.am_j[slot][w];
        if (v < b || (v == b && jw < j)) {
            b = v;
            j = jw;
        }
    }
    slot ^= 1;
    return j;
}

// CF_s += point x (n = 1, LS = x, SS = xx); c = LS / n, sqn = dot(c, c).  All threads.
__device__ void cf_add_point(const TreeDev& t, int s, const double* xs, double xx) {
    const int d = t.d;
    const double nn = t.n[s] + 1.0;
    for (int k = threadIdx.x; k < d; k += kFitThreads) {
        const double l = t.ls[(int64_t)s * d + k] + xs[k];
        t.ls[(int64_t)s * d + k] = l;
        t.cen[(int64_t)s * t.ldc + k] = l / nn;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        const double q = dot2(t.cen + (int64_t)s * t.ldc, t.cen + (int64_t)s * t.ldc, d, threadIdx.x, 0x3u);
        if (threadIdx.x == 0) {
            t.n[s] = nn;
            t.ss[s] = t.ss[s] + xx;
            t.sqn[s] = q;
        }
    }
    __syncthreads();
}

// a new zero entry (thread 0 only; returns its index)
__device__ int new_entry(const TreeDev& t) {
    const int s = (int)t.hdr[H_NS]++;
    t.n[s] = 0.0;
    t.ss[s] = 0.0;
    t.sqn[s] = 0.0;
    t.child[s] = -1;
    return s;
}
__device__ int new_node(const TreeDev& t, int leaf) {
    const int v = (int)t.hdr[H_NN]++;
    t.is_leaf[v] = leaf;
    t.nsub[v] = 0;
    t.prev[v] = t.next[v] = -1;
    return v;
}

// split node v (all threads).  Returns the two halves' entries in sh.scal-free ints via out.
__device__ void split_node(const TreeDev& t, int v, double* D, FitShared& sh, int* h_out) {
    const int d = t.d, B1 = t.B + 1;
    const int m = t.nsub[v];
    const int32_t* ent = t.sub + (int64_t)v * B1;
    const int g = threadIdx.x >> 1, r = threadIdx.x & 1;
    // pairwise d2 for a < b (one 2-lane group per pair), mirrored; diagonal 0
    const int P = m * (m - 1) / 2;
    for (int p0 = 0; p0 < P; p0 += kFitThreads / 2) {
        const int p = p0 + g;
        int a = 0, b = 0;
        if (p < P) {  // pair index p -> (a, b) in row-major order of the upper triangle
            int rem = p;
            a = 0;
            while (rem >= m - 1 - a) {
                rem -= m - 1 - a;
                ++a;
            }
            b = a + 1 + rem;
        }
        const int sa = ent[a], sb = ent[b];  // (a, b) = (0, 0) past the last pair: computed, discarded
        const double x = dot2(t.cen + (int64_t)sa * t.ldc, t.cen + (int64_t)sb * t.ldc, d, r);
        if (p < P && r == 0) {
            double v2 = __dadd_rn(__dadd_rn(-2.0 * x, t.sqn[sa]), t.sqn[sb]);
            v2 = v2 > 0.0 ? v2 : 0.0;
            D[a * m + b] = v2;
            D[b * m + a] = v2;
        }
    }
    for (int a = threadIdx.x; a < m; a += kFitThreads) D[a * m + a] = 0.0;
    __syncthreads();
    // first maximum in row-major order (over the upper triangle: a < b comes first)
    {
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int idx = threadIdx.x; idx < m * m; idx += kFitThreads)
            if (D[idx] > bv) {  // ascending idx per thread: keeps the first of equal maxima
                bv = D[idx];
                bi = idx;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(kFullMask, bv, o);
            const int oi = __shfl_xor_sync(kFullMask, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            sh.best_d[warp] = bv;
            sh.best_j[warp] = bi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double b = sh.best_d[0];
            int j = sh.best_j[0];
            for (int w = 1; w < kFitThreads / 32; ++w)
                if (sh.best_d[w] > b || (sh.best_d[w] == b && sh.best_j[w] < j)) {
                    b = sh.best_d[w];
                    j = sh.best_j[w];
                }
            // the new nodes and halves (thread 0)
            const int ia = j / m, ib = j % m;
            const int leaf = t.is_leaf[v];
            const int n1 = new_node(t, leaf), n2 = new_node(t, leaf);
            const int s1 = new_entry(t), s2 = new_entry(t);
            t.child[s1] = n1;
            t.child[s2] = n2;
            if (leaf) {  // n1 takes v's place in the leaf chain, n2 follows it
                const int pv = t.prev[v], qv = t.next[v];
                t.prev[n1] = pv;
                t.next[n1] = n2;
                t.prev[n2] = n1;
                t.next[n2] = qv;
                if (pv >= 0) t.next[pv] = n1; else t.hdr[H_FIRST_LEAF] = n1;
                if (qv >= 0) t.prev[qv] = n2;
            }
            double c1 = 0.0, c2 = 0.0, q1 = 0.0, q2 = 0.0;
            for (int i = 0; i < m; ++i) {
                const bool to1 = (i == ia) || (D[ia * m + i] < D[ib * m + i]);
                const int nd = to1 ? n1 : n2;
                t.sub[(int64_t)nd * B1 + t.nsub[nd]++] = ent[i];
                if (to1) {
                    c1 = c1 + t.n[ent[i]];
                    q1 = q1 + t.ss[ent[i]];
                } else {
                    c2 = c2 + t.n[ent[i]];
                    q2 = q2 + t.ss[ent[i]];
                }
            }
            t.n[s1] = c1;
            t.n[s2] = c2;
            t.ss[s1] = q1;
            t.ss[s2] = q2;
            sh.best_j[0] = s1;
            sh.best_j[1] = s2;
            sh.best_j[2] = n1;
            sh.best_j[3] = ia;
            sh.best_j[4] = ib;
        }
        __syncthreads();
    }
    const int s1 = sh.best_j[0], s2 = sh.best_j[1], ia = sh.best_j[3], ib = sh.best_j[4];
    // the halves' LS in entry order, then c = LS / n
    for (int k = threadIdx.x; k < d; k += kFitThreads) {
        double l1 = 0.0, l2 = 0.0;
        for (int i = 0; i < m; ++i) {
            const bool to1 = (i == ia) || (D[ia * m + i] < D[ib * m + i]);
            const double v2 = t.ls[(int64_t)ent[i] * d + k];
            if (to1) l1 = l1 + v2; else l2 = l2 + v2;
        }
        t.ls[(int64_t)s1 * d + k] = l1;
        t.ls[(int64_t)s2 * d + k] = l2;
        t.cen[(int64_t)s1 * t.ldc + k] = l1 / t.n[s1];
        t.cen[(int64_t)s2 * t.ldc + k] = l2 / t.n[s2];
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        const int s = threadIdx.x < 2 ? s1 : s2;
        const double q = dot2(t.cen + (int64_t)s * t.ldc, t.cen + (int64_t)s * t.ldc, d, threadIdx.x & 1, 0xfu);
        if ((threadIdx.x & 1) == 0) t.sqn[s] = q;
    }
    __syncthreads();
    h_out[0] = s1;
    h_out[1] = s2;
    __syncthreads();
}

// Insert rows [start, m) of X in order.  One CTA.  Stops (hdr[H_STOP] = i) before a point whose
// worst-case growth (one leaf entry, two entries and two nodes per split level, a new root)
// could overflow a pool.
// copy the live part of a tree (entries [0, ns), nodes [0, nn), header) between two layouts
__device__ void copy_tree(const TreeDev& dst, const TreeDev& src, long long ns, long long nn) {
    const int d = src.d, B1 = src.B + 1;
    for (long long e = threadIdx.x; e < ns; e += kFitThreads) {
        dst.n[e] = src.n[e];
        dst.ss[e] = src.ss[e];
        dst.sqn[e] = src.sqn[e];
        dst.child[e] = src.child[e];
    }
    for (long long e = threadIdx.x; e < ns * d; e += kFitThreads) {
        dst.ls[e] = src.ls[e];
        dst.cen[(e / d) * dst.ldc + e % d] = src.cen[(e / d) * src.ldc + e % d];
    }
    for (long long v = threadIdx.x; v < nn; v += kFitThreads) {
        dst.is_leaf[v] = src.is_leaf[v];
        dst.nsub[v] = src.nsub[v];
        dst.prev[v] = src.prev[v];
        dst.next[v] = src.next[v];
    }
    for (long long e = threadIdx.x; e < nn * B1; e += kFitThreads) dst.sub[e] = src.sub[e];
    for (int w = threadIdx.x; w < H_WORDS; w += kFitThreads) dst.hdr[w] = src.hdr[w];
}

// The insertion loop over rows [start, m).  Instantiated twice: SM = true with every tree pointer
// derived from the kernel's shared-memory pool inside the same inlined body (the compiler then
// emits shared-memory loads / stores instead of generic ones on the descent's dependent chain),
// SM = false for trees left in global memory.
#ifdef IGP_FIT_PROFILE  // phase cycle counts of thread 0, printed at the end of a launch (tooling builds only)
#define FIT_MARK(k)                                  \
    do {                                             \
        const long long _t = clock64();              \
        prof[k] += _t - prof_t;                      \
        prof_t = _t;                                 \
    } while (0)
#else
#define FIT_MARK(k) ((void)0)
#endif

template <bool SM>
__device__ __forceinline__ void fit_rows(TreeDev T, const float* __restrict__ X, int64_t m, int64_t start, double* xs,
                                         double* tmp, double* D, float* xring, FitShared& sh) {
    const int d = T.d, B1 = T.B + 1;
    const int CH = ring_rows(d);
    const int g = threadIdx.x >> 1, r = threadIdx.x & 1;
#ifdef IGP_FIT_PROFILE
    long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long prof_t = clock64();
#endif
    if (threadIdx.x == 0) T.hdr[H_STOP] = m;
    auto issue_chunk = [&](int64_t c) {  // rows [start + c CH, ...) into ring slot c & 1
        const int64_t r0 = start + c * CH;
        const int64_t r1 = r0 + CH < m ? r0 + CH : m;
        float* dst = xring + (size_t)(c & 1) * CH * d;
        const uint32_t sdst = (uint32_t)__cvta_generic_to_shared(dst);
        for (int64_t e = threadIdx.x; e < (r1 - r0) * d; e += kFitThreads)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sdst + 4u * (uint32_t)e), "l"(X + r0 * d + e)
                         : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    issue_chunk(0);
    int am_slot = 0;
    int64_t c = -1;  // current chunk of staged rows
    int in_chunk = CH;
    for (int64_t i = start; i < m; ++i) {
        if (in_chunk == CH) {  // entering chunk c + 1: queue the one after, wait for this one
            ++c;
            in_chunk = 0;
            issue_chunk(c + 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        }
        const int row_in_chunk = in_chunk++;
        // capacity (all threads read the same header values)
        __syncthreads();
        const long long ns = T.hdr[H_NS], nn = T.hdr[H_NN], dep = T.hdr[H_DEPTH];
        if (ns + 1 + 2 * (dep + 1) > T.cap_s || nn + 2 * (dep + 1) + 1 > T.cap_n || dep + 1 >= kMaxDepth) {
            if (threadIdx.x == 0) T.hdr[H_STOP] = i;
            break;
        }
        {
            const float* xr = xring + (size_t)(c & 1) * CH * d + (size_t)row_in_chunk * d;
            for (int k = threadIdx.x; k < d; k += kFitThreads) xs[k] = (double)xr[k];
        }
        __syncthreads();
        FIT_MARK(0);
        double xx = 0.0;  // |x|^2: computed beside the leaf's merge test (not on the descent's path)
        const int root = (int)T.hdr[H_ROOT];
        if (T.nsub[root] == 0) {  // the empty root leaf takes the first point
            if (threadIdx.x < 2) {
                xx = dot2(xs, xs, d, threadIdx.x, 0x3u);
                if (threadIdx.x == 0) sh.scal[0] = xx;
            }
            __syncthreads();
            xx = sh.scal[0];
            if (threadIdx.x == 0) sh.cur = new_entry(T);
            __syncthreads();
            const int s = sh.cur;
            for (int k = threadIdx.x; k < d; k += kFitThreads) T.ls[(int64_t)s * d + k] = 0.0;
            __syncthreads();
            cf_add_point(T, s, xs, xx);
            if (threadIdx.x == 0) {
                T.sub[(int64_t)root * B1 + T.nsub[root]++] = s;
                T.hdr[H_NPOINTS]++;
            }
            continue;
        }
        // descend: closest entry at every level
        int depth = 0, v = root;
        while (true) {
            const int cnt = T.nsub[v];
            const int leafv = T.is_leaf[v];
            // one 2-lane group per entry; groups past the node's entries stay idle
            double dist = INFINITY;
            const unsigned act = __ballot_sync(kFullMask, g < cnt);
            if (g < cnt) {
                const int s = T.sub[(int64_t)v * B1 + g];
                // a tree in global memory: every entry's next hop is fetched beside its distance
                // (the child and, into L1, that node's count / leaf flag / entry list; at a leaf,
                // the entry's LS row and counts for the merge test), so the winner's path costs L1
                // hits instead of dependent L2 round trips after the argmin
                const int ch = (!SM && !leafv) ? T.child[s] : -1;
                const double dt = dot2(T.cen + (int64_t)s * T.ldc, xs, d, r, act);
                dist = __dadd_rn(T.sqn[s], -2.0 * dt);
                if (!SM) {
                    if (!leafv) {
                        if (r == 0) {
                            sh.ch[am_slot][g] = ch;
                            prefetch_l1(T.nsub + ch);
                            prefetch_l1(T.is_leaf + ch);
                            prefetch_l1(T.sub + (int64_t)ch * B1);
                            prefetch_l1(T.sub + (int64_t)ch * B1 + B1 - 1);
                        }
                    } else {
                        for (int k = 16 * r; k < d; k += 32) prefetch_l1(T.ls + (int64_t)s * d + k);
                        if (r == 0) {
                            prefetch_l1(T.n + s);
                            prefetch_l1(T.ss + s);
                        }
                    }
                }
            }
            const int slot = am_slot;  // the ch slot this level wrote (block_argmin toggles am_slot)
            const int j = block_argmin(dist, g, cnt, sh, am_slot);
            if (threadIdx.x == 0) {
                sh.path_node[depth] = v;
                sh.path_j[depth] = j;
            }
            ++depth;
            if (leafv) break;
            v = SM ? T.child[T.sub[(int64_t)v * B1 + j]] : sh.ch[slot][j];
        }
        __syncthreads();
        FIT_MARK(1);
        // leaf: merge into the closest entry if the merged radius^2 <= T^2, else append
        const int leaf = v;
        const int sj = T.sub[(int64_t)leaf * B1 + sh.path_j[depth - 1]];
        const double nn1 = T.n[sj] + 1.0;
        const double inv = 1.0 / nn1;
        for (int k = threadIdx.x; k < d; k += kFitThreads) {
            const double l = T.ls[(int64_t)sj * d + k] + xs[k];
            tmp[k] = l;
            tmp[d + k] = inv * l;
        }
        __syncthreads();
        if (threadIdx.x < 2) {
            xx = dot2(xs, xs, d, threadIdx.x, 0x3u);  // independent of the next dot: the two overlap
            const double nsq = dot2(tmp + d, tmp + d, d, threadIdx.x, 0x3u);
            if (threadIdx.x == 0) {
                sh.scal[0] = xx;
                const double nss = T.ss[sj] + xx;
                const double r2 = nss / nn1 - nsq;
                sh.flag = r2 <= T.T2;
                sh.scal[1] = nsq;
                sh.scal[2] = nss;
            }
        }
        __syncthreads();
        xx = sh.scal[0];
        FIT_MARK(2);
        int split = 0;
        if (sh.flag) {
            for (int k = threadIdx.x; k < d; k += kFitThreads) {
                T.ls[(int64_t)sj * d + k] = tmp[k];
                T.cen[(int64_t)sj * T.ldc + k] = tmp[d + k];
            }
            if (threadIdx.x == 0) {
                T.n[sj] = nn1;
                T.ss[sj] = sh.scal[2];
                T.sqn[sj] = sh.scal[1];
            }
            __syncthreads();
        } else {
            if (threadIdx.x == 0) sh.cur = new_entry(T);
            __syncthreads();
            const int s = sh.cur;
            for (int k = threadIdx.x; k < d; k += kFitThreads) T.ls[(int64_t)s * d + k] = 0.0;
            __syncthreads();
            cf_add_point(T, s, xs, xx);
            if (threadIdx.x == 0) T.sub[(int64_t)leaf * B1 + T.nsub[leaf]++] = s;
            __syncthreads();
            split = T.nsub[leaf] > T.B;
        }
        FIT_MARK(3);
        // back up the path: splits bottom-up while they propagate, then one batched CF update of
        // every remaining ancestor entry (distinct entries: their order does not matter)
        int l = depth - 2;
        for (; l >= 0 && split; --l) {
            const int pv = sh.path_node[l], pj = sh.path_j[l];
            const int se = T.sub[(int64_t)pv * B1 + pj];
            int h[2];
            split_node(T, T.child[se], D, sh, h);
            if (threadIdx.x == 0) {
                T.sub[(int64_t)pv * B1 + pj] = h[0];
                T.sub[(int64_t)pv * B1 + T.nsub[pv]++] = h[1];
            }
            __syncthreads();
            split = T.nsub[pv] > T.B;
        }
        FIT_MARK(5);
        if (l >= 0) {  // levels 0..l: CF_e += x, c = LS / n, sqn = |c|^2
            const int nl = l + 1;
            for (int idx = threadIdx.x; idx < nl * d; idx += kFitThreads) {
                const int lv = idx / d, k = idx % d;
                const int se = T.sub[(int64_t)sh.path_node[lv] * B1 + sh.path_j[lv]];
                const double nn = T.n[se] + 1.0;
                const double lsum = T.ls[(int64_t)se * d + k] + xs[k];
                T.ls[(int64_t)se * d + k] = lsum;
                T.cen[(int64_t)se * T.ldc + k] = lsum / nn;
            }
            __syncthreads();
            for (int lv0 = 0; lv0 < nl; lv0 += kFitThreads / 2) {  // one 2-lane group per level
                const int lv = lv0 + g;
                const int se = T.sub[(int64_t)sh.path_node[lv < nl ? lv : 0] * B1 + sh.path_j[lv < nl ? lv : 0]];
                const double q = dot2(T.cen + (int64_t)se * T.ldc, T.cen + (int64_t)se * T.ldc, d, r);
                if (lv < nl && r == 0) {
                    T.n[se] = T.n[se] + 1.0;
                    T.ss[se] = T.ss[se] + xx;
                    T.sqn[se] = q;
                }
            }
            __syncthreads();
        }
        if (split) {  // the root itself split: a new internal root holds the two halves
            int h[2];
            split_node(T, root, D, sh, h);
            if (threadIdx.x == 0) {
                const int nr = new_node(T, 0);
                T.sub[(int64_t)nr * B1 + T.nsub[nr]++] = h[0];
                T.sub[(int64_t)nr * B1 + T.nsub[nr]++] = h[1];
                T.hdr[H_ROOT] = nr;
                T.hdr[H_DEPTH] = T.hdr[H_DEPTH] + 1;
            }
        }
        if (threadIdx.x == 0) T.hdr[H_NPOINTS]++;
        FIT_MARK(4);
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
#ifdef IGP_FIT_PROFILE
    if (threadIdx.x == 0)
        printf("fit profile (cycles, thread 0; rows %lld..%lld, smem tree %d): top+stage %lld descent %lld merge-test %lld "
               "write %lld ancestors+root %lld split %lld\n",
               (long long)start, (long long)T.hdr[H_STOP], (int)SM, prof[0], prof[1], prof[2], prof[3], prof[4], prof[5]);
#endif
}

// Insert rows [start, m) of X in order.  One CTA.  When the whole tree (plus the growth one
// launch may need) fits in the cap_s_sm / cap_n_sm pool carved from shared memory, the tree is
// moved there for the launch and written back at its end (every dependent lookup of the descent
// then costs a shared-memory access instead of an L2 round trip); otherwise it is used in place.
__global__ void __launch_bounds__(kFitThreads, 1) birch_fit_kernel(TreeDev t, const float* __restrict__ X, int64_t m,
                                                                    int64_t start, int64_t cap_s_sm, int64_t cap_n_sm) {
    extern __shared__ double fit_smem[];
    __shared__ FitShared sh;
    __shared__ int use_sm;
    const int d = t.d, B1 = t.B + 1;
    double* xs = fit_smem;              // [d] the point
    double* tmp = fit_smem + d;         // [2d] merge candidate LS', c'
    double* D = fit_smem + 3 * d;       // [(B+1)^2] split distances
    float* xring = reinterpret_cast<float*>(D + (((size_t)B1 * B1 + 1) & ~(size_t)1));  // [2][CH][d] staged rows
    const int CH = ring_rows(d);
    // shared-memory pool (if it holds the tree with room for at least a few hundred inserts)
    if (threadIdx.x == 0) {
        const long long ns0 = t.hdr[H_NS], nn0 = t.hdr[H_NN], dep0 = t.hdr[H_DEPTH];
        use_sm = cap_s_sm > 0 && ns0 + 64 + 2 * (dep0 + 2) <= cap_s_sm && nn0 + 2 * (dep0 + 2) + 8 <= cap_n_sm;
    }
    __syncthreads();
    if (use_sm) {
        TreeDev T = t;  // every pointer derived from fit_smem in this branch only
        char* p = reinterpret_cast<char*>(xring + (size_t)2 * CH * d);
        T.n = reinterpret_cast<double*>(p);
        T.ss = T.n + cap_s_sm;
        T.sqn = T.ss + cap_s_sm;
        T.ls = T.sqn + cap_s_sm;
        T.cen = T.ls + cap_s_sm * d;
        T.ldc = (d & 1) ? d : d + 2;
        T.hdr = reinterpret_cast<long long*>(T.cen + cap_s_sm * T.ldc);
        T.child = reinterpret_cast<int32_t*>(T.hdr + H_WORDS);
        T.is_leaf = T.child + cap_s_sm;
        T.nsub = T.is_leaf + cap_n_sm;
        T.prev = T.nsub + cap_n_sm;
        T.next = T.prev + cap_n_sm;
        T.sub = T.next + cap_n_sm;
        T.cap_s = cap_s_sm;
        T.cap_n = cap_n_sm;
        copy_tree(T, t, t.hdr[H_NS], t.hdr[H_NN]);
        __syncthreads();
        fit_rows<true>(T, X, m, start, xs, tmp, D, xring, sh);
        __syncthreads();
        copy_tree(t, T, T.hdr[H_NS], T.hdr[H_NN]);
    } else {
        fit_rows<false>(t, X, m, start, xs, tmp, D, xring, sh);
    }
}

// leaf entries in leaf-chain order -> idx[K], K -> *count.  The chain walk is a pointer chase
// (one dependent load per leaf); with the tree's next / nsub arrays staged in shared memory
// (nodes <= smem_nodes) a hop costs a shared-memory latency instead of an L2 one, thread 0
// records each leaf's rank and output offset, and the block then writes the entries in parallel.
// Larger trees walk global memory (one thread).
__global__ void __launch_bounds__(1024) birch_list_kernel(TreeDev t, int32_t* idx, long long* count, int smem_nodes) {
    extern __shared__ int32_t list_smem[];
    const int B1 = t.B + 1;
    const int nn = (int)t.hdr[H_NN];
    if (nn > smem_nodes) {
        if (threadIdx.x != 0) return;
        long long k = 0;
        for (int v = (int)t.hdr[H_FIRST_LEAF]; v >= 0; v = t.next[v])
            for (int j = 0; j < t.nsub[v]; ++j) {
                if (idx) idx[k] = t.sub[(int64_t)v * B1 + j];
                ++k;
            }
        *count = k;
        return;
    }
    int32_t* nxt = list_smem;       // [nn]
    int32_t* nsb = nxt + nn;        // [nn]
    int32_t* ord = nsb + nn;        // [nn] leaves in chain order
    int32_t* off = ord + nn;        // [nn] their first output position
    __shared__ int nleaves;
    for (int v = threadIdx.x; v < nn; v += blockDim.x) {
        nxt[v] = t.next[v];
        nsb[v] = t.nsub[v];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int r = 0, k = 0;
        for (int v = (int)t.hdr[H_FIRST_LEAF]; v >= 0; v = nxt[v]) {
            ord[r] = v;
            off[r++] = k;
            k += nsb[v];
        }
        nleaves = r;
        *count = k;
    }
    __syncthreads();
    if (!idx) return;
    const int L = nleaves;
    for (int e = threadIdx.x; e < L * B1; e += blockDim.x) {  // (leaf rank, slot) pairs
        const int r = e / B1, j = e - r * B1;
        const int v = ord[r];
        if (j < nsb[v]) idx[off[r] + j] = t.sub[(int64_t)v * B1 + j];
    }
}

// gather the listed entries: centroids, sqn, n, LS, SS (any output may be null)
__global__ void birch_gather_kernel(TreeDev t, const int32_t* __restrict__ idx, int64_t K, double* cen, double* sqn,
                                    double* n, double* ls, double* ss) {
    const int d = t.d;
    const int64_t total = K * d;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / d, k = e % d;
        const int s = idx[j];
        if (cen) cen[e] = t.cen[(int64_t)s * t.ldc + k];
        if (ls) ls[e] = t.ls[(int64_t)s * d + k];
        if (k == 0) {
            if (sqn) sqn[j] = t.sqn[s];
            if (n) n[j] = t.n[s];
            if (ss) ss[j] = t.ss[s];
        }
    }
}

// label_i = argmin_j sqn_j - 2 dot(c_j, x_i) (first minimum; the oracle's dot order).  128 points per block (one per
// thread), cluster tiles of kPT centroids staged in shared memory; the point's row lives in
// shared memory too (stride d + 1).  Rows: 0 .. n-1, or list[0 .. n) (the rows the tensor-core
// pass could not certify, birch_tc.cu).  Clusters: blockIdx.y's range [y kchunk, (y+1) kchunk);
// with several ranges (few rows: the grid would not fill the GPU) each block writes its range's
// (distance, index) to part_d / part_j [y][n] and birch_argmin_merge_kernel picks the minimum.
constexpr int kPredThreads = 128;  // points per block (fewer for wide rows, see launch_predict_fp64)
constexpr int kPT = 16;            // centroids per shared-memory tile
// XS: the block's rows are staged in shared memory (stride d + 1); otherwise (very wide rows)
// each thread reads its row from global memory (L1-cached)
template <bool XS>
__global__ void __launch_bounds__(kPredThreads) birch_predict_kernel(const double* __restrict__ cen,
                                                                    const double* __restrict__ sqn, int64_t K, int d,
                                                                    const float* __restrict__ X, int64_t n,
                                                                    const int32_t* __restrict__ list, int64_t kchunk,
                                                                    int32_t* __restrict__ labels,
                                                                    double* __restrict__ part_d,
                                                                    int32_t* __restrict__ part_j) {
    extern __shared__ double pred_smem[];
    const int P = blockDim.x;
    const int64_t i0 = (int64_t)blockIdx.x * P;
    auto row_of = [&](int64_t i) -> int64_t { return list ? (int64_t)list[i] : i; };
    double* cs = pred_smem;                   // [kPT][d]
    double* xs = pred_smem + (size_t)kPT * d;  // [P][d + 1] (XS)
    if (XS) {
        for (int e = threadIdx.x; e < P * d; e += P) {
            const int p = e / d, k = e % d;
            xs[p * (d + 1) + k] = (i0 + p < n) ? (double)X[row_of(i0 + p) * d + k] : 0.0;
        }
    }
    const int64_t i = i0 + threadIdx.x < n ? i0 + threadIdx.x : n - 1;
    const double* x = XS ? xs + threadIdx.x * (d + 1) : nullptr;
    const float* xg = X + row_of(i) * d;
    const int64_t jb = (int64_t)blockIdx.y * kchunk, je = jb + kchunk < K ? jb + kchunk : K;
    double best = INFINITY;
    int64_t bj = jb;
    for (int64_t j0 = jb; j0 < je; j0 += kPT) {
        const int nt = (int)(je - j0 < kPT ? je - j0 : kPT);
        __syncthreads();
        for (int e = threadIdx.x; e < nt * d; e += P) cs[e] = cen[j0 * d + e];
        __syncthreads();
        for (int jj = 0; jj < nt; ++jj) {
            const double* c = cs + jj * d;
            double p[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            int k = 0;
            for (; k + 8 <= d; k += 8) {
#pragma unroll
                for (int q = 0; q < 8; ++q) p[q] = __fma_rn(c[k + q], XS ? x[k + q] : (double)xg[k + q], p[q]);
            }
            for (; k < d; ++k) p[k & 7] = __fma_rn(c[k], XS ? x[k] : (double)xg[k], p[k & 7]);
            const double dt = __dadd_rn(__dadd_rn(__dadd_rn(p[0], p[1]), __dadd_rn(p[2], p[3])),
                                        __dadd_rn(__dadd_rn(p[4], p[5]), __dadd_rn(p[6], p[7])));
            const double dist = __dadd_rn(sqn[j0 + jj], -2.0 * dt);
            if (dist < best) {  // strict: keeps the first minimum
                best = dist;
                bj = j0 + jj;
            }
        }
    }
    if (i0 + threadIdx.x < n) {
        if (part_d) {
            part_d[(int64_t)blockIdx.y * n + i] = best;
            part_j[(int64_t)blockIdx.y * n + i] = (int32_t)bj;
        } else {
            labels[row_of(i)] = (int32_t)bj;
        }
    }
}

// the minimum over the cluster ranges, first range on ties (= the first minimum overall)
__global__ void birch_argmin_merge_kernel(const double* __restrict__ part_d, const int32_t* __restrict__ part_j, int ks,
                                          int64_t n, const int32_t* __restrict__ list, int32_t* __restrict__ labels) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double best = part_d[i];
        int32_t bj = part_j[i];
        for (int y = 1; y < ks; ++y) {
            const double v = part_d[(int64_t)y * n + i];
            if (v < best) {
                best = v;
                bj = part_j[(int64_t)y * n + i];
            }
        }
        labels[list ? (int64_t)list[i] : i] = bj;
    }
}

__global__ void nonfinite_kernel(const float* __restrict__ X, int64_t count, int32_t* bad) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(X[e])) *bad = 1;
}

igp_status launch_nonfinite_check(const float* X, int64_t count, int32_t* bad, cudaStream_t s) {
    IGP_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), s), "memset");
    const int grid = (int)std::min<int64_t>((count + 255) / 256, 8192);
    nonfinite_kernel<<<grid > 0 ? grid : 1, 256, 0, s>>>(X, count, bad);
    return launch_status("nonfinite_kernel");
}

}  // namespace
}  // namespace igp

using namespace igp;

// ------------------------------------------------------------------------------ host handle
struct igp_birch_s {
    TreeDev t{};
    int device = 0;
    void* pool = nullptr;
    int64_t points = 0;
    // the clusters' entry indices in label order, valid until the next partial fit
    int32_t* list = nullptr;
    int64_t list_cap = 0;
    int64_t list_k = 0;
    bool list_valid = false;
};

namespace {

// dynamic shared memory of the fit kernel before the tree pool: x, the merge candidate, the split
// distances (rounded to an even count: every array below stays 16-byte aligned), the staged rows
size_t smem_fit(int d, int B) {
    const size_t dd = ((size_t)(B + 1) * (B + 1) + 1) & ~(size_t)1;
    return sizeof(double) * ((size_t)3 * d + dd) + ((sizeof(float) * 2 * (size_t)ring_rows(d) * d + 15) & ~(size_t)15);
}
// shared-memory pool capacities (entries, nodes) that fit beside the fit kernel's scratch
void smem_pool_caps(int d, int B, int max_optin, int64_t* cs, int64_t* cn, size_t* bytes) {
    const size_t base = smem_fit(d, B) + 2048;  // + static shared memory
    const size_t ldc = (d & 1) ? (size_t)d : (size_t)d + 2;  // the kernel's padded centroid stride
    const size_t per_e = sizeof(double) * ((size_t)d + ldc + 3) + sizeof(int32_t);
    const size_t per_n = sizeof(int32_t) * ((size_t)B + 1 + 4);
    *cs = *cn = 0;
    *bytes = 0;
    if ((size_t)max_optin <= base) return;
    const size_t avail = (size_t)max_optin - base - sizeof(long long) * H_WORDS - 64;
    int64_t c = (int64_t)(avail / (per_e + per_n / 4 + 1));
    while (c > 0 && (size_t)c * per_e + (size_t)(c / 4 + 8) * per_n > avail) --c;
    if (c < 128) return;  // too small to be worth a launch-long residency
    c &= ~(int64_t)3;     // even entry count: the LS / centroid rows stay 16-byte aligned
    *cs = c;
    *cn = c / 4 + 8;
    *bytes = (size_t)c * per_e + (size_t)(*cn) * per_n + sizeof(long long) * H_WORDS;
}

// (re)allocate the pools with capacities (cs entries, cn nodes), copying the first (ns, nn) rows
igp_status grow(igp_birch_s* b, int64_t cs, int64_t cn, cudaStream_t s) {
    const int d = b->t.d, B1 = b->t.B + 1;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t off = 0;
    const size_t o_n = off; off = al(off + 8 * (size_t)cs);
    const size_t o_ls = off; off = al(off + 8 * (size_t)cs * d);
    const size_t o_ss = off; off = al(off + 8 * (size_t)cs);
    const size_t o_cen = off; off = al(off + 8 * (size_t)cs * d);
    const size_t o_sqn = off; off = al(off + 8 * (size_t)cs);
    const size_t o_child = off; off = al(off + 4 * (size_t)cs);
    const size_t o_leaf = off; off = al(off + 4 * (size_t)cn);
    const size_t o_nsub = off; off = al(off + 4 * (size_t)cn);
    const size_t o_sub = off; off = al(off + 4 * (size_t)cn * B1);
    const size_t o_prev = off; off = al(off + 4 * (size_t)cn);
    const size_t o_next = off; off = al(off + 4 * (size_t)cn);
    const size_t o_hdr = off; off = al(off + 8 * (size_t)H_WORDS);
    char* p = nullptr;
    IGP_CUDA(alloc_async((void**)&p, off, s), "birch pool alloc");
    TreeDev n = b->t;
    n.n = (double*)(p + o_n);
    n.ls = (double*)(p + o_ls);
    n.ss = (double*)(p + o_ss);
    n.cen = (double*)(p + o_cen);
    n.sqn = (double*)(p + o_sqn);
    n.child = (int32_t*)(p + o_child);
    n.is_leaf = (int32_t*)(p + o_leaf);
    n.nsub = (int32_t*)(p + o_nsub);
    n.sub = (int32_t*)(p + o_sub);
    n.prev = (int32_t*)(p + o_prev);
    n.next = (int32_t*)(p + o_next);
    n.hdr = (long long*)(p + o_hdr);
    n.cap_s = cs;
    n.cap_n = cn;
    if (b->pool) {
        long long h[H_WORDS];
        IGP_CUDA(cudaMemcpyAsync(h, b->t.hdr, sizeof(h), cudaMemcpyDeviceToHost, s), "birch header");
        IGP_CUDA(cudaStreamSynchronize(s), "birch sync");
        const int64_t ns = h[H_NS], nn = h[H_NN];
        const TreeDev& o = b->t;
        auto cp = [&](void* dst, const void* src, size_t bytes) {
            return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s) : cudaSuccess;
        };
        cudaError_t e = cudaSuccess;
        if (e == cudaSuccess) e = cp(n.n, o.n, 8 * ns);
        if (e == cudaSuccess) e = cp(n.ls, o.ls, 8 * ns * d);
        if (e == cudaSuccess) e = cp(n.ss, o.ss, 8 * ns);
        if (e == cudaSuccess) e = cp(n.cen, o.cen, 8 * ns * d);
        if (e == cudaSuccess) e = cp(n.sqn, o.sqn, 8 * ns);
        if (e == cudaSuccess) e = cp(n.child, o.child, 4 * ns);
        if (e == cudaSuccess) e = cp(n.is_leaf, o.is_leaf, 4 * nn);
        if (e == cudaSuccess) e = cp(n.nsub, o.nsub, 4 * nn);
        if (e == cudaSuccess) e = cp(n.sub, o.sub, 4 * nn * B1);
        if (e == cudaSuccess) e = cp(n.prev, o.prev, 4 * nn);
        if (e == cudaSuccess) e = cp(n.next, o.next, 4 * nn);
        if (e == cudaSuccess) e = cp(n.hdr, o.hdr, sizeof(h));
        if (e != cudaSuccess) {
            free_async(p, s);
            return cuda_status(e, "birch pool copy");
        }
        free_async(b->pool, s);
    }
    b->pool = p;
    b->t = n;
    return IGP_OK;
}

igp_status read_hdr(igp_birch_s* b, long long* h, cudaStream_t s) {
    IGP_CUDA(cudaMemcpyAsync(h, b->t.hdr, sizeof(long long) * H_WORDS, cudaMemcpyDeviceToHost, s), "birch header");
    IGP_CUDA(cudaStreamSynchronize(s), "birch sync");
    return IGP_OK;
}

// (re)build the cached cluster list (entry indices in leaf-chain order) after a fit; synchronous
igp_status refresh_list(igp_birch_s* b, const long long* h, cudaStream_t s) {
    if (b->list_valid) return IGP_OK;
    const int64_t ns = h[H_NS];  // entries of every node: an upper bound of the leaf entries
    if (b->list_cap < ns || !b->list) {
        if (b->list) free_async(b->list, s);
        b->list = nullptr;
        b->list_cap = 0;
        // capacity: 1.5x the entries (fewer reallocations as the tree grows), even (the count below is 8-B aligned)
        const int64_t cap = (std::max<int64_t>(ns + ns / 2, 1024) + 1) & ~(int64_t)1;
        IGP_CUDA(alloc_async((void**)&b->list, sizeof(int32_t) * (size_t)(cap + 2), s), "alloc");
        b->list_cap = cap;
    }
    long long* cnt = reinterpret_cast<long long*>(b->list + b->list_cap);  // past the entries
    DeviceInfo di;
    if (!device_info(&di)) return IGP_ERR_CUDA;
    const int smem_nodes = (int)std::min<int64_t>((di.max_smem_optin - 1024) / 16, INT32_MAX);
    const int nn = (int)h[H_NN];
    const size_t smem = nn <= smem_nodes ? (size_t)16 * nn : 0;
    IGP_CUDA(cudaFuncSetAttribute(birch_list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
             "birch list smem attribute");
    birch_list_kernel<<<1, 1024, smem, s>>>(b->t, b->list, cnt, smem_nodes);
    IGP_TRY(launch_status("birch_list_kernel"));
    long long k = 0;
    IGP_CUDA(cudaMemcpyAsync(&k, cnt, sizeof(k), cudaMemcpyDeviceToHost, s), "readback");
    IGP_CUDA(cudaStreamSynchronize(s), "birch sync");
    b->list_k = k;
    b->list_valid = true;
    return IGP_OK;
}

// the fp64 kernel over n rows (all rows, or the listed ones): points per block as many (<= 128,
// multiple of 32) as fit in shared memory with their rows; when the row blocks alone would not
// fill the GPU, the clusters are split into ranges (grid y) and merged by a second kernel
igp_status launch_predict_fp64(const double* cen, const double* sqn, int64_t K, int d, const float* X, int64_t n,
                               const int32_t* list, int32_t* labels, cudaStream_t s) {
    const size_t budget = 200 * 1024, tile = sizeof(double) * (size_t)kPT * d;
    int P = kPredThreads;
    while (P > 32 && tile + sizeof(double) * (size_t)P * (d + 1) > budget) P -= 32;
    const bool xs = tile + sizeof(double) * (size_t)P * (d + 1) <= budget;
    if (!xs) P = kPredThreads;
    const size_t smem = tile + (xs ? sizeof(double) * (size_t)P * (d + 1) : 0);
    auto kern = xs ? birch_predict_kernel<true> : birch_predict_kernel<false>;
    IGP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "predict smem attribute");
    DeviceInfo di;
    if (!device_info(&di)) return IGP_ERR_CUDA;
    const int64_t rb = (n + P - 1) / P, want = (int64_t)di.num_sms * 4;
    int64_t ks = rb >= want ? 1 : std::min<int64_t>((want + rb - 1) / rb, (K + 255) / 256);
    if (ks < 1) ks = 1;
    if (ks > 65535) ks = 65535;
    int64_t kchunk = (K + ks - 1) / ks;
    kchunk = (kchunk + kPT - 1) / kPT * kPT;
    ks = (K + kchunk - 1) / kchunk;
    double* pd = nullptr;
    int32_t* pj = nullptr;
    if (ks > 1) {
        IGP_CUDA(alloc_async((void**)&pd, sizeof(double) * (size_t)ks * n, s), "alloc");
        igp_status st = cuda_status(alloc_async((void**)&pj, sizeof(int32_t) * (size_t)ks * n, s), "alloc");
        if (st != IGP_OK) {
            free_async(pd, s);
            return st;
        }
    }
    kern<<<dim3((unsigned)rb, (unsigned)ks), P, smem, s>>>(cen, sqn, K, d, X, n, list, kchunk, labels, pd, pj);
    igp_status st = launch_status("birch_predict_kernel");
    if (st == IGP_OK && ks > 1) {
        birch_argmin_merge_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, s>>>(pd, pj, (int)ks, n,
                                                                                                   list, labels);
        st = launch_status("birch_argmin_merge_kernel");
    }
    if (pd) free_async(pd, s);
    if (pj) free_async(pj, s);
    return st;
}

}  // namespace

extern "C" {

igp_status igp_birch_create(int32_t d, double threshold, int32_t branching, igp_birch_t* out) {
    set_error("");
    if (!out) {
        set_error("out handle pointer is NULL");
        return IGP_ERR_INPUT;
    }
    *out = nullptr;
    if (d < 1 || d > kMaxBirchD || !(threshold > 0.0) || !std::isfinite(threshold) || branching < 2 ||
        branching > kMaxBirchBranching) {
        set_error("birch: need 1 <= d <= 1024, finite threshold > 0, 2 <= branching <= 63");
        return IGP_ERR_INPUT;
    }
    DeviceInfo di;
    if (!device_info(&di)) return IGP_ERR_CUDA;
    igp_birch_s* b = new (std::nothrow) igp_birch_s();
    if (!b) return IGP_ERR_OOM;
    b->device = di.device;
    b->t.d = d;
    b->t.ldc = d;
    b->t.B = branching;
    b->t.T2 = threshold * threshold;
    cudaStream_t s = 0;
    igp_status st = grow(b, 1024, 256, s);
    if (st == IGP_OK) {
        // header: ns 0, nn 1 (the empty root leaf 0), root 0, first leaf 0, depth 1
        long long h[H_WORDS] = {0, 1, 0, 0, 0, 0, 1};
        int32_t root[3] = {1, 0, -1};  // is_leaf, nsub, prev/next
        st = cuda_status(cudaMemcpyAsync(b->t.hdr, h, sizeof(h), cudaMemcpyHostToDevice, s), "birch init");
        if (st == IGP_OK) st = cuda_status(cudaMemcpyAsync(b->t.is_leaf, &root[0], 4, cudaMemcpyHostToDevice, s), "init");
        if (st == IGP_OK) st = cuda_status(cudaMemcpyAsync(b->t.nsub, &root[1], 4, cudaMemcpyHostToDevice, s), "init");
        if (st == IGP_OK) st = cuda_status(cudaMemcpyAsync(b->t.prev, &root[2], 4, cudaMemcpyHostToDevice, s), "init");
        if (st == IGP_OK) st = cuda_status(cudaMemcpyAsync(b->t.next, &root[2], 4, cudaMemcpyHostToDevice, s), "init");
        if (st == IGP_OK) st = cuda_status(cudaStreamSynchronize(s), "birch sync");
    }
    if (st != IGP_OK) {
        if (b->pool) {
            free_async(b->pool, s);
            cudaStreamSynchronize(s);
        }
        delete b;
        return st;
    }
    *out = b;
    return IGP_OK;
}

igp_status igp_birch_partial_fit(igp_birch_t b, const float* d_X, int64_t m, igp_stream_t stream) {
    set_error("");
    if (!b || m < 0 || (m > 0 && !d_X)) {
        set_error("birch handle or rows invalid");
        return IGP_ERR_INPUT;
    }
    if (m == 0) return IGP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int d = b->t.d;
    // non-finite rows are an input error: checked on the device before any insert
    int32_t* bad = nullptr;
    IGP_CUDA(alloc_async((void**)&bad, sizeof(int32_t), s), "alloc");
    igp_status st = launch_nonfinite_check(d_X, m * (int64_t)d, bad, s);
    int32_t hbad = 0;
    if (st == IGP_OK) st = cuda_status(cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s), "readback");
    if (st == IGP_OK) st = cuda_status(cudaStreamSynchronize(s), "sync");
    free_async(bad, s);
    if (st != IGP_OK) return st;
    if (hbad) {
        set_error("birch: non-finite value in the rows");
        return IGP_ERR_INPUT;
    }
    DeviceInfo di;
    if (!device_info(&di)) return IGP_ERR_CUDA;
    int64_t cs_sm = 0, cn_sm = 0;
    size_t pool_bytes = 0;
    smem_pool_caps(d, b->t.B, di.max_smem_optin, &cs_sm, &cn_sm, &pool_bytes);
    // never more than the global pools hold (the tree is written back into them)
    if (cs_sm > b->t.cap_s || cn_sm > b->t.cap_n) cs_sm = cn_sm = 0;
    const size_t smem = smem_fit(d, b->t.B) + (cs_sm ? pool_bytes : 0);
    IGP_CUDA(cudaFuncSetAttribute(birch_fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
             "birch smem attribute");
    int64_t start = 0;
    while (start < m) {
        birch_fit_kernel<<<1, kFitThreads, smem, s>>>(b->t, d_X, m, start, cs_sm, cn_sm);
        IGP_TRY(launch_status("birch_fit_kernel"));
        long long h[H_WORDS];
        IGP_TRY(read_hdr(b, h, s));
        start = h[H_STOP];
        if (start < m) {  // a pool would overflow: double both and continue from row `start`
            IGP_TRY(grow(b, 2 * b->t.cap_s + (int64_t)2 * (h[H_DEPTH] + 2), 2 * b->t.cap_n + 2 * (h[H_DEPTH] + 2), s));
        }
    }
    b->points += m;
    b->list_valid = false;
    return IGP_OK;
}

igp_status igp_birch_info(igp_birch_t b, int64_t* num_clusters, int32_t* depth, int64_t* nodes, int64_t* points) {
    set_error("");
    if (!b) {
        set_error("birch handle is NULL");
        return IGP_ERR_INPUT;
    }
    cudaStream_t s = 0;
    long long h[H_WORDS] = {0};
    IGP_TRY(read_hdr(b, h, s));
    IGP_TRY(refresh_list(b, h, s));
    if (num_clusters) *num_clusters = b->list_k;
    if (depth) *depth = (int32_t)h[H_DEPTH];
    if (nodes) *nodes = h[H_NN];
    if (points) *points = h[H_NPOINTS];
    return IGP_OK;
}

igp_status igp_birch_clusters(igp_birch_t b, double* d_centroids, double* d_sqn, double* d_n, double* d_ls,
                              double* d_ss, igp_stream_t stream) {
    set_error("");
    if (!b) {
        set_error("birch handle is NULL");
        return IGP_ERR_INPUT;
    }
    int64_t K = 0;
    IGP_TRY(igp_birch_info(b, &K, nullptr, nullptr, nullptr));  // the list is current after this
    if (K == 0) return IGP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int grid = (int)std::min<int64_t>((K * b->t.d + 255) / 256, 4096);
    birch_gather_kernel<<<grid, 256, 0, s>>>(b->t, b->list, K, d_centroids, d_sqn, d_n, d_ls, d_ss);
    return launch_status("birch_gather_kernel");
}

igp_status igp_birch_predict_ex(igp_birch_t b, const float* d_X, int64_t m, int32_t* d_labels, int32_t path,
                                int64_t* ambiguous, igp_stream_t stream) {
    set_error("");
    if (!b || m < 0 || (m > 0 && (!d_X || !d_labels))) {
        set_error("birch handle or buffers invalid");
        return IGP_ERR_INPUT;
    }
    if (path != IGP_PREDICT_AUTO && path != IGP_PREDICT_FP64 && path != IGP_PREDICT_TENSOR) {
        set_error("birch: unknown predict path");
        return IGP_ERR_INPUT;
    }
#ifdef IGP_TC_STATS
    auto now = [] { cudaDeviceSynchronize(); return std::chrono::steady_clock::now(); };
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto t0 = now();
#endif
    int64_t K = 0;
    IGP_TRY(igp_birch_info(b, &K, nullptr, nullptr, nullptr));
#ifdef IGP_TC_STATS
    const auto t1 = now();
#endif
    if (K == 0) {
        set_error("birch: predict on an empty tree");
        return IGP_ERR_INPUT;
    }
    const int d = b->t.d;
    const bool tc_ok = birch_tc_eligible(d, K);
    if (path == IGP_PREDICT_TENSOR && !tc_ok) {
        set_error("birch: the tensor-core predict needs d a multiple of 8 in [8, 64]");
        return IGP_ERR_INPUT;
    }
    const bool tc = path != IGP_PREDICT_FP64 && tc_ok;
    if (ambiguous) *ambiguous = tc ? 0 : m;
    if (m == 0) return IGP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    double* cen = nullptr;
    double* sqn = nullptr;
    int32_t* amb_rows = nullptr;
    unsigned long long* amb_count = nullptr;
    IGP_CUDA(alloc_async_class((void**)&cen, 8 * ((size_t)K * d + (size_t)K), s), "alloc");  // centroids, then sqn
    sqn = cen + (size_t)K * d;
    igp_status st = igp_birch_clusters(b, cen, sqn, nullptr, nullptr, nullptr, stream);
#ifdef IGP_TC_STATS
    const auto t2 = now();
#endif
    int64_t n = m;  // rows left for the fp64 kernel
    if (st == IGP_OK && tc) {
        st = cuda_status(alloc_async_class((void**)&amb_rows, 4 * (size_t)m, s), "alloc");
        if (st == IGP_OK) st = cuda_status(alloc_async((void**)&amb_count, 2 * sizeof(unsigned long long), s), "alloc");
        if (st == IGP_OK) st = launch_birch_tc(cen, sqn, K, d, d_X, m, d_labels, amb_rows, amb_count, s);
        unsigned long long h[2] = {0, 0};  // the grid of the fp64 pass is sized by the uncertified count
        if (st == IGP_OK) st = cuda_status(cudaMemcpyAsync(h, amb_count, sizeof(h), cudaMemcpyDeviceToHost, s), "readback");
        if (st == IGP_OK) st = cuda_status(cudaStreamSynchronize(s), "sync");
        n = (int64_t)h[0];
        if (ambiguous) *ambiguous = (int64_t)(h[0] + h[1]);
#ifdef IGP_TC_STATS  // diagnostics builds: how the tensor-core pass settled the rows
        const auto t3 = now();
        fprintf(stderr, "birch tc predict: %lld rows, K %lld: %llu re-checked in the kernel, %llu to the fp64 pass; "
                "host ms: info %.2f clusters %.2f tensor passes %.2f\n",
                (long long)m, (long long)K, h[1], h[0], ms(t0, t1), ms(t1, t2), ms(t2, t3));
#endif
    }
    if (st == IGP_OK && n > 0) st = launch_predict_fp64(cen, sqn, K, d, d_X, n, tc ? amb_rows : nullptr, d_labels, s);
    free_async(cen, s);
    if (amb_rows) free_async(amb_rows, s);
    if (amb_count) free_async(amb_count, s);
    return st;
}

igp_status igp_birch_predict(igp_birch_t b, const float* d_X, int64_t m, int32_t* d_labels, igp_stream_t stream) {
    return igp_birch_predict_ex(b, d_X, m, d_labels, IGP_PREDICT_AUTO, nullptr, stream);
}

igp_status igp_birch_destroy(igp_birch_t b) {
    if (!b) return IGP_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != b->device) cudaSetDevice(b->device);
    cudaStreamSynchronize(0);  // the tree's calls are synchronous or ordered on the caller's stream
    if (b->pool) free_async(b->pool, 0);
    if (b->list) free_async(b->list, 0);
    if (prev >= 0 && prev != b->device) cudaSetDevice(prev);
    delete b;
    return IGP_OK;
}

}  // extern "C"
