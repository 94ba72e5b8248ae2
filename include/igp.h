/*
 * igp.h — C ABI of the B200-native InfraredGP feed-forward-propagation (FFP) library.
 *
 * InfraredGP (arXiv 2508.19737) embeds the nodes of an undirected, unweighted
 * graph by pushing random Gaussian noise through L layers of a low-pass
 * spectral-GNN filter on the negatively corrected graph Laplacian, with no
 * training (§III).  This library implements Alg. 1 lines
 * 1-6 on one GPU:
 *
 *   igp_build_graph   the problem statement's graph G = (V, E), A symmetric
 *                     binary with no self loops, as a
 *                     canonical device CSR;
 *   igp_embed         Alg. 1 l.1-6: D_tau by Eq. (1) or
 *                     D + tau I; Theta ~ N(0, 1/d) (PAPER.md:161,
 *                     :186); L layers Z <- ZNorm(tanh(phi * Z)) with
 *                     phi * Z = theta Z + alpha D^-1/2 A D^-1/2 Z (Eq. (2)/(3),
 *                     PAPER.md:143-157; Eq. (4)); output
 *                     Z~ = sigmoid(Z^(L)).
 *
 * Conventions (all functions):
 *   - extern "C", no exceptions cross the ABI; every call returns igp_status.
 *   - Pointers named d_* are DEVICE pointers (CUDA global memory of the current
 *     device); h_* are HOST pointers (pageable or pinned).
 *   - `stream` is a cudaStream_t (a CUstream handle) passed as void*; NULL means
 *     the legacy default stream.  Work is enqueued on it; unless stated
 *     otherwise the call returns before the work completes (asynchronous, like a
 *     kernel launch) and device faults surface at the caller's next sync.
 *   - On any non-OK status no output is written and no handle is created;
 *     igp_last_error_message() gives a thread-local detail string.
 *   - The library never falls back to the CPU: with no usable CUDA device every
 *     call returns IGP_ERR_CUDA.
 *   - Development knobs (read from the environment at each embed; measurement tooling
 *     only, results are bitwise independent of all of them): IGP_SLICE_WIDTH (16/32/64/128
 *     columns per slice), IGP_LAYER_OCC (2/3/4 blocks per SM), IGP_IDX_EF / IGP_ST_EF
 *     (fraction of index loads / output stores marked L2 evict_first).
 */
#ifndef IGP_H_
#define IGP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define IGP_API __attribute__((visibility("default")))
#else
#define IGP_API
#endif

typedef struct igp_graph_s* igp_graph_t;
typedef void* igp_stream_t; /* cudaStream_t */

typedef enum {
    IGP_OK = 0,
    IGP_ERR_INPUT = 2,       /* invalid argument or edge index out of range */
    IGP_ERR_NUMERICAL = 4,   /* reserved */
    IGP_ERR_CUDA = 5,        /* CUDA runtime/launch error (detail in igp_last_error_message) */
    IGP_ERR_OOM = 6,         /* device allocation failed */
    IGP_ERR_UNSUPPORTED = 7  /* valid request outside this build's envelope (e.g. d not a multiple of 16) */
} igp_status;

/* ---------------------------------------------------------------------------
 * Graph construction  (§II: A_ij = A_ji = 1 iff (v_i,v_j) in E)
 * ------------------------------------------------------------------------- */

/* Build the canonical CSR of the undirected simple graph on num_nodes nodes.
 *   d_edges    device, int32 [num_edges][2] row-major (u, v) pairs; borrowed until the
 *              build's work on `stream` has completed.  Duplicates, both orientations
 *              and self loops are allowed: self loops are dropped, each unordered pair
 *              {u, v}, u != v, becomes A_uv = A_vu = 1 once.
 *   num_edges  >= 0 (0 is valid: M = 0, all degrees 0); 2*num_edges must be
 *              <= INT32_MAX - 64 (int32 CSR offsets; else IGP_ERR_UNSUPPORTED).
 *   num_nodes  N >= 1 (else IGP_ERR_INPUT) and <= 2^30 - 4096 (else IGP_ERR_UNSUPPORTED: the
 *              builder's int32 scans and digit histograms cover ~2N entries).
 *   out        receives a new handle owning device row_ptr int32[N+1] and
 *              col_idx int32[2M] (rows ascending, columns strictly ascending); the
 *              column arrays are allocated for the 2*num_edges directed entries before
 *              deduplication (no host round trip is needed to size them).
 * Errors: any index outside [0, N) -> IGP_ERR_INPUT (detected on the device; the
 * offending edges are skipped).
 * Synchronisation: every kernel is enqueued first, then the call waits once for the
 * build to complete (to report the error flag and nnz).  With IGP_BUILD_ASYNC it does
 * not wait at all: see igp_graph_status. */
IGP_API igp_status igp_build_graph(const int32_t* d_edges, int64_t num_edges, int32_t num_nodes,
                           igp_stream_t stream, igp_graph_t* out);

#define IGP_BUILD_DEFAULT 0u    /* row order chosen by size: IGP_BUILD_REORDER_COMMUNITY when a 32-column
                                   feature slice (N x 128 B) exceeds half the L2, else IGP_BUILD_REORDER_DEGREE */
#define IGP_BUILD_NO_REORDER 1u /* keep the original node order for the filter steps (no relabelling;
                                   results differ only by fp32 summation order) */
#define IGP_BUILD_REORDER_DEGREE 8u /* rows by descending degree (ties by ascending id) */
#define IGP_BUILD_REORDER_COMMUNITY 4u /* rows grouped by label-propagation communities (8 synchronous
                                   sweeps, mode of <= 31 neighbour labels and the node's own, ties to the
                                   smallest label), descending degree within a community: neighbour gathers
                                   stay local in L2 on graphs whose feature slice exceeds it.
                                   At most one of NO_REORDER / REORDER_DEGREE / REORDER_COMMUNITY. */
#define IGP_BUILD_ASYNC 2u      /* fully asynchronous build (and later igp_graph_add_edges): the call
                                   returns after enqueueing; a range error is reported by the first
                                   igp_graph_status / igp_graph_info / igp_graph_copy_csr call, which
                                   waits for the build.  Embeds may be enqueued behind it right away. */

/* As igp_build_graph; `flags` selects the filter steps' row order and the synchronisation.
 * Unless IGP_BUILD_NO_REORDER is given, the handle also holds a relabelled copy of the CSR
 * (rows in the chosen order, each row's neighbours in canonical order) which the embed kernels
 * traverse; the canonical CSR, the output row order and the results' meaning do not change.
 * Unknown or conflicting flags -> IGP_ERR_INPUT. */
IGP_API igp_status igp_build_graph_ex(const int32_t* d_edges, int64_t num_edges, int32_t num_nodes, uint32_t flags,
                                      igp_stream_t stream, igp_graph_t* out);

/* Streaming update (Alg. 2 l.1): merge a batch of new edges (same rules as
 * igp_build_graph, node ids in [0, N)) into the graph in place, on the device: the result
 * is the canonical CSR of the union, as if built from all edges at once, with the row
 * order (relabelling) recomputed.  The previous CSR is released in stream order.  Waits
 * once for the merge, and on a range error leaves the graph unchanged; a graph built with
 * IGP_BUILD_ASYNC does not wait, skips the bad edges and reports IGP_ERR_INPUT from
 * igp_graph_status.  Not safe concurrently with an embed of g on another stream. */
IGP_API igp_status igp_graph_add_edges(igp_graph_t g, const int32_t* d_edges, int64_t num_edges,
                                       igp_stream_t stream);

/* Query a graph: N, nnz = 2M (directed CSR entries) and M.  Any output pointer may be NULL.
 * Waits for an outstanding IGP_BUILD_ASYNC build/merge; returns its range error, if any. */
IGP_API igp_status igp_graph_info(igp_graph_t g, int32_t* num_nodes, int64_t* nnz, int64_t* num_undirected_edges);

/* Wait for the graph's build / last merge and return IGP_OK or IGP_ERR_INPUT (an edge
 * index outside [0, N) was skipped).  Immediate for graphs built without IGP_BUILD_ASYNC. */
IGP_API igp_status igp_graph_status(igp_graph_t g);

/* Copy the canonical CSR (original node ids) into caller-owned device buffers
 * d_row_ptr int32[N+1], d_col_idx int32[nnz] and d_deg int32[N] (deg_i = row_ptr[i+1] -
 * row_ptr[i], the degree diagonal D of PAPER.md:82); d_deg may be NULL.  Asynchronous on
 * `stream`. */
IGP_API igp_status igp_graph_copy_csr(igp_graph_t g, int32_t* d_row_ptr, int32_t* d_col_idx, int32_t* d_deg,
                                      igp_stream_t stream);

/* Release a graph.  Waits only for the work this library enqueued on the graph (its build /
 * merges and every embed's use of it, tracked by events), never for unrelated streams; the
 * memory is released in stream order behind those uses.  NULL is a no-op. */
IGP_API igp_status igp_destroy_graph(igp_graph_t g);

/* Release a graph in stream order on `stream` without any host synchronisation: all
 * work that reads g must be on `stream` or ordered before it (e.g. by events).
 * NULL g is a no-op. */
IGP_API igp_status igp_destroy_graph_async(igp_graph_t g, igp_stream_t stream);

/* ---------------------------------------------------------------------------
 * Embedding  (Alg. 1 lines 1-6)
 * ------------------------------------------------------------------------- */

#define IGP_MODE_FULL 0        /* Z~ = sigmoid(Z^(L))                      (Eq. (4)) */
#define IGP_MODE_PRE_SIGMOID 1 /* Z^(L) (column z-scored), debug/test      */
#define IGP_MODE_LINEAR 2      /* Z^(l) = phi * Z^(l-1): no tanh/ZNorm/sigmoid, debug/test */

#define IGP_FLAG_ROW_L2 2u      /* post-op, NOT part of the paper's method (Eq. (4) ends with the sigmoid):
                                   each output row scaled to unit L2 norm (fp64 norm), zero rows unchanged;
                                   for consumers that want the north star's "rows normalised" reading (A12) */
#define IGP_FLAG_TIME_LAYERS 1u /* record CUDA events on `stream` around each slice's L filter-step
                                   launches into the process-wide layer timer (igp_layer_timer_*) */

typedef struct {
    float tau;            /* degree correction tau (Eq. (1) for tau < 0; D + tau I otherwise); finite */
    int32_t d;            /* embedding dimensionality: a multiple of 16 in [16, 1024] (the paper uses 16-64) */
    int32_t steps;        /* L >= 0 filter steps (layers) */
    uint64_t seed;        /* Philox key for Theta */
    uint64_t subsequence; /* Philox subsequence (e.g. streaming stage t, Alg. 2 l.3) */
    float theta;          /* Eq. (2) theta, default 0.1 */
    float alpha;          /* Eq. (2) alpha, default 1.0 */
    float eps;            /* Eq. (1) epsilon > 0, default 0.001 */
    int32_t mode;         /* IGP_MODE_* */
    uint32_t flags;       /* IGP_FLAG_* */
    const float* d_z0;    /* NULL (default): Z^(0) = Theta from Philox (Alg. 1 l.2).  Otherwise a
                             caller-owned device fp32 [N][d] row-major Z^(0) (row i = node id i), 16-byte
                             aligned, used instead of Theta: an inspection / verification hook (e.g.
                             layer-by-layer checks from a given state, Alg. 1 l.3 "Z^(0) <- Theta" replaced) */
    int32_t ddof;         /* ZNorm's standard deviation divides by N - ddof: 0 (default) = population std
                             (reading A2; PAPER.md:166 does not say), 1 = sample std.  0 <= ddof <= 1;
                             a column with N <= ddof is treated as constant (reading A3) */
} igp_embed_opts;

/* Fill opts with the paper's defaults: theta 0.1, alpha 1, eps 1e-3, subsequence 0,
 * mode FULL, flags 0, d_z0 NULL (tau/d/steps/seed left at 0 for the caller to set). */
IGP_API void igp_embed_opts_default(igp_embed_opts* opts);

/* Z~ for graph g written to d_out, device fp32 [N][d] row-major, caller-owned,
 * row i = node id i, values in (0, 1).  Input Theta = X / sqrt(d) with X the
 * Philox4x32-10/Box-Muller stream (seed, subsequence 0) of element k = i*d + c
 * (readings A1, A11).  Fully asynchronous on `stream`; workspace is
 * allocated stream-ordered (cudaMallocAsync) and released before return, so the
 * handle is read-only and concurrent embeds on different streams are safe.
 * Errors (host-validated, nothing enqueued): NULL g/d_out, d_out (or opts.d_z0) not 16-byte
 * aligned, or non-finite tau -> IGP_ERR_INPUT; d not a multiple of 16 in [16, 1024] ->
 * IGP_ERR_UNSUPPORTED; steps < 0 -> IGP_ERR_INPUT.  Deterministic: identical arguments give
 * bitwise-identical output.  (There is no separate "stop after layer k" mode: steps = k is
 * that run; DESIGN.md §8(b) deviations.) */
IGP_API igp_status igp_embed(igp_graph_t g, float tau, int32_t d, int32_t steps, uint64_t seed,
                     float* d_out, igp_stream_t stream);

/* As igp_embed with all options (theta, alpha, eps, subsequence, debug modes, timing). */
IGP_API igp_status igp_embed_ex(igp_graph_t g, const igp_embed_opts* opts, float* d_out, igp_stream_t stream);

/* End-to-end convenience on HOST buffers: copies h_edges (int32 [num_edges][2])
 * to the device, builds the graph, embeds, copies Z~ back into h_out (fp32 [N][d])
 * and synchronises `stream` before returning.  Same argument rules as above. */
IGP_API igp_status igp_embed_host(const int32_t* h_edges, int64_t num_edges, int32_t num_nodes,
                          const igp_embed_opts* opts, float* h_out, igp_stream_t stream);

/* Process-wide filter-step timer fed by embeds with IGP_FLAG_TIME_LAYERS (thread safe).
 * reset: forget all recorded intervals.  read: wait for the recorded intervals to
 * complete and return their summed device time (ms) and the number of filter-step
 * launches they bracket.  Recording adds no host synchronisation to an embed. */
IGP_API igp_status igp_layer_timer_reset(void);
IGP_API igp_status igp_layer_timer_read(float* total_ms, int64_t* launches);

/* ---------------------------------------------------------------------------
 * Random input (test / inspection entry points)
 * ------------------------------------------------------------------------- */

/* Raw Philox4x32-10 words r[k], k < count: block b = k/4, counter
 * (lo32 b, hi32 b, lo32 subsequence, hi32 subsequence), key (lo32 seed, hi32 seed),
 * word k%4 (identical to cuRAND curand_init(seed, subsequence, 4b) + curand4).
 * d_out device uint32[count]. */
IGP_API igp_status igp_philox_bits(uint64_t seed, uint64_t subsequence, int64_t count, uint32_t* d_out,
                           igp_stream_t stream);

/* X ~ N(0,1) fp32 (unscaled): Box-Muller on word pairs (r0,r1), (r2,r3):
 * u = (r_even + 1/2) 2^-32, v = (r_odd + 1/2) 2^-32, X_even = sqrt(-2 ln u) sin(2 pi v),
 * X_odd = sqrt(-2 ln u) cos(2 pi v), evaluated in fp64 and rounded.
 * count must be a multiple of 4.  d_out device float[count]. */
IGP_API igp_status igp_philox_normal(uint64_t seed, uint64_t subsequence, int64_t count, float* d_out,
                             igp_stream_t stream);

/* ---------------------------------------------------------------------------
 * BIRCH clustering of the embeddings  (Alg. 1 l.7; streaming Alg. 2
 * l.9-11; BIRCH as the paper invokes it)
 *
 * A CF tree (clustering features n, LS, SS per entry; at most `branching` entries per
 * node; leaf entries of radius <= threshold) built by single-pass insertion of rows in
 * row order; its leaf entries, in leaf-chain order, are the K-agnostic clusters, and a
 * row's label is the index of its nearest leaf centroid.  fp64 on the device, with the
 * exact operation order of oracle/birch_oracle.c (readings B1-B6), so trees,
 * clusters and labels are bitwise reproducible.  A tree is single-writer: calls on the same
 * igp_birch_t must not run concurrently (predict is read-only once fitting stops).
 * ------------------------------------------------------------------------- */
typedef struct igp_birch_s* igp_birch_t;

/* New empty tree on the current device for rows of width d (1 <= d <= 1024), radius
 * threshold T > 0 (finite) and branching factor 2 <= B <= 63 (scikit-learn's defaults,
 * T = 0.5 and B = 50).  Invalid arguments -> IGP_ERR_INPUT. */
IGP_API igp_status igp_birch_create(int32_t d, double threshold, int32_t branching, igp_birch_t* out);

/* Insert rows d_X (device fp32 [m][d] row-major, e.g. igp_embed's output, widened to
 * fp64 exactly) in row order: fit on a new tree (Alg. 1 l.7), partial fit on an existing
 * one (Alg. 2 l.9).  Synchronous: returns after the tree is updated (the insertion is a
 * sequential process; the device pools grow as needed).  m = 0 is a no-op.  A non-finite
 * value -> IGP_ERR_INPUT (tree unchanged). */
IGP_API igp_status igp_birch_partial_fit(igp_birch_t b, const float* d_X, int64_t m, igp_stream_t stream);

/* Tree statistics: number of clusters K (leaf entries), depth (levels), nodes, points
 * inserted.  Any output may be NULL.  Synchronous. */
IGP_API igp_status igp_birch_info(igp_birch_t b, int64_t* num_clusters, int32_t* depth, int64_t* nodes,
                                  int64_t* points);

/* The K clusters in label order: device fp64 centroids [K][d], |centroid|^2 [K], point
 * counts n [K], linear sums LS [K][d], square sums SS [K] (caller-owned; any may be NULL).
 * Asynchronous on `stream` (after a synchronous count). */
IGP_API igp_status igp_birch_clusters(igp_birch_t b, double* d_centroids, double* d_sqn, double* d_n, double* d_ls,
                                      double* d_ss, igp_stream_t stream);

/* Labels (Alg. 2 l.11): d_labels[i] = argmin_j |c_j|^2 - 2 c_j . x_i over the K clusters
 * (first minimum; |x_i|^2 is common to all j, reading B5; fp64, bit-identical to the oracle),
 * device int32 [m].  Does not modify the tree.  Empty tree -> IGP_ERR_INPUT.  Runs the
 * tensor-core path where d allows (igp_birch_predict_ex, IGP_PREDICT_AUTO), which synchronises
 * `stream` once to size its fp64 pass; the fp64 path is asynchronous on `stream`. */
IGP_API igp_status igp_birch_predict(igp_birch_t b, const float* d_X, int64_t m, int32_t* d_labels,
                                     igp_stream_t stream);

/* igp_birch_predict with a choice of arithmetic (same labels either way):
 *   IGP_PREDICT_FP64   every distance in fp64 on the CUDA cores, in the oracle's order;
 *   IGP_PREDICT_TENSOR the scores c_j . x_i on the tensor cores (tcgen05, 3xTF32 split),
 *                      each row's argmin certified by an error margin; where other clusters
 *                      come within twice the margin of the best (near or exact ties) the
 *                      candidates' distances are evaluated in fp64 as above (all clusters when
 *                      the candidates cannot be isolated).  Needs d a multiple of 8 in [8, 64]
 *                      (else IGP_ERR_INPUT);
 *   IGP_PREDICT_AUTO   TENSOR where eligible, else FP64 (what igp_birch_predict does).
 * ambiguous (host, may be NULL) receives the number of rows whose label was decided by fp64
 * distances: the rows the tensor scores alone did not settle, m on the FP64 path. */
#define IGP_PREDICT_AUTO 0
#define IGP_PREDICT_FP64 1
#define IGP_PREDICT_TENSOR 2
IGP_API igp_status igp_birch_predict_ex(igp_birch_t b, const float* d_X, int64_t m, int32_t* d_labels, int32_t path,
                                        int64_t* ambiguous, igp_stream_t stream);

/* Release the tree (waits for the legacy default stream).  NULL is a no-op. */
IGP_API igp_status igp_birch_destroy(igp_birch_t b);

/* ---------------------------------------------------------------------------
 * Diagnostics
 * ------------------------------------------------------------------------- */
IGP_API const char* igp_status_string(igp_status s);
IGP_API const char* igp_last_error_message(void);
/* Number of kernels this library has launched in this process (all threads). */
IGP_API uint64_t igp_kernel_launch_count(void);
/* Library version string. */
IGP_API const char* igp_version(void);
/* Return the library's cached device memory to the driver.  Every workspace (builds, embeds)
 * comes from a memory pool private to this library (never the device's default pool), which
 * keeps freed blocks for reuse by later calls; this trims it on the current device. */
IGP_API igp_status igp_trim_memory(void);

#ifdef __cplusplus
}
#endif

#endif /* IGP_H_ */
