// igp_internal.cuh — host-side plumbing shared by the library's translation units.
// (Product code only; shares nothing with oracle/.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/igp.h"

// Debug builds (IGP_DEBUG=1 python paper_2508_19737_b200/_build.py --force) check every index a
// kernel dereferences with device asserts (compute-sanitizer is unavailable on the GPU pool);
// release builds compile the checks away.
#ifdef IGP_DEBUG
#include <cassert>
#define IGP_DASSERT(cond) assert(cond)
#else
#define IGP_DASSERT(cond) ((void)0)
#endif

namespace igp {

// error detail string, thread-local
void set_error(const std::string& msg);
std::string& error_slot();

// kernel launch accounting (igp_kernel_launch_count)
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

struct DeviceInfo {
    int device = -1;
    int num_sms = 0;
    int max_smem_optin = 0;
    size_t l2_bytes = 0;
};
// cached per current device; returns false (and sets the error) if no device
bool device_info(DeviceInfo* out);

// a non-blocking side stream per device (library-internal fork/join of independent work;
// every use joins back to the caller's stream before returning)
cudaStream_t side_stream(int dev);

// stream-ordered allocation helpers: a memory pool private to the library per device (freed
// blocks are kept for reuse; igp_trim_memory releases them), never the device's default pool
cudaError_t alloc_async(void** p, size_t bytes, cudaStream_t s);
cudaError_t alloc_async_class(void** p, size_t bytes, cudaStream_t s);  // rounded up to a size class
void free_async(void* p, cudaStream_t s);
cudaError_t trim_pool();  // synchronises the device, then trims the current device's pool

inline igp_status cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return IGP_OK;
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? IGP_ERR_OOM : IGP_ERR_CUDA;
}

// check the launch that was just enqueued
inline igp_status launch_status(const char* what) {
    count_launch();
    return cuda_status(cudaGetLastError(), what);
}

#define IGP_TRY(expr)                                   \
    do {                                                \
        igp_status _st = (expr);                        \
        if (_st != IGP_OK) return _st;                  \
    } while (0)

#define IGP_CUDA(expr, what) IGP_TRY(::igp::cuda_status((expr), (what)))

// ---------------------------------------------------------------------------
// csr_build.cu
// ---------------------------------------------------------------------------
struct CsrDevice {
    int32_t* row_ptr = nullptr;  // [N+1]
    int32_t* col_idx = nullptr;  // [cap + kColPad] (vector index loads may overrun a row's end)
    int32_t* order = nullptr;    // [N] order[r] = original id of relabelled row r (degree or community order)
    int32_t* rp_perm = nullptr;  // [N+5] CSR of the relabelled graph (row r = node order[r]) ...
    int32_t* col_perm = nullptr; // [cap + kColPad]  ... neighbour ids relabelled, in canonical order
    int32_t* meta = nullptr;     // device [4]: [0] range-error flag (nnz is row_ptr[N])
    int32_t* labels = nullptr;   // [N] label-propagation communities (community order only): the warm
                                 // start of the next streaming merge's propagation
    bool perm_alias = false;     // no relabelling: rp_perm/col_perm alias row_ptr/col_idx, order = identity
    int32_t n = 0;
    int64_t cap = 0;             // allocated column entries (>= nnz; 2E + base entries before dedup)
};
// release every array of c in stream order on s
void free_csr(const CsrDevice& c, cudaStream_t s);
constexpr int kColPad = 16;
// row-pointer arrays carry kRpPad entries past [N]: the filter step's bulk copies of a row-pointer
// slice are rounded up to 16 bytes and may start below / end past the batch's rows
constexpr int kRpPad = 64;
// largest CSR entry count (before dedup): int32 offsets with headroom for the kernels' chunk
// arithmetic (a chunk start + 2 chunks of 16 must not overflow)
constexpr int64_t kMaxEntries = (int64_t)INT32_MAX - 64;
// largest node count: the row-order sorts scan kDigits x ceil(N / kSortTile) ~ 2N int32 histogram
// entries and scan lengths are padded by a 2048-element tile, all inside int32
constexpr int64_t kMaxNodes = ((int64_t)1 << 30) - 4096;
// row order of the relabelled CSR the filter steps traverse
enum RowOrder { kOrderNone = 0, kOrderDegree = 1, kOrderCommunity = 2 };
constexpr int kLabelPropIters = 8;  // label-propagation sweeps of the community order (measured best of
                                    // 4-14 on headline and Large: profiles/r01b/lp_sweep.txt)
constexpr int kLabelPropWarmIters = 2;  // sweeps after a streaming merge, from the previous labels
// canonical CSR of the new edges, merged with `base` (an existing canonical CSR on the same
// node set) when base != nullptr
igp_status build_csr(const int32_t* d_edges, int64_t num_edges, int32_t n, RowOrder order, cudaStream_t s,
                     CsrDevice* out, const CsrDevice* base = nullptr);

// deg[i] = rp[i + 1] - rp[i] (the degree diagonal D) into a caller buffer
igp_status launch_degrees(const int32_t* rp, int32_t n, int32_t* deg, cudaStream_t s);

// exclusive scan of n int32 counts: out[0..n], out[n] = total (int32 range checked by caller)
igp_status scan_exclusive(const int32_t* in, int32_t* out, int32_t n, cudaStream_t s);

// ---------------------------------------------------------------------------
// philox.cu
// ---------------------------------------------------------------------------
igp_status launch_philox_bits(uint64_t seed, uint64_t sub, int64_t count, uint32_t* out, cudaStream_t s);
igp_status launch_philox_normal(uint64_t seed, uint64_t sub, int64_t count, float* out, cudaStream_t s);

// ---------------------------------------------------------------------------
// embed.cu
// ---------------------------------------------------------------------------
constexpr int kMaxD = 1024;                // embedding widths: multiples of 16 up to this
constexpr int kMaxSlices = kMaxD / 16;     // column slices of width W in {16, 32, 64, 128} dividing d
// process-wide filter-step timer (igp_layer_timer_*): a pair of events per timed slice
struct TimerSlot {
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};
// an event pair (created on the current device) for `launches` filter steps; nullptr on failure
TimerSlot* timer_acquire(int64_t launches);
// optional device->host copy of each column slice as soon as it is final (igp_embed_host):
// slice k's columns go to h_out on stream cs while slice k+1 computes
struct HostCopy {
    float* h_out = nullptr;  // host [N][d]
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[kMaxSlices] = {};
};
igp_status run_embed(const CsrDevice& g, const igp_embed_opts& o, float* out, cudaStream_t s,
                     HostCopy* hc = nullptr);

// ---------------------------------------------------------------------------
// birch_tc.cu: BIRCH predict's nearest-centroid search on the tensor cores (3xTF32 tcgen05.mma,
// certified by a margin; near-ties among a few candidates are re-checked in fp64 in the kernel
// (counted in amb_count[1]); rows it cannot settle get label -1 and are listed in amb_rows /
// amb_count[0] for the fp64 kernel in birch.cu)
// ---------------------------------------------------------------------------
constexpr int kBirchTcMaxD = 64;
bool birch_tc_eligible(int d, int64_t K);
igp_status launch_birch_tc(const double* cen, const double* sqn, int64_t K, int d, const float* X, int64_t m,
                           int32_t* labels, int32_t* amb_rows, unsigned long long* amb_count, cudaStream_t s);

}  // namespace igp

struct igp_graph_s {
    igp::CsrDevice csr;
    // embeds that read the graph: one event per stream used (recorded after the embed's work),
    // so igp_destroy_graph waits for exactly the work that uses the graph
    std::mutex use_mu;
    struct Use {
        cudaStream_t stream;
        cudaEvent_t ev;
    };
    std::vector<Use> uses;
    igp::RowOrder order = igp::kOrderDegree;
    bool async = false;        // IGP_BUILD_ASYNC: nnz / range errors resolved lazily
    int device = 0;
    cudaEvent_t ready = nullptr;  // recorded after the last build / merge
    std::mutex mu;             // guards the lazy resolution below (queries may race across threads)
    bool resolved = false;     // nnz / err below are valid
    int64_t nnz = -1;
    int32_t err = 0;
};
