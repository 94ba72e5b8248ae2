// igp_api.cu — the C ABI declared in include/igp.h: argument validation, handle
// ownership, status codes, stream-ordered workspace, and the host-buffer
// end-to-end entry point.  All compute is in csr_build.cu / philox.cu / embed.cu.
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "igp_internal.cuh"

namespace igp {

std::atomic<uint64_t> g_launches{0};

std::string& error_slot() {
    thread_local std::string msg;
    return msg;
}

void set_error(const std::string& msg) { error_slot() = msg; }

bool device_info(DeviceInfo* out) {
    static std::mutex mu;
    static DeviceInfo cache[64];
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess || dev < 0) {
        set_error(std::string("no usable CUDA device: ") + cudaGetErrorString(e));
        return false;
    }
    std::lock_guard<std::mutex> lock(mu);
    DeviceInfo& di = cache[dev & 63];
    if (di.device != dev) {
        DeviceInfo n;
        n.device = dev;
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
            set_error("cudaDeviceGetAttribute(MultiProcessorCount) failed");
            return false;
        }
        n.num_sms = v;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        n.max_smem_optin = v;
        cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev);
        n.l2_bytes = (size_t)v;
        di = n;
    }
    *out = di;
    return true;
}

// the library's private stream-ordered pool of a device: freed blocks stay cached for the next
// build / embed (release threshold raised on THIS pool only; the device's default pool and other
// allocators in the process are untouched); igp_trim_memory returns them to the driver
static cudaMemPool_t library_pool(int dev) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    cudaMemPool_t& p = pools[dev & 63];
    if (!p) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
            p = nullptr;
            return nullptr;
        }
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    return p;
}

cudaError_t alloc_async(void** p, size_t bytes, cudaStream_t s) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = library_pool(dev);
    if (!pool) return cudaErrorMemoryAllocation;
    return cudaMallocFromPoolAsync(p, bytes > 0 ? bytes : 16, pool, s);
}

// a size class above `bytes` (>= 1 MiB: 2^k x {1, 1.25, 1.5, 1.75}, at most 25% over): workspaces
// whose size creeps up call by call (BIRCH predict as clusters accrue) then reuse the pool's block
// instead of growing the pool on every call
cudaError_t alloc_async_class(void** p, size_t bytes, cudaStream_t s) {
    if (bytes >= ((size_t)1 << 20)) {
        size_t k = (size_t)1 << 20;
        while (k * 2 <= bytes) k *= 2;
        const size_t q = k / 4;
        size_t c = k;
        while (c < bytes) c += q;
        bytes = c;
    }
    return alloc_async(p, bytes, s);
}

cudaError_t trim_pool() {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    cudaMemPool_t pool = library_pool(dev);
    if (!pool) return cudaErrorMemoryAllocation;
    e = cudaDeviceSynchronize();
    return e != cudaSuccess ? e : cudaMemPoolTrimTo(pool, 0);
}

void free_async(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

cudaStream_t side_stream(int dev) {
    static std::mutex mu;
    static cudaStream_t st[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    cudaStream_t& x = st[dev & 63];
    if (!x && cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking) != cudaSuccess) x = nullptr;
    return x;
}

// ---------------------------------------------------------------- layer timer
namespace {
struct TimerEntry {
    TimerSlot slot;
    int device = -1;
    int64_t launches = 0;
};
std::mutex g_timer_mu;
std::vector<TimerEntry*> g_timer;  // entries [0, g_timer_used) are recorded intervals
size_t g_timer_used = 0;
}  // namespace

TimerSlot* timer_acquire(int64_t launches) {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(g_timer_mu);
    // reuse a free entry of this device, else create one
    for (size_t k = g_timer_used; k < g_timer.size(); ++k) {
        if (g_timer[k]->device == dev) {
            std::swap(g_timer[k], g_timer[g_timer_used]);
            TimerEntry* e = g_timer[g_timer_used++];
            e->launches = launches;
            return &e->slot;
        }
    }
    TimerEntry* e = new (std::nothrow) TimerEntry();
    if (!e) return nullptr;
    if (cudaEventCreate(&e->slot.ev0) != cudaSuccess || cudaEventCreate(&e->slot.ev1) != cudaSuccess) {
        if (e->slot.ev0) cudaEventDestroy(e->slot.ev0);
        delete e;
        return nullptr;
    }
    e->device = dev;
    e->launches = launches;
    g_timer.push_back(e);
    std::swap(g_timer.back(), g_timer[g_timer_used]);
    return &g_timer[g_timer_used++]->slot;
}

// ---------------------------------------------------------------- lazy graph status
// a private non-blocking stream per device for the few-byte status reads (so a query does not
// serialise behind unrelated work on the legacy default stream)
static cudaStream_t status_stream(int dev) {
    static std::mutex mu;
    static cudaStream_t st[64] = {};
    std::lock_guard<std::mutex> lock(mu);
    cudaStream_t& x = st[dev & 63];
    if (!x) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    return x;
}

// wait for g's last build / merge and read nnz = row_ptr[N] and the range-error flag
igp_status resolve_graph(igp_graph_s* g) {
    std::lock_guard<std::mutex> lock(g->mu);
    if (g->resolved) return IGP_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != g->device) cudaSetDevice(g->device);
    igp_status st = cuda_status(cudaEventSynchronize(g->ready), "graph build");
    int32_t vals[2] = {0, 0};
    if (st == IGP_OK) {
        cudaStream_t ps = status_stream(g->device);
        st = cuda_status(cudaMemcpyAsync(&vals[0], g->csr.row_ptr + g->csr.n, sizeof(int32_t), cudaMemcpyDeviceToHost, ps),
                         "nnz readback");
        if (st == IGP_OK)
            st = cuda_status(cudaMemcpyAsync(&vals[1], g->csr.meta, sizeof(int32_t), cudaMemcpyDeviceToHost, ps),
                             "flag readback");
        if (st == IGP_OK) st = cuda_status(cudaStreamSynchronize(ps), "status sync");
    }
    if (prev != g->device && prev >= 0) cudaSetDevice(prev);
    if (st != IGP_OK) return st;
    g->nnz = vals[0];
    g->err = vals[1];
    g->resolved = true;
    return IGP_OK;
}

igp_status graph_error(const igp_graph_s* g) {
    if (g->err) {
        set_error("edge index outside [0, num_nodes) (the offending edges were skipped)");
        return IGP_ERR_INPUT;
    }
    return IGP_OK;
}

}  // namespace igp

using namespace igp;

static igp_status check_opts(const igp_embed_opts* o) {
    if (!o) {
        set_error("opts is NULL");
        return IGP_ERR_INPUT;
    }
    if (!std::isfinite(o->tau) || !std::isfinite(o->theta) || !std::isfinite(o->alpha)) {
        set_error("tau, theta and alpha must be finite");
        return IGP_ERR_INPUT;
    }
    if (!(o->eps > 0.0f) || !std::isfinite(o->eps)) {
        set_error("eps must be positive (Eq. (1))");
        return IGP_ERR_INPUT;
    }
    if (o->steps < 0) {
        set_error("steps must be >= 0");
        return IGP_ERR_INPUT;
    }
    if (o->flags & ~(uint32_t)(IGP_FLAG_TIME_LAYERS | IGP_FLAG_ROW_L2)) {
        set_error("unknown embed flags");
        return IGP_ERR_INPUT;
    }
    if (o->mode != IGP_MODE_FULL && o->mode != IGP_MODE_PRE_SIGMOID && o->mode != IGP_MODE_LINEAR) {
        set_error("unknown mode");
        return IGP_ERR_INPUT;
    }
    if (o->ddof < 0 || o->ddof > 1) {
        set_error("ddof must be 0 (population std) or 1 (sample std)");
        return IGP_ERR_INPUT;
    }
    if ((reinterpret_cast<uintptr_t>(o->d_z0) & 15) != 0) {
        set_error("opts.d_z0 must be 16-byte aligned");
        return IGP_ERR_INPUT;
    }
    if (o->d < 16 || o->d > kMaxD || o->d % 16 != 0) {
        set_error("d must be a multiple of 16 in [16, 1024]");
        return IGP_ERR_UNSUPPORTED;
    }
    return IGP_OK;
}

// remember that `s` uses g (an event recorded behind the work just enqueued on s)
static igp_status note_use(igp_graph_s* g, cudaStream_t s) {
    std::lock_guard<std::mutex> lock(g->use_mu);
    for (auto& u : g->uses)
        if (u.stream == s) return cuda_status(cudaEventRecord(u.ev, s), "event record");
    igp_graph_s::Use u{s, nullptr};
    IGP_CUDA(cudaEventCreateWithFlags(&u.ev, cudaEventDisableTiming), "event");
    igp_status st = cuda_status(cudaEventRecord(u.ev, s), "event record");
    if (st != IGP_OK) {
        cudaEventDestroy(u.ev);
        return st;
    }
    g->uses.push_back(u);
    return IGP_OK;
}

extern "C" {

const char* igp_version(void) { return "igp 0.1 (sm_100a)"; }

const char* igp_status_string(igp_status s) {
    switch (s) {
        case IGP_OK: return "IGP_OK";
        case IGP_ERR_INPUT: return "IGP_ERR_INPUT";
        case IGP_ERR_NUMERICAL: return "IGP_ERR_NUMERICAL";
        case IGP_ERR_CUDA: return "IGP_ERR_CUDA";
        case IGP_ERR_OOM: return "IGP_ERR_OOM";
        case IGP_ERR_UNSUPPORTED: return "IGP_ERR_UNSUPPORTED";
        default: return "IGP_ERR_UNKNOWN";
    }
}

const char* igp_last_error_message(void) { return error_slot().c_str(); }

uint64_t igp_kernel_launch_count(void) { return g_launches.load(); }

igp_status igp_build_graph(const int32_t* d_edges, int64_t num_edges, int32_t num_nodes, igp_stream_t stream,
                           igp_graph_t* out) {
    return igp_build_graph_ex(d_edges, num_edges, num_nodes, IGP_BUILD_DEFAULT, stream, out);
}

igp_status igp_build_graph_ex(const int32_t* d_edges, int64_t num_edges, int32_t num_nodes, uint32_t flags,
                              igp_stream_t stream, igp_graph_t* out) {
    set_error("");
    const uint32_t order_flags = flags & (IGP_BUILD_NO_REORDER | IGP_BUILD_REORDER_DEGREE | IGP_BUILD_REORDER_COMMUNITY);
    if ((flags & ~(uint32_t)(IGP_BUILD_NO_REORDER | IGP_BUILD_ASYNC | IGP_BUILD_REORDER_COMMUNITY |
                             IGP_BUILD_REORDER_DEGREE)) ||
        (order_flags & (order_flags - 1))) {
        if (out) *out = nullptr;
        set_error("unknown or conflicting build flags");
        return IGP_ERR_INPUT;
    }
    if (!out) {
        set_error("out handle pointer is NULL");
        return IGP_ERR_INPUT;
    }
    *out = nullptr;
    if (num_nodes <= 0) {
        set_error("num_nodes must be >= 1");
        return IGP_ERR_INPUT;
    }
    if (num_edges < 0 || (num_edges > 0 && !d_edges)) {
        set_error("num_edges must be >= 0 and d_edges non-NULL when num_edges > 0");
        return IGP_ERR_INPUT;
    }
    if (num_edges > kMaxEntries / 2) {
        set_error("2*num_edges exceeds the int32 CSR index range");
        return IGP_ERR_UNSUPPORTED;
    }
    if (num_nodes > kMaxNodes) {  // the builder's int32 scans / digit histograms cover ~2N entries
        set_error("num_nodes exceeds 2^30 - 4096");
        return IGP_ERR_UNSUPPORTED;
    }
    igp_graph_s* g = new (std::nothrow) igp_graph_s();
    if (!g) return IGP_ERR_OOM;
    cudaStream_t s = (cudaStream_t)stream;
    if (flags & IGP_BUILD_NO_REORDER) {
        g->order = kOrderNone;
    } else if (flags & IGP_BUILD_REORDER_COMMUNITY) {
        g->order = kOrderCommunity;
    } else if (flags & IGP_BUILD_REORDER_DEGREE) {
        g->order = kOrderDegree;
    } else {
        // default: communities once a 32-column slice of the features no longer fits half the L2
        // (measured: headline +2%, Large +20% per step incl. the build)
        DeviceInfo di;
        if (!device_info(&di)) {
            delete g;
            return IGP_ERR_CUDA;
        }
        g->order = (double)num_nodes * 128.0 > 0.5 * (double)di.l2_bytes ? kOrderCommunity : kOrderDegree;
    }
    g->async = (flags & IGP_BUILD_ASYNC) != 0;
    igp_status st = cuda_status(cudaGetDevice(&g->device), "cudaGetDevice");
    if (st == IGP_OK) st = cuda_status(cudaEventCreateWithFlags(&g->ready, cudaEventDisableTiming), "event");
    if (st == IGP_OK) st = build_csr(d_edges, num_edges, num_nodes, g->order, s, &g->csr);
    if (st != IGP_OK) {
        if (g->ready) cudaEventDestroy(g->ready);
        delete g;
        return st;
    }
    st = cuda_status(cudaEventRecord(g->ready, s), "event record");
    if (st == IGP_OK && !g->async) {
        st = resolve_graph(g);
        if (st == IGP_OK) st = graph_error(g);
    }
    if (st != IGP_OK) {
        std::string msg = igp_last_error_message();
        igp_destroy_graph_async(g, stream);
        set_error(msg);
        return st;
    }
    *out = g;
    return IGP_OK;
}

igp_status igp_graph_add_edges(igp_graph_t g, const int32_t* d_edges, int64_t num_edges, igp_stream_t stream) {
    set_error("");
    if (!g) {
        set_error("graph is NULL");
        return IGP_ERR_INPUT;
    }
    if (num_edges < 0 || (num_edges > 0 && !d_edges)) {
        set_error("num_edges must be >= 0 and d_edges non-NULL when num_edges > 0");
        return IGP_ERR_INPUT;
    }
    if (num_edges > (kMaxEntries - g->csr.cap) / 2) {
        set_error("merged edge count exceeds the int32 CSR index range");
        return IGP_ERR_UNSUPPORTED;
    }
    cudaStream_t s = (cudaStream_t)stream;
    // the merge reads the current CSR: order it behind the build / merge that wrote it
    IGP_CUDA(cudaStreamWaitEvent(s, g->ready, 0), "stream wait");
    CsrDevice merged;
    IGP_TRY(build_csr(d_edges, num_edges, g->csr.n, g->order, s, &merged, &g->csr));
    IGP_CUDA(cudaEventRecord(g->ready, s), "event record");
    if (!g->async) {
        // check the merge before replacing the graph: on a range error g stays as it was
        igp_graph_s tmp;
        tmp.csr = merged;
        tmp.device = g->device;
        tmp.ready = g->ready;
        igp_status st = resolve_graph(&tmp);
        if (st == IGP_OK) st = graph_error(&tmp);
        tmp.ready = nullptr;
        if (st != IGP_OK) {
            free_csr(merged, s);
            return st;
        }
        g->nnz = tmp.nnz;
        g->err = 0;
        g->resolved = true;
    } else {
        g->resolved = false;
    }
    // the old CSR is released in stream order behind the merge that read it
    free_csr(g->csr, s);
    g->csr = merged;
    return IGP_OK;
}

igp_status igp_graph_status(igp_graph_t g) {
    if (!g) {
        set_error("graph is NULL");
        return IGP_ERR_INPUT;
    }
    IGP_TRY(resolve_graph(g));
    return graph_error(g);
}

igp_status igp_graph_info(igp_graph_t g, int32_t* num_nodes, int64_t* nnz, int64_t* m) {
    IGP_TRY(igp_graph_status(g));
    if (num_nodes) *num_nodes = g->csr.n;
    if (nnz) *nnz = g->nnz;
    if (m) *m = g->nnz / 2;
    return IGP_OK;
}

igp_status igp_graph_copy_csr(igp_graph_t g, int32_t* d_row_ptr, int32_t* d_col_idx, int32_t* d_deg,
                              igp_stream_t stream) {
    if (!g || !d_row_ptr) {
        set_error("graph or output pointer is NULL");
        return IGP_ERR_INPUT;
    }
    IGP_TRY(igp_graph_status(g));
    if (g->nnz > 0 && !d_col_idx) {
        set_error("d_col_idx is NULL");
        return IGP_ERR_INPUT;
    }
    cudaStream_t s = (cudaStream_t)stream;
    IGP_CUDA(cudaMemcpyAsync(d_row_ptr, g->csr.row_ptr, sizeof(int32_t) * ((size_t)g->csr.n + 1),
                             cudaMemcpyDeviceToDevice, s),
             "copy row_ptr");
    if (g->nnz > 0)
        IGP_CUDA(cudaMemcpyAsync(d_col_idx, g->csr.col_idx, sizeof(int32_t) * (size_t)g->nnz,
                                 cudaMemcpyDeviceToDevice, s),
                 "copy col_idx");
    if (d_deg) IGP_TRY(launch_degrees(g->csr.row_ptr, g->csr.n, d_deg, s));
    return IGP_OK;
}

static void release_graph(igp_graph_t g, cudaStream_t s) {
    free_csr(g->csr, s);
    if (g->ready) cudaEventDestroy(g->ready);  // deferred by the runtime until the event completes
    for (auto& u : g->uses) cudaEventDestroy(u.ev);
    delete g;
}

igp_status igp_destroy_graph(igp_graph_t g) {
    if (!g) return IGP_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != g->device) cudaSetDevice(g->device);
    // wait for the graph's own build / merges and embeds only (not the whole device), then
    // release in stream order on the library's private status stream
    igp_status st = cuda_status(cudaEventSynchronize(g->ready), "graph build");
    {
        std::lock_guard<std::mutex> lock(g->use_mu);
        for (auto& u : g->uses)
            if (st == IGP_OK) st = cuda_status(cudaEventSynchronize(u.ev), "graph use");
    }
    release_graph(g, status_stream(g->device));
    if (prev >= 0 && prev != g->device) cudaSetDevice(prev);
    return st;
}

igp_status igp_destroy_graph_async(igp_graph_t g, igp_stream_t stream) {
    if (!g) return IGP_OK;
    cudaStream_t s = (cudaStream_t)stream;
    cudaStreamWaitEvent(s, g->ready, 0);  // never free under an unfinished build / merge ...
    {
        std::lock_guard<std::mutex> lock(g->use_mu);
        for (auto& u : g->uses) cudaStreamWaitEvent(s, u.ev, 0);  // ... or an embed on another stream
    }
    release_graph(g, s);
    return IGP_OK;
}

igp_status igp_trim_memory(void) { return cuda_status(trim_pool(), "trim memory"); }

void igp_embed_opts_default(igp_embed_opts* o) {
    if (!o) return;
    std::memset(o, 0, sizeof(*o));
    o->theta = 0.1f;
    o->alpha = 1.0f;
    o->eps = 1e-3f;
    o->mode = IGP_MODE_FULL;
    o->ddof = 0;     // population std (reading A2)
}

igp_status igp_embed_ex(igp_graph_t g, const igp_embed_opts* opts, float* d_out, igp_stream_t stream) {
    set_error("");
    if (!g || !d_out) {
        set_error("graph or d_out is NULL");
        return IGP_ERR_INPUT;
    }
    IGP_TRY(check_opts(opts));
    if ((reinterpret_cast<uintptr_t>(d_out) & 15) != 0) {
        set_error("d_out must be 16-byte aligned");
        return IGP_ERR_INPUT;
    }
    cudaStream_t s = (cudaStream_t)stream;
    // order the embed behind the build / merge (a no-op wait when it is on the same stream)
    IGP_CUDA(cudaStreamWaitEvent(s, g->ready, 0), "stream wait");
    igp_status st = run_embed(g->csr, *opts, d_out, s);
    igp_status su = note_use(g, s);  // igp_destroy_graph waits for this embed (even after an error)
    return st != IGP_OK ? st : su;
}

igp_status igp_embed(igp_graph_t g, float tau, int32_t d, int32_t steps, uint64_t seed, float* d_out,
                     igp_stream_t stream) {
    igp_embed_opts o;
    igp_embed_opts_default(&o);
    o.tau = tau;
    o.d = d;
    o.steps = steps;
    o.seed = seed;
    return igp_embed_ex(g, &o, d_out, stream);
}

igp_status igp_layer_timer_reset(void) {
    std::lock_guard<std::mutex> lock(g_timer_mu);
    g_timer_used = 0;
    return IGP_OK;
}

igp_status igp_layer_timer_read(float* total_ms, int64_t* launches) {
    std::lock_guard<std::mutex> lock(g_timer_mu);
    double ms = 0.0;
    int64_t nl = 0;
    int prev = -1;
    cudaGetDevice(&prev);
    igp_status st = IGP_OK;
    for (size_t k = 0; k < g_timer_used && st == IGP_OK; ++k) {
        TimerEntry* e = g_timer[k];
        if (e->device != prev) cudaSetDevice(e->device);
        float t = 0.0f;
        st = cuda_status(cudaEventSynchronize(e->slot.ev1), "cudaEventSynchronize");
        if (st == IGP_OK) st = cuda_status(cudaEventElapsedTime(&t, e->slot.ev0, e->slot.ev1), "cudaEventElapsedTime");
        if (e->device != prev && prev >= 0) cudaSetDevice(prev);
        ms += t;
        nl += e->launches;
    }
    if (st != IGP_OK) return st;
    if (total_ms) *total_ms = (float)ms;
    if (launches) *launches = nl;
    return IGP_OK;
}

igp_status igp_embed_host(const int32_t* h_edges, int64_t num_edges, int32_t num_nodes, const igp_embed_opts* opts,
                          float* h_out, igp_stream_t stream) {
    set_error("");
    if (!h_out || (num_edges > 0 && !h_edges) || num_edges < 0 || num_nodes <= 0) {
        set_error("invalid host buffers or sizes");
        return IGP_ERR_INPUT;
    }
    IGP_TRY(check_opts(opts));
    cudaStream_t s = (cudaStream_t)stream;
    int32_t* d_edges = nullptr;
    float* d_out = nullptr;
    const size_t eb = sizeof(int32_t) * 2 * (size_t)num_edges;
    const size_t ob = sizeof(float) * (size_t)num_nodes * (size_t)opts->d;
    IGP_CUDA(alloc_async((void**)&d_edges, eb, s), "edges alloc");
    igp_status st = eb ? cuda_status(cudaMemcpyAsync(d_edges, h_edges, eb, cudaMemcpyHostToDevice, s), "edges H2D")
                       : IGP_OK;
    // everything is enqueued before the single wait at the end
    igp_graph_t g = nullptr;
    if (st == IGP_OK) st = igp_build_graph_ex(d_edges, num_edges, num_nodes, IGP_BUILD_ASYNC, stream, &g);
    free_async(d_edges, s);  // stream-ordered: after the build that reads it (or the failed copy)
    if (st != IGP_OK) {
        cudaStreamSynchronize(s);
        return st;
    }
    // each column slice is copied to h_out on a second stream as soon as it is final, so all
    // but the last slice's device->host transfer overlaps the remaining filter steps
    HostCopy hc;
    hc.h_out = h_out;
    st = cuda_status(cudaStreamCreateWithFlags(&hc.cs, cudaStreamNonBlocking), "copy stream");
    for (int k = 0; k < opts->d / 16 && st == IGP_OK; ++k)  // at most d/16 column slices
        st = cuda_status(cudaEventCreateWithFlags(&hc.ev[k], cudaEventDisableTiming), "event");
    if (st == IGP_OK) st = cuda_status(alloc_async((void**)&d_out, ob, s), "out alloc");
    if (st == IGP_OK) st = cuda_status(cudaStreamWaitEvent(s, g->ready, 0), "stream wait");
    if (st == IGP_OK) st = run_embed(g->csr, *opts, d_out, s, &hc);
    // d_out is released only after every slice copy queued on hc.cs has read it -- also when
    // the embed failed after queuing some of them (then the copy stream is simply drained)
    if (d_out) {
        cudaEvent_t copied = nullptr;
        bool ordered = hc.cs == nullptr;
        if (!ordered && cudaEventCreateWithFlags(&copied, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventRecord(copied, hc.cs) == cudaSuccess && cudaStreamWaitEvent(s, copied, 0) == cudaSuccess)
            ordered = true;
        if (!ordered) cudaStreamSynchronize(hc.cs);
        free_async(d_out, s);
        if (copied) cudaEventDestroy(copied);  // released by the runtime once complete
    }
    // the range check ran with the build (early on `s`); its flag is read after the work is queued
    if (st == IGP_OK) st = igp_graph_status(g);
    std::string msg = igp_last_error_message();
    igp_destroy_graph_async(g, stream);  // its only user is `s`
    igp_status st2 = cuda_status(cudaStreamSynchronize(s), "stream sync");
    if (hc.cs) cudaStreamSynchronize(hc.cs);
    for (int k = 0; k < kMaxSlices; ++k)
        if (hc.ev[k]) cudaEventDestroy(hc.ev[k]);
    if (hc.cs) cudaStreamDestroy(hc.cs);
    if (st != IGP_OK) set_error(msg);
    return st != IGP_OK ? st : st2;
}

igp_status igp_philox_bits(uint64_t seed, uint64_t sub, int64_t count, uint32_t* d_out, igp_stream_t stream) {
    set_error("");
    if (count < 0 || (count > 0 && !d_out)) {
        set_error("invalid count or NULL output");
        return IGP_ERR_INPUT;
    }
    DeviceInfo di;
    if (!device_info(&di)) return IGP_ERR_CUDA;
    return launch_philox_bits(seed, sub, count, d_out, (cudaStream_t)stream);
}

igp_status igp_philox_normal(uint64_t seed, uint64_t sub, int64_t count, float* d_out, igp_stream_t stream) {
    set_error("");
    if (count < 0 || count % 4 != 0 || (count > 0 && !d_out)) {
        set_error("count must be a non-negative multiple of 4 and d_out non-NULL");
        return IGP_ERR_INPUT;
    }
    DeviceInfo di;
    if (!device_info(&di)) return IGP_ERR_CUDA;
    return launch_philox_normal(seed, sub, count, d_out, (cudaStream_t)stream);
}

}  // extern "C"
