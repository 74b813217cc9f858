// handle.h — the opaque vol_s handle and host helpers shared by vol_api.cu and shard.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdarg.h>

#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX 3: ranges show up in nsys / ncu timelines

#include "../../include/vol.h"
#include "internal.h"

struct ShardRuntime;

// ------------------------------------------------------------------------------ error reporting

vol_status fail(vol_status st, const char *fmt, ...) __attribute__((format(printf, 2, 3)));

#define CK(call)                                                                                    \
    do {                                                                                            \
        cudaError_t e_ = (call);                                                                    \
        if (e_ != cudaSuccess)                                                                      \
            return fail(e_ == cudaErrorMemoryAllocation ? VOL_ENOMEM : VOL_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                         \
    } while (0)

#define CKL(n)                                                                                 \
    do {                                                                                       \
        if ((n) < 0) {                                                                         \
            cudaError_t e_ = cudaGetLastError();                                               \
            return fail(VOL_ECUDA, "kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                   \
        }                                                                                      \
    } while (0)

// NVTX range for the lifetime of a scope (one per ABI call; SURVEY §5 tracing)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

// ------------------------------------------------------------------------------ workspace carving
struct Carve {
    size_t off = 0;
    char *base = nullptr;
    template <class T>
    T *take(size_t count) {
        off = (off + 255) & ~(size_t)255;
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

struct Layout {
    int64_t S, n_global, n_local;
    uint32_t T;
};

// An instantiated CUDA graph of an iteration loop, kept by the volume and reused by later calls with
// the same key (kernel parameters, buffer parity, schedule); destroyed in vol_destroy after the stream is
// idle — destroying an executable graph right after launching it makes the host wait for it.
struct GraphEntry {
    std::string key;
    cudaGraphExec_t exec = nullptr;
    int64_t per = 0;   // kernel launches per replay
};

struct vol_s {
    std::vector<GraphEntry> graphs;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t cap = nullptr;  // private stream used only for graph capture
    bool owns_ws = false;
    void *ws = nullptr;
    size_t ws_bytes = 0;
    Layout L{};
    hvg::Fields F{};
    int cur = 0;
    bool initialised = false;
    int64_t n_omega_local = 0, n_omega_global = 0;
    int32_t *d_xyz = nullptr;          // [n_global][3]
    uint32_t *d_hash = nullptr;        // [n_global]
    uint32_t *d_count = nullptr;       // [T]
    uint32_t *d_start = nullptr;       // [T+1]
    int32_t *d_entry = nullptr;        // [n_global]
    uint32_t *d_scan = nullptr;        // scan scratch
    int32_t *d_nbr = nullptr;          // [S][12] store indices (6 faces + 6 edge neighbours)
    uint32_t *d_frozen = nullptr;      // [n_local][16] frozen-voxel bits of the current call
    const uint32_t *pending_frozen = nullptr;
    uint8_t *d_w8 = nullptr;           // [S][512] exact 8-bit weights (used when F.W8 != null)
    int32_t *d_perm = nullptr;         // [n_local] caller index of store row r
    float *d_tmp = nullptr;            // [n_local][512] scratch for caller-order I/O
    float *d_u2 = nullptr;             // [S][512] second u buffer of the skewed schedule
    unsigned long long *d_misc = nullptr;  // [4]: dup, bad, n_omega, spare
    double *d_part = nullptr;          // [S][5]
    double *d_eout = nullptr;          // [8]
    int64_t last_launches = 0;
    // the state is the warm initial state (u = ū = f in both ū buffers, p = 0, cur = 0) — set by vol_create,
    // cleared by any iteration, a zero initialisation or vol_load_state; a restart with the warm
    // initialisation then has nothing to rewrite
    bool pristine = false;
    // sharded state (world > 1)
    ShardRuntime *shard = nullptr;
    char *extra = nullptr;             // workspace tail for the sharded runtime
    bool shard_nccl() const;
    hvg::IterParams pending{};         // parameters of the current vol_regularise call
    int pending_kernel = 0;
    int pending_exchange = 1;          // opts.exchange of the current call (sharded only)
};

// Validates the parameters, fills v->pending, initialises the state unless opts->resume.
vol_status vol_regularise_prepare(vol_s *v, float lambda, float eps, float tau, float sigma, int32_t iters,
                                  const vol_opts *opts);
// Fills the 8-bit weight copy (or disables it) once all held W, ghosts included, are final.
vol_status finalize_w8(vol_s *v);
// Dual value from the five reduced energy terms (see energy.cu).
double energy_dual_value(const double *o, float eps, int data_term);

bool is_device_ptr(const void *p);

// Key bytes of a graph: any trivially copyable values, appended in order.
struct GraphKey {
    std::string bytes;
    template <class T>
    GraphKey &add(const T &x) {
        bytes.append(reinterpret_cast<const char *>(&x), sizeof x);
        return *this;
    }
};

// The volume's graph for `key`: a cached executable, or `body(cap_stream, per)` captured on the volume's
// private capture stream and instantiated (the kernels it launches during capture are not counted:
// they run at replay, counted by the caller).
template <class Body>
vol_status cached_graph(vol_s *v, const GraphKey &key, Body body, cudaGraphExec_t *exec, int64_t *per) {
    for (const GraphEntry &e : v->graphs)
        if (e.key == key.bytes) {
            *exec = e.exec;
            *per = e.per;
            return VOL_OK;
        }
    if (v->graphs.size() >= 8) {   // bounded: evict the oldest once the stream has drained it
        CK(cudaStreamSynchronize(v->stream));
        cudaGraphExecDestroy(v->graphs.front().exec);
        v->graphs.erase(v->graphs.begin());
    }
    cudaGraph_t g = nullptr;
    const long long before = hvg::g_launches.load();
    int64_t n = 0;
    CK(cudaStreamBeginCapture(v->cap, cudaStreamCaptureModeThreadLocal));
    vol_status st = body(v->cap, n);
    cudaError_t e = cudaStreamEndCapture(v->cap, &g);
    hvg::g_launches.fetch_sub(hvg::g_launches.load() - before);
    if (st != VOL_OK || e != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        if (st != VOL_OK) return st;
        return fail(VOL_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
    }
    cudaGraphExec_t ge = nullptr;
    e = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(VOL_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
    v->graphs.push_back(GraphEntry{key.bytes, ge, n});
    *exec = ge;
    *per = n;
    return VOL_OK;
}
