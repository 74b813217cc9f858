// vol_api.cu — the C ABI of include/vol.h (host runtime: validation, workspace carving, store build
// orchestration, iteration scheduling with CUDA graphs, read-back, energy).  All arithmetic of the
// method runs in the kernels of store.cu / iterate.cu / energy.cu; the host only plans and launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/vol.h"
#include "handle.h"
#include "internal.h"
#include "shard.h"

#include <cstdarg>

using namespace hvg;

std::atomic<long long> hvg::g_launches{0};

extern "C" int64_t vol_total_launches(void) { return (int64_t)g_launches.load(); }

static thread_local std::string g_err;

vol_status fail(vol_status st, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

extern "C" const char *vol_last_error(void) { return g_err.c_str(); }

extern "C" void vol_default_opts(vol_opts *o) {
    if (!o) return;
    o->theta = 1.0f;
    o->data_term = 0;
    o->init = 0;
    o->resume = 0;
    o->kernel = 0;
    o->freeze = 1;
    o->exchange = 1;
}

extern "C" uint32_t vol_block_hash(int32_t x, int32_t y, int32_t z, uint32_t T) { return host_hash(x, y, z, T); }

static uint32_t table_size(int64_t n) {
    uint32_t T = 1;
    while ((int64_t)T < 2 * n) T <<= 1;
    return T;
}

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static void carve_all(Carve &c, vol_s *v, const Layout &L) {
    const int64_t nv = L.S * kBlockVox;
    float *fields[11];
    for (int k = 0; k < 11; k++) fields[k] = c.take<float>(nv);
    if (v) {
        v->F.f = fields[0];
        v->F.W = fields[1];
        v->F.u = fields[2];
        for (int k = 0; k < 2; k++) {
            v->F.ub[k] = fields[3 + k];
            v->F.px[k] = fields[5 + k];
            v->F.py[k] = fields[7 + k];
            v->F.pz[k] = fields[9 + k];
        }
    }
    auto xyz = c.take<int32_t>(3 * (size_t)L.n_global + 3);
    auto hash = c.take<uint32_t>((size_t)L.n_global + 1);
    auto count = c.take<uint32_t>((size_t)L.T + 1);
    auto start = c.take<uint32_t>((size_t)L.T + 1);
    auto entry = c.take<int32_t>((size_t)L.n_global + 1);
    auto scan = c.take<uint32_t>((size_t)L.T / 4096 + 4);
    auto nbr = c.take<int32_t>(kNbr * (size_t)L.S);
    auto w8 = c.take<uint8_t>((size_t)L.S * kBlockVox + 16);
    auto frozen = c.take<uint32_t>((size_t)L.n_local * 16 + 16);
    auto perm = c.take<int32_t>((size_t)L.n_local + 1);
    auto tmp = c.take<float>((size_t)L.n_local * kBlockVox + 4);
    auto u2 = c.take<float>((size_t)L.S * kBlockVox + 4);   // second u buffer of the skewed schedule
    auto misc = c.take<unsigned long long>(6);
    auto part = c.take<double>(5 * (size_t)L.S + 5);
    auto eout = c.take<double>(8);
    if (v) {
        v->d_xyz = xyz;
        v->d_hash = hash;
        v->d_count = count;
        v->d_start = start;
        v->d_entry = entry;
        v->d_scan = scan;
        v->d_nbr = nbr;
        v->d_w8 = w8;
        v->d_frozen = frozen;
        v->d_perm = perm;
        v->d_tmp = tmp;
        v->d_u2 = u2;
        v->d_misc = misc;
        v->d_part = part;
        v->d_eout = eout;
        v->F.u2 = u2;
    }
}

static size_t layout_bytes(const Layout &L) {
    Carve c;
    carve_all(c, nullptr, L);
    return c.off + 512;
}

// The shard plan is needed twice per volume (workspace size, then creation) and, in a loop that creates one
// volume per step, again and again for the same blocks; the last plan is cached per thread, keyed by an
// order-independent digest of the coordinates computed where they live (device coordinates are not copied
// to the host on a hit) and a digest of the owner map.  The store's row maps come with it.
namespace {
struct PlanCache {
    bool valid = false;
    int64_t n = 0;
    int world = 0, rank = 0;
    uint64_t cdig = 0, pdig = 0;
    ShardPlan plan;
};
thread_local PlanCache g_plan_cache;
}  // namespace

static uint64_t part_digest(const int32_t *part, int64_t n) {
    uint64_t h = 1469598103934665603ull;
    for (int64_t i = 0; i < n; i++) h = (h ^ (uint32_t)part[i]) * 1099511628211ull;
    return h;
}

// Device coordinates are read on stream s (vol_create: the caller's stream; vol_workspace_bytes, which has no
// stream: the legacy default stream).
static vol_status get_shard_plan(const int32_t *block_xyz, int64_t n, const vol_dist *d, ShardPlan &out,
                                 cudaStream_t s) {
    const bool dev = is_device_ptr(block_xyz);
    unsigned long long cd = 0;
    if (dev) {
        if (!coord_digest_device(block_xyz, n, &cd, s)) return fail(VOL_ECUDA, "coordinate digest failed");
    } else {
        cd = coord_digest_host(block_xyz, n);
    }
    const uint64_t pd = part_digest(d->part, n);
    PlanCache &c = g_plan_cache;
    if (c.valid && c.n == n && c.world == d->world && c.rank == d->rank && c.cdig == cd && c.pdig == pd) {
        out = c.plan;
        return VOL_OK;
    }
    std::vector<int32_t> h;
    const int32_t *xyz = block_xyz;
    if (dev) {
        h.resize(3 * (size_t)n);
        if (cudaMemcpyAsync(h.data(), block_xyz, h.size() * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return fail(VOL_ECUDA, "copy of block_xyz failed");
        xyz = h.data();
    }
    // block coordinates must leave room for the ±1 neighbour offsets in int32 arithmetic
    for (int64_t k = 0; k < 3 * n; k++)
        if (xyz[k] <= -(1 << 30) || xyz[k] >= (1 << 30))
            return fail(VOL_EDATA, "block %lld: coordinate %d outside (-2^30, 2^30)", (long long)(k / 3), xyz[k]);
    if (!make_shard_plan(xyz, n, d->part, d->world, d->rank, out))
        return fail(VOL_EDATA, "vol_create: shard plan failed: %s", out.error.c_str());
    out.digest = (cd ^ (pd * 0x9E3779B97F4A7C15ull)) | 1ull;
    out.rows = out.local;
    out.rows.insert(out.rows.end(), out.ghost.begin(), out.ghost.end());
    out.store_of_global.assign(n, -1);
    for (size_t r = 0; r < out.rows.size(); r++) out.store_of_global[out.rows[r]] = (int32_t)r;
    c.valid = true;
    c.n = n;
    c.world = d->world;
    c.rank = d->rank;
    c.cdig = cd;
    c.pdig = pd;
    c.plan = out;
    return VOL_OK;
}

extern "C" size_t vol_workspace_bytes(const int32_t *block_xyz, int64_t n_global, const vol_dist *dist) {
    if (n_global < 1) return 0;
    Layout L{};
    L.n_global = n_global;
    L.T = table_size(n_global);
    if (!dist || (dist->world <= 1 && !dist->nccl_id)) {
        L.S = n_global;
        L.n_local = n_global;
        return layout_bytes(L);
    }
    if (!block_xyz || !dist->part) return 0;
    ShardPlan plan;
    if (get_shard_plan(block_xyz, n_global, dist, plan, cudaStreamLegacy) != VOL_OK) return 0;
    L.n_local = plan.n_local();
    L.S = plan.n_local() + plan.n_ghost();
    return layout_bytes(L) + shard_extra_bytes(plan);
}

static vol_status copy_in(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    return VOL_OK;
}

static vol_status create_impl(const int32_t *block_xyz, int64_t n_global, const float *f, const float *W,
                              const uint8_t *W8in, const vol_dist *dist, void *workspace, size_t workspace_bytes,
                              void *stream, vol_t *out);

extern "C" vol_status vol_create(const int32_t *block_xyz, int64_t n_global, const float *f, const float *W,
                                 const vol_dist *dist, void *workspace, size_t workspace_bytes, void *stream,
                                 vol_t *out) {
    NvtxRange nvtx_range_("vol_create");
    return create_impl(block_xyz, n_global, f, W, nullptr, dist, workspace, workspace_bytes, stream, out);
}

extern "C" vol_status vol_create_w8(const int32_t *block_xyz, int64_t n_global, const float *f, const uint8_t *W8,
                                    const vol_dist *dist, void *workspace, size_t workspace_bytes, void *stream,
                                    vol_t *out) {
    NvtxRange nvtx_range_("vol_create_w8");
    if (!W8) return fail(VOL_EINVAL, "vol_create_w8: W8 is NULL");
    return create_impl(block_xyz, n_global, f, nullptr, W8, dist, workspace, workspace_bytes, stream, out);
}

// HVG_TRACE_CREATE=1: host time of each phase of vol_create on stderr (development aid)
namespace {
struct PhaseTrace {
    bool on = std::getenv("HVG_TRACE_CREATE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void operator()(const char *what) {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[create] %-24s %8.1f us\n", what, std::chrono::duration<double, std::micro>(n - t).count());
        t = n;
    }
};
}  // namespace

static vol_status create_impl(const int32_t *block_xyz, int64_t n_global, const float *f, const float *W,
                              const uint8_t *W8in, const vol_dist *dist, void *workspace, size_t workspace_bytes,
                              void *stream, vol_t *out) {
    PhaseTrace trace;
    if (!out) return fail(VOL_EINVAL, "vol_create: out is NULL");
    *out = nullptr;
    if (n_global < 1) return fail(VOL_EINVAL, "vol_create: n_global must be >= 1 (got %lld)", (long long)n_global);
    if (n_global > (int64_t)1 << 30) return fail(VOL_EINVAL, "vol_create: n_global too large");
    if (!block_xyz || !f || !(W || W8in)) return fail(VOL_EINVAL, "vol_create: NULL input pointer");
    // a dist with world > 1, or any dist carrying an NCCL id (world 1 runs the sharded runtime with no
    // peers, which exercises the NCCL set-up and the two-launch schedule on a single GPU)
    const bool sharded = dist && (dist->world > 1 || dist->nccl_id != nullptr);
    if (dist && (dist->world < 1 || dist->rank < 0 || dist->rank >= dist->world))
        return fail(VOL_EINVAL, "vol_create: bad rank/world");
    if (sharded && !dist->part) return fail(VOL_EINVAL, "vol_create: dist->part is NULL");

    vol_s *v = new vol_s();
    auto bail = [&](vol_status st) {
        vol_destroy(v);
        return st;
    };
    CK(cudaGetDevice(&v->device));
    v->stream = (cudaStream_t)stream;
    if (cudaStreamCreateWithFlags(&v->cap, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(VOL_ECUDA, "cudaStreamCreate failed"));

    // the shard plan is a host-side schedule (sharded volumes; cached across volumes of the same blocks — the
    // coordinates are copied to the host only to build it); one GPU orders and checks the blocks on the
    // device (order.cu)
    ShardPlan plan;
    if (sharded) {
        vol_status pst = get_shard_plan(block_xyz, n_global, dist, plan, v->stream);
        if (pst != VOL_OK) return bail(pst);
    }
    trace("stream (+ coords D2H)");

    Layout L{};
    L.n_global = n_global;
    L.T = table_size(n_global);
    if (sharded) {
        L.n_local = plan.n_local();
        L.S = plan.n_local() + plan.n_ghost();
    } else {
        L.n_local = n_global;
        L.S = n_global;
    }
    // the iteration kernels index voxels with 32 bits (one GPU holds < 2^32 voxels: 2^23 blocks of
    // 41 B per voxel are already 176 GB)
    if (L.S >= ((int64_t)1 << 23))
        return bail(fail(VOL_EINVAL, "vol_create: %lld store rows (local + ghost) on one GPU; at most 2^23 - 1 "
                                     "(32-bit voxel indexing) — shard the volume over more GPUs",
                         (long long)L.S));
    v->L = L;
    size_t need = layout_bytes(L) + (sharded ? shard_extra_bytes(plan) : 0);
    if (workspace) {
        if (workspace_bytes < need)
            return bail(fail(VOL_ENOMEM, "vol_create: workspace %zu bytes < %zu needed", workspace_bytes, need));
        v->ws = workspace;
        v->ws_bytes = workspace_bytes;
    } else {
        cudaError_t e = cudaMalloc(&v->ws, need);
        if (e != cudaSuccess) return bail(fail(VOL_ENOMEM, "cudaMalloc(%zu) failed: %s", need, cudaGetErrorString(e)));
        v->owns_ws = true;
        v->ws_bytes = need;
    }
    Carve c;
    c.base = (char *)(((uintptr_t)v->ws + 255) & ~(uintptr_t)255);
    carve_all(c, v, L);
    v->extra = c.base + ((c.off + 255) & ~(size_t)255);
    cudaStream_t s = v->stream;
    // status words: [0] duplicate pair, [1] first invalid voxel, [2] |Ω|, [3] W8 unusable, [4] first block
    // with an out-of-range coordinate
    if (cudaMemsetAsync(v->d_misc, 0, 6 * 8, s) != cudaSuccess || cudaMemsetAsync(v->d_misc, 0xFF, 2 * 8, s) != cudaSuccess ||
        cudaMemsetAsync(&v->d_misc[4], 0xFF, 8, s) != cudaSuccess)
        return bail(fail(VOL_ECUDA, "memset failed"));

    // store order: Morton order of the blocks (single GPU, on the device) or the shard plan's
    // [launch A | launch B] rows + ghosts; d_perm[r] is the block's index in the caller's f / W / u arrays
    vol_status st;
    if ((st = copy_in(v->d_xyz, block_xyz, 3 * (size_t)n_global * 4, s)) != VOL_OK) return bail(st);
    if (!sharded) {
        const size_t ms = morton_order_scratch_bytes(n_global);
        void *scr = v->d_tmp;
        const bool own = ms > (size_t)L.n_local * kBlockVox * 4;
        if (own && cudaMallocAsync(&scr, ms, s) != cudaSuccess) return bail(fail(VOL_ENOMEM, "order scratch"));
        const int r = launch_morton_order(v->d_xyz, n_global, scr, v->d_perm, &v->d_misc[4], s);
        if (own) cudaFreeAsync(scr, s);
        if (r < 0) return bail(fail(VOL_ECUDA, "store order launch failed: %s", cudaGetErrorString(cudaGetLastError())));
    } else {
        if (cudaMemcpyAsync(v->d_perm, plan.local_caller.data(), (size_t)L.n_local * 4, cudaMemcpyHostToDevice, s) !=
            cudaSuccess)
            return bail(fail(VOL_ECUDA, "permutation upload failed"));
    }
    trace("store order queued");

    // inputs: f and W through a staging copy, then permuted into store order
    const size_t fbytes = (size_t)L.n_local * kBlockVox * 4;
    if ((st = copy_in(v->d_tmp, f, fbytes, s)) != VOL_OK) return bail(st);
    if (W8in) {   // 8-bit counts: a quarter of the bytes to copy, widened on the device (exact)
        if ((st = copy_in(v->F.u, W8in, (size_t)L.n_local * kBlockVox, s)) != VOL_OK) return bail(st);
        if (launch_permute_blocks(v->d_tmp, const_cast<float *>(v->F.f), v->d_perm, L.n_local, true, s) < 0 ||
            launch_permute_w8_to_f32(reinterpret_cast<const uint8_t *>(v->F.u), const_cast<float *>(v->F.W),
                                     v->d_perm, L.n_local, s) < 0)
            return bail(fail(VOL_ECUDA, "input permutation failed"));
    } else {
        if ((st = copy_in(v->F.u, W, fbytes, s)) != VOL_OK) return bail(st);
        if (launch_permute_blocks(v->d_tmp, const_cast<float *>(v->F.f), v->d_perm, L.n_local, true, s) < 0 ||
            launch_permute_blocks(v->F.u, const_cast<float *>(v->F.W), v->d_perm, L.n_local, true, s) < 0)
            return bail(fail(VOL_ECUDA, "input permutation failed"));
    }

    // K1: hash + CSR bucket table over all n_global blocks
    if (cudaMemsetAsync(v->d_count, 0, ((size_t)L.T + 1) * 4, s) != cudaSuccess)
        return bail(fail(VOL_ECUDA, "memset failed"));
    if (launch_hash_count(v->d_xyz, n_global, L.T, v->d_hash, v->d_count, s) < 0 ||
        launch_exclusive_scan_u32(v->d_count, v->d_start, L.T, v->d_scan, s) < 0)
        return bail(fail(VOL_ECUDA, "store build launch failed: %s", cudaGetErrorString(cudaGetLastError())));
    if (cudaMemcpyAsync(v->d_count, v->d_start, (size_t)L.T * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return bail(fail(VOL_ECUDA, "cursor copy failed"));
    if (launch_bucket_fill(v->d_hash, n_global, v->d_count, v->d_entry, s) < 0 ||
        launch_bucket_sort_and_dups(v->d_xyz, v->d_start, v->d_entry, L.T, n_global, &v->d_misc[0], s) < 0 ||
        launch_validate(v->F.f, v->F.W, (int64_t)L.n_local * kBlockVox, &v->d_misc[1], &v->d_misc[2], s) < 0)
        return bail(fail(VOL_ECUDA, "store build launch failed: %s", cudaGetErrorString(cudaGetLastError())));
    // the row maps reuse build scratch (d_hash is free once the buckets are filled)
    int32_t *d_sog = reinterpret_cast<int32_t *>(v->d_hash);
    int64_t *d_rows = reinterpret_cast<int64_t *>(v->d_part);

    // reports the first input error the status words hold (caller block indices and coordinates fetched on
    // demand), else records |Ω|
    auto check_inputs = [&](const unsigned long long *misc) -> vol_status {
        auto coord = [&](long long i, int32_t *xyz3) {   // fetched from the device copy, on error only
            if (cudaMemcpy(xyz3, v->d_xyz + 3 * i, 12, cudaMemcpyDeviceToHost) != cudaSuccess)
                xyz3[0] = xyz3[1] = xyz3[2] = 0;
        };
        int32_t q[3];
        if (misc[4] != ~0ULL) {
            coord((long long)misc[4], q);
            return fail(VOL_EDATA, "block %lld: coordinate (%d, %d, %d) outside (-2^30, 2^30)", (long long)misc[4],
                        q[0], q[1], q[2]);
        }
        if (misc[0] != ~0ULL) {
            long long i = (long long)(misc[0] >> 32), j = (long long)(misc[0] & 0xFFFFFFFFu);
            coord(i, q);
            return fail(VOL_EDATA, "duplicate block coordinates: blocks %lld and %lld are both (%d, %d, %d)", j, i,
                        q[0], q[1], q[2]);
        }
        if (misc[1] != ~0ULL) {
            long long i = (long long)misc[1];
            int32_t blk = 0;
            if (cudaMemcpy(&blk, v->d_perm + i / kBlockVox, 4, cudaMemcpyDeviceToHost) != cudaSuccess) blk = -1;
            return fail(VOL_EDATA, "invalid input in block %lld, voxel %lld: f must be finite, W finite and >= 0",
                        (long long)blk, i % kBlockVox);
        }
        v->n_omega_local = (int64_t)misc[2];
        v->n_omega_global = v->n_omega_local;
        return VOL_OK;
    };

    if (!sharded) {
        // K2: neighbour table; K3: initial state (warm start) so read_u / energy are defined before the first
        // iteration; 8-bit weights — all queued, then one synchronisation reads every status word
        if (launch_row_maps(v->d_perm, n_global, d_sog, d_rows, s) < 0 ||
            launch_neighbours(v->d_xyz, n_global, v->d_start, v->d_entry, L.T, d_sog, d_rows, L.S, v->d_nbr, s) < 0 ||
            launch_init_state(v->F, L.S * kBlockVox, 0, s) < 0 ||
            launch_pack_w8(v->F.W, v->d_w8, L.S * kBlockVox, reinterpret_cast<unsigned *>(&v->d_misc[3]), s) < 0)
            return bail(fail(VOL_ECUDA, "store build launch failed: %s", cudaGetErrorString(cudaGetLastError())));
        unsigned long long misc[5];
        if (cudaMemcpyAsync(misc, v->d_misc, 5 * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return bail(fail(VOL_ECUDA, "store build failed: %s", cudaGetErrorString(cudaGetLastError())));
        trace("build + init + sync");
        if ((st = check_inputs(misc)) != VOL_OK) return bail(st);
        v->F.W8 = (misc[3] & 0xFFFFFFFFull) ? nullptr : v->d_w8;
    } else {
        unsigned long long misc[5];
        if (cudaMemcpyAsync(misc, v->d_misc, 5 * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            return bail(fail(VOL_ECUDA, "store build failed: %s", cudaGetErrorString(cudaGetLastError())));
        trace("store build + sync");
        if ((st = check_inputs(misc)) != VOL_OK) return bail(st);
        // K2: neighbour table in store rows (faces + edges)
        if (cudaMemcpyAsync(d_sog, plan.store_of_global.data(), (size_t)n_global * 4, cudaMemcpyHostToDevice, s) !=
                cudaSuccess ||
            cudaMemcpyAsync(d_rows, plan.rows.data(), (size_t)L.S * 8, cudaMemcpyHostToDevice, s) != cudaSuccess)
            return bail(fail(VOL_ECUDA, "row map upload failed"));
        // (copies from pageable host memory return once the data is staged: the host row maps may go)
        if (launch_neighbours(v->d_xyz, n_global, v->d_start, v->d_entry, L.T, d_sog, d_rows, L.S, v->d_nbr, s) < 0)
            return bail(fail(VOL_ECUDA, "neighbour launch failed"));
        trace("neighbours");
        st = shard_setup(v, plan, dist);
        if (st != VOL_OK) return bail(st);
        // K3: initial state (warm start) so read_u / energy are defined before the first iteration (NCCL
        // shards initialise in shard_after_create, once the ghosts' f and W have arrived)
        if (!v->shard_nccl() && launch_init_state(v->F, L.S * kBlockVox, 0, s) < 0)
            return bail(fail(VOL_ECUDA, "init launch failed"));
        st = shard_after_create(v);
        if (st != VOL_OK) return bail(st);
        trace("shard setup + init");
        // (NCCL shards set up their 8-bit weights in shard_after_create; loopback shards in vol_group_connect)
    }
    v->cur = 0;
    v->initialised = true;
    v->pristine = true;
    *out = v;
    return VOL_OK;
}

// Store W additionally as exact 8-bit counts when every held W (ghosts included) is an integer in
// [0, 255]; the fused kernel then reads 1 B instead of 4 B per voxel for W.
vol_status finalize_w8(vol_s *v) {
    unsigned *d_bad = reinterpret_cast<unsigned *>(&v->d_misc[3]);
    unsigned bad = 0;
    CK(cudaMemsetAsync(d_bad, 0, sizeof(unsigned), v->stream));
    CKL(launch_pack_w8(v->F.W, v->d_w8, v->L.S * kBlockVox, d_bad, v->stream));
    CK(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    v->F.W8 = bad ? nullptr : v->d_w8;
    return VOL_OK;
}

extern "C" void vol_destroy(vol_t v) {
    if (!v) return;
    PhaseTrace trace;
    if (v->shard) shard_destroy(v);
    trace("destroy: shard");
    if (v->stream) cudaStreamSynchronize(v->stream);
    trace("destroy: sync");
    for (GraphEntry &e : v->graphs) cudaGraphExecDestroy(e.exec);
    v->graphs.clear();
    trace("destroy: graphs");
    if (v->cap) cudaStreamDestroy(v->cap);
    trace("destroy: stream");
    if (v->owns_ws && v->ws) cudaFree(v->ws);
    delete v;
}

// ------------------------------------------------------------------------------- iterations

// Skewed schedule (opts.kernel = 0/2, single GPU): k_dual (p^1 from ū^0), iters − 1 launches of k_skew
// (primal k + dual k+1), k_primal (u^iters, ū^iters).  u is double-buffered with d_u2; both buffers start equal to u^0 so voxels that are never
// written (Ω̄, frozen) hold the same value in both, and the buffer order is chosen so that the epilogue
// updates F.u in place.
static vol_status run_iterations_skew(vol_s *v, const IterParams &P, int32_t iters) {
    cudaStream_t s = v->stream;
    const int cur = v->cur;
    const int64_t n = v->L.n_local;
    const size_t ubytes = (size_t)n * kBlockVox * 4;
    int64_t launches = 0;
    CK(cudaMemcpyAsync(v->d_u2, v->F.u, ubytes, cudaMemcpyDeviceToDevice, s));
    float *B[2];
    B[(iters - 1) & 1] = v->F.u;
    B[iters & 1] = v->d_u2;
    {
        View V = view_of(v->F, cur);   // ū^0 = ub[cur], p^0 = p[cur] → p^1 = p[cur ^ 1]
        int r = launch_dual_only(V, v->d_nbr, n, P, s);
        CKL(r);
        launches += r;
    }
    auto skew = [&](cudaStream_t st, int j) -> int {
        return launch_skew_loop(v->F, B[j & 1], B[(j + 1) & 1], cur ^ ((j + 1) & 1), v->pending_frozen, v->d_nbr, n,
                                P, st);
    };
    int j = 0;
    const int total = iters - 1;
    const int m = std::min<int>(16, total / 2);
    if (m >= 1) {   // a graph of 2m launches (buffer parities repeat every 2), replayed
        GraphKey key;
        key.add('S').add(cur).add(m).add(iters & 1).add(v->pending_frozen).add(P);
        cudaGraphExec_t ge = nullptr;
        int64_t per = 0;
        vol_status st = cached_graph(
            v, key,
            [&](cudaStream_t cs, int64_t &n) -> vol_status {
                for (int k = 0; k < 2 * m; k++) {
                    int r = skew(cs, k);
                    if (r < 0) return fail(VOL_ECUDA, "skew launch failed during capture");
                    n += r;
                }
                return VOL_OK;
            },
            &ge, &per);
        if (st != VOL_OK) return st;
        const int reps = total / (2 * m);
        for (int r = 0; r < reps; r++) {
            CK(cudaGraphLaunch(ge, s));
            launches += per;
            g_launches.fetch_add(per);
        }
        j = reps * 2 * m;
    }
    for (; j < total; j++) {
        int r = skew(s, j);
        CKL(r);
        launches += r;
    }
    {
        const int c2 = cur ^ (iters & 1);   // p^iters and the final ū live at index c2
        View V = view_of(v->F, c2 ^ 1);     // px_out = p[c2], ub_out = ub[c2]
        V.u = B[(iters - 1) & 1];           // == F.u
        int r = launch_primal_only(V, v->d_nbr, n, P, s);
        CKL(r);
        launches += r;
        v->cur = c2;
    }
    v->last_launches += launches;
    return VOL_OK;
}

static vol_status run_iterations_single(vol_s *v, const IterParams &P, int32_t iters, int kernel) {
    // kernel 0 (product): the skewed schedule on one GPU; 3: the one-pass fused kernel
    if (kernel == 0 || kernel == 2) return run_iterations_skew(v, P, iters);
    cudaStream_t s = v->stream;
    int64_t launches = 0;
    auto one = [&](cudaStream_t st, int cur) -> int {
        View V = view_of(v->F, cur);
        V.frozen = v->pending_frozen;
        if (kernel == 1) return launch_two_kernel(V, v->d_nbr, nullptr, v->L.n_local, P, st);
        return launch_fused(V, v->d_nbr, nullptr, 0, v->L.n_local, P, st);
    };
    // CUDA graph of 2·m iterations (ū parity returns to the start), replayed; remainder launched directly.
    const int m = std::min<int>(16, iters / 2);
    if (m >= 1) {
        GraphKey key;
        key.add('F').add(kernel).add(v->cur).add(m).add(v->pending_frozen).add(P);
        cudaGraphExec_t ge = nullptr;
        int64_t per = 0;
        const int cur0 = v->cur;
        vol_status st = cached_graph(
            v, key,
            [&](cudaStream_t cs, int64_t &n) -> vol_status {
                int cur = cur0;
                for (int k = 0; k < 2 * m; k++) {
                    int r = one(cs, cur);
                    if (r < 0) return fail(VOL_ECUDA, "launch failed during capture");
                    n += r;
                    cur ^= 1;
                }
                return VOL_OK;
            },
            &ge, &per);
        if (st != VOL_OK) return st;
        const int reps = iters / (2 * m);
        for (int r = 0; r < reps; r++) {
            CK(cudaGraphLaunch(ge, s));
            launches += per;
            g_launches.fetch_add(per);
        }
        iters -= reps * 2 * m;
    }
    for (int k = 0; k < iters; k++) {
        int r = one(s, v->cur);
        CKL(r);
        launches += r;
        v->cur ^= 1;
    }
    v->last_launches += launches;
    return VOL_OK;
}

vol_status vol_regularise_prepare(vol_s *v, float lambda, float eps, float tau, float sigma, int32_t iters,
                                  const vol_opts *opts) {
    if (!v) return fail(VOL_EINVAL, "vol_regularise: NULL handle");
    vol_opts o;
    vol_default_opts(&o);
    if (opts) o = *opts;
    if (!(lambda > 0.0f) || !std::isfinite(lambda)) return fail(VOL_EINVAL, "lambda must be > 0 (got %g)", lambda);
    if (!(eps >= 0.0f) || !std::isfinite(eps)) return fail(VOL_EINVAL, "eps must be >= 0 (got %g)", eps);
    if (!(tau > 0.0f) || !(sigma > 0.0f) || !std::isfinite(tau) || !std::isfinite(sigma))
        return fail(VOL_EINVAL, "tau and sigma must be > 0");
    if ((double)tau * (double)sigma * 12.0 > 1.0 + 1e-6)
        return fail(VOL_EINVAL, "step sizes violate 12*tau*sigma <= 1 (||grad||^2 <= 12): %g", (double)tau * sigma * 12.0);
    if (iters < 0) return fail(VOL_EINVAL, "iters must be >= 0");
    if (!(o.theta >= 0.0f) || !std::isfinite(o.theta)) return fail(VOL_EINVAL, "theta must be >= 0");
    if (o.data_term != 0 && o.data_term != 1) return fail(VOL_EINVAL, "data_term must be 0 (L1) or 1 (L2)");
    if (o.init != 0 && o.init != 1) return fail(VOL_EINVAL, "init must be 0 (warm) or 1 (zero)");
    if (o.kernel < 0 || o.kernel > 3)
        return fail(VOL_EINVAL, "kernel must be 0 (product), 1 (two-kernel), 2 (skewed) or 3 (one-pass fused)");
    if (v->shard && o.kernel == 1) return fail(VOL_ENOTSUP, "the two-kernel baseline is single-GPU only");
    if (o.exchange != 0 && o.exchange != 1) return fail(VOL_EINVAL, "exchange must be 0 (no-op, timing only) or 1");
    if (v->shard) {
        vol_status st = shard_reset(v);
        if (st != VOL_OK) return st;
    }
    if (v->n_omega_global == 0) return fail(VOL_EDATA, "empty Omega: no voxel with W > 0 (S:261)");

    IterParams &P = v->pending;
    P.sigma = sigma;
    P.tau = tau;
    volatile float tl = tau * lambda;  // fl(τ·λ)
    volatile float se = sigma * eps;   // fl(σ·ε)
    volatile float dn = 1.0f + se;     // fl(1 + σε)
    volatile float kp = 1.0f / dn;     // κ = fl(1 / fl(1 + σε))
    P.tl = tl;
    P.kappa = kp;
    P.theta = o.theta;
    P.data_term = o.data_term;
    P.one = 1.0f;
    v->pending_kernel = o.kernel;
    v->pending_exchange = o.exchange;
    v->last_launches = 0;
    if (!o.resume) {
        if (!(v->pristine && o.init == 0)) {   // (the warm initial state needs no rewrite)
            CKL(launch_init_state(v->F, v->L.S * kBlockVox, o.init, v->stream));
            v->last_launches = 1;
        }
        v->cur = 0;
        v->pristine = o.init == 0;
    }
    if (iters > 0) v->pristine = false;
    v->pending_frozen = nullptr;
    if (o.freeze && o.data_term == 0 && o.kernel != 1 && iters > 0) {
        CKL(launch_freeze_mask(v->F, v->cur, P, v->L.n_local, v->d_frozen, v->stream));
        v->pending_frozen = v->d_frozen;
        v->last_launches += 1;
    }
    return VOL_OK;
}

extern "C" vol_status vol_regularise(vol_t v, float lambda, float eps, float tau, float sigma, int32_t iters,
                                     const vol_opts *opts) {
    NvtxRange nvtx_range_("vol_regularise");
    vol_status st = vol_regularise_prepare(v, lambda, eps, tau, sigma, iters, opts);
    if (st != VOL_OK) return st;
    if (iters == 0) return VOL_OK;
    if (v->shard) return shard_iterate(v, v->pending, iters);
    return run_iterations_single(v, v->pending, iters, v->pending_kernel);
}

extern "C" int64_t vol_last_launches(vol_t v) { return v ? v->last_launches : -1; }

extern "C" vol_status vol_sync(vol_t v) {
    if (!v) return fail(VOL_EINVAL, "NULL handle");
    CK(cudaStreamSynchronize(v->stream));
    return VOL_OK;
}

static vol_status copy_out(void *dst, const void *src, size_t bytes, cudaStream_t s) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s));
    if (!is_device_ptr(dst)) CK(cudaStreamSynchronize(s));
    return VOL_OK;
}

// store order → caller order: scatter straight into a device destination, or through the scratch
// buffer for a host destination
static vol_status read_field(vol_s *v, float *dst, const float *src) {
    cudaStream_t s = v->stream;
    const int64_t n = v->L.n_local;
    if (is_device_ptr(dst)) {
        CKL(launch_permute_blocks(src, dst, v->d_perm, n, false, s));
        return VOL_OK;
    }
    CKL(launch_permute_blocks(src, v->d_tmp, v->d_perm, n, false, s));
    return copy_out(dst, v->d_tmp, (size_t)n * kBlockVox * 4, s);
}

// caller order → store order, through the scratch buffer
static vol_status write_field(vol_s *v, float *dst, const float *src) {
    cudaStream_t s = v->stream;
    const int64_t n = v->L.n_local;
    vol_status st = copy_in(v->d_tmp, src, (size_t)n * kBlockVox * 4, s);
    if (st != VOL_OK) return st;
    CKL(launch_permute_blocks(v->d_tmp, dst, v->d_perm, n, true, s));
    return VOL_OK;
}

extern "C" vol_status vol_read_u(vol_t v, float *u_out) {
    NvtxRange nvtx_range_("vol_read_u");
    if (!v || !u_out) return fail(VOL_EINVAL, "vol_read_u: NULL argument");
    return read_field(v, u_out, v->F.u);
}

extern "C" vol_status vol_read_state(vol_t v, float *u, float *ubar, float *p) {
    NvtxRange nvtx_range_("vol_read_state");
    if (!v) return fail(VOL_EINVAL, "vol_read_state: NULL handle");
    const size_t nv = (size_t)v->L.n_local * kBlockVox;
    const int c = v->cur;
    vol_status st;
    if (u && (st = read_field(v, u, v->F.u)) != VOL_OK) return st;
    if (ubar && (st = read_field(v, ubar, v->F.ub[c])) != VOL_OK) return st;
    if (p) {
        if ((st = read_field(v, p, v->F.px[c])) != VOL_OK) return st;
        if ((st = read_field(v, p + nv, v->F.py[c])) != VOL_OK) return st;
        if ((st = read_field(v, p + 2 * nv, v->F.pz[c])) != VOL_OK) return st;
    }
    return VOL_OK;
}

extern "C" vol_status vol_load_state(vol_t v, const float *u, const float *ubar, const float *p) {
    NvtxRange nvtx_range_("vol_load_state");
    if (!v) return fail(VOL_EINVAL, "vol_load_state: NULL handle");
    if (v->shard) return fail(VOL_ENOTSUP, "vol_load_state: single-GPU volumes only");
    v->pristine = false;
    const size_t nv = (size_t)v->L.n_local * kBlockVox;
    const int c = v->cur;
    vol_status st;
    if (u && (st = write_field(v, v->F.u, u)) != VOL_OK) return st;
    if (ubar && (st = write_field(v, v->F.ub[c], ubar)) != VOL_OK) return st;
    if (p) {
        if ((st = write_field(v, v->F.px[c], p)) != VOL_OK) return st;
        if ((st = write_field(v, v->F.py[c], p + nv)) != VOL_OK) return st;
        if ((st = write_field(v, v->F.pz[c], p + 2 * nv)) != VOL_OK) return st;
    }
    CKL(launch_sanitize_state(v->F, c, v->d_nbr, v->L.n_local, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    return VOL_OK;
}

extern "C" vol_status vol_energy(vol_t v, float lambda, float eps, int data_term, double *primal, double *dual) {
    NvtxRange nvtx_range_("vol_energy");
    if (!v || !primal) return fail(VOL_EINVAL, "vol_energy: NULL argument");
    if (!(lambda > 0.0f) || !(eps >= 0.0f) || (data_term != 0 && data_term != 1))
        return fail(VOL_EINVAL, "vol_energy: bad parameters");
    if (v->shard) {
        vol_status st = shard_refresh_for_energy(v);
        if (st != VOL_OK) return st;
    }
    CKL(launch_energy(view_of(v->F, v->cur), v->d_nbr, nullptr, v->L.n_local, lambda, eps, data_term, v->d_part,
                      v->d_eout, v->stream));
    double o[5];
    if (v->shard) {
        vol_status st = shard_allreduce_energy(v, v->d_eout);
        if (st != VOL_OK) return st;
    }
    CK(cudaMemcpyAsync(o, v->d_eout, sizeof o, cudaMemcpyDeviceToHost, v->stream));
    CK(cudaStreamSynchronize(v->stream));
    *primal = o[0];
    if (dual) *dual = energy_dual_value(o, eps, data_term);
    return VOL_OK;
}

double energy_dual_value(const double *o, float eps, int data_term) {
    const double e = (double)eps;
    if (data_term == 0) {
        const double sc = std::min(1.0, o[4]);
        return -0.5 * e * sc * sc * o[1] - sc * o[2];
    }
    return -0.5 * e * o[1] - o[2] - o[3];
}

extern "C" vol_status vol_read_tables(vol_t v, uint32_t *T, uint32_t *bucket_start, int32_t *bucket_entry,
                                      int32_t *nbr) {
    if (!v) return fail(VOL_EINVAL, "vol_read_tables: NULL handle");
    if (T) *T = v->L.T;
    vol_status st;
    if (bucket_start && (st = copy_out(bucket_start, v->d_start, ((size_t)v->L.T + 1) * 4, v->stream)) != VOL_OK)
        return st;
    if (bucket_entry && (st = copy_out(bucket_entry, v->d_entry, (size_t)v->L.n_global * 4, v->stream)) != VOL_OK)
        return st;
    if (nbr) {
        if (v->shard) return fail(VOL_ENOTSUP, "vol_read_tables: nbr of a sharded volume is in store indices");
        std::vector<int32_t> all((size_t)v->L.S * kNbr), perm((size_t)v->L.n_local);
        CK(cudaMemcpyAsync(all.data(), v->d_nbr, all.size() * 4, cudaMemcpyDeviceToHost, v->stream));
        CK(cudaMemcpyAsync(perm.data(), v->d_perm, perm.size() * 4, cudaMemcpyDeviceToHost, v->stream));
        CK(cudaStreamSynchronize(v->stream));
        std::vector<int32_t> faces((size_t)v->L.S * 6);
        for (int64_t r = 0; r < v->L.S; r++)
            for (int d = 0; d < 6; d++) {
                const int32_t q = all[kNbr * r + d];
                faces[6 * (size_t)perm[r] + d] = q < 0 ? -1 : perm[q];
            }
        if ((st = copy_out(nbr, faces.data(), faces.size() * 4, v->stream)) != VOL_OK) return st;
    }
    return VOL_OK;
}

extern "C" vol_status vol_info(vol_t v, int64_t *n_local, int64_t *n_ghost, int64_t *n_omega) {
    if (!v) return fail(VOL_EINVAL, "vol_info: NULL handle");
    if (n_local) *n_local = v->L.n_local;
    if (n_ghost) *n_ghost = v->L.S - v->L.n_local;
    if (n_omega) *n_omega = v->n_omega_local;
    return VOL_OK;
}

extern "C" vol_status vol_shard_timing(vol_t v, float *interior_ms, float *exchange_ms, float *boundary_ms) {
    if (!v) return fail(VOL_EINVAL, "vol_shard_timing: NULL handle");
    return shard_timing(v, interior_ms, exchange_ms, boundary_ms);
}
