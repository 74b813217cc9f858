// shard.cu — route-axis spatial sharding across GPUs (north_star (c)).
//
// Every rank holds the blocks it owns (caller-supplied owner map `part`: contiguous ranges along the
// route arc length) plus ghost copies of the remote blocks its stencil reads: every remote block among
// the 12 neighbours (6 faces + 6 edges) of a local block.  The fused kernel (iterate.cu) recomputes the
// −face duals itself, so one halo message per peer and iteration — ū^k, p^k (x, y, z) of the ghost
// blocks; W and f once at set-up — makes every local block computable without any other
// inter-GPU dependency.  Per iteration:
//   pack (send blocks' ū^k, p^k → send buffer) on the compute stream;
//   [comm stream]    ncclSend/ncclRecv with each peer in one group → unpack into the ghost rows;
//   [compute stream] launch A = local blocks with no remote neighbour (overlaps the exchange),
//                    wait for the halo, launch B = the remaining local blocks.
// Reads and writes never alias: the kernels read buffers [cur] and write [cur^1]; ghost rows are
// only written by unpack and only read by launch B.  The result is bitwise equal to the single-GPU
// result (no reduction crosses GPUs inside the iteration).
// Transports: NCCL point-to-point, or for tests on one GPU a loopback of device-to-device copies
// between handles of one process (vol_group_connect / vol_regularise_group / vol_group_energy).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <climits>
#include <cstring>
#include <future>
#include <memory>
#include <mutex>
#include <numeric>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "handle.h"
#include "peer.cuh"
#include "shard.h"

using namespace hvg;

// ------------------------------------------------------------------------------ host planning

static uint64_t spread3(uint32_t v) {  // 21 bits → every third bit
    uint64_t x = v & 0x1FFFFFu;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

// Morton (Z-order) of the block coordinates (offset by 2^20): consecutive CTAs work on spatially
// close blocks, so the halo a CTA reads was recently brought into L2 by its neighbours' CTAs.
void hvg::morton_sort_rows(const int32_t *xyz, const std::vector<int64_t> &g, std::vector<int32_t> &rows) {
    // Morton key relative to the bounding box (fewer significant bits), then a stable LSD radix sort
    // (11-bit digits) of (key, index): linear time, and ties keep the input order (deterministic).
    const size_t n = g.size();
    rows.resize(n);
    if (n == 0) return;
    int32_t lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX};
    for (size_t k = 0; k < n; k++)
        for (int a = 0; a < 3; a++) lo[a] = std::min(lo[a], xyz[3 * g[k] + a]);
    std::vector<uint64_t> key(n), key2(n);
    std::vector<int32_t> idx2(n);
    uint64_t kmax = 0;
    for (size_t k = 0; k < n; k++) {
        const int32_t *c = xyz + 3 * g[k];
        key[k] = spread3((uint32_t)(c[0] - lo[0])) | (spread3((uint32_t)(c[1] - lo[1])) << 1) |
                 (spread3((uint32_t)(c[2] - lo[2])) << 2);
        kmax = std::max(kmax, key[k]);
        rows[k] = (int32_t)k;
    }
    constexpr int kBits = 11, kRadix = 1 << kBits;
    std::vector<uint32_t> cnt(kRadix + 1);
    for (int shift = 0; shift < 64 && (kmax >> shift) != 0; shift += kBits) {
        std::fill(cnt.begin(), cnt.end(), 0u);
        for (size_t k = 0; k < n; k++) cnt[((key[k] >> shift) & (kRadix - 1)) + 1]++;
        for (int d = 0; d < kRadix; d++) cnt[d + 1] += cnt[d];
        for (size_t k = 0; k < n; k++) {
            const uint32_t pos = cnt[(key[k] >> shift) & (kRadix - 1)]++;
            key2[pos] = key[k];
            idx2[pos] = rows[k];
        }
        key.swap(key2);
        rows.swap(idx2);
    }
}

namespace {
struct Key {
    int32_t x, y, z;
    bool operator==(const Key &o) const { return x == o.x && y == o.y && z == o.z; }
};
struct KeyHash {
    size_t operator()(const Key &k) const {
        uint64_t h = (uint64_t)(uint32_t)k.x * 0x9E3779B97F4A7C15ull;
        h ^= (uint64_t)(uint32_t)k.y * 0xC2B2AE3D27D4EB4Full + (h << 6) + (h >> 2);
        h ^= (uint64_t)(uint32_t)k.z * 0x165667B19E3779F9ull + (h << 6) + (h >> 2);
        return (size_t)h;
    }
};
}  // namespace

bool hvg::make_shard_plan(const int32_t *xyz, int64_t n, const int32_t *part, int world, int rank, ShardPlan &P) {
    P = ShardPlan();
    P.rank = rank;
    P.world = world;
    if (world < 1 || rank < 0 || rank >= world || n < 1 || !xyz || !part) {
        P.error = "bad arguments";
        return false;
    }
    // open-addressing table (linear probing, power-of-two capacity >= 2n) of the global block set
    size_t cap = 1;
    while (cap < 2 * (size_t)n) cap <<= 1;
    std::vector<int32_t> slot(cap, -1);
    KeyHash hasher;
    auto find = [&](int32_t x, int32_t y, int32_t z) -> int64_t {
        for (size_t h = hasher(Key{x, y, z}) & (cap - 1);; h = (h + 1) & (cap - 1)) {
            const int32_t g = slot[h];
            if (g < 0) return -1;
            if (xyz[3 * g] == x && xyz[3 * g + 1] == y && xyz[3 * g + 2] == z) return g;
        }
    };
    for (int64_t g = 0; g < n; g++) {
        if (part[g] < 0 || part[g] >= world) {
            P.error = "part[" + std::to_string(g) + "] out of range";
            return false;
        }
        const int32_t x = xyz[3 * g], y = xyz[3 * g + 1], z = xyz[3 * g + 2];
        size_t h = hasher(Key{x, y, z}) & (cap - 1);
        for (;; h = (h + 1) & (cap - 1)) {
            const int32_t o = slot[h];
            if (o < 0) break;
            if (xyz[3 * o] == x && xyz[3 * o + 1] == y && xyz[3 * o + 2] == z) {
                P.error = "duplicate block coordinates at block " + std::to_string(g);
                return false;
            }
        }
        slot[h] = (int32_t)g;
    }
    static const int OFF[kNbr][3] = {{-1, 0, 0}, {1, 0, 0},  {0, -1, 0}, {0, 1, 0},  {0, 0, -1}, {0, 0, 1},
                                     {-1, 1, 0}, {-1, 0, 1}, {1, -1, 0}, {0, -1, 1}, {1, 0, -1}, {0, 1, -1}};
    auto nb = [&](int64_t g, int d) -> int64_t {
        return find(xyz[3 * g] + OFF[d][0], xyz[3 * g + 1] + OFF[d][1], xyz[3 * g + 2] + OFF[d][2]);
    };
    // One pass over the rank's own blocks.  The 12-neighbour relation is symmetric (each edge offset's
    // inverse is in the set: 6 ↔ 8, 7 ↔ 10, 9 ↔ 11), so the blocks rank q needs from this rank are
    // exactly this rank's blocks that have a neighbour owned by q: no other rank's plan is needed.
    std::vector<int64_t> ghosts;
    std::vector<std::vector<int64_t>> send_g(world);
    std::vector<int64_t> ga, gb, ca, cb;
    int64_t nl = 0;
    for (int64_t g = 0; g < n; g++) {
        if (part[g] != rank) continue;
        bool remote = false;
        for (int d = 0; d < kNbr; d++) {
            const int64_t c = nb(g, d);
            if (c < 0 || part[c] == rank) continue;
            remote = true;
            ghosts.push_back(c);
            send_g[part[c]].push_back(g);
        }
        // store order of the local blocks: launch A (no remote neighbour) then launch B, each in Morton
        // order, so both launches are contiguous row ranges; local_caller maps a row to the block's
        // position among the rank's blocks in global order (the caller's f / W / u layout)
        (remote ? gb : ga).push_back(g);
        (remote ? cb : ca).push_back(nl++);
    }
    std::sort(ghosts.begin(), ghosts.end(), [&](int64_t a, int64_t b) {
        return part[a] != part[b] ? part[a] < part[b] : a < b;
    });
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    std::vector<int32_t> ord;
    for (auto pr : {std::make_pair(&ga, &ca), std::make_pair(&gb, &cb)}) {
        morton_sort_rows(xyz, *pr.first, ord);
        for (int32_t k : ord) {
            P.local.push_back((*pr.first)[k]);
            P.local_caller.push_back((int32_t)(*pr.second)[k]);
        }
    }
    P.nA = (int64_t)ga.size();
    P.ghost = ghosts;
    P.recv_off.assign(world, 0);
    P.recv_cnt.assign(world, 0);
    for (size_t k = 0; k < P.ghost.size(); k++) P.recv_cnt[part[P.ghost[k]]]++;
    for (int q = 1; q < world; q++) P.recv_off[q] = P.recv_off[q - 1] + P.recv_cnt[q - 1];
    std::vector<int32_t> row(n, -1);
    for (size_t r = 0; r < P.local.size(); r++) row[P.local[r]] = (int32_t)r;
    // send lists in each peer's receive order (ascending global index within an owner)
    P.send_off.assign(world, 0);
    P.send_cnt.assign(world, 0);
    for (int q = 0; q < world; q++) {
        P.send_off[q] = (int64_t)P.send_rows.size();
        std::vector<int64_t> &sg = send_g[q];
        std::sort(sg.begin(), sg.end());
        sg.erase(std::unique(sg.begin(), sg.end()), sg.end());
        for (int64_t g : sg) P.send_rows.push_back(row[g]);
        P.send_cnt[q] = (int64_t)P.send_rows.size() - P.send_off[q];
    }
    return true;
}

extern "C" vol_status vol_plan_shard(const int32_t *xyz, int64_t n, const int32_t *part, int world, int rank,
                                     int64_t *n_local, int64_t *n_ghost, int64_t *n_send, int64_t *ghost_global,
                                     int64_t *send_global, int64_t *peer_send, int64_t *peer_recv) {
    ShardPlan P;
    if (!make_shard_plan(xyz, n, part, world, rank, P)) return fail(VOL_EINVAL, "vol_plan_shard: %s", P.error.c_str());
    if (n_local) *n_local = P.n_local();
    if (n_ghost) *n_ghost = P.n_ghost();
    if (n_send) *n_send = (int64_t)P.send_rows.size();
    if (ghost_global) std::copy(P.ghost.begin(), P.ghost.end(), ghost_global);
    if (send_global)
        for (size_t k = 0; k < P.send_rows.size(); k++) send_global[k] = P.local[P.send_rows[k]];
    if (peer_send) std::copy(P.send_cnt.begin(), P.send_cnt.end(), peer_send);
    if (peer_recv) std::copy(P.recv_cnt.begin(), P.recv_cnt.end(), peer_recv);
    return VOL_OK;
}

// Route-axis partition: order the blocks by the arc length of the point of the route
// polyline nearest to the block centre (ties by (x, y, z)) and cut the order into `world` contiguous
// ranges of equal block count.  The paper's regulariser is block-local with boundary conditions taken
// from the neighbours, so the cut surface is the halo: cutting across the route keeps it
// to one canyon cross-section per rank boundary, and a route that never comes back to itself gives
// every rank at most the two peers r - 1 and r + 1.
extern "C" vol_status vol_partition_route(const int32_t *xyz, int64_t n, const double *route, int32_t n_route,
                                          double block_edge, int world, int32_t *part, double *arc_out) {
    if (!xyz || n < 1 || !route || n_route < 1 || !(block_edge > 0.0) || world < 1 || !part)
        return fail(VOL_EINVAL, "vol_partition_route: bad arguments");
    // cumulative arc length at every polyline vertex
    std::vector<double> cum(n_route, 0.0);
    for (int k = 1; k < n_route; k++) {
        const double *a = route + 3 * (k - 1), *b = route + 3 * k;
        cum[k] = cum[k - 1] + std::sqrt((b[0] - a[0]) * (b[0] - a[0]) + (b[1] - a[1]) * (b[1] - a[1]) +
                                        (b[2] - a[2]) * (b[2] - a[2]));
    }
    std::vector<double> arc(n);
    for (int64_t g = 0; g < n; g++) {
        double c[3];
        for (int a = 0; a < 3; a++) c[a] = ((double)xyz[3 * g + a] + 0.5) * block_edge;
        double best_d2 = INFINITY, best_s = 0.0;
        if (n_route == 1) {
            best_s = 0.0;
        } else {
            for (int k = 0; k + 1 < n_route; k++) {   // first segment with the strictly smallest distance wins
                const double *a = route + 3 * k, *b = route + 3 * (k + 1);
                const double d[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
                const double len2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
                double t = 0.0;
                if (len2 > 0.0) {
                    t = ((c[0] - a[0]) * d[0] + (c[1] - a[1]) * d[1] + (c[2] - a[2]) * d[2]) / len2;
                    t = std::min(1.0, std::max(0.0, t));
                }
                double d2 = 0.0;
                for (int q = 0; q < 3; q++) {
                    const double e = c[q] - (a[q] + t * d[q]);
                    d2 += e * e;
                }
                if (d2 < best_d2) {
                    best_d2 = d2;
                    best_s = cum[k] + t * (cum[k + 1] - cum[k]);
                }
            }
        }
        arc[g] = best_s;
        if (arc_out) arc_out[g] = best_s;
    }
    std::vector<int64_t> order(n);
    std::iota(order.begin(), order.end(), (int64_t)0);
    std::sort(order.begin(), order.end(), [&](int64_t i, int64_t j) {
        if (arc[i] != arc[j]) return arc[i] < arc[j];
        for (int a = 0; a < 3; a++)
            if (xyz[3 * i + a] != xyz[3 * j + a]) return xyz[3 * i + a] < xyz[3 * j + a];
        return i < j;
    });
    for (int r = 0; r < world; r++) {
        const int64_t lo = (int64_t)r * n / world, hi = (int64_t)(r + 1) * n / world;
        for (int64_t k = lo; k < hi; k++) part[order[k]] = r;
    }
    return VOL_OK;
}

// ------------------------------------------------------------------------------ device runtime

constexpr int64_t kMsgFloats = 4 * kBlockVox;  // ū (or W), p_x (or f), p_y, p_z per block

struct ShardRuntime {
    ShardPlan plan;
    bool nccl = false;
    ncclComm_t comm = nullptr;
    cudaStream_t cs = nullptr;       // communication stream
    cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
    // timing events of the last iteration (vol_shard_timing): A start/end, chain start/end, B start/end
    cudaEvent_t ev_t[6] = {};
    bool timed = false;
    float *sendbuf = nullptr, *recvbuf = nullptr;
    int32_t *send_rows = nullptr;
    unsigned long long *omega = nullptr;  // [2] device scratch for the Ω count all-reduce
    bool connected = false;
    bool graphs = true;              // capture the skewed loop into a CUDA graph (HVG_SHARD_NO_GRAPH=1: eager)
    // direct-store transport (peer.cuh): connected peers, their mapped buffers, destinations, counters
    bool p2p = false;
    std::vector<int> peers;                          // ranks this rank exchanges with (send_cnt > 0)
    std::vector<int64_t> peer_slot;                  // [world] slot of a connected peer, −1
    std::vector<PeerOut> peer_out;                   // [slot]
    std::vector<std::vector<int64_t>> peer_info;     // [slot] the peer's vol_peer_info
    std::vector<void *> peer_ipc;                    // IPC mappings to close at destroy
    PeerOut *d_peers = nullptr;                      // [world]
    PeerDst *d_dst = nullptr;                        // [n_local − nA] destinations of each launch-B row
    int2 *d_push = nullptr;                          // [n_send] (slot, peer row) of each send entry
    unsigned long long *flags = nullptr;             // [world] arrivals from each rank (written by peers)
    unsigned long long *expect = nullptr;            // [world] arrivals consumed so far (local)
    int *d_peer_ranks = nullptr;                     // [n_peers]
    int *d_peer_slots = nullptr;                     // [n_peers]
};

size_t hvg::shard_extra_bytes(const ShardPlan &P) {
    Carve c;
    c.take<float>((size_t)P.send_rows.size() * kMsgFloats + 4);
    c.take<float>((size_t)P.ghost.size() * kMsgFloats + 4);
    c.take<int32_t>(P.send_rows.size() + 1);
    c.take<unsigned long long>(4);
    c.take<unsigned long long>(2 * (size_t)P.world + 2);          // flags, expect
    c.take<PeerOut>((size_t)P.world + 1);
    c.take<PeerDst>((size_t)(P.n_local() - P.nA) + 1);
    c.take<int2>(P.send_rows.size() + 1);
    c.take<int>(2 * (size_t)P.world + 2);
    return c.off + 512;
}

__global__ void k_pack(const int32_t *__restrict__ rows, const float *a, const float *b, const float *c,
                       const float *d, float *__restrict__ buf) {
    const int64_t r = rows[blockIdx.x];
    const float *src[4] = {a, b, c, d};
    float4 *dst = reinterpret_cast<float4 *>(buf + (int64_t)blockIdx.x * kMsgFloats);
#pragma unroll
    for (int f = 0; f < 4; f++) {
        const float4 *s = reinterpret_cast<const float4 *>(src[f] + r * kBlockVox);
        dst[f * 128 + threadIdx.x] = s[threadIdx.x];
    }
}

__global__ void k_unpack(int64_t first_row, const float *__restrict__ buf, float *a, float *b, float *c, float *d) {
    const int64_t r = first_row + blockIdx.x;
    float *dst[4] = {a, b, c, d};
    const float4 *src = reinterpret_cast<const float4 *>(buf + (int64_t)blockIdx.x * kMsgFloats);
#pragma unroll
    for (int f = 0; f < 4; f++) reinterpret_cast<float4 *>(dst[f] + r * kBlockVox)[threadIdx.x] = src[f * 128 + threadIdx.x];
}

static vol_status pack(vol_s *v, const float *a, const float *b, const float *c, const float *d, cudaStream_t s) {
    ShardRuntime *R = v->shard;
    const int64_t n = (int64_t)R->plan.send_rows.size();
    if (n > 0) {
        k_pack<<<(unsigned)n, 128, 0, s>>>(R->send_rows, a, b, c, d, R->sendbuf);
        counted(1);
    }
    CK(cudaPeekAtLastError());
    return VOL_OK;
}

static vol_status unpack(vol_s *v, float *a, float *b, float *c, float *d, cudaStream_t s) {
    ShardRuntime *R = v->shard;
    const int64_t n = R->plan.n_ghost();
    if (n > 0) {
        k_unpack<<<(unsigned)n, 128, 0, s>>>(R->plan.n_local(), R->recvbuf, a, b, c, d);
        counted(1);
    }
    CK(cudaPeekAtLastError());
    return VOL_OK;
}

#define NCK(call)                                                                                      \
    do {                                                                                               \
        ncclResult_t r_ = (call);                                                                      \
        if (r_ != ncclSuccess) return fail(VOL_ENCCL, "%s: %s (%s:%d)", #call, ncclGetErrorString(r_), \
                                           __FILE__, __LINE__);                                        \
    } while (0)

static vol_status nccl_exchange(vol_s *v, cudaStream_t s) {
    NvtxRange nvtx_range_("halo_exchange");
    ShardRuntime *R = v->shard;
    const ShardPlan &P = R->plan;
    // the group is always closed, even when a send/recv fails inside it: an open group would defer
    // every later NCCL call of this thread
    ncclResult_t first = ncclGroupStart();
    if (first != ncclSuccess) return fail(VOL_ENCCL, "ncclGroupStart: %s", ncclGetErrorString(first));
    const char *what = nullptr;
    for (int q = 0; q < P.world && !what; q++) {
        if (q == P.rank) continue;
        if (P.send_cnt[q] > 0) {
            const ncclResult_t r = ncclSend(R->sendbuf + P.send_off[q] * kMsgFloats, (size_t)(P.send_cnt[q] * kMsgFloats),
                                            ncclFloat, q, R->comm, s);
            if (r != ncclSuccess) first = r, what = "ncclSend";
        }
        if (!what && P.recv_cnt[q] > 0) {
            const ncclResult_t r = ncclRecv(R->recvbuf + P.recv_off[q] * kMsgFloats, (size_t)(P.recv_cnt[q] * kMsgFloats),
                                            ncclFloat, q, R->comm, s);
            if (r != ncclSuccess) first = r, what = "ncclRecv";
        }
    }
    const ncclResult_t end = ncclGroupEnd();
    if (what) return fail(VOL_ENCCL, "%s: %s", what, ncclGetErrorString(first));
    if (end != ncclSuccess) return fail(VOL_ENCCL, "ncclGroupEnd: %s", ncclGetErrorString(end));
    return VOL_OK;
}

// NCCL communicators are cached by (unique id, world, rank, device): creating a communicator costs
// hundreds of milliseconds, and a process typically builds many volumes over one process group (the
// Python binding reuses one unique id per torch.distributed group).  The first caller of a key inserts
// a placeholder (a shared future) under the lock and runs ncclCommInitRank outside it — so threads of
// one process driving different ranks of one id cannot deadlock each other — and later callers of the
// same key wait on the placeholder instead of initialising the same rank twice.  A failed init removes
// the placeholder (its waiters see the failure); a communicator that reports an asynchronous error is
// aborted and evicted (comm_evict), so later volumes of the group build a fresh one.
namespace {
struct CommEntry {
    unsigned char id[NCCL_UNIQUE_ID_BYTES];
    int world, rank, device;
    std::shared_future<ncclComm_t> comm;   // nullptr once ready = init failed
};
std::vector<std::shared_ptr<CommEntry>> g_comms;
std::mutex g_comms_mu;

bool same_comm_key(const CommEntry &e, const void *id_bytes, int world, int rank, int device) {
    return e.world == world && e.rank == rank && e.device == device && !memcmp(e.id, id_bytes, NCCL_UNIQUE_ID_BYTES);
}
}  // namespace

static vol_status comm_acquire(const void *id_bytes, int world, int rank, int device, ncclComm_t *out) {
    std::promise<ncclComm_t> made;
    std::shared_ptr<CommEntry> mine;
    std::shared_future<ncclComm_t> wait;
    {
        std::lock_guard<std::mutex> lk(g_comms_mu);
        for (const auto &e : g_comms)
            if (same_comm_key(*e, id_bytes, world, rank, device)) wait = e->comm;
        if (!wait.valid()) {
            mine = std::make_shared<CommEntry>();
            memcpy(mine->id, id_bytes, NCCL_UNIQUE_ID_BYTES);
            mine->world = world;
            mine->rank = rank;
            mine->device = device;
            mine->comm = made.get_future().share();
            g_comms.push_back(mine);
        }
    }
    if (!mine) {   // another thread owns (or owned) the initialisation of this key
        ncclComm_t c = wait.get();
        if (!c) return fail(VOL_ENCCL, "ncclCommInitRank of this (id, rank) failed in another thread");
        *out = c;
        return VOL_OK;
    }
    ncclUniqueId id;
    memcpy(&id, id_bytes, sizeof id);
    ncclComm_t comm = nullptr;
    const ncclResult_t r = ncclCommInitRank(&comm, world, id, rank);
    if (r != ncclSuccess) {
        {
            std::lock_guard<std::mutex> lk(g_comms_mu);
            g_comms.erase(std::remove(g_comms.begin(), g_comms.end(), mine), g_comms.end());
        }
        made.set_value(nullptr);
        return fail(VOL_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
    made.set_value(comm);
    *out = comm;
    return VOL_OK;
}

// Process-wide cache of the sharded loop's graphs.  A graph with NCCL nodes is expensive to instantiate and
// to destroy (~1.6 ms: NCCL's resources for captured work), and bench.py / an application creating one
// volume per step would pay both every step.  The graph only holds device addresses inside the volume's
// workspace and the communicator, so it is reused by any later volume whose key — workspace address and
// size, layout, shard-plan digest, communicator, rank, device and the loop's parameters — is identical:
// that volume's buffers sit at the same addresses with the same sizes and counts.  Entries of a
// communicator are destroyed when it is evicted or released; at most kSharedGraphs are kept.
// The executable is reference-counted: a call holds its own reference from lookup through its launches, so an
// eviction by another thread (a 9th key, or the communicator's release) cannot destroy an exec that call is
// about to launch; the last reference synchronises the device and destroys it.
namespace {
using SharedExec = std::shared_ptr<CUgraphExec_st>;
SharedExec shared_exec(cudaGraphExec_t e) {
    return SharedExec(e, [](cudaGraphExec_t x) {
        if (x) {
            cudaDeviceSynchronize();   // the exec may still run on some volume's stream
            cudaGraphExecDestroy(x);
        }
    });
}
struct SharedGraph {
    std::string key;
    SharedExec exec;
    int64_t per;
    ncclComm_t comm;
};
std::mutex g_sg_mu;
// heap-allocated and never destroyed: no graph destruction (device synchronisation, NCCL resources) runs
// during static destruction at process exit, after the CUDA runtime or a communicator may be gone
std::vector<SharedGraph> &g_sg = *new std::vector<SharedGraph>();
constexpr size_t kSharedGraphs = 8;

void shared_graphs_drop(ncclComm_t comm) {   // comm == nullptr: all
    std::vector<SharedGraph> dead;
    {
        std::lock_guard<std::mutex> lk(g_sg_mu);
        for (auto it = g_sg.begin(); it != g_sg.end();) {
            if (!comm || it->comm == comm) {
                dead.push_back(*it);
                it = g_sg.erase(it);
            } else {
                ++it;
            }
        }
    }
    dead.clear();   // each exec is destroyed with its last reference
}
}  // namespace

template <class Body>
static vol_status cached_graph_shared(vol_s *v, const GraphKey &key, ncclComm_t comm, Body body, SharedExec *hold,
                                      cudaGraphExec_t *exec, int64_t *per) {
    {
        std::lock_guard<std::mutex> lk(g_sg_mu);
        for (const SharedGraph &e : g_sg)
            if (e.key == key.bytes) {
                *hold = e.exec;
                *exec = e.exec.get();
                *per = e.per;
                return VOL_OK;
            }
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
    SharedExec ref = shared_exec(ge);
    SharedGraph old{};
    {
        std::lock_guard<std::mutex> lk(g_sg_mu);
        if (g_sg.size() >= kSharedGraphs) {
            old = std::move(g_sg.front());   // released below, outside the lock
            g_sg.erase(g_sg.begin());
        }
        g_sg.push_back(SharedGraph{key.bytes, ref, n, comm});
    }
    old = SharedGraph{};
    *hold = std::move(ref);
    *exec = ge;
    *per = n;
    return VOL_OK;
}

// A communicator with an asynchronous error is unusable: abort it and drop it from the cache.
static void comm_evict(ncclComm_t comm) {
    bool found = false;
    {
        std::lock_guard<std::mutex> lk(g_comms_mu);
        for (auto it = g_comms.begin(); it != g_comms.end(); ++it) {
            const std::shared_future<ncclComm_t> &f = (*it)->comm;
            if (f.wait_for(std::chrono::seconds(0)) == std::future_status::ready && f.get() == comm) {
                g_comms.erase(it);
                found = true;
                break;
            }
        }
    }
    if (found) {
        shared_graphs_drop(comm);
        ncclCommAbort(comm);
    }
}

// Asynchronous NCCL failures of earlier work (SURVEY §5 failure detection): evict the communicator.
static vol_status check_async(ncclComm_t comm) {
    ncclResult_t async = ncclSuccess;
    if (ncclCommGetAsyncError(comm, &async) == ncclSuccess && async != ncclSuccess && async != ncclInProgress) {
        comm_evict(comm);
        return fail(VOL_ENCCL, "NCCL asynchronous error: %s (communicator aborted)", ncclGetErrorString(async));
    }
    return VOL_OK;
}

extern "C" vol_status vol_release_comms(void) {
    shared_graphs_drop(nullptr);
    std::vector<std::shared_ptr<CommEntry>> all;
    {
        std::lock_guard<std::mutex> lk(g_comms_mu);
        all.swap(g_comms);
    }
    ncclResult_t first = ncclSuccess;
    for (auto &e : all) {
        ncclComm_t c = e->comm.get();
        if (!c) continue;
        const ncclResult_t r = ncclCommDestroy(c);
        if (first == ncclSuccess) first = r;
    }
    if (first != ncclSuccess) return fail(VOL_ENCCL, "ncclCommDestroy: %s", ncclGetErrorString(first));
    return VOL_OK;
}

extern "C" vol_status vol_nccl_unique_id(void *out128) {
    if (!out128) return fail(VOL_EINVAL, "vol_nccl_unique_id: NULL");
    ncclUniqueId id;
    NCK(ncclGetUniqueId(&id));
    memcpy(out128, &id, sizeof id);
    return VOL_OK;
}

vol_status shard_setup(vol_s *v, const ShardPlan &plan, const vol_dist *dist) {
    ShardRuntime *R = new ShardRuntime();
    v->shard = R;
    R->plan = plan;
    const ShardPlan &P = R->plan;
    cudaStream_t s = v->stream;
    Carve c;
    c.base = v->extra;
    R->sendbuf = c.take<float>((size_t)P.send_rows.size() * kMsgFloats + 4);
    R->recvbuf = c.take<float>((size_t)P.ghost.size() * kMsgFloats + 4);
    R->send_rows = c.take<int32_t>(P.send_rows.size() + 1);
    R->omega = c.take<unsigned long long>(4);
    R->flags = c.take<unsigned long long>(2 * (size_t)P.world + 2);
    R->expect = R->flags + P.world;
    R->d_peers = c.take<PeerOut>((size_t)P.world + 1);
    R->d_dst = c.take<PeerDst>((size_t)(P.n_local() - P.nA) + 1);
    R->d_push = c.take<int2>(P.send_rows.size() + 1);
    R->d_peer_ranks = c.take<int>(2 * (size_t)P.world + 2);
    R->d_peer_slots = R->d_peer_ranks + P.world;
    CK(cudaMemsetAsync(R->flags, 0, (2 * (size_t)P.world + 2) * sizeof(unsigned long long), s));
    R->peer_slot.assign(P.world, -1);
    for (int q = 0; q < P.world; q++)
        if (q != P.rank && P.send_cnt[q] > 0) R->peers.push_back(q);
    std::vector<int32_t> send32(P.send_rows.begin(), P.send_rows.end());
    // (a copy from pageable host memory returns once the data is staged: the host vector may go)
    CK(cudaMemcpyAsync(R->send_rows, send32.data(), send32.size() * 4, cudaMemcpyHostToDevice, s));
    CK(cudaStreamCreateWithFlags(&R->cs, cudaStreamNonBlocking));
    R->graphs = getenv("HVG_SHARD_NO_GRAPH") == nullptr;
    CK(cudaEventCreateWithFlags(&R->ev_pack, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&R->ev_halo, cudaEventDisableTiming));
    for (auto &e : R->ev_t) CK(cudaEventCreate(&e));
    if (dist->nccl_id) {
        R->nccl = true;
        vol_status st = comm_acquire(dist->nccl_id, P.world, P.rank, v->device, &R->comm);
        if (st != VOL_OK) return st;
    }
    return VOL_OK;
}

// Static ghost data (W, f) and the global Ω count.  NCCL: now; loopback: in vol_group_connect.
vol_status shard_after_create(vol_s *v) {
    ShardRuntime *R = v->shard;
    if (!R->nccl) return VOL_OK;
    cudaStream_t s = v->stream;
    float *W = const_cast<float *>(v->F.W), *f = const_cast<float *>(v->F.f);
    vol_status st = pack(v, W, f, W, f, s);
    if (st != VOL_OK) return st;
    if ((st = nccl_exchange(v, s)) != VOL_OK) return st;
    if ((st = unpack(v, W, f, v->F.ub[0], v->F.ub[1], s)) != VOL_OK) return st;
    CKL(launch_init_state(v->F, v->L.S * kBlockVox, 0, s));
    // the 8-bit weight copy (finalize_w8) in the same synchronisation: every held W, ghosts included, is final
    unsigned *d_bad = reinterpret_cast<unsigned *>(&v->d_misc[3]);
    unsigned bad = 0;
    CK(cudaMemsetAsync(d_bad, 0, sizeof(unsigned), s));
    CKL(launch_pack_w8(v->F.W, v->d_w8, v->L.S * kBlockVox, d_bad, s));
    CK(cudaMemcpyAsync(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost, s));
    unsigned long long cnt = (unsigned long long)v->n_omega_local, tot = 0;
    CK(cudaMemcpyAsync(R->omega, &cnt, 8, cudaMemcpyHostToDevice, s));
    NCK(ncclAllReduce(R->omega, R->omega + 1, 1, ncclUint64, ncclSum, R->comm, s));
    CK(cudaMemcpyAsync(&tot, R->omega + 1, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    v->F.W8 = bad ? nullptr : v->d_w8;
    v->n_omega_global = (int64_t)tot;
    R->connected = true;
    return VOL_OK;
}

bool vol_s::shard_nccl() const { return shard && shard->nccl; }

vol_status shard_reset(vol_s *v) {
    if (!v->shard->connected) return fail(VOL_EINVAL, "sharded volume not connected (call vol_group_connect)");
    return VOL_OK;
}

// One sharded iteration on one rank with the NCCL transport.  `timed`: record the per-stream timing
// events (the last iteration of a call).  exchange == 0 replaces the halo chain by a no-op (timing only).
static vol_status nccl_iteration(vol_s *v, const IterParams &P, int64_t &launches, bool timed) {
    ShardRuntime *R = v->shard;
    cudaStream_t s = v->stream;
    const int cur = v->cur;
    const bool xchg = v->pending_exchange != 0;
    CK(cudaEventRecord(R->ev_pack, s));
    CK(cudaStreamWaitEvent(R->cs, R->ev_pack, 0));
    if (timed) CK(cudaEventRecord(R->ev_t[2], R->cs));
    if (xchg) {
        // pack on the communication stream: it reads ū^k, p^k, final once the previous iteration's
        // launch B (ordered before ev_pack on the compute stream) has finished
        vol_status st = pack(v, v->F.ub[cur], v->F.px[cur], v->F.py[cur], v->F.pz[cur], R->cs);
        if (st != VOL_OK) return st;
        if ((st = nccl_exchange(v, R->cs)) != VOL_OK) return st;
        if ((st = unpack(v, v->F.ub[cur], v->F.px[cur], v->F.py[cur], v->F.pz[cur], R->cs)) != VOL_OK) return st;
    }
    if (timed) CK(cudaEventRecord(R->ev_t[3], R->cs));
    CK(cudaEventRecord(R->ev_halo, R->cs));
    View V = view_of(v->F, cur);
    V.frozen = v->pending_frozen;
    const ShardPlan &SP = R->plan;
    if (timed) CK(cudaEventRecord(R->ev_t[0], s));
    int r = launch_fused(V, v->d_nbr, nullptr, 0, SP.nA, P, s);
    CKL(r);
    if (timed) CK(cudaEventRecord(R->ev_t[1], s));
    CK(cudaStreamWaitEvent(s, R->ev_halo, 0));
    if (timed) CK(cudaEventRecord(R->ev_t[4], s));
    int r2 = launch_fused(V, v->d_nbr, nullptr, SP.nA, SP.n_local() - SP.nA, P, s);
    CKL(r2);
    if (timed) CK(cudaEventRecord(R->ev_t[5], s));
    if (timed) R->timed = true;
    launches += r + r2 + (xchg ? 2 : 0);  // + pack + unpack
    v->cur ^= 1;
    return VOL_OK;
}

vol_status shard_timing(vol_s *v, float *interior_ms, float *exchange_ms, float *boundary_ms) {
    ShardRuntime *R = v->shard;
    if (!R || !R->nccl) return fail(VOL_EINVAL, "vol_shard_timing: the volume is not NCCL-sharded");
    if (!R->timed) return fail(VOL_EINVAL, "vol_shard_timing: no sharded iteration has run yet");
    CK(cudaEventSynchronize(R->ev_t[5]));
    float a = 0.f, c = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, R->ev_t[0], R->ev_t[1]));
    CK(cudaEventElapsedTime(&c, R->ev_t[2], R->ev_t[3]));
    CK(cudaEventElapsedTime(&b, R->ev_t[4], R->ev_t[5]));
    if (interior_ms) *interior_ms = a;
    if (exchange_ms) *exchange_ms = c;
    if (boundary_ms) *boundary_ms = b;
    return VOL_OK;
}

// ---- skewed schedule on a sharded volume (opts.kernel = 2), NCCL transport.  The same sequence as the
// single-GPU run_iterations_skew, with a halo exchange in front of every launch that reads ghosts:
//   X(ū^0, p^0) · k_dual · { X(u^j, p^{j+1}) ∥ k_skew A ; k_skew B }_{j < iters−1} · X(p^iters) · k_primal
// (A = local blocks without a remote neighbour, launched while the exchange runs; B the others).  The
// exchange moves four fields per boundary block (a u field and p), like the one-pass schedule's (ū, p).
// The halo chain of one exchange: fork from the compute stream `s` to the communication stream, pack →
// ncclSend/ncclRecv → unpack there, and record ev_halo for launch B to wait on.  Returns the number of
// kernels it launches (pack, unpack).
static vol_status nccl_exchange_fields(vol_s *v, cudaStream_t s, float *a, float *px, float *py, float *pz,
                                       int64_t &launches, bool timed = false) {
    ShardRuntime *R = v->shard;
    CK(cudaEventRecord(R->ev_pack, s));
    CK(cudaStreamWaitEvent(R->cs, R->ev_pack, 0));
    if (timed) CK(cudaEventRecord(R->ev_t[2], R->cs));
    if (v->pending_exchange) {   // opts.exchange = 0: no-op chain (timing only)
        vol_status st = pack(v, a, px, py, pz, R->cs);
        if (st != VOL_OK) return st;
        if ((st = nccl_exchange(v, R->cs)) != VOL_OK) return st;
        if ((st = unpack(v, a, px, py, pz, R->cs)) != VOL_OK) return st;
        launches += (R->plan.send_rows.empty() ? 0 : 1) + (R->plan.ghost.empty() ? 0 : 1);
    }
    if (timed) CK(cudaEventRecord(R->ev_t[3], R->cs));
    CK(cudaEventRecord(R->ev_halo, R->cs));
    return VOL_OK;
}

// Skewed schedule on a sharded volume, NCCL transport — the single-GPU run_iterations_skew with a halo
// exchange in front of every launch that reads ghosts:
//   X(ū^0, p^0) · k_dual · { X(u^j, p^{j+1}) ∥ k_skew A ; k_skew B }_{j < iters−1} · X(p^iters) · k_primal
// (A = local blocks without a remote neighbour, launched while the exchange runs; B the others).  The
// exchange moves four fields per boundary block (a u field and p).  The loop body is captured once per
// call into a CUDA graph of 2m iterations (the buffer parities repeat every 2) — the compute stream
// forks to the communication stream and joins back through ev_pack / ev_halo inside the graph, NCCL's
// send/recv are captured as graph nodes — and replayed, so the host issues one graph launch per 2m
// iterations instead of ~10 API calls and an NCCL group per iteration ("careful synchronization
// between subsequent primal and dual variable updates": here it is the graph's dependency edges).  The
// last skewed iteration runs eagerly with the timing events (vol_shard_timing).
static vol_status nccl_skew(vol_s *v, const IterParams &P, int32_t iters) {
    ShardRuntime *R = v->shard;
    const ShardPlan &SP = R->plan;
    cudaStream_t s = v->stream;
    const int c = v->cur;
    const int64_t nl = SP.n_local(), nA = SP.nA;
    int64_t launches = 0;
    CK(cudaMemcpyAsync(v->d_u2, v->F.u, (size_t)v->L.S * kBlockVox * 4, cudaMemcpyDeviceToDevice, s));
    float *B[2];
    B[(iters - 1) & 1] = v->F.u;
    B[iters & 1] = v->d_u2;
    vol_status st = nccl_exchange_fields(v, s, v->F.ub[c], v->F.px[c], v->F.py[c], v->F.pz[c], launches);
    if (st != VOL_OK) return st;
    CK(cudaStreamWaitEvent(s, R->ev_halo, 0));
    int r = launch_dual_only(view_of(v->F, c), v->d_nbr, nl, P, s);
    CKL(r);
    launches += r;
    // one skewed iteration j on compute stream `cs_` (the chain on R->cs)
    auto skew_iter = [&](cudaStream_t cs_, int j, bool timed, int64_t &n) -> vol_status {
        const int pin = c ^ ((j + 1) & 1);
        vol_status st2 = nccl_exchange_fields(v, cs_, B[j & 1], v->F.px[pin], v->F.py[pin], v->F.pz[pin], n, timed);
        if (st2 != VOL_OK) return st2;
        if (timed) CK(cudaEventRecord(R->ev_t[0], cs_));
        int a = launch_skew(v->F, B[j & 1], B[(j + 1) & 1], pin, v->pending_frozen, v->d_nbr, 0, nA, P, cs_);
        CKL(a);
        if (timed) CK(cudaEventRecord(R->ev_t[1], cs_));
        CK(cudaStreamWaitEvent(cs_, R->ev_halo, 0));
        if (timed) CK(cudaEventRecord(R->ev_t[4], cs_));
        int b = launch_skew(v->F, B[j & 1], B[(j + 1) & 1], pin, v->pending_frozen, v->d_nbr, nA, nl - nA, P, cs_);
        CKL(b);
        if (timed) {
            CK(cudaEventRecord(R->ev_t[5], cs_));
            R->timed = true;
        }
        n += a + b;
        return VOL_OK;
    };
    const int total = iters - 1;            // skewed launches
    const int body = total - 1;             // all but the last (timed, eager)
    const int m = std::min(16, body / 2);
    int j = 0;
    if (m >= 1 && R->graphs) {
        GraphKey key;
        key.add('N').add(c).add(m).add(iters & 1).add(v->pending_frozen).add(v->pending_exchange).add(P);
        cudaGraphExec_t ge = nullptr;
        SharedExec hold;   // keeps a shared exec alive through the launches below
        int64_t per = 0;
        auto capture = [&](cudaStream_t cap, int64_t &n) -> vol_status {
            for (int k = 0; k < 2 * m; k++) {
                vol_status s2 = skew_iter(cap, k, false, n);
                if (s2 != VOL_OK) return s2;
            }
            return VOL_OK;
        };
        if (SP.digest != 0 && R->comm) {   // reusable by later volumes with the same workspace and plan
            key.add(v->ws).add(v->ws_bytes).add(v->L.n_global).add(v->L.n_local).add(v->L.S).add(v->L.T)
                .add(SP.digest).add(SP.rank).add(SP.world).add(R->comm).add(v->device);
            st = cached_graph_shared(v, key, R->comm, capture, &hold, &ge, &per);
        } else {
            st = cached_graph(v, key, capture, &ge, &per);
        }
        if (st != VOL_OK) return st;
        const int reps = body / (2 * m);
        for (int q = 0; q < reps; q++) {
            CK(cudaGraphLaunch(ge, s));
            launches += per;
            g_launches.fetch_add(per);
        }
        j = reps * 2 * m;
    }
    for (; j < total; j++)
        if ((st = skew_iter(s, j, j == total - 1, launches)) != VOL_OK) return st;
    if (iters < 2) {   // no skewed launch: the timing events record an empty interval
        for (int k = 0; k < 6; k++) CK(cudaEventRecord(R->ev_t[k], k == 2 || k == 3 ? R->cs : s));
        R->timed = true;
    }
    const int c2 = c ^ (iters & 1);
    if ((st = nccl_exchange_fields(v, s, v->F.ub[c2], v->F.px[c2], v->F.py[c2], v->F.pz[c2], launches)) != VOL_OK)
        return st;
    CK(cudaStreamWaitEvent(s, R->ev_halo, 0));
    View V = view_of(v->F, c2 ^ 1);   // px_out = p[c2] (p^iters), ub_out = ub[c2]
    V.u = B[(iters - 1) & 1];         // == F.u
    r = launch_primal_only(V, v->d_nbr, nl, P, s);
    CKL(r);
    launches += r;
    v->cur = c2;
    v->last_launches = launches;
    return VOL_OK;
}

static int p2p_signal(vol_s *v, cudaStream_t s);
static int p2p_wait(vol_s *v, cudaStream_t s);
static int p2p_push(vol_s *v, const float *a, int which_a, int pidx, cudaStream_t s);

// The skewed schedule with the direct-store transport (one rank; its peers run the same sequence):
//   ready · push(ū⁰, p⁰) · k_dual · push(u⁰, p¹) · { A_j · wait · B_j (+ stores into the peers) · signal } · wait · k_primal
// with a signal after every push and a wait before every consumer of ghost data (see above).
static vol_status p2p_skew(vol_s *v, const IterParams &P, int32_t iters) {
    ShardRuntime *R = v->shard;
    const ShardPlan &SP = R->plan;
    cudaStream_t s = v->stream;
    const int c = v->cur;
    const int64_t nl = SP.n_local(), nA = SP.nA;
    int64_t launches = 0;
    CK(cudaMemcpyAsync(v->d_u2, v->F.u, (size_t)v->L.S * kBlockVox * 4, cudaMemcpyDeviceToDevice, s));
    float *B[2];
    B[(iters - 1) & 1] = v->F.u;
    B[iters & 1] = v->d_u2;
    auto uidx = [&](const float *p) { return p == v->F.u ? 0 : 1; };
    auto step = [&](int r) -> vol_status {
        CKL(r);
        launches += r;
        return VOL_OK;
    };
    vol_status st;
    if ((st = step(p2p_signal(v, s))) != VOL_OK || (st = step(p2p_wait(v, s))) != VOL_OK) return st;   // ready
    if ((st = step(p2p_push(v, v->F.ub[c], 2 + c, c, s))) != VOL_OK || (st = step(p2p_signal(v, s))) != VOL_OK ||
        (st = step(p2p_wait(v, s))) != VOL_OK)
        return st;
    if ((st = step(launch_dual_only(view_of(v->F, c), v->d_nbr, nl, P, s))) != VOL_OK) return st;
    if ((st = step(p2p_push(v, B[0], uidx(B[0]), c ^ 1, s))) != VOL_OK || (st = step(p2p_signal(v, s))) != VOL_OK)
        return st;
    auto skew_iter = [&](cudaStream_t cs_, int j, bool timed, int64_t &n) -> vol_status {
        const int pin = c ^ ((j + 1) & 1);
        if (timed) CK(cudaEventRecord(R->ev_t[0], cs_));
        int a = launch_skew(v->F, B[j & 1], B[(j + 1) & 1], pin, v->pending_frozen, v->d_nbr, 0, nA, P, cs_);
        CKL(a);
        if (timed) {
            CK(cudaEventRecord(R->ev_t[1], cs_));
            CK(cudaEventRecord(R->ev_t[2], cs_));
        }
        int w = p2p_wait(v, cs_);
        CKL(w);
        if (timed) {
            CK(cudaEventRecord(R->ev_t[3], cs_));
            CK(cudaEventRecord(R->ev_t[4], cs_));
        }
        int b = launch_skew_peers(v->F, B[j & 1], B[(j + 1) & 1], pin, v->pending_frozen, v->d_nbr, nA, nl - nA, P,
                                  R->d_peers, R->d_dst, cs_);
        CKL(b);
        if (timed) {
            CK(cudaEventRecord(R->ev_t[5], cs_));
            R->timed = true;
        }
        int g = p2p_signal(v, cs_);
        CKL(g);
        n += a + w + b + g;
        return VOL_OK;
    };
    const int total = iters - 1;
    const int body = total - 1;
    const int m = std::min(16, body / 2);
    int j = 0;
    if (m >= 1 && R->graphs) {
        GraphKey key;
        key.add('Q').add(c).add(m).add(iters & 1).add(v->pending_frozen).add(P);
        cudaGraphExec_t ge = nullptr;
        int64_t per = 0;
        st = cached_graph(
            v, key,
            [&](cudaStream_t cap, int64_t &n) -> vol_status {
                for (int k = 0; k < 2 * m; k++) {
                    vol_status s2 = skew_iter(cap, k, false, n);
                    if (s2 != VOL_OK) return s2;
                }
                return VOL_OK;
            },
            &ge, &per);
        if (st != VOL_OK) return st;
        const int reps = body / (2 * m);
        for (int q = 0; q < reps; q++) {
            CK(cudaGraphLaunch(ge, s));
            launches += per;
            g_launches.fetch_add(per);
        }
        j = reps * 2 * m;
    }
    for (; j < total; j++)
        if ((st = skew_iter(s, j, j == total - 1, launches)) != VOL_OK) return st;
    if (iters < 2) {
        for (int k = 0; k < 6; k++) CK(cudaEventRecord(R->ev_t[k], s));
        R->timed = true;
    }
    if ((st = step(p2p_wait(v, s))) != VOL_OK) return st;
    const int c2 = c ^ (iters & 1);
    View V = view_of(v->F, c2 ^ 1);   // px_out = p[c2] (p^iters), ub_out = ub[c2]
    V.u = B[(iters - 1) & 1];         // == F.u
    if ((st = step(launch_primal_only(V, v->d_nbr, nl, P, s))) != VOL_OK) return st;
    v->cur = c2;
    v->last_launches = launches;
    return VOL_OK;
}

vol_status shard_iterate(vol_s *v, const IterParams &P, int32_t iters) {
    ShardRuntime *R = v->shard;
    if (!R->nccl) return fail(VOL_EINVAL, "loopback-sharded volume: use vol_regularise_group");
    if (v->pending_kernel == 0 || v->pending_kernel == 2) {   // the product path: the skewed schedule
        vol_status st = (R->p2p && v->pending_exchange) ? p2p_skew(v, P, iters) : nccl_skew(v, P, iters);
        if (st != VOL_OK) return st;
        return check_async(R->comm);
    }
    int64_t launches = 0;
    for (int32_t k = 0; k < iters; k++) {
        vol_status st = nccl_iteration(v, P, launches, k == iters - 1);
        if (st != VOL_OK) return st;
    }
    v->last_launches = launches;
    return check_async(R->comm);
}

// Refresh every ghost's u and p (energy needs u of +neighbours and p of −neighbours), then the
// per-rank partial sums are all-reduced (sum of 4 terms, min of the L1 dual scale).
vol_status shard_refresh_for_energy(vol_s *v) {
    ShardRuntime *R = v->shard;
    if (!R->nccl) return VOL_OK;  // loopback: vol_group_energy refreshes
    cudaStream_t s = v->stream;
    const int c = v->cur;
    vol_status st = pack(v, v->F.u, v->F.px[c], v->F.py[c], v->F.pz[c], s);
    if (st != VOL_OK) return st;
    if ((st = nccl_exchange(v, s)) != VOL_OK) return st;
    return unpack(v, v->F.u, v->F.px[c], v->F.py[c], v->F.pz[c], s);
}

vol_status shard_allreduce_energy(vol_s *v, double *d_eout) {
    ShardRuntime *R = v->shard;
    if (!R->nccl) return VOL_OK;
    NCK(ncclAllReduce(d_eout, d_eout, 4, ncclDouble, ncclSum, R->comm, v->stream));
    NCK(ncclAllReduce(d_eout + 4, d_eout + 4, 1, ncclDouble, ncclMin, R->comm, v->stream));
    return VOL_OK;
}

void shard_destroy(vol_s *v) {
    ShardRuntime *R = v->shard;
    if (!R) return;
    if (v->stream) cudaStreamSynchronize(v->stream);
    if (R->cs) {
        cudaStreamSynchronize(R->cs);
        cudaStreamDestroy(R->cs);
    }
    if (R->ev_pack) cudaEventDestroy(R->ev_pack);
    if (R->ev_halo) cudaEventDestroy(R->ev_halo);
    for (auto &e : R->ev_t)
        if (e) cudaEventDestroy(e);
    // the communicator stays cached for later volumes of the same process group (comm_acquire)
    for (void *p : R->peer_ipc) cudaIpcCloseMemHandle(p);
    delete R;
    v->shard = nullptr;
}

// ---------------------------------------------------------------- direct-store transport (peers)
// The boundary launch writes each block a peer reads straight into the peer's ghost rows (k_skew<…, true>,
// peer.cuh); the prologue / post-dual exchanges copy with k_push.  Completion is a per-source arrival
// counter in the receiver's memory (k_signal: system-scope fence, then an atomic add into every peer's
// counter for this rank) and a device-side expected count (k_wait spins until every peer's counter
// reaches it), so the same graph can be replayed.  Waits before every consumer of ghost data also order
// the writes against the peer's previous reads of the same buffers (the rank only writes buffer parity
// j + 1 after every peer has signalled the end of its launch j − 1), and a "ready" handshake at the start
// of a call orders the first pushes after the peer's previous call.

__global__ void k_push(const int32_t *__restrict__ rows, const int2 *__restrict__ push, const PeerOut *__restrict__ peers,
                       const float *a, const float *px, const float *py, const float *pz, int which_a, int pidx) {
    const int64_t e = blockIdx.x;
    const int64_t r = rows[e];
    const int2 d = push[e];
    const PeerOut &Q = peers[d.x];
    float *dst[4] = {which_a == 0 ? Q.u[0] : (which_a == 1 ? Q.u[1] : (which_a == 2 ? Q.ub[0] : Q.ub[1])),
                     Q.px[pidx], Q.py[pidx], Q.pz[pidx]};
    const float *src[4] = {a, px, py, pz};
#pragma unroll
    for (int f = 0; f < 4; f++)
        reinterpret_cast<float4 *>(dst[f] + (int64_t)d.y * kBlockVox)[threadIdx.x] =
            reinterpret_cast<const float4 *>(src[f] + r * kBlockVox)[threadIdx.x];
    __threadfence_system();
}

__global__ void k_signal(const PeerOut *__restrict__ peers, const int *__restrict__ slots, int n, int me) {
    __threadfence_system();
    const int i = threadIdx.x;
    if (i < n) atomicAdd_system(peers[slots[i]].flags + me, 1ull);
}

// Spins at most ~10 s (a peer that never signals is a broken peer, not a slow one): then it records the
// failure in expect[world] (read back by the host after loopback calls) and gives up.
__global__ void k_wait(unsigned long long *flags, unsigned long long *expect, const int *__restrict__ ranks, int n,
                       int world) {
    const int i = threadIdx.x;
    if (i < n) {
        const int q = ranks[i];
        const unsigned long long target = expect[q] + 1;
        const long long t0 = clock64();
        unsigned long long v;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + q) : "memory");
            if (v < target && clock64() - t0 > 20000000000ll) {
                atomicExch(expect + world, 1ull);
                break;
            }
        } while (v < target);
        expect[q] = target;
    }
    __syncwarp();
}

static int p2p_signal(vol_s *v, cudaStream_t s) {
    ShardRuntime *R = v->shard;
    const int n = (int)R->peers.size();
    if (n == 0) return 0;
    k_signal<<<1, 32, 0, s>>>(R->d_peers, R->d_peer_slots, n, R->plan.rank);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

static int p2p_wait(vol_s *v, cudaStream_t s) {
    ShardRuntime *R = v->shard;
    const int n = (int)R->peers.size();
    if (n == 0) return 0;
    k_wait<<<1, 32, 0, s>>>(R->flags, R->expect, R->d_peer_ranks, n, R->plan.world);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// which_a: 0/1 = the peer's u / u2 buffer, 2/3 = its ū[0] / ū[1]; pidx: the peer's p parity
static int p2p_push(vol_s *v, const float *a, int which_a, int pidx, cudaStream_t s) {
    ShardRuntime *R = v->shard;
    const int64_t n = (int64_t)R->plan.send_rows.size();
    if (n == 0) return 0;
    k_push<<<(unsigned)n, 128, 0, s>>>(R->send_rows, R->d_push, R->d_peers, a, v->F.px[pidx], v->F.py[pidx],
                                       v->F.pz[pidx], which_a, pidx);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

static constexpr int kPeerInfoFixed = 6, kPeerInfoOffsets = 11;

extern "C" vol_status vol_peer_info(vol_t v, int64_t *info, int64_t cap, int64_t *n) {
    if (!v || !v->shard || !n) return fail(VOL_EINVAL, "vol_peer_info: not a sharded volume");
    const ShardPlan &P = v->shard->plan;
    const int64_t need = kPeerInfoFixed + P.world + kPeerInfoOffsets;
    *n = need;
    if (!info) return VOL_OK;
    if (cap < need) return fail(VOL_EINVAL, "vol_peer_info: %lld entries needed", (long long)need);
    const char *base = (const char *)v->ws;
    int64_t k = 0;
    info[k++] = 1;   // version
    info[k++] = P.rank;
    info[k++] = P.world;
    info[k++] = P.n_local();
    info[k++] = v->L.S;
    info[k++] = need;
    for (int q = 0; q < P.world; q++) info[k++] = P.recv_off[q];
    const void *ptrs[kPeerInfoOffsets] = {v->F.u,     v->d_u2,    v->F.ub[0], v->F.ub[1], v->F.px[0], v->F.px[1],
                                          v->F.py[0], v->F.py[1], v->F.pz[0], v->F.pz[1], v->shard->flags};
    for (const void *p : ptrs) info[k++] = (int64_t)((const char *)p - base);
    return VOL_OK;
}

// All peers connected: build the destination tables and switch the volume to direct stores.
static vol_status p2p_finalize(vol_s *v) {
    ShardRuntime *R = v->shard;
    const ShardPlan &P = R->plan;
    const int64_t nB = P.n_local() - P.nA;
    std::vector<PeerDst> dst((size_t)std::max<int64_t>(nB, 1));
    for (auto &d : dst)
        for (int k = 0; k < kMaxDst; k++) d.slot[k] = -1, d.row[k] = 0;
    std::vector<int2> push(P.send_rows.size());
    for (int q : R->peers) {
        const int64_t slot = R->peer_slot[q];
        const std::vector<int64_t> &I = R->peer_info[slot];
        const int64_t q_nlocal = I[3], q_recv_off_me = I[kPeerInfoFixed + P.rank];
        for (int64_t i = 0; i < P.send_cnt[q]; i++) {
            const int64_t e = P.send_off[q] + i;
            const int64_t row = P.send_rows[e];
            const int64_t prow = q_nlocal + q_recv_off_me + i;
            push[e] = make_int2((int)slot, (int)prow);
            if (row < P.nA || row >= P.n_local()) return fail(VOL_EINVAL, "peer transport: send row outside launch B");
            PeerDst &d = dst[row - P.nA];
            int k = 0;
            while (k < kMaxDst && d.slot[k] >= 0) k++;
            if (k == kMaxDst) return fail(VOL_ENOTSUP, "peer transport: a block is read by more than %d peers", kMaxDst);
            d.slot[k] = (int)slot;
            d.row[k] = (int)prow;
        }
    }
    std::vector<int> ranks(R->peers.begin(), R->peers.end()), slots;
    for (int q : R->peers) slots.push_back((int)R->peer_slot[q]);
    cudaStream_t s = v->stream;
    CK(cudaMemcpyAsync(R->d_peers, R->peer_out.data(), R->peer_out.size() * sizeof(PeerOut), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(R->d_dst, dst.data(), dst.size() * sizeof(PeerDst), cudaMemcpyHostToDevice, s));
    if (!push.empty()) CK(cudaMemcpyAsync(R->d_push, push.data(), push.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
    if (!ranks.empty()) {
        CK(cudaMemcpyAsync(R->d_peer_ranks, ranks.data(), ranks.size() * sizeof(int), cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(R->d_peer_slots, slots.data(), slots.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    }
    CK(cudaStreamSynchronize(s));
    R->p2p = true;
    return VOL_OK;
}

static vol_status connect_peer_impl(vol_s *v, int peer, char *peer_ws, const int64_t *info, int64_t n) {
    if (!v || !v->shard) return fail(VOL_EINVAL, "vol_connect_peer: not a sharded volume");
    ShardRuntime *R = v->shard;
    const ShardPlan &P = R->plan;
    if (peer < 0 || peer >= P.world || peer == P.rank || !peer_ws || !info)
        return fail(VOL_EINVAL, "vol_connect_peer: bad peer %d", peer);
    if (n != kPeerInfoFixed + P.world + kPeerInfoOffsets || info[0] != 1 || info[1] != peer || info[2] != P.world ||
        info[5] != n)
        return fail(VOL_EINVAL, "vol_connect_peer: peer info does not match (rank %d of %d)", peer, P.world);
    if (std::find(R->peers.begin(), R->peers.end(), peer) == R->peers.end()) return VOL_OK;   // no halo with it
    if (R->peer_slot[peer] < 0) {
        R->peer_slot[peer] = (int64_t)R->peer_out.size();
        R->peer_out.push_back(PeerOut{});
        R->peer_info.emplace_back();
    }
    const int64_t slot = R->peer_slot[peer];
    R->peer_info[slot].assign(info, info + n);
    const int64_t *off = info + kPeerInfoFixed + P.world;
    PeerOut &Q = R->peer_out[slot];
    Q.u[0] = (float *)(peer_ws + off[0]);
    Q.u[1] = (float *)(peer_ws + off[1]);
    Q.ub[0] = (float *)(peer_ws + off[2]);
    Q.ub[1] = (float *)(peer_ws + off[3]);
    Q.px[0] = (float *)(peer_ws + off[4]);
    Q.px[1] = (float *)(peer_ws + off[5]);
    Q.py[0] = (float *)(peer_ws + off[6]);
    Q.py[1] = (float *)(peer_ws + off[7]);
    Q.pz[0] = (float *)(peer_ws + off[8]);
    Q.pz[1] = (float *)(peer_ws + off[9]);
    Q.flags = (unsigned long long *)(peer_ws + off[10]);
    for (int q : R->peers)
        if (R->peer_slot[q] < 0) return VOL_OK;   // more peers to come
    return p2p_finalize(v);
}

extern "C" vol_status vol_connect_peer(vol_t v, int peer, void *peer_workspace, const int64_t *info, int64_t n) {
    return connect_peer_impl(v, peer, (char *)peer_workspace, info, n);
}

extern "C" vol_status vol_ipc_handle(vol_t v, void *handle64, int64_t *offset) {
    if (!v || !handle64 || !offset) return fail(VOL_EINVAL, "vol_ipc_handle: NULL argument");
    static PFN_cuMemGetAddressRange_v3020 range = nullptr;
    if (!range) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", (void **)&range, cudaEnableDefault, &q) != cudaSuccess || !range)
            return fail(VOL_ENOTSUP, "vol_ipc_handle: cuMemGetAddressRange unavailable");
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)v->ws) != CUDA_SUCCESS) return fail(VOL_ECUDA, "vol_ipc_handle: address range");
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, (void *)base));
    memcpy(handle64, &h, sizeof h);
    *offset = (int64_t)((char *)v->ws - (char *)base);
    return VOL_OK;
}

extern "C" vol_status vol_connect_peer_ipc(vol_t v, int peer, const void *handle64, int64_t offset, const int64_t *info,
                                          int64_t n) {
    if (!v || !v->shard || !handle64) return fail(VOL_EINVAL, "vol_connect_peer_ipc: NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof h);
    void *base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    v->shard->peer_ipc.push_back(base);
    return connect_peer_impl(v, peer, (char *)base + offset, info, n);
}

extern "C" int vol_transport(vol_t v) {
    if (!v || !v->shard) return 0;
    if (v->shard->p2p) return 3;
    return v->shard->nccl ? 1 : 2;
}

// ------------------------------------------------------------------------- loopback transport

static vol_status loopback_exchange(vol_t *h, int world, cudaStream_t s) {
    for (int r = 0; r < world; r++) {
        const ShardPlan &Pr = h[r]->shard->plan;
        for (int q = 0; q < world; q++) {
            if (q == r || Pr.send_cnt[q] == 0) continue;
            const ShardPlan &Pq = h[q]->shard->plan;
            if (Pq.recv_cnt[r] != Pr.send_cnt[q])
                return fail(VOL_EINVAL, "loopback: rank %d sends %lld blocks to %d, which expects %lld", r,
                            (long long)Pr.send_cnt[q], q, (long long)Pq.recv_cnt[r]);
            CK(cudaMemcpyAsync(h[q]->shard->recvbuf + Pq.recv_off[r] * kMsgFloats,
                               h[r]->shard->sendbuf + Pr.send_off[q] * kMsgFloats,
                               (size_t)Pr.send_cnt[q] * kMsgFloats * 4, cudaMemcpyDeviceToDevice, s));
        }
    }
    return VOL_OK;
}

static vol_status check_group(vol_t *h, int world) {
    if (!h || world < 2) return fail(VOL_EINVAL, "group: need >= 2 handles");
    for (int r = 0; r < world; r++) {
        if (!h[r] || !h[r]->shard) return fail(VOL_EINVAL, "group: handle %d is not sharded", r);
        if (h[r]->shard->nccl) return fail(VOL_EINVAL, "group: handle %d uses NCCL", r);
        if (h[r]->shard->plan.rank != r || h[r]->shard->plan.world != world)
            return fail(VOL_EINVAL, "group: handle %d has rank %d of %d", r, h[r]->shard->plan.rank,
                        h[r]->shard->plan.world);
    }
    return VOL_OK;
}

extern "C" vol_status vol_group_connect(vol_t *h, int world) {
    vol_status st = check_group(h, world);
    if (st != VOL_OK) return st;
    cudaStream_t s = h[0]->stream;
    for (int r = 0; r < world; r++) CK(cudaStreamSynchronize(h[r]->stream));
    for (int r = 0; r < world; r++) {
        float *W = const_cast<float *>(h[r]->F.W), *f = const_cast<float *>(h[r]->F.f);
        if ((st = pack(h[r], W, f, W, f, s)) != VOL_OK) return st;
    }
    if ((st = loopback_exchange(h, world, s)) != VOL_OK) return st;
    int64_t tot = 0;
    for (int r = 0; r < world; r++) {
        float *W = const_cast<float *>(h[r]->F.W), *f = const_cast<float *>(h[r]->F.f);
        if ((st = unpack(h[r], W, f, h[r]->F.ub[0], h[r]->F.ub[1], s)) != VOL_OK) return st;
        CKL(launch_init_state(h[r]->F, h[r]->L.S * kBlockVox, 0, s));
        tot += h[r]->n_omega_local;
    }
    CK(cudaStreamSynchronize(s));
    for (int r = 0; r < world; r++) {
        h[r]->n_omega_global = tot;
        h[r]->shard->connected = true;
        h[r]->cur = 0;
        if ((st = finalize_w8(h[r])) != VOL_OK) return st;
    }
    return VOL_OK;
}

extern "C" vol_status vol_regularise_group(vol_t *h, int world, float lambda, float eps, float tau, float sigma,
                                           int32_t iters, const vol_opts *opts) {
    NvtxRange nvtx_range_("vol_regularise_group");
    vol_status st = check_group(h, world);
    if (st != VOL_OK) return st;
    for (int r = 0; r < world; r++)
        if (!h[r]->shard->connected) return fail(VOL_EINVAL, "group: call vol_group_connect first");
    // parameter validation + initialisation through the single-handle entry with iters = 0
    for (int r = 0; r < world; r++)
        if ((st = vol_regularise_prepare(h[r], lambda, eps, tau, sigma, iters, opts)) != VOL_OK) return st;
    IterParams P = h[0]->pending;
    cudaStream_t s = h[0]->stream;
    for (int r = 1; r < world; r++) CK(cudaStreamSynchronize(h[r]->stream));
    int64_t launches = 0;
    bool all_p2p = true;
    for (int r = 0; r < world; r++) all_p2p = all_p2p && h[r]->shard->p2p;
    if ((h[0]->pending_kernel == 0 || h[0]->pending_kernel == 2) && iters > 0 && all_p2p && h[0]->pending_exchange) {
        // the direct-store transport, as p2p_skew, every stage issued for all shards before the next stage
        // (one stream: every wait finds its peers' signals already counted)
        const int c = h[0]->cur;
        float *Bu[64][2];
        if (world > 64) return fail(VOL_EINVAL, "group: at most 64 loopback shards");
        for (int r = 0; r < world; r++) {
            CK(cudaMemcpyAsync(h[r]->d_u2, h[r]->F.u, (size_t)h[r]->L.S * kBlockVox * 4, cudaMemcpyDeviceToDevice, s));
            Bu[r][(iters - 1) & 1] = h[r]->F.u;
            Bu[r][iters & 1] = h[r]->d_u2;
        }
        auto all = [&](auto fn) -> vol_status {
            for (int r = 0; r < world; r++) {
                const int n = fn(r);
                CKL(n);
                launches += n;
            }
            return VOL_OK;
        };
        auto sig = [&](int r) { return p2p_signal(h[r], s); };
        auto wt = [&](int r) { return p2p_wait(h[r], s); };
        if ((st = all(sig)) != VOL_OK || (st = all(wt)) != VOL_OK) return st;   // ready
        if ((st = all([&](int r) { return p2p_push(h[r], h[r]->F.ub[c], 2 + c, c, s); })) != VOL_OK ||
            (st = all(sig)) != VOL_OK || (st = all(wt)) != VOL_OK)
            return st;
        if ((st = all([&](int r) {
                 return launch_dual_only(view_of(h[r]->F, c), h[r]->d_nbr, h[r]->shard->plan.n_local(), P, s);
             })) != VOL_OK)
            return st;
        if ((st = all([&](int r) {
                 return p2p_push(h[r], Bu[r][0], Bu[r][0] == h[r]->F.u ? 0 : 1, c ^ 1, s);
             })) != VOL_OK ||
            (st = all(sig)) != VOL_OK)
            return st;
        for (int j = 0; j < iters - 1; j++) {
            const int pin = c ^ ((j + 1) & 1);
            if ((st = all([&](int r) {
                     return launch_skew(h[r]->F, Bu[r][j & 1], Bu[r][(j + 1) & 1], pin, h[r]->pending_frozen,
                                        h[r]->d_nbr, 0, h[r]->shard->plan.nA, P, s);
                 })) != VOL_OK ||
                (st = all(wt)) != VOL_OK)
                return st;
            if ((st = all([&](int r) {
                     const ShardPlan &SP = h[r]->shard->plan;
                     return launch_skew_peers(h[r]->F, Bu[r][j & 1], Bu[r][(j + 1) & 1], pin, h[r]->pending_frozen,
                                              h[r]->d_nbr, SP.nA, SP.n_local() - SP.nA, P, h[r]->shard->d_peers,
                                              h[r]->shard->d_dst, s);
                 })) != VOL_OK ||
                (st = all(sig)) != VOL_OK)
                return st;
        }
        if ((st = all(wt)) != VOL_OK) return st;
        const int c2 = c ^ (iters & 1);
        if ((st = all([&](int r) {
                 View V = view_of(h[r]->F, c2 ^ 1);
                 V.u = Bu[r][(iters - 1) & 1];
                 return launch_primal_only(V, h[r]->d_nbr, h[r]->shard->plan.n_local(), P, s);
             })) != VOL_OK)
            return st;
        for (int r = 0; r < world; r++) h[r]->cur = c2;
        CK(cudaStreamSynchronize(s));
        for (int r = 0; r < world; r++) {
            h[r]->last_launches = launches;
            unsigned long long err = 0;
            CK(cudaMemcpy(&err, h[r]->shard->expect + world, 8, cudaMemcpyDeviceToHost));
            if (err) return fail(VOL_ECUDA, "peer transport: shard %d waited for a peer that never signalled", r);
        }
        return VOL_OK;
    }
    if ((h[0]->pending_kernel == 0 || h[0]->pending_kernel == 2) && iters > 0) {   // skewed, as nccl_skew
        const int c = h[0]->cur;
        float *Bu[64][2];
        if (world > 64) return fail(VOL_EINVAL, "group: at most 64 loopback shards");
        auto X = [&](auto field_of) -> vol_status {
            vol_status st2;
            for (int r = 0; r < world; r++) {
                float *f4[4];
                field_of(r, f4);
                if ((st2 = pack(h[r], f4[0], f4[1], f4[2], f4[3], s)) != VOL_OK) return st2;
            }
            if ((st2 = loopback_exchange(h, world, s)) != VOL_OK) return st2;
            for (int r = 0; r < world; r++) {
                float *f4[4];
                field_of(r, f4);
                if ((st2 = unpack(h[r], f4[0], f4[1], f4[2], f4[3], s)) != VOL_OK) return st2;
            }
            launches += 2 * world;
            return VOL_OK;
        };
        for (int r = 0; r < world; r++) {
            CK(cudaMemcpyAsync(h[r]->d_u2, h[r]->F.u, (size_t)h[r]->L.S * kBlockVox * 4, cudaMemcpyDeviceToDevice, s));
            Bu[r][(iters - 1) & 1] = h[r]->F.u;
            Bu[r][iters & 1] = h[r]->d_u2;
        }
        if ((st = X([&](int r, float **f4) {
                 f4[0] = h[r]->F.ub[c], f4[1] = h[r]->F.px[c], f4[2] = h[r]->F.py[c], f4[3] = h[r]->F.pz[c];
             })) != VOL_OK)
            return st;
        for (int r = 0; r < world; r++) {
            int a = launch_dual_only(view_of(h[r]->F, c), h[r]->d_nbr, h[r]->shard->plan.n_local(), P, s);
            CKL(a);
            launches += a;
        }
        for (int j = 0; j < iters - 1; j++) {
            const int pin = c ^ ((j + 1) & 1);
            if ((st = X([&](int r, float **f4) {
                     f4[0] = Bu[r][j & 1], f4[1] = h[r]->F.px[pin], f4[2] = h[r]->F.py[pin], f4[3] = h[r]->F.pz[pin];
                 })) != VOL_OK)
                return st;
            for (int r = 0; r < world; r++) {
                const ShardPlan &SP = h[r]->shard->plan;
                const int64_t nl = SP.n_local(), nA = SP.nA;
                int a = launch_skew(h[r]->F, Bu[r][j & 1], Bu[r][(j + 1) & 1], pin, h[r]->pending_frozen, h[r]->d_nbr,
                                    0, nA, P, s);
                CKL(a);
                int b = launch_skew(h[r]->F, Bu[r][j & 1], Bu[r][(j + 1) & 1], pin, h[r]->pending_frozen, h[r]->d_nbr,
                                    nA, nl - nA, P, s);
                CKL(b);
                launches += a + b;
            }
        }
        const int c2 = c ^ (iters & 1);
        if ((st = X([&](int r, float **f4) {
                 f4[0] = h[r]->F.ub[c2], f4[1] = h[r]->F.px[c2], f4[2] = h[r]->F.py[c2], f4[3] = h[r]->F.pz[c2];
             })) != VOL_OK)
            return st;
        for (int r = 0; r < world; r++) {
            View V = view_of(h[r]->F, c2 ^ 1);
            V.u = Bu[r][(iters - 1) & 1];
            int a = launch_primal_only(V, h[r]->d_nbr, h[r]->shard->plan.n_local(), P, s);
            CKL(a);
            launches += a;
            h[r]->cur = c2;
        }
        CK(cudaStreamSynchronize(s));
        for (int r = 0; r < world; r++) h[r]->last_launches = launches;
        return VOL_OK;
    }
    for (int32_t k = 0; k < iters; k++) {
        const int cur = h[0]->cur;
        for (int r = 0; r < world; r++)
            if ((st = pack(h[r], h[r]->F.ub[cur], h[r]->F.px[cur], h[r]->F.py[cur], h[r]->F.pz[cur], s)) != VOL_OK)
                return st;
        if ((st = loopback_exchange(h, world, s)) != VOL_OK) return st;
        for (int r = 0; r < world; r++) {
            ShardRuntime *R = h[r]->shard;
            if ((st = unpack(h[r], h[r]->F.ub[cur], h[r]->F.px[cur], h[r]->F.py[cur], h[r]->F.pz[cur], s)) != VOL_OK)
                return st;
            View V = view_of(h[r]->F, cur);
            V.frozen = h[r]->pending_frozen;
            int a = launch_fused(V, h[r]->d_nbr, nullptr, 0, R->plan.nA, P, s);
            CKL(a);
            int b = launch_fused(V, h[r]->d_nbr, nullptr, R->plan.nA, R->plan.n_local() - R->plan.nA, P, s);
            CKL(b);
            launches += a + b + 2;
        }
        for (int r = 0; r < world; r++) h[r]->cur ^= 1;
    }
    CK(cudaStreamSynchronize(s));
    for (int r = 0; r < world; r++) h[r]->last_launches = launches;
    return VOL_OK;
}

// Energy of a loopback group: refresh ghost u/p, local partial sums, combined on the host.
extern "C" vol_status vol_group_energy(vol_t *h, int world, float lambda, float eps, int data_term, double *primal,
                                       double *dual) {
    vol_status st = check_group(h, world);
    if (st != VOL_OK) return st;
    if (!primal) return fail(VOL_EINVAL, "vol_group_energy: primal is NULL");
    cudaStream_t s = h[0]->stream;
    for (int r = 0; r < world; r++) {
        const int c = h[r]->cur;
        if ((st = pack(h[r], h[r]->F.u, h[r]->F.px[c], h[r]->F.py[c], h[r]->F.pz[c], s)) != VOL_OK) return st;
    }
    if ((st = loopback_exchange(h, world, s)) != VOL_OK) return st;
    double acc[5] = {0, 0, 0, 0, 1.0};
    for (int r = 0; r < world; r++) {
        const int c = h[r]->cur;
        if ((st = unpack(h[r], h[r]->F.u, h[r]->F.px[c], h[r]->F.py[c], h[r]->F.pz[c], s)) != VOL_OK) return st;
        CKL(launch_energy(view_of(h[r]->F, c), h[r]->d_nbr, nullptr, h[r]->L.n_local, lambda, eps, data_term, h[r]->d_part,
                          h[r]->d_eout, s));
        double o[5];
        CK(cudaMemcpyAsync(o, h[r]->d_eout, sizeof o, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int k = 0; k < 4; k++) acc[k] += o[k];
        acc[4] = std::min(acc[4], o[4]);
    }
    *primal = acc[0];
    if (dual) *dual = energy_dual_value(acc, eps, data_term);
    return VOL_OK;
}
