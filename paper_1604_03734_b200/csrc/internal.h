// internal.h — shared declarations of the libvol CUDA implementation (not part of the C ABI).
//
// Layout in HBM: structure of arrays, one float32 field per quantity,
// [S][512] with S = local + ghost blocks ("store order" = the caller's block order, ghosts last),
// voxel index x + 8y + 64z inside a block.  Each 8^3 block of one field is a contiguous,
// 256 B-aligned 2 KiB run: one TMA bulk copy per field per block, 128 contiguous bytes per warp load.
// ū and p are double-buffered (in = [cur], out = [cur ^ 1]) so a launch only reads values that no
// CTA of the same launch writes.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace hvg {

// Process-wide count of kernels this library has launched (graph replays count every node).
extern std::atomic<long long> g_launches;
inline int counted(int r) {
    if (r > 0) g_launches.fetch_add(r, std::memory_order_relaxed);
    return r;
}

constexpr int kBlockVox = 512;     // 8^3 voxels per block
constexpr int kThreads = 128;      // CTA size of the per-block kernels: 4 voxels per thread
constexpr int kNbr = 12;           // 6 face neighbours (−x,+x,−y,+y,−z,+z) + 6 edge (diagonal) neighbours
// Edge neighbours read by the −face halo recompute, as block-coordinate offsets (iterate.cu):
//   6: (−1,+1,0)  7: (−1,0,+1)  8: (+1,−1,0)  9: (0,−1,+1)  10: (+1,0,−1)  11: (0,+1,−1)

struct Fields {
    const float *f;        // fused TSDF (read only)
    const float *W;        // fusion weight (read only), Ω ⇔ W > 0
    const uint8_t *W8;     // W as exact 8-bit counts when every W is an integer in [0, 255], else null
    float *u;              // primal u (in place: only its own CTA touches a voxel's u)
    float *ub[2];          // relaxed primal ū, double-buffered
    float *px[2], *py[2], *pz[2];  // dual p, double-buffered
    float *u2 = nullptr;           // second u buffer of the skewed schedule
};

// The buffers of one iteration, selected on the host (no dynamic indexing in kernels).
struct View {
    const float *f, *W;
    const uint8_t *W8;
    const uint32_t *frozen;   // [rows][16] bit per voxel: primal step is the identity this call (or null)
    float *u;
    const float *ub_in;
    float *ub_out;
    const float *px_in, *py_in, *pz_in;
    float *px_out, *py_out, *pz_out;
};

inline View view_of(const Fields &F, int cur) {
    const int o = cur ^ 1;
    return View{F.f, F.W, F.W8, nullptr, F.u, F.ub[cur], F.ub[o], F.px[cur], F.py[cur], F.pz[cur], F.px[o], F.py[o],
                F.pz[o]};
}

struct IterParams {
    float sigma;     // σ
    float tau;       // τ
    float tl;        // fl(τ·λ) (data-term threshold per unit weight)
    float theta;     // θ
    float kappa;     // fl(1 / fl(1 + σ·ε)) (Huber damping factor, reading c-18)
    int data_term;   // 0 L1, 1 L2
    float one;       // 1.0f, as a runtime value: the paired sums a + b = fma(a, one, b) (see iterate.cu)
};

// Iteration launchers (return the number of kernel launches, or -1 on a launch error).
// work == nullptr means blocks 0 .. n_work-1.
// Fused iteration over work items [first, first + n_work) (work == nullptr: store rows).
int launch_fused(const View &V, const int32_t *nbr, const int32_t *work, int64_t first, int64_t n_work,
                 const IterParams &P, cudaStream_t s);
// The two halves of the two-kernel baseline on their own (the skewed schedule's prologue / epilogue):
// k_dual reads ū_in, p_in, W and writes p_out; k_primal reads p_out (p^{k+1}), u, f, W and writes u, ū_out.
int launch_dual_only(const View &V, const int32_t *nbr, int64_t n_work, const IterParams &P, cudaStream_t s);
int launch_primal_only(const View &V, const int32_t *nbr, int64_t n_work, const IterParams &P, cudaStream_t s);
// Skewed schedule (iterate.cu): one launch = primal step k + dual step k+1 of store rows
// [first, first + n_blocks); reads u_in and p[p_in] (p^{k+1}), writes u_out and p[p_in ^ 1] (p^{k+2}).
int launch_skew(const Fields &F, const float *u_in, float *u_out, int p_in, const uint32_t *frozen,
                const int32_t *nbr, int64_t first, int64_t n_blocks, const IterParams &P, cudaStream_t s);
// The single-GPU loop's launch of all rows: launch_skew, or with HVG_SKEW_PDL (off: measured ±0)
// the programmatic-dependent-launch form whose static prologue overlaps the previous launch's tail.
int launch_skew_loop(const Fields &F, const float *u_in, float *u_out, int p_in, const uint32_t *frozen,
                    const int32_t *nbr, int64_t n_blocks, const IterParams &P, cudaStream_t s);
// The same launch for the boundary rows of a peer-connected shard: every output of a row is also stored
// into its peer destinations (peer.cuh), followed by a system-scope fence.
struct PeerOut;
struct PeerDst;
int launch_skew_peers(const Fields &F, const float *u_in, float *u_out, int p_in, const uint32_t *frozen,
                      const int32_t *nbr, int64_t first, int64_t n_blocks, const IterParams &P, const PeerOut *peers,
                      const PeerDst *dst, cudaStream_t s);
int launch_two_kernel(const View &V, const int32_t *nbr, const int32_t *work, int64_t n_work, const IterParams &P,
                      cudaStream_t s);

// store build
int launch_hash_count(const int32_t *xyz, int64_t n, uint32_t T, uint32_t *hash, uint32_t *count,
                      cudaStream_t s);
int launch_exclusive_scan_u32(const uint32_t *in, uint32_t *out, int64_t n, uint32_t *scratch,
                              cudaStream_t s);
int launch_bucket_fill(const uint32_t *hash, int64_t n, uint32_t *cursor, int32_t *entry, cudaStream_t s);
int launch_bucket_sort_and_dups(const int32_t *xyz, const uint32_t *start, int32_t *entry, uint32_t T,
                                int64_t n, unsigned long long *dup, cudaStream_t s);
int launch_neighbours(const int32_t *xyz, int64_t n, const uint32_t *start, const int32_t *entry, uint32_t T,
                      const int32_t *store_of_global, const int64_t *rows, int64_t n_rows, int32_t *nbr,
                      cudaStream_t s);
int launch_validate(const float *f, const float *W, int64_t nvox, unsigned long long *bad,
                    unsigned long long *n_omega, cudaStream_t s);
int launch_init_state(const Fields &F, int64_t nvox, int init, cudaStream_t s);
// frozen: 64 bytes per row, byte c (column c = x + 8y) bit z set iff voxel c + 64z has an identity primal step
// for this call (L1 only)
int launch_freeze_mask(const Fields &F, int cur, const IterParams &P, int64_t n_blocks, uint32_t *frozen,
                       cudaStream_t s);
// W8[i] = W[i] for W integer in [0, 255]; *bad = 1 if some W is not (W8 then unusable)
int launch_pack_w8(const float *W, uint8_t *W8, int64_t nvox, unsigned *bad, cudaStream_t s);
// gather: dst[r] = src[perm[r]] (caller → store order); scatter: dst[perm[r]] = src[r] (store → caller)
int launch_permute_blocks(const float *src, float *dst, const int32_t *perm, int64_t n, bool gather, cudaStream_t s);
// W given as 8-bit counts [n][512] in caller order → fp32 W in store order (gather by perm)
int launch_permute_w8_to_f32(const uint8_t *src, float *dst, const int32_t *perm, int64_t n, cudaStream_t s);
int launch_sanitize_state(const Fields &F, int cur, const int32_t *nbr, int64_t n_blocks, cudaStream_t s);

// energy: per-block partial sums, then one deterministic final reduction into out[5]
int launch_energy(const View &V, const int32_t *nbr, const int32_t *blocks, int64_t n_blocks, float lam,
                  float eps, int data_term, double *partials, double *out, cudaStream_t s);

// single-GPU store order on the device (order.cu): perm[r] = caller index of store row r (Morton order of the
// coordinates relative to their bounding box, ties in caller order); *bad = lowest block index with a
// coordinate outside (−2^30, 2^30) (*bad must be preset to ~0).  scratch: morton_order_scratch_bytes(n).
size_t morton_order_scratch_bytes(int64_t n);
int launch_morton_order(const int32_t *xyz, int64_t n, void *scratch, int32_t *perm, unsigned long long *bad,
                        cudaStream_t s);
// store_of_global[perm[r]] = r, rows[r] = perm[r]
int launch_row_maps(const int32_t *perm, int64_t n, int32_t *sog, int64_t *rows, cudaStream_t s);

// order-independent 64-bit digest of n block coordinates ([n][3] int32), the same value on host and device
unsigned long long coord_digest_host(const int32_t *xyz, int64_t n);
// (computed on stream s, returns when done)
bool coord_digest_device(const int32_t *xyz, int64_t n, unsigned long long *out, cudaStream_t s);

uint32_t host_hash(int32_t x, int32_t y, int32_t z, uint32_t T);

}  // namespace hvg
