// internal.h — shared declarations of the libvol CUDA implementation (not part of the C ABI).
//
// Layout in HBM: structure of arrays, one float32 field per quantity,
// [S][512] with S = local + ghost blocks ("store order" = the caller's block order, ghosts last),
// voxel index x + 8y + 64z inside a block.  Each 8^3 block of one field is a contiguous,
// 2 KiB-aligned run, so one warp reads 128 contiguous bytes per instruction.
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
constexpr int kVoxPerThread = 4;

// Work-item modes of the fused kernel (SURVEY §8(e) two-launch schedule).
enum : uint8_t { MODE_FULL = 0, MODE_DUAL = 1, MODE_PRIMAL = 2 };

struct Fields {
    const float *f;       // fused TSDF (read only)
    const float *W;       // fusion weight (read only), Ω ⇔ W > 0
    float *u;             // primal u
    float *ub[2];         // relaxed primal ū, ping-pong (in = ub[cur], out = ub[cur ^ 1])
    float *px, *py, *pz;  // dual p, in place
};

struct IterParams {
    float sigma;     // σ
    float tau;       // τ
    float tl;        // fl(τ·λ) (data-term threshold per unit weight)
    float theta;     // θ
    float denom;     // fl(1 + σ·ε) (Huber damping divisor)
    int data_term;   // 0 L1, 1 L2
};

// Launchers (return the number of kernel launches issued, or -1 on a launch error).
int launch_fused(const Fields &F, int cur, const int32_t *nbr, const int32_t *work, const uint8_t *mode,
                 int64_t n_work, uint32_t *flags, uint32_t *ticket, const IterParams &P, cudaStream_t s);
int launch_two_kernel(const Fields &F, int cur, const int32_t *nbr, const int32_t *work, int64_t n_work,
                      const IterParams &P, cudaStream_t s);

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
int launch_sanitize_state(const Fields &F, int cur, const int32_t *nbr, int64_t n_blocks, cudaStream_t s);

// energy: per-block partial sums, then one deterministic final reduction into out[5]
int launch_energy(const Fields &F, const int32_t *nbr, const int32_t *blocks, int64_t n_blocks, float lam,
                  float eps, int data_term, double *partials, double *out, cudaStream_t s);

uint32_t host_hash(int32_t x, int32_t y, int32_t z, uint32_t T);

}  // namespace hvg
