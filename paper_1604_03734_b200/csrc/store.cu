// store.cu — device build of the hashed voxel-block store (K1, K2, K3).
//
// "The HVG subdivides the world into an infinite, uniform grid of voxel blocks ... Applying
// a hash function to coordinates in world space gives an index within the hash table".  The hash is
// the Teschner spatial hash of S:56 evaluated in uint32 wrap-around arithmetic (reading c-14):
//     h(x, y, z) = ((u32)x·73856093 ⊕ (u32)y·19349669 ⊕ (u32)z·83492791) mod T,  T = 2^k >= 2n.
// The table is a CSR bucket array: bucket_start[T+1] (exclusive scan of bucket counts) and
// bucket_entry[n] holding caller indices in ascending order inside each bucket.  The order inside a
// bucket is fixed by a per-bucket sort after an atomic scatter, so the table is bit-identical on
// every run (and to the oracle's counting sort).  The 6-neighbour table (−x,+x,−y,+y,−z,+z) is one
// lookup per (block, direction) (block boundary conditions come from the neighbours).
#include <math.h>

#include "internal.h"

namespace hvg {

__host__ __device__ __forceinline__ uint32_t hash3(int32_t x, int32_t y, int32_t z, uint32_t T) {
    uint32_t hx = (uint32_t)x * 73856093u;
    uint32_t hy = (uint32_t)y * 19349669u;
    uint32_t hz = (uint32_t)z * 83492791u;
    return (hx ^ hy ^ hz) % T;
}

uint32_t host_hash(int32_t x, int32_t y, int32_t z, uint32_t T) { return hash3(x, y, z, T); }

static inline unsigned grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    return (unsigned)(g < 1 ? 1 : g);
}

__global__ void k_hash_count(const int32_t *__restrict__ xyz, int64_t n, uint32_t T, uint32_t *__restrict__ hash,
                             uint32_t *__restrict__ count) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t h = hash3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], T);
    hash[i] = h;
    atomicAdd(&count[h], 1u);
}

int launch_hash_count(const int32_t *xyz, int64_t n, uint32_t T, uint32_t *hash, uint32_t *count, cudaStream_t s) {
    if (n == 0) return 0;
    k_hash_count<<<grid_for(n, 256), 256, 0, s>>>(xyz, n, T, hash, count);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// ---------------------------------------------------------------- exclusive scan of uint32 counts
constexpr int kScanThreads = 1024;
constexpr int kScanChunk = 4 * kScanThreads;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t *smem_warp, uint32_t *total) {
    // warp inclusive scan
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) smem_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        uint32_t w = lane < (int)(blockDim.x >> 5) ? smem_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        smem_warp[lane] = w;  // inclusive warp totals
    }
    __syncthreads();
    uint32_t base = wid > 0 ? smem_warp[wid - 1] : 0u;
    if (total) *total = smem_warp[(blockDim.x >> 5) - 1];
    uint32_t r = base + x - v;
    __syncthreads();
    return r;
}

__global__ void k_chunk_sums(const uint32_t *__restrict__ in, int64_t n, uint32_t *__restrict__ sums) {
    __shared__ uint32_t sw[32];
    int64_t base = (int64_t)blockIdx.x * kScanChunk;
    uint32_t acc = 0;
    for (int k = 0; k < 4; k++) {
        int64_t i = base + (int64_t)threadIdx.x * 4 + k;
        if (i < n) acc += in[i];
    }
    uint32_t tot;
    block_exclusive_scan(acc, sw, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void k_scan_sums(uint32_t *sums, int64_t m) {
    // single CTA: exclusive scan of m chunk sums in place, sums[m] = total
    __shared__ uint32_t sw[32];
    int64_t per = (m + blockDim.x - 1) / blockDim.x;
    int64_t lo = threadIdx.x * per, hi = lo + per < m ? lo + per : m;
    uint32_t acc = 0;
    for (int64_t i = lo; i < hi; i++) acc += sums[i];
    uint32_t tot;
    uint32_t off = block_exclusive_scan(acc, sw, &tot);
    for (int64_t i = lo; i < hi; i++) {
        uint32_t v = sums[i];
        sums[i] = off;
        off += v;
    }
    if (threadIdx.x == 0) sums[m] = tot;
}

__global__ void k_chunk_scan(const uint32_t *__restrict__ in, int64_t n, const uint32_t *__restrict__ sums,
                             uint32_t *__restrict__ out) {
    __shared__ uint32_t sw[32];
    int64_t base = (int64_t)blockIdx.x * kScanChunk + (int64_t)threadIdx.x * 4;
    uint32_t v[4];
    uint32_t acc = 0;
    for (int k = 0; k < 4; k++) {
        v[k] = base + k < n ? in[base + k] : 0u;
        acc += v[k];
    }
    uint32_t off = block_exclusive_scan(acc, sw, nullptr) + sums[blockIdx.x];
    for (int k = 0; k < 4; k++) {
        if (base + k < n) out[base + k] = off;
        off += v[k];
    }
}

__global__ void k_write_total(const uint32_t *sums, int64_t m, int64_t n, uint32_t *out) { out[n] = sums[m]; }

// out[0..n] = exclusive scan of in[0..n), out[n] = total; scratch needs n/kScanChunk + 2 entries.
int launch_exclusive_scan_u32(const uint32_t *in, uint32_t *out, int64_t n, uint32_t *scratch, cudaStream_t s) {
    int64_t m = (n + kScanChunk - 1) / kScanChunk;
    if (m < 1) m = 1;
    k_chunk_sums<<<(unsigned)m, kScanThreads, 0, s>>>(in, n, scratch);
    k_scan_sums<<<1, kScanThreads, 0, s>>>(scratch, m);
    k_chunk_scan<<<(unsigned)m, kScanThreads, 0, s>>>(in, n, scratch, out);
    k_write_total<<<1, 1, 0, s>>>(scratch, m, n, out);
    return cudaPeekAtLastError() == cudaSuccess ? counted(4) : -1;
}

__global__ void k_bucket_fill(const uint32_t *__restrict__ hash, int64_t n, uint32_t *__restrict__ cursor,
                              int32_t *__restrict__ entry) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t pos = atomicAdd(&cursor[hash[i]], 1u);
    entry[pos] = (int32_t)i;
}

int launch_bucket_fill(const uint32_t *hash, int64_t n, uint32_t *cursor, int32_t *entry, cudaStream_t s) {
    if (n == 0) return 0;
    k_bucket_fill<<<grid_for(n, 256), 256, 0, s>>>(hash, n, cursor, entry);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// One thread per bucket: insertion sort of its caller indices (buckets hold ~0.5 entries on average
// at T >= 2n), then the duplicate check ("No duplicate block_coords keys"): the smallest caller
// index i repeating an earlier j is reported as (i << 32 | j) through atomicMin.
__global__ void k_bucket_sort_dups(const int32_t *__restrict__ xyz, const uint32_t *__restrict__ start,
                                   int32_t *__restrict__ entry, uint32_t T, unsigned long long *dup) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= T) return;
    uint32_t lo = start[b], hi = start[b + 1];
    for (uint32_t k = lo + 1; k < hi; k++) {
        int32_t key = entry[k];
        uint32_t j = k;
        while (j > lo && entry[j - 1] > key) {
            entry[j] = entry[j - 1];
            j--;
        }
        entry[j] = key;
    }
    for (uint32_t k = lo + 1; k < hi; k++) {
        int32_t i = entry[k];
        for (uint32_t m = lo; m < k; m++) {
            int32_t j = entry[m];
            if (xyz[3 * j] == xyz[3 * i] && xyz[3 * j + 1] == xyz[3 * i + 1] && xyz[3 * j + 2] == xyz[3 * i + 2]) {
                atomicMin(dup, ((unsigned long long)(uint32_t)i << 32) | (uint32_t)j);
                break;
            }
        }
    }
}

int launch_bucket_sort_and_dups(const int32_t *xyz, const uint32_t *start, int32_t *entry, uint32_t T, int64_t n,
                                unsigned long long *dup, cudaStream_t s) {
    (void)n;
    k_bucket_sort_dups<<<grid_for(T, 256), 256, 0, s>>>(xyz, start, entry, T, dup);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// nbr[12r + d] for store row r (global block index rows[r], or r itself when rows == NULL): the store
// index of the neighbour at offset d — faces (−x,+x,−y,+y,−z,+z), then the six edge neighbours of
// internal.h — or −1 if unallocated (Ω̄) or not held by this rank.
__constant__ int8_t c_nbr_off[kNbr][3] = {{-1, 0, 0}, {1, 0, 0},  {0, -1, 0}, {0, 1, 0},  {0, 0, -1}, {0, 0, 1},
                                          {-1, 1, 0}, {-1, 0, 1}, {1, -1, 0}, {0, -1, 1}, {1, 0, -1}, {0, 1, -1}};

__global__ void k_neighbours(const int32_t *__restrict__ xyz, const uint32_t *__restrict__ start,
                             const int32_t *__restrict__ entry, uint32_t T, const int32_t *__restrict__ store_of_global,
                             const int64_t *__restrict__ rows, int64_t n_rows, int32_t *__restrict__ nbr) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= kNbr * n_rows) return;
    int64_t r = k / kNbr;
    int d = (int)(k % kNbr);
    int64_t g = rows ? rows[r] : r;
    int32_t q[3] = {xyz[3 * g] + c_nbr_off[d][0], xyz[3 * g + 1] + c_nbr_off[d][1], xyz[3 * g + 2] + c_nbr_off[d][2]};
    uint32_t h = hash3(q[0], q[1], q[2], T);
    int32_t found = -1;
    for (uint32_t m = start[h]; m < start[h + 1]; m++) {
        int32_t j = entry[m];
        if (xyz[3 * j] == q[0] && xyz[3 * j + 1] == q[1] && xyz[3 * j + 2] == q[2]) {
            found = j;
            break;
        }
    }
    if (found >= 0 && store_of_global) found = store_of_global[found];
    nbr[k] = found;
}

int launch_neighbours(const int32_t *xyz, int64_t n, const uint32_t *start, const int32_t *entry, uint32_t T,
                      const int32_t *store_of_global, const int64_t *rows, int64_t n_rows, int32_t *nbr,
                      cudaStream_t s) {
    (void)n;
    if (n_rows == 0) return 0;
    k_neighbours<<<grid_for(kNbr * n_rows, 256), 256, 0, s>>>(xyz, start, entry, T, store_of_global, rows, n_rows,
                                                              nbr);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// f finite, W finite and >= 0 (VOL_EDATA otherwise); counts Ω = {W > 0}: one atomic per CTA.
__global__ void k_validate(const float *__restrict__ f, const float *__restrict__ W, int64_t nvox,
                           unsigned long long *bad, unsigned long long *n_omega) {
    __shared__ unsigned s_cnt;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    unsigned om = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvox; i += (int64_t)gridDim.x * blockDim.x) {
        const float fv = f[i], wv = W[i];
        if (!(isfinite(fv) && isfinite(wv) && wv >= 0.0f)) atomicMin(bad, (unsigned long long)i);
        om += wv > 0.0f ? 1u : 0u;
    }
    for (int o = 16; o > 0; o >>= 1) om += __shfl_xor_sync(0xffffffffu, om, o);
    if ((threadIdx.x & 31) == 0 && om) atomicAdd(&s_cnt, om);
    __syncthreads();
    if (threadIdx.x == 0 && s_cnt) atomicAdd(n_omega, (unsigned long long)s_cnt);
}

int launch_validate(const float *f, const float *W, int64_t nvox, unsigned long long *bad, unsigned long long *n_omega,
                    cudaStream_t s) {
    if (nvox == 0) return 0;
    int64_t g = grid_for(nvox, 256);
    k_validate<<<(unsigned)(g < 148 * 16 ? g : 148 * 16), 256, 0, s>>>(f, W, nvox, bad, n_omega);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// Initialisation (P:291 step 1 / S:276, reading c-4): p = 0; u = ū = f (warm) or 0 on Ω (zero init);
// Ω̄ keeps u = ū = f in both ū buffers forever (never written by the iteration kernels).
__global__ void k_init_state(Fields F, int64_t nvox, int init) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nvox) return;
    float fv = F.f[i];
    float u0 = (init == 1 && F.W[i] > 0.0f) ? 0.0f : fv;
    F.u[i] = u0;
    F.ub[0][i] = u0;
    F.ub[1][i] = u0;
    F.px[0][i] = 0.0f;
    F.py[0][i] = 0.0f;
    F.pz[0][i] = 0.0f;
    F.px[1][i] = 0.0f;
    F.py[1][i] = 0.0f;
    F.pz[1][i] = 0.0f;
}

int launch_init_state(const Fields &F, int64_t nvox, int init, cudaStream_t s) {
    if (nvox == 0) return 0;
    k_init_state<<<grid_for(nvox, 256), 256, 0, s>>>(F, nvox, init);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// After vol_load_state: Ω̄ voxels get u = ū = f (both ū buffers) and p = 0 (both buffers); on Ω
// voxels the components of p that live on invalid edges are set to 0 (the invariant the iteration
// keeps, see iterate.cu), so a loaded state behaves exactly like one produced by the iteration.
__global__ void k_sanitize_state(Fields F, int cur, const int32_t *__restrict__ nbr, int64_t nvox) {
    int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nvox) return;
    const int64_t b = v / kBlockVox;
    const int i = (int)(v % kBlockVox);
    float *ubc = cur ? F.ub[1] : F.ub[0];
    float *ubo = cur ? F.ub[0] : F.ub[1];
    float *pc[3] = {cur ? F.px[1] : F.px[0], cur ? F.py[1] : F.py[0], cur ? F.pz[1] : F.pz[0]};
    float *po[3] = {cur ? F.px[0] : F.px[1], cur ? F.py[0] : F.py[1], cur ? F.pz[0] : F.pz[1]};
    if (!(F.W[v] > 0.0f)) {
        float fv = F.f[v];
        F.u[v] = fv;
        ubc[v] = fv;
        ubo[v] = fv;
        for (int a = 0; a < 3; a++) pc[a][v] = po[a][v] = 0.0f;
        return;
    }
    ubo[v] = ubc[v];
    int c[3] = {i & 7, (i >> 3) & 7, i >> 6};
    for (int a = 0; a < 3; a++) {
        int q[3] = {c[0], c[1], c[2]};
        q[a] += 1;
        int64_t w;
        if (q[a] > 7) {
            int32_t nb = nbr[kNbr * b + 2 * a + 1];
            q[a] = 0;
            w = nb < 0 ? -1 : (int64_t)nb * kBlockVox + q[0] + 8 * q[1] + 64 * q[2];
        } else {
            w = b * kBlockVox + q[0] + 8 * q[1] + 64 * q[2];
        }
        if (w < 0 || !(F.W[w] > 0.0f)) pc[a][v] = 0.0f;
        po[a][v] = pc[a][v];
    }
}

int launch_sanitize_state(const Fields &F, int cur, const int32_t *nbr, int64_t n_blocks, cudaStream_t s) {
    int64_t nvox = n_blocks * kBlockVox;
    if (nvox == 0) return 0;
    k_sanitize_state<<<grid_for(nvox, 256), 256, 0, s>>>(F, cur, nbr, nvox);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// Block permutation between the caller's order and the store order (one 2 KiB row per block):
// gather: dst[r] = src[perm[r]];  scatter: dst[perm[r]] = src[r].
__global__ void k_permute_blocks(const float4 *__restrict__ src, float4 *__restrict__ dst,
                                 const int32_t *__restrict__ perm, int gather) {
    const int64_t r = blockIdx.x;
    const int64_t p = perm[r];
    const int64_t from = gather ? p : r, to = gather ? r : p;
    dst[to * 128 + threadIdx.x] = src[from * 128 + threadIdx.x];
}

int launch_permute_blocks(const float *src, float *dst, const int32_t *perm, int64_t n, bool gather, cudaStream_t s) {
    if (n == 0) return 0;
    k_permute_blocks<<<(unsigned)n, 128, 0, s>>>(reinterpret_cast<const float4 *>(src), reinterpret_cast<float4 *>(dst),
                                                 perm, gather ? 1 : 0);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// 8-bit weights given by the caller (vol_create_w8), gathered into store order and widened to fp32:
// dst[r][i] = (float)src[perm[r]][i]
__global__ void k_permute_w8_to_f32(const uint8_t *__restrict__ src, float *__restrict__ dst,
                                    const int32_t *__restrict__ perm) {
    const int64_t r = blockIdx.x;
    const int64_t c = perm[r];
    const uchar4 w = reinterpret_cast<const uchar4 *>(src + c * kBlockVox)[threadIdx.x];
    reinterpret_cast<float4 *>(dst + r * kBlockVox)[threadIdx.x] = make_float4((float)w.x, (float)w.y, (float)w.z,
                                                                               (float)w.w);
}

int launch_permute_w8_to_f32(const uint8_t *src, float *dst, const int32_t *perm, int64_t n, cudaStream_t s) {
    if (n == 0) return 0;
    k_permute_w8_to_f32<<<(unsigned)n, 128, 0, s>>>(src, dst, perm);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// The fusion weight is an observation count (Eq. 1: w_k = w_{k-1} + 1), so it is usually an
// exact small integer; then the fused kernel reads it as one byte instead of four (exact: the kernel
// converts back to the same float).
__global__ void k_pack_w8(const float *__restrict__ W, uint8_t *__restrict__ W8, int64_t nvox, unsigned *bad) {
    bool ok = true;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvox; i += (int64_t)gridDim.x * blockDim.x) {
        const float w = W[i];
        const bool e = w >= 0.0f && w <= 255.0f && w == truncf(w);
        W8[i] = e ? (uint8_t)w : 0;
        ok &= e;
    }
    if (__any_sync(0xffffffffu, !ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

int launch_pack_w8(const float *W, uint8_t *W8, int64_t nvox, unsigned *bad, cudaStream_t s) {
    if (nvox == 0) return 0;
    int64_t g = grid_for(nvox, 256);
    k_pack_w8<<<(unsigned)(g < 148 * 16 ? g : 148 * 16), 256, 0, s>>>(W, W8, nvox, bad);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// Frozen voxels (opts.freeze): with the L1 data term the primal step of a voxel with u = f is
//   ũ = fl(f + fl(τ·d)),  r = fl(ũ − f),  u' = f  whenever |r| <= t = fl(fl(τλ)·W),
// and |d| = |Σ_a p_a(v) − p_a(v−ê_a)| <= √3 + 3 because every p the primal step reads was just projected
// onto the unit ball (‖p‖₂ <= 1 up to a few ulps).  |r| <= τ|d|(1 + 2^-21) + |f|·2^-23, so
// t >= τ(3+√3)(1 + 2^-19) + |f|·2^-22 guarantees u' = f and then ū' = f + θ·(f − f) = f, at every
// iteration of the call.  A voxel that satisfies it with u = ū = f in both ū buffers at the start of the
// call therefore never changes during the call; the fused kernel skips its primal step and stores.
// Layout of a row's 64 bytes: byte c (column c = x + 8y) holds bit z for voxel c + 64z — the layout the
// iteration kernels read, where a thread owns one column and a run of z (one byte load per thread).
__global__ void k_freeze_mask(Fields F, int cur, IterParams P, uint32_t *__restrict__ frozen) {
    __shared__ uint32_t part[128];
    const int64_t b = blockIdx.x;
    const int t = threadIdx.x;
    const float *ubc = cur ? F.ub[1] : F.ub[0];
    const float *ubo = cur ? F.ub[0] : F.ub[1];
    uint32_t bits = 0;
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const int i = t + 128 * j;   // column t & 63, z = (t >> 6) + 2j
        const int64_t v = b * 512 + i;
        const float fv = F.f[v], w = F.W[v];
        const float tt = P.tl * w;
        const float bound = P.tau * (4.7320508f * 1.0000019f) + fabsf(fv) * 2.3841858e-7f;
        // bitwise equality, and f ≠ −0 (ū' = f + (+0) would turn −0 into +0)
        const uint32_t fb = __float_as_uint(fv);
        const bool fz = P.data_term == 0 && w > 0.0f && tt >= bound && fb != 0x80000000u &&
                        __float_as_uint(F.u[v]) == fb && __float_as_uint(ubc[v]) == fb && __float_as_uint(ubo[v]) == fb;
        bits |= (fz ? 1u : 0u) << (i >> 6);
    }
    part[t] = bits;
    __syncthreads();
    if (t < 64) reinterpret_cast<uint8_t *>(frozen + b * 16)[t] = (uint8_t)(part[t] | part[t + 64]);
}

int launch_freeze_mask(const Fields &F, int cur, const IterParams &P, int64_t n_blocks, uint32_t *frozen,
                       cudaStream_t s) {
    if (n_blocks == 0) return 0;
    k_freeze_mask<<<(unsigned)n_blocks, 128, 0, s>>>(F, cur, P, frozen);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

}  // namespace hvg
