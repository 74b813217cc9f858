// fuse.cu — TSDF fusion of posed depth maps into the hashed voxel-block grid on the device
// (arXiv 1604.03734 §III-A, Eq. 1).  Readings F-1 … F-10: DESIGN.md §11.
//
// The paper fuses frame by frame: allocate the blocks where frame k observes a surface,
// then update every voxel of every allocated block with frame k (P:152-176 steps 1-4, Eq. 1).
// The update of one voxel depends only on its own (f, w) and the frame, so the sequential result is
// reproduced exactly by (i) one allocation launch over all pixels of all frames that records, per
// block, the FIRST frame that allocates it (atomicMin — order-independent), and (ii) one update
// launch in which every voxel runs its Eq. 1 recurrence over frames first(b) … K−1 in order, in
// registers, writing f and W once.  The block set, the canonical (x, y, z) order (radix sort of the
// packed keys) and every value are therefore independent of thread scheduling.
//
//   k_fuse_alloc      one thread per (frame, pixel): the pixel ray between camera depths
//                     max(d − μ, 0) and d + μ (the truncation band, reading F-5) walked over the
//                     block lattice (reading F-7), each block inserted into an open-addressing
//                     device hash set of packed keys (atomicCAS) with atomicMin of the frame;
//   k_fuse_compact    occupied slots → (key, first frame) list;  CUB radix sort by key;
//   k_fuse_integrate  one 128-thread CTA per block, 4 voxels per thread: for k = first … K−1, a
//                     conservative block-level frustum / range cull (never skips a voxel the exact
//                     per-voxel test would update), then steps 1-4 and Eq. 1 per voxel.
//
// Every floating-point decision and value follows the written order of the readings (compiled
// with --fmad=false, IEEE division): bit-identical to the oracle in the same precision.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "../../include/vol.h"
#include "handle.h"
#include "internal.h"

namespace hvg {

constexpr unsigned long long kEmpty = ~0ull;
constexpr int kWalkMax = 4096;        // longest accepted block walk (cells)
constexpr int32_t kCoordLim = 1 << 20;

// packed key: (x + 2^20, y + 2^20, z + 2^20) in 21 bits each, x most significant → sorting the keys
// sorts blocks by (x, y, z) lexicographically (reading F-9)
__device__ __forceinline__ unsigned long long pack_key(int32_t x, int32_t y, int32_t z) {
    return ((unsigned long long)(uint32_t)(x + kCoordLim) << 42) | ((unsigned long long)(uint32_t)(y + kCoordLim) << 21) |
           (unsigned long long)(uint32_t)(z + kCoordLim);
}

struct FuseSet {
    unsigned long long *keys;   // [cap], kEmpty = free
    int32_t *first;             // [cap], INT_MAX = none
    unsigned long long *count;  // [0] inserted keys, [1] error flags (bit0 table full, bit1 coordinate range /
                                // walk), [2] compaction cursor, [3] valid pixels, [4] evaluated block-frames,
                                // [5] Eq. 1 voxel updates
    uint32_t mask;              // cap − 1
    unsigned long long limit;   // max_blocks: past it the call fails with VOL_ENOMEM, so inserting stops
    int32_t *prev;              // [cap] row of the block in the previous fusion's arrays, −1 = new (F-11)
};

__device__ __forceinline__ void set_insert(const FuseSet &S, int32_t x, int32_t y, int32_t z, int32_t frame) {
    if (x <= -kCoordLim || x >= kCoordLim || y <= -kCoordLim || y >= kCoordLim || z <= -kCoordLim || z >= kCoordLim) {
        atomicOr(&S.count[1], 2ull);
        return;
    }
    const unsigned long long key = pack_key(x, y, z);
    uint32_t h = ((uint32_t)x * 73856093u ^ (uint32_t)y * 19349669u ^ (uint32_t)z * 83492791u) & S.mask;
    for (uint32_t probe = 0; probe <= S.mask; probe++) {
        // capacity reached: the call will fail (VOL_ENOMEM), so stop probing a table that keeps filling
        // (checked only on long probe sequences: below the capacity the load factor is <= 1/2)
        if (probe >= 32 && (probe & 15) == 0) {
            if (*((volatile unsigned long long *)&S.count[0]) > S.limit) {
                atomicOr(&S.count[1], 1ull);
                return;
            }
        }
        // plain load: a slot only ever goes EMPTY -> key and first only decreases, so a stale value is
        // an older state — EMPTY falls through to the CAS, a larger first costs one extra atomicMin
        unsigned long long cur = S.keys[h];
        if (cur == kEmpty) {
            cur = atomicCAS(&S.keys[h], kEmpty, key);
            if (cur == kEmpty) {
                atomicAdd(&S.count[0], 1ull);
                atomicMin(&S.first[h], frame);
                return;
            }
        }
        if (cur == key) {
            if (S.first[h] > frame) atomicMin(&S.first[h], frame);
            return;
        }
        h = (h + 1) & S.mask;
    }
    atomicOr(&S.count[1], 1ull);
}

// Reading F-11: the blocks of an earlier fusion enter the set before frame 0 (first frame −1) and
// remember their row in the caller's previous arrays.  Flags: bit1 coordinate range, bit2 repeated block.
__global__ void k_fuse_seed(const int32_t *__restrict__ xyz, int64_t n, FuseSet S) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    if (x <= -kCoordLim || x >= kCoordLim || y <= -kCoordLim || y >= kCoordLim || z <= -kCoordLim || z >= kCoordLim) {
        atomicOr(&S.count[1], 2ull);
        return;
    }
    const unsigned long long key = pack_key(x, y, z);
    uint32_t h = ((uint32_t)x * 73856093u ^ (uint32_t)y * 19349669u ^ (uint32_t)z * 83492791u) & S.mask;
    for (uint32_t probe = 0; probe <= S.mask; probe++) {
        const unsigned long long cur = atomicCAS(&S.keys[h], kEmpty, key);
        if (cur == kEmpty) {
            atomicAdd(&S.count[0], 1ull);
            S.first[h] = -1;
            S.prev[h] = (int32_t)i;
            return;
        }
        if (cur == key) {
            atomicOr(&S.count[1], 4ull);
            return;
        }
        h = (h + 1) & S.mask;
    }
    atomicOr(&S.count[1], 1ull);
}

__device__ __forceinline__ bool depth_ok(float d, float max_range) {
    return isfinite(d) && d > 0.0f && d <= max_range;
}

// Reading F-6: p_c = (xr·z, yr·z, z) with xr = (i − cx)/fx, yr = (j − cy)/fy; p_g = R p_c + t, row sums left
// to right.  (xr, yr) are computed once per pixel (same operations as evaluating them per point.)
__device__ __forceinline__ void ray_point(const float *T, float xr, float yr, float z, float &gx, float &gy, float &gz) {
    const float xc = __fmul_rn(xr, z);
    const float yc = __fmul_rn(yr, z);
    const float zc = z;
    gx = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(T[0], xc), __fmul_rn(T[1], yc)), __fmul_rn(T[2], zc)), T[3]);
    gy = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(T[4], xc), __fmul_rn(T[5], yc)), __fmul_rn(T[6], zc)), T[7]);
    gz = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(T[8], xc), __fmul_rn(T[9], yc)), __fmul_rn(T[10], zc)), T[11]);
}

// One axis of the reading F-7 walk set-up.  tMax and tDelta are only ever read for an axis with
// remaining steps (n > 0), so they are computed only then (n > 0 implies dir != 0).
__device__ __forceinline__ void walk_axis(float a, float b, float inv_bm, int32_t &c, int32_t &n, int32_t &step,
                                          float &tmax, float &tdel) {
    const float sa = __fmul_rn(a, inv_bm);   // reading F-12: s = p·fl(1/Bm)
    const float sb = __fmul_rn(b, inv_bm);
    const float fa = floorf(sa);
    const float fb = floorf(sb);
    // coordinates far outside the packable range are clamped here and rejected by set_insert
    const float lim = 2.0e9f;
    c = (int32_t)fminf(fmaxf(fa, -lim), lim);
    const int32_t e = (int32_t)fminf(fmaxf(fb, -lim), lim);
    const long long dn = (long long)e - (long long)c;
    n = (int32_t)(dn < 0 ? (-dn > kWalkMax ? kWalkMax + 1 : -dn) : (dn > kWalkMax ? kWalkMax + 1 : dn));
    step = dn > 0 ? 1 : (dn < 0 ? -1 : 0);
    tmax = INFINITY;
    tdel = INFINITY;
    if (n > 0) {
        const float dir = __fsub_rn(sb, sa);
        if (dir > 0.0f) {
            tdel = __frcp_rn(dir);
            tmax = __fmul_rn(__fsub_rn(__fadd_rn(fa, 1.0f), sa), tdel);
        } else {
            tdel = __frcp_rn(-dir);
            tmax = __fmul_rn(__fsub_rn(sa, fa), tdel);
        }
    }
}

struct FuseArgs {
    const float *depth;   // [K][H][W]
    const float *poses;   // [K][12] T_gc row-major
    int32_t K, H, W;
    float fx, fy, cx, cy;
    float voxel, mu, max_range, w_max;
};

// One thread per pixel, grid-stride.  IDX is uint32_t when K·H·W < 2^32 (cheap index arithmetic), else
// 64-bit.  A lane's walk is independent of its neighbours' (no lockstep): repeated inserts of a block
// by neighbouring pixels mostly hit the block's slot in L1/L2 and skip the atomics (set_insert).
template <class IDX>
__global__ void __launch_bounds__(256) k_fuse_alloc(FuseArgs A, FuseSet S) {
    const IDX HW = (IDX)A.H * (IDX)A.W;
    const IDX total = HW * (IDX)A.K;
    const float inv_bm = __fdiv_rn(1.0f, __fmul_rn(8.0f, A.voxel));   // fl(1/Bm), Bm = fl(8v)
    const float inv_fx = __fdiv_rn(1.0f, A.fx), inv_fy = __fdiv_rn(1.0f, A.fy);
    unsigned long long n_valid = 0;
    for (IDX pix = (IDX)blockIdx.x * blockDim.x + threadIdx.x; pix < total; pix += (IDX)gridDim.x * blockDim.x) {
        const float d = __ldg(A.depth + pix);
        if (!depth_ok(d, A.max_range)) continue;
        n_valid++;
        const int32_t k = (int32_t)(pix / HW);
        const IDX rem = pix - (IDX)k * HW;
        const int32_t j = (int32_t)(rem / (IDX)A.W);
        const int32_t i = (int32_t)(rem - (IDX)j * (IDX)A.W);
        float T[12];
#pragma unroll
        for (int q = 0; q < 12; q++) T[q] = __ldg(A.poses + 12 * k + q);
        float za = __fsub_rn(d, A.mu);
        if (za < 0.0f) za = 0.0f;
        const float zb = __fadd_rn(d, A.mu);
        const float xr = __fmul_rn(__fsub_rn((float)i, A.cx), inv_fx);   // reading F-12
        const float yr = __fmul_rn(__fsub_rn((float)j, A.cy), inv_fy);
        float ax, ay, az, bx, by, bz;
        ray_point(T, xr, yr, za, ax, ay, az);
        ray_point(T, xr, yr, zb, bx, by, bz);
        int32_t cx_, cy_, cz_, nx, ny, nz, sx, sy, sz;
        float tx, ty, tz, dx, dy, dz;
        walk_axis(ax, bx, inv_bm, cx_, nx, sx, tx, dx);
        walk_axis(ay, by, inv_bm, cy_, ny, sy, ty, dy);
        walk_axis(az, bz, inv_bm, cz_, nz, sz, tz, dz);
        if (nx + ny + nz + 1 > kWalkMax) {
            atomicOr(&S.count[1], 2ull);
            continue;
        }
        set_insert(S, cx_, cy_, cz_, k);
        while (nx + ny + nz > 0) {
            // the axis with remaining steps and the smallest tMax; ties → lowest axis (reading F-7)
            if (nx > 0 && (ny == 0 || tx <= ty) && (nz == 0 || tx <= tz)) {
                cx_ += sx;
                tx = __fadd_rn(tx, dx);
                nx--;
            } else if (ny > 0 && (nz == 0 || ty <= tz)) {
                cy_ += sy;
                ty = __fadd_rn(ty, dy);
                ny--;
            } else {
                cz_ += sz;
                tz = __fadd_rn(tz, dz);
                nz--;
            }
            set_insert(S, cx_, cy_, cz_, k);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_valid += __shfl_xor_sync(0xffffffffu, n_valid, o);
    if ((threadIdx.x & 31) == 0 && n_valid) atomicAdd(&S.count[3], n_valid);
}

__global__ void k_fuse_compact(FuseSet S, uint32_t cap, unsigned long long *out_keys, unsigned long long *out_val,
                               unsigned long long *cursor, unsigned long long limit) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= cap) return;
    const unsigned long long key = S.keys[s];
    if (key == kEmpty) return;
    const unsigned long long r = atomicAdd(cursor, 1ull);
    if (r < limit) {
        out_keys[r] = key;
        // value: (first frame, previous row), both int32, first in the high half
        out_val[r] = ((unsigned long long)(uint32_t)S.first[s] << 32) | (uint32_t)S.prev[s];
    }
}

// Conservative cull of one block against one frame: true only if no voxel of the block can pass the
// per-voxel test (z_c > 0, nearest pixel inside the image, u_SDF >= −μ with d <= max_range).  The
// block's voxel centres lie in the sphere of centre c (block centre) and radius 3.5·v·√3; the
// margins below absorb the fp32 rounding of the per-voxel path (relative ~1e-6) many times over.
__device__ __forceinline__ bool block_culled(const float *T, const FuseArgs &A, float cxg, float cyg, float czg) {
    const float d0 = cxg - T[3], d1 = cyg - T[7], d2 = czg - T[11];
    const float xc = (T[0] * d0 + T[4] * d1) + T[8] * d2;
    const float yc = (T[1] * d0 + T[5] * d1) + T[9] * d2;
    const float zc = (T[2] * d0 + T[6] * d1) + T[10] * d2;
    const float ext = fabsf(d0) + fabsf(d1) + fabsf(d2);
    const float r = 3.5f * 1.7320508f * A.voxel * 1.001f + 1e-3f + 1e-5f * ext;
    if (zc + r <= 0.0f) return true;                            // behind the camera
    if (zc - r > A.max_range + A.mu) return true;               // behind every admissible surface by > μ
    const float pad = 2.0f;                                     // pixels
    // in-image half-spaces for z_c > 0:  fx·x + (cx + ½ + pad)·z >= 0,  −fx·x + (W − cx − ½ + pad)·z > 0
    const float l0 = A.cx + 0.5f + pad, r0 = (float)A.W - A.cx - 0.5f + pad;
    const float t0 = A.cy + 0.5f + pad, b0 = (float)A.H - A.cy - 0.5f + pad;
    if (A.fx * xc + l0 * zc + sqrtf(A.fx * A.fx + l0 * l0) * r < 0.0f) return true;
    if (-A.fx * xc + r0 * zc + sqrtf(A.fx * A.fx + r0 * r0) * r < 0.0f) return true;
    if (A.fy * yc + t0 * zc + sqrtf(A.fy * A.fy + t0 * t0) * r < 0.0f) return true;
    if (-A.fy * yc + b0 * zc + sqrtf(A.fy * A.fy + b0 * b0) * r < 0.0f) return true;
    return false;
}

// Frames are taken in chunks of 128 (one per thread): each thread loads one frame's pose into shared
// memory and runs the block cull for it; the CTA then walks the surviving frames of the chunk in
// increasing order (the Eq. 1 recurrence order is unchanged).
constexpr int kFrameChunk = 128;

__global__ void __launch_bounds__(128) k_fuse_integrate(FuseArgs A, const unsigned long long *__restrict__ keys,
                                                        const unsigned long long *__restrict__ vals, int64_t n,
                                                        const float *__restrict__ prev_f,
                                                        const float *__restrict__ prev_w,
                                                        int32_t *__restrict__ xyz_out, int32_t *__restrict__ first_out,
                                                        float *__restrict__ f_out, float *__restrict__ w_out,
                                                        int cull, unsigned long long *stats) {
    __shared__ float4 sT[kFrameChunk][3];
    __shared__ uint32_t sMask[kFrameChunk / 32];
    const int64_t b = blockIdx.x;
    if (b >= n) return;
    const unsigned long long key = keys[b];
    const int32_t bx = (int32_t)((key >> 42) & 0x1FFFFF) - kCoordLim;
    const int32_t by = (int32_t)((key >> 21) & 0x1FFFFF) - kCoordLim;
    const int32_t bz = (int32_t)(key & 0x1FFFFF) - kCoordLim;
    const unsigned long long val = vals[b];
    const int32_t kfirst = (int32_t)(uint32_t)(val >> 32);
    const int32_t prow = (int32_t)(uint32_t)(val & 0xFFFFFFFFull);
    const int32_t k0 = kfirst < 0 ? 0 : kfirst;
    const int t = threadIdx.x;
    if (t == 0) {
        xyz_out[3 * b] = bx;
        xyz_out[3 * b + 1] = by;
        xyz_out[3 * b + 2] = bz;
        if (first_out) first_out[b] = kfirst;
    }
    // voxels 4t … 4t+3: x = 4(t&1) + q, y = (t>>1)&7, z = t>>4
    const int lx0 = 4 * (t & 1), ly = (t >> 1) & 7, lz = t >> 4;
    // voxel centre (8B + i + ½)·v (SURVEY §8(d) frame convention)
    float px[4];
#pragma unroll
    for (int q = 0; q < 4; q++) px[q] = __fmul_rn(__fadd_rn((float)(8 * bx + lx0 + q), 0.5f), A.voxel);
    const float py = __fmul_rn(__fadd_rn((float)(8 * by + ly), 0.5f), A.voxel);
    const float pz = __fmul_rn(__fadd_rn((float)(8 * bz + lz), 0.5f), A.voxel);
    const float cxg = (8.0f * (float)bx + 4.0f) * A.voxel;
    const float cyg = (8.0f * (float)by + 4.0f) * A.voxel;
    const float czg = (8.0f * (float)bz + 4.0f) * A.voxel;
    float f[4] = {0.f, 0.f, 0.f, 0.f}, w[4] = {0.f, 0.f, 0.f, 0.f};
    if (prow >= 0) {   // a block of the previous fusion continues from its (f, W) (reading F-11)
        const float4 pf = *reinterpret_cast<const float4 *>(prev_f + (int64_t)prow * kBlockVox + 4 * t);
        const float4 pw = *reinterpret_cast<const float4 *>(prev_w + (int64_t)prow * kBlockVox + 4 * t);
        f[0] = pf.x; f[1] = pf.y; f[2] = pf.z; f[3] = pf.w;
        w[0] = pw.x; w[1] = pw.y; w[2] = pw.z; w[3] = pw.w;
    }
    const long long HW = (long long)A.H * A.W;
    unsigned n_frames = 0, n_upd = 0;
    const float Wf = (float)A.W, Hf = (float)A.H;
    const float inv_mu = __fdiv_rn(1.0f, A.mu);
    for (int32_t kb = k0; kb < A.K; kb += kFrameChunk) {
        {
            const int32_t k = kb + t;
            bool keep = false;
            if (k < A.K) {
                float T[12];
#pragma unroll
                for (int q = 0; q < 12; q++) T[q] = __ldg(A.poses + 12 * k + q);
                keep = !cull || !block_culled(T, A, cxg, cyg, czg);
                sT[t][0] = make_float4(T[0], T[1], T[2], T[3]);
                sT[t][1] = make_float4(T[4], T[5], T[6], T[7]);
                sT[t][2] = make_float4(T[8], T[9], T[10], T[11]);
            }
            const uint32_t m = __ballot_sync(0xffffffffu, keep);
            if ((t & 31) == 0) sMask[t >> 5] = m;
        }
        __syncthreads();
#pragma unroll 1
        for (int wq = 0; wq < kFrameChunk / 32; wq++) {
            uint32_t m = sMask[wq];
            while (m) {
                const int idx = 32 * wq + __ffs(m) - 1;
                m &= m - 1;
                n_frames++;
                const float4 r0 = sT[idx][0], r1 = sT[idx][1], r2 = sT[idx][2];
                const float *D = A.depth + (long long)(kb + idx) * HW;
                // step 1: p_c = R^T (p_g − t); the y and z parts of p_g − t are shared by the 4 voxels
                const float d1 = __fsub_rn(py, r1.w);
                const float d2 = __fsub_rn(pz, r2.w);
                const float e1x = __fmul_rn(r1.x, d1), e1y = __fmul_rn(r1.y, d1), e1z = __fmul_rn(r1.z, d1);
                const float e2x = __fmul_rn(r2.x, d2), e2y = __fmul_rn(r2.y, d2), e2z = __fmul_rn(r2.z, d2);
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const float d0 = __fsub_rn(px[q], r0.w);
                    const float xc = __fadd_rn(__fadd_rn(__fmul_rn(r0.x, d0), e1x), e2x);
                    const float yc = __fadd_rn(__fadd_rn(__fmul_rn(r0.y, d0), e1y), e2y);
                    const float zc = __fadd_rn(__fadd_rn(__fmul_rn(r0.z, d0), e1z), e2z);
                    if (!(zc > 0.0f)) continue;
                    // step 2: nearest pixel (reading F-1)
                    const float rz = __frcp_rn(zc);   // reading F-12: one correctly rounded reciprocal of z_c
                    const float ix = __fadd_rn(__fmul_rn(A.fx, __fmul_rn(xc, rz)), A.cx);
                    const float iy = __fadd_rn(__fmul_rn(A.fy, __fmul_rn(yc, rz)), A.cy);
                    const float fi = floorf(__fadd_rn(ix, 0.5f));
                    const float fj = floorf(__fadd_rn(iy, 0.5f));
                    if (!(fi >= 0.0f && fi < Wf && fj >= 0.0f && fj < Hf)) continue;
                    const float d = __ldg(D + (int32_t)fj * A.W + (int32_t)fi);
                    if (!depth_ok(d, A.max_range)) continue;
                    // step 3: u_SDF = d − z_c;  step 4, Eq. 1, readings F-3/F-4
                    const float sdf = __fsub_rn(d, zc);
                    if (sdf < -A.mu) continue;
                    const float c = fminf(fmaxf(sdf, -A.mu), A.mu);
                    const float tsdf = __fmul_rn(c, inv_mu);   // reading F-12: ·fl(1/μ)
                    const float num = __fadd_rn(tsdf, __fmul_rn(w[q], f[q]));
                    const float den = __fadd_rn(w[q], 1.0f);
                    f[q] = __fdiv_rn(num, den);
                    w[q] = fminf(den, A.w_max);
                    n_upd++;
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n_upd += __shfl_xor_sync(0xffffffffu, n_upd, o);
    if ((t & 31) == 0 && n_upd) atomicAdd(&stats[1], (unsigned long long)n_upd);
    if (t == 0 && n_frames) atomicAdd(&stats[0], (unsigned long long)n_frames);
    const int64_t o = b * kBlockVox + 4 * t;
    *reinterpret_cast<float4 *>(f_out + o) = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4 *>(w_out + o) = make_float4(w[0], w[1], w[2], w[3]);
}

}  // namespace hvg

using namespace hvg;

namespace {

uint32_t fuse_table_cap(int64_t max_blocks) {
    uint64_t c = 1024;
    while ((int64_t)c < 2 * max_blocks) c <<= 1;
    return (uint32_t)c;
}

size_t cub_sort_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                    (const unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                    (int)(n > 0 ? n : 1), 0, 63);
    return bytes;
}

struct FuseLayout {
    float *depth;
    float *poses;
    unsigned long long *keys;
    int32_t *first;
    int32_t *prev;
    unsigned long long *count;
    unsigned long long *ckeys[2];
    unsigned long long *cval[2];
    void *sort_tmp;
    size_t sort_bytes;
    int32_t *xyz;
    int32_t *ofirst;
    float *f, *w;
};

size_t fuse_layout(Carve &c, FuseLayout &L, int64_t max_blocks, int32_t K, int32_t H, int32_t W, bool dev_depth,
                   bool dev_poses, bool dev_out) {
    const uint32_t cap = fuse_table_cap(max_blocks);
    L.depth = dev_depth ? nullptr : c.take<float>((size_t)K * H * W);
    L.poses = dev_poses ? nullptr : c.take<float>((size_t)K * 12);
    L.keys = c.take<unsigned long long>(cap);
    L.first = c.take<int32_t>(cap);
    L.prev = c.take<int32_t>(cap);
    L.count = c.take<unsigned long long>(8);
    for (int q = 0; q < 2; q++) {
        L.ckeys[q] = c.take<unsigned long long>(max_blocks);
        L.cval[q] = c.take<unsigned long long>(max_blocks);
    }
    L.sort_bytes = cub_sort_bytes(max_blocks);
    L.sort_tmp = c.take<char>(L.sort_bytes);
    if (!dev_out) {
        L.xyz = c.take<int32_t>(3 * max_blocks);
        L.ofirst = c.take<int32_t>(max_blocks);
        L.f = c.take<float>((size_t)max_blocks * kBlockVox);
        L.w = c.take<float>((size_t)max_blocks * kBlockVox);
    } else {
        L.xyz = nullptr;
        L.ofirst = nullptr;
        L.f = L.w = nullptr;
    }
    return c.off + 256;
}

vol_status check_fuse_args(int32_t K, const vol_camera *cam, const vol_fusion_params *p, int64_t max_blocks) {
    if (K < 1) return fail(VOL_EINVAL, "vol_fuse: n_frames must be >= 1 (got %d)", K);
    if (!cam || !p) return fail(VOL_EINVAL, "vol_fuse: camera and params must not be NULL");
    if (cam->width < 1 || cam->height < 1) return fail(VOL_EINVAL, "vol_fuse: image size must be positive");
    if ((long long)K * cam->width * cam->height > (1ll << 40)) return fail(VOL_EINVAL, "vol_fuse: too many pixels");
    if (!(cam->fx > 0.0f) || !(cam->fy > 0.0f) || !std::isfinite(cam->fx) || !std::isfinite(cam->fy) ||
        !std::isfinite(cam->cx) || !std::isfinite(cam->cy))
        return fail(VOL_EINVAL, "vol_fuse: intrinsics must be finite with fx, fy > 0");
    if (!(p->voxel > 0.0f) || !std::isfinite(p->voxel)) return fail(VOL_EINVAL, "vol_fuse: voxel must be > 0");
    if (!(p->mu > 0.0f) || !std::isfinite(p->mu)) return fail(VOL_EINVAL, "vol_fuse: mu must be > 0");
    if (!(p->max_range > 0.0f)) return fail(VOL_EINVAL, "vol_fuse: max_range must be > 0");
    if (!(p->w_max >= 1.0f)) return fail(VOL_EINVAL, "vol_fuse: w_max must be >= 1");
    if (max_blocks < 1 || max_blocks > (1ll << 30)) return fail(VOL_EINVAL, "vol_fuse: max_blocks out of range");
    return VOL_OK;
}

}  // namespace

extern "C" size_t vol_fuse_workspace_bytes(int64_t max_blocks, int32_t n_frames, const vol_camera *cam) {
    if (!cam || max_blocks < 1 || n_frames < 1) return 0;
    Carve c;
    FuseLayout L;
    // worst case: host depth, host poses, host outputs
    return fuse_layout(c, L, max_blocks, n_frames, cam->height, cam->width, false, false, false);
}

extern "C" vol_status vol_fuse_incremental(const int32_t *prev_xyz, const float *prev_f, const float *prev_W,
                                           int64_t n_prev, const float *depth, int32_t n_frames, const vol_camera *cam,
                                           const float *poses, const vol_fusion_params *prm, int64_t max_blocks,
                                           void *workspace, size_t workspace_bytes, void *stream, int32_t *block_xyz,
                                           int32_t *first_frame, float *f, float *W, int64_t *n_blocks,
                                           vol_fusion_stats *stats) {
    NvtxRange nvtx_range_("vol_fuse");
    vol_status st = check_fuse_args(n_frames, cam, prm, max_blocks);
    if (st != VOL_OK) return st;
    if (n_prev < 0 || (n_prev > 0 && (!prev_xyz || !prev_f || !prev_W)))
        return fail(VOL_EINVAL, "vol_fuse: n_prev < 0 or NULL previous arrays");
    if (!depth || !poses || !block_xyz || !f || !W || !n_blocks)
        return fail(VOL_EINVAL, "vol_fuse: depth, poses, block_xyz, f, W and n_blocks must not be NULL");
    *n_blocks = 0;
    if (stats) memset(stats, 0, sizeof *stats);
    cudaStream_t s = (cudaStream_t)stream;
    const bool dev_depth = is_device_ptr(depth), dev_poses = is_device_ptr(poses);
    const bool dev_out = is_device_ptr(block_xyz) && is_device_ptr(f) && is_device_ptr(W) &&
                         (!first_frame || is_device_ptr(first_frame));
    const bool any_dev_out = is_device_ptr(block_xyz) || is_device_ptr(f) || is_device_ptr(W) ||
                             (first_frame && is_device_ptr(first_frame));
    if (any_dev_out && !dev_out) return fail(VOL_EINVAL, "vol_fuse: outputs must be all device or all host pointers");
    const int32_t K = n_frames, H = cam->height, Wd = cam->width;
    Carve probe;
    FuseLayout L;
    const size_t need = fuse_layout(probe, L, max_blocks, K, H, Wd, dev_depth, dev_poses, dev_out);
    void *ws = workspace;
    bool owns = false;
    if (ws) {
        if (workspace_bytes < need)
            return fail(VOL_ENOMEM, "vol_fuse: workspace of %zu bytes < %zu needed", workspace_bytes, need);
    } else {
        CK(cudaMalloc(&ws, need));
        owns = true;
    }
    struct Free {
        void *p;
        bool own;
        ~Free() {
            if (own && p) cudaFree(p);
        }
    } guard{ws, owns};
    Carve c;
    c.base = (char *)ws;
    fuse_layout(c, L, max_blocks, K, H, Wd, dev_depth, dev_poses, dev_out);
    const float *d_depth = dev_depth ? depth : L.depth;
    const float *d_poses = dev_poses ? poses : L.poses;
    if (!dev_depth) CK(cudaMemcpyAsync(L.depth, depth, sizeof(float) * (size_t)K * H * Wd, cudaMemcpyDefault, s));
    if (!dev_poses) CK(cudaMemcpyAsync(L.poses, poses, sizeof(float) * (size_t)K * 12, cudaMemcpyDefault, s));
    const uint32_t cap = fuse_table_cap(max_blocks);
    CK(cudaMemsetAsync(L.keys, 0xFF, sizeof(unsigned long long) * cap, s));
    CK(cudaMemsetAsync(L.first, 0x7F, sizeof(int32_t) * cap, s));   // 0x7F7F7F7F > any frame index
    CK(cudaMemsetAsync(L.prev, 0xFF, sizeof(int32_t) * cap, s));    // −1: a new block
    CK(cudaMemsetAsync(L.count, 0, sizeof(unsigned long long) * 8, s));
    FuseArgs A{d_depth, d_poses, K, H, Wd, cam->fx, cam->fy, cam->cx, cam->cy,
               prm->voxel, prm->mu, prm->max_range, prm->w_max};
    FuseSet S{L.keys, L.first, L.count, cap - 1, (unsigned long long)max_blocks, L.prev};
    // previous blocks (reading F-11), staged to the device if they are host arrays
    const int32_t *d_pxyz = prev_xyz;
    const float *d_pf = prev_f, *d_pw = prev_W;
    struct Stage {
        void *p = nullptr;
        cudaStream_t s;
        ~Stage() {
            if (p) cudaFreeAsync(p, s);
        }
    } pstage{nullptr, s};
    if (n_prev > 0) {
        if (n_prev > max_blocks) return fail(VOL_ENOMEM, "vol_fuse: n_prev = %lld > max_blocks", (long long)n_prev);
        if (!(is_device_ptr(prev_xyz) && is_device_ptr(prev_f) && is_device_ptr(prev_W))) {
            const size_t bx = (size_t)n_prev * 12, bf = (size_t)n_prev * kBlockVox * 4;
            CK(cudaMallocAsync(&pstage.p, bx + 2 * bf + 512, s));
            char *base = (char *)pstage.p;
            float *sf = (float *)(base + ((bx + 255) & ~(size_t)255));
            float *sw = sf + (size_t)n_prev * kBlockVox;
            CK(cudaMemcpyAsync(base, prev_xyz, bx, cudaMemcpyDefault, s));
            CK(cudaMemcpyAsync(sf, prev_f, bf, cudaMemcpyDefault, s));
            CK(cudaMemcpyAsync(sw, prev_W, bf, cudaMemcpyDefault, s));
            d_pxyz = (const int32_t *)base;
            d_pf = sf;
            d_pw = sw;
        }
        k_fuse_seed<<<(unsigned)((n_prev + 255) / 256), 256, 0, s>>>(d_pxyz, n_prev, S);
        CK(cudaPeekAtLastError());
        counted(1);
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long total = (long long)K * H * Wd;
    long long grid = (total + 255) / 256;
    if (grid > (long long)sms * 16) grid = (long long)sms * 16;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    if (stats)
        for (auto &e : ev) CK(cudaEventCreate(&e));
    struct EvFree {
        cudaEvent_t *e;
        ~EvFree() {
            for (int q = 0; q < 4; q++)
                if (e[q]) cudaEventDestroy(e[q]);
        }
    } ev_guard{ev};
    if (stats) CK(cudaEventRecord(ev[0], s));
    if (total < (1ll << 32) - 1 - (long long)grid * 256)
        k_fuse_alloc<uint32_t><<<(unsigned)grid, 256, 0, s>>>(A, S);
    else
        k_fuse_alloc<unsigned long long><<<(unsigned)grid, 256, 0, s>>>(A, S);
    CK(cudaPeekAtLastError());
    counted(1);
    if (stats) CK(cudaEventRecord(ev[1], s));
    unsigned long long hc[4];
    CK(cudaMemcpyAsync(hc, L.count, sizeof hc, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *n_blocks = (int64_t)hc[0];
    if (stats) {
        stats->pixels_valid = (int64_t)hc[3];
        stats->blocks = (int64_t)hc[0];
    }
    if (hc[1] & 4ull) return fail(VOL_EDATA, "vol_fuse: the previous blocks repeat a block coordinate");
    if (hc[1] & 2ull)
        return fail(VOL_EDATA, "vol_fuse: a block walk leaves the block-coordinate range (-2^20, 2^20) or is longer "
                               "than %d blocks (check poses, voxel size and max_range)", kWalkMax);
    if ((hc[1] & 1ull) || (int64_t)hc[0] > max_blocks)
        return fail(VOL_ENOMEM, "vol_fuse: %lld blocks allocated (at least) > max_blocks = %lld",
                    (long long)hc[0], (long long)max_blocks);
    const int64_t n = (int64_t)hc[0];
    if (n == 0) return VOL_OK;
    CK(cudaMemsetAsync(L.count + 2, 0, sizeof(unsigned long long), s));
    k_fuse_compact<<<(cap + 255) / 256, 256, 0, s>>>(S, cap, L.ckeys[0], L.cval[0], L.count + 2,
                                                      (unsigned long long)max_blocks);
    CK(cudaPeekAtLastError());
    counted(1);
    size_t sb = L.sort_bytes;
    CK(cub::DeviceRadixSort::SortPairs(L.sort_tmp, sb, L.ckeys[0], L.ckeys[1], L.cval[0], L.cval[1], (int)n, 0, 63,
                                       s));   // library sort (CUB): not counted as this library's launches
    int32_t *oxyz = dev_out ? block_xyz : L.xyz;
    int32_t *ofirst = dev_out ? first_frame : (first_frame ? L.ofirst : nullptr);
    float *of = dev_out ? f : L.f;
    float *ow = dev_out ? W : L.w;
    const int cull = getenv("HVG_FUSE_NOCULL") ? 0 : 1;   // experiments only: the cull never changes results
    if (stats) CK(cudaEventRecord(ev[2], s));
    k_fuse_integrate<<<(unsigned)n, 128, 0, s>>>(A, L.ckeys[1], L.cval[1], n, d_pf, d_pw, oxyz, ofirst, of, ow, cull,
                                                  L.count + 4);
    CK(cudaPeekAtLastError());
    counted(1);
    if (stats) CK(cudaEventRecord(ev[3], s));
    if (!dev_out) {
        CK(cudaMemcpyAsync(block_xyz, L.xyz, sizeof(int32_t) * 3 * n, cudaMemcpyDeviceToHost, s));
        if (first_frame) CK(cudaMemcpyAsync(first_frame, L.ofirst, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(f, L.f, sizeof(float) * kBlockVox * n, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(W, L.w, sizeof(float) * kBlockVox * n, cudaMemcpyDeviceToHost, s));
    }
    if (stats) {
        unsigned long long hs[2];
        CK(cudaMemcpyAsync(hs, L.count + 4, sizeof hs, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        stats->block_frames = (int64_t)hs[0];
        stats->voxel_updates = (int64_t)hs[1];
        CK(cudaEventElapsedTime(&stats->ms_alloc, ev[0], ev[1]));
        CK(cudaEventElapsedTime(&stats->ms_integrate, ev[2], ev[3]));
    }
    if (owns || !dev_out) CK(cudaStreamSynchronize(s));
    return VOL_OK;
}

extern "C" vol_status vol_fuse(const float *depth, int32_t n_frames, const vol_camera *cam, const float *poses,
                               const vol_fusion_params *prm, int64_t max_blocks, void *workspace,
                               size_t workspace_bytes, void *stream, int32_t *block_xyz, int32_t *first_frame,
                               float *f, float *W, int64_t *n_blocks, vol_fusion_stats *stats) {
    return vol_fuse_incremental(nullptr, nullptr, nullptr, 0, depth, n_frames, cam, poses, prm, max_blocks, workspace,
                                workspace_bytes, stream, block_xyz, first_frame, f, W, n_blocks, stats);
}
