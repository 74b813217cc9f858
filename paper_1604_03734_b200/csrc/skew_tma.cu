// skew_tma.cu — the skewed Chambolle–Pock launch with the halo planes read by the tensor memory accelerator
// (SURVEY §8(a) rows a-3 … a-5; arXiv 1604.03734 §III-C; the schedule of iterate.cu's k_skew).
//
// Launch k computes, for one 8³ block per 128-thread CTA, the primal step k + relaxation of its own voxels,
// the primal step of the 3×64 voxels of its +x/+y/+z neighbour faces (recomputed: same function, same
// inputs ⇒ bit-identical to the owner), then the dual step k+1 of its own voxels.  What
// differs from k_skew is how the halo arrives.  k_skew gathers all of it with per-thread loads through the
// L1 load pipe, which ncu shows ~72 % busy (the limiter next to DRAM).  Here warp 0 issues tensor TMA
// copies (cp.async.bulk.tensor.4d) of the +y / +z face planes (u^k, f, W, p^{k+1}), the −y / −z normal
// p components and the four edge lines the y / z recomputes need, into shared memory, completing on the
// block's own mbarrier; only the +x plane (and the −x p_x) keep per-thread register loads.  The x=0
// plane of a block is 64 rows of one float, every 32-byte row a separate TMA request — measured 1.55x
// slower when fetched by TMA (probe and A/B in DESIGN.md §10), the TMA unit being row-rate bound.
// An absent neighbour is block coordinate −1: the box is out of bounds, TMA fills zeros (W = 0 ⇒ Ω̄, p = 0)
// and still completes the full byte count (probed on B200: scripts/probes/tma_probe.cu), so the barrier's
// transaction count is a per-launch constant and no thread tests neighbour existence.
// The tensor maps (one per field buffer and box shape) are encoded once per volume (skew_tma_build_maps).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "device_common.cuh"
#include "internal.h"

#ifndef HVG_TMA_MINB
#define HVG_TMA_MINB 8   // CTAs per SM k_skew_tma is compiled for (register budget)
#endif

namespace hvg {

// map table: index = box * kMapFields + field
enum { kFieldF = 0, kFieldW = 1, kFieldU = 2 /* + buffer */, kFieldPX = 4, kFieldPY = 6, kFieldPZ = 8, kMapFields = 10 };
enum { kBoxX = 0, kBoxY = 1, kBoxZ = 2, kBoxD = 3, kBoxE = 4, kBoxF = 5, kBoxShapes = 6 };
// box dims {x, y, z, block} per shape: the +x/−x planes, +y/−y planes, +z/−z planes, and edge lines
static const uint32_t kBoxDim[kBoxShapes][4] = {{4, 8, 8, 1}, {8, 1, 8, 1}, {8, 8, 1, 1},
                                                {4, 1, 8, 1}, {4, 8, 1, 1}, {8, 1, 1, 1}};
constexpr uint32_t kNbrTx = 6 * 256 + 6 * 256 + 256 + 256 + 128 + 128 + 32 + 32;   // +y, +z planes; −y, −z; 4 edge lines

size_t skew_tma_map_bytes() { return (size_t)kBoxShapes * kMapFields * sizeof(CUtensorMap); }

// Encodes the 60 tensor maps of a volume's fields (4-D {8, 8, 8, S} float32 views, row strides 32 / 256 /
// 2048 bytes) into host memory and copies them to `d_maps` (64-byte aligned device memory).
int skew_tma_build_maps(const Fields &F, int64_t S, void *d_maps, cudaStream_t s) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !enc)
            return -1;
    }
    const float *fld[kMapFields] = {F.f, F.W, F.u, F.u2, F.px[0], F.px[1], F.py[0], F.py[1], F.pz[0], F.pz[1]};
    CUtensorMap h[kBoxShapes * kMapFields];
    const cuuint64_t dim[4] = {8, 8, 8, (cuuint64_t)S};
    const cuuint64_t str[3] = {32, 256, 2048};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    for (int b = 0; b < kBoxShapes; b++)
        for (int q = 0; q < kMapFields; q++) {
            const cuuint32_t box[4] = {kBoxDim[b][0], kBoxDim[b][1], kBoxDim[b][2], kBoxDim[b][3]};
            CUresult r = enc(&h[b * kMapFields + q], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(fld[q]), dim,
                             str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return -1;
        }
    if (cudaMemcpyAsync(d_maps, h, sizeof h, cudaMemcpyHostToDevice, s) != cudaSuccess) return -1;
    return cudaStreamSynchronize(s) == cudaSuccess ? 0 : -1;
}

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_addr(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar))
        : "memory");
}

struct SkewTmaView {
    const float *f, *W;
    const uint8_t *W8;
    const uint32_t *frozen;
    const float *u_in;
    float *u_out;
    const float *px_in, *py_in, *pz_in;   // p^{k+1}
    float *px_out, *py_out, *pz_out;      // p^{k+2}
    const CUtensorMap *maps;
    int ui, pi;                           // in-buffer of u (0: F.u, 1: F.u2) and of p
};

template <bool W8>
struct __align__(128) TStage {
    float f[kBlockVox];
    float u[kBlockVox + 192];    // u^k own → ū^{k+1} own (in place); [512 + 64a + entry): ū^{k+1} of +face a
    float Wf[kBlockVox + 192];   // W own (fp32); [512 + 64a + entry): W of +face a
    float px[kBlockVox], py[kBlockVox], pz[kBlockVox];   // p^{k+1} own
    float yf[6][64];             // +y face plane: [z·8 + x]
    float zf[6][64];             // +z face plane: [y·8 + x]
    float mx[64];                // −x neighbour p_x at x = 7: [z·8 + y] (per-thread loads)
    float my[64];                // −y neighbour p_y at y = 7: [z·8 + x]
    float mz[64];                // −z neighbour p_z at z = 7: [y·8 + x]
    float e6[32];                // (−1,+1,0) p_x at (4+x, 0, z): [z·4 + x]
    float e7[32];                // (−1,0,+1) p_x at (4+x, y, 0): [y·4 + x]
    __align__(128) float e11[8];  // (0,+1,−1) p_z at (x, 0, 7)
    __align__(128) float e9[8];   // (0,−1,+1) p_y at (x, 7, 0)
    __align__(128) uint8_t W8b[W8 ? kBlockVox : 16];
    uint32_t fz[16];
    int32_t snb[kNbr];
};

// +x face entry k = y + 8z (voxel (0, y, z) of the +x neighbour): its u^k, f, W, p^{k+1} and the p_y, p_z of
// its in-face −neighbours (same block, or the edge neighbours (+1,−1,0) / (+1,0,−1) for y = 0 / z = 0),
// loaded into registers before the own primal step and consumed after it
struct XReg {
    float u, f, w, px, py, pz, m1, m2;
};
template <bool W8>
__device__ __forceinline__ XReg xface_load(const SkewTmaView &V, const int32_t *nb, int k) {
    const int y = k & 7, z = k >> 3;
    const int32_t b = nb[1];
    const uint32_t idx = b >= 0 ? (uint32_t)b * (uint32_t)kBlockVox + (uint32_t)(8 * k) : 0u;
    XReg r;
    r.u = V.u_in[idx];
    r.f = V.f[idx];
    r.w = W8 ? (float)V.W8[idx] : V.W[idx];
    r.px = V.px_in[idx];
    r.py = V.py_in[idx];
    r.pz = V.pz_in[idx];
    const int32_t b1 = y > 0 ? b : nb[8], b2 = z > 0 ? b : nb[10];
    const uint32_t i1 = b1 >= 0 ? (uint32_t)b1 * (uint32_t)kBlockVox + (uint32_t)(y > 0 ? 8 * k - 8 : 56 + 64 * z) : 0u;
    const uint32_t i2 = b2 >= 0 ? (uint32_t)b2 * (uint32_t)kBlockVox + (uint32_t)(z > 0 ? 8 * k - 64 : 8 * y + 448) : 0u;
    r.m1 = V.py_in[i1];
    r.m2 = V.pz_in[i2];
    if (b < 0) r.w = 0.0f;
    if (b1 < 0) r.m1 = 0.0f;
    if (b2 < 0) r.m2 = 0.0f;
    return r;
}

template <bool W8>
__global__ void __launch_bounds__(128, HVG_TMA_MINB) k_skew_tma(SkewTmaView V, const int32_t *__restrict__ nbr, int64_t first,
                                                     IterParams P) {
    __shared__ TStage<W8> S;
    __shared__ uint64_t bar;
    const int tid = threadIdx.x;
    // reverse store (Morton) order: the neighbours whose faces this launch reads tend to be L2-resident
    const int64_t row = first + (int64_t)gridDim.x - 1 - blockIdx.x;
    const uint32_t base = (uint32_t)row * (uint32_t)kBlockVox;
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_arrive_expect_tx(&bar, 5u * kBlockVox * 4u + (W8 ? kBlockVox : kBlockVox * 4u) + (V.frozen ? 64u : 0u) +
                                        kNbrTx);
    }
    if (!V.frozen && tid >= 32 && tid < 48) S.fz[tid - 32] = 0u;
    __syncwarp();
    if (tid < 32) {
        // warp 0: lanes 12-18 the block's own fields (no dependency), lanes 0-11 the neighbour row entry,
        // then lanes 2-11 that neighbour's planes / lines
        int32_t nb = -1;
        if (tid < kNbr) nb = ld_hint(nbr + kNbr * row + tid, policy_evict_last());
        switch (tid) {
            case 12: bulk_copy_g2s(S.f, V.f + base, kBlockVox * 4, &bar); break;
            case 13:
                if (W8)
                    bulk_copy_g2s(S.W8b, V.W8 + base, kBlockVox, &bar);
                else
                    bulk_copy_g2s(S.Wf, V.W + base, kBlockVox * 4, &bar);
                break;
            case 14: bulk_copy_g2s(S.u, V.u_in + base, kBlockVox * 4, &bar); break;
            case 15: bulk_copy_g2s(S.px, V.px_in + base, kBlockVox * 4, &bar); break;
            case 16: bulk_copy_g2s(S.py, V.py_in + base, kBlockVox * 4, &bar); break;
            case 17: bulk_copy_g2s(S.pz, V.pz_in + base, kBlockVox * 4, &bar); break;
            case 18:
                if (V.frozen) bulk_copy_g2s(S.fz, V.frozen + base / 32, 64, &bar);
                break;
            default: break;
        }
        if (tid < kNbr) {
            S.snb[tid] = nb;
            const CUtensorMap *M = V.maps;
            const int fu = kFieldU + V.ui, fx = kFieldPX + V.pi, fy = kFieldPY + V.pi, fz = kFieldPZ + V.pi;
            if (tid == 3 || tid == 5) {   // +y / +z face planes: u, f, W, p_x, p_y, p_z
                const int box = tid >> 1;
                float *dst = tid == 3 ? S.yf[0] : S.zf[0];
                const int fl[6] = {fu, kFieldF, kFieldW, fx, fy, fz};
#pragma unroll
                for (int q = 0; q < 6; q++) tma_load_4d(dst + q * 64, M + box * kMapFields + fl[q], 0, 0, 0, nb, &bar);
            } else if (tid != 0 && tid != 1 && tid != 8 && tid != 10) {   // x-face data: per-thread loads
                float *dst;
                int map, c0 = 0, c1 = 0, c2 = 0;
                switch (tid) {
                    case 2: dst = S.my; map = kBoxY * kMapFields + fy; c1 = 7; break;
                    case 4: dst = S.mz; map = kBoxZ * kMapFields + fz; c2 = 7; break;
                    case 6: dst = S.e6; map = kBoxD * kMapFields + fx; c0 = 4; break;
                    case 7: dst = S.e7; map = kBoxE * kMapFields + fx; c0 = 4; break;
                    case 9: dst = S.e9; map = kBoxF * kMapFields + fy; c1 = 7; break;
                    default: dst = S.e11; map = kBoxF * kMapFields + fz; c2 = 7; break;
                }
                tma_load_4d(dst, M + map, c0, c1, c2, nb, &bar);
            }
        }
    }
    __syncthreads();   // snb
    XReg xr;
    if (tid < 64) {
        xr = xface_load<W8>(V, S.snb, tid);
    } else {
        // −x neighbour p_x at (7, y, z), entry y + 8z
        const int k = tid - 64;
        const int32_t b = S.snb[0];
        const uint32_t idx = b >= 0 ? (uint32_t)b * (uint32_t)kBlockVox + (uint32_t)(7 + 8 * k) : 0u;
        const float v = V.px_in[idx];
        S.mx[k] = b >= 0 ? v : 0.0f;
    }
    mbar_wait(&bar, 0);
    __syncthreads();   // mx
    constexpr int NV = 4;
    const int x = tid & 7, y = (tid >> 3) & 7, z0 = (tid >> 6) * NV;
    const int c = tid & 63;
    const uint32_t vb = base + (uint32_t)(c + 64 * z0);
    const Add2 A2{P.one};
    float px[NV], py[NV], pz[NV], W[NV + 1];
    bool om[NV + 1];
#pragma unroll
    for (int k = 0; k < NV; k++) {
        const int i = c + 64 * (z0 + k);
        px[k] = S.px[i];
        py[k] = S.py[i];
        pz[k] = S.pz[i];
        if (W8) {
            W[k] = (float)S.W8b[i];
            S.Wf[i] = W[k];
        } else {
            W[k] = S.Wf[i];
        }
        om[k] = W[k] > 0.0f;
    }
    // 1a. primal step k + relaxation of the own voxels; ū^{k+1} in place of u^k in shared memory
    float pzm = z0 == 0 ? S.mz[x + 8 * y] : S.pz[c + 64 * (z0 - 1)];
#pragma unroll
    for (int k = 0; k < NV; k += 2) {
        const int i0 = c + 64 * (z0 + k), i1 = i0 + 64;
        const bool upd0 = om[k] && !((S.fz[i0 >> 5] >> (i0 & 31)) & 1u);
        const bool upd1 = om[k + 1] && !((S.fz[i1 >> 5] >> (i1 & 31)) & 1u);
        const float2 u = f2(S.u[i0], S.u[i1]);
        if (__any_sync(0xffffffffu, upd0 || upd1)) {
            const int z = z0 + k;
            const float2 pxm = f2(x > 0 ? S.px[i0 - 1] : S.mx[y + 8 * z], x > 0 ? S.px[i1 - 1] : S.mx[y + 8 * (z + 1)]);
            const float2 pym = f2(y > 0 ? S.py[i0 - 8] : S.my[x + 8 * z], y > 0 ? S.py[i1 - 8] : S.my[x + 8 * (z + 1)]);
            const float2 d = A2.add(A2.add(A2.sub(f2(px[k], px[k + 1]), pxm), A2.sub(f2(py[k], py[k + 1]), pym)),
                                    A2.sub(f2(pz[k], pz[k + 1]), f2(pzm, pz[k])));
            float2 ub2;
            const float2 un = primal_update2(u, f2(S.f[i0], S.f[i1]), f2(W[k], W[k + 1]), d, ub2, P);
            st_pred(V.u_out + (vb + 64 * k), un.x, upd0);
            st_pred(V.u_out + (vb + 64 * (k + 1)), un.y, upd1);
            if (upd0) S.u[i0] = ub2.x;
            if (upd1) S.u[i1] = ub2.y;
        }
        pzm = pz[k + 1];
    }
    // 1b. the primal step at the +face voxels (recomputed from the TMA'd planes): threads 0-63 the +x and
    // +z faces, 64-127 the +y face.  Same order as the owner: d = ((p_x − p_x(−x̂)) + (p_y − p_y(−ŷ))) + ...
    {
        auto face = [&](int A, int k) {
            const int c0 = k & 7, c1 = k >> 3;
            float u, f, w, qx, qy, qz, pxm, pym, pzm2;
            if (A == 0) {        // v = (0, y, z) of the +x neighbour, y = c0, z = c1 (registers)
                u = xr.u, f = xr.f, w = xr.w, qx = xr.px, qy = xr.py, qz = xr.pz;
                pxm = S.px[7 + 8 * c0 + 64 * c1];
                pym = xr.m1;
                pzm2 = xr.m2;
            } else if (A == 1) { // v = (x, 0, z) of the +y neighbour, x = c0, z = c1
                u = S.yf[0][k], f = S.yf[1][k], w = S.yf[2][k], qx = S.yf[3][k], qy = S.yf[4][k], qz = S.yf[5][k];
                pxm = c0 > 0 ? S.yf[3][k - 1] : S.e6[4 * c1 + 3];
                pym = S.py[c0 + 56 + 64 * c1];
                pzm2 = c1 > 0 ? S.yf[5][k - 8] : S.e11[c0];
            } else {             // v = (x, y, 0) of the +z neighbour, x = c0, y = c1
                u = S.zf[0][k], f = S.zf[1][k], w = S.zf[2][k], qx = S.zf[3][k], qy = S.zf[4][k], qz = S.zf[5][k];
                pxm = c0 > 0 ? S.zf[3][k - 1] : S.e7[4 * c1 + 3];
                pym = c1 > 0 ? S.zf[4][k - 8] : S.e9[c0];
                pzm2 = S.pz[c0 + 8 * c1 + 448];
            }
            float ub = u;
            if (w > 0.0f) {
                const float d = ((qx - pxm) + (qy - pym)) + (qz - pzm2);
                (void)primal_update(u, f, w, d, ub, P);
            }
            S.u[kBlockVox + 64 * A + k] = ub;
            S.Wf[kBlockVox + 64 * A + k] = w;
        };
        if (tid < 64) {
            face(0, tid);
            face(2, tid);
        } else {
            face(1, tid - 64);
        }
    }
    __syncthreads();
    // 2. dual step k + 1 of the own voxels from ū^{k+1} (shared) and p^{k+1} (registers)
    {
        const int iz = z0 + NV < 8 ? c + 64 * (z0 + NV) : kBlockVox + 128 + (x + 8 * y);
        W[NV] = S.Wf[iz];
        om[NV] = W[NV] > 0.0f;
    }
    const int fxo = kBlockVox + (y + 8 * z0);
    const int fyo = kBlockVox + 64 + (x + 8 * z0);
    const int fzo = kBlockVox + 128 + (x + 8 * y);
#pragma unroll
    for (int k = 0; k < NV; k += 2) {
        if (!__any_sync(0xffffffffu, om[k] || om[k + 1])) continue;
        const int i0 = c + 64 * (z0 + k), i1 = i0 + 64;
        const int ix0 = x < 7 ? i0 + 1 : fxo + 8 * k, ix1 = x < 7 ? i1 + 1 : fxo + 8 * (k + 1);
        const int iy0 = y < 7 ? i0 + 8 : fyo + 8 * k, iy1 = y < 7 ? i1 + 8 : fyo + 8 * (k + 1);
        const int iz1 = z0 + k + 2 < 8 ? i1 + 64 : fzo;
        const float2 ubx = f2(S.u[ix0], S.u[ix1]), uby = f2(S.u[iy0], S.u[iy1]);
        const bool ex0 = om[k] && S.Wf[ix0] > 0.0f, ex1 = om[k + 1] && S.Wf[ix1] > 0.0f;
        const bool ey0 = om[k] && S.Wf[iy0] > 0.0f, ey1 = om[k + 1] && S.Wf[iy1] > 0.0f;
        const bool ez0 = om[k] && om[k + 1], ez1 = om[k + 1] && om[k + 2];
        float2 qx = f2(px[k], px[k + 1]), qy = f2(py[k], py[k + 1]), qz = f2(pz[k], pz[k + 1]);
        dual_update2(f2(S.u[i0], S.u[i1]), ubx, uby, f2(S.u[i1], S.u[iz1]), ex0, ex1, ey0, ey1, ez0, ez1, qx, qy, qz,
                     P);
        st_pred(V.px_out + (vb + 64 * k), qx.x, om[k]);
        st_pred(V.py_out + (vb + 64 * k), qy.x, om[k]);
        st_pred(V.pz_out + (vb + 64 * k), qz.x, om[k]);
        st_pred(V.px_out + (vb + 64 * (k + 1)), qx.y, om[k + 1]);
        st_pred(V.py_out + (vb + 64 * (k + 1)), qy.y, om[k + 1]);
        st_pred(V.pz_out + (vb + 64 * (k + 1)), qz.y, om[k + 1]);
    }
}

int launch_skew_tma(const Fields &F, int ui, int p_in, const uint32_t *frozen, const int32_t *nbr, int64_t first,
                    int64_t n_blocks, const IterParams &P, cudaStream_t s) {
    if (n_blocks == 0) return 0;
    const int o = p_in ^ 1;
    const float *u_in = ui ? F.u2 : F.u;
    float *u_out = ui ? F.u : F.u2;
    SkewTmaView V{F.f,       F.W,       F.W8,      frozen,    u_in,
                  u_out,     F.px[p_in], F.py[p_in], F.pz[p_in], F.px[o],
                  F.py[o],   F.pz[o],   reinterpret_cast<const CUtensorMap *>(F.tmaps), ui, p_in};
    if (F.W8)
        k_skew_tma<true><<<(unsigned)n_blocks, 128, 0, s>>>(V, nbr, first, P);
    else
        k_skew_tma<false><<<(unsigned)n_blocks, 128, 0, s>>>(V, nbr, first, P);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

}  // namespace hvg
