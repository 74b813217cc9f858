// extract.cu — Ω-restricted isosurface extraction of the regularised TSDF (paper
// P:102 "regularise the model in 3D space, extract the surface", P:132-133 zero-crossing level set).
// Readings X-1 … X-7: marching tetrahedra over the cells of fully observed voxels.
//
//   k_extract<false>  one 128-thread CTA per store row: stage the 9×9×9 tile of values and
//                     "usable" flags (allocated ∧ W > 0 ∧ W >= w_min) of the block and its +x/+y/+z
//                     neighbours (face, edge and corner blocks reached by neighbour-table chains: if an
//                     intermediate block is missing, every cell needing the chained block has a corner
//                     in the missing one, so it is skipped anyway); each thread counts the triangles of
//                     its 4 cells; per-thread counts go to scratch, the block total to counts[caller].
//   exclusive scan of the per-block totals in caller order → triangle offsets (deterministic output
//   order X-7: caller block order, cell order, tetrahedron order, triangle order).
//   k_extract<true>   same CTA layout: block scan of the per-thread counts, then each thread writes
//                     its triangles at offset[caller] + prefix.
// Vertex arithmetic is fp32 in the written order of X-4 (bit-identical to the oracle).
#include <cuda_runtime.h>

#include "../../include/vol.h"
#include "handle.h"
#include "internal.h"

namespace hvg {

namespace {

constexpr int kT = 9;             // tile edge: 8 own voxels + 1 from the + neighbours
constexpr int kTile = kT * kT * kT;

struct ExArgs {
    const float *val;      // [S][512] field (u or f), store rows
    const float *W;        // [S][512]
    const int32_t *nbr;    // [S][12]
    const int32_t *perm;   // [n] caller index of store row
    const int32_t *xyz;    // [n][3] caller order
    float voxel, w_min;
};

// Cube corners are coded c = i + 2j + 4k for the offset (i, j, k) ∈ {0,1}^3 from the cell origin.

// Voxel-centre coordinates of one cell: X[b][k] = fl(fl((float)(o_k + b) + ½)·v) for the cell origin o
// and b ∈ {0, 1}, and dX[k] = fl(X[1][k] − X[0][k]).  Every quantity of X-4 is one of these: P_lo and
// P_hi of an edge are corner coordinates, and P_hi − P_lo is ±dX[k] on an axis where the ends differ
// (fl(a − b) = −fl(b − a)) and 0 where they agree — where p = P_lo + t·0 = P_lo exactly (P_lo ≠ 0).
struct CellGeom {
    float X[2][3];
    float dX[3];
};
__device__ __forceinline__ CellGeom cell_geom(int ox, int oy, int oz, float voxel) {
    CellGeom G;
    const int o[3] = {ox, oy, oz};
#pragma unroll
    for (int k = 0; k < 3; k++) {
        G.X[0][k] = __fmul_rn(__fadd_rn((float)o[k], 0.5f), voxel);
        G.X[1][k] = __fmul_rn(__fadd_rn((float)(o[k] + 1), 0.5f), voxel);
        G.dX[k] = __fsub_rn(G.X[1][k], G.X[0][k]);
    }
    return G;
}

// X-4: vertex on the edge between cell corners ca and cb (values ua, ub).  The ends are ordered by global
// voxel coordinate, lexicographically in (x, y, z).  The corners of a Freudenthal tetrahedron are nested
// (000 ⊂ e_a ⊂ e_a + e_b ⊂ 111), so of any two corners one is a bitwise subset of the other — the lower end,
// lexicographically first as well: lo = ca & cb, and the axes where the ends differ are d = ca ^ cb.
// t = u_lo/(u_lo − u_hi), p = P_lo + t·(P_hi − P_lo) per coordinate, in fp32 (the oracle's written order):
// on an axis in d, P_lo = X[0] and P_hi − P_lo = dX; elsewhere p = P_lo exactly.
__device__ __forceinline__ void edge_vertex(const CellGeom &G, int ca, float ua, int cb, float ub, float *p) {
    const int lo = ca & cb, d = ca ^ cb;
    const float ulo = lo == ca ? ua : ub, uhi = lo == ca ? ub : ua;
    const float t = __fdiv_rn(ulo, __fsub_rn(ulo, uhi));
#pragma unroll
    for (int k = 0; k < 3; k++)
        p[k] = ((d >> k) & 1) ? __fadd_rn(G.X[0][k], __fmul_rn(t, G.dX[k])) : G.X[(lo >> k) & 1][k];
}

// X-6: a triangle is dropped iff its area is zero in exact arithmetic, decided on the corner values (an
// edge vertex sits on its outside corner iff that corner's value is exactly 0), never on rounded vertices.
template <bool EMIT>
__device__ __forceinline__ void put(float *out, unsigned &m, const float *p0, const float *p1, const float *p2,
                                    bool degenerate) {
    if (degenerate) return;   // X-6
    if (EMIT) {
        float *o = out + 9ull * m;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            o[k] = p0[k];
            o[3 + k] = p1[k];
            o[6 + k] = p2[k];
        }
    }
    m++;
}

__device__ __forceinline__ float sel4f(int i, float a0, float a1, float a2, float a3) {
    return i == 0 ? a0 : (i == 1 ? a1 : (i == 2 ? a2 : a3));
}

// One tetrahedron with corner codes (k0, k1, k2, k3) in positively oriented order (X-2) and values
// (v0 … v3).  X-5: the lone corner (nin = 1: the inside one, nin = 3: the outside one) or the inside pair
// goes first, the remaining corners follow in tetrahedron order, and the last two are swapped when that
// permutation is odd, so (a, b, c, d) stays positively oriented.
template <bool EMIT>
__device__ __forceinline__ void tet(int k0, int k1, int k2, int k3, float v0, float v1, float v2, float v3,
                                    const CellGeom &G, float *out, unsigned &m) {
    const int mask = (v0 < 0.0f) | ((v1 < 0.0f) << 1) | ((v2 < 0.0f) << 2) | ((v3 < 0.0f) << 3);   // X-3
    if (mask == 0 || mask == 15) return;
    const int nin = __popc(mask);
    int pa, pb, pc, pd;
    if (nin == 2) {
        // inside positions i < j first, then outside k < l; parity = inversions between the two groups
        const int i = __ffs(mask) - 1, j = 31 - __clz(mask);
        const int om = (~mask) & 15;
        const int k = __ffs(om) - 1, l = 31 - __clz(om);
        const int inv = (k < i) + (l < i) + (k < j) + (l < j);
        pa = i;
        pb = j;
        pc = (inv & 1) ? l : k;
        pd = (inv & 1) ? k : l;
    } else {
        const int lone = nin == 1 ? mask : ((~mask) & 15);
        const int a = __ffs(lone) - 1;
        // remaining positions in order; moving a to the front costs a transpositions
        const int r0 = a == 0 ? 1 : 0, r1 = a <= 1 ? 2 : 1, r2 = a <= 2 ? 3 : 2;
        pa = a;
        pb = r0;
        pc = (a & 1) ? r2 : r1;
        pd = (a & 1) ? r1 : r2;
    }
    const int packed = k0 | (k1 << 4) | (k2 << 8) | (k3 << 12);   // corner code of position i at bits 4i
    const int ca = (packed >> (4 * pa)) & 15, cb = (packed >> (4 * pb)) & 15;
    const int cc = (packed >> (4 * pc)) & 15, cd = (packed >> (4 * pd)) & 15;
    const float ua = sel4f(pa, v0, v1, v2, v3), ub = sel4f(pb, v0, v1, v2, v3);
    const float uc = sel4f(pc, v0, v1, v2, v3), ud = sel4f(pd, v0, v1, v2, v3);
    float e1[3], e2[3], e3[3];
    if (nin != 2) {
        edge_vertex(G, ca, ua, cb, ub, e1);
        edge_vertex(G, ca, ua, cc, uc, e2);
        edge_vertex(G, ca, ua, cd, ud, e3);
        // 1 inside: never degenerate; 1 outside (a): all three vertices sit on a iff u_a = 0
        if (nin == 1) put<EMIT>(out, m, e1, e2, e3, false);
        else put<EMIT>(out, m, e1, e3, e2, ua == 0.0f);
    } else {
        float e4[3];
        edge_vertex(G, ca, ua, cc, uc, e1);   // E_ac
        edge_vertex(G, ca, ua, cd, ud, e2);   // E_ad
        edge_vertex(G, cb, ub, cd, ud, e3);   // E_bd
        edge_vertex(G, cb, ub, cc, uc, e4);   // E_bc
        put<EMIT>(out, m, e1, e2, e3, ud == 0.0f);   // E_ad = E_bd iff u_d = 0
        put<EMIT>(out, m, e1, e3, e4, uc == 0.0f);   // E_ac = E_bc iff u_c = 0
    }
}

// X-2: the 6 Freudenthal tetrahedra 000 → e_a → e_a + e_b → 111 for the axis permutations (a, b, c) in
// lexicographic order; odd permutations list their last two corners swapped (positive orientation):
//   (0,1,2): 0 1 3 7   (0,2,1): 0 1 7 5   (1,0,2): 0 2 7 3   (1,2,0): 0 2 6 7   (2,0,1): 0 4 5 7   (2,1,0): 0 4 7 6
// corner codes k1 k2 k3 of tetrahedron q, 4 bits each (k1 lowest), 12 bits per tetrahedron
constexpr unsigned long long kTetLo = 0x731ull | (0x571ull << 12) | (0x372ull << 24);
constexpr unsigned long long kTetHi = 0x762ull | (0x754ull << 12) | (0x674ull << 24);
__device__ __forceinline__ int tet_code(int q, int r) {   // r = 1, 2, 3
    const unsigned long long w = q < 3 ? kTetLo : kTetHi;
    return (int)((w >> (12 * (q < 3 ? q : q - 3) + 4 * (r - 1))) & 0xF);
}

__device__ __forceinline__ int tile_index(int cx, int cy, int cz, int code) {
    return (cx + (code & 1)) + kT * (cy + ((code >> 1) & 1)) + kT * kT * (cz + (code >> 2));
}

constexpr int kMaxItems = 512 * 6;   // (cell, tetrahedron) pairs of one block
constexpr int kItemWords = 2 * kMaxItems / 32;   // 2 count bits per item

// Two phases per CTA: (A) every thread tests its 4 cells (all corners usable, mixed signs) and their
// 6 tetrahedra (mixed signs) and appends the crossing (cell, tetrahedron) items to a shared list in
// cell, tetrahedron order; (B) the 128 threads process the items round-robin — the same code path for
// every lane, instead of each lane walking its own cells' varying tetrahedra.  The count pass stores
// the triangles of every item (0, 1 or 2 after the X-6 drop) for the emit pass as 2 bits per item:
// item_bits[row][2·(4·round + warp) + b] = bit b of the counts of the warp's 32 items (ballots).
template <bool EMIT>
__global__ void __launch_bounds__(128) k_extract(ExArgs A, int64_t n_rows, uint32_t *__restrict__ block_counts,
                                                 uint32_t *__restrict__ item_bits,
                                                 const uint32_t *__restrict__ offsets, float *__restrict__ out) {
    __shared__ float su[kTile];
    __shared__ uint8_t sok[kTile];
    __shared__ uint16_t sitem[kMaxItems];   // cell (9 bits) << 3 | tetrahedron (3 bits)
    __shared__ int32_t srow[8];
    __shared__ uint32_t swarp[4];
    // emit pass: one round's triangles (≤ 2 per item) staged here, then written out by the whole CTA
    // with consecutive lanes on consecutive floats (coalesced) instead of 9 scattered 4-byte stores
    // per triangle 36 B apart
    __shared__ float sout[EMIT ? 2 * 128 * 9 : 1];   // 4 warp slices of 2 triangles x 32 lanes
    __shared__ uint32_t goff[EMIT ? kMaxItems / 32 : 1];   // triangle offset of each 32-item group
    const int64_t r = blockIdx.x;
    if (r >= n_rows) return;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    if (t == 0) {
        // blocks of the tile: index dx + 2dy + 4dz; chains +x → +y → +z (a missing intermediate block
        // holds a corner of every cell that needs the chained block, so such cells are skipped anyway)
        const int32_t *N = A.nbr;
        const int32_t bx = N[12 * r + 1], by = N[12 * r + 3], bz = N[12 * r + 5];
        const int32_t bxy = bx >= 0 ? N[12 * bx + 3] : -1;
        const int32_t bxz = bx >= 0 ? N[12 * bx + 5] : -1;
        const int32_t byz = by >= 0 ? N[12 * by + 5] : -1;
        const int32_t bxyz = bxy >= 0 ? N[12 * bxy + 5] : -1;
        srow[0] = (int32_t)r;
        srow[1] = bx;
        srow[2] = by;
        srow[3] = bxy;
        srow[4] = bz;
        srow[5] = bxz;
        srow[6] = byz;
        srow[7] = bxyz;
    }
    __syncthreads();
    for (int i = t; i < kTile; i += 128) {
        const int x = i % kT, y = (i / kT) % kT, z = i / (kT * kT);
        const int blk = srow[(x >> 3) + 2 * (y >> 3) + 4 * (z >> 3)];
        float uv = 0.0f;
        uint8_t ok = 0;
        if (blk >= 0) {
            const int64_t o = (int64_t)blk * kBlockVox + (x & 7) + 8 * (y & 7) + 64 * (z & 7);
            const float w = A.W[o];
            uv = A.val[o];
            ok = (w > 0.0f && w >= A.w_min) ? 1 : 0;   // X-1
        }
        su[i] = uv;
        sok[i] = ok;
    }
    __syncthreads();
    const int32_t ci = A.perm[r];
    const int gx = 8 * A.xyz[3 * ci], gy = 8 * A.xyz[3 * ci + 1], gz = 8 * A.xyz[3 * ci + 2];
    // (A) cells 4t … 4t+3 (voxel order): x = 4(t&1) + q, y = (t>>1)&7, z = t>>4
    const int cy = (t >> 1) & 7, cz = t >> 4;
    uint32_t tets = 0;   // bit 6q + k: tetrahedron k of cell q crosses the level set
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int cx = 4 * (t & 1) + q;
        bool ok = true;
        int neg = 0;
#pragma unroll
        for (int c8 = 0; c8 < 8; c8++) {
            const int idx = tile_index(cx, cy, cz, c8);
            ok = ok && sok[idx];
            neg |= (su[idx] < 0.0f) << c8;   // X-3
        }
        if (!ok || neg == 0 || neg == 255) continue;
        uint32_t tm = 0;
#pragma unroll
        for (int k = 0; k < 6; k++) {
            const int m4 = (neg & 1) | (((neg >> tet_code(k, 1)) & 1) << 1) | (((neg >> tet_code(k, 2)) & 1) << 2) |
                           (((neg >> tet_code(k, 3)) & 1) << 3);
            tm |= (uint32_t)(m4 != 0 && m4 != 15) << k;
        }
        tets |= tm << (6 * q);
    }
    const uint32_t mine = __popc(tets);
    uint32_t x = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) swarp[wid] = x;
    __syncthreads();
    uint32_t pos = x - mine;
    for (int w = 0; w < wid; w++) pos += swarp[w];
    const uint32_t n_items = swarp[0] + swarp[1] + swarp[2] + swarp[3];
    while (tets) {
        const int bit = __ffs(tets) - 1;
        tets &= tets - 1;
        const int q = bit / 6, k = bit - 6 * q;
        sitem[pos++] = (uint16_t)(((4 * t + q) << 3) | k);
    }
    __syncthreads();
    // (B) items in list order.  Count pass: round-robin, item i = t + 128·round, 2 count bits per item
    // stored per 32-item group (ballots).  Emit pass: the group totals (popcounts of those bits) are scanned
    // once per block; then each warp takes whole groups (w, w + 4, …), places its lanes' triangles with a
    // warp scan at the group's offset, stages them in its own slice of shared memory and writes them out
    // with consecutive lanes on consecutive floats — no block-wide barrier inside the loop.
    uint32_t block_total = 0;    // count pass: triangles of this thread's items
    if (EMIT) {
        const uint32_t ng = (n_items + 31) / 32;   // <= kMaxItems / 32 = 96
        const uint32_t *wbb = item_bits + (size_t)r * kItemWords;
        if (wid == 0) {
            uint32_t c3[3], sum = 0;
#pragma unroll
            for (int j = 0; j < 3; j++) {
                const uint32_t g = 3 * lane + j;
                c3[j] = g < ng ? __popc(wbb[2 * g]) + 2 * __popc(wbb[2 * g + 1]) : 0u;
                sum += c3[j];
            }
            uint32_t inc = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            uint32_t ex = inc - sum;
#pragma unroll
            for (int j = 0; j < 3; j++) {
                goff[3 * lane + j] = ex;
                ex += c3[j];
            }
        }
        __syncthreads();
        float *wsout = sout + wid * (2 * 32 * 9);
        float *base_out = out + 9ull * offsets[ci];
        for (uint32_t g = wid; g < ng; g += 4) {
            const uint32_t i = 32 * g + lane;
            const uint32_t w0 = wbb[2 * g], w1 = wbb[2 * g + 1];
            const uint32_t cnt = i < n_items ? (((w0 >> lane) & 1u) | (((w1 >> lane) & 1u) << 1)) : 0u;
            uint32_t y = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) y += z;
            }
            const uint32_t gtot = __shfl_sync(0xffffffffu, y, 31);
            if (cnt) {
                const int cell = sitem[i] >> 3, k = sitem[i] & 7;
                const int cx = cell & 7, cyy = (cell >> 3) & 7, czz = cell >> 6;
                const int k1 = tet_code(k, 1), k2 = tet_code(k, 2), k3 = tet_code(k, 3);
                unsigned m = 0;
                const CellGeom G = cell_geom(gx + cx, gy + cyy, gz + czz, A.voxel);
                tet<true>(0, k1, k2, k3, su[tile_index(cx, cyy, czz, 0)], su[tile_index(cx, cyy, czz, k1)],
                          su[tile_index(cx, cyy, czz, k2)], su[tile_index(cx, cyy, czz, k3)], G,
                          wsout + 9 * (y - cnt), m);
            }
            __syncwarp();
            float *dst = base_out + 9ull * goff[g];
            for (uint32_t j = lane; j < 9 * gtot; j += 32) dst[j] = wsout[j];
            __syncwarp();
        }
    } else {
        for (uint32_t i0 = 0; i0 < n_items; i0 += 128) {
            const uint32_t i = i0 + t;
            int cell = 0, k = 0;
            if (i < n_items) {
                cell = sitem[i] >> 3;
                k = sitem[i] & 7;
            }
            const int cx = cell & 7, cyy = (cell >> 3) & 7, czz = cell >> 6;
            const int k1 = tet_code(k, 1), k2 = tet_code(k, 2), k3 = tet_code(k, 3);
            unsigned m = 0;
            if (i < n_items)
                tet<false>(0, k1, k2, k3, su[tile_index(cx, cyy, czz, 0)], su[tile_index(cx, cyy, czz, k1)],
                           su[tile_index(cx, cyy, czz, k2)], su[tile_index(cx, cyy, czz, k3)], CellGeom{}, nullptr, m);
            const uint32_t b0 = __ballot_sync(0xffffffffu, m & 1u), b1 = __ballot_sync(0xffffffffu, (m >> 1) & 1u);
            if (lane == 0 && i0 + 32 * wid < n_items) {
                uint32_t *wb = item_bits + (size_t)r * kItemWords + 2 * ((i0 >> 5) + wid);
                wb[0] = b0;
                wb[1] = b1;
            }
            block_total += m;
        }
    }
    if (!EMIT) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) block_total += __shfl_xor_sync(0xffffffffu, block_total, o);
        __syncthreads();
        if (lane == 0) swarp[wid] = block_total;
        __syncthreads();
        if (t == 0) block_counts[ci] = swarp[0] + swarp[1] + swarp[2] + swarp[3];
    }
}

}  // namespace

}  // namespace hvg

using namespace hvg;

extern "C" vol_status vol_extract(vol_t v, int field, float voxel, float w_min, float *tris, int64_t max_tris,
                                  int64_t *n_tris) {
    NvtxRange nvtx_range_("vol_extract");
    if (!v || !n_tris) return fail(VOL_EINVAL, "vol_extract: NULL argument");
    *n_tris = 0;
    if (v->shard) return fail(VOL_ENOTSUP, "vol_extract: sharded volumes are not supported (extract per GPU volume)");
    if (field != 0 && field != 1) return fail(VOL_EINVAL, "vol_extract: field must be 0 (u) or 1 (f)");
    if (!(voxel > 0.0f) || !(voxel < 1e30f)) return fail(VOL_EINVAL, "vol_extract: voxel must be > 0");
    if (!(w_min >= 0.0f) || !(w_min < 1e30f)) return fail(VOL_EINVAL, "vol_extract: w_min must be finite and >= 0");
    if (tris && max_tris < 0) return fail(VOL_EINVAL, "vol_extract: max_tris < 0");
    const int64_t n = v->L.n_local;
    cudaStream_t s = v->stream;
    uint32_t *counts = v->d_count;                                   // [n] (build scratch, T >= 2n)
    uint32_t *offs = v->d_hash;                                      // [n + 1] (build scratch)
    // [n][192] words: 2 bits per (cell, tetrahedron) item (768 B per block <= the 2 KiB per block of d_tmp)
    uint32_t *tcounts = reinterpret_cast<uint32_t *>(v->d_tmp);
    ExArgs A{field == 0 ? v->F.u : v->F.f, v->F.W, v->d_nbr, v->d_perm, v->d_xyz, voxel, w_min};
    k_extract<false><<<(unsigned)n, 128, 0, s>>>(A, n, counts, tcounts, nullptr, nullptr);
    CK(cudaPeekAtLastError());
    counted(1);
    CKL(launch_exclusive_scan_u32(counts, offs, n, v->d_scan, s));
    uint32_t total = 0;
    CK(cudaMemcpyAsync(&total, offs + n, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *n_tris = (int64_t)total;
    if (!tris) return VOL_OK;
    if ((int64_t)total > max_tris)
        return fail(VOL_ENOMEM, "vol_extract: %lld triangles > max_tris = %lld", (long long)total, (long long)max_tris);
    if (total == 0) return VOL_OK;
    const bool dev = is_device_ptr(tris);
    float *out = tris;
    if (!dev) CK(cudaMallocAsync((void **)&out, (size_t)total * 36, s));
    k_extract<true><<<(unsigned)n, 128, 0, s>>>(A, n, nullptr, tcounts, offs, out);
    cudaError_t e = cudaPeekAtLastError();
    if (e == cudaSuccess) counted(1);
    if (!dev) {
        if (e == cudaSuccess) e = cudaMemcpyAsync(tris, out, (size_t)total * 36, cudaMemcpyDeviceToHost, s);
        cudaFreeAsync(out, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
    if (e != cudaSuccess) return fail(VOL_ECUDA, "vol_extract: %s", cudaGetErrorString(e));
    return VOL_OK;
}
