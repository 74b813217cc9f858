// extract.cu — Ω-restricted isosurface extraction of the regularised TSDF (paper
// P:102 "regularise the model in 3D space, extract the surface", P:132-133 zero-crossing level set).
// Readings X-1 … X-7: marching tetrahedra over the cells of fully observed voxels.
//
//   k_extract<true>   the ordered single pass: CTAs take caller blocks in ticket order; each stages the
//                     9×9×9 tile of values and "usable" flags (allocated ∧ W > 0 ∧ W >= w_min) of its block
//                     and the +x/+y/+z neighbours (face, edge and corner blocks reached by neighbour-table
//                     chains: if an intermediate block is missing, every cell needing the chained block has
//                     a corner in the missing one, so it is skipped anyway), counts the triangles of every
//                     (cell, tetrahedron) from corner signs and zeros alone, finds the triangle offset of its
//                     block by decoupled look-back over its predecessors in caller order (deterministic
//                     output order X-7: caller block, cell, tetrahedron, triangle) and writes its triangles.
//   k_extract<false>  the counting half alone (count-only calls; sizing a host buffer's staging copy).
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
        p[k] = ((d >> k) & 1) ? __fadd_rn(G.X[0][k], __fmul_rn(t, G.dX[k])) : (((lo >> k) & 1) ? G.X[1][k] : G.X[0][k]);
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

// Triangles of one tetrahedron (X-5, X-6), from its 4-bit inside mask (bit i: corner i has value < 0, X-3)
// and its 4-bit mask of corners with value ≠ 0: one for a lone inside corner; otherwise one per outside
// corner whose value is not exactly 0 (X-6: with 3 inside, the triangle degenerates iff the outside corner is
// 0; with 2 inside, the quad's (E_ac, E_ad, E_bd) iff u_d = 0 and (E_ac, E_bd, E_bc) iff u_c = 0).
__device__ __forceinline__ uint32_t tet_triangles(int m4, int nz4) {
    if (m4 == 0 || m4 == 15) return 0u;
    return __popc(m4) == 1 ? 1u : (uint32_t)__popc(nz4 & ~m4 & 15);
}

// Corner codes and tile offsets of the 4 corners of tetrahedron q, one byte per corner (corner 0 first):
// code c ↔ tile offset (c & 1) + 9·((c >> 1) & 1) + 81·(c >> 2) from the cell's origin in the 9³ tile.
__host__ __device__ constexpr int tile_off(int c) { return (c & 1) + kT * ((c >> 1) & 1) + kT * kT * (c >> 2); }
__device__ __forceinline__ uint2 tet_words(int q) {
    const int k1 = tet_code(q, 1), k2 = tet_code(q, 2), k3 = tet_code(q, 3);
    return make_uint2((uint32_t)((k1 << 8) | (k2 << 16) | (k3 << 24)),
                      (uint32_t)((tile_off(k1) << 8) | (tile_off(k2) << 16) | (tile_off(k3) << 24)));
}
__device__ __forceinline__ uint32_t byte_of(uint32_t w, int i) { return __byte_perm(w, 0u, 0x4440u | (uint32_t)i); }

// One tetrahedron (corner codes and tile offsets TW = tet_words, positively oriented order, X-2) of the
// cell whose origin is sb[0] in the staged tile, values v0 … v3.  X-5: the lone corner (nin = 1: the inside
// one, nin = 3: the outside one) or the inside pair goes first, the remaining corners follow in tetrahedron
// order, and the last two are swapped when that permutation is odd, so (a, b, c, d) stays positively
// oriented.  Triangles: 1 inside (E_ab, E_ac, E_ad), 3 inside (E_ab, E_ad, E_ac), 2 inside (E_ac, E_ad, E_bd)
// + (E_ac, E_bd, E_bc); with the edges
//   E0 = (a, quad ? c : b), E1 = (a, quad ? d : c), E2 = (quad ? b : a, d), E3 = (b, c)
// these are (E0, E1, E2) [(E0, E2, E1) for 3 inside] and (E0, E2, E3): one code path for every case (the
// lanes of a warp hold mixed cases).  The surviving triangles (X-6) are written to o[0 …], 9 floats each.
__device__ __forceinline__ void tet_emit(uint2 TW, const float *sb, float v0, float v1, float v2, float v3,
                                         const CellGeom &G, float *o) {
    const int mask = (v0 < 0.0f) | ((v1 < 0.0f) << 1) | ((v2 < 0.0f) << 2) | ((v3 < 0.0f) << 3);   // X-3
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
    const int ca = (int)byte_of(TW.x, pa), cb = (int)byte_of(TW.x, pb);
    const int cc = (int)byte_of(TW.x, pc), cd = (int)byte_of(TW.x, pd);
    const float ua = sb[byte_of(TW.y, pa)], ub = sb[byte_of(TW.y, pb)];
    const float uc = sb[byte_of(TW.y, pc)], ud = sb[byte_of(TW.y, pd)];
    const bool quad = nin == 2;
    float e0[3], e1[3], e2[3];
    edge_vertex(G, ca, ua, quad ? cc : cb, quad ? uc : ub, e0);
    edge_vertex(G, ca, ua, quad ? cd : cc, quad ? ud : uc, e1);
    edge_vertex(G, quad ? cb : ca, quad ? ub : ua, cd, ud, e2);
    const bool drop1 = quad ? ud == 0.0f : (nin == 3 && ua == 0.0f);   // X-6
    const bool sw = nin == 3;
    if (!drop1) {
#pragma unroll
        for (int k = 0; k < 3; k++) {
            o[k] = e0[k];
            o[3 + k] = sw ? e2[k] : e1[k];
            o[6 + k] = sw ? e1[k] : e2[k];
        }
        o += 9;
    }
    if (quad && uc != 0.0f) {   // X-6
        float e3[3];
        edge_vertex(G, cb, ub, cc, uc, e3);
#pragma unroll
        for (int k = 0; k < 3; k++) {
            o[k] = e0[k];
            o[3 + k] = e2[k];
            o[6 + k] = e3[k];
        }
    }
}

constexpr int kMaxItems = 512 * 6;   // (cell, tetrahedron) pairs of one block
constexpr int kSlice = 64 * 9 + 4;   // floats of one warp's staging slice: 64 triangles + alignment shift

// Output of one call.  Count pass (EMIT = false): only *total (atomic sum of the block totals).  Emit pass:
// CTAs take caller blocks in ticket order and find their triangle offset by decoupled look-back over the
// per-block words state[i] = flag << 62 | value (flag 1: the block's own total, 2: inclusive prefix), so one
// pass both counts and writes in the deterministic order of X-7; triangles at index >= max_tris are not
// written.
struct ExOut {
    const int32_t *inv;                  // [n] store row of caller block i
    unsigned long long *state;           // [n] look-back words (zeroed)
    unsigned *ticket;                    // CTA ticket (zeroed)
    unsigned long long *total;           // triangles of the call (zeroed)
    float *out;                          // 16-byte aligned when vec
    long long max_tris;
    int vec;
};

constexpr unsigned long long kAgg = 1ull << 62, kInc = 2ull << 62, kVal = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p) {
    return *reinterpret_cast<const volatile unsigned long long *>(p);
}
__device__ __forceinline__ void st_volatile(unsigned long long *p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long *>(p) = v;
}

// One 128-thread CTA per block: stage the 9³ tile; (A) every thread tests its 4 cells (all corners usable,
// mixed signs) and their 6 tetrahedra and counts each one's triangles (tet_triangles: a function of the
// corner signs and zeros alone); a block scan places the (cell, tetrahedron) items with triangles in a shared
// list in cell, tetrahedron order, each with its triangle offset inside the block; (B, emit pass) after the
// look-back, each warp takes whole 32-item groups (w, w + 4, …), computes their triangles into its own
// slice of shared memory and writes them out with consecutive lanes on consecutive floats.
template <bool EMIT>
__global__ void __launch_bounds__(128) k_extract(ExArgs A, int64_t n_rows, ExOut O) {
    __shared__ float su[kTile];
    __shared__ uint8_t sok[kTile];
    __shared__ uint16_t sitem[EMIT ? kMaxItems : 1];       // cell (9 bits) << 3 | tetrahedron (3 bits)
    __shared__ uint16_t soff[EMIT ? kMaxItems + 1 : 1];    // triangle offset of each item in the block
    __shared__ int32_t srow[8];
    __shared__ uint32_t swarp[4];
    __shared__ __align__(16) float sout[EMIT ? 4 * kSlice : 1];   // 4 warp slices of 64 triangles (+ align)
    __shared__ uint2 stw[6];                                 // tet_words of the 6 tetrahedra
    __shared__ unsigned long long s_base;
    __shared__ int64_t s_ci;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    int64_t r, ci = 0;
    if (EMIT) {
        if (t == 0) s_ci = (int64_t)atomicAdd(O.ticket, 1u);
        __syncthreads();
        ci = s_ci;
        r = O.inv[ci];
    } else {
        r = blockIdx.x;
    }
    if (EMIT && t < 6) stw[t] = tet_words(t);
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
    // the caller block's origin (emit pass), loaded before the tile so its latency overlaps the staging
    int gx = 0, gy = 0, gz = 0;
    if (EMIT) {
        const int32_t cidx = A.perm[r];
        gx = 8 * A.xyz[3 * cidx];
        gy = 8 * A.xyz[3 * cidx + 1];
        gz = 8 * A.xyz[3 * cidx + 2];
    }
    {
        constexpr int kIt = (kTile + 127) / 128;   // 6 loads of u and W per thread, all issued before use
        float uv[kIt], wv[kIt];
#pragma unroll
        for (int it = 0; it < kIt; it++) {
            const int i = t + 128 * it;
            uv[it] = 0.0f;
            wv[it] = 0.0f;
            if (i < kTile) {
                const int x = i % kT, y = (i / kT) % kT, z = i / (kT * kT);
                const int blk = srow[(x >> 3) + 2 * (y >> 3) + 4 * (z >> 3)];
                if (blk >= 0) {
                    const int64_t o = (int64_t)blk * kBlockVox + (x & 7) + 8 * (y & 7) + 64 * (z & 7);
                    wv[it] = A.W[o];
                    uv[it] = A.val[o];
                }
            }
        }
#pragma unroll
        for (int it = 0; it < kIt; it++) {
            const int i = t + 128 * it;
            if (i < kTile) {
                su[i] = uv[it];
                sok[i] = (wv[it] > 0.0f && wv[it] >= A.w_min) ? 1 : 0;   // X-1 (unallocated: W = 0)
            }
        }
    }
    __syncthreads();
    // (A) cells 4t … 4t+3 (voxel order): x = 4(t&1) + q, y = (t>>1)&7, z = t>>4
    const int cy = (t >> 1) & 7, cz = t >> 4;
    uint32_t tets = 0;             // bit 6q + k: tetrahedron k of cell q has triangles
    unsigned long long tc = 0;     // its triangle count (1 or 2) at bits 2(6q + k)
    uint32_t ntri = 0;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int cx = 4 * (t & 1) + q;
        bool ok = true;
        int neg = 0, nz = 0;
#pragma unroll
        for (int c8 = 0; c8 < 8; c8++) {
            const int idx = tile_index(cx, cy, cz, c8);
            ok = ok && sok[idx];
            const float v = su[idx];
            neg |= (v < 0.0f) << c8;    // X-3
            nz |= (v != 0.0f) << c8;
        }
        if (!ok || neg == 0 || neg == 255) continue;
#pragma unroll
        for (int k = 0; k < 6; k++) {
            const int k1 = tet_code(k, 1), k2 = tet_code(k, 2), k3 = tet_code(k, 3);
            const int m4 = (neg & 1) | (((neg >> k1) & 1) << 1) | (((neg >> k2) & 1) << 2) | (((neg >> k3) & 1) << 3);
            const int z4 = (nz & 1) | (((nz >> k1) & 1) << 1) | (((nz >> k2) & 1) << 2) | (((nz >> k3) & 1) << 3);
            const uint32_t c = tet_triangles(m4, z4);
            tets |= (uint32_t)(c != 0) << (6 * q + k);
            tc |= (unsigned long long)c << (2 * (6 * q + k));
            ntri += c;
        }
    }
    if (!EMIT) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ntri += __shfl_xor_sync(0xffffffffu, ntri, o);
        if (lane == 0 && ntri) atomicAdd(O.total, (unsigned long long)ntri);
        return;
    }
    // block scan of (items, triangles), packed as items | triangles << 16 (≤ 3072 items, ≤ 6144 triangles)
    const uint32_t mine = __popc(tets) | (ntri << 16);
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
    const uint32_t all = swarp[0] + swarp[1] + swarp[2] + swarp[3];
    const uint32_t n_items = all & 0xFFFFu, block_total = all >> 16;
    uint32_t ip = pos & 0xFFFFu, tp = pos >> 16;
    // publish this block's total for its successors' look-back before writing the item list
    if (t == 0) st_volatile(&O.state[ci], (ci == 0 ? kInc : kAgg) | block_total);
    while (tets) {
        const int bit = __ffs(tets) - 1;
        tets &= tets - 1;
        const int q = bit / 6, k = bit - 6 * q;
        sitem[ip] = (uint16_t)(((4 * t + q) << 3) | k);
        soff[ip++] = (uint16_t)tp;
        tp += (uint32_t)(tc >> (2 * bit)) & 3u;
    }
    if (t == 0) soff[n_items] = (uint16_t)block_total;
    __syncthreads();   // the item list is complete
    const uint32_t ng = (n_items + 31) / 32;
    float *wsout = sout + wid * kSlice;
    // triangles of 32-item group g into this warp's slice at float offset `shift`
    auto compute_group = [&](uint32_t g, uint32_t shift) {
        const uint32_t i = 32 * g + lane;
        if (i < n_items) {
            const uint32_t g0 = soff[32 * g];
            const int cell = sitem[i] >> 3, k = sitem[i] & 7;
            const int cx = cell & 7, cyy = (cell >> 3) & 7, czz = cell >> 6;
            const uint2 TW = stw[k];
            const float *sb = su + tile_index(cx, cyy, czz, 0);
            const CellGeom G = cell_geom(gx + cx, gy + cyy, gz + czz, A.voxel);
            tet_emit(TW, sb, sb[0], sb[byte_of(TW.y, 1)], sb[byte_of(TW.y, 2)], sb[byte_of(TW.y, 3)], G,
                     wsout + shift + 9 * (soff[i] - g0));
        }
        __syncwarp();
    };
    // warps 1-3 compute their first group (staged unshifted: its offset is not known yet) while warp 0
    // runs the look-back
    const bool pre = wid > 0 && wid < ng;
    if (pre) compute_group(wid, 0u);
    // look-back (warp 0): sum the predecessors' words back to the nearest inclusive one
    if (wid == 0) {
        unsigned long long excl = 0;
        if (ci > 0) {
            int64_t end = ci - 1;   // predecessor read by lane 0
            while (true) {
                const int64_t j = end - lane;
                unsigned long long w = j >= 0 ? ld_volatile(&O.state[j]) : kInc;
                while (__any_sync(0xffffffffu, (w >> 62) == 0))
                    if ((w >> 62) == 0) w = ld_volatile(&O.state[j]);
                const uint32_t inc = __ballot_sync(0xffffffffu, (w >> 62) == 2);
                // lanes up to (and including) the nearest inclusive word contribute
                const int stop = inc ? __ffs(inc) - 1 : 31;
                unsigned long long v = lane <= stop ? (w & kVal) : 0ull;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                excl += v;
                if (inc) break;
                end -= 32;
            }
            if (lane == 0) st_volatile(&O.state[ci], kInc | (excl + block_total));
        }
        if (lane == 0) {
            s_base = excl;
            if (ci == n_rows - 1) *O.total = excl + block_total;
        }
    }
    __syncthreads();
    const unsigned long long base = s_base;
    const long long cap = O.max_tris;
    for (uint32_t g = wid; g < ng; g += 4) {
        const uint32_t g0 = soff[32 * g], g1 = soff[min(32 * g + 32, n_items)];
        const long long first = (long long)(base + g0);
        const long long room = cap - first;
        const uint32_t nt = room <= 0 ? 0u : (room < (long long)(g1 - g0) ? (uint32_t)room : g1 - g0);
        if (pre && g == (uint32_t)wid) {   // staged unshifted: scalar copy-out
            float *dst = O.out + 9ull * (unsigned long long)first;
            for (uint32_t j = lane; j < 9 * nt; j += 32) dst[j] = wsout[j];
            __syncwarp();
            continue;
        }
        // stage at the global address's offset within 16 bytes, so that whole float4s copy out
        const uint32_t shift = O.vec ? (uint32_t)(9ull * (unsigned long long)first) & 3u : 0u;
        compute_group(g, shift);
        float *dst = O.out + 9ull * (unsigned long long)first - shift;   // element e ↔ wsout[e], e ∈ [shift, end)
        const uint32_t end = shift + 9 * nt;
        if (O.vec) {
            const uint32_t q_lo = (shift + 3) / 4, q_hi = end / 4;
            for (uint32_t q = q_lo + lane; q < q_hi; q += 32)
                reinterpret_cast<float4 *>(dst)[q] = reinterpret_cast<const float4 *>(wsout)[q];
            const uint32_t head_end = min(4 * q_lo, end), tail = max(4 * q_hi, head_end);
            const uint32_t e = lane < 4 ? shift + lane : tail + (lane - 4);
            if (lane < 8 && e < (lane < 4 ? head_end : end)) dst[e] = wsout[e];
        } else {
            for (uint32_t j = lane; j < end; j += 32) dst[j] = wsout[j];
        }
        __syncwarp();
    }
}

__global__ void k_invert_perm(const int32_t *__restrict__ perm, int32_t *__restrict__ inv, int64_t n) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) inv[perm[r]] = (int32_t)r;
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
    if (n == 0) return VOL_OK;
    // scratch in d_tmp (n × 2 KiB): look-back words [n] u64, ticket, total, inverse permutation [n] i32
    unsigned long long *state = reinterpret_cast<unsigned long long *>(v->d_tmp);
    unsigned *ticket = reinterpret_cast<unsigned *>(state + n);
    unsigned long long *total = state + n + 1;
    int32_t *inv = reinterpret_cast<int32_t *>(state + n + 2);
    ExArgs A{field == 0 ? v->F.u : v->F.f, v->F.W, v->d_nbr, v->d_perm, v->d_xyz, voxel, w_min};
    const bool dev = tris && is_device_ptr(tris);
    unsigned long long m = 0;
    float *out = tris;
    if (!dev) {
        // count pass (count only, or a host buffer: the device staging buffer is sized by it)
        CK(cudaMemsetAsync(total, 0, 8, s));
        k_extract<false><<<(unsigned)n, 128, 0, s>>>(A, n, ExOut{nullptr, nullptr, nullptr, total, nullptr, 0, 0});
        CK(cudaPeekAtLastError());
        counted(1);
        CK(cudaMemcpyAsync(&m, total, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        *n_tris = (int64_t)m;
        if (!tris) return VOL_OK;
        if ((int64_t)m > max_tris)
            return fail(VOL_ENOMEM, "vol_extract: %lld triangles > max_tris = %lld", (long long)m, (long long)max_tris);
        if (m == 0) return VOL_OK;
        CK(cudaMallocAsync((void **)&out, (size_t)m * 36, s));
        max_tris = (int64_t)m;
    }
    // single ordered pass: count, look-back, emit
    cudaError_t e = cudaMemsetAsync(state, 0, ((size_t)n + 2) * 8, s);
    if (e == cudaSuccess) {
        k_invert_perm<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(v->d_perm, inv, n);
        k_extract<true><<<(unsigned)n, 128, 0, s>>>(A, n, ExOut{inv, state, ticket, total, out, max_tris, ((uintptr_t)out & 15) == 0});
        e = cudaPeekAtLastError();
        if (e == cudaSuccess) counted(2);
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&m, total, 8, cudaMemcpyDeviceToHost, s);
    if (!dev) {
        if (e == cudaSuccess) e = cudaMemcpyAsync(tris, out, (size_t)max_tris * 36, cudaMemcpyDeviceToHost, s);
        cudaFreeAsync(out, s);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(VOL_ECUDA, "vol_extract: %s", cudaGetErrorString(e));
    *n_tris = (int64_t)m;
    if ((int64_t)m > max_tris)
        return fail(VOL_ENOMEM, "vol_extract: %lld triangles > max_tris = %lld (the first max_tris written)",
                    (long long)m, (long long)max_tris);
    return VOL_OK;
}
