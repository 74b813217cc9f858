/*
 * oracle/extract_oracle.c — plain, slow, obviously-correct CPU oracle of the Ω-restricted isosurface
 * extraction of the regularised TSDF (paper P:102 "regularise the model in 3D
 * space, extract the surface", "solve for the zero-crossing level set (isosurface)").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path (paper_1604_03734_b200/csrc).
 *
 * The paper names no extraction algorithm ("algorithm choice is invented").  Readings
 * X-1 … X-7:
 *   X-1 cells     every voxel g of an allocated block spans the cell with corners g + {0,1}^3 (voxel
 *                 centres (g + ½)·v); a cell is extracted iff all 8 corners are allocated voxels with
 *                 W > 0 (Ω) and W >= w_min — no geometry next to Ω̄;
 *   X-2 tetrahedra each cell is split into the 6 Freudenthal (Kuhn) tetrahedra around its main
 *                 diagonal: for each permutation (a, b, c) of the axes, 000 → e_a → e_a + e_b → 111
 *                 (permutations in lexicographic order); this triangulates space consistently, so the
 *                 surface has no cracks across cells and blocks (marching tetrahedra, no case table);
 *   X-3 inside    corner value u < 0 is inside (behind the surface, P:158 sign), u >= 0 outside;
 *   X-4 vertices  on every tet edge with one inside and one outside end: with the edge's ends ordered
 *                 by global voxel coordinate (lo < hi lexicographically in (x, y, z)),
 *                 t = u_lo/(u_lo − u_hi), p = P_lo + t·(P_hi − P_lo) per axis (fp32, written order), so
 *                 every occurrence of an edge yields bit-identical vertices;
 *   X-5 triangles 1 inside corner a (or 1 outside, orientation reversed) → triangle (E_ab, E_ac, E_ad);
 *                 2 inside a, b → (E_ac, E_ad, E_bd), (E_ac, E_bd, E_bc); with (a, b, c, d) a
 *                 positively oriented ordering of the tet — normals point toward u > 0 (free space);
 *   X-6 degenerate a triangle whose area is zero in exact arithmetic is dropped ("no
 *                 degenerate"): an edge vertex lies on its outside corner iff that corner's value is
 *                 exactly 0 (the inside value is < 0), so two vertices coincide iff they share an
 *                 outside corner of value 0 — the 1-outside triangle when that corner is 0, the quad's
 *                 (E_ac, E_ad, E_bd) when u_d = 0 and (E_ac, E_bd, E_bc) when u_c = 0; the 1-inside
 *                 triangle never degenerates.  A decision on the corner values alone, not on rounded
 *                 vertices;
 *   X-7 order     blocks in caller order, cells in voxel order (x fastest), tets in X-2 order,
 *                 triangles in X-5 order.  Output: float [m][3][3] triangle soup (S:325 allows
 *                 duplicated seam vertices).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* from hvg_oracle.c (the oracle's own block store) */
uint32_t orc_table_size(int64_t n);
int64_t orc_build_table(const int32_t *xyz, int64_t n, uint32_t T, uint32_t *bucket_start, int32_t *bucket_entry,
                        int64_t *dup_j);
int64_t orc_lookup(const int32_t *xyz, const uint32_t *bucket_start, const int32_t *bucket_entry, uint32_t T,
                   int32_t x, int32_t y, int32_t z);

static int64_t floordiv8(int64_t a) { return a >= 0 ? a / 8 : -((-a + 7) / 8); }

typedef struct {
    const int32_t *xyz;
    const uint32_t *bs;
    const int32_t *be;
    uint32_t T;
    const float *u, *W;
} store;

/* value and weight of the voxel at global coordinate g; returns 0 if its block is not allocated */
static int voxel_at(const store *S, const int64_t g[3], float *u, float *w)
{
    int64_t b[3], l[3];
    for (int k = 0; k < 3; k++) {
        b[k] = floordiv8(g[k]);
        l[k] = g[k] - 8 * b[k];
    }
    int64_t j = orc_lookup(S->xyz, S->bs, S->be, S->T, (int32_t)b[0], (int32_t)b[1], (int32_t)b[2]);
    if (j < 0) return 0;
    int64_t v = l[0] + 8 * l[1] + 64 * l[2];
    *u = S->u[512 * j + v];
    *w = S->W[512 * j + v];
    return 1;
}

static int lex_less(const int64_t a[3], const int64_t b[3])
{
    for (int k = 0; k < 3; k++) {
        if (a[k] != b[k]) return a[k] < b[k];
    }
    return 0;
}

/* X-4: vertex on the edge between corners i and j of the cell (both given by global coordinates) */
static void edge_vertex(const int64_t gi[3], float ui, const int64_t gj[3], float uj, float voxel, float *p)
{
    const int64_t *glo = gi, *ghi = gj;
    float ulo = ui, uhi = uj;
    if (lex_less(gj, gi)) { glo = gj; ghi = gi; ulo = uj; uhi = ui; }
    float t = ulo / (ulo - uhi);
    for (int k = 0; k < 3; k++) {
        float plo = ((float)glo[k] + 0.5f) * voxel;
        float phi = ((float)ghi[k] + 0.5f) * voxel;
        p[k] = plo + t * (phi - plo);
    }
}

static int64_t emit(float *out, int64_t m, int64_t max, const float *p0, const float *p1, const float *p2,
                    int degenerate)
{
    if (degenerate) return m;    /* X-6 */
    if (out && m < max) {
        memcpy(out + 9 * m, p0, 3 * sizeof(float));
        memcpy(out + 9 * m + 3, p1, 3 * sizeof(float));
        memcpy(out + 9 * m + 6, p2, 3 * sizeof(float));
    }
    return m + 1;
}

/* Extract the triangles of all cells.  coords [n][3], u, W [n][512] in caller order.  Writes up to
 * max_tris triangles [.][3][3] into out (may be NULL) and returns the number of triangles.         */
int64_t orc_extract(const int32_t *xyz, int64_t n, const float *u, const float *W, float voxel, float w_min,
                    float *out, int64_t max_tris)
{
    uint32_t T = orc_table_size(n);
    uint32_t *bs = (uint32_t *)malloc(sizeof(uint32_t) * ((size_t)T + 1));
    int32_t *be = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
    int64_t dj;
    orc_build_table(xyz, n, T, bs, be, &dj);
    store S = {xyz, bs, be, T, u, W};
    /* X-2: the 6 permutations of the axes in lexicographic order, and their parity */
    static const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    static const int EVEN[6] = {1, 0, 0, 1, 1, 0};
    int64_t m = 0;
    for (int64_t b = 0; b < n; b++) {
        for (int v = 0; v < 512; v++) {
            int64_t g0[3] = {8 * (int64_t)xyz[3 * b] + v % 8, 8 * (int64_t)xyz[3 * b + 1] + (v / 8) % 8,
                             8 * (int64_t)xyz[3 * b + 2] + v / 64};
            /* X-1: the 8 corners, all allocated, in Ω and with W >= w_min */
            float cu[2][2][2];
            int ok = 1;
            for (int k = 0; k < 2 && ok; k++)
                for (int j = 0; j < 2 && ok; j++)
                    for (int i = 0; i < 2 && ok; i++) {
                        int64_t g[3] = {g0[0] + i, g0[1] + j, g0[2] + k};
                        float uu, ww;
                        if (!voxel_at(&S, g, &uu, &ww) || !(ww > 0.0f) || !(ww >= w_min)) ok = 0;
                        else cu[i][j][k] = uu;
                    }
            if (!ok) continue;
            for (int q = 0; q < 6; q++) {
                /* tet vertices as cube offsets: 000, e_a, e_a + e_b, 111 */
                int off[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {1, 1, 1}};
                off[1][PERM[q][0]] = 1;
                off[2][PERM[q][0]] = 1;
                off[2][PERM[q][1]] = 1;
                int ord[4] = {0, 1, 2, 3};
                if (!EVEN[q]) { ord[2] = 3; ord[3] = 2; }       /* positively oriented ordering */
                int64_t g[4][3];
                float val[4];
                int in[4], nin = 0;
                for (int r = 0; r < 4; r++) {
                    const int *o = off[ord[r]];
                    for (int k = 0; k < 3; k++) g[r][k] = g0[k] + o[k];
                    val[r] = cu[o[0]][o[1]][o[2]];
                    in[r] = val[r] < 0.0f;                        /* X-3 */
                    nin += in[r];
                }
                if (nin == 0 || nin == 4) continue;
                /* reorder (keeping the orientation) so that the lone / paired vertices come first */
                int a, bb, c, d, flip = 0;
                int sel = (nin == 3) ? 0 : 1;                      /* lone vertex has in == sel */
                int p[4], np = 0;
                if (nin == 1 || nin == 3) {
                    for (int r = 0; r < 4; r++) if (in[r] == sel) p[np++] = r;
                    for (int r = 0; r < 4; r++) if (in[r] != sel) p[np++] = r;
                } else {
                    for (int r = 0; r < 4; r++) if (in[r]) p[np++] = r;
                    for (int r = 0; r < 4; r++) if (!in[r]) p[np++] = r;
                }
                /* parity of the permutation p of (0,1,2,3): count inversions */
                int inv = 0;
                for (int x = 0; x < 4; x++)
                    for (int y = x + 1; y < 4; y++) inv += p[x] > p[y];
                if (inv & 1) { int t = p[2]; p[2] = p[3]; p[3] = t; }
                a = p[0]; bb = p[1]; c = p[2]; d = p[3];
                if (nin == 3) flip = 1;
                float e1[3], e2[3], e3[3], e4[3];
                if (nin == 1 || nin == 3) {
                    edge_vertex(g[a], val[a], g[bb], val[bb], voxel, e1);
                    edge_vertex(g[a], val[a], g[c], val[c], voxel, e2);
                    edge_vertex(g[a], val[a], g[d], val[d], voxel, e3);
                    /* 1 inside: never degenerate; 1 outside (a): all three vertices at a iff u_a = 0 */
                    int deg = flip && val[a] == 0.0f;
                    if (!flip) m = emit(out, m, max_tris, e1, e2, e3, deg);
                    else m = emit(out, m, max_tris, e1, e3, e2, deg);
                } else {
                    edge_vertex(g[a], val[a], g[c], val[c], voxel, e1);   /* E_ac */
                    edge_vertex(g[a], val[a], g[d], val[d], voxel, e2);   /* E_ad */
                    edge_vertex(g[bb], val[bb], g[d], val[d], voxel, e3); /* E_bd */
                    edge_vertex(g[bb], val[bb], g[c], val[c], voxel, e4); /* E_bc */
                    m = emit(out, m, max_tris, e1, e2, e3, val[d] == 0.0f);   /* E_ad = E_bd iff u_d = 0 */
                    m = emit(out, m, max_tris, e1, e3, e4, val[c] == 0.0f);   /* E_ac = E_bc iff u_c = 0 */
                }
            }
        }
    }
    free(bs);
    free(be);
    return m;
}
