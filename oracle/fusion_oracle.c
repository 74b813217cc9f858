/*
 * oracle/fusion_oracle.c — plain, slow, obviously-correct CPU oracle of the TSDF fusion of depth maps
 * into the hashed voxel-block grid (arXiv 1604.03734 §III-A, Eq. 1).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant with
 * the CUDA path (paper_1604_03734_b200/csrc) and never imports it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n.  The readings F-1 … F-10
 * of silent or ambiguous passages are listed in DESIGN.md ("Fusion readings").
 *
 * The algorithm, in the paper's order, for every depth map k = 0 … K−1 in sequence:
 *   allocation  P:144-145 "Anytime a surface is observed within a given voxel block, all the voxels in
 *               that block are allocated" (reading F-5): for every valid pixel (i, j) with depth d,
 *               the blocks met by the pixel's viewing ray between camera depths max(d − μ, 0) and
 *               d + μ (the truncation band |u_SDF| <= μ) are allocated, visited by the 6-connected
 *               lattice walk of reading F-7;
 *   update      P:152-176 steps 1-4 for every voxel of every allocated block (reading F-8: blocks
 *               allocated by frame k are updated from frame k on):
 *               1. p_c = T_gc^{-1} p_g = R^T (p_g − t)                         (reading F-2)
 *               2. nearest pixel (i, j) = (floor(fx·x/z + cx + ½), floor(fy·y/z + cy + ½))  (F-1)
 *               3. if (i, j) is inside D and d_{i,j} valid: u_SDF = d_{i,j} − z_c
 *               4. Eq. 1: if u_SDF >= −μ: u_TSDF = clamp(u_SDF, −μ, μ)/μ (F-3),
 *                  f = (u_TSDF + w·f)/(w + 1), w = min(w + 1, w_max) (F-4); else unchanged.
 *
 * Every floating-point decision (pixel choice, block walk) and every value is evaluated in IEEE
 * fp32 in the order written here; divisions by per-call constants (1/fx, 1/fy, 1/Bm, 1/μ) and the two
 * divisions by z_c are products with a correctly rounded reciprocal (reading F-12) (reading F-10, "where floating point decides an integer, both sides
 * take that decision in the same precision"); compile with -ffp-contract=off.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ Eq. 1 for one voxel */

/* sdf = u_SDF = d − z_c.  Updates (*f, *w) in place per Eq. 1 with the weight cap of F-4.
 * Returns 1 if the voxel was updated, 0 if the carve-protection branch left it unchanged.         */
int orc_tsdf_update(float *f, float *w, float sdf, float mu, float w_max)
{
    if (sdf < -mu) return 0;                         /* Eq. 1 case u_SDF < −μ: unchanged     */
    float c = sdf;
    if (c < -mu) c = -mu;
    if (c > mu) c = mu;
    float tsdf = c * (1.0f / mu);                    /* reading F-3 (F-12: ·fl(1/μ)), in [−1, 1] */
    float num = tsdf + (*w) * (*f);                  /* u_TSDF + w_{k−1} f_{k−1}              */
    float den = (*w) + 1.0f;                         /* w_{k−1} + 1                           */
    *f = num / den;
    float wn = (*w) + 1.0f;
    *w = wn < w_max ? wn : w_max;
    return 1;
}

static int depth_valid(float d, float max_range)
{
    return isfinite(d) && d > 0.0f && d <= max_range;
}

/* Steps 1-2: global point -> camera frame -> nearest pixel.  pose = T_gc row-major 3x4
 * (camera-to-global: p_g = R p_c + t).  Returns 1 and (i, j, z_c) if z_c > 0 and the pixel lies in
 * the W×H image (reading F-1: pixel (i, j) is the square of centre (i, j)).                       */
int orc_project(const float *pose, const float *intr, int32_t H, int32_t Wd, float px, float py, float pz,
                int32_t *pi, int32_t *pj, float *pzc)
{
    float d0 = px - pose[3];
    float d1 = py - pose[7];
    float d2 = pz - pose[11];
    /* R^T d: column c of R dotted with d, summed in row order (reading F-2) */
    float xc = (pose[0] * d0 + pose[4] * d1) + pose[8] * d2;
    float yc = (pose[1] * d0 + pose[5] * d1) + pose[9] * d2;
    float zc = (pose[2] * d0 + pose[6] * d1) + pose[10] * d2;
    if (!(zc > 0.0f)) return 0;
    float rz = 1.0f / zc;                            /* reading F-12: one reciprocal of z_c  */
    float a = xc * rz;
    float b = yc * rz;
    float ix = intr[0] * a + intr[2];
    float iy = intr[1] * b + intr[3];
    float fi = floorf(ix + 0.5f);
    float fj = floorf(iy + 0.5f);
    if (!(fi >= 0.0f && fi < (float)Wd && fj >= 0.0f && fj < (float)H)) return 0;
    *pi = (int32_t)fi;
    *pj = (int32_t)fj;
    *pzc = zc;
    return 1;
}

/* Ray point of pixel (i, j) at camera depth z, in the global frame (reading F-6):
 * p_c = ((i − cx)/fx · z, (j − cy)/fy · z, z);  p_g = R p_c + t (row sums left to right).        */
static void ray_point(const float *pose, const float *intr, int32_t i, int32_t j, float z, float *g)
{
    float xc = (((float)i - intr[2]) * (1.0f / intr[0])) * z;   /* reading F-12: ·fl(1/fx) */
    float yc = (((float)j - intr[3]) * (1.0f / intr[1])) * z;
    float zc = z;
    for (int r = 0; r < 3; r++) g[r] = ((pose[4 * r + 0] * xc + pose[4 * r + 1] * yc) + pose[4 * r + 2] * zc) + pose[4 * r + 3];
}

/* ------------------------------------------------------------------ block walk (reading F-7) */

/* 6-connected lattice walk from the block of point a to the block of point b (points in metres,
 * block edge Bm metres).  s = p·fl(1/Bm) (F-12); start cell floor(s_a), end cell floor(s_b); per axis
 * dir = s_b − s_a, tMax = distance in t to the first face crossing, tDelta = 1/|dir|; each step
 * advances the axis with remaining steps and the smallest tMax (ties: lowest axis), exactly
 * |Δcell|_1 steps.  Writes up to max_cells cells [.][3]; returns the number of cells of the walk. */
int64_t orc_block_walk(const float *a, const float *b, float Bm, int32_t *cells, int64_t max_cells)
{
    float sa[3], sb[3], tmax[3], tdel[3];
    int64_t c[3], n[3], step[3];
    const float inv = 1.0f / Bm;                     /* reading F-12: s = p·fl(1/Bm) */
    for (int k = 0; k < 3; k++) {
        sa[k] = a[k] * inv;
        sb[k] = b[k] * inv;
        float fa = floorf(sa[k]);
        float fb = floorf(sb[k]);
        c[k] = (int64_t)fa;
        int64_t e = (int64_t)fb;
        float dir = sb[k] - sa[k];
        if (dir > 0.0f) {
            step[k] = 1;
            tdel[k] = 1.0f / dir;
            tmax[k] = ((fa + 1.0f) - sa[k]) * tdel[k];
        } else if (dir < 0.0f) {
            step[k] = -1;
            tdel[k] = 1.0f / (-dir);
            tmax[k] = (sa[k] - fa) * tdel[k];
        } else {
            step[k] = 0;
            tdel[k] = INFINITY;
            tmax[k] = INFINITY;
        }
        n[k] = e > c[k] ? e - c[k] : c[k] - e;
    }
    int64_t m = 0;
    if (m < max_cells) { cells[3 * m] = (int32_t)c[0]; cells[3 * m + 1] = (int32_t)c[1]; cells[3 * m + 2] = (int32_t)c[2]; }
    m++;
    while (n[0] + n[1] + n[2] > 0) {
        int best = -1;
        for (int k = 0; k < 3; k++) {
            if (n[k] == 0) continue;
            if (best < 0 || tmax[k] < tmax[best]) best = k;
        }
        c[best] += step[best];
        tmax[best] = tmax[best] + tdel[best];
        n[best] -= 1;
        if (m < max_cells) { cells[3 * m] = (int32_t)c[0]; cells[3 * m + 1] = (int32_t)c[1]; cells[3 * m + 2] = (int32_t)c[2]; }
        m++;
    }
    return m;
}

/* ------------------------------------------------------------------ a plain block set */

typedef struct {
    int64_t cap;       /* power of two */
    int64_t n;
    int64_t *key;      /* packed coordinates, -1 = empty */
    int64_t *idx;      /* index into the block list */
    int32_t *xyz;      /* [n][3] in insertion order */
    int32_t *first;    /* [n] frame of allocation */
    float *f, *w;      /* [n][512] */
    int64_t list_cap;
} blockset;

static int64_t pack(int32_t x, int32_t y, int32_t z)
{
    const int64_t o = (int64_t)1 << 20, m = ((int64_t)1 << 21) - 1;
    return (((int64_t)x + o) & m) << 42 | (((int64_t)y + o) & m) << 21 | (((int64_t)z + o) & m);
}

static uint64_t mix(int64_t k)
{
    uint64_t z = (uint64_t)k + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static void set_init(blockset *s)
{
    memset(s, 0, sizeof(*s));
    s->cap = 1024;
    s->key = (int64_t *)malloc(sizeof(int64_t) * s->cap);
    s->idx = (int64_t *)malloc(sizeof(int64_t) * s->cap);
    for (int64_t i = 0; i < s->cap; i++) s->key[i] = -1;
}

static void set_free(blockset *s)
{
    free(s->key); free(s->idx); free(s->xyz); free(s->first); free(s->f); free(s->w);
}

static int64_t set_find(const blockset *s, int64_t k)
{
    int64_t h = (int64_t)(mix(k) & (uint64_t)(s->cap - 1));
    while (s->key[h] != -1) {
        if (s->key[h] == k) return s->idx[h];
        h = (h + 1) & (s->cap - 1);
    }
    return -1;
}

static void set_put(blockset *s, int64_t k, int64_t v)
{
    int64_t h = (int64_t)(mix(k) & (uint64_t)(s->cap - 1));
    while (s->key[h] != -1) h = (h + 1) & (s->cap - 1);
    s->key[h] = k;
    s->idx[h] = v;
}

/* Insert block (x, y, z) allocated by frame `frame` (no-op if present); f = w = 0 for a new block. */
static void set_insert(blockset *s, int32_t x, int32_t y, int32_t z, int32_t frame, int with_data)
{
    int64_t k = pack(x, y, z);
    if (set_find(s, k) >= 0) return;
    if (2 * (s->n + 1) > s->cap) {
        int64_t oc = s->cap;
        int64_t *ok = s->key, *oi = s->idx;
        s->cap = 2 * oc;
        s->key = (int64_t *)malloc(sizeof(int64_t) * s->cap);
        s->idx = (int64_t *)malloc(sizeof(int64_t) * s->cap);
        for (int64_t i = 0; i < s->cap; i++) s->key[i] = -1;
        for (int64_t i = 0; i < oc; i++)
            if (ok[i] != -1) set_put(s, ok[i], oi[i]);
        free(ok); free(oi);
    }
    if (s->n == s->list_cap) {
        s->list_cap = s->list_cap ? 2 * s->list_cap : 1024;
        s->xyz = (int32_t *)realloc(s->xyz, sizeof(int32_t) * 3 * s->list_cap);
        s->first = (int32_t *)realloc(s->first, sizeof(int32_t) * s->list_cap);
        if (with_data) {
            s->f = (float *)realloc(s->f, sizeof(float) * 512 * s->list_cap);
            s->w = (float *)realloc(s->w, sizeof(float) * 512 * s->list_cap);
        }
    }
    int64_t i = s->n++;
    s->xyz[3 * i] = x; s->xyz[3 * i + 1] = y; s->xyz[3 * i + 2] = z;
    s->first[i] = frame;
    if (with_data) {
        for (int v = 0; v < 512; v++) { s->f[512 * i + v] = 0.0f; s->w[512 * i + v] = 0.0f; }
    }
    set_put(s, k, i);
}

/* ------------------------------------------------------------------ the two passes of one frame */

#define WALK_MAX 4096

/* Allocation pass of frame k (reading F-5).  Returns 0, or -1 if a walk leaves the coordinate range. */
static int alloc_frame(blockset *s, const float *depth, int32_t k, int32_t H, int32_t Wd, const float *intr,
                       const float *pose, float voxel, float mu, float max_range, int with_data)
{
    const float Bm = 8.0f * voxel;
    int32_t *cells = (int32_t *)malloc(sizeof(int32_t) * 3 * WALK_MAX);
    int rc = 0;
    for (int32_t j = 0; j < H && rc == 0; j++) {
        for (int32_t i = 0; i < Wd; i++) {
            float d = depth[(int64_t)j * Wd + i];
            if (!depth_valid(d, max_range)) continue;
            float za = d - mu;
            if (za < 0.0f) za = 0.0f;
            float zb = d + mu;
            float ga[3], gb[3];
            ray_point(pose, intr, i, j, za, ga);
            ray_point(pose, intr, i, j, zb, gb);
            int64_t m = orc_block_walk(ga, gb, Bm, cells, WALK_MAX);
            if (m > WALK_MAX) { rc = -1; break; }
            for (int64_t q = 0; q < m; q++) {
                int32_t x = cells[3 * q], y = cells[3 * q + 1], z = cells[3 * q + 2];
                if (x <= -(1 << 20) || x >= (1 << 20) || y <= -(1 << 20) || y >= (1 << 20) || z <= -(1 << 20) ||
                    z >= (1 << 20)) { rc = -1; break; }
                set_insert(s, x, y, z, k, with_data);
            }
            if (rc) break;
        }
    }
    free(cells);
    return rc;
}

/* Update pass of frame k over blocks [0, nb) of (xyz, f, w) (P:152-176 steps 1-4). */
static void update_blocks(const int32_t *xyz, float *f, float *w, int64_t nb, const float *depth, int32_t H,
                          int32_t Wd, const float *intr, const float *pose, float voxel, float mu, float max_range,
                          float w_max)
{
    for (int64_t b = 0; b < nb; b++) {
        for (int v = 0; v < 512; v++) {
            int32_t lx = v % 8, ly = (v / 8) % 8, lz = v / 64;
            /* voxel centre (8B + i + ½)·v (SURVEY §8(d) frame convention) */
            float px = ((float)(8 * xyz[3 * b] + lx) + 0.5f) * voxel;
            float py = ((float)(8 * xyz[3 * b + 1] + ly) + 0.5f) * voxel;
            float pz = ((float)(8 * xyz[3 * b + 2] + lz) + 0.5f) * voxel;
            int32_t i, j;
            float zc;
            if (!orc_project(pose, intr, H, Wd, px, py, pz, &i, &j, &zc)) continue;
            float d = depth[(int64_t)j * Wd + i];
            if (!depth_valid(d, max_range)) continue;
            float sdf = d - zc;                              /* u_SDF = d_{x,y} − z_c */
            orc_tsdf_update(&f[512 * b + v], &w[512 * b + v], sdf, mu, w_max);
        }
    }
}

static int cmp_key(const void *a, const void *b)
{
    int64_t x = ((const int64_t *)a)[0], y = ((const int64_t *)b)[0];
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* Sort the set's blocks by (x, y, z) lexicographically (reading F-9) and copy them out. */
static void emit_sorted(const blockset *s, int32_t *xyz, int32_t *first, float *f, float *w, int with_data)
{
    int64_t *kv = (int64_t *)malloc(sizeof(int64_t) * 2 * (s->n ? s->n : 1));
    for (int64_t i = 0; i < s->n; i++) {
        kv[2 * i] = pack(s->xyz[3 * i], s->xyz[3 * i + 1], s->xyz[3 * i + 2]);
        kv[2 * i + 1] = i;
    }
    qsort(kv, (size_t)s->n, 2 * sizeof(int64_t), cmp_key);
    for (int64_t r = 0; r < s->n; r++) {
        int64_t i = kv[2 * r + 1];
        if (xyz) { xyz[3 * r] = s->xyz[3 * i]; xyz[3 * r + 1] = s->xyz[3 * i + 1]; xyz[3 * r + 2] = s->xyz[3 * i + 2]; }
        if (first) first[r] = s->first[i];
        if (with_data) {
            if (f) memcpy(f + 512 * r, s->f + 512 * i, 512 * sizeof(float));
            if (w) memcpy(w + 512 * r, s->w + 512 * i, 512 * sizeof(float));
        }
    }
    free(kv);
}

/* ------------------------------------------------------------------ entry points */

/* The whole fusion, frame by frame (allocation then update), continuing from an existing
 * set of fused blocks ("New incoming data can be added at any time"; reading F-11): the
 * n_prev blocks prev_xyz with their (f, W) are in the set before frame 0 (allocating frame −1), and
 * new depth maps update them exactly as they would have after the frames that produced them.
 *   depth [K][H][Wd] metres (invalid: non-finite, <= 0 or > max_range);  intr = (fx, fy, cx, cy);
 *   pose [K][12] row-major T_gc (camera-to-global).
 * Returns the number of blocks n (or -1 if a block walk leaves the coordinate range or is longer than
 * the oracle's walk buffer, -2 if prev_xyz repeats a block).  Outputs (sorted by (x, y, z)) are
 * written only when n <= max_blocks: xyz [n][3], first [n] (allocating frame, −1 for the previous
 * blocks), f, W [n][512].                                                                          */
int64_t orc_fuse_incremental(const int32_t *prev_xyz, const float *prev_f, const float *prev_W, int64_t n_prev,
                             const float *depth, int32_t K, int32_t H, int32_t Wd, const float *intr,
                             const float *pose, float voxel, float mu, float max_range, float w_max,
                             int64_t max_blocks, int32_t *xyz, int32_t *first, float *f, float *W)
{
    blockset s;
    set_init(&s);
    for (int64_t b = 0; b < n_prev; b++) {
        int64_t before = s.n;
        set_insert(&s, prev_xyz[3 * b], prev_xyz[3 * b + 1], prev_xyz[3 * b + 2], -1, 1);
        if (s.n == before) { set_free(&s); return -2; }
        memcpy(s.f + 512 * before, prev_f + 512 * b, 512 * sizeof(float));
        memcpy(s.w + 512 * before, prev_W + 512 * b, 512 * sizeof(float));
    }
    for (int32_t k = 0; k < K; k++) {
        const float *D = depth + (int64_t)k * H * Wd;
        if (alloc_frame(&s, D, k, H, Wd, intr, pose + 12 * k, voxel, mu, max_range, 1)) { set_free(&s); return -1; }
        update_blocks(s.xyz, s.f, s.w, s.n, D, H, Wd, intr, pose + 12 * k, voxel, mu, max_range, w_max);
    }
    int64_t n = s.n;
    if (n <= max_blocks) emit_sorted(&s, xyz, first, f, W, 1);
    set_free(&s);
    return n;
}

int64_t orc_fuse(const float *depth, int32_t K, int32_t H, int32_t Wd, const float *intr, const float *pose,
                 float voxel, float mu, float max_range, float w_max, int64_t max_blocks, int32_t *xyz,
                 int32_t *first, float *f, float *W)
{
    return orc_fuse_incremental(NULL, NULL, NULL, 0, depth, K, H, Wd, intr, pose, voxel, mu, max_range, w_max,
                                max_blocks, xyz, first, f, W);
}

/* Allocation passes only (every frame in sequence): the allocated blocks sorted by (x, y, z) and the
 * frame that allocated each.  Same return convention as orc_fuse.                                   */
int64_t orc_fuse_alloc(const float *depth, int32_t K, int32_t H, int32_t Wd, const float *intr, const float *pose,
                       float voxel, float mu, float max_range, int64_t max_blocks, int32_t *xyz, int32_t *first)
{
    blockset s;
    set_init(&s);
    for (int32_t k = 0; k < K; k++)
        if (alloc_frame(&s, depth + (int64_t)k * H * Wd, k, H, Wd, intr, pose + 12 * k, voxel, mu, max_range, 0)) {
            set_free(&s);
            return -1;
        }
    int64_t n = s.n;
    if (n <= max_blocks) emit_sorted(&s, xyz, first, NULL, NULL, 0);
    set_free(&s);
    return n;
}

/* Update passes for a chosen subset of blocks: block b (allocated by frame first[b]) receives the
 * updates of frames first[b] … K−1 in order, exactly as in orc_fuse (the update of a voxel depends
 * only on its own (f, w) and the frame).  f, W [nb][512] are initialised to 0 here.  Used to check
 * sampled blocks of full-size volumes.                                                              */
void orc_fuse_update_blocks(const float *depth, int32_t K, int32_t H, int32_t Wd, const float *intr,
                            const float *pose, float voxel, float mu, float max_range, float w_max,
                            const int32_t *xyz, const int32_t *first, int64_t nb, float *f, float *W)
{
    for (int64_t q = 0; q < 512 * nb; q++) { f[q] = 0.0f; W[q] = 0.0f; }
    for (int32_t k = 0; k < K; k++)
        for (int64_t b = 0; b < nb; b++)
            if (first[b] <= k)
                update_blocks(xyz + 3 * b, f + 512 * b, W + 512 * b, 1, depth + (int64_t)k * H * Wd, H, Wd, intr,
                              pose + 12 * k, voxel, mu, max_range, w_max);
}
