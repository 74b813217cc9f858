/*
 * oracle/hvg_oracle.c — plain, slow, obviously-correct CPU oracle of the hashed-voxel-grid
 * primal–dual TV regulariser of arXiv 1604.03734 (§III-B/C).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header, table or constant with
 * the CUDA path (paper_1604_03734_b200/csrc) and never imports it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n (spec of a CPU program,
 * used for interfaces and worked examples only).  Readings of ambiguous passages are the ones of
 * SURVEY.md §8(c) and are listed in DESIGN.md ("Readings").
 *
 *   block store     P:143 (8^3 blocks), P:147-148 (hash of block coords indexes the table),
 *                   S:49-57/S:83 (Teschner primes).  Reading c-14: uint32 wrap-around, T = next
 *                   power of two >= 2n, buckets in CSR form ordered by caller index.
 *   Ω               P:232-234: observed voxels; unallocated blocks are in Ω̄.  Reading c-13: Ω ⇔ W>0.
 *   gradient        P:240-250 (Eq. 3): forward difference, 0 if either end is in Ω̄ (or absent).
 *   divergence      P:252-263 (Eq. 4): "the dual of the new gradient"; reading c-8: edge-based
 *                   negative adjoint, each edge term present iff the edge is valid.
 *   dual step       P:293-302 (Eq. 7) + Huber damping (north_star, reading c-12):
 *                   q = (p + σ∇ū)/(1+σε);  p = q / max(1, ‖q‖₂).
 *   primal step     P:304-313 (Eq. 8) with the sign of reading c-2: ũ = u + τ·div p; then
 *                   L1 (north_star): weighted shrinkage toward f by t = τλW, or
 *                   L2 (paper Eq. 8): u = (ũ + τλW f)/(1 + τλW).
 *   relaxation      P:315-321 (Eq. 9) with reading c-3: ū = u' + θ(u' − u).
 *   init            P:291 (zero) or warm u = ū = f, reading c-4.
 *   energy          P:216-222 (Eq. 2) with the W-weighted data term (c-1) and Huber TV.
 *
 * Arithmetic is written out in one fixed order (reading c-18); compile with -ffp-contract=off.
 * The whole file is compiled twice: REAL=double (the parity oracle) and REAL=float (same formula
 * order in fp32, used to show the GPU path reproduces the written order).
 */
#include <math.h>
#include <stdint.h>

/* Voxel loops of one phase are independent (each phase reads a frozen snapshot of the previous one),
 * so the timing build (liboracle_omp.so, -fopenmp; bench.py cpu_baseline_omp only) runs them over all
 * host cores.  The parity build has no -fopenmp and the pragma is empty: same arithmetic either way. */
#ifdef _OPENMP
#define ORC_PAR _Pragma("omp parallel for schedule(static)")
#else
#define ORC_PAR
#endif
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- block store (precision-free) */

/* h(x,y,z) = ((u32)x·73856093 ⊕ (u32)y·19349669 ⊕ (u32)z·83492791) mod T */
uint32_t orc_hash(int32_t x, int32_t y, int32_t z, uint32_t T)
{
    uint32_t hx = (uint32_t)x * 73856093u;
    uint32_t hy = (uint32_t)y * 19349669u;
    uint32_t hz = (uint32_t)z * 83492791u;
    return (hx ^ hy ^ hz) % T;
}

/* T = smallest power of two with T >= 2n (at least 1). */
uint32_t orc_table_size(int64_t n)
{
    uint32_t T = 1;
    while ((int64_t)T < 2 * n) T <<= 1;
    return T;
}

/* CSR bucket table by counting sort in caller order.
 * bucket_start[T+1]: bucket b holds bucket_entry[bucket_start[b] .. bucket_start[b+1]).
 * Returns -1 if all coordinates are distinct, else the caller index i of the first block (smallest i)
 * that repeats an earlier block j < i; *dup_j receives j.                                        */
int64_t orc_build_table(const int32_t *xyz, int64_t n, uint32_t T, uint32_t *bucket_start,
                        int32_t *bucket_entry, int64_t *dup_j)
{
    uint32_t *cursor = (uint32_t *)calloc((size_t)T + 1, sizeof(uint32_t));
    for (uint32_t b = 0; b <= T; b++) bucket_start[b] = 0;
    for (int64_t i = 0; i < n; i++) {
        uint32_t h = orc_hash(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], T);
        bucket_start[h + 1] += 1;
    }
    for (uint32_t b = 0; b < T; b++) bucket_start[b + 1] += bucket_start[b];
    for (uint32_t b = 0; b <= T; b++) cursor[b] = bucket_start[b];
    for (int64_t i = 0; i < n; i++) {
        uint32_t h = orc_hash(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], T);
        bucket_entry[cursor[h]] = (int32_t)i;
        cursor[h] += 1;
    }
    free(cursor);
    /* duplicates: an earlier entry of the same bucket with equal coordinates */
    for (int64_t i = 0; i < n; i++) {
        uint32_t h = orc_hash(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], T);
        for (uint32_t k = bucket_start[h]; k < bucket_start[h + 1]; k++) {
            int64_t j = bucket_entry[k];
            if (j >= i) break;
            if (xyz[3 * j] == xyz[3 * i] && xyz[3 * j + 1] == xyz[3 * i + 1] && xyz[3 * j + 2] == xyz[3 * i + 2]) {
                if (dup_j) *dup_j = j;
                return i;
            }
        }
    }
    return -1;
}

/* Caller index of block (x,y,z), or -1 if not allocated (S:67-75 locate with allocate=false). */
int64_t orc_lookup(const int32_t *xyz, const uint32_t *bucket_start, const int32_t *bucket_entry,
                   uint32_t T, int32_t x, int32_t y, int32_t z)
{
    uint32_t h = orc_hash(x, y, z, T);
    for (uint32_t k = bucket_start[h]; k < bucket_start[h + 1]; k++) {
        int64_t j = bucket_entry[k];
        if (xyz[3 * j] == x && xyz[3 * j + 1] == y && xyz[3 * j + 2] == z) return j;
    }
    return -1;
}

/* nbr[6i + d], d = (−x,+x,−y,+y,−z,+z): caller index of the face neighbour or -1. */
void orc_neighbours(const int32_t *xyz, int64_t n, uint32_t T, const uint32_t *bucket_start,
                    const int32_t *bucket_entry, int32_t *nbr)
{
    static const int D[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};
    for (int64_t i = 0; i < n; i++)
        for (int d = 0; d < 6; d++)
            nbr[6 * i + d] = (int32_t)orc_lookup(xyz, bucket_start, bucket_entry, T, xyz[3 * i] + D[d][0],
                                                 xyz[3 * i + 1] + D[d][1], xyz[3 * i + 2] + D[d][2]);
}

/* Linear index (block·512 + x + 8y + 64z) of the voxel one step along `axis` (0,1,2) in direction
 * `dir` (+1/−1) from voxel v, or -1 if that voxel lies in an unallocated block.                  */
static int64_t orc_step(const int32_t *nbr, int64_t v, int axis, int dir)
{
    int64_t b = v / 512;
    int loc = (int)(v % 512);
    int c[3] = {loc % 8, (loc / 8) % 8, loc / 64};
    c[axis] += dir;
    if (c[axis] < 0 || c[axis] > 7) {
        int32_t nb = nbr[6 * b + 2 * axis + (dir > 0 ? 1 : 0)];
        if (nb < 0) return -1;
        c[axis] = (c[axis] + 8) % 8;
        b = nb;
    }
    return b * 512 + c[0] + 8 * c[1] + 64 * c[2];
}

/* ------------------------------------------- precision-dependent part, compiled twice */
#define REAL double
#define SQRT sqrt
#define SFX(name) name##_f64
#include "hvg_oracle_real.inc"
#undef REAL
#undef SQRT
#undef SFX
#define REAL float
#define SQRT sqrtf
#define SFX(name) name##_f32
#include "hvg_oracle_real.inc"
#undef REAL
#undef SQRT
#undef SFX


/* ------------------------------------------------------------------------ energy (fp64 only) */

/* Primal energy (Eq. 2, with Huber TV and the W-weighted data term of reading c-1):
 *   P(u) = Σ_Ω H_ε(‖∇_Ω u‖₂) + λ Σ_Ω W|u − f|            (data_term 0, L1)
 *   P(u) = Σ_Ω H_ε(‖∇_Ω u‖₂) + (λ/2) Σ_Ω W (u − f)²      (data_term 1, L2)
 *   H_ε(s) = s²/(2ε) if s ≤ ε else s − ε/2  (H_0(s) = s).
 * Dual value, p given: L2  D = −(ε/2)Σ‖p‖² − Σ_Ω [f·div p + (div p)²/(2λW)];
 * L1: D = −(ε/2)Σ‖p̂‖² − Σ_Ω f·div p̂ at p̂ = s·p, s = min(1, min_v λW_v/|div p(v)|).
 * u is double [N]; p double [3][N] or NULL (then *dual is not written).                          */
void orc_energy(int64_t n, const int32_t *nbr, const float *f, const float *W, const double *u,
                const double *p, double lam, double eps, int data_term, double *primal, double *dual)
{
    int64_t N = 512 * n;
    double *g = (double *)malloc(sizeof(double) * 3 * (size_t)N);
    orc_gradient_f64(n, nbr, W, u, g);
    double P = 0.0;
    for (int64_t v = 0; v < N; v++) {
        if (!(W[v] > 0.0f)) continue;
        double s = sqrt(g[v] * g[v] + g[N + v] * g[N + v] + g[2 * N + v] * g[2 * N + v]);
        double h = (eps > 0.0 && s <= eps) ? s * s / (2.0 * eps) : s - eps / 2.0;
        double r = u[v] - (double)f[v];
        double dt = data_term == 0 ? lam * (double)W[v] * fabs(r) : 0.5 * lam * (double)W[v] * r * r;
        P += h + dt;
    }
    *primal = P;
    free(g);
    if (!p || !dual) return;
    double *d = (double *)malloc(sizeof(double) * (size_t)N);
    orc_divergence_f64(n, nbr, W, p, d);
    double scale = 1.0;
    if (data_term == 0) {
        for (int64_t v = 0; v < N; v++) {
            if (!(W[v] > 0.0f)) continue;
            double lim = lam * (double)W[v];
            if (fabs(d[v]) > lim) {
                double s = lim / fabs(d[v]);
                if (s < scale) scale = s;
            }
        }
    }
    double D = 0.0;
    for (int64_t v = 0; v < N; v++) {
        if (!(W[v] > 0.0f)) continue;
        double p0 = scale * p[v], p1 = scale * p[N + v], p2 = scale * p[2 * N + v];
        double dv = scale * d[v];
        D -= 0.5 * eps * (p0 * p0 + p1 * p1 + p2 * p2);
        D -= (double)f[v] * dv;
        if (data_term == 1) D -= dv * dv / (2.0 * lam * (double)W[v]);
    }
    *dual = D;
    free(d);
}
