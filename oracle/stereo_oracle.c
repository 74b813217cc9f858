/*
 * oracle/stereo_oracle.c — plain, slow, obviously-correct CPU oracle of the depth-map estimation module
 * (arXiv 1604.03734 §IV: census-transform data term, tensor-weighted TGV regulariser; SURVEY.md §8(f)
 * NEXT-4).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py may load this library.
 * It shares no code, header, table or constant with the CUDA path (paper_1604_03734_b200/csrc).
 *
 * Citations: P:n = PAPER.md line n (§IV: P:492-552), S:n = SPEC.md line n (stereo-depth module,
 * S:342-438, used for interfaces, worked examples and the gap ledger).  Readings S-1 … S-12: DESIGN.md
 * §13.  All arithmetic is IEEE fp32 in the order written here (compile with -ffp-contract=off), except
 * the tensor, evaluated in fp64 and rounded once to fp32 (S-5).
 *
 *   census    P:515-518: a bit per window pixel, "set to 1 if the corresponding pixel has a lower
 *             intensity than the pixel of interest"; window w×w (odd, default 5), bits in
 *             row-major window order without the centre, bit k = (k-th neighbour < centre), borders
 *             clamp to the edge;
 *   data term P:510-513: ρ(d, x, y) = Sim(I_L(x + d, y), I_R(x, y)) — the right image is the reference;
 *             Sim = Hamming distance of the signatures, used as is (reading S-3: not normalised,
 *             so λ_2D = 0.5 of Table I weighs bit counts); x + d outside the image → maximal cost
 *             w² − 1;
 *   tensor    P:540-546: T = exp(−γ|∇I|^β) n nᵀ + n⊥ n⊥ᵀ, n = ∇I/|∇I|, ∇I by central differences of I_R
 *             (clamp to edge), T = identity if |∇I| < 1e-6;
 *   TGV       P:524-529, Eq. reg_2D: α₁ Σ|T∇d − w|₂ + α₂ Σ|∇w|_F (S-6), forward differences with
 *             Neumann boundary (zero difference on the last column / row), divergences their negative
 *             adjoints;
 *   solver    S:398 / S:422 (the paper defers to Ranftl et al. [ranftl2012pushing]): quadratic
 *             relaxation E = TGV(d, w) + 1/(2θ) Σ(d − a)² + λ Σ ρ(a); `outer` rounds of `inner`
 *             Chambolle–Pock iterations on (d, w) with a fixed, then the exact point-wise minimisation
 *             of 1/(2θ)(d − a)² + λρ(a) over the integer disparities with a 3-point parabola sub-pixel
 *             step; θ decreases geometrically from θ₀ to θ_end.  Reading S-13: the ball
 *             projections are p·fl(α/‖p‖) when ‖p‖ > α and the coupling prox divides by (1 + τ/θ) as a
 *             product with fl(1/(1 + τ/θ)) — the same real numbers as Eq.'s prox steps.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* ------------------------------------------------------------------------------------ census */

/* sig [H][W]: bit k (row-major over the window, centre skipped) = neighbour < centre. */
void orc_census(const float *I, int H, int W, int win, uint32_t *sig)
{
    int r = win / 2;
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            float c = I[y * W + x];
            uint32_t s = 0;
            int k = 0;
            for (int dy = -r; dy <= r; dy++)
                for (int dx = -r; dx <= r; dx++) {
                    if (dx == 0 && dy == 0) continue;
                    float v = I[clampi(y + dy, 0, H - 1) * W + clampi(x + dx, 0, W - 1)];
                    if (v < c) s |= 1u << k;
                    k++;
                }
            sig[y * W + x] = s;
        }
}

static int popcount32(uint32_t v)
{
    int c = 0;
    while (v) { c += (int)(v & 1u); v >>= 1; }
    return c;
}

/* cost [H][W][D] (integer Hamming distances): cost(x, y, d) = |sig_R(x, y) ⊕ sig_L(x + d, y)|,
 * win² − 1 when x + d >= W. */
void orc_cost(const uint32_t *sigL, const uint32_t *sigR, int H, int W, int D, int win, uint8_t *cost)
{
    int maxc = win * win - 1;
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++)
            for (int d = 0; d < D; d++) {
                int c = maxc;
                if (x + d < W) c = popcount32(sigR[y * W + x] ^ sigL[y * W + x + d]);
                cost[((size_t)y * W + x) * D + d] = (uint8_t)c;
            }
}

/* ------------------------------------------------------------------------------------ tensor */

/* T [H][W][3] = (T11, T12, T22) of P:544, evaluated in fp64 and rounded to fp32 (reading S-5). */
void orc_tensor(const float *I, int H, int W, float beta, float gamma, float *T)
{
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            double gx = ((double)I[y * W + clampi(x + 1, 0, W - 1)] - (double)I[y * W + clampi(x - 1, 0, W - 1)]) / 2.0;
            double gy = ((double)I[clampi(y + 1, 0, H - 1) * W + x] - (double)I[clampi(y - 1, 0, H - 1) * W + x]) / 2.0;
            double g = sqrt(gx * gx + gy * gy);
            double t11 = 1.0, t12 = 0.0, t22 = 1.0;
            if (g >= 1e-6) {
                double nx = gx / g, ny = gy / g;
                double e = exp(-(double)gamma * pow(g, (double)beta));
                t11 = e * nx * nx + ny * ny;          /* e·n nᵀ + n⊥ n⊥ᵀ, n⊥ = (−ny, nx) */
                t12 = e * nx * ny - nx * ny;
                t22 = e * ny * ny + nx * nx;
            }
            T[3 * (y * W + x)] = (float)t11;
            T[3 * (y * W + x) + 1] = (float)t12;
            T[3 * (y * W + x) + 2] = (float)t22;
        }
}

/* ------------------------------------------------------------------------------------ TGV operators */

/* forward differences with Neumann boundary (zero on the last column / row) */
static float fdx(const float *f, int H, int W, int x, int y) { (void)H; return x < W - 1 ? f[y * W + x + 1] - f[y * W + x] : 0.0f; }
static float fdy(const float *f, int H, int W, int x, int y) { return y < H - 1 ? f[(y + 1) * W + x] - f[y * W + x] : 0.0f; }
/* backward divergence: the negative adjoint of (fdx, fdy) */
static float bdx(const float *f, int H, int W, int x, int y)
{
    (void)H;
    float a = x < W - 1 ? f[y * W + x] : 0.0f;
    float b = x > 0 ? f[y * W + x - 1] : 0.0f;
    return a - b;
}
static float bdy(const float *f, int H, int W, int x, int y)
{
    float a = y < H - 1 ? f[y * W + x] : 0.0f;
    float b = y > 0 ? f[(y - 1) * W + x] : 0.0f;
    return a - b;
}

/* K(d, w) = (T∇d − w, ∇w):  u [2][H][W], v [4][H][W] = (∂x w1, ∂y w1, ∂x w2, ∂y w2). */
void orc_tgv_K(const float *T, const float *d, const float *w, int H, int W, float *u, float *v)
{
    size_t n = (size_t)H * W;
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            size_t i = (size_t)y * W + x;
            float gx = fdx(d, H, W, x, y), gy = fdy(d, H, W, x, y);
            float tx = T[3 * i] * gx + T[3 * i + 1] * gy;
            float ty = T[3 * i + 1] * gx + T[3 * i + 2] * gy;
            u[i] = tx - w[i];
            u[n + i] = ty - w[n + i];
            v[i] = fdx(w, H, W, x, y);
            v[n + i] = fdy(w, H, W, x, y);
            v[2 * n + i] = fdx(w + n, H, W, x, y);
            v[3 * n + i] = fdy(w + n, H, W, x, y);
        }
}

/* Kᵀ(p, q) = (−div(T p), −p − div q):  kd [H][W], kw [2][H][W].  tp is scratch [2][H][W]. */
void orc_tgv_KT(const float *T, const float *p, const float *q, int H, int W, float *kd, float *kw, float *tp)
{
    size_t n = (size_t)H * W;
    for (size_t i = 0; i < n; i++) {
        tp[i] = T[3 * i] * p[i] + T[3 * i + 1] * p[n + i];
        tp[n + i] = T[3 * i + 1] * p[i] + T[3 * i + 2] * p[n + i];
    }
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            size_t i = (size_t)y * W + x;
            kd[i] = -(bdx(tp, H, W, x, y) + bdy(tp + n, H, W, x, y));
            kw[i] = -(p[i] + (bdx(q, H, W, x, y) + bdy(q + n, H, W, x, y)));
            kw[n + i] = -(p[n + i] + (bdx(q + 2 * n, H, W, x, y) + bdy(q + 3 * n, H, W, x, y)));
        }
}

/* ------------------------------------------------------------------------------------ data step */

/* a = argmin_k c·(d − k)² + λ·ρ_k over k = 0 … D−1 (ties: smallest k), then the parabola step
 * δ = (E₋ − E₊)/(2·((E₋ − 2E₀) + E₊)) for 0 < k* < D−1 when the denominator is > 0, clamped to
 * [−½, ½] (reading S-9).  rho [D] normalised costs.                                                */
float orc_data_step(float d, const float *rho, int D, float c, float lambda)
{
    int best = 0;
    float eb = 0.0f;
    for (int k = 0; k < D; k++) {
        float diff = d - (float)k;
        float e = c * (diff * diff) + lambda * rho[k];
        if (k == 0 || e < eb) { eb = e; best = k; }
    }
    float a = (float)best;
    if (best > 0 && best < D - 1) {
        float dm = d - (float)(best - 1), dp = d - (float)(best + 1);
        float em = c * (dm * dm) + lambda * rho[best - 1];
        float ep = c * (dp * dp) + lambda * rho[best + 1];
        float den = (em - 2.0f * eb) + ep;
        if (den > 0.0f) {
            float delta = (em - ep) / (2.0f * den);
            if (delta > 0.5f) delta = 0.5f;
            if (delta < -0.5f) delta = -0.5f;
            a = a + delta;
        }
    }
    return a;
}

/* ------------------------------------------------------------------------------------ the solver */

typedef struct {
    int win, D, outer, inner;
    float lambda, alpha1, alpha2, beta, gamma, theta0, theta_end, tau, sigma;
} orc_stereo_params;

/* θ of outer round o (fp64, rounded to fp32): θ₀·(θ_end/θ₀)^(o/(outer−1)). */
float orc_stereo_theta(const orc_stereo_params *P, int o)
{
    if (P->outer <= 1) return P->theta0;
    double r = (double)o / (double)(P->outer - 1);
    return (float)((double)P->theta0 * pow((double)P->theta_end / (double)P->theta0, r));
}

/* Full solve of one rectified pair.  Outputs: d [H][W], w [2][H][W] (may be NULL), a [H][W] (the last
 * data-step result, may be NULL).  Returns 0, or -1 on bad parameters.                            */
int orc_stereo(const float *IL, const float *IR, int H, int W, const orc_stereo_params *P, float *d_out,
               float *w_out, float *a_out)
{
    if (H < 1 || W < 1 || P->D < 1 || (P->win != 3 && P->win != 5)) return -1;   /* 24-bit signatures at most */
    size_t n = (size_t)H * W;
    int D = P->D;
    uint32_t *sL = malloc(n * 4), *sR = malloc(n * 4);
    uint8_t *cost = malloc(n * (size_t)D);
    float *T = malloc(n * 12), *rho = malloc(n * (size_t)D * 4);
    float *d = malloc(n * 4), *db = malloc(n * 4), *a = malloc(n * 4), *dn = malloc(n * 4);
    float *w = calloc(2 * n, 4), *wb = calloc(2 * n, 4), *wn = malloc(2 * n * 4);
    float *p = calloc(2 * n, 4), *q = calloc(4 * n, 4);
    float *u = malloc(2 * n * 4), *v = malloc(4 * n * 4), *kd = malloc(n * 4), *kw = malloc(2 * n * 4),
          *tp = malloc(2 * n * 4);
    orc_census(IL, H, W, P->win, sL);
    orc_census(IR, H, W, P->win, sR);
    orc_cost(sL, sR, H, W, D, P->win, cost);
    orc_tensor(IR, H, W, P->beta, P->gamma, T);
    for (size_t i = 0; i < n * (size_t)D; i++) rho[i] = (float)cost[i];   /* S-3: the Hamming distance */
    /* init (S-8): winner-take-all a = d = argmin ρ (ties: smallest), w = p = q = 0 */
    for (size_t i = 0; i < n; i++) {
        int best = 0;
        for (int k = 1; k < D; k++)
            if (cost[i * D + k] < cost[i * D + best]) best = k;
        a[i] = d[i] = db[i] = (float)best;
    }
    for (int o = 0; o < P->outer; o++) {
        float theta = orc_stereo_theta(P, o);
        float tt = P->tau / theta;                 /* τ/θ */
        float kd_inv = 1.0f / (1.0f + tt);         /* the prox divisor as a reciprocal (reading S-13) */
        for (int it = 0; it < P->inner; it++) {
            /* dual ascent on the frozen relaxed primal (d̄, w̄), projections onto the α-balls */
            orc_tgv_K(T, db, wb, H, W, u, v);
            for (size_t i = 0; i < n; i++) {
                float p1 = p[i] + P->sigma * u[i], p2 = p[n + i] + P->sigma * u[n + i];
                /* projection onto the α₁-ball, p·(α₁/‖p‖) when ‖p‖ > α₁ (reading S-13) */
                float nrm = sqrtf(p1 * p1 + p2 * p2);
                if (nrm > P->alpha1) { float r = P->alpha1 / nrm; p1 = p1 * r; p2 = p2 * r; }
                p[i] = p1;
                p[n + i] = p2;
                float q1 = q[i] + P->sigma * v[i], q2 = q[n + i] + P->sigma * v[n + i];
                float q3 = q[2 * n + i] + P->sigma * v[2 * n + i], q4 = q[3 * n + i] + P->sigma * v[3 * n + i];
                float nq = sqrtf(((q1 * q1 + q2 * q2) + q3 * q3) + q4 * q4);
                if (nq > P->alpha2) { float r = P->alpha2 / nq; q1 = q1 * r; q2 = q2 * r; q3 = q3 * r; q4 = q4 * r; }
                q[i] = q1; q[n + i] = q2; q[2 * n + i] = q3; q[3 * n + i] = q4;
            }
            /* primal descent: prox of the coupling for d, plain step for w; over-relaxation θ = 1 */
            orc_tgv_KT(T, p, q, H, W, kd, kw, tp);
            for (size_t i = 0; i < n; i++) {
                dn[i] = ((d[i] - P->tau * kd[i]) + tt * a[i]) * kd_inv;
                wn[i] = w[i] - P->tau * kw[i];
                wn[n + i] = w[n + i] - P->tau * kw[n + i];
            }
            for (size_t i = 0; i < n; i++) {
                db[i] = dn[i] + (dn[i] - d[i]);
                wb[i] = wn[i] + (wn[i] - w[i]);
                wb[n + i] = wn[n + i] + (wn[n + i] - w[n + i]);
                d[i] = dn[i];
                w[i] = wn[i];
                w[n + i] = wn[n + i];
            }
        }
        /* data step (exact point-wise minimisation over the integer disparities + parabola) */
        float c = 1.0f / (2.0f * theta);
        for (size_t i = 0; i < n; i++) a[i] = orc_data_step(d[i], rho + i * D, D, c, P->lambda);
    }
    memcpy(d_out, d, n * 4);
    if (w_out) memcpy(w_out, w, 2 * n * 4);
    if (a_out) memcpy(a_out, a, n * 4);
    free(sL); free(sR); free(cost); free(T); free(rho); free(d); free(db); free(a); free(dn);
    free(w); free(wb); free(wn); free(p); free(q); free(u); free(v); free(kd); free(kw); free(tp);
    return 0;
}
