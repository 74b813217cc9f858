// stereo.cu — depth-map estimation on the device (arXiv 1604.03734 §IV): census
// signatures, Hamming matching cost with the right image as reference, the
// anisotropic tensor T = exp(−γ|∇I|^β) n nᵀ + n⊥ n⊥ᵀ and the tensor-TGV energy
// minimised by quadratic relaxation: `outer` rounds of `inner` Chambolle–Pock iterations on (d, w)
// followed by the exact point-wise data step with parabola sub-pixel refinement.  Readings S-1 … S-12:
// DESIGN.md §13.  Batched over frames: every field is [F][H][W] (structure of arrays).
//
// Kernels (one thread per pixel of the batch):
//   k_census        both images, window 3 or 5, clamp-to-edge;
//   k_tensor        T from central differences of I_R, in fp64, rounded to fp32 (S-5);
//   k_wta           winner-take-all init a = d = d̄ = argmin cost (ties: smallest), w = w̄ = p = q = 0;
//   k_dual          p ← P_α1(p + σ(T∇d̄ − w̄)),  q ← P_α2(q + σ∇w̄);
//   k_primal        d ← ((d − τ·kd) + (τ/θ)a)/(1 + τ/θ),  w ← w − τ·kw  with (kd, kw) = Kᵀ(p, q);
//                   d̄ = 2d' − d, w̄ = 2w' − w;
//   k_data          a ← argmin_k 1/(2θ)(d − k)² + λρ_k, ρ_k = Hamming distance (S-3), parabola step.
// All fp32 arithmetic in the written order of the readings (--fmad=false; explicit _rn intrinsics).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>

#include "../../include/vol.h"
#include "handle.h"
#include "internal.h"

namespace hvg {
namespace {

struct Img {
    int F, H, W;
    __device__ __forceinline__ long long n() const { return (long long)F * H * W; }
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

__global__ void k_census(const float *__restrict__ I, Img g, int win, uint32_t *__restrict__ sig) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n()) return;
    const int x = (int)(i % g.W);
    const long long fy = i / g.W;
    const int y = (int)(fy % g.H);
    const float *If = I + (fy / g.H) * (long long)g.H * g.W;
    const float c = If[(long long)y * g.W + x];
    const int r = win / 2;
    uint32_t s = 0;
    int k = 0;
    for (int dy = -r; dy <= r; dy++)
        for (int dx = -r; dx <= r; dx++) {
            if (dx == 0 && dy == 0) continue;
            const float v = __ldg(If + (long long)clampi(y + dy, 0, g.H - 1) * g.W + clampi(x + dx, 0, g.W - 1));
            s |= (uint32_t)(v < c) << k;   // bit set iff the neighbour is darker than the centre
            k++;
        }
    sig[i] = s;
}

__global__ void k_tensor(const float *__restrict__ I, Img g, float beta, float gamma, float *__restrict__ T11,
                         float *__restrict__ T12, float *__restrict__ T22) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n()) return;
    const int x = (int)(i % g.W);
    const long long fy = i / g.W;
    const int y = (int)(fy % g.H);
    const float *If = I + (fy / g.H) * (long long)g.H * g.W;
    const double gx = __ddiv_rn(__dsub_rn((double)If[(long long)y * g.W + clampi(x + 1, 0, g.W - 1)],
                                          (double)If[(long long)y * g.W + clampi(x - 1, 0, g.W - 1)]), 2.0);
    const double gy = __ddiv_rn(__dsub_rn((double)If[(long long)clampi(y + 1, 0, g.H - 1) * g.W + x],
                                          (double)If[(long long)clampi(y - 1, 0, g.H - 1) * g.W + x]), 2.0);
    const double gn = __dsqrt_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)));
    double t11 = 1.0, t12 = 0.0, t22 = 1.0;
    if (gn >= 1e-6) {
        const double nx = __ddiv_rn(gx, gn), ny = __ddiv_rn(gy, gn);
        const double e = exp(-(double)gamma * pow(gn, (double)beta));
        t11 = __dadd_rn(__dmul_rn(__dmul_rn(e, nx), nx), __dmul_rn(ny, ny));
        t12 = __dsub_rn(__dmul_rn(__dmul_rn(e, nx), ny), __dmul_rn(nx, ny));
        t22 = __dadd_rn(__dmul_rn(__dmul_rn(e, ny), ny), __dmul_rn(nx, nx));
    }
    T11[i] = (float)t11;
    T12[i] = (float)t12;
    T22[i] = (float)t22;
}

struct State {
    float *d, *db, *a, *w1, *w2, *wb1, *wb2, *p1, *p2, *q1, *q2, *q3, *q4;
    const float *T11, *T12, *T22;
    const uint32_t *sL, *sR;
};

__device__ __forceinline__ int cost_at(const uint32_t *sL, uint32_t sr, int x, int W, long long rowL, int k,
                                       int maxc) {
    return x + k < W ? __popc(sr ^ sL[rowL + x + k]) : maxc;
}

__global__ void k_wta(State S, Img g, int D, int maxc) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n()) return;
    const int x = (int)(i % g.W);
    const long long row = i - x;
    const uint32_t sr = S.sR[i];
    int best = 0, cb = cost_at(S.sL, sr, x, g.W, row, 0, maxc);
    for (int k = 1; k < D; k++) {
        const int c = cost_at(S.sL, sr, x, g.W, row, k, maxc);
        if (c < cb) {
            cb = c;
            best = k;
        }
    }
    const float v = (float)best;
    S.a[i] = v;
    S.d[i] = v;
    S.db[i] = v;
    S.w1[i] = S.w2[i] = S.wb1[i] = S.wb2[i] = 0.0f;
    S.p1[i] = S.p2[i] = 0.0f;
    S.q1[i] = S.q2[i] = S.q3[i] = S.q4[i] = 0.0f;
}

struct Steps {
    float sigma, tau, alpha1, alpha2, tt;   // tt = fl(τ/θ)
    float kinv;                             // fl(1/fl(1 + tt)): the coupling prox divisor (reading S-13)
};

// Projections onto the α-balls: p·fl(α/‖p‖) when ‖p‖ > α (reading S-13), sums in the written order.
// ‖p‖² <= α²·(1 − 2·10⁻⁶) (fp32, every rounding far inside that margin) proves fl(√‖p‖²) < α: no square root
// is needed to know that the projection is the identity (same bits as the written order).
__device__ __forceinline__ void project2(float &p1, float &p2, float alpha) {
    const float n2 = __fadd_rn(__fmul_rn(p1, p1), __fmul_rn(p2, p2));
    if (n2 <= alpha * alpha * 0.999998f) return;
    const float nrm = __fsqrt_rn(n2);
    if (nrm > alpha) {
        const float r = __fdiv_rn(alpha, nrm);
        p1 = __fmul_rn(p1, r);
        p2 = __fmul_rn(p2, r);
    }
}
__device__ __forceinline__ void project4(float &q1, float &q2, float &q3, float &q4, float alpha) {
    const float n2 = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(q1, q1), __fmul_rn(q2, q2)), __fmul_rn(q3, q3)),
                               __fmul_rn(q4, q4));
    if (n2 <= alpha * alpha * 0.999998f) return;
    const float nrm = __fsqrt_rn(n2);
    if (nrm > alpha) {
        const float r = __fdiv_rn(alpha, nrm);
        q1 = __fmul_rn(q1, r);
        q2 = __fmul_rn(q2, r);
        q3 = __fmul_rn(q3, r);
        q4 = __fmul_rn(q4, r);
    }
}

// forward differences with Neumann boundary (zero on the last column / row)
__device__ __forceinline__ float fdx(const float *f, long long i, int x, int W) {
    return x < W - 1 ? __fsub_rn(f[i + 1], f[i]) : 0.0f;
}
__device__ __forceinline__ float fdy(const float *f, long long i, int y, int H, int W) {
    return y < H - 1 ? __fsub_rn(f[i + W], f[i]) : 0.0f;
}

__global__ void k_dual(State S, Img g, Steps P) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n()) return;
    const int x = (int)(i % g.W);
    const int y = (int)((i / g.W) % g.H);
    // u = T∇d̄ − w̄
    const float gx = fdx(S.db, i, x, g.W), gy = fdy(S.db, i, y, g.H, g.W);
    const float t11 = S.T11[i], t12 = S.T12[i], t22 = S.T22[i];
    const float tx = __fadd_rn(__fmul_rn(t11, gx), __fmul_rn(t12, gy));
    const float ty = __fadd_rn(__fmul_rn(t12, gx), __fmul_rn(t22, gy));
    const float u1 = __fsub_rn(tx, S.wb1[i]), u2 = __fsub_rn(ty, S.wb2[i]);
    float p1 = __fadd_rn(S.p1[i], __fmul_rn(P.sigma, u1));
    float p2 = __fadd_rn(S.p2[i], __fmul_rn(P.sigma, u2));
    project2(p1, p2, P.alpha1);
    S.p1[i] = p1;
    S.p2[i] = p2;
    // v = ∇w̄
    float q1 = __fadd_rn(S.q1[i], __fmul_rn(P.sigma, fdx(S.wb1, i, x, g.W)));
    float q2 = __fadd_rn(S.q2[i], __fmul_rn(P.sigma, fdy(S.wb1, i, y, g.H, g.W)));
    float q3 = __fadd_rn(S.q3[i], __fmul_rn(P.sigma, fdx(S.wb2, i, x, g.W)));
    float q4 = __fadd_rn(S.q4[i], __fmul_rn(P.sigma, fdy(S.wb2, i, y, g.H, g.W)));
    project4(q1, q2, q3, q4, P.alpha2);
    S.q1[i] = q1;
    S.q2[i] = q2;
    S.q3[i] = q3;
    S.q4[i] = q4;
}

// backward divergence term of one component at pixel i: (x < W−1 ? f(i) : 0) − (x > 0 ? f(i−1) : 0)
__device__ __forceinline__ float bd(float here, float before, bool has_here, bool has_before) {
    return __fsub_rn(has_here ? here : 0.0f, has_before ? before : 0.0f);
}

__global__ void k_primal(State S, Img g, Steps P) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n()) return;
    const int x = (int)(i % g.W);
    const int y = (int)((i / g.W) % g.H);
    // T p at this pixel and at the −x / −y neighbours (same operations everywhere)
    auto tp = [&](long long j, float &a1, float &a2) {
        const float p1 = S.p1[j], p2 = S.p2[j];
        a1 = __fadd_rn(__fmul_rn(S.T11[j], p1), __fmul_rn(S.T12[j], p2));
        a2 = __fadd_rn(__fmul_rn(S.T12[j], p1), __fmul_rn(S.T22[j], p2));
    };
    float h1, h2, l1 = 0.f, l2 = 0.f, u1 = 0.f, u2 = 0.f;
    tp(i, h1, h2);
    if (x > 0) tp(i - 1, l1, l2);
    if (y > 0) tp(i - g.W, u1, u2);
    const bool hx = x < g.W - 1, bx = x > 0, hy = y < g.H - 1, by = y > 0;
    const float kd = -__fadd_rn(bd(h1, l1, hx, bx), bd(h2, u2, hy, by));
    (void)u1;
    (void)l2;
    const float dq1 = __fadd_rn(bd(S.q1[i], bx ? S.q1[i - 1] : 0.f, hx, bx), bd(S.q2[i], by ? S.q2[i - g.W] : 0.f, hy, by));
    const float dq2 = __fadd_rn(bd(S.q3[i], bx ? S.q3[i - 1] : 0.f, hx, bx), bd(S.q4[i], by ? S.q4[i - g.W] : 0.f, hy, by));
    const float kw1 = -__fadd_rn(S.p1[i], dq1);
    const float kw2 = -__fadd_rn(S.p2[i], dq2);
    const float d = S.d[i], w1 = S.w1[i], w2 = S.w2[i];
    const float dn = __fmul_rn(__fadd_rn(__fsub_rn(d, __fmul_rn(P.tau, kd)), __fmul_rn(P.tt, S.a[i])), P.kinv);
    const float wn1 = __fsub_rn(w1, __fmul_rn(P.tau, kw1));
    const float wn2 = __fsub_rn(w2, __fmul_rn(P.tau, kw2));
    S.db[i] = __fadd_rn(dn, __fsub_rn(dn, d));
    S.wb1[i] = __fadd_rn(wn1, __fsub_rn(wn1, w1));
    S.wb2[i] = __fadd_rn(wn2, __fsub_rn(wn2, w2));
    S.d[i] = dn;
    S.w1[i] = wn1;
    S.w2[i] = wn2;
}

// Quad forms of k_dual / k_primal (widths divisible by 4): four consecutive pixels of a row per thread,
// 128-bit loads and stores, 32-bit index arithmetic once per quad.  Per pixel the operations, their
// operands and their order are exactly those of k_dual / k_primal (bit-identical results).
__device__ __forceinline__ void ld4(const float *p, float (&a)[4]) {
    const float4 v = *reinterpret_cast<const float4 *>(p);
    a[0] = v.x; a[1] = v.y; a[2] = v.z; a[3] = v.w;
}
__device__ __forceinline__ void st4(float *p, const float (&a)[4]) {
    *reinterpret_cast<float4 *>(p) = make_float4(a[0], a[1], a[2], a[3]);
}

struct Quad {
    unsigned i;      // pixel index of the first pixel of the quad
    int x0, y;
    bool hasx;       // the quad's last pixel has a +x neighbour (x0 + 3 < W − 1)
    bool hasy;       // y < H − 1
};
__device__ __forceinline__ bool quad_of(const Img &g, Quad &q) {
    const unsigned Wq = (unsigned)g.W >> 2;
    const unsigned qi = blockIdx.x * blockDim.x + threadIdx.x;
    if (qi >= (unsigned)(g.n() >> 2)) return false;
    const unsigned row = qi / Wq;
    q.x0 = 4 * (int)(qi - row * Wq);
    q.y = (int)(row % (unsigned)g.H);
    q.i = 4u * qi;
    q.hasx = q.x0 + 4 < g.W;
    q.hasy = q.y < g.H - 1;
    return true;
}

#ifndef HVG_DUAL4_MINB
#define HVG_DUAL4_MINB 1
#endif
#ifndef HVG_PRIMAL4_MINB
#define HVG_PRIMAL4_MINB 1
#endif
__global__ void __launch_bounds__(256, HVG_DUAL4_MINB) k_dual4(State S, Img g, Steps P) {
    Quad Q;
    if (!quad_of(g, Q)) return;
    const unsigned i = Q.i, W = (unsigned)g.W;
    float db[5], dbd[4] = {0.f, 0.f, 0.f, 0.f}, wb1[5], wb2[5], wd1[4] = {0.f, 0.f, 0.f, 0.f},
                 wd2[4] = {0.f, 0.f, 0.f, 0.f};
    float t11[4], t12[4], t22[4], p1[4], p2[4], q1[4], q2[4], q3[4], q4[4];
    ld4(S.db + i, reinterpret_cast<float(&)[4]>(db));
    ld4(S.wb1 + i, reinterpret_cast<float(&)[4]>(wb1));
    ld4(S.wb2 + i, reinterpret_cast<float(&)[4]>(wb2));
    db[4] = Q.hasx ? S.db[i + 4] : 0.f;
    wb1[4] = Q.hasx ? S.wb1[i + 4] : 0.f;
    wb2[4] = Q.hasx ? S.wb2[i + 4] : 0.f;
    if (Q.hasy) {
        ld4(S.db + i + W, dbd);
        ld4(S.wb1 + i + W, wd1);
        ld4(S.wb2 + i + W, wd2);
    }
    ld4(S.T11 + i, t11); ld4(S.T12 + i, t12); ld4(S.T22 + i, t22);
    ld4(S.p1 + i, p1); ld4(S.p2 + i, p2);
    ld4(S.q1 + i, q1); ld4(S.q2 + i, q2); ld4(S.q3 + i, q3); ld4(S.q4 + i, q4);
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const bool hx = j < 3 || Q.hasx;   // x < W − 1
        // u = T∇d̄ − w̄
        const float gx = hx ? __fsub_rn(db[j + 1], db[j]) : 0.0f;
        const float gy = Q.hasy ? __fsub_rn(dbd[j], db[j]) : 0.0f;
        const float tx = __fadd_rn(__fmul_rn(t11[j], gx), __fmul_rn(t12[j], gy));
        const float ty = __fadd_rn(__fmul_rn(t12[j], gx), __fmul_rn(t22[j], gy));
        const float u1 = __fsub_rn(tx, wb1[j]), u2 = __fsub_rn(ty, wb2[j]);
        float a1 = __fadd_rn(p1[j], __fmul_rn(P.sigma, u1));
        float a2 = __fadd_rn(p2[j], __fmul_rn(P.sigma, u2));
        project2(a1, a2, P.alpha1);
        p1[j] = a1;
        p2[j] = a2;
        // v = ∇w̄
        float b1 = __fadd_rn(q1[j], __fmul_rn(P.sigma, hx ? __fsub_rn(wb1[j + 1], wb1[j]) : 0.0f));
        float b2 = __fadd_rn(q2[j], __fmul_rn(P.sigma, Q.hasy ? __fsub_rn(wd1[j], wb1[j]) : 0.0f));
        float b3 = __fadd_rn(q3[j], __fmul_rn(P.sigma, hx ? __fsub_rn(wb2[j + 1], wb2[j]) : 0.0f));
        float b4 = __fadd_rn(q4[j], __fmul_rn(P.sigma, Q.hasy ? __fsub_rn(wd2[j], wb2[j]) : 0.0f));
        project4(b1, b2, b3, b4, P.alpha2);
        q1[j] = b1;
        q2[j] = b2;
        q3[j] = b3;
        q4[j] = b4;
    }
    st4(S.p1 + i, p1); st4(S.p2 + i, p2);
    st4(S.q1 + i, q1); st4(S.q2 + i, q2); st4(S.q3 + i, q3); st4(S.q4 + i, q4);
}

__global__ void __launch_bounds__(256, HVG_PRIMAL4_MINB) k_primal4(State S, Img g, Steps P) {
    Quad Q;
    if (!quad_of(g, Q)) return;
    const unsigned i = Q.i, W = (unsigned)g.W;
    const bool has_left = Q.x0 > 0, by = Q.y > 0;
    // T p at the quad's pixels and at the pixel before it (index 0 = i − 1), a1 component
    float p1[5], p2[5], t11[5], t12[5], t22[4];
    ld4(S.p1 + i, reinterpret_cast<float(&)[4]>(p1[1]));
    ld4(S.p2 + i, reinterpret_cast<float(&)[4]>(p2[1]));
    ld4(S.T11 + i, reinterpret_cast<float(&)[4]>(t11[1]));
    ld4(S.T12 + i, reinterpret_cast<float(&)[4]>(t12[1]));
    ld4(S.T22 + i, t22);
    p1[0] = has_left ? S.p1[i - 1] : 0.f;
    p2[0] = has_left ? S.p2[i - 1] : 0.f;
    t11[0] = has_left ? S.T11[i - 1] : 0.f;
    t12[0] = has_left ? S.T12[i - 1] : 0.f;
    float up1[4] = {0.f, 0.f, 0.f, 0.f}, up2[4] = {0.f, 0.f, 0.f, 0.f}, ut12[4] = {0.f, 0.f, 0.f, 0.f},
          ut22[4] = {0.f, 0.f, 0.f, 0.f}, uq2[4] = {0.f, 0.f, 0.f, 0.f}, uq4[4] = {0.f, 0.f, 0.f, 0.f};
    if (by) {
        ld4(S.p1 + i - W, up1); ld4(S.p2 + i - W, up2);
        ld4(S.T12 + i - W, ut12); ld4(S.T22 + i - W, ut22);
        ld4(S.q2 + i - W, uq2); ld4(S.q4 + i - W, uq4);
    }
    float q1[5], q2[4], q3[5], q4[4];
    ld4(S.q1 + i, reinterpret_cast<float(&)[4]>(q1[1]));
    ld4(S.q3 + i, reinterpret_cast<float(&)[4]>(q3[1]));
    ld4(S.q2 + i, q2);
    ld4(S.q4 + i, q4);
    q1[0] = has_left ? S.q1[i - 1] : 0.f;
    q3[0] = has_left ? S.q3[i - 1] : 0.f;
    float d[4], w1[4], w2[4], a[4];
    ld4(S.d + i, d); ld4(S.w1 + i, w1); ld4(S.w2 + i, w2); ld4(S.a + i, a);
    float h1[5];
#pragma unroll
    for (int j = 0; j < 5; j++) h1[j] = __fadd_rn(__fmul_rn(t11[j], p1[j]), __fmul_rn(t12[j], p2[j]));
    float dbo[4], wbo1[4], wbo2[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
        const bool hx = j < 3 || Q.hasx, bx = j > 0 || has_left, hy = Q.hasy;
        const float h2 = __fadd_rn(__fmul_rn(t12[j + 1], p1[j + 1]), __fmul_rn(t22[j], p2[j + 1]));
        const float l1 = bx ? h1[j] : 0.f;
        const float u2 = by ? __fadd_rn(__fmul_rn(ut12[j], up1[j]), __fmul_rn(ut22[j], up2[j])) : 0.f;
        const float kd = -__fadd_rn(bd(h1[j + 1], l1, hx, bx), bd(h2, u2, hy, by));
        const float dq1 = __fadd_rn(bd(q1[j + 1], bx ? q1[j] : 0.f, hx, bx), bd(q2[j], by ? uq2[j] : 0.f, hy, by));
        const float dq2 = __fadd_rn(bd(q3[j + 1], bx ? q3[j] : 0.f, hx, bx), bd(q4[j], by ? uq4[j] : 0.f, hy, by));
        const float kw1 = -__fadd_rn(p1[j + 1], dq1);
        const float kw2 = -__fadd_rn(p2[j + 1], dq2);
        const float dn = __fmul_rn(__fadd_rn(__fsub_rn(d[j], __fmul_rn(P.tau, kd)), __fmul_rn(P.tt, a[j])), P.kinv);
        const float wn1 = __fsub_rn(w1[j], __fmul_rn(P.tau, kw1));
        const float wn2 = __fsub_rn(w2[j], __fmul_rn(P.tau, kw2));
        dbo[j] = __fadd_rn(dn, __fsub_rn(dn, d[j]));
        wbo1[j] = __fadd_rn(wn1, __fsub_rn(wn1, w1[j]));
        wbo2[j] = __fadd_rn(wn2, __fsub_rn(wn2, w2[j]));
        d[j] = dn;
        w1[j] = wn1;
        w2[j] = wn2;
    }
    st4(S.db + i, dbo); st4(S.wb1 + i, wbo1); st4(S.wb2 + i, wbo2);
    st4(S.d + i, d); st4(S.w1 + i, w1); st4(S.w2 + i, w2);
}

// Fused iteration: dual then primal in one launch.  A CTA owns a TX×TY tile; it recomputes the dual
// update of the −x column and −y row next to the tile (same function, same inputs ⇒ bit-identical to
// the owner's), so the primal step needs no grid-wide synchronisation.  Ping-pong buffers: every field
// another CTA may read (d̄, w̄, p, q) is read from set `in` and written to set `out`; d, w, a are only
// touched by their owner and stay in place.
constexpr int TX = 32, TY = 8;
constexpr int SX = TX + 2, SY = TY + 2;   // staged box x0−1 … x0+TX, y0−1 … y0+TY

struct PP {
    const float *db, *wb1, *wb2, *p1, *p2, *q1, *q2, *q3, *q4;   // in
    float *dbo, *wb1o, *wb2o, *p1o, *p2o, *q1o, *q2o, *q3o, *q4o;  // out
    float *d, *w1, *w2;
    const float *a, *T11, *T12, *T22;
};

__global__ void __launch_bounds__(TX * TY) k_tgv_iter(PP S, Img g, Steps P) {
    __shared__ float s_db[SY][SX], s_w1[SY][SX], s_w2[SY][SX];
    __shared__ float s_p1[SY][SX], s_p2[SY][SX], s_q1[SY][SX], s_q2[SY][SX], s_q3[SY][SX], s_q4[SY][SX];
    __shared__ float s_t11[SY][SX], s_t12[SY][SX], s_t22[SY][SX];
    const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
    const long long fo = (long long)blockIdx.z * g.H * g.W;
    const int tid = threadIdx.x;
    // stage d̄, w̄ over the whole box, T, p, q over the box (−1 … +TX/TY is enough for the dual region)
    for (int k = tid; k < SX * SY; k += TX * TY) {
        const int sx = k % SX, sy = k / SX;
        const int x = x0 - 1 + sx, y = y0 - 1 + sy;
        float db = 0.f, w1 = 0.f, w2 = 0.f, p1 = 0.f, p2 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f, q4 = 0.f;
        float t11 = 0.f, t12 = 0.f, t22 = 0.f;
        if (x >= 0 && x < g.W && y >= 0 && y < g.H) {
            const long long i = fo + (long long)y * g.W + x;
            db = S.db[i];
            w1 = S.wb1[i];
            w2 = S.wb2[i];
            p1 = S.p1[i];
            p2 = S.p2[i];
            q1 = S.q1[i];
            q2 = S.q2[i];
            q3 = S.q3[i];
            q4 = S.q4[i];
            t11 = S.T11[i];
            t12 = S.T12[i];
            t22 = S.T22[i];
        }
        s_db[sy][sx] = db;
        s_w1[sy][sx] = w1;
        s_w2[sy][sx] = w2;
        s_p1[sy][sx] = p1;
        s_p2[sy][sx] = p2;
        s_q1[sy][sx] = q1;
        s_q2[sy][sx] = q2;
        s_q3[sy][sx] = q3;
        s_q4[sy][sx] = q4;
        s_t11[sy][sx] = t11;
        s_t12[sy][sx] = t12;
        s_t22[sy][sx] = t22;
    }
    __syncthreads();
    // dual step on the tile, its −x column and its −y row (reading order of k_dual); results overwrite
    // p, q in shared memory only after every thread has read its inputs
    float np1[2], np2[2], nq1[2], nq2[2], nq3[2], nq4[2];
    int ssx[2], ssy[2];
    const int n_dual = TX * TY + TX + TY;
#pragma unroll
    for (int r = 0; r < 2; r++) {
        const int k = tid + r * TX * TY;
        ssx[r] = -1;
        if (k >= n_dual) continue;
        int sx, sy;
        if (k < TX * TY) {
            sx = 1 + k % TX;
            sy = 1 + k / TX;
        } else if (k < TX * TY + TX) {
            sx = 1 + (k - TX * TY);
            sy = 0;
        } else {
            sx = 0;
            sy = 1 + (k - TX * TY - TX);
        }
        const int x = x0 - 1 + sx, y = y0 - 1 + sy;
        if (x < 0 || x >= g.W || y < 0 || y >= g.H) continue;
        ssx[r] = sx;
        ssy[r] = sy;
        const bool hx = x < g.W - 1, hy = y < g.H - 1;
        const float gx = hx ? __fsub_rn(s_db[sy][sx + 1], s_db[sy][sx]) : 0.0f;
        const float gy = hy ? __fsub_rn(s_db[sy + 1][sx], s_db[sy][sx]) : 0.0f;
        const float t11 = s_t11[sy][sx], t12 = s_t12[sy][sx], t22 = s_t22[sy][sx];
        const float tx = __fadd_rn(__fmul_rn(t11, gx), __fmul_rn(t12, gy));
        const float ty = __fadd_rn(__fmul_rn(t12, gx), __fmul_rn(t22, gy));
        const float u1 = __fsub_rn(tx, s_w1[sy][sx]), u2 = __fsub_rn(ty, s_w2[sy][sx]);
        float p1 = __fadd_rn(s_p1[sy][sx], __fmul_rn(P.sigma, u1));
        float p2 = __fadd_rn(s_p2[sy][sx], __fmul_rn(P.sigma, u2));
        project2(p1, p2, P.alpha1);
        const float v1 = hx ? __fsub_rn(s_w1[sy][sx + 1], s_w1[sy][sx]) : 0.0f;
        const float v2 = hy ? __fsub_rn(s_w1[sy + 1][sx], s_w1[sy][sx]) : 0.0f;
        const float v3 = hx ? __fsub_rn(s_w2[sy][sx + 1], s_w2[sy][sx]) : 0.0f;
        const float v4 = hy ? __fsub_rn(s_w2[sy + 1][sx], s_w2[sy][sx]) : 0.0f;
        float q1 = __fadd_rn(s_q1[sy][sx], __fmul_rn(P.sigma, v1));
        float q2 = __fadd_rn(s_q2[sy][sx], __fmul_rn(P.sigma, v2));
        float q3 = __fadd_rn(s_q3[sy][sx], __fmul_rn(P.sigma, v3));
        float q4 = __fadd_rn(s_q4[sy][sx], __fmul_rn(P.sigma, v4));
        project4(q1, q2, q3, q4, P.alpha2);
        np1[r] = p1;
        np2[r] = p2;
        nq1[r] = q1;
        nq2[r] = q2;
        nq3[r] = q3;
        nq4[r] = q4;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 2; r++) {
        if (ssx[r] < 0) continue;
        const int sx = ssx[r], sy = ssy[r];
        s_p1[sy][sx] = np1[r];
        s_p2[sy][sx] = np2[r];
        s_q1[sy][sx] = nq1[r];
        s_q2[sy][sx] = nq2[r];
        s_q3[sy][sx] = nq3[r];
        s_q4[sy][sx] = nq4[r];
    }
    __syncthreads();
    // primal step on the tile pixel of this thread (reading order of k_primal)
    const int tx_ = tid % TX, ty_ = tid / TX;
    const int x = x0 + tx_, y = y0 + ty_;
    if (x >= g.W || y >= g.H) return;
    const int sx = tx_ + 1, sy = ty_ + 1;
    const long long i = fo + (long long)y * g.W + x;
    auto tp = [&](int cx, int cy, float &a1, float &a2) {
        const float p1 = s_p1[cy][cx], p2 = s_p2[cy][cx];
        a1 = __fadd_rn(__fmul_rn(s_t11[cy][cx], p1), __fmul_rn(s_t12[cy][cx], p2));
        a2 = __fadd_rn(__fmul_rn(s_t12[cy][cx], p1), __fmul_rn(s_t22[cy][cx], p2));
    };
    float h1, h2, l1 = 0.f, l2 = 0.f, u1 = 0.f, u2 = 0.f;
    tp(sx, sy, h1, h2);
    const bool hx = x < g.W - 1, bx = x > 0, hy = y < g.H - 1, by = y > 0;
    if (bx) tp(sx - 1, sy, l1, l2);
    if (by) tp(sx, sy - 1, u1, u2);
    (void)l2;
    (void)u1;
    const float kd = -__fadd_rn(bd(h1, l1, hx, bx), bd(h2, u2, hy, by));
    const float dq1 = __fadd_rn(bd(s_q1[sy][sx], bx ? s_q1[sy][sx - 1] : 0.f, hx, bx),
                                bd(s_q2[sy][sx], by ? s_q2[sy - 1][sx] : 0.f, hy, by));
    const float dq2 = __fadd_rn(bd(s_q3[sy][sx], bx ? s_q3[sy][sx - 1] : 0.f, hx, bx),
                                bd(s_q4[sy][sx], by ? s_q4[sy - 1][sx] : 0.f, hy, by));
    const float kw1 = -__fadd_rn(s_p1[sy][sx], dq1);
    const float kw2 = -__fadd_rn(s_p2[sy][sx], dq2);
    const float d = S.d[i], w1 = S.w1[i], w2 = S.w2[i];
    const float dn = __fmul_rn(__fadd_rn(__fsub_rn(d, __fmul_rn(P.tau, kd)), __fmul_rn(P.tt, S.a[i])), P.kinv);
    const float wn1 = __fsub_rn(w1, __fmul_rn(P.tau, kw1));
    const float wn2 = __fsub_rn(w2, __fmul_rn(P.tau, kw2));
    S.dbo[i] = __fadd_rn(dn, __fsub_rn(dn, d));
    S.wb1o[i] = __fadd_rn(wn1, __fsub_rn(wn1, w1));
    S.wb2o[i] = __fadd_rn(wn2, __fsub_rn(wn2, w2));
    S.d[i] = dn;
    S.w1[i] = wn1;
    S.w2[i] = wn2;
    S.p1o[i] = s_p1[sy][sx];
    S.p2o[i] = s_p2[sy][sx];
    S.q1o[i] = s_q1[sy][sx];
    S.q2o[i] = s_q2[sy][sx];
    S.q3o[i] = s_q3[sy][sx];
    S.q4o[i] = s_q4[sy][sx];
}

__global__ void k_data(State S, Img g, int D, int maxc, float c, float lambda) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.n()) return;
    const int x = (int)(i % g.W);
    const long long row = i - x;
    const uint32_t sr = S.sR[i];
    const float d = S.d[i];
    auto energy = [&](int k) {
        const float rho = (float)cost_at(S.sL, sr, x, g.W, row, k, maxc);   // S-3: the Hamming distance
        const float diff = __fsub_rn(d, (float)k);
        return __fadd_rn(__fmul_rn(c, __fmul_rn(diff, diff)), __fmul_rn(lambda, rho));
    };
    // Exact pruning of the scan: E(k) = fl(fl(c·fl((d−k)²)) + fl(λρ)) >= fl(c·fl((d−k)²)) (λρ >= 0,
    // rounding is monotone), so every k with c(d−k)² > E(k₀) for the nearest integer k₀ has
    // E(k) > E(k₀) >= min E and can be neither the minimiser nor tied with it.  The window below
    // contains every other k with a margin of two disparities; scanning it in increasing k with the
    // strict < keeps the "smallest k among equal minima" rule of the full scan.
    int lo = 0, hi = D - 1;
    if (c > 0.0f) {
        const int k0 = (int)fminf(fmaxf(rintf(d), 0.0f), (float)(D - 1));
        const float r = __fmul_rn(sqrtf(__fdiv_rn(energy(k0), c)), 1.001f) + 2.0f;
        if (r < (float)D) {
            lo = (int)fmaxf(floorf(d - r), 0.0f);
            hi = (int)fminf(ceilf(d + r), (float)(D - 1));
        }
    }
    int best = lo;
    float eb = energy(lo);
    for (int k = lo + 1; k <= hi; k++) {
        const float e = energy(k);
        if (e < eb) {
            eb = e;
            best = k;
        }
    }
    float a = (float)best;
    if (best > 0 && best < D - 1) {
        const float em = energy(best - 1), ep = energy(best + 1);
        const float den = __fadd_rn(__fsub_rn(em, __fmul_rn(2.0f, eb)), ep);
        if (den > 0.0f) {
            float delta = __fdiv_rn(__fsub_rn(em, ep), __fmul_rn(2.0f, den));
            if (delta > 0.5f) delta = 0.5f;
            if (delta < -0.5f) delta = -0.5f;
            a = __fadd_rn(a, delta);
        }
    }
    S.a[i] = a;
}

__global__ void k_depth(const float *__restrict__ disp, long long n, float fb, float dmin, float *__restrict__ depth) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float d = disp[i];
    depth[i] = d > dmin ? __fdiv_rn(fb, d) : 0.0f;   // z = f·B/d, invalid (0) for d <= d_min
}

unsigned blocks_for(long long n, int t) { return (unsigned)((n + t - 1) / t); }

struct StereoLayout {
    float *IL, *IR;
    uint32_t *sL, *sR;
    float *T[3];
    float *f[13];
    float *g2[9];      // second buffer of d̄, w̄1, w̄2, p1, p2, q1 … q4 (fused kernel ping-pong)
    size_t bytes;
};

StereoLayout stereo_layout(char *base, long long n, bool stage_in) {
    Carve c;
    c.base = base;
    StereoLayout L{};
    L.IL = stage_in ? c.take<float>(n) : nullptr;
    L.IR = stage_in ? c.take<float>(n) : nullptr;
    L.sL = c.take<uint32_t>(n);
    L.sR = c.take<uint32_t>(n);
    for (auto &t : L.T) t = c.take<float>(n);
    for (auto &f : L.f) f = c.take<float>(n);
    for (auto &f : L.g2) f = c.take<float>(n);
    L.bytes = c.off + 256;
    return L;
}

vol_status check_params(int32_t F, const vol_stereo_params *p) {
    if (!p) return fail(VOL_EINVAL, "vol_stereo: params is NULL");
    if (F < 1) return fail(VOL_EINVAL, "vol_stereo: n_frames must be >= 1");
    if (p->width < 2 || p->height < 2) return fail(VOL_EINVAL, "vol_stereo: images must be at least 2x2");
    if ((long long)F * p->width * p->height > (1ll << 34)) return fail(VOL_EINVAL, "vol_stereo: batch too large");
    if (p->n_disp < 1 || p->n_disp > 4096) return fail(VOL_EINVAL, "vol_stereo: n_disp must be in [1, 4096]");
    if (p->window != 3 && p->window != 5) return fail(VOL_EINVAL, "vol_stereo: window must be 3 or 5");
    if (p->outer < 0 || p->inner < 0) return fail(VOL_EINVAL, "vol_stereo: negative iteration counts");
    if (!(p->lambda >= 0.0f) || !(p->alpha1 > 0.0f) || !(p->alpha2 > 0.0f) || !(p->gamma >= 0.0f) ||
        !(p->beta > 0.0f) || !(p->theta0 > 0.0f) || !(p->theta_end > 0.0f) || !(p->tau > 0.0f) || !(p->sigma > 0.0f))
        return fail(VOL_EINVAL, "vol_stereo: lambda >= 0, alpha1/alpha2/beta/theta/tau/sigma > 0, gamma >= 0 required");
    if ((double)p->tau * p->sigma * 12.0 > 1.0 + 1e-6)
        return fail(VOL_EINVAL, "vol_stereo: tau*sigma*12 must be <= 1 (||K||^2 < 12, reading S-10)");
    return VOL_OK;
}

}  // namespace
}  // namespace hvg

using namespace hvg;

extern "C" void vol_stereo_default_params(vol_stereo_params *p) {
    if (!p) return;
    p->width = 1240;
    p->height = 376;
    p->n_disp = 128;
    p->window = 5;
    p->outer = 10;
    p->inner = 20;
    p->lambda = 0.5f;    // Table I λ_2D
    p->alpha1 = 1.0f;    // Table I α₁
    p->alpha2 = 5.0f;    // Table I α₂
    p->beta = 1.0f;      // Table I β
    p->gamma = 4.0f;     // Table I γ
    p->theta0 = 1.0f;
    p->theta_end = 0.01f;
    p->tau = 1.0f / sqrtf(12.0f);
    p->sigma = 1.0f / sqrtf(12.0f);
}

extern "C" size_t vol_stereo_workspace_bytes(int32_t n_frames, const vol_stereo_params *p) {
    if (!p || n_frames < 1) return 0;
    return stereo_layout(nullptr, (long long)n_frames * p->width * p->height, true).bytes;
}

// θ of outer round o, evaluated on the host in fp64 and rounded once (reading S-8)
static float theta_of(const vol_stereo_params *P, int o) {
    if (P->outer <= 1) return P->theta0;
    const double r = (double)o / (double)(P->outer - 1);
    return (float)((double)P->theta0 * std::pow((double)P->theta_end / (double)P->theta0, r));
}

namespace {

// The whole solve of frames [c0, c0 + C) of the batch, for each chunk of `chunk` frames in turn: a chunk's
// state (~116 B per pixel) is sized to stay resident in the 126 MB L2 across its iterations.
// mode: 0 fused k_tgv_iter, 1 k_dual + k_primal, 2 k_dual4 + k_primal4 where the width allows (product)
void enqueue_solve(const StereoLayout &L, const vol_stereo_params *prm, int32_t F, int chunk, int mode,
                   const cudaStream_t *streams, int n_streams, long long &launches) {
    const long long HW = (long long)prm->width * prm->height;
    const int maxc = prm->window * prm->window - 1;
    const int TPB = 256;
    for (int c0 = 0, ci = 0; c0 < F; c0 += chunk, ci++) {
        cudaStream_t s = streams[ci % n_streams];   // chunks are independent: round-robin over the streams
        const int C = F - c0 < chunk ? F - c0 : chunk;
        const long long o = (long long)c0 * HW, n = (long long)C * HW;
        const unsigned nb = blocks_for(n, TPB);
        // quad kernels: widths divisible by 4 (16-byte aligned rows) and 32-bit pixel indices
        const bool two_kernel = mode != 0;
        const bool quads = mode == 2 && prm->width % 4 == 0 && n < (1ll << 31);
        const unsigned nq = blocks_for(n / 4, TPB);
        Img g{C, prm->height, prm->width};
        State S{L.f[0] + o, L.f[1] + o, L.f[2] + o, L.f[3] + o, L.f[4] + o, L.f[5] + o, L.f[6] + o, L.f[7] + o,
                L.f[8] + o, L.f[9] + o, L.f[10] + o, L.f[11] + o, L.f[12] + o, L.T[0] + o, L.T[1] + o, L.T[2] + o,
                L.sL + o, L.sR + o};
        k_census<<<nb, TPB, 0, s>>>(L.IL + o, g, prm->window, L.sL + o);
        k_census<<<nb, TPB, 0, s>>>(L.IR + o, g, prm->window, L.sR + o);
        k_tensor<<<nb, TPB, 0, s>>>(L.IR + o, g, prm->beta, prm->gamma, L.T[0] + o, L.T[1] + o, L.T[2] + o);
        k_wta<<<nb, TPB, 0, s>>>(S, g, prm->n_disp, maxc);
        launches += 4;
        // set 0 = the State fields (k_wta / k_dual / k_primal), set 1 = L.g2; d, w, a single
        float *set[2][9] = {{S.db, S.wb1, S.wb2, S.p1, S.p2, S.q1, S.q2, S.q3, S.q4},
                            {L.g2[0] + o, L.g2[1] + o, L.g2[2] + o, L.g2[3] + o, L.g2[4] + o, L.g2[5] + o,
                             L.g2[6] + o, L.g2[7] + o, L.g2[8] + o}};
        const dim3 tgrid((prm->width + TX - 1) / TX, (prm->height + TY - 1) / TY, C);
        int cur = 0;
        for (int oi = 0; oi < prm->outer; oi++) {
            const float theta = theta_of(prm, oi);
            const float tt = prm->tau / theta;
            Steps P{prm->sigma, prm->tau, prm->alpha1, prm->alpha2, tt, 1.0f / (1.0f + tt)};
            for (int it = 0; it < prm->inner; it++) {
                if (two_kernel && quads) {
                    k_dual4<<<nq, TPB, 0, s>>>(S, g, P);
                    k_primal4<<<nq, TPB, 0, s>>>(S, g, P);
                    launches += 2;
                } else if (two_kernel) {
                    k_dual<<<nb, TPB, 0, s>>>(S, g, P);
                    k_primal<<<nb, TPB, 0, s>>>(S, g, P);
                    launches += 2;
                } else {
                    float *const *in = set[cur], *const *out = set[cur ^ 1];
                    PP pp{in[0], in[1], in[2], in[3], in[4], in[5], in[6], in[7], in[8],
                          out[0], out[1], out[2], out[3], out[4], out[5], out[6], out[7], out[8],
                          S.d, S.w1, S.w2, S.a, S.T11, S.T12, S.T22};
                    k_tgv_iter<<<tgrid, TX * TY, 0, s>>>(pp, g, P);
                    cur ^= 1;
                    launches++;
                }
            }
            const float c = 1.0f / (2.0f * theta);
            k_data<<<nb, TPB, 0, s>>>(S, g, prm->n_disp, maxc, c, prm->lambda);
            launches++;
        }
    }
}

struct StereoGraphKey {
    void *ws;
    int32_t F;
    int chunk;
    int mode;
    int device;
    vol_stereo_params p;
};

// The executable graph is reference-counted: a call holds its own reference from lookup to launch, so
// evicting the entry (another thread inserting a 9th key) cannot destroy an exec about to be launched.
using ExecRef = std::shared_ptr<CUgraphExec_st>;
ExecRef exec_ref(cudaGraphExec_t e) {
    return ExecRef(e, [](cudaGraphExec_t x) {
        if (x) cudaGraphExecDestroy(x);
    });
}

struct StereoGraphEntry {
    StereoGraphKey key;
    ExecRef exec;
    long long launches;
};

std::mutex g_graph_mu;
// most recent last; at most 8 (heap-allocated and never destroyed: no graph destruction at process exit)
std::vector<StereoGraphEntry> &g_graphs = *new std::vector<StereoGraphEntry>();

bool same_key(const StereoGraphKey &a, const StereoGraphKey &b) {
    return a.ws == b.ws && a.F == b.F && a.chunk == b.chunk && a.mode == b.mode && a.device == b.device &&
           memcmp(&a.p, &b.p, sizeof a.p) == 0;
}

}  // namespace

// θ of outer round o is evaluated on the host (theta_of), so a captured graph holds the same values.
extern "C" vol_status vol_stereo(const float *left, const float *right, int32_t n_frames,
                                 const vol_stereo_params *prm, void *workspace, size_t workspace_bytes, void *stream,
                                 float *disparity, float *w_out, float *a_out) {
    NvtxRange nvtx_range_("vol_stereo");
    vol_status st = check_params(n_frames, prm);
    if (st != VOL_OK) return st;
    if (!left || !right || !disparity) return fail(VOL_EINVAL, "vol_stereo: NULL image or output pointer");
    const long long n = (long long)n_frames * prm->width * prm->height;
    const bool dev_out = is_device_ptr(disparity);
    if ((w_out && is_device_ptr(w_out) != dev_out) || (a_out && is_device_ptr(a_out) != dev_out))
        return fail(VOL_EINVAL, "vol_stereo: outputs must be all host or all device pointers");
    const size_t need = stereo_layout(nullptr, n, true).bytes;
    void *ws = workspace;
    bool owns = false;
    if (ws) {
        if (workspace_bytes < need)
            return fail(VOL_ENOMEM, "vol_stereo: workspace of %zu bytes < %zu needed", workspace_bytes, need);
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
    StereoLayout L = stereo_layout((char *)ws, n, true);
    cudaStream_t s = (cudaStream_t)stream;
    // inputs are always staged into the workspace, so a captured solve depends only on the workspace
    CK(cudaMemcpyAsync(L.IL, left, n * 4, cudaMemcpyDefault, s));
    CK(cudaMemcpyAsync(L.IR, right, n * 4, cudaMemcpyDefault, s));
    // Product path: the two per-pixel kernels (k_dual, k_primal) on chunks of frames whose iteration
    // working set (16 fp32 fields ≈ 64 B per pixel) stays in L2 — measured faster than the fused
    // halo-recompute kernel once the state is L2-resident.  The fused kernel stays
    // selectable (experiments only).
    // HVG_STEREO_FUSED / HVG_STEREO_SCALAR select the other kernel forms (bit-identical; tests, experiments)
    const int mode = getenv("HVG_STEREO_FUSED") ? 0 : (getenv("HVG_STEREO_SCALAR") ? 1 : 2);
    // Two chunks in flight on two streams (forked inside the graph), each half of the L2 budget: the
    // iteration kernels of one chunk are ~1 wave, so two independent chunks fill the GPU and hide each
    // other's launch gaps and tails (8 pairs 1240x376: 2 streams x 1 frame 11.1 ms, 1 stream x 2 frames
    // 13.5 ms, 3 x 1 12.4 ms, 2 x 2 15.5 ms — DESIGN.md §13)
    const long long per_frame = (long long)prm->width * prm->height * 64;
    const bool graph = !(owns || getenv("HVG_STEREO_NO_GRAPH"));   // the extra streams live inside the graph
    int n_streams = graph ? 2 : 1;
    if (const char *e = getenv("HVG_STEREO_STREAMS"); e && graph) n_streams = std::max(1, std::min(4, atoi(e)));
    int chunk = (int)((80ll << 20) / (per_frame > 0 ? per_frame : 1)) / n_streams;
    if (const char *e = getenv("HVG_STEREO_CHUNK")) chunk = atoi(e);      // experiments only
    if (chunk < 1) chunk = 1;
    if (chunk > n_frames) chunk = n_frames;
    if (n_streams > (n_frames + chunk - 1) / chunk) n_streams = (n_frames + chunk - 1) / chunk;
    long long launches = 0;
    if (!graph) {
        enqueue_solve(L, prm, n_frames, chunk, mode, &s, 1, launches);
        CK(cudaPeekAtLastError());
    } else {
        int dev = 0;
        cudaGetDevice(&dev);
        StereoGraphKey key{ws, n_frames, chunk, mode * 8 + n_streams, dev, *prm};
        ExecRef exec;
        {
            std::lock_guard<std::mutex> lk(g_graph_mu);
            for (auto &e : g_graphs)
                if (same_key(e.key, key)) {
                    exec = e.exec;
                    launches = e.launches;
                }
        }
        if (!exec) {
            cudaStream_t cs;
            CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            cudaGraph_t graph;
            cudaGraphExec_t ge = nullptr;
            cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
            if (e == cudaSuccess) {
                // extra streams fork from the capture stream and join back (graph edges)
                cudaStream_t ss[4] = {cs, nullptr, nullptr, nullptr};
                cudaEvent_t fork = nullptr, join[4] = {};
                cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
                cudaEventRecord(fork, cs);
                for (int k = 1; k < n_streams; k++) {
                    cudaStreamCreateWithFlags(&ss[k], cudaStreamNonBlocking);
                    cudaStreamWaitEvent(ss[k], fork, 0);
                }
                enqueue_solve(L, prm, n_frames, chunk, mode, ss, n_streams, launches);
                for (int k = 1; k < n_streams; k++) {
                    cudaEventCreateWithFlags(&join[k], cudaEventDisableTiming);
                    cudaEventRecord(join[k], ss[k]);
                    cudaStreamWaitEvent(cs, join[k], 0);
                }
                e = cudaStreamEndCapture(cs, &graph);
                for (int k = 1; k < n_streams; k++) {
                    cudaEventDestroy(join[k]);
                    cudaStreamDestroy(ss[k]);
                }
                cudaEventDestroy(fork);
            }
            if (e == cudaSuccess) {
                e = cudaGraphInstantiate(&ge, graph, 0);
                cudaGraphDestroy(graph);
            }
            cudaStreamDestroy(cs);
            if (e != cudaSuccess) return fail(VOL_ECUDA, "vol_stereo: graph capture failed: %s", cudaGetErrorString(e));
            exec = exec_ref(ge);
            std::lock_guard<std::mutex> lk(g_graph_mu);
            if (g_graphs.size() >= 8) g_graphs.erase(g_graphs.begin());   // freed once no call holds it
            g_graphs.push_back(StereoGraphEntry{key, exec, launches});
        }
        CK(cudaGraphLaunch(exec.get(), s));
    }
    counted((int)launches);
    const cudaMemcpyKind kind = dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(cudaMemcpyAsync(disparity, L.f[0], n * 4, kind, s));
    if (w_out) {
        CK(cudaMemcpyAsync(w_out, L.f[3], n * 4, kind, s));
        CK(cudaMemcpyAsync(w_out + n, L.f[4], n * 4, kind, s));
    }
    if (a_out) CK(cudaMemcpyAsync(a_out, L.f[2], n * 4, kind, s));
    if (owns || !dev_out) CK(cudaStreamSynchronize(s));
    return VOL_OK;
}

extern "C" vol_status vol_stereo_census(const float *img, int32_t n_frames, int32_t height, int32_t width,
                                        int32_t window, void *stream, uint32_t *sig) {
    if (!img || !sig || n_frames < 1 || height < 1 || width < 1 || (window != 3 && window != 5))
        return fail(VOL_EINVAL, "vol_stereo_census: bad arguments");
    if (!is_device_ptr(img) || !is_device_ptr(sig)) return fail(VOL_EINVAL, "vol_stereo_census: device pointers required");
    Img g{n_frames, height, width};
    const long long n = (long long)n_frames * height * width;
    k_census<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(img, g, window, sig);
    CK(cudaPeekAtLastError());
    counted(1);
    return VOL_OK;
}

extern "C" vol_status vol_stereo_tensor(const float *img, int32_t n_frames, int32_t height, int32_t width, float beta,
                                        float gamma, void *stream, float *T) {
    if (!img || !T || n_frames < 1 || height < 1 || width < 1 || !(beta > 0.0f) || !(gamma >= 0.0f))
        return fail(VOL_EINVAL, "vol_stereo_tensor: bad arguments");
    if (!is_device_ptr(img) || !is_device_ptr(T)) return fail(VOL_EINVAL, "vol_stereo_tensor: device pointers required");
    Img g{n_frames, height, width};
    const long long n = (long long)n_frames * height * width;
    k_tensor<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(img, g, beta, gamma, T, T + n, T + 2 * n);
    CK(cudaPeekAtLastError());
    counted(1);
    return VOL_OK;
}

extern "C" vol_status vol_disparity_to_depth(const float *disparity, int64_t n, float fx_baseline, float d_min,
                                             void *stream, float *depth) {
    if (!disparity || !depth || n < 0 || !(fx_baseline > 0.0f) || !(d_min >= 0.0f))
        return fail(VOL_EINVAL, "vol_disparity_to_depth: bad arguments");
    if (!is_device_ptr(disparity) || !is_device_ptr(depth))
        return fail(VOL_EINVAL, "vol_disparity_to_depth: device pointers required");
    if (n == 0) return VOL_OK;
    k_depth<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(disparity, n, fx_baseline, d_min, depth);
    CK(cudaPeekAtLastError());
    counted(1);
    return VOL_OK;
}
