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
#include <cstring>
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
};

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
    const float s = __fdiv_rn(__fsqrt_rn(__fadd_rn(__fmul_rn(p1, p1), __fmul_rn(p2, p2))), P.alpha1);
    if (s > 1.0f) {
        p1 = __fdiv_rn(p1, s);
        p2 = __fdiv_rn(p2, s);
    }
    S.p1[i] = p1;
    S.p2[i] = p2;
    // v = ∇w̄
    float q1 = __fadd_rn(S.q1[i], __fmul_rn(P.sigma, fdx(S.wb1, i, x, g.W)));
    float q2 = __fadd_rn(S.q2[i], __fmul_rn(P.sigma, fdy(S.wb1, i, y, g.H, g.W)));
    float q3 = __fadd_rn(S.q3[i], __fmul_rn(P.sigma, fdx(S.wb2, i, x, g.W)));
    float q4 = __fadd_rn(S.q4[i], __fmul_rn(P.sigma, fdy(S.wb2, i, y, g.H, g.W)));
    const float n2 = __fadd_rn(__fadd_rn(__fadd_rn(__fmul_rn(q1, q1), __fmul_rn(q2, q2)), __fmul_rn(q3, q3)),
                               __fmul_rn(q4, q4));
    const float sq = __fdiv_rn(__fsqrt_rn(n2), P.alpha2);
    if (sq > 1.0f) {
        q1 = __fdiv_rn(q1, sq);
        q2 = __fdiv_rn(q2, sq);
        q3 = __fdiv_rn(q3, sq);
        q4 = __fdiv_rn(q4, sq);
    }
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
    const float dn = __fdiv_rn(__fadd_rn(__fsub_rn(d, __fmul_rn(P.tau, kd)), __fmul_rn(P.tt, S.a[i])),
                               __fadd_rn(1.0f, P.tt));
    const float wn1 = __fsub_rn(w1, __fmul_rn(P.tau, kw1));
    const float wn2 = __fsub_rn(w2, __fmul_rn(P.tau, kw2));
    S.db[i] = __fadd_rn(dn, __fsub_rn(dn, d));
    S.wb1[i] = __fadd_rn(wn1, __fsub_rn(wn1, w1));
    S.wb2[i] = __fadd_rn(wn2, __fsub_rn(wn2, w2));
    S.d[i] = dn;
    S.w1[i] = wn1;
    S.w2[i] = wn2;
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
    int best = 0;
    float eb = energy(0);
    for (int k = 1; k < D; k++) {
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

extern "C" vol_status vol_stereo(const float *left, const float *right, int32_t n_frames,
                                 const vol_stereo_params *prm, void *workspace, size_t workspace_bytes, void *stream,
                                 float *disparity, float *w_out, float *a_out) {
    vol_status st = check_params(n_frames, prm);
    if (st != VOL_OK) return st;
    if (!left || !right || !disparity) return fail(VOL_EINVAL, "vol_stereo: NULL image or output pointer");
    const long long n = (long long)n_frames * prm->width * prm->height;
    const bool dev_in = is_device_ptr(left) && is_device_ptr(right);
    if (!dev_in && (is_device_ptr(left) || is_device_ptr(right)))
        return fail(VOL_EINVAL, "vol_stereo: both images must be host or both device pointers");
    const bool dev_out = is_device_ptr(disparity);
    if ((w_out && is_device_ptr(w_out) != dev_out) || (a_out && is_device_ptr(a_out) != dev_out))
        return fail(VOL_EINVAL, "vol_stereo: outputs must be all host or all device pointers");
    const size_t need = stereo_layout(nullptr, n, !dev_in).bytes;
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
    StereoLayout L = stereo_layout((char *)ws, n, !dev_in);
    cudaStream_t s = (cudaStream_t)stream;
    const float *IL = left, *IR = right;
    if (!dev_in) {
        CK(cudaMemcpyAsync(L.IL, left, n * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(L.IR, right, n * 4, cudaMemcpyHostToDevice, s));
        IL = L.IL;
        IR = L.IR;
    }
    Img g{n_frames, prm->height, prm->width};
    const int TPB = 256;
    const unsigned nb = blocks_for(n, TPB);
    State S{L.f[0], L.f[1], L.f[2], L.f[3], L.f[4], L.f[5], L.f[6], L.f[7], L.f[8], L.f[9], L.f[10], L.f[11], L.f[12],
            L.T[0], L.T[1], L.T[2], L.sL, L.sR};
    const int maxc = prm->window * prm->window - 1;
    long long launches = 0;
    k_census<<<nb, TPB, 0, s>>>(IL, g, prm->window, L.sL);
    k_census<<<nb, TPB, 0, s>>>(IR, g, prm->window, L.sR);
    k_tensor<<<nb, TPB, 0, s>>>(IR, g, prm->beta, prm->gamma, L.T[0], L.T[1], L.T[2]);
    k_wta<<<nb, TPB, 0, s>>>(S, g, prm->n_disp, maxc);
    launches += 4;
    CK(cudaPeekAtLastError());
    for (int o = 0; o < prm->outer; o++) {
        const float theta = theta_of(prm, o);
        Steps P{prm->sigma, prm->tau, prm->alpha1, prm->alpha2, prm->tau / theta};
        for (int it = 0; it < prm->inner; it++) {
            k_dual<<<nb, TPB, 0, s>>>(S, g, P);
            k_primal<<<nb, TPB, 0, s>>>(S, g, P);
            launches += 2;
        }
        const float c = 1.0f / (2.0f * theta);
        k_data<<<nb, TPB, 0, s>>>(S, g, prm->n_disp, maxc, c, prm->lambda);
        launches++;
        CK(cudaPeekAtLastError());
    }
    counted((int)launches);
    const cudaMemcpyKind kind = dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    CK(cudaMemcpyAsync(disparity, S.d, n * 4, kind, s));
    if (w_out) {
        CK(cudaMemcpyAsync(w_out, S.w1, n * 4, kind, s));
        CK(cudaMemcpyAsync(w_out + n, S.w2, n * 4, kind, s));
    }
    if (a_out) CK(cudaMemcpyAsync(a_out, S.a, n * 4, kind, s));
    if (owns || !dev_out || !dev_in) CK(cudaStreamSynchronize(s));
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
