// energy.cu — primal energy and dual value of the current state (off the
// iteration loop).  Eq. 2 with Huber TV and the W-weighted data term (reading c-1):
//   P(u) = Σ_Ω H_ε(‖∇_Ω u‖₂) + λ Σ_Ω W|u − f|   (L1)   or   + (λ/2) Σ_Ω W (u − f)²   (L2),
//   H_ε(s) = s²/(2ε) if s ≤ ε else s − ε/2.
// Dual value: D = −(ε/2)Σ_Ω‖p̂‖² − Σ_Ω f·div p̂ − [L2] Σ_Ω (div p̂)²/(2λW), with
// p̂ = s·p, s = min(1, min_v λW_v/|div p(v)|) for L1 and s = 1 for L2.
// Per-voxel terms are evaluated in fp64 from the fp32 state; sums use a fixed per-thread order, a
// fixed shared-memory tree per block and a fixed tree over blocks, so the result is deterministic.
#include "internal.h"

namespace hvg {

constexpr int kNPart = 5;  // [0] primal, [1] Σ‖p‖², [2] Σ f·div p, [3] Σ (div p)²/(2λW), [4] min λW/|div p|

__device__ __forceinline__ int64_t step_voxel(const int32_t *nbr, int64_t b, int i, int axis, int dir) {
    int c[3] = {i & 7, (i >> 3) & 7, i >> 6};
    c[axis] += dir;
    if (c[axis] < 0 || c[axis] > 7) {
        int32_t nb = nbr[6 * b + 2 * axis + (dir > 0 ? 1 : 0)];
        if (nb < 0) return -1;
        c[axis] &= 7;
        b = nb;
    }
    return b * kBlockVox + c[0] + 8 * c[1] + 64 * c[2];
}

__global__ void __launch_bounds__(kThreads)
k_energy_blocks(Fields F, const int32_t *__restrict__ nbr, const int32_t *__restrict__ blocks, double lam, double eps,
                int data_term, double *__restrict__ partials) {
    __shared__ double red[kNPart][kThreads];
    const int tid = threadIdx.x;
    const int64_t b = blocks ? blocks[blockIdx.x] : blockIdx.x;
    double acc[kNPart] = {0.0, 0.0, 0.0, 0.0, 1.0};
    for (int j = 0; j < 4; j++) {
        const int i = tid + kThreads * j;
        const int64_t v = b * kBlockVox + i;
        const float Wv = F.W[v];
        if (!(Wv > 0.0f)) continue;
        const double uv = F.u[v], fv = F.f[v], Wd = Wv;
        double g2 = 0.0, dv = 0.0, p2 = 0.0;
        const float *pc[3] = {F.px, F.py, F.pz};
        for (int a = 0; a < 3; a++) {
            const int64_t w = step_voxel(nbr, b, i, a, +1);
            const bool fwd = w >= 0 && F.W[w] > 0.0f;
            const double ga = fwd ? (double)F.u[w] - uv : 0.0;
            g2 += ga * ga;
            const int64_t m = step_voxel(nbr, b, i, a, -1);
            const bool bwd = m >= 0 && F.W[m] > 0.0f;
            const double own = fwd ? (double)pc[a][v] : 0.0;
            const double prv = bwd ? (double)pc[a][m] : 0.0;
            dv += own - prv;
            const double pa = pc[a][v];
            p2 += pa * pa;
        }
        const double s = sqrt(g2);
        const double h = (eps > 0.0 && s <= eps) ? s * s / (2.0 * eps) : s - eps / 2.0;
        const double r = uv - fv;
        const double dt = data_term == 0 ? lam * Wd * fabs(r) : 0.5 * lam * Wd * r * r;
        acc[0] += h + dt;
        acc[1] += p2;
        acc[2] += fv * dv;
        acc[3] += dv * dv / (2.0 * lam * Wd);
        const double lim = lam * Wd;
        if (fabs(dv) > lim) acc[4] = fmin(acc[4], lim / fabs(dv));
    }
    for (int k = 0; k < kNPart; k++) red[k][tid] = acc[k];
    __syncthreads();
    for (int o = kThreads / 2; o > 0; o >>= 1) {
        if (tid < o) {
            for (int k = 0; k < 4; k++) red[k][tid] += red[k][tid + o];
            red[4][tid] = fmin(red[4][tid], red[4][tid + o]);
        }
        __syncthreads();
    }
    if (tid == 0)
        for (int k = 0; k < kNPart; k++) partials[(int64_t)blockIdx.x * kNPart + k] = red[k][0];
}

__global__ void __launch_bounds__(1024) k_energy_final(const double *__restrict__ partials, int64_t n, double *out) {
    __shared__ double red[kNPart][1024];
    const int tid = threadIdx.x;
    double acc[kNPart] = {0.0, 0.0, 0.0, 0.0, 1.0};
    for (int64_t k = tid; k < n; k += 1024) {
        for (int q = 0; q < 4; q++) acc[q] += partials[k * kNPart + q];
        acc[4] = fmin(acc[4], partials[k * kNPart + 4]);
    }
    for (int q = 0; q < kNPart; q++) red[q][tid] = acc[q];
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if (tid < o) {
            for (int q = 0; q < 4; q++) red[q][tid] += red[q][tid + o];
            red[4][tid] = fmin(red[4][tid], red[4][tid + o]);
        }
        __syncthreads();
    }
    if (tid == 0)
        for (int q = 0; q < kNPart; q++) out[q] = red[q][0];
}

int launch_energy(const Fields &F, const int32_t *nbr, const int32_t *blocks, int64_t n_blocks, float lam, float eps,
                  int data_term, double *partials, double *out, cudaStream_t s) {
    if (n_blocks > 0)
        k_energy_blocks<<<(unsigned)n_blocks, kThreads, 0, s>>>(F, nbr, blocks, (double)lam, (double)eps, data_term,
                                                                  partials);
    k_energy_final<<<1, 1024, 0, s>>>(partials, n_blocks, out);
    return cudaPeekAtLastError() == cudaSuccess ? counted(2) : -1;
}

}  // namespace hvg
