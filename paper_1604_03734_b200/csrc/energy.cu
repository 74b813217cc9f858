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

__device__ __forceinline__ int face_idx(int a, int k, int c) {
    return a == 0 ? c + 8 * k : (a == 1 ? (k & 7) + 8 * c + 64 * (k >> 3) : k + 64 * c);
}

// One CTA per block; the block and its face halos are staged in shared memory (u, W of the +faces;
// p_a of the −faces, which is 0 on invalid edges by the iteration's invariant, see iterate.cu).
__global__ void __launch_bounds__(kThreads)
k_energy_blocks(View F, const int32_t *__restrict__ nbr, const int32_t *__restrict__ blocks, double lam, double eps,
                int data_term, double *__restrict__ partials) {
    __shared__ float su[kBlockVox + 192], sW[kBlockVox + 192];
    __shared__ float sp[3][64 + kBlockVox];
    __shared__ double red[kNPart][kThreads];
    const int tid = threadIdx.x;
    const int64_t b = blocks ? blocks[blockIdx.x] : blockIdx.x;
    const int64_t base = b * kBlockVox;
    for (int j = 0; j < 4; j++) {
        const int i = tid + kThreads * j;
        su[i] = F.u[base + i];
        sW[i] = F.W[base + i];
        sp[0][64 + i] = F.px_in[base + i];
        sp[1][64 + i] = F.py_in[base + i];
        sp[2][64 + i] = F.pz_in[base + i];
    }
    for (int it = tid; it < 384; it += kThreads) {
        const int a = (it >> 6) % 3, k = it & 63;
        if (it < 192) {                                   // + faces: u, W
            const int32_t nb = nbr[kNbr * b + 2 * a + 1];
            const int64_t idx = nb < 0 ? 0 : (int64_t)nb * kBlockVox + face_idx(a, k, 0);
            su[kBlockVox + it] = nb < 0 ? 0.0f : F.u[idx];
            sW[kBlockVox + it] = nb < 0 ? 0.0f : F.W[idx];
        } else {                                          // − faces: p_a
            const int32_t nb = nbr[kNbr * b + 2 * a];
            const float *pa = a == 0 ? F.px_in : (a == 1 ? F.py_in : F.pz_in);
            sp[a][k] = nb < 0 ? 0.0f : pa[(int64_t)nb * kBlockVox + face_idx(a, k, 7)];
        }
    }
    __syncthreads();
    double acc[kNPart] = {0.0, 0.0, 0.0, 0.0, 1.0};
    for (int j = 0; j < 4; j++) {
        const int i = tid + kThreads * j;
        const float Wv = sW[i];
        if (!(Wv > 0.0f)) continue;
        const int x = i & 7, y = (i >> 3) & 7, z = i >> 6;
        const int nx = x < 7 ? i + 1 : kBlockVox + (y + 8 * z);
        const int ny = y < 7 ? i + 8 : kBlockVox + 64 + (x + 8 * z);
        const int nz = z < 7 ? i + 64 : kBlockVox + 128 + (x + 8 * y);
        const double uv = su[i], fv = F.f[base + i], Wd = Wv;
        const double gx = sW[nx] > 0.0f ? (double)su[nx] - uv : 0.0;
        const double gy = sW[ny] > 0.0f ? (double)su[ny] - uv : 0.0;
        const double gz = sW[nz] > 0.0f ? (double)su[nz] - uv : 0.0;
        const double pxv = sp[0][64 + i], pyv = sp[1][64 + i], pzv = sp[2][64 + i];
        const double dv = (pxv - (double)sp[0][x > 0 ? 64 + i - 1 : y + 8 * z]) +
                          (pyv - (double)sp[1][y > 0 ? 64 + i - 8 : x + 8 * z]) +
                          (pzv - (double)sp[2][z > 0 ? i : x + 8 * y]);
        // H_ε(s), s = ‖∇u‖: the quadratic branch from s² directly (no square root; H is continuous at s = ε,
        // so deciding s ≤ ε on s² ≤ ε² moves the value by rounding only)
        const double s2 = gx * gx + gy * gy + gz * gz;
        const double h = (eps > 0.0 && s2 <= eps * eps) ? s2 / (2.0 * eps) : sqrt(s2) - eps / 2.0;
        const double r = uv - fv;
        const double dt = data_term == 0 ? lam * Wd * fabs(r) : 0.5 * lam * Wd * r * r;
        acc[0] += h + dt;
        acc[1] += pxv * pxv + pyv * pyv + pzv * pzv;
        acc[2] += fv * dv;
        if (data_term == 1) {   // Σ (div p)²/(2λW) enters only the L2 dual value
            acc[3] += dv * dv / (2.0 * lam * Wd);
        } else {                // the L1 dual's feasibility scale s = min λW/|div p| (1 for L2)
            const double lim = lam * Wd;
            if (fabs(dv) > lim) acc[4] = fmin(acc[4], lim / fabs(dv));
        }
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

int launch_energy(const View &F, const int32_t *nbr, const int32_t *blocks, int64_t n_blocks, float lam, float eps,
                  int data_term, double *partials, double *out, cudaStream_t s) {
    if (n_blocks > 0)
        k_energy_blocks<<<(unsigned)n_blocks, kThreads, 0, s>>>(F, nbr, blocks, (double)lam, (double)eps, data_term,
                                                                  partials);
    k_energy_final<<<1, 1024, 0, s>>>(partials, n_blocks, out);
    return cudaPeekAtLastError() == cudaSuccess ? counted(2) : -1;
}

}  // namespace hvg
