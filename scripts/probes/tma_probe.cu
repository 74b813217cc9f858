// TMA capability probe (one-off, B200): tensor-map boxes used by the skewed kernel's face loads.
//  (1) x-face with elementStrides {4,1,1,1}: does the encode accept it, and what lands in smem?
//  (2) a box entirely out of bounds (block coordinate -1): zero fill, and does complete_tx count
//      the full box?  (a hang here would mean it does not; the probe is run under `timeout`)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const CUtensorMap *mA, const CUtensorMap *mS, const __grid_constant__ CUtensorMap pA, float *out,
                  int blk, int use_s, int *ok) {
    __shared__ __align__(128) float buf[256];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = -7.0f;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t bytes = use_s == 1 ? 256u : 1024u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
        const CUtensorMap *m = use_s == 2 ? &pA : (use_s ? mS : mA);
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
                "r"(sa(buf)), "l"(m), "r"(0), "r"(0), "r"(0), "r"(blk), "r"(sa(&bar))
            : "memory");
    }
    uint32_t done = 0;
    for (int it = 0; it < 2000000 && !done; it++)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(sa(&bar)), "r"(0) : "memory");
    if (threadIdx.x == 0) *ok = done;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}

int main() {
    const int S = 4;
    float *d, *o;
    cudaMalloc(&d, S * 512 * 4);
    cudaMalloc(&o, 256 * 4);
    float h[S * 512];
    for (int i = 0; i < S * 512; i++) h[i] = (float)i;
    cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no entry point\n"); return 1; }
    cuuint64_t dim[4] = {8, 8, 8, (cuuint64_t)S};
    cuuint64_t str[3] = {32, 256, 2048};
    cuuint32_t boxA[4] = {4, 8, 8, 1}, es1[4] = {1, 1, 1, 1};
    cuuint32_t boxS[4] = {4, 8, 8, 1}, es4[4] = {4, 1, 1, 1};
    CUtensorMap hA, hS;
    CUresult rA = enc(&hA, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dim, str, boxA, es1, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUresult rS = enc(&hS, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, dim, str, boxS, es4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode A (box 4x8x8, stride 1): %d   encode S (box 4x8x8, elementStrides 4): %d\n", (int)rA, (int)rS);
    CUtensorMap *dm;
    cudaMalloc(&dm, 2 * sizeof(CUtensorMap));
    cudaMemcpy(dm, &hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dm + 1, &hS, sizeof hS, cudaMemcpyHostToDevice);
    float out[256];
    int *dok;
    cudaMalloc(&dok, 4);
    setvbuf(stdout, nullptr, _IONBF, 0);
    for (int use_s = 0; use_s < 3; use_s++) {
        if (use_s == 1 && rS != 0) continue;
        for (int blk : {1, -1, S}) {
            k<<<1, 128>>>(dm, dm + 1, hA, o, blk, use_s, dok);
            cudaError_t e = cudaDeviceSynchronize();
            int okh = -1;
            cudaMemcpy(out, o, sizeof out, cudaMemcpyDeviceToHost);
            cudaMemcpy(&okh, dok, 4, cudaMemcpyDeviceToHost);
            printf("map %s blk %2d: err=%s completed=%d out[0..8] = ", use_s == 1 ? "S" : (use_s == 2 ? "param-A" : "A"), blk,
                   cudaGetErrorString(e), okh);
            for (int i = 0; i < 9; i++) printf("%g ", out[i]);
            printf(" ... out[63]=%g out[64]=%g out[255]=%g\n", out[63], out[64], out[255]);
        }
    }
    return 0;
}
