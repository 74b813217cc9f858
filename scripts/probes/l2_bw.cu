// L2 read-bandwidth probe (one-off, B200): every SM streams a buffer that fits in L2 (the 126 MB L2 holds
// it after the first pass) with 16-byte ld.global.cg loads (L1 bypassed), timed with CUDA events.  The
// number is the roofline denominator of the L2-resident stereo iteration (bench.py l2_peak).
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void rd(const float4 *__restrict__ a, size_t n4, int reps, float *sink) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int r = 0; r < reps; r++)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
            float4 v;
            asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a + i));
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    if (acc.x + acc.y + acc.z + acc.w == 1.2345f) *sink = acc.x;
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *sink;
    cudaMalloc(&sink, 4);
    for (size_t mb : {16, 32, 48, 64, 96, 512}) {
        const size_t bytes = mb << 20, n4 = bytes / 16;
        float4 *a;
        cudaMalloc(&a, bytes);
        cudaMemset(a, 0, bytes);
        const int reps = mb >= 512 ? 2 : 20;
        for (int blocks_per_sm : {4, 8}) {
            rd<<<sms * blocks_per_sm, 512>>>(a, n4, 1, sink);   // warm: bring into L2
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            float best = 1e30f;
            for (int t = 0; t < 5; t++) {
                cudaEventRecord(e0);
                rd<<<sms * blocks_per_sm, 512>>>(a, n4, reps, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("buffer %4zu MB, %d CTAs/SM x 512 threads: %.0f GB/s\n", mb, blocks_per_sm,
                   (double)bytes * reps / (best * 1e-3) / 1e9);
        }
        cudaFree(a);
    }
    return 0;
}
