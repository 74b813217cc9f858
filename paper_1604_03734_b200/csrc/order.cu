// order.cu — the single-GPU store order on the device (vol_create): blocks sorted along a Morton (Z-order)
// curve of their coordinates relative to the bounding box, ties in caller order — the same order as the
// host planner's morton_sort_rows (shard.cu), computed without a host round trip of the coordinates:
//   k_coord_min      bounding-box minimum (atomicMin per axis) and the first block whose coordinate
//                    leaves (−2^30, 2^30) (the neighbour offsets need that room in int32 arithmetic);
//   k_morton_keys    key = spread3(x − lo_x) | spread3(y − lo_y) << 1 | spread3(z − lo_z) << 2 (21 bits
//                    per axis), value = caller index;
//   CUB radix sort   stable, so equal keys keep the caller order;
//   k_row_maps       store_of_global[perm[r]] = r and rows[r] = perm[r] for the neighbour-table build.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <mutex>

#include "internal.h"

namespace hvg {

namespace {

__device__ __forceinline__ unsigned long long spread3_dev(uint32_t v) {   // 21 bits → every third bit
    unsigned long long x = v & 0x1FFFFFu;
    x = (x | (x << 32)) & 0x1F00000000FFFFull;
    x = (x | (x << 16)) & 0x1F0000FF0000FFull;
    x = (x | (x << 8)) & 0x100F00F00F00F00Full;
    x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
    x = (x | (x << 2)) & 0x1249249249249249ull;
    return x;
}

__global__ void k_coord_min(const int32_t *__restrict__ xyz, int64_t n, int32_t *lo, unsigned long long *bad) {
    __shared__ int32_t s_lo[3];
    if (threadIdx.x < 3) s_lo[threadIdx.x] = INT32_MAX;
    __syncthreads();
    int32_t m[3] = {INT32_MAX, INT32_MAX, INT32_MAX};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        bool out = false;
#pragma unroll
        for (int a = 0; a < 3; a++) {
            const int32_t c = xyz[3 * i + a];
            m[a] = min(m[a], c);
            out = out || c <= -(1 << 30) || c >= (1 << 30);
        }
        if (out) atomicMin(bad, (unsigned long long)i);
    }
#pragma unroll
    for (int a = 0; a < 3; a++) atomicMin(&s_lo[a], m[a]);
    __syncthreads();
    if (threadIdx.x < 3) atomicMin(&lo[threadIdx.x], s_lo[threadIdx.x]);
}

__global__ void k_morton_keys(const int32_t *__restrict__ xyz, int64_t n, const int32_t *__restrict__ lo,
                              unsigned long long *__restrict__ key, int32_t *__restrict__ val) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t *c = xyz + 3 * i;
    key[i] = spread3_dev((uint32_t)(c[0] - lo[0])) | (spread3_dev((uint32_t)(c[1] - lo[1])) << 1) |
             (spread3_dev((uint32_t)(c[2] - lo[2])) << 2);
    val[i] = (int32_t)i;
}

__global__ void k_row_maps(const int32_t *__restrict__ perm, int64_t n, int32_t *__restrict__ sog,
                           int64_t *__restrict__ rows) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int32_t g = perm[r];
    sog[g] = (int32_t)r;
    rows[r] = g;
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

size_t cub_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                    (const int32_t *)nullptr, (int32_t *)nullptr, (int)n, 0, 63);
    return bytes;
}

}  // namespace

size_t morton_order_scratch_bytes(int64_t n) {
    return 256 + 2 * align256((size_t)n * 8) + align256((size_t)n * 4) + align256(cub_bytes(n));
}

int launch_morton_order(const int32_t *xyz, int64_t n, void *scratch, int32_t *perm, unsigned long long *bad,
                        cudaStream_t s) {
    if (n == 0) return 0;
    char *p = static_cast<char *>(scratch);
    int32_t *lo = reinterpret_cast<int32_t *>(p);
    p += 256;
    unsigned long long *k0 = reinterpret_cast<unsigned long long *>(p);
    p += align256((size_t)n * 8);
    unsigned long long *k1 = reinterpret_cast<unsigned long long *>(p);
    p += align256((size_t)n * 8);
    int32_t *v0 = reinterpret_cast<int32_t *>(p);
    p += align256((size_t)n * 4);
    size_t tb = cub_bytes(n);
    if (cudaMemsetAsync(lo, 0x7F, 12, s) != cudaSuccess) return -1;   // 0x7F7F7F7F > any valid coordinate
    const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 4);
    k_coord_min<<<g, 256, 0, s>>>(xyz, n, lo, bad);
    k_morton_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(xyz, n, lo, k0, v0);
    if (cudaPeekAtLastError() != cudaSuccess) return -1;
    if (cub::DeviceRadixSort::SortPairs(p, tb, k0, k1, v0, perm, (int)n, 0, 63, s) != cudaSuccess) return -1;
    return counted(2);   // our two kernels (the CUB sort is library code)
}

int launch_row_maps(const int32_t *perm, int64_t n, int32_t *sog, int64_t *rows, cudaStream_t s) {
    if (n == 0) return 0;
    k_row_maps<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(perm, n, sog, rows);
    return cudaPeekAtLastError() == cudaSuccess ? counted(1) : -1;
}

// Order-independent 64-bit digest of block coordinates: Σ_i mix(i, x_i, y_i, z_i) mod 2^64 (splitmix64 rounds),
// the same function on the host (coord_digest_host) and the device (one reduction, no host copy of the
// coordinates).
__host__ __device__ inline unsigned long long dig_mix(unsigned long long z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ inline unsigned long long dig_term(int64_t i, int32_t x, int32_t y, int32_t z) {
    const unsigned long long a = dig_mix((unsigned long long)i);
    const unsigned long long b = dig_mix(a ^ (unsigned long long)(uint32_t)x);
    return dig_mix(b ^ (((unsigned long long)(uint32_t)y << 32) | (uint32_t)z));
}

namespace {
__global__ void k_coord_digest(const int32_t *__restrict__ xyz, int64_t n, unsigned long long *out) {
    unsigned long long acc = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += dig_term(i, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}
}  // namespace

unsigned long long coord_digest_host(const int32_t *xyz, int64_t n) {
    unsigned long long acc = 0;
    for (int64_t i = 0; i < n; i++) acc += dig_term(i, xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    return acc ^ dig_mix((unsigned long long)n);
}

bool coord_digest_device(const int32_t *xyz, int64_t n, unsigned long long *out, cudaStream_t s) {
    // one scratch word per device, kept for the process; runs on `s` — the caller's stream in vol_create, so
    // coordinates still being written there are read after they are complete — and returns synchronously
    // (it gates the shard plan); serialised by a mutex
    static std::mutex mu;
    static unsigned long long *words[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
    std::lock_guard<std::mutex> lk(mu);
    if (!words[dev] && cudaMalloc(&words[dev], 8) != cudaSuccess) return false;
    unsigned long long *d = words[dev], h = 0;
    bool ok = cudaMemsetAsync(d, 0, 8, s) == cudaSuccess;
    if (ok && n > 0) {
        const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 8);
        k_coord_digest<<<g, 256, 0, s>>>(xyz, n, d);
        ok = cudaPeekAtLastError() == cudaSuccess;
        if (ok) counted(1);
    }
    ok = ok && cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, s) == cudaSuccess && cudaStreamSynchronize(s) == cudaSuccess;
    *out = h ^ dig_mix((unsigned long long)n);
    return ok;
}

}  // namespace hvg
