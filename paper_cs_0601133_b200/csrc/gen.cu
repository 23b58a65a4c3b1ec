// gen.cu -- device twin of ffgen/__init__.py (seeded synthetic inputs).
// Holds none of the method's arithmetic; the tests compare it bit-for-bit
// with the numpy generator.
#include <cuda_runtime.h>

#include "internal.h"

namespace ff {

namespace {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void fill_uniform_kernel(int32_t* __restrict__ X, int64_t rows, int64_t cols, int64_t ld, uint32_t p,
                                    uint64_t key, int64_t index0) {
    const int64_t total = rows * cols;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / cols, c = idx - r * cols;
        const uint64_t i = static_cast<uint64_t>(index0 + idx);
        const uint64_t v = (mix64(key + (i + 1) * kGamma) >> 11) % p;
        X[r * ld + c] = static_cast<int32_t>(v);
    }
}

}  // namespace

cudaError_t launch_fill_uniform(int32_t* X, int64_t rows, int64_t cols, int64_t ld, uint32_t p, uint64_t seed,
                                uint32_t stream_id, int64_t index0, cudaStream_t st) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    const uint64_t key = mix64(seed * 16 + stream_id);
    int64_t g = (rows * cols + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 32;
    if (g > cap) g = cap;
    fill_uniform_kernel<<<static_cast<int>(g), 256, 0, st>>>(X, rows, cols, ld, p, key, index0);
    return cudaGetLastError();
}

}  // namespace ff
