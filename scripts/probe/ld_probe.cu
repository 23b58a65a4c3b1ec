// Probe: latency of the epilogue's C-row loads (each thread 8 x 16 B of its own row;
// a warp = 32 rows) with ~198 KB of dynamic shared memory, cold vs warm.
#include <cstdio>
#include <cstdint>
__global__ void k(const int32_t* C, int ldc, long long* out, int32_t* sink) {
    extern __shared__ uint8_t smem[];
    const int row = threadIdx.x & 127, col0 = (threadIdx.x >> 7) * 32;
    const int32_t* cr = C + row * ldc + col0;
    long long t0 = clock64();
    int4 x[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) x[t] = *reinterpret_cast<const int4*>(cr + 4 * t);
    int s = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) s += x[t].x + x[t].y + x[t].z + x[t].w;
    long long t1 = clock64();
    if (s == 999) smem[0] = 1;
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (s == 12345) sink[0] = s;
}
int main() {
    int32_t* C; long long* d; int32_t* sink;
    cudaMalloc(&C, 128 * 128 * 4); cudaMalloc(&d, 8); cudaMalloc(&sink, 4);
    cudaMemset(C, 1, 128 * 128 * 4);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 198 * 1024);
    long long h;
    for (int smem : {0, 198 * 1024}) {
        for (int i = 0; i < 3; ++i) {
            k<<<1, 512, smem>>>(C, 128, d, sink);
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("smem %d run %d: %lld cycles\n", smem, i, h);
        }
    }
    return 0;
}
