// fe_probe.cu -- throughput of the fused-encode chunk loop in isolation: 148 CTAs
// x 16 warps transposing + packing an int32 [k][n] source into int8 planes
// [n][k] in chunks of 128 rows x 512 k taken from an atomic counter, with a
// configurable dynamic-SMEM carve-out (the GEMM kernel leaves ~26 KB of L1),
// items in flight per warp D, and L1-allocating or streaming loads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fe_probe fe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kFeK = 512;

template <bool NA>
__device__ __forceinline__ int32_t ld1(const int32_t* p) {
    if (NA) {
        int32_t v;
        asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
        return v;
    }
    return __ldg(p);
}

template <int D, bool NA>
__global__ void __launch_bounds__(512, 1) probe(const int32_t* X, int64_t k, int rows, int8_t* P, int* ctr,
                                                  int total, int nkc, uint32_t p, uint32_t mu) {
    extern __shared__ uint8_t smem[];
    __shared__ int cmd;
    if (threadIdx.x == 0) smem[0] = 0;
    const int et = threadIdx.x, lane = et & 31, w = et >> 5;
    for (;;) {
        if (et == 0) cmd = atomicAdd(ctr, 1);
        __syncthreads();
        const int c = cmd;
        __syncthreads();
        if (c >= total) break;
        const int blk = c % (rows / 128), kc = c / (rows / 128);
        const int64_t kbase = (int64_t)kc * kFeK;
        int32_t v[D][16];
        auto load = [&](int i, int32_t (&vv)[16]) {
            const int r = blk * 128 + (w & 3) * 32 + lane;
            const int64_t kk0 = kbase + (int64_t)((w >> 2) + 4 * i) * 16;
            const int32_t* src = X + r + kk0 * rows;
#pragma unroll
            for (int j = 0; j < 16; ++j) { vv[j] = ld1<NA>(src); src += rows; }
        };
        auto store = [&](int i, const int32_t (&vv)[16]) {
            const int r = blk * 128 + (w & 3) * 32 + lane;
            const int64_t kk0 = kbase + (int64_t)((w >> 2) + 4 * i) * 16;
            uint32_t wd[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t x = static_cast<uint32_t>(vv[j]) ^ 0x80000000u;
                uint32_t rr = x - __umulhi(x, mu) * p;
                if (rr >= p) rr -= p;
                const int32_t cc = rr > p / 2 ? (int32_t)rr - (int32_t)p : (int32_t)rr;
                wd[j >> 2] |= (static_cast<uint32_t>(cc) & 0xFF) << (8 * (j & 3));
            }
            *reinterpret_cast<uint4*>(P + (int64_t)r * k + kk0) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
        };
#pragma unroll
        for (int d = 0; d < D; ++d) load(d, v[d]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            store(i, v[i % D]);
            if (i + D < 8) load(i + D, v[i % D]);
        }
    }
}

template <int D, bool NA>
void run(const int32_t* X, int64_t k, int rows, int8_t* P, int* ctr, int smem, const char* name) {
    const int nkc = (int)(k / kFeK), total = nkc * (rows / 128);
    cudaFuncSetAttribute(probe<D, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(ctr, 0, 4);
        cudaEventRecord(e0);
        probe<D, NA><<<148, 512, smem>>>(X, k, rows, P, ctr, total, nkc, 251u, (uint32_t)((1ull << 32) / 251));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double bytes = (double)k * rows * 5;
    printf("%-28s smem %6d KB: %.3f ms  %.2f TB/s  (%.0f us per chunk per CTA)  %s\n", name, smem / 1024, best,
           bytes / best / 1e9, best * 1e3 / ((double)total / 148), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int64_t k = 16384;
    const int rows = 8192;
    int32_t* X;
    int8_t* P;
    int* ctr;
    cudaMalloc(&X, k * rows * 4);
    cudaMalloc(&P, k * rows);
    cudaMalloc(&ctr, 4);
    cudaMemset(X, 1, k * rows * 4);
    for (int smem : {0, 200 * 1024}) {
        run<2, false>(X, k, rows, P, ctr, smem, "D=2 ldg");
        run<2, true>(X, k, rows, P, ctr, smem, "D=2 no_allocate");
        run<4, false>(X, k, rows, P, ctr, smem, "D=4 ldg");
        run<4, true>(X, k, rows, P, ctr, smem, "D=4 no_allocate");
    }
    return 0;
}
