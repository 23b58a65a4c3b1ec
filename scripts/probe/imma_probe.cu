// Probe: legacy warp-level int8 MMA (mma.sync m16n8k32 u8 -> s32) on sm_100a:
// fragment layout check against a host product, and throughput (one CTA).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ __forceinline__ void imma(int (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
// A: 16 x 32 row-major bytes, B: 8 columns x 32 k (k contiguous per column), D: 16 x 8 int
__global__ void layout(const uint8_t* A, const uint8_t* B, int* D) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    uint32_t a[4], b[2];
    a[0] = *reinterpret_cast<const uint32_t*>(A + g * 32 + t * 4);
    a[1] = *reinterpret_cast<const uint32_t*>(A + (g + 8) * 32 + t * 4);
    a[2] = *reinterpret_cast<const uint32_t*>(A + g * 32 + t * 4 + 16);
    a[3] = *reinterpret_cast<const uint32_t*>(A + (g + 8) * 32 + t * 4 + 16);
    b[0] = *reinterpret_cast<const uint32_t*>(B + g * 32 + t * 4);
    b[1] = *reinterpret_cast<const uint32_t*>(B + g * 32 + t * 4 + 16);
    int d[4] = {0, 0, 0, 0};
    imma(d, a, b);
    D[g * 8 + t * 2] = d[0];
    D[g * 8 + t * 2 + 1] = d[1];
    D[(g + 8) * 8 + t * 2] = d[2];
    D[(g + 8) * 8 + t * 2 + 1] = d[3];
}
__global__ void tput(int iters, int* out) {
    uint32_t a[4] = {threadIdx.x, 2u, 3u, 4u}, b[2] = {5u, threadIdx.x};
    int d0[4] = {0, 0, 0, 0}, d1[4] = {0, 0, 0, 0}, d2[4] = {0, 0, 0, 0}, d3[4] = {0, 0, 0, 0};
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { imma(d0, a, b); imma(d1, a, b); imma(d2, a, b); imma(d3, a, b); }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (int)(t1 - t0); }
    out[1 + threadIdx.x] = d0[0] + d1[1] + d2[2] + d3[3];
}
int main() {
    uint8_t hA[16 * 32], hB[8 * 32];
    for (int i = 0; i < 16 * 32; ++i) hA[i] = rand() & 255;
    for (int i = 0; i < 8 * 32; ++i) hB[i] = rand() & 255;
    uint8_t *dA, *dB; int* dD; int hD[128];
    cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, 4096 * 4);
    cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
    layout<<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 8; ++c) {
            int s = 0;
            for (int k = 0; k < 32; ++k) s += hA[r * 32 + k] * hB[c * 32 + k];
            if (s != hD[r * 8 + c]) ++bad;
        }
    printf("layout check: %d mismatches (%s)\n", bad, cudaGetErrorString(cudaGetLastError()));
    for (int warps : {1, 8, 32}) {
        tput<<<1, 32 * warps>>>(2000, dD);
        int h[1]; cudaMemcpy(h, dD, 4, cudaMemcpyDeviceToHost);
        const double macs = 2000.0 * 4 * 16 * 8 * 32 * warps;
        printf("warps %2d: %.0f cycles, %.0f MAC/clk/SM\n", warps, (double)h[0], macs / h[0]);
    }
    return 0;
}
