// Probe: cycles per iteration of a (LDS -> mul -> STS -> barrier) loop, by thread count.
#include <cstdio>
#include <cstdint>
__global__ void k(int iters, int nbar, long long* out, uint32_t p) {
    __shared__ uint32_t buf[1024];
    buf[threadIdx.x] = threadIdx.x;
    __syncthreads();
    uint32_t x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t v = buf[(i + threadIdx.x) & 1023];
        x = (x * v + 7) % p;
        buf[(threadIdx.x * 7 + i) & 1023] = x;
        if (nbar == 0) __syncthreads();
        else asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = x; }
}
__global__ void k2(int iters, long long* out) {   // barrier only
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
}
int main() {
    long long* d; cudaMalloc(&d, 16); long long h[2];
    for (int nt : {32, 256, 1024}) {
        for (int nb = 0; nb < 2; ++nb) {
            k<<<1, nt>>>(1000, nb, d, 65521); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            printf("threads %4d %s: %.1f cyc/iter\n", nt, nb ? "named" : "sync ", h[0] / 1000.0);
        }
        k2<<<1, nt>>>(1000, d); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
        printf("threads %4d barrier only: %.1f cyc/iter\n", nt, h[0] / 1000.0);
    }
    return 0;
}
