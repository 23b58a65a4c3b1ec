// Probe: dependent-chain latency (cycles per op, one warp) of the modular primitives used by the LQUP panel.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t shoup_m(uint32_t x, uint32_t w, uint32_t wsh, uint32_t p) {
    const uint32_t q = __umulhi(x, wsh);
    const uint32_t r = x * w - q * p;
    return r >= p ? r - p : r;
}
__device__ __forceinline__ uint32_t residue_u64(unsigned long long x, unsigned long long mu64, uint32_t p) {
    const unsigned long long q = __umul64hi(x, mu64);
    unsigned long long r = x - q * p;
    return static_cast<uint32_t>(r >= p ? r - p : r);
}
__device__ __forceinline__ uint32_t shoup_c(uint32_t w, uint32_t p, unsigned long long mu64) {
    const unsigned long long lo = static_cast<unsigned long long>(w) * static_cast<uint32_t>(mu64);
    const unsigned long long hi = static_cast<unsigned long long>(w) * static_cast<uint32_t>(mu64 >> 32);
    uint64_t c = (hi + (lo >> 32));
    if ((c + 1) * p <= (static_cast<uint64_t>(w) << 32)) ++c;
    return static_cast<uint32_t>(c);
}
__global__ void k(int iters, long long* out, uint32_t p, uint32_t w, uint32_t wsh, unsigned long long mu, uint32_t seed) {
    uint32_t x = seed + threadIdx.x;
    unsigned long long acc = x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) acc += static_cast<unsigned long long>(static_cast<uint32_t>(acc)) * w;
    long long t1 = clock64();
    for (int i = 0; i < iters; ++i) x = shoup_m(x, w, wsh, p);
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) x = residue_u64(static_cast<unsigned long long>(x) * w + acc, mu, p);
    long long t3 = clock64();
    __shared__ uint32_t s[64];
    s[threadIdx.x] = x;
    __syncwarp();
    for (int i = 0; i < iters; ++i) { x = s[x & 63]; }
    long long t4 = clock64();
    for (int i = 0; i < iters; ++i) { x = shoup_c(x % p, p, mu); }
    long long t5 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = x + acc; out[5] = t5 - t4; }
}
int main() {
    long long* d; cudaMalloc(&d, 64); long long h[6];
    uint32_t p = 65521, w = 12345; uint32_t wsh = (uint32_t)(((unsigned long long)w << 32) / p);
    unsigned long long mu = (unsigned long long)(((unsigned __int128)1 << 64) / p);
    k<<<1, 32>>>(1000, d, p, w, wsh, mu, 1); cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
    k<<<1, 32>>>(1000, d, p, w, wsh, mu, 1); cudaMemcpy(h, d, 48, cudaMemcpyDeviceToHost);
    printf("shoup_c(+mod) chain %.1f\n", h[5] / 1000.0);
    printf("IMAD.WIDE chain %.1f  shoup_m chain %.1f  residue_u64(mad) chain %.1f  LDS chain %.1f cyc/op\n",
           h[0] / 1000.0, h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0);
    return 0;
}
