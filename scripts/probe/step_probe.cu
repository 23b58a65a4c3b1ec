// Probe: the speculative LQUP panel's fraction-free LDU step loop on one 16 x 16 block
// (256 threads, named barrier), cycles per pivot.  Variant bits: 1 = no shoup_c
// production (constants recomputed by the consumers), 2 = __syncthreads instead of the
// named barrier, 4 = skip E tracking.
#include <cstdio>
#include <cstdint>
constexpr int kB = 16, kH = 128;
__device__ __forceinline__ uint32_t shoup_c(uint32_t w, uint32_t p, unsigned long long mu64) {
    const unsigned long long lo = static_cast<unsigned long long>(w) * static_cast<uint32_t>(mu64);
    const unsigned long long hi = static_cast<unsigned long long>(w) * static_cast<uint32_t>(mu64 >> 32);
    uint64_t c = (hi + (lo >> 32));
    if ((c + 1) * p <= (static_cast<uint64_t>(w) << 32)) ++c;
    return static_cast<uint32_t>(c);
}
__device__ __forceinline__ uint32_t shoup_m(uint32_t x, uint32_t w, uint32_t wsh, uint32_t p) {
    const uint32_t q = __umulhi(x, wsh);
    const uint32_t r = x * w - q * p;
    return r >= p ? r - p : r;
}
__device__ __forceinline__ uint32_t subm_u(uint32_t a, uint32_t b, uint32_t p) { return a >= b ? a - b : a + p - b; }

__global__ void k(uint32_t p, unsigned long long mu, int variant, long long* out, uint32_t* res) {
    extern __shared__ uint32_t sm[];
    uint32_t* D = sm; uint32_t* El = D + kH * kH; uint32_t* Eu = El + kH * kH;
    __shared__ uint32_t ash[2][kB], bsh[2][kB];
    const int tid = threadIdx.x, er = tid / kB, ec = tid % kB;
    uint32_t x = (er * 2654435761u + ec * 40503u + 17u) % p;
    if (x == 0) x = 1;
    if (er == ec) x = (x | 1u) % p + 1;
    D[er * kH + ec] = x;
    uint32_t el = 0, eu = 0;
    if (ec == 0) ash[0][er] = shoup_c(x, p, mu);
    if (er == 0) bsh[0][ec] = shoup_c(x, p, mu);
    uint32_t S = 1;
    __syncthreads();
    long long t0 = clock64();
    for (int rep = 0; rep < 8; ++rep)
    for (int t = 0; t < kB; ++t) {
        const int par = t & 1;
        const uint32_t pk = D[t * kH + t];
        if (!(variant & 32) && pk == 0u) break;
        const uint32_t pk_sh = (variant & 1) ? shoup_c(pk, p, mu) : ash[par][t];
        if (variant & 8) {
        } else if (variant & 16) {
            if (er > t && ec > t) { x = subm_u(shoup_m(x, pk, pk_sh, p), shoup_m(D[t * kH + ec], 77, 3456789, p), p); D[er * kH + ec] = x; }
        } else if (er > t) {
            const uint32_t a = D[er * kH + t];
            const uint32_t a_sh = (variant & 1) ? shoup_c(a, p, mu) : ash[par][er];
            if (ec > t) {
                x = subm_u(shoup_m(x, pk, pk_sh, p), shoup_m(D[t * kH + ec], a, a_sh, p), p);
                D[er * kH + ec] = x;
                if (!(variant & 1)) {
                    if (ec == t + 1) ash[par ^ 1][er] = shoup_c(x, p, mu);
                    if (er == t + 1) bsh[par ^ 1][ec] = shoup_c(x, p, mu);
                }
            } else if (!(variant & 4)) {
                const uint32_t g = (ec == t) ? S : El[t * kH + ec];
                el = subm_u(shoup_m(el, pk, pk_sh, p), shoup_m(g, a, a_sh, p), p);
                El[er * kH + ec] = el;
            }
        } else if (ec > t && !(variant & 4)) {
            const uint32_t h = (er == t) ? S : Eu[er * kH + t];
            const uint32_t b = D[t * kH + ec];
            const uint32_t b_sh = (variant & 1) ? shoup_c(b, p, mu) : bsh[par][ec];
            eu = subm_u(shoup_m(eu, pk, pk_sh, p), shoup_m(h, b, b_sh, p), p);
            Eu[er * kH + ec] = eu;
        }
        S = shoup_m(S, pk, pk_sh, p);
        if (variant & 64) { }
        else if (variant & 2) __syncthreads();
        else asm volatile("bar.sync 1, 256;" ::: "memory");
    }
    long long t1 = clock64();
    if (tid == 0) out[0] = t1 - t0;
    res[tid] = x + el + eu;
}
int main() {
    long long* d; uint32_t* r; cudaMalloc(&d, 16); cudaMalloc(&r, 4096); long long h;
    const uint32_t p = 65521;
    const unsigned long long mu = (unsigned long long)(((unsigned __int128)1 << 64) / p);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * kH * kH * 4);
    for (int v : {0, 32, 64, 96, 4, 36}) {
        for (int nt : {256, 1024}) {
            if (nt == 1024 && !(v & 2)) continue;
            k<<<1, nt, 3 * kH * kH * 4>>>(p, mu, v, d, r);
            k<<<1, nt, 3 * kH * kH * 4>>>(p, mu, v, d, r);
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            printf("variant %d threads %d: %.1f cyc/step  (%s)\n", v, nt, h / 128.0, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
