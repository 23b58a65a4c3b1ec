// Experiment: can the SM -> die map be recovered from L2 hit latency?
// One CTA per SM (forced by a large dynamic SMEM request); thread 0 of each CTA
// times a dependent chain of L2 hits inside one 2 KB granule, for several granules.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ int ld_cg(const int* p) {
    int v;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__global__ void probe(const int* buf, int ngran, unsigned* lat, int* smid_out) {
    extern __shared__ int dummy[];
    if (threadIdx.x != 0) return;
    int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    smid_out[blockIdx.x] = smid;
    for (int g = 0; g < ngran; ++g) {
        const int* base = buf + g * 512 * 64;   // granules 128 KB apart
        int idx = 0;
        for (int i = 0; i < 64; ++i) idx = ld_cg(base + idx);   // warm
        long long t0 = clock64();
        for (int i = 0; i < 256; ++i) idx = ld_cg(base + idx);
        long long t1 = clock64();
        lat[blockIdx.x * ngran + g] = (unsigned)((t1 - t0) / 256) + (idx == -1 ? 1 : 0);
    }
    dummy[0] = 0;
}

int main() {
    const int ngran = 16, nsm = 148;
    std::vector<int> h(512 * 64 * ngran);
    for (int g = 0; g < ngran; ++g)
        for (int j = 0; j < 512; ++j) h[g * 512 * 64 + j] = (j + 32) % 512;   // 16-line chain in 2 KB
    int* d; unsigned* dl; int* ds;
    cudaMalloc(&d, h.size() * 4); cudaMalloc(&dl, nsm * ngran * 4); cudaMalloc(&ds, nsm * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int rep = 0; rep < 2; ++rep) {
        probe<<<nsm, 32, 200 * 1024>>>(d, ngran, dl, ds);
        cudaDeviceSynchronize();
    }
    std::vector<unsigned> lat(nsm * ngran); std::vector<int> sm(nsm);
    cudaMemcpy(lat.data(), dl, lat.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(sm.data(), ds, nsm * 4, cudaMemcpyDeviceToHost);
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    std::vector<std::pair<int,int>> order;
    for (int b = 0; b < nsm; ++b) order.push_back({sm[b], b});
    std::sort(order.begin(), order.end());
    for (auto& o : order) {
        printf("sm %3d:", o.first);
        for (int g = 0; g < ngran; ++g) printf(" %4u", lat[o.second * ngran + g]);
        printf("\n");
    }
    return 0;
}
