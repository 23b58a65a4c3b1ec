// dies.cu -- SM -> die map of a B200 (two dies of 74 SMs, each with half of the
// L2), measured once per device from L2-hit latency.
//
// Why: a line touched by SMs of both dies ends up cached in both L2 halves,
// so the usable L2 for operands shared by the whole GPU is ~half of 126 MB
// (measured: DRAM traffic appears at a ~48-64 MiB shared working set;
// DESIGN.md §4.8).  The GEMM therefore gives each die its own contiguous part
// of the tile raster, so each die's L2 holds only its own operands.
//
// How: one CTA per SM (forced by a large SMEM request) times dependent L2 hits
// inside several 2 KB granules; a granule is homed on one die, and SMs of that
// die see ~266 cycles vs ~305 for the other die.  SMs are classified by the
// agreement of their near/far pattern with the first SM's.  Any doubt (an SM
// not seen, a pattern that is neither clearly equal nor clearly opposite, a
// lopsided split) disables the die-aware schedule; it never affects results.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.h"

namespace ff {

namespace {

constexpr int kGran = 12;
constexpr int kChain = 256;

__device__ __forceinline__ int ld_cg(const int* p) {
    int v;
    asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

__global__ void die_probe_kernel(const int* buf, unsigned* lat, int* smid_out) {
    extern __shared__ int pad[];
    if (threadIdx.x != 0) return;
    int smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    smid_out[blockIdx.x] = smid;
    for (int g = 0; g < kGran; ++g) {
        const int* base = buf + g * 512 * 64;     // granules 128 KB apart
        int idx = 0;
        for (int i = 0; i < 64; ++i) idx = ld_cg(base + idx);
        const long long t0 = clock64();
        for (int i = 0; i < kChain; ++i) idx = ld_cg(base + idx);
        const long long t1 = clock64();
        lat[blockIdx.x * kGran + g] = static_cast<unsigned>((t1 - t0) / kChain) + (idx < 0 ? 1u : 0u);
    }
    pad[0] = 0;
}

struct DieInfo {
    bool done = false;
    bool ok = false;
    uint8_t* d_map = nullptr;   // device: die of each %smid (0/1), 255 unknown
    int* d_sched = nullptr;     // device: per-launch counters (reset before every launch)
    int count[2] = {0, 0};
};
DieInfo g_die[64];

void calibrate(int dev, DieInfo& D) {
    D.done = true;
    // Off unless requested: measured 4-6% slower than the plain raster on c4/c5
    // (DESIGN.md §4.8), kept as an experiment.
    if (!knobs().die_aware) return;
    const int nsm = num_sms();
    std::vector<int> h(512 * 64 * kGran);
    for (int g = 0; g < kGran; ++g)
        for (int j = 0; j < 512; ++j) h[g * 512 * 64 + j] = (j + 32) % 512;  // 16-line chain in 2 KB
    int *d = nullptr, *ds = nullptr;
    unsigned* dl = nullptr;
    bool ok = cudaMalloc(&d, h.size() * 4) == cudaSuccess && cudaMalloc(&dl, nsm * kGran * 4) == cudaSuccess &&
              cudaMalloc(&ds, nsm * 4) == cudaSuccess &&
              cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess &&
              cudaFuncSetAttribute(die_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024) ==
                  cudaSuccess;
    std::vector<unsigned> lat(nsm * kGran);
    std::vector<int> sm(nsm, -1);
    if (ok) {
        for (int rep = 0; rep < 2 && ok; ++rep) {
            die_probe_kernel<<<nsm, 32, 160 * 1024>>>(d, dl, ds);
            ok = cudaDeviceSynchronize() == cudaSuccess;
        }
        ok = ok && cudaMemcpy(lat.data(), dl, lat.size() * 4, cudaMemcpyDeviceToHost) == cudaSuccess &&
             cudaMemcpy(sm.data(), ds, nsm * 4, cudaMemcpyDeviceToHost) == cudaSuccess;
    }
    cudaFree(d);
    cudaFree(dl);
    cudaFree(ds);
    cudaGetLastError();
    if (!ok) return;
    // Classify by the first principal component of the per-SM latency vectors
    // (centred): its sign separates the two dies; a per-granule threshold is
    // confused by the smaller latency differences inside a die.
    std::vector<double> mean(kGran, 0.0);
    for (int b = 0; b < nsm; ++b)
        for (int g = 0; g < kGran; ++g) mean[g] += lat[b * kGran + g] / double(nsm);
    std::vector<double> cov(kGran * kGran, 0.0);
    for (int b = 0; b < nsm; ++b)
        for (int i = 0; i < kGran; ++i)
            for (int j = 0; j < kGran; ++j)
                cov[i * kGran + j] += (lat[b * kGran + i] - mean[i]) * (lat[b * kGran + j] - mean[j]);
    std::vector<double> v(kGran, 1.0), w(kGran);
    for (int it = 0; it < 200; ++it) {                       // power iteration
        double nrm = 0;
        for (int i = 0; i < kGran; ++i) {
            w[i] = 0;
            for (int j = 0; j < kGran; ++j) w[i] += cov[i * kGran + j] * v[j];
            nrm += w[i] * w[i];
        }
        nrm = std::sqrt(nrm);
        if (nrm <= 0) return;
        for (int i = 0; i < kGran; ++i) v[i] = w[i] / nrm;
    }
    std::vector<double> proj(nsm);
    double lo = 1e30, hi = -1e30;
    for (int b = 0; b < nsm; ++b) {
        double s = 0;
        for (int g = 0; g < kGran; ++g) s += (lat[b * kGran + g] - mean[g]) * v[g];
        proj[b] = s;
        lo = std::min(lo, s);
        hi = std::max(hi, s);
    }
    std::vector<uint8_t> map(1024, 255);
    std::vector<char> seen(1024, 0);
    int cnt[2] = {0, 0};
    double gap_in = 1e30;                                    // smallest |projection|
    for (int b = 0; b < nsm; ++b) {
        if (sm[b] < 0 || sm[b] >= 1024 || seen[sm[b]]) return;   // each SM exactly once
        seen[sm[b]] = 1;
        map[sm[b]] = proj[b] < 0 ? 0 : 1;
        ++cnt[map[sm[b]]];
        gap_in = std::min(gap_in, std::fabs(proj[b]));
    }
    // require a clear separation: every SM at least 25% of the half-range from 0
    if (gap_in < 0.25 * std::min(-lo, hi)) return;
    if (cnt[0] * 4 < nsm || cnt[1] * 4 < nsm) return;            // implausible split
    if (cudaMalloc(&D.d_map, 1024) != cudaSuccess || cudaMalloc(&D.d_sched, 4096 * 4 * sizeof(int)) != cudaSuccess ||
        cudaMemcpy(D.d_map, map.data(), 1024, cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    D.count[0] = cnt[0];
    D.count[1] = cnt[1];
    D.ok = true;
    if (getenv("FF_DIE_VERBOSE")) fprintf(stderr, "[ff] device %d: die-aware schedule on, %d + %d SMs\n", dev, cnt[0], cnt[1]);
}

}  // namespace

// Device pointers for the die-aware schedule of the current device, or false.
bool die_schedule(const uint8_t** die_map, int** sched) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return false;
    DieInfo& D = g_die[dev];
    if (!D.done) calibrate(dev, D);
    if (!D.ok) return false;
    *die_map = D.d_map;
    *sched = D.d_sched;
    return true;
}

}  // namespace ff
