// ceiling.cu -- the int8 tensor-core ceiling of this B200, measured (SURVEY §8(d):
// "an MMA-only microbenchmark ceiling measured on the box").  The same
// instruction the hot kernel issues -- tcgen05.mma.cta_group::2.kind::i8,
// M = 256, N = 256, K = 32, s32 accumulators in TMEM, operands K-major with
// the 128-byte swizzle -- issued back to back by one thread per CTA pair from
// SMEM-resident operands (no TMA traffic, no epilogue, two TMEM accumulators
// alternating as in the product kernel), one CTA per SM.  It is the analogue of
// the paper's fgemm / dgemm comparison: the numerical
// kernel's own speed on the same machine.
#include <cuda.h>
#include <cuda_runtime.h>

#include "internal.h"
#include "ptx.cuh"

namespace ff {
namespace {

constexpr int kStagesC = 4;                 // distinct SMEM operand tiles cycled through
constexpr int kStageBytes = 2 * 128 * kBK;  // A 128 rows + B 128 rows of 128 bytes (per CTA)
constexpr int kSmemC = kStagesC * kStageBytes + 1024 + 64;

__global__ void __launch_bounds__(128, 1) mma_ceiling_kernel(int iters, uint32_t idesc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* done = reinterpret_cast<uint64_t*>(smem + kStagesC * kStageBytes);
    uint32_t* holder = reinterpret_cast<uint32_t*>(done + 1);
    // random operand bytes: the tensor core's power (hence the clock it sustains
    // under the 1 kW cap) depends on how many operand bits toggle
    for (int i = threadIdx.x; i < kStagesC * kStageBytes / 4; i += blockDim.x) {
        uint32_t z = static_cast<uint32_t>(i) * 0x9E3779B9u + blockIdx.x * 0x85EBCA6Bu;
        z ^= z >> 16; z *= 0x7FEB352Du; z ^= z >> 15; z *= 0x846CA68Bu; z ^= z >> 16;
        reinterpret_cast<uint32_t*>(smem)[i] = z;
    }
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        ptx::mbar_init(done, 1);
        ptx::fence_barrier_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 1) ptx::tmem_alloc_pair(holder, 512);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = *holder;
    if (warp == 1 && ptx::lane_id() == 0 && ptx::cluster_ctarank() == 0) {
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = tmem + (it & 1) * 256;
            const uint32_t sa = ptx::smem_u32(smem + (it % kStagesC) * kStageBytes);
            const uint64_t da = ptx::smem_desc_sw128(sa);
            const uint64_t db = ptx::smem_desc_sw128(sa + 128 * kBK);
#pragma unroll
            for (int kk = 0; kk < kBK / kMmaK; ++kk) ptx::mma_i8_pair(d, da + 2 * kk, db + 2 * kk, idesc, it > 1 || kk);
        }
        ptx::tc_commit_pair(done);
    }
    if (threadIdx.x == 0) ptx::mbar_wait(done, 0);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair(tmem, 512);
    }
}

}  // namespace
}  // namespace ff

extern "C" int ff_mma_ceiling(int32_t iters, double* tops) {
    using namespace ff;
    if (iters <= 0 || !tops) return -1;
    int e = check_device();
    if (e) return e;
    if (set_smem_attr(reinterpret_cast<const void*>(mma_ceiling_kernel), kSmemC) != cudaSuccess) return FF_ERR_CUDA;
    // s8 x s8 -> s32, M = 256 (cta pair), N = 256, K-major operands (the hot kernel's descriptor)
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
    const int grid = (num_sms() / 2) * 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = kSmemC;
    cfg.stream = nullptr;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t e0, e1;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return FF_ERR_CUDA;
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {          // first launch warms up (clock ramp, TMEM)
        cudaEventRecord(e0, nullptr);
        if (cudaLaunchKernelEx(&cfg, mma_ceiling_kernel, static_cast<int>(iters), idesc) != cudaSuccess) {
            cudaGetLastError();
            return FF_ERR_CUDA;
        }
        cudaEventRecord(e1, nullptr);
        if (cudaEventSynchronize(e1) != cudaSuccess) return FF_ERR_CUDA;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // per iteration and CTA pair: 4 MMAs of 256 x 256 x 32 (2 ops per MAC)
    const double ops = static_cast<double>(iters) * (grid / 2) * 4.0 * 256.0 * 256.0 * 32.0 * 2.0;
    *tops = ops / (best * 1e-3) / 1e12;
    return 0;
}
