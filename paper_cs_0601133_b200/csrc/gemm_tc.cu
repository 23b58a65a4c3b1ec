// gemm_tc.cu -- the hot kernel: exact limb-product accumulation on the sm_100a
// tensor cores (tcgen05.mma.kind::i8 -> s32 in TMEM) with the delayed modular
// reduction, limb recombination and alpha/beta epilogue fused in.
//
// What it computes, per 128x256 output tile:
//   op(A) = sum_i 256^i Ad_i,  op(B) = sum_j 256^j Bd_j   (int8 limb planes)
//   A B   = sum_w 256^w S_w,   S_w = sum_{i+j=w} Ad_i Bd_j^T   (weight groups)
//   Horner over w from 2L-2 down to 0, one TMEM accumulator per tile:
//     R <- S_{2L-2};  R <- 256 (R mod p) + S_w  ...;  out = alpha (R mod p) + beta C
// The accumulator is reduced mod p and re-centred ("delayed reduction",
// PAPER.md l.145-159) only (a) between weight groups, where it is also scaled
// by 256 mod p, and (b) every kb elements of k (the Eq. (2) analogue computed
// by the planner).  Nothing is ever rounded: the result is exact.
//
// Structure (one CTA per SM, persistent, warp-specialised, 320 threads):
//   warp 0      TMA producer: limb tiles A_i[128 x 128B], B_j[256 x 128B] -> 4-stage SMEM ring
//   warp 1      TMEM owner + single-thread MMA issuer (4 x K=32 MMAs per stage)
//   warps 2..9  epilogue: tcgen05.ld -> mod p / Horner / alpha,beta -> tcgen05.st or global
// Two tiles are in flight per CTA, one per 256-column TMEM accumulator ("slot"):
// while the epilogue reduces slot s between two steps, the MMA runs the other
// slot, so the tensor pipe never waits for the modular reduction.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "internal.h"
#include "modp.cuh"
#include "ptx.cuh"

namespace ff {

namespace {

constexpr int kStages = 4;
constexpr int kABytes = kTileM * kBK;          // 16 KB
constexpr int kBBytes = kTileN * kBK;          // 32 KB
constexpr int kStageBytes = kABytes + kBBytes; // 48 KB
constexpr int kNumEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kNumEpiWarps);
constexpr int kTmemCols = 512;                 // two 256-column s32 accumulators
constexpr int kSmemBytes = kStages * kStageBytes + 256 + 1024;
constexpr int kRasterGroup = 16;               // m-tiles per raster band (L2 reuse)

struct GemmArgs {
    ModP mp;
    int32_t* C;
    int64_t ldc;
    int32_t m, n;
    int32_t tiles_m, tiles_n, num_tiles;
    int32_t k_iters;   // ceil(k / 128)
    int32_t kb_iters;  // k-block length / 128
    int32_t nkb;       // number of k-blocks
    int32_t G;         // weight groups
    int8_t pair_i[16], pair_j[16];
    int8_t group_first[8], group_len[8];
    uint32_t idesc[16];
    int32_t vec_store;  // 1 if C rows are 16-byte aligned
};

struct Smem {
    uint64_t full[kStages];
    uint64_t empty[kStages];
    uint64_t accfull[2];
    uint64_t accempty[2];
    uint32_t tmem_base;
};

__device__ __forceinline__ void tile_coords(const GemmArgs& a, int t, int& tm, int& tn) {
    const int band_size = kRasterGroup * a.tiles_n;
    const int band = t / band_size;
    const int idx = t - band * band_size;
    const int rows_in_band = min(kRasterGroup, a.tiles_m - band * kRasterGroup);
    tm = band * kRasterGroup + idx % rows_in_band;
    tn = idx / rows_in_band;
}

// The common schedule every role walks: tiles in pairs (one per TMEM slot),
// groups from the highest weight down, k-blocks in order, then the slots.
template <class F>
__device__ __forceinline__ void for_each_step(const GemmArgs& a, F&& f) {
    for (int t0 = blockIdx.x; t0 < a.num_tiles; t0 += 2 * gridDim.x) {
        const int t1 = t0 + gridDim.x;
        const int nslots = t1 < a.num_tiles ? 2 : 1;
        for (int g = a.G - 1; g >= 0; --g)
            for (int kb = 0; kb < a.nkb; ++kb)
                for (int s = 0; s < nslots; ++s) f(s == 0 ? t0 : t1, s, g, kb);
    }
}

__global__ void __launch_bounds__(kThreads, 1)
    ffgemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ GemmArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Smem* sh = reinterpret_cast<Smem*>(smem + kStages * kStageBytes);
    const int warp = threadIdx.x / 32;
    const uint32_t lane = ptx::lane_id();

    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&sh->full[s], 1);
            ptx::mbar_init(&sh->empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&sh->accfull[s], 1);
            ptx::mbar_init(&sh->accempty[s], kNumEpiWarps);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc(&sh->tmem_base, kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = sh->tmem_base;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            for_each_step(a, [&](int tile, int, int g, int kb) {
                int tm, tn;
                tile_coords(a, tile, tm, tn);
                const int ks0 = kb * a.kb_iters;
                const int ks1 = min(ks0 + a.kb_iters, a.k_iters);
                for (int pi = a.group_first[g]; pi < a.group_first[g] + a.group_len[g]; ++pi) {
                    const int li = a.pair_i[pi], lj = a.pair_j[pi];
                    for (int ks = ks0; ks < ks1; ++ks) {
                        ptx::mbar_wait(&sh->empty[stage], phase ^ 1);
                        uint8_t* sa = smem + stage * kStageBytes;
                        ptx::mbar_arrive_expect_tx(&sh->full[stage], kStageBytes);
                        ptx::tma_load_3d(sa, &tmA, &sh->full[stage], ks * kBK, tm * kTileM, li);
                        ptx::tma_load_3d(sa + kABytes, &tmB, &sh->full[stage], ks * kBK, tn * kTileN, lj);
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                }
            });
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (one thread)
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            uint32_t acc_par[2] = {0, 0};
            for_each_step(a, [&](int, int slot, int g, int kb) {
                ptx::mbar_wait(&sh->accempty[slot], acc_par[slot] ^ 1);
                acc_par[slot] ^= 1;
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + slot * kTileN;
                uint32_t acc = (g == a.G - 1 && kb == 0) ? 0u : 1u;  // first MMA of a tile overwrites
                const int ks0 = kb * a.kb_iters;
                const int ks1 = min(ks0 + a.kb_iters, a.k_iters);
                for (int pi = a.group_first[g]; pi < a.group_first[g] + a.group_len[g]; ++pi) {
                    const uint32_t idesc = a.idesc[pi];
                    for (int ks = ks0; ks < ks1; ++ks) {
                        ptx::mbar_wait(&sh->full[stage], phase);
                        ptx::tc_fence_after();
                        const uint32_t sa = ptx::smem_u32(smem + stage * kStageBytes);
                        const uint64_t da = ptx::smem_desc_sw128(sa);
                        const uint64_t db = ptx::smem_desc_sw128(sa + kABytes);
#pragma unroll
                        for (int kk = 0; kk < kBK / kMmaK; ++kk) {
                            ptx::mma_i8(d, da + 2 * kk, db + 2 * kk, idesc, acc);
                            acc = 1u;
                        }
                        ptx::tc_commit(&sh->empty[stage]);  // frees the SMEM stage when these MMAs finish
                        if (++stage == kStages) { stage = 0; phase ^= 1; }
                    }
                }
                ptx::tc_commit(&sh->accfull[slot]);  // accumulator ready for the epilogue
            });
        }
    } else {
        // ------------------------------------------------ epilogue warps
        const int q = warp & 3;                 // TMEM lane quadrant this warp may access
        const int h = (warp - 2) >> 2;          // which 128-column half of the tile
        const ModP M = a.mp;
        uint32_t acc_par[2] = {0, 0};
        for_each_step(a, [&](int tile, int slot, int g, int kb) {
            ptx::mbar_wait(&sh->accfull[slot], acc_par[slot]);
            acc_par[slot] ^= 1;
            ptx::tc_fence_after();
            const bool last_kb = (kb == a.nkb - 1);
            const bool final_step = last_kb && g == 0;
            const bool horner = last_kb && g > 0;
            const uint32_t tcol = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + slot * kTileN + h * 128;
            int tm, tn;
            tile_coords(a, tile, tm, tn);
            const int row = tm * kTileM + q * 32 + static_cast<int>(lane);
            for (int c = 0; c < 4; ++c) {
                uint32_t v[32];
                ptx::tmem_ld32(tcol + c * 32, v);
                ptx::tmem_wait_ld();
                if (!final_step) {
#pragma unroll
                    for (int t = 0; t < 32; ++t) {
                        uint32_t r = residue_i32(static_cast<int32_t>(v[t]), M);
                        if (horner) r = mulmod_shoup(r, M.w256, M.w256_sh, M.p);
                        v[t] = static_cast<uint32_t>(centre(r, M));
                    }
                    ptx::tmem_st32(tcol + c * 32, v);
                } else if (row < a.m) {
                    const int col0 = tn * kTileN + h * 128 + c * 32;
                    int32_t* crow = a.C + static_cast<int64_t>(row) * a.ldc + col0;
                    const bool full = a.vec_store && (col0 + 32 <= a.n);
                    uint32_t cin[32];
                    if (M.beta != 0) {
                        if (full) {
#pragma unroll
                            for (int t = 0; t < 8; ++t) {
                                const int4 x = *reinterpret_cast<const int4*>(crow + 4 * t);
                                cin[4 * t] = x.x; cin[4 * t + 1] = x.y; cin[4 * t + 2] = x.z; cin[4 * t + 3] = x.w;
                            }
                        } else {
#pragma unroll
                            for (int t = 0; t < 32; ++t) cin[t] = (col0 + t < a.n) ? crow[t] : 0;
                        }
                    }
#pragma unroll
                    for (int t = 0; t < 32; ++t) {
                        uint32_t r = mulmod_shoup(residue_i32(static_cast<int32_t>(v[t]), M), M.alpha, M.alpha_sh, M.p);
                        if (M.beta != 0) {
                            const uint32_t cr = residue_i32(static_cast<int32_t>(cin[t]), M);
                            r = addmod(r, mulmod_shoup(cr, M.beta, M.beta_sh, M.p), M.p);
                        }
                        v[t] = r;
                    }
                    if (full) {
#pragma unroll
                        for (int t = 0; t < 8; ++t)
                            *reinterpret_cast<int4*>(crow + 4 * t) =
                                make_int4(v[4 * t], v[4 * t + 1], v[4 * t + 2], v[4 * t + 3]);
                    } else {
#pragma unroll
                        for (int t = 0; t < 32; ++t)
                            if (col0 + t < a.n) crow[t] = static_cast<int32_t>(v[t]);
                    }
                }
            }
            if (!final_step) ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&sh->accempty[slot]);
        });
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// Limb planes [L][rows][k_pad] int8 as a 3-D tensor (k fastest), box 128 x box_rows x 1, 128B swizzle.
bool make_plane_map(CUtensorMap* map, const int8_t* base, int L, int64_t rows, int64_t k_pad, int box_rows) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(k_pad), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(L)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(k_pad), static_cast<cuuint64_t>(rows * k_pad)};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

uint32_t make_idesc(bool a_signed, bool b_signed, bool saturate) {
    uint32_t d = 0;
    d |= (saturate ? 1u : 0u) << 3;          // saturate (s8 only)
    d |= 2u << 4;                             // D format: S32
    d |= (a_signed ? 1u : 0u) << 7;           // A: 0 = u8, 1 = s8
    d |= (b_signed ? 1u : 0u) << 10;          // B: 0 = u8, 1 = s8
    // bits 15/16: A/B K-major (0); no negate
    d |= static_cast<uint32_t>(kTileN >> 3) << 17;  // N / 8
    d |= static_cast<uint32_t>(kTileM >> 4) << 24;  // M / 16
    return d;
}

}  // namespace

int launch_gemm_tc(const Plan& pl, int64_t m, int64_t n, int64_t k, const int8_t* A_limbs, const int8_t* B_limbs,
                   int32_t* C, int64_t ldc, cudaStream_t st) {
    const ff_plan_info& I = pl.info;
    if (m > INT32_MAX - kTileM || n > INT32_MAX - kTileN) return -2;
    GemmArgs a;
    std::memset(&a, 0, sizeof(a));
    a.mp = pl.mp;
    a.C = C;
    a.ldc = ldc;
    a.m = static_cast<int32_t>(m);
    a.n = static_cast<int32_t>(n);
    a.tiles_m = static_cast<int32_t>((m + kTileM - 1) / kTileM);
    a.tiles_n = static_cast<int32_t>((n + kTileN - 1) / kTileN);
    const int64_t nt = static_cast<int64_t>(a.tiles_m) * a.tiles_n;
    if (nt > INT32_MAX / 2) return -2;
    a.num_tiles = static_cast<int32_t>(nt);
    a.k_iters = static_cast<int32_t>((k + kBK - 1) / kBK);
    a.kb_iters = static_cast<int32_t>(I.kb / kBK);
    a.nkb = (a.k_iters + a.kb_iters - 1) / a.kb_iters;
    a.G = I.groups;
    for (int pi = 0; pi < pl.npairs; ++pi) {
        a.pair_i[pi] = static_cast<int8_t>(pl.pair_i[pi]);
        a.pair_j[pi] = static_cast<int8_t>(pl.pair_j[pi]);
        a.idesc[pi] = make_idesc(I.limb_signed[pl.pair_i[pi]] != 0, I.limb_signed[pl.pair_j[pi]] != 0, pl.saturate);
    }
    for (int w = 0; w < I.groups; ++w) {
        a.group_first[w] = static_cast<int8_t>(pl.group_first[w]);
        a.group_len[w] = static_cast<int8_t>(pl.group_len[w]);
    }
    a.vec_store = ((ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0) ? 1 : 0;

    CUtensorMap mapA, mapB;
    if (!make_plane_map(&mapA, A_limbs, I.L, m, I.k_pad, kTileM)) return FF_ERR_CUDA;
    if (!make_plane_map(&mapB, B_limbs, I.L, n, I.k_pad, kTileN)) return FF_ERR_CUDA;

    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(ffgemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes) !=
            cudaSuccess)
            return FF_ERR_CUDA;
        attr_set = true;
    }
    const int grid = static_cast<int>(nt < num_sms() ? nt : num_sms());
    ffgemm_tc_kernel<<<grid, kThreads, kSmemBytes, st>>>(mapA, mapB, a);
    return cudaGetLastError() == cudaSuccess ? 0 : FF_ERR_CUDA;
}

}  // namespace ff
