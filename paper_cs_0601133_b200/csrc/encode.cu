// encode.cu -- normalise + centre + limb-encode an int32 operand into K-major
// int8 limb planes [L][rows][k_pad]; plus the beta*C quick-return kernel.
//
// PAPER.md l.139-141 (Sec. 2.1.2): "any prime field Z_p can be naturally
// embedded into Z by representing its elements with an integer of an interval
// [m, M], such that M - m = p - 1"; l.153: the centred interval
// [-(p-1)/2, (p-1)/2] halves the worst-case magnitude (Eq. (2)).  We take the
// centred representative c of x mod p and split it into L int8 digits with
// c = sum_i d_i 256^i exactly, so that every limb product is
// an exact 8x8-bit integer product on the tensor cores.
//
// HBM-bound: each element is read once (4 B) and written once per limb (L B).
// Both kernels are templated on (L, scheme) so the digits live in registers,
// and both write whole 128-byte lines of every limb plane per warp.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "internal.h"
#include "modp.cuh"
#include "ptx.cuh"

namespace ff {

namespace {

// Digits of one centred residue, packed into byte `pos` of w[i] (limb i).
// S: balanced bytes (low byte reinterpreted as s8, subtract, shift);
// T: two's-complement bytes (low limbs u8, top limb s8).  Subtract-then-shift
// is an exact division by 256.
template <int L, int SCHEME>
__device__ __forceinline__ void put_digits(int32_t c, int pos, uint32_t (&w)[L]) {
#pragma unroll
    for (int i = 0; i < L; ++i) {
        const int32_t lo = (SCHEME == FF_SCHEME_S) ? static_cast<int32_t>(static_cast<int8_t>(c & 0xFF)) : (c & 0xFF);
        w[i] |= static_cast<uint32_t>(lo & 0xFF) << (8 * pos);
        c = (c - lo) >> 8;
    }
}

// Source already K-major: limb row r = X[r*ldx + 0..k).  One thread encodes 4
// consecutive elements of a row into one 32-bit word per limb plane, so a warp
// reads 512 contiguous bytes and writes 128 contiguous bytes per plane.  Each
// thread handles kRowsInFlight rows per pass with all their loads issued first
// (one 16-byte load per thread in flight left this HBM-bound pass at ~4.3 TB/s).
constexpr int kRowsInFlight = 4;
template <int L, int SCHEME>
__global__ void __launch_bounds__(256) encode_direct_kernel(ModP M, int64_t rows, int64_t k, int64_t k_pad,
                                                            const int32_t* __restrict__ X, int64_t ldx,
                                                            int8_t* __restrict__ limbs, int vec_ok) {
    ptx::pdl_trigger();   // the GEMM that consumes these limbs may start its prologue
    const int64_t groups = k_pad / 4;
    const int64_t plane = rows * k_pad;
    const int64_t rstep = gridDim.y;
    for (int64_t r0 = blockIdx.y; r0 < rows; r0 += rstep * kRowsInFlight) {
        for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
             g += (int64_t)gridDim.x * blockDim.x) {
            const int64_t kk = 4 * g;
            int32_t x[kRowsInFlight][4];
#pragma unroll
            for (int u = 0; u < kRowsInFlight; ++u) {
                const int64_t r = r0 + u * rstep;
                const int32_t* src = X + (r < rows ? r : rows - 1) * ldx;
                if (vec_ok && kk + 4 <= k) {
                    const int4 v = __ldg(reinterpret_cast<const int4*>(src + kk));
                    x[u][0] = v.x; x[u][1] = v.y; x[u][2] = v.z; x[u][3] = v.w;
                } else {
#pragma unroll
                    for (int t = 0; t < 4; ++t) x[u][t] = (kk + t < k) ? __ldg(src + kk + t) : 0;
                }
            }
#pragma unroll
            for (int u = 0; u < kRowsInFlight; ++u) {
                const int64_t r = r0 + u * rstep;
                if (r >= rows) break;
                uint32_t w[L];
#pragma unroll
                for (int i = 0; i < L; ++i) w[i] = 0;
                centre_all(x[u], M);
#pragma unroll
                for (int t = 0; t < 4; ++t) put_digits<L, SCHEME>(x[u][t], t, w);
                uint32_t* dst = reinterpret_cast<uint32_t*>(limbs + r * k_pad);
#pragma unroll
                for (int i = 0; i < L; ++i) dst[g + i * (plane / 4)] = w[i];
            }
        }
    }
}

// Source transposed: limb row r, column kk = X[kk*ldx + r].  Tiles of 32 rows
// (r) x 128 columns (kk): the load phase reads 128-byte rows of X (a warp =
// 32 consecutive r at one kk); each thread holds 4 groups of 4 consecutive kk
// of its row, so the digits of a group pack into one 32-bit word per plane,
// stored into SMEM tiles [L][32][132] (row pitch 33 words: the word stores
// and the 16-byte reads below are bank-conflict free); the write phase then
// emits whole 128-byte limb rows, four rows per warp per plane.
constexpr int kTR = 32, kTK = 128, kPitch = kTK + 4;
template <int L, int SCHEME>
__global__ void __launch_bounds__(256) encode_trans_kernel(ModP M, int64_t rows, int64_t k, int64_t k_pad,
                                                           const int32_t* __restrict__ X, int64_t ldx,
                                                           int8_t* __restrict__ limbs) {
    ptx::pdl_trigger();   // the GEMM that consumes these limbs may start its prologue
    __shared__ __align__(16) uint8_t tile[L][kTR][kPitch];
    const int64_t plane = rows * k_pad;
    const int64_t tiles_r = (rows + kTR - 1) / kTR;
    const int64_t tiles_k = (k_pad + kTK - 1) / kTK;
    const int lr = threadIdx.x % kTR;       // load: r offset
    const int lk = threadIdx.x / kTR;       // load: kk offset 0..7 (+8 i)
    const int wr = (threadIdx.x / 32) * 4 + (threadIdx.x % 32) / 8;   // write: row 0..31
    const int wc = (threadIdx.x % 8) * 16;                            // write: column 0..112
    // Software-pipelined: the next tile's 16 loads are issued before this
    // tile's write phase, so HBM reads overlap the SMEM transpose and stores.
    int32_t xv[kTK / 8];
    auto load_tile = [&](int64_t t) {
        const int64_t r0 = (t % tiles_r) * kTR;
        const int64_t kk0 = (t / tiles_r) * kTK;
        const bool rin = (r0 + lr) < rows;
        const int32_t* col = X + (r0 + lr);
#pragma unroll
        for (int i = 0; i < kTK / 8; ++i) {        // all 16 loads in flight first
            const int64_t kk = kk0 + 4 * lk + 32 * (i >> 2) + (i & 3);
            xv[i] = (kk < k && rin) ? __ldg(col + kk * ldx) : 0;
        }
    };
    const int64_t ntiles = tiles_r * tiles_k;
    if (static_cast<int64_t>(blockIdx.x) < ntiles) load_tile(blockIdx.x);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t r0 = (t % tiles_r) * kTR;
        const int64_t kk0 = (t / tiles_r) * kTK;
        __syncthreads();
        centre_all(xv, M);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            uint32_t w[L];
#pragma unroll
            for (int l = 0; l < L; ++l) w[l] = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e) put_digits<L, SCHEME>(xv[4 * g + e], e, w);
#pragma unroll
            for (int l = 0; l < L; ++l) *reinterpret_cast<uint32_t*>(&tile[l][lr][4 * lk + 32 * g]) = w[l];
        }
        if (t + gridDim.x < ntiles) load_tile(t + gridDim.x);
        __syncthreads();
        const int64_t r = r0 + wr;
        const int64_t kc = kk0 + wc;
        if (r < rows && kc < k_pad) {
            int8_t* dst = limbs + r * k_pad + kc;
#pragma unroll
            for (int l = 0; l < L; ++l) {
                const uint32_t* src = reinterpret_cast<const uint32_t*>(&tile[l][wr][wc]);
                *reinterpret_cast<uint4*>(dst + l * plane) = make_uint4(src[0], src[1], src[2], src[3]);
            }
        }
    }
}

// TMA-fed variant of the transposed encoder (limb schemes): tiles of 128 k-rows
// x 32 columns of X (16 KB) stream into a 4-stage shared-memory ring by TMA
// (one thread issues, zero fill beyond the matrix = the K padding), so the
// loads no longer wait on the per-thread load latency.  Thread (r, kg) reads
// the 16 values X[kg*16 .. +16][r] of its row r (bank r: conflict-free), packs
// their digits and stages them as [L][32][132] bytes; whole 128-byte limb rows
// are then written as before.
constexpr int kTmaStages = 4;
constexpr int kTmaTileBytes = kTK * kTR * 4;     // 128 k-rows x 32 columns of int32
constexpr int kTmaSmem = kTmaStages * kTmaTileBytes + 4 * kTR * kPitch + 2 * kTmaStages * 8 + 1024;

template <int L, int SCHEME>
__global__ void __launch_bounds__(256) encode_trans_tma_kernel(const __grid_constant__ CUtensorMap tmX, ModP M,
                                                               int64_t rows, int64_t k_pad,
                                                               int8_t* __restrict__ limbs) {
    ptx::pdl_trigger();   // the GEMM that consumes these limbs may start its prologue
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int32_t* ring = reinterpret_cast<const int32_t*>(sm);
    uint8_t (*tile)[kTR][kPitch] = reinterpret_cast<uint8_t (*)[kTR][kPitch]>(sm + kTmaStages * kTmaTileBytes);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kTmaStages * kTmaTileBytes + 4 * kTR * kPitch);
    uint64_t* empty = full + kTmaStages;
    const int64_t plane = rows * k_pad;
    const int64_t tiles_r = (rows + kTR - 1) / kTR;
    const int64_t tiles_k = (k_pad + kTK - 1) / kTK;
    const int64_t ntiles = tiles_r * tiles_k;
    const int tid = threadIdx.x, r = tid % kTR, kg = tid / kTR;          // kg: 16 k-values each
    const int wr = (tid / 32) * 4 + (tid % 32) / 8, wc = (tid % 8) * 16;
    if (tid == 0) {
        for (int s = 0; s < kTmaStages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 256); }
        ptx::fence_barrier_init();
    }
    __syncthreads();
    const uint64_t pol = ptx::policy_evict_normal();
    auto issue = [&](int64_t j) {                       // j-th tile of this CTA into stage j % S
        const int64_t t = blockIdx.x + j * gridDim.x;
        const int s = static_cast<int>(j % kTmaStages);
        ptx::mbar_arrive_expect_tx(&full[s], kTmaTileBytes);
        ptx::tma_load_2d(const_cast<int32_t*>(ring) + s * (kTmaTileBytes / 4), &tmX, &full[s],
                         static_cast<int32_t>((t % tiles_r) * kTR), static_cast<int32_t>((t / tiles_r) * kTK), pol);
    };
    const int64_t mine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    if (tid == 0)
        for (int64_t j = 0; j < kTmaStages && j < mine; ++j) issue(j);
    for (int64_t j = 0; j < mine; ++j) {
        const int64_t t = blockIdx.x + j * gridDim.x;
        const int s = static_cast<int>(j % kTmaStages);
        const uint32_t par = static_cast<uint32_t>((j / kTmaStages) & 1);
        ptx::mbar_wait(&full[s], par);
        const int32_t* T = ring + s * (kTmaTileBytes / 4);     // [128][32]
        uint32_t w[4][L];
#pragma unroll
        for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int l = 0; l < L; ++l) w[g][l] = 0;
        int32_t xv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) xv[i] = T[(kg * 16 + i) * kTR + r];
        centre_all(xv, M);
#pragma unroll
        for (int i = 0; i < 16; ++i) put_digits<L, SCHEME>(xv[i], i & 3, w[i >> 2]);
        ptx::mbar_arrive(&empty[s]);                            // this stage may be refilled
        if (tid == 0 && j + kTmaStages < mine) {
            ptx::mbar_wait(&empty[s], par);
            issue(j + kTmaStages);
        }
        __syncthreads();                                        // previous tile's write-out done with `tile`
#pragma unroll
        for (int l = 0; l < L; ++l)
#pragma unroll
            for (int g = 0; g < 4; ++g) *reinterpret_cast<uint32_t*>(&tile[l][r][kg * 16 + 4 * g]) = w[g][l];
        __syncthreads();
        const int64_t rr = (t % tiles_r) * kTR + wr;
        const int64_t kc = (t / tiles_r) * kTK + wc;
        if (rr < rows && kc < k_pad) {
            int8_t* dst = limbs + rr * k_pad + kc;
#pragma unroll
            for (int l = 0; l < L; ++l) {
                const uint32_t* src = reinterpret_cast<const uint32_t*>(&tile[l][wr][wc]);
                *reinterpret_cast<uint4*>(dst + l * plane) = make_uint4(src[0], src[1], src[2], src[3]);
            }
        }
    }
}

typedef CUresult (*EncodeTiledFnE)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// X stored [k][ld] int32 (the transposed source) as a 2-D tensor map, box 32 x 128.
bool make_src_map(CUtensorMap* map, const int32_t* X, int64_t rows, int64_t k, int64_t ldx) {
    static EncodeTiledFnE fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
        fn = reinterpret_cast<EncodeTiledFnE>(p);
    }
    if ((reinterpret_cast<uintptr_t>(X) & 15) || ((ldx * 4) % 16) || rows <= 0 || k <= 0) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(k)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx * 4)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kTR), static_cast<cuuint32_t>(kTK)};
    cuuint32_t estr[2] = {1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<int32_t*>(X), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- multi-modular (CRT) planes: plane i holds the centred
// residue of c (the centred residue of x mod p) modulo q_i, as s8.  The same
// two access patterns as the limb encoders; the moduli are runtime constants.

// Centred residue of c mod q as a byte, in fp32 (full-rate FFMA instead of
// integer Barrett).  c = h1 2^15 + h0 with h0 in [0, 2^15): s = h1 (2^15 mod q)
// + h0 satisfies |s| < 2^23 for odd q <= 255, so s is exact in fp32 and
// t = fl(s fl(1/q)) rounded to an integer equals round(s/q): its error is below
// |s/q| 2^-24 < 1/(2q), while s/q is at least 1/(2q) away from any half-integer
// (q odd).  r = s - q t is then the exact centred residue, and the low byte of
// the float r + 1.5 2^23 is its two's-complement byte.  q = 256: the low byte of c.
struct CrtDigitsIn {
    float h0, h1;
};

__device__ __forceinline__ CrtDigitsIn crt_split(int32_t c) {
    const uint32_t h0 = static_cast<uint32_t>(c) & 0x7FFFu;
    const uint32_t h1 = static_cast<uint32_t>((c >> 15) + 32768);          // in [0, 2^16)
    CrtDigitsIn d;
    d.h0 = __uint_as_float(0x4B000000u | h0) - 8388608.0f;
    d.h1 = __uint_as_float(0x4B000000u | h1) - (8388608.0f + 32768.0f);
    return d;
}

// The low bytes of four words, in order, in one word (three byte permutes).
__device__ __forceinline__ uint32_t pack_lo4(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3) {
    return __byte_perm(__byte_perm(x0, x1, 0x0040), __byte_perm(x2, x3, 0x0040), 0x5410);
}

__device__ __forceinline__ uint32_t crt_digit(int32_t c, const CrtDigitsIn& d, const CrtConsts& C, int i) {
    if (C.q[i] == 256u) return static_cast<uint32_t>(c) & 0xFFu;
    const float s = fmaf(d.h1, C.fw15[i], d.h0);
    const float t = fmaf(s, C.finv[i], 12582912.0f) - 12582912.0f;
    const float r = fmaf(-C.fq[i], t, s);
    return __float_as_uint(r + 12582912.0f) & 0xFFu;
}

// 16 consecutive elements per thread: four 16-byte loads, one 16-byte store per
// plane (the per-element residue arithmetic dominates; wide accesses amortise
// the address and store instructions).
__global__ void __launch_bounds__(256) encode_crt_direct_kernel(ModP M, CrtConsts C, int64_t rows, int64_t k,
                                                                int64_t k_pad, const int32_t* __restrict__ X,
                                                                int64_t ldx, int8_t* __restrict__ planes,
                                                                int vec_ok) {
    ptx::pdl_trigger();   // the GEMM that consumes these limbs may start its prologue
    const int64_t groups = k_pad / 16;
    const int64_t plane = rows * k_pad;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
        const int32_t* src = X + r * ldx;
        for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups;
             g += (int64_t)gridDim.x * blockDim.x) {
            const int64_t kk = 16 * g;
            int32_t c[16];
            if (vec_ok && kk + 16 <= k) {
#pragma unroll
                for (int v4 = 0; v4 < 4; ++v4) {
                    const int4 v = __ldg(reinterpret_cast<const int4*>(src + kk) + v4);
                    c[4 * v4] = v.x; c[4 * v4 + 1] = v.y; c[4 * v4 + 2] = v.z; c[4 * v4 + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int t = 0; t < 16; ++t) c[t] = (kk + t < k) ? __ldg(src + kk + t) : 0;
            }
            CrtDigitsIn dg[16];
            centre_all(c, M);
#pragma unroll
            for (int t = 0; t < 16; ++t) dg[t] = crt_split(c[t]);
            int8_t* dst = planes + r * k_pad + kk;
            // plane 0 is q = 256 (the planner picks 256 first): the low byte of c
            uint32_t w0[4];
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
                w0[q4] = pack_lo4(c[4 * q4], c[4 * q4 + 1], c[4 * q4 + 2], c[4 * q4 + 3]);
            *reinterpret_cast<uint4*>(dst) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
#pragma unroll 1
            for (int i = 1; i < C.nq; ++i) {
                const float fq = C.fq[i], fi = C.finv[i], fw = C.fw15[i];
                uint32_t b[16];
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const float sv = fmaf(dg[t].h1, fw, dg[t].h0);
                    const float tq = fmaf(sv, fi, 12582912.0f) - 12582912.0f;
                    const float rr = fmaf(-fq, tq, sv);
                    b[t] = __float_as_uint(rr + 12582912.0f);      // the residue's byte is the low byte
                }
                *reinterpret_cast<uint4*>(dst + i * plane) =
                    make_uint4(pack_lo4(b[0], b[1], b[2], b[3]), pack_lo4(b[4], b[5], b[6], b[7]),
                               pack_lo4(b[8], b[9], b[10], b[11]), pack_lo4(b[12], b[13], b[14], b[15]));
            }
        }
    }
}

// Transposed source: as encode_trans_kernel, the moduli in batches of 4 planes
// through the SMEM byte tile (the centred values stay in registers).
__global__ void __launch_bounds__(256) encode_crt_trans_kernel(ModP M, CrtConsts C, int64_t rows, int64_t k,
                                                               int64_t k_pad, const int32_t* __restrict__ X,
                                                               int64_t ldx, int8_t* __restrict__ planes) {
    ptx::pdl_trigger();   // the GEMM that consumes these limbs may start its prologue
    __shared__ __align__(16) uint8_t tile[4][kTR][kPitch];
    const int64_t plane = rows * k_pad;
    const int64_t tiles_r = (rows + kTR - 1) / kTR;
    const int64_t tiles_k = (k_pad + kTK - 1) / kTK;
    const int lr = threadIdx.x % kTR;
    const int lk = threadIdx.x / kTR;
    const int wr = (threadIdx.x / 32) * 4 + (threadIdx.x % 32) / 8;
    const int wc = (threadIdx.x % 8) * 16;
    int32_t xv[kTK / 8];
    auto load_tile = [&](int64_t t) {
        const int64_t r0 = (t % tiles_r) * kTR;
        const int64_t kk0 = (t / tiles_r) * kTK;
        const bool rin = (r0 + lr) < rows;
        const int32_t* col = X + (r0 + lr);
#pragma unroll
        for (int i = 0; i < kTK / 8; ++i) {
            const int64_t kk = kk0 + 4 * lk + 32 * (i >> 2) + (i & 3);
            xv[i] = (kk < k && rin) ? __ldg(col + kk * ldx) : 0;
        }
    };
    const int64_t ntiles = tiles_r * tiles_k;
    if (static_cast<int64_t>(blockIdx.x) < ntiles) load_tile(blockIdx.x);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t r0 = (t % tiles_r) * kTR;
        const int64_t kk0 = (t / tiles_r) * kTK;
        int32_t cv[kTK / 8];
#pragma unroll
        for (int i = 0; i < kTK / 8; ++i) cv[i] = xv[i];
        centre_all(cv, M);
        if (t + gridDim.x < ntiles) load_tile(t + gridDim.x);     // next tile's loads in flight
        const int64_t r = r0 + wr;
        const int64_t kc = kk0 + wc;
        for (int b0 = 0; b0 < C.nq; b0 += 4) {
            // this batch's constants in registers (runtime-indexed parameter
            // loads inside the digit loop dominated the instruction count)
            float fq[4], fi[4], fw[4];
            bool q256[4], live[4];
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const int pl = b0 + l < C.nq ? b0 + l : 0;
                live[l] = b0 + l < C.nq;
                q256[l] = C.q[pl] == 256u;
                fq[l] = C.fq[pl]; fi[l] = C.finv[pl]; fw[l] = C.fw15[pl];
            }
            __syncthreads();
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int32_t c = cv[4 * g + e];
                    const CrtDigitsIn d = crt_split(c);
#pragma unroll
                    for (int l = 0; l < 4; ++l) {
                        const float sv = fmaf(d.h1, fw[l], d.h0);
                        const float t = fmaf(sv, fi[l], 12582912.0f) - 12582912.0f;
                        const float rr = fmaf(-fq[l], t, sv);
                        const uint32_t byte = q256[l] ? (static_cast<uint32_t>(c) & 0xFFu)
                                                      : (__float_as_uint(rr + 12582912.0f) & 0xFFu);
                        w[l] |= byte << (8 * e);
                    }
                }
#pragma unroll
                for (int l = 0; l < 4; ++l)
                    if (live[l]) *reinterpret_cast<uint32_t*>(&tile[l][lr][4 * lk + 32 * g]) = w[l];
            }
            __syncthreads();
            if (r < rows && kc < k_pad) {
                int8_t* dst = planes + r * k_pad + kc;
#pragma unroll
                for (int l = 0; l < 4; ++l) {
                    if (b0 + l < C.nq) {
                        const uint32_t* src = reinterpret_cast<const uint32_t*>(&tile[l][wr][wc]);
                        *reinterpret_cast<uint4*>(dst + (b0 + l) * plane) = make_uint4(src[0], src[1], src[2], src[3]);
                    }
                }
            }
        }
    }
}

// TMA-fed transposed CRT encoder: as encode_trans_tma_kernel, all n_q planes
// staged at once ([n_q][32][132] bytes) so each tile needs two barriers, and
// the per-plane constants are loaded once per plane.
constexpr int kCrtStages = 2;   // 2 CTAs per SM: the residue arithmetic needs the warps
constexpr int kCrtTmaSmem = kCrtStages * kTmaTileBytes + kMaxMod * kTR * kPitch + 2 * kCrtStages * 8 + 1024;

__global__ void __launch_bounds__(256) encode_crt_trans_tma_kernel(const __grid_constant__ CUtensorMap tmX, ModP M,
                                                                   CrtConsts C, int64_t rows, int64_t k_pad,
                                                                   int8_t* __restrict__ planes) {
    ptx::pdl_trigger();   // the GEMM that consumes these limbs may start its prologue
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int32_t* ring = reinterpret_cast<const int32_t*>(sm);
    uint8_t (*tile)[kTR][kPitch] = reinterpret_cast<uint8_t (*)[kTR][kPitch]>(sm + kCrtStages * kTmaTileBytes);
    const int nq = C.nq;   // staging for nq planes only (dynamic SMEM sized by the launch)
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + kCrtStages * kTmaTileBytes + nq * kTR * kPitch);
    uint64_t* empty = full + kCrtStages;
    const int64_t plane = rows * k_pad;
    const int64_t tiles_r = (rows + kTR - 1) / kTR;
    const int64_t tiles_k = (k_pad + kTK - 1) / kTK;
    const int64_t ntiles = tiles_r * tiles_k;
    const int tid = threadIdx.x, r = tid % kTR, kg = tid / kTR;
    const int wr = (tid / 32) * 4 + (tid % 32) / 8, wc = (tid % 8) * 16;
    if (tid == 0) {
        for (int s = 0; s < kCrtStages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 256); }
        ptx::fence_barrier_init();
    }
    __syncthreads();
    const uint64_t pol = ptx::policy_evict_normal();
    auto issue = [&](int64_t j) {
        const int64_t t = blockIdx.x + j * gridDim.x;
        const int s = static_cast<int>(j % kCrtStages);
        ptx::mbar_arrive_expect_tx(&full[s], kTmaTileBytes);
        ptx::tma_load_2d(const_cast<int32_t*>(ring) + s * (kTmaTileBytes / 4), &tmX, &full[s],
                         static_cast<int32_t>((t % tiles_r) * kTR), static_cast<int32_t>((t / tiles_r) * kTK), pol);
    };
    const int64_t mine = (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x;
    if (tid == 0)
        for (int64_t j = 0; j < kCrtStages && j < mine; ++j) issue(j);
    for (int64_t j = 0; j < mine; ++j) {
        const int64_t t = blockIdx.x + j * gridDim.x;
        const int s = static_cast<int>(j % kCrtStages);
        const uint32_t par = static_cast<uint32_t>((j / kCrtStages) & 1);
        ptx::mbar_wait(&full[s], par);
        const int32_t* T = ring + s * (kTmaTileBytes / 4);
        int32_t c[16];
        CrtDigitsIn dg[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) c[i] = T[(kg * 16 + i) * kTR + r];
        centre_all(c, M);
#pragma unroll
        for (int i = 0; i < 16; ++i) dg[i] = crt_split(c[i]);
        ptx::mbar_arrive(&empty[s]);
        if (tid == 0 && j + kCrtStages < mine) {
            ptx::mbar_wait(&empty[s], par);
            issue(j + kCrtStages);
        }
        __syncthreads();                                  // previous tile's write-out is done with `tile`
        {   // plane 0: q = 256, the low byte of c
#pragma unroll
            for (int g = 0; g < 4; ++g)
                *reinterpret_cast<uint32_t*>(&tile[0][r][kg * 16 + 4 * g]) =
                    pack_lo4(c[4 * g], c[4 * g + 1], c[4 * g + 2], c[4 * g + 3]);
        }
#pragma unroll 1
        for (int pl = 1; pl < nq; ++pl) {
            const float fq = C.fq[pl], fi = C.finv[pl], fw = C.fw15[pl];
            uint32_t b[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float sv = fmaf(dg[i].h1, fw, dg[i].h0);
                const float tq = fmaf(sv, fi, 12582912.0f) - 12582912.0f;
                const float rr = fmaf(-fq, tq, sv);
                b[i] = __float_as_uint(rr + 12582912.0f);
            }
#pragma unroll
            for (int g = 0; g < 4; ++g)
                *reinterpret_cast<uint32_t*>(&tile[pl][r][kg * 16 + 4 * g]) =
                    pack_lo4(b[4 * g], b[4 * g + 1], b[4 * g + 2], b[4 * g + 3]);
        }
        __syncthreads();
        const int64_t rr = (t % tiles_r) * kTR + wr;
        const int64_t kc = (t / tiles_r) * kTK + wc;
        if (rr < rows && kc < k_pad) {
            int8_t* dst = planes + rr * k_pad + kc;
            for (int pl = 0; pl < nq; ++pl) {
                const uint32_t* src = reinterpret_cast<const uint32_t*>(&tile[pl][wr][wc]);
                *reinterpret_cast<uint4*>(dst + pl * plane) = make_uint4(src[0], src[1], src[2], src[3]);
            }
        }
    }
}

// C <- beta * C mod p (k = 0 or alpha = 0); C <- 0 when beta = 0 (C not read).
// Rows on grid.y, 4 columns per thread (16-byte accesses when aligned).
__global__ void __launch_bounds__(256) scale_c_kernel(ModP M, int64_t m, int64_t n, int32_t* __restrict__ C,
                                                      int64_t ldc, int vec_ok) {
    for (int64_t r = blockIdx.y; r < m; r += gridDim.y) {
        int32_t* row = C + r * ldc;
        for (int64_t c = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x); c < n;
             c += 4 * (int64_t)gridDim.x * blockDim.x) {
            if (vec_ok && c + 4 <= n) {
                int4 v = make_int4(0, 0, 0, 0);
                if (M.beta != 0) {
                    v = *reinterpret_cast<const int4*>(row + c);
                    v.x = static_cast<int32_t>(mulmod_shoup(residue_i32(v.x, M), M.beta, M.beta_sh, M.p));
                    v.y = static_cast<int32_t>(mulmod_shoup(residue_i32(v.y, M), M.beta, M.beta_sh, M.p));
                    v.z = static_cast<int32_t>(mulmod_shoup(residue_i32(v.z, M), M.beta, M.beta_sh, M.p));
                    v.w = static_cast<int32_t>(mulmod_shoup(residue_i32(v.w, M), M.beta, M.beta_sh, M.p));
                }
                *reinterpret_cast<int4*>(row + c) = v;
            } else {
                for (int64_t t = c; t < c + 4 && t < n; ++t)
                    row[t] = M.beta == 0 ? 0
                                         : static_cast<int32_t>(mulmod_shoup(residue_i32(row[t], M), M.beta,
                                                                             M.beta_sh, M.p));
            }
        }
    }
}

int grid_for(int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (g > cap) g = cap;
    return static_cast<int>(g < 1 ? 1 : g);
}

template <int L, int SCHEME>
void launch_encode_t(const Plan& pl, int kmajor_src, int64_t rows, int64_t k, int64_t k_pad, const int32_t* X,
                     int64_t ldx, int8_t* limbs, cudaStream_t st) {
    if (kmajor_src) {
        const int64_t groups = k_pad / 4;
        int gx = static_cast<int>((groups + 255) / 256);
        if (gx > 64) gx = 64;
        int64_t gy = (int64_t)num_sms() * 8 / gx;
        if (gy > rows) gy = rows;
        if (gy > 65535) gy = 65535;
        if (gy < 1) gy = 1;
        const int vec_ok = ((ldx % 4) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) ? 1 : 0;
        note_launch();
        encode_direct_kernel<L, SCHEME><<<dim3(gx, static_cast<unsigned>(gy)), 256, 0, st>>>(
            pl.mp, rows, k, k_pad, X, ldx, limbs, vec_ok);
    } else {
        const int64_t tiles = ((rows + kTR - 1) / kTR) * ((k_pad + kTK - 1) / kTK);
        CUtensorMap map;
        if (!knobs().enc_notma && make_src_map(&map, X, rows, k, ldx)) {   // FF_ENC_NOTMA: the LSU-load version
            set_smem_attr(reinterpret_cast<const void*>(encode_trans_tma_kernel<L, SCHEME>), kTmaSmem);
            const int64_t cap = (int64_t)num_sms() * 2;
            note_launch();
            encode_trans_tma_kernel<L, SCHEME><<<static_cast<int>(tiles < cap ? tiles : cap), 256, kTmaSmem, st>>>(
                map, pl.mp, rows, k_pad, limbs);
            return;
        }
        const int64_t cap = (int64_t)num_sms() * 8;
        note_launch();
        encode_trans_kernel<L, SCHEME><<<static_cast<int>(tiles < cap ? tiles : cap), 256, 0, st>>>(
            pl.mp, rows, k, k_pad, X, ldx, limbs);
    }
}

}  // namespace

cudaError_t launch_encode(const Plan& pl, int kmajor_src, int64_t rows, int64_t k, const int32_t* X, int64_t ldx,
                          int8_t* limbs, cudaStream_t st) {
    const int64_t k_pad = pl.info.k_pad;
    if (rows == 0 || k_pad == 0) return cudaSuccess;
    if (pl.crt) {
        if (kmajor_src) {
            const int64_t groups = k_pad / 16;
            int gx = static_cast<int>((groups + 255) / 256);
            if (gx > 64) gx = 64;
            int64_t gy = (int64_t)num_sms() * 8 / gx;
            if (gy > rows) gy = rows;
            if (gy > 65535) gy = 65535;
            if (gy < 1) gy = 1;
            const int vec_ok = ((ldx % 4) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0) ? 1 : 0;
            note_launch();
            encode_crt_direct_kernel<<<dim3(gx, static_cast<unsigned>(gy)), 256, 0, st>>>(
                pl.mp, pl.cc, rows, k, k_pad, X, ldx, limbs, vec_ok);
        } else {
            const int64_t tiles = ((rows + kTR - 1) / kTR) * ((k_pad + kTK - 1) / kTK);
            CUtensorMap map;
            if (!knobs().enc_notma && make_src_map(&map, X, rows, k, ldx)) {
                const cudaError_t ea = set_smem_attr(reinterpret_cast<const void*>(encode_crt_trans_tma_kernel), kCrtTmaSmem);
                if (ea != cudaSuccess) return ea;
                // SMEM for this plan's nq planes only: 3 CTAs per SM for nq = 9 (2 at kMaxMod)
                const int smem = kCrtStages * kTmaTileBytes + pl.cc.nq * kTR * kPitch + 2 * kCrtStages * 8 + 1024;
                int per_sm = 0;
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, encode_crt_trans_tma_kernel, 256, smem) !=
                        cudaSuccess || per_sm < 1) {
                    cudaGetLastError();
                    per_sm = 2;
                }
                const int64_t capt = (int64_t)num_sms() * per_sm;
                note_launch();
                encode_crt_trans_tma_kernel<<<static_cast<int>(tiles < capt ? tiles : capt), 256, smem, st>>>(
                    map, pl.mp, pl.cc, rows, k_pad, limbs);
                return cudaGetLastError();
            }
            const int64_t cap = (int64_t)num_sms() * 8;
            note_launch();
            encode_crt_trans_kernel<<<static_cast<int>(tiles < cap ? tiles : cap), 256, 0, st>>>(
                pl.mp, pl.cc, rows, k, k_pad, X, ldx, limbs);
        }
        return cudaGetLastError();
    }
    const bool S = pl.info.scheme == FF_SCHEME_S;
    switch (pl.info.L) {
        case 1: S ? launch_encode_t<1, FF_SCHEME_S>(pl, kmajor_src, rows, k, k_pad, X, ldx, limbs, st)
                  : launch_encode_t<1, FF_SCHEME_T>(pl, kmajor_src, rows, k, k_pad, X, ldx, limbs, st); break;
        case 2: S ? launch_encode_t<2, FF_SCHEME_S>(pl, kmajor_src, rows, k, k_pad, X, ldx, limbs, st)
                  : launch_encode_t<2, FF_SCHEME_T>(pl, kmajor_src, rows, k, k_pad, X, ldx, limbs, st); break;
        case 3: S ? launch_encode_t<3, FF_SCHEME_S>(pl, kmajor_src, rows, k, k_pad, X, ldx, limbs, st)
                  : launch_encode_t<3, FF_SCHEME_T>(pl, kmajor_src, rows, k, k_pad, X, ldx, limbs, st); break;
        case 4: S ? launch_encode_t<4, FF_SCHEME_S>(pl, kmajor_src, rows, k, k_pad, X, ldx, limbs, st)
                  : launch_encode_t<4, FF_SCHEME_T>(pl, kmajor_src, rows, k, k_pad, X, ldx, limbs, st); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_scale_c(const ModP& mp, int64_t m, int64_t n, int32_t* C, int64_t ldc, cudaStream_t st) {
    if (m == 0 || n == 0) return cudaSuccess;
    int gx = static_cast<int>((n + 4 * 256 - 1) / (4 * 256));
    if (gx > 64) gx = 64;
    int64_t gy = (int64_t)num_sms() * 8 / gx;
    if (gy > m) gy = m;
    if (gy > 65535) gy = 65535;
    if (gy < 1) gy = 1;
    const int vec_ok = ((ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0) ? 1 : 0;
    note_launch();
    scale_c_kernel<<<dim3(gx, static_cast<unsigned>(gy)), 256, 0, st>>>(mp, m, n, C, ldc, vec_ok);
    return cudaGetLastError();
}

}  // namespace ff
