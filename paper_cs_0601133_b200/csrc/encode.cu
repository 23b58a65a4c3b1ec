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
#include <cuda_runtime.h>

#include "internal.h"
#include "modp.cuh"

namespace ff {

namespace {

constexpr int kVec = 16;  // K elements per thread-chunk (one 16-byte store per limb plane)

// Digits of one centred residue.  S: balanced bytes (reinterpret the low byte
// as s8, subtract, shift); T: two's-complement bytes (top byte signed).  Both
// subtract-then-shift steps are exact divisions by 256.
__device__ __forceinline__ void digits(int32_t c, int L, int scheme, uint8_t* d) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (i < L) {
            const int32_t lo = (scheme == FF_SCHEME_S) ? static_cast<int32_t>(static_cast<int8_t>(c & 0xFF))
                                                       : (c & 0xFF);
            d[i] = static_cast<uint8_t>(lo & 0xFF);
            c = (c - lo) >> 8;
        }
    }
}

// 16 residues -> L packed 16-byte limb vectors.
__device__ __forceinline__ void encode16(const int32_t (&x)[kVec], const ModP& M, int L, int scheme,
                                         uint4 (&out)[4]) {
    uint8_t b[4][kVec];
#pragma unroll
    for (int t = 0; t < kVec; ++t) {
        uint8_t d[4] = {0, 0, 0, 0};
        digits(centre(residue_i32(x[t], M), M), L, scheme, d);
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i][t] = d[i];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
            w[q] = static_cast<uint32_t>(b[i][4 * q]) | (static_cast<uint32_t>(b[i][4 * q + 1]) << 8) |
                   (static_cast<uint32_t>(b[i][4 * q + 2]) << 16) | (static_cast<uint32_t>(b[i][4 * q + 3]) << 24);
        out[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// Source already K-major: limb row r = X[r*ldx + 0..k).
__global__ void __launch_bounds__(256) encode_direct_kernel(ModP M, int L, int scheme, int64_t rows,
                                                            int64_t k, int64_t k_pad,
                                                            const int32_t* __restrict__ X, int64_t ldx,
                                                            int8_t* __restrict__ limbs) {
    const int64_t cpr = k_pad / kVec;
    const int64_t total = rows * cpr;
    const int64_t plane = rows * k_pad;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / cpr;
        const int64_t kk0 = (idx - r * cpr) * kVec;
        const int32_t* src = X + r * ldx + kk0;
        int32_t x[kVec];
        if (kk0 + kVec <= k && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int4 v = __ldg(reinterpret_cast<const int4*>(src) + q);
                x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int t = 0; t < kVec; ++t) x[t] = (kk0 + t < k) ? __ldg(src + t) : 0;
        }
        uint4 out[4];
        encode16(x, M, L, scheme, out);
        int8_t* dst = limbs + r * k_pad + kk0;
        for (int i = 0; i < L; ++i) *reinterpret_cast<uint4*>(dst + i * plane) = out[i];
    }
}

// Source transposed: limb row r, column kk = X[kk*ldx + r].  64x64 tile through SMEM.
constexpr int kT = 64;
__global__ void __launch_bounds__(256) encode_trans_kernel(ModP M, int L, int scheme, int64_t rows,
                                                           int64_t k, int64_t k_pad,
                                                           const int32_t* __restrict__ X, int64_t ldx,
                                                           int8_t* __restrict__ limbs) {
    __shared__ int32_t tile[kT][kT + 1];
    const int64_t plane = rows * k_pad;
    const int c = threadIdx.x % kT;   // r offset within the tile
    const int rr = threadIdx.x / kT;  // 0..3
    const int64_t tiles_r = (rows + kT - 1) / kT;
    const int64_t tiles_k = (k_pad + kT - 1) / kT;
    for (int64_t t = blockIdx.x; t < tiles_r * tiles_k; t += gridDim.x) {
        const int64_t r0 = (t % tiles_r) * kT;
        const int64_t kk0 = (t / tiles_r) * kT;
        __syncthreads();
#pragma unroll 4
        for (int i = 0; i < 16; ++i) {
            const int kl = rr * 16 + i;
            const int64_t kk = kk0 + kl, r = r0 + c;
            tile[kl][c] = (kk < k && r < rows) ? __ldg(X + kk * ldx + r) : 0;
        }
        __syncthreads();
        const int64_t r = r0 + c;
        const int64_t kc = kk0 + rr * 16;
        if (r < rows && kc < k_pad) {
            int32_t x[kVec];
#pragma unroll
            for (int i = 0; i < kVec; ++i) x[i] = tile[rr * 16 + i][c];
            uint4 out[4];
            encode16(x, M, L, scheme, out);
            int8_t* dst = limbs + r * k_pad + kc;
            for (int i = 0; i < L; ++i) *reinterpret_cast<uint4*>(dst + i * plane) = out[i];
        }
    }
}

// C <- beta * C mod p (k = 0 or alpha = 0); C <- 0 when beta = 0 (C not read).
__global__ void scale_c_kernel(ModP M, int64_t m, int64_t n, int32_t* __restrict__ C, int64_t ldc) {
    const int64_t total = m * n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx / n, j = idx - i * n;
        int32_t* c = C + i * ldc + j;
        *c = M.beta == 0 ? 0
                         : static_cast<int32_t>(mulmod_shoup(residue_i32(*c, M), M.beta, M.beta_sh, M.p));
    }
}

int grid_for(int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (g > cap) g = cap;
    return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t launch_encode(const Plan& pl, int kmajor_src, int64_t rows, int64_t k, const int32_t* X,
                          int64_t ldx, int8_t* limbs, cudaStream_t st) {
    const int64_t k_pad = (k + 15) / 16 * 16;
    if (rows == 0 || k_pad == 0) return cudaSuccess;
    if (kmajor_src) {
        encode_direct_kernel<<<grid_for(rows * (k_pad / kVec), 256), 256, 0, st>>>(
            pl.mp, pl.info.L, pl.info.scheme, rows, k, k_pad, X, ldx, limbs);
    } else {
        const int64_t tiles = ((rows + kT - 1) / kT) * ((k_pad + kT - 1) / kT);
        int64_t g = tiles < (int64_t)num_sms() * 8 ? tiles : (int64_t)num_sms() * 8;
        encode_trans_kernel<<<static_cast<int>(g), 256, 0, st>>>(pl.mp, pl.info.L, pl.info.scheme, rows, k,
                                                                k_pad, X, ldx, limbs);
    }
    return cudaGetLastError();
}

cudaError_t launch_scale_c(const ModP& mp, int64_t m, int64_t n, int32_t* C, int64_t ldc, cudaStream_t st) {
    if (m == 0 || n == 0) return cudaSuccess;
    scale_c_kernel<<<grid_for(m * n, 256), 256, 0, st>>>(mp, m, n, C, ldc);
    return cudaGetLastError();
}

}  // namespace ff
