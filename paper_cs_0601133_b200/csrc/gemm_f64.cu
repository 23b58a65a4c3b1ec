// gemm_f64.cu -- the paper-literal engine: "Zpz-double"
// residues multiplied by a floating-point kernel with delayed modular
// reduction, on the B200's fp64 tensor cores.
//
// tcgen05 has no f64 kind, so this is the warp-level DMMA path
// (mma.sync.m8n8k4.f64).  Operands are the centred residues as doubles
// (Eq. (2), l.153-157: the balanced representation halves the magnitude);
// products are accumulated in fp64 registers exactly while the partial sums
// stay below 2^53, i.e. for lambda terms with lambda ((p-1)/2)^2 < 2^52
// (Eq. (2) with gamma = 53; the planner's kb), after which each accumulator is
// reduced "using the floating point inverse" (l.125-127): x - p rint(x / p),
// which may be off by one multiple of p -- harmless for an intermediate, and
// corrected at the end.  The int8 engine (gemm_tc.cu) is the product; this one
// is the paper's own method measured on the same hardware.
//
// Tiling: CTA 64 x 64 outputs, 4 warps of 32 x 32 (4 x 4 m8n8 tiles, 32
// doubles of accumulator per thread), K staged 16 at a time through a 2-deep
// cp.async double buffer; operands are K-major double planes [rows][k_pad].
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "modp.cuh"

namespace ff {

namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16, kPitch = 20, kStages = 2;   // pitch in doubles (bank spread); 40 KB SMEM

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const int sz = pred ? 16 : 0;   // zero-fill when out of range
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

struct F64Args {
    const double* A;      // [m][k_pad] centred residues of op(A)
    const double* B;      // [n][k_pad] centred residues of op(B)^T
    int32_t* C;
    int64_t ldc;
    int64_t m, n, k_pad;
    int32_t kb4;          // reduce the accumulators every kb4 k-steps of 4 (lambda / 4)
    double p, invp;       // p and fl(1/p)
    uint32_t up, alpha, beta;
};

// x - p rint(x / p): exact (fma), |result| <= p/2 + p (the quotient may be off by one).
__device__ __forceinline__ double fp_reduce(double x, double p, double invp) {
    return fma(-rint(x * invp), p, x);
}

__global__ void __launch_bounds__(128) f64_gemm_kernel(F64Args a) {
    __shared__ __align__(16) double As[kStages][kBM][kPitch];
    __shared__ __align__(16) double Bs[kStages][kBN][kPitch];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int wm = warp >> 1, wn = warp & 1;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kBM, n0 = static_cast<int64_t>(blockIdx.x) * kBN;
    const int ktiles = static_cast<int>((a.k_pad + kBK - 1) / kBK);
    auto load = [&](int kt, int stage) {
        // 64 rows x 16 doubles per operand = 512 chunks of 16 B; 4 per thread each
        for (int c = threadIdx.x; c < kBM * 8; c += 128) {
            const int r = c >> 3, ch = c & 7;
            const int64_t kk = static_cast<int64_t>(kt) * kBK + ch * 2;
            const bool inA = (m0 + r) < a.m && kk < a.k_pad;
            const bool inB = (n0 + r) < a.n && kk < a.k_pad;
            cp_async16(&As[stage][r][ch * 2], a.A + (inA ? (m0 + r) * a.k_pad + kk : 0), inA);
            cp_async16(&Bs[stage][r][ch * 2], a.B + (inB ? (n0 + r) * a.k_pad + kk : 0), inB);
        }
    };
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < ktiles) load(s, s);
        cp_async_commit();
    }
    int ksteps = 0;
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        const int st = kt % kStages;
        if (kt + kStages - 1 < ktiles) load(kt + kStages - 1, (kt + kStages - 1) % kStages);
        cp_async_commit();
#pragma unroll
        for (int kk = 0; kk < kBK; kk += 4) {
            double fa[4], fb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) fa[i] = As[st][wm * 32 + i * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int j = 0; j < 4; ++j) fb[j] = Bs[st][wn * 32 + j * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(acc[i][j], fa[i], fb[j]);
            // delayed reduction: every lambda products (Eq. (2), the planner's kb)
            if (++ksteps == a.kb4) {
                ksteps = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        acc[i][j][0] = fp_reduce(acc[i][j][0], a.p, a.invp);
                        acc[i][j][1] = fp_reduce(acc[i][j][1], a.p, a.invp);
                    }
            }
        }
    }
    cp_async_wait<0>();
    // epilogue: exact residue, then (alpha R + beta C) mod p in 64-bit integers
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t r = m0 + wm * 32 + i * 8 + (lane >> 2);
                const int64_t c = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
                if (r >= a.m || c >= a.n) continue;
                double x = fp_reduce(acc[i][j][h], a.p, a.invp);
                int64_t v = static_cast<int64_t>(x);
                v %= static_cast<int64_t>(a.up);
                if (v < 0) v += a.up;
                uint64_t o = static_cast<uint64_t>(v) * a.alpha % a.up;
                int32_t* cp = a.C + r * a.ldc + c;
                if (a.beta) {
                    int64_t cin = static_cast<int64_t>(*cp) % static_cast<int64_t>(a.up);
                    if (cin < 0) cin += a.up;
                    o = (o + static_cast<uint64_t>(cin) * a.beta) % a.up;
                }
                *cp = static_cast<int32_t>(o);
            }
}

// int32 -> centred residue as double, K-major [rows][k_pad] (zero padded).
// kmajor_src: X[r * ldx + kk]; else X[kk * ldx + r] (transposed through SMEM).
__global__ void __launch_bounds__(256) f64_encode_kernel(ModP M, int kmajor_src, int64_t rows, int64_t k,
                                                         int64_t k_pad, const int32_t* __restrict__ X,
                                                         int64_t ldx, double* __restrict__ out) {
    __shared__ double tile[32][33];
    const int64_t tiles_r = (rows + 31) / 32, tiles_k = (k_pad + 31) / 32;
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;   // 32 x 8
    for (int64_t t = blockIdx.x; t < tiles_r * tiles_k; t += gridDim.x) {
        const int64_t r0 = (t % tiles_r) * 32, k0 = (t / tiles_r) * 32;
        __syncthreads();
        for (int yy = ty; yy < 32; yy += 8) {
            // tile[rr][kk] = value of (row r0 + rr, column k0 + kk)
            int64_t r, kk;
            if (kmajor_src) { r = r0 + yy; kk = k0 + tx; } else { r = r0 + tx; kk = k0 + yy; }
            double v = 0.0;
            if (r < rows && kk < k) {
                const int32_t x = kmajor_src ? X[r * ldx + kk] : X[kk * ldx + r];
                v = static_cast<double>(centre(residue_i32(x, M), M));
            }
            if (kmajor_src) tile[yy][tx] = v; else tile[tx][yy] = v;
        }
        __syncthreads();
        for (int yy = ty; yy < 32; yy += 8) {
            const int64_t r = r0 + yy, kk = k0 + tx;
            if (r < rows && kk < k_pad) out[r * k_pad + kk] = tile[yy][tx];
        }
    }
}

}  // namespace

size_t f64_ws_bytes(const Plan& pl, int64_t m, int64_t n) {
    const size_t kp = static_cast<size_t>(pl.info.k_pad);
    return ((8 * static_cast<size_t>(m) * kp + 255) & ~size_t(255)) + 8 * static_cast<size_t>(n) * kp;
}

int run_f64(const Plan& pl, bool transA, bool transB, int64_t m, int64_t n, int64_t k, const int32_t* A,
            int64_t lda, const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, void* ws, cudaStream_t st) {
    const int64_t kp = pl.info.k_pad;
    double* Ad = static_cast<double*>(ws);
    double* Bd = reinterpret_cast<double*>(static_cast<uint8_t*>(ws) + ((8 * static_cast<size_t>(m) * kp + 255) & ~size_t(255)));
    auto enc_grid = [&](int64_t rows) {
        const int64_t t = ((rows + 31) / 32) * ((kp + 31) / 32);
        const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
        return static_cast<int>(t < cap ? t : cap);
    };
    f64_encode_kernel<<<enc_grid(m), 256, 0, st>>>(pl.mp, transA ? 0 : 1, m, k, kp, A, lda, Ad);
    f64_encode_kernel<<<enc_grid(n), 256, 0, st>>>(pl.mp, transB ? 1 : 0, n, k, kp, B, ldb, Bd);
    F64Args a;
    a.A = Ad;
    a.B = Bd;
    a.C = C;
    a.ldc = ldc;
    a.m = m;
    a.n = n;
    a.k_pad = kp;
    a.kb4 = static_cast<int32_t>(pl.info.kb / 4);
    a.p = static_cast<double>(pl.mp.p);
    a.invp = 1.0 / static_cast<double>(pl.mp.p);
    a.up = pl.mp.p;
    a.alpha = pl.mp.alpha;
    a.beta = pl.mp.beta;
    const dim3 grid(static_cast<unsigned>((n + kBN - 1) / kBN), static_cast<unsigned>((m + kBM - 1) / kBM));
    f64_gemm_kernel<<<grid, 128, 0, st>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : FF_ERR_CUDA;
}

}  // namespace ff
