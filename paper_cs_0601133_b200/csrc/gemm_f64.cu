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

// int32 -> centred residue as double, K-major [rows_out][k_pad] (zero padded:
// columns k..k_pad-1 and rows rows..rows_out-1).
// kmajor_src: X[r * ldx + kk]; else X[kk * ldx + r] (transposed through SMEM).
__global__ void __launch_bounds__(256) f64_encode_kernel(ModP M, int kmajor_src, int64_t rows, int64_t rows_out,
                                                         int64_t k, int64_t k_pad, const int32_t* __restrict__ X,
                                                         int64_t ldx, double* __restrict__ out) {
    __shared__ double tile[32][33];
    const int64_t tiles_r = (rows_out + 31) / 32, tiles_k = (k_pad + 31) / 32;
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
            if (r < rows_out && kk < k_pad) out[r * k_pad + kk] = tile[yy][tx];
        }
    }
}

// ---------------------------------------------------------------- delayed Winograd (Sec. 3.2.3)
//
// l recursive levels of Winograd's algorithm over Z in doubles, with no
// modular reduction anywhere -- the pre-additions S1..S4, T1..T4 are NOT
// reduced, the seven products are exact dot products, the post-additions
// U1..U7 are exact sums -- which Theorem 3.1 / Corollary 3.4 (PAPER.md
// l.278-312) allow while floor(k / 2^l) v_l^2 < 2^53 (the planner's
// k_winograd).  The schedule is Appendix A.2's (l.935-951): the intermediates
// are exactly the ones the theorem bounds.  One reduction at the very end.

// O[i][j] = (E ? E[i][j] : 0) + sum_{t < K} X[i][t] Y[j][t]  for i < m, j < n, in
// doubles, no reduction (a leaf product of the recursion, or the peeled
// rank-(k mod 2^l) update).  X, Y, E, O row-major with their own leading
// dimensions (any alignment: 8-byte cp.async, zero fill past m, n, K).
struct F64Raw {
    const double* X;
    const double* Y;
    const double* E;
    double* O;
    int64_t ldx, ldy, lde, ldo;
    int64_t m, n, K;
};

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}

__device__ __forceinline__ void cp_async16n(void* smem, const void* gmem, int bytes) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(bytes) : "memory");
}

// kV16: X, Y 16-byte aligned with even leading dimensions (16-byte chunks of two
// doubles, a ragged last chunk zero-filled); else 8-byte chunks.
template <bool kV16>
__global__ void __launch_bounds__(128) f64_raw_gemm_kernel(F64Raw a) {
    __shared__ __align__(16) double As[kStages][kBM][kPitch];
    __shared__ __align__(16) double Bs[kStages][kBN][kPitch];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int wm = warp >> 1, wn = warp & 1;
    const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kBM, n0 = static_cast<int64_t>(blockIdx.x) * kBN;
    const int ktiles = static_cast<int>((a.K + kBK - 1) / kBK);
    auto load = [&](int kt, int stage) {
        if (kV16) {
            for (int c = threadIdx.x; c < kBM * (kBK / 2); c += 128) {
                const int r = c / (kBK / 2), kc = 2 * (c % (kBK / 2));
                const int64_t kk = static_cast<int64_t>(kt) * kBK + kc;
                const int left = kk < a.K ? (a.K - kk >= 2 ? 16 : 8) : 0;
                const int ba = (m0 + r) < a.m ? left : 0, bb = (n0 + r) < a.n ? left : 0;
                cp_async16n(&As[stage][r][kc], a.X + (ba ? (m0 + r) * a.ldx + kk : 0), ba);
                cp_async16n(&Bs[stage][r][kc], a.Y + (bb ? (n0 + r) * a.ldy + kk : 0), bb);
            }
        } else {
            for (int c = threadIdx.x; c < kBM * kBK; c += 128) {
                const int r = c / kBK, kc = c % kBK;
                const int64_t kk = static_cast<int64_t>(kt) * kBK + kc;
                const bool inA = (m0 + r) < a.m && kk < a.K;
                const bool inB = (n0 + r) < a.n && kk < a.K;
                cp_async8(&As[stage][r][kc], a.X + (inA ? (m0 + r) * a.ldx + kk : 0), inA);
                cp_async8(&Bs[stage][r][kc], a.Y + (inB ? (n0 + r) * a.ldy + kk : 0), inB);
            }
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
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int64_t r = m0 + wm * 32 + i * 8 + (lane >> 2);
                const int64_t c = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
                if (r >= a.m || c >= a.n) continue;
                double v = acc[i][j][h];
                if (a.E) v += a.E[r * a.lde + c];
                a.O[r * a.ldo + c] = v;
            }
}

// O = X + s Y elementwise (s = +1 / -1) over rows x cols, all with their own
// leading dimensions: one pre- or post-addition of the schedule, exact in
// doubles because every value involved is below Theorem 3.1's bound.
__global__ void __launch_bounds__(256) f64_add_kernel(int64_t rows, int64_t cols, const double* __restrict__ X,
                                                      int64_t ldx, const double* __restrict__ Y, int64_t ldy,
                                                      double s, double* __restrict__ O, int64_t ldo) {
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
        for (int64_t c = blockIdx.x * 256 + threadIdx.x; c < cols; c += static_cast<int64_t>(gridDim.x) * 256)
            O[r * ldo + c] = X[r * ldx + c] + s * Y[r * ldy + c];
}

// The only reduction: C = (alpha (X mod p) + beta C) mod p, X an exact integer
// in a double (|X| < 2^53), in 64-bit integers.
__global__ void __launch_bounds__(256) f64_final_kernel(int64_t m, int64_t n, const double* __restrict__ X,
                                                        int64_t ldx, uint32_t p, uint32_t alpha, uint32_t beta,
                                                        int32_t* __restrict__ C, int64_t ldc) {
    for (int64_t r = blockIdx.y; r < m; r += gridDim.y)
        for (int64_t c = blockIdx.x * 256 + threadIdx.x; c < n; c += static_cast<int64_t>(gridDim.x) * 256) {
            int64_t v = static_cast<int64_t>(X[r * ldx + c]) % static_cast<int64_t>(p);
            if (v < 0) v += p;
            uint64_t o = static_cast<uint64_t>(v) * alpha % p;
            int32_t* cp = C + r * ldc + c;
            if (beta) {
                int64_t cin = static_cast<int64_t>(*cp) % static_cast<int64_t>(p);
                if (cin < 0) cin += p;
                o = (o + static_cast<uint64_t>(cin) * beta) % p;
            }
            *cp = static_cast<int32_t>(o);
        }
}

struct DMat {
    double* p;
    int64_t ld;
    DMat at(int64_t r, int64_t c) const { return {p + r * ld + c, ld}; }
};

dim3 grid2d(int64_t rows, int64_t cols) {
    int64_t gx = (cols + 255) / 256;
    if (gx > 64) gx = 64;
    if (gx < 1) gx = 1;
    int64_t gy = rows < 4096 ? rows : 4096;
    if (gy < 1) gy = 1;
    return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
}

int f64_add(int64_t rows, int64_t cols, DMat X, DMat Y, double s, DMat O, cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return 0;
    note_launch();
    f64_add_kernel<<<grid2d(rows, cols), 256, 0, st>>>(rows, cols, X.p, X.ld, Y.p, Y.ld, s, O.p, O.ld);
    return cudaGetLastError() == cudaSuccess ? 0 : FF_ERR_CUDA;
}

// O = [E +] X Y^T (m x n, inner K)
int f64_raw(int64_t m, int64_t n, int64_t K, DMat X, DMat Y, const DMat* E, DMat O, cudaStream_t st) {
    if (m <= 0 || n <= 0) return 0;
    F64Raw a;
    a.X = X.p; a.ldx = X.ld;
    a.Y = Y.p; a.ldy = Y.ld;
    a.E = E ? E->p : nullptr; a.lde = E ? E->ld : 0;
    a.O = O.p; a.ldo = O.ld;
    a.m = m; a.n = n; a.K = K;
    const dim3 grid(static_cast<unsigned>((n + kBN - 1) / kBN), static_cast<unsigned>((m + kBM - 1) / kBM));
    const bool v16 = (X.ld % 2 == 0) && (Y.ld % 2 == 0) && (reinterpret_cast<uintptr_t>(X.p) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(Y.p) % 16 == 0);
    note_launch();
    prof_gemm_begin(st);
    if (v16) f64_raw_gemm_kernel<true><<<grid, 128, 0, st>>>(a);
    else f64_raw_gemm_kernel<false><<<grid, 128, 0, st>>>(a);
    prof_gemm_end(st);
    return cudaGetLastError() == cudaSuccess ? 0 : FF_ERR_CUDA;
}

int64_t even(int64_t x) { return (x + 1) & ~int64_t(1); }

// Doubles of scratch the recursion needs below level j (sizes of level j's operands).
size_t wino_scratch(int j, int64_t m, int64_t n, int64_t k) {
    if (j == 0) return 0;
    const int64_t hm = m / 2, hn = n / 2, hk = k / 2;
    const size_t here = 4 * static_cast<size_t>(hm) * even(hk) + 4 * static_cast<size_t>(hn) * even(hk) +
                        3 * static_cast<size_t>(hm) * even(hn);
    return here + wino_scratch(j - 1, hm, hn, hk);
}

// O (m x n) = X (m x k) Y^T (Y: n x k, the K-major form of the right operand)
// with j recursive levels; m, n, k divisible by 2^j.  `ws` holds wino_scratch(j)
// doubles.  Appendix A.2's schedule with B = Y^T: B11 = Y11^T, B12 = Y21^T,
// B21 = Y12^T, B22 = Y22^T.
int wino_rec(int j, int64_t m, int64_t n, int64_t k, DMat X, DMat Y, DMat O, double* ws, cudaStream_t st) {
    if (j == 0) return f64_raw(m, n, k, X, Y, nullptr, O, st);
    const int64_t hm = m / 2, hn = n / 2, hk = k / 2;
    const int64_t ldk = even(hk), ldn = even(hn);
    DMat S[4], T[4], R[3];
    double* w = ws;
    for (int i = 0; i < 4; ++i) { S[i] = {w, ldk}; w += hm * ldk; }
    for (int i = 0; i < 4; ++i) { T[i] = {w, ldk}; w += hn * ldk; }
    for (int i = 0; i < 3; ++i) { R[i] = {w, ldn}; w += hm * ldn; }
    double* sub = w;
    const DMat X11 = X.at(0, 0), X12 = X.at(0, hk), X21 = X.at(hm, 0), X22 = X.at(hm, hk);
    const DMat B11 = Y.at(0, 0), B12 = Y.at(hn, 0), B21 = Y.at(0, hk), B22 = Y.at(hn, hk);   // K-major blocks
    const DMat O11 = O.at(0, 0), O12 = O.at(0, hn), O21 = O.at(hm, 0), O22 = O.at(hm, hn);
    int e;
    // pre-additions, unreduced
    if ((e = f64_add(hm, hk, X21, X22, +1.0, S[0], st))) return e;    // S1 = A21 + A22
    if ((e = f64_add(hm, hk, S[0], X11, -1.0, S[1], st))) return e;   // S2 = S1 - A11
    if ((e = f64_add(hm, hk, X11, X21, -1.0, S[2], st))) return e;    // S3 = A11 - A21
    if ((e = f64_add(hm, hk, X12, S[1], -1.0, S[3], st))) return e;   // S4 = A12 - S2
    if ((e = f64_add(hn, hk, B12, B11, -1.0, T[0], st))) return e;    // T1 = B12 - B11
    if ((e = f64_add(hn, hk, B22, T[0], -1.0, T[1], st))) return e;   // T2 = B22 - T1
    if ((e = f64_add(hn, hk, B22, B12, -1.0, T[2], st))) return e;    // T3 = B22 - B12
    if ((e = f64_add(hn, hk, T[1], B21, -1.0, T[3], st))) return e;   // T4 = T2 - B21
    // products and post-additions (U1..U7 of A.2), three temporaries
    if ((e = wino_rec(j - 1, hm, hn, hk, X11, B11, R[0], sub, st))) return e;      // R0 = P1 = A11 B11
    if ((e = wino_rec(j - 1, hm, hn, hk, X12, B21, O11, sub, st))) return e;       // O11 = P2 = A12 B21
    if ((e = f64_add(hm, hn, O11, R[0], +1.0, O11, st))) return e;                 // C11 = U1 = P1 + P2
    if ((e = wino_rec(j - 1, hm, hn, hk, S[1], T[1], R[1], sub, st))) return e;    // R1 = P6 = S2 T2
    if ((e = f64_add(hm, hn, R[0], R[1], +1.0, R[1], st))) return e;               // R1 = U2 = P1 + P6
    if ((e = wino_rec(j - 1, hm, hn, hk, S[2], T[2], R[0], sub, st))) return e;    // R0 = P7 = S3 T3
    if ((e = f64_add(hm, hn, R[1], R[0], +1.0, R[0], st))) return e;               // R0 = U3 = U2 + P7
    if ((e = wino_rec(j - 1, hm, hn, hk, S[0], T[0], R[2], sub, st))) return e;    // R2 = P5 = S1 T1
    if ((e = f64_add(hm, hn, R[1], R[2], +1.0, O12, st))) return e;                // O12 = U4 = U2 + P5
    if ((e = f64_add(hm, hn, R[0], R[2], +1.0, O22, st))) return e;                // C22 = U7 = U3 + P5
    if ((e = wino_rec(j - 1, hm, hn, hk, S[3], B22, R[1], sub, st))) return e;    // R1 = P3 = S4 B22
    if ((e = f64_add(hm, hn, O12, R[1], +1.0, O12, st))) return e;                 // C12 = U5 = U4 + P3
    if ((e = wino_rec(j - 1, hm, hn, hk, X22, T[3], R[1], sub, st))) return e;    // R1 = P4 = A22 T4
    return f64_add(hm, hn, R[0], R[1], -1.0, O21, st);                              // C21 = U6 = U3 - P4
}

}  // namespace

size_t f64_ws_bytes(const Plan& pl, int64_t m, int64_t n, int64_t k, int levels) {
    const size_t kp = static_cast<size_t>(pl.info.k_pad);
    if (levels <= 0)
        return ((8 * static_cast<size_t>(m) * kp + 255) & ~size_t(255)) + 8 * static_cast<size_t>(n) * kp;
    const int64_t g = int64_t{1} << levels;
    const int64_t mp = (m + g - 1) / g * g, np = (n + g - 1) / g * g, ke = k / g * g;
    const size_t a = (8 * static_cast<size_t>(mp) * kp + 255) & ~size_t(255);
    const size_t b = (8 * static_cast<size_t>(np) * kp + 255) & ~size_t(255);
    const size_t o = (8 * static_cast<size_t>(mp) * np + 255) & ~size_t(255);
    return a + b + o + 8 * wino_scratch(levels, mp, np, ke);
}

int run_f64(const Plan& pl, int levels, bool transA, bool transB, int64_t m, int64_t n, int64_t k, const int32_t* A,
            int64_t lda, const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, void* ws, cudaStream_t st) {
    const int64_t kp = pl.info.k_pad;
    const int64_t g = int64_t{1} << (levels > 0 ? levels : 0);
    const int64_t mp = (m + g - 1) / g * g, np = (n + g - 1) / g * g;
    uint8_t* w = static_cast<uint8_t*>(ws);
    double* Ad = reinterpret_cast<double*>(w);
    w += (8 * static_cast<size_t>(mp) * kp + 255) & ~size_t(255);
    double* Bd = reinterpret_cast<double*>(w);
    w += (8 * static_cast<size_t>(np) * kp + 255) & ~size_t(255);
    auto enc_grid = [&](int64_t rows) {
        const int64_t t = ((rows + 31) / 32) * ((kp + 31) / 32);
        const int64_t cap = static_cast<int64_t>(num_sms()) * 8;
        return static_cast<int>(t < cap ? t : cap);
    };
    note_launch(2);
    f64_encode_kernel<<<enc_grid(mp), 256, 0, st>>>(pl.mp, transA ? 0 : 1, m, mp, k, kp, A, lda, Ad);
    f64_encode_kernel<<<enc_grid(np), 256, 0, st>>>(pl.mp, transB ? 1 : 0, n, np, k, kp, B, ldb, Bd);
    if (levels > 0) {
        // Winograd on the first ke = 2^l floor(k / 2^l) columns of k, no reduction;
        // the last k - ke columns as one more unreduced product added on top
        // (Appendix A.5's peeling; its values stay below the bound, l.1068-1085).
        const int64_t ke = k / g * g;
        double* O = reinterpret_cast<double*>(w);
        w += (8 * static_cast<size_t>(mp) * np + 255) & ~size_t(255);
        const DMat Xa = {Ad, kp}, Yb = {Bd, kp}, Om = {O, np};
        int e = 0;
        if (ke > 0) {
            if ((e = wino_rec(levels, mp, np, ke, Xa, Yb, Om, reinterpret_cast<double*>(w), st))) return e;
            if (k > ke && (e = f64_raw(mp, np, k - ke, Xa.at(0, ke), Yb.at(0, ke), &Om, Om, st))) return e;
        } else if ((e = f64_raw(mp, np, k, Xa, Yb, nullptr, Om, st))) {
            return e;
        }
        note_launch();
        f64_final_kernel<<<grid2d(m, n), 256, 0, st>>>(m, n, O, np, pl.mp.p, pl.mp.alpha, pl.mp.beta, C, ldc);
        return cudaGetLastError() == cudaSuccess ? 0 : FF_ERR_CUDA;
    }
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
    note_launch();
    prof_gemm_begin(st);
    f64_gemm_kernel<<<grid, 128, 0, st>>>(a);
    prof_gemm_end(st);
    return cudaGetLastError() == cudaSuccess ? 0 : FF_ERR_CUDA;
}

}  // namespace ff
