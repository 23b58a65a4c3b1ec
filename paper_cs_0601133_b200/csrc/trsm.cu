// trsm.cu -- ftrsm on the tensor-core fgemm.
//
// PAPER.md Sec. 4: the triangular solve with a matrix right-hand side
// ("B <- U^{-1} B", l.346-356) by the block recursive Algorithm 1
// (l.366-384): X2 := trsm(A3, B2); B1 := B1 - A2 X2; X1 := trsm(A1, B1), so
// that almost all the work is matrix multiplication (Lemma 4.1, l.388-394:
// trsm costs 1/2 of a multiplication of the same size with omega = 3).
//
// B200 design:
//   * every update B1 <- B1 - A2 X2 is one ff_gemm (alpha = p-1, beta = 1):
//     exact int8 tensor-core products with the modular reduction fused into the
//     epilogue.  The paper's cascades (t_del: solve small blocks over Z without
//     reductions; t_update: accumulate several updates over Z) exist to amortise
//     reductions on a CPU; here the reduction is free in the GEMM epilogue, so
//     every update is reduced and no threshold is needed.
//   * the terminal case (the paper's t_del blocks solved by BLAS dtrsm) is
//     replaced by inverting each nb x nb diagonal block once (exact over the
//     field: no stability issue) with a small kernel, so the leaf solve
//     X_d = D^{-1} B_d is a GEMM on the tensor cores too.
//   * op(A) with transA = 'T' and side = 'R' are handled by the GEMM's own
//     transpose flags on the blocks; nothing is copied or transposed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "internal.h"
#include "modp.cuh"

namespace ff {

namespace {

constexpr int kNb = 64;             // diagonal block size inverted by trsm_diag_inv_kernel
constexpr int kLeaf = 512;          // leaf size of the recursion: inverses doubled 64 -> 128 -> 256 -> 512

struct InvArgs {
    const int32_t* A;
    int64_t lda;
    int64_t d;                      // dimension of A
    int32_t upper;                  // A's referenced triangle (not op(A)'s)
    int32_t unit;
    uint32_t p;
    unsigned long long mu64;        // floor(2^64 / p)
    int32_t* W;                     // out: [nblk][kNb][kNb] inverses of the diagonal blocks of A
};

__device__ uint32_t inv32(uint32_t a, uint32_t p) {        // a^-1 mod p, extended Euclid in 32 bits
    int32_t r0 = static_cast<int32_t>(p), r1 = static_cast<int32_t>(a), s0 = 0, s1 = 1;
    while (r1 != 0) {
        const int32_t q = r0 / r1, t = r0 - q * r1, u = s0 - q * s1;
        r0 = r1; r1 = t; s0 = s1; s1 = u;
    }
    return static_cast<uint32_t>(s0 < 0 ? s0 + static_cast<int32_t>(p) : s0);
}

constexpr int kInvThreads = 1024;
constexpr int kInvSmem = (2 * kNb * kNb + kNb) * 4;

// One CTA (32 x 32 threads) per diagonal block D (db x db, db <= kNb):
// W = D^-1 by Gauss-Jordan phases on [D | I] (D and the identity in shared
// memory).  Upper D: for k = db-1 .. 1, rows r < k: E_r -= (D_rk / D_kk) E_k
// (the multipliers use the original D: eliminating columns to the right of k
// never changes column k); then W_k = E_k / D_kk.  Lower D mirrors it.  One
// barrier per phase; the dependent chain per phase is a single product.
// Shoup's constant floor(w 2^32 / p) for w < p < 2^31 from mu64 = floor(2^64 / p)
// ((w mu64) >> 32 is the floor or one less; one 64-bit check makes it exact)
__device__ __forceinline__ uint32_t shoup_mu(uint32_t w, uint32_t p, unsigned long long mu64) {
    const unsigned long long lo = static_cast<unsigned long long>(w) * static_cast<uint32_t>(mu64);
    const unsigned long long hi = static_cast<unsigned long long>(w) * static_cast<uint32_t>(mu64 >> 32);
    unsigned long long c = hi + (lo >> 32);
    if ((c + 1) * p <= (static_cast<unsigned long long>(w) << 32)) ++c;
    return static_cast<uint32_t>(c);
}

__global__ void __launch_bounds__(kInvThreads) trsm_diag_inv_kernel(InvArgs a) {
    extern __shared__ uint32_t sm[];
    uint32_t* D = sm;                    // [kNb][kNb]
    uint32_t* E = sm + kNb * kNb;        // [kNb][kNb]
    uint32_t* dinv = E + kNb * kNb;      // [kNb]
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * kNb;
    const int db = static_cast<int>(a.d - r0 < kNb ? a.d - r0 : kNb);
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const uint32_t p = a.p;
    for (int e = tid; e < kNb * kNb; e += kInvThreads) {
        const int i = e / kNb, j = e % kNb;
        uint32_t v = 0;
        if (i < db && j < db) {
            const bool inside = a.upper ? (j >= i) : (j <= i);
            if (inside) {
                v = residue_i32_64(a.A[(r0 + i) * a.lda + r0 + j], a.mu64, p);
            }
        }
        D[e] = v;
        E[e] = (i == j && i < db) ? 1u : 0u;
    }
    __syncthreads();
    for (int i = tid; i < db; i += kInvThreads) dinv[i] = a.unit ? 1u : inv32(D[i * kNb + i], p);
    __syncthreads();
    if (a.upper) {
        for (int k = db - 1; k >= 1; --k) {
            for (int r = ty; r < k; r += 32) {
                const uint32_t d = D[r * kNb + k];
                if (d == 0u) continue;
                const uint32_t mlt = residue_u64(static_cast<unsigned long long>(d) * dinv[k], a.mu64, p);
                const uint32_t mlt_sh = shoup_mu(mlt, p, a.mu64);     // per-row Shoup constant
                for (int c = k + tx; c < db; c += 32) {
                    const uint32_t t = mulmod_shoup(E[k * kNb + c], mlt, mlt_sh, p);
                    const uint32_t x = E[r * kNb + c];
                    E[r * kNb + c] = x >= t ? x - t : x + p - t;
                }
            }
            __syncthreads();
        }
    } else {
        for (int k = 0; k + 1 < db; ++k) {
            for (int r = k + 1 + ty; r < db; r += 32) {
                const uint32_t d = D[r * kNb + k];
                if (d == 0u) continue;
                const uint32_t mlt = residue_u64(static_cast<unsigned long long>(d) * dinv[k], a.mu64, p);
                const uint32_t mlt_sh = shoup_mu(mlt, p, a.mu64);
                for (int c = tx; c <= k; c += 32) {
                    const uint32_t t = mulmod_shoup(E[k * kNb + c], mlt, mlt_sh, p);
                    const uint32_t x = E[r * kNb + c];
                    E[r * kNb + c] = x >= t ? x - t : x + p - t;
                }
            }
            __syncthreads();
        }
    }
    int32_t* W = a.W + static_cast<int64_t>(blockIdx.x) * kNb * kNb;
    for (int e = tid; e < kNb * kNb; e += kInvThreads) {
        const int i = e / kNb;
        W[e] = (i < db) ? static_cast<int32_t>(residue_u64(static_cast<unsigned long long>(E[e]) * dinv[i], a.mu64, p)) : 0;
    }
}

// ---- doubling the inverted diagonal blocks ----------------
// inv([D1 D2; 0 D3]) = [W1, -W1 D2 W3; 0, W3] (upper; lower: [W1 0; -W3 D2 W1, W3]),
// from the inverses of the halves: two h x h products mod p per block, on the
// CUDA cores (batched over the blocks; small next to the solve's GEMMs).

struct MatDesc {
    const int32_t* ptr;
    int64_t bstride;     // elements between consecutive batch entries
    int64_t ld;
    int64_t rows_lim;    // rows/cols beyond these (absolute, for A) read as 0
    int64_t cols_lim;
    int64_t row0_step;   // absolute row offset of batch b = b * row0_step (for the limits)
    int64_t col0_step;
    int32_t reduce;      // 1: reduce raw int32 mod p on load
    unsigned long long mu64;   // floor(2^64 / p) (for reduce)
};

__device__ __forceinline__ uint32_t load_md(const MatDesc& d, int64_t b, int64_t i, int64_t j, uint32_t p) {
    if (b * d.row0_step + i >= d.rows_lim || b * d.col0_step + j >= d.cols_lim) return 0u;
    const int32_t x = d.ptr[b * d.bstride + i * d.ld + j];
    if (!d.reduce) return static_cast<uint32_t>(x);
    return residue_i32_64(x, d.mu64, p);
}

// C[b] = (neg ? -1 : 1) * X[b] Y[b] mod p, all n x n (zero outside the limits);
// 32 x 32 output tile per CTA, 256 threads, 4 outputs each.
__global__ void __launch_bounds__(256) batched_modmul_kernel(MatDesc X, MatDesc Y, int32_t* C, int64_t c_bstride,
                                                             int64_t ldc, int n, int neg, uint32_t p,
                                                             unsigned long long mu64) {
    __shared__ uint32_t xs[32][33], ys[32][33];
    const int64_t b = blockIdx.z;
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
    const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    unsigned long long acc[4] = {0, 0, 0, 0};
    for (int k0 = 0; k0 < n; k0 += 32) {
        for (int r = ty; r < 32; r += 8) {
            xs[r][tx] = (i0 + r < n && k0 + tx < n) ? load_md(X, b, i0 + r, k0 + tx, p) : 0u;
            ys[r][tx] = (k0 + r < n && j0 + tx < n) ? load_md(Y, b, k0 + r, j0 + tx, p) : 0u;
        }
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < 32; kk += 2) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int r = ty + 8 * q;
                const unsigned long long s2 = static_cast<unsigned long long>(xs[r][kk]) * ys[kk][tx] +
                                              static_cast<unsigned long long>(xs[r][kk + 1]) * ys[kk + 1][tx];
                acc[q] = residue_u64(acc[q] + s2, mu64, p);     // s2 < 2^63, acc < p
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = i0 + ty + 8 * q, j = j0 + tx;
        if (i < n && j < n) {
            const uint32_t v = static_cast<uint32_t>(acc[q]);
            C[b * c_bstride + static_cast<int64_t>(i) * ldc + j] = static_cast<int32_t>(neg && v ? p - v : v);
        }
    }
}

// The same on the warp-level tensor cores for p < 2^16 (as gemm_small.cu):
// residues split into two bytes, four mma.sync m16n8k32 u8 products per 32-wide
// k slice, recombined exactly in 64 bits (n <= kLeaf: each byte product stays
// below n 255^2 < 2^31) and reduced once.  8 warps, one m16n8 tile each.
__device__ __forceinline__ void imma_t(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                       uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void split4_t(uint32_t x, uint32_t y, uint32_t z, uint32_t w, uint32_t& lo, uint32_t& hi) {
    const uint32_t t0 = __byte_perm(x, y, 0x5140), t1 = __byte_perm(z, w, 0x5140);
    lo = __byte_perm(t0, t1, 0x5410);
    hi = __byte_perm(t0, t1, 0x7632);
}
__global__ void __launch_bounds__(256) batched_modmul_tc_kernel(MatDesc X, MatDesc Y, int32_t* C, int64_t c_bstride,
                                                                int64_t ldc, int n, int neg, uint32_t p,
                                                                unsigned long long mu64) {
    __shared__ uint32_t xs[32][36], ys[32][40];
    const int64_t b = blockIdx.z;
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
    const int warp = ty, g = tx >> 2, t = tx & 3;
    const int wm = warp & 1, wn = warp >> 1;                 // 2 x 4 tiles of 16 x 8
    const int i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;
    int P[4][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}, {0, 0, 0, 0}};
    for (int k0 = 0; k0 < n; k0 += 32) {
        for (int r = ty; r < 32; r += 8) {
            xs[r][tx] = (i0 + r < n && k0 + tx < n) ? load_md(X, b, i0 + r, k0 + tx, p) : 0u;
            ys[r][tx] = (k0 + r < n && j0 + tx < n) ? load_md(Y, b, k0 + r, j0 + tx, p) : 0u;
        }
        __syncthreads();
        uint32_t alo[4], ahi[4], blo[2], bhi[2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = wm * 16 + g + ((q & 1) ? 8 : 0), k = ((q & 2) ? 16 : 0) + 4 * t;
            const uint4 v = *reinterpret_cast<const uint4*>(&xs[r][k]);
            split4_t(v.x, v.y, v.z, v.w, alo[q], ahi[q]);
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int k = (q ? 16 : 0) + 4 * t, c = wn * 8 + g;
            split4_t(ys[k][c], ys[k + 1][c], ys[k + 2][c], ys[k + 3][c], blo[q], bhi[q]);
        }
        imma_t(P[0], alo[0], alo[1], alo[2], alo[3], blo[0], blo[1]);
        imma_t(P[1], alo[0], alo[1], alo[2], alo[3], bhi[0], bhi[1]);
        imma_t(P[2], ahi[0], ahi[1], ahi[2], ahi[3], blo[0], blo[1]);
        imma_t(P[3], ahi[0], ahi[1], ahi[2], ahi[3], bhi[0], bhi[1]);
        __syncthreads();
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int i = i0 + wm * 16 + g + ((e & 2) ? 8 : 0), j = j0 + wn * 8 + 2 * t + (e & 1);
        if (i < n && j < n) {
            const unsigned long long S =
                static_cast<unsigned long long>(static_cast<uint32_t>(P[0][e])) +
                (static_cast<unsigned long long>(static_cast<uint32_t>(P[1][e]) + static_cast<uint32_t>(P[2][e])) << 8) +
                (static_cast<unsigned long long>(static_cast<uint32_t>(P[3][e])) << 16);
            const uint32_t v = residue_u64(S, mu64, p);
            C[b * c_bstride + static_cast<int64_t>(i) * ldc + j] = static_cast<int32_t>(neg && v ? p - v : v);
        }
    }
}

// W_s[b] (s x s) <- the diagonal quadrants W_h[2b], W_h[2b+1] and a zero quadrant
// (the off-diagonal one is written by the second product).
__global__ void assemble_kernel(const int32_t* Wh, int64_t nblk_h, int32_t* Ws, int s, int upper) {
    const int h = s / 2;
    const int64_t b = blockIdx.y;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < static_cast<int64_t>(s) * s;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int i = static_cast<int>(e / s), j = static_cast<int>(e % s);
        const bool top = i < h, left = j < h;
        int32_t v = 0;
        if (top == left) {
            const int64_t hb = 2 * b + (top ? 0 : 1);
            if (hb < nblk_h) v = Wh[hb * h * h + static_cast<int64_t>(top ? i : i - h) * h + (left ? j : j - h)];
        } else if ((upper && top) || (!upper && !top)) {
            continue;                       // off-diagonal quadrant: written by the product
        }
        Ws[b * s * s + e] = v;
    }
}

struct Ctx {
    uint32_t p;
    bool left, t_upper, tA;
    const int32_t* A;
    int64_t lda;
    int32_t* B;
    int64_t ldb;
    int64_t m, n;
    const int32_t* W;               // inverted kLeaf x kLeaf diagonal blocks (of A)
    void* gws;                      // GEMM workspace
    const ff_opts* opts;
    cudaStream_t st;
};

// GEMM on device pointers: C <- (alpha op(X) op(Y) + beta C) mod p.
int gemm(const Ctx& c, char tX, char tY, int64_t m, int64_t n, int64_t k, uint32_t alpha, const int32_t* X,
         int64_t ldx, const int32_t* Y, int64_t ldy, uint32_t beta, int32_t* C, int64_t ldc) {
    if (m == 0 || n == 0 || k == 0) return 0;
    ff_opts o;
    std::memset(&o, 0, sizeof(o));
    if (c.opts) o = *c.opts;
    Plan pl;
    int e = make_plan(c.p, k, &o, &pl);
    if (e) return e;
    set_scalars(&pl, alpha, beta);
    return gemm_dev(pl, tX, tY, m, n, k, X, ldx, Y, ldy, C, ldc, c.gws, c.st);
}

// Block [r0, r1) x [c0, c1) of op(A) as a GEMM operand (pointer, trans flag).
void opA_block(const Ctx& c, int64_t r0, int64_t c0, const int32_t** ptr, char* tr) {
    if (!c.tA) { *ptr = c.A + r0 * c.lda + c0; *tr = 'N'; }
    else { *ptr = c.A + c0 * c.lda + r0; *tr = 'T'; }
}

// Leaf: the diagonal block [i0, i1) (i0 a multiple of kLeaf): X_d = D^{-1} B_d
// (side L) or X_d = B_d D^{-1} (side R), written over B_d.  The output may
// alias the B_d operand here: gemm_dev encodes both operands into limb planes
// before the GEMM kernel runs, and with beta = 0 that kernel reads only the
// planes (never C), so the in-place write is ordered after every read.
int leaf(const Ctx& c, int64_t i0, int64_t i1) {
    const int64_t db = i1 - i0;
    const int32_t* Wb = c.W + (i0 / kLeaf) * kLeaf * kLeaf;   // inverse of A's block; op(A)'s is its transpose if tA
    const char tw = c.tA ? 'T' : 'N';
    if (c.left)
        return gemm(c, tw, 'N', db, c.n, db, 1, Wb, kLeaf, c.B + i0 * c.ldb, c.ldb, 0, c.B + i0 * c.ldb, c.ldb);
    return gemm(c, 'N', tw, c.m, db, db, 1, c.B + i0, c.ldb, Wb, kLeaf, 0, c.B + i0, c.ldb);
}

// Algorithm 1 on the index range [i0, i1) of op(A) (split at a multiple of kLeaf).
int solve(const Ctx& c, int64_t i0, int64_t i1) {
    if (i1 - i0 <= kLeaf) return leaf(c, i0, i1);
    const int64_t nblk = (i1 - i0 + kLeaf - 1) / kLeaf;
    const int64_t mid = i0 + ((nblk + 1) / 2) * kLeaf;
    const uint32_t neg1 = c.p - 1;
    const int32_t* Ab;
    char ta;
    int e;
    if (c.left) {
        if (c.t_upper) {          // [A1 A2; 0 A3] [X1; X2] = [B1; B2]
            if ((e = solve(c, mid, i1))) return e;                                  // X2 := trsm(A3, B2)
            opA_block(c, i0, mid, &Ab, &ta);                                        // B1 := B1 - A2 X2
            if ((e = gemm(c, ta, 'N', mid - i0, c.n, i1 - mid, neg1, Ab, c.lda, c.B + mid * c.ldb, c.ldb, 1,
                          c.B + i0 * c.ldb, c.ldb)))
                return e;
            return solve(c, i0, mid);                                               // X1 := trsm(A1, B1)
        }
        if ((e = solve(c, i0, mid))) return e;                                      // lower: X1 first
        opA_block(c, mid, i0, &Ab, &ta);                                            // B2 := B2 - A21 X1
        if ((e = gemm(c, ta, 'N', i1 - mid, c.n, mid - i0, neg1, Ab, c.lda, c.B + i0 * c.ldb, c.ldb, 1,
                      c.B + mid * c.ldb, c.ldb)))
            return e;
        return solve(c, mid, i1);
    }
    // side R: X op(A) = B, column blocks
    if (c.t_upper) {              // [X1 X2] [A1 A2; 0 A3] = [B1 B2]
        if ((e = solve(c, i0, mid))) return e;                                      // X1 A1 = B1
        opA_block(c, i0, mid, &Ab, &ta);                                            // B2 := B2 - X1 A2
        if ((e = gemm(c, 'N', ta, c.m, i1 - mid, mid - i0, neg1, c.B + i0, c.ldb, Ab, c.lda, 1, c.B + mid,
                      c.ldb)))
            return e;
        return solve(c, mid, i1);
    }
    if ((e = solve(c, mid, i1))) return e;                                          // lower: X2 first
    opA_block(c, mid, i0, &Ab, &ta);                                                // B1 := B1 - X2 A21
    if ((e = gemm(c, 'N', ta, c.m, mid - i0, i1 - mid, neg1, c.B + mid, c.ldb, Ab, c.lda, 1, c.B + i0, c.ldb)))
        return e;
    return solve(c, i0, mid);
}

bool is_side_l(char s) { return s == 'L' || s == 'l'; }
bool is_side_r(char s) { return s == 'R' || s == 'r'; }

int validate_trsm(uint32_t p, char side, char uplo, char transA, char diag, int64_t m, int64_t n, const void* A,
                  int64_t lda, const void* B, int64_t ldb) {
    if (p < 2 || p >= (1u << 31)) return -1;
    if (!is_side_l(side) && !is_side_r(side)) return -2;
    if (!(uplo == 'U' || uplo == 'u' || uplo == 'L' || uplo == 'l')) return -3;
    if (!(transA == 'N' || transA == 'n' || transA == 'T' || transA == 't')) return -4;
    if (!(diag == 'N' || diag == 'n' || diag == 'U' || diag == 'u')) return -5;
    if (m < 0) return -6;
    if (n < 0) return -7;
    const int64_t d = is_side_l(side) ? m : n;
    if (!A && d > 0) return -9;
    if (lda < (d > 1 ? d : 1)) return -10;
    if (!B && m > 0 && n > 0) return -11;
    if (ldb < (n > 1 ? n : 1)) return -12;
    return 0;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct TrsmWs {
    size_t w_bytes, t_bytes, g_bytes;
    size_t lvl_off[8];              // offset of the inverse blocks of size kNb << l
    int nlvl;
    size_t total() const { return w_bytes + t_bytes + g_bytes; }
};

int trsm_ws(uint32_t p, bool left, int64_t m, int64_t n, const ff_opts* opts, TrsmWs* out) {
    const int64_t d = left ? m : n;
    size_t off = 0;
    out->nlvl = 0;
    for (int s = kNb; s <= kLeaf; s *= 2) {
        out->lvl_off[out->nlvl++] = off;
        off += align256(static_cast<size_t>((d + s - 1) / s) * s * s * 4);
    }
    out->w_bytes = off;
    // product temporaries of the doubling (h x h per block at the last level);
    // the leaves write in place (see leaf())
    out->t_bytes = align256(static_cast<size_t>((d + kLeaf - 1) / kLeaf) * (kLeaf / 2) * (kLeaf / 2) * 4);
    // The largest GEMM: k <= d, operand rows <= d and <= n (L) / m (R); the plan for
    // k = d has the most planes (CRT) and the longest rows.
    // AUTO may pick CRT for short k and limbs for long k (the moduli count
    // grows with k), so bound over the plans at k = d, k = kNb and forced CRT.
    const int64_t M = left ? d : m, N = left ? n : d;
    size_t g = 0;
    const int64_t ks[2] = {d > 0 ? d : 1, std::min<int64_t>(kLeaf, d > 0 ? d : 1)};
    for (int i = 0; i < 2; ++i) {
        Plan pl;
        int e = make_plan(p, ks[i], opts, &pl);
        if (e) return e;
        g = std::max(g, gemm_ws_bytes(pl, M, N));
        ff_opts oc;
        std::memset(&oc, 0, sizeof(oc));
        if (opts) oc = *opts;
        oc.scheme = FF_SCHEME_CRT;
        oc.kb_override = 0;
        if (make_plan(p, ks[i], &oc, &pl) == 0) {
            // planes of the CRT plan at k = d with the row length of k = d
            Plan pd;
            if (make_plan(p, ks[0], &oc, &pd) == 0) g = std::max(g, gemm_ws_bytes(pd, M, N));
        }
    }
    out->g_bytes = align256(g);
    return 0;
}

}  // namespace

}  // namespace ff

using namespace ff;

extern "C" {

size_t ff_trsm_workspace_size(uint32_t p, char side, int64_t m, int64_t n, const ff_opts* opts) {
    if (p < 2 || p >= (1u << 31) || m < 0 || n < 0 || (!is_side_l(side) && !is_side_r(side))) return 0;
    TrsmWs w;
    if (trsm_ws(p, is_side_l(side), m, n, opts, &w)) return 0;
    return w.total();
}

int ff_trsm_ex(uint32_t p, char side, char uplo, char transA, char diag, int64_t m, int64_t n, uint32_t alpha,
               const int32_t* A, int64_t lda, int32_t* B, int64_t ldb, const ff_opts* opts, void* workspace,
               size_t workspace_bytes, void* stream) {
    int e = validate_trsm(p, side, uplo, transA, diag, m, n, A, lda, B, ldb);
    if (e) return e;
    if (m == 0 || n == 0) return 0;
    if ((e = check_device())) return e;
    const bool left = is_side_l(side);
    TrsmWs w;
    if ((e = trsm_ws(p, left, m, n, opts, &w))) return e;
    if (!workspace || workspace_bytes < w.total() || (reinterpret_cast<uintptr_t>(workspace) & 255)) return -15;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Plan pl0;
    if ((e = make_plan(p, 1, opts, &pl0))) return e;
    // B <- alpha B mod p; alpha = 0 gives X = 0.  Skipped for alpha = 1: every
    // read of B below reduces it (the encoders, and the beta = 1 epilogue).
    set_scalars(&pl0, 1, alpha);
    if (pl0.mp.beta != 1 % p && launch_scale_c(pl0.mp, m, n, B, ldb, st) != cudaSuccess) return FF_ERR_CUDA;
    if (pl0.mp.beta == 0) return 0;
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    Ctx c;
    c.p = p;
    c.left = left;
    c.tA = (transA == 'T' || transA == 't');
    const bool upper = (uplo == 'U' || uplo == 'u');
    c.t_upper = upper != c.tA;
    c.A = A;
    c.lda = lda;
    c.B = B;
    c.ldb = ldb;
    c.m = m;
    c.n = n;
    c.W = reinterpret_cast<int32_t*>(ws + w.lvl_off[w.nlvl - 1]);
    c.gws = ws + w.w_bytes + w.t_bytes;
    c.opts = opts;
    c.st = st;
    // invert the diagonal blocks of A (one CTA each)
    const int64_t d = left ? m : n;
    InvArgs ia;
    ia.A = A;
    ia.lda = lda;
    ia.d = d;
    ia.upper = upper ? 1 : 0;
    ia.unit = (diag == 'U' || diag == 'u') ? 1 : 0;
    ia.p = p;
    ia.mu64 = static_cast<unsigned long long>((static_cast<unsigned __int128>(1) << 64) / p);
    ia.W = reinterpret_cast<int32_t*>(ws + w.lvl_off[0]);
    const size_t smem = kInvSmem;
    if (set_smem_attr(reinterpret_cast<const void*>(trsm_diag_inv_kernel), (int)smem) != cudaSuccess)
        return FF_ERR_CUDA;
    trsm_diag_inv_kernel<<<static_cast<unsigned>((d + kNb - 1) / kNb), kInvThreads, smem, st>>>(ia);
    if (cudaGetLastError() != cudaSuccess) return FF_ERR_CUDA;
    // double the inverted blocks up to kLeaf: W_s = [W1, X; 0, W3] (upper)
    int32_t* T = reinterpret_cast<int32_t*>(ws + w.w_bytes);
    for (int l = 1; l < w.nlvl; ++l) {
        const int sz = kNb << l, h = sz / 2;
        const int64_t nb_s = (d + sz - 1) / sz, nb_h = (d + h - 1) / h;
        const int32_t* Wh = reinterpret_cast<const int32_t*>(ws + w.lvl_off[l - 1]);
        int32_t* Ws = reinterpret_cast<int32_t*>(ws + w.lvl_off[l]);
        assemble_kernel<<<dim3(64, static_cast<unsigned>(nb_s)), 256, 0, st>>>(Wh, nb_h, Ws, sz, upper ? 1 : 0);
        const int64_t big = INT64_MAX / 4;
        MatDesc W1 = {Wh, 2LL * h * h, h, big, big, 0, 0, 0, ia.mu64};
        MatDesc W3 = {Wh + static_cast<int64_t>(h) * h, 2LL * h * h, h, (nb_h - 1) * h, big, sz, 0, 0, ia.mu64};
        MatDesc Tm = {T, static_cast<int64_t>(h) * h, h, big, big, 0, 0, 0, ia.mu64};
        const dim3 g(h / 32, h / 32, static_cast<unsigned>(nb_s));
        auto modmul = [&](dim3 gg, cudaStream_t ss, MatDesc X, MatDesc Y, int32_t* Cc, int64_t cb, int64_t ldcc,
                          int nn, int ng, uint32_t pp, unsigned long long mu) {
            if (pp < 65536u) batched_modmul_tc_kernel<<<gg, 256, 0, ss>>>(X, Y, Cc, cb, ldcc, nn, ng, pp, mu);
            else batched_modmul_kernel<<<gg, 256, 0, ss>>>(X, Y, Cc, cb, ldcc, nn, ng, pp, mu);
        };
        if (upper) {
            MatDesc A12 = {A + h, sz * lda + sz, lda, d, d - h, sz, sz, 1, ia.mu64};      // A[r0 + i][r0 + h + j]
            modmul(g, st, W1, A12, T, static_cast<int64_t>(h) * h, h, h, 0, p, ia.mu64);
            modmul(g, st, Tm, W3, Ws + h, static_cast<int64_t>(sz) * sz, sz, h, 1, p,
                                                     ia.mu64);
        } else {
            MatDesc A21 = {A + h * lda, sz * lda + sz, lda, d - h, d, sz, sz, 1, ia.mu64};  // A[r0 + h + i][r0 + j]
            modmul(g, st, A21, W1, T, static_cast<int64_t>(h) * h, h, h, 0, p, ia.mu64);
            modmul(g, st, W3, Tm, Ws + static_cast<int64_t>(h) * sz,
                                                     static_cast<int64_t>(sz) * sz, sz, h, 1, p, ia.mu64);
        }
        if (cudaGetLastError() != cudaSuccess) return FF_ERR_CUDA;
    }
    return solve(c, 0, d);
}

int ff_trsm(uint32_t p, char side, char uplo, char transA, char diag, int64_t m, int64_t n, uint32_t alpha,
            const int32_t* A, int64_t lda, int32_t* B, int64_t ldb) {
    int e = validate_trsm(p, side, uplo, transA, diag, m, n, A, lda, B, ldb);
    if (e) return e;
    if (m == 0 || n == 0) return 0;
    const size_t need = ff_trsm_workspace_size(p, side, m, n, nullptr);
    if (need == 0) return FF_ERR_INTERNAL;
    void* ws = nullptr;
    if (cudaMalloc(&ws, need) != cudaSuccess) {
        cudaGetLastError();
        return FF_ERR_NOMEM;
    }
    e = ff_trsm_ex(p, side, uplo, transA, diag, m, n, alpha, A, lda, B, ldb, nullptr, ws, need, nullptr);
    cudaFree(ws);   // synchronises with the legacy stream's work
    return e;
}

}  // extern "C"
