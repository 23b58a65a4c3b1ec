// lqup.cu -- rank-revealing triangular factorization on the tensor-core fgemm
// (Sec. 5.1, l.575-590), with rank and
// determinant (Sec. 6, l.655-657).
//
// The paper's LQUP (A = L Q U P, after Ibarra-Moran-Hui) recurses on row
// halves and reduces to trsm + fgemm.  On the B200 the same reduction is done
// right-looking by panels of kH rows, because the GPU pays per
// launch and per pivot decision, not per flop:
//   1. panel kernel (one CTA): factor the kH panel rows restricted to a column
//      window [c, c+W) with "first non-zero in the row" pivoting (column swaps),
//      in a workspace copy; it also inverts the panel's L11 (unit lower) and
//      U11 (upper).  If a panel row has no pivot inside the window the window
//      is widened (ultimately to all remaining columns) and the panel redone.
//   2. U of the pivot rows beyond the window: U_rest = L11^-1 A_rest  (fgemm).
//   3. trailing rows: G = X U11^-1 (their L entries, fgemm), Z <- Z - G U12 (fgemm,
//      alpha = p-1, beta = 1) -- the paper's "GT = X via trsm ... Z = Z - GY".
//   4. rows that reduced to zero (rank deficiency) move to the bottom.
// Output, in place: with the row permutation Q (rows Q[0..m) of A) and column
// permutation P (columns P[0..n)),  (QAP)[i][j] = sum_k L[i][k] U[k][j],  L unit
// lower (m x r, stored strictly below the diagonal of the first r columns), U
// upper (r x n, on and above the diagonal of the first r rows); rows >= r hold
// only their L entries (zeros elsewhere).  This is the "PLUQ" arrangement of the
// paper's LQUP (reading R20).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>
#include <cstdio>
#include <cstdlib>

#include "internal.h"
#include "modp.cuh"
#include "ptx.cuh"

namespace ff {

namespace {

constexpr int kH = 128;          // panel rows
constexpr int kThr = 1024;
constexpr int kMaxSwaps = 2 * kH;
constexpr int kSmemBytes = 2 * kH * kH * 4;   // the window + the inverse scratch in shared memory (uint32)

int fail_cuda_now() {
    cudaGetLastError();
    return FF_ERR_CUDA;
}

struct PanelArgs {
    int32_t* A;
    int64_t lda;
    int64_t i0, hr;              // panel rows [i0, i0 + hr)
    int64_t c, W;                // window columns [c, c + W)
    int32_t full;                // 1: the window reaches the last column (zero rows allowed)
    uint32_t p;
    double dp, invp;             // p, fl(1/p)
    unsigned long long mu64;     // floor(2^64 / p)
    double* win;                 // workspace hr x W (ld W): the window, residues as exact doubles
    int32_t* Linv;               // kH x kH
    int32_t* Uinv;               // kH x kH
    double* tmp;                 // kH x kH scratch for the inverses
    int32_t* out;                // [0] kk, [1] fail, [2] ncol, [3] nrow, then col swaps (a,b)..., row swaps (a,b)...
};

// a b mod p for residues a, b < p < 2^31 held as doubles: the product is split
// exactly (hi + lo, fma), the quotient estimated with the fp reciprocal (the
// paper's "floating point inverse": off by at most one),
// and corrected.  No integer<->float conversions.
__device__ __forceinline__ double mulm(double a, double b, double p, double invp) {
    const double hi = a * b;
    const double lo = fma(a, b, -hi);
    const double q = rint(hi * invp);
    double r = fma(-q, p, hi) + lo;
    if (r < 0) r += p;
    if (r >= p) r -= p;
    return r;
}
__device__ __forceinline__ double subm(double x, double t, double p) {
    const double r = x - t;
    return r < 0 ? r + p : r;
}

// a^-1 mod p by the extended Euclid algorithm in 32-bit integers (p < 2^31:
// remainders < 2^31, Bezout coefficients |s| < p); on the panel's critical path.
__device__ uint32_t inv_dev(uint32_t a, uint32_t p) {
    int32_t r0 = static_cast<int32_t>(p), r1 = static_cast<int32_t>(a), s0 = 0, s1 = 1;
    while (r1 != 0) {
        const int32_t q = r0 / r1, t = r0 - q * r1, u = s0 - q * s1;
        r0 = r1; r1 = t; s0 = s1; s1 = u;
    }
    return static_cast<uint32_t>(s0 < 0 ? s0 + static_cast<int32_t>(p) : s0);
}

// Shoup's constant floor(w 2^32 / p) for w < p < 2^31 from mu64 = floor(2^64 / p):
// (w mu64) >> 32 is the floor or one less (w eps / 2^32 < 1/2); one 64-bit check
// makes it exact.  Integer instructions only.
__device__ __forceinline__ uint32_t shoup_c(uint32_t w, uint32_t p, unsigned long long mu64) {
    const unsigned long long lo = static_cast<unsigned long long>(w) * static_cast<uint32_t>(mu64);
    const unsigned long long hi = static_cast<unsigned long long>(w) * static_cast<uint32_t>(mu64 >> 32);
    uint64_t c = (hi + (lo >> 32)) ;     // (w mu64) >> 32  (w < 2^31: no overflow of the sum)
    if ((c + 1) * p <= (static_cast<uint64_t>(w) << 32)) ++c;
    return static_cast<uint32_t>(c);
}
// x w mod p for x, w < p (Shoup): one mulhi, two multiplies, one correction.
__device__ __forceinline__ uint32_t shoup_m(uint32_t x, uint32_t w, uint32_t wsh, uint32_t p) {
    const uint32_t q = __umulhi(x, wsh);
    const uint32_t r = x * w - q * p;
    return r >= p ? r - p : r;
}
__device__ __forceinline__ uint32_t subm_u(uint32_t a, uint32_t b, uint32_t p) { return a >= b ? a - b : a + p - b; }

// One CTA of 32 x 32 threads factors the panel window (see the file header).
// kSmem: the window (<= kH x kH residues) and the inverse scratch live in
// shared memory (the generic case); otherwise in the global workspace.
//
// Fraction-free elimination keeps the modular inverse off the critical path:
// at pivot k (raw value pi_k) every unprocessed row becomes
// pi_k row_s - a_s row_k, so all rows below and the next pivot row carry the
// same scale S_k = prod_{k'<k} pi_k'; hence the true multiplier is
// L_sk = a_s / pi_k (the scales cancel) and the true U row k is row_k / S_k.
// After the elimination the pi_k are inverted in parallel and the raw
// multipliers and U rows rescaled.  L11^-1 and U11^-1 are then formed by
// Gauss-Jordan phases (one barrier and a few products per phase).  All
// products are Shoup multiplications by a per-row or per-step constant.
template <bool kSmem>
__global__ void __launch_bounds__(kThr) panel_kernel(PanelArgs P) {
    extern __shared__ uint32_t dyn_smem[];
    __shared__ int s_j;
    __shared__ int s_ncol, s_nrow, s_kk, s_fail;
    __shared__ int colsw[kMaxSwaps][2];
    __shared__ int rowsw[kMaxSwaps][2];
    __shared__ uint32_t piv[kH], pinv[kH], sinv[kH], sfw[kH];
    __shared__ int orig[kH];                      // original panel row now at each position
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const int64_t hr = P.hr, W = P.W;
    const uint32_t p = P.p;
    const unsigned long long c32 = P.mu64;             // floor(2^64 / p), for shoup_c
    uint32_t* w = kSmem ? dyn_smem : reinterpret_cast<uint32_t*>(P.win);
    uint32_t* E = kSmem ? dyn_smem + kH * kH : reinterpret_cast<uint32_t*>(P.tmp);   // kH x kH
    long long t_0 = clock64();
    // copy in (canonical residues)
    for (int64_t r = ty; r < hr; r += 32)
        for (int64_t cc = tx; cc < W; cc += 32) {
            const int64_t v = static_cast<int64_t>(P.A[(P.i0 + r) * P.lda + P.c + cc]) % static_cast<int64_t>(p);
            w[r * W + cc] = static_cast<uint32_t>(v < 0 ? v + p : v);
        }
    // E = I (kH x kH): the same row operations turn it into S L^-1 (see below)
    for (int e = tid; e < kH * kH; e += kThr) E[e] = ((e / kH) == (e % kH)) ? 1u : 0u;
    for (int e = tid; e < kH; e += kThr) orig[e] = e;
    if (tid == 0) { s_ncol = 0; s_nrow = 0; s_kk = 0; s_fail = 0; s_j = INT32_MAX; }
    __syncthreads();
    for (int64_t i = 0; i < hr; ++i) {
        const int kk = s_kk;
        // first non-zero of row i in columns [kk, W): ballot per warp, one atomic per warp
        for (int64_t c0 = kk + 32 * ty; c0 < W; c0 += kThr) {
            const int64_t cc = c0 + tx;
            const unsigned bal = __ballot_sync(0xffffffffu, cc < W && w[i * W + cc] != 0u);
            if (bal) { if (tx == 0) atomicMin(&s_j, static_cast<int>(c0) + __ffs(bal) - 1); break; }
        }
        __syncthreads();
        const int j = s_j;
        if (j == INT32_MAX) {                      // no pivot in the window
            if (!P.full) { if (tid == 0) s_fail = 1; __syncthreads(); break; }
            __syncthreads();                       // (everyone has read s_j before the next search)
            continue;                              // a zero row (stays below the pivot rows)
        }
        if (j != kk || i != kk) {                  // (uniform: rare for generic inputs)
            // column swap kk <-> j (all panel rows) and row swap i <-> kk, disjoint cells first
            if (j != kk)
                for (int64_t r = tid; r < hr; r += kThr) {
                    const uint32_t t = w[r * W + kk]; w[r * W + kk] = w[r * W + j]; w[r * W + j] = t;
                }
            if (i != kk) {
                for (int64_t cc = tid; cc < W; cc += kThr) {
                    if (cc == kk || cc == j) continue;
                    const uint32_t t = w[i * W + cc]; w[i * W + cc] = w[kk * W + cc]; w[kk * W + cc] = t;
                }
                for (int c = tid; c < kH; c += kThr) {     // E rows follow (rows i, kk)
                    const uint32_t t = E[i * kH + c]; E[i * kH + c] = E[kk * kH + c]; E[kk * kH + c] = t;
                }
            }
            __syncthreads();
            if (tid == 0) {
                if (i != kk) {                         // the swapped columns of the swapped rows
                    uint32_t t = w[i * W + kk]; w[i * W + kk] = w[kk * W + kk]; w[kk * W + kk] = t;
                    if (j != kk) { t = w[i * W + j]; w[i * W + j] = w[kk * W + j]; w[kk * W + j] = t; }
                }
                if (j != kk) { colsw[s_ncol][0] = kk; colsw[s_ncol][1] = j; ++s_ncol; }
                if (i != kk) {
                    rowsw[s_nrow][0] = kk; rowsw[s_nrow][1] = static_cast<int>(i); ++s_nrow;
                    const int t = orig[kk]; orig[kk] = orig[i]; orig[i] = t;
                }
            }
            __syncthreads();
        }
        const uint32_t pk = w[kk * W + kk];
        const uint32_t pk_sh = shoup_c(pk, p, c32);
        if (tid == 0) piv[kk] = pk;
        // fraction-free update of the unprocessed rows i+1..hr-1 (raw a_s stays in column kk)
        for (int64_t r = i + 1 + ty; r < hr; r += 32) {
            const uint32_t as = w[r * W + kk];
            if (as == 0u) {
                for (int64_t cc = kk + 1 + tx; cc < W; cc += 32) w[r * W + cc] = shoup_m(w[r * W + cc], pk, pk_sh, p);
                for (int c = tx; c <= static_cast<int>(i); c += 32) E[r * kH + c] = shoup_m(E[r * kH + c], pk, pk_sh, p);
                if (tx == 0) E[r * kH + r] = shoup_m(E[r * kH + r], pk, pk_sh, p);   // E_r's own column r > i
            } else {
                const uint32_t as_sh = shoup_c(as, p, c32);
                for (int64_t cc = kk + 1 + tx; cc < W; cc += 32)
                    w[r * W + cc] = subm_u(shoup_m(w[r * W + cc], pk, pk_sh, p), shoup_m(w[kk * W + cc], as, as_sh, p), p);
                for (int c = tx; c <= static_cast<int>(i); c += 32)
                    E[r * kH + c] = subm_u(shoup_m(E[r * kH + c], pk, pk_sh, p), shoup_m(E[kk * kH + c], as, as_sh, p), p);
                if (tx == 0) E[r * kH + r] = shoup_m(E[r * kH + r], pk, pk_sh, p);   // (E_kk has no column r)
            }
        }
        if (tid == 0) { s_kk = kk + 1; s_j = INT32_MAX; }   // (all threads read s_j before the update)
        __syncthreads();
    }
    const int kk = s_kk;
    long long t_1 = clock64(), t_2 = 0, t_3 = 0, t_4 = 0;
    if (!s_fail) {
        // pivot inverses (parallel), prefix products S_k^-1 and S_k
        for (int k = tid; k < kk; k += kThr) pinv[k] = inv_dev(piv[k], p);
        __syncthreads();
        if (tid == 0) {
            uint32_t sacc = 1 % p, facc = 1 % p;
            for (int k = 0; k < kk; ++k) {
                sinv[k] = sacc; sacc = shoup_m(sacc, pinv[k], shoup_c(pinv[k], p, c32), p);
                sfw[k] = facc; facc = shoup_m(facc, piv[k], shoup_c(piv[k], p, c32), p);
            }
        }
        __syncthreads();
        // true L (w[s][k] = a_s / pi_k for k < min(s, kk)) and true U (row k / S_k)
        for (int64_t r = ty; r < hr; r += 32) {
            const uint32_t si = r < kk ? sinv[r] : 0u;
            const uint32_t si_sh = r < kk ? shoup_c(si, p, c32) : 0u;
            for (int64_t cc = tx; cc < W; cc += 32) {
                const uint32_t x = w[r * W + cc];
                if (cc < r && cc < kk) w[r * W + cc] = shoup_m(x, pinv[cc], shoup_c(pinv[cc], p, c32), p);
                else if (r < kk && cc >= r) w[r * W + cc] = shoup_m(x, si, si_sh, p);
            }
        }
        t_2 = clock64();
        // Linv = L11^-1: E = S L^-1 Pi with Pi the panel's row permutation (E's columns
        // are original row indices), so Linv[r][c] = E[r][orig[c]] / S_r
        for (int e = tid; e < kk * kk; e += kThr) {
            const int r = e / kk, c = e % kk;
            P.Linv[r * kH + c] =
                static_cast<int32_t>(c <= r ? shoup_m(E[r * kH + orig[c]], sinv[r], shoup_c(sinv[r], p, c32), p) : 0u);
        }
        __syncthreads();
        t_3 = clock64();
        // Uinv: F <- I; phase k = kk-1..0: rows r < k: F_r -= (u_rk / u_kk) F_k; at the end
        // F_k *= 1/u_kk (the true u_kk = pi_k / S_k, so 1/u_kk = pi_k^-1 S_k)
        for (int e = tid; e < kk * kH; e += kThr) E[e] = ((e / kH) == (e % kH)) ? 1u : 0u;
        __syncthreads();
        for (int k = kk - 1; k > 0; --k) {
            const uint32_t iu = shoup_m(pinv[k], sfw[k], shoup_c(sfw[k], p, c32), p);
            for (int r = ty; r < k; r += 32) {
                const uint32_t u = w[r * W + k];
                if (u == 0u) continue;
                const uint32_t m = shoup_m(u, iu, shoup_c(iu, p, c32), p);
                const uint32_t m_sh = shoup_c(m, p, c32);
                for (int c = k + tx; c < kk; c += 32) E[r * kH + c] = subm_u(E[r * kH + c], shoup_m(E[k * kH + c], m, m_sh, p), p);
            }
            __syncthreads();
        }
        for (int e = tid; e < kk * kk; e += kThr) {
            const int r = e / kk;
            const uint32_t iu = shoup_m(pinv[r], sfw[r], shoup_c(sfw[r], p, c32), p);
            E[r * kH + e % kk] = shoup_m(E[r * kH + e % kk], iu, shoup_c(iu, p, c32), p);
        }
        __syncthreads();
        for (int e = tid; e < kk * kk; e += kThr) P.Uinv[(e / kk) * kH + e % kk] = static_cast<int32_t>(E[(e / kk) * kH + e % kk]);
        t_4 = clock64();
        // copy back
        for (int64_t r = ty; r < hr; r += 32)
            for (int64_t cc = tx; cc < W; cc += 32)
                P.A[(P.i0 + r) * P.lda + P.c + cc] = static_cast<int32_t>(w[r * W + cc]);
    }
    if (tid == 0) {
        long long* tt = reinterpret_cast<long long*>(P.out + 4 + 4 * kMaxSwaps);
        tt[0] = t_1 - t_0; tt[1] = t_2 - t_1; tt[2] = t_3 - t_2; tt[3] = t_4 - t_3; tt[4] = clock64() - t_4;
        P.out[0] = kk;
        P.out[1] = s_fail;
        P.out[2] = s_ncol;
        P.out[3] = s_nrow;
        for (int s = 0; s < s_ncol; ++s) { P.out[4 + 2 * s] = colsw[s][0]; P.out[5 + 2 * s] = colsw[s][1]; }
        for (int s = 0; s < s_nrow; ++s) {
            P.out[4 + 2 * kMaxSwaps + 2 * s] = rowsw[s][0];
            P.out[5 + 2 * kMaxSwaps + 2 * s] = rowsw[s][1];
        }
    }
}

// ---- the same panel on a CTA pair (cluster of 2) ------------------------------
// Generic case only (window of kH columns in shared memory, no zero rows): CTA
// rho owns window columns [64 rho, 64 rho + 64) and the same columns of E.  Per
// pivot: each CTA searches its columns, one cluster barrier exchanges the two
// minima (DSMEM), the non-owner of the pivot column reads the pivot and the
// multipliers a_s from the owner's shared memory, and each CTA updates its own
// half -- half the work of panel_kernel per SM, one cluster barrier per pivot.
// A zero row returns fail (the host then runs panel_kernel on this panel).
constexpr int kHalf = kH / 2;
constexpr int kPanel2Smem = (3 * kH * kHalf + 2 * kH) * 4;   // w, E, peer U columns, colbuf(+pad)

__device__ __forceinline__ uint32_t dsmem_ld_u32(const void* local_ptr, uint32_t peer) {
    const uint32_t ra = ptx::mapa(ptx::smem_u32(local_ptr), peer);
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
    return v;
}

__global__ void __launch_bounds__(kThr) panel2_kernel(PanelArgs P) {
    extern __shared__ uint32_t dyn2[];
    uint32_t* w = dyn2;                       // [kH][kHalf]: this CTA's window columns
    uint32_t* E = w + kH * kHalf;             // [kH][kHalf]: this CTA's columns of E (S L^-1, then F for U^-1)
    uint32_t* Up = E + kH * kHalf;            // [kH][kHalf]: the peer's U columns (Uinv phases)
    uint32_t* colbuf = Up + kH * kHalf;       // [kH]: the pivot column (multipliers), from its owner
    __shared__ int s_jloc[2], s_fail, s_kk, s_ncol;
    __shared__ int colsw[kMaxSwaps][2];
    __shared__ uint32_t piv[kH], pinv[kH], sinv[kH], sfw[kH];
    const uint32_t rho = ptx::cluster_ctarank(), peer = rho ^ 1u;
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const int64_t hr = P.hr;
    const uint32_t p = P.p;
    const unsigned long long c32 = P.mu64;
    const int c0 = static_cast<int>(rho) * kHalf;            // first global window column of this CTA
    long long t_0 = clock64();
    for (int e = tid; e < kH * kHalf; e += kThr) {
        const int r = e / kHalf, cl = e % kHalf;
        uint32_t v = 0;
        if (r < hr) {
            const int64_t x = static_cast<int64_t>(P.A[(P.i0 + r) * P.lda + P.c + c0 + cl]) % static_cast<int64_t>(p);
            v = static_cast<uint32_t>(x < 0 ? x + p : x);
        }
        w[e] = v;
        E[e] = (r == c0 + cl) ? 1u : 0u;
    }
    if (tid == 0) { s_jloc[0] = s_jloc[1] = INT32_MAX; s_fail = 0; s_kk = 0; s_ncol = 0; }
    __syncthreads();
    ptx::cluster_sync();
    for (int i = 0; i < hr; ++i) {
        const int kk = i;                                    // no zero rows on this path: kk == i
        const int par = i & 1;
        // local search over this CTA's columns >= kk
        if (ty == 0) {
            const int cl = tx + 32 * 0, cl2 = tx + 32;       // kHalf = 64: two columns per lane
            int best = INT32_MAX;
            if (c0 + cl >= kk && w[i * kHalf + cl] != 0u) best = c0 + cl;
            if (c0 + cl2 >= kk && w[i * kHalf + cl2] != 0u && c0 + cl2 < best) best = c0 + cl2;
            for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
            if (tx == 0) s_jloc[par] = best;     // (the peer read step i-2's value before cluster barrier i-1)
        }
        __syncthreads();
        ptx::cluster_sync();                                 // both minima written; pivot columns final
        const int j = min(s_jloc[par], static_cast<int>(dsmem_ld_u32(&s_jloc[par], peer)));
        if (j == INT32_MAX) { if (tid == 0) s_fail = 1; break; }
        const uint32_t own_k = static_cast<uint32_t>(kk / kHalf), own_j = static_cast<uint32_t>(j / kHalf);
        if (j != kk) {                                       // column swap kk <-> j (rare)
            if (own_k == own_j) {
                if (own_k == rho)
                    for (int r = tid; r < hr; r += kThr) {
                        const uint32_t t = w[r * kHalf + kk - c0];
                        w[r * kHalf + kk - c0] = w[r * kHalf + j - c0];
                        w[r * kHalf + j - c0] = t;
                    }
            } else {                                         // across the pair: read the peer's column, then write
                const int mine = (own_k == rho) ? kk : j, theirs = (own_k == rho) ? j : kk;
                for (int r = tid; r < hr; r += kThr)
                    colbuf[r] = dsmem_ld_u32(&w[r * kHalf + theirs - static_cast<int>(peer) * kHalf], peer);
                __syncthreads();
                ptx::cluster_sync();
                for (int r = tid; r < hr; r += kThr) w[r * kHalf + mine - c0] = colbuf[r];
            }
            if (tid == 0 && rho == 0) { colsw[s_ncol][0] = kk; colsw[s_ncol][1] = j; ++s_ncol; }
            __syncthreads();
            ptx::cluster_sync();
        }
        // the pivot column (multipliers a_s, and pi_k) into colbuf
        if (own_k == rho) {
            for (int r = kk + tid; r < hr; r += kThr) colbuf[r] = w[r * kHalf + kk - c0];
        } else {
            for (int r = kk + tid; r < hr; r += kThr) colbuf[r] = dsmem_ld_u32(&w[r * kHalf + kk - static_cast<int>(peer) * kHalf], peer);
        }
        __syncthreads();
        const uint32_t pk = colbuf[kk];
        const uint32_t pk_sh = shoup_c(pk, p, c32);
        if (tid == 0) piv[kk] = pk;
        // fraction-free update of rows i+1.. on this CTA's columns > kk, and of E; the
        // (up to 4) rows of a warp are processed together for instruction-level parallelism
        const int clo = max(kk + 1 - c0, 0);
        uint32_t as[4], as_sh[4];
        bool ok[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = i + 1 + ty + 32 * q;
            ok[q] = r < hr;
            as[q] = ok[q] ? colbuf[r] : 0u;
            as_sh[q] = shoup_c(as[q], p, c32);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int cl = tx + 32 * h;
            const uint32_t pw = w[kk * kHalf + cl], pe = E[kk * kHalf + cl];
            const int e = c0 + cl;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!ok[q]) continue;
                const int r = i + 1 + ty + 32 * q;
                if (cl >= clo)
                    w[r * kHalf + cl] = subm_u(shoup_m(w[r * kHalf + cl], pk, pk_sh, p), shoup_m(pw, as[q], as_sh[q], p), p);
                if (e <= i)
                    E[r * kHalf + cl] = subm_u(shoup_m(E[r * kHalf + cl], pk, pk_sh, p), shoup_m(pe, as[q], as_sh[q], p), p);
                else if (e == r)
                    E[r * kHalf + cl] = shoup_m(E[r * kHalf + cl], pk, pk_sh, p);
            }
        }
        __syncthreads();
    }
    int kk = s_fail ? 0 : static_cast<int>(hr);
    long long t_1 = clock64(), t_2 = 0, t_3 = 0, t_4 = 0;
    ptx::cluster_sync();
    const int fail = s_fail | static_cast<int>(dsmem_ld_u32(&s_fail, peer));
    if (!fail) {
        for (int k = tid; k < kk; k += kThr) pinv[k] = inv_dev(piv[k], p);
        __syncthreads();
        if (tid == 0) {
            uint32_t sacc = 1 % p, facc = 1 % p;
            for (int k = 0; k < kk; ++k) {
                sinv[k] = sacc; sacc = shoup_m(sacc, pinv[k], shoup_c(pinv[k], p, c32), p);
                sfw[k] = facc; facc = shoup_m(facc, piv[k], shoup_c(piv[k], p, c32), p);
            }
        }
        __syncthreads();
        for (int r = ty; r < hr; r += 32) {              // true L and U on this CTA's columns
            const uint32_t si = r < kk ? sinv[r] : 0u;
            const uint32_t si_sh = r < kk ? shoup_c(si, p, c32) : 0u;
            for (int cl = tx; cl < kHalf; cl += 32) {
                const int cc = c0 + cl;
                const uint32_t x = w[r * kHalf + cl];
                if (cc < r && cc < kk) w[r * kHalf + cl] = shoup_m(x, pinv[cc], shoup_c(pinv[cc], p, c32), p);
                else if (r < kk && cc >= r) w[r * kHalf + cl] = shoup_m(x, si, si_sh, p);
            }
        }
        t_2 = clock64();
        // Linv columns of this CTA: E[r][e] / S_r (no row swaps on this path)
        for (int e = tid; e < kk * kHalf; e += kThr) {
            const int r = e / kHalf, cl = e % kHalf, cc = c0 + cl;
            if (cc < kk)
                P.Linv[r * kH + cc] = static_cast<int32_t>(cc <= r ? shoup_m(E[r * kHalf + cl], sinv[r], shoup_c(sinv[r], p, c32), p) : 0u);
        }
        __syncthreads();
        ptx::cluster_sync();                                 // both CTAs' U rescaled: copy the peer's U columns
        for (int e = tid; e < kH * kHalf; e += kThr) Up[e] = dsmem_ld_u32(&w[e], peer);
        for (int e = tid; e < kH * kHalf; e += kThr) E[e] = ((e / kHalf) == c0 + (e % kHalf)) ? 1u : 0u;
        __syncthreads();
        t_3 = clock64();
        // Uinv (this CTA's columns c >= k): F_r -= (u_rk / u_kk) F_k for r < k, then F_k /= u_kk
        for (int k = kk - 1; k > 0; --k) {
            const uint32_t own = static_cast<uint32_t>(k / kHalf);
            const uint32_t* Ucol = (own == rho) ? w : Up;
            const int kl = k - static_cast<int>(own) * kHalf;
            const uint32_t iu = shoup_m(pinv[k], sfw[k], shoup_c(sfw[k], p, c32), p);
            const int clo = max(k - c0, 0);
            if (clo < kHalf) {
                for (int r = ty; r < k; r += 32) {
                    const uint32_t u = Ucol[r * kHalf + kl];
                    if (u == 0u) continue;
                    const uint32_t m = shoup_m(u, iu, shoup_c(iu, p, c32), p);
                    const uint32_t m_sh = shoup_c(m, p, c32);
                    for (int cl = clo + tx; cl < kHalf; cl += 32)
                        E[r * kHalf + cl] = subm_u(E[r * kHalf + cl], shoup_m(E[k * kHalf + cl], m, m_sh, p), p);
                }
            }
            __syncthreads();
        }
        for (int e = tid; e < kk * kHalf; e += kThr) {
            const int r = e / kHalf, cl = e % kHalf, cc = c0 + cl;
            if (cc < kk) {
                const uint32_t iu = shoup_m(pinv[r], sfw[r], shoup_c(sfw[r], p, c32), p);
                P.Uinv[r * kH + cc] = static_cast<int32_t>(shoup_m(E[r * kHalf + cl], iu, shoup_c(iu, p, c32), p));
            }
        }
        t_4 = clock64();
        for (int e = tid; e < hr * kHalf; e += kThr) {
            const int r = e / kHalf, cl = e % kHalf;
            P.A[(P.i0 + r) * P.lda + P.c + c0 + cl] = static_cast<int32_t>(w[e]);
        }
    } else {
        kk = 0;
    }
    if (tid == 0 && rho == 0) {
        long long* tt = reinterpret_cast<long long*>(P.out + 4 + 4 * kMaxSwaps);
        tt[0] = t_1 - t_0; tt[1] = t_2 - t_1; tt[2] = 0; tt[3] = t_4 - t_3; tt[4] = clock64() - t_4;
        P.out[0] = kk;
        P.out[1] = fail;
        P.out[2] = s_ncol;
        P.out[3] = 0;
        for (int s = 0; s < s_ncol; ++s) { P.out[4 + 2 * s] = colsw[s][0]; P.out[5 + 2 * s] = colsw[s][1]; }
    }
    ptx::cluster_sync();                                     // the peer is done reading this CTA's shared memory
}

// Column transpositions (in order) applied to the rows outside [skip0, skip1).
__global__ void colswap_kernel(int32_t* A, int64_t lda, int64_t m, int64_t skip0, int64_t skip1,
                               const int* sw, int nsw, int64_t c) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x) {
        if (r >= skip0 && r < skip1) continue;
        int32_t* row = A + r * lda + c;
        for (int s = 0; s < nsw; ++s) {
            const int a = sw[2 * s], b = sw[2 * s + 1];
            const int32_t t = row[a]; row[a] = row[b]; row[b] = t;
        }
    }
}

// Swap columns [c0, c1) of rows ra and rb, for each pair.
__global__ void rowswap_kernel(int32_t* A, int64_t lda, const int64_t* pairs, int npairs, int64_t c0, int64_t c1) {
    for (int s = 0; s < npairs; ++s) {
        int32_t* a = A + pairs[2 * s] * lda;
        int32_t* b = A + pairs[2 * s + 1] * lda;
        for (int64_t cc = c0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cc < c1;
             cc += (int64_t)gridDim.x * blockDim.x) {
            const int32_t t = a[cc]; a[cc] = b[cc]; b[cc] = t;
        }
    }
}

// Zero the columns [c0, n) of rows [r0, r1) (the U part of rows that reduced to zero).
__global__ void zero_kernel(int32_t* A, int64_t lda, int64_t r0, int64_t r1, int64_t c0, int64_t n) {
    for (int64_t r = r0 + blockIdx.y; r < r1; r += gridDim.y)
        for (int64_t cc = c0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; cc < n;
             cc += (int64_t)gridDim.x * blockDim.x)
            A[r * lda + cc] = 0;
}

int gemm_plain(uint32_t p, const ff_opts* opts, char tX, char tY, int64_t m, int64_t n, int64_t k, uint32_t alpha,
               const int32_t* X, int64_t ldx, const int32_t* Y, int64_t ldy, uint32_t beta, int32_t* C, int64_t ldc,
               void* ws, cudaStream_t st, int reserve_sms = 0) {
    if (m == 0 || n == 0) return 0;
    Plan pl;
    int e = make_plan(p, k, opts, &pl);
    if (e) return e;
    set_scalars(&pl, alpha, beta);
    pl.reserve_sms = reserve_sms;
    return gemm_dev(pl, tX, tY, m, n, k, X, ldx, Y, ldy, C, ldc, ws, st);
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct LqupWs {
    size_t win, linv, uinv, out, pairs, gemm;
    size_t total() const { return win + linv + uinv + out + pairs + gemm; }
};

int lqup_ws(uint32_t p, int64_t m, int64_t n, const ff_opts* opts, LqupWs* w) {
    w->win = align256(static_cast<size_t>(kH) * std::max<int64_t>(n, 1) * 8 + static_cast<size_t>(kH) * kH * 8);
    w->linv = w->uinv = align256(2 * static_cast<size_t>(kH) * kH * 4);          // double-buffered (lookahead)
    w->out = align256(2 * ((4 + 4 * kMaxSwaps) * 4 + 64));
    w->pairs = align256(4 * kMaxSwaps * 8);
    // GEMMs: K <= kH; M <= m, N <= n (a CRT plan for short K has the most planes)
    size_t g = 0;
    for (int crt = 0; crt < 2; ++crt) {
        ff_opts o;
        std::memset(&o, 0, sizeof(o));
        if (opts) o = *opts;
        if (crt) { o.scheme = FF_SCHEME_CRT; o.kb_override = 0; }
        Plan pl;
        if (make_plan(p, kH, &o, &pl) == 0) g = std::max(g, gemm_ws_bytes(pl, m, n));
        else if (!crt) return FF_ERR_OPTS;
    }
    w->gemm = align256(g);
    return 0;
}

// product of the first r diagonal entries of A mod p (one CTA: tree of Barrett products)
__global__ void diag_prod_kernel(const int32_t* A, int64_t lda, int64_t r, uint32_t p, unsigned long long mu64,
                                 uint32_t* out) {
    __shared__ uint32_t part[256];
    unsigned long long acc = 1 % p;
    for (int64_t i = threadIdx.x; i < r; i += 256)
        acc = residue_u64(acc * static_cast<uint32_t>(A[i * lda + i]), mu64, p);
    part[threadIdx.x] = static_cast<uint32_t>(acc);
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            part[threadIdx.x] = static_cast<uint32_t>(
                residue_u64(static_cast<unsigned long long>(part[threadIdx.x]) * part[threadIdx.x + s], mu64, p));
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = part[0];
}

int perm_parity(const int64_t* v, int64_t n) {   // 0 even, 1 odd (cycle decomposition)
    std::vector<char> seen(static_cast<size_t>(n), 0);
    int par = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (seen[i]) continue;
        int64_t len = 0;
        for (int64_t j = i; !seen[j]; j = v[j]) { seen[j] = 1; ++len; }
        par ^= static_cast<int>((len - 1) & 1);
    }
    return par;
}
}  // namespace

}  // namespace ff

using namespace ff;

extern "C" {

size_t ff_lqup_workspace_size(uint32_t p, int64_t m, int64_t n, const ff_opts* opts) {
    if (p < 2 || p >= (1u << 31) || m < 0 || n < 0) return 0;
    LqupWs w;
    if (lqup_ws(p, m, n, opts, &w)) return 0;
    return w.total();
}

int ff_lqup_ex(uint32_t p, int64_t m, int64_t n, int32_t* A, int64_t lda, int64_t* Q, int64_t* P, int64_t* rank,
               const ff_opts* opts, void* workspace, size_t workspace_bytes, void* stream) {
    if (p < 2 || p >= (1u << 31)) return -1;
    if (m < 0) return -2;
    if (n < 0) return -3;
    if (!A && m > 0 && n > 0) return -4;
    if (lda < (n > 1 ? n : 1)) return -5;
    if (!Q && m > 0) return -6;
    if (!P && n > 0) return -7;
    if (!rank) return -8;
    for (int64_t i = 0; i < m; ++i) Q[i] = i;
    for (int64_t j = 0; j < n; ++j) P[j] = j;
    *rank = 0;
    if (m == 0 || n == 0) return 0;
    int e = check_device();
    if (e) return e;
    LqupWs w;
    if ((e = lqup_ws(p, m, n, opts, &w))) return e;
    if (!workspace || workspace_bytes < w.total() || (reinterpret_cast<uintptr_t>(workspace) & 255)) return -10;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    double* win = reinterpret_cast<double*>(ws);
    double* tmpd = win + static_cast<size_t>(kH) * std::max<int64_t>(n, 1);
    int32_t* Linv2 = reinterpret_cast<int32_t*>(ws + w.win);
    int32_t* Uinv2 = reinterpret_cast<int32_t*>(ws + w.win + w.linv);
    int32_t* dout2 = reinterpret_cast<int32_t*>(ws + w.win + w.linv + w.uinv);
    const size_t out_stride = ((4 + 4 * kMaxSwaps) * 4 + 64) / 4;
    int64_t* dpairs = reinterpret_cast<int64_t*>(ws + w.win + w.linv + w.uinv + w.out);
    void* gws = ws + w.win + w.linv + w.uinv + w.out + w.pairs;
    std::vector<int32_t> hout(4 + 4 * kMaxSwaps);
    std::vector<int64_t> hp(4 * kMaxSwaps);
    const uint32_t neg1 = p - 1;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(panel_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes) !=
                cudaSuccess ||
            cudaFuncSetAttribute(panel2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanel2Smem) !=
                cudaSuccess)
            return fail_cuda_now();
        attr = true;
    }
    static const bool use_pair = getenv("FF_LQUP_ONECTA") == nullptr;   // experiment: one-CTA panels only
    int64_t i0 = 0, c = 0, m_active = m, r = 0;
    int64_t W = std::min<int64_t>(n, kH);
    auto fail_cuda = [&]() { cudaGetLastError(); return FF_ERR_CUDA; };
    // Lookahead: the panel kernel of the next panel runs on its own stream, on
    // SMs the big trailing GEMM leaves free (kReserve), as soon as the next
    // panel's rows are updated; Linv/Uinv/out are double-buffered for that.
    constexpr int kReserve = 2;
    cudaStream_t ps = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_panel = nullptr;
    if (cudaStreamCreateWithFlags(&ps, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev_panel, cudaEventDisableTiming) != cudaSuccess)
        return fail_cuda();
    struct Cleanup {
        cudaStream_t s; cudaEvent_t a, b;
        ~Cleanup() { cudaStreamSynchronize(s); cudaStreamDestroy(s); cudaEventDestroy(a); cudaEventDestroy(b); }
    } cleanup{ps, ev_ready, ev_panel};
    if (cudaEventRecord(ev_ready, st) != cudaSuccess) return fail_cuda();
    int buf = 0;
    while (i0 < m_active && c < n) {
        int32_t* Linv = Linv2 + static_cast<size_t>(buf) * kH * kH;
        int32_t* Uinv = Uinv2 + static_cast<size_t>(buf) * kH * kH;
        int32_t* dout = dout2 + static_cast<size_t>(buf) * out_stride;
        const int64_t hr = std::min<int64_t>(kH, m_active - i0);
        const int64_t Wc = std::min<int64_t>(W, n - c);
        PanelArgs pa;
        pa.A = A; pa.lda = lda; pa.i0 = i0; pa.hr = hr; pa.c = c; pa.W = Wc;
        pa.full = (c + Wc == n) ? 1 : 0;
        pa.p = p; pa.dp = static_cast<double>(p); pa.invp = 1.0 / static_cast<double>(p);
        pa.mu64 = static_cast<unsigned long long>((static_cast<unsigned __int128>(1) << 64) / p);
        pa.win = win; pa.tmp = tmpd; pa.Linv = Linv; pa.Uinv = Uinv; pa.out = dout;
        if (cudaStreamWaitEvent(ps, ev_ready, 0) != cudaSuccess) return fail_cuda();
        bool used_pair = false;
        if (Wc == kH && use_pair) {
            // the panel on a CTA pair (generic case); a zero row makes it report fail
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(2);
            cfg.blockDim = dim3(kThr);
            cfg.dynamicSmemBytes = kPanel2Smem;
            cfg.stream = ps;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            if (cudaLaunchKernelEx(&cfg, panel2_kernel, pa) != cudaSuccess) return fail_cuda();
            if (cudaMemcpyAsync(hout.data(), dout, hout.size() * 4, cudaMemcpyDeviceToHost, ps) != cudaSuccess ||
                cudaStreamSynchronize(ps) != cudaSuccess)
                return fail_cuda();
            used_pair = !hout[1];
        }
        if (!used_pair) {
            if (Wc <= kH) panel_kernel<true><<<1, kThr, kSmemBytes, ps>>>(pa);
            else panel_kernel<false><<<1, kThr, 0, ps>>>(pa);
            if (cudaGetLastError() != cudaSuccess) return fail_cuda();
            if (cudaMemcpyAsync(hout.data(), dout, hout.size() * 4, cudaMemcpyDeviceToHost, ps) != cudaSuccess)
                return fail_cuda();
        }
        if (cudaEventRecord(ev_panel, ps) != cudaSuccess || cudaStreamSynchronize(ps) != cudaSuccess)
            return fail_cuda();
        if (cudaStreamWaitEvent(st, ev_panel, 0) != cudaSuccess) return fail_cuda();
        const int64_t kk = hout[0];
        if (getenv("FF_LQUP_TRACE")) {
            long long tt[5];
            cudaMemcpy(tt, dout + 4 + 4 * kMaxSwaps, sizeof(tt), cudaMemcpyDeviceToHost);
            fprintf(stderr, "[lqup panel i0=%lld kk=%lld W=%lld] cycles: elim %lld  rescale %lld  Linv %lld  Uinv %lld  copy %lld\n",
                    (long long)i0, (long long)kk, (long long)Wc, tt[0], tt[1], tt[2], tt[3], tt[4]);
        }
        if (hout[1]) {                       // a row without pivot in the window: widen and redo
            W = std::min<int64_t>(n, 4 * Wc);
            continue;
        }
        buf ^= 1;
        const int ncol = hout[2], nrow = hout[3];
        // column swaps (window coordinates) on all rows outside the panel + bookkeeping
        if (ncol > 0) {
            colswap_kernel<<<static_cast<unsigned>(std::min<int64_t>((m + 255) / 256, 4096)), 256, 0, st>>>(
                A, lda, m, i0, i0 + hr, dout + 4, ncol, c);
            for (int s = 0; s < ncol; ++s) std::swap(P[c + hout[4 + 2 * s]], P[c + hout[5 + 2 * s]]);
        }
        // row swaps inside the panel: the L parts (columns [0, c)) of those rows follow
        if (nrow > 0) {
            for (int s = 0; s < nrow; ++s) {
                const int64_t a = i0 + hout[4 + 2 * kMaxSwaps + 2 * s], b = i0 + hout[5 + 2 * kMaxSwaps + 2 * s];
                hp[2 * s] = a; hp[2 * s + 1] = b;
                std::swap(Q[a], Q[b]);
            }
            if (c > 0) {
                if (cudaMemcpyAsync(dpairs, hp.data(), 2 * nrow * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
                    return fail_cuda();
                rowswap_kernel<<<static_cast<unsigned>(std::min<int64_t>((c + 255) / 256, 1024)), 256, 0, st>>>(
                    A, lda, dpairs, nrow, 0, c);
            }
        }
        const int64_t z = hr - kk;
        bool ready_recorded = false;
        if (kk > 0) {
            // U of the pivot rows beyond the window: U_rest = L11^-1 A_rest (in place, beta = 0)
            if (c + Wc < n) {
                int32_t* Ar = A + i0 * lda + c + Wc;
                if ((e = gemm_plain(p, opts, 'N', 'N', kk, n - c - Wc, kk, 1, Linv, kH, Ar, lda, 0, Ar, lda, gws, st)))
                    return e;
            }
            // trailing rows [i0 + hr, m_active): G = X U11^-1, Z <- Z - G U12; without zero
            // rows the next panel's rows go first and release the next panel kernel
            auto trailing = [&](int64_t r0, int64_t r1, int reserve) -> int {
                if (r1 <= r0) return 0;
                int32_t* X = A + r0 * lda + c;
                int ee = gemm_plain(p, opts, 'N', 'N', r1 - r0, kk, kk, 1, X, lda, Uinv, kH, 0, X, lda, gws, st, reserve);
                if (ee) return ee;
                if (c + kk < n)
                    ee = gemm_plain(p, opts, 'N', 'N', r1 - r0, n - c - kk, kk, neg1, X, lda, A + i0 * lda + c + kk,
                                    lda, 1, X + kk, lda, gws, st, reserve);
                return ee;
            };
            const int64_t t0 = i0 + hr;
            if (z == 0) {
                const int64_t t1 = std::min<int64_t>(m_active, t0 + kH);
                if ((e = trailing(t0, t1, 0))) return e;
                if (cudaEventRecord(ev_ready, st) != cudaSuccess) return fail_cuda();
                ready_recorded = true;
                if ((e = trailing(t1, m_active, kReserve))) return e;
            } else if ((e = trailing(t0, m_active, 0))) {
                return e;
            }
        }
        // rows of the panel that reduced to zero (full window only): to the bottom of the active rows
        if (z > 0) {
            zero_kernel<<<dim3(64, static_cast<unsigned>(std::min<int64_t>(z, 1024))), 256, 0, st>>>(
                A, lda, i0 + kk, i0 + hr, c + kk, n);
            // zero rows Zs = [i0+kk, i0+hr) go to Tb = [m_active-z, m_active): swap
            // Zs \ Tb with Tb \ Zs (trailing rows, already updated above)
            const int64_t dst0 = m_active - z;
            const int64_t b0 = std::max(dst0, i0 + hr);
            int np = 0;
            for (int64_t a = i0 + kk, b = b0; a < std::min(dst0, i0 + hr); ++a, ++b) {
                hp[2 * np] = a; hp[2 * np + 1] = b; ++np;
                std::swap(Q[a], Q[b]);
            }
            if (np > 0) {
                if (cudaMemcpyAsync(dpairs, hp.data(), 2 * np * 8, cudaMemcpyHostToDevice, st) != cudaSuccess)
                    return fail_cuda();
                rowswap_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 1024)), 256, 0, st>>>(
                    A, lda, dpairs, np, 0, n);
            }
            m_active -= z;
        }
        if (!ready_recorded && cudaEventRecord(ev_ready, st) != cudaSuccess) return fail_cuda();
        i0 += kk;
        c += kk;
        r += kk;
        W = std::min<int64_t>(n, kH);
    }
    // rows that never got a pivot (c reached n): their U part is already zero
    *rank = r;
    return cudaStreamSynchronize(st) == cudaSuccess ? 0 : FF_ERR_CUDA;
}

int ff_rank_det(uint32_t p, int64_t m, int64_t n, const int32_t* A, int64_t lda, int64_t* rank, uint32_t* det) {
    if (p < 2 || p >= (1u << 31)) return -1;
    if (m < 0) return -2;
    if (n < 0) return -3;
    if (!A && m > 0 && n > 0) return -4;
    if (lda < (n > 1 ? n : 1)) return -5;
    if (!rank) return -6;
    if (det && m != n) return -7;
    const size_t need = ff_lqup_workspace_size(p, m, n, nullptr);
    if (need == 0) return FF_ERR_INTERNAL;
    const size_t abytes = (static_cast<size_t>(m) * std::max<int64_t>(n, 1) * 4 + 255) & ~size_t(255);
    void* ws = nullptr;
    if (cudaMalloc(&ws, need + abytes + 256) != cudaSuccess) {
        cudaGetLastError();
        return FF_ERR_NOMEM;
    }
    int32_t* Ac = static_cast<int32_t*>(ws);
    uint32_t* dprod = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + abytes);
    std::vector<int64_t> Q(static_cast<size_t>(std::max<int64_t>(m, 1))), P(static_cast<size_t>(std::max<int64_t>(n, 1)));
    int e = 0;
    if (m > 0 && n > 0 && cudaMemcpy2D(Ac, n * 4, A, lda * 4, n * 4, m, cudaMemcpyDeviceToDevice) != cudaSuccess)
        e = FF_ERR_CUDA;
    if (!e) e = ff_lqup_ex(p, m, n, Ac, n, Q.data(), P.data(), rank, nullptr, static_cast<uint8_t*>(ws) + abytes + 256,
                           need, nullptr);
    if (!e && det) {
        if (*rank < m) {
            *det = 0;
        } else {
            // det A = sign(Q) sign(P) prod_i U_ii  (Q A P = L U, L unit lower)
            const unsigned long long mu64 = static_cast<unsigned long long>((static_cast<unsigned __int128>(1) << 64) / p);
            diag_prod_kernel<<<1, 256>>>(Ac, n, *rank, p, mu64, dprod);
            uint32_t d = 0;
            if (cudaMemcpy(&d, dprod, 4, cudaMemcpyDeviceToHost) != cudaSuccess) e = FF_ERR_CUDA;
            const int odd = perm_parity(Q.data(), m) ^ perm_parity(P.data(), n);
            *det = (odd && d) ? p - d : d;
        }
    }
    cudaFree(ws);
    return e;
}

int ff_lqup(uint32_t p, int64_t m, int64_t n, int32_t* A, int64_t lda, int64_t* Q, int64_t* P, int64_t* rank) {
    if (p < 2 || p >= (1u << 31)) return -1;
    if (m < 0) return -2;
    if (n < 0) return -3;
    const size_t need = ff_lqup_workspace_size(p, m, n, nullptr);
    if (need == 0) return FF_ERR_INTERNAL;
    void* ws = nullptr;
    if (cudaMalloc(&ws, need) != cudaSuccess) {
        cudaGetLastError();
        return FF_ERR_NOMEM;
    }
    const int e = ff_lqup_ex(p, m, n, A, lda, Q, P, rank, nullptr, ws, need, nullptr);
    cudaFree(ws);
    return e;
}

}  // extern "C"
