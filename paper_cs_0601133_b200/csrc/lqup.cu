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
#include <array>
#include <chrono>
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
constexpr int kGroup = 8;        // panels per deferred trailing update (ff_lqup_ex)
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
    unsigned long long mu64;     // floor(2^64 / p)
    int32_t red;                 // panel_spec_kernel: reduce 64-bit sums every red products
    volatile int32_t* note;      // panel_spec_kernel: host-mapped [seq, fail] written last (or null)
    int32_t seq;
    double* win;                 // workspace hr x W (ld W): the window, residues as exact doubles
    int32_t* Linv;               // kH x kH
    int32_t* Uinv;               // kH x kH
    double* tmp;                 // kH x kH scratch for the inverses
    int32_t* out;                // [0] kk, [1] fail, [2] ncol, [3] nrow, then col swaps (a,b)..., row swaps (a,b)...
};

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
            w[r * W + cc] = residue_i32_64(P.A[(P.i0 + r) * P.lda + P.c + cc], P.mu64, p);
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
    __shared__ int s_jloc[2], s_fail, s_ncol;
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
            v = residue_i32_64(P.A[(P.i0 + r) * P.lda + P.c + c0 + cl], P.mu64, p);
        }
        w[e] = v;
        E[e] = (r == c0 + cl) ? 1u : 0u;
    }
    if (tid == 0) { s_jloc[0] = s_jloc[1] = INT32_MAX; s_fail = 0; s_ncol = 0; }
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

// ---- speculative blocked panel -----------------------------------------------
// For a full kH x kH window the paper's pivot rule ("first non-zero of the row",
// P:583-588) selects the diagonal entry unless it is zero, which for a random
// matrix over a large field happens with probability about kH/p per panel.  This
// kernel assumes no swap at all and factors the window as a blocked LU, kB
// columns at a time:
//   (1) fraction-free LDU elimination of the kB x kB diagonal block D (one
//       element per thread, one barrier per pivot): row operations below the
//       pivot, tracked in E_L (-> S L_D^-1), and column operations right of it,
//       tracked in E_U (-> U'^-1 S, U' = the unit upper factor);
//   (2) the kB pivots inverted together (prefix / suffix products in one warp,
//       one modular inverse); D, E_L, E_U rescaled to L_D, U_D, L_D^-1, U_D^-1;
//   (3) U12 = L_D^-1 A12 and L21 = A21 U_D^-1, then A22 <- A22 - L21 U12, as
//       shared-memory products with delayed reduction (Eq. (1) in 64 bits).
// The full L11^-1 and U11^-1 follow from the diagonal blocks' inverses by block
// back-substitution waves.  A zero pivot reports fail and nothing is written:
// the host then runs panel2_kernel / panel_kernel, whose output is what this
// kernel produces when no swap occurs (the LU without pivoting is unique).
constexpr int kB = 16;                                            // block size (kB^2 threads eliminate)
constexpr int kNb = kH / kB;
constexpr int kSpecScratch = 2 * kB * (kH - kB);                  // u32: U12 (kB x R) + L21 (R x kB); 2 (kNb-1) blocks
constexpr int kSpecSmem = (3 * kH * kH + kSpecScratch) * 4;       // window, Linv, Uinv, scratch: 206 KB
static_assert(kB == 16 || kB == 32, "block size");

__device__ __forceinline__ uint32_t mulm_b(uint32_t a, uint32_t b, uint32_t p, unsigned long long mu64) {
    return residue_u64(static_cast<unsigned long long>(a) * b, mu64, p);
}

// C = A B (mode 0), C - A B (mode 1) or -(A B) (mode 2) mod p on shared-memory
// residue matrices; M multiple of 4, N and K of 32; rows of A 16-byte aligned.
struct MmJob {
    uint32_t* C;
    const uint32_t* A;
    const uint32_t* B;
    int ldc, lda, ldb, M, N, K, mode;
};

__device__ __forceinline__ MmJob mm_job(uint32_t* C, int ldc, const uint32_t* A, int lda, const uint32_t* B, int ldb,
                                        int M, int N, int K, int mode) {
    MmJob j;
    j.C = C; j.A = A; j.B = B; j.ldc = ldc; j.lda = lda; j.ldb = ldb; j.M = M; j.N = N; j.K = K; j.mode = mode;
    return j;
}

// One job on a group of nthr threads (lt: index in the group).  An item is 4 x 1
// output cells; a warp takes 4 rows x 32 consecutive columns, so the A reads are
// broadcasts (16 B: four k at once) and the B reads conflict-free.  Products are
// summed in 64 bits: kBig reduces every 4 products (any p < 2^31: 4 (p-1)^2 + p
// < 2^64), otherwise every kB (the host checks kB (p-1)^2 + p < 2^64).  K is a
// multiple of kB.
template <bool kBig>
__device__ __forceinline__ void mm_one(const MmJob J, int lt, int nthr, uint32_t p, unsigned long long mu64) {
    const int items = (J.M / 4) * J.N;
    for (int e = lt; e < items; e += nthr) {
        const int i = (e / J.N) * 4, j = e % J.N;
        const uint32_t* Ab = J.A + i * J.lda;
        const uint32_t* Bb = J.B + j;
        unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
        for (int k0 = 0; k0 < J.K; k0 += kB) {
#pragma unroll
            for (int kk = 0; kk < kB; kk += 4) {
                const int k = k0 + kk;
                const uint32_t b0 = Bb[(k + 0) * J.ldb], b1 = Bb[(k + 1) * J.ldb];
                const uint32_t b2 = Bb[(k + 2) * J.ldb], b3 = Bb[(k + 3) * J.ldb];
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) {
                    const uint4 a = *reinterpret_cast<const uint4*>(Ab + ii * J.lda + k);
                    acc[ii] += static_cast<unsigned long long>(a.x) * b0 + static_cast<unsigned long long>(a.y) * b1 +
                               static_cast<unsigned long long>(a.z) * b2 + static_cast<unsigned long long>(a.w) * b3;
                    if (kBig) acc[ii] = residue_u64(acc[ii], mu64, p);
                }
            }
            if (!kBig) {
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) acc[ii] = residue_u64(acc[ii], mu64, p);
            }
        }
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
            const uint32_t r = static_cast<uint32_t>(acc[ii]);     // already reduced
            uint32_t* c = J.C + (i + ii) * J.ldc + j;
            if (J.mode == 0) *c = r;
            else if (J.mode == 1) *c = subm_u(*c, r, p);
            else *c = r ? p - r : 0u;
        }
    }
}
// The same job on the tensor cores (warp-level mma.sync m16n8k32 u8 x u8 -> s32),
// for p < 2^16: residues split into two bytes, x = x0 + 256 x1, so that
// A B = P00 + 256 (P01 + P10) + 65536 P11 with four byte products, each exact in
// s32 (K <= 128: K 255^2 < 2^24), recombined in 64 bits and reduced once.  A
// warp computes a 16 x 8 tile; the fragments are built straight from the u32
// matrices (A: one 16 B load gives four k of a row; B: four loads down a column)
// and their bytes gathered with byte permutes.  K is zero-padded to 32.
__device__ __forceinline__ void imma16832(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                          uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// bytes 0 (lo) and 1 (hi) of four residues < 2^16, packed in order
__device__ __forceinline__ void split4(uint32_t x, uint32_t y, uint32_t z, uint32_t w, uint32_t& lo, uint32_t& hi) {
    const uint32_t t0 = __byte_perm(x, y, 0x5140), t1 = __byte_perm(z, w, 0x5140);   // x0 y0 x1 y1 | z0 w0 z1 w1
    lo = __byte_perm(t0, t1, 0x5410);
    hi = __byte_perm(t0, t1, 0x7632);
}
__device__ void mm_tc(const MmJob J, int wg, int nw, uint32_t p, unsigned long long mu64) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int tiles_n = J.N / 8, tiles = (J.M / 16) * tiles_n;
    for (int tile = wg; tile < tiles; tile += nw) {
        const int r0 = (tile / tiles_n) * 16, c0 = (tile % tiles_n) * 8;
        int P00[4] = {0, 0, 0, 0}, P01[4] = {0, 0, 0, 0}, P10[4] = {0, 0, 0, 0}, P11[4] = {0, 0, 0, 0};
        for (int k0 = 0; k0 < J.K; k0 += 32) {
            uint32_t alo[4], ahi[4], blo[2], bhi[2];
#pragma unroll
            for (int q = 0; q < 4; ++q) {              // a0: row g, a1: row g+8; a2, a3: k + 16
                const int row = r0 + g + ((q & 1) ? 8 : 0), k = k0 + ((q & 2) ? 16 : 0) + 4 * t;
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (k < J.K) v = *reinterpret_cast<const uint4*>(J.A + row * J.lda + k);
                split4(v.x, v.y, v.z, v.w, alo[q], ahi[q]);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {              // b0: column g, k = 4t..; b1: k + 16
                const int k = k0 + (q ? 16 : 0) + 4 * t;
                const uint32_t* bp = J.B + k * J.ldb + c0 + g;
                uint32_t x = 0, y = 0, z = 0, w = 0;
                if (k < J.K) { x = bp[0]; y = bp[J.ldb]; z = bp[2 * J.ldb]; w = bp[3 * J.ldb]; }
                split4(x, y, z, w, blo[q], bhi[q]);
            }
            imma16832(P00, alo[0], alo[1], alo[2], alo[3], blo[0], blo[1]);
            imma16832(P01, alo[0], alo[1], alo[2], alo[3], bhi[0], bhi[1]);
            imma16832(P10, ahi[0], ahi[1], ahi[2], ahi[3], blo[0], blo[1]);
            imma16832(P11, ahi[0], ahi[1], ahi[2], ahi[3], bhi[0], bhi[1]);
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {                  // d0, d1: row g, cols 2t, 2t+1; d2, d3: row g+8
            const unsigned long long S = static_cast<unsigned long long>(static_cast<uint32_t>(P00[e])) +
                                         (static_cast<unsigned long long>(static_cast<uint32_t>(P01[e]) +
                                                                          static_cast<uint32_t>(P10[e])) << 8) +
                                         (static_cast<unsigned long long>(static_cast<uint32_t>(P11[e])) << 16);
            const uint32_t r = residue_u64(S, mu64, p);
            uint32_t* c = J.C + (r0 + g + ((e & 2) ? 8 : 0)) * J.ldc + c0 + 2 * t + (e & 1);
            if (J.mode == 0) *c = r;
            else if (J.mode == 1) *c = subm_u(*c, r, p);
            else *c = r ? p - r : 0u;
        }
    }
}

__device__ __forceinline__ void mm_any(bool big, const MmJob& J, int lt, int nthr, uint32_t p, unsigned long long mu64) {
    if (p < 65536u) mm_tc(J, lt >> 5, nthr >> 5, p, mu64);     // (groups are whole warps)
    else if (big) mm_one<true>(J, lt, nthr, p, mu64);
    else mm_one<false>(J, lt, nthr, p, mu64);
}

// Block row b of L11^-1 and block column b of U11^-1 once blocks 0..b are final
// (left-looking):
//   Li[b][j] = -Li[b][b] (sum_{k=j}^{b-1} L[b][k] Li[k][j]),
//   Ui[j][b] = -(sum_{k=j}^{b-1} Ui[j][k] U[k][b]) Ui[b][b],   j < b,
// two dependent products over the thread group [g0, g0 + gn) (whole warps),
// synchronised by `bar` (a named barrier for the group, or the CTA barrier).
template <class Bar>
__device__ __forceinline__ void inv_block(int b, const uint32_t* W, uint32_t* Li, uint32_t* Ui, uint32_t* T, int gtid,
                                          int gn, bool big, uint32_t p, unsigned long long mu, Bar bar) {
    if (b == 0) return;
    const int n = 2 * b, gw = gn / 32, wpj = gw / n;
    const int q = (gtid >> 5) / wpj, lt = gtid - q * wpj * 32;
    const bool on = q < n;
    const int j = q >> 1;
    uint32_t* Tq = T + q * kB * kB;
    if (on) {
        if ((q & 1) == 0)       // T_L = [L[b][j] .. L[b][b-1]] [Li[j][j] ; .. ; Li[b-1][j]]
            mm_any(big, mm_job(Tq, kB, W + b * kB * kH + j * kB, kH, Li + j * kB * kH + j * kB, kH, kB, kB, (b - j) * kB, 0),
                   lt, wpj * 32, p, mu);
        else                    // T_U = [Ui[j][j] .. Ui[j][b-1]] [U[j][b] ; .. ; U[b-1][b]]
            mm_any(big, mm_job(Tq, kB, Ui + j * kB * kH + j * kB, kH, W + j * kB * kH + b * kB, kH, kB, kB, (b - j) * kB, 0),
                   lt, wpj * 32, p, mu);
    }
    bar();
    if (on) {
        if ((q & 1) == 0)
            mm_any(big, mm_job(Li + b * kB * kH + j * kB, kH, Li + b * kB * kH + b * kB, kH, Tq, kB, kB, kB, kB, 2),
                   lt, wpj * 32, p, mu);
        else
            mm_any(big, mm_job(Ui + j * kB * kH + b * kB, kH, Tq, kB, Ui + b * kB * kH + b * kB, kH, kB, kB, kB, 2),
                   lt, wpj * 32, p, mu);
    }
    bar();
}

__global__ void __launch_bounds__(kThr) panel_spec_kernel(PanelArgs P) {
    extern __shared__ __align__(16) uint32_t dyn3[];
    uint32_t* W = dyn3;                       // [kH][kH] the window -> L (strict lower) and U
    uint32_t* Li = W + kH * kH;               // [kH][kH] L11^-1
    uint32_t* Ui = Li + kH * kH;              // [kH][kH] U11^-1
    uint32_t* T = Ui + kH * kH;               // scratch
    __shared__ uint32_t ipk[kH], isc[kH], iu[kH];
    __shared__ uint32_t ash[2][kB], bsh[2][kB];   // Shoup constants of the pivot column / row (by parity)
    __shared__ int s_fail;
    const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
    const uint32_t p = P.p;
    const unsigned long long mu = P.mu64;
    const bool big = P.red < kB;
    long long t_0 = clock64();
    {
        const int32_t* src = P.A + P.i0 * P.lda + P.c;
        const bool vec = (P.lda % 4) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
        if (vec) {                                // 16-byte rows: 4 loads per thread, all in flight
            int4 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = (tid + q * kThr) * 4;
                v[q] = *reinterpret_cast<const int4*>(src + static_cast<int64_t>(e / kH) * P.lda + e % kH);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int e = (tid + q * kThr) * 4;
                *reinterpret_cast<uint4*>(W + e) =
                    make_uint4(residue_i32_64(v[q].x, mu, p), residue_i32_64(v[q].y, mu, p), residue_i32_64(v[q].z, mu, p),
                               residue_i32_64(v[q].w, mu, p));
                *reinterpret_cast<uint4*>(Li + e) = make_uint4(0u, 0u, 0u, 0u);
                *reinterpret_cast<uint4*>(Ui + e) = make_uint4(0u, 0u, 0u, 0u);
            }
        } else {
            constexpr int kPer = kH * kH / kThr;  // all loads in flight before any use
            int32_t v[kPer];
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                const int e = tid + q * kThr;
                v[q] = src[static_cast<int64_t>(e / kH) * P.lda + e % kH];
            }
#pragma unroll
            for (int q = 0; q < kPer; ++q) {
                const int e = tid + q * kThr;
                W[e] = residue_i32_64(v[q], mu, p);
                Li[e] = 0u;
                Ui[e] = 0u;
            }
        }
    }
    if (tid == 0) s_fail = 0;
    __syncthreads();
    bool fail = false;
    // the kB x kB diagonal block is eliminated by threads [0, kB^2), cell (er, ec),
    // synchronised by named barrier 1; the other warps wait at the next CTA barrier
    const bool elim = tid < kB * kB;
    const int er = tid / kB, ec = tid % kB;
    for (int kb = 0; kb < kNb; ++kb) {
        const int o = kb * kB;
        uint32_t* D = W + o * kH + o;          // the diagonal block (ld kH)
        uint32_t* El = Li + o * kH + o;        // E_L, then L_D^-1
        uint32_t* Eu = Ui + o * kH + o;        // E_U, then U_D^-1
        uint32_t x = 0u, el = 0u, eu = 0u;
        if (!elim) {
            // the other 24 warps: block kb - 1's row of L11^-1 / column of U11^-1 meanwhile
            inv_block(kb - 1, W, Li, Ui, T, tid - kB * kB, kThr - kB * kB, big, p, mu,
                      [] { ptx::named_bar_sync(2, kThr - kB * kB); });
        } else {
            x = D[er * kH + ec];
            if (ec == 0) ash[0][er] = shoup_c(x, p, mu);
            if (er == 0) bsh[0][ec] = shoup_c(x, p, mu);
            uint32_t S = 1u % p;                   // S_t = prod_{t' < t} pk_t' (uniform)
            ptx::named_bar_sync(1, kB * kB);
            // (1) pivot t (pk = D[t][t], scale S_t): rows r > t become pk row_r - a_r row_t
            // -- on D's columns > t (column t keeps the raw a_r) and on E_L's columns <= t;
            // the columns c > t of E_U become pk col_c - D[t][c] col_t on its rows <= t.
            // The diagonals of E_L and E_U are implicitly S_r (never stored), every other
            // entry outside these ranges stays zero, so each thread updates exactly one
            // cell (er, ec) of one of D, E_L, E_U per pivot.  Step t reads row t and
            // column t only and writes rows / columns > t: one barrier per pivot.  All
            // products are Shoup multiplications; the constants of the next pivot's row
            // and column (ash: a_r and the pivot, bsh: D[t][c]) come from the threads
            // that produce them.
            for (int t = 0; t < kB; ++t) {
                const int par = t & 1;
                const uint32_t pk = D[t * kH + t];
                if (pk == 0u) { fail = true; if (tid == 0) s_fail = 1; break; }   // uniform: speculation failed
                const uint32_t pk_sh = ash[par][t];
                // one update per thread, v <- pk v - X Y, without divergence: all
                // operands are loaded and the role (D, E_L or E_U cell) selects them
                const uint32_t a = D[er * kH + t], a_sh = ash[par][er];          // D[r][t] and its constant
                const uint32_t u = D[t * kH + ec], u_sh = bsh[par][ec];          // D[t][c] and its constant
                const uint32_t elt = El[t * kH + ec], eut = Eu[er * kH + t];
                const bool rowop = er > t, colgt = ec > t;
                const uint32_t v = rowop ? (colgt ? x : el) : eu;
                const uint32_t X = rowop ? (colgt ? u : (ec == t ? S : elt)) : (er == t ? S : eut);
                const uint32_t Y = rowop ? a : u, Ysh = rowop ? a_sh : u_sh;
                const uint32_t nv = subm_u(shoup_m(v, pk, pk_sh, p), shoup_m(X, Y, Ysh, p), p);
                if (rowop || colgt) {
                    uint32_t* dst = rowop ? (colgt ? D : El) : Eu;
                    dst[er * kH + ec] = nv;
                    if (rowop && colgt) x = nv;
                    else if (rowop) el = nv;
                    else eu = nv;
                    if (rowop && colgt) {
                        if (ec == t + 1) ash[par ^ 1][er] = shoup_c(nv, p, mu);
                        if (er == t + 1) bsh[par ^ 1][ec] = shoup_c(nv, p, mu);
                    }
                }
                if (er == t && ec == t) { El[t * kH + t] = S; Eu[t * kH + t] = S; }   // the implicit diagonals S_t
                S = shoup_m(S, pk, pk_sh, p);
                ptx::named_bar_sync(1, kB * kB);
            }
        }
        __syncthreads();
        fail = s_fail != 0;
        if (fail) break;
        // (2) warp 0: prefix P_t and suffix Q_t products of the pivots, one inverse of
        // P_{kB-1}: 1/S_t = inv Q_t, 1/pk_t = (1/S_{t+1}) P_{t-1}, 1/u_tt = S_t / pk_t.
        // Meanwhile warps 1..31 form the raw products E_L A12 and A21 E_U (E_L = S L_D^-1,
        // E_U = U_D^-1-ish with column scales S_c), scaled to U12 and L21 once the
        // inverses are known: U12 = diag(1/S_r) (E_L A12), L21 = (A21 E_U) diag(1/pk_c).
        const int R = kH - o - kB;
        uint32_t* T1 = T;
        uint32_t* T2 = T + kB * R;
        if (ty == 0) {
            const uint32_t v = tx < kB ? D[tx * kH + tx] : 1u;
            uint32_t pre = v, suf = v;
#pragma unroll
            for (int d = 1; d < kB; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, pre, d);
                const uint32_t z = __shfl_down_sync(0xffffffffu, suf, d);
                if (tx >= d) pre = mulm_b(pre, y, p, mu);
                if (tx + d < kB) suf = mulm_b(suf, z, p, mu);
            }
            const uint32_t total = __shfl_sync(0xffffffffu, pre, kB - 1);
            const uint32_t inv = inv_dev(total, p);
            const uint32_t is = mulm_b(inv, suf, p, mu);              // 1 / S_tx
            uint32_t is_next = __shfl_down_sync(0xffffffffu, is, 1);  // 1 / S_{tx+1} = 1 / P_tx
            if (tx == kB - 1) is_next = inv;
            uint32_t pprev = __shfl_up_sync(0xffffffffu, pre, 1);    // P_{tx-1} = S_tx
            if (tx == 0) pprev = 1u % p;
            const uint32_t ip = mulm_b(is_next, pprev, p, mu);
            if (tx < kB) {
                isc[o + tx] = is;
                ipk[o + tx] = ip;
                iu[o + tx] = mulm_b(pprev, ip, p, mu);
            }
        } else if (R > 0) {
            const int gw = 31, w1 = 15;                                  // warps 1..15 | 16..31
            const int wi = ty - 1;
            if (wi < w1) mm_any(big, mm_job(T1, R, El, kH, W + o * kH + o + kB, kH, kB, R, kB, 0), wi * 32 + tx, w1 * 32, p, mu);
            else mm_any(big, mm_job(T2, kB, W + (o + kB) * kH + o, kH, Eu, kH, R, kB, kB, 0), (wi - w1) * 32 + tx,
                        (gw - w1) * 32, p, mu);
        }
        __syncthreads();
        // true L_D (a / pk_c), U_D (row / S_r); L_D^-1 = E_L / S_r (unit diagonal);
        // U_D^-1 = E_U / pk_c (E_U col c = S_c U'^-1 col c, U_D^-1 = U'^-1 diag(S_c / pk_c));
        // U12 rows and L21 columns scaled alike
        if (elim) {
            D[er * kH + ec] = mulm_b(x, er > ec ? ipk[o + ec] : isc[o + er], p, mu);
            El[er * kH + ec] = ec < er ? mulm_b(el, isc[o + er], p, mu) : (ec == er ? 1u : 0u);
            Eu[er * kH + ec] = er < ec ? mulm_b(eu, ipk[o + ec], p, mu) : (ec == er ? iu[o + ec] : 0u);
        } else if (R > 0) {
            for (int e = tid - kB * kB; e < kB * R; e += kThr - kB * kB) {
                T1[e] = mulm_b(T1[e], isc[o + e / R], p, mu);
                T2[e] = mulm_b(T2[e], ipk[o + e % kB], p, mu);
            }
        }
        __syncthreads();
        // (3) A22 -= L21 U12 while U12 (T1, kB x R) and L21 (T2, R x kB) are copied into the window
        if (R > 0) {
            mm_any(big, mm_job(W + (o + kB) * kH + o + kB, kH, T2, kB, T1, R, R, R, kB, 1), tid, kThr, p, mu);
            for (int e = tid; e < kB * R; e += kThr) {
                W[(o + e / R) * kH + o + kB + e % R] = T1[e];
                W[(o + kB + e / kB) * kH + o + e % kB] = T2[e];
            }
            __syncthreads();
        }
    }
    long long t_1 = clock64(), t_2 = 0;
    if (!fail) {
        // the last block's row of L11^-1 / column of U11^-1 (the earlier ones ran
        // beside the eliminations)
        inv_block(kNb - 1, W, Li, Ui, T, tid, kThr, big, p, mu, [] { __syncthreads(); });
        t_2 = clock64();
        int32_t* dst = P.A + P.i0 * P.lda + P.c;
        if ((P.lda % 4) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
            for (int e = tid * 4; e < kH * kH; e += kThr * 4) {
                *reinterpret_cast<uint4*>(dst + static_cast<int64_t>(e / kH) * P.lda + e % kH) = *reinterpret_cast<const uint4*>(W + e);
                *reinterpret_cast<uint4*>(P.Linv + e) = *reinterpret_cast<const uint4*>(Li + e);
                *reinterpret_cast<uint4*>(P.Uinv + e) = *reinterpret_cast<const uint4*>(Ui + e);
            }
        } else {
            for (int e = tid; e < kH * kH; e += kThr) {
                dst[static_cast<int64_t>(e / kH) * P.lda + e % kH] = static_cast<int32_t>(W[e]);
                P.Linv[e] = static_cast<int32_t>(Li[e]);
                P.Uinv[e] = static_cast<int32_t>(Ui[e]);
            }
        }
    }
    if (tid == 0) {
        long long* tt = reinterpret_cast<long long*>(P.out + 4 + 4 * kMaxSwaps);
        tt[0] = t_1 - t_0; tt[1] = 0; tt[2] = 0; tt[3] = t_2 - t_1; tt[4] = clock64() - t_2;
        P.out[0] = fail ? 0 : kH;
        P.out[1] = fail ? 1 : 0;
        P.out[2] = 0;
        P.out[3] = 0;
        if (P.note) {                 // the host polls this instead of synchronising the stream
            P.note[1] = fail ? 1 : 0;
            __threadfence_system();
            P.note[0] = P.seq;
        }
    }
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
               void* ws, cudaStream_t st, int reserve_sms = 0, bool canon = false) {
    if (m == 0 || n == 0) return 0;
    static const bool host_t = getenv("FF_LQUP_HOSTTIME") != nullptr;   // development aid
    const auto h0 = std::chrono::steady_clock::now();
    Plan pl;
    int e = make_plan(p, k, opts, &pl);
    if (e) return e;
    set_scalars(&pl, alpha, beta);
    pl.reserve_sms = reserve_sms;
    pl.canonical_ab = canon;         // the caller guarantees X, Y canonical (products of earlier steps)
    const auto h1 = std::chrono::steady_clock::now();
    e = gemm_dev(pl, tX, tY, m, n, k, X, ldx, Y, ldy, C, ldc, ws, st);
    if (host_t) {
        const auto h2 = std::chrono::steady_clock::now();
        static double tp = 0, tg = 0;
        static long cnt = 0;
        tp += std::chrono::duration<double, std::micro>(h1 - h0).count();
        tg += std::chrono::duration<double, std::micro>(h2 - h1).count();
        if (++cnt % 200 == 0) fprintf(stderr, "[gemm_plain host] %ld calls: plan %.1f us, enqueue %.1f us (avg)\n", cnt, tp / cnt, tg / cnt);
    }
    return e;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct LqupWs {
    size_t win, linv, uinv, out, pairs, gemm, obuf;
    size_t total() const { return win + linv + uinv + out + pairs + gemm + obuf; }
};

int lqup_ws(uint32_t p, int64_t m, int64_t n, const ff_opts* opts, LqupWs* w) {
    w->win = align256(static_cast<size_t>(kH) * std::max<int64_t>(n, 1) * 8 + static_cast<size_t>(kH) * kH * 8);
    w->linv = w->uinv = align256(2 * static_cast<size_t>(kH) * kH * 4);          // double-buffered (lookahead)
    w->out = align256(2 * ((4 + 4 * kMaxSwaps) * 4 + 64));
    w->pairs = align256(4 * kMaxSwaps * 8);
    // GEMMs: K <= kH kGroup; M <= m, N <= n (a CRT plan for short K has the most planes)
    size_t g = 0;
    for (int crt = 0; crt < 2; ++crt) {
        ff_opts o;
        std::memset(&o, 0, sizeof(o));
        if (opts) o = *opts;
        if (crt) { o.scheme = FF_SCHEME_CRT; o.kb_override = 0; }
        Plan pl;
        for (int64_t K : {static_cast<int64_t>(kH), static_cast<int64_t>(kH) * kGroup}) {
            if (make_plan(p, K, &o, &pl) == 0) g = std::max(g, gemm_ws_bytes(pl, m, n));
            else if (!crt) return FF_ERR_OPTS;
        }
    }
    w->gemm = align256(g);
    // out-of-place destination of the wide U_rest / G products (copied back)
    w->obuf = align256(static_cast<size_t>(kH) * std::max<int64_t>(std::max<int64_t>(m, n), 1) * 4);
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
    int32_t* obuf = reinterpret_cast<int32_t*>(ws + w.win + w.linv + w.uinv + w.out + w.pairs + w.gemm);
    std::vector<int32_t> hout(4 + 4 * kMaxSwaps);
    std::vector<int64_t> hp(4 * kMaxSwaps);
    const uint32_t neg1 = p - 1;
    if (set_smem_attr(reinterpret_cast<const void*>(panel_kernel<true>), kSmemBytes) != cudaSuccess ||
        set_smem_attr(reinterpret_cast<const void*>(panel2_kernel), kPanel2Smem) != cudaSuccess ||
        set_smem_attr(reinterpret_cast<const void*>(panel_spec_kernel), kSpecSmem) != cudaSuccess)
        return fail_cuda_now();
    static const bool use_pair = getenv("FF_LQUP_ONECTA") == nullptr;   // experiment: one-CTA panels only
    // speculative no-swap panels; given up after kSpecGiveUp failures (small fields)
    constexpr int kSpecGiveUp = 2;
    int spec_fails = getenv("FF_LQUP_NOSPEC") ? kSpecGiveUp : 0;
    // delayed reduction in panel_spec_kernel: red (p-1)^2 + p < 2^64, a multiple of 4, <= 128
    int red = 4;
    {
        const unsigned __int128 lim = (static_cast<unsigned __int128>(1) << 64) - p;
        const unsigned __int128 sq = static_cast<unsigned __int128>(p - 1) * (p - 1);
        while (red < 128 && static_cast<unsigned __int128>(red + 4) * sq < lim) red += 4;
    }
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
    // host-mapped note for the speculative panel's outcome (one per process)
    static volatile int32_t* note_h = nullptr;
    static int32_t* note_d = nullptr;
    static int32_t note_seq = 0;
    if (!note_h) {
        void* hp_ = nullptr;
        if (cudaHostAlloc(&hp_, 64, cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess &&
            cudaHostGetDevicePointer(reinterpret_cast<void**>(&note_d), hp_, 0) == cudaSuccess) {
            note_h = static_cast<volatile int32_t*>(hp_);
            note_h[0] = 0;
        } else {
            cudaGetLastError();
            note_d = nullptr;
        }
    }
    // FF_LQUP_TIMELINE=1 (development aid): per-panel event timestamps, printed at the end
    const bool tl = getenv("FF_LQUP_TIMELINE") != nullptr;
    std::vector<std::array<cudaEvent_t, 6>> tl_ev;
    const int group = [] {
        const char* g = getenv("FF_LQUP_GROUP");                // experiment knob (1 = no deferral)
        const int v = g ? atoi(g) : kGroup;
        return v < 1 ? 1 : (v > kGroup ? kGroup : v);
    }();
    int npend = 0;
    int64_t pi0 = 0, pc0 = 0;
    static const bool chain_fuse = getenv("FF_LQUP_NOCHAIN") == nullptr;   // A/B knob
    // rows [ra, rb) x columns [ca, cb) -= A[ra.., pc0 .. pc0 + K) A[pi0 .. pi0 + K, ca..cb)
    auto upd = [&](int64_t ra, int64_t rb, int64_t ca, int64_t cb, int64_t K, int reserve) -> int {
        rb = std::min<int64_t>(rb, m_active);
        cb = std::min<int64_t>(cb, n);
        if (rb <= ra || cb <= ca || K <= 0) return 0;
        return gemm_plain(p, opts, 'N', 'N', rb - ra, cb - ca, K, neg1, A + ra * lda + pc0, lda, A + pi0 * lda + ca, lda,
                          1, A + ra * lda + ca, lda, gws, st, reserve, true);   // L and U entries: canonical
    };
    while (i0 < m_active && c < n) {
        int32_t* Linv = Linv2 + static_cast<size_t>(buf) * kH * kH;
        int32_t* Uinv = Uinv2 + static_cast<size_t>(buf) * kH * kH;
        int32_t* dout = dout2 + static_cast<size_t>(buf) * out_stride;
        const int64_t hr = std::min<int64_t>(kH, m_active - i0);
        const int64_t Wc = std::min<int64_t>(W, n - c);
        PanelArgs pa;
        pa.note = nullptr;
        pa.seq = 0;
        pa.A = A; pa.lda = lda; pa.i0 = i0; pa.hr = hr; pa.c = c; pa.W = Wc;
        pa.full = (c + Wc == n) ? 1 : 0;
        pa.p = p;
        pa.mu64 = static_cast<unsigned long long>((static_cast<unsigned __int128>(1) << 64) / p);
        pa.win = win; pa.tmp = tmpd; pa.Linv = Linv; pa.Uinv = Uinv; pa.out = dout;
        pa.red = red;
        if (cudaStreamWaitEvent(ps, ev_ready, 0) != cudaSuccess) return fail_cuda();
        if (tl) { tl_ev.emplace_back(); for (auto& x : tl_ev.back()) cudaEventCreate(&x); cudaEventRecord(tl_ev.back()[0], ps); }
        bool used_pair = false;
        bool waited = false;
        if (Wc == kH && hr == kH && spec_fails < kSpecGiveUp) {
            pa.note = note_d;
            pa.seq = ++note_seq;
            panel_spec_kernel<<<1, kThr, kSpecSmem, ps>>>(pa);
            pa.note = nullptr;
            if (cudaGetLastError() != cudaSuccess) return fail_cuda();
            if (note_h) {
                // poll the host-mapped note (lower latency than a stream synchronisation
                // plus a copy); the stream is queried now and then for errors
                if (tl) cudaEventRecord(tl_ev.back()[1], ps);
                if (cudaEventRecord(ev_panel, ps) != cudaSuccess) return fail_cuda();
                for (long spins = 1; note_h[0] != pa.seq; ++spins) {
                    if ((spins & 4095) == 0) {
                        const cudaError_t q = cudaStreamQuery(ps);
                        if (q == cudaSuccess && note_h[0] != pa.seq) return FF_ERR_INTERNAL;
                        if (q != cudaSuccess && q != cudaErrorNotReady) return fail_cuda();
                    }
                }
                hout[1] = note_h[1];
                hout[0] = hout[1] ? 0 : kH;
                hout[2] = hout[3] = 0;
                waited = !hout[1];
            } else if (cudaMemcpyAsync(hout.data(), dout, hout.size() * 4, cudaMemcpyDeviceToHost, ps) != cudaSuccess ||
                       cudaStreamSynchronize(ps) != cudaSuccess) {
                return fail_cuda();
            }
            used_pair = !hout[1];
            if (hout[1]) ++spec_fails;
        }
        if (!used_pair && Wc == kH && use_pair) {
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
        if (!waited) {
            if (tl) cudaEventRecord(tl_ev.back()[1], ps);
            if (cudaEventRecord(ev_panel, ps) != cudaSuccess || cudaStreamSynchronize(ps) != cudaSuccess)
                return fail_cuda();
        }
        if (tl) cudaEventRecord(tl_ev.back()[2], st);   // host turnaround: GEMM work enqueued from here
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
            // the wider window reaches columns whose update was queued after the
            // release of this panel: wait for all of it
            if (cudaEventRecord(ev_ready, st) != cudaSuccess) return fail_cuda();
            continue;
        }
        buf ^= 1;
        const bool generic = group > 1 && kk == kH && hr == kH && Wc == kH;
        // A non-generic panel first brings the pending region up to date -- before its
        // column swaps, which may reach beyond the 128-column window (widened window)
        // and would otherwise exchange pending and up-to-date columns.
        if (npend > 0 && !generic) {
            if ((e = upd(i0 + kH, m_active, c + kH, n, c - pc0, 0))) return e;
            npend = 0;
        }
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
        // Deferred trailing updates: for a group of up to `group` generic
        // panels (kk = hr = W = kH) the Schur-complement updates of the rows and columns
        // beyond the group are applied once, as one GEMM with K = kH x (panels); only the
        // next panel's rows and window columns are brought up to date in between.  The
        // short-K update GEMM is bound by its epilogue (the C read / write and the
        // reduction), not by K, so this divides the dominant cost by the group size.
        // Invariant while npend > 0: the pending panels (rows [pi0, i0), L columns
        // [pc0, c)) have not yet updated rows >= i0 + kH at columns >= c + kH.
        if (generic) {
            // The next panel kernel needs only its own 128 x 128 window up to date, so the
            // chain that releases it is three 128-column products (U_rest's first window,
            // G of the next panel's rows, the window's update); everything wider runs
            // while that panel kernel does.
            const int64_t r1 = i0 + kH, c1 = c + kH, rn = std::min<int64_t>(m_active, r1 + kH);
            const int64_t cw = std::min<int64_t>(n, c1 + kH);                     // end of the next window
            auto urest = [&](int64_t ca, int64_t cb) -> int {                     // U_rest = L11^-1 A_rest
                if (cb <= ca) return 0;
                int32_t* Ar = A + i0 * lda + ca;    // (canonical once an earlier panel has updated these rows)
                return gemm_plain(p, opts, 'N', 'N', kk, cb - ca, kk, 1, Linv, kH, Ar, lda, 0, Ar, lda, gws, st, 0, i0 > 0);
            };
            auto gmul = [&](int64_t ra, int64_t rb) -> int {                      // G = X U11^-1
                rb = std::min<int64_t>(rb, m_active);
                if (rb <= ra) return 0;
                int32_t* X = A + ra * lda + c;
                return gemm_plain(p, opts, 'N', 'N', rb - ra, kk, kk, 1, X, lda, Uinv, kH, 0, X, lda, gws, st, 0, i0 > 0);
            };
            if (npend == 0) { pi0 = i0; pc0 = c; }
            ++npend;
            const int64_t K = c1 - pc0;
            // The three chain products in one cooperative launch when they take the
            // small-field path anyway (p < 2^16, canonical operands): U_rest's window,
            // G of the next rows (both in place), then the window's update from them.
            int fused = FF_ERR_INTERNAL;
            if (chain_fuse && i0 > 0 && !tl && kk == kH) {
                const int64_t rnm = std::min<int64_t>(rn, m_active);
                SmallChainProduct pr[3] = {
                    {kk, cw - c1, kk, Linv, kH, A + i0 * lda + c1, lda, A + i0 * lda + c1, lda},
                    {rnm - r1, kk, kk, A + r1 * lda + c, lda, Uinv, kH, A + r1 * lda + c, lda},
                    {rnm - r1, cw - c1, K, A + r1 * lda + pc0, lda, A + pi0 * lda + c1, lda, A + r1 * lda + c1, lda}};
                Plan p01, p2;
                if (cw > c1 && rnm > r1 && make_plan(p, kk, opts, &p01) == 0 && make_plan(p, K, opts, &p2) == 0 &&
                    p01.all_auto && p2.all_auto) {
                    set_scalars(&p01, 1, 0);
                    set_scalars(&p2, neg1, 1);
                    p01.canonical_ab = p2.canonical_ab = true;
                    fused = launch_small_chain(p01, p2, pr, st);
                    if (fused != 0 && fused != FF_ERR_INTERNAL) return fused;
                }
            }
            if (fused != 0) {
                if ((e = urest(c1, cw))) return e;
                if (tl) cudaEventRecord(tl_ev.back()[4], st);
                if ((e = gmul(r1, rn))) return e;
                if (tl) cudaEventRecord(tl_ev.back()[5], st);
                if ((e = upd(r1, rn, c1, cw, K, 0))) return e;                  // the next window
            }
            if (cudaEventRecord(ev_ready, st) != cudaSuccess) return fail_cuda();
            // the wide U_rest and G products: out of place (a small-field product may not
            // run in place without a grid barrier, which these grids are too large for),
            // then copied back
            if (i0 > 0 && cw < n) {
                if ((e = gemm_plain(p, opts, 'N', 'N', kk, n - cw, kk, 1, Linv, kH, A + i0 * lda + cw, lda, 0, obuf, n - cw,
                                    gws, st, 0, true)))
                    return e;
                if (cudaMemcpy2DAsync(A + i0 * lda + cw, lda * 4, obuf, (n - cw) * 4, (n - cw) * 4, kk,
                                      cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                    return fail_cuda();
            } else if ((e = urest(cw, n))) {
                return e;
            }
            if ((e = upd(r1, rn, cw, n, K, 0))) return e;                        // the rest of its rows
            if (i0 > 0 && rn < m_active) {
                if ((e = gemm_plain(p, opts, 'N', 'N', m_active - rn, kk, kk, 1, A + rn * lda + c, lda, Uinv, kH, 0, obuf, kk,
                                    gws, st, 0, true)))
                    return e;
                if (cudaMemcpy2DAsync(A + rn * lda + c, lda * 4, obuf, kk * 4, kk * 4, m_active - rn,
                                      cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                    return fail_cuda();
            } else if ((e = gmul(rn, m_active))) {
                return e;
            }
            if (npend == group || r1 + kH >= m_active || c1 + kH >= n) {
                if ((e = upd(rn, m_active, c1, n, K, kReserve))) return e;      // flush the group
                npend = 0;
            } else if ((e = upd(rn, m_active, c1, cw, K, 0))) {                 // the next window's columns below
                return e;
            }
            ready_recorded = true;
        } else if (kk > 0) {
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
        if (tl) cudaEventRecord(tl_ev.back()[3], st);   // (after the whole iteration's work)
        i0 += kk;
        c += kk;
        r += kk;
        W = std::min<int64_t>(n, kH);
    }
    if (npend > 0) {                                            // (not reached: the last group flushes)
        if ((e = upd(i0 + kH, m_active, c + kH, n, c - pc0, 0))) return e;
        npend = 0;
    }
    if (tl) {
        cudaStreamSynchronize(st);
        cudaStreamSynchronize(ps);
        double sp = 0, sg = 0, sc = 0, su = 0, sgg = 0, si = 0;
        for (size_t i = 0; i < tl_ev.size(); ++i) {
            float a = 0, b = 0, c2 = 0, u = 0, g = 0, ii = 0;
            if (cudaEventElapsedTime(&u, tl_ev[i][2], tl_ev[i][4]) != cudaSuccess) { u = 0; cudaGetLastError(); }
            if (cudaEventElapsedTime(&g, tl_ev[i][4], tl_ev[i][5]) != cudaSuccess) { g = 0; cudaGetLastError(); }
            if (i + 1 < tl_ev.size() && cudaEventElapsedTime(&ii, tl_ev[i][5], tl_ev[i + 1][0]) != cudaSuccess) { ii = 0; cudaGetLastError(); }
            su += u; sgg += g; si += ii;
            cudaEventElapsedTime(&a, tl_ev[i][0], tl_ev[i][1]);              // panel kernel
            cudaEventElapsedTime(&b, tl_ev[i][1], tl_ev[i][2]);              // panel end -> host enqueues
            if (i + 1 < tl_ev.size()) cudaEventElapsedTime(&c2, tl_ev[i][1], tl_ev[i + 1][0]);   // panel end -> next panel start
            sp += a; sg += b; sc += c2;
        }
        const double np = tl_ev.empty() ? 1.0 : static_cast<double>(tl_ev.size());
        fprintf(stderr, "[lqup timeline] panels %zu: panel kernel %.1f us, panel end -> host enqueue %.1f us, "
                "panel end -> next panel start %.1f us (averages); chain: U_rest %.1f us, G(next rows) %.1f us, "
                "lookahead row update -> next panel start %.1f us\n", tl_ev.size(), 1e3 * sp / np, 1e3 * sg / np,
                1e3 * sc / np, 1e3 * su / np, 1e3 * sgg / np, 1e3 * si / np);
        for (auto& e4 : tl_ev) for (auto& x : e4) cudaEventDestroy(x);
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
