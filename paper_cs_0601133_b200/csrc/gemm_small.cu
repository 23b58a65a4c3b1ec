// gemm_small.cu -- fgemm for small fields (p < 2^16) on the warp-level tensor
// cores (mma.sync m16n8k32 u8 x u8 -> s32), without encoders: the latency path
// for short-K and small problems.
//
// Every residue x < p < 2^16 is split into two bytes, x = x0 + 256 x1, so that
// one dot product of length K is
//     sum_k a_k b_k = P00 + 256 (P01 + P10) + 65536 P11,   P_ij = sum_k a_ki b_kj,
// four byte products, each exact in s32 while K 255^2 < 2^31 (K <= 32768), and
// recombined exactly in 64 bits before one modular reduction -- the delayed
// reduction of PAPER.md Eq. (1) with the whole K in one block.
// The tcgen05 kernel (gemm_tc.cu) is the throughput path; this one has no
// encode pass, no TMEM round trips between weight groups and a light epilogue,
// which is what short-K products (LQUP / ftrsm updates, K = 128 .. 1024) and
// small matrices are bound by.
//
// Three kernels:
//  * small_gemm_kernel: any int32 inputs (reduced on load, reading R3), any
//    transposes; CTA of 256 threads (8 warps) owns a 64 x 64 tile of C, warp w
//    computes rows 16 (w & 3) .. +16 and columns 32 (w >> 2) .. +32 (four
//    m16n8 tiles); K staged 32 at a time in shared memory as canonical u32
//    residues, the next slice loaded into registers meanwhile;
//  * small_gemm_canon_kernel: canonical, non-transposed operands streamed raw by
//    cp.async through a 4-deep ring (same tile);
//  * small_gemm_wide_kernel<L>: the same for 2^16 <= p < 2^31 with L = 3 or 4
//    bytes per residue (64 x 16 tiles for the L^2 accumulators).
// Fragments are built from the u32 residues with byte permutes.  None of them
// may run with C overlapping A or B unless launched with `alias` (the two
// canonical kernels only): a cooperative launch whose grid barrier separates
// every CTA's reads from the first write.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"
#include "modp.cuh"

namespace ff {

namespace {

constexpr int kSM = 64, kSN = 64, kSK = 32;
constexpr int kSThreads = 256;
constexpr int kApitch = kSK + 4;   // u32; 16 B aligned rows
constexpr int kBpitch = kSN + 4;

struct SmallArgs {
    ModP M;
    unsigned long long mu64;       // floor(2^64 / p)
    const int32_t* A;
    const int32_t* B;
    int32_t* C;
    int64_t lda, ldb, ldc;
    int32_t m, n, k;
    int32_t tA, tB;                // 1: op(X) = X^T
    int32_t alias;                 // 1: C overlaps A or B: grid-wide barrier between reads and writes
    int32_t reduce;                // small_gemm_canon_kernel: 1: A, B raw int32, reduced in shared memory
};

__device__ __forceinline__ void imma(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// bytes 0 (lo) and 1 (hi) of four values < 2^16, in order
__device__ __forceinline__ void split4(uint32_t x, uint32_t y, uint32_t z, uint32_t w, uint32_t& lo, uint32_t& hi) {
    const uint32_t t0 = __byte_perm(x, y, 0x5140), t1 = __byte_perm(z, w, 0x5140);
    lo = __byte_perm(t0, t1, 0x5410);
    hi = __byte_perm(t0, t1, 0x7632);
}

__device__ __forceinline__ int32_t ld_a(const SmallArgs& a, int r, int kk) {   // op(A)[r][kk], 0 outside
    if (r >= a.m || kk >= a.k) return 0;
    return a.tA ? a.A[static_cast<int64_t>(kk) * a.lda + r] : a.A[static_cast<int64_t>(r) * a.lda + kk];
}
__device__ __forceinline__ int32_t ld_b(const SmallArgs& a, int kk, int c) {   // op(B)[kk][c], 0 outside
    if (kk >= a.k || c >= a.n) return 0;
    return a.tB ? a.B[static_cast<int64_t>(c) * a.ldb + kk] : a.B[static_cast<int64_t>(kk) * a.ldb + c];
}

__global__ void __launch_bounds__(kSThreads) small_gemm_kernel(const __grid_constant__ SmallArgs a) {
    __shared__ __align__(16) uint32_t As[kSM][kApitch];
    __shared__ __align__(16) uint32_t Bs[kSK][kBpitch];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const int m0 = blockIdx.y * kSM, n0 = blockIdx.x * kSN;
    // staging: 2048 values per operand slice, 8 per thread, mapped so that the
    // global reads are coalesced along the stored (fastest) dimension
    int32_t ra[8], rb[8];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int e = tid + j * kSThreads;
            if (a.tA) ra[j] = ld_a(a, m0 + e % kSM, k0 + e / kSM);      // A stored [k][m]: along m
            else ra[j] = ld_a(a, m0 + e / kSK, k0 + e % kSK);           // A stored [m][k]: along k
            if (a.tB) rb[j] = ld_b(a, k0 + e % kSK, n0 + e / kSK);      // B stored [n][k]: along k
            else rb[j] = ld_b(a, k0 + e / kSN, n0 + e % kSN);           // B stored [k][n]: along n
        }
    };
    auto stage = [&]() {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int e = tid + j * kSThreads;
            const uint32_t va = residue_i32(ra[j], a.M), vb = residue_i32(rb[j], a.M);
            if (a.tA) As[e % kSM][e / kSM] = va; else As[e / kSK][e % kSK] = va;
            if (a.tB) Bs[e % kSK][e / kSK] = vb; else Bs[e / kSN][e % kSN] = vb;
        }
    };
    int P[4][4][4];                     // [n-tile][byte product 00, 01, 10, 11][fragment]
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) P[i][j][e] = 0;
    fetch(0);
    for (int k0 = 0; k0 < a.k; k0 += kSK) {
        __syncthreads();                // the previous slice is consumed
        stage();
        __syncthreads();
        if (k0 + kSK < a.k) fetch(k0 + kSK);   // in flight during the products
        uint32_t alo[4], ahi[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {   // a0: row g, a1: row g + 8; a2, a3: k + 16
            const uint4 v = *reinterpret_cast<const uint4*>(&As[wm * 16 + g + ((q & 1) ? 8 : 0)][((q & 2) ? 16 : 0) + 4 * t]);
            split4(v.x, v.y, v.z, v.w, alo[q], ahi[q]);
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int c = wn * 32 + nt * 8 + g;
            uint32_t blo[2], bhi[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int kk = (q ? 16 : 0) + 4 * t;
                split4(Bs[kk][c], Bs[kk + 1][c], Bs[kk + 2][c], Bs[kk + 3][c], blo[q], bhi[q]);
            }
            imma(P[nt][0], alo[0], alo[1], alo[2], alo[3], blo[0], blo[1]);
            imma(P[nt][1], alo[0], alo[1], alo[2], alo[3], bhi[0], bhi[1]);
            imma(P[nt][2], ahi[0], ahi[1], ahi[2], ahi[3], blo[0], blo[1]);
            imma(P[nt][3], ahi[0], ahi[1], ahi[2], ahi[3], bhi[0], bhi[1]);
        }
    }
    // epilogue: R = P00 + 256 (P01 + P10) + 65536 P11 (exact, < 2^48), one
    // reduction, then alpha R + beta C mod p
    const uint32_t p = a.M.p;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int r = m0 + wm * 16 + g + ((e & 2) ? 8 : 0);
            const int c = n0 + wn * 32 + nt * 8 + 2 * t + (e & 1);
            if (r >= a.m || c >= a.n) continue;
            const unsigned long long S =
                static_cast<unsigned long long>(static_cast<uint32_t>(P[nt][0][e])) +
                (static_cast<unsigned long long>(static_cast<uint32_t>(P[nt][1][e]) + static_cast<uint32_t>(P[nt][2][e])) << 8) +
                (static_cast<unsigned long long>(static_cast<uint32_t>(P[nt][3][e])) << 16);
            uint32_t x = mulmod_shoup(residue_u64(S, a.mu64, p), a.M.alpha, a.M.alpha_sh, p);
            int32_t* cp = a.C + static_cast<int64_t>(r) * a.ldc + c;
            if (a.M.beta) x = addmod(x, mulmod_shoup(residue_i32(*cp, a.M), a.M.beta, a.M.beta_sh, p), p);
            *cp = static_cast<int32_t>(x);
        }
}

// Variant for internal callers whose A and B are canonical residues (LQUP's
// panel chain: outputs of earlier products), both not transposed, rows 16 B
// aligned: the slices are copied raw with cp.async into a 4-deep ring, so the
// whole K streams with several slices in flight (the register-staged kernel
// above waits one load latency per slice).
constexpr int kCStages = 4;
constexpr int kCApitch = kSK + 4, kCBpitch = kSN + 4;
constexpr int kCSmem = kCStages * (kSM * kCApitch + kSK * kCBpitch) * 4;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}

// The 64 x 64 output tile (m0, n0) of one canonical product: byte-split partial
// products accumulated in P (compute), then recombined, alpha/beta applied and
// stored (store).  Split so that a kernel may put a grid barrier in between
// (in-place products) or run several products in phases (small_chain_kernel).
__device__ __forceinline__ void canon_compute(const SmallArgs& a, int m0, int n0, int (&P)[4][4][4], uint32_t* csm) {
    uint32_t* As = csm;                                  // [kCStages][kSM][kCApitch]
    uint32_t* Bs = csm + kCStages * kSM * kCApitch;      // [kCStages][kSK][kCBpitch]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const int nsl = (a.k + kSK - 1) / kSK;
    auto issue = [&](int sl) {
        if (sl < nsl) {
            const int st = sl % kCStages, k0 = sl * kSK;
#pragma unroll
            for (int j = 0; j < 2; ++j) {                // A: 64 rows x 8 chunks of 4
                const int e = tid + j * kSThreads, r = e >> 3, kc = (e & 7) * 4;
                const int row = m0 + r, kk = k0 + kc;
                const int nb = (row < a.m && kk < a.k) ? 4 * min(4, a.k - kk) : 0;
                const int32_t* src = nb ? a.A + static_cast<int64_t>(row) * a.lda + kk : a.A;
                cp_async16(As + (st * kSM + r) * kCApitch + kc, src, nb);
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {                // B: 32 rows x 16 chunks of 4
                const int e = tid + j * kSThreads, r = e >> 4, cc = (e & 15) * 4;
                const int kk = k0 + r, col = n0 + cc;
                const int nb = (kk < a.k && col < a.n) ? 4 * min(4, a.n - col) : 0;
                const int32_t* src = nb ? a.B + static_cast<int64_t>(kk) * a.ldb + col : a.B;
                cp_async16(Bs + (st * kSK + r) * kCBpitch + cc, src, nb);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) P[i][j][e] = 0;
    for (int s = 0; s < kCStages - 1; ++s) issue(s);
    for (int sl = 0; sl < nsl; ++sl) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kCStages - 2) : "memory");
        if (a.reduce) {                                  // raw int32 inputs: this thread's own chunks of
            const int st = sl % kCStages;                // slice sl have landed -> residues (R3)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int e = tid + j * kSThreads;
                uint4* qa = reinterpret_cast<uint4*>(As + (st * kSM + (e >> 3)) * kCApitch + (e & 7) * 4);
                uint4* qb = reinterpret_cast<uint4*>(Bs + (st * kSK + (e >> 4)) * kCBpitch + (e & 15) * 4);
                uint4 va = *qa, vb = *qb;
                va.x = residue_i32(static_cast<int32_t>(va.x), a.M); va.y = residue_i32(static_cast<int32_t>(va.y), a.M);
                va.z = residue_i32(static_cast<int32_t>(va.z), a.M); va.w = residue_i32(static_cast<int32_t>(va.w), a.M);
                vb.x = residue_i32(static_cast<int32_t>(vb.x), a.M); vb.y = residue_i32(static_cast<int32_t>(vb.y), a.M);
                vb.z = residue_i32(static_cast<int32_t>(vb.z), a.M); vb.w = residue_i32(static_cast<int32_t>(vb.w), a.M);
                *qa = va;
                *qb = vb;
            }
        }
        __syncthreads();                                 // slice sl visible; slice sl-1's stage is free
        issue(sl + kCStages - 1);
        const uint32_t* A_ = As + (sl % kCStages) * kSM * kCApitch;
        const uint32_t* B_ = Bs + (sl % kCStages) * kSK * kCBpitch;
        uint32_t alo[4], ahi[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 v = *reinterpret_cast<const uint4*>(A_ + (wm * 16 + g + ((q & 1) ? 8 : 0)) * kCApitch +
                                                            ((q & 2) ? 16 : 0) + 4 * t);
            split4(v.x, v.y, v.z, v.w, alo[q], ahi[q]);
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int c = wn * 32 + nt * 8 + g;
            uint32_t blo[2], bhi[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int kk = (q ? 16 : 0) + 4 * t;
                split4(B_[kk * kCBpitch + c], B_[(kk + 1) * kCBpitch + c], B_[(kk + 2) * kCBpitch + c],
                       B_[(kk + 3) * kCBpitch + c], blo[q], bhi[q]);
            }
            imma(P[nt][0], alo[0], alo[1], alo[2], alo[3], blo[0], blo[1]);
            imma(P[nt][1], alo[0], alo[1], alo[2], alo[3], bhi[0], bhi[1]);
            imma(P[nt][2], ahi[0], ahi[1], ahi[2], ahi[3], blo[0], blo[1]);
            imma(P[nt][3], ahi[0], ahi[1], ahi[2], ahi[3], bhi[0], bhi[1]);
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();                                     // the shared stages may be reused by the caller
}

__device__ __forceinline__ void canon_store(const SmallArgs& a, int m0, int n0, const int (&P)[4][4][4]) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const uint32_t p = a.M.p;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int r = m0 + wm * 16 + g + ((e & 2) ? 8 : 0);
            const int c = n0 + wn * 32 + nt * 8 + 2 * t + (e & 1);
            if (r >= a.m || c >= a.n) continue;
            const unsigned long long S =
                static_cast<unsigned long long>(static_cast<uint32_t>(P[nt][0][e])) +
                (static_cast<unsigned long long>(static_cast<uint32_t>(P[nt][1][e]) + static_cast<uint32_t>(P[nt][2][e])) << 8) +
                (static_cast<unsigned long long>(static_cast<uint32_t>(P[nt][3][e])) << 16);
            uint32_t x = mulmod_shoup(residue_u64(S, a.mu64, p), a.M.alpha, a.M.alpha_sh, p);
            int32_t* cp = a.C + static_cast<int64_t>(r) * a.ldc + c;
            if (a.M.beta) x = addmod(x, mulmod_shoup(residue_i32(*cp, a.M), a.M.beta, a.M.beta_sh, p), p);
            *cp = static_cast<int32_t>(x);
        }
}

__global__ void __launch_bounds__(kSThreads) small_gemm_canon_kernel(const __grid_constant__ SmallArgs a) {
    extern __shared__ __align__(16) uint32_t csm[];
    const int m0 = blockIdx.y * kSM, n0 = blockIdx.x * kSN;
    int P[4][4][4];
    canon_compute(a, m0, n0, P, csm);
    if (a.alias) cooperative_groups::this_grid().sync();   // every CTA has read its A, B before C is written
    canon_store(a, m0, n0, P);
}

// LQUP's panel chain in one cooperative launch (lqup.cu): phase 1
// runs products 0 and 1 (both in place: every CTA computes its tile, a grid
// barrier, then stores), phase 2 product 2, which reads their outputs.  Each
// product is at most 128 x 128 (four 64 x 64 tiles): CTAs 0-3 take product 0's
// tiles, 4-7 product 1's, and CTAs 0-3 product 2's.
struct ChainArgs {
    SmallArgs p[3];
};

__global__ void __launch_bounds__(kSThreads) small_chain_kernel(const __grid_constant__ ChainArgs c) {
    extern __shared__ __align__(16) uint32_t csm[];
    const int b = blockIdx.x;
    int P[4][4][4];
    {
        const SmallArgs& a = c.p[b >> 2];
        const int m0 = ((b >> 1) & 1) * kSM, n0 = (b & 1) * kSN;
        const bool live = m0 < a.m && n0 < a.n;
        if (live) canon_compute(a, m0, n0, P, csm);
        cooperative_groups::this_grid().sync();            // products 0, 1 read before they are written
        if (live) canon_store(a, m0, n0, P);
    }
    cooperative_groups::this_grid().sync();                // their outputs are product 2's operands
    if (b < 4) {
        const SmallArgs& a = c.p[2];
        const int m0 = (b >> 1) * kSM, n0 = (b & 1) * kSN;
        if (m0 < a.m && n0 < a.n) {
            canon_compute(a, m0, n0, P, csm);
            canon_store(a, m0, n0, P);
        }
    }
}


// Wider fields (2^16 <= p < 2^31), canonical operands: L = 3 or 4 bytes per
// residue and all L^2 byte products per K slice (each exact in s32 for K <= 33025),
// recombined at the end as sum_{i,j} (P_ij mod p) (256^(i+j) mod p) mod p.  The
// L^2 accumulators need a narrower tile: 64 x 16 per CTA, one m16n8 tile per warp.
constexpr int kWN = 16;
constexpr int kWBpitch = kWN + 4;
constexpr int kWSmem = kCStages * (kSM * kCApitch + kSK * kWBpitch) * 4;

__device__ __forceinline__ uint32_t pack_byte(uint32_t x, uint32_t y, uint32_t z, uint32_t w, int b) {
    const uint32_t s = static_cast<uint32_t>(b) | (static_cast<uint32_t>(4 + b) << 4);
    return __byte_perm(__byte_perm(x, y, s), __byte_perm(z, w, s), 0x5410);
}

// The 64 x 16 tile (m0, n0) of one wide-field product, split into compute and
// store like canon_compute / canon_store.
template <int L>
__device__ __forceinline__ void wide_compute(const SmallArgs& a, int m0, int n0, int (&P)[L * L][4], uint32_t* wsm) {
    uint32_t* As = wsm;                                  // [kCStages][kSM][kCApitch]
    uint32_t* Bs = wsm + kCStages * kSM * kCApitch;      // [kCStages][kSK][kWBpitch]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const int nsl = (a.k + kSK - 1) / kSK;
    auto issue = [&](int sl) {
        if (sl < nsl) {
            const int st = sl % kCStages, k0 = sl * kSK;
#pragma unroll
            for (int j = 0; j < 2; ++j) {                // A: 64 rows x 8 chunks of 4
                const int e = tid + j * kSThreads, r = e >> 3, kc = (e & 7) * 4;
                const int row = m0 + r, kk = k0 + kc;
                const int nb = (row < a.m && kk < a.k) ? 4 * min(4, a.k - kk) : 0;
                const int32_t* src = nb ? a.A + static_cast<int64_t>(row) * a.lda + kk : a.A;
                cp_async16(As + (st * kSM + r) * kCApitch + kc, src, nb);
            }
            if (tid < kSK * kWN / 4) {                  // B: 32 rows x 4 chunks of 4
                const int r = tid >> 2, cc = (tid & 3) * 4;
                const int kk = k0 + r, col = n0 + cc;
                const int nb = (kk < a.k && col < a.n) ? 4 * min(4, a.n - col) : 0;
                const int32_t* src = nb ? a.B + static_cast<int64_t>(kk) * a.ldb + col : a.B;
                cp_async16(Bs + (st * kSK + r) * kWBpitch + cc, src, nb);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#pragma unroll
    for (int q = 0; q < L * L; ++q)
#pragma unroll
        for (int e = 0; e < 4; ++e) P[q][e] = 0;
    for (int s = 0; s < kCStages - 1; ++s) issue(s);
    for (int sl = 0; sl < nsl; ++sl) {
        asm volatile("cp.async.wait_group %0;" ::"n"(kCStages - 2) : "memory");
        __syncthreads();
        issue(sl + kCStages - 1);
        const uint32_t* A_ = As + (sl % kCStages) * kSM * kCApitch;
        const uint32_t* B_ = Bs + (sl % kCStages) * kSK * kWBpitch;
        uint32_t av[4][4], bv[2][4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 v = *reinterpret_cast<const uint4*>(A_ + (wm * 16 + g + ((q & 1) ? 8 : 0)) * kCApitch +
                                                            ((q & 2) ? 16 : 0) + 4 * t);
            av[q][0] = v.x; av[q][1] = v.y; av[q][2] = v.z; av[q][3] = v.w;
        }
        const int c = wn * 8 + g;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int kk = (q ? 16 : 0) + 4 * t;
#pragma unroll
            for (int i = 0; i < 4; ++i) bv[q][i] = B_[(kk + i) * kWBpitch + c];
        }
#pragma unroll
        for (int i = 0; i < L; ++i) {
            const uint32_t a0 = pack_byte(av[0][0], av[0][1], av[0][2], av[0][3], i);
            const uint32_t a1 = pack_byte(av[1][0], av[1][1], av[1][2], av[1][3], i);
            const uint32_t a2 = pack_byte(av[2][0], av[2][1], av[2][2], av[2][3], i);
            const uint32_t a3 = pack_byte(av[3][0], av[3][1], av[3][2], av[3][3], i);
#pragma unroll
            for (int j = 0; j < L; ++j) {
                const uint32_t b0 = pack_byte(bv[0][0], bv[0][1], bv[0][2], bv[0][3], j);
                const uint32_t b1 = pack_byte(bv[1][0], bv[1][1], bv[1][2], bv[1][3], j);
                imma(P[i * L + j], a0, a1, a2, a3, b0, b1);
            }
        }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();                                     // the shared stages may be reused by the caller
}

template <int L>
__device__ __forceinline__ void wide_store(const SmallArgs& a, int m0, int n0, const int (&P)[L * L][4]) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const uint32_t p = a.M.p;
    uint32_t w[2 * L - 1];                               // 256^s mod p
    w[0] = 1u % p;
#pragma unroll
    for (int q = 1; q < 2 * L - 1; ++q) w[q] = residue_u64(static_cast<unsigned long long>(w[q - 1]) * 256u, a.mu64, p);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const int r = m0 + wm * 16 + g + ((e & 2) ? 8 : 0);
        const int cc = n0 + wn * 8 + 2 * t + (e & 1);
        if (r >= a.m || cc >= a.n) continue;
        uint32_t S = 0u;
#pragma unroll
        for (int i = 0; i < L; ++i)
#pragma unroll
            for (int j = 0; j < L; ++j)
                S = residue_u64(static_cast<unsigned long long>(S) +
                                    static_cast<unsigned long long>(static_cast<uint32_t>(P[i * L + j][e])) * w[i + j],
                                a.mu64, p);
        uint32_t x = mulmod_shoup(S, a.M.alpha, a.M.alpha_sh, p);
        int32_t* cp = a.C + static_cast<int64_t>(r) * a.ldc + cc;
        if (a.M.beta) x = addmod(x, mulmod_shoup(residue_i32(*cp, a.M), a.M.beta, a.M.beta_sh, p), p);
        *cp = static_cast<int32_t>(x);
    }
}

template <int L>
__global__ void __launch_bounds__(kSThreads) small_gemm_wide_kernel(const __grid_constant__ SmallArgs a) {
    extern __shared__ __align__(16) uint32_t wsm[];
    const int m0 = blockIdx.y * kSM, n0 = blockIdx.x * kWN;
    int P[L * L][4];
    wide_compute<L>(a, m0, n0, P, wsm);
    if (a.alias) cooperative_groups::this_grid().sync();   // every CTA has read its A, B before C is written
    wide_store<L>(a, m0, n0, P);
}

// small_chain_kernel for 2^16 <= p < 2^31: 64 x 16 tiles, 16 per 128 x 128
// product; CTAs 0-15 product 0, 16-31 product 1, then CTAs 0-15 product 2.
template <int L>
__global__ void __launch_bounds__(kSThreads) small_chain_wide_kernel(const __grid_constant__ ChainArgs c) {
    extern __shared__ __align__(16) uint32_t wsm[];
    const int b = blockIdx.x;
    int P[L * L][4];
    {
        const SmallArgs& a = c.p[b >> 4];
        const int m0 = ((b >> 3) & 1) * kSM, n0 = (b & 7) * kWN;
        const bool live = m0 < a.m && n0 < a.n;
        if (live) wide_compute<L>(a, m0, n0, P, wsm);
        cooperative_groups::this_grid().sync();
        if (live) wide_store<L>(a, m0, n0, P);
    }
    cooperative_groups::this_grid().sync();
    if (b < 16) {
        const SmallArgs& a = c.p[2];
        const int m0 = (b >> 3) * kSM, n0 = (b & 7) * kWN;
        if (m0 < a.m && n0 < a.n) {
            wide_compute<L>(a, m0, n0, P, wsm);
            wide_store<L>(a, m0, n0, P);
        }
    }
}

}  // namespace

// Plain launch, or (alias) a cooperative one with every CTA co-resident for the
// grid barrier; FF_ERR_INTERNAL if the grid cannot be co-resident (the caller
// then takes the tcgen05 path).
int launch_small(const void* fn, dim3 grid, int smem, SmallArgs& a, bool alias, cudaStream_t st) {
    if (set_smem_attr(fn, smem) != cudaSuccess) return FF_ERR_CUDA;
    void* args[] = {&a};
    if (!alias) {
        note_launch();
        prof_gemm_begin(st);
        const cudaError_t le = cudaLaunchKernel(fn, grid, dim3(kSThreads), args, static_cast<size_t>(smem), st);
        prof_gemm_end(st);
        if (le != cudaSuccess) {
            cudaGetLastError();
            return FF_ERR_CUDA;
        }
        return 0;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kSThreads, static_cast<size_t>(smem)) != cudaSuccess) {
        cudaGetLastError();
        return FF_ERR_INTERNAL;
    }
    if (static_cast<int64_t>(per_sm) * num_sms() < static_cast<int64_t>(grid.x) * grid.y) return FF_ERR_INTERNAL;
    note_launch();
    prof_gemm_begin(st);
    const cudaError_t le = cudaLaunchCooperativeKernel(fn, grid, dim3(kSThreads), args, static_cast<size_t>(smem), st);
    prof_gemm_end(st);
    if (le != cudaSuccess) {
        cudaGetLastError();
        return FF_ERR_CUDA;
    }
    return 0;
}

bool small_wide_ok(const Plan& pl, bool tA, bool tB, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                   const int32_t* B, int64_t ldb) {
    return pl.canonical_ab && !tA && !tB && pl.mp.p >= 65536u && k > 0 && k <= 32768 && m > 0 && n > 0 &&
           m < (1ll << 30) && n < (1ll << 30) && (lda % 4) == 0 && (ldb % 4) == 0 &&
           (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
}

int launch_gemm_small_wide(const Plan& pl, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                           const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, bool alias, cudaStream_t st) {
    SmallArgs a;
    a.M = pl.mp;
    a.mu64 = static_cast<unsigned long long>((static_cast<unsigned __int128>(1) << 64) / pl.mp.p);
    a.A = A; a.B = B; a.C = C;
    a.lda = lda; a.ldb = ldb; a.ldc = ldc;
    a.m = static_cast<int32_t>(m); a.n = static_cast<int32_t>(n); a.k = static_cast<int32_t>(k);
    a.tA = 0; a.tB = 0;
    const dim3 grid(static_cast<unsigned>((n + kWN - 1) / kWN), static_cast<unsigned>((m + kSM - 1) / kSM));
    if (grid.y > 65535u) return FF_ERR_INTERNAL;
    a.alias = alias ? 1 : 0;
    a.reduce = 0;
    const void* fn = pl.mp.p < (1u << 24) ? reinterpret_cast<const void*>(small_gemm_wide_kernel<3>)
                                          : reinterpret_cast<const void*>(small_gemm_wide_kernel<4>);
    return launch_small(fn, grid, kWSmem, a, alias, st);
}

bool small_canon_ok(const Plan& pl, bool tA, bool tB, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                    const int32_t* B, int64_t ldb) {
    return pl.canonical_ab && !tA && !tB && pl.mp.p < 65536u && k > 0 && k <= 32768 && m > 0 && n > 0 &&
           m < (1ll << 30) && n < (1ll << 30) && (lda % 4) == 0 && (ldb % 4) == 0 &&
           (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0;
}

int launch_gemm_small_canon(const Plan& pl, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                            const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, bool alias, cudaStream_t st,
                            bool reduce) {
    SmallArgs a;
    a.M = pl.mp;
    a.mu64 = static_cast<unsigned long long>((static_cast<unsigned __int128>(1) << 64) / pl.mp.p);
    a.A = A; a.B = B; a.C = C;
    a.lda = lda; a.ldb = ldb; a.ldc = ldc;
    a.m = static_cast<int32_t>(m); a.n = static_cast<int32_t>(n); a.k = static_cast<int32_t>(k);
    a.tA = 0; a.tB = 0;
    const dim3 grid(static_cast<unsigned>((n + kSN - 1) / kSN), static_cast<unsigned>((m + kSM - 1) / kSM));
    if (grid.y > 65535u) return FF_ERR_INTERNAL;
    a.alias = alias ? 1 : 0;
    a.reduce = reduce ? 1 : 0;
    return launch_small(reinterpret_cast<const void*>(small_gemm_canon_kernel), grid, kCSmem, a, alias, st);
}

int launch_small_chain(const Plan& pl0, const Plan& pl2, const SmallChainProduct (&pr)[3], cudaStream_t st) {
    ChainArgs c;
    for (int i = 0; i < 3; ++i) {
        const Plan& pl = i < 2 ? pl0 : pl2;
        SmallArgs& a = c.p[i];
        const int64_t mm = pr[i].m > 0 ? pr[i].m : 1, nn = pr[i].n > 0 ? pr[i].n : 1;
        const bool ok = pl.mp.p < 65536u
                            ? small_canon_ok(pl, false, false, mm, nn, pr[i].k, pr[i].A, pr[i].lda, pr[i].B, pr[i].ldb)
                            : small_wide_ok(pl, false, false, mm, nn, pr[i].k, pr[i].A, pr[i].lda, pr[i].B, pr[i].ldb);
        if (pr[i].m > 2 * kSM || pr[i].n > 2 * kSN || pr[i].m < 0 || pr[i].n < 0 || pr[i].k <= 0 || pr[i].k > 32768 ||
            !ok || (pl.mp.p < 65536u) != (pl0.mp.p < 65536u))
            return FF_ERR_INTERNAL;
        a.M = pl.mp;
        a.mu64 = static_cast<unsigned long long>((static_cast<unsigned __int128>(1) << 64) / pl.mp.p);
        a.A = pr[i].A; a.B = pr[i].B; a.C = pr[i].C;
        a.lda = pr[i].lda; a.ldb = pr[i].ldb; a.ldc = pr[i].ldc;
        a.m = static_cast<int32_t>(pr[i].m); a.n = static_cast<int32_t>(pr[i].n); a.k = static_cast<int32_t>(pr[i].k);
        a.tA = 0; a.tB = 0;
        a.alias = 1;
        a.reduce = 0;
    }
    const bool narrow = pl0.mp.p < 65536u;
    const void* fn = narrow ? reinterpret_cast<const void*>(small_chain_kernel)
                   : pl0.mp.p < (1u << 24) ? reinterpret_cast<const void*>(small_chain_wide_kernel<3>)
                                           : reinterpret_cast<const void*>(small_chain_wide_kernel<4>);
    const int smem = narrow ? kCSmem : kWSmem;
    if (set_smem_attr(fn, smem) != cudaSuccess) return FF_ERR_CUDA;
    void* args[] = {&c};
    note_launch();
    prof_gemm_begin(st);
    const cudaError_t le = cudaLaunchCooperativeKernel(fn, dim3(narrow ? 8 : 32), dim3(kSThreads), args,
                                                       static_cast<size_t>(smem), st);
    prof_gemm_end(st);
    if (le != cudaSuccess) {
        cudaGetLastError();
        return FF_ERR_CUDA;
    }
    return 0;
}

bool small_stream_ok(const Plan& pl, bool tA, bool tB, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                     const int32_t* B, int64_t ldb) {
    return !tA && !tB && pl.mp.p < 65536u && k > 0 && k <= 32768 && m > 0 && n > 0 && m < (1ll << 30) &&
           n < (1ll << 30) && (lda % 4) == 0 && (ldb % 4) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(B) & 15) == 0;
}

bool small_path_ok(const Plan& pl, int64_t m, int64_t n, int64_t k) {
    return pl.mp.p < 65536u && k > 0 && k <= 32768 && m > 0 && n > 0 && m < (1ll << 30) && n < (1ll << 30);
}

int launch_gemm_small(const Plan& pl, bool tA, bool tB, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                      const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, cudaStream_t st) {
    if (!small_path_ok(pl, m, n, k)) return FF_ERR_INTERNAL;
    SmallArgs a;
    a.M = pl.mp;
    a.mu64 = static_cast<unsigned long long>((static_cast<unsigned __int128>(1) << 64) / pl.mp.p);
    a.A = A; a.B = B; a.C = C;
    a.lda = lda; a.ldb = ldb; a.ldc = ldc;
    a.m = static_cast<int32_t>(m); a.n = static_cast<int32_t>(n); a.k = static_cast<int32_t>(k);
    a.tA = tA ? 1 : 0; a.tB = tB ? 1 : 0;
    a.alias = 0;
    a.reduce = 0;
    const dim3 grid(static_cast<unsigned>((n + kSN - 1) / kSN), static_cast<unsigned>((m + kSM - 1) / kSM));
    if (grid.y > 65535u) return FF_ERR_INTERNAL;
    note_launch();
    prof_gemm_begin(st);
    small_gemm_kernel<<<grid, kSThreads, 0, st>>>(a);
    prof_gemm_end(st);
    return cudaGetLastError() == cudaSuccess ? 0 : FF_ERR_CUDA;
}

}  // namespace ff
