// modp.cuh -- 32-bit residue arithmetic used by the encoder and the GEMM epilogue.
//
// The paper's "floating point inverse" representation:
// "precompute the inverse of the characteristic p ... only two floating point
// multiplications and some rounding are necessary.  However, floating point
// rounding may induce a +-1 error and then an adjustment is required".  We use
// the integer form of that idea: a precomputed fixed-point inverse (Barrett's
// mu = floor(2^32/p), Shoup's w' = floor(w 2^32/p)), one __umulhi, and one
// conditional correction.  Valid for 2 <= p < 2^31.
#pragma once
#include <cstdint>

#include "internal.h"

namespace ff {

// Any int32 -> its Euclidean residue in [0, p).
// x = a + 2^31 in [0, 2^32); q = floor(x mu / 2^32) is floor(x/p) or one less,
// so x - q p is in [0, 2p); then remove 2^31 mod p.
__device__ __forceinline__ uint32_t residue_i32(int32_t a, const ModP& M) {
    const uint32_t x = static_cast<uint32_t>(a) ^ 0x80000000u;
    const uint32_t q = __umulhi(x, M.mu);
    uint32_t r = x - q * M.p;
    if (r >= M.p) r -= M.p;
    return r >= M.off31 ? r - M.off31 : r + (M.p - M.off31);
}

// a * w mod p for a, w in [0, p), w_sh = floor(w 2^32 / p)  (Shoup).
__device__ __forceinline__ uint32_t mulmod_shoup(uint32_t a, uint32_t w, uint32_t w_sh, uint32_t p) {
    const uint32_t q = __umulhi(a, w_sh);
    uint32_t r = a * w - q * p;
    return r >= p ? r - p : r;
}

// [0,p) -> centred [-(p-1)/2, (p-1)/2]  (balanced representation).
__device__ __forceinline__ int32_t centre(uint32_t r, const ModP& M) {
    return r > M.half ? static_cast<int32_t>(r) - static_cast<int32_t>(M.p) : static_cast<int32_t>(r);
}

// Centred residues of N values in place.  Canonical inputs (every value already
// in [0, p): the usual case, e.g. all five BASELINE configs) take the short path
// -- one compare each, then centre -- and any other int32 the Barrett reduction;
// the branch is per thread and group, so only a thread holding a non-canonical
// value pays for the reduction.
template <int N>
__device__ __forceinline__ void centre_all(int32_t (&x)[N], const ModP& M) {
    bool canon = true;
#pragma unroll
    for (int i = 0; i < N; ++i) canon &= static_cast<uint32_t>(x[i]) < M.p;
    if (canon) {
#pragma unroll
        for (int i = 0; i < N; ++i) x[i] = centre(static_cast<uint32_t>(x[i]), M);
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) x[i] = centre(residue_i32(x[i], M), M);
    }
}

// Intermediate write-back value: a centred-ish representative of (a * w) mod p
// for the s32 accumulator a and w in {1, 256} (Horner scaling), with the
// quotient estimated through the fp32 reciprocal w/p (PAPER.md l.125-127:
// "precompute the inverse of the characteristic p within a floating point
// number ... rounding may induce a +-1 error").  No correction is applied:
// v = a*w - q*p is exact in wrapping 32-bit arithmetic and
// |v| <= p/2 + 385*w, a carry the planner's k-block bound
// includes.  Used only between steps; the final output uses residue_i32.
__device__ __forceinline__ int32_t reduce_approx(int32_t a, int32_t w, float w_over_p, int32_t p) {
    const int32_t q = __float2int_rn(__int2float_rn(a) * w_over_p);
    return static_cast<int32_t>(static_cast<uint32_t>(a) * static_cast<uint32_t>(w) -
                                static_cast<uint32_t>(q) * static_cast<uint32_t>(p));
}

// Same purpose with integer instructions only (no int<->float conversions,
// which issue at quarter rate): q = floor(a * m / 2^32) with
// m = round(w 2^32 / p) (clamped to 2^31-1) estimates a*w/p within [-1.5, +0.5],
// so v = a*w - q*p (wrapping 32-bit) lies in [-p/2, 3p/2].  Valid while
// 2p < 2^31 (the planner uses it for p < 2^29); DESIGN.md §4.4.
__device__ __forceinline__ int32_t reduce_mulhi(int32_t a, uint32_t w, int32_t m, uint32_t p) {
    const int32_t q = __mulhi(a, m);
    return static_cast<int32_t>(static_cast<uint32_t>(a) * w - static_cast<uint32_t>(q) * p);
}

// ---- small moduli q <= 256 of the multi-modular scheme

// Any int32 -> its residue in [0, q), the same Barrett form as residue_i32
// (mu = floor(2^32/q), off31 = 2^31 mod q).
__device__ __forceinline__ uint32_t residue_small(int32_t a, uint32_t q, uint32_t mu, uint32_t off31) {
    const uint32_t x = static_cast<uint32_t>(a) ^ 0x80000000u;
    uint32_t r = x - __umulhi(x, mu) * q;
    if (r >= q) r -= q;
    return r >= off31 ? r - off31 : r + (q - off31);
}

// r in [0, q) -> centred representative: r - q if r > (q-1)/2 (q = 256: [-128, 127]).
__device__ __forceinline__ int32_t centre_small(uint32_t r, uint32_t q, uint32_t half) {
    return r > half ? static_cast<int32_t>(r) - static_cast<int32_t>(q) : static_cast<int32_t>(r);
}

// (r v) mod q for r, v in [0, q): r v < 2^16, one Barrett step + one correction.
__device__ __forceinline__ uint32_t mulmod_small(uint32_t r, uint32_t v, uint32_t q, uint32_t mu) {
    const uint32_t y = r * v;
    uint32_t u = y - __umulhi(y, mu) * q;
    return u >= q ? u - q : u;
}

// x mod p for x < 2^64 (Barrett with mu64 = floor(2^64/p): the quotient
// estimate is floor(x/p) or one less, so one correction).
__device__ __forceinline__ uint32_t residue_u64(unsigned long long x, unsigned long long mu64, uint32_t p) {
    const unsigned long long q = __umul64hi(x, mu64);
    unsigned long long r = x - q * p;
    return static_cast<uint32_t>(r >= p ? r - p : r);
}

// Any int32 -> its Euclidean residue in [0, p), with mu64 = floor(2^64 / p):
// x + p 2^31 > 0 and < 2^62, one Barrett step.
__device__ __forceinline__ uint32_t residue_i32_64(int32_t x, unsigned long long mu64, uint32_t p) {
    return residue_u64(static_cast<unsigned long long>(static_cast<long long>(x) + (static_cast<long long>(p) << 31)),
                       mu64, p);
}

__device__ __forceinline__ uint32_t addmod(uint32_t a, uint32_t b, uint32_t p) {
    const uint32_t s = a + b;  // < 2p < 2^32
    return s >= p ? s - p : s;
}

}  // namespace ff
