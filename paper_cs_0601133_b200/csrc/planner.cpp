// planner.cpp -- host planner: limb scheme, digit bounds, k-block length.
//
// The paper bounds delayed reduction by the accumulator width: for centred
// residues, lambda ((p-1)/2)^2 < 2^(gamma-1) (Eq. (2)), so
// that ceil(n/lambda) reductions suffice per dot product (l.159).  Here the
// products are of int8 limbs d_i in [-D_i, D_i] and the accumulator is the
// s32 TMEM cell (gamma = 32), which also carries one centred residue written
// back between k-blocks / weight groups (|carry| <= (p-1)/2).  So a k-block
// of kb terms of weight group w = i+j is safe iff
//
//      kb * B_w + (p-1)/2 <= 2^31 - 1,      B_w = sum_{i+j=w} D_i D_j,
//
// giving kb_max = floor((2^31 - 1 - carry_max) / max_w B_w)  (
// the "one extra carried term" form matches the paper's own t_update values,
// l.524-527, which satisfy (t+1)(p-1)^2 < 2^53 exactly).
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace ff {

namespace {

// Digit stripping.  Both maps are monotone non-decreasing in
// c, so the range of the top digit is [top(-half), top(half)].
//   S: d = ((c+128) mod 256) - 128, c <- (c - d)/256 = floor((c+128)/256)
//   T: d = c mod 256 (u8),          c <- floor(c/256)
int64_t floor_div(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b) != 0 && ((a < 0) != (b < 0))) --q;
    return q;
}

int64_t strip(int64_t c, int scheme) {
    return scheme == FF_SCHEME_S ? floor_div(c + 128, 256) : floor_div(c, 256);
}

int64_t top_digit(int64_t c, int L, int scheme) {
    for (int i = 0; i + 1 < L; ++i) c = strip(c, scheme);
    return c;
}

bool feasible(int64_t half, int64_t neg, int L, int scheme) {
    int64_t hi = top_digit(half, L, scheme), lo = top_digit(-neg, L, scheme);
    return hi <= 127 && lo >= -128;
}

int min_limbs(int64_t half, int64_t neg, int scheme) {
    for (int L = 1; L <= kMaxLimbs; ++L)
        if (feasible(half, neg, L, scheme)) return L;
    return 0;
}

uint32_t shoup(uint32_t w, uint32_t p) {
    return (uint32_t)(((uint64_t)w << 32) / p);
}

typedef unsigned __int128 u128;

uint32_t gcd32(uint32_t a, uint32_t b) {
    while (b) { const uint32_t t = a % b; a = b; b = t; }
    return a;
}

// x^-1 mod q for gcd(x, q) = 1 (extended Euclid).
uint32_t inv_mod(uint32_t x, uint32_t q) {
    int64_t r0 = q, r1 = x % q, s0 = 0, s1 = 1;
    while (r1 != 0) {
        const int64_t qq = r0 / r1, t = r0 - qq * r1, u = s0 - qq * s1;
        r0 = r1; r1 = t; s0 = s1; s1 = u;
    }
    return (uint32_t)(((s0 % (int64_t)q) + q) % q);
}

int ceil_log2_u128(u128 x) {   // smallest e with 2^e >= x (x >= 1)
    int e = 0;
    while (((u128)1 << e) < x) ++e;
    return e;
}

int floor_log2_u128(u128 x) {  // largest e with 2^e <= x (x >= 1)
    int e = 0;
    while (e < 127 && ((u128)1 << (e + 1)) <= x) ++e;
    return e;
}

// Multi-modular moduli.  The exact integer dot product X of
// two centred residue vectors of length k satisfies |X| <= k cmax^2; it is
// recovered from its residues modulo pairwise-coprime q_i <= 256 when
// M = prod q_i >= 4 k cmax^2 (so |X| / M <= 1/4: the CRT quotient is then the
// nearest integer to sum_i u_i / q_i with a 1/4 margin for its fixed-point
// evaluation).  Greedy from 256 down: the fewest moduli (each one int8 GEMM).
// Returns the count (0 if more than kMaxMod would be needed).
int crt_select(int64_t cmax, int64_t k, uint32_t* q, u128* Mout, u128* Bout) {
    const u128 kk = (u128)(k > 0 ? k : 1);
    const u128 B = (u128)4 * kk * (u128)cmax * (u128)cmax;
    u128 M = 1;
    int n = 0;
    for (uint32_t c = 256; c >= 2 && M < B; --c) {
        bool ok = true;
        for (int i = 0; i < n && ok; ++i) ok = gcd32(c, q[i]) == 1;
        if (!ok) continue;
        if (n == kMaxMod) return 0;
        q[n++] = c;
        M *= c;
    }
    if (M < B) return 0;
    if (n == 0) { q[n++] = 256; M = 256; }
    *Mout = M;
    *Bout = B;
    return n;
}

// Fill the CRT part of a plan (one group = one modulus = one pair (i, i)).
int make_crt_plan(uint32_t p, int64_t k, const ff_opts& o, int64_t cmax, Plan& pl) {
    ff_plan_info& I = pl.info;
    uint32_t q[kMaxMod];
    u128 M = 0, B = 0;
    const int nq = crt_select(cmax, k, q, &M, &B);
    if (nq == 0) return FF_ERR_OPTS;
    pl.crt = true;
    I.scheme = FF_SCHEME_CRT;
    I.L = nq;
    I.groups = nq;
    I.nmod = nq;
    I.log2_M_floor = floor_log2_u128(M);
    I.log2_bound_ceil = ceil_log2_u128(B);
    int64_t bmax = 0;
    for (int i = 0; i < nq; ++i) {
        I.moduli[i] = q[i];
        const int64_t D = q[i] / 2;            // |centred residue| <= q/2 (q = 256: [-128, 127])
        if (i < 4) { I.digit_max[i] = (int32_t)D; I.limb_signed[i] = 1; }
        if (i < 7) I.group_bound[i] = D * D;
        if (D * D > bmax) bmax = D * D;
    }
    I.group_bound_max = bmax;
    // The carry written back between k-blocks is a centred residue mod q_i.
    I.carry_max = q[0] / 2;
    I.kb_max = (((int64_t)1 << 31) - 1 - I.carry_max) / bmax;
    pl.korder = 1;
    I.korder = 1;
    int64_t kb = I.kb_max;
    if (o.kb_override > 0) {
        if (o.kb_override > I.kb_max || o.kb_override < kBK) return FF_ERR_OPTS;
        kb = o.kb_override;
    }
    kb = (kb / kBK) * kBK;
    I.kb = kb;
    I.k_pad = (k + 15) / 16 * 16;
    I.num_kblocks = k > 0 ? (k + kb - 1) / kb : 0;
    // Groups are processed from index G-1 down to 0 (as the limb groups): the
    // last one (modulus 0) is the final step that reconstructs.
    for (int i = 0; i < nq; ++i) {
        pl.group_first[i] = i;
        pl.group_len[i] = 1;
        pl.pair_i[i] = i;
        pl.pair_j[i] = i;
    }
    pl.npairs = nq;
    CrtConsts& C = pl.cc;
    C.nq = nq;
    const u128 Mp = M % p;
    C.Mneg = (uint32_t)((p - (uint32_t)Mp) % p);
    C.mu64 = (unsigned long long)((((u128)1) << 64) / p);
    for (int i = 0; i < nq; ++i) {
        const uint32_t qi = q[i];
        const u128 Mi = M / qi;
        C.q[i] = qi;
        C.mu[i] = (uint32_t)((((uint64_t)1) << 32) / qi);
        C.off31[i] = (uint32_t)((((uint64_t)1) << 31) % qi);
        C.half[i] = (qi - 1) / 2;
        C.v[i] = inv_mod((uint32_t)(Mi % qi), qi);
        C.W[i] = (uint32_t)(Mi % p);
        C.R[i] = (uint32_t)(((((uint64_t)1) << 25) / qi + 1) / 2);   // round(2^24 / q)
        C.fq[i] = (float)qi;
        C.finv[i] = (float)(1.0 / (double)qi);
        C.fw15[i] = (float)(32768u % qi);
    }
    return 0;
}

// The paper-literal fp64 engine: Eq. (2) with gamma = 53,
// lambda ((p-1)/2)^2 < 2^52, lambda >= 4 (one DMMA k-step);
// the accumulator also carries one reduced value (|r| <= p), which the factor-2
// headroom of 2^52 < 2^53 covers.  kb is a multiple of 4 (the DMMA k).
int make_f64_plan(int64_t k, const ff_opts& o, int64_t cmax, Plan& pl) {
    ff_plan_info& I = pl.info;
    const int64_t c2 = cmax * cmax;
    const int64_t lam = c2 > 0 ? ((((int64_t)1) << 52) - 1) / c2 : ((int64_t)1 << 40);
    if (lam < 4) return FF_ERR_OPTS;
    pl.fp64 = true;
    I.scheme = FF_SCHEME_FP64;
    I.L = 1;
    I.groups = 1;
    I.digit_max[0] = (int32_t)cmax;
    I.limb_signed[0] = 1;
    I.group_bound[0] = c2;
    I.group_bound_max = c2;
    I.carry_max = 2 * cmax + 1;
    I.kb_max = lam;
    int64_t kb = lam;
    if (o.kb_override > 0) {
        if ((o.kb_override > lam && !o.debug_unchecked_kb) || o.kb_override < 4) return FF_ERR_OPTS;
        kb = o.kb_override;
    }
    kb = (kb / 4) * 4;
    if (kb > ((int64_t)1 << 30)) kb = (int64_t)1 << 30;
    I.kb = kb;
    I.k_pad = (k + 15) / 16 * 16;
    I.num_kblocks = k > 0 ? (k + kb - 1) / kb : 0;
    pl.korder = 1;
    I.korder = 1;
    pl.npairs = 0;
    // Corollary 3.4, exact form (reading R21): l
    // recursive Winograd levels without any reduction are safe while
    // floor(k / 2^l) v_l^2 < 2^53, v_l = 3^l cmax (Theorem 3.1 on the balanced
    // range [-cmax, cmax]), i.e. for k < k_winograd[l] = ceil(2^53 / v_l^2) 2^l.
    for (int l = 1; l <= 3; ++l) {
        const u128 v = (u128)cmax * (l == 1 ? 3 : l == 2 ? 9 : 27);
        const u128 v2 = v * v;
        const u128 two53 = (u128)1 << 53;
        const u128 d = (two53 + v2 - 1) / v2;               // ceil(2^53 / v^2)
        const u128 kw = d << l;
        I.k_winograd[l] = kw > (u128)INT64_MAX ? INT64_MAX : (int64_t)kw;
    }
    I.k_winograd[0] = lam + 1;                              // l = 0: the dot-product bound, k <= lambda
    return 0;
}

// Limb schemes S / T: digit bounds, group bounds, the
// Eq. (2) k-block and the (i, j) pairs of each weight group.
int make_limb_plan(uint32_t p, int64_t k, const ff_opts& o, int64_t half, int64_t neg, int64_t cmax, int scheme,
                   int L, Plan& pl, bool& int_wb) {
    ff_plan_info& I = pl.info;
    if (L == 0) return FF_ERR_INTERNAL;
    I.L = L;
    I.scheme = scheme;
    I.groups = 2 * L - 1;

    // Digit magnitude bounds D_i.
    for (int i = 0; i < L; ++i) {
        const bool top = (i == L - 1);
        if (top) {
            int64_t hi = top_digit(half, L, scheme), lo = top_digit(-neg, L, scheme);
            I.digit_max[i] = (int32_t)(hi > -lo ? hi : -lo);
            I.limb_signed[i] = 1;
        } else {
            I.digit_max[i] = scheme == FF_SCHEME_S ? 128 : 255;
            I.limb_signed[i] = scheme == FF_SCHEME_S ? 1 : 0;
        }
    }
    int64_t bmax = 0;
    for (int w = 0; w < I.groups; ++w) {
        int64_t b = 0;
        for (int i = 0; i < L; ++i) {
            int j = w - i;
            if (j >= 0 && j < L) b += (int64_t)I.digit_max[i] * I.digit_max[j];
        }
        I.group_bound[w] = b;
        if (b > bmax) bmax = b;
    }
    I.group_bound_max = bmax;
    // Carry written back between steps (modp.cuh): integer write-back
    // (p < 2^29) leaves |v| <= 3p/2; the fp32-reciprocal one |v| <= p/2 + 385 w
    // with w = 256 for the Horner scaling (L >= 2) and w = 1 otherwise.
    // (m = round(w 2^32/p) must fit in int32 for every w used: p >= 512 when the
    // Horner factor w = 256 occurs, i.e. L >= 2.)
    int_wb = p < (1u << 29) && (L == 1 || p >= 512);
    const int64_t carry = int_wb ? (3 * (int64_t)p + 1) / 2 : cmax + (L >= 2 ? 385 * 256 : 385);
    I.carry_max = carry;
    I.kb_max = bmax > 0 ? (((int64_t)1 << 31) - 1 - carry) / bmax : ((int64_t)1 << 40);
    // Step order: k-outer needs 256 invertible mod p when there are several groups.
    int korder = o.korder == 0 ? 2 : o.korder;
    pl.korder_auto = (o.korder == 0 && o.kb_override == 0);
    if (knobs().korder > 0) { korder = knobs().korder == 1 ? 1 : 2; pl.korder_auto = false; }  // experiment only
    if (korder == 2 && L > 1 && (p % 2) == 0) korder = 1;
    pl.korder = korder;
    I.korder = korder;
    int64_t kb = I.kb_max;
    if (o.kb_override > 0) {
        if (o.kb_override > I.kb_max || o.kb_override < kBK) return FF_ERR_OPTS;
        kb = o.kb_override;
    } else if (korder == 2) {
        int64_t loc = (kKbLocalityBytes / L + kBK - 1) / kBK * kBK;   // L=1: 8192, 2: 4096, 3: 2816, 4: 2048
        if (knobs().kbloc > 0) loc = knobs().kbloc;  // experiment only
        kb = loc < kb ? loc : kb;
    }
    kb = (kb / kBK) * kBK;
    if (kb < kBK) return FF_ERR_INTERNAL;
    I.kb = kb;
    I.k_pad = (k + 15) / 16 * 16;
    I.num_kblocks = k > 0 ? (k + kb - 1) / kb : 0;

    // Pairs (i,j) ordered by weight group, highest w first (Horner order).
    int np = 0;
    for (int w = I.groups - 1; w >= 0; --w) {
        pl.group_first[w] = np;
        for (int i = 0; i < L; ++i) {
            int j = w - i;
            if (j >= 0 && j < L) {
                pl.pair_i[np] = i;
                pl.pair_j[np] = j;
                ++np;
            }
        }
        pl.group_len[w] = np - pl.group_first[w];
    }
    pl.npairs = np;
    return 0;
}

}  // namespace

int make_plan(uint32_t p, int64_t k, const ff_opts* opts, Plan* out) {
    if (p < 2 || p >= (1u << 31)) return -1;
    if (k < 0) return -6;
    ff_opts o;
    std::memset(&o, 0, sizeof(o));
    if (opts) o = *opts;
    if (o.scheme < FF_SCHEME_AUTO || o.scheme > FF_SCHEME_FP64) return FF_ERR_OPTS;
    if (o.winograd < -1 || o.winograd > 3) return FF_ERR_OPTS;
    if (o.winograd > 1 && o.scheme != FF_SCHEME_FP64) return FF_ERR_OPTS;   // several levels: fp64 only
    if (o.kb_override < 0) return FF_ERR_OPTS;
    if (o.cta_group < 0 || o.cta_group > 2) return FF_ERR_OPTS;
    if (o.korder < 0 || o.korder > 2) return FF_ERR_OPTS;
    if (o.inputs_canonical < 0 || o.inputs_canonical > 1) return FF_ERR_OPTS;
    if (o.small_path < -1 || o.small_path > 2) return FF_ERR_OPTS;
    if (o.wide_tiles < -1 || o.wide_tiles > 1) return FF_ERR_OPTS;

    Plan pl;
    std::memset(&pl, 0, sizeof(pl));
    pl.all_auto = o.scheme == FF_SCHEME_AUTO && o.winograd == 0 && o.kb_override == 0 && o.cta_group == 0 &&
                  o.korder == 0 && o.debug_saturate == 0 && o.debug_unchecked_kb == 0;
    pl.canonical_ab = o.inputs_canonical != 0;
    pl.small_mode = o.small_path != 0 ? (o.small_path > 0 ? o.small_path : 0) : knobs().small;
    pl.wide = knobs().wide ? o.wide_tiles : -1;
    ff_plan_info& I = pl.info;
    // Centred residues lie in [-neg, half]: neg = half for odd p, half + 1 for p = 2.
    const int64_t half = (int64_t)(p - 1) / 2;
    const int64_t neg = (int64_t)(p - 1) - half;
    const int64_t cmax = neg > half ? neg : half;
    I.p = p;
    I.centre_max = (int32_t)cmax;

    const int LS = min_limbs(half, neg, FF_SCHEME_S), LT = min_limbs(half, neg, FF_SCHEME_T);
    int scheme = o.scheme;
    if (scheme == FF_SCHEME_AUTO) {
        scheme = (LS != 0 && (LT == 0 || LS <= LT)) ? FF_SCHEME_S : FF_SCHEME_T;
        // Multi-modular when it needs clearly fewer int8 products than the
        // limbs (L^2): c5 (p ~ 2^26, k = 16384) takes 9 instead of 16.  The
        // margin of 2 charges its extra encoder planes and residue scratch
        // (DESIGN.md §4.9): c2 (8 vs 9) stays on limbs.
        const int Ll = scheme == FF_SCHEME_S ? LS : LT;
        uint32_t q[kMaxMod];
        u128 M, B;
        const int nq = crt_select(cmax, k, q, &M, &B);
        if (nq > 0 && nq + 2 < Ll * Ll) scheme = FF_SCHEME_CRT;
    }
    if (scheme == FF_SCHEME_CRT) {
        const int e = make_crt_plan(p, k, o, cmax, pl);
        if (e) return e;
    }
    if (scheme == FF_SCHEME_FP64) {
        const int e = make_f64_plan(k, o, cmax, pl);
        if (e) return e;
    }
    const int L = scheme == FF_SCHEME_S ? LS : scheme == FF_SCHEME_T ? LT : 0;
    bool int_wb = false;
    if (scheme == FF_SCHEME_S || scheme == FF_SCHEME_T) {
        const int e = make_limb_plan(p, k, o, half, neg, cmax, scheme, L, pl, int_wb);
        if (e) return e;
    }
    pl.saturate = o.debug_saturate != 0;
    pl.force_pair = o.cta_group;

    ModP& M = pl.mp;
    M.p = p;
    M.half = (uint32_t)half;
    M.mu = (uint32_t)((((uint64_t)1) << 32) / p);
    M.off31 = (uint32_t)((((uint64_t)1) << 31) % p);
    M.w256 = 256u % p;
    M.w256_sh = shoup(M.w256, p);
    M.inv_p = (float)(1.0 / (double)p);
    M.w256_over_p = (float)(256.0 / (double)p);
    auto mround = [&](double w) {
        const double v = w * 4294967296.0 / (double)p + 0.5;
        return (int32_t)(v >= 2147483647.0 ? 2147483647.0 : v);
    };
    M.m1 = mround(1.0);
    M.m256 = mround(256.0);
    M.int_wb = int_wb ? 1 : 0;
    // 256^-(G-1) mod p (k-outer carry between k-blocks); 1 when G = 1.
    pl.kinv = 1 % p;
    if (pl.korder == 2 && I.groups > 1 && !pl.crt) {
        int64_t r0 = p, r1 = 256 % p, s0 = 0, s1 = 1;     // extended Euclid: s1 * 256 = r1 (mod p)
        while (r1 != 0) {
            const int64_t qq = r0 / r1, t = r0 - qq * r1, u = s0 - qq * s1;
            r0 = r1; r1 = t; s0 = s1; s1 = u;
        }
        int64_t inv = ((s0 % (int64_t)p) + p) % p;          // r0 == 1 since p is odd
        uint64_t acc = 1;
        for (int g = 0; g < I.groups - 1; ++g) acc = acc * (uint64_t)inv % p;
        pl.kinv = (uint32_t)acc;
    }
    pl.kinv_sh = shoup(pl.kinv, p);
    *out = pl;
    set_scalars(out, 1, 0);
    return 0;
}

void set_scalars(Plan* pl, uint32_t alpha, uint32_t beta) {
    const uint32_t p = pl->mp.p;
    pl->mp.alpha = alpha % p;
    pl->mp.beta = beta % p;
    pl->mp.alpha_sh = shoup(pl->mp.alpha, p);
    pl->mp.beta_sh = shoup(pl->mp.beta, p);
}

}  // namespace ff
