// gemm_tc.cu -- the hot kernel: exact limb-product accumulation on the sm_100a
// tensor cores (tcgen05.mma.kind::i8 -> s32 in TMEM) with the delayed modular
// reduction, limb recombination and alpha/beta epilogue fused in.
//
// What it computes, per output tile:
//   op(A) = sum_i 256^i Ad_i,  op(B) = sum_j 256^j Bd_j   (int8 limb planes)
//   A B   = sum_w 256^w S_w,   S_w = sum_{i+j=w} Ad_i Bd_j^T   (weight groups)
//   Horner over w from 2L-2 down to 0, one TMEM accumulator per tile:
//     R <- S_{2L-2};  R <- 256 (R mod p) + S_w  ...;  out = alpha (R mod p) + beta C
// The accumulator is reduced mod p and re-centred ("delayed reduction",
// PAPER.md l.145-159) only (a) between weight groups, where it is also scaled
// by 256 mod p, and (b) every kb elements of k (the Eq. (2) analogue computed
// by the planner).  Nothing is ever rounded: the result is exact.
//
// Structure (persistent, warp-specialised, 576 threads per CTA):
//   warp 0      TMA producer: limb tiles A_i[128 x 128B], B_j[BN x 128B] -> SMEM ring
//   warp 1      TMEM owner + single-thread MMA issuer (4 x K=32 MMAs per stage)
//   warps 2..17 epilogue: tcgen05.ld -> mod p / Horner / alpha,beta -> tcgen05.st or global
// Two tiles are in flight per CTA (pair), one per 256-column TMEM accumulator
// ("slot"): while the epilogue reduces slot s between two steps, the MMA runs
// the other slot, so the tensor pipe never waits for the modular reduction.
//
// kPair = 2 (the production configuration): a cluster of two CTAs on one TPC
// computes 256 x 256 tiles with tcgen05.mma.cta_group::2 (M = 256): each CTA
// stages its own 128 rows of A and 128 of the 256 rows of B, the leader CTA
// issues the MMAs, each CTA's TMEM holds its 128 output rows.  This halves
// the SMEM operand traffic per MMA versus kPair = 1 (128 x 256 tiles).  The
// kWide variant (Cfg) widens the pair's tile to 256 x 512.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"
#include "modp.cuh"
#include "ptx.cuh"

namespace ff {

namespace {

constexpr int kNumEpiWarps = 16;  // 4 per TMEM lane quadrant, 64 columns each
constexpr int kThreads = 32 * (2 + kNumEpiWarps);
constexpr int kTmemCols = 512;  // two 256-column s32 accumulators
constexpr double kL2PlanesBytes = 192.0 * (1 << 20);   // operand planes "fit the L2" (launch_impl)
constexpr int kWideDelta = 32;     // wide tiles: staggered k-steps before the final output (swept on c3)
constexpr int kWideDeltaWb = 6;    //   before a TMEM write-back step (swept on c2)
constexpr int kRasterDefault = 12;  // tile-rows per raster band (L2 reuse; swept on c4: DESIGN.md §16)

// kWide (CTA pair only): 256 x 512 tiles, two N = 256 MMAs per k-step sharing the
// A stage, one accumulator in all 512 TMEM columns (no second slot): up to 25%
// less L2->SMEM operand traffic per MMA; the two halves are staggered
// (wide_phases) so each half's epilogue overlaps MMAs of the other.  Default for
// one-limb plans (c3), ff_opts.wide_tiles = 1 for any limb plan.
template <int kPair, bool kWide = false>
struct Cfg {
    static constexpr int BM = 128 * kPair;         // tile rows (per cluster)
    static constexpr int BN = kWide ? 2 * kTileN : kTileN;   // tile columns
    static constexpr int A_BYTES = 128 * kBK;      // per CTA: 128 rows of A
    static constexpr int B_BYTES = (BN / kPair) * kBK;  // per CTA: BN/kPair rows of B (wide: two 128-row halves)
    static constexpr int STAGE = A_BYTES + B_BYTES;
    static constexpr int STAGES = kWide ? 4 : (kPair == 2 ? 7 : 4);
    static constexpr int SMEM = STAGES * STAGE + 256 + 1024;
};

// One output of the fused epilogue: C_q <- (a * R + b * C_q) mod p.  A plain
// fgemm has one output (a = alpha, b = beta); a Winograd product adds +-alpha*P
// into up to four quadrants of C.
struct GemmOut {
    int32_t* C;
    int64_t ld;        // leading dimension of this output
    uint32_t a, a_sh, b, b_sh;
    int32_t vec;       // 1 if rows of C are 16-byte aligned
    int32_t add;       // 1: this output takes R + addend (mod p) instead of R
};

struct GemmArgs {
    ModP mp;
    GemmOut out[4];
    int32_t nout;
    int64_t ldc;
    int32_t m, n;
    int32_t tiles_m, tiles_n, num_tiles;
    int32_t k_iters;   // ceil(k / 128)
    int32_t kb_iters;  // k-block length / 128
    int32_t nkb;       // number of k-blocks
    int32_t G;         // weight groups
    int8_t pair_i[kMaxPairs], pair_j[kMaxPairs];
    int8_t group_first[kMaxGroups], group_len[kMaxGroups];
    uint32_t idesc[kMaxPairs];
    int32_t raster;     // tile-rows per raster band
    int32_t hints;      // bit0: TMA loads evict_last; bit1: C stores evict_first
    int32_t last_use;   // 1 if no later launch reads these outputs (streaming stores allowed)
    unsigned long long* trace;  // optional per-CTA cycle counters (FF_TRACE=1), else null
    int32_t korder;             // 1 group-outer, 2 k-outer
    uint32_t kinv, kinv_sh;     // k-outer: 256^-(G-1) mod p
    const uint8_t* die_map;     // die-aware schedule (dies.cu): die of each %smid, or null
    int* sched;                 // per-launch counters: [0],[1] clusters per die, [2] arrivals
    int* progress;              // throttle (FF_THROTTLE=S): tile pairs started, all clusters
    int32_t throttle;           // slack S in tile pairs (0: off)
    int32_t crt;                // 1: groups are CRT moduli
    const int32_t* addend;      // optional: residues in [0, p) added to R (mod p) for the outputs
    int64_t ld_add;             //   with `add` set (Winograd temporaries U2 = P1 + P6)
    int32_t add_vec;            //   1 if the addend's rows are 16-byte aligned
    CrtConsts cc;
    uint8_t* scratch;           // CRT: per CTA and slot, G byte planes of kCrtPlane bytes
    int32_t wdelta;             // wide tiles: k-steps of the staggered halves (wide_phases), final steps
    int32_t wdelta_wb;          //   the same before a write-back step
};

// Wide tiles (kWide): the two 256-column halves are staggered by D MMA k-steps so
// the epilogue of one half overlaps MMAs of the other.  A step's MMA k-steps are
// its (limb pair, k-slice) list, sigma = 0 .. S-1 (pair-major); per step: sigma in
// [0, D) for the low half only, [D, S) for both (one A stage feeds two MMAs), then
// [0, D) for the high half only.  The low half completes D k-steps before the
// high half; the next step (or tile) starts on the low half while the epilogue
// drains the high one.  Producer and MMA walk the same (pair, k-slice, lo, hi)
// sequence.  D: wdelta after the last step of a tile (final output), wdelta_wb
// after the others (TMEM write-back only).
template <class F>
__device__ __forceinline__ void wide_phases(const GemmArgs& a, int g, int kb, F&& f) {
    const int ks0 = kb * a.kb_iters;
    const int nks = min(ks0 + a.kb_iters, a.k_iters) - ks0;
    const int S = a.group_len[g] * nks;
    const bool final_step = (kb == a.nkb - 1) && g == 0;
    const int D = min(final_step ? a.wdelta : a.wdelta_wb, S / 2);
    auto run = [&](int s0, int s1, bool lo, bool hi) {   // one division per phase, not per k-step
        int q = s0 / nks, ks = s0 - q * nks;
        for (int sg = s0; sg < s1; ++sg) {
            f(a.group_first[g] + q, ks0 + ks, lo, hi);
            if (++ks == nks) { ks = 0; ++q; }
        }
    };
    run(0, D, true, false);
    run(D, S, true, true);
    run(0, D, false, true);
}

// CRT residue scratch: one 128 x 256 byte plane per (CTA, slot, modulus 0..G-1),
// laid out [h: 64-column quarter][grp: 8-column group][row 0..127][8 bytes] so
// that a warp's 32 rows store / load 256 contiguous bytes per instruction, and
// the final step's per-group reads (crt_group) use every byte of their sectors.
constexpr int kCrtPlane = 128 * kTileN;
constexpr int kCrtBatch = 5;    // scratch bytes of this many moduli loaded together in the final step

__device__ __forceinline__ uint8_t* crt_plane(const GemmArgs& a, int slot, int g) {
    return a.scratch + (static_cast<size_t>(blockIdx.x * 2 + slot) * a.G + g) * kCrtPlane;
}

__device__ __forceinline__ unsigned long long clk() {
    unsigned long long c;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
    return c;
}

struct Smem {
    uint64_t full[8];
    uint64_t empty[8];
    uint64_t accfull[2];
    uint64_t accempty[2];
    uint32_t tmem_base;
    int32_t sched[4];   // unit, nunits, first tile, tile count of this cluster's die
};

__device__ __forceinline__ void tile_coords(const GemmArgs& a, int t, int& tm, int& tn) {
    const int band_size = a.raster * a.tiles_n;
    const int band = t / band_size;
    const int idx = t - band * band_size;
    const int rows_in_band = min(a.raster, a.tiles_m - band * a.raster);
    tm = band * a.raster + idx % rows_in_band;
    tn = idx / rows_in_band;
}

// The common schedule every role walks: tiles in pairs (one per TMEM slot);
// per tile pair either groups (highest weight first) outer and k-blocks inner
// (group-outer), or k-blocks outer and all groups inner (k-outer, so a k-slice
// of every limb is reused from L2 by all groups); the two slots innermost.
// Tiles of this cluster: base + unit + j * nunits for j = 0, 1, ... < count.
template <bool kWide = false, class F>
__device__ __forceinline__ void for_each_step(const GemmArgs& a, int unit, int nunits, int base, int count, F&& f) {
    for (int t0 = unit; t0 < count; t0 += (kWide ? 1 : 2) * nunits) {
        const int t1 = t0 + nunits;
        const int nslots = (!kWide && t1 < count) ? 2 : 1;   // wide tiles use both TMEM halves
        if (a.korder == 2) {
            for (int kb = 0; kb < a.nkb; ++kb)
                for (int g = a.G - 1; g >= 0; --g)
                    for (int s = 0; s < nslots; ++s) f(base + (s == 0 ? t0 : t1), s, g, kb);
        } else {
            for (int g = a.G - 1; g >= 0; --g)
                for (int kb = 0; kb < a.nkb; ++kb)
                    for (int s = 0; s < nslots; ++s) f(base + (s == 0 ? t0 : t1), s, g, kb);
        }
    }
}

// C values for beta * C: Shoup's product w * x mod p is exact for any unsigned
// x < 2^32 (the quotient estimate errs by less than 2), so non-negative int32 C
// (canonical C in particular) is used as it is; only a group holding a negative
// value is reduced first (its unsigned reading would be off by 2^32).
template <int N>
__device__ __forceinline__ void c_nonneg(uint32_t (&o)[N], const ModP& M) {
    uint32_t any = 0;
#pragma unroll
    for (int t = 0; t < N; ++t) any |= o[t];
    if (static_cast<int32_t>(any) < 0) {
#pragma unroll
        for (int t = 0; t < N; ++t) o[t] = residue_i32(static_cast<int32_t>(o[t]), M);
    }
}

// One 8-column group of the final step of a CRT tile, for one thread (one row of
// its 64-column quarter), after the accumulator has been released: X = sum_i u_i
// M_i - t M exactly, t = round(sum_i u_i / q_i) (|X| <= M/4), X mod p =
// sum_i u_i (M_i mod p) + t (p - M mod p), every u_i from this thread's scratch
// bytes; then every output C_q <- (a_q X + b_q C_q) mod p for these columns.
// plane0: this thread's bytes in modulus 0's scratch plane; grp = 0..7.
__device__ __forceinline__ void crt_group(const GemmArgs& a, const ModP& M, const uint8_t* plane0, int row, int col_q,
                                          int grp) {
    if (row >= a.m) return;
    const int col0 = col_q + grp * 8;
    const uint8_t* src = plane0 + grp * 128 * 8;
    unsigned long long S[8];
    uint32_t F[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { S[j] = 0; F[j] = 0; }
#pragma unroll 1
    for (int g0 = 0; g0 < a.G; g0 += kCrtBatch) {
        // a batch of moduli's bytes in flight together (one L2 round trip per batch)
        uint2 xb[kCrtBatch];
#pragma unroll
        for (int b = 0; b < kCrtBatch; ++b)
            xb[b] = (g0 + b < a.G) ? *reinterpret_cast<const uint2*>(src + static_cast<size_t>(g0 + b) * kCrtPlane)
                                   : make_uint2(0, 0);
#pragma unroll
        for (int b = 0; b < kCrtBatch; ++b) {
            if (g0 + b >= a.G) break;
            const uint32_t W = a.cc.W[g0 + b], R = a.cc.R[g0 + b];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t u = ((j < 4 ? xb[b].x : xb[b].y) >> (8 * (j & 3))) & 0xFFu;
                S[j] += static_cast<unsigned long long>(u) * W;
                F[j] += u * R;
            }
        }
    }
    uint32_t X[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t t = (F[j] + (1u << 23)) >> 24;
        X[j] = residue_u64(S[j] + static_cast<unsigned long long>(t) * a.cc.Mneg, a.cc.mu64, M.p);
    }
    bool added = false;    // outputs with `add` come last (sorted on the host)
#pragma unroll 1
    for (int qo = 0; qo < a.nout; ++qo) {
        const GemmOut O = a.out[qo];
        int32_t* cr = O.C + static_cast<int64_t>(row) * O.ld + col0;
        const bool full = O.vec && (col0 + 8 <= a.n);
        if (O.add && !added) {
            const int32_t* ad = a.addend + static_cast<int64_t>(row) * a.ld_add + col0;
            if (a.add_vec && col0 + 8 <= a.n) {   // two 16-byte loads instead of eight scalar ones
                const int4 y0 = *reinterpret_cast<const int4*>(ad), y1 = *reinterpret_cast<const int4*>(ad + 4);
                const uint32_t y[8] = {(uint32_t)y0.x, (uint32_t)y0.y, (uint32_t)y0.z, (uint32_t)y0.w,
                                       (uint32_t)y1.x, (uint32_t)y1.y, (uint32_t)y1.z, (uint32_t)y1.w};
#pragma unroll
                for (int j = 0; j < 8; ++j) X[j] = addmod(X[j], y[j], M.p);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (col0 + j < a.n) X[j] = addmod(X[j], static_cast<uint32_t>(ad[j]), M.p);
            }
            added = true;
        }
        uint32_t o[8];
        if (O.b != 0) {
            if (full) {
                const int4 x0 = *reinterpret_cast<const int4*>(cr), x1 = *reinterpret_cast<const int4*>(cr + 4);
                o[0] = x0.x; o[1] = x0.y; o[2] = x0.z; o[3] = x0.w; o[4] = x1.x; o[5] = x1.y; o[6] = x1.z; o[7] = x1.w;
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] = (col0 + j < a.n) ? cr[j] : 0;
            }
            c_nonneg(o, M);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            uint32_t r = mulmod_shoup(X[j], O.a, O.a_sh, M.p);
            if (O.b != 0) r = addmod(r, mulmod_shoup(o[j], O.b, O.b_sh, M.p), M.p);
            o[j] = r;
        }
        if (full) {
            *reinterpret_cast<int4*>(cr) = make_int4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<int4*>(cr + 4) = make_int4(o[4], o[5], o[6], o[7]);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (col0 + j < a.n) cr[j] = static_cast<int32_t>(o[j]);
        }
    }
}

// Hand a TMEM accumulator slot back to the MMA issuer (all epilogue warps of
// both CTAs arrive on the leader's barrier).
template <int kPair>
__device__ __forceinline__ void release_slot(Smem* sh, int slot, uint32_t lane, uint32_t leader0, uint32_t leader1) {
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) {
        if (kPair == 2) ptx::mbar_arrive_cluster(slot ? leader1 : leader0);
        else ptx::mbar_arrive(&sh->accempty[slot]);
    }
}

template <int kPair, bool kTrace, bool kWide = false>
__global__ void __launch_bounds__(kThreads, 1)
    ffgemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ GemmArgs a) {
    using K = Cfg<kPair, kWide>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    Smem* sh = reinterpret_cast<Smem*>(smem + K::STAGES * K::STAGE);
    const int warp = threadIdx.x / 32;
    const uint32_t lane = ptx::lane_id();
    const uint32_t rank = kPair == 2 ? ptx::cluster_ctarank() : 0;
    const bool leader = (rank == 0);

    if (threadIdx.x == 0) {
        ptx::tma_prefetch(&tmA);
        ptx::tma_prefetch(&tmB);
        for (int s = 0; s < K::STAGES; ++s) {
            ptx::mbar_init(&sh->full[s], 1);
            ptx::mbar_init(&sh->empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(&sh->accfull[s], 1);
            ptx::mbar_init(&sh->accempty[s], kNumEpiWarps * kPair);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) {
        if (kPair == 2) ptx::tmem_alloc_pair(&sh->tmem_base, kTmemCols);
        else ptx::tmem_alloc(&sh->tmem_base, kTmemCols);
    }
    // Work assignment.  Plain: cluster c takes tiles c, c + C, ...  Die-aware: each
    // cluster registers on its die's counter, waits until every cluster of the
    // launch has registered (co-residency is guaranteed by the cooperative launch),
    // and the tile raster is split between the dies in proportion to their cluster
    // counts, so each die's L2 holds only its own operands.
    if (threadIdx.x == 0 && leader) {
        const int nclusters = gridDim.x / kPair;
        int unit = blockIdx.x / kPair, nunits = nclusters, base = 0, count = a.num_tiles;
#ifdef FF_EXPERIMENTS
        if (a.die_map) {
            uint32_t smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            const int d = a.die_map[smid] ? 1 : 0;
            unit = atomicAdd(&a.sched[d], 1);
            __threadfence();
            atomicAdd(&a.sched[2], 1);
            while (atomicAdd(&a.sched[2], 0) < nclusters) __nanosleep(64);
            const int n0 = atomicAdd(&a.sched[0], 0), n1 = nclusters - n0;
            const int T0 = n1 == 0 ? a.num_tiles
                                   : (n0 == 0 ? 0 : static_cast<int>(static_cast<long long>(a.num_tiles) * n0 / nclusters));
            nunits = d ? n1 : n0;
            base = d ? T0 : 0;
            count = d ? a.num_tiles - T0 : T0;
        }
#endif
        sh->sched[0] = unit; sh->sched[1] = nunits; sh->sched[2] = base; sh->sched[3] = count;
    }
    ptx::tc_fence_before();
    if (kPair == 2) ptx::cluster_sync();
    else __syncthreads();
    ptx::tc_fence_after();
    if (kPair == 2) {   // the peer CTA takes the leader's assignment (DSMEM read)
        if (threadIdx.x == 0 && !leader) {
            for (int i = 0; i < 4; ++i) {
                const uint32_t ra = ptx::mapa(ptx::smem_u32(&sh->sched[i]), 0);
                int v;
                asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(ra) : "memory");
                sh->sched[i] = v;
            }
        }
        ptx::cluster_sync();
    }
    const int unit = sh->sched[0], nunits = sh->sched[1], tbase = sh->sched[2], tcount = sh->sched[3];
    const uint32_t tmem_base = sh->tmem_base;
    // launched programmatically after the encoders: everything above overlapped
    // them; the limb planes (TMA), C and the scratch are read only from here on
    ptx::pdl_wait();

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (both CTAs)
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            // L2 policies (experiment bits, FF_HINTS): bit0 both operands evict_last;
            // bit2 A evict_last + B evict_first; bit3 A evict_first + B evict_last.
            uint64_t polA = (a.hints & 1) ? ptx::policy_evict_last() : ptx::policy_evict_normal();
            uint64_t polB = polA;
            if (a.hints & 4) { polA = ptx::policy_evict_last(); polB = ptx::policy_evict_first(); }
            if (a.hints & 8) { polA = ptx::policy_evict_first(); polB = ptx::policy_evict_last(); }
#ifdef FF_EXPERIMENTS
            int pair_idx = 0;
#endif
            for_each_step<kWide>(a, unit, nunits, tbase, tcount, [&](int tile, int slot, int g, int kb) {
#ifdef FF_EXPERIMENTS
                if (a.throttle && leader && slot == 0 && kb == 0 && g == a.G - 1) {
                    // soft lockstep: start tile pair j only once every cluster (on
                    // average) has started pair j - S, so the tiles in flight stay a
                    // compact part of the raster and share their operands in L2
                    atomicAdd(a.progress, 1);
                    const int need = (pair_idx + 1 - a.throttle) * nunits;
                    if (need > 0)
                        while (*reinterpret_cast<volatile int*>(a.progress) < need) __nanosleep(128);
                    ++pair_idx;
                }
#endif
                int tm, tn;
                tile_coords(a, tile, tm, tn);
                const int arow = tm * K::BM + static_cast<int>(rank) * 128;
                // wide: this CTA's 128 rows of each of the two 256-row B halves
                const int brow = tn * K::BN + static_cast<int>(rank) * (kWide ? 128 : K::BN / kPair);
                if constexpr (kWide) {   // staggered halves (wide_phases)
                    wide_phases(a, g, kb, [&](int pi, int ks, bool lo, bool hi) {
                        const int li = a.pair_i[pi], lj = a.pair_j[pi];
                        ptx::mbar_wait_sleep(&sh->empty[stage], phase ^ 1);
                        uint8_t* sa = smem + stage * K::STAGE;
                        const int bytes = K::A_BYTES + (lo ? 128 * kBK : 0) + (hi ? 128 * kBK : 0);
                        if (leader) ptx::mbar_arrive_expect_tx(&sh->full[stage], 2 * bytes);
                        const uint32_t bar = ptx::mapa(ptx::smem_u32(&sh->full[stage]), 0);
                        ptx::tma_load_3d_pair(sa, &tmA, bar, ks * kBK, arow, li, polA);
                        if (lo) ptx::tma_load_3d_pair(sa + K::A_BYTES, &tmB, bar, ks * kBK, brow, lj, polB);
                        if (hi)
                            ptx::tma_load_3d_pair(sa + K::A_BYTES + 128 * kBK, &tmB, bar, ks * kBK, brow + kTileN, lj,
                                                  polB);
                        if (++stage == K::STAGES) { stage = 0; phase ^= 1; }
                    });
                    return;
                }
                const int ks0 = kb * a.kb_iters;
                const int ks1 = min(ks0 + a.kb_iters, a.k_iters);
                for (int pi = a.group_first[g]; pi < a.group_first[g] + a.group_len[g]; ++pi) {
                    const int li = a.pair_i[pi], lj = a.pair_j[pi];
                    for (int ks = ks0; ks < ks1; ++ks) {
                        ptx::mbar_wait_sleep(&sh->empty[stage], phase ^ 1);
                        uint8_t* sa = smem + stage * K::STAGE;
                        if (kPair == 1) {
                            ptx::mbar_arrive_expect_tx(&sh->full[stage], K::STAGE);
                            ptx::tma_load_3d(sa, &tmA, &sh->full[stage], ks * kBK, arow, li, polA);
                            ptx::tma_load_3d(sa + K::A_BYTES, &tmB, &sh->full[stage], ks * kBK, brow, lj, polB);
                        } else {
                            // both CTAs' bytes are counted on the leader's full barrier
                            if (leader) ptx::mbar_arrive_expect_tx(&sh->full[stage], 2 * K::STAGE);
                            const uint32_t bar = ptx::mapa(ptx::smem_u32(&sh->full[stage]), 0);
                            ptx::tma_load_3d_pair(sa, &tmA, bar, ks * kBK, arow, li, polA);
                            ptx::tma_load_3d_pair(sa + K::A_BYTES, &tmB, bar, ks * kBK, brow, lj, polB);
                        }
                        if (++stage == K::STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            });
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (one thread of the leader)
        if (lane == 0 && leader) {
            uint32_t stage = 0, phase = 0;
            uint32_t acc_par[2] = {0, 0};
            unsigned long long t_start = clk(), w_acc = 0, w_full = 0, nsteps = 0;
            for_each_step<kWide>(a, unit, nunits, tbase, tcount, [&](int, int slot, int g, int kb) {
                if constexpr (kWide) {   // staggered halves (wide_phases): slot 0 = low, 1 = high half
                    const unsigned long long tw = kTrace ? clk() : 0;
                    ptx::mbar_wait_cluster(&sh->accempty[0], acc_par[0] ^ 1);
                    acc_par[0] ^= 1;
                    if (kTrace) { w_acc += clk() - tw; ++nsteps; }
                    ptx::tc_fence_after();
                    // the first step of a tile overwrites; later ones accumulate onto the write-back
                    const uint32_t acc0 = (g == a.G - 1 && kb == 0) ? 0u : 1u;
                    uint32_t acc_lo = acc0, acc_hi = acc0;
                    bool hi_ready = false;
                    int done = 0;
                    const int ks0 = kb * a.kb_iters;
                    const int nlo = a.group_len[g] * (min(ks0 + a.kb_iters, a.k_iters) - ks0);
                    wide_phases(a, g, kb, [&](int pi, int, bool lo, bool hi) {
                        const uint32_t idesc = a.idesc[pi];
                        if (hi && !hi_ready) {   // first high-half MMA: its TMEM half must be free
                            const unsigned long long th = kTrace ? clk() : 0;
                            ptx::mbar_wait_cluster(&sh->accempty[1], acc_par[1] ^ 1);
                            acc_par[1] ^= 1;
                            if (kTrace) w_acc += clk() - th;
                            ptx::tc_fence_after();
                            hi_ready = true;
                        }
                        const unsigned long long t1 = kTrace ? clk() : 0;
                        ptx::mbar_wait(&sh->full[stage], phase);
                        if (kTrace) w_full += clk() - t1;
                        ptx::tc_fence_after();
                        const uint32_t sa = ptx::smem_u32(smem + stage * K::STAGE);
                        const uint64_t da = ptx::smem_desc_sw128(sa);
                        const uint64_t dbl = ptx::smem_desc_sw128(sa + K::A_BYTES);
                        const uint64_t dbh = ptx::smem_desc_sw128(sa + K::A_BYTES + 128 * kBK);
#pragma unroll
                        for (int kk = 0; kk < kBK / kMmaK; ++kk) {
                            if (lo) ptx::mma_i8_pair(tmem_base, da + 2 * kk, dbl + 2 * kk, idesc, acc_lo);
                            if (hi) ptx::mma_i8_pair(tmem_base + kTileN, da + 2 * kk, dbh + 2 * kk, idesc, acc_hi);
                            if (lo) acc_lo = 1u;
                            if (hi) acc_hi = 1u;
                        }
                        ptx::tc_commit_pair(&sh->empty[stage]);
                        if (++stage == K::STAGES) { stage = 0; phase ^= 1; }
                        // the low half is complete after its last k-step (end of the shared phase)
                        if (lo && ++done == nlo) ptx::tc_commit_pair(&sh->accfull[0]);
                    });
                    ptx::tc_commit_pair(&sh->accfull[1]);
                    return;
                }
                const unsigned long long t0 = kTrace ? clk() : 0;
                if (kPair == 2) ptx::mbar_wait_cluster(&sh->accempty[slot], acc_par[slot] ^ 1);
                else ptx::mbar_wait(&sh->accempty[slot], acc_par[slot] ^ 1);
                if (kTrace) { w_acc += clk() - t0; ++nsteps; }
                acc_par[slot] ^= 1;
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + slot * kTileN;
                // The first MMA of a tile (limbs: Horner continues in the accumulator)
                // or of each modulus (CRT: independent products) overwrites.
                uint32_t acc = (a.crt ? kb == 0 : (g == a.G - 1 && kb == 0)) ? 0u : 1u;
                const int ks0 = kb * a.kb_iters;
                const int ks1 = min(ks0 + a.kb_iters, a.k_iters);
                for (int pi = a.group_first[g]; pi < a.group_first[g] + a.group_len[g]; ++pi) {
                    const uint32_t idesc = a.idesc[pi];
                    for (int ks = ks0; ks < ks1; ++ks) {
                        const unsigned long long t1 = kTrace ? clk() : 0;
                        ptx::mbar_wait(&sh->full[stage], phase);
                        if (kTrace) w_full += clk() - t1;
                        ptx::tc_fence_after();
                        const uint32_t sa = ptx::smem_u32(smem + stage * K::STAGE);
                        const uint64_t da = ptx::smem_desc_sw128(sa);
                        const uint64_t db = ptx::smem_desc_sw128(sa + K::A_BYTES);
#pragma unroll
                        for (int kk = 0; kk < kBK / kMmaK; ++kk) {
                            if (kPair == 2) ptx::mma_i8_pair(d, da + 2 * kk, db + 2 * kk, idesc, acc);
                            else ptx::mma_i8(d, da + 2 * kk, db + 2 * kk, idesc, acc);
                            acc = 1u;
                        }
                        // frees the SMEM stage (in both CTAs) when these MMAs finish
                        if (kPair == 2) ptx::tc_commit_pair(&sh->empty[stage]);
                        else ptx::tc_commit(&sh->empty[stage]);
                        if (++stage == K::STAGES) { stage = 0; phase ^= 1; }
                    }
                }
                // accumulator ready for the epilogue (of both CTAs)
                if (kPair == 2) ptx::tc_commit_pair(&sh->accfull[slot]);
                else ptx::tc_commit(&sh->accfull[slot]);
            });
            if (kTrace) {
                unsigned long long* tr = a.trace + blockIdx.x * 8;
                tr[0] = clk() - t_start;  // MMA thread lifetime (cycles)
                tr[1] = w_acc;            // waiting for the epilogue to free a TMEM slot
                tr[2] = w_full;           // waiting for TMA data
                tr[3] = nsteps;
            }
        }
    } else {
        // ------------------------------------------------ epilogue warps (both CTAs)
        const int q = warp & 3;                 // TMEM lane quadrant this warp may access
        const int h = (warp - 2) >> 2;          // which 64-column quarter of the tile
        const ModP M = a.mp;
        const uint32_t accempty_leader0 = kPair == 2 ? ptx::mapa(ptx::smem_u32(&sh->accempty[0]), 0) : 0;
        const uint32_t accempty_leader1 = kPair == 2 ? ptx::mapa(ptx::smem_u32(&sh->accempty[1]), 0) : 0;
        uint32_t acc_par[2] = {0, 0};
        unsigned long long e_wait = 0, e_busy = 0, e_final = 0;
        // CRT plans: the final step of a tile only stores u_0 and releases TMEM; its
        // reconstruction + outputs (8 groups of 8 columns) are deferred and done while
        // this thread would otherwise wait for the next accumulator, so that they never
        // hold back the release of a slot the MMA needs.
        int pend_tile[2] = {0, 0}, pend_grp[2] = {8, 8};
        auto pend_work = [&](int ps) {
            int tm, tn;
            tile_coords(a, pend_tile[ps], tm, tn);
            const int row = tm * K::BM + static_cast<int>(rank) * 128 + q * 32 + static_cast<int>(lane);
            const int crow = q * 32 + static_cast<int>(lane);
            crt_group(a, M, crt_plane(a, ps, 0) + (h * 8 * 128 + crow) * 8, row, tn * K::BN + h * 64, pend_grp[ps]);
            ++pend_grp[ps];
        };
        for_each_step<kWide>(a, unit, nunits, tbase, tcount, [&](int tile, int slot, int g, int kb) {
            const unsigned long long t0 = kTrace ? clk() : 0;
            if (a.crt) {
                // this slot's pending work must finish before its scratch is reused
                for (;;) {
                    const bool ready = ptx::mbar_test(&sh->accfull[slot], acc_par[slot]);
                    const int ps = pend_grp[slot] < 8 ? slot : (pend_grp[slot ^ 1] < 8 ? (slot ^ 1) : -1);
                    if (ready && ps != slot) break;
                    if (ps < 0) {
                        ptx::mbar_wait_sleep(&sh->accfull[slot], acc_par[slot]);
                        break;
                    }
                    pend_work(ps);
                }
            } else {
                ptx::mbar_wait_sleep(&sh->accfull[slot], acc_par[slot]);
            }
            const unsigned long long t1 = kTrace ? clk() : 0;
            acc_par[slot] ^= 1;
            ptx::tc_fence_after();
            const bool last_kb = (kb == a.nkb - 1);
            const bool final_step = last_kb && g == 0;
            // Write-back factor: x256 (Horner) when the next step is the next-lower group;
            // k-outer order: 256^-(G-1) (exact) when the next step restarts the groups
            // on the next k-block; group-outer order: x1 between k-blocks of a group.
            const bool horner = (a.korder == 2) ? (g > 0) : last_kb;
            const bool rescale = (a.korder == 2) && g == 0 && !last_kb;
            const uint32_t tcol = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + slot * kTileN + h * 64;
            const int crow = q * 32 + static_cast<int>(lane);   // row of this thread within the CTA tile
            // The TMEM slot is handed back to the MMA as soon as the accumulator has been
            // read; for CRT plans that happens BEFORE the final step's reconstruction and
            // output stores, which then overlap the next tile's MMAs on this slot.
            const bool crt_final = a.crt && final_step;
            if (a.crt) {
                // CRT: between k-blocks keep the centred residue
                // mod q_g; after the last one store u_g = (S_g mod q_g) v_g mod q_g
                // to this CTA's scratch (read back by the final step of the tile,
                // modulus 0 included).
                uint32_t v[64];
                ptx::tmem_ld64(tcol, v);
                ptx::tmem_wait_ld();
                const uint32_t qg = a.cc.q[g], mu = a.cc.mu[g], off = a.cc.off31[g];
                if (!last_kb) {
                    const uint32_t hf = a.cc.half[g];
#pragma unroll
                    for (int t = 0; t < 64; ++t)
                        v[t] = static_cast<uint32_t>(centre_small(residue_small(static_cast<int32_t>(v[t]), qg, mu, off), qg, hf));
                    ptx::tmem_st64(tcol, v);
                    ptx::tmem_wait_st();
                } else {
                    const uint32_t vg = a.cc.v[g];
                    uint8_t* dst = crt_plane(a, slot, g) + (h * 8 * 128 + crow) * 8;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t w[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            w[j] = 0;
#pragma unroll
                            for (int b = 0; b < 4; ++b) {
                                const uint32_t r = residue_small(static_cast<int32_t>(v[c * 16 + j * 4 + b]), qg, mu, off);
                                w[j] |= mulmod_small(r, vg, qg, mu) << (8 * b);
                            }
                        }
                        // columns 16c .. 16c+15 = groups 2c and 2c+1 of this quarter
                        *reinterpret_cast<uint2*>(dst + (2 * c) * 128 * 8) = make_uint2(w[0], w[1]);
                        *reinterpret_cast<uint2*>(dst + (2 * c + 1) * 128 * 8) = make_uint2(w[2], w[3]);
                    }
                }
            }
            if (crt_final) release_slot<kPair>(sh, slot, lane, accempty_leader0, accempty_leader1);
            if (a.crt && !final_step) {
                // (done above)
            } else if (rescale) {
#pragma unroll 1
              for (int hs = 0; hs < (kWide ? 2 : 1); ++hs) {   // wide: low half, hand-off, high half
                if (kWide && hs == 1) {
                    release_slot<kPair>(sh, 0, lane, accempty_leader0, accempty_leader1);
                    ptx::mbar_wait_sleep(&sh->accfull[1], acc_par[1]);
                    acc_par[1] ^= 1;
                    ptx::tc_fence_after();
                }
                const uint32_t tcw = tcol + hs * kTileN;
                uint32_t v[64];
                ptx::tmem_ld64(tcw, v);
                ptx::tmem_wait_ld();
#pragma unroll
                for (int t = 0; t < 64; ++t)
                    v[t] = static_cast<uint32_t>(centre(mulmod_shoup(residue_i32(static_cast<int32_t>(v[t]), M),
                                                                     a.kinv, a.kinv_sh, M.p), M));
                ptx::tmem_st64(tcw, v);
                ptx::tmem_wait_st();
              }
            } else if (!final_step) {
                // delayed reduction between steps (+ Horner x256 before the next-lower group);
                // wide tiles: the low half, hand it back, then the high half (wide_phases)
#pragma unroll 1
              for (int hs = 0; hs < (kWide ? 2 : 1); ++hs) {
                if (kWide && hs == 1) {
                    release_slot<kPair>(sh, 0, lane, accempty_leader0, accempty_leader1);
                    ptx::mbar_wait_sleep(&sh->accfull[1], acc_par[1]);
                    acc_par[1] ^= 1;
                    ptx::tc_fence_after();
                }
                const uint32_t tcw = tcol + hs * kTileN;
                uint32_t v[64];
                ptx::tmem_ld64(tcw, v);
                ptx::tmem_wait_ld();
                const int32_t w = horner ? 256 : 1;
                if (M.int_wb) {
                    const int32_t mm = horner ? M.m256 : M.m1;
#pragma unroll
                    for (int t = 0; t < 64; ++t)
                        v[t] = static_cast<uint32_t>(reduce_mulhi(static_cast<int32_t>(v[t]), w, mm, M.p));
                } else {
                    const float f = horner ? M.w256_over_p : M.inv_p;
#pragma unroll
                    for (int t = 0; t < 64; ++t)
                        v[t] = static_cast<uint32_t>(reduce_approx(static_cast<int32_t>(v[t]), w, f,
                                                                   static_cast<int32_t>(M.p)));
                }
                ptx::tmem_st64(tcw, v);
                ptx::tmem_wait_st();
              }
            } else if (a.crt) {
                pend_tile[slot] = tile;        // deferred: see pend_work
                pend_grp[slot] = 0;
            } else {
                int tm, tn;
                tile_coords(a, tile, tm, tn);
                const int row = tm * K::BM + static_cast<int>(rank) * 128 + q * 32 + static_cast<int>(lane);
                // 32-column chunks of this thread's quarter; wide tiles: the same quarter of
                // both 256-column halves (TMEM columns 0..255 and 256..511)
#pragma unroll 1
                for (int half = 0; half < (kWide ? 4 : 2); ++half) {
                    if (kWide && half == 2) {
                        // low half done: hand it to the next tile's first k-steps, then
                        // wait for the high half (wide_phases)
                        release_slot<kPair>(sh, 0, lane, accempty_leader0, accempty_leader1);
                        ptx::mbar_wait_sleep(&sh->accfull[1], acc_par[1]);
                        acc_par[1] ^= 1;
                        ptx::tc_fence_after();
                    }
                    uint32_t v[32];
                    const int coff = (half >> 1) * kTileN + (half & 1) * 32;
                    ptx::tmem_ld32(tcol + coff, v);
                    ptx::tmem_wait_ld();
                    if (row >= a.m) continue;
                    const int col0 = tn * K::BN + h * 64 + coff;
#pragma unroll
                    for (int t = 0; t < 32; ++t) v[t] = residue_i32(static_cast<int32_t>(v[t]), M);  // exact R

                    bool added = false;    // outputs with `add` come last (sorted on the host)
#pragma unroll 1
                    for (int qo = 0; qo < a.nout; ++qo) {
                        const GemmOut O = a.out[qo];
                        int32_t* crow = O.C + static_cast<int64_t>(row) * O.ld + col0;
                        if (O.add && !added) {
                            const int32_t* ad = a.addend + static_cast<int64_t>(row) * a.ld_add + col0;
#pragma unroll
                            for (int t = 0; t < 32; ++t)
                                if (col0 + t < a.n) v[t] = addmod(v[t], static_cast<uint32_t>(ad[t]), M.p);
                            added = true;
                        }
                        const bool full = O.vec && (col0 + 32 <= a.n);
                        uint32_t o[32];
                        if (O.b != 0) {
                            if (full) {
#pragma unroll
                                for (int t = 0; t < 8; ++t) {
                                    const int4 x = *reinterpret_cast<const int4*>(crow + 4 * t);
                                    o[4 * t] = x.x; o[4 * t + 1] = x.y; o[4 * t + 2] = x.z; o[4 * t + 3] = x.w;
                                }
                            } else {
#pragma unroll
                                for (int t = 0; t < 32; ++t) o[t] = (col0 + t < a.n) ? crow[t] : 0;
                            }
                            c_nonneg(o, M);
                        }
#pragma unroll
                        for (int t = 0; t < 32; ++t) {
                            uint32_t r = mulmod_shoup(v[t], O.a, O.a_sh, M.p);
                            if (O.b != 0) r = addmod(r, mulmod_shoup(o[t], O.b, O.b_sh, M.p), M.p);
                            o[t] = r;
                        }
                        if (full && (a.hints & 2) && qo == a.nout - 1 && a.last_use) {
#pragma unroll
                            for (int t = 0; t < 8; ++t)
                                ptx::st_global_v4_stream(crow + 4 * t, o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]);
                        } else if (full) {
#pragma unroll
                            for (int t = 0; t < 8; ++t)
                                *reinterpret_cast<int4*>(crow + 4 * t) = make_int4(o[4 * t], o[4 * t + 1], o[4 * t + 2], o[4 * t + 3]);
                        } else {
#pragma unroll
                            for (int t = 0; t < 32; ++t)
                                if (col0 + t < a.n) crow[t] = static_cast<int32_t>(o[t]);
                        }
                    }
                }
            }
            if (!crt_final) release_slot<kPair>(sh, kWide ? 1 : slot, lane, accempty_leader0, accempty_leader1);
            if (kTrace) {
                const unsigned long long t2 = clk();
                e_wait += t1 - t0;
                if (final_step) e_final += t2 - t1; else e_busy += t2 - t1;
            }
        });
        for (int ps = 0; ps < 2; ++ps)
            while (pend_grp[ps] < 8) pend_work(ps);
        if (kTrace && warp == 2 && lane == 0) {
            unsigned long long* tr = a.trace + blockIdx.x * 8;
            tr[4] = e_wait;   // epilogue waiting for an accumulator
            tr[5] = e_busy;   // epilogue work on intermediate steps
            tr[6] = e_final;  // epilogue work on final steps (stores)
        }
    }

    ptx::tc_fence_before();
    if (kPair == 2) ptx::cluster_sync();
    else __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        if (kPair == 2) ptx::tmem_dealloc_pair(tmem_base, kTmemCols);
        else ptx::tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ---------------------------------------------------------------- host side

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// Limb planes [L][rows][k_pad] int8 as a 3-D tensor (k fastest), box 128 x box_rows x 1, 128B swizzle.
bool make_plane_map(CUtensorMap* map, const int8_t* base, int L, int64_t rows, int64_t k_pad, int box_rows) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(k_pad), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(L)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(k_pad), static_cast<cuuint64_t>(rows * k_pad)};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

uint32_t make_idesc(bool a_signed, bool b_signed, bool saturate, int M, int N) {
    uint32_t d = 0;
    d |= (saturate ? 1u : 0u) << 3;          // saturate (s8 only)
    d |= 2u << 4;                             // D format: S32
    d |= (a_signed ? 1u : 0u) << 7;           // A: 0 = u8, 1 = s8
    d |= (b_signed ? 1u : 0u) << 10;          // B: 0 = u8, 1 = s8
    // bits 15/16: A/B K-major (0); no negate
    d |= static_cast<uint32_t>(N >> 3) << 17;  // N / 8
    d |= static_cast<uint32_t>(M >> 4) << 24;  // M / 16
    return d;
}

uint32_t shoup_host(uint32_t w, uint32_t p) { return static_cast<uint32_t>((static_cast<uint64_t>(w) << 32) / p); }

template <int kPair, bool kWide = false>
int launch_impl(const Plan& pl, int64_t m, int64_t n, int64_t k, const int8_t* A_limbs, const int8_t* B_limbs,
                const OutSpec* outs, int nout, int64_t ldc, int last_use, void* scratch, cudaStream_t st,
                const int32_t* addend, int64_t ld_add) {
    using K = Cfg<kPair, kWide>;
    const ff_plan_info& I = pl.info;
    if (m > INT32_MAX - K::BM || n > INT32_MAX - K::BN) return -2;
    GemmArgs a;
    std::memset(&a, 0, sizeof(a));
    a.mp = pl.mp;
    if (nout < 1 || nout > 4) return -10;
    a.nout = nout;
    // the kernels add the addend in place before the first output that takes it,
    // so the outputs that do come last
    OutSpec so[4];
    int ns = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (int q = 0; q < nout; ++q)
            if ((outs[q].add && addend ? 1 : 0) == pass) so[ns++] = outs[q];
    outs = so;
    for (int q = 0; q < nout; ++q) {
        const uint32_t p = pl.mp.p;
        a.out[q].C = outs[q].C;
        a.out[q].ld = outs[q].ld > 0 ? outs[q].ld : ldc;
        a.out[q].a = outs[q].a % p;
        a.out[q].a_sh = shoup_host(a.out[q].a, p);
        a.out[q].b = outs[q].b % p;
        a.out[q].b_sh = shoup_host(a.out[q].b, p);
        a.out[q].vec = ((a.out[q].ld % 4) == 0 && (reinterpret_cast<uintptr_t>(outs[q].C) & 15) == 0) ? 1 : 0;
        a.out[q].add = (outs[q].add && addend) ? 1 : 0;
    }
    a.addend = addend;
    a.ld_add = ld_add;
    a.add_vec = (addend && (ld_add % 4) == 0 && (reinterpret_cast<uintptr_t>(addend) & 15) == 0) ? 1 : 0;
    a.last_use = last_use;
    a.ldc = ldc;
    a.m = static_cast<int32_t>(m);
    a.n = static_cast<int32_t>(n);
    a.tiles_m = static_cast<int32_t>((m + K::BM - 1) / K::BM);
    a.tiles_n = static_cast<int32_t>((n + K::BN - 1) / K::BN);
    const int64_t nt = static_cast<int64_t>(a.tiles_m) * a.tiles_n;
    if (nt > INT32_MAX / 2) return -2;
    a.num_tiles = static_cast<int32_t>(nt);
    a.k_iters = static_cast<int32_t>((k + kBK - 1) / kBK);
    a.kb_iters = static_cast<int32_t>(I.kb / kBK);
    a.korder = pl.korder;
    // k-outer pays off only when the operand planes do not fit the L2 (it trades
    // more steps, each costing TMEM traffic, for DRAM locality; measured: c4
    // (1 GiB of planes) -5% with k-outer, c2 (100 MB) +6%, c1/c3 equal or better
    // group-outer).  Below kL2Planes the default falls back to group-outer with
    // the safe k-block.
    if (pl.korder_auto && pl.korder == 2 &&
        static_cast<double>(I.L) * static_cast<double>(m + n) * static_cast<double>(I.k_pad) <= kL2PlanesBytes) {
        a.korder = 1;
        a.kb_iters = static_cast<int32_t>((I.kb_max / kBK) > 0 ? I.kb_max / kBK : 1);
    }
    if (kWide && pl.wide == 0) {   // auto (one weight group): one safe k-block, group-outer
        a.korder = 1;
        if (pl.korder_auto) a.kb_iters = static_cast<int32_t>((I.kb_max / kBK) > 0 ? I.kb_max / kBK : 1);
    }
    a.wdelta = knobs().wdelta > 0 ? knobs().wdelta : kWideDelta;
    a.wdelta_wb = knobs().wdelta_wb > 0 ? knobs().wdelta_wb : kWideDeltaWb;
    a.nkb = (a.k_iters + a.kb_iters - 1) / a.kb_iters;
    a.G = I.groups;
    for (int pi = 0; pi < pl.npairs; ++pi) {
        a.pair_i[pi] = static_cast<int8_t>(pl.pair_i[pi]);
        a.pair_j[pi] = static_cast<int8_t>(pl.pair_j[pi]);
        const bool sa = pl.crt || I.limb_signed[pl.pair_i[pi]] != 0;   // CRT residues are s8
        const bool sb = pl.crt || I.limb_signed[pl.pair_j[pi]] != 0;
        a.idesc[pi] = make_idesc(sa, sb, pl.saturate, K::BM, kWide ? kTileN : K::BN);   // wide: two N = 256 MMAs
    }
    for (int w = 0; w < I.groups; ++w) {
        a.group_first[w] = static_cast<int8_t>(pl.group_first[w]);
        a.group_len[w] = static_cast<int8_t>(pl.group_len[w]);
    }
    a.throttle = 0;
    a.progress = nullptr;
#ifdef FF_EXPERIMENTS
    if (knobs().throttle > 0) {        // experiment: soft lockstep of the clusters
        static int* ring = nullptr;
        static unsigned slot = 0;
        if (!ring && cudaMalloc(&ring, 4096 * sizeof(int)) != cudaSuccess) ring = nullptr;
        if (ring) {
            int* c = ring + (slot++ % 4096);
            if (cudaMemsetAsync(c, 0, sizeof(int), st) == cudaSuccess) {
                a.progress = c;
                a.throttle = knobs().throttle;
            }
        }
    }
#endif
    a.crt = pl.crt ? 1 : 0;
    a.cc = pl.cc;
    a.scratch = static_cast<uint8_t*>(scratch);
    if (pl.crt && !scratch) return FF_ERR_INTERNAL;
    a.trace = nullptr;
    static unsigned long long* trace_buf = nullptr;
    const bool tracing = knobs().trace;
    if (tracing) {
        if (!trace_buf) cudaMalloc(&trace_buf, 8 * 1024 * sizeof(unsigned long long));
        cudaMemsetAsync(trace_buf, 0, 8 * 1024 * sizeof(unsigned long long), st);
        a.trace = trace_buf;
    }
    a.die_map = nullptr;
    a.sched = nullptr;
#ifdef FF_EXPERIMENTS
    {
        const uint8_t* dm = nullptr;
        int* ring = nullptr;
        const int64_t units_total = (nt < num_sms() / kPair) ? nt : num_sms() / kPair;
        if (kPair == 2 && units_total >= 8 && die_schedule(&dm, &ring)) {
            static unsigned slot = 0;                 // fresh counters per launch (ring of 4096)
            int* c = ring + 4 * (slot++ % 4096);
            if (cudaMemsetAsync(c, 0, 4 * sizeof(int), st) == cudaSuccess) {
                a.die_map = dm;
                a.sched = c;
            }
        }
    }
#endif
    a.kinv = pl.kinv;
    a.kinv_sh = pl.kinv_sh;
    a.raster = kRasterDefault;
    a.hints = 3;  // TMA loads evict_last, C stores streaming (swept on c4)
    if (knobs().raster > 0) a.raster = knobs().raster;
    if (knobs().hints >= 0) a.hints = knobs().hints;

    CUtensorMap mapA, mapB;
    if (!make_plane_map(&mapA, A_limbs, I.L, m, I.k_pad, 128)) return FF_ERR_CUDA;
    if (!make_plane_map(&mapB, B_limbs, I.L, n, I.k_pad, kWide ? 128 : K::BN / kPair)) return FF_ERR_CUDA;

    if (set_smem_attr(reinterpret_cast<const void*>(ffgemm_tc_kernel<kPair, false, kWide>), K::SMEM) != cudaSuccess ||
        set_smem_attr(reinterpret_cast<const void*>(ffgemm_tc_kernel<kPair, true, kWide>), K::SMEM) != cudaSuccess)
        return FF_ERR_CUDA;
    const int64_t units = (num_sms() - pl.reserve_sms) / kPair;
    const int grid = static_cast<int>((nt < units ? nt : units) * kPair);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = K::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[3];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kPair;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // prologue overlaps the encoders
    attr[1].val.programmaticStreamSerializationAllowed = knobs().pdl ? 1 : 0;
    attr[2].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident (die-aware registration)
    attr[2].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = a.die_map ? 3 : 2;
    note_launch();
    prof_gemm_begin(st);
    const cudaError_t lerr = tracing ? cudaLaunchKernelEx(&cfg, ffgemm_tc_kernel<kPair, true, kWide>, mapA, mapB, a)
                                     : cudaLaunchKernelEx(&cfg, ffgemm_tc_kernel<kPair, false, kWide>, mapA, mapB, a);
    prof_gemm_end(st);
    if (lerr != cudaSuccess) return FF_ERR_CUDA;
    if (tracing) {  // development aid: per-CTA cycle counters, averaged over MMA-issuing CTAs
        unsigned long long h[8 * 1024];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, trace_buf, sizeof(unsigned long long) * 8 * grid, cudaMemcpyDeviceToHost);
        double s[8] = {0};
        int nl = 0, ne = 0;
        for (int b = 0; b < grid; ++b) {
            if (h[8 * b] > 0) { ++nl; for (int i = 0; i < 4; ++i) s[i] += h[8 * b + i]; }
            if (h[8 * b + 4] + h[8 * b + 5] > 0) { ++ne; for (int i = 4; i < 7; ++i) s[i] += h[8 * b + i]; }
        }
        for (int i = 0; i < 4; ++i) s[i] /= nl > 0 ? nl : 1;
        for (int i = 4; i < 7; ++i) s[i] /= ne > 0 ? ne : 1;
        fprintf(stderr, "[ff trace] kPair=%d m=%lld n=%lld k=%lld steps/CTA=%.0f  MMA thread: life %.3g cyc, "
                "wait slot %.1f%%, wait data %.1f%% | epilogue: wait %.1f%%, step work %.1f%% (%.0f cyc/step), "
                "final %.1f%%\n", kPair, (long long)m, (long long)n, (long long)k, s[3], s[0], 100 * s[1] / s[0],
                100 * s[2] / s[0], 100 * s[4] / s[0], 100 * s[5] / s[0], s[5] / (s[3] > 0 ? s[3] : 1), 100 * s[6] / s[0]);
    }
    return cudaGetLastError() == cudaSuccess ? 0 : FF_ERR_CUDA;
}

}  // namespace

size_t crt_scratch_bytes(const Plan& pl) {
    if (!pl.crt) return 0;
    // grid <= num_sms() CTAs (both kernels), 2 TMEM slots each
    return static_cast<size_t>(num_sms()) * 2 * static_cast<size_t>(pl.cc.nq) * kCrtPlane;
}

int launch_gemm_tc_multi(const Plan& pl, int64_t m, int64_t n, int64_t k, const int8_t* A_limbs,
                         const int8_t* B_limbs, const OutSpec* outs, int nout, int64_t ldc, int last_use,
                         void* scratch, cudaStream_t st, const int32_t* addend, int64_t ld_add) {
    // The CTA-pair kernel unless the problem has too few 256 x 256 tiles to
    // occupy the GPU (then the 128 x 256 single-CTA kernel gives more CTAs).
    const int64_t pair_tiles = ((m + 255) / 256) * ((n + 255) / 256);
    if (pl.force_pair == 1 || (pl.force_pair == 0 && pair_tiles * 2 < num_sms()))
        return launch_impl<1>(pl, m, n, k, A_limbs, B_limbs, outs, nout, ldc, last_use, scratch, st, addend, ld_add);
    // 256 x 512 tiles (limb plans) when the steps may run group-outer -- one weight
    // group, or operand planes that fit the L2 (else k-outer order is kept for DRAM
    // locality, launch_impl) -- and the wide tiles fill the GPU
    const ff_plan_info& I = pl.info;
    const int64_t wide_tiles = ((m + 255) / 256) * ((n + 511) / 512);
    const bool group_outer_ok =
        pl.korder == 1 ||
        (pl.korder_auto && (I.groups == 1 ||
                            static_cast<double>(I.L) * static_cast<double>(m + n) * static_cast<double>(I.k_pad) <=
                                kL2PlanesBytes));
    // auto: one weight group only (c3: -4%); with several groups the write-back
    // steps' staggered k-steps re-read A and it measured neutral (c2) or slower
    // (ftrsm 8192 +2%), so that is opt-in (ff_opts.wide_tiles = 1)
    const bool wide = (pl.wide > 0 && !pl.crt) ||
                      (pl.wide == 0 && !pl.crt && group_outer_ok && I.groups == 1 && wide_tiles * 2 >= num_sms());
    if (wide)
        return launch_impl<2, true>(pl, m, n, k, A_limbs, B_limbs, outs, nout, ldc, last_use, scratch, st, addend,
                                    ld_add);
    return launch_impl<2>(pl, m, n, k, A_limbs, B_limbs, outs, nout, ldc, last_use, scratch, st, addend, ld_add);
}

int launch_gemm_tc(const Plan& pl, int64_t m, int64_t n, int64_t k, const int8_t* A_limbs, const int8_t* B_limbs,
                   int32_t* C, int64_t ldc, void* scratch, cudaStream_t st) {
    const OutSpec o = {C, pl.mp.alpha, pl.mp.beta, 0, 0};
    return launch_gemm_tc_multi(pl, m, n, k, A_limbs, B_limbs, &o, 1, ldc, 1, scratch, st);
}

}  // namespace ff
