// internal.h -- host-side structures shared by the library's translation units.
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

#include "../../include/ffgemm.h"

namespace ff {

constexpr int kMaxLimbs = 4;
constexpr int kMaxMod = FF_MAX_MODULI;       // CRT moduli
constexpr int kMaxGroups = kMaxMod;          // >= 2 kMaxLimbs - 1 weight groups
constexpr int kMaxPairs = 16;                // >= kMaxLimbs^2 limb pairs, >= kMaxMod moduli
constexpr int kBK = 128;        // bytes (= int8 elements) of K per pipeline stage (one 128B swizzle row)
constexpr int kMmaK = 32;       // K per tcgen05.mma.kind::i8 instruction
constexpr int kTileM = 128;     // rows of op(A) per CTA tile (= TMEM lanes)
constexpr int kTileN = 256;     // columns of C per CTA tile (= TMEM columns per accumulator)

// Residue-arithmetic constants for one p (all 32-bit; see modp.cuh for the
// algorithms: Barrett for int32 -> [0,p), Shoup for a*w mod p).
struct ModP {
    uint32_t p;
    uint32_t half;        // (p-1)/2: centred residues are in [-half, half]
    uint32_t mu;          // floor(2^32 / p)
    uint32_t off31;       // 2^31 mod p
    uint32_t w256;        // 256 mod p
    uint32_t w256_sh;     // floor(w256 * 2^32 / p)
    uint32_t alpha, alpha_sh;
    uint32_t beta, beta_sh;
    float inv_p;          // fl(1/p)
    float w256_over_p;    // fl(256/p)
    int32_t m1, m256;     // round(w 2^32 / p) for w = 1, 256 (clamped to 2^31-1), integer write-back
    int32_t int_wb;       // 1: integer write-back (p < 2^29), 0: fp32-reciprocal write-back
};

// Multi-modular (CRT) constants.  M = prod q_i, M_i = M / q_i.
// Small-modulus residues use the same Barrett form as residue_i32 (modp.cuh).
struct CrtConsts {
    int32_t nq;
    uint32_t q[kMaxMod];       // moduli, pairwise coprime, <= 256
    uint32_t mu[kMaxMod];      // floor(2^32 / q)
    uint32_t off31[kMaxMod];   // 2^31 mod q
    uint32_t half[kMaxMod];    // (q-1)/2: residues r > half are centred to r - q
    uint32_t v[kMaxMod];       // (M_i mod q_i)^-1 mod q_i
    uint32_t W[kMaxMod];       // M_i mod p
    uint32_t R[kMaxMod];       // round(2^24 / q_i): fixed-point 1/q_i for the quotient t
    float fq[kMaxMod];         // q as float (encoder, fp32 residue path)
    float finv[kMaxMod];       // fl(1/q)
    float fw15[kMaxMod];       // 2^15 mod q, as float
    uint32_t Mneg;             // (p - M mod p) mod p
    unsigned long long mu64;   // floor(2^64 / p) (Barrett for the 64-bit sum)
};

struct Plan {
    ff_plan_info info;
    ModP mp;
    bool crt;                        // FF_SCHEME_CRT: groups are moduli, one pair (i, i) each
    bool fp64;                       // FF_SCHEME_FP64: the paper-literal DMMA engine (gemm_f64.cu)
    CrtConsts cc;
    int npairs;                      // L*L (limbs) or L (CRT)
    int pair_i[kMaxPairs];
    int pair_j[kMaxPairs];
    int group_first[kMaxGroups];     // pairs of group w are [group_first[w], group_first[w]+group_len[w])
    int group_len[kMaxGroups];
    bool saturate;
    int force_pair;                  // 0 auto, 1 single-CTA kernel, 2 CTA-pair kernel
    int reserve_sms;                 // leave this many SMs free (LQUP lookahead: a panel kernel co-runs)
    int korder;                      // 1 group-outer, 2 k-outer step order
    bool korder_auto;                // k-outer chosen by default (no option, no kb_override):
                                     // the launch may fall back to group-outer for L2-sized operands
    uint32_t kinv, kinv_sh;          // 256^-(G-1) mod p and its Shoup constant (k-outer carry)
    bool all_auto;                   // no option forced: the planner may route to the small-field path
    bool canonical_ab;               // (internal callers) A, B hold canonical residues in [0, p)
    int small_mode;                  // small-field kernels: -1 size rule, 0 never, 1 mma.sync kernels
                                     // whenever valid, 2 the tcgen05 latency kernel whenever valid
    int wide;                        // ff_opts.wide_tiles: 0 auto, 1 force, -1 never (gemm_tc.cu)
};

constexpr int64_t kKbLocalityBytes = 8192;  // L * kb per row-slice in k-outer order (swept on c4, c5)

// planner.cpp
int make_plan(uint32_t p, int64_t k, const ff_opts* opts, Plan* out);
void set_scalars(Plan* pl, uint32_t alpha, uint32_t beta);

// encode.cu
cudaError_t launch_encode(const Plan& pl, int kmajor_src, int64_t rows, int64_t k,
                          const int32_t* X, int64_t ldx, int8_t* limbs, cudaStream_t st);
// CRT scratch of the GEMM kernel: per CTA and TMEM slot, the (nq-1) byte planes
// of u_i = r_i v_i mod q_i for a 128 x 256 tile (0 for limb plans).
size_t crt_scratch_bytes(const Plan& pl);
cudaError_t launch_scale_c(const ModP& mp, int64_t m, int64_t n, int32_t* C, int64_t ldc,
                           cudaStream_t st);

// gemm_small.cu: p < 2^16 on warp-level tensor cores, no encoders (latency path)
bool small_path_ok(const Plan& pl, int64_t m, int64_t n, int64_t k);
int launch_gemm_small(const Plan& pl, bool tA, bool tB, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                      const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, cudaStream_t st);

bool small_canon_ok(const Plan& pl, bool tA, bool tB, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                    const int32_t* B, int64_t ldb);
// LQUP's panel chain (three canonical products of at most 128 x 128, p < 2^16, the
// third reading the first two's outputs; products 0 and 1 in place) in one
// cooperative launch; FF_ERR_INTERNAL if it does not apply (the caller then runs
// the three products one by one).
struct SmallChainProduct {
    int64_t m, n, k;
    const int32_t* A;
    int64_t lda;
    const int32_t* B;
    int64_t ldb;
    int32_t* C;
    int64_t ldc;
};
int launch_small_chain(const Plan& pl01, const Plan& pl2, const SmallChainProduct (&pr)[3], cudaStream_t st);
// alias: C overlaps A or B (in-place products): a cooperative launch with a grid barrier between the
// reads and the writes; FF_ERR_INTERNAL if the grid cannot be co-resident
// reduce: A, B are raw int32 (any value), reduced per slice in shared memory (small_stream_ok)
int launch_gemm_small_canon(const Plan& pl, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                            const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, bool alias, cudaStream_t st,
                            bool reduce = false);
bool small_stream_ok(const Plan& pl, bool tA, bool tB, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                     const int32_t* B, int64_t ldb);
bool small_wide_ok(const Plan& pl, bool tA, bool tB, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                   const int32_t* B, int64_t ldb);
int launch_gemm_small_wide(const Plan& pl, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                           const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, bool alias, cudaStream_t st);

// gemm_lat.cu: p < 2^16 latency path on tcgen05 (one kernel, split-K cluster, no encoders)
bool lat_path_ok(const Plan& pl, int64_t m, int64_t n, int64_t k);
int launch_gemm_lat(const Plan& pl, bool tA, bool tB, int64_t m, int64_t n, int64_t k, const int32_t* A, int64_t lda,
                    const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, cudaStream_t st);

// gemm_tc.cu
struct OutSpec {          // C <- (a * A B + b * C) mod p for one output block
    int32_t* C;
    uint32_t a, b;
    int64_t ld;           // leading dimension of C (0: the launch's ldc)
    int32_t add;          // 1: C <- (a * (A B + addend) + b * C) mod p (the launch's addend)
};
// `scratch`: crt_scratch_bytes(pl) bytes of device memory (ignored for limb plans).
// `addend` (optional, residues in [0, p), leading dimension ld_add): added to the
// product mod p for the outputs with `add` set (a Winograd temporary).
int launch_gemm_tc_multi(const Plan& pl, int64_t m, int64_t n, int64_t k, const int8_t* A_limbs,
                         const int8_t* B_limbs, const OutSpec* outs, int nout, int64_t ldc, int last_use,
                         void* scratch, cudaStream_t st, const int32_t* addend = nullptr, int64_t ld_add = 0);
int launch_gemm_tc(const Plan& pl, int64_t m, int64_t n, int64_t k, const int8_t* A_limbs,
                   const int8_t* B_limbs, int32_t* C, int64_t ldc, void* scratch, cudaStream_t st);

// winograd.cu
size_t winograd_ws_bytes(const Plan& half, int64_t m, int64_t n, int64_t k);
int run_winograd(const Plan& half, bool transA, bool transB, int64_t m, int64_t n, int64_t k, const int32_t* A,
                 int64_t lda, const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, void* ws, cudaStream_t st);

// gemm_f64.cu: the paper-literal fp64 engine (workspace = two double planes; with
// `levels` > 0 recursive Winograd levels without reduction, Sec. 3.2.3,
// also the unreduced result and the recursion's temporaries)
size_t f64_ws_bytes(const Plan& pl, int64_t m, int64_t n, int64_t k, int levels);
int run_f64(const Plan& pl, int levels, bool transA, bool transB, int64_t m, int64_t n, int64_t k, const int32_t* A,
            int64_t lda, const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, void* ws, cudaStream_t st);

// gen.cu
cudaError_t launch_fill_uniform(int32_t* X, int64_t rows, int64_t cols, int64_t ld, uint32_t p,
                                uint64_t seed, uint32_t stream_id, int64_t index0,
                                cudaStream_t st);

int num_sms();

// Per-device, thread-safe cudaFuncSetAttribute(MaxDynamicSharedMemorySize) on the
// current device, done once per (device, kernel): the attribute is per device
// context, so a process-wide "done" flag would skip it on a second GPU.
cudaError_t set_smem_attr(const void* fn, int bytes);

// Developer knobs, read from the environment ONCE per process.
// None changes a result: they pick between exact code paths or turn on
// diagnostics.  Experiments that needed extra machinery (cluster throttling,
// the die-aware schedule) are compiled only with -DFF_EXPERIMENTS.
struct Knobs {
    int small;          // FF_SMALL: -1 default rule, 0 never, 1 whenever valid
    bool pdl;           // !FF_NOPDL: programmatic dependent launch of the GEMM
    bool trace;         // FF_TRACE: per-CTA cycle counters (diagnostic kernel build)
    int raster;         // FF_RASTER: tile rows per raster band (0 = default)
    int hints;          // FF_HINTS: L2 policy bits (-1 = default)
    int korder;         // FF_KORDER: 0 default, 1 group-outer, 2 k-outer
    int64_t kbloc;      // FF_KBLOC: k-outer locality bytes (0 = default)
    bool enc_notma;     // FF_ENC_NOTMA: LSU-load transposing encoders
    bool wide;          // !FF_NOWIDE: 256 x 512 tiles for single-step GEMMs (gemm_tc.cu)
    int wdelta;         // FF_WDELTA: staggered k-steps of the wide tiles' halves (0 = default)
    int wdelta_wb;      // FF_WDELTA_WB: the same before write-back steps (0 = default)
    int throttle;       // FF_THROTTLE (FF_EXPERIMENTS builds only)
    bool die_aware;     // FF_DIE_AWARE (FF_EXPERIMENTS builds only)
};
const Knobs& knobs();

// Benchmark instrumentation (ff_prof_start/stop, include/ffgemm.h): count every
// kernel launch of the fgemm path, and bracket each GEMM-kernel launch with
// two CUDA events on its stream while recording is on.  No-ops otherwise.
void note_launch(int n = 1);
void prof_gemm_begin(cudaStream_t st);
void prof_gemm_end(cudaStream_t st);

// api.cu: the classical device path (encode A, encode B, tcgen05 GEMM) for
// callers inside the library (trsm.cu), and its workspace size.
int gemm_dev(const Plan& pl, char transA, char transB, int64_t m, int64_t n, int64_t k, const int32_t* A,
             int64_t lda, const int32_t* B, int64_t ldb, int32_t* C, int64_t ldc, void* ws, cudaStream_t st);
size_t gemm_ws_bytes(const Plan& pl, int64_t m, int64_t n);
int check_device();

// dies.cu: SM -> die map and per-launch counter ring for the die-aware schedule
bool die_schedule(const uint8_t** die_map, int** sched);

}  // namespace ff
