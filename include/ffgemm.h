/*
 * ffgemm.h -- C ABI of the B200 (sm_100a) fgemm library: exact modular matrix
 * multiplication over a word-size prime field,
 *
 *     C <- (alpha * op(A) * op(B) + beta * C) mod p,        results in [0, p).
 *
 * The operation is the paper's fgemm ("we named our routine
 * over a word-size finite field fgemm"; Table 2 caption l.276, "operation
 * C <- alpha A x B + beta C").  The paper computes it over Z with a numerical
 * BLAS kernel and delayed modular reduction (Sec. 2.1.2, l.139-159, Eq. (1)/(2));
 * this library does the same with int8 "limbs" on the 5th-generation tensor
 * cores (tcgen05.mma.kind::i8, exact int32 accumulation in TMEM), blocking k
 * by the Eq. (2) analogue of the int32 accumulator.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Storage is row-major with a leading dimension (elements), as in
 *    SPEC.md l.22-26 / l.89.  op(A) is m x k: transA = 'N'/'n' means A is
 *    stored m x k with lda >= max(1,k); 'T'/'t' means A is stored k x m with
 *    lda >= max(1,m).  Likewise op(B) is k x n with ldb, and C is m x n with
 *    ldc >= max(1,n).  Indices and sizes are 64-bit; elements are int32.
 *  - Inputs are meant to be canonical residues in [0,p) (BASELINE.json
 *    north_star (1)); any int32 is accepted and reduced (Euclidean) mod p
 *    (reading R3).  alpha and beta are reduced mod p (reading R4);
 *    alpha = p-1 means -1.  Output is always canonical [0,p).
 *  - beta = 0 (mod p): C is write-only and never read (BLAS convention,
 *    reading R5).  k = 0 or alpha = 0 (mod p): C <- beta*C mod p.
 *    m = 0 or n = 0: no-op.
 *  - p: 2 <= p < 2^31 (primality is not required: the result is exact in
 *    the ring Z/pZ).
 *  - Device pointers ("dev") must be device memory of the current CUDA device;
 *    they are owned by the caller.  A and B are read only; C is updated in
 *    place and must not overlap A or B.  Work is asynchronous with respect to
 *    the host (like cuBLAS): errors from kernels surface at the next sync.
 *  - Return value: 0 on success.  A negative value -i means argument i is
 *    invalid, in BLAS xerbla order of ff_gemm's signature (1 p, 2 transA,
 *    3 transB, 4 m, 5 n, 6 k, 8 A, 9 lda, 10 B, 11 ldb, 13 C, 14 ldc;
 *    15+ for the extra arguments of the _ex / split entry points).  A positive
 *    value is one of the FF_ERR_* runtime codes below.  ff_strerror() names it.
 *  - There is no CPU fallback: without an sm_100 device every compute entry
 *    point returns FF_ERR_ARCH (or FF_ERR_CUDA).
 */
#ifndef FFGEMM_H
#define FFGEMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FF_OK 0
#define FF_ERR_CUDA 1     /* a CUDA runtime/driver call failed */
#define FF_ERR_NOMEM 2    /* device or pinned allocation failed / workspace too small */
#define FF_ERR_ARCH 3     /* current device is not sm_100 (B200) */
#define FF_ERR_OPTS 4     /* ff_opts invalid (e.g. kb_override above the safe bound) */
#define FF_ERR_INTERNAL 5 /* planner could not represent p (should not happen for p < 2^31) */

/* Limb schemes.  S: balanced signed digits in [-128,127];
 * T: two's-complement bytes (low limbs u8 in [0,255], top limb s8).
 * CRT: multi-modular (the paper's "Chinese remainder
 * algorithm" for large fields): the centred residue c is
 * replaced by its centred residues modulo pairwise-coprime q_i <= 256, one
 * exact int8 product per modulus, and the exact integer dot product is
 * reconstructed from them before the final reduction mod p.  AUTO uses it
 * when it needs fewer int8 products than the limb schemes (large p). */
#define FF_SCHEME_AUTO 0
#define FF_SCHEME_S 1
#define FF_SCHEME_T 2
#define FF_SCHEME_CRT 3
#define FF_MAX_MODULI 16
/* FP64: the paper-literal "Zpz-double" engine: centred
 * residues as doubles on the fp64 tensor cores (DMMA), lambda products
 * accumulated exactly between floating-point reductions, lambda from Eq. (2)
 * with gamma = 53, or l recursive Winograd levels with no reduction at all
 * under Corollary 3.4 (ff_opts.winograd = l).  Only when chosen explicitly;
 * needs lambda >= 4, i.e. p <= 2^26 + 1 (the paper's feasibility bound,
 * l.882).  Not available for ff_encode / ff_gemm_limbs / ff_gemm_host
 * (FF_ERR_OPTS). */
#define FF_SCHEME_FP64 4

/* Options for the _ex / split entry points.  Zero-initialise and set fields;
 * a NULL pointer means all defaults. */
typedef struct ff_opts {
    int32_t winograd;       /* 0 auto, 1 one Winograd level (Table 2; needs even
                               m, n, k with m, n >= 512 and k >= 256, else FF_ERR_OPTS),
                               -1 never.  FF_SCHEME_FP64: l = 1, 2 or 3 recursive levels
                               with unreduced pre-additions (Sec. 3.2.3; any
                               shape: m, n zero-padded to multiples of 2^l, the last
                               k mod 2^l columns peeled), accepted iff k < k_winograd[l]
                               of ff_plan_info, else FF_ERR_OPTS */
    int32_t scheme;         /* FF_SCHEME_*; AUTO picks the fewest int8 products: limbs
                               (S on ties) unless CRT needs clearly fewer */
    int64_t kb_override;    /* 0: planner k-block; else k-block length in elements,
                               rounded down to a multiple of 128; must not exceed the
                               safe bound (else FF_ERR_OPTS).  Forces mid-k reductions. */
    int32_t debug_saturate; /* 1: set the MMA saturate bit (test builds only; a clamp
                               then shows as a mismatch instead of a silent wrap) */
    int32_t cta_group;      /* 0 auto; 1 force the 128x256 single-CTA kernel; 2 force the
                               256x256 CTA-pair (tcgen05 cta_group::2) kernel */
    int32_t host_block;     /* ff_gemm_host only: rows/columns of C per pipelined block
                               (rounded up to 256); 0 = auto (~4096) */
    int32_t korder;         /* step order of the kernel: 0 auto (k-outer when the operand
                               planes exceed ~192 MB, else group-outer), 1 group-outer (each
                               weight group over all of k), 2 k-outer (each k-block through
                               all groups: L2 locality) */
    int32_t debug_unchecked_kb; /* test builds only: accept a kb_override above the safe
                               bound, or (FF_SCHEME_FP64) Winograd levels with k past
                               k_winograd (to show that the bounds are needed); results
                               are then not guaranteed */
    int32_t inputs_canonical; /* 1: the caller guarantees every element of op(A), op(B) is a
                               canonical residue in [0, p) (C may still be any int32): for
                               p < 2^16 short-K products may then stream A and B raw
                               (DESIGN.md §4.10).  Results are undefined if violated. */
    int32_t small_path;     /* latency kernels for small fields: 0 by the
                               size rule, 1 the mma.sync kernels whenever they apply, 2 the
                               tcgen05 split-K kernel whenever it applies, -1 never (results
                               are identical) */
    int32_t wide_tiles;     /* tcgen05 GEMM tile shape: 0 auto (256 x 512 CTA-pair tiles with
                               staggered halves for one-limb plans, p < 256, when they fill
                               the GPU), 1 256 x 512 for every limb plan on the
                               CTA-pair kernel (ignored for CRT plans and with cta_group = 1),
                               -1 never (256 x 256).  Results are identical. */
} ff_opts;

/* The plan the library derives from (p, k, opts): host-only, no GPU needed. */
typedef struct ff_plan_info {
    uint32_t p;
    int32_t L;               /* int8 planes per operand: limbs (1..4) or, for
                                FF_SCHEME_CRT, moduli (2..FF_MAX_MODULI) */
    int32_t scheme;          /* FF_SCHEME_S, FF_SCHEME_T, FF_SCHEME_CRT or FF_SCHEME_FP64 */
    int32_t groups;          /* accumulation groups: 2L-1 weight groups w = i+j
                                (limbs) or L moduli (CRT) */
    int32_t limb_signed[4];  /* 1 if limb i is s8, 0 if u8 (limb schemes) */
    int32_t digit_max[4];    /* D_i = max |limb i| over all centred residues
                                (limb schemes; CRT: max |residue| of plane i, i < 4) */
    int64_t group_bound[7];  /* B_w = sum_{i+j=w} D_i D_j  (per unit of k; CRT: D_w^2) */
    int64_t group_bound_max; /* max_w B_w */
    int64_t kb_max;          /* floor((2^31-1-carry_max) / max_w B_w): Eq. (2) analogue */
    int64_t kb;              /* k-block actually used (multiple of 128, <= kb_max) */
    int64_t k_pad;           /* k rounded up to a multiple of 16 (limb plane row length) */
    int64_t num_kblocks;     /* ceil(k / kb); 1 for every BASELINE config */
    int32_t centre_max;      /* (p-1)/2 (p/2 for p = 2) */
    int32_t reserved0;
    int64_t carry_max;       /* bound on |value| written back into the accumulator
                                between steps */
    int32_t korder;          /* 1 group-outer, 2 k-outer (CRT: always 1) */
    int32_t nmod;            /* FF_SCHEME_CRT: number of moduli (= L); else 0 */
    uint32_t moduli[FF_MAX_MODULI]; /* CRT moduli q_0 > q_1 > ..., pairwise coprime,
                                q_i <= 256, with prod q_i >= 4 k centre_max^2 */
    int32_t log2_M_floor;    /* CRT: floor(log2(prod q_i)) */
    int32_t log2_bound_ceil; /* CRT: ceil(log2(4 k centre_max^2)) (<= log2_M_floor) */
    int64_t k_winograd[4];   /* FF_SCHEME_FP64: l = 1..3 Winograd levels without any
                                reduction are accepted iff k < k_winograd[l] (Corollary 3.4,
                                PAPER.md l.304-312, exact form: ceil(2^53 / v_l^2) 2^l with
                                v_l = 3^l centre_max, Theorem 3.1 on the balanced range);
                                [0] = lambda + 1 (Eq. (2)); 0 for the int8 schemes */
} ff_plan_info;

/* Library version (major*10000 + minor*100 + patch). Host only. */
int ff_version(void);

/* Name of a return code. Host only; never NULL. */
const char *ff_strerror(int code);

/* 0 if `device` is an sm_100 GPU usable by this library, else FF_ERR_ARCH /
 * FF_ERR_CUDA. */
int ff_device_check(int device);

/* Derive the plan for (p, k, opts) (Eq. (2), l.155, generalised to
 * limbs: DESIGN.md §4.2).  Host only.  Returns -1 (p), -6 (k) or FF_ERR_OPTS. */
int ff_plan_query(uint32_t p, int64_t k, const ff_opts *opts, ff_plan_info *out);

/* Core call, on the legacy default stream with a library-owned cached
 * workspace (not thread-safe across host threads).  A, B, C: dev. */
int ff_gemm(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k,
            uint32_t alpha, const int32_t *A, int64_t lda, const int32_t *B, int64_t ldb,
            uint32_t beta, int32_t *C, int64_t ldc);

/* Bytes of device workspace ff_gemm_ex needs for this problem. Host only. */
size_t ff_gemm_workspace_size(uint32_t p, char transA, char transB, int64_t m, int64_t n,
                              int64_t k, const ff_opts *opts);

/* As ff_gemm, on `stream` (a cudaStream_t; NULL = legacy default), with
 * options and a caller workspace (dev, >= ff_gemm_workspace_size bytes,
 * 256-byte aligned; NULL = library pool).  Reentrant with distinct workspaces.
 * Extra argument codes: -15 opts, -16 workspace. */
int ff_gemm_ex(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k,
               uint32_t alpha, const int32_t *A, int64_t lda, const int32_t *B, int64_t ldb,
               uint32_t beta, int32_t *C, int64_t ldc, const ff_opts *opts,
               void *workspace, size_t workspace_bytes, void *stream);

/* *levels <- the Winograd levels ff_gemm_ex would run for this problem with
 * these options (host only, no GPU needed): 0 classical, 1 one level (int8
 * engines: forced by opts->winograd or, by default, where it was measured to
 * win -- DESIGN.md §7), 1..3 (FF_SCHEME_FP64 with opts->winograd = l).
 * Returns 0, -1 p, -2 m, -3 n, -4 k, -6 levels NULL, or FF_ERR_OPTS (options
 * invalid, or a forced level the shape or Corollary 3.4 does not allow).  The
 * multi-GPU driver uses it to decide whether a rank multiplies its panel in
 * one call. */
int ff_gemm_winograd_levels(uint32_t p, int64_t m, int64_t n, int64_t k, const ff_opts *opts, int32_t *levels);

/* As ff_gemm, but A, B and C are HOST pointers (pinned for full PCIe speed;
 * pageable works).  Copies in, computes on the current device, copies C back
 * and synchronises before returning.  Device buffers are library-owned and
 * cached.  The work is pipelined over blocks of C on three library streams
 * (host->device copies, compute, device->host copies), so the PCIe transfers
 * of one block overlap the encode/GEMM of others.  This is
 * the end-to-end entry point the bench's "e2e" number uses. */
int ff_gemm_host(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k,
                 uint32_t alpha, const int32_t *A, int64_t lda, const int32_t *B, int64_t ldb,
                 uint32_t beta, int32_t *C, int64_t ldc, const ff_opts *opts);

/* ---- split entry points (multi-GPU row-panel path) ----------
 * Limb planes: int8, layout [L][rows][k_pad] (plane l, row r, column kk at
 * byte l*rows*k_pad + r*k_pad + kk), where L and k_pad come from
 * ff_plan_query(p, k, opts) and rows is the operand's row count in K-major
 * form (m for op(A), n for op(B)^T).  Size: L*rows*k_pad bytes, dev,
 * 16-byte aligned.  Under FF_SCHEME_CRT plane l holds the centred residues
 * modulo moduli[l] (s8) instead of a limb. */

/* Encode `rows` K-major rows of an operand into limb planes: row r, column
 * kk of the K-major view is X[r*ldx + kk] if kmajor_src = 1 (op(A) with
 * transA='N', or op(B)^T with transB='T'), else X[kk*ldx + r] (the
 * transposed cases).  Columns k..k_pad-1 are written as zero.
 * X: dev int32; limbs: dev.  Codes: -1 p, -2 k, -4 rows, -5 X, -6 ldx, -7 limbs. */
int ff_encode(uint32_t p, int64_t k, const ff_opts *opts, int kmajor_src, int64_t rows,
              const int32_t *X, int64_t ldx, int8_t *limbs, void *stream);

/* C (m x n, ldc) <- (alpha * op(A) * op(B) + beta * C) mod p from limb planes
 * produced by ff_encode with the same (p, k, opts): A_limbs has m rows,
 * B_limbs has n rows.  Under FF_SCHEME_CRT the kernel's per-CTA residue
 * scratch comes from a library-owned per-device buffer (so concurrent calls
 * on different streams of one device are not reentrant for CRT plans).
 * Codes: -1 p, -2 m, -3 n, -4 k, -7 A_limbs, -8 B_limbs, -10 C, -11 ldc. */
int ff_gemm_limbs(uint32_t p, int64_t m, int64_t n, int64_t k, const ff_opts *opts,
                  uint32_t alpha, const int8_t *A_limbs, const int8_t *B_limbs,
                  uint32_t beta, int32_t *C, int64_t ldc, void *stream);

/* ---- ftrsm: triangular solve with a matrix right-hand side ---------------
 * PAPER.md Sec. 4 (l.346-356, the BLAS trsm operation over Z/pZ) by the
 * block recursive Algorithm 1 (l.366-384) on the tensor-core fgemm, with the
 * nb x nb diagonal blocks inverted once so the leaves are GEMMs too
 * (DESIGN.md §13):
 *
 *   side = 'L':  op(A) X = alpha B,  op(A) m x m;   side = 'R':  X op(A) = alpha B,  op(A) n x n;
 *
 * X (m x n) overwrites B.  op(A) = A ('N') or A^T ('T'); uplo ('U'/'L')
 * names the triangle of A that is read -- the other one is never
 * referenced; diag = 'U': unit diagonal, not read; 'N': the diagonal must be
 * invertible mod p (not checked: as in BLAS, a singular A gives an
 * undefined X).  A (lda >= max(1, dim)) and B (ldb >= max(1, n)) are dev,
 * row-major, int32, any values (reduced mod p); A must not overlap B.
 * Output canonical in [0, p).  Codes, BLAS order: -1 p, -2 side, -3 uplo,
 * -4 transA, -5 diag, -6 m, -7 n, -9 A, -10 lda, -11 B, -12 ldb,
 * -15 workspace; positive FF_ERR_*.  ff_trsm allocates its workspace
 * (cudaMalloc/cudaFree: synchronous); ff_trsm_ex takes a caller workspace
 * (>= ff_trsm_workspace_size bytes, 256-byte aligned) and a stream and is
 * asynchronous. */
int ff_trsm(uint32_t p, char side, char uplo, char transA, char diag, int64_t m, int64_t n,
            uint32_t alpha, const int32_t *A, int64_t lda, int32_t *B, int64_t ldb);

size_t ff_trsm_workspace_size(uint32_t p, char side, int64_t m, int64_t n, const ff_opts *opts);

int ff_trsm_ex(uint32_t p, char side, char uplo, char transA, char diag, int64_t m, int64_t n,
               uint32_t alpha, const int32_t *A, int64_t lda, int32_t *B, int64_t ldb,
               const ff_opts *opts, void *workspace, size_t workspace_bytes, void *stream);

/* ---- LQUP, rank, determinant -----------------------------------------------
 * The rank-revealing triangular factorization of PAPER.md Sec. 5.1 (l.575-590)
 * reduced to the tensor-core fgemm, returned in place in the
 * PLUQ arrangement (reading R20): with Q[i] = the original row now at row i
 * and P[j] = the original column now at column j,
 *     A[Q[i]][P[j]] = sum_{k < r} L[i][k] U[k][j]  (mod p),
 * L (m x r) unit lower triangular, stored strictly below the diagonal of the
 * first r columns of A; U (r x n) upper triangular with a non-zero diagonal,
 * stored on and above the diagonal of the first r rows; rows >= r hold their
 * L entries and zeros.  Pivoting: the first non-zero entry of each row (rows in
 * order), so the pivot columns are the row-echelon pivots.  A: dev, int32,
 * any values (reduced mod p), lda >= max(1, n).  Q (m), P (n), rank: HOST
 * outputs.  Synchronous (the host needs each panel's rank).  p prime (pivots
 * are inverted).  Codes: -1 p, -2 m, -3 n, -4 A, -5 lda, -6 Q, -7 P, -8 rank,
 * -10 workspace.  ff_lqup allocates its workspace; ff_lqup_ex takes one
 * (>= ff_lqup_workspace_size bytes, 256-byte aligned) and a stream. */
int ff_lqup(uint32_t p, int64_t m, int64_t n, int32_t *A, int64_t lda, int64_t *Q, int64_t *P,
            int64_t *rank);

size_t ff_lqup_workspace_size(uint32_t p, int64_t m, int64_t n, const ff_opts *opts);

int ff_lqup_ex(uint32_t p, int64_t m, int64_t n, int32_t *A, int64_t lda, int64_t *Q, int64_t *P,
               int64_t *rank, const ff_opts *opts, void *workspace, size_t workspace_bytes, void *stream);

/* Rank (and, for m == n, the determinant in [0, p)) of A (dev, not modified),
 * PAPER.md Sec. 6 (l.655-657): "the rank is the number of non-zero rows in U;
 * the determinant is the product of the diagonal elements of U" (times the
 * signs of the permutations).  det may be NULL.  Codes: -1 p, -2 m, -3 n, -4 A,
 * -5 lda, -6 rank, -7 det requested for m != n. */
int ff_rank_det(uint32_t p, int64_t m, int64_t n, const int32_t *A, int64_t lda, int64_t *rank,
                uint32_t *det);

/* ---- kernel timing for benchmarks (host) -----------------------------------
 * ff_prof_start(capacity): from now on every GEMM-kernel launch of the library
 * (tcgen05 limb/CRT, small-field, fp64 -- on the current device, any stream) is
 * bracketed by two CUDA events recorded on that launch's own stream, for the
 * first `capacity` launches, and every kernel launch of the fgemm path
 * (encoders, pre-additions, GEMMs, scaling) is counted.  Returns 0, -1
 * (capacity outside [0, 2^20]) or FF_ERR_CUDA.
 * ff_prof_stop(gemm_ms, cap, launches): stops recording, waits for the
 * recorded events, writes min(cap, recorded) per-launch durations in ms to
 * gemm_ms (host, may be NULL), stores the number of kernel launches counted
 * since ff_prof_start in *launches (may be NULL) and returns the number of
 * GEMM launches recorded (or -FF_ERR_CUDA).  Process-wide state: not for
 * concurrent use by several host threads. */
int ff_prof_start(int32_t capacity);
int ff_prof_stop(float *gemm_ms, int32_t cap, int64_t *launches);

/* The int8 tensor-core ceiling of the current device, measured: the hot
 * kernel's instruction (tcgen05.mma.cta_group::2.kind::i8, 256 x 256 x 32,
 * s32 in TMEM) issued back to back from SMEM-resident operands by every CTA
 * pair, no data movement, no epilogue; `iters` x 4 MMAs per pair, best of 3
 * timed launches on the legacy default stream (synchronous).  *tops receives
 * int8 tera-ops/s (2 per multiply-add).  The analogue of the paper's dgemm
 * yardstick for fgemm.  Codes: -1 iters <= 0 or tops
 * NULL; FF_ERR_ARCH / FF_ERR_CUDA. */
int ff_mma_ceiling(int32_t iters, double *tops);

/* ---- synthetic inputs (device twin of ffgen/__init__.py) -----------------
 * X[r*ld + c] = v[index0 + r*cols + c] for r < rows, c < cols, where v is the
 * (seed, stream_id) sequence of ffgen: v[i] = (mix64(key + (i+1)*GAMMA) >> 11)
 * mod p, key = mix64(seed*16 + stream_id).  X: dev. */
int ff_fill_uniform(int32_t *X, int64_t rows, int64_t cols, int64_t ld, uint32_t p,
                    uint64_t seed, uint32_t stream_id, int64_t index0, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FFGEMM_H */
