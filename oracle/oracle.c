/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for fgemm.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, constant or helper with the CUDA product path
 * (paper_cs_0601133_b200/csrc); it knows nothing of limbs, centring,
 * Barrett/Shoup reduction, k-blocking or Winograd.
 *
 * What it computes (the plain definition the method reaches exactly):
 *
 *   C_out[i,j] = ( (alpha mod p) * sum_{l<k} a'(i,l) * b'(l,j)
 *                  + (beta mod p) * c'(i,j) ) mod p        in [0, p)
 *
 *   a'(i,l) = A[i*lda + l] (transA = N) or A[l*lda + i] (transA = T), reduced mod p
 *   b'(l,j) = B[l*ldb + j] (transB = N) or B[j*ldb + l] (transB = T), reduced mod p
 *   c'(i,j) = C_in[i*ldc + j] reduced mod p; not read when beta = 0 mod p.
 *
 * Passages followed (PAPER.md line numbers):
 *   - l.139-143 (Sec. 2.1.2): Z_p embeds in Z, "the ring structure being
 *     preserved", so compute over Z and reduce once at the end;
 *   - l.261 (Sec. 3.2.2, Table 2): the operation is C <- alpha*A*B + beta*C;
 *   - l.117 (Sec. 2.1.1): residues are integers in [0, p-1] (our output range);
 *   - SPEC.md l.323 post-condition "C = alpha*A*B + beta*C (mod p), canonical";
 *   - BLAS conventions for trans/ld (row-major per SPEC.md l.23, l.89) --
 *     DESIGN.md reading R1; inputs outside [0,p) are reduced (reading R3);
 *     alpha/beta reduced mod p (reading R4); beta = 0 never reads C (R5).
 *
 * Arithmetic: a', b' < 2^31 so a'*b' < 2^62 fits uint64; a sum of k <= 2^40
 * such terms fits unsigned __int128 (no overflow is possible for any k this
 * library accepts).  The sum is reduced mod p once, then alpha*s + beta*c'
 * is formed in unsigned __int128 and reduced.  Nothing is reordered: each
 * output is the dot product over l = 0..k-1 in order.
 *
 * oracle_trsm (below) is the triangular solve of PAPER.md Sec. 4 written as
 * plain substitution; see its own header.
 *
 * Parity status: pinned (see tests/test_oracle_pins.py): SPEC worked example,
 * exhaustive GF(2)/GF(3) brute force, random shapes vs Python big integers,
 * identity/permutation matrices, closed forms, transpose identity,
 * Freivalds, linearity.
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* Euclidean residue of a signed integer ("the reverse
 * conversion consists in applying a reduction modulo p"). */
static uint64_t residue(int64_t x, int64_t p)
{
    int64_t r = x % p;
    if (r < 0) r += p;
    return (uint64_t)r;
}

static int is_n(char t) { return t == 'N' || t == 'n'; }
static int is_t(char t) { return t == 'T' || t == 't'; }

/* a'(i,l) */
static uint64_t a_elem(const int32_t *A, int64_t lda, int transA, int64_t i, int64_t l, int64_t p)
{
    return residue(transA ? A[l * lda + i] : A[i * lda + l], p);
}

/* b'(l,j) */
static uint64_t b_elem(const int32_t *B, int64_t ldb, int transB, int64_t l, int64_t j, int64_t p)
{
    return residue(transB ? B[j * ldb + l] : B[l * ldb + j], p);
}

/* One output entry: the definition above, written out. */
static int32_t entry(uint64_t p, int tA, int tB, int64_t k, uint64_t alpha,
                     const int32_t *A, int64_t lda, const int32_t *B, int64_t ldb,
                     uint64_t beta, int32_t cin, int64_t i, int64_t j)
{
    u128 s = 0;
    for (int64_t l = 0; l < k; ++l)
        s += (u128)(a_elem(A, lda, tA, i, l, (int64_t)p) * b_elem(B, ldb, tB, l, j, (int64_t)p));
    uint64_t sp = (uint64_t)(s % p);
    u128 t = (u128)alpha * sp;
    if (beta != 0)
        t += (u128)beta * residue(cin, (int64_t)p);
    return (int32_t)(uint64_t)(t % p);
}

static int check_args(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k)
{
    if (p < 2 || p >= (1u << 31)) return -1;
    if (!is_n(transA) && !is_t(transA)) return -2;
    if (!is_n(transB) && !is_t(transB)) return -3;
    if (m < 0) return -4;
    if (n < 0) return -5;
    if (k < 0) return -6;
    return 0;
}

/*
 * Full product: C (m x n, row-major, ldc) is overwritten in place with
 * (alpha*op(A)*op(B) + beta*C) mod p.  nthreads <= 0 means "all".
 */
int oracle_fgemm(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k,
                 uint32_t alpha, const int32_t *A, int64_t lda,
                 const int32_t *B, int64_t ldb, uint32_t beta,
                 int32_t *C, int64_t ldc, int nthreads)
{
    int e = check_args(p, transA, transB, m, n, k);
    if (e) return e;
    const int tA = is_t(transA), tB = is_t(transB);
    const uint64_t al = alpha % p, be = beta % p;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for collapse(2) schedule(dynamic, 64) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) {
            int32_t cin = be ? C[i * ldc + j] : 0;
            C[i * ldc + j] = entry(p, tA, tB, k, al, A, lda, B, ldb, be, cin, i, j);
        }
    return 0;
}

/*
 * Sampled rows: for r < nrows, Cout[r*ldo + j] = C_out[rows[r], j] for all
 * j < n, where C_in row rows[r] is supplied as Cin[r*ldi + j] (ignored when
 * beta = 0 mod p).  Same definition as oracle_fgemm, restricted to rows.
 */
int oracle_fgemm_rows(uint32_t p, char transA, char transB, int64_t m, int64_t n, int64_t k,
                      uint32_t alpha, const int32_t *A, int64_t lda,
                      const int32_t *B, int64_t ldb, uint32_t beta,
                      const int32_t *Cin, int64_t ldi,
                      const int64_t *rows, int64_t nrows,
                      int32_t *Cout, int64_t ldo, int nthreads)
{
    int e = check_args(p, transA, transB, m, n, k);
    if (e) return e;
    for (int64_t r = 0; r < nrows; ++r)
        if (rows[r] < 0 || rows[r] >= m) return -16;
    const int tA = is_t(transA), tB = is_t(transB);
    const uint64_t al = alpha % p, be = beta % p;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for collapse(2) schedule(dynamic, 64) num_threads(nthreads)
#endif
    for (int64_t r = 0; r < nrows; ++r)
        for (int64_t j = 0; j < n; ++j) {
            int32_t cin = be ? Cin[r * ldi + j] : 0;
            Cout[r * ldo + j] = entry(p, tA, tB, k, al, A, lda, B, ldb, be, cin, rows[r], j);
        }
    return 0;
}

/*
 * Matrix-vector product mod p: out[i] = (sum_l x'(i,l) * v[l]) mod p for the
 * rows x cols matrix op(X) (trans = T reads X[l*ld + i]).  v entries are
 * reduced mod p.  Used by the tests' Freivalds check (C*x vs A*(B*x)).
 */
int oracle_matvec(uint32_t p, char trans, int64_t rows, int64_t cols,
                  const int32_t *X, int64_t ld, const int32_t *v, int32_t *out, int nthreads)
{
    if (p < 2 || p >= (1u << 31)) return -1;
    if (!is_n(trans) && !is_t(trans)) return -2;
    const int t = is_t(trans);
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(nthreads)
#endif
    for (int64_t i = 0; i < rows; ++i) {
        u128 s = 0;
        for (int64_t l = 0; l < cols; ++l) {
            uint64_t x = residue(t ? X[l * ld + i] : X[i * ld + l], (int64_t)p);
            s += (u128)(x * residue(v[l], (int64_t)p));
        }
        out[i] = (int32_t)(uint64_t)(s % p);
    }
    return 0;
}

/* ------------------------------------------------------------------------
 * ftrsm: triangular solve with a matrix right-hand side (Sec. 4,
 * l.346-356: "the operation B <- U^{-1} B, where U is m x m upper triangular
 * and B is m x n", in the BLAS trsm convention l.348).  Written out as plain
 * substitution over Z/pZ, one right-hand side at a time -- the definition
 * the block-recursive Algorithm 1 (l.366-384) reaches exactly:
 *
 *   side = 'L':  op(A) X = alpha B   (op(A) m x m, X and B m x n)
 *   side = 'R':  X op(A) = alpha B   (op(A) n x n)
 *
 * op(A) = A (transA = 'N') or A^T ('T'); uplo names the triangle of A that is
 * read (the other one is never referenced); diag = 'U' means a unit diagonal
 * that is not read.  Divisions by the diagonal are multiplications by its
 * inverse mod p (extended Euclid), the field operations of l.398-400.
 * X overwrites B.  Returns 0, -i for an invalid argument i, or 1 when a
 * diagonal entry is not invertible mod p (B is then left partially solved).
 * ------------------------------------------------------------------------ */
static int64_t inv_mod(uint64_t a, int64_t p)
{
    int64_t r0 = p, r1 = (int64_t)(a % (uint64_t)p), s0 = 0, s1 = 1;
    while (r1 != 0) {
        int64_t q = r0 / r1, t = r0 - q * r1, u = s0 - q * s1;
        r0 = r1; r1 = t; s0 = s1; s1 = u;
    }
    if (r0 != 1) return -1;
    return ((s0 % p) + p) % p;
}

/* T(i, l) = op(A)[i][l], reduced mod p. */
static uint64_t t_elem(const int32_t *A, int64_t lda, int tA, int64_t i, int64_t l, int64_t p)
{
    return residue(tA ? A[l * lda + i] : A[i * lda + l], p);
}

int oracle_trsm(uint32_t p, char side, char uplo, char transA, char diag, int64_t m, int64_t n,
                uint32_t alpha, const int32_t *A, int64_t lda, int32_t *B, int64_t ldb, int nthreads)
{
    if (p < 2 || p >= (1u << 31)) return -1;
    const int left = (side == 'L' || side == 'l'), right = (side == 'R' || side == 'r');
    if (!left && !right) return -2;
    const int up = (uplo == 'U' || uplo == 'u'), lo = (uplo == 'L' || uplo == 'l');
    if (!up && !lo) return -3;
    if (!is_n(transA) && !is_t(transA)) return -4;
    const int unit = (diag == 'U' || diag == 'u');
    if (!unit && !(diag == 'N' || diag == 'n')) return -5;
    if (m < 0) return -6;
    if (n < 0) return -7;
    const int64_t dim = left ? m : n;
    if (lda < (dim > 1 ? dim : 1)) return -10;
    if (ldb < (n > 1 ? n : 1)) return -12;
    const int tA = is_t(transA);
    const int t_upper = up ^ tA;           /* op(A) is upper triangular */
    const int64_t P = (int64_t)p;
    const uint64_t al = alpha % p;
    /* inverses of the diagonal of op(A) */
    int singular = 0;
    int64_t *inv = NULL;
    if (dim > 0) {
        inv = (int64_t *)malloc((size_t)dim * sizeof(int64_t));
        if (!inv) return 2;
        for (int64_t i = 0; i < dim; ++i) {
            inv[i] = unit ? 1 : inv_mod(t_elem(A, lda, tA, i, i, P), P);
            if (inv[i] < 0) singular = 1;
        }
    }
    if (singular) { free(inv); return 1; }
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#endif
    if (left) {
        /* columns of B are independent right-hand sides */
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
#endif
        for (int64_t j = 0; j < n; ++j) {
            for (int64_t s = 0; s < m; ++s) {
                const int64_t i = t_upper ? m - 1 - s : s;      /* back / forward substitution */
                u128 acc = (u128)al * residue(B[i * ldb + j], P);
                u128 sub = 0;
                const int64_t l0 = t_upper ? i + 1 : 0, l1 = t_upper ? m : i;
                for (int64_t l = l0; l < l1; ++l)
                    sub += (u128)t_elem(A, lda, tA, i, l, P) * (uint64_t)B[l * ldb + j];
                const uint64_t v = (uint64_t)((acc % P + (P - sub % P)) % P);
                B[i * ldb + j] = (int32_t)(uint64_t)(((u128)v * (uint64_t)inv[i]) % P);
            }
        }
    } else {
        /* rows of B are independent: x_i op(A) = alpha b_i */
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads)
#endif
        for (int64_t i = 0; i < m; ++i) {
            for (int64_t s = 0; s < n; ++s) {
                const int64_t j = t_upper ? s : n - 1 - s;
                u128 acc = (u128)al * residue(B[i * ldb + j], P);
                u128 sub = 0;
                const int64_t l0 = t_upper ? 0 : j + 1, l1 = t_upper ? j : n;
                for (int64_t l = l0; l < l1; ++l)
                    sub += (u128)(uint64_t)B[i * ldb + l] * t_elem(A, lda, tA, l, j, P);
                const uint64_t v = (uint64_t)((acc % P + (P - sub % P)) % P);
                B[i * ldb + j] = (int32_t)(uint64_t)(((u128)v * (uint64_t)inv[j]) % P);
            }
        }
    }
    free(inv);
    return 0;
}

/* ------------------------------------------------------------------------
 * rank and determinant over Z/pZ (Sec. 6, l.655-657: "the rank is
 * the number of non-zero rows in U; the determinant is the product of the
 * diagonal elements of U"), by plain Gaussian elimination: for each column,
 * the first row (from the current one down) with a non-zero entry is the
 * pivot; rows are swapped (each swap flips the sign of the determinant) and
 * the rows below are eliminated.  X (m x n, row-major, ld) is copied, never
 * modified.  Returns 0, -i for an invalid argument i, 1 if a pivot is not
 * invertible mod p (p not prime), 2 on allocation failure.  det is written
 * only for m == n (0 when singular).
 * ------------------------------------------------------------------------ */
int oracle_rank_det(uint32_t p, int64_t m, int64_t n, const int32_t *X, int64_t ld,
                    int64_t *rank_out, int64_t *det_out)
{
    if (p < 2 || p >= (1u << 31)) return -1;
    if (m < 0) return -2;
    if (n < 0) return -3;
    if (ld < (n > 1 ? n : 1)) return -5;
    const int64_t P = (int64_t)p;
    uint64_t *a = (uint64_t *)malloc((size_t)(m * n > 0 ? m * n : 1) * sizeof(uint64_t));
    if (!a) return 2;
    for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) a[i * n + j] = residue(X[i * ld + j], P);
    int64_t r = 0;
    uint64_t det = 1;
    int neg = 0;
    for (int64_t col = 0; col < n && r < m; ++col) {
        int64_t piv = -1;
        for (int64_t i = r; i < m; ++i)
            if (a[i * n + col]) { piv = i; break; }
        if (piv < 0) { det = 0; continue; }
        if (piv != r) {
            for (int64_t j = 0; j < n; ++j) { uint64_t t = a[r * n + j]; a[r * n + j] = a[piv * n + j]; a[piv * n + j] = t; }
            neg ^= 1;
        }
        const int64_t iv = inv_mod(a[r * n + col], P);
        if (iv < 0) { free(a); return 1; }
        det = (uint64_t)(((u128)det * a[r * n + col]) % P);
        for (int64_t i = r + 1; i < m; ++i) {
            const uint64_t f = (uint64_t)(((u128)a[i * n + col] * (uint64_t)iv) % P);
            if (!f) continue;
            for (int64_t j = col; j < n; ++j)
                a[i * n + j] = (uint64_t)((a[i * n + j] + (u128)(P - f) * a[r * n + j]) % P);
        }
        ++r;
    }
    if (rank_out) *rank_out = r;
    if (det_out && m == n) *det_out = (r < m) ? 0 : (int64_t)(neg && det ? P - det : det);
    free(a);
    return 0;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
