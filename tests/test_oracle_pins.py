"""Pins for the CPU oracle (oracle/): checks against what the paper and the
mathematics fix, never against the oracle's own formula.

Each check is chosen so that a plausible slip in oracle.c -- a dropped term
(beta*C, the last l), a transposed operand, a wrong ld/index, a sign, an
overflow of the accumulator, a wrong residue of negative input -- fails at
least one of them.
"""
import itertools
import os
import random

import numpy as np
import pytest

import ffgen
import oracle
from oracle import winograd

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CONFIG_PRIMES = [251, 65521, 8388593, 67108859]
PRIMES = [2, 3, 5, 7] + CONFIG_PRIMES + [2 ** 31 - 1]


def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([int(t) for t in line.split()])
    return rows


def _linear_map_product(p, alpha, A, B, beta, C):
    """Brute force by a different route: column j of A*B is A applied to B*e_j
    (composition of linear maps), in Python integers, reduced at the end."""
    m, k = len(A), len(A[0]) if A else 0
    n = len(B[0]) if B else (len(C[0]) if C else 0)
    out = [[0] * n for _ in range(m)]
    for j in range(n):
        y = [B[l][j] for l in range(k)]                 # B e_j
        z = [sum(A[i][l] * y[l] for l in range(k)) for i in range(m)]   # A y
        for i in range(m):
            out[i][j] = (alpha * z[i] + beta * C[i][j]) % p
    return out


def _as_np(M):
    return np.array(M, dtype=np.int32).reshape(len(M), len(M[0]) if M else 0)


# ---------------------------------------------------------------- paper / SPEC values

def test_spec_worked_example():
    rows = _golden_rows("spec_fgemm_example.txt")
    (p, alpha, beta), (m, k, n) = rows[0], rows[1]
    A = _as_np(rows[2:2 + m])
    B = _as_np(rows[2 + m:2 + m + k])
    want = _as_np(rows[2 + m + k:2 + 2 * m + k])
    got = oracle.fgemm(p, "N", "N", alpha, A, B, beta)
    assert np.array_equal(got, want)


def test_table1_opcounts_all_25_cells():
    cells = 0
    for row in _golden_rows("table1_opcounts.txt"):
        n, counts = row[0], row[1:]
        for l, c in enumerate(counts):
            assert winograd.opcount(n, l) == c, (n, l)
            cells += 1
    assert cells == 25


def _rand_mat(rng, r, c, lo, hi):
    return [[rng.randrange(lo, hi) for _ in range(c)] for _ in range(r)]


def test_table2_schedule_with_A22_is_alpha_AB_plus_beta_C():
    rng = random.Random(7)
    for _ in range(20):
        m, k, n = (2 * rng.randint(1, 4) for _ in range(3))
        A, B, C = _rand_mat(rng, m, k, -9, 10), _rand_mat(rng, k, n, -9, 10), _rand_mat(rng, m, n, -9, 10)
        alpha, beta = rng.randint(-5, 5), rng.randint(-5, 5)
        want = _linear_map_product(10 ** 30, alpha, A, B, beta, C)   # modulus > any value
        want = [[v if v < 10 ** 29 else v - 10 ** 30 for v in r] for r in want]
        assert winograd.schedule_table2(alpha, A, B, beta, C, "A22") == want


def test_table2_step16_as_printed_is_wrong():
    # DESIGN.md reading R9: PAPER.md l.268 prints A12 in step 16; App. A.2
    # (l.935) has P4 = A22 x (...).  The printed operand gives a wrong product.
    rng = random.Random(8)
    A, B, C = _rand_mat(rng, 4, 4, -9, 10), _rand_mat(rng, 4, 4, -9, 10), _rand_mat(rng, 4, 4, -9, 10)
    want = winograd.schedule_table2(3, A, B, 2, C, "A22")
    assert winograd.schedule_table2(3, A, B, 2, C, "A12") != want


def _is_prime_trial(n):
    if n < 2:
        return False
    d = 2
    while d * d <= n:
        if n % d == 0:
            return False
        d += 1
    return True


def _miller_rabin(n):
    if n < 2:
        return False
    bases = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37]
    for b in bases:
        if n % b == 0:
            return n == b
    d, s = n - 1, 0
    while d % 2 == 0:
        d, s = d // 2, s + 1
    for a in bases:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def test_config_primes_are_largest_below_powers_of_two():
    for bits, q in _golden_rows("paper_primes.txt"):
        assert _is_prime_trial(q) and _miller_rabin(q)
        assert all(not _miller_rabin(x) for x in range(q + 1, 2 ** bits))


# ---------------------------------------------------------------- brute force

def test_exhaustive_gf2_2x2():
    p = 2
    mats = [np.array(v, dtype=np.int32).reshape(2, 2) for v in itertools.product(range(p), repeat=4)]
    for A in mats:
        for B in mats:
            for C in mats[::3]:
                for alpha, beta in itertools.product(range(p), repeat=2):
                    want = _linear_map_product(p, alpha, A.tolist(), B.tolist(), beta, C.tolist())
                    got = oracle.fgemm(p, "N", "N", alpha, A, B, beta, C)
                    assert got.tolist() == want


def test_exhaustive_gf3_2x2_products():
    p = 3
    mats = [np.array(v, dtype=np.int32).reshape(2, 2) for v in itertools.product(range(p), repeat=4)]
    C = np.array([[2, 1], [0, 2]], dtype=np.int32)
    for A in mats:
        for B in mats:
            for alpha, beta in ((1, 0), (2, 1), (1, 2)):
                want = _linear_map_product(p, alpha, A.tolist(), B.tolist(), beta, C.tolist())
                assert oracle.fgemm(p, "N", "N", alpha, A, B, beta, C).tolist() == want


def _stored(rng, rows, cols, p, ld_extra, lo=None):
    """A stored rows x cols int32 matrix inside a wider buffer (ld = cols + ld_extra)."""
    lo = 0 if lo is None else lo
    buf = rng.integers(lo, p, size=(rows, cols + ld_extra), dtype=np.int64).astype(np.int32)
    return buf[:, :cols]


@pytest.mark.parametrize("p", PRIMES)
def test_random_shapes_vs_bigint(p):
    rng = np.random.default_rng(p % 1000)
    for trial in range(25):
        m, k, n = (int(x) for x in rng.integers(1, 40, size=3))
        tA, tB = rng.choice(["N", "T"]), rng.choice(["N", "T"])
        # non-canonical inputs too: negative and >= p (reading R3)
        lo = -p if trial % 3 == 0 else 0
        A = _stored(rng, *( (k, m) if tA == "T" else (m, k) ), p, trial % 3, lo)
        B = _stored(rng, *( (n, k) if tB == "T" else (k, n) ), p, trial % 2, lo)
        C = _stored(rng, m, n, p, 1, lo)
        alpha = int(rng.integers(0, 2 ** 32))   # reduced mod p (reading R4)
        beta = int(rng.integers(0, 2 ** 32)) if trial % 4 else 0
        opA = (A.T if tA == "T" else A).astype(object)
        opB = (B.T if tB == "T" else B).astype(object)
        want = (alpha * (opA.dot(opB)) + beta * C.astype(object)) % p
        got = oracle.fgemm(p, tA, tB, alpha, A, B, beta, C, m=m, n=n, k=k)
        assert np.array_equal(got.astype(object), want), (p, trial)


# ---------------------------------------------------------------- identities / closed forms

@pytest.mark.parametrize("p", CONFIG_PRIMES)
def test_identity_and_alpha_zero(p):
    rng = np.random.default_rng(1)
    A = rng.integers(0, p, size=(9, 9), dtype=np.int64).astype(np.int32)
    C = rng.integers(0, p, size=(9, 9), dtype=np.int64).astype(np.int32)
    I = np.eye(9, dtype=np.int32)
    # B = I  =>  C = alpha*A + beta*C
    got = oracle.fgemm(p, "N", "N", 3, A, I, 5, C)
    assert np.array_equal(got.astype(np.int64), (3 * A.astype(np.int64) + 5 * C.astype(np.int64)) % p)
    # alpha = 0  =>  C = beta*C
    got = oracle.fgemm(p, "N", "N", 0, A, A, 7, C)
    assert np.array_equal(got.astype(np.int64), (7 * C.astype(np.int64)) % p)
    # beta = 0 never reads C: garbage C gives the same answer as zero C
    junk = np.full_like(C, -12345)
    assert np.array_equal(oracle.fgemm(p, "N", "N", 1, A, A, 0, junk),
                          oracle.fgemm(p, "N", "N", 1, A, A, 0, np.zeros_like(C)))


@pytest.mark.parametrize("p", CONFIG_PRIMES)
def test_permutation_matrix_permutes_rows(p):
    rng = np.random.default_rng(2)
    sigma = rng.permutation(13)
    P = np.zeros((13, 13), dtype=np.int32)
    P[np.arange(13), sigma] = 1
    B = rng.integers(0, p, size=(13, 6), dtype=np.int64).astype(np.int32)
    got = oracle.fgemm(p, "N", "N", 1, P, B, 0)
    assert np.array_equal(got, B[sigma])


@pytest.mark.parametrize("p,k,quarter", [(65521, 8192, 2048), (8388593, 4096, 1024),
                                         (251, 16384, 80), (67108859, 16384, 4096)])
def test_closed_forms_max_magnitude(p, k, quarter):
    # (p-1)^2 = 1 mod p  =>  (AB)_ij = k mod p.  These are also the largest
    # terms the positive representation can produce (Eq (1)),
    # so an accumulator overflow would show here.
    A = np.full((3, k), p - 1, dtype=np.int32)
    B = np.full((k, 2), p - 1, dtype=np.int32)
    assert (oracle.fgemm(p, "N", "N", 1, A, B, 0) == k % p).all()
    # alpha = p-1 (i.e. -1, BASELINE config 5)
    assert (oracle.fgemm(p, "N", "N", p - 1, A, B, 0) == (-k) % p).all()
    # ((p+1)/2)^2 = 1/4 mod p: the centred extreme -(p-1)/2 (Eq (2), l.155)
    h = (p + 1) // 2
    A[:] = h
    B[:] = h
    got = oracle.fgemm(p, "N", "N", 1, A, B, 0)
    assert (got == (k * pow(4, -1, p)) % p).all()
    assert (got == quarter).all()      # SURVEY.md §8(c) values, recomputed by hand


def test_transpose_identity_and_ld():
    p = 65521
    rng = np.random.default_rng(3)
    A = _stored(rng, 37, 29, p, 5)      # m x k, lda = 34
    B = _stored(rng, 29, 41, p, 3)      # k x n, ldb = 44
    C1 = oracle.fgemm(p, "N", "N", 1, A, B, 0)
    # (AB)^T = B^T A^T : read B as op(B_stored)=B^T with transA=T, A with transB=T
    C2 = oracle.fgemm(p, "T", "T", 1, B, A, 0)
    assert np.array_equal(C1.T, C2)
    # transposed storage of the same operands gives the same product
    At = np.ascontiguousarray(A.T)
    Bt = np.ascontiguousarray(B.T)
    assert np.array_equal(oracle.fgemm(p, "T", "T", 1, At, Bt, 0), C1)
    assert np.array_equal(oracle.fgemm(p, "T", "N", 1, At, B, 0), C1)
    assert np.array_equal(oracle.fgemm(p, "N", "T", 1, A, Bt, 0), C1)


def test_linearity_in_B_and_residue_invariance():
    p = 8388593
    rng = np.random.default_rng(4)
    A = _stored(rng, 20, 30, p, 0)
    B1 = _stored(rng, 30, 10, p, 0)
    B2 = _stored(rng, 30, 10, p, 0)
    s = ((B1.astype(np.int64) + B2) % p).astype(np.int32)
    lhs = oracle.fgemm(p, "N", "N", 1, A, s, 0).astype(np.int64)
    rhs = (oracle.fgemm(p, "N", "N", 1, A, B1, 0).astype(np.int64)
           + oracle.fgemm(p, "N", "N", 1, A, B2, 0)) % p
    assert np.array_equal(lhs, rhs)
    # adding a multiple of p to inputs changes nothing (reduction on load)
    Ash = (A.astype(np.int64) - p).astype(np.int32)
    assert np.array_equal(oracle.fgemm(p, "N", "N", 1, Ash, B1, 0),
                          oracle.fgemm(p, "N", "N", 1, A, B1, 0))


def test_rows_entry_point_matches_full():
    p = 67108859
    rng = np.random.default_rng(5)
    A, B, C = _stored(rng, 50, 33, p, 0), _stored(rng, 33, 21, p, 0), _stored(rng, 50, 21, p, 0)
    full = oracle.fgemm(p, "N", "N", p - 1, A, B, 1, C)
    rows = [0, 7, 49, 13]
    part = oracle.fgemm_rows(p, "N", "N", p - 1, A, B, 1, C[rows], rows, 50, 21, 33)
    assert np.array_equal(part, full[rows])


def test_matvec_vs_bigint_and_freivalds():
    p = 67108859
    rng = np.random.default_rng(6)
    A, B, C = _stored(rng, 40, 60, p, 0), _stored(rng, 60, 30, p, 0), _stored(rng, 40, 30, p, 0)
    x = rng.integers(0, p, size=30, dtype=np.int64).astype(np.int32)
    assert np.array_equal(oracle.matvec(p, "N", B, x).astype(object),
                          B.astype(object).dot(x.astype(object)) % p)
    assert np.array_equal(oracle.matvec(p, "T", A, A[:, 0].copy()).astype(object),
                          A.T.astype(object).dot(A[:, 0].astype(object)) % p)
    alpha, beta = p - 1, 1
    out = oracle.fgemm(p, "N", "N", alpha, A, B, beta, C)
    lhs = oracle.matvec(p, "N", out, x).astype(object)
    rhs = (alpha * oracle.matvec(p, "N", A, oracle.matvec(p, "N", B, x)).astype(object)
           + beta * oracle.matvec(p, "N", C, x).astype(object)) % p
    assert np.array_equal(lhs, rhs)
    # a single corrupted entry is caught
    out[3, 4] = (out[3, 4] + 1) % p
    lhs = oracle.matvec(p, "N", out, x).astype(object)
    assert not np.array_equal(lhs, rhs)


def test_empty_and_degenerate_shapes():
    p = 251
    A = np.zeros((3, 0), dtype=np.int32)
    B = np.zeros((0, 4), dtype=np.int32)
    C = np.full((3, 4), 100, dtype=np.int32)
    # k = 0: C = beta*C mod p (SPEC.md l.327 reading R5)
    assert (oracle.fgemm(p, "N", "N", 1, A, B, 2, C, m=3, n=4, k=0) == 200).all()
    assert oracle.fgemm(p, "N", "N", 1, np.zeros((0, 5), np.int32), np.zeros((5, 4), np.int32),
                        0, m=0, n=4, k=5).shape == (0, 4)


# ---------------------------------------------------------------- input generator

def test_generator_matches_splitmix64_reference_stream():
    # splitmix64 with state 0: the first outputs are the published reference
    # values of Vigna's splitmix64.c (state += GAMMA; return mix64(state)).
    want = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    got = [ffgen.mix64_int((i + 1) * ffgen.GAMMA) for i in range(3)]
    assert got == want


def test_generator_vector_matches_scalar_and_blocks():
    p = 67108859
    key = ffgen.seed_key(5, ffgen.STREAM_A)
    v = ffgen.uniform_flat(p, 5, ffgen.STREAM_A, 0, 1000)
    ref = [(ffgen.mix64_int(key + (i + 1) * ffgen.GAMMA) >> 11) % p for i in range(1000)]
    assert v.tolist() == ref
    M = ffgen.uniform_matrix(p, 5, ffgen.STREAM_A, 40, 25)
    assert np.array_equal(M.ravel(), v[:1000])
    assert np.array_equal(ffgen.uniform_matrix(p, 5, ffgen.STREAM_A, 40, 25, row0=7, nrows=3), M[7:10])
    assert v.min() >= 0 and v.max() < p


def test_generator_c_twin_matches_numpy():
    # ffgen/gen.c (OpenMP, used for large host inputs) against the numpy recipe,
    # including an index window past 2^32 and every config prime
    for p in [2, 251, 65521, 8388593, 67108859, 2 ** 31 - 1]:
        for start in (0, 12345, (1 << 32) - 1000):
            a = ffgen.uniform_flat(p, 3, ffgen.STREAM_B, start, 1 << 17)
            b = ffgen.uniform_flat_numpy(p, 3, ffgen.STREAM_B, start, 1 << 17)
            assert np.array_equal(a, b)
    assert ffgen._c_gen() is not None
