"""Pins for the trsm oracle (oracle.trsm, Sec. 4) and for the
paper's delayed-reduction thresholds (oracle/bounds.py): checked against
brute force, the defining residual, the triangle/diagonal conventions and
the values the paper prints -- never against the oracle's own formula."""
import itertools
import os
import random

import numpy as np
import pytest

import oracle
from oracle import bounds

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
COMBOS = list(itertools.product("LR", "UL", "NT", "NU"))


def _rand_tri(rng, p, d, uplo, diag, garbage=True):
    """Random d x d matrix whose referenced triangle is uplo (+ invertible
    diagonal unless diag = 'U'); the unreferenced part holds garbage."""
    A = rng.integers(-2 ** 31, 2 ** 31, size=(d, d), dtype=np.int64) if garbage else np.zeros((d, d), np.int64)
    for i in range(d):
        for j in range(d):
            inside = (j > i) if uplo == "U" else (j < i)
            if inside:
                A[i, j] = rng.integers(0, p)
        if diag == "N":
            A[i, i] = rng.integers(1, p)
            while np.gcd(int(A[i, i]), p) != 1:
                A[i, i] = rng.integers(1, p)
    return A.astype(np.int32)


def _op_dense(A, p, uplo, trans, diag):
    """op(A) as Python ints, with the unreferenced triangle zeroed and a unit
    diagonal made explicit."""
    d = A.shape[0]
    T = [[0] * d for _ in range(d)]
    for i in range(d):
        for j in range(d):
            inside = (j > i) if uplo == "U" else (j < i)
            if inside:
                T[i][j] = int(A[i, j]) % p
        T[i][i] = 1 if diag == "U" else int(A[i, i]) % p
    if trans == "T":
        T = [list(r) for r in zip(*T)]
    return T


def _residual_ok(p, side, uplo, trans, diag, alpha, A, B, X):
    T = _op_dense(A, p, uplo, trans, diag)
    Xi = [[int(v) for v in r] for r in X]
    Bi = [[int(v) for v in r] for r in B]
    m, n = len(Bi), len(Bi[0]) if Bi else 0
    for i in range(m):
        for j in range(n):
            if side == "L":
                s = sum(T[i][l] * Xi[l][j] for l in range(m))
            else:
                s = sum(Xi[i][l] * T[l][j] for l in range(n))
            if (s - alpha * Bi[i][j]) % p:
                return False
    return True


@pytest.mark.parametrize("p", [2, 3, 5])
def test_trsm_brute_force_tiny(p):
    """Every combination of side/uplo/trans/diag on 2 x 2 systems: the unique X
    with op(A) X = alpha B (or X op(A) = alpha B), found by exhaustive search."""
    rng = np.random.default_rng(p)
    for side, uplo, trans, diag in COMBOS:
        for trial in range(4):
            m, n = (2, 2) if trial % 2 == 0 else ((2, 1) if side == "L" else (1, 2))
            d = m if side == "L" else n
            A = _rand_tri(rng, p, d, uplo, diag)
            B = rng.integers(0, p, size=(m, n)).astype(np.int32)
            alpha = int(rng.integers(0, p))
            X = oracle.trsm(p, side, uplo, trans, diag, alpha, A, B)
            sols = []
            for cand in itertools.product(range(p), repeat=m * n):
                Xc = np.array(cand, dtype=np.int64).reshape(m, n)
                if _residual_ok(p, side, uplo, trans, diag, alpha, A, B, Xc):
                    sols.append(Xc)
            assert len(sols) == 1, (side, uplo, trans, diag)
            np.testing.assert_array_equal(X, sols[0])


@pytest.mark.parametrize("p", [3, 251, 65521, 8388593, 67108859, 2 ** 31 - 1])
def test_trsm_residual_and_conventions(p):
    rng = np.random.default_rng(p % 1000)
    for side, uplo, trans, diag in COMBOS:
        m, n = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        d = m if side == "L" else n
        A = _rand_tri(rng, p, d, uplo, diag)
        B = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
        alpha = int(rng.integers(0, p))
        X = oracle.trsm(p, side, uplo, trans, diag, alpha, A, B)
        assert X.min() >= 0 and X.max() < p
        assert _residual_ok(p, side, uplo, trans, diag, alpha, A, B, X), (side, uplo, trans, diag)
        # the unreferenced triangle (and a unit diagonal) is never read
        A2 = A.copy()
        for i in range(d):
            for j in range(d):
                inside = (j > i) if uplo == "U" else (j < i)
                if not inside and (i != j or diag == "U"):
                    A2[i, j] = rng.integers(-2 ** 31, 2 ** 31)
        np.testing.assert_array_equal(oracle.trsm(p, side, uplo, trans, diag, alpha, A2, B), X)


def test_trsm_identity_singular_and_empty():
    p = 65521
    rng = np.random.default_rng(1)
    B = rng.integers(0, p, size=(5, 7)).astype(np.int32)
    I5 = np.eye(5, dtype=np.int32)
    np.testing.assert_array_equal(oracle.trsm(p, "L", "U", "N", "N", 3, I5, B), (3 * B.astype(np.int64)) % p)
    I7 = np.eye(7, dtype=np.int32)
    np.testing.assert_array_equal(oracle.trsm(p, "R", "L", "T", "N", 2, I7, B), (2 * B.astype(np.int64)) % p)
    S = np.triu(rng.integers(1, p, size=(5, 5))).astype(np.int32)
    S[2, 2] = p                                     # = 0 mod p
    with pytest.raises(ZeroDivisionError):
        oracle.trsm(p, "L", "U", "N", "N", 1, S, B)
    np.testing.assert_array_equal(oracle.trsm(p, "L", "U", "N", "U", 1, S, B),
                                  oracle.trsm(p, "L", "U", "N", "U", 1, S + np.eye(5, dtype=np.int32), B))
    assert oracle.trsm(p, "L", "U", "N", "N", 1, np.zeros((0, 0), np.int32), np.zeros((0, 4), np.int32)).shape == (0, 4)


def _golden(name):
    rows = []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line.split())
    return rows


def test_paper_thresholds_table_l522():
    rows = [r for r in _golden("trsm_thresholds.txt") if len(r) == 4]
    assert len(rows) == 3
    for p, lg, td, tu in rows:
        p = int(p)
        # the printed "ceil(log2 p)" column reads 3, 20, 23: p = 2^20 + 7 and
        # 2^23 + 9 are just above powers of two, so it is the field's nominal
        # size, not ceil(log2 p) (= 21, 24): a label, not used by the formulas
        assert int(lg) in (p.bit_length() - 1, p.bit_length())
        assert bounds.t_del(p, 53) == int(td)
        assert bounds.t_update(p, 53) == int(tu)


def test_paper_thresholds_text_l482():
    rows = [r for r in _golden("trsm_thresholds.txt") if len(r) == 3]
    for p, pos, bal in rows:
        assert bounds.t_del(int(p), 53) == int(pos)
        if bal != "-":
            assert bounds.t_del(int(p), 53, balanced=True) == int(bal)
    # "n <= 6" for balanced p = 1001 is reproduced by neither Eq. (5) (n) nor
    # Cor. 4.5 (n - 1): 4 and 5 (reading recorded in DESIGN.md)
    assert bounds.t_del(1001, 53, balanced=True) == 4


def test_trsm_bound_theorem_4_2_holds_and_is_attained_balanced():
    rng = random.Random(7)
    for M, m in [(7, -7), (5, -5), (7, 0), (10, 0), (7, -3), (4, -1)]:
        for trial in range(200):
            n = rng.randint(1, 8)
            T = [[0] * n for _ in range(n)]
            for i in range(n):
                T[i][i] = 1
                for j in range(i + 1, n):
                    T[i][j] = rng.randint(m, M)
            b = [rng.randint(m, M) for _ in range(n)]
            x = bounds.solve_unit_upper_over_Z(T, b)
            for k in range(n):
                u, v = bounds.trsm_u_v(M, m, k)
                lo, hi = (-u, v) if k % 2 == 0 else (-v, u)
                assert lo <= x[n - 1 - k] <= hi, (M, m, k)
        if m == -M:     # Cor. 4.3's system attains v_k exactly (balanced representation)
            T, b = bounds.trsm_worst_case(M, m, 9)
            x = bounds.solve_unit_upper_over_Z(T, b)
            assert [abs(x[9 - 1 - k]) for k in range(9)] == [bounds.trsm_u_v(M, m, k)[1] for k in range(9)]
            # Cor. 4.5: |x| <= (p-1)/2 ((p+1)/2)^(n-1) with M = (p-1)/2
            assert max(abs(v) for v in x) == M * (M + 1) ** 8


def test_theorem_4_2_display_as_printed_is_wrong():
    """The display at l.412-416 swaps (M+m) and (M-m): with M = 7, m = -3 the
    system x_n = 7, x_(n-1) = -3 - 7*7 = -52 already exceeds its v_1 = 46."""
    M, m = 7, -3
    printed_v1 = (M + m) // 2 * (M + 1) + (M - m) // 2 * (M - 1)
    assert printed_v1 == 46
    x = bounds.solve_unit_upper_over_Z([[1, M], [0, 1]], [m, M])
    assert x == [-52, 7] and abs(x[0]) > printed_v1
    assert bounds.trsm_u_v(M, m, 1)[1] == 52


def test_dot_product_and_winograd_bounds():
    # Eq. (1): lambda (p-1)^2 < 2^53 is the largest such lambda
    for p in [3, 65521, 1048583, 8388617, 67108859]:
        lam = bounds.lambda_dot(p, 53)
        assert lam * (p - 1) ** 2 < 2 ** 53 <= (lam + 1) * (p - 1) ** 2
        lb = bounds.lambda_dot(p, 53, balanced=True)
        h = (p - 1) // 2
        assert lb * h * h < 2 ** 52 <= (lb + 1) * h * h
    # Cor. 3.4 at l = 0 is Eq. (1) + 1 (k < k_W): the classical dot-product bound
    for p in [65521, 1048583, 8388617]:            # (2^53 / (p-1)^2 not an integer)
        assert bounds.k_winograd(p, 53, 0) == bounds.lambda_dot(p, 53) + 1
    # Theorem 3.1 / Cor 3.2 at l = 1 with the positive representation: the bound
    # ((1+3)/2)^2 floor(k/2) (p-1)^2 fits gamma bits just below k_W (here the
    # printed formula's quotient is such that it equals the exact threshold)
    p, g = 65521, 53
    kw = bounds.k_winograd(p, g, 1)
    assert 4 * ((kw - 1) // 2) * (p - 1) ** 2 < 2 ** g
    assert 4 * (kw // 2) * (p - 1) ** 2 >= 2 ** g


# ---------------------------------------------------------------- rank / det oracle (Sec. 6)

def _span_size(rows, p):
    """|row space| by enumerating every linear combination (tiny cases only)."""
    n = len(rows[0]) if rows else 0
    seen = set()
    for coeffs in itertools.product(range(p), repeat=len(rows)):
        v = tuple(sum(c * r[j] for c, r in zip(coeffs, rows)) % p for j in range(n))
        seen.add(v)
    return len(seen)


def _leibniz_det(M, p):
    n = len(M)
    tot = 0
    for perm in itertools.permutations(range(n)):
        inv = sum(1 for i in range(n) for j in range(i + 1, n) if perm[i] > perm[j])
        term = 1
        for i in range(n):
            term *= M[i][perm[i]]
        tot += -term if inv % 2 else term
    return tot % p


@pytest.mark.parametrize("p", [2, 3, 5])
def test_rank_det_brute_force(p):
    """rank = log_p |row space| (enumerated); det = Leibniz's permutation sum."""
    rng = np.random.default_rng(p)
    for trial in range(60):
        m, n = int(rng.integers(1, 4)), int(rng.integers(1, 5))
        X = rng.integers(0, p, size=(m, n))
        if trial % 3 == 0 and m > 1:
            X[-1] = (X[0] * int(rng.integers(0, p))) % p       # a dependent row
        r, d = oracle.rank_det(p, X.astype(np.int32))
        assert p ** r == _span_size(X.tolist(), p)
        if m == n:
            assert d == _leibniz_det(X.tolist(), p)
        else:
            assert d is None


@pytest.mark.parametrize("p", [65521, 8388593, 2 ** 31 - 1])
def test_rank_det_structured(p):
    rng = np.random.default_rng(p % 997)
    n = 40
    assert oracle.rank_det(p, np.eye(n, dtype=np.int32)) == (n, 1)
    assert oracle.rank_det(p, np.zeros((n, n + 3), np.int32))[0] == 0
    # det of a product is the product of dets; det of a triangular matrix is its diagonal product
    U = np.triu(rng.integers(0, p, size=(n, n))).astype(np.int64)
    U[np.arange(n), np.arange(n)] = rng.integers(1, p, size=n)
    dU = 1
    for i in range(n):
        dU = dU * int(U[i, i]) % p
    assert oracle.rank_det(p, U.astype(np.int32))[1] == dU
    # a row swap flips the sign; rank of an outer product u v^T (u, v != 0) is 1
    S = U.copy()
    S[[0, 5]] = S[[5, 0]]
    assert oracle.rank_det(p, S.astype(np.int32))[1] == (p - dU) % p
    u = rng.integers(1, p, size=(n, 1))
    v = rng.integers(1, p, size=(1, n + 7))
    assert oracle.rank_det(p, ((u * v) % p).astype(np.int32))[0] == 1
    # non-canonical input is reduced
    assert oracle.rank_det(p, (U.astype(np.int64) - p).astype(np.int32))[1] == dU
