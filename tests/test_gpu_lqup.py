"""GPU LQUP / rank / determinant (Sec. 5.1 and 6)
against the oracle.  The factorization is not unique, so the tests check
what is unique (rank, determinant) against oracle.rank_det and that the rest
is valid: Q, P permutations, L unit lower, U upper with a non-zero diagonal,
zero rows beyond the rank, and A[Q][:, P] = L U (mod p) exactly."""
import numpy as np
import pytest

import ffgen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_cs_0601133_b200 as ff
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return torch, ff


def _factor(torch, ff, p, A):
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    Q, P, r = ff.lqup(p, dA)
    torch.cuda.synchronize()
    return dA.cpu().numpy(), Q, P, r


def _check_valid(p, A, F, Q, P, r, full_product=True):
    m, n = A.shape
    assert sorted(Q.tolist()) == list(range(m)) and sorted(P.tolist()) == list(range(n))
    assert 0 <= r <= min(m, n)
    assert F.min() >= 0 and F.max() < p
    L = np.zeros((m, r), np.int64)
    for k in range(r):
        L[k + 1:, k] = F[k + 1:, k]
        L[k, k] = 1
    U = np.triu(F[:r, :].astype(np.int64))
    assert (np.diagonal(U[:, :r]) != 0).all()                 # U_kk != 0 for k < r
    assert (F[r:, r:] == 0).all()                             # zero rows beyond the rank
    Ap = np.ascontiguousarray(np.mod(A.astype(np.int64), p)[Q][:, P].astype(np.int32))
    if full_product:
        LU = oracle.fgemm(p, "N", "N", 1, L.astype(np.int32), U.astype(np.int32), 0, m=m, n=n, k=r) if r \
            else np.zeros((m, n), np.int32)
        np.testing.assert_array_equal(LU, Ap)
    else:                                                     # Freivalds: A' x = L (U x)
        for t in range(3):
            x = ffgen.uniform_vector(p, 77, 30 + t, n)
            lhs = oracle.matvec(p, "N", Ap, x)
            ux = oracle.matvec(p, "N", U.astype(np.int32), x) if r else np.zeros(0, np.int32)
            rhs = oracle.matvec(p, "N", L.astype(np.int32), ux) if r else np.zeros(m, np.int32)
            np.testing.assert_array_equal(lhs, rhs)


def _low_rank(rng, p, m, n, r):
    X = rng.integers(0, p, size=(m, r)).astype(np.int32)
    Y = rng.integers(0, p, size=(r, n)).astype(np.int32)
    return oracle.fgemm(p, "N", "N", 1, X, Y, 0, m=m, n=n, k=r) if r else np.zeros((m, n), np.int32)


@pytest.mark.parametrize("p", [3, 65521, 8388593, 67108859])
@pytest.mark.parametrize("m,n,r", [(300, 300, None), (200, 530, None), (530, 200, None), (400, 400, 0),
                                   (400, 400, 1), (400, 380, 5), (520, 600, 130), (257, 1000, 256)])
def test_lqup_vs_oracle_rank(env, p, m, n, r):
    torch, ff = env
    rng = np.random.default_rng(m * 3 + n + (r or 0) + p % 101)
    A = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32) if r is None \
        else _low_rank(rng, p, m, n, r)
    F, Q, P, rk = _factor(torch, ff, p, A)
    want_r, want_d = oracle.rank_det(p, A)
    assert rk == want_r
    _check_valid(p, A, F, Q, P, rk)
    dA = torch.from_numpy(A).cuda()
    got_r, got_d = ff.rank_det(p, dA)
    assert got_r == want_r and got_d == want_d
    assert torch.equal(dA.cpu(), torch.from_numpy(A))        # rank_det leaves A untouched


def test_lqup_structured_rank_deficiency(env):
    """Zero rows, repeated rows, zero leading columns, a rank-deficient first
    panel and a window that must be widened (pivots beyond 256 columns)."""
    torch, ff = env
    p = 65521
    rng = np.random.default_rng(5)
    m, n = 300, 900
    A = rng.integers(0, p, size=(m, n)).astype(np.int32)
    A[0] = 0
    A[3] = A[1]
    A[10] = (2 * A[2].astype(np.int64) % p).astype(np.int32)
    A[:, :40] = 0
    A[20:60, :] = 0
    A[70, :700] = 0                                           # first non-zero beyond the initial window
    A[130:260, :] = A[0:130, :]                               # the second panel repeats the first
    F, Q, P, rk = _factor(torch, ff, p, A)
    assert rk == oracle.rank_det(p, A)[0]
    _check_valid(p, A, F, Q, P, rk)


@pytest.mark.parametrize("p", [65521, 67108859])
def test_det_small_and_signs(env, p):
    torch, ff = env
    rng = np.random.default_rng(p % 31)
    for n in [1, 2, 3, 7, 129, 260]:
        A = rng.integers(0, p, size=(n, n)).astype(np.int32)
        assert ff.rank_det(p, torch.from_numpy(A).cuda()) == oracle.rank_det(p, A)
        S = A.copy()
        S[:, [0, n - 1]] = S[:, [n - 1, 0]]
        if n > 1:
            assert ff.rank_det(p, torch.from_numpy(S).cuda())[1] == (p - oracle.rank_det(p, A)[1]) % p


def test_lqup_large_freivalds(env):
    torch, ff = env
    p = 65521
    N = 2048
    A = ffgen.uniform_matrix(p, 21, ffgen.STREAM_A, N, N)
    F, Q, P, rk = _factor(torch, ff, p, A)
    assert rk == oracle.rank_det(p, A)[0]
    _check_valid(p, A, F, Q, P, rk, full_product=False)


@pytest.mark.parametrize("p", [65521, 8388593, 2147483647])
def test_lqup_speculative_panel_matches_pivoting_panel(env, p, monkeypatch):
    """Full 128 x 128 windows go to the speculative blocked panel (no pivot
    search).  Without swaps the LU is unique, so the result must
    be bit-identical to the pivoting panels' (FF_LQUP_NOSPEC), including the
    trailing GEMMs that consume its L11^-1 / U11^-1; p = 2^31 - 1 exercises
    the shortest delayed-reduction cadence (4 products)."""
    torch, ff = env
    m, n = 640, 520
    A = ffgen.uniform_matrix(p, 33, ffgen.STREAM_A, m, n)
    F1, Q1, P1, r1 = _factor(torch, ff, p, A)
    monkeypatch.setenv("FF_LQUP_NOSPEC", "1")
    F2, Q2, P2, r2 = _factor(torch, ff, p, A)
    assert r1 == r2 == min(m, n)
    np.testing.assert_array_equal(Q1, Q2)
    np.testing.assert_array_equal(P1, P2)
    np.testing.assert_array_equal(F1, F2)
    _check_valid(p, A, F1, Q1, P1, r1)


@pytest.mark.parametrize("row", [1, 31, 32, 70, 127, 128 + 64])
def test_lqup_speculation_fails_mid_panel(env, row):
    """A zero pivot at `row` (its leading minor vanishes but the row does not):
    the speculative panel must report failure without touching A, and the
    pivoting panel takes over (a column swap)."""
    torch, ff = env
    p = 65521
    rng = np.random.default_rng(row)
    m, n = 384, 384
    A = rng.integers(0, p, size=(m, n)).astype(np.int32)
    A[row, :row + 1] = A[row - 1, :row + 1]                   # row - 1 and row agree up to the diagonal
    F, Q, P, rk = _factor(torch, ff, p, A)
    assert rk == oracle.rank_det(p, A)[0] == n
    assert (P != np.arange(n)).any()                          # a column swap happened
    _check_valid(p, A, F, Q, P, rk)


@pytest.mark.parametrize("dep_row", [None, 700, 1000])
def test_lqup_deferred_updates_match_immediate(env, dep_row, monkeypatch):
    """Groups of generic panels defer their trailing updates into one GEMM with
    K = 128 x (panels).  The arithmetic is exact, so the result
    must be bit-identical to immediate updates (FF_LQUP_GROUP=1); a dependent
    row inside a later panel (rank deficiency: zero row) forces a flush in the
    middle of a group."""
    torch, ff = env
    p = 65521
    m, n = 1100, 1060
    A = ffgen.uniform_matrix(p, 41, ffgen.STREAM_A, m, n)
    if dep_row is not None:
        A[dep_row] = ((A[100].astype(np.int64) + 3 * A[200]) % p).astype(np.int32)
    F1, Q1, P1, r1 = _factor(torch, ff, p, A)
    monkeypatch.setenv("FF_LQUP_GROUP", "1")
    F2, Q2, P2, r2 = _factor(torch, ff, p, A)
    assert r1 == r2 == oracle.rank_det(p, A)[0]
    np.testing.assert_array_equal(Q1, Q2)
    np.testing.assert_array_equal(P1, P2)
    np.testing.assert_array_equal(F1, F2)
    _check_valid(p, A, F1, Q1, P1, r1)


@pytest.mark.parametrize("seed", range(12))
def test_lqup_random_sweep(env, seed):
    """Seeded random shapes, ranks and primes (incl. tiny fields where the
    speculative panel fails and the pivoting panels take over): rank and
    determinant against the oracle, the factorization valid."""
    torch, ff = env
    rng = np.random.default_rng(777 + seed)
    primes = [2, 3, 7, 29, 251, 4099, 65521, 8388593, 2 ** 31 - 1]
    for _ in range(3):
        p = int(rng.choice(primes))
        m, n = (int(x) for x in rng.integers(1, 900, size=2))
        if rng.random() < 0.5:
            r = int(rng.integers(0, min(m, n) + 1))
            A = _low_rank(rng, p, m, n, r)
        else:
            A = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
        if rng.random() < 0.5:                       # structure: zero / repeated rows, zero columns
            i, j, c0 = int(rng.integers(0, m)), int(rng.integers(0, m)), int(rng.integers(0, n))
            A[i] = A[j]
            A[:, c0:c0 + int(rng.integers(1, 150))] = 0
            A[j] = 0
        F, Q, P, rk = _factor(torch, ff, p, A)
        want_r, want_d = oracle.rank_det(p, A)
        assert rk == want_r, (p, m, n)
        _check_valid(p, A, F, Q, P, rk)
        if m == n:
            assert ff.rank_det(p, torch.from_numpy(A).cuda())[1] == want_d


@pytest.mark.parametrize("p,m,n,seed", [(3, 700, 700, 6), (2, 844, 341, 1), (29, 423, 836, 3), (5, 1000, 1000, 7)])
def test_lqup_small_fields_widened_windows_with_pending_updates(env, p, m, n, seed):
    """Regression: in small fields a panel often needs a widened window; its
    column swaps then reach beyond the 128-column window into the region whose
    deferred updates are still pending, so the pending group must be flushed
    before those swaps (a found-by-fuzzing bug: rank 699 instead of 700 for
    p = 3, 700 x 700)."""
    torch, ff = env
    rng = np.random.default_rng(seed)
    A = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
    F, Q, P, rk = _factor(torch, ff, p, A)
    want_r, want_d = oracle.rank_det(p, A)
    assert rk == want_r
    _check_valid(p, A, F, Q, P, rk)
    if m == n:
        assert ff.rank_det(p, torch.from_numpy(A).cuda())[1] == want_d
