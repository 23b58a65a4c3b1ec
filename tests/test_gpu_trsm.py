"""GPU parity of ftrsm (Sec. 4, Algorithm 1 on the tensor-core
fgemm) against the substitution oracle, bit-exact."""
import itertools

import numpy as np
import pytest

import ffgen
import oracle

pytestmark = pytest.mark.gpu

COMBOS = list(itertools.product("LR", "UL", "NT", "NU"))


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_cs_0601133_b200 as ff
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return torch, ff


def _tri(rng, p, d, uplo, diag, garbage=True, ld_extra=0):
    """d x d (+ld_extra columns) with the referenced triangle uniform in [0,p),
    an invertible diagonal (diag N), and garbage everywhere else."""
    A = rng.integers(-2 ** 31, 2 ** 31, size=(d, d + ld_extra), dtype=np.int64) if garbage \
        else np.zeros((d, d + ld_extra), np.int64)
    iu = np.triu_indices(d, 1) if uplo == "U" else np.tril_indices(d, -1)
    A[iu] = rng.integers(0, p, size=len(iu[0]))
    if diag == "N":
        dg = rng.integers(1, p, size=d)
        if p > 2:
            while True:
                bad = np.gcd(dg, p) != 1
                if not bad.any():
                    break
                dg[bad] = rng.integers(1, p, size=int(bad.sum()))
        A[np.arange(d), np.arange(d)] = dg
    return A.astype(np.int32)


def _run(torch, ff, p, side, uplo, trans, diag, alpha, A, B, opts=None):
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    m, n = B.shape[0], B.shape[1]
    ff.ftrsm(p, dA, dB, side, uplo, trans, diag, alpha, opts)
    torch.cuda.synchronize()
    return dB.cpu().numpy()


@pytest.mark.parametrize("p", [65521, 67108859, 251, 3])
@pytest.mark.parametrize("side,uplo,trans,diag", COMBOS)
def test_trsm_all_combinations_vs_oracle(env, p, side, uplo, trans, diag):
    torch, ff = env
    rng = np.random.default_rng(p % 997 + 31 * COMBOS.index((side, uplo, trans, diag)))
    m, n = (1100, 200) if side == "L" else (150, 1100)   # 3 leaves (512, 512, 76), ragged
    d = m if side == "L" else n
    A = _tri(rng, p, d, uplo, diag, ld_extra=3)
    B = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
    alpha = int(rng.integers(0, p)) if p > 3 else 2
    got = _run(torch, ff, p, side, uplo, trans, diag, alpha, A, B)
    want = oracle.trsm(p, side, uplo, trans, diag, alpha, A[:, :d], B)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("p,side,uplo,trans,diag,m,n", [
    (65521, "L", "U", "N", "N", 1000, 700),
    (8388593, "L", "L", "T", "N", 777, 513),
    (67108859, "R", "U", "N", "U", 600, 1029),
    (65521, "R", "L", "T", "N", 257, 1100),
    (65521, "L", "U", "N", "N", 1, 1),
    (65521, "L", "L", "N", "N", 128, 5),
    (65521, "L", "U", "N", "N", 300, 77),                # one ragged leaf
    (67108859, "L", "L", "N", "N", 2100, 300),           # 5 leaves, CRT GEMMs
    (2 ** 31 - 1, "L", "U", "T", "N", 500, 260),
])
def test_trsm_medium_vs_oracle(env, p, side, uplo, trans, diag, m, n):
    torch, ff = env
    rng = np.random.default_rng(m * 7 + n)
    d = m if side == "L" else n
    A = _tri(rng, p, d, uplo, diag)
    # alpha = 1 skips the scaling pass: B may be any int32 (reduced where it is read)
    B = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
    got = _run(torch, ff, p, side, uplo, trans, diag, 1, A, B)
    np.testing.assert_array_equal(got, oracle.trsm(p, side, uplo, trans, diag, 1, A, B))


def test_trsm_alpha_zero_identity_and_ld(env):
    torch, ff = env
    p = 65521
    rng = np.random.default_rng(2)
    m, n = 300, 170
    Bbuf = rng.integers(0, p, size=(m, n + 9)).astype(np.int32)
    I = np.eye(m, dtype=np.int32)
    dB = torch.from_numpy(Bbuf).cuda()
    ff.ftrsm(p, torch.from_numpy(I).cuda(), dB[:, :n], "L", "U", "N", "N", 5)
    torch.cuda.synchronize()
    out = dB.cpu().numpy()
    np.testing.assert_array_equal(out[:, :n], (5 * Bbuf[:, :n].astype(np.int64)) % p)
    np.testing.assert_array_equal(out[:, n:], Bbuf[:, n:])            # ld padding untouched
    A = _tri(rng, p, m, "U", "N")
    dB = torch.from_numpy(Bbuf).cuda()
    ff.ftrsm(p, torch.from_numpy(A).cuda(), dB[:, :n], "L", "U", "N", "N", 0)
    torch.cuda.synchronize()
    assert (dB[:, :n] == 0).all().item()
    with pytest.raises(ff.FFError):
        ff.ff_trsm(p, "X", "U", "N", "N", 2, 2, 1, dB, 2, dB, 2)


@pytest.mark.parametrize("side", ["L", "R"])
def test_trsm_large_residual_freivalds(env, side):
    """m = n = 8192 over Z/65521Z: op(A) X = B checked on the whole output by
    Freivalds' test (A (X r) = B r for random r), A holding zeros off its triangle."""
    torch, ff = env
    p, N = 65521, 8192
    rng = np.random.default_rng(9)
    A = _tri(rng, p, N, "U", "N", garbage=False)
    B = ffgen.uniform_matrix(p, 13, ffgen.STREAM_B, N, N)
    got = _run(torch, ff, p, side, "U", "N", "N", 1, A, B)
    assert got.min() >= 0 and got.max() < p
    for t in range(3):
        r = ffgen.uniform_vector(p, 13, 20 + t, N)
        if side == "L":
            lhs = oracle.matvec(p, "N", A, oracle.matvec(p, "N", got, r))
            rhs = oracle.matvec(p, "N", B, r)
        else:                           # X A = B  =>  r^T X A = r^T B  ->  A^T (X^T r) = B^T r
            lhs = oracle.matvec(p, "T", A, oracle.matvec(p, "T", got, r))
            rhs = oracle.matvec(p, "T", B, r)
        np.testing.assert_array_equal(lhs, rhs)
