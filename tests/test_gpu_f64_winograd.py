"""Delayed multi-level Winograd on the fp64 engine (SURVEY §8(f) NEXT-3,
PAPER.md Sec. 3.2.3): l = 1..3 recursive levels whose pre-additions are NOT
reduced, accepted while Corollary 3.4 allows it (k < k_winograd[l], the exact
reading R21), bit-exact against the oracle; rejected at k_winograd; the
Appendix A.6 witnesses run exactly at the bound's scale; and past the bound
(test knob) the same construction gives wrong residues -- the theorem's
bound is what keeps the delayed Winograd exact on this hardware.

The host-side planner pin (k_winograd against oracle/bounds.py) runs without
a GPU (not marked)."""
import numpy as np
import pytest

import oracle
from oracle import bounds, winograd

PRIMES = [2, 3, 251, 65521, 8388593, 67108859]


@pytest.mark.parametrize("p", PRIMES + [5, 1048583, 16777259])
def test_planner_k_winograd_is_corollary_34(p):
    """ff_plan_query's k_winograd[l] (host only) equals the oracle's exact
    Corollary 3.4 threshold for the balanced representation, gamma = 53."""
    import paper_cs_0601133_b200 as ff
    info = ff.ff_plan_query(p, 1000, {"scheme": 4})
    for l in (1, 2, 3):
        assert info["k_winograd"][l] == bounds.k_winograd_exact(p, 53, l, balanced=True), (p, l)
    assert info["k_winograd"][0] == info["kb_max"] + 1
    # several levels are an fp64-engine option only
    with pytest.raises(ff.FFError):
        ff.ff_plan_query(p, 1000, {"winograd": 2})


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_cs_0601133_b200 as ff
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return torch, ff


def _run(torch, ff, p, tA, tB, m, n, k, alpha, A, B, beta, C, opts):
    dA, dB, dC = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (A, B, C))
    ff.ff_gemm_ex(p, tA, tB, m, n, k, alpha, dA, A.shape[1], dB, B.shape[1], beta, dC, C.shape[1], opts)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


def _shapes(p, l):
    kw = bounds.k_winograd_exact(p, 53, l, balanced=True)
    ks = [k for k in (1, 2, 3, 7, 8, 27, 33, 113, 640, 1000, 4097) if k < kw]
    ms = [(1, 1), (8, 8), (65, 130), (200, 300), (256, 512)]
    return [(m, n, ks[i % len(ks)]) for i, (m, n) in enumerate(ms)] + [(64, 64, max(ks))]


@pytest.mark.gpu
@pytest.mark.parametrize("p", PRIMES)
@pytest.mark.parametrize("l", [1, 2, 3])
@pytest.mark.parametrize("tA,tB", [("N", "N"), ("T", "T")])
def test_f64_winograd_vs_oracle(env, p, l, tA, tB):
    torch, ff = env
    rng = np.random.default_rng(p % 997 + 31 * l + ord(tA))
    for si, (m, n, k) in enumerate(_shapes(p, l)):
        A = rng.integers(-2 ** 31, 2 ** 31, size=(m, k) if tA == "N" else (k, m), dtype=np.int64).astype(np.int32)
        B = rng.integers(0, p, size=(k, n) if tB == "N" else (n, k)).astype(np.int32)
        C = rng.integers(0, p, size=(m, n)).astype(np.int32)
        alpha = [1, p - 1, int(rng.integers(0, p))][si % 3]
        beta = [0, 1, int(rng.integers(0, p))][(si + 1) % 3]
        got = _run(torch, ff, p, tA, tB, m, n, k, alpha, A, B, beta, C, {"scheme": 4, "winograd": l})
        np.testing.assert_array_equal(got, oracle.fgemm(p, tA, tB, alpha, A, B, beta, C),
                                      err_msg="p=%d l=%d %dx%dx%d" % (p, l, m, n, k))


@pytest.mark.gpu
@pytest.mark.parametrize("p", [65521, 8388593, 67108859])
@pytest.mark.parametrize("l", [1, 2, 3])
def test_f64_winograd_rejected_at_k_winograd(env, p, l):
    torch, ff = env
    kw = bounds.k_winograd_exact(p, 53, l, balanced=True)
    if kw > 20000:
        pytest.skip("k_winograd too large to allocate here")
    m = n = 16
    A = np.ones((m, kw), np.int32)
    B = np.ones((kw, n), np.int32)
    C = np.zeros((m, n), np.int32)
    with pytest.raises(ff.FFError) as ei:
        _run(torch, ff, p, "N", "N", m, n, kw, 1, A, B, 0, C, {"scheme": 4, "winograd": l})
    assert ei.value.code == 4            # FF_ERR_OPTS
    # one less is accepted and exact (the largest k Corollary 3.4 admits)
    got = _run(torch, ff, p, "N", "N", m, n, kw - 1, 1, A[:, :kw - 1], B[:kw - 1], 0, C,
               {"scheme": 4, "winograd": l})
    np.testing.assert_array_equal(got, oracle.fgemm(p, "N", "N", 1, A[:, :kw - 1], B[:kw - 1], 0, C))


@pytest.mark.gpu
@pytest.mark.parametrize("p,l,d", [(65521, 1, 1), (65521, 2, 1), (65521, 3, 1), (65521, 1, 1000),
                                   (65521, 2, 1000), (8388593, 1, 56), (8388593, 2, 6), (251, 3, 4000)])
def test_appendix_a6_witnesses_on_the_gpu(env, p, l, d):
    """The witnesses A_l, B_l on the balanced range
    [-(p-1)/2, (p-1)/2], stretched to k = 2^l d: their largest Winograd
    intermediate equals Theorem 3.1's bound (pinned in
    test_oracle_winograd_bound.py); below k_winograd the GPU result is exact."""
    torch, ff = env
    h = (p - 1) // 2
    Aw, Bw = winograd.witness(l, h, -h, h, -h)
    A = np.array([[x for x in r for _ in range(d)] for r in Aw], dtype=np.int64)
    B = np.array([list(r) for r in Bw for _ in range(d)], dtype=np.int64)
    k = 2 ** l * d
    assert k < bounds.k_winograd_exact(p, 53, l, balanced=True)
    assert bounds.thm31_bound(h, -h, h, -h, k, l) < 2 ** 53
    A32, B32 = (A % p).astype(np.int32), (B % p).astype(np.int32)
    C = np.zeros((A.shape[0], B.shape[1]), np.int32)
    got = _run(torch, ff, p, "N", "N", A.shape[0], B.shape[1], k, 1, A32, B32, 0, C,
               {"scheme": 4, "winograd": l})
    np.testing.assert_array_equal(got, oracle.fgemm(p, "N", "N", 1, A32, B32, 0, C))


def _p6_adversary(p, m, n, d, rng):
    """A (m x 2d), B (2d x n) with A.6's one-level block structure on every row /
    column: A = [[-M_i, 0], [M_i, M_i]], B = [[N_j, -N_j], [0, N_j]] (blocks of
    d columns / rows), M_i, N_j odd and close to (p-1)/2, so P6 = S2 T2 =
    9 M_i N_j d at the leaf reaches Theorem 3.1's bound and its partial sums
    are odd multiples of 9 M_i N_j -- not representable in a double past 2^53."""
    h = (p - 1) // 2
    Mi = h - 1 - 2 * rng.integers(0, 50, size=m // 2)
    Nj = h - 1 - 2 * rng.integers(0, 50, size=n // 2)
    assert (Mi % 2 == 1).all() and (Nj % 2 == 1).all()
    A = np.zeros((m, 2 * d), np.int64)
    A[:m // 2, :d] = -Mi[:, None]
    A[m // 2:, :d] = Mi[:, None]
    A[m // 2:, d:] = Mi[:, None]
    B = np.zeros((2 * d, n), np.int64)
    B[:d, :n // 2] = Nj[None, :]
    B[:d, n // 2:] = -Nj[None, :]
    B[d:, n // 2:] = Nj[None, :]
    return (A % p).astype(np.int32), (B % p).astype(np.int32)


@pytest.mark.gpu
def test_f64_winograd_past_the_bound_is_wrong(env):
    """p = 8388593, one level: k_winograd = 114.  The adversary is exact at
    k = 112 (bound below 2^53) and, with the bound lifted (debug_unchecked_kb),
    wrong at k = 4 * 114, where P6 reaches ~3.6e16 > 2^53 with odd partial sums;
    the classical fp64 engine (Eq. (2) reductions) stays exact there."""
    torch, ff = env
    p = 8388593
    rng = np.random.default_rng(7)
    m = n = 64
    for d, expect_exact in [(56, True), (228, False)]:
        A, B = _p6_adversary(p, m, n, d, rng)
        k = 2 * d
        C = np.zeros((m, n), np.int32)
        want = oracle.fgemm(p, "N", "N", 1, A, B, 0, C)
        opts = {"scheme": 4, "winograd": 1}
        if not expect_exact:
            with pytest.raises(ff.FFError):
                _run(torch, ff, p, "N", "N", m, n, k, 1, A, B, 0, C, opts)
            opts["debug_unchecked_kb"] = 1
        got = _run(torch, ff, p, "N", "N", m, n, k, 1, A, B, 0, C, opts)
        if expect_exact:
            np.testing.assert_array_equal(got, want)
        else:
            assert (got != want).any(), "past Corollary 3.4's bound the unreduced Winograd must round"
            classical = _run(torch, ff, p, "N", "N", m, n, k, 1, A, B, 0, C, {"scheme": 4})
            np.testing.assert_array_equal(classical, want)
