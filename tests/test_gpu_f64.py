"""GPU parity of the paper-literal fp64 engine (FF_SCHEME_FP64, DESIGN.md
§14: centred residues as doubles on DMMA, Eq. (2) delayed reduction) against
the oracle, bit-exact; plus a demonstration that the Eq. (2) bound is needed."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

PRIMES = [2, 3, 251, 65521, 8388593, 67108859]
SHAPES = [(1, 1, 1), (3, 5, 7), (64, 64, 16), (65, 130, 33), (200, 300, 1000), (256, 512, 640)]


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


@pytest.mark.parametrize("p", PRIMES)
@pytest.mark.parametrize("tA,tB", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_f64_engine_vs_oracle(env, p, tA, tB):
    torch, ff = env
    rng = np.random.default_rng(p % 1013 + ord(tA) + 3 * ord(tB))
    for si, (m, n, k) in enumerate(SHAPES):
        A = rng.integers(-2 ** 31, 2 ** 31, size=(m, k) if tA == "N" else (k, m), dtype=np.int64).astype(np.int32)
        B = rng.integers(0, p, size=(k, n) if tB == "N" else (n, k)).astype(np.int32)
        C = rng.integers(0, p, size=(m, n)).astype(np.int32)
        alpha = [1, p - 1, int(rng.integers(0, p))][si % 3]
        beta = [0, 1, int(rng.integers(0, p))][(si + 1) % 3]
        got = _run(torch, ff, p, tA, tB, m, n, k, alpha, A, B, beta, C, {"scheme": 4})
        np.testing.assert_array_equal(got, oracle.fgemm(p, tA, tB, alpha, A, B, beta, C))


@pytest.mark.parametrize("p", [65521, 8388593, 67108859])
@pytest.mark.parametrize("kb", [4, 16, 100])
def test_f64_forced_reductions(env, p, kb):
    torch, ff = env
    rng = np.random.default_rng(kb)
    m, n, k = 130, 70, 777
    A = rng.integers(0, p, size=(m, k)).astype(np.int32)
    B = rng.integers(0, p, size=(k, n)).astype(np.int32)
    C = rng.integers(0, p, size=(m, n)).astype(np.int32)
    info = ff.ff_plan_query(p, k, {"scheme": 4})
    kbo = min(kb, info["kb_max"])
    got = _run(torch, ff, p, "N", "N", m, n, k, 3, A, B, 5, C, {"scheme": 4, "kb_override": kbo})
    np.testing.assert_array_equal(got, oracle.fgemm(p, "N", "N", 3, A, B, 5, C))


@pytest.mark.parametrize("p", [65521, 8388593, 67108859])
def test_f64_at_the_eq2_bound_and_beyond(env, p):
    """All entries (p+1)/2 (centred -(p-1)/2): k lambda-blocks of the largest
    products Eq. (2) admits are exact; with the bound lifted (test knob) the
    fp64 accumulator must round and the result is wrong -- Eq. (2) is needed."""
    torch, ff = env
    info = ff.ff_plan_query(p, 1, {"scheme": 4})
    lam = info["kb_max"]
    cm = (p - 1) // 2
    assert lam * cm * cm < 2 ** 52 <= (lam + 1) * cm * cm            # PAPER.md Eq. (2), gamma = 53
    k = 4096
    m, n = 64, 64
    A = np.full((m, k), (p + 1) // 2, np.int32)
    B = np.full((k, n), (p + 1) // 2, np.int32)
    C = np.zeros((m, n), np.int32)
    got = _run(torch, ff, p, "N", "N", m, n, k, 1, A, B, 0, C, {"scheme": 4})
    assert (got == (k * cm * cm) % p).all()
    # beyond the bound: an odd centred value c (so the partial sums j c^2 are odd
    # for odd j and stop being representable past 2^53); one unreduced block of k
    c = cm if cm % 2 else cm - 1
    if k * c * c >= 2 ** 54:
        A2 = np.full((m, k), p - c, np.int32)
        B2 = np.full((k, n), p - c, np.int32)
        bad = _run(torch, ff, p, "N", "N", m, n, k, 1, A2, B2, 0, C,
                   {"scheme": 4, "kb_override": k, "debug_unchecked_kb": 1})
        assert (bad != (k * c * c) % p).any()
        good = _run(torch, ff, p, "N", "N", m, n, k, 1, A2, B2, 0, C, {"scheme": 4})
        assert (good == (k * c * c) % p).all()
