"""The small-field latency path (gemm_small.cu: p < 2^16, warp-level mma.sync on
byte-split residues, no encoders) against the oracle, forced on
with FF_SMALL=1 for every shape, and bit-identical to the tcgen05 path."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

PRIMES = [2, 3, 251, 257, 4099, 65521]


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_cs_0601133_b200 as ff
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return torch, ff


@pytest.mark.parametrize("p", PRIMES)
@pytest.mark.parametrize("tA,tB", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_small_path_vs_oracle(env, p, tA, tB, monkeypatch):
    torch, ff = env
    rng = np.random.default_rng(p + ord(tA) * 7 + ord(tB))
    for (m, n, k) in [(1, 1, 1), (5, 3, 7), (64, 64, 32), (65, 63, 33), (128, 300, 128), (200, 70, 1000),
                      (17, 129, 4100)]:
        ar, ac = (m, k) if tA == "N" else (k, m)
        br, bc = (k, n) if tB == "N" else (n, k)
        A = rng.integers(-2 ** 31, 2 ** 31, size=(ar, ac + 1), dtype=np.int64).astype(np.int32)
        B = rng.integers(-2 ** 31, 2 ** 31, size=(br, bc + 2), dtype=np.int64).astype(np.int32)
        C = rng.integers(-2 ** 31, 2 ** 31, size=(m, n + 3), dtype=np.int64).astype(np.int32)
        for alpha, beta in [(1, 0), (p - 1, 1), (int(rng.integers(0, p)), int(rng.integers(0, p)))]:
            want = oracle.fgemm(p, tA, tB, alpha, A[:, :ac], B[:, :bc], beta, C[:, :n], m=m, n=n, k=k)
            outs = []
            for mode in ("1", "0"):
                monkeypatch.setenv("FF_SMALL", mode)
                dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
                ff.ff_gemm_ex(p, tA, tB, m, n, k, alpha, dA, A.shape[1], dB, B.shape[1], beta, dC, C.shape[1])
                torch.cuda.synchronize()
                got = dC.cpu().numpy()
                np.testing.assert_array_equal(got[:, :n], want, err_msg="FF_SMALL=%s m=%d n=%d k=%d" % (mode, m, n, k))
                np.testing.assert_array_equal(got[:, n:], C[:, n:])
                outs.append(got)
            np.testing.assert_array_equal(outs[0], outs[1])


def test_small_path_k_at_the_s32_bound(env, monkeypatch):
    """K = 32768 with every byte 255 (x = 65535 is not a residue mod 65521, but
    p - 1 = 65520 = 0xFFF0 maximises the high bytes): each byte product sum
    reaches 32768 * 255^2 < 2^31, the largest K the path accepts."""
    torch, ff = env
    p = 65521
    m, n, k = 64, 64, 32768
    A = np.full((m, k), p - 1, np.int32)
    B = np.full((k, n), p - 1, np.int32)
    C = np.zeros((m, n), np.int32)
    want = oracle.fgemm(p, "N", "N", 1, A, B, 0, C, m=m, n=n, k=k)
    monkeypatch.setenv("FF_SMALL", "1")
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    ff.ff_gemm_ex(p, "N", "N", m, n, k, 1, dA, k, dB, n, 0, dC, n)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(dC.cpu().numpy(), want)
