"""The small-field latency path (gemm_small.cu: p < 2^16, warp-level mma.sync on
byte-split residues, no encoders) against the oracle, forced on
with ff_opts.small_path = 1 for every shape, and bit-identical to the tcgen05 path
(small_path = -1)."""
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
def test_small_path_vs_oracle(env, p, tA, tB):
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
            for mode in (1, -1):
                dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
                ff.ff_gemm_ex(p, tA, tB, m, n, k, alpha, dA, A.shape[1], dB, B.shape[1], beta, dC, C.shape[1],
                              {"small_path": mode})
                torch.cuda.synchronize()
                got = dC.cpu().numpy()
                np.testing.assert_array_equal(got[:, :n], want, err_msg="small_path=%s m=%d n=%d k=%d" % (mode, m, n, k))
                np.testing.assert_array_equal(got[:, n:], C[:, n:])
                outs.append(got)
            np.testing.assert_array_equal(outs[0], outs[1])


def test_small_path_k_at_the_s32_bound(env):
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
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    ff.ff_gemm_ex(p, "N", "N", m, n, k, 1, dA, k, dB, n, 0, dC, n, {"small_path": 1})
    torch.cuda.synchronize()
    np.testing.assert_array_equal(dC.cpu().numpy(), want)


@pytest.mark.parametrize("p", [2, 251, 65521, 65537, 8388593, 16777259, 67108859, 2 ** 31 - 1])
def test_small_path_canonical_inputs(env, p):
    """inputs_canonical = 1 (A, B already in [0, p)): the cp.async variants
    stream them raw (p < 2^16: two bytes, four byte products; larger p: three
    or four bytes, 9 or 16 byte products); ragged K and n exercise its partial (zero-filled) 16-byte
    chunks, transposed operands fall back to the reducing kernel.  C stays any
    int32.  Bit-exact vs the oracle, forced on and under the default rule."""
    torch, ff = env
    rng = np.random.default_rng(p * 3 + 1)
    for (m, n, k, tA, tB) in [(5, 3, 7, "N", "N"), (64, 64, 32, "N", "N"), (65, 63, 33, "N", "N"),
                              (128, 301, 130, "N", "N"), (200, 70, 1000, "N", "N"), (17, 129, 4101, "N", "N"),
                              (128, 128, 1024, "N", "N"), (40, 50, 60, "T", "N"), (40, 50, 60, "N", "T")]:
        ar, ac = (m, k) if tA == "N" else (k, m)
        br, bc = (k, n) if tB == "N" else (n, k)
        la, lb = (ac + 3) // 4 * 4 + 4, (bc + 3) // 4 * 4     # leading dimensions: multiples of 4
        A = rng.integers(0, p, size=(ar, la), dtype=np.int64).astype(np.int32)
        B = rng.integers(0, p, size=(br, lb), dtype=np.int64).astype(np.int32)
        C = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
        alpha, beta = p - 1, 1
        want = oracle.fgemm(p, tA, tB, alpha, A[:, :ac], B[:, :bc], beta, C, m=m, n=n, k=k)
        for mode in (1, 0):
            dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
            ff.ff_gemm_ex(p, tA, tB, m, n, k, alpha, dA, la, dB, lb, beta, dC, n,
                          {"inputs_canonical": 1, "small_path": mode})
            torch.cuda.synchronize()
            np.testing.assert_array_equal(dC.cpu().numpy(), want, err_msg="m=%d n=%d k=%d %s%s small_path=%s" % (
                m, n, k, tA, tB, mode))


@pytest.mark.parametrize("p", [65521, 8388593])
@pytest.mark.parametrize("canonical", [0, 1])
def test_in_place_products(env, p, canonical):
    """C aliasing B (X <- W X) or A (X <- X W), as LQUP's U_rest / G products
    do: the small paths read A and B while other CTAs write C, so an overlap
    must either take the grid-barrier variant (canonical inputs) or the
    tcgen05 path (which reads only its encoded planes).  Forced small paths
    (small_path = 1) included; results bit-exact."""
    torch, ff = env
    rng = np.random.default_rng(p + canonical)
    for mode in (1, 0):
        for (r, c) in [(128, 1000), (300, 128), (128, 128)]:
            k = r if c >= r else c
            W = rng.integers(0, p, size=(k, k), dtype=np.int64).astype(np.int32)
            X = rng.integers(0, p, size=(r, c), dtype=np.int64).astype(np.int32)
            opts = {"inputs_canonical": canonical, "small_path": mode}
            dW = torch.from_numpy(W).cuda()
            if c >= r:      # X <- W X  (C = B)
                dX = torch.from_numpy(X).cuda()
                ff.ff_gemm_ex(p, "N", "N", r, c, r, 1, dW, k, dX, c, 0, dX, c, opts)
                want = oracle.fgemm(p, "N", "N", 1, W, X, 0, None, m=r, n=c, k=r)
            else:           # X <- X W  (C = A)
                dX = torch.from_numpy(X).cuda()
                ff.ff_gemm_ex(p, "N", "N", r, c, c, 1, dX, c, dW, k, 0, dX, c, opts)
                want = oracle.fgemm(p, "N", "N", 1, X, W, 0, None, m=r, n=c, k=c)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(dX.cpu().numpy(), want, err_msg="%dx%d small_path=%s" % (r, c, mode))


@pytest.mark.parametrize("p", [251, 65521])
def test_streaming_kernel_reduces_raw_operands(env, p):
    """The default rule's raw-input branch of the streaming kernel (non-transposed
    A and B with 16-byte rows: leading dimensions multiples of 4, any int32
    values, each K slice reduced in shared memory), ragged m, n, k, and an
    in-place call (C aliasing A) with raw inputs; bit-exact vs the oracle, with
    the size rule (small_path = 0) and forced (1)."""
    torch, ff = env
    rng = np.random.default_rng(p + 99)
    for (m, n, k) in [(65, 63, 33), (200, 70, 1000), (128, 256, 512), (1, 4, 4)]:
        la, lb = (k + 3) // 4 * 4, (n + 3) // 4 * 4
        A = rng.integers(-2 ** 31, 2 ** 31, size=(m, la), dtype=np.int64).astype(np.int32)
        B = rng.integers(-2 ** 31, 2 ** 31, size=(k, lb), dtype=np.int64).astype(np.int32)
        C = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
        for alpha, beta in [(1, 0), (p - 1, 1)]:
            want = oracle.fgemm(p, "N", "N", alpha, A[:, :k], B[:, :n], beta, C, m=m, n=n, k=k)
            for mode in (0, 1):
                dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
                ff.ff_gemm_ex(p, "N", "N", m, n, k, alpha, dA, la, dB, lb, beta, dC, n, {"small_path": mode})
                torch.cuda.synchronize()
                np.testing.assert_array_equal(dC.cpu().numpy(), want, err_msg="%dx%dx%d mode %d" % (m, n, k, mode))
    # in place, raw inputs: X <- X W with X m x k (ld multiple of 4), W k x k
    m, k = 96, 64
    X = rng.integers(-2 ** 31, 2 ** 31, size=(m, k), dtype=np.int64).astype(np.int32)
    W = rng.integers(-2 ** 31, 2 ** 31, size=(k, k), dtype=np.int64).astype(np.int32)
    want = oracle.fgemm(p, "N", "N", 1, X, W, 0, None, m=m, n=k, k=k)
    for mode in (0, 1):
        dX, dW = torch.from_numpy(X).cuda(), torch.from_numpy(W).cuda()
        ff.ff_gemm_ex(p, "N", "N", m, k, k, 1, dX, k, dW, k, 0, dX, k, {"small_path": mode})
        torch.cuda.synchronize()
        np.testing.assert_array_equal(dX.cpu().numpy(), want, err_msg="in place, mode %d" % mode)


# ---------------------------------------------------------------- tcgen05 latency kernel (gemm_lat.cu)

@pytest.mark.parametrize("p", [2, 3, 251, 257, 4099, 65521])
@pytest.mark.parametrize("tA,tB", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_lat_kernel_vs_oracle(env, p, tA, tB):
    """The one-launch tcgen05 kernel (split-K cluster, DSMEM reduction, coalesced
    epilogue) forced on (small_path = 2): any int32 inputs, ragged shapes across
    tile / chunk / cluster boundaries, every transpose; bit-exact vs the oracle
    and bit-identical to the encoder + tcgen05 path (small_path = -1)."""
    torch, ff = env
    rng = np.random.default_rng(p * 7 + ord(tA) + 3 * ord(tB))
    for (m, n, k) in [(1, 1, 1), (5, 3, 7), (128, 64, 128), (129, 65, 129), (512, 512, 512), (200, 300, 1000),
                      (64, 1000, 2048), (300, 70, 5000)]:
        ar, ac = (m, k) if tA == "N" else (k, m)
        br, bc = (k, n) if tB == "N" else (n, k)
        A = rng.integers(-2 ** 31, 2 ** 31, size=(ar, ac + 3), dtype=np.int64).astype(np.int32)
        B = rng.integers(-2 ** 31, 2 ** 31, size=(br, bc + 1), dtype=np.int64).astype(np.int32)
        C = rng.integers(-2 ** 31, 2 ** 31, size=(m, n + 2), dtype=np.int64).astype(np.int32)
        for alpha, beta in [(1, 0), (p - 1, 1), (int(rng.integers(0, p)), int(rng.integers(0, p)))]:
            want = oracle.fgemm(p, tA, tB, alpha, A[:, :ac], B[:, :bc], beta, C[:, :n], m=m, n=n, k=k)
            outs = []
            for mode in (2, -1):
                dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
                ff.ff_gemm_ex(p, tA, tB, m, n, k, alpha, dA, A.shape[1], dB, B.shape[1], beta, dC, C.shape[1],
                              {"small_path": mode})
                torch.cuda.synchronize()
                got = dC.cpu().numpy()
                np.testing.assert_array_equal(got[:, :n], want, err_msg="mode %d %dx%dx%d" % (mode, m, n, k))
                np.testing.assert_array_equal(got[:, n:], C[:, n:])
                outs.append(got)
            np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("m,n", [(64, 64), (1024, 1024)])
def test_lat_kernel_at_the_s32_bound(env, m, n):
    """K = 16384 (the kernel's limit) with every residue p - 1 = 0xFFF0: the middle
    weight group of a CTA reaches 2 K 240 255 ~ 2^31 when one CTA takes all of K
    (1024^2: enough tiles that the cluster is 1 CTA); (p-1)^2 = 1 mod p gives
    the closed form (AB)_ij = K mod p (oracle pin, tests/test_oracle_pins.py)."""
    torch, ff = env
    p, k = 65521, 16384
    dA = torch.full((m, k), p - 1, dtype=torch.int32, device="cuda")
    dB = torch.full((k, n), p - 1, dtype=torch.int32, device="cuda")
    dC = torch.zeros((m, n), dtype=torch.int32, device="cuda")
    ff.ff_gemm_ex(p, "N", "N", m, n, k, 1, dA, k, dB, n, 0, dC, n, {"small_path": 2})
    torch.cuda.synchronize()
    assert bool((dC == k % p).all())
