"""Seeded random sweep of ff_gemm_ex against the oracle (bit-exact): random
primes (2 .. 2^31 - 1), shapes with ragged tails, transposes, leading
dimensions, alpha / beta (incl. 0, 1, p - 1), non-canonical int32 inputs and
every option the planner accepts (scheme S / T / CRT / FP64, kernel, step
order, forced k-blocks, one Winograd level).  A combination the planner
rejects must be rejected by ff_plan_query too (and is then skipped)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _is_prime(n):
    if n < 2:
        return False
    for q in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if n % q == 0:
            return n == q
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17):          # deterministic below 3.4e14
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


def _random_prime(rng):
    bits = int(rng.choice([2, 5, 8, 12, 16, 20, 23, 26, 28, 31]))
    while True:
        c = int(rng.integers(2 ** (bits - 1), 2 ** bits))
        if _is_prime(c):
            return c


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_cs_0601133_b200 as ff
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    return torch, ff


@pytest.mark.parametrize("block", range(8))
def test_gemm_random_sweep(env, block):
    torch, ff = env
    rng = np.random.default_rng(20261019 + block)
    done = 0
    for case in range(40):
        p = _random_prime(rng)
        dims = [int(x) for x in rng.choice([1, 2, 7, 31, 64, 127, 128, 129, 200, 255, 256, 300, 383], size=3)]
        m, n, k = dims
        tA, tB = str(rng.choice(["N", "T"])), str(rng.choice(["N", "T"]))
        opts = {}
        r = rng.random()
        if r < 0.2:
            opts["scheme"] = 1
        elif r < 0.4:
            opts["scheme"] = 2
        elif r < 0.6:
            opts["scheme"] = 3
        elif r < 0.7:
            opts["scheme"] = 4
        if rng.random() < 0.4:
            opts["cta_group"] = int(rng.choice([1, 2]))
        if rng.random() < 0.25 and opts.get("scheme", 0) != 4:
            opts["korder"] = int(rng.choice([1, 2]))
        if rng.random() < 0.2 and opts.get("scheme", 0) in (1, 2):
            opts["kb_override"] = int(rng.choice([128, 256]))
        if rng.random() < 0.15 and m % 2 == 0 and n % 2 == 0 and k % 2 == 0 and min(m, n, k) >= 64 \
                and opts.get("scheme", 0) != 4:
            opts["winograd"] = 1
        try:
            ff.ff_plan_query(p, k, opts)
        except Exception:
            continue                                   # the planner rejects this combination
        ar, ac = (m, k) if tA == "N" else (k, m)
        br, bc = (k, n) if tB == "N" else (n, k)
        la, lb, lc = ac + int(rng.integers(0, 3)), bc + int(rng.integers(0, 3)), n + int(rng.integers(0, 3))
        lo = -2 ** 31 if rng.random() < 0.3 else 0
        hi = 2 ** 31 if lo else p
        Abuf = rng.integers(lo, hi, size=(ar, la), dtype=np.int64).astype(np.int32)
        Bbuf = rng.integers(lo, hi, size=(br, lb), dtype=np.int64).astype(np.int32)
        Cbuf = rng.integers(lo, hi, size=(m, lc), dtype=np.int64).astype(np.int32)
        alpha = int(rng.choice([0, 1, p - 1, int(rng.integers(0, p))]))
        beta = int(rng.choice([0, 1, p - 1, int(rng.integers(0, p))]))
        A = torch.from_numpy(Abuf).cuda()
        B = torch.from_numpy(Bbuf).cuda()
        C = torch.from_numpy(Cbuf).cuda()
        ff.ff_gemm_ex(p, tA, tB, m, n, k, alpha, A, la, B, lb, beta, C, lc, opts)
        torch.cuda.synchronize()
        got = C.cpu().numpy()
        want = oracle.fgemm(p, tA, tB, alpha, Abuf[:, :ac], Bbuf[:, :bc], beta, Cbuf[:, :n], m=m, n=n, k=k)
        ctx = "p=%d m=%d n=%d k=%d %s%s alpha=%d beta=%d opts=%s" % (p, m, n, k, tA, tB, alpha, beta, opts)
        np.testing.assert_array_equal(got[:, :n], want, err_msg=ctx)
        np.testing.assert_array_equal(got[:, n:], Cbuf[:, n:], err_msg=ctx)   # ld padding untouched
        done += 1
    assert done >= 20
