"""Extended random sweep of ftrsm and LQUP against the oracle.  Development aid."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402
from test_gpu_fuzz import _random_prime  # noqa: E402
from test_gpu_lqup import _check_valid, _low_rank  # noqa: E402
from test_gpu_trsm import _tri  # noqa: E402

torch.cuda.set_device(0)
n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 4242)
bad = 0
for case in range(n_cases):
    p = _random_prime(rng)
    side, uplo, trans, diag = (str(rng.choice(list(x))) for x in ("LR", "UL", "NT", "NU"))
    m, n = (int(x) for x in rng.integers(1, 1300, size=2))
    d = m if side == "L" else n
    A = _tri(rng, p, d, uplo, diag, ld_extra=int(rng.integers(0, 3)))
    B = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
    alpha = int(rng.integers(0, p))
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    opts = {"scheme": int(rng.choice([1, 2, 3]))} if (os.environ.get("FUZZ_OPTS") and rng.random() < 0.7) else None
    try:
        ff.ftrsm(p, dA, dB, side, uplo, trans, diag, alpha, opts)
    except ff.FFError:
        continue
    torch.cuda.synchronize()
    want = oracle.trsm(p, side, uplo, trans, diag, alpha, A[:, :d], B)
    if not np.array_equal(dB.cpu().numpy(), want):
        bad += 1
        print("TRSM MISMATCH p=%d %s%s%s%s m=%d n=%d" % (p, side, uplo, trans, diag, m, n), flush=True)
for case in range(n_cases):
    p = _random_prime(rng)
    m, n = (int(x) for x in rng.integers(1, int(os.environ.get("FUZZ_MAXN", 900)), size=2))
    if rng.random() < 0.4:
        A = _low_rank(rng, p, m, n, int(rng.integers(0, min(m, n) + 1)))
    else:
        A = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
    if rng.random() < 0.5:                               # structure: zero / repeated rows and columns
        for _ in range(int(rng.integers(1, 6))):
            kind = int(rng.integers(0, 4))
            i, j = int(rng.integers(0, m)), int(rng.integers(0, m))
            c0 = int(rng.integers(0, n))
            if kind == 0: A[i] = 0
            elif kind == 1: A[i] = A[j]
            elif kind == 2: A[:, c0:c0 + int(rng.integers(1, 200))] = 0
            else: A[i:i + int(rng.integers(1, 200)), :] = A[j]
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    opts = {"scheme": int(rng.choice([1, 2, 3]))} if (os.environ.get("FUZZ_OPTS") and rng.random() < 0.7) else None
    try:
        Q, P, rk = ff.lqup(p, dA, opts)
    except ff.FFError:
        continue
    torch.cuda.synchronize()
    F = dA.cpu().numpy()
    want_r, want_d = oracle.rank_det(p, A)
    try:
        assert rk == want_r
        _check_valid(p, A, F, Q, P, rk)
        if m == n:
            assert ff.rank_det(p, torch.from_numpy(A).cuda())[1] == want_d
    except AssertionError as ex:
        bad += 1
        print("LQUP MISMATCH p=%d m=%d n=%d: %s" % (p, m, n, str(ex)[:200]), flush=True)
print("solver fuzz: %d trsm + %d lqup cases, %d failures" % (n_cases, n_cases, bad))
