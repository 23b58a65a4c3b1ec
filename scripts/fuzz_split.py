"""Randomized sweep of the split entry points (ff_encode + ff_gemm_limbs: encode
A once, multiply by random column chunks of B, as the multi-GPU driver does)
against the oracle.  Development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402
from test_gpu_fuzz import _random_prime  # noqa: E402

torch.cuda.set_device(0)
n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
bad = done = 0
for case in range(n_cases):
    p = _random_prime(rng)
    m, n, k = (int(x) for x in rng.integers(1, 1200, size=3))
    opts = {}
    if rng.random() < 0.5:
        opts["scheme"] = int(rng.choice([1, 2, 3]))
    try:
        info = ff.ff_plan_query(p, k, opts)
    except Exception:
        continue
    L, kp = info["L"], info["k_pad"]
    A = rng.integers(-2 ** 31, 2 ** 31, size=(m, k), dtype=np.int64).astype(np.int32)
    B = rng.integers(-2 ** 31, 2 ** 31, size=(k, n), dtype=np.int64).astype(np.int32)
    C = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
    alpha, beta = int(rng.integers(0, p)), int(rng.choice([0, 1, int(rng.integers(0, p))]))
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    Al = torch.empty((L, m, kp), dtype=torch.int8, device="cuda")
    ff.ff_encode(p, k, opts, 1, m, dA, k, Al)
    cuts = sorted(set([0, n] + [int(x) for x in rng.integers(0, n, size=int(rng.integers(0, 4)))]))
    for n0, n1 in zip(cuts[:-1], cuts[1:]):
        if n1 <= n0:
            continue
        Bl = torch.empty((L, n1 - n0, kp), dtype=torch.int8, device="cuda")
        ff.ff_encode(p, k, opts, 0, n1 - n0, dB[:, n0:], n, Bl)
        ff.ff_gemm_limbs(p, m, n1 - n0, k, opts, alpha, Al, Bl, beta, dC[:, n0:], n)
    torch.cuda.synchronize()
    want = oracle.fgemm(p, "N", "N", alpha, A, B, beta, C)
    done += 1
    if not np.array_equal(dC.cpu().numpy(), want):
        bad += 1
        print("MISMATCH p=%d m=%d n=%d k=%d opts=%s cuts=%s" % (p, m, n, k, opts, cuts), flush=True)
print("split fuzz: %d cases, %d failures" % (done, bad))
