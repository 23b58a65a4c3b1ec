"""Randomized sweep of the other fgemm entry points against the oracle:
ff_gemm_host (pipelined host buffers, random block sizes) and one Winograd
level (even shapes, random schemes).  Development aid: prints failures."""
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
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
bad = done = 0
for case in range(n_cases):
    p = _random_prime(rng)
    host = case % 2 == 0
    if host:
        m, n, k = (int(x) for x in rng.integers(1, 1500, size=3))
        opts = {"host_block": int(rng.choice([0, 256, 512, 1024]))}
    else:
        m, n, k = 2 * int(rng.integers(256, 700)), 2 * int(rng.integers(256, 700)), 2 * int(rng.integers(128, 700))
        opts = {"winograd": 1}
        if rng.random() < 0.5:
            opts["scheme"] = int(rng.choice([1, 2, 3]))
    try:
        ff.ff_plan_query(p, k, opts)
    except Exception:
        continue
    tA, tB = str(rng.choice(["N", "T"])), str(rng.choice(["N", "T"]))
    ar, ac = (m, k) if tA == "N" else (k, m)
    br, bc = (k, n) if tB == "N" else (n, k)
    A = rng.integers(-2 ** 31, 2 ** 31, size=(ar, ac), dtype=np.int64).astype(np.int32)
    B = rng.integers(-2 ** 31, 2 ** 31, size=(br, bc), dtype=np.int64).astype(np.int32)
    C = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
    alpha, beta = int(rng.integers(0, p)), int(rng.choice([0, 1, int(rng.integers(0, p))]))
    want = oracle.fgemm(p, tA, tB, alpha, A, B, beta, C, m=m, n=n, k=k)
    if host:
        out = C.copy()
        ff.ff_gemm_host(p, tA, tB, m, n, k, alpha, A, ac, B, bc, beta, out, n, opts)
    else:
        dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
        try:
            ff.ff_gemm_ex(p, tA, tB, m, n, k, alpha, dA, ac, dB, bc, beta, dC, n, opts)
        except ff.FFError as ex:
            print("REJECTED winograd p=%d m=%d n=%d k=%d %s%s opts=%s: %s" % (p, m, n, k, tA, tB, opts, ex), flush=True)
            continue
        torch.cuda.synchronize()
        out = dC.cpu().numpy()
    done += 1
    if not np.array_equal(out, want):
        bad += 1
        print("MISMATCH %s p=%d m=%d n=%d k=%d %s%s opts=%s" % ("host" if host else "winograd", p, m, n, k, tA, tB, opts),
              flush=True)
print("paths fuzz: %d cases, %d failures" % (done, bad))
