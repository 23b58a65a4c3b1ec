"""Extended random sweep of ff_gemm_ex against the oracle (same generator as
tests/test_gpu_fuzz.py, many more seeds).  Development aid: prints failures."""
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
nblocks = int(sys.argv[1]) if len(sys.argv) > 1 else 50
bad = done = 0
for block in range(100, 100 + nblocks):
    rng = np.random.default_rng(20261019 + block)
    for case in range(40):
        p = _random_prime(rng)
        m, n, k = (int(x) for x in rng.choice([1, 2, 7, 31, 64, 127, 128, 129, 200, 255, 256, 300, 383, 513, 1000] + ([1024, 1536, 2047, 2304] if os.environ.get("FUZZ_BIG") else []), size=3))
        tA, tB = str(rng.choice(["N", "T"])), str(rng.choice(["N", "T"]))
        opts = {}
        r = rng.random()
        if r < 0.15: opts["scheme"] = 1
        elif r < 0.3: opts["scheme"] = 2
        elif r < 0.45: opts["scheme"] = 3
        elif r < 0.5: opts["scheme"] = 4
        if rng.random() < 0.3: opts["cta_group"] = int(rng.choice([1, 2]))
        if rng.random() < 0.2 and opts.get("scheme", 0) != 4: opts["korder"] = int(rng.choice([1, 2]))
        if rng.random() < 0.2 and opts.get("scheme", 0) in (1, 2): opts["kb_override"] = int(rng.choice([128, 256]))
        canon = rng.random() < 0.3
        if canon: opts["inputs_canonical"] = 1
        try:
            ff.ff_plan_query(p, k, opts)
        except Exception:
            continue
        ar, ac = (m, k) if tA == "N" else (k, m)
        br, bc = (k, n) if tB == "N" else (n, k)
        la, lb, lc = ac + int(rng.integers(0, 5)), bc + int(rng.integers(0, 5)), n + int(rng.integers(0, 3))
        lo = 0 if canon else (-2 ** 31 if rng.random() < 0.3 else 0)
        hi = p if lo == 0 else 2 ** 31
        Abuf = rng.integers(lo, hi, size=(ar, la), dtype=np.int64).astype(np.int32)
        Bbuf = rng.integers(lo, hi, size=(br, lb), dtype=np.int64).astype(np.int32)
        Cbuf = rng.integers(-2 ** 31, 2 ** 31, size=(m, lc), dtype=np.int64).astype(np.int32)
        alpha = int(rng.choice([0, 1, p - 1, int(rng.integers(0, p))]))
        beta = int(rng.choice([0, 1, p - 1, int(rng.integers(0, p))]))
        A, B, C = (torch.from_numpy(x).cuda() for x in (Abuf, Bbuf, Cbuf))
        ff.ff_gemm_ex(p, tA, tB, m, n, k, alpha, A, la, B, lb, beta, C, lc, opts)
        torch.cuda.synchronize()
        got = C.cpu().numpy()
        want = oracle.fgemm(p, tA, tB, alpha, Abuf[:, :ac], Bbuf[:, :bc], beta, Cbuf[:, :n], m=m, n=n, k=k)
        done += 1
        if not (np.array_equal(got[:, :n], want) and np.array_equal(got[:, n:], Cbuf[:, n:])):
            bad += 1
            print("MISMATCH p=%d m=%d n=%d k=%d %s%s a=%d b=%d opts=%s" % (p, m, n, k, tA, tB, alpha, beta, opts), flush=True)
print("fuzz: %d cases, %d mismatches" % (done, bad))
