"""Randomized sweep of the 256 x 512 CTA-pair tiles (ff_opts.wide_tiles = 1)
against the square tiles (wide_tiles = -1) and the oracle: random primes,
shapes, transposes, alpha/beta, limb schemes, step orders and forced k-blocks.
Development aid: prints failures.
    python scripts/fuzz_wide.py [cases] [seed]"""
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
n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 60
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 512)
bad = 0
for case in range(n_cases):
    p = _random_prime(rng)
    m, n, k = (int(rng.integers(1, 2600)), int(rng.integers(1, 2600)), int(rng.integers(1, 3000)))
    tA, tB = str(rng.choice(["N", "T"])), str(rng.choice(["N", "T"]))
    opts = {"scheme": int(rng.choice([0, 1, 2])), "small_path": -1}
    if rng.random() < 0.5:
        opts["cta_group"] = 2          # the pair kernel (and so the wide tiles) even for small outputs
    if rng.random() < 0.3:
        opts["korder"] = int(rng.choice([1, 2]))
        info = ff.ff_plan_query(p, k, {"scheme": opts["scheme"]})
        if info["scheme"] != "CRT" and info["kb_max"] >= 256:
            opts["kb_override"] = int(rng.integers(128, min(info["kb_max"], 4 * k + 256)))
    try:
        ff.ff_plan_query(p, k, opts)
    except ff.FFError:
        opts.pop("kb_override", None)
    ar, ac = (m, k) if tA == "N" else (k, m)
    br, bc = (k, n) if tB == "N" else (n, k)
    A = rng.integers(0, p, size=(ar, ac), dtype=np.int64).astype(np.int32)
    B = rng.integers(0, p, size=(br, bc), dtype=np.int64).astype(np.int32)
    C = rng.integers(0, p, size=(m, n), dtype=np.int64).astype(np.int32)
    alpha, beta = int(rng.integers(0, p)), int(rng.integers(0, p))
    outs = []
    for w in (1, -1):
        dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
        ff.ff_gemm_ex(p, tA, tB, m, n, k, alpha, dA, ac, dB, bc, beta, dC, n, dict(opts, wide_tiles=w))
        torch.cuda.synchronize()
        outs.append(dC.cpu().numpy())
    rows = sorted(set([0, m - 1] + rng.integers(0, m, size=3).tolist()))
    want = oracle.fgemm_rows(p, tA, tB, alpha, A, B, beta, C[rows], rows, m, n, k)
    ok = np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0][rows], want)
    if not ok:
        bad += 1
        print("MISMATCH p=%d m=%d n=%d k=%d %s%s opts=%s wide==square %s" % (
            p, m, n, k, tA, tB, opts, np.array_equal(outs[0], outs[1])), flush=True)
print("fuzz_wide: %d cases, %d mismatches" % (n_cases, bad), flush=True)
