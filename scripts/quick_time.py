"""Quick per-config timing (CUDA events) of ff_gemm on device-resident inputs.
Development aid; the contract benchmark is bench.py."""
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ffgen  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402

CONFIGS = {
    "c1": (65521, 512, 512, 512, "N", "N", 1, 0, 1),
    "c2": (8388593, 4096, 4096, 4096, "N", "N", 3, 1, 2),
    "c3": (251, 8192, 8192, 16384, "T", "N", 1, 0, 3),
    "c4": (65521, 32768, 32768, 8192, "N", "N", 1, 0, 4),
    "c5": (67108859, 16384, 16384, 16384, "N", "N", 67108858, 1, 5),
}


def main(names, reps=5):
    torch.cuda.set_device(0)
    for name in names:
        p, m, n, k, tA, tB, alpha, beta, seed = CONFIGS[name]
        ar, ac = (m, k) if tA == "N" else (k, m)
        A = torch.empty((ar, ac), dtype=torch.int32, device="cuda")
        B = torch.empty((k, n), dtype=torch.int32, device="cuda")
        C = torch.zeros((m, n), dtype=torch.int32, device="cuda")
        ff.ff_fill_uniform(A, ar, ac, ac, p, seed, 0)
        ff.ff_fill_uniform(B, k, n, n, p, seed, 1)
        info = ff.ff_plan_query(p, k)
        for _ in range(2):
            ff.fgemm(p, A, B, C, alpha, beta, tA, tB)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ff.fgemm(p, A, B, C, alpha, beta, tA, tB)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = min(ts) / 1e3
        useful = 2.0 * m * n * k
        mma = useful * (info["L"] if info["scheme"] == "CRT" else info["L"] ** 2)   # int8 products per output
        print("%s p=%d L=%d  t=%.3f ms  useful %.1f TOPS  int8-MMA %.1f TOPS (%.1f%% of 3305)" % (
            name, p, info["L"], t * 1e3, useful / t / 1e12, mma / t / 1e12, 100 * mma / t / 3.305e15),
            flush=True)
        del A, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIGS))
