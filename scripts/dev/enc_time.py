"""Time the limb encoders (direct / transposed) on config-sized operands. Development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_cs_0601133_b200 as ff  # noqa: E402

torch.cuda.set_device(0)
for p, rows, k in [(65521, 32768, 8192), (251, 8192, 16384), (67108859, 16384, 16384)]:
    info = ff.ff_plan_query(p, k)
    L = info["L"]
    for kmaj in (1, 0):
        X = torch.randint(0, p, (rows, k) if kmaj else (k, rows), dtype=torch.int32, device="cuda")
        Y = torch.empty((L, rows, info["k_pad"]), dtype=torch.int8, device="cuda")
        for _ in range(3):
            ff.ff_encode(p, k, None, kmaj, rows, X, X.shape[1], Y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ff.ff_encode(p, k, None, kmaj, rows, X, X.shape[1], Y)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 10 / 1e3
        by = rows * k * (4 + L)
        print("p=%d rows=%d k=%d L=%d %s: %.3f ms  %.0f GB/s" % (p, rows, k, L, "direct" if kmaj else "trans ", t * 1e3, by / t / 1e9))
        del X, Y
