"""Tiny fgemm kernel time by alpha/beta and shape (CUDA events around 20 calls).  Development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_cs_0601133_b200 as ff  # noqa: E402

p = 65521
torch.cuda.set_device(0)
for m, n, k in [(128, 128, 128), (128, 256, 128), (256, 256, 128)]:
    X = torch.randint(0, p, (m, k), dtype=torch.int32, device="cuda")
    Y = torch.randint(0, p, (k, n), dtype=torch.int32, device="cuda")
    C = torch.randint(0, p, (m, n), dtype=torch.int32, device="cuda")
    for al, be in [(1, 0), (p - 1, 1), (5, 7)]:
        for _ in range(3):
            ff.fgemm(p, X, Y, C, al, be)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            ff.fgemm(p, X, Y, C, al, be)
        e1.record()
        torch.cuda.synchronize()
        print("m=%d n=%d k=%d alpha=%d beta=%d: %.1f us" % (m, n, k, al, be, e0.elapsed_time(e1) / 20 * 1e3), flush=True)
