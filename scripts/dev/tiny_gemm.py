"""Latency of small fgemm calls (the LQUP panel-chain GEMMs).  Development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_cs_0601133_b200 as ff  # noqa: E402

p = 65521
torch.cuda.set_device(0)
for m, n, k in [(128, 128, 128), (128, 8192, 128), (8192, 128, 128), (128, 16384, 512), (16384, 128, 512)]:
    X = torch.randint(0, p, (m, k), dtype=torch.int32, device="cuda")
    Y = torch.randint(0, p, (k, n), dtype=torch.int32, device="cuda")
    C = torch.randint(0, p, (m, n), dtype=torch.int32, device="cuda")
    for _ in range(3):
        ff.fgemm(p, X, Y, C, p - 1, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ff.fgemm(p, X, Y, C, p - 1, 1)
    e1.record()
    torch.cuda.synchronize()
    t_b2b = e0.elapsed_time(e1) / 20
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        e0.record()
        ff.fgemm(p, X, Y, C, p - 1, 1)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print("m=%5d n=%5d k=%4d  back-to-back %.1f us   single %.1f us" % (m, n, k, t_b2b * 1e3, min(ts) * 1e3), flush=True)
