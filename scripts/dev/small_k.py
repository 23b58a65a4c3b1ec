"""Small-K update GEMMs (the LQUP / ftrsm trailing updates): C <- (-X Y + C) mod p,
timed with CUDA events; reports the C read+write bandwidth.  Development aid.
    python scripts/small_k.py [once]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_cs_0601133_b200 as ff  # noqa: E402

p = int(os.environ.get("P", 65521))
once = "once" in sys.argv
torch.cuda.set_device(0)
shapes = [(8192, 8192, 128)] if once else [(8192, 8192, 128), (16384, 16384, 128), (8192, 8192, 256), (8192, 8192, 512)]
for m, n, k in shapes:
    X = torch.empty((m, k), dtype=torch.int32, device="cuda")
    Y = torch.empty((k, n), dtype=torch.int32, device="cuda")
    C = torch.empty((m, n), dtype=torch.int32, device="cuda")
    ff.ff_fill_uniform(X, m, k, k, p, 1, 0)
    ff.ff_fill_uniform(Y, k, n, n, p, 1, 1)
    ff.ff_fill_uniform(C, m, n, n, p, 1, 2)
    if once:
        ff.fgemm(p, X, Y, C, p - 1, 1)
        torch.cuda.synchronize()
        break
    for _ in range(2):
        ff.fgemm(p, X, Y, C, p - 1, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        ff.fgemm(p, X, Y, C, p - 1, 1)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    print("m=%d n=%d k=%d  %.1f us  C r+w %.2f TB/s" % (m, n, k, t * 1e3, 8 * m * n / t / 1e9), flush=True)
    del X, Y, C
