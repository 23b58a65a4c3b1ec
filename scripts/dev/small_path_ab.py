"""A/B of the small-field path (FF_SMALL=1) against the tcgen05 path (FF_SMALL=0)
on a grid of shapes (p = 65521), CUDA events.  Run once per setting.  Development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_cs_0601133_b200 as ff  # noqa: E402

p = 65521
torch.cuda.set_device(0)
shapes = [(128, 128, 128), (512, 512, 512), (128, 8192, 128), (8192, 128, 128), (128, 8192, 1024),
          (1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 128), (8192, 8192, 128), (8192, 8192, 512),
          (4096, 4096, 4096), (16384, 16384, 128)]
for m, n, k in shapes:
    X = torch.randint(0, p, (m, k), dtype=torch.int32, device="cuda")
    Y = torch.randint(0, p, (k, n), dtype=torch.int32, device="cuda")
    C = torch.randint(0, p, (m, n), dtype=torch.int32, device="cuda")
    canon = os.environ.get("CANON") == "1"
    opts = {"inputs_canonical": 1} if canon else None
    for _ in range(3):
        ff.fgemm(p, X, Y, C, p - 1, 1, opts=opts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        ff.fgemm(p, X, Y, C, p - 1, 1, opts=opts)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps
    print("CANON=%d FF_SMALL=%s m=%5d n=%5d k=%5d  %9.1f us  %7.1f TOPS" % (canon, os.environ.get("FF_SMALL", "-"), m, n, k, t * 1e3,
                                                                2 * m * n * k / t / 1e9), flush=True)
    del X, Y, C
