"""Host-side cost of one ff.fgemm call (ctypes + planning + launches), no sync.  Development aid."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402
p = 65521
torch.cuda.set_device(0)
X = torch.randint(0, p, (128, 128), dtype=torch.int32, device="cuda")
C = torch.randint(0, p, (128, 128), dtype=torch.int32, device="cuda")
for opts in (None, {"inputs_canonical": 1}):
    for _ in range(20):
        ff.fgemm(p, X, X, C, p - 1, 1, opts=opts)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        ff.fgemm(p, X, X, C, p - 1, 1, opts=opts)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("opts=%s: host %.1f us/call, wall incl. drain %.1f us/call" % (opts, (t1 - t0) / 200 * 1e6, (t2 - t0) / 200 * 1e6))
