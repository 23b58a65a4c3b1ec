"""Time the LQUP U_rest GEMM shape in isolation: (128 x 128) x (128 x N) with B a
row block of an n x n matrix (ld = n), in place (C = B).  Development aid."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_cs_0601133_b200 as ff  # noqa: E402

p = 65521
torch.cuda.set_device(0)
n = 8192
M = torch.randint(0, p, (n, n), dtype=torch.int32, device="cuda")
L = torch.randint(0, p, (128, 128), dtype=torch.int32, device="cuda")
for N in [4096, 8064]:
    Ar = M[1024:1152, n - N:]
    for inplace in [True, False]:
        C = Ar if inplace else torch.empty((128, N), dtype=torch.int32, device="cuda")
        for _ in range(3):
            ff.ff_gemm_ex(p, "N", "N", 128, N, 128, 1, L, 128, Ar, n, 0, C, n if inplace else N)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ff.ff_gemm_ex(p, "N", "N", 128, N, 128, 1, L, 128, Ar, n, 0, C, n if inplace else N)
        e1.record()
        torch.cuda.synchronize()
        print("N=%d inplace=%d: %.1f us" % (N, inplace, e0.elapsed_time(e1) / 10 * 1e3), flush=True)
