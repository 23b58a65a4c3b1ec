"""LQUP timing vs fgemm of the same size (Sec. 5.3: classical ratio
1/3).  Development aid; CUDA events on device-resident inputs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0601133_b200 as ff  # noqa: E402

p = int(os.environ.get("P", 65521))
torch.cuda.set_device(0)
for N in [int(x) for x in (sys.argv[1:] or ["2048", "4096", "8192", "10000"])]:
    A0 = torch.empty((N, N), dtype=torch.int32, device="cuda")
    ff.ff_fill_uniform(A0, N, N, N, p, 3, 0)
    A = A0.clone()
    ff.lqup(p, A)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        A.copy_(A0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, _, r = ff.lqup(p, A)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    C = torch.empty_like(A0)
    ff.fgemm(p, A0, A0, C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ff.fgemm(p, A0, A0, C); e1.record(); torch.cuda.synchronize()
    tg = e0.elapsed_time(e1)
    print("p=%d N=%d rank=%d  lqup %.2f ms  fgemm %.3f ms  ratio %.2f  (2/3 N^3 / t = %.1f TOPS)" % (
        p, N, r, best * 1e3, tg, best * 1e3 / tg, 2 * N ** 3 / 3 / best / 1e12), flush=True)
    del A, A0, C
    torch.cuda.empty_cache()
