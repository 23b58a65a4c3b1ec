"""c1 latency kernel: phase timestamps (FF_TRACE=1) with a cold and a warm L2.  Development aid."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FF_TRACE"] = "1"
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402

torch.cuda.set_device(0)
p = 65521
flush = torch.empty(64 * 2 ** 20, dtype=torch.int32, device="cuda")
for (m, n, k) in [(512, 512, 512)]:
    A = torch.randint(0, p, (m, k), dtype=torch.int32, device="cuda")
    B = torch.randint(0, p, (k, n), dtype=torch.int32, device="cuda")
    C = torch.zeros((m, n), dtype=torch.int32, device="cuda")
    for cold in (True, False, True, False):
        if cold:
            flush.fill_(1)
        torch.cuda.synchronize()
        print("cold" if cold else "warm", flush=True)
        ff.fgemm(p, A, B, C, 1, 0)
        torch.cuda.synchronize()
