"""LQUP of an N x N uniform matrix, `reps` times (for ncu launch lists and the
FF_LQUP_TIMELINE / FF_LQUP_HOSTTIME traces: the last repetition is warm).
Development aid.   python scripts/run_lqup_once.py N [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = 65521
torch.cuda.set_device(0)
A0 = torch.empty((N, N), dtype=torch.int32, device="cuda")
ff.ff_fill_uniform(A0, N, N, N, p, 3, 0)
for _ in range(reps):
    A = A0.clone()
    r = ff.lqup(p, A)[2]
print(r)
