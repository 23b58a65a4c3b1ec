"""One LQUP of an N x N uniform matrix (for ncu launch lists). Development aid."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
p = 65521
torch.cuda.set_device(0)
A = torch.empty((N, N), dtype=torch.int32, device="cuda")
ff.ff_fill_uniform(A, N, N, N, p, 3, 0)
print(ff.lqup(p, A)[2])
