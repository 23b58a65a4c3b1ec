"""One ftrsm (L, U, N, N) of size N x N over Z/pZ, for ncu launch lists. Development aid."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = int(os.environ.get("P", 65521))
torch.cuda.set_device(0)
A = torch.empty((N, N), dtype=torch.int32, device="cuda")
ff.ff_fill_uniform(A, N, N, N, p, 1, 0)
A.diagonal().clamp_(min=1)
B = torch.empty((N, N), dtype=torch.int32, device="cuda")
ff.ff_fill_uniform(B, N, N, N, p, 1, 1)
ff.ftrsm(p, A, B)
torch.cuda.synchronize()
print("ok")
