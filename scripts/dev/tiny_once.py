import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_cs_0601133_b200 as ff
p = 65521
torch.cuda.set_device(0)
m, n, k = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (128, 128, 128)
X = torch.randint(0, p, (m, k), dtype=torch.int32, device="cuda")
Y = torch.randint(0, p, (k, n), dtype=torch.int32, device="cuda")
C = torch.randint(0, p, (m, n), dtype=torch.int32, device="cuda")
for _ in range(3):
    ff.fgemm(p, X, Y, C, p - 1, 1)
torch.cuda.synchronize()
