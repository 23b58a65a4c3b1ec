"""Run small fgemm shapes once per mode (for ncu launch lists).  Development aid."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402

torch.cuda.set_device(0)
p = 65521
for (m, n, k) in [(128, 128, 128), (512, 512, 512), (128, 8192, 1024)]:
    A = torch.randint(0, p, (m, k), dtype=torch.int32, device="cuda")
    B = torch.randint(0, p, (k, n), dtype=torch.int32, device="cuda")
    C = torch.randint(0, p, (m, n), dtype=torch.int32, device="cuda")
    for mode in (2, 1):
        for _ in range(2):
            ff.fgemm(p, A, B, C, p - 1, 1, opts={"small_path": mode})
torch.cuda.synchronize()
print("ok")
