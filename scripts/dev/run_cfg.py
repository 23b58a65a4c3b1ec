"""Run fgemm once on a config with default options (for ncu launch lists). Development aid."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402
from paper_cs_0601133_b200.configs import CONFIGS  # noqa: E402
cfg = CONFIGS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
torch.cuda.set_device(0)
A = torch.empty(cfg.a_shape, dtype=torch.int32, device="cuda")
B = torch.empty(cfg.b_shape, dtype=torch.int32, device="cuda")
C = torch.zeros((cfg.m, cfg.n), dtype=torch.int32, device="cuda")
ff.ff_fill_uniform(A, *cfg.a_shape, cfg.a_shape[1], cfg.p, cfg.seed, 0)
ff.ff_fill_uniform(B, *cfg.b_shape, cfg.b_shape[1], cfg.p, cfg.seed, 1)
if cfg.beta:
    ff.ff_fill_uniform(C, cfg.m, cfg.n, cfg.n, cfg.p, cfg.seed, 2)
for _ in range(reps):
    ff.fgemm(cfg.p, A, B, C, cfg.alpha, cfg.beta, cfg.transA, cfg.transB)
torch.cuda.synchronize()
print("ok")
