#!/bin/bash
# round-2 baseline: per-config timing + launch lists of c3 and c5 + torch._int_mm ceiling
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2b_smi.txt
timeout 600 python scripts/quick_time.py c1 c2 c3 c4 c5 > gpurun_out/r2b_times.txt 2>&1
timeout 300 python - > gpurun_out/r2b_intmm.txt 2>&1 <<'PY'
import torch
a = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device="cuda").t()
for _ in range(3): torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); torch._int_mm(a, b); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print("torch._int_mm 8192^3: %.3f ms = %.1f TOPS" % (best, 2 * 8192**3 / best / 1e9))
PY
for c in c3 c5 c1; do bash scripts/launch_list.sh $c '{}' r2b_$c > gpurun_out/r2b_ll_$c.txt 2>&1; done
