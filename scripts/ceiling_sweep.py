"""tcgen05 MMA-only ceiling at several durations, with nvidia-smi clocks (power-cap lag)."""
import os
import subprocess
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402

torch.cuda.set_device(0)
for iters in (20000, 200000, 2000000, 8000000):
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                            "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    t0 = time.time()
    tops = ff.ff_mma_ceiling(iters)
    dt = time.time() - t0
    time.sleep(0.1)
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    print("iters=%d  %.0f TOPS  wall %.2f s  smi: %s" % (iters, tops, dt, " | ".join(out[-12:])), flush=True)
