"""Sustained timing of one config on the default path with given ff_opts
(JSON) and steps; prints ms/step, median SM clock and power (nvidia-smi during
the timed region).  Development aid for power-cap-sensitive sweeps:
    python scripts/cfg_sustained.py c4 '{"kb_override": 2048}' 20"""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402

cfg = bench._load_configs()[sys.argv[1]]
opts = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {}
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
torch.cuda.set_device(0)
eng = bench.SingleGpu(ff, cfg, torch.device("cuda", 0))
if opts:
    ws = ff.ff_gemm_workspace_size(cfg.p, cfg.transA, cfg.transB, cfg.m, cfg.n, cfg.k, opts)
    eng.ws = torch.empty(max(1, ws), dtype=torch.uint8, device="cuda")
    eng.ws_bytes = ws

    def step():
        c = cfg
        ff.ff_gemm_ex(c.p, c.transA, c.transB, c.m, c.n, c.k, c.alpha, eng.A, eng.A.stride(0), eng.B,
                      eng.B.stride(0), c.beta, eng.C, eng.C.stride(0), opts, eng.ws, eng.ws_bytes)
else:
    step = eng.step
for _ in range(3):
    step()
torch.cuda.synchronize()
with bench.ClockSampler(0) as clk:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / steps
c = clk.summary()
print("%s %s env=%s  %.3f ms/step  %.1f TOPS useful  sm %s MHz  pw %s W  %s" % (
    cfg.name, json.dumps(opts), os.environ.get("FF_RASTER", "-"), ms, cfg.useful_ops() / ms / 1e9,
    c.get("sm_mhz"), c.get("power_w_max"), ",".join(c.get("reasons", []))), flush=True)
