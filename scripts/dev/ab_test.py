"""A/B timing of kernel variants with the SM clock sampled (NVML) during each
timed loop, so variants can be compared per clock cycle.  Development aid.

    python scripts/ab_test.py c4 '{"cta_group":1}' '{"cta_group":2}' ...
"""
import json
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_cs_0601133_b200 as ff  # noqa: E402
from paper_cs_0601133_b200.configs import CONFIGS  # noqa: E402

try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:  # pragma: no cover
    pynvml = None


class Sampler:
    def __init__(self):
        self.v, self.p, self.stop = [], [], False

    def run(self):
        while not self.stop:
            if pynvml:
                self.v.append(pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM))
                self.p.append(pynvml.nvmlDeviceGetPowerUsage(_h) / 1000.0)
            time.sleep(0.005)

    def __enter__(self):
        self.t = threading.Thread(target=self.run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop = True
        self.t.join()


def main():
    name = sys.argv[1]
    variants = [json.loads(s) for s in sys.argv[2:]] or [{}]
    reps = int(os.environ.get("REPS", "10"))
    rounds = int(os.environ.get("ROUNDS", "2"))
    cfg = CONFIGS[name]
    torch.cuda.set_device(0)
    A = torch.empty(cfg.a_shape, dtype=torch.int32, device="cuda")
    B = torch.empty(cfg.b_shape, dtype=torch.int32, device="cuda")
    C = torch.zeros((cfg.m, cfg.n), dtype=torch.int32, device="cuda")
    ff.ff_fill_uniform(A, *cfg.a_shape, cfg.a_shape[1], cfg.p, cfg.seed, 0)
    ff.ff_fill_uniform(B, *cfg.b_shape, cfg.b_shape[1], cfg.p, cfg.seed, 1)
    info = ff.ff_plan_query(cfg.p, cfg.k)
    ops = cfg.useful_ops() * (info["L"] if info["scheme"] == "CRT" else info["L"] ** 2)
    ref = None
    for rnd in range(rounds):
        for vi, opts in enumerate(variants):
            for _ in range(2):
                ff.fgemm(cfg.p, A, B, C, cfg.alpha, cfg.beta, cfg.transA, cfg.transB, opts=opts)
            torch.cuda.synchronize()
            if rnd == 0 and vi == 0:
                ref = C.clone()
            elif not torch.equal(ref, C) and cfg.beta % cfg.p == 0:
                print("MISMATCH between variants", opts, flush=True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with Sampler() as s:
                e0.record()
                for _ in range(reps):
                    ff.fgemm(cfg.p, A, B, C, cfg.alpha, cfg.beta, cfg.transA, cfg.transB, opts=opts)
                e1.record()
                torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / reps / 1e3
            mhz = sum(s.v) / len(s.v) if s.v else float("nan")
            pw = max(s.p) if s.p else float("nan")
            print("%s round %d %-40s t=%8.3f ms  %7.1f TOPS int8  clk %6.0f MHz  power<=%5.0f W  "
                  "ops/cycle/SM %7.0f (peak 16384)" % (
                      name, rnd, json.dumps(opts), t * 1e3, ops / t / 1e12, mhz, pw,
                      ops / t / (mhz * 1e6) / 148), flush=True)


if __name__ == "__main__":
    main()
