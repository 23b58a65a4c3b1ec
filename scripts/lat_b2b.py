"""Back-to-back latency-kernel calls (no kernels in between) vs interleaved with a fill."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402

torch.cuda.set_device(0)
p = 65521
flush = torch.empty(64 * 2 ** 20, dtype=torch.int32, device="cuda")
for (m, n, k) in [(128, 128, 128), (512, 512, 512)]:
    A = torch.randint(0, p, (m, k), dtype=torch.int32, device="cuda")
    B = torch.randint(0, p, (k, n), dtype=torch.int32, device="cuda")
    C = torch.randint(0, p, (m, n), dtype=torch.int32, device="cuda")
    for mode in (2, 1):
        o = {"small_path": mode}
        for _ in range(3):
            ff.fgemm(p, A, B, C, p - 1, 1, opts=o)
        torch.cuda.synchronize()
        # back to back: the host enqueues 200 calls, the GPU runs them without gaps once queued
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ff.fgemm(p, A, B, C, p - 1, 1, opts=o)
            g.capture_begin()
            for _ in range(50):
                ff.fgemm(p, A, B, C, p - 1, 1, opts=o)
            g.capture_end()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        print("%dx%dx%d mode %d: graph of 50 back-to-back calls: %.2f us per call" % (
            m, n, k, mode, 1e3 * e0.elapsed_time(e1) / 50), flush=True)
