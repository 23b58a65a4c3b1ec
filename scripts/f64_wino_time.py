"""Time the fp64 engine classical vs delayed Winograd l = 1, 2, 3."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402

torch.cuda.set_device(0)
for (p, n) in [(65521, 4096), (65521, 8192)]:
    A = torch.empty((n, n), dtype=torch.int32, device="cuda")
    B = torch.empty((n, n), dtype=torch.int32, device="cuda")
    C = torch.zeros((n, n), dtype=torch.int32, device="cuda")
    ff.ff_fill_uniform(A, n, n, n, p, 1, 0)
    ff.ff_fill_uniform(B, n, n, n, p, 1, 1)
    ref = None
    for l in (0, 1, 2, 3):
        opts = {"scheme": 4, "winograd": l}
        for _ in range(2):
            ff.fgemm(p, A, B, C, 1, 0, opts=opts)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ff.fgemm(p, A, B, C, 1, 0, opts=opts)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        same = None
        if ref is None:
            ref = C.clone()
        else:
            same = bool(torch.equal(ref, C))
        t = min(ts)
        print("p=%d n=%d l=%d: %.2f ms  %.1f TFLOP/s-equivalent (2n^3)  identical-to-classical=%s" % (
            p, n, l, t, 2 * n ** 3 / t / 1e9, same), flush=True)
