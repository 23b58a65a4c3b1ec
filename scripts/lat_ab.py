"""A/B timing of the small-field paths: tcgen05 latency kernel (small_path 2), mma.sync
kernels (1), encoder + tcgen05 GEMM (-1), default (0).  Development aid."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402

torch.cuda.set_device(0)
p = 65521
flush = torch.empty(64 * 2 ** 20, dtype=torch.int32, device="cuda")
for (m, n, k) in [(512, 512, 512), (128, 128, 128), (128, 8192, 128), (128, 8192, 1024), (1024, 1024, 1024),
                  (4096, 4096, 128), (2048, 2048, 512), (256, 256, 4096), (8192, 128, 128)]:
    A = torch.randint(0, p, (m, k), dtype=torch.int32, device="cuda")
    B = torch.randint(0, p, (k, n), dtype=torch.int32, device="cuda")
    C = torch.randint(0, p, (m, n), dtype=torch.int32, device="cuda")
    res = []
    for mode in (2, 1, -1, 0):
        o = {"small_path": mode}
        for _ in range(3):
            ff.fgemm(p, A, B, C, p - 1, 1, opts=o)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ff.fgemm(p, A, B, C, p - 1, 1, opts=o)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        res.append("%s %.1f" % (mode, 1e3 * ts[len(ts) // 2]))
    print("%5d x %5d x %5d   us (median): %s" % (m, n, k, "   ".join(res)), flush=True)
