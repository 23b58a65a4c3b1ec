"""Host-side cost of one c1 call (development aid): wall time per ff_gemm_ex over
many back-to-back calls (host-bound if above the kernel time), and its parts."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_cs_0601133_b200 as ff  # noqa: E402
from paper_cs_0601133_b200 import ffgemm as b  # noqa: E402

cfg = bench._load_configs()[sys.argv[1] if len(sys.argv) > 1 else "c1"]
torch.cuda.set_device(0)
eng = bench.SingleGpu(ff, cfg, torch.device("cuda", 0))
N = 2000
for _ in range(50):
    eng.step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(N):
    eng.step()
t_enq = (time.perf_counter() - t) / N
torch.cuda.synchronize()
t_all = (time.perf_counter() - t) / N
t = time.perf_counter()
for _ in range(N):
    torch.cuda.current_stream().cuda_stream
t_stream = (time.perf_counter() - t) / N
A, B, C = eng.A, eng.B, eng.C
t = time.perf_counter()
for _ in range(N):
    A.data_ptr(); B.data_ptr(); C.data_ptr()
t_ptr = (time.perf_counter() - t) / N
print("%s: enqueue %.2f us/call, with sync %.2f us/call; current_stream %.2f us; 3x data_ptr %.2f us" % (
    cfg.name, t_enq * 1e6, t_all * 1e6, t_stream * 1e6, t_ptr * 1e6))
import torch as _t  # noqa: E402
t = time.perf_counter()
for _ in range(N):
    _t._C._cuda_getCurrentRawStream(_t._C._cuda_getDevice())
print("raw stream accessor %.2f us; matches current_stream: %s" % (
    (time.perf_counter() - t) / N * 1e6,
    _t._C._cuda_getCurrentRawStream(_t._C._cuda_getDevice()) == _t.cuda.current_stream().cuda_stream))
s2 = _t.cuda.Stream()
with _t.cuda.stream(s2):
    print("inside a stream context: %s" % (b._stream(None) == s2.cuda_stream))
