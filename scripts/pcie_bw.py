"""PCIe bandwidth of this box: H2D, D2H, and both at once (pinned). Development aid."""
import torch
torch.cuda.set_device(0)
n = 1 << 30  # 4 GiB of int32
h1 = torch.empty(n, dtype=torch.int32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.int32, pin_memory=True)
d1 = torch.empty(n, dtype=torch.int32, device="cuda")
d2 = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); f(); e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / 1e3
for _ in range(2):
    th = t(lambda: d1.copy_(h1, non_blocking=True))
    td = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    tb = t(both)
    print("H2D %.1f GB/s  D2H %.1f GB/s  both: %.1f ms for 4+4 GiB (%.1f GB/s each)" % (4*n/th/1e9, 4*n/td/1e9, tb*1e3, 4*n/tb/1e9))
