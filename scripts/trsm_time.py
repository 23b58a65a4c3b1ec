"""ftrsm timing vs fgemm of the same size (the trsm/fgemm
ratio is 1/2 with omega = 3).  Development aid; CUDA events, device-resident."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0601133_b200 as ff  # noqa: E402


def t_ms(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    p = int(os.environ.get("P", 65521))
    torch.cuda.set_device(0)
    for N in [int(x) for x in (sys.argv[1:] or ["4096", "8192", "10000", "16384"])]:
        A = torch.empty((N, N), dtype=torch.int32, device="cuda")
        ff.ff_fill_uniform(A, N, N, N, p, 1, 0)
        A.diagonal().clamp_(min=1)            # nonzero diagonal (p prime: invertible)
        B0 = torch.empty((N, N), dtype=torch.int32, device="cuda")
        ff.ff_fill_uniform(B0, N, N, N, p, 1, 1)
        B = B0.clone()
        nbytes = ff.ff_trsm_workspace_size(p, "L", N, N)
        ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")

        def trsm():
            B.copy_(B0)
            ff.ff_trsm_ex(p, "L", "U", "N", "N", N, N, 1, A, N, B, N, None, ws, nbytes)
        copy_ms = t_ms(lambda: B.copy_(B0))
        ts = t_ms(trsm) - copy_ms
        C = torch.empty((N, N), dtype=torch.int32, device="cuda")
        tg = t_ms(lambda: ff.fgemm(p, A, B0, C))
        useful = float(N) ** 3            # m^2 n field multiply-adds x2 / 2 (classical trsm)
        print("p=%d N=%d  ftrsm %.3f ms (%.1f TOPS, N^3/t)  fgemm %.3f ms  ratio %.3f" % (
            p, N, ts, useful / ts / 1e9, tg, ts / tg), flush=True)
        del A, B, B0, C, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
