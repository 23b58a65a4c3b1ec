"""Row-panel data parallelism over the GPUs of one box.

Rank r owns rows [row0_r, row1_r) of op(A) and of C; B (k x n) starts on rank
0 only.  One fgemm step is:

  rank 0, comm stream:   for each column chunk j of op(B):
                           ff_encode(B[:, chunk j]) -> limb planes Bl[j]  (int8, [L][n_j][k_pad])
                           NCCL broadcast Bl[j] from rank 0          (the only exchange step)
  every rank, compute:   ff_encode(A panel) -> Al                    (overlaps broadcast of chunk 0)
                           for each chunk j: wait Bl[j];  ff_gemm_limbs(Al, Bl[j]) -> C[:, chunk j]

Broadcasting the *encoded* limbs, not int32, moves L bytes per element instead
of 4 (c3: 128 MiB instead of 512).  k is never split, so no reduction
collective is needed.  The paper has no parallel algorithm (PAPER.md l.883,
"parallel library ... sequential-first" is future work); this is our design.

All arithmetic runs in the CUDA library; torch provides memory, streams and the
NCCL process group.  For CPU tests the per-chunk kernels can be swapped for
injected callables (``backend=``) so the partition / chunk / broadcast logic is
exercised with gloo.
"""
from __future__ import annotations

from dataclasses import dataclass


def panel_bounds(m: int, world: int, rank: int, align: int = 128) -> tuple[int, int]:
    """Rows of op(A)/C owned by `rank`: contiguous, balanced in units of `align`
    rows (the GEMM tile height), covering [0, m) exactly once across ranks."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    units = (m + align - 1) // align
    lo_u = units * rank // world
    hi_u = units * (rank + 1) // world
    return min(m, lo_u * align), min(m, hi_u * align)


def chunk_bounds(n: int, chunks: int, align: int = 256) -> list[tuple[int, int]]:
    """Column chunks of op(B) (multiples of the 256-wide tile except the last)."""
    units = (n + align - 1) // align
    chunks = max(1, min(chunks, units))
    out = []
    for j in range(chunks):
        a = min(n, units * j // chunks * align)
        b = min(n, units * (j + 1) // chunks * align)
        if b > a:
            out.append((a, b))
    return out


@dataclass
class Problem:
    p: int
    m: int
    n: int
    k: int
    transA: str = "N"
    transB: str = "N"
    alpha: int = 1
    beta: int = 0


class RowPanelGemm:
    """One rank's share of a row-panel-sharded fgemm (see module docstring)."""

    def __init__(self, prob: Problem, group=None, chunks: int = 4, opts=None, device=None,
                 backend=None, world: int | None = None, rank: int | None = None):
        """`world`/`rank` override the process group's ("virtual ranks" on one GPU
        for testing: no broadcast is issued, the caller fills non-zero ranks' B limbs)."""
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.prob = prob
        self.group = group
        self.virtual = world is not None
        self.world = world if world is not None else (dist.get_world_size(group) if dist.is_initialized() else 1)
        self.rank = rank if rank is not None else (dist.get_rank(group) if dist.is_initialized() else 0)
        self.row0, self.row1 = panel_bounds(prob.m, self.world, self.rank)
        self.mr = self.row1 - self.row0
        self.chunks = chunk_bounds(prob.n, chunks if self.world > 1 else 1)
        self.opts = opts
        if backend is None:
            from . import ffgemm as backend
        self.be = backend
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        info = backend.ff_plan_query(prob.p, prob.k, opts)
        self.L, self.k_pad = info["L"], info["k_pad"]
        self.Al = torch.empty((self.L, max(self.mr, 1), self.k_pad), dtype=torch.int8, device=self.device)
        self.Bl = [torch.empty((self.L, b - a, self.k_pad), dtype=torch.int8, device=self.device)
                   for a, b in self.chunks]
        is_cuda = self.device.type == "cuda"
        self.comm_stream = torch.cuda.Stream(self.device) if is_cuda else None
        self.launches_per_step = 0
        self.gemm_events = []

    # --------------------------------------------------------------- helpers
    def a_panel_view(self, A):
        """This rank's rows of op(A) as a view of the stored A (any rank may hold full A)."""
        if self.prob.transA in "Nn":
            return A[self.row0:self.row1, :]
        return A[:, self.row0:self.row1]

    def step(self, A_panel, B, C_panel, time_gemm: bool = False):
        """Run one sharded fgemm step.  A_panel: this rank's stored rows of A
        (transA=N: mr x k, ld = A_panel.stride(0); transA=T: k x mr view);
        B: stored B on rank 0 (ignored elsewhere); C_panel: mr x n, updated in place."""
        torch, pr = self.torch, self.prob
        cur = torch.cuda.current_stream(self.device) if self.comm_stream is not None else None
        launches = 0
        works = []
        # B: encode + broadcast each chunk on the comm stream (rank 0 encodes).
        ctx = torch.cuda.stream(self.comm_stream) if self.comm_stream is not None else _null()
        if self.comm_stream is not None:
            self.comm_stream.wait_stream(cur)
        with ctx:
            for (n0, n1), bl in zip(self.chunks, self.Bl):
                if self.rank == 0:
                    if pr.transB in "Nn":       # stored k x n: chunk = columns n0..n1, transposed read
                        src, kmaj, ldx = B[:, n0:n1], 0, B.stride(0)
                    else:                        # stored n x k: chunk = rows n0..n1, K-major already
                        src, kmaj, ldx = B[n0:n1, :], 1, B.stride(0)
                    self.be.ff_encode(pr.p, pr.k, self.opts, kmaj, n1 - n0, src, ldx, bl,
                                      stream=self.comm_stream)
                    launches += 1
                if self.world > 1 and not self.virtual:
                    works.append(self.dist.broadcast(bl, src=0, group=self.group, async_op=True))
                else:
                    works.append(None)
        # A panel: encode on the compute stream (overlaps the first broadcast).
        if self.mr > 0:
            kmaj = 1 if pr.transA in "Nn" else 0
            self.be.ff_encode(pr.p, pr.k, self.opts, kmaj, self.mr, A_panel, max(1, A_panel.stride(0)),
                              self.Al, stream=cur)
            launches += 1
        evs = []
        for (n0, n1), bl, w in zip(self.chunks, self.Bl, works):
            if w is not None:
                w.wait()                         # compute stream waits for this chunk's broadcast
            elif self.comm_stream is not None:
                cur.wait_stream(self.comm_stream)
            if self.mr == 0:
                continue
            if time_gemm and cur is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(cur)
            self.be.ff_gemm_limbs(pr.p, self.mr, n1 - n0, pr.k, self.opts, pr.alpha, self.Al, bl,
                                  pr.beta, C_panel[:, n0:n1], max(1, C_panel.stride(0)), stream=cur)
            launches += 1
            if time_gemm and cur is not None:
                e1.record(cur)
                evs.append((e0, e1))
        self.launches_per_step = launches
        self.gemm_events = evs
        return C_panel

    def gemm_ms(self) -> float:
        """Device time of this step's GEMM launches (after synchronisation)."""
        return sum(e0.elapsed_time(e1) for e0, e1 in self.gemm_events)


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
