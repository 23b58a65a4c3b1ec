"""Row-panel data parallelism over the GPUs of one box.

Rank r owns rows [row0_r, row1_r) of op(A) and of C; B (k x n) starts on rank
0 only.  k is never split, so no reduction collective is needed: the one
exchange step is the broadcast of B, done one of two ways (``mode``):

* ``"planes"`` -- when the plan's int8 planes per element are fewer than 4
  (limb schemes with L <= 3: c1-c4), rank 0 encodes B once and broadcasts the
  ENCODED planes, L bytes per element instead of 4 (c3: 128 MiB instead of
  512):

    rank 0, comm stream:  for each column chunk j of op(B):
                            ff_encode(B[:, chunk j]) -> Bl[j]   (int8, [L][n_j][k_pad])
                            NCCL broadcast Bl[j] from rank 0
    every rank, compute:  ff_encode(A panel) -> Al              (overlaps chunk 0)
                          for each chunk j: wait Bl[j]; ff_gemm_limbs(Al, Bl[j]) -> C[:, chunk j]

* ``"int32"`` -- when planes >= 4 (c5: CRT with 9 moduli, or 4 limbs), the
  int32 matrix is the smaller payload, so rank 0 broadcasts int32 chunks of B
  and every rank encodes what it receives itself ("encoding may
  be done per rank").  If the library would multiply the rank's panel with a
  Winograd level (ff_gemm_winograd_levels: the measured rule of DESIGN.md §7,
  e.g. c5 at 2 GPUs), the rank waits for all of B and runs ONE ff_gemm_ex on
  its panel -- the local one-level Winograd of §8(e); otherwise chunk j is
  encoded and multiplied as soon as it lands (broadcast overlapped with
  compute).

All arithmetic runs in the CUDA library; torch provides memory, streams and the
NCCL process group.  For CPU tests the per-chunk kernels can be swapped for
injected callables (``backend=``) so the partition / chunk / broadcast logic is
exercised with gloo.  The paper has no parallel algorithm;
this is our design.
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


def choose_mode(planes: int) -> str:
    """Broadcast encoded planes only when they are smaller than the int32 matrix."""
    return "planes" if planes < 4 else "int32"


class RowPanelGemm:
    """One rank's share of a row-panel-sharded fgemm (see module docstring)."""

    def __init__(self, prob: Problem, group=None, chunks: int = 4, opts=None, device=None,
                 backend=None, world: int | None = None, rank: int | None = None, mode: str = "auto"):
        """`world`/`rank` override the process group's ("virtual ranks" on one GPU
        for testing: no broadcast is issued, the caller copies rank 0's broadcast
        buffers (``bcast_buffers()``) to the others)."""
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
        self.opts = opts
        if backend is None:
            from . import ffgemm as backend
        self.be = backend
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        info = backend.ff_plan_query(prob.p, prob.k, opts)
        self.L, self.k_pad = info["L"], info["k_pad"]
        self.mode = choose_mode(self.L) if mode == "auto" else mode
        if self.mode not in ("planes", "int32"):
            raise ValueError("mode must be auto, planes or int32")
        # int32 mode: one call on the whole panel when the library would use Winograd
        # there -- decided on rank 0's panel so that every rank chunks the broadcast alike
        r0a, r0b = panel_bounds(prob.m, self.world, 0)
        self.whole = (self.mode == "int32" and r0b > r0a and
                      backend.ff_gemm_winograd_levels(prob.p, r0b - r0a, prob.n, prob.k, opts) > 0)
        dev = self.device
        if self.mode == "planes":
            self.chunks = chunk_bounds(prob.n, chunks if self.world > 1 else 1)
            self.Al = torch.empty((self.L, max(self.mr, 1), self.k_pad), dtype=torch.int8, device=dev)
            self.Bl = [torch.empty((self.L, b - a, self.k_pad), dtype=torch.int8, device=dev)
                       for a, b in self.chunks]
        elif self.whole:
            # all of B, received in row chunks of the STORED array (contiguous)
            rows = prob.k if prob.transB in "Nn" else prob.n
            self.chunks = chunk_bounds(rows, chunks if self.world > 1 else 1, align=1)
            self.Bfull = torch.empty((prob.k, prob.n) if prob.transB in "Nn" else (prob.n, prob.k),
                                     dtype=torch.int32, device=dev)
        else:
            # int32 column chunks of op(B), K-major (n_j x k) so every chunk is contiguous
            self.chunks = chunk_bounds(prob.n, chunks if self.world > 1 else 1)
            self.Bi = [torch.empty((b - a, prob.k), dtype=torch.int32, device=dev) for a, b in self.chunks]
            self.Al = torch.empty((self.L, max(self.mr, 1), self.k_pad), dtype=torch.int8, device=dev)
            wmax = max(b - a for a, b in self.chunks)
            self.Bl1 = torch.empty((self.L, wmax, self.k_pad), dtype=torch.int8, device=dev)
        is_cuda = dev.type == "cuda"
        self.comm_stream = torch.cuda.Stream(dev) if is_cuda else None
        self.launches_per_step = 0
        self.gemm_events = []

    # --------------------------------------------------------------- helpers
    def a_panel_view(self, A):
        """This rank's rows of op(A) as a view of the stored A (any rank may hold full A)."""
        if self.prob.transA in "Nn":
            return A[self.row0:self.row1, :]
        return A[:, self.row0:self.row1]

    def bcast_buffers(self):
        """The tensors the broadcast fills, in chunk order (rank 0's are the source)."""
        if self.mode == "planes":
            return list(self.Bl)
        if self.whole:
            return [self.Bfull[a:b] for a, b in self.chunks]
        return list(self.Bi)

    def _bcast(self, buf):
        if self.world > 1 and not self.virtual:
            return self.dist.broadcast(buf, group=self.group, group_src=0, async_op=True)
        return None

    def step(self, A_panel, B, C_panel, time_gemm: bool = False):
        """Run one sharded fgemm step.  A_panel: this rank's stored rows of A
        (transA=N: mr x k, ld = A_panel.stride(0); transA=T: k x mr view);
        B: stored B on rank 0 (ignored elsewhere); C_panel: mr x n, updated in place."""
        torch, pr = self.torch, self.prob
        cur = torch.cuda.current_stream(self.device) if self.comm_stream is not None else None
        launches = 0
        works = []
        ctx = torch.cuda.stream(self.comm_stream) if self.comm_stream is not None else _null()
        if self.comm_stream is not None:
            self.comm_stream.wait_stream(cur)
        # ---- B: produce (rank 0) and broadcast each chunk on the comm stream
        with ctx:
            for (n0, n1), buf in zip(self.chunks, self.bcast_buffers()):
                if self.rank == 0:
                    if self.mode == "planes":
                        if pr.transB in "Nn":       # stored k x n: chunk = columns n0..n1, transposed read
                            src, kmaj, ldx = B[:, n0:n1], 0, B.stride(0)
                        else:                        # stored n x k: chunk = rows n0..n1, K-major already
                            src, kmaj, ldx = B[n0:n1, :], 1, B.stride(0)
                        self.be.ff_encode(pr.p, pr.k, self.opts, kmaj, n1 - n0, src, ldx, buf,
                                          stream=self.comm_stream)
                        launches += 1
                    elif self.whole:
                        buf.copy_(B[n0:n1])          # row chunk of the stored B
                    else:                            # K-major int32 chunk (n_j x k)
                        buf.copy_(B[:, n0:n1].t() if pr.transB in "Nn" else B[n0:n1, :])
                works.append(self._bcast(buf))
        # ---- A panel: encode on the compute stream (overlaps the first broadcast)
        if self.mode in ("planes", "int32") and not self.whole and self.mr > 0:
            kmaj = 1 if pr.transA in "Nn" else 0
            self.be.ff_encode(pr.p, pr.k, self.opts, kmaj, self.mr, A_panel, max(1, A_panel.stride(0)),
                              self.Al, stream=cur)
            launches += 1
        evs = []

        def wait(w):
            if w is not None:
                w.wait()                         # compute stream waits for this chunk's broadcast
            elif self.comm_stream is not None:
                cur.wait_stream(self.comm_stream)

        def timed(fn):
            if time_gemm and cur is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(cur)
                fn()
                e1.record(cur)
                evs.append((e0, e1))
            else:
                fn()

        if self.whole:
            for w in works:
                wait(w)
            if self.mr > 0:
                Bf = self.Bfull
                timed(lambda: self.be.ff_gemm_ex(pr.p, pr.transA, pr.transB, self.mr, pr.n, pr.k, pr.alpha,
                                                 A_panel, max(1, A_panel.stride(0)), Bf, Bf.stride(0), pr.beta,
                                                 C_panel, max(1, C_panel.stride(0)), self.opts, None, 0, cur))
                launches += 1
        else:
            for j, ((n0, n1), w) in enumerate(zip(self.chunks, works)):
                wait(w)
                if self.mr == 0:
                    continue
                if self.mode == "planes":
                    bl = self.Bl[j]
                else:   # the chunk's planes [L][n_j][k_pad], packed at the front of the buffer
                    bl = self.Bl1.view(-1)[:self.L * (n1 - n0) * self.k_pad].view(self.L, n1 - n0, self.k_pad)
                    self.be.ff_encode(pr.p, pr.k, self.opts, 1, n1 - n0, self.Bi[j], pr.k, bl, stream=cur)
                    launches += 1
                timed(lambda: self.be.ff_gemm_limbs(pr.p, self.mr, n1 - n0, pr.k, self.opts, pr.alpha, self.Al, bl,
                                                    pr.beta, C_panel[:, n0:n1], max(1, C_panel.stride(0)),
                                                    stream=cur))
                launches += 1
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
