"""Row-panel sharding (paper_cs_0601133_b200/sharded.py) on CPU with gloo,
world_size 2: partitioning, B-chunk encode/broadcast ordering and the per-chunk
output placement.  The GPU kernels are replaced by a CPU stand-in backend whose
"limbs" are the 4 bytes of each residue and whose GEMM is the oracle, so any
mis-sliced panel, mis-ordered chunk or corrupted broadcast shows up as a
mismatch against the oracle's full product.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_cs_0601133_b200.sharded import Problem, RowPanelGemm, chunk_bounds, panel_bounds


def test_panel_bounds_cover_exactly_once():
    for m in (1, 127, 128, 129, 1000, 32768):
        for world in (1, 2, 3, 4, 8):
            spans = [panel_bounds(m, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == m
            for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                assert a1 == b0 and a0 <= a1
            for a0, a1 in spans:
                assert a0 % 128 == 0
    assert panel_bounds(32768, 8, 3) == (12288, 16384)   # c4 at 8 GPUs: 4096-row panels


def test_chunk_bounds():
    for n in (1, 255, 256, 700, 32768):
        for c in (1, 2, 4, 8):
            ch = chunk_bounds(n, c)
            assert ch[0][0] == 0 and ch[-1][1] == n
            assert all(b0 == a1 for (_, a1), (b0, _) in zip(ch, ch[1:]))
            assert all(a % 256 == 0 for a, _ in ch)
    assert chunk_bounds(32768, 4) == [(0, 8192), (8192, 16384), (16384, 24576), (24576, 32768)]


class ByteBackend:
    """CPU stand-in for the CUDA library with the same call signatures.
    ``wino`` is what ff_gemm_winograd_levels reports (1: the rank multiplies
    its whole panel with one ff_gemm_ex call)."""

    def __init__(self, wino=0):
        self.calls = []
        self.wino = wino

    def ff_gemm_winograd_levels(self, p, m, n, k, opts=None):
        return self.wino

    def ff_gemm_ex(self, p, tA, tB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, opts=None,
                   workspace=None, workspace_bytes=0, stream=None):
        self.calls.append(("gemm_ex", m, n))
        a = A.numpy() if tA in "Nn" else A.numpy()
        out = oracle.fgemm(p, tA, tB, alpha, np.ascontiguousarray(a), np.ascontiguousarray(B.numpy()), beta,
                           np.ascontiguousarray(C[:m, :n].numpy()), m=m, n=n, k=k)
        C[:m, :n].copy_(torch.from_numpy(out))

    def ff_plan_query(self, p, k, opts=None):
        return {"L": 4, "k_pad": (k + 15) // 16 * 16}

    def ff_encode(self, p, k, opts, kmajor_src, rows, X, ldx, limbs, stream=None):
        self.calls.append(("encode", rows))
        x = X[:rows, :k] if kmajor_src else X[:k, :rows].t()
        r = torch.remainder(x.to(torch.int64), p).to(torch.int32)
        b = r.contiguous().view(torch.uint8).view(rows, k, 4).permute(2, 0, 1)
        limbs.zero_()
        limbs[:, :, :k] = b.view(torch.int8)

    def ff_gemm_limbs(self, p, m, n, k, opts, alpha, Al, Bl, beta, C, ldc, stream=None):
        self.calls.append(("gemm", m, n))
        a = Al[:, :m, :k].contiguous().view(torch.uint8).permute(1, 2, 0).contiguous().view(torch.int32)
        b = Bl[:, :n, :k].contiguous().view(torch.uint8).permute(1, 2, 0).contiguous().view(torch.int32)
        A = a.view(m, k).numpy()
        Bt = b.view(n, k).numpy()
        Cv = C[:m, :n]
        out = oracle.fgemm(p, "N", "T", alpha, A, Bt, beta, np.ascontiguousarray(Cv.numpy()))
        Cv.copy_(torch.from_numpy(out))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASES = [
    # encoded planes broadcast (forced: the stand-in has 4 planes per element)
    (65521, 300, 700, 257, "N", "N", 1, 0, 3, "planes", 0),
    (67108859, 257, 520, 100, "T", "N", 67108858, 1, 2, "planes", 0),
    (251, 129, 300, 64, "N", "T", 3, 2, 4, "planes", 0),
    # int32 broadcast, per-rank encode of every chunk (auto: 4 planes >= 4 bytes)
    (67108859, 257, 520, 100, "T", "N", 67108858, 1, 3, "auto", 0),
    (8388593, 300, 700, 257, "N", "T", 5, 7, 2, "auto", 0),
    # int32 broadcast of all of B, one call per panel (the library would use Winograd)
    (67108859, 300, 520, 129, "N", "N", 67108858, 1, 3, "auto", 1),
    (251, 257, 300, 64, "T", "T", 3, 2, 2, "auto", 1),
    # a rank with no rows (m smaller than one 128-row unit per rank)
    (65521, 100, 300, 40, "N", "N", 1, 0, 2, "auto", 0),
]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for ci, case in enumerate(CASES):
            p, m, n, k, tA, tB, alpha, beta, chunks, mode, wino = case
            rng = np.random.default_rng(123 + ci)
            A = rng.integers(0, p, size=(m, k) if tA == "N" else (k, m), dtype=np.int64).astype(np.int32)
            B = rng.integers(0, p, size=(k, n) if tB == "N" else (n, k), dtype=np.int64).astype(np.int32)
            C = rng.integers(0, p, size=(m, n), dtype=np.int64).astype(np.int32)
            be = ByteBackend(wino)
            eng = RowPanelGemm(Problem(p, m, n, k, tA, tB, alpha, beta), chunks=chunks,
                               device=torch.device("cpu"), backend=be, mode=mode)
            At = torch.from_numpy(A)
            Ap = eng.a_panel_view(At)
            Bt = torch.from_numpy(B) if rank == 0 else None      # B lives on rank 0 only
            Cp = torch.from_numpy(C[eng.row0:eng.row1].copy())
            eng.step(Ap, Bt, Cp)
            want = oracle.fgemm(p, tA, tB, alpha, A, B, beta, C)[eng.row0:eng.row1]
            ok = np.array_equal(Cp.numpy(), want)
            n_enc = sum(1 for c in be.calls if c[0] == "encode")
            n_ex = sum(1 for c in be.calls if c[0] == "gemm_ex")
            q.put((ci, rank, ok, eng.row0, eng.row1, len(eng.chunks), n_enc, n_ex, eng.mode, eng.whole))
    finally:
        dist.destroy_process_group()


def test_row_panel_world2_gloo():
    """All CASES in one pair of gloo processes (spawn + torch import once)."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world * len(CASES))]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for ci, case in enumerate(CASES):
        rr = sorted(r[1:] for r in res if r[0] == ci)
        m = case[1]
        assert rr[0][2] == 0 and rr[-1][3] == m and rr[0][3] == rr[1][2], case
        assert rr[0][4] == rr[1][4] and rr[0][8] == rr[1][8], case      # same chunking / mode on both ranks
        for rank, ok, r0, r1, nchunks, n_enc, n_ex, mode, whole in rr:
            assert ok, (case, rank, r0, r1)
            has_rows = r1 > r0
            if mode == "planes":
                # only rank 0 encodes B (one encode per chunk); the others receive planes
                assert n_enc == (nchunks if rank == 0 else 0) + (1 if has_rows else 0) and n_ex == 0, case
            elif not whole:
                # int32 chunks: every rank encodes its A panel and each chunk it receives
                assert mode == "int32" and n_ex == 0, case
                assert n_enc == ((1 + nchunks) if has_rows else 0), case
            else:
                assert mode == "int32" and n_enc == 0 and n_ex == (1 if has_rows else 0), case
