"""Thin Python binding of the C ABI in include/ffgemm.h (ctypes).

Argument marshalling only: every step of the path runs in the CUDA library
``lib/libffgemm.so``.  If that library is missing this module raises at import
(there is no CPU fallback of any kind).  Functions keep the C names; the
``fgemm`` convenience wrapper derives m, n, k and the leading dimensions from
torch tensors and launches on torch's current stream.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libffgemm.so")
# development A/B runs only: load another build of the same library (same ABI)
if os.environ.get("FF_LIB_OVERRIDE"):
    LIB_PATH = os.environ["FF_LIB_OVERRIDE"]

if not os.path.exists(LIB_PATH):
    raise ImportError(
        "paper_cs_0601133_b200: CUDA library %s is missing; build it with "
        "`python paper_cs_0601133_b200/build.py` (there is no CPU fallback)" % LIB_PATH)

_lib = ctypes.CDLL(LIB_PATH)

FF_OK, FF_ERR_CUDA, FF_ERR_NOMEM, FF_ERR_ARCH, FF_ERR_OPTS, FF_ERR_INTERNAL = 0, 1, 2, 3, 4, 5
FF_SCHEME_AUTO, FF_SCHEME_S, FF_SCHEME_T, FF_SCHEME_CRT, FF_SCHEME_FP64 = 0, 1, 2, 3, 4
FF_MAX_MODULI = 16

_i32, _i64, _u32, _u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
_p, _ch, _sz = ctypes.c_void_p, ctypes.c_char, ctypes.c_size_t


class ff_opts(ctypes.Structure):
    _fields_ = [("winograd", _i32), ("scheme", _i32), ("kb_override", _i64),
                ("debug_saturate", _i32), ("cta_group", _i32), ("host_block", _i32),
                ("korder", _i32), ("debug_unchecked_kb", _i32), ("inputs_canonical", _i32),
                ("small_path", _i32), ("wide_tiles", _i32)]


class ff_plan_info(ctypes.Structure):
    _fields_ = [("p", _u32), ("L", _i32), ("scheme", _i32), ("groups", _i32),
                ("limb_signed", _i32 * 4), ("digit_max", _i32 * 4), ("group_bound", _i64 * 7),
                ("group_bound_max", _i64), ("kb_max", _i64), ("kb", _i64), ("k_pad", _i64),
                ("num_kblocks", _i64), ("centre_max", _i32), ("reserved0", _i32),
                ("carry_max", _i64), ("korder", _i32), ("nmod", _i32), ("moduli", _u32 * 16),
                ("log2_M_floor", _i32), ("log2_bound_ceil", _i32), ("k_winograd", _i64 * 4)]


_OPTS_P = ctypes.POINTER(ff_opts)
_SIGS = {
    "ff_version": ([], ctypes.c_int),
    "ff_strerror": ([ctypes.c_int], ctypes.c_char_p),
    "ff_device_check": ([ctypes.c_int], ctypes.c_int),
    "ff_plan_query": ([_u32, _i64, _OPTS_P, ctypes.POINTER(ff_plan_info)], ctypes.c_int),
    "ff_gemm": ([_u32, _ch, _ch, _i64, _i64, _i64, _u32, _p, _i64, _p, _i64, _u32, _p, _i64],
                ctypes.c_int),
    "ff_gemm_workspace_size": ([_u32, _ch, _ch, _i64, _i64, _i64, _OPTS_P], _sz),
    "ff_gemm_ex": ([_u32, _ch, _ch, _i64, _i64, _i64, _u32, _p, _i64, _p, _i64, _u32, _p, _i64,
                    _OPTS_P, _p, _sz, _p], ctypes.c_int),
    "ff_gemm_host": ([_u32, _ch, _ch, _i64, _i64, _i64, _u32, _p, _i64, _p, _i64, _u32, _p, _i64,
                      _OPTS_P], ctypes.c_int),
    "ff_encode": ([_u32, _i64, _OPTS_P, ctypes.c_int, _i64, _p, _i64, _p, _p], ctypes.c_int),
    "ff_gemm_limbs": ([_u32, _i64, _i64, _i64, _OPTS_P, _u32, _p, _p, _u32, _p, _i64, _p],
                      ctypes.c_int),
    "ff_fill_uniform": ([_p, _i64, _i64, _i64, _u32, _u64, _u32, _i64, _p], ctypes.c_int),
    "ff_trsm": ([_u32, _ch, _ch, _ch, _ch, _i64, _i64, _u32, _p, _i64, _p, _i64], ctypes.c_int),
    "ff_trsm_workspace_size": ([_u32, _ch, _i64, _i64, _OPTS_P], _sz),
    "ff_trsm_ex": ([_u32, _ch, _ch, _ch, _ch, _i64, _i64, _u32, _p, _i64, _p, _i64, _OPTS_P, _p, _sz, _p],
                   ctypes.c_int),
    "ff_lqup": ([_u32, _i64, _i64, _p, _i64, _p, _p, _p], ctypes.c_int),
    "ff_lqup_workspace_size": ([_u32, _i64, _i64, _OPTS_P], _sz),
    "ff_lqup_ex": ([_u32, _i64, _i64, _p, _i64, _p, _p, _p, _OPTS_P, _p, _sz, _p], ctypes.c_int),
    "ff_rank_det": ([_u32, _i64, _i64, _p, _i64, _p, _p], ctypes.c_int),
    "ff_prof_start": ([_i32], ctypes.c_int),
    "ff_prof_stop": ([_p, _i32, _p], ctypes.c_int),
    "ff_mma_ceiling": ([_i32, _p], ctypes.c_int),
    "ff_gemm_winograd_levels": ([_u32, _i64, _i64, _i64, _OPTS_P, _p], ctypes.c_int),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


class FFError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__("%s: %s (code %d)" % (where, ff_strerror(code), code))


def _check(code: int, where: str) -> None:
    if code != 0:
        raise FFError(code, where)


def _opts(opts):
    if opts is None:
        return None
    if isinstance(opts, ff_opts):
        return ctypes.byref(opts)
    o = ff_opts()
    for key, val in dict(opts).items():
        setattr(o, key, val)
    return ctypes.byref(o)


def _tr(t: str) -> bytes:
    return t.encode() if isinstance(t, str) else bytes(t)


def ff_version() -> int:
    return _lib.ff_version()


def ff_strerror(code: int) -> str:
    return _lib.ff_strerror(code).decode()


def ff_device_check(device: int = 0) -> int:
    return _lib.ff_device_check(device)


def ff_plan_query(p: int, k: int, opts=None) -> dict:
    info = ff_plan_info()
    _check(_lib.ff_plan_query(p, k, _opts(opts), ctypes.byref(info)), "ff_plan_query")
    L, G = info.L, info.groups
    return {"p": info.p, "L": L, "scheme": {1: "S", 2: "T", 3: "CRT", 4: "FP64"}[info.scheme], "groups": G,
            "limb_signed": list(info.limb_signed[:min(L, 4)]), "digit_max": list(info.digit_max[:min(L, 4)]),
            "group_bound": list(info.group_bound[:min(G, 7)]), "group_bound_max": info.group_bound_max,
            "kb_max": info.kb_max, "kb": info.kb, "k_pad": info.k_pad,
            "num_kblocks": info.num_kblocks, "centre_max": info.centre_max,
            "carry_max": info.carry_max, "korder": info.korder, "nmod": info.nmod,
            "moduli": list(info.moduli[:info.nmod]), "log2_M_floor": info.log2_M_floor,
            "log2_bound_ceil": info.log2_bound_ceil, "k_winograd": list(info.k_winograd)}


def ff_gemm(p, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc) -> None:
    """Raw C call; A, B, C are device pointers (ints) or tensors (``data_ptr()`` is used)."""
    _check(_lib.ff_gemm(p, _tr(transA), _tr(transB), m, n, k, alpha % 2 ** 32, _ptr(A), lda,
                        _ptr(B), ldb, beta % 2 ** 32, _ptr(C), ldc), "ff_gemm")


def ff_gemm_workspace_size(p, transA, transB, m, n, k, opts=None) -> int:
    return _lib.ff_gemm_workspace_size(p, _tr(transA), _tr(transB), m, n, k, _opts(opts))


def ff_gemm_ex(p, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, opts=None,
               workspace=None, workspace_bytes=0, stream=None) -> None:
    _check(_lib.ff_gemm_ex(p, _tr(transA), _tr(transB), m, n, k, alpha % 2 ** 32, _ptr(A), lda,
                           _ptr(B), ldb, beta % 2 ** 32, _ptr(C), ldc, _opts(opts),
                           _ptr(workspace), workspace_bytes, _stream(stream)), "ff_gemm_ex")


def ff_gemm_winograd_levels(p, m, n, k, opts=None) -> int:
    """Winograd levels ff_gemm_ex would use for this shape (host only)."""
    lv = ctypes.c_int32(0)
    _check(_lib.ff_gemm_winograd_levels(p, m, n, k, _opts(opts), ctypes.byref(lv)), "ff_gemm_winograd_levels")
    return lv.value


def ff_gemm_host(p, transA, transB, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, opts=None) -> None:
    """Host-buffer entry point: A, B, C are host pointers / numpy arrays / CPU tensors."""
    _check(_lib.ff_gemm_host(p, _tr(transA), _tr(transB), m, n, k, alpha % 2 ** 32, _ptr(A), lda,
                             _ptr(B), ldb, beta % 2 ** 32, _ptr(C), ldc, _opts(opts)),
           "ff_gemm_host")


def ff_encode(p, k, opts, kmajor_src, rows, X, ldx, limbs, stream=None) -> None:
    _check(_lib.ff_encode(p, k, _opts(opts), int(kmajor_src), rows, _ptr(X), ldx, _ptr(limbs),
                          _stream(stream)), "ff_encode")


def ff_gemm_limbs(p, m, n, k, opts, alpha, A_limbs, B_limbs, beta, C, ldc, stream=None) -> None:
    _check(_lib.ff_gemm_limbs(p, m, n, k, _opts(opts), alpha % 2 ** 32, _ptr(A_limbs),
                              _ptr(B_limbs), beta % 2 ** 32, _ptr(C), ldc, _stream(stream)),
           "ff_gemm_limbs")


def ff_fill_uniform(X, rows, cols, ld, p, seed, stream_id, index0=0, stream=None) -> None:
    _check(_lib.ff_fill_uniform(_ptr(X), rows, cols, ld, p, seed, stream_id, index0,
                                _stream(stream)), "ff_fill_uniform")


def ff_trsm(p, side, uplo, transA, diag, m, n, alpha, A, lda, B, ldb) -> None:
    _check(_lib.ff_trsm(p, _tr(side), _tr(uplo), _tr(transA), _tr(diag), m, n, alpha % 2 ** 32, _ptr(A), lda,
                        _ptr(B), ldb), "ff_trsm")


def ff_trsm_workspace_size(p, side, m, n, opts=None) -> int:
    return _lib.ff_trsm_workspace_size(p, _tr(side), m, n, _opts(opts))


def ff_trsm_ex(p, side, uplo, transA, diag, m, n, alpha, A, lda, B, ldb, opts=None, workspace=None,
               workspace_bytes=0, stream=None) -> None:
    _check(_lib.ff_trsm_ex(p, _tr(side), _tr(uplo), _tr(transA), _tr(diag), m, n, alpha % 2 ** 32, _ptr(A),
                           lda, _ptr(B), ldb, _opts(opts), _ptr(workspace), workspace_bytes, _stream(stream)),
           "ff_trsm_ex")


def ff_prof_start(capacity: int) -> None:
    """Start bracketing the library's GEMM-kernel launches with CUDA events (benchmarks)."""
    _check(_lib.ff_prof_start(capacity), "ff_prof_start")


def ff_prof_stop(capacity: int):
    """Stop recording; returns (per-launch GEMM kernel times in ms, kernel launches counted)."""
    buf = (ctypes.c_float * max(1, capacity))()
    launches = ctypes.c_int64(0)
    n = _lib.ff_prof_stop(buf, capacity, ctypes.byref(launches))
    if n < 0:
        raise FFError(-n, "ff_prof_stop")
    return [buf[i] for i in range(min(n, capacity))], launches.value


def ff_mma_ceiling(iters: int = 200000) -> float:
    """Measured int8 tcgen05 MMA-only throughput of the current device (TOPS)."""
    out = ctypes.c_double(0.0)
    _check(_lib.ff_mma_ceiling(iters, ctypes.byref(out)), "ff_mma_ceiling")
    return out.value


# ---------------------------------------------------------------- marshalling helpers

def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):          # numpy
        return x.ctypes.data
    raise TypeError("cannot take the address of %r" % type(x))


_cur_stream = None


def _stream(s):
    """Raw cudaStream_t of `s` (None: torch's current stream on the current device,
    read through torch's two C accessors -- torch.cuda.current_stream() builds a
    Python Stream object per call, ~3 us of the ~15 us a small call takes)."""
    global _cur_stream
    if s is None:
        if _cur_stream is None:
            import torch
            if not torch.cuda.is_available():
                return None
            get_dev, get_raw = torch._C._cuda_getDevice, torch._C._cuda_getCurrentRawStream
            _cur_stream = lambda: get_raw(get_dev())  # noqa: E731
        return _cur_stream()
    if isinstance(s, int):
        return s
    return s.cuda_stream


def _ld(t) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("need a 2-D row-major tensor with unit column stride")
    return max(1, t.stride(0))


def fgemm(p: int, A, B, C=None, alpha: int = 1, beta: int = 0, transA: str = "N",
          transB: str = "N", opts=None, stream=None):
    """C <- (alpha op(A) op(B) + beta C) mod p on torch int32 CUDA tensors; returns C.

    A, B, C are 2-D int32 CUDA tensors (row-major, any leading dimension).  If C is
    None a new (m x n) tensor is allocated (beta must then be 0 mod p).
    """
    import torch
    m = A.shape[1] if transA in "Tt" else A.shape[0]
    k = A.shape[0] if transA in "Tt" else A.shape[1]
    n = B.shape[0] if transB in "Tt" else B.shape[1]
    kb = B.shape[1] if transB in "Tt" else B.shape[0]
    if kb != k:
        raise ValueError("inner dimensions differ: %d vs %d" % (k, kb))
    if C is None:
        if beta % p:
            raise ValueError("beta != 0 needs C")
        C = torch.empty((m, n), dtype=torch.int32, device=A.device)
    for t in (A, B, C):
        if t.dtype != torch.int32 or not t.is_cuda:
            raise TypeError("fgemm takes int32 CUDA tensors")
    ff_gemm_ex(p, transA, transB, m, n, k, alpha, A, _ld(A), B, _ld(B), beta, C, _ld(C), opts,
               None, 0, stream)
    return C


def ftrsm(p: int, A, B, side: str = "L", uplo: str = "U", transA: str = "N", diag: str = "N",
          alpha: int = 1, opts=None, stream=None):
    """B <- X with op(A) X = alpha B (side 'L') or X op(A) = alpha B ('R'), mod p,
    on int32 CUDA tensors (Sec. 4); the workspace is a torch tensor
    from the caching allocator, the work runs on torch's current stream."""
    import torch
    m, n = B.shape
    d = m if side in "Ll" else n
    if A.shape[0] < d or A.shape[1] < d:
        raise ValueError("A must be at least %d x %d" % (d, d))
    for t in (A, B):
        if t.dtype != torch.int32 or not t.is_cuda:
            raise TypeError("ftrsm takes int32 CUDA tensors")
    nbytes = ff_trsm_workspace_size(p, side, m, n, opts)
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=B.device)
    ff_trsm_ex(p, side, uplo, transA, diag, m, n, alpha, A, _ld(A), B, _ld(B), opts, ws, nbytes, stream)
    return B


def lqup(p: int, A, opts=None, stream=None):
    """In-place LQUP (PLUQ arrangement, include/ffgemm.h) of the int32 CUDA
    tensor A; returns (Q, P, rank) with Q, P numpy int64 permutation arrays."""
    import numpy as np
    import torch
    if A.dtype != torch.int32 or not A.is_cuda:
        raise TypeError("lqup takes an int32 CUDA tensor")
    m, n = A.shape
    Q = np.zeros(max(m, 1), dtype=np.int64)
    P = np.zeros(max(n, 1), dtype=np.int64)
    r = ctypes.c_int64(0)
    nbytes = _lib.ff_lqup_workspace_size(p, m, n, _opts(opts))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=A.device)
    _check(_lib.ff_lqup_ex(p, m, n, _ptr(A), _ld(A), Q.ctypes.data, P.ctypes.data, ctypes.byref(r), _opts(opts),
                           _ptr(ws), nbytes, _stream(stream)), "ff_lqup_ex")
    return Q[:m], P[:n], r.value


def rank_det(p: int, A):
    """(rank, det or None) of the int32 CUDA tensor A (not modified)."""
    m, n = A.shape
    r = ctypes.c_int64(0)
    d = ctypes.c_uint32(0)
    _check(_lib.ff_rank_det(p, m, n, _ptr(A), _ld(A), ctypes.byref(r), ctypes.byref(d) if m == n else None),
           "ff_rank_det")
    return r.value, (d.value if m == n else None)
