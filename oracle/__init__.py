"""CPU oracle for fgemm -- TEST INFRASTRUCTURE, not the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_cs_0601133_b200``) never imports it and shares no code with it.

``oracle.c`` holds the definitions (fgemm, and the triangular solve ``trsm``
of PAPER.md Sec. 4; see its header for the passages followed); this module
only marshals numpy arrays into it, plus ``winograd.py`` (Table 1 op counts
and the Table 2 schedule) and ``bounds.py`` (the paper's
delayed-reduction thresholds: Eq. (1)/(2), Cor. 3.4, Thm. 4.2, Eq. (4)/(5))
in exact Python ints.

Parity status: every function here is pinned (tests/test_oracle_pins.py,
test_oracle_trsm_pins.py, test_oracle_winograd_bound.py); none is "parity
unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64 = ctypes.c_int64
_u32 = ctypes.c_uint32
_p = ctypes.c_void_p
_char = ctypes.c_char


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain C, -O2, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-Wall", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_fgemm.argtypes = [_u32, _char, _char, _i64, _i64, _i64, _u32, _p, _i64,
                                     _p, _i64, _u32, _p, _i64, ctypes.c_int]
        lib.oracle_fgemm.restype = ctypes.c_int
        lib.oracle_fgemm_rows.argtypes = [_u32, _char, _char, _i64, _i64, _i64, _u32, _p, _i64,
                                          _p, _i64, _u32, _p, _i64, _p, _i64, _p, _i64,
                                          ctypes.c_int]
        lib.oracle_fgemm_rows.restype = ctypes.c_int
        lib.oracle_matvec.argtypes = [_u32, _char, _i64, _i64, _p, _i64, _p, _p, ctypes.c_int]
        lib.oracle_matvec.restype = ctypes.c_int
        lib.oracle_max_threads.restype = ctypes.c_int
        lib.oracle_trsm.argtypes = [_u32, _char, _char, _char, _char, _i64, _i64, _u32, _p, _i64,
                                    _p, _i64, ctypes.c_int]
        lib.oracle_trsm.restype = ctypes.c_int
        lib.oracle_rank_det.argtypes = [_u32, _i64, _i64, _p, _i64, _p, _p]
        lib.oracle_rank_det.restype = ctypes.c_int
        _lib = lib
    return _lib


def _c32(x: np.ndarray) -> np.ndarray:
    if x.dtype != np.int32:
        raise TypeError("oracle takes int32 arrays")
    return x


def _ptr(x: np.ndarray):
    return x.ctypes.data_as(ctypes.c_void_p)


def _ld(x: np.ndarray) -> int:
    """Leading dimension (elements) of a 2-D int32 array with unit inner stride."""
    if x.ndim == 2 and x.size == 0:
        return max(1, x.shape[1])
    if x.ndim != 2 or x.strides[1] != 4 or x.strides[0] % 4:
        raise ValueError("need a 2-D row-major int32 view with unit column stride")
    return max(1, x.strides[0] // 4)


def max_threads() -> int:
    return _load().oracle_max_threads()


def fgemm(p: int, transA: str, transB: str, alpha: int, A: np.ndarray, B: np.ndarray,
          beta: int, C: np.ndarray | None = None, m: int | None = None, n: int | None = None,
          k: int | None = None, nthreads: int = 0) -> np.ndarray:
    """Return (alpha*op(A)*op(B) + beta*C) mod p as a new int32 array (C untouched)."""
    lib = _load()
    A, B = _c32(A), _c32(B)
    if m is None:
        m = A.shape[1] if transA in "Tt" else A.shape[0]
    if k is None:
        k = A.shape[0] if transA in "Tt" else A.shape[1]
    if n is None:
        n = B.shape[0] if transB in "Tt" else B.shape[1]
    out = np.zeros((m, n), dtype=np.int32) if C is None else np.array(_c32(C)[:m, :n], copy=True)
    if m == 0 or n == 0:
        return out
    e = lib.oracle_fgemm(p, transA.encode(), transB.encode(), m, n, k, alpha % (1 << 32),
                         _ptr(A), _ld(A), _ptr(B), _ld(B), beta % (1 << 32),
                         _ptr(out), _ld(out) if n else 1, nthreads)
    if e:
        raise ValueError("oracle_fgemm argument %d invalid" % -e)
    return out


def fgemm_rows(p: int, transA: str, transB: str, alpha: int, A: np.ndarray, B: np.ndarray,
               beta: int, Cin_rows: np.ndarray | None, rows, m: int, n: int, k: int,
               nthreads: int = 0) -> np.ndarray:
    """Rows ``rows`` of the output (Cin_rows holds the matching input rows of C)."""
    lib = _load()
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    out = np.zeros((len(rows), n), dtype=np.int32)
    if Cin_rows is None:
        Cin_rows = np.zeros((len(rows), max(n, 1)), dtype=np.int32)
    Cin_rows = np.ascontiguousarray(_c32(Cin_rows))
    e = lib.oracle_fgemm_rows(p, transA.encode(), transB.encode(), m, n, k, alpha % (1 << 32),
                              _ptr(_c32(A)), _ld(A), _ptr(_c32(B)), _ld(B), beta % (1 << 32),
                              _ptr(Cin_rows), _ld(Cin_rows), _ptr(rows), len(rows),
                              _ptr(out), max(n, 1), nthreads)
    if e:
        raise ValueError("oracle_fgemm_rows argument %d invalid" % -e)
    return out


def matvec(p: int, trans: str, X: np.ndarray, v: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """(op(X) @ v) mod p, exactly."""
    lib = _load()
    X = _c32(X)
    v = np.ascontiguousarray(_c32(v))
    rows, cols = (X.shape[1], X.shape[0]) if trans in "Tt" else X.shape
    out = np.zeros(rows, dtype=np.int32)
    e = lib.oracle_matvec(p, trans.encode(), rows, cols, _ptr(X), _ld(X), _ptr(v), _ptr(out),
                          nthreads)
    if e:
        raise ValueError("oracle_matvec argument %d invalid" % -e)
    return out


def trsm(p: int, side: str, uplo: str, transA: str, diag: str, alpha: int, A: np.ndarray,
         B: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """X with op(A) X = alpha B (side 'L') or X op(A) = alpha B (side 'R'), mod p,
    as a new int32 array (Sec. 4, plain substitution; see oracle.c)."""
    lib = _load()
    A = _c32(A)
    X = np.array(_c32(B), copy=True)
    m, n = X.shape
    e = lib.oracle_trsm(p, side.encode(), uplo.encode(), transA.encode(), diag.encode(), m, n,
                        alpha % (1 << 32), _ptr(A), _ld(A), _ptr(X), _ld(X), nthreads)
    if e < 0:
        raise ValueError("oracle_trsm argument %d invalid" % -e)
    if e == 1:
        raise ZeroDivisionError("oracle_trsm: a diagonal entry is not invertible mod p")
    if e:
        raise MemoryError("oracle_trsm")
    return X


def rank_det(p: int, X: np.ndarray):
    """(rank, det) of X over Z/pZ by plain Gaussian elimination (det is None
    unless X is square).  PAPER.md Sec. 6 (l.655-657)."""
    lib = _load()
    X = _c32(X)
    m, n = X.shape
    r = ctypes.c_int64(0)
    d = ctypes.c_int64(-1)
    e = lib.oracle_rank_det(p, m, n, _ptr(X), _ld(X), ctypes.byref(r), ctypes.byref(d))
    if e < 0:
        raise ValueError("oracle_rank_det argument %d invalid" % -e)
    if e == 1:
        raise ZeroDivisionError("oracle_rank_det: pivot not invertible (p not prime)")
    if e:
        raise MemoryError("oracle_rank_det")
    return r.value, (d.value if m == n else None)
