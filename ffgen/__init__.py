"""Seeded, counter-based synthetic input generator (shared by both sides).

This module is the ONE piece of code that both the CPU oracle side (``oracle/``,
``tests/``) and the CUDA product side may rely on.  It contains none of the
method's arithmetic: it only draws i.i.d. integers in ``[0, p)`` from a seed, as
BASELINE.json's configs require ("A,B i.i.d. uniform integers in [0,p) from a
seed, stored as int32").  The paper itself never states its input distribution
(§3.3, l.320: "modulo 65521 on these tables", random dense matrices);
the recipe below is our reading, recorded in DESIGN.md §3.

Recipe; every element is a pure function of its index, so any
sub-block can be generated independently (row panels for multi-GPU, sampled
rows for parity) and the CUDA twin (``ff_fill_uniform`` in the product library)
is compared with this one bit-for-bit in the tests:

    GAMMA     = 0x9E3779B97F4A7C15
    mix64(z)  = splitmix64 output function:
                z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
                z = (z ^ (z >> 27)) * 0x94D049BB133111EB
                return z ^ (z >> 31)                       (all mod 2^64)
    seed_key  = mix64(seed * 16 + stream)                  stream: A=0, B=1, C=2
    v[i]      = (mix64(seed_key + (i + 1) * GAMMA) >> 11) mod p

where ``i`` is the row-major index over the STORED array (``i = r * cols + c``)
and the stored array is dense (``ld == cols``).  ``>> 11`` keeps 53 bits, so the
modulo bias is below 2^-27 for every p < 2^26 used here; it is irrelevant to
correctness because both sides consume the same stored integers.
"""
from __future__ import annotations

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1

STREAM_A, STREAM_B, STREAM_C = 0, 1, 2


def mix64_int(z: int) -> int:
    """splitmix64 output function on one Python int (reference for the vector form)."""
    z &= _MASK
    z = ((z ^ (z >> 30)) * _M1) & _MASK
    z = ((z ^ (z >> 27)) * _M2) & _MASK
    return z ^ (z >> 31)


def seed_key(seed: int, stream: int) -> int:
    return mix64_int((seed * 16 + stream) & _MASK)


def _mix64_vec(z: np.ndarray) -> np.ndarray:
    # numpy uint64 arithmetic wraps mod 2^64, which is exactly what we want.
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        return z ^ (z >> np.uint64(31))


def uniform_flat_numpy(p: int, seed: int, stream: int, start: int, count: int,
                       chunk: int = 1 << 22) -> np.ndarray:
    """Elements ``v[start : start+count]`` of the (seed, stream) sequence, as int32
    (plain numpy; the reference form of the recipe)."""
    if not (2 <= p < 2 ** 31):
        raise ValueError("p must be in [2, 2^31)")
    key = np.uint64(seed_key(seed, stream))
    out = np.empty(count, dtype=np.int32)
    pu = np.uint64(p)
    for off in range(0, count, chunk):
        n = min(chunk, count - off)
        idx = np.arange(start + off + 1, start + off + 1 + n, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = key + idx * np.uint64(GAMMA)
        v = (_mix64_vec(z) >> np.uint64(11)) % pu
        out[off:off + n] = v.astype(np.int32)
    return out


_clib = None


def _c_gen():
    """ffgen/gen.c (the same recipe in C with OpenMP), built on first use with gcc;
    None if it cannot be built (the numpy form is then used)."""
    global _clib
    if _clib is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        src, lib = os.path.join(here, "gen.c"), os.path.join(here, "libffgen.so")
        try:
            if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
                tmp = lib + ".tmp%d" % os.getpid()
                subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, src])
                os.replace(tmp, lib)
            c = ctypes.CDLL(lib)
            c.ffgen_uniform_flat.argtypes = [ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_void_p]
            c.ffgen_uniform_flat.restype = None
            c.ffgen_set_threads.argtypes = [ctypes.c_int]
            c.ffgen_set_threads.restype = None
            _clib = c
        except Exception:
            _clib = False
    return _clib or None


def set_threads(n: int) -> None:
    """Threads of the C generator (no-op without it)."""
    c = _c_gen()
    if c is not None:
        c.ffgen_set_threads(int(n))


def uniform_flat(p: int, seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """Elements ``v[start : start+count]`` of the (seed, stream) sequence, as int32
    (C + OpenMP when available; bit-identical to ``uniform_flat_numpy``, tested)."""
    if not (2 <= p < 2 ** 31):
        raise ValueError("p must be in [2, 2^31)")
    c = _c_gen() if count >= 1 << 16 else None
    if c is None:
        return uniform_flat_numpy(p, seed, stream, start, count)
    out = np.empty(count, dtype=np.int32)
    c.ffgen_uniform_flat(p, seed_key(seed, stream), start, count, out.ctypes.data)
    return out


def uniform_matrix(p: int, seed: int, stream: int, rows: int, cols: int,
                   row0: int = 0, nrows: int | None = None) -> np.ndarray:
    """Rows ``[row0, row0+nrows)`` of the dense stored ``rows x cols`` matrix (int32)."""
    if nrows is None:
        nrows = rows - row0
    if row0 < 0 or nrows < 0 or row0 + nrows > rows:
        raise ValueError("row window out of range")
    flat = uniform_flat(p, seed, stream, row0 * cols, nrows * cols)
    return flat.reshape(nrows, cols)


def uniform_vector(p: int, seed: int, stream: int, n: int) -> np.ndarray:
    """A length-n vector from the same recipe (Freivalds probes use stream >= 8)."""
    return uniform_flat(p, seed, stream, 0, n)
