"""Host-side checks of the CUDA library (no GPU needed): it loads, exports
every symbol include/ffgemm.h declares, validates arguments in BLAS xerbla
order, and its planner reproduces the delayed-reduction bounds derived
independently here from the paper's Eq. (2)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ff():
    from paper_cs_0601133_b200 import build
    build.build()
    import paper_cs_0601133_b200 as ff
    return ff


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "ffgemm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ff_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(ff):
    lib = ctypes.CDLL(ff.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 11
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(ff.EXPORTED)


def test_binary_is_sm100a_tcgen05(ff):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", ff.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", ff.LIB_PATH],
                                       capture_output=True, text=True).stdout
    for mnemonic in ("UTCIMMA", "UTMALDG", "LDTM", "STTM"):
        assert mnemonic in out, mnemonic


def test_version_and_strerror(ff):
    assert ff.ff_version() >= 100
    for code in (0, 1, 2, 3, 4, 5, -1, -9, -14, 99):
        assert isinstance(ff.ff_strerror(code), str) and ff.ff_strerror(code)


@pytest.mark.parametrize("args,code", [
    ((1, b"N", b"N", 2, 2, 2), -1),            # p < 2
    ((2 ** 31, b"N", b"N", 2, 2, 2), -1),      # p >= 2^31
    ((5, b"X", b"N", 2, 2, 2), -2),
    ((5, b"N", b"Q", 2, 2, 2), -3),
    ((5, b"N", b"N", -1, 2, 2), -4),
    ((5, b"N", b"N", 2, -1, 2), -5),
    ((5, b"N", b"N", 2, 2, -1), -6),
])
def test_argument_errors_in_xerbla_order(ff, args, code):
    lib = ctypes.CDLL(ff.LIB_PATH)
    lib.ff_gemm.argtypes = ff.ffgemm._lib.ff_gemm.argtypes
    p, ta, tb, m, n, k = args
    dummy = 4096
    assert lib.ff_gemm(p, ta, tb, m, n, k, 1, dummy, 8, dummy, 8, 0, dummy, 8) == code


def test_ld_and_null_errors(ff):
    g = ff.ffgemm._lib.ff_gemm
    d = 4096
    assert g(5, b"N", b"N", 4, 3, 6, 1, None, 6, d, 3, 0, d, 3) == -8
    assert g(5, b"N", b"N", 4, 3, 6, 1, d, 5, d, 3, 0, d, 3) == -9     # lda < k
    assert g(5, b"T", b"N", 4, 3, 6, 1, d, 3, d, 3, 0, d, 3) == -9     # lda < m
    assert g(5, b"N", b"N", 4, 3, 6, 1, d, 6, None, 3, 0, d, 3) == -10
    assert g(5, b"N", b"N", 4, 3, 6, 1, d, 6, d, 2, 0, d, 3) == -11    # ldb < n
    assert g(5, b"N", b"T", 4, 3, 6, 1, d, 6, d, 5, 0, d, 3) == -11    # ldb < k
    assert g(5, b"N", b"N", 4, 3, 6, 1, d, 6, d, 3, 0, None, 3) == -13
    assert g(5, b"N", b"N", 4, 3, 6, 1, d, 6, d, 3, 0, d, 2) == -14
    # m = 0 or n = 0 is a successful no-op that never touches the GPU
    assert g(5, b"N", b"N", 0, 3, 6, 1, None, 6, d, 3, 0, None, 3) == 0


# ---------------------------------------------------------------- planner vs Eq. (2)

def _balanced_digits(c, L):
    """Test-side digit split, written from the definition c = sum d_i 256^i with
    d_i in [-128, 127] chosen as the residue of c mod 256 nearest to zero."""
    out = []
    for _ in range(L):
        d = ((c + 128) % 256) - 128
        out.append(d)
        c = (c - d) // 256
    return out, c


def _twos_digits(c, L):
    out = []
    for i in range(L - 1):
        out.append(c % 256)
        c //= 256
    out.append(c)
    return out, 0 if -128 <= c <= 127 else c


def _centred_all(p):
    r = np.arange(p, dtype=np.int64)
    return np.where(r > (p - 1) // 2, r - p, r)


@pytest.mark.parametrize("p,L,scheme,D,kb_max", [
    (65521, 2, "T", [255, 128], 32896),          # c1, c4
    (8388593, 3, "S", [128, 128, 64], 65408),    # c2
    (251, 1, "S", [125], 137438),                # c3
    (67108859, 4, "S", [128, 128, 128, 2], 43008),  # c5
])
def test_planner_matches_paper_bound(ff, p, L, scheme, D, kb_max):
    lopt = {"scheme": {"S": 1, "T": 2}[scheme]}      # the limb scheme (AUTO may pick CRT for c5)
    info = ff.ff_plan_query(p, 1000, lopt)
    assert info["L"] == L and info["scheme"] == scheme
    assert info["digit_max"] == D
    # Eq. (2) with gamma = 32 for the s32 accumulator, per weight group, plus one
    # centred carry: kb * max_w B_w + (p-1)/2 <= 2^31 - 1.
    B = [sum(D[i] * D[w - i] for i in range(L) if 0 <= w - i < L) for w in range(2 * L - 1)]
    assert info["group_bound"] == B
    half = (p - 1) // 2
    # with an exactly centred carry the bound is SURVEY §8(a)'s kb_max ...
    assert kb_max == (2 ** 31 - 1 - half) // max(B)
    # ... the kernel writes back an integer-Barrett estimate (modp.cuh reduce_mulhi)
    # with |carry| <= 3p/2 for p < 2^29 (else a float-reciprocal one: (p-1)/2 + 385 w)
    carry = (3 * p + 1) // 2 if p < 2 ** 29 and (L == 1 or p >= 512) else half + 385 * (256 if L >= 2 else 1)
    assert info["carry_max"] == carry
    kbm = info["kb_max"]
    assert kbm == (2 ** 31 - 1 - carry) // max(B)
    assert kbm * max(B) + carry <= 2 ** 31 - 1 < (kbm + 1) * max(B) + carry
    assert 0.95 * kb_max <= kbm <= kb_max
    assert info["kb"] % 128 == 0 and info["kb"] <= kbm
    # every config fits one safe k-block ("none of the 5 needs it") in
    # group-outer order; the default k-outer order blocks k by 8192/L for L2 locality
    for k in (512, 4096, 8192, 16384):
        assert ff.ff_plan_query(p, k, dict(lopt, korder=1))["num_kblocks"] == 1
        d = ff.ff_plan_query(p, k, lopt)
        loc = -(-(8192 // L) // 128) * 128
        assert d["korder"] == 2 and d["kb"] == min(loc, info["kb"]) and d["num_kblocks"] == -(-k // d["kb"])


@pytest.mark.parametrize("p", [2, 3, 5, 251, 257, 65279, 65521, 65537])
def test_digit_bounds_exhaustive_small_primes(ff, p):
    info = ff.ff_plan_query(p, 64)
    if info["scheme"] == "CRT":          # 65537 (+-32768 needs 3 limbs): AUTO is multi-modular
        info = ff.ff_plan_query(p, 64, {"scheme": 1})
    L = info["L"]
    split = _balanced_digits if info["scheme"] == "S" else _twos_digits
    seen = [0] * L
    for c in _centred_all(p).tolist():
        d, rest = split(c, L)
        assert rest == 0, (p, c)
        assert sum(di * 256 ** i for i, di in enumerate(d)) == c
        seen = [max(s, abs(di)) for s, di in zip(seen, d)]
    # the planner's bound is attained (tight) for the top digit and safe elsewhere
    assert seen[-1] == info["digit_max"][-1]
    assert all(s <= dm for s, dm in zip(seen, info["digit_max"]))
    # minimality of L: one limb fewer cannot represent all residues
    if L > 1:
        for other in (_balanced_digits, _twos_digits):
            assert any(other(c, L - 1)[1] != 0 for c in _centred_all(p).tolist())


def test_scheme_choice_rule(ff):
    # S is used unless only T reaches the smaller L:
    assert ff.ff_plan_query(65279, 8)["scheme"] == "S"   # 2 balanced digits reach +-32639
    assert ff.ff_plan_query(65521, 8)["scheme"] == "T"   # centred +-32760 needs T for L=2
    assert ff.ff_plan_query(65521, 8, {"scheme": 1})["L"] == 3
    assert ff.ff_plan_query(2 ** 31 - 1, 8, {"scheme": 1})["L"] == 4
    # multi-modular when it needs >= 3 fewer int8 products than L^2
    assert ff.ff_plan_query(2 ** 31 - 1, 8)["scheme"] == "CRT"
    assert ff.ff_plan_query(67108859, 16384)["scheme"] == "CRT"      # c5: 9 moduli vs 16
    assert ff.ff_plan_query(67108859, 16384)["L"] == 9
    assert ff.ff_plan_query(8388593, 4096)["scheme"] == "S"          # c2: 8 vs 9, stays on limbs
    assert ff.ff_plan_query(65521, 8192)["scheme"] == "T"            # c4: 6 vs 4


def test_kb_override_rules(ff):
    info = ff.ff_plan_query(65521, 5000, {"kb_override": 1000})
    assert info["kb"] == 896 and info["num_kblocks"] == 6
    with pytest.raises(ff.FFError):
        ff.ff_plan_query(65521, 5000, {"kb_override": 40000})   # above the safe bound
    with pytest.raises(ff.FFError):
        ff.ff_plan_query(65521, 5000, {"kb_override": 64})      # below one stage


def test_f64_plan_is_paper_eq2(ff):
    """The fp64 engine's lambda is Eq. (2) with gamma = 53,
    SURVEY §8(f) NEXT-3: 4196352 (p = 65521), 256 (8388593), 4 (67108859)."""
    from oracle import bounds
    for p, lam in [(65521, 4196352), (8388593, 256), (67108859, 4)]:
        info = ff.ff_plan_query(p, 1000, {"scheme": 4})
        assert info["scheme"] == "FP64" and info["kb_max"] == lam
        assert lam == bounds.lambda_dot(p, 53, balanced=True)
        assert info["kb"] == lam // 4 * 4 and info["kb"] % 4 == 0
    with pytest.raises(ff.FFError):
        ff.ff_plan_query(2 ** 27 - 39, 10, {"scheme": 4})       # lambda < 4: beyond the paper's 2^26 bound
    with pytest.raises(ff.FFError):
        ff.ff_plan_query(65521, 10, {"scheme": 4, "kb_override": 2 ** 23})


def test_wide_tiles_option_rules(ff):
    for v in (-1, 0, 1):
        ff.ff_plan_query(251, 5000, {"wide_tiles": v})
    for v in (-2, 2):
        with pytest.raises(ff.FFError):
            ff.ff_plan_query(251, 5000, {"wide_tiles": v})


def test_struct_layouts_match_the_header(ff, tmp_path):
    """The ctypes mirrors of ff_opts and ff_plan_info (the Python binding) have
    the header's size and field offsets: compiled and measured with the host C
    compiler from include/ffgemm.h itself."""
    import subprocess
    from paper_cs_0601133_b200 import ffgemm as binding
    structs = {"ff_opts": binding.ff_opts, "ff_plan_info": binding.ff_plan_info}
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "ffgemm.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append('printf("%s sizeof %%zu\\n", sizeof(%s));' % (name, name))
        for fname, _ in cls._fields_:
            lines.append('printf("%s %s %%zu\\n", offsetof(%s, %s));' % (name, fname, name, fname))
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", str(src),
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for name, cls in structs.items():
        assert got[(name, "sizeof")] == ctypes.sizeof(cls), name
        for fname, _ in cls._fields_:
            assert got[(name, fname)] == getattr(cls, fname).offset, (name, fname)


def test_winograd_levels_query_host_only():
    """ff_gemm_winograd_levels (host only): the measured default rule (one level
    for several limbs / CRT planes on large shapes), forced levels,
    the fp64 engine's Corollary 3.4 limit, and argument errors."""
    import paper_cs_0601133_b200 as ff
    lv = ff.ff_gemm_winograd_levels
    assert lv(67108859, 16384, 16384, 16384) == 1          # c5: CRT + one level by default
    assert lv(67108859, 8192, 16384, 16384) == 1           # c5 panel at 2 GPUs: local Winograd
    assert lv(67108859, 2048, 16384, 16384) == 0           # c5 panel at 8 GPUs: too few half tiles
    assert lv(65521, 32768, 32768, 8192) == 0              # c4: two limbs, measured to lose
    assert lv(65521, 4096, 4096, 4096, {"winograd": 1}) == 1
    assert lv(65521, 4096, 4096, 4096, {"winograd": -1}) == 0
    assert lv(65521, 1000, 1000, 1000, {"scheme": 4, "winograd": 3}) == 3
    with pytest.raises(ff.FFError):
        lv(8388593, 64, 64, 114, {"scheme": 4, "winograd": 1})   # k = k_winograd: Cor 3.4 refuses
    assert lv(8388593, 64, 64, 113, {"scheme": 4, "winograd": 1}) == 1
    with pytest.raises(ff.FFError):
        lv(65521, 511, 512, 512, {"winograd": 1})           # odd / too small for the int8 level
    with pytest.raises(ff.FFError):
        lv(1, 10, 10, 10)                                    # p out of range
