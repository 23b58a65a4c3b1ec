"""Host-side checks of the multi-modular (CRT) plan (the
paper's "Chinese remainder algorithm" for fields beyond the BLAS bound,
PAPER.md l.882).  No GPU needed.

The planner's moduli are checked against the number theory directly (Python
big integers): pairwise coprime, q <= 256 so every centred residue is an s8,
M = prod q >= 4 k ((p-1)/2)^2 so the exact integer dot product X is determined
by its residues with |X|/M <= 1/4, and no modulus is superfluous.  The
reconstruction formula the kernel's final epilogue evaluates is then checked
end to end on extreme and random X, with its fixed-point quotient estimate
written out here from the CRT definition (not from the CUDA source)."""
import math
import random

import pytest


@pytest.fixture(scope="module")
def ff():
    import paper_cs_0601133_b200 as ff
    return ff


CASES = [(67108859, 16384), (67108859, 8192), (67108859, 1), (8388593, 4096), (65521, 8192),
         (2 ** 31 - 1, 1), (2 ** 31 - 1, 65536), (251, 16384), (3, 5), (2, 1000), (16711423, 100000)]


@pytest.mark.parametrize("p,k", CASES)
def test_crt_moduli_cover_the_dot_product_bound(ff, p, k):
    info = ff.ff_plan_query(p, k, {"scheme": 3})
    q = info["moduli"]
    assert info["scheme"] == "CRT" and info["L"] == info["nmod"] == info["groups"] == len(q) >= 1
    assert all(2 <= x <= 256 for x in q) and q == sorted(q, reverse=True)
    assert q[0] == 256                         # the encoders take plane 0 as the low byte
    for i in range(len(q)):
        for j in range(i):
            assert math.gcd(q[i], q[j]) == 1, (q[i], q[j])
    cmax = max((p - 1) // 2, (p - 1) - (p - 1) // 2)
    assert info["centre_max"] == cmax
    B = 4 * max(k, 1) * cmax * cmax
    M = math.prod(q)
    assert M >= B                              # |X| <= k cmax^2 <= M/4
    if len(q) > 1:
        assert M // q[-1] < B                  # the last modulus is needed
    assert info["log2_M_floor"] == M.bit_length() - 1
    assert info["log2_bound_ceil"] == (B - 1).bit_length()
    # s32 accumulator: kb products of centred residues (|r| <= q/2) plus one
    # centred residue carried between k-blocks (Eq. (2) analogue, gamma = 32)
    D = max(x // 2 for x in q)
    assert info["group_bound_max"] == D * D
    assert info["kb_max"] * D * D + info["carry_max"] <= 2 ** 31 - 1
    assert (info["kb_max"] + 1) * D * D + info["carry_max"] > 2 ** 31 - 1
    assert info["kb"] % 128 == 0 and info["kb"] <= info["kb_max"]
    assert info["korder"] == 1
    assert info["num_kblocks"] == (-(-k // info["kb"]) if k else 0)


def test_crt_config_counts(ff):
    """int8 products per output tile (SURVEY §8(f) NEXT-1 estimates)."""
    assert ff.ff_plan_query(67108859, 16384, {"scheme": 3})["nmod"] == 9    # c5 (vs 16 limb products)
    assert ff.ff_plan_query(67108859, 8192, {"scheme": 3})["nmod"] == 9     # c5 Winograd half size
    assert ff.ff_plan_query(8388593, 4096, {"scheme": 3})["nmod"] == 8      # c2 (vs 9)
    assert ff.ff_plan_query(65521, 8192, {"scheme": 3})["nmod"] == 6        # c4 (vs 4)
    assert ff.ff_plan_query(251, 16384, {"scheme": 3})["nmod"] == 4         # c3 (vs 1)


def test_crt_extremes(ff):
    # 16 moduli (prod ~ 2^125.4) cover every p < 2^31 up to k ~ 2^63
    info = ff.ff_plan_query(2 ** 31 - 1, 2 ** 62, {"scheme": 3})
    assert info["nmod"] == 16 and info["log2_M_floor"] >= info["log2_bound_ceil"] == 124
    with pytest.raises(ff.FFError):
        ff.ff_plan_query(67108859, 16384, {"scheme": 3, "kb_override": 10 ** 9})


def _reconstruct(X, q, p):
    """The final-epilogue formula, from the CRT definition: u_i = (X mod q_i)
    (M_i^-1 mod q_i) mod q_i; t = round(sum_i u_i / q_i) evaluated in 24-bit
    fixed point; X mod p = sum_i u_i (M_i mod p) - t (M mod p)  (mod p)."""
    M = math.prod(q)
    S, F = 0, 0
    for qi in q:
        Mi = M // qi
        u = (X % qi) * pow(Mi % qi, -1, qi) % qi
        S += u * (Mi % p)
        F += u * ((2 ** 25 // qi + 1) // 2)           # round(2^24 / q_i)
        assert F < 2 ** 32
    t = (F + 2 ** 23) >> 24
    assert t == round(sum(((X % qi) * pow((M // qi) % qi, -1, qi) % qi) / qi for qi in q))
    S += t * ((p - M % p) % p)
    assert S < 2 ** 64
    return S % p


@pytest.mark.parametrize("p,k", CASES)
def test_crt_reconstruction_formula_exact(ff, p, k):
    info = ff.ff_plan_query(p, k, {"scheme": 3})
    q = info["moduli"]
    cmax = info["centre_max"]
    X_max = max(k, 1) * cmax * cmax
    rng = random.Random(p ^ k)
    xs = [0, 1, -1, X_max, -X_max, X_max - 1, -X_max + 1, cmax * cmax, -cmax * cmax]
    xs += [rng.randint(-X_max, X_max) for _ in range(300)]
    for X in xs:
        assert _reconstruct(X, q, p) == X % p, X
