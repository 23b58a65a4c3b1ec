"""Property tests of the host planner (no GPU): for random primes-or-not p and
k, whatever scheme the planner picks must satisfy the exactness conditions
derived here from first principles (Eq. (2) generalised to limbs,
and the CRT bound of DESIGN.md §4.9)."""
import math

import pytest
from hypothesis import given, settings, strategies as st


@pytest.fixture(scope="module")
def ff():
    import paper_cs_0601133_b200 as ff
    return ff


def _limb_check(info, p):
    L = info["L"]
    half = (p - 1) // 2
    neg = (p - 1) - half
    # every centred residue in [-neg, half] is representable: decode of the extreme digits
    D = info["digit_max"]
    if info["scheme"] == "S":
        reach_hi = sum(127 * 256 ** i for i in range(L - 1)) + D[-1] * 256 ** (L - 1)
        reach_lo = -sum(128 * 256 ** i for i in range(L - 1)) - D[-1] * 256 ** (L - 1)
    else:
        reach_hi = sum(255 * 256 ** i for i in range(L - 1)) + D[-1] * 256 ** (L - 1)
        reach_lo = -D[-1] * 256 ** (L - 1)
    assert reach_hi >= half and reach_lo <= -neg
    # the k-block keeps every group's partial sum (plus the carried value) in s32
    B = [sum(D[i] * D[w - i] for i in range(L) if 0 <= w - i < L) for w in range(2 * L - 1)]
    assert info["kb"] * max(B) + info["carry_max"] <= 2 ** 31 - 1
    assert info["kb"] % 128 == 0 and info["kb"] >= 128


def _crt_check(info, p, k):
    q = info["moduli"]
    assert all(math.gcd(a, b) == 1 for i, a in enumerate(q) for b in q[:i])
    cmax = max((p - 1) // 2, (p - 1) - (p - 1) // 2)
    assert math.prod(q) >= 4 * max(k, 1) * cmax * cmax
    D = max(x // 2 for x in q)
    assert info["kb"] * D * D + info["carry_max"] <= 2 ** 31 - 1


@settings(max_examples=300, deadline=None)
@given(p=st.integers(min_value=2, max_value=2 ** 31 - 1), k=st.integers(min_value=0, max_value=1 << 22))
def test_auto_plan_is_exact(ff, p, k):
    info = ff.ff_plan_query(p, k)
    if info["scheme"] == "CRT":
        _crt_check(info, p, k)
    else:
        _limb_check(info, p)
    assert info["k_pad"] % 16 == 0 and info["k_pad"] >= k
    assert info["num_kblocks"] == (-(-k // info["kb"]) if k else 0)


@settings(max_examples=200, deadline=None)
@given(p=st.integers(min_value=2, max_value=2 ** 31 - 1), k=st.integers(min_value=1, max_value=1 << 20),
       scheme=st.sampled_from([1, 2, 3]))
def test_forced_schemes_are_exact(ff, p, k, scheme):
    info = ff.ff_plan_query(p, k, {"scheme": scheme})
    if scheme == 3:
        assert info["scheme"] == "CRT"
        _crt_check(info, p, k)
    else:
        assert info["scheme"] == {1: "S", 2: "T"}[scheme]
        _limb_check(info, p)
