"""Pins for Theorem 3.1 / Corollaries 3.2-3.4 and the
optimality witnesses of Appendix A.6 (l.1087-1117): oracle/bounds.py
(winograd_v, thm31_bound, k_winograd, k_winograd_exact) and
oracle/winograd.py (witness, winograd_traced).

What pins what (none of these re-types a formula against itself):
* the traced Winograd recursion is pinned to the plain product (any slip in
  the A.2 pre-/post-additions changes the product) and, exhaustively over
  every 2 x 2 pair with entries in a small range, its maximum intermediate is
  the theorem's bound -- attained and never exceeded (brute force);
* on the A.6 witnesses the traced maximum equals thm31_bound for l = 1..3 and
  several ranges (optimality, the paper's own construction);
* Cor 3.2 / 3.3 are the theorem specialised to [0, p-1] / [-(p-1)/2, (p-1)/2]
  (asserted on the theorem's value, not on a restated corollary formula);
* Cor 3.4: SURVEY §8(f)'s [calc] values of the printed formula, and the
  defining property of the threshold checked against thm31_bound at the
  boundary -- which the printed formula fails for p = 65521 (reading R21).
"""
import itertools
import random

import pytest

from oracle import bounds, winograd


def _mm(X, Y):
    return [[sum(X[i][t] * Y[t][j] for t in range(len(Y))) for j in range(len(Y[0]))]
            for i in range(len(X))]


def _kron_ones(X, d, axis):
    """Replicate every entry d times along the inner dimension (axis 1 for A:
    columns, axis 0 for B: rows): the witness stretched to k = 2^l d."""
    if axis == 1:
        return [[x for x in r for _ in range(d)] for r in X]
    return [list(r) for r in X for _ in range(d)]


@pytest.mark.parametrize("l", [1, 2, 3])
def test_traced_winograd_is_the_product(l):
    rng = random.Random(31 + l)
    n = 2 ** l
    for shape in [(n, n, n), (2 * n, n, 3 * n), (n, 4 * n, 2 * n)]:
        m, k, nn = shape
        A = [[rng.randint(-50, 50) for _ in range(k)] for _ in range(m)]
        B = [[rng.randint(-50, 50) for _ in range(nn)] for _ in range(k)]
        P, peak = winograd.winograd_traced(A, B, l)
        assert P == _mm(A, B)
        assert peak <= bounds.thm31_bound(50, -50, 50, -50, k, l)


def test_exhaustive_2x2_max_intermediate_is_the_bound():
    # every A, B in [m, M]^{2x2}: the theorem's bound is never exceeded and is
    # attained (optimality) -- brute force over 4^8 pairs per range
    for (MA, mA, MB, mB) in [(2, -1, 2, -1), (2, 0, 1, -1), (1, -1, 2, -2)]:
        vals_a = range(mA, MA + 1)
        vals_b = range(mB, MB + 1)
        best = 0
        for a in itertools.product(vals_a, repeat=4):
            A = [[a[0], a[1]], [a[2], a[3]]]
            for b in itertools.product(vals_b, repeat=4):
                B = [[b[0], b[1]], [b[2], b[3]]]
                P, peak = winograd.winograd_traced(A, B, 1)
                assert peak <= bounds.thm31_bound(MA, mA, MB, mB, 2, 1)
                best = max(best, peak)
        assert best == bounds.thm31_bound(MA, mA, MB, mB, 2, 1)


@pytest.mark.parametrize("l", [1, 2, 3])
@pytest.mark.parametrize("rng_", [(7, -3, 5, -2), (3, -3, 3, -3), (10, 0, 10, 0), (4, -1, 6, -6)])
def test_appendix_a6_witnesses_attain_the_bound(l, rng_):
    MA, mA, MB, mB = rng_
    A, B = winograd.witness(l, MA, mA, MB, mB)
    assert len(A) == len(B) == 2 ** l
    assert all(mA <= x <= MA for r in A for x in r)
    assert all(mB <= x <= MB for r in B for x in r)
    P, peak = winograd.winograd_traced(A, B, l)
    assert P == _mm(A, B)
    assert peak == bounds.thm31_bound(MA, mA, MB, mB, 2 ** l, l)
    # stretched along k (k = 2^l d): the bound's floor(k / 2^l) factor is attained too
    for d in (2, 3):
        Ad, Bd = _kron_ones(A, d, 1), _kron_ones(B, d, 0)
        P, peak = winograd.winograd_traced(Ad, Bd, l)
        assert P == _mm(Ad, Bd)
        assert peak == bounds.thm31_bound(MA, mA, MB, mB, 2 ** l * d, l)


def test_witness_recursion_first_steps():
    # A.6's definition written out for l = 2 (conj(x) = M + m - x)
    A, B = winograd.witness(2, 5, -2, 4, -1)
    assert A == [[-2 + 5 - (-2), 5 - 2 - 0, 0, 0],
                 [5 - 2 - 5, 5 - 2 - 5, 0, 0],
                 [-2, 0, -2, 0],
                 [5, 5, 5, 5]]
    assert B == [[4, -1, 4 - 1 - 4, 4 - 1 + 1],
                 [0, 4, 3, 4 - 1 - 4],
                 [0, 0, 4, -1],
                 [0, 0, 0, 4]]


@pytest.mark.parametrize("p", [3, 251, 65521, 8388593, 67108859])
@pytest.mark.parametrize("l", [1, 2, 3])
def test_corollaries_32_33_are_the_theorem_on_the_two_representations(p, l):
    k = 2 ** l * 5
    pos = bounds.thm31_bound(p - 1, 0, p - 1, 0, k, l)
    h = (p - 1) // 2
    bal = bounds.thm31_bound(h, -h, h, -h, k, l)
    # Cor 3.2: ((1+3^l)/2)^2 floor(k/2^l) (p-1)^2 ; Cor 3.3: (3^l/2)^2 floor(k/2^l) (p-1)^2
    assert 4 * pos == (1 + 3 ** l) ** 2 * 5 * (p - 1) ** 2
    assert 4 * bal == 9 ** l * 5 * (p - 1) ** 2
    # the balanced bound is smaller for l >= 1 (Cor 3.3 "can be improved")
    assert bal < pos


def test_k_winograd_printed_formula_survey_values():
    # SURVEY §8(f) NEXT-3 [calc]: k_Winograd(l = 1), balanced, gamma = 53
    assert [bounds.k_winograd(p, 53, 1, balanced=True) for p in (65521, 8388593, 67108859)] == \
        [1865047, 115, 3]
    assert [bounds.k_winograd(p, 53, 1) for p in (65521, 8388593, 67108859)] == [1049090, 66, 3]


@pytest.mark.parametrize("gamma", [24, 31, 53])
@pytest.mark.parametrize("p", [3, 5, 251, 65521, 1048583, 8388593, 67108859])
@pytest.mark.parametrize("l", [1, 2, 3])
@pytest.mark.parametrize("balanced", [False, True])
def test_k_winograd_exact_is_the_threshold_of_theorem_31(gamma, p, l, balanced):
    kw = bounds.k_winograd_exact(p, gamma, l, balanced)
    if balanced:
        h = (p - 1) // 2
        b = lambda k: bounds.thm31_bound(h, -h, h, -h, k, l)  # noqa: E731
    else:
        b = lambda k: bounds.thm31_bound(p - 1, 0, p - 1, 0, k, l)  # noqa: E731
    # defining property: k_W - 1 fits gamma bits, k_W does not (and k_W is the
    # first such k: the bound is monotone in k)
    assert b(kw) >= 2 ** gamma
    if kw - 1 >= 2 ** l:
        assert b(kw - 1) < 2 ** gamma
    # the printed formula never admits less than the exact threshold, and at
    # most 2^l more values of k (its "+1" stands for the ceiling)
    kp = bounds.k_winograd(p, gamma, l, balanced)
    assert kw <= kp <= kw + 2 ** l


def test_printed_cor34_admits_an_unsafe_k_at_p_65521():
    # reading R21: for p = 65521, l = 1, balanced, gamma = 53 the printed
    # k_Winograd = 1865047 admits k = 1865046, whose Theorem 3.1 bound exceeds 2^53
    h = 65520 // 2
    kp = bounds.k_winograd(65521, 53, 1, balanced=True)
    assert kp == 1865047
    assert bounds.thm31_bound(h, -h, h, -h, kp - 1, 1) >= 2 ** 53
    assert bounds.k_winograd_exact(65521, 53, 1, balanced=True) == 1865046
    assert bounds.thm31_bound(h, -h, h, -h, 1865045, 1) < 2 ** 53
    # and a witness-shaped input at k = kp - 1 really reaches past 2^53: the
    # l = 1 witness stretched to k = 2 d has peak v^2 d (attained, as above)
    d = (kp - 1) // 2
    assert (3 * h) ** 2 * d >= 2 ** 53
