"""The paper's delayed-reduction thresholds, in exact Python integers --
TEST INFRASTRUCTURE (pins for the planner and for the trsm cascade thresholds).

* ``lambda_dot(p, gamma, balanced)`` -- Eq. (1)/(2): the
  largest number lambda of products of residues that can be accumulated
  without reduction, lambda (p-1)^2 < 2^gamma (positive) or
  lambda ((p-1)/2)^2 < 2^(gamma-1) (balanced).
* ``k_winograd(p, gamma, l, balanced)`` -- Corollary 3.4 (l.302-312) as printed.
* ``winograd_v``, ``thm31_bound`` -- Theorem 3.1's v_l and bound (l.284-290,
  App. A.1-A.2); ``k_winograd_exact`` -- the corollary's exact threshold
  (reading R21: the printed "+1" admits up to 2^l unsafe k).
* ``trsm_u_v(M, m, k)`` -- Theorem 4.2 (l.404-420): the bounds u_k, v_k on the
  entries of the integer solution of a unit upper triangular system.
* ``trsm_worst_case(M, m, n)`` -- the system of Corollary 4.3 (l.448-458); it
  attains the bound for the balanced representation m = -M (reading R17).
* ``t_del(p, gamma, balanced)`` -- Eq. (4) (positive) / Eq. (5) (balanced)
  (l.470-482): the largest dimension of a unit triangular system solvable
  over Z with gamma-bit integers.
* ``t_update(p, gamma)`` -- the update threshold of Sec. 4.3 (l.488-496, Table
  at l.522-527): the number of accumulated update products.

Readings: the table's t_update values are reproduced by the
dot-product bound with one carried term, (t+1)(p-1)^2 < 2^53 (reading R6),
capped at 2^31 - 1 - p (an int-sized dimension: p = 5 gives 2147483642 as
printed); t_del is the positive-representation Eq. (4), which reproduces the
table (23, 2, 2) and the text's "34 for Z_3" and "n <= 5 for p = 1001"; the
balanced Eq. (5) with exponent n (not Cor. 4.5's n-1) reproduces "52 for Z_3";
the text's "n <= 6" for balanced p = 1001 is reproduced by neither (garble,
SURVEY §8(c).15).

Parity status: pinned (tests/test_oracle_pins.py::test_paper_thresholds_*,
test_trsm_bound_*; tests/test_oracle_trsm_pins.py; Theorem 3.1 / Cor. 3.2-3.4 by
tests/test_oracle_winograd_bound.py: the App. A.6 witnesses attain thm31_bound
exactly, brute force over all 2 x 2 pairs, SURVEY's k_Winograd values).
"""
from __future__ import annotations


def lambda_dot(p: int, gamma: int = 53, balanced: bool = False) -> int:
    """Largest lambda with lambda (p-1)^2 < 2^gamma (or the balanced Eq. (2))."""
    if balanced:
        h = (p - 1) // 2
        return (2 ** (gamma - 1) - 1) // (h * h)
    return (2 ** gamma - 1) // ((p - 1) ** 2)


def k_winograd(p: int, gamma: int, l: int, balanced: bool = False) -> int:
    """Corollary 3.4: l Winograd levels are safe while k < k_Winograd (returned,
    rounded down: the largest real bound's floor)."""
    if balanced:
        den = (3 ** l * (p - 1)) ** 2
    else:
        den = ((1 + 3 ** l) * (p - 1)) ** 2
    # (2^(gamma+2)/den + 1) 2^l, floor of the exact rational
    return ((2 ** (gamma + 2) + den) * 2 ** l) // den


def trsm_u_v(M: int, m: int, k: int):
    """Theorem 4.2's bounds, in the form its proof (l.430-436), Corollary 4.3
    (l.446) and Corollary 4.5 (m = -M) use:
        u_k = (M-m)/2 (M+1)^k - (M+m)/2 (M-1)^k,
        v_k = (M-m)/2 (M+1)^k + (M+m)/2 (M-1)^k.
    The theorem's own display (l.412-416) swaps (M+m) and (M-m) between the
    two terms; that form fails already at k = 1 (reading R16)."""
    u2 = (M - m) * (M + 1) ** k - (M + m) * (M - 1) ** k      # 2 u_k
    v2 = (M - m) * (M + 1) ** k + (M + m) * (M - 1) ** k      # 2 v_k
    assert u2 % 2 == 0 and v2 % 2 == 0
    return u2 // 2, v2 // 2


def trsm_worst_case(M: int, m: int, n: int):
    """Corollary 4.3's unit upper triangular T (rows ... 1 M m M ...) and b
    (... m M m M from the bottom), over Z, as lists of Python ints."""
    T = [[0] * n for _ in range(n)]
    for i in range(n):
        T[i][i] = 1
        for j in range(i + 1, n):
            T[i][j] = M if (j - i) % 2 == 1 else m
    b = [M if (n - 1 - i) % 2 == 0 else m for i in range(n)]
    return T, b


def solve_unit_upper_over_Z(T, b):
    """Plain back substitution over Z (no division: unit diagonal)."""
    n = len(b)
    x = [0] * n
    for i in range(n - 1, -1, -1):
        x[i] = b[i] - sum(T[i][j] * x[j] for j in range(i + 1, n))
    return x


def t_del(p: int, gamma: int = 53, balanced: bool = False) -> int:
    """Largest n with Eq. (4) (p-1)/2 (p^(n-1) + (p-1)^(n-1)) < 2^gamma, or with
    Eq. (5) (p-1)/2 ((p+1)/2)^n < 2^gamma (balanced)."""
    n = 1
    while True:
        m = n + 1
        if balanced:       # (p-1)/2 ((p+1)/2)^m < 2^gamma, cleared of denominators
            ok = (p - 1) * (p + 1) ** m < 2 ** gamma * 2 ** (m + 1)
        else:
            ok = (p - 1) * (p ** (m - 1) + (p - 1) ** (m - 1)) < 2 ** (gamma + 1)
        if not ok:
            return n
        n = m


def t_update(p: int, gamma: int = 53) -> int:
    """Largest t with (t+1)(p-1)^2 < 2^gamma, capped at 2^31 - 1 - p."""
    t = (2 ** gamma - 1) // ((p - 1) ** 2) - 1
    return min(t, 2 ** 31 - 1 - p)


# ---------------------------------------------------------------- Thm 3.1 / Cor 3.4

def winograd_v(M: int, m: int, l: int) -> int:
    """v_l of Appendix A.1: v_l = (1+3^l)/2 M + (1-3^l)/2 m
    (both halves are integers since 3^l is odd)."""
    return (1 + 3 ** l) // 2 * M + (1 - 3 ** l) // 2 * m


def thm31_bound(MA: int, mA: int, MB: int, mB: int, k: int, l: int) -> int:
    """Theorem 3.1: every intermediate value z of A x B with
    l >= 1 recursive Winograd levels has |z| <= v_l^A v_l^B floor(k / 2^l)."""
    return winograd_v(MA, mA, l) * winograd_v(MB, mB, l) * (k // 2 ** l)


def k_winograd_exact(p: int, gamma: int, l: int, balanced: bool = False) -> int:
    """The exact form of Corollary 3.4 (reading R21): the smallest k for
    which Theorem 3.1's bound reaches 2^gamma, so l levels are safe iff k < it.

    With X = 2^gamma / v_l^2 (= the paper's 2^(gamma+2)/((1+3^l)(p-1))^2, or
    2^(gamma+2)/(3^l (p-1))^2 balanced), floor(k/2^l) v_l^2 < 2^gamma holds iff
    floor(k/2^l) < X iff k < ceil(X) 2^l.  The paper's (X + 1) 2^l (floored)
    agrees only when 0 < frac(X) 2^l < 1; otherwise it admits up to 2^l values
    of k whose bound reaches 2^gamma (p = 65521, l = 1, balanced: 1865047 by
    the printed formula vs 1865046)."""
    if balanced:
        h = (p - 1) // 2 if p % 2 else p // 2
        v = winograd_v(h, -h, l)
    else:
        v = winograd_v(p - 1, 0, l)
    return -(-(2 ** gamma) // (v * v)) * 2 ** l
