"""Winograd-level oracle pieces, in exact Python integers -- TEST INFRASTRUCTURE.

* ``opcount(n, l)`` -- the arithmetic-operation count behind PAPER.md Table 1
  (l.245-253): the classical algorithm on n x n matrices costs n^3
  multiplications and n^2 (n-1) additions, 2n^3 - n^2 in total (l.239:
  "MM(n) = 2n^3 ... means ... 2n^3 + O(n^2)"); one Winograd level replaces it
  by 7 half-size products plus 15 half-size additions (Winograd's variant,
  l.235-243; Table 2 lists its 8 pre-additions S1..S4, T1..T4 and 7 post-
  additions U1..U7).  Pinned against all 25 printed cells of Table 1.

* ``schedule_table2(...)`` -- PAPER.md Table 2 (l.263-276), "Schedule for
  operation C <- alpha A x B + beta C with 3 temporaries", executed step by
  step over Z on quadrants.  Step 16 is printed "P4 = alpha A12 T4 - beta C21";
  Appendix A.2 (l.935) and the algebra require A22 (reading R9).
  ``step16_operand`` selects which, so the tests can show the printed form is
  wrong and the fixed form equals alpha*A*B + beta*C.

* ``witness(l, MA, mA, MB, mB)`` -- the optimality witnesses A_l, B_l of
  Appendix A.6 (l.1087-1117); ``winograd_traced(A, B, l)`` -- l levels of
  App. A.2's form over Z returning the product and the largest |intermediate|
  (the quantity Theorem 3.1 bounds).

Parity status: pinned (tests/test_oracle_pins.py::test_table1_*, test_table2_*;
tests/test_oracle_winograd_bound.py: traced product = plain product, witnesses
attain Theorem 3.1's bound, exhaustive 2 x 2 optimality).
"""
from __future__ import annotations


def opcount(n: int, l: int) -> int:
    """Field operations for n x n times n x n with l Winograd levels (Table 1)."""
    if l == 0:
        return 2 * n ** 3 - n ** 2
    if n % 2:
        raise ValueError("n must be even at every Winograd level")
    h = n // 2
    return 7 * opcount(h, l - 1) + 15 * h * h


def _mm(X, Y):
    k = len(Y)
    return [[sum(X[i][t] * Y[t][j] for t in range(k)) for j in range(len(Y[0]))]
            for i in range(len(X))]


def _add(X, Y, s=1):
    return [[x + s * y for x, y in zip(rx, ry)] for rx, ry in zip(X, Y)]


def _scale(a, X):
    return [[a * x for x in r] for r in X]


def _quad(M, r, c):
    h, w = len(M) // 2, len(M[0]) // 2
    return [row[c * w:(c + 1) * w] for row in M[r * h:(r + 1) * h]]


def schedule_table2(alpha, A, B, beta, C, step16_operand="A22"):
    """One Winograd level of Table 2 over Z; returns the new C (lists of ints).

    A is m x k, B is k x n, C is m x n, all even dimensions.  The three
    temporaries X1, X2, X3 of the "loc." column are kept as named variables.
    """
    A11, A12, A21, A22 = _quad(A, 0, 0), _quad(A, 0, 1), _quad(A, 1, 0), _quad(A, 1, 1)
    B11, B12, B21, B22 = _quad(B, 0, 0), _quad(B, 0, 1), _quad(B, 1, 0), _quad(B, 1, 1)
    C11, C12, C21, C22 = _quad(C, 0, 0), _quad(C, 0, 1), _quad(C, 1, 0), _quad(C, 1, 1)
    A4 = {"A22": A22, "A12": A12}[step16_operand]

    X1 = _add(A21, A22)                               # 1  S1 = A21 + A22
    X2 = _add(B12, B11, -1)                           # 2  T1 = B12 - B11
    X3 = _scale(alpha, _mm(X1, X2))                   # 3  P5 = alpha S1 T1
    C22 = _add(X3, _scale(beta, C22))                 # 4  C22 = P5 + beta C22
    C12 = _add(X3, _scale(beta, C12))                 # 5  C12 = P5 + beta C12
    X1 = _add(X1, A11, -1)                            # 6  S2 = S1 - A11
    X2 = _add(B22, X2, -1)                            # 7  T2 = B22 - T1
    X3 = _scale(alpha, _mm(A11, B11))                 # 8  P1 = alpha A11 B11
    C11 = _add(X3, _scale(beta, C11))                 # 9  C11 = P1 + beta C11
    X3 = _add(_scale(alpha, _mm(X1, X2)), X3)         # 10 U2 = alpha S2 T2 + P1
    C11 = _add(_scale(alpha, _mm(A12, B21)), C11)     # 11 U1 = alpha A12 B21 + C11
    X1 = _add(A12, X1, -1)                            # 12 S4 = A12 - S2
    X2 = _add(X2, B21, -1)                            # 13 T4 = T2 - B21
    C12 = _add(_scale(alpha, _mm(X1, B22)), C12)      # 14 C12 = alpha S4 B22 + C12
    C12 = _add(X3, C12)                               # 15 U5 = U2 + C12
    C21 = _add(_scale(alpha, _mm(A4, X2)), _scale(beta, C21), -1)  # 16 P4 = alpha A22 T4 - beta C21
    X1 = _add(A11, A21, -1)                           # 17 S3 = A11 - A21
    X2 = _add(B22, B12, -1)                           # 18 T3 = B22 - B12
    X3 = _add(_scale(alpha, _mm(X1, X2)), X3)         # 19 U3 = alpha S3 T3 + U2
    C22 = _add(X3, C22)                               # 20 U7 = U3 + C22
    C21 = _add(X3, C21, -1)                           # 21 U6 = U3 - C21

    top = [r1 + r2 for r1, r2 in zip(C11, C12)]
    bot = [r1 + r2 for r1, r2 in zip(C21, C22)]
    return top + bot


# ---------------------------------------------------------------- Thm 3.1 traced

def witness(l: int, MA: int, mA: int, MB: int, mB: int):
    """Appendix A.6: the square matrices A_l, B_l of order
    2^l on which l recursive Winograd levels reach Theorem 3.1's bound:
        A_1 = [[mA, 0], [MA, MA]],  B_1 = [[MB, mB], [0, MB]],
        A_{l+1} = [[conj(A_l), 0], [A_l, A_l]],  B_{l+1} = [[B_l, conj(B_l)], [0, B_l]],
    conj(x) = M + m - x."""
    A = [[mA, 0], [MA, MA]]
    B = [[MB, mB], [0, MB]]
    for _ in range(l - 1):
        n = len(A)
        Ab = [[MA + mA - x for x in r] for r in A]
        Bb = [[MB + mB - x for x in r] for r in B]
        A = [Ab[i] + [0] * n for i in range(n)] + [A[i] + A[i] for i in range(n)]
        B = [B[i] + Bb[i] for i in range(n)] + [[0] * n + B[i] for i in range(n)]
    return A, B


def _sub(X, Y):
    return _add(X, Y, -1)


def winograd_traced(A, B, l: int):
    """A x B over Z with l recursive levels of Winograd's algorithm in the form of
    Appendix A.2, classical products at the leaves.

    Returns (product, max |z|) where z runs over EVERY intermediate value: the
    pre-additions S1..S4 / T1..T4 (and the partial sums inside them), the seven
    recursive products P1..P7, the post-additions U1..U7, and the partial sums
    of every leaf dot product (in order of the inner index).  No reduction
    anywhere: this is the quantity Theorem 3.1 bounds.  Dimensions of A (m x k)
    and B (k x n) must be divisible by 2^l."""
    peak = [0]

    def note(X):
        for r in X:
            for x in r:
                if abs(x) > peak[0]:
                    peak[0] = abs(x)
        return X

    def classic(X, Y):
        k = len(Y)
        out = []
        for i in range(len(X)):
            row = []
            for j in range(len(Y[0])):
                s = 0
                for t in range(k):
                    s += X[i][t] * Y[t][j]
                    if abs(s) > peak[0]:
                        peak[0] = abs(s)
                row.append(s)
            out.append(row)
        return out

    def rec(X, Y, j):
        if j == 0:
            return classic(X, Y)
        A11, A12, A21, A22 = _quad(X, 0, 0), _quad(X, 0, 1), _quad(X, 1, 0), _quad(X, 1, 1)
        B11, B12, B21, B22 = _quad(Y, 0, 0), _quad(Y, 0, 1), _quad(Y, 1, 0), _quad(Y, 1, 1)
        S1 = note(_add(A21, A22))
        S2 = note(_sub(S1, A11))
        S3 = note(_sub(A11, A21))
        S4 = note(_sub(A12, S2))
        T1 = note(_sub(B12, B11))
        T2 = note(_sub(B22, T1))
        T3 = note(_sub(B22, B12))
        T4 = note(_sub(T2, B21))
        P1 = note(rec(A11, B11, j - 1))
        P2 = note(rec(A12, B21, j - 1))
        P3 = note(rec(S4, B22, j - 1))
        P4 = note(rec(A22, T4, j - 1))
        P5 = note(rec(S1, T1, j - 1))
        P6 = note(rec(S2, T2, j - 1))
        P7 = note(rec(S3, T3, j - 1))
        U1 = note(_add(P1, P2))
        U2 = note(_add(P1, P6))
        U3 = note(_add(U2, P7))
        U4 = note(_add(U2, P5))
        U5 = note(_add(U4, P3))
        U6 = note(_sub(U3, P4))
        U7 = note(_add(U3, P5))
        top = [r1 + r2 for r1, r2 in zip(U1, U5)]
        bot = [r1 + r2 for r1, r2 in zip(U6, U7)]
        return top + bot

    return rec(A, B, l), peak[0]
