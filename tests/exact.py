"""Exact rational helpers for the pins (Python fractions; tests only).

Every binary64 is a dyadic rational, so sums and products of limbs are
formed exactly with fractions.Fraction; float(Fraction) is correctly rounded
(round-to-nearest-even), which gives an independent greedy L-limb rounding.
"""
import math
from fractions import Fraction
from typing import List, Sequence

import numpy as np


def F(x) -> Fraction:
    return Fraction(float(x))


def value(limbs: Sequence[float]) -> Fraction:
    return sum((Fraction(float(v)) for v in limbs), Fraction(0))


def greedy(X: Fraction, L: int) -> List[float]:
    """limb_0 = RN(X), limb_1 = RN(X - limb_0), ... (L limbs)."""
    out = []
    for _ in range(L):
        v = float(X)
        out.append(v)
        X -= Fraction(v)
    return out


def series_value(s: np.ndarray):
    """[2][L][D] float array -> list of complex Fractions (re, im) per coefficient."""
    _, L, D = s.shape
    return [(value(s[0, :, k]), value(s[1, :, k])) for k in range(D)]


def series_from_exact(coefs, L: int) -> np.ndarray:
    """list of (re, im) Fractions -> greedy-rounded [2][L][D] array."""
    D = len(coefs)
    out = np.zeros((2, L, D))
    for k, (re, im) in enumerate(coefs):
        out[0, :, k] = greedy(Fraction(re), L)
        out[1, :, k] = greedy(Fraction(im), L)
    return out


def cmul(a, b):
    return (a[0] * b[0] - a[1] * b[1], a[0] * b[1] + a[1] * b[0])


def cadd(a, b):
    return (a[0] + b[0], a[1] + b[1])


def conv(x, y, D):
    """exact truncated product of coefficient lists."""
    z = []
    for k in range(D):
        acc = (Fraction(0), Fraction(0))
        for i in range(k + 1):
            acc = cadd(acc, cmul(x[i], y[k - i]))
        z.append(acc)
    return z


def series_err_exact(approx: np.ndarray, exact) -> float:
    """max_k |approx_k - exact_k| / max(max_k |exact_k|, 1), complex modulus,
    computed from exact differences (SURVEY C2.9 reading)."""
    _, L, D = approx.shape
    maxd, maxe = 0.0, 0.0
    for k in range(D):
        dr = value(approx[0, :, k]) - exact[k][0]
        di = value(approx[1, :, k]) - exact[k][1]
        maxd = max(maxd, math.hypot(float(dr), float(di)))
        maxe = max(maxe, math.hypot(float(exact[k][0]), float(exact[k][1])))
    return maxd / max(maxe, 1.0)


def csub(a, b):
    return (a[0] - b[0], a[1] - b[1])


def cdiv(a, b):
    den = b[0] * b[0] + b[1] * b[1]
    return ((a[0] * b[0] + a[1] * b[1]) / den, (a[1] * b[0] - a[0] * b[1]) / den)


def solve_exact(A, b):
    """x with A x = b over complex Fractions (Gauss-Jordan, any nonzero pivot)."""
    n = len(A)
    M = [list(A[i]) + [b[i]] for i in range(n)]
    for k in range(n):
        p = next(i for i in range(k, n) if M[i][k] != (0, 0))
        M[k], M[p] = M[p], M[k]
        for i in range(n):
            if i != k and M[i][k] != (0, 0):
                f = cdiv(M[i][k], M[k][k])
                M[i] = [csub(M[i][c], cmul(f, M[k][c])) for c in range(n + 1)]
    return [cdiv(M[i][n], M[i][i]) for i in range(n)]


def toeplitz_exact(jac: np.ndarray, rhs: np.ndarray):
    """Exact forward substitution on float inputs:
    returns dx[q] = list of D complex Fractions."""
    n, _, _, L, D = jac.shape
    A = [[[(value(jac[p, q, 0, :, k]), value(jac[p, q, 1, :, k])) for q in range(n)] for p in range(n)]
         for k in range(D)]
    b = [[(value(rhs[p, 0, :, k]), value(rhs[p, 1, :, k])) for p in range(n)] for k in range(D)]
    dx = []
    for j in range(D):
        r = list(b[j])
        for i in range(1, j + 1):
            for p in range(n):
                for q in range(n):
                    r[p] = csub(r[p], cmul(A[i][p][q], dx[j - i][q]))
        dx.append(solve_exact(A[0], r))
    return [[dx[j][q] for j in range(D)] for q in range(n)]
