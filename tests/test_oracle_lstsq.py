"""Pins for the oracle's least-squares forward substitution (N > n equations;
PAPER.md:258-262; reading R18): exact rational least squares on tiny
systems, the square case, a consistent overdetermined system, and the
normal-equation residual."""
from fractions import Fraction

import numpy as np
import pytest

import mdinputs
import oracle
from tests.exact import cadd, cdiv, cmul, csub, series_err_exact, solve_exact, value

U = {L: 2.0 ** (-53 * L) for L in (2, 3, 4, 5, 8, 10)}


def conj(a):
    return (a[0], -a[1])


def exact_lstsq(jac, rhs):
    """dx_j = (A_0^H A_0)^-1 A_0^H (b_j - sum_{i>=1} A_i dx_{j-i}) with Fractions."""
    N, n, _, L, D = jac.shape
    A = [[[(value(jac[p, q, 0, :, k]), value(jac[p, q, 1, :, k])) for q in range(n)] for p in range(N)]
         for k in range(D)]
    b = [[(value(rhs[p, 0, :, k]), value(rhs[p, 1, :, k])) for p in range(N)] for k in range(D)]
    G = [[(Fraction(0), Fraction(0))] * n for _ in range(n)]
    for p in range(n):
        for q in range(n):
            acc = (Fraction(0), Fraction(0))
            for r in range(N):
                acc = cadd(acc, cmul(conj(A[0][r][p]), A[0][r][q]))
            G[p][q] = acc
    dx = []
    for j in range(D):
        r = list(b[j])
        for i in range(1, j + 1):
            for p in range(N):
                for q in range(n):
                    r[p] = csub(r[p], cmul(A[i][p][q], dx[j - i][q]))
        y = []
        for p in range(n):
            acc = (Fraction(0), Fraction(0))
            for t in range(N):
                acc = cadd(acc, cmul(conj(A[0][t][p]), r[t]))
            y.append(acc)
        dx.append(solve_exact(G, y))
    return [[dx[j][q] for j in range(D)] for q in range(n)]


@pytest.mark.parametrize("N,n,degree,L", [(3, 2, 0, 2), (3, 2, 2, 4), (4, 2, 3, 2), (5, 3, 1, 3)])
def test_exact_rational_tiny(N, n, degree, L):
    t = mdinputs.random_toeplitz_rect(300 + N * 10 + n, N, n, degree, L)
    dx = oracle.toeplitz_lstsq(t.jac, t.rhs)
    ex = exact_lstsq(t.jac, t.rhs)
    for q in range(n):
        assert series_err_exact(dx[q], ex[q]) <= 64 * U[L], series_err_exact(dx[q], ex[q]) / U[L]


def test_square_case_equals_the_solve():
    t = mdinputs.random_toeplitz(17, 6, 7, 4)
    a, _ = oracle.toeplitz_solve(t.jac, t.rhs)
    b = oracle.toeplitz_lstsq(t.jac, t.rhs)
    assert oracle.series_err(a, b).max() <= 16 * U[4]


def test_consistent_overdetermined_system_recovers_the_solution():
    """b(t) = A(t) x*(t) mod t^D, formed exactly: the least-squares solution is x*."""
    N, n, d, L = 6, 3, 4, 3
    t = mdinputs.random_toeplitz_rect(21, N, n, d, L)
    xs = mdinputs.unit_circle_series(mdinputs.SplitMix64(21, "extra"), n, d + 1, L, "random")
    D = d + 1
    A = [[[(value(t.jac[p, q, 0, :, k]), value(t.jac[p, q, 1, :, k])) for k in range(D)] for q in range(n)]
         for p in range(N)]
    X = [[(value(xs[q, 0, :, k]), value(xs[q, 1, :, k])) for k in range(D)] for q in range(n)]
    rhs = np.zeros((N, 2, L, D))
    from tests.exact import greedy
    for p in range(N):
        for k in range(D):
            acc = (Fraction(0), Fraction(0))
            for q in range(n):
                for i in range(k + 1):
                    acc = cadd(acc, cmul(A[p][q][i], X[q][k - i]))
            rhs[p, 0, :, k] = greedy(acc[0], L)
            rhs[p, 1, :, k] = greedy(acc[1], L)
    dx = oracle.toeplitz_lstsq(t.jac, rhs)
    assert oracle.series_err(dx, xs).max() <= 2.0 ** (-53 * L + 16)
