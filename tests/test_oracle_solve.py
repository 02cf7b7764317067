"""Pins for the oracle's block lower-triangular Toeplitz forward substitution
(§4).

The oracle factors A_0 once (LU, partial pivoting) and solves
A_0 dx_j = b_j - sum_{i=1..j} A_i dx_{j-i} for j = 0..d.  It is pinned to
exact rational forward substitution on tiny systems, an exactly solvable
permutation case (which also fixes the pivot order), the truncation
invariant, the residual A(t) dx(t) - b(t) formed exactly, and the precision
ladder L vs L+2.
"""
from fractions import Fraction

import numpy as np
import pytest

import mdinputs
import oracle
from tests.exact import cmul, csub, series_err_exact, toeplitz_exact, value

U = {L: 2.0 ** (-53 * L) for L in (2, 3, 4, 5, 8, 10)}


@pytest.mark.parametrize("n,degree,L", [(1, 0, 2), (1, 4, 4), (2, 0, 3), (2, 3, 2), (3, 2, 4), (3, 3, 8),
                                        (2, 2, 10)])
def test_exact_rational_tiny(n, degree, L):
    """Against exact Fraction forward substitution: a few units of 2^-53L."""
    t = mdinputs.random_toeplitz(100 + 7 * n + degree, n, degree, L)
    dx, piv = oracle.toeplitz_solve(t.jac, t.rhs, nthreads=1)
    ex = toeplitz_exact(t.jac, t.rhs)
    for q in range(n):
        assert series_err_exact(dx[q], ex[q]) <= 64 * U[L], (q, series_err_exact(dx[q], ex[q]) / U[L])
    assert sorted(set(piv.tolist()) | set(range(n))) == list(range(n))
    assert all(k <= piv[k] < n for k in range(n))


@pytest.mark.parametrize("L", [2, 5, 10])
def test_permutation_case_exact(L):
    """A_0 = P diag(s) with s_k = +-2^e or +-i 2^e, A_i = 0 (i >= 1): dx_j =
    diag(s)^-1 P^T b_j exactly, and partial pivoting must pick row sigma(k)
    at step k (the only nonzero in column k among the remaining rows)."""
    n, D = 5, 4
    rng = np.random.default_rng(3)
    sigma = [2, 0, 4, 1, 3]                      # A_0[sigma[k]][k] = s_k
    s = [(2.0 ** e, 0.0) if k % 2 == 0 else (0.0, -(2.0 ** e)) for k, e in enumerate([1, -3, 0, 5, -2])]
    jac = np.zeros((n, n, 2, L, D))
    for k in range(n):
        jac[sigma[k], k, 0, 0, 0], jac[sigma[k], k, 1, 0, 0] = s[k]
    rhs = np.zeros((n, 2, L, D))
    rhs[:, :, 0, :] = rng.integers(-50, 50, size=(n, 2, D)).astype(np.float64)
    dx, piv = oracle.toeplitz_solve(jac, rhs, nthreads=1)
    # expected pivot rows: LAPACK-style swaps realising sigma
    rows = list(range(n))
    exp_piv = []
    for k in range(n):
        r = rows.index(sigma[k])
        exp_piv.append(r)
        rows[k], rows[r] = rows[r], rows[k]
    assert piv.tolist() == exp_piv
    for k in range(n):
        for j in range(D):
            b = (Fraction(rhs[sigma[k], 0, 0, j]), Fraction(rhs[sigma[k], 1, 0, j]))
            den = s[k][0] ** 2 + s[k][1] ** 2
            want = ((b[0] * Fraction(s[k][0]) + b[1] * Fraction(s[k][1])) / Fraction(den),
                    (b[1] * Fraction(s[k][0]) - b[0] * Fraction(s[k][1])) / Fraction(den))
            assert value(dx[k, 0, :, j]) == want[0] and value(dx[k, 1, :, j]) == want[1]


def test_truncation_invariant():
    """dx_0..dx_{d'} depend only on A_0..A_{d'} and b_0..b_{d'}: solving the
    truncated system reproduces the leading coefficients bit for bit."""
    t = mdinputs.random_toeplitz(11, 6, 9, 4)
    full, p1 = oracle.toeplitz_solve(t.jac, t.rhs)
    part, p2 = oracle.toeplitz_solve(*(lambda u: (u.jac, u.rhs))(t.truncate(4)))
    assert np.array_equal(p1, p2)
    assert np.array_equal(full[..., :5], part)


def test_scalar_case_is_series_division():
    """n = 1: dx = b / a, the series quotient — compared
    with the exact rational quotient b * a^-1 mod t^D."""
    L, D = 3, 7
    t = mdinputs.random_toeplitz(12, 1, D - 1, L)
    dx, _ = oracle.toeplitz_solve(t.jac, t.rhs)
    a = [(value(t.jac[0, 0, 0, :, k]), value(t.jac[0, 0, 1, :, k])) for k in range(D)]
    b = [(value(t.rhs[0, 0, :, k]), value(t.rhs[0, 1, :, k])) for k in range(D)]
    # exact quotient by the recurrence q_k = (b_k - sum_{i>=1} a_i q_{k-i}) / a_0
    from tests.exact import cdiv
    q = []
    for k in range(D):
        r = b[k]
        for i in range(1, k + 1):
            r = csub(r, cmul(a[i], q[k - i]))
        q.append(cdiv(r, a[0]))
    assert series_err_exact(dx[0], q) <= 16 * U[L]


def test_residual_exact():
    """A(t) dx(t) - b(t) = O(u) coefficientwise, formed exactly (dd config shape
    at d = 7): |res_k| <= 64 u (|b_k| + sum_q sum_i |A_i||dx_{k-i}|)."""
    t = mdinputs.toeplitz_config("dd").truncate(7)
    n, D, L = t.n, t.D, t.limbs
    dx, _ = oracle.toeplitz_solve(t.jac, t.rhs)
    X = [[(value(dx[q, 0, :, k]), value(dx[q, 1, :, k])) for k in range(D)] for q in range(n)]
    for p in range(n):
        for k in range(D):
            res = (value(t.rhs[p, 0, :, k]), value(t.rhs[p, 1, :, k]))
            scale = abs(complex(float(res[0]), float(res[1])))
            for q in range(n):
                for i in range(k + 1):
                    a = (value(t.jac[p, q, 0, :, i]), value(t.jac[p, q, 1, :, i]))
                    prod = cmul(a, X[q][k - i])
                    res = csub(res, prod)
                    scale += abs(complex(float(prod[0]), float(prod[1])))
            assert abs(complex(float(res[0]), float(res[1]))) <= 64 * U[L] * scale


@pytest.mark.parametrize("name,degree", [("dd", 15), ("qd", 15)])
def test_precision_ladder(name, degree):
    """Oracle at L against the same inputs solved at L+2: within tol(L)/4
    (the GPU parity tolerance, reading R12)."""
    tol = {2: 1e-29, 4: 1e-61}
    t = mdinputs.toeplitz_config(name).truncate(degree)
    dx, _ = oracle.toeplitz_solve(t.jac, t.rhs)
    hi, _ = oracle.toeplitz_solve(t.jac, t.rhs, limbs=t.limbs + 2)
    err = oracle.series_err(dx, np.ascontiguousarray(hi[:, :, :t.limbs]))
    assert err.max() <= tol[t.limbs] / 4


def test_singular_detected():
    t = mdinputs.random_toeplitz(13, 3, 2, 2)
    jac = t.jac.copy()
    jac[:, 1, :, :, 0] = 0.0       # column 1 of A_0 is zero
    with pytest.raises(oracle.SingularError):
        oracle.toeplitz_solve(jac, t.rhs)
