"""Pins for Newton's method on power series (oracle.newton; PAPER.md:253-265,
§3 circle demo PAPER.md:183-208).

The circle system f = (s(t) - y, x^2 + y^2 - 1), s the degree-7 Taylor
polynomial of sin, started at (1, 0) with truncation degree 8: the paper
prints the x-series 1 - 0.5 t^2 + 4.16666666666667E-02 t^4 -
1.38888888888889E-03 t^6 + 2.48015873015868E-05 t^8, the
Taylor series of cos.  A linear system converges in one
step (the second update is at the rounding level).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import mdinputs
import oracle
from tests.exact import series_err_exact, value
from tests.test_oracle_evaldiff import const_series, make_si

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))["circle"]


def circle_system(L, x0=(1, 0)):
    d = GOLD["degree"]
    D = d + 1
    s_coef = [Fraction(c) for c in GOLD["s_coefficients"]]
    polys = [[[], [(1, 1)]], [[(0, 2)], [(1, 2)], []]]
    coeffs = [const_series(s_coef, L, D), const_series([-1], L, D), const_series([1], L, D),
              const_series([1], L, D), const_series([-1], L, D)]
    x = [const_series([x0[0]], L, D), const_series([x0[1]], L, D)]
    return make_si(2, polys, coeffs, x, d, L)


@pytest.mark.parametrize("L", (2, 4, 8))
def test_circle_demo_converges_to_cos(L):
    si = circle_system(L)
    x, norms = oracle.newton(si, 8, nthreads=2)   # the paper's cap for degree 8 (§6)
    cos = [(Fraction(c), Fraction(0)) for c in GOLD["cos_coefficients"]]
    sin = [(Fraction(c), Fraction(0)) for c in GOLD["s_coefficients"]]
    assert series_err_exact(x[0], cos) <= 64 * 2.0 ** (-53 * L)
    assert series_err_exact(x[1], sin) <= 64 * 2.0 ** (-53 * L)
    # quadratic convergence: the correct degree doubles per step; the updates
    # shrink to the rounding level
    assert norms[-1] <= 64 * 2.0 ** (-53 * L)
    assert norms[0] > norms[1] > norms[2]


def test_circle_demo_matches_printed_output():
    """The paper's printed coefficients come from a run in
    DOUBLE precision, and the paper points at their roundoff:
    the printed t^8 coefficient 2.48015873015868E-05 differs from 1/40320 by
    2.0e-14 relative.  The dd result agrees with every printed value within
    1e-13 relative (double-precision roundoff of a 9-coefficient Newton run),
    and with 1/40320 to dd precision (test above)."""
    x, _ = oracle.newton(circle_system(2), 8, nthreads=2)
    pr = GOLD["printed_newton_cos"]
    for k in (0, 2, 4, 6, 8):
        got = float(value(x[0, 0, :, k]))
        want = pr[f"t^{k}"]
        assert abs(got - want) <= 1e-13 * abs(want), (k, got, want)
    for k in (1, 3, 5, 7):
        assert abs(float(value(x[0, 0, :, k]))) <= 1e-30


def test_linear_system_converges_in_one_step():
    """f(x) = C(t) x - b(t) (degree-1 monomials and a constant): the first
    update solves the system, the second is at the rounding level."""
    n, d, L = 4, 6, 3
    rng = mdinputs.SplitMix64(77, "extra")
    C = mdinputs.unit_circle_series(rng, n * n, d + 1, L, "random")
    b = mdinputs.unit_circle_series(rng, n, d + 1, L, "random")
    polys = [[[(j, 1)] for j in range(n)] + [[]] for _ in range(n)]
    coeffs = []
    for i in range(n):
        coeffs += [C[i * n + j] for j in range(n)] + [-b[i]]
    si = make_si(n, polys, coeffs, [np.zeros((2, L, d + 1))] * n, d, L)
    x, norms = oracle.newton(si, 2, nthreads=2)
    assert norms[0] > 0.1
    assert norms[1] <= 2.0 ** (-53 * L + 20)
    want, _ = oracle.toeplitz_solve(C.reshape(n, n, 2, L, d + 1), b)
    assert oracle.series_err(x, want).max() <= 2.0 ** (-53 * L + 20)
