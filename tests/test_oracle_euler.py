"""Pins of the oracle functions behind the full-size output checks (SURVEY
§8(c) C3 "eval/diff identities", R19):

  * eval_entries' (i, -2) entries: the degree-weighted value
    g_i = sum_r deg(r) c_r x^{a_r} (Euler's identity for polynomials:
    sum_j x_j df_i/dx_j = g_i);
  * euler_residual: |sum_j (x_j * J_ij)_k - g_ik| formed exactly.

Pinned against exact rationals (tests/exact.py: Fractions, no oracle code),
closed forms (exact-integer inputs, homogeneous systems of power-of-two
degree) and detection of a known perturbation.
"""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import mdinputs
import oracle
from tests.exact import conv, greedy, series_value, value
from tests.test_oracle_evaldiff import const_series, make_si

LEVELS = (2, 3, 4, 5, 8, 10)


def exact_weighted_values(si):
    """brute force g_i = sum_r deg(r) c_r x^{a_r} mod t^D (Fractions)."""
    D = si.degree + 1
    X = [series_value(si.x[j]) for j in range(si.n)]
    out = []
    for i in range(len(si.poly_ptr) - 1):
        acc = [(Fraction(0), Fraction(0))] * D
        for r in range(si.poly_ptr[i], si.poly_ptr[i + 1]):
            t = series_value(si.coeffs[r])
            deg = 0
            for v, a in zip(si.vars[si.mono_ptr[r]:si.mono_ptr[r + 1]], si.exps[si.mono_ptr[r]:si.mono_ptr[r + 1]]):
                deg += int(a)
                for _ in range(int(a)):
                    t = conv(t, X[int(v)], D)
            acc = [(p[0] + deg * q[0], p[1] + deg * q[1]) for p, q in zip(acc, t)]
        out.append(acc)
    return out


@pytest.mark.parametrize("L", LEVELS)
def test_weighted_value_vs_exact(L):
    """tiny systems with constants and exponents 1..3: g within the oracle's
    rounding bound of the exact sum (the chains are rounded per product)."""
    for seed in range(2):
        si = mdinputs.random_system(2000 + 10 * L + seed, n=3, monos=4, m_range=(0, 3), exps=(1, 2, 3),
                                    degree=4, limbs=L)
        g, _ = oracle.eval_entries(si, [(i, -2) for i in range(3)], nthreads=2)
        ex = exact_weighted_values(si)
        for i in range(3):
            scale = max(1.0, max(math.hypot(float(a), float(b)) for a, b in ex[i]))
            for k in range(si.degree + 1):
                d = math.hypot(float(value(g[i, 0, :, k]) - ex[i][k][0]), float(value(g[i, 1, :, k]) - ex[i][k][1]))
                assert d <= 64 * 2.0 ** (-53 * L) * scale * 16


@pytest.mark.parametrize("L", (2, 8, 10))
def test_weighted_value_homogeneous_is_degree_times_value(L):
    """every monomial of degree 8 (the sweep's shape) or 16 (deca's): g = deg * f
    bit for bit (a power-of-two scaling commutes with rounding)."""
    for m, seed in ((8, 1), (16, 2)):
        si = mdinputs.random_system(2100 + seed + L, n=m + 2, monos=3, m_range=(m, m), exps=(1,), degree=6, limbs=L)
        out, _ = oracle.eval_entries(si, [(i, -1) for i in range(si.n)] + [(i, -2) for i in range(si.n)])
        f, g = out[:si.n], out[si.n:]
        assert np.array_equal(g, m * f)


def exact_residual(x, J, g):
    n, _, L, D = x.shape
    X = [series_value(x[j]) for j in range(n)]
    Jv = [series_value(J[j]) for j in range(n)]
    G = series_value(g)
    acc = [(Fraction(0), Fraction(0))] * D
    for j in range(n):
        p = conv(X[j], Jv[j], D)
        acc = [(a[0] + b[0], a[1] + b[1]) for a, b in zip(acc, p)]
    return [math.hypot(float(a[0] - b[0]), float(a[1] - b[1])) for a, b in zip(acc, G)]


@pytest.mark.parametrize("L", LEVELS)
def test_euler_residual_vs_exact(L):
    """random x, J rows and g (overlapping limbs too): the residual equals the
    exact one rounded per part (up to the last bit of hypot)."""
    rng = random.Random(300 + L)
    for rep in range(4):
        n, D = rng.randint(1, 3), rng.randint(1, 4)
        x = np.zeros((n, 2, L, D))
        J = np.zeros((2, n, 2, L, D))
        g = np.zeros((2, 2, L, D))
        for arr in (x, J, g):
            flat = arr.reshape(-1, L)
            for t in range(flat.shape[0]):
                flat[t] = greedy(Fraction(rng.getrandbits(64 * L) - (1 << (64 * L - 1)), 1 << (64 * L - 3)), L)
        # make row 1 nearly consistent: g = the exact sum rounded (tiny residual)
        X = [series_value(x[j]) for j in range(n)]
        acc = [(Fraction(0), Fraction(0))] * D
        for j in range(n):
            acc = [(a[0] + b[0], a[1] + b[1]) for a, b in zip(acc, conv(X[j], series_value(J[1, j]), D))]
        for k in range(D):
            g[1, 0, :, k] = greedy(acc[k][0], L)
            g[1, 1, :, k] = greedy(acc[k][1], L)
        res = oracle.euler_residual(x, J, g, nthreads=2)
        for c in range(2):
            want = exact_residual(x, J[c], g[c])
            for k in range(D):
                assert res[c, k] == pytest.approx(want[k], rel=2.0 ** -50, abs=0.0)
        assert res[1].max() <= 4.0 * 2.0 ** (-53 * L) * 2 ** 6


@pytest.mark.parametrize("m,L", [(3, 2), (8, 4), (16, 10)])
def test_euler_residual_zero_on_exact_integers(m, L):
    """x_j = 1 + alpha_j t, c = 1 (the exact-integer case): the
    oracle's J and g are exact integers, so the Euler residual is exactly 0;
    changing one coefficient of one Jacobian entry by 1 shows up there."""
    D = m + 1
    alphas = list(range(1, m + 1))
    xs = [const_series([1, a], L, D) for a in alphas]
    si = make_si(m, [[[(v, 1) for v in range(m)]]] + [[] for _ in range(m - 1)],
                 [const_series([1], L, D)], xs, m, L)
    f, J, _ = oracle.eval_diff(si)
    g, _ = oracle.eval_entries(si, [(0, -2)])
    assert np.array_equal(g[0], m * f[0])
    res = oracle.euler_residual(si.x, J[:1], g)
    assert not res.any()
    J2 = J[:1].copy()
    J2[0, 2, 0, 0, 1] += 1.0  # J_{0,2} coefficient 1 (an integer < 2^53)
    res2 = oracle.euler_residual(si.x, J2, g)
    # (x_2 * dJ)_k = t (1 + alpha_2 t): residual 1 at k = 1, alpha_2 = 3 at k = 2
    assert res2[0, 1] == 1.0 and res2[0, 2] == 3.0 and res2[0, 0] == 0.0 and not res2[0, 3:].any()


@pytest.mark.parametrize("L", (2, 8))
def test_euler_residual_on_oracle_output_and_detection(L):
    """on the oracle's own f, J of a random system the residual is at the
    rounding level; a perturbation of one Jacobian coefficient by eps
    (relative) is reported at >= 0.5 * eps * |x_j,0| * |J| at that k."""
    si = mdinputs.random_system(2200 + L, n=5, monos=6, m_range=(1, 4), exps=(1, 2), degree=9, limbs=L)
    _, J, _ = oracle.eval_diff(si)
    g, _ = oracle.eval_entries(si, [(i, -2) for i in range(si.n)])
    res = oracle.euler_residual(si.x, J, g)
    scale = np.abs(J[:, :, :, 0, :]).max() * si.n * (si.degree + 1) * 4
    assert res.max() <= 64 * 2.0 ** (-53 * L) * max(scale, 1.0)
    i, j, k = 1, int(si.vars[si.mono_ptr[si.poly_ptr[1]]]), 4
    eps = 2.0 ** (-20 * L)
    J2 = J.copy()
    J2[i, j, 0, :, k] = greedy(value(J[i, j, 0, :, k]) * (1 + Fraction(eps)), L)
    res2 = oracle.euler_residual(si.x, J2, g)
    want = eps * abs(float(value(J[i, j, 0, :, k]))) * math.hypot(si.x[j, 0, 0, 0], si.x[j, 1, 0, 0])
    assert res2[i, k] >= 0.5 * want
    assert np.array_equal(res2[np.arange(si.n) != i], res[np.arange(si.n) != i])


def test_values_weighted_equals_entries():
    """the fused (f, g) pass equals the separate (i, -1) and (i, -2) entries bit for bit."""
    si = mdinputs.random_system(2300, n=5, monos=6, m_range=(0, 4), exps=(1, 2, 3), degree=7, limbs=3)
    f, g = oracle.values_weighted(si, [4, 0, 2], nthreads=2)
    out, _ = oracle.eval_entries(si, [(4, -1), (0, -1), (2, -1), (4, -2), (0, -2), (2, -2)])
    assert np.array_equal(f, out[:3]) and np.array_equal(g, out[3:])
