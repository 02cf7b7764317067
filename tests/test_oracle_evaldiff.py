"""Pins for the oracle's evaluation and differentiation of a polynomial
system with series coefficients.

Closed forms (exact-integer inputs), the paper's circle system
(PAPER.md:183-208), exact rational brute force on tiny systems, and
invariants (Euler's identity, truncation, linearity, L vs L+2).
"""
import itertools
import json
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import mdinputs
import oracle
from tests.exact import conv, greedy, series_err_exact, series_from_exact, series_value, value

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))
LEVELS = (2, 3, 4, 5, 8, 10)


def const_series(coefs, L, D):
    """real series from exact coefficient list (padded with zeros)."""
    c = [(Fraction(v), Fraction(0)) for v in coefs] + [(Fraction(0), Fraction(0))] * (D - len(coefs))
    return series_from_exact(c[:D], L)


def make_si(n, polys, coeff_series, x_series, degree, L, name="t"):
    pp, mp, vv, ee = mdinputs.structure_from_monomials(len(polys), polys) if len(polys) == n else \
        _structure_rect(polys)
    return mdinputs.SystemInputs(name, n, degree, L, pp, mp, vv, ee,
                                 np.ascontiguousarray(np.stack(coeff_series)) if coeff_series else
                                 np.zeros((0, 2, L, degree + 1)),
                                 np.ascontiguousarray(np.stack(x_series)))


def _structure_rect(polys):
    pp, mp, vv, ee = [0], [0], [], []
    for poly in polys:
        for mono in poly:
            for v, a in mono:
                vv.append(v)
                ee.append(a)
            mp.append(len(vv))
        pp.append(len(mp) - 1)
    return (np.asarray(pp, np.int32), np.asarray(mp, np.int32), np.asarray(vv, np.int32),
            np.asarray(ee, np.int32))


def esym(alphas, k):
    return sum(math.prod(c) for c in itertools.combinations(alphas, k)) if k <= len(alphas) else 0


@pytest.mark.parametrize("m,L", [(3, 2), (8, 4), (16, 8), (16, 10)])
def test_exact_integer_speelpenning(m, L):
    """x_j = 1 + alpha_j t, c = 1: the value coefficients are the elementary
    symmetric numbers e_k(alpha), d/dx_l gives e_k(alpha without alpha_l);
    all integers < 2^53, so the result is exact."""
    D = m + 2
    alphas = list(range(1, m + 1))
    xs = [const_series([1, a], L, D) for a in alphas]
    si = make_si(m, [[[(j, 1) for j in range(m)]]] + [[] for _ in range(m - 1)],
                 [const_series([1], L, D)], xs, D - 1, L)
    vals, jac, _ = oracle.eval_diff(si)
    want = [esym(alphas, k) for k in range(D)]
    assert np.array_equal(vals[0], const_series(want, L, D))
    for l in range(m):
        rest = alphas[:l] + alphas[l + 1:]
        assert np.array_equal(jac[0, l], const_series([esym(rest, k) for k in range(D)], L, D))
    # structurally zero rows (empty polynomials) are exactly zero
    assert not vals[1:].any() and not jac[1:].any()


def test_exact_integer_complex_and_exponents():
    """x = 1 + i alpha t (complex), exponents 2 and 3:
    f = c x1^2 x2^3, df/dx1 = 2 c x1 x2^3, df/dx2 = 3 c x1^2 x2^2."""
    L, D = 4, 7
    a1, a2 = 3, 5
    X1 = [(Fraction(1), Fraction(0)), (Fraction(0), Fraction(a1))] + [(Fraction(0),) * 2] * (D - 2)
    X2 = [(Fraction(1), Fraction(0)), (Fraction(0), Fraction(a2))] + [(Fraction(0),) * 2] * (D - 2)
    C = [(Fraction(2), Fraction(-1))] + [(Fraction(0),) * 2] * (D - 1)
    si = make_si(2, [[[(0, 2), (1, 3)]], []], [series_from_exact(C, L)],
                 [series_from_exact(X1, L), series_from_exact(X2, L)], D - 1, L)
    vals, jac, _ = oracle.eval_diff(si)

    def P(*fs):
        acc = [(Fraction(1), Fraction(0))] + [(Fraction(0),) * 2] * (D - 1)
        for f in fs:
            acc = conv(acc, f, D)
        return acc

    def scale(s, w):
        return [(w * a, w * b) for a, b in s]

    assert np.array_equal(vals[0], series_from_exact(P(C, X1, X1, X2, X2, X2), L))
    assert np.array_equal(jac[0, 0], series_from_exact(scale(P(C, X1, X2, X2, X2), 2), L))
    assert np.array_equal(jac[0, 1], series_from_exact(scale(P(C, X1, X1, X2, X2), 3), L))


@pytest.mark.parametrize("L", LEVELS)
def test_circle_system(L):
    """f1 = s(t) - y, f2 = x^2 + y^2 - 1 with s the degree-7
    Taylor polynomial of sin.  At x = cos_8(t), y = sin_8(t)
    f1 = 0 exactly, f2 = 0 mod t^9 to working precision, J = [[0,-1],[2x,2y]]."""
    g = GOLD["circle"]
    d = g["degree"]
    D = d + 1
    s_coef = [Fraction(c) for c in g["s_coefficients"]]
    cos_coef = [Fraction(c) for c in g["cos_coefficients"]]
    sin_coef = s_coef  # sin_8 = t - t^3/6 + t^5/120 - t^7/5040 (its t^9 term is beyond d)
    polys = [[[], [(1, 1)]], [[(0, 2)], [(1, 2)], []]]   # f1: s(t)*1 + (-1)*y ; f2: x^2 + y^2 + (-1)
    coeffs = [const_series(s_coef, L, D), const_series([-1], L, D),
              const_series([1], L, D), const_series([1], L, D), const_series([-1], L, D)]
    x = const_series(cos_coef, L, D)
    y = const_series(sin_coef, L, D)
    si = make_si(2, polys, coeffs, [x, y], d, L)
    vals, jac, _ = oracle.eval_diff(si)
    assert not vals[0].any()                          # f1 = s - sin_8 = 0 exactly
    zero = [(Fraction(0), Fraction(0))] * D
    assert series_err_exact(vals[1], zero) <= 2.0 ** (-53 * L + 4)   # cos^2 + sin^2 - 1 = O(t^9)
    assert not jac[0, 0].any()                        # structural zero
    assert np.array_equal(jac[0, 1], const_series([-1], L, D))
    assert np.array_equal(jac[1, 0], 2 * x)           # 2x: exact scaling
    assert np.array_equal(jac[1, 1], 2 * y)
    # at the constant point (1, 0): A_0 = [[0, -1], [2, 0]]
    si0 = make_si(2, polys, coeffs, [const_series([1], L, D), const_series([0], L, D)], d, L)
    _, jac0, _ = oracle.eval_diff(si0)
    assert [[jac0[i, j, 0, 0, 0] for j in range(2)] for i in range(2)] == [[0.0, -1.0], [2.0, 0.0]]


def exact_eval(si):
    """brute-force exact f and J (Fractions) of a tiny system."""
    D = si.degree + 1
    X = [series_value(si.x[j]) for j in range(si.n)]
    zero = [(Fraction(0), Fraction(0))] * D
    n_polys = len(si.poly_ptr) - 1
    vals = [list(zero) for _ in range(n_polys)]
    jac = [[list(zero) for _ in range(si.n)] for _ in range(n_polys)]
    for i in range(n_polys):
        for r in range(si.poly_ptr[i], si.poly_ptr[i + 1]):
            C = series_value(si.coeffs[r])
            mono = list(zip(si.vars[si.mono_ptr[r]:si.mono_ptr[r + 1]].tolist(),
                            si.exps[si.mono_ptr[r]:si.mono_ptr[r + 1]].tolist()))
            t = C
            for v, a in mono:
                for _ in range(a):
                    t = conv(t, X[v], D)
            vals[i] = [(p[0] + q[0], p[1] + q[1]) for p, q in zip(vals[i], t)]
            for l, (vl, al) in enumerate(mono):
                t = C
                for v, a in mono:
                    for _ in range(a - (1 if v == vl else 0)):
                        t = conv(t, X[v], D)
                jac[i][vl] = [(p[0] + al * q[0], p[1] + al * q[1]) for p, q in zip(jac[i][vl], t)]
    return vals, jac


@pytest.mark.parametrize("L", LEVELS)
def test_tiny_systems_vs_exact(L):
    """n <= 3, d <= 4, m <= 3, exponents <= 3: the oracle is within its
    rounding bound of the exact result (SURVEY §8(c) C3 'eval/diff tiny')."""
    for seed in range(3):
        si = mdinputs.random_system(1000 + 10 * L + seed, n=3, monos=3, m_range=(0, 3), exps=(1, 2, 3),
                                    degree=4, limbs=L)
        vals, jac, _ = oracle.eval_diff(si)
        ev, ej = exact_eval(si)
        bound = 64 * 2.0 ** (-53 * L)
        for i in range(3):
            assert series_err_exact(vals[i], ev[i]) <= bound
            for j in range(3):
                if all(c == (0, 0) for c in ej[i][j]) and not any(
                        j in si.vars[si.mono_ptr[r]:si.mono_ptr[r + 1]] for r in range(si.poly_ptr[i], si.poly_ptr[i + 1])):
                    assert not jac[i, j].any()   # structural zero is exactly 0
                assert series_err_exact(jac[i, j], ej[i][j]) <= bound


def test_euler_identity_homogeneous():
    """for a system homogeneous of degree delta: sum_j x_j J_ij = delta f_i
    (Euler; BASELINE.json 'exponent-weighted monomial quotients')."""
    L, delta = 4, 10
    si = mdinputs.random_system(77, n=5, monos=6, m_range=(2, 4), exps=(1, 2, 3), degree=7, limbs=L)
    # make every monomial homogeneous of degree delta by adjusting the last exponent
    exps = si.exps.copy()
    for r in range(len(si.mono_ptr) - 1):
        a, b = si.mono_ptr[r], si.mono_ptr[r + 1]
        if b > a:
            exps[b - 1] = delta - int(exps[a:b - 1].sum())
            assert exps[b - 1] >= 1 or (exps[a:b - 1].sum() >= delta)
    if (exps < 1).any():
        pytest.skip("degree overflow in draw")
    si.exps[:] = exps
    vals, jac, _ = oracle.eval_diff(si)
    for i in range(si.n):
        ms = [r for r in range(si.poly_ptr[i], si.poly_ptr[i + 1]) if si.mono_ptr[r + 1] > si.mono_ptr[r]]
        acc = np.zeros_like(vals[i])
        for j in range(si.n):
            acc = oracle.series_add(acc, oracle.series_mul(si.x[j], jac[i, j]))
        const = [r for r in range(si.poly_ptr[i], si.poly_ptr[i + 1]) if si.mono_ptr[r + 1] == si.mono_ptr[r]]
        D = si.degree + 1
        dser = const_series([delta], L, D)           # delta * s formed exactly by the oracle
        target = oracle.series_mul(dser, vals[i])
        for r in const:  # a constant monomial has degree 0
            target = oracle.series_add(target, -oracle.series_mul(dser, si.coeffs[r]))
        assert oracle.series_err(acc, target) <= 2.0 ** (-53 * L + 20)


def test_truncation_and_self_consistency():
    """eval at d truncated to d' == eval at d' (bit-exact); eval at L vs L+2
    limbs agree to the L-limb rounding (SURVEY C3 'self-consistency')."""
    si = mdinputs.random_system(5, n=4, monos=5, m_range=(1, 4), exps=(1, 2), degree=10, limbs=3)
    vals, jac, _ = oracle.eval_diff(si)
    sit = mdinputs.truncate(si, 5, 3)
    vt, jt, _ = oracle.eval_diff(sit)
    assert np.array_equal(vt, vals[..., :6]) and np.array_equal(jt, jac[..., :6])
    v5, j5, _ = oracle.eval_diff(si, limbs=5)
    assert oracle.series_err(vals, v5[:, :, :3]).max() <= 2.0 ** (-53 * 3 + 8)
    assert oracle.series_err(jac, j5[:, :, :, :3]).max() <= 2.0 ** (-53 * 3 + 8)


def test_linearity_in_coefficients():
    """f and J are linear in the coefficient series."""
    L = 4
    si = mdinputs.random_system(11, n=3, monos=4, m_range=(1, 3), exps=(1, 2), degree=6, limbs=L)
    v1, j1, _ = oracle.eval_diff(si)
    si2 = mdinputs.SystemInputs(**{**si.__dict__, "coeffs": 2.0 * si.coeffs})
    v2, j2, _ = oracle.eval_diff(si2)
    assert np.array_equal(v2, 2.0 * v1) and np.array_equal(j2, 2.0 * j1)  # power-of-2 scaling is exact
    c3 = oracle.series_add(si.coeffs, 2.0 * si.coeffs)     # c + 2c, md-rounded
    si3 = mdinputs.SystemInputs(**{**si.__dict__, "coeffs": c3})
    v3, _, _ = oracle.eval_diff(si3)
    assert oracle.series_err(v3, oracle.series_add(v1, v2)).max() <= 2.0 ** (-53 * L + 8)


def test_entries_match_full_eval():
    si = mdinputs.random_system(3, n=4, monos=4, m_range=(1, 3), exps=(1,), degree=5, limbs=2)
    vals, jac, prods = oracle.eval_diff(si, nthreads=3)
    out, _ = oracle.eval_entries(si, [(2, -1), (1, 3), (0, 0)], nthreads=1)
    assert np.array_equal(out[0], vals[2]) and np.array_equal(out[1], jac[1, 3]) and np.array_equal(out[2], jac[0, 0])


@pytest.mark.parametrize("L", (2, 4, 8))
def test_constant_series_reduce_to_polynomial_values(L):
    """SURVEY §8(c) C3 'eval/diff special case': at
    constant series (only t^0 nonzero) with constant coefficients, every
    coefficient t^k, k >= 1, of f and J is exactly 0 and t^0 is the plain
    complex polynomial value and derivative — written out here with exact
    rationals on scalars (no series arithmetic)."""
    si = mdinputs.random_system(300 + L, n=4, monos=5, m_range=(0, 4), exps=(1, 2, 3), degree=6, limbs=L)
    si.x[..., 1:] = 0.0
    si.coeffs[..., 1:] = 0.0
    vals, jac, _ = oracle.eval_diff(si)
    assert not vals[..., 1:].any() and not jac[..., 1:].any()
    xs = [(value(si.x[j, 0, :, 0]), value(si.x[j, 1, :, 0])) for j in range(si.n)]

    def cmul_(a, b):
        return (a[0] * b[0] - a[1] * b[1], a[0] * b[1] + a[1] * b[0])

    bound = 64 * 2.0 ** (-53 * L)
    for i in range(si.n):
        f = (Fraction(0), Fraction(0))
        df = [(Fraction(0), Fraction(0)) for _ in range(si.n)]
        for r in range(si.poly_ptr[i], si.poly_ptr[i + 1]):
            c = (value(si.coeffs[r, 0, :, 0]), value(si.coeffs[r, 1, :, 0]))
            mono = list(zip(si.vars[si.mono_ptr[r]:si.mono_ptr[r + 1]].tolist(),
                            si.exps[si.mono_ptr[r]:si.mono_ptr[r + 1]].tolist()))
            term = c
            for v, a in mono:
                for _ in range(a):
                    term = cmul_(term, xs[v])
            f = (f[0] + term[0], f[1] + term[1])
            for vl, al in mono:  # d/dx_vl: al * c * x_vl^(al-1) * prod_{v != vl} x_v^a
                term = (al * c[0], al * c[1])
                for v, a in mono:
                    for _ in range(a - (1 if v == vl else 0)):
                        term = cmul_(term, xs[v])
                df[vl] = (df[vl][0] + term[0], df[vl][1] + term[1])
        assert series_err_exact(vals[i][..., :1], [f]) <= bound
        for j in range(si.n):
            assert series_err_exact(jac[i, j][..., :1], [df[j]]) <= bound


@pytest.mark.parametrize("L", (2, 5, 10))
def test_monomial_quotient_identity(L):
    """Per monomial f = c prod x_l^(a_l): x_l * df/dx_l = a_l * f exactly
    (SURVEY §8(c) C3 'eval/diff identities'; the north star's
    exponent-weighted monomial quotients), checked on the oracle's rounded
    outputs with exact rational series products."""
    for seed in range(3):
        si = mdinputs.random_system(400 + 10 * L + seed, n=5, monos=1, m_range=(3, 5), exps=(1, 2, 3),
                                    degree=5, limbs=L)
        vals, jac, _ = oracle.eval_diff(si)
        D = si.degree + 1
        F0 = series_value(vals[0])
        scale = max(max(abs(a), abs(b)) for a, b in F0) + 1
        r = si.poly_ptr[0]
        for v, a in zip(si.vars[si.mono_ptr[r]:si.mono_ptr[r + 1]].tolist(),
                        si.exps[si.mono_ptr[r]:si.mono_ptr[r + 1]].tolist()):
            lhs = conv(series_value(si.x[v]), series_value(jac[0, v]), D)
            diff = max(max(abs(p[0] - a * q[0]), abs(p[1] - a * q[1])) for p, q in zip(lhs, F0))
            assert diff <= 256 * 2.0 ** (-53 * L) * scale, (seed, v, float(diff))
