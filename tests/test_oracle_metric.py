"""Pins of the parity metric itself, oracle.series_err (oracle/mdoracle.c
mdo_series_err, R8):

    e_s = max_k |a_{s,k} - b_{s,k}| / max(max_k |b_{s,k}|, 1)

with the complex difference of every coefficient formed exactly.  Every
non-bit-exact GPU parity assertion is `series_err(gpu, oracle) <= TOL[L]`, so
a metric that under-reports (a sign slip in the rounding of a negative
difference, the wrong part in the modulus, the clamp on the wrong side) would
leave them all green.  Here it is compared with an independent computation
from exact rationals (tests/exact.series_err_exact: Python Fractions, no
oracle code) on adversarial pairs, and checked to DETECT known differences.
"""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import mdinputs
import oracle
from tests.exact import greedy, series_err_exact, value

LEVELS = (2, 3, 4, 5, 8, 10)
D = 3


def rand_md(rng, L, scale=1.0, canonical=True):
    """an L-limb number near `scale`: canonical (greedy rounding of a random
    rational) or overlapping limbs (each limb random at 2^-40 of the last)."""
    if canonical:
        X = Fraction(rng.getrandbits(60 * L) - (1 << (60 * L - 1)), 1 << (60 * L - 1)) * Fraction(scale)
        return greedy(X, L)
    out, s = [], float(scale)
    for _ in range(L):
        out.append(rng.uniform(-1, 1) * s)
        s *= 2.0 ** -40
    return out


def rand_series(rng, L, scale=1.0, canonical=True):
    s = np.zeros((2, L, D))
    for part in range(2):
        for k in range(D):
            s[part, :, k] = rand_md(rng, L, scale, canonical)
    return s


def perturbed(rng, b, L, kind):
    """a close to b, with a difference of the requested kind."""
    a = b.copy()
    k = rng.randrange(D)
    if kind == "ulp_last":  # one unit in the last limb of one part
        part = rng.randrange(2)
        a[part, L - 1, k] = math.nextafter(a[part, L - 1, k], math.inf if rng.random() < 0.5 else -math.inf)
    elif kind == "tiny":  # exact difference 10^-e, e across the tolerance range
        part = rng.randrange(2)
        e = rng.choice([29, 45, 61, 77, 124, 156, 200])
        sign = rng.choice([-1, 1])
        X = value(b[part, :, k]) + sign * Fraction(rng.randint(1, 9), 10 ** e)
        a[part, :, k] = greedy(X, L)
    elif kind == "imag_only":  # the real parts equal, imaginary ones differ
        X = value(b[1, :, k]) - Fraction(rng.randint(1, 1000), 1 << (53 * L - 20))
        a[1, :, k] = greedy(X, L)
    elif kind == "cancel":  # a's limbs cancel in pairs: [u, -u, greedy(b + d)]
        part = rng.randrange(2)
        u = 2.0 ** rng.randrange(20, 400)
        if L >= 3:
            d = Fraction(rng.choice([-1, 1]), 1 << (53 * (L - 2) + rng.randrange(0, 30)))
            a[part, :, k] = [u, -u] + greedy(value(b[part, :, k]) + d, L - 2)
        else:
            a[part, :, k] = [u, -u]
    return a


def check_pair(a, b):
    got = float(oracle.series_err(a[None], b[None])[0])
    want = series_err_exact(a, [(value(b[0, :, k]), value(b[1, :, k])) for k in range(b.shape[2])])
    # same exact difference rounded once per part; the two hypot calls (libm,
    # Python) may differ in the last bit
    assert got == pytest.approx(want, rel=2.0 ** -50, abs=0.0), (got, want)
    return got, want


@pytest.mark.parametrize("L", LEVELS)
def test_series_err_matches_exact_random(L):
    """>= 200 pairs per L: independent, 1-ulp, 10^-e, imaginary-only and
    cancelling differences; |b| below 1 (the clamp) and above 1; canonical
    and overlapping limbs."""
    rng = random.Random(1000 + L)
    kinds = ["indep", "ulp_last", "tiny", "imag_only", "cancel"]
    npairs = 0
    for rep in range(44):
        for kind in kinds:
            scale = rng.choice([2.0 ** -30, 2.0 ** -3, 1.0, 2.0 ** 3, 2.0 ** 40])
            canonical = rep % 4 != 3
            b = rand_series(rng, L, scale, canonical)
            a = rand_series(rng, L, scale, canonical) if kind == "indep" else perturbed(rng, b, L, kind)
            got, want = check_pair(a, b)
            if kind != "indep":
                assert got > 0.0 or want == 0.0
            npairs += 1
    assert npairs >= 200


@pytest.mark.parametrize("L", LEVELS)
def test_series_err_known_values(L):
    """closed forms: equal series give 0; b = 0 and a = 3+4i at one
    coefficient gives 5 (the clamp at 1, the complex modulus); a scale below 1
    uses the clamp, above 1 divides by max|b|; negative differences count."""
    z = np.zeros((2, L, D))
    assert oracle.series_err(z[None], z[None])[0] == 0.0
    a = z.copy()
    a[0, 0, 1], a[1, 0, 1] = 3.0, 4.0
    assert oracle.series_err(a[None], z[None])[0] == 5.0
    assert oracle.series_err(z[None], a[None])[0] == 1.0  # |0 - (3+4i)| / |3+4i|
    b = z.copy()
    b[0, 0, 0] = 0.25
    c = b.copy()
    c[0, 1, 0] = -2.0 ** -60  # negative difference, |b| < 1: divided by 1
    assert oracle.series_err(c[None], b[None])[0] == 2.0 ** -60
    b[0, 0, 0] = 64.0
    c[0, 0, 0] = 64.0
    c[0, 1, 0] = 0.0
    c[1, L - 1, 2] = -2.0 ** -500  # imaginary-only, last limb, |b| = 64
    assert oracle.series_err(c[None], b[None])[0] == 2.0 ** -506
    # the maximum is over coefficients, not the first or the last
    d = b.copy()
    d[0, 1, 1] = 2.0 ** -70
    d[0, 1, 2] = 2.0 ** -80
    assert oracle.series_err(d[None], b[None])[0] == 2.0 ** -76


@pytest.mark.parametrize("L,tol", [(2, 1e-29), (4, 1e-61), (8, 1e-124), (10, 1e-156)])
def test_series_err_detects_perturbation(L, tol):
    """an od-shaped series (D = 64, unit-circle data, full random limbs)
    perturbed by 10 x the tolerance in ONE coefficient of ONE part is reported
    at >= that size, for every position of the perturbation tried; a
    perturbation of 1e-120 on an octo-double series is reported >= 1e-121."""
    si = mdinputs.random_system(7, n=4, monos=1, m_range=(1, 1), exps=(1,), degree=63, limbs=L)
    b = si.x[0]
    rng = random.Random(L)
    for _ in range(8):
        part, k = rng.randrange(2), rng.randrange(64)
        for size in (10 * tol, 1e-120 if L == 8 else 10 * tol):
            for sign in (-1, 1):
                a = b.copy()
                a[part, :, k] = greedy(value(b[part, :, k]) + sign * Fraction(size), L)
                e = float(oracle.series_err(a[None], b[None])[0])
                assert e >= 0.9 * size, (part, k, size, e)
                assert e <= 1.1 * size + 2.0 ** (-53 * L), (part, k, size, e)
