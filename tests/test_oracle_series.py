"""Pins for the oracle's truncated power-series arithmetic.

Truncated product z_k = sum_{i<=k} x_i y_{k-i}, series
add and inverse, pinned to closed
forms, the paper's operation counts and exact rational convolution.
"""
import json
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests.exact import conv, greedy, series_err_exact, series_from_exact, series_value

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))
LEVELS = (2, 3, 4, 5, 8, 10)


def real_series(coefs, L):
    return series_from_exact([(Fraction(c), Fraction(0)) for c in coefs], L)


@pytest.mark.parametrize("L", LEVELS)
def test_one_plus_t_times_one_minus_t(L):
    """(1+t)(1-t) = 1 - t^2 exactly."""
    D = 6
    a = real_series([1, 1] + [0] * (D - 2), L)
    b = real_series([1, -1] + [0] * (D - 2), L)
    z = oracle.series_mul(a, b)
    assert np.array_equal(z, real_series([1, 0, -1] + [0] * (D - 3), L))


@pytest.mark.parametrize("D", [1, 2, 9, 33])
def test_geometric_series_closed_form(D):
    """(1 - t) * sum_k t^k = 1 mod t^D and 1/(1-t) = sum_k t^k."""
    L = 4
    one_minus_t = real_series([1, -1] + [0] * (D - 2), L) if D > 1 else real_series([1], L)
    geo = real_series([1] * D, L)
    assert np.array_equal(oracle.series_mul(one_minus_t, geo), real_series([1] + [0] * (D - 1), L))
    assert np.array_equal(oracle.series_inv(one_minus_t), geo)


def test_product_operation_counts_match_paper():
    """45 mul / 36 add at d=8, 561 / 528 at d=32."""
    g = GOLD["series_product_counts"]
    for d in (8, 32):
        counts = np.zeros(2, dtype=np.int64)
        x = np.zeros((2, 2, d + 1))
        oracle.series_mul(x, x, counts)
        assert counts.tolist() == g[str(d)]
    for d in range(0, 20):  # closed form for all d
        counts = np.zeros(2, dtype=np.int64)
        x = np.zeros((2, 2, d + 1))
        oracle.series_mul(x, x, counts)
        assert counts.tolist() == [(d + 2) * (d + 1) // 2, (d + 1) * d // 2]


def rand_series(rng, D, L):
    coefs = []
    for _ in range(D):
        coefs.append((Fraction(rng.getrandbits(64 * L), 1 << (64 * L - 1)) - 1,
                      Fraction(rng.getrandbits(64 * L), 1 << (64 * L - 1)) - 1))
    return series_from_exact(coefs, L)


@pytest.mark.parametrize("L", LEVELS)
def test_product_is_exact_convolution_rounded(L):
    """brute force: every coefficient equals the exact convolution rounded
    greedily to L limbs (d <= 4)."""
    rng = random.Random(L)
    for D in (1, 2, 3, 5):
        x, y = rand_series(rng, D, L), rand_series(rng, D, L)
        z = oracle.series_mul(x, y)
        want = series_from_exact(conv(series_value(x), series_value(y), D), L)
        assert np.array_equal(z, want)
        assert np.array_equal(oracle.series_mul(y, x), z)  # commutativity, bit-exact


@pytest.mark.parametrize("L", LEVELS)
def test_add_exact_rounded(L):
    rng = random.Random(30 + L)
    x, y = rand_series(rng, 5, L), rand_series(rng, 5, L)
    z = oracle.series_add(x, y)
    xv, yv = series_value(x), series_value(y)
    assert np.array_equal(z, series_from_exact([(a[0] + b[0], a[1] + b[1]) for a, b in zip(xv, yv)], L))


@pytest.mark.parametrize("L", [2, 4, 8, 10])
def test_inverse_invariant(L):
    """x * (1/x) = 1 + O(u) (BASELINE.json north_star)."""
    rng = random.Random(40 + L)
    D = 12
    x = rand_series(rng, D, L)
    x[0, 0, 0] += 4.0  # keep x_0 well away from 0
    y = oracle.series_inv(x)
    z = oracle.series_mul(x, y)
    one = [(Fraction(1), Fraction(0))] + [(Fraction(0), Fraction(0))] * (D - 1)
    assert series_err_exact(z, one) <= 2.0 ** (-53 * L + 12)


def test_truncation_consistency():
    """coefficient k of a product depends only on coefficients <= k."""
    rng = random.Random(9)
    L, D = 3, 9
    x, y = rand_series(rng, D, L), rand_series(rng, D, L)
    z = oracle.series_mul(x, y)
    for Dp in (1, 4, 8):
        assert np.array_equal(oracle.series_mul(x[:, :, :Dp].copy(), y[:, :, :Dp].copy()), z[:, :, :Dp])
