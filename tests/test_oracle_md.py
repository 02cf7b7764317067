"""Pins for the oracle's multiple-double arithmetic (oracle/mdoracle.c).

Each md operation of the oracle is specified as "exact result, rounded
greedily to L limbs" (round-to-nearest-even per limb).  These tests pin it
to exact rational arithmetic (every double is a dyadic rational; Python's
float(Fraction) is correctly rounded) and to the paper's worked example
(PAPER.md:82-95).
"""
import json
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests.exact import greedy, value

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))
LEVELS = (2, 3, 4, 5, 8, 10)


def rand_md(rng: random.Random, L: int, scale_exp: int = 0, sparse: bool = False):
    """a random canonical L-limb expansion built from exact rationals."""
    X = Fraction(rng.getrandbits(60 * L + 10), 1 << (60 * L)) * (1 if rng.random() < .5 else -1)
    X *= Fraction(2) ** scale_exp
    if sparse:  # 1 + tiny: limbs far apart
        X = Fraction(rng.choice([-1, 1])) + Fraction(rng.getrandbits(50) | 1, 1 << (rng.randrange(120, 300)))
    return greedy(X, L)


def adversarial_values(rng):
    vals = [0.0, 1.0, -1.0, 2.0 ** -1074, 2.0 ** 600, -(2.0 ** -600), 1.0 + 2.0 ** -52, 1.5,
            2.0 ** 53 + 2, 3.0 * 2.0 ** -60]
    for _ in range(40):
        vals.append(rng.uniform(-1, 1) * 2.0 ** rng.randrange(-200, 200))
    return vals


def test_round_is_greedy_rn_exactly():
    rng = random.Random(7)
    for trial in range(400):
        L = rng.choice(LEVELS)
        n = rng.randrange(1, 3 * L + 2)
        pool = adversarial_values(rng)
        v = [rng.choice(pool) for _ in range(n)]
        if trial % 5 == 0:  # heavy cancellation
            v = v + [-x for x in v[: n // 2]] + [2.0 ** -300]
        got = oracle.md_round(v, L)
        want = greedy(value(v), L)
        assert list(got) == want, (v, L)


def test_round_ties_to_even():
    # 1 + 2^-53 is a tie between 1 and 1+2^-52: RN picks the even mantissa (1.0)
    assert list(oracle.md_round([1.0, 2.0 ** -53], 1)) == [1.0]
    assert list(oracle.md_round([1.0 + 2.0 ** -52, 2.0 ** -53], 1)) == [1.0 + 2.0 ** -51]
    # sticky bit below the tie breaks it upward
    assert list(oracle.md_round([1.0, 2.0 ** -53, 2.0 ** -200], 1)) == [1.0 + 2.0 ** -52]


@pytest.mark.parametrize("L", LEVELS)
def test_add_mul_exactly_rounded(L):
    rng = random.Random(100 + L)
    for t in range(60):
        a = rand_md(rng, L, rng.randrange(-20, 20), sparse=(t % 7 == 0))
        b = rand_md(rng, L, rng.randrange(-20, 20), sparse=(t % 11 == 0))
        if t % 13 == 0:
            b = [-x for x in a]  # exact cancellation
        assert list(oracle.md_add(a, b)) == greedy(value(a) + value(b), L)
        assert list(oracle.md_mul(a, b)) == greedy(value(a) * value(b), L)


@pytest.mark.parametrize("L", LEVELS)
def test_div_sqrt_accuracy(L):
    rng = random.Random(200 + L)
    u = Fraction(1, 2 ** (53 * L))
    for t in range(30):
        a = rand_md(rng, L, rng.randrange(-5, 5))
        b = rand_md(rng, L, rng.randrange(-5, 5))
        q = oracle.md_div(a, b)
        exact = value(a) / value(b)
        assert abs(value(q) - exact) <= 2 * u * abs(exact)
        pa = [abs(x) for x in a] if a[0] > 0 else [-x for x in a]
        s = oracle.md_sqrt(pa)
        # |s^2 - a| <= 4u|a|  (s faithful to ~u)
        assert abs(value(s) ** 2 - value(pa)) <= 4 * u * abs(value(pa))
    assert list(oracle.md_sqrt([64.0] + [0.0] * (L - 1))) == [8.0] + [0.0] * (L - 1)
    assert list(oracle.md_div([1.0] + [0.0] * (L - 1), [1.0] + [0.0] * (L - 1))) == [1.0] + [0.0] * (L - 1)


def unit_circle_md(rng, count, L):
    """complex entries ((1-s^2) + 2is)/(1+s^2), |.| = 1 exactly, rounded to L limbs
    (unit modulus to working precision without md sin/cos)."""
    v = np.zeros((count, 2, L))
    for i in range(count):
        s = Fraction(rng.randrange(-10 ** 9, 10 ** 9), 10 ** 9 + rng.randrange(1, 10 ** 6))
        re = (1 - s * s) / (1 + s * s)
        im = 2 * s / (1 + s * s)
        v[i, 0] = greedy(re, L)
        v[i, 1] = greedy(im, L)
    return v


@pytest.mark.parametrize("L", LEVELS)
def test_ex1_norm_of_64_unit_complex_is_8(L):
    """||v||_2 = 8 for 64 entries cos(theta)+i sin(theta)."""
    g = GOLD["ex1_norm"]
    v = unit_circle_md(random.Random(64 + L), g["dimension"], L)
    nrm = oracle.md_norm2(v)
    assert nrm[0] == g["norm"]
    err = abs(value(nrm) - 8)
    # bound from the arithmetic: each |v_j|^2 = 1 + delta, |delta| <= 4*2^-53L
    assert err <= Fraction(32, 2 ** (53 * L))
    # at least as accurate as the paper's printed residual (x10 slack: the
    # paper's angles are unknown)
    assert float(err) <= 10 * abs(g["second_limb_printed"][str(L)])


def test_precision_ladder():
    """error vs exact is non-increasing in L (same rational inputs)."""
    rng = random.Random(5)
    for _ in range(20):
        A = Fraction(rng.getrandbits(700), 1 << 700)
        B = Fraction(rng.getrandbits(700), 1 << 699)
        errs = []
        for L in LEVELS:
            a, b = greedy(A, L), greedy(B, L)
            errs.append(abs(value(oracle.md_mul(a, b)) - value(a) * value(b)) / (value(a) * value(b)))
        assert all(errs[i + 1] <= errs[i] for i in range(len(errs) - 1))
        assert errs[-1] < Fraction(1, 2 ** 529)
