"""Host-side checks of the seeded input generator (mdinputs): determinism,
structure recipe and canonical limbs (C2.12)."""
import random
from fractions import Fraction

import numpy as np
import pytest

import mdinputs
from tests.exact import greedy, value


def test_deterministic_and_seeded():
    a = mdinputs.make_system(mdinputs.CONFIGS["dd"])
    b = mdinputs.make_system(mdinputs.CONFIGS["dd"])
    assert a.sha256() == b.sha256()
    c = mdinputs.random_system(2, 8, 16, (3, 3), (1,), 15, 2, "zero")
    assert c.sha256() != a.sha256()


@pytest.mark.parametrize("name", ["dd", "qd"])
def test_structure_recipe(name):
    cfg = mdinputs.CONFIGS[name]
    si = mdinputs.make_config(name)
    assert si.poly_ptr.tolist() == [cfg.monos * i for i in range(cfg.n + 1)]
    for i in range(cfg.n):
        seen = set()
        for r in range(si.poly_ptr[i], si.poly_ptr[i + 1]):
            v = si.vars[si.mono_ptr[r]:si.mono_ptr[r + 1]].tolist()
            e = si.exps[si.mono_ptr[r]:si.mono_ptr[r + 1]].tolist()
            assert cfg.m_range[0] <= len(v) <= cfg.m_range[1]
            assert v == sorted(set(v)) and all(0 <= t < cfg.n for t in v)
            assert set(e) <= set(cfg.exps)
            assert (tuple(v), tuple(e)) not in seen
            seen.add((tuple(v), tuple(e)))
    assert si.coeffs.shape == (si.M, 2, cfg.limbs, cfg.degree + 1)
    assert si.x.shape == (cfg.n, 2, cfg.limbs, cfg.degree + 1)


def test_unit_circle_leading_limbs_and_zero_lower_limbs():
    si = mdinputs.make_config("dd")
    lead = si.x[:, 0, 0, :] ** 2 + si.x[:, 1, 0, :] ** 2
    assert np.allclose(lead, 1.0, atol=4e-16)
    assert not si.x[:, :, 1, :].any() and not si.coeffs[:, :, 1, :].any()


def test_random_lower_limbs_are_canonical():
    """limb_j = RN(X - sum_{q<j} limb_q): the expansion is its own greedy
    rounding, so truncation to fewer limbs equals rounding (sweep cells)."""
    si = mdinputs.make_config("od")
    rng = random.Random(1)
    for _ in range(200):
        r, part, k = rng.randrange(si.M), rng.randrange(2), rng.randrange(si.D)
        limbs = si.coeffs[r, part, :, k].tolist()
        assert greedy(value(limbs), len(limbs)) == limbs
        for L in (2, 5):
            assert greedy(value(limbs), L) == limbs[:L]
        # lower limbs are about 2^-53 apart (full random limbs)
        assert all(0 < abs(limbs[j + 1]) <= abs(limbs[j]) * 2.0 ** -52 for j in range(len(limbs) - 1))


def test_sweep_cells_share_data():
    c = mdinputs.sweep_cell(15, 2)
    big = mdinputs.make_config("sweep")
    assert c.coeffs.shape[-2:] == (2, 16) and np.array_equal(c.x, big.x[:, :, :2, :16])
    assert c.n == 64 and c.M == 64 * 64
