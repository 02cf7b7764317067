"""CUDA parity of Newton's method on power series (mdps_newton_step /
mdps_newton) against the oracle's Newton iteration, and
the paper's circle demo at every limb count."""
from fractions import Fraction

import numpy as np
import pytest

import mdinputs
import oracle
from tests.exact import series_err_exact
from tests.gpu_util import NTHREADS, TOL
from tests.test_oracle_evaldiff import make_si
from tests.test_oracle_newton import GOLD, circle_system

pytestmark = pytest.mark.gpu
LEVELS = (2, 3, 4, 5, 8, 10)


@pytest.fixture(scope="module")
def mdps():
    import torch
    import paper_2012_06607_b200 as m
    assert torch.cuda.is_available()
    m.lib()
    return m


def cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("L", LEVELS)
def test_circle_demo(mdps, L):
    """From (1, 0), degree 8, tolerance 1e-32, at most 8 steps (§6):
    x -> the Taylor series of cos, y -> s(t); GPU iterate = oracle iterate."""
    import torch
    si = circle_system(L)
    with mdps.System.from_inputs(si) as sys_, mdps.Solver(si.n, si.degree, L) as sol:
        x = cuda(si.x)
        steps, norm = sol.newton(sys_, x, 8, 1e-32)
        torch.cuda.synchronize()
        xg = x.cpu().numpy()
    cos = [(Fraction(c), Fraction(0)) for c in GOLD["cos_coefficients"]]
    sin = [(Fraction(c), Fraction(0)) for c in GOLD["s_coefficients"]]
    assert series_err_exact(xg[0], cos) <= TOL[L]
    assert series_err_exact(xg[1], sin) <= TOL[L]
    assert 4 <= steps <= 8
    xo, norms = oracle.newton(si, steps, nthreads=NTHREADS)
    assert oracle.series_err(xg, xo).max() <= TOL[L]


@pytest.mark.parametrize("L", (2, 4, 10))
def test_steps_match_oracle_small_system(mdps, L):
    """Two Newton steps on a small random system (exponents 1 and 2,
    constants), GPU against the oracle step by step."""
    import torch
    si = mdinputs.random_system(31 + L, 4, 5, (1, 3), (1, 2), 6, L)
    with mdps.System.from_inputs(si) as sys_, mdps.Solver(si.n, si.degree, L) as sol:
        x = cuda(si.x)
        dx = torch.empty_like(x)
        nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
        got = []
        for _ in range(2):
            sol.newton_step(sys_, x, dx, nrm)
            torch.cuda.synchronize()
            got.append(x.cpu().numpy().copy())
    for k in (1, 2):
        xo, norms = oracle.newton(si, k, nthreads=NTHREADS)
        assert oracle.series_err(got[k - 1], xo).max() <= TOL[L], k
    assert abs(float(nrm.item()) - norms[-1]) <= 1e-12 * norms[-1]


def test_shape_mismatch_rejected(mdps):
    si = circle_system(2)
    with mdps.System.from_inputs(si) as sys_, mdps.Solver(si.n, si.degree + 1, 2) as sol:
        with pytest.raises(mdps.MdpsError, match="differ"):
            sol.newton_step(sys_, cuda(si.x))


@pytest.mark.parametrize("L", (2, 4, 8))
def test_overdetermined_circle(mdps, L):
    """The circle system plus the redundant equation f_0 + f_1 (N = 3 > n = 2):
    Newton with least-squares steps still converges to (cos, sin)."""
    import torch
    from fractions import Fraction as Fr
    from tests.test_oracle_evaldiff import const_series
    si = circle_system(L)
    D = si.D
    s_coef = [Fr(c) for c in GOLD["s_coefficients"]]
    # f2 = s(t) - y + x^2 + y^2 - 1
    pp = np.concatenate([si.poly_ptr, [si.poly_ptr[-1] + 5]]).astype(np.int32)
    mono_vars = [[], [(1, 1)], [(0, 2)], [(1, 2)], []]
    mp, vv, ee = list(si.mono_ptr), list(si.vars), list(si.exps)
    for mono in mono_vars:
        for v, a in mono:
            vv.append(v)
            ee.append(a)
        mp.append(len(vv))
    coeffs = np.concatenate([si.coeffs, np.stack([const_series(s_coef, L, D), const_series([-1], L, D),
                                                  const_series([1], L, D), const_series([1], L, D),
                                                  const_series([-1], L, D)])])
    sys_in = mdinputs.SystemInputs("circle3", 2, si.degree, L, pp, np.asarray(mp, np.int32),
                                   np.asarray(vv, np.int32), np.asarray(ee, np.int32), coeffs, si.x)
    with mdps.System.from_inputs(sys_in) as sys_, mdps.Solver(2, si.degree, L, n_eqs=3) as sol:
        x = cuda(si.x)
        steps, norm = sol.newton(sys_, x, 10, 1e-32)
        torch.cuda.synchronize()
        xg = x.cpu().numpy()
    cos = [(Fr(c), Fr(0)) for c in GOLD["cos_coefficients"]]
    sin = [(Fr(c), Fr(0)) for c in GOLD["s_coefficients"]]
    assert series_err_exact(xg[0], cos) <= TOL[L]
    assert series_err_exact(xg[1], sin) <= TOL[L]
