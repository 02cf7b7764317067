"""Edge cases of eval/diff on the GPU against the oracle: degree 0 (constant
series), n = 1, zero inputs, polynomials of constants only, a monomial whose
variable has a large exponent (a long common-factor chain), cancellation to
exact zeros, and tiny / huge magnitudes."""
import numpy as np
import pytest

import mdinputs
import oracle
from tests.gpu_util import TOL, gpu_eval, structural_support
from tests.test_oracle_evaldiff import make_si

pytestmark = pytest.mark.gpu


def full_check(si, L):
    vals, jac, _ = gpu_eval(si)
    ov, oj, _ = oracle.eval_diff(si)
    assert oracle.series_err(vals, ov).max() <= TOL[L]
    assert oracle.series_err(jac, oj).max() <= TOL[L]
    assert not jac[~structural_support(si)].any()
    return vals, jac


@pytest.mark.parametrize("L", (2, 5, 10))
def test_degree_zero(L):
    si = mdinputs.random_system(700 + L, n=6, monos=5, m_range=(0, 4), exps=(1, 2), degree=0, limbs=L)
    full_check(si, L)


@pytest.mark.parametrize("L", (2, 8))
def test_single_variable(L):
    si = mdinputs.random_system(710 + L, n=1, monos=4, m_range=(0, 1), exps=(1, 2, 3), degree=9, limbs=L)
    full_check(si, L)


@pytest.mark.parametrize("L", (3, 8))
def test_zero_input_series(L):
    si = mdinputs.random_system(720 + L, n=4, monos=6, m_range=(0, 3), exps=(1, 2), degree=11, limbs=L)
    si.x[:] = 0.0
    vals, jac = full_check(si, L)


def test_constants_only_polynomial():
    L, D = 4, 8
    rng = mdinputs.SplitMix64(730, "c")
    c = mdinputs.unit_circle_series(rng, 3, D, L, "random")
    x = mdinputs.unit_circle_series(mdinputs.SplitMix64(730, "x"), 2, D, L, "random")
    si = make_si(2, [[[], []], [[(0, 1)], []]], [c[0], c[1], c[2], c[0]], [x[0], x[1]], D - 1, L)
    vals, jac = full_check(si, L)
    assert not jac[0].any()


@pytest.mark.parametrize("L", (2, 10))
def test_high_exponent(L):
    """x0^7 x1^3: common factor chains of 8 products."""
    D = 12
    x = mdinputs.unit_circle_series(mdinputs.SplitMix64(740, "x"), 2, D, L, "random")
    c = mdinputs.unit_circle_series(mdinputs.SplitMix64(740, "c"), 1, D, L, "random")
    si = make_si(2, [[[(0, 7), (1, 3)]], [[(1, 1)]]], [c[0], c[0]], [x[0], x[1]], D - 1, L)
    full_check(si, L)


def test_exact_cancellation_to_zero():
    """f = c x0 - c x0 (duplicate monomials with opposite coefficients): the
    value and the Jacobian are exactly zero."""
    L, D = 4, 10
    x = mdinputs.unit_circle_series(mdinputs.SplitMix64(750, "x"), 2, D, L, "random")
    c = mdinputs.unit_circle_series(mdinputs.SplitMix64(750, "c"), 1, D, L, "random")[0]
    si = make_si(2, [[[(0, 1), (1, 1)], [(0, 1), (1, 1)]], [[(1, 1)]]], [c, -c, c], [x[0], x[1]], D - 1, L)
    vals, jac, _ = gpu_eval(si)
    assert not vals[0].any() and not jac[0].any()


@pytest.mark.parametrize("scale_exp", [-200, 150])
def test_tiny_and_huge_magnitudes(scale_exp):
    """inputs scaled by 2^scale (exact): the outputs scale exactly as the
    oracle's; the tolerance is relative to each series."""
    L = 5
    si = mdinputs.random_system(760, n=4, monos=5, m_range=(1, 3), exps=(1,), degree=7, limbs=L)
    si.x[:] *= 2.0 ** scale_exp
    vals, jac, _ = gpu_eval(si)
    ov, oj, _ = oracle.eval_diff(si)
    for got, want in ((vals, ov), (jac, oj)):
        g = got.reshape(-1, 2, L, si.D)
        w = want.reshape(-1, 2, L, si.D)
        for a, b in zip(g, w):
            s = np.abs(b[:, 0]).max()
            if s == 0:
                assert not a.any()
                continue
            e = 2.0 ** -int(np.floor(np.log2(s)))        # rescale to O(1), exactly
            assert oracle.series_err(a * e, b * e).max() <= TOL[L]


@pytest.mark.parametrize("algo", (1, 2))
@pytest.mark.parametrize("L", (2, 4, 8))
def test_constant_series_inputs(algo, L):
    """Constant series (only t^0 nonzero) and constant coefficients at D > 1:
    every higher coefficient of f and J is exactly 0 on the GPU (every term
    of z_k, k >= 1, has an exact-zero factor), t^0 matches the oracle (which is
    pinned to plain polynomial evaluation, test_oracle_evaldiff)."""
    si = mdinputs.random_system(300 + L, n=4, monos=5, m_range=(0, 4), exps=(1, 2, 3), degree=6, limbs=L)
    si.x[..., 1:] = 0.0
    si.coeffs[..., 1:] = 0.0
    vals, jac, _ = gpu_eval(si, algo)
    assert not vals[..., 1:].any() and not jac[..., 1:].any()
    ov, oj, _ = oracle.eval_diff(si)
    assert oracle.series_err(vals, ov).max() <= TOL[L]
    assert oracle.series_err(jac, oj).max() <= TOL[L]


def test_binding_rejects_wrong_buffers():
    """The binding checks sizes, dtype and device before the C ABI (which only
    sees pointers): a short output, a wrong-size input or host array raises
    MdpsError instead of letting the kernels or the copies overrun memory."""
    import torch
    import paper_2012_06607_b200 as mdps
    si = mdinputs.random_system(740, n=3, monos=4, m_range=(1, 3), exps=(1,), degree=7, limbs=2)
    with mdps.System.from_inputs(si) as s:
        x = torch.from_numpy(si.x).cuda()
        vals, jac = s.eval_diff(x)
        with pytest.raises(mdps.MdpsError, match="values_out"):
            s.eval_diff(x, vals[:-1].contiguous(), jac)
        with pytest.raises(mdps.MdpsError, match="jacobian_out"):
            s.eval_diff(x, vals, jac.reshape(-1)[:-1].contiguous())
        with pytest.raises(mdps.MdpsError, match="series_in"):
            s.eval_diff(x[:2].contiguous(), vals, jac)
        with pytest.raises(mdps.MdpsError, match="float64"):
            s.eval_diff(x.float(), vals, jac)
        with pytest.raises(mdps.MdpsError, match="series_in"):
            mdps.mdps_eval_diff_host(s.handle, si.x[:2].copy(), np.empty(vals.shape), np.empty(jac.shape))
        with pytest.raises(mdps.MdpsError, match="jacobian_out"):
            mdps.mdps_eval_diff_host(s.handle, si.x, np.empty(vals.shape), np.empty(jac.shape)[:-1].copy())
    with mdps.Solver(3, 7, 2) as sol:
        with pytest.raises(mdps.MdpsError, match="rhs"):
            sol.solve(jac, vals[:2].contiguous())
        with pytest.raises(mdps.MdpsError, match="jacobian"):
            sol.solve(jac[:2].contiguous(), vals)


@pytest.mark.parametrize("L", (3, 8))
def test_parts_of_very_different_magnitude(L):
    """DESIGN R20: the digit pool holds both parts of a complex coefficient on
    the grid of the larger one.  Inputs whose imaginary parts are 2^-200 of
    their real parts and coefficients whose real parts are 2^-90 of their
    imaginary parts (exact power-of-two scalings) stay within the md
    tolerance normwise (the metric R8); purely real inputs give exactly zero
    imaginary outputs."""
    si = mdinputs.random_system(770 + L, n=4, monos=5, m_range=(1, 3), exps=(1, 2), degree=9, limbs=L)
    si.x[:, 1] *= 2.0 ** -200
    si.coeffs[:, 0] *= 2.0 ** -90
    full_check(si, L)
    sr = mdinputs.random_system(780 + L, n=4, monos=5, m_range=(0, 3), exps=(1, 2), degree=9, limbs=L)
    sr.x[:, 1] = 0.0
    sr.coeffs[:, 1] = 0.0
    vals, jac = full_check(sr, L)
    assert not vals[:, 1].any() and not jac[:, :, 1].any()
