"""Randomised stress of the product kernels on inputs with a wide exponent
range inside every series: each coefficient of x and of the monomial
coefficients scaled by its own 2^k, k uniform in [-60, 60] (exact), a tenth
of the complex coefficients exactly zero and a tenth of the parts zero.
Terms of one output then differ by up to ~10 radix digits, so the digit
kernel's alignment shifts leave the PADZ window (the select-based slow path),
leading digits of outputs are zero (the emit's leading-digit exchange between
the part lanes, DESIGN R20), and zero coefficients take the ZERO_E encoding.
Both algorithms against the oracle, every output, the north-star tolerance."""
import numpy as np
import pytest

import mdinputs
import oracle
from tests.gpu_util import TOL, gpu_eval, structural_support

pytestmark = pytest.mark.gpu


def scramble(si, seed):
    rng = np.random.default_rng(seed)
    for arr in (si.x, si.coeffs):
        nser, _, L, D = arr.shape
        k = rng.integers(-60, 61, size=(nser, 1, 1, D))
        arr *= np.ldexp(1.0, k)                       # exact per-coefficient scaling
    for arr in (si.x, si.coeffs):
        nser, _, L, D = arr.shape
        zc = rng.random((nser, D)) < 0.1
        for s, kk in zip(*np.nonzero(zc)):
            arr[s, :, :, kk] = 0.0
        zp = rng.random((nser, 2, D)) < 0.1
        for s, p, kk in zip(*np.nonzero(zp)):
            arr[s, p, :, kk] = 0.0
    return si


@pytest.mark.parametrize("seed,L,degree", [(1, 3, 15), (2, 5, 31), (3, 8, 20), (4, 4, 63), (5, 10, 9), (6, 2, 17)])
def test_wide_exponent_range(seed, L, degree):
    si = mdinputs.random_system(990 + seed, n=5, monos=6, m_range=(0, 4), exps=(1, 2, 3), degree=degree, limbs=L)
    si = scramble(si, seed)
    ov, oj, _ = oracle.eval_diff(si)
    sup = structural_support(si)
    for algo in (1, 2):
        vals, jac, _ = gpu_eval(si, algo)
        ev = oracle.series_err(vals, ov).max()
        ej = oracle.series_err(jac, oj).max()
        assert ev <= TOL[L] and ej <= TOL[L], (algo, ev, ej)
        assert not jac[~sup].any()
