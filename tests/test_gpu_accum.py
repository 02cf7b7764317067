"""The addition jobs on lanes (8 lanes per value coefficient,
2 or 1 per Jacobian coefficient, merged in a fixed tree): polynomials of 1 to
70 monomials — entry counts below, at and across the lane counts, odd and even
—, weighted entries (exponents 2 and 3), odd D (lane groups straddling rows of
the thread layout), both algorithms, every output against the oracle; the
structural zeros exact; and the same outputs run after run."""
import numpy as np
import pytest

import mdinputs
import oracle
from tests.gpu_util import TOL, gpu_eval, structural_support

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("monos", [1, 2, 7, 8, 9, 17, 33, 70])
@pytest.mark.parametrize("L,degree", [(2, 6), (4, 15), (8, 20)])
def test_entry_counts_around_the_lane_counts(monos, L, degree):
    si = mdinputs.random_system(4000 + 10 * monos + L, n=4, monos=monos, m_range=(0 if monos > 2 else 1, 3),
                                exps=(1, 2, 3), degree=degree, limbs=L)
    ov, oj, _ = oracle.eval_diff(si)
    sup = structural_support(si)
    for algo in (1, 2):
        vals, jac, _ = gpu_eval(si, algo)
        assert oracle.series_err(vals, ov).max() <= TOL[L], (algo, monos)
        assert oracle.series_err(jac, oj).max() <= TOL[L], (algo, monos)
        assert not jac[~sup].any()
        v2, j2, _ = gpu_eval(si, algo)
        assert np.array_equal(vals, v2) and np.array_equal(jac, j2)
