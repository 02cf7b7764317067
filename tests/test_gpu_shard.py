"""Rectangular systems (N != n) and row sharding on the GPU: each shard's
outputs equal the full system's rows bit for bit (the product jobs of a row
do not depend on the other rows), and a row subset matches the oracle."""
import numpy as np
import pytest

import mdinputs
import oracle
from paper_2012_06607_b200 import shard
from tests.gpu_util import TOL, gpu_eval

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,parts", [("dd", 3), ("qd", 2), ("sweep_d31_L4", 4)])
def test_shards_reassemble_bitwise(name, parts):
    si = (mdinputs.sweep_cell(31, 4) if name.startswith("sweep") else mdinputs.make_config(name))
    vals, jac, _ = gpu_eval(si)
    rows = shard.partition_rows(shard.row_products(si.poly_ptr, si.mono_ptr, si.exps), parts)
    for part in rows:
        pp, mp_, vv, ee, cc = shard.subsystem(si.poly_ptr, si.mono_ptr, si.vars, si.exps, si.coeffs, part)
        sub = mdinputs.SystemInputs("part", si.n, si.degree, si.limbs, pp, mp_, vv, ee, cc, si.x)
        v, j, st = gpu_eval(sub)
        assert v.shape == (len(part),) + vals.shape[1:] and j.shape == (len(part),) + jac.shape[1:]
        assert np.array_equal(v, vals[part]) and np.array_equal(j, jac[part])


@pytest.mark.parametrize("L", (2, 8))
@pytest.mark.parametrize("N,n", [(3, 7), (9, 5)])
def test_rectangular_against_oracle(L, N, n):
    """N polynomials in n variables, N < n and N > n."""
    si = mdinputs.rect_system(40 + N, N, n, 4, (1, 3), (1, 2), 7, L)
    vals, jac, _ = gpu_eval(si)
    ov, oj, _ = oracle.eval_diff(si)
    assert vals.shape == ov.shape == (N, 2, L, si.D) and jac.shape == oj.shape == (N, n, 2, L, si.D)
    assert oracle.series_err(vals, ov).max() <= TOL[L]
    assert oracle.series_err(jac, oj).max() <= TOL[L]
