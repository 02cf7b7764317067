"""The digit product kernel under every launch geometry that fits
(mdps_test_force_geometry: F lanes per output pair x P jobs per block; one
lane set per part),
including F > D + 1 (lanes without terms), odd D (the generic-D build, scalar
staging) and several jobs per block: every geometry matches the oracle within
the tolerance, and the tuned defaults are among them; a complex system
rejects NP = 1."""
import numpy as np
import pytest

import mdinputs
import oracle
from tests.gpu_util import TOL

pytestmark = pytest.mark.gpu

GEOMS = [(f, p, 2) for f in (1, 2, 4, 8) for p in (1, 2, 4)]  # complex: one lane set per part


@pytest.mark.parametrize("L,degree", [(2, 6), (4, 15), (8, 31), (10, 15), (3, 63)])
def test_every_fitting_geometry_matches_the_oracle(L, degree):
    import torch
    import paper_2012_06607_b200 as mdps
    si = mdinputs.random_system(900 + L + degree, n=5, monos=6, m_range=(1, 4), exps=(1, 2), degree=degree,
                                limbs=L)
    ov, oj, _ = oracle.eval_diff(si)
    ran = 0
    try:
        with mdps.System.from_inputs(si, algo=mdps.MDPS_ALGO_DIGITS) as s:
            x = torch.from_numpy(si.x).cuda()
            for f, p, q in GEOMS:
                mdps.force_geometry(f, p, q)
                try:
                    v, j = s.eval_diff(x)
                except mdps.MdpsError:
                    continue  # does not fit this kernel's thread / shared-memory limits
                torch.cuda.synchronize()
                v, j = v.cpu().numpy(), j.cpu().numpy()
                assert oracle.series_err(v, ov).max() <= TOL[L], (f, p, q)
                assert oracle.series_err(j, oj).max() <= TOL[L], (f, p, q)
                ran += 1
    finally:
        mdps.force_geometry(0, 0, 0)
    assert ran >= 3


def test_complex_systems_reject_one_lane_set():
    import torch
    import paper_2012_06607_b200 as mdps
    si = mdinputs.random_system(950, n=3, monos=3, m_range=(1, 3), exps=(1,), degree=7, limbs=4)
    with mdps.System.from_inputs(si, algo=mdps.MDPS_ALGO_DIGITS) as s:
        x = torch.from_numpy(si.x).cuda()
        try:
            mdps.force_geometry(2, 1, 1)
            with pytest.raises(mdps.MdpsError, match="NP = 2"):
                s.eval_diff(x)
        finally:
            mdps.force_geometry(0, 0, 0)
