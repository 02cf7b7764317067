"""Real systems (mdps_options.real; SURVEY §8(f) #3 "a real md path"): one real
md product per term.  For real inputs the complex path accumulates the same
exact real parts (its imaginary products are exact zeros); the two modes may
pick different launch geometries, hence different (equally exact) digit
representations and a last-place difference after rounding — so real mode must
agree with the complex mode to a few units of 2^-53L, have exactly zero
imaginary outputs, and match the oracle within the tolerance."""
import numpy as np
import pytest

import mdinputs
import oracle
from tests.gpu_util import TOL, gpu_eval, sample_entries, check_against_oracle

pytestmark = pytest.mark.gpu


def gpu_eval_real(si):
    import torch
    import paper_2012_06607_b200 as mdps
    with mdps.System.from_inputs(si, real=True) as sys_:
        x = torch.from_numpy(si.x).cuda()
        vals, jac = sys_.eval_diff(x)
        torch.cuda.synchronize()
        return vals.cpu().numpy(), jac.cpu().numpy(), sys_.stats()


@pytest.mark.parametrize("name", ["dd", "qd", "sweep_d31_L5", "sweep_d15_L10"])
def test_real_mode_equals_complex_mode(name):
    si = mdinputs.realify(mdinputs.sweep_cell(int(name.split("_")[1][1:]), int(name.split("_")[2][1:]))
                          if name.startswith("sweep") else mdinputs.make_config(name))
    v1, j1, st1 = gpu_eval(si, 2)  # the complex digit path (the default is EFT at L = 2)
    v2, j2, st2 = gpu_eval_real(si)
    assert not v2[:, 1].any() and not j2[:, :, 1].any()
    L = si.limbs
    assert oracle.series_err(v2, v1).max() <= 8 * 2.0 ** (-53 * L)
    assert oracle.series_err(j2, j1).max() <= 8 * 2.0 ** (-53 * L)
    assert st2["fp64_ops_conv"] * 4 == st1["fp64_ops_conv"]


@pytest.mark.parametrize("name,nv,nj", [("dd", 8, 40), ("od", 1, 3)])
def test_real_mode_against_oracle(name, nv, nj):
    si = mdinputs.realify(mdinputs.make_config(name))
    vals, jac, _ = gpu_eval_real(si)
    ent = sample_entries(si, nv, nj, seed=3)
    err, _ = check_against_oracle(si, vals, jac, ent, TOL[si.limbs])
    assert err <= TOL[si.limbs]
