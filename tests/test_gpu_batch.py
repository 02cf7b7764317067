"""Batched evaluation (mdps_options.batch): one system at B points per call,
the B copies of every product level in one launch.  The batch must equal B
separate evaluations bit for bit (the jobs are the same computations), for
both product algorithms and the real path."""
import numpy as np
import pytest

import mdinputs
import oracle
from tests.gpu_util import TOL, gpu_eval

pytestmark = pytest.mark.gpu


def points(si, B, seed):
    xs = [mdinputs.unit_circle_series(mdinputs.SplitMix64(seed + b, "x"), si.n, si.D, si.limbs,
                                      "zero" if si.name == "dd" else "random") for b in range(B)]
    return np.ascontiguousarray(np.stack(xs))


def gpu_eval_batch(si, X, algo=0, real=False):
    import torch
    import paper_2012_06607_b200 as mdps
    with mdps.System.from_inputs(si, algo=algo, real=real, batch=X.shape[0]) as s:
        v, j = s.eval_diff(torch.from_numpy(X).cuda())
        torch.cuda.synchronize()
        return v.cpu().numpy(), j.cpu().numpy(), s.stats()


@pytest.mark.parametrize("name,B,algo", [("dd", 5, 0), ("dd", 3, 1), ("qd", 3, 0)])
def test_batch_equals_separate_evaluations(name, B, algo):
    import dataclasses
    si = mdinputs.make_config(name)
    X = points(si, B, 900)
    vb, jb, st = gpu_eval_batch(si, X, algo)
    assert vb.shape == (B,) + (si.n, 2, si.limbs, si.D) and jb.shape == (B, si.n, si.n, 2, si.limbs, si.D)
    for b in range(B):
        v, j, st1 = gpu_eval(dataclasses.replace(si, x=X[b]), algo)
        assert np.array_equal(vb[b], v) and np.array_equal(jb[b], j), b
    assert st["products"] == B * st1["products"]


def test_batch_real_and_rectangular_against_oracle():
    import dataclasses
    si = mdinputs.realify(mdinputs.rect_system(61, 3, 5, 4, (1, 3), (1, 2), 9, 4))
    X = points(si, 4, 950)
    X[:, :, 1] = 0.0
    vb, jb, _ = gpu_eval_batch(si, X, real=True)
    for b in range(4):
        ov, oj, _ = oracle.eval_diff(dataclasses.replace(si, x=X[b]))
        assert oracle.series_err(vb[b], ov).max() <= TOL[4]
        assert oracle.series_err(jb[b], oj).max() <= TOL[4]
        assert not vb[b][:, 1].any()
