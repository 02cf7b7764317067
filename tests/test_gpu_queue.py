"""The device-side job queue (MDPS_SCHED_QUEUE, PAPER.md:367-378
Fig. 1 job queue, 411-424 stages): one persistent launch, jobs claimed from a
device counter in topological order, each waiting only on its own inputs'
ready flags.  Checked against the oracle (every output) on the dd config and
on small systems with every structural case, for bitwise run-to-run
determinism, for the epoch handling across evaluations (no reset between
calls), under a CUDA graph and with batches."""
import numpy as np
import pytest

import mdinputs
import oracle
from tests.gpu_util import TOL, structural_support
from tests.test_oracle_newton import circle_system

pytestmark = pytest.mark.gpu
LEVELS = (2, 3, 4, 5, 8, 10)


@pytest.fixture(scope="module")
def mdps():
    import paper_2012_06607_b200 as m
    m.lib()
    return m


def run(mdps, si, xs, **kw):
    import torch
    with mdps.System.from_inputs(si, **kw) as s:
        st = s.stats()
        outs = []
        for x in xs:
            v, j = s.eval_diff(torch.from_numpy(np.ascontiguousarray(x)).cuda())
            torch.cuda.synchronize()
            outs.append((v.cpu().numpy(), j.cpu().numpy()))
        return outs, st


def check(si, v, j, L):
    ov, oj, _ = oracle.eval_diff(si)
    assert oracle.series_err(v, ov).max() <= TOL[L]
    assert oracle.series_err(j, oj).max() <= TOL[L]
    assert not j[~structural_support(si)].any()


def test_dd_auto_uses_queue_and_matches_oracle(mdps):
    si = mdinputs.make_config("dd")
    (out,), st = run(mdps, si, [si.x])
    assert st["schedule"] == mdps.MDPS_SCHED_QUEUE and st["launches"] == 1 and st["algo"] == mdps.MDPS_ALGO_EFT
    check(si, *out, 2)
    # the leveled schedule agrees within the tolerance (a different summation order)
    (lv,), st2 = run(mdps, si, [si.x], schedule=mdps.MDPS_SCHED_LEVELS)
    assert st2["schedule"] == mdps.MDPS_SCHED_LEVELS
    assert oracle.series_err(out[1], lv[1]).max() <= TOL[2]


@pytest.mark.parametrize("L", LEVELS)
def test_small_systems_every_case(mdps, L):
    """constants, m = 1, exponents 2 and 3, odd degree, forced queue."""
    si = mdinputs.random_system(900 + L, n=5, monos=7, m_range=(0, 5), exps=(1, 2, 3), degree=12, limbs=L)
    (out,), st = run(mdps, si, [si.x], algo=mdps.MDPS_ALGO_EFT, schedule=mdps.MDPS_SCHED_QUEUE)
    assert st["launches"] == 1
    check(si, *out, L)


@pytest.mark.parametrize("degree", (0, 1, 2, 15, 31, 64, 127))
def test_degrees(mdps, degree):
    L = 3
    si = mdinputs.random_system(950 + degree, n=4, monos=5, m_range=(1, 4), exps=(1, 2), degree=degree, limbs=L)
    (out,), _ = run(mdps, si, [si.x], algo=mdps.MDPS_ALGO_EFT, schedule=mdps.MDPS_SCHED_QUEUE)
    check(si, *out, L)


def test_circle_system(mdps):
    si = circle_system(8)
    (out,), _ = run(mdps, si, [si.x], algo=mdps.MDPS_ALGO_EFT, schedule=mdps.MDPS_SCHED_QUEUE)
    check(si, *out, 8)


def test_determinism_and_epochs(mdps):
    """30 evaluations at alternating points: every result bitwise equal to the
    first evaluation at the same point (flags are never reset: epochs)."""
    si = mdinputs.make_config("dd")
    x2 = si.x.copy()
    x2[:, 0, 0, 1] *= 0.5
    outs, _ = run(mdps, si, [si.x if k % 2 == 0 else x2 for k in range(30)])
    for k in range(2, 30):
        assert np.array_equal(outs[k][0], outs[k % 2][0]) and np.array_equal(outs[k][1], outs[k % 2][1])
    assert not np.array_equal(outs[0][0], outs[1][0])


def test_graph_and_batch(mdps):
    import torch
    si = mdinputs.make_config("dd")
    (ref,), _ = run(mdps, si, [si.x])
    with mdps.System.from_inputs(si, use_graph=True) as s:
        x = torch.from_numpy(si.x).cuda()
        for _ in range(4):
            v, j = s.eval_diff(x)
        torch.cuda.synchronize()
        assert np.array_equal(v.cpu().numpy(), ref[0]) and np.array_equal(j.cpu().numpy(), ref[1])
    B = 3
    xb = np.stack([si.x * (1.0 if b == 0 else 0.5 ** b) for b in range(B)])
    (outb,), st = run(mdps, si, [xb], batch=B, schedule=mdps.MDPS_SCHED_QUEUE, algo=mdps.MDPS_ALGO_EFT)
    assert st["schedule"] == mdps.MDPS_SCHED_QUEUE
    for b in range(B):
        (one,), _ = run(mdps, si, [xb[b]])
        assert np.array_equal(outb[0][b], one[0]) and np.array_equal(outb[1][b], one[1])


def test_rectangular_and_larger(mdps):
    """N != n, and a system of ~86k products forced through the queue (sweep
    d = 15, L = 2: many waves of tickets), sampled against the oracle."""
    from tests.gpu_util import check_against_oracle, sample_entries
    si = mdinputs.random_system(990, n=6, monos=4, m_range=(1, 4), exps=(1, 2), degree=9, limbs=4)
    sub = mdinputs.subsystem(si, [0, 2, 5])
    (out,), _ = run(mdps, sub, [sub.x], algo=mdps.MDPS_ALGO_EFT, schedule=mdps.MDPS_SCHED_QUEUE)
    check(sub, *out, 4)
    sw = mdinputs.sweep_cell(15, 2)
    (out,), _ = run(mdps, sw, [sw.x], algo=mdps.MDPS_ALGO_EFT, schedule=mdps.MDPS_SCHED_QUEUE)
    err, _ = check_against_oracle(sw, out[0], out[1], sample_entries(sw, 4, 12, seed=3), TOL[2])
    assert err <= TOL[2]


def test_queue_needs_eft(mdps):
    si = mdinputs.make_config("dd")
    with pytest.raises(mdps.MdpsError, match="EFT"):
        mdps.System.from_inputs(si, algo=mdps.MDPS_ALGO_DIGITS, schedule=mdps.MDPS_SCHED_QUEUE)
