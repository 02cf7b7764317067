"""The digit product kernel under every launch geometry that fits
(mdps_test_force_geometry: F lanes per output pair x P jobs per block; NP = 2
one lane set per part, NP = 1 both parts on one thread — the fused-parts
kernel of L <= 5 —, NP = 3 the same with the fold parked in local memory), including F > D + 1 (lanes without terms), odd D (the
generic-D build) and several jobs per block: every geometry matches the
oracle within the tolerance, and the tuned defaults are among them; the
fused-parts kernel and the part-lane kernel give the same bits (both
accumulate exactly and round once)."""
import numpy as np
import pytest

import mdinputs
import oracle
from tests.gpu_util import TOL

pytestmark = pytest.mark.gpu

GEOMS = [(f, p, q) for q in (2, 1, 3) for f in (1, 2, 4, 8) for p in (1, 2, 4)]


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


@pytest.mark.parametrize("L,degree", [(2, 9), (3, 15), (4, 31), (4, 12), (5, 63), (5, 127)])
def test_fused_parts_kernel_equals_the_part_lane_kernel_bitwise(L, degree):
    import torch
    import paper_2012_06607_b200 as mdps
    si = mdinputs.random_system(950 + L + degree, n=4, monos=5, m_range=(1, 4), exps=(1, 2), degree=degree,
                                limbs=L)
    with mdps.System.from_inputs(si, algo=mdps.MDPS_ALGO_DIGITS) as s:
        x = torch.from_numpy(si.x).cuda()
        outs = {}
        try:
            for q in (2, 1, 3):
                for f in (1, 2, 4):
                    mdps.force_geometry(f, 0, q)
                    try:
                        v, j = s.eval_diff(x)
                    except mdps.MdpsError:
                        continue  # this F does not fit the kernel's thread limit
                    torch.cuda.synchronize()
                    outs[(q, f)] = (v.cpu().numpy(), j.cpu().numpy())
        finally:
            mdps.force_geometry(0, 0, 0)
    ref = outs[(2, 1)]
    assert len(outs) >= 7
    for key, (v, j) in outs.items():
        assert np.array_equal(v, ref[0]) and np.array_equal(j, ref[1]), key


@pytest.mark.parametrize("L,degree,graph", [(4, 31, False), (4, 31, True), (8, 15, False), (3, 63, True), (10, 31, False)])
def test_programmatic_dependent_launch_changes_nothing(L, degree, graph):
    """The product levels launched with programmatic stream serialization (the
    default: a level's blocks are scheduled while the previous level drains and
    wait for it before reading the pools), small levels on the wider launch
    geometry, give the same bits as plain stream order on the default geometry,
    evaluation after evaluation (a level reading a slot before its
    producer finished, or overwriting one still being read, would show up)."""
    import torch
    import paper_2012_06607_b200 as mdps
    si = mdinputs.random_system(970 + L + degree, n=12, monos=10, m_range=(2, 6), exps=(1, 2), degree=degree,
                                limbs=L)
    x = torch.from_numpy(si.x).cuda()
    try:
        mdps.set_pdl(False, small_levels=False, balance=False)
        with mdps.System.from_inputs(si, algo=mdps.MDPS_ALGO_DIGITS) as s:
            v, j = s.eval_diff(x)
            torch.cuda.synchronize()
            ref = (v.cpu().numpy(), j.cpu().numpy())
        mdps.set_pdl(True)
        with mdps.System.from_inputs(si, algo=mdps.MDPS_ALGO_DIGITS, use_graph=graph) as s:
            v = torch.empty_like(v)
            j = torch.empty_like(j)
            for _ in range(25):
                v.zero_()
                j.zero_()
                s.eval_diff(x, v, j)
                torch.cuda.synchronize()
                assert np.array_equal(v.cpu().numpy(), ref[0]) and np.array_equal(j.cpu().numpy(), ref[1])
    finally:
        mdps.set_pdl(True)


def test_level_balancing_changes_nothing():
    """Summed-only products moved into later, emptier levels (balance_levels):
    the qd config's last levels fill up to one wave, the outputs stay bit for
    bit those of the earliest-level schedule."""
    import torch
    import paper_2012_06607_b200 as mdps
    si = mdinputs.make_config("qd")
    x = torch.from_numpy(si.x).cuda()
    try:
        mdps.set_pdl(True, balance=False)
        with mdps.System.from_inputs(si) as s:
            lv0 = s.level_jobs()
            v, j = s.eval_diff(x)
            torch.cuda.synchronize()
            ref = (v.cpu().numpy(), j.cpu().numpy())
        mdps.set_pdl(True)
        with mdps.System.from_inputs(si) as s:
            lv1 = s.level_jobs()
            v, j = s.eval_diff(x)
            torch.cuda.synchronize()
            assert np.array_equal(v.cpu().numpy(), ref[0]) and np.array_equal(j.cpu().numpy(), ref[1])
    finally:
        mdps.set_pdl(True)
    assert sum(lv0) == sum(lv1) and len(lv0) == len(lv1)
    assert min(lv1) > min(lv0) and lv1 != lv0


@pytest.mark.parametrize("name,mb", [("qd", 48), ("qd", 24)])
def test_row_chunks_change_nothing(name, mb):
    """Under a workspace bound (mdps_options.workspace_mb) the rows run in
    chunks, each its (balanced) levels then its own addition jobs, with the
    pool slots reused across chunks: the outputs equal the unchunked
    evaluation's bit for bit."""
    import torch
    import paper_2012_06607_b200 as mdps
    si = mdinputs.make_config(name)
    x = torch.from_numpy(si.x).cuda()
    with mdps.System.from_inputs(si) as s:
        assert s.stats()["chunks"] == 1
        v, j = s.eval_diff(x)
        torch.cuda.synchronize()
        ref = (v.cpu().numpy(), j.cpu().numpy())
    with mdps.System.from_inputs(si, workspace_mb=mb) as s:
        st = s.stats()
        assert st["chunks"] >= 2 and st["workspace_bytes"] <= (mb << 20) * 1.05
        for _ in range(2):
            v, j = s.eval_diff(x)
            torch.cuda.synchronize()
            assert np.array_equal(v.cpu().numpy(), ref[0]) and np.array_equal(j.cpu().numpy(), ref[1])
