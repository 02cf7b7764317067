"""Host-only checks of the job schedule and its memory plan (no GPU; the
C-ABI library's mdps_test_plan): every slot index in range, every product
input written by an EARLIER launch, no slot read and written in one launch,
no live slot overwritten, every summed series intact until its addition jobs
(schedule.hpp check_schedule) — the bounds and race-freedom invariants of the
kernels' global-memory traffic, which compute-sanitizer would otherwise be
asked to find (it is closed on this GPU pool).  Also: the checker catches
deliberately damaged plans, and liveness reuse bounds the workspace."""
import pytest

import mdinputs
import paper_2012_06607_b200 as mdps
from paper_2012_06607_b200 import build as mdps_build


@pytest.fixture(scope="module", autouse=True)
def built():
    mdps_build.build()
    mdps.lib()


CASES = [("dd", None), ("qd", None), ("od", None), ("deca", None), ("sweep", None),
         ("rand_consts", dict(seed=5, n=9, monos=7, m_range=(0, 6), exps=(1, 2, 3), degree=9, limbs=4)),
         ("rand_m1", dict(seed=6, n=5, monos=9, m_range=(1, 2), exps=(1, 4), degree=3, limbs=8))]


def system(name, kw):
    if kw is None:
        return mdinputs.make_config(name) if name != "sweep" else mdinputs.sweep_cell(63, 8)
    return mdinputs.random_system(kw["seed"], n=kw["n"], monos=kw["monos"], m_range=kw["m_range"],
                                  exps=kw["exps"], degree=kw["degree"], limbs=kw["limbs"])


@pytest.mark.parametrize("name,kw", CASES)
@pytest.mark.parametrize("eft", (False, True))
def test_plans_check(name, kw, eft):
    si = system(name, kw)
    for chunks in (1, 2, 3, 7):
        rc, info, msg = mdps.test_plan(si, eft, chunks=chunks)
        assert rc == 0, (chunks, msg)
        assert info["planned_bytes"] <= info["unplanned_bytes"]
        assert 1 <= info["chunks"] <= chunks
    if name in ("dd", "rand_consts"):
        rc, info, msg = mdps.test_plan(si, eft, batch=3)
        assert rc == 0, msg


@pytest.mark.parametrize("corrupt", (1, 2, 3))
@pytest.mark.parametrize("eft", (False, True))
def test_checker_catches_damaged_plans(corrupt, eft):
    si = mdinputs.make_config("qd")
    rc, _, msg = mdps.test_plan(si, eft, corrupt=corrupt)
    assert rc == mdps.MDPS_EINVAL and "schedule check" in msg, (rc, msg)


def test_workspace_bounds():
    """liveness reuse (one chunk) and row chunks shrink the pools."""
    out = {}
    for name in ("od", "deca"):
        si = mdinputs.make_config(name)
        rc, one, _ = mdps.test_plan(si, False, chunks=1)
        rc4, four, _ = mdps.test_plan(si, False, chunks=4)
        assert rc == 0 and rc4 == 0
        assert one["planned_bytes"] < 0.5 * one["unplanned_bytes"]
        assert four["planned_bytes"] < 0.45 * one["planned_bytes"]
        out[name] = (one, four)
    assert out["od"][1]["planned_bytes"] < 1 << 30
    assert out["deca"][1]["planned_bytes"] < 3 << 30


@pytest.mark.parametrize("name,min_jobs", [("qd", 1776), ("qd", 4000), ("dd", 100), ("od", 20000), ("qd", 10 ** 6)])
def test_level_balancing_keeps_the_jobs_and_passes_the_checks(name, min_jobs):
    """balance_levels (schedule.hpp): the balanced levels hold exactly the
    original jobs, none moved to an earlier level, every moved job summed
    only; later levels below the target fill up to it while earlier levels
    above it have such jobs to give; the balanced schedule passes the schedule
    check and the memory plan's check."""
    import mdinputs
    import paper_2012_06607_b200 as mdps
    si = mdinputs.make_config(name)
    rc, before, after, moved, same, msg = mdps.test_balance(si, min_jobs)
    assert rc > 0, msg
    assert same == 1
    assert sum(before) == sum(after) and len(before) == len(after) == rc
    assert moved == sum(max(0, a - b) for a, b in zip(after, before))
    for b, a in zip(before, after):
        assert a <= max(b, min_jobs)          # a level grows at most to the target
        assert a >= min(b, min_jobs)          # and gives only what it holds above it
    if name == "qd" and min_jobs == 1776:
        assert before[-3:] == [1476, 856, 270] and after[-3:] == [1776, 1776, 1776] and moved == 2726
