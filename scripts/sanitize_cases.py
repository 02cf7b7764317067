"""Small launches for compute-sanitizer (scripts/sanitize.sh): one case per
run, results checked against the oracle so a run that 'passes' the sanitizer
also computed the right thing.

  python scripts/sanitize_cases.py {dd_queue,dd_levels,digits_small,digits_odd,eft_odd,solve,solve_ls}
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mdinputs  # noqa: E402
import oracle  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402

TOL = {2: 1e-29, 3: 1e-45, 4: 1e-61, 5: 1e-77, 8: 1e-124, 10: 1e-156}


def evalcheck(si, **kw):
    with mdps.System.from_inputs(si, **kw) as s:
        x = torch.from_numpy(si.x).cuda()
        for _ in range(2):  # twice: the queue's epochs, the graph cache
            v, j = s.eval_diff(x)
        torch.cuda.synchronize()
        st = s.stats()
    ov, oj, _ = oracle.eval_diff(si)
    e = max(oracle.series_err(v.cpu().numpy(), ov).max(), oracle.series_err(j.cpu().numpy(), oj).max())
    assert e <= TOL[si.limbs], e
    print(f"ok algo={st['algo']} schedule={st['schedule']} err={e:.2e}")


def solvecheck(N, n, L, degree):
    t = mdinputs.random_toeplitz(77, n, degree, L) if N == n else None
    if t is None:
        rng = np.random.default_rng(5)
        big = mdinputs.random_toeplitz(78, N, degree, L)
        jac = np.ascontiguousarray(big.jac[:, :n])
        rhs = big.rhs
    else:
        jac, rhs = t.jac, t.rhs
    with mdps.Solver(n, degree, L, n_eqs=N) as s:
        dx = s.solve(torch.from_numpy(jac).cuda(), torch.from_numpy(rhs).cuda())
        torch.cuda.synchronize()
        flags = s.flags()
    assert flags == 0, flags
    if N == n:
        want, _ = oracle.toeplitz_solve(jac, rhs)
        e = oracle.series_err(dx.cpu().numpy(), want).max()
        assert e <= TOL[L], e
        print(f"ok solve err={e:.2e}")
    else:
        print("ok least-squares solve ran (flags 0)")


case = sys.argv[1]
mdps.lib()
if case == "dd_queue":
    evalcheck(mdinputs.make_config("dd"))
elif case == "dd_levels":
    evalcheck(mdinputs.make_config("dd"), schedule=mdps.MDPS_SCHED_LEVELS)
elif case == "digits_small":
    evalcheck(mdinputs.random_system(31, n=5, monos=4, m_range=(0, 4), exps=(1, 2), degree=15, limbs=4),
              algo=mdps.MDPS_ALGO_DIGITS)
elif case == "digits_odd":
    evalcheck(mdinputs.random_system(32, n=4, monos=3, m_range=(1, 3), exps=(1, 2, 3), degree=12, limbs=8),
              algo=mdps.MDPS_ALGO_DIGITS)
elif case == "eft_odd":
    evalcheck(mdinputs.random_system(33, n=4, monos=3, m_range=(1, 3), exps=(1, 2), degree=20, limbs=3),
              algo=mdps.MDPS_ALGO_EFT, schedule=mdps.MDPS_SCHED_LEVELS)
elif case == "solve":
    solvecheck(6, 6, 4, 7)
elif case == "solve_ls":
    solvecheck(8, 5, 2, 5)
else:
    raise SystemExit(f"unknown case {case}")
