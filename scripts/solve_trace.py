"""Phase trace of one mdps_solve per config (grid-barrier completion times):
refinement phases, M, then the (dx, update) pairs of the substitution loop."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdinputs  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402

for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["od", "deca"]):
    t = mdinputs.toeplitz_config(name)
    with mdps.Solver(t.n, t.degree, t.limbs) as s:
        J, b = torch.from_numpy(t.jac).cuda(), torch.from_numpy(t.rhs).cuda()
        for _ in range(3):
            dx = s.solve(J, b)
        torch.cuda.synchronize()
        ts, refine = s.trace()
    d = [round((b_ - a) / 1e3, 1) for a, b_ in zip(ts, ts[1:])]
    print(json.dumps({"config": name, "refine_steps": refine, "total_us": round(ts[-1] / 1e3, 1),
                      "phase_us": d}))
