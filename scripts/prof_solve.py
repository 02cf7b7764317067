"""One mdps_solve on a config's shape (profiling driver for ncu; not a bench)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdinputs  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402

t = mdinputs.toeplitz_config(sys.argv[1] if len(sys.argv) > 1 else "od")
with mdps.Solver(t.n, t.degree, t.limbs) as s:
    J, b = torch.from_numpy(t.jac).cuda(), torch.from_numpy(t.rhs).cuda()
    dx = s.solve(J, b)
    torch.cuda.synchronize()
print("ok", float(dx.abs().sum()))
