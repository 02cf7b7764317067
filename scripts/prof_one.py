"""One system, `--evals` evaluations (profiling driver for ncu; not a bench)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdinputs  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="od")
ap.add_argument("--algo", type=int, default=0)
ap.add_argument("--evals", type=int, default=2)
ap.add_argument("--geom", default="", help="forced product-kernel geometry F,P,NP (mdps_test_force_geometry)")
a = ap.parse_args()
if a.geom:
    mdps.force_geometry(*[int(v) for v in a.geom.split(",")])
si = (mdinputs.sweep_cell(int(a.config.split("_")[1][1:]), int(a.config.split("_")[2][1:]))
      if a.config.startswith("sweep") else mdinputs.make_config(a.config))
s = mdps.System.from_inputs(si, algo=a.algo)
print("levels:", s.level_jobs(), "stats:", s.stats(), flush=True)
x = torch.from_numpy(si.x).cuda()
for _ in range(a.evals):
    v, j = s.eval_diff(x)
torch.cuda.synchronize()
print("ok", float(v.abs().sum()), flush=True)
