"""eval_diff time with and without the CUDA graph (small systems are launch bound)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdinputs  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402


def run(si, graph, iters=50):
    with mdps.System.from_inputs(si, use_graph=graph) as s:
        x = torch.from_numpy(si.x).cuda()
        v = torch.empty((si.n, 2, si.limbs, si.D), dtype=torch.float64, device="cuda")
        j = torch.empty((si.n, si.n, 2, si.limbs, si.D), dtype=torch.float64, device="cuda")
        for _ in range(5):
            s.eval_diff(x, v, j)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            s.eval_diff(x, v, j)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters


for name in sys.argv[1:] or ["dd", "qd", "sweep_d15_L2", "sweep_d15_L4"]:
    si = (mdinputs.sweep_cell(int(name.split("_")[1][1:]), int(name.split("_")[2][1:]))
          if name.startswith("sweep") else mdinputs.make_config(name))
    print(json.dumps({"config": name, "ms_plain": run(si, False), "ms_graph": run(si, True)}), flush=True)
