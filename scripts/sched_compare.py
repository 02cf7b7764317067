"""Leveled launches vs the digit job queue on mid-size configurations:
back-to-back time per evaluation (CUDA events, 20 evaluations after warm-up,
L2 not flushed) and the product kernel's FP64 fraction.

  python scripts/sched_compare.py [configs...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402

PEAK = 148 * 64 * 1965e6

names = sys.argv[1:] or ["qd", "sweep_d15_L4", "sweep_d15_L5", "sweep_d31_L4", "sweep_d31_L5", "sweep_d15_L8",
                         "sweep_d15_L10", "sweep_d31_L8", "sweep_d63_L4"]
for name in names:
    si = bench.workload(name)
    for sched in (1, 2):
        try:
            with mdps.System.from_inputs(si, algo=2, schedule=sched) as s:
                st = s.stats()
                x = torch.from_numpy(si.x).cuda()
                v, j = s.eval_diff(x)
                for _ in range(3):
                    s.eval_diff(x, v, j)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(20):
                    s.eval_diff(x, v, j)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 20
            print(json.dumps({"config": name, "schedule": {1: "levels", 2: "queue"}[sched], "ms": ms,
                              "products": st["products"], "frac_conv_alg": st["fp64_ops_conv"] / (ms * 1e-3) / PEAK,
                              "launches": st["launches"]}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"config": name, "schedule": sched, "error": str(e)}), flush=True)
