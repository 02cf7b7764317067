"""Whole-step time of mdps_eval_diff with the product levels launched by
programmatic dependent launch (default) against plain stream order, with and
without the CUDA graph: CUDA events around each evaluation, L2 flushed, no
per-kernel instrumentation."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdinputs  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402

CELLS = sys.argv[1].split(",") if len(sys.argv) > 1 else [
    "qd", "sweep_d15_L3", "sweep_d15_L4", "sweep_d15_L5", "sweep_d15_L8", "sweep_d31_L4", "sweep_d63_L4", "od"]


def workload(c):
    if c.startswith("sweep"):
        _, d, L = c.split("_")
        return mdinputs.sweep_cell(int(d[1:]), int(L[1:]))
    return mdinputs.make_config(c)


flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for c in CELLS:
    si = workload(c)
    x = torch.from_numpy(si.x).cuda()
    v = torch.empty((si.n, 2, si.limbs, si.D), dtype=torch.float64, device="cuda")
    j = torch.empty((si.n, si.n, 2, si.limbs, si.D), dtype=torch.float64, device="cuda")
    row = {"cell": c}
    for graph in (False, True):
        # 2: programmatic launch, but every level on the default geometry; 3: no level balancing
        for pdl in (False, True, 2, 3):
            mdps.set_pdl(bool(pdl), small_levels=pdl != 2, balance=pdl != 3)
            with mdps.System.from_inputs(si, algo=mdps.MDPS_ALGO_DIGITS, use_graph=graph) as s:
                for _ in range(3):
                    s.eval_diff(x, v, j)
                torch.cuda.synchronize()
                ts = []
                for _ in range(10 if si.limbs * si.D <= 512 else 4):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    s.eval_diff(x, v, j)
                    b.record()
                    torch.cuda.synchronize()
                    ts.append(a.elapsed_time(b))
                ts.sort()
                row[f"graph={int(graph)},pdl={int(bool(pdl))}" + (",default_geometry" if pdl == 2 else ",unbalanced_levels" if pdl == 3 else "")] = ts[len(ts) // 2]
    mdps.set_pdl(True)
    print(json.dumps(row), flush=True)
