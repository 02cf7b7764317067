"""Critical path of one job-queue evaluation (mdps_test_queue_trace): per DAG
level, when its jobs were claimed, got their inputs and finished, relative to
the first claim; then the addition tickets.

  python scripts/queue_trace.py [config]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "dd"
si = bench.workload(name)
with mdps.System.from_inputs(si, algo=1, schedule=2) as s:
    x = torch.from_numpy(si.x).cuda()
    v, j = s.eval_diff(x)
    s.queue_trace(enable=True)
    for _ in range(5):
        s.eval_diff(x, v, j)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s.eval_diff(x, v, j)
    e1.record()
    torch.cuda.synchronize()
    tr = s.queue_trace(read=True).astype(np.float64)
    levels = s.level_jobs()
    t0 = tr[:, 0].min()
    tr -= t0
    out = {"config": name, "event_ms": e0.elapsed_time(e1), "span_us": float(tr.max() / 1e3), "levels": []}
    off = 0
    for lv, cnt in enumerate(levels):
        seg = tr[off:off + cnt] / 1e3
        out["levels"].append({"level": lv + 1, "jobs": cnt, "claim_us": [float(seg[:, 0].min()), float(seg[:, 0].max())],
                              "ready_us": [float(seg[:, 1].min()), float(seg[:, 1].max())],
                              "done_us": [float(seg[:, 4].min()), float(seg[:, 4].max())],
                              "median_us": {"stage": float(np.median(seg[:, 2] - seg[:, 1])),
                                            "compute": float(np.median(seg[:, 3] - seg[:, 2])),
                                            "release": float(np.median(seg[:, 4] - seg[:, 3]))}})
        off += cnt
    seg = tr[off:] / 1e3
    out["add"] = {"tickets": len(seg), "claim_us": [float(seg[:, 0].min()), float(seg[:, 0].max())],
                  "ready_us": [float(seg[:, 1].min()), float(seg[:, 1].max())],
                  "done_us": [float(seg[:, 4].min()), float(seg[:, 4].max())]}
    print(json.dumps(out, indent=1))
