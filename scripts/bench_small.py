"""Latency of one small evaluation (dd and small sweep cells) under each
schedule: the device-side job queue (one persistent launch) vs one launch per
level, each with and without a CUDA graph.  Per configuration: the median of
single evaluations each bracketed by CUDA events with a synchronize (the
latency of one call), and back-to-back evaluations (throughput).

  python scripts/bench_small.py [configs...]   -> one JSON line per (config, schedule)
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402


def measure(si, **kw):
    with mdps.System.from_inputs(si, **kw) as s:
        st = s.stats()
        x = torch.from_numpy(si.x).cuda()
        v, j = s.eval_diff(x)
        for _ in range(20):
            s.eval_diff(x, v, j)
        torch.cuda.synchronize()
        single = []
        for _ in range(50):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            s.eval_diff(x, v, j)
            e1.record()
            torch.cuda.synchronize()
            single.append(e0.elapsed_time(e1))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            s.eval_diff(x, v, j)
        e1.record()
        torch.cuda.synchronize()
        return st, statistics.median(single), min(single), e0.elapsed_time(e1) / 200


def main():
    names = sys.argv[1:] or ["dd", "sweep_d15_L2", "sweep_d15_L3", "sweep_d31_L2"]
    for name in names:
        si = bench.workload(name)
        for label, kw in (("queue", dict(algo=1, schedule=2)), ("queue+graph", dict(algo=1, schedule=2, use_graph=True)),
                          ("levels", dict(algo=1, schedule=1)), ("levels+graph", dict(algo=1, schedule=1, use_graph=True))):
            try:
                st, med, mn, b2b = measure(si, **kw)
                print(json.dumps({"config": name, "schedule": label, "products": st["products"],
                                  "launches": st["launches"], "single_ms_median": med, "single_ms_min": mn,
                                  "back_to_back_ms": b2b, "products_per_s_b2b": st["products"] / (b2b * 1e-3)}),
                      flush=True)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"config": name, "schedule": label, "error": str(e)}), flush=True)


if __name__ == "__main__":
    main()
