"""Job-queue geometry on a small configuration: grid cap x lanes per output
pair; single-evaluation latency (CUDA events + synchronize, median of 50) and
back-to-back time, each with and without a CUDA graph.

  python scripts/queue_tune.py [config]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402
from scripts.bench_small import measure  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "dd"
si = bench.workload(name)
for blocks in (0, 1184, 592, 296):
    for lanes in (4, 8, 16):
        mdps.queue_config(blocks, lanes)
        for graph in (False, True):
            st, med, mn, b2b = measure(si, algo=1, schedule=2, use_graph=graph)
            print(json.dumps({"config": name, "max_blocks": blocks, "lanes": lanes, "graph": graph,
                              "single_ms_median": med, "single_ms_min": mn, "back_to_back_ms": b2b}), flush=True)
mdps.queue_config(0, 0)
