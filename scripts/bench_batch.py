"""Batched evaluation (mdps_options.batch): one system at B points per call.
CUDA events on the stream, L2 flushed between calls; products/s and the
product kernel's FP64 fraction per (config, B, algorithm)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mdinputs  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402

PEAK = 148 * 64 * 1.965e9


def run(name, B, algo, steps=5):
    si = mdinputs.make_config(name)
    X = np.ascontiguousarray(np.stack([si.x] * B))
    with mdps.System.from_inputs(si, algo=algo, batch=B) as s:
        x = torch.from_numpy(X).cuda()
        v, j = s.eval_diff(x)
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        s.set_timing(True)
        s.timing(reset=True)
        st = torch.cuda.current_stream()
        tot = 0.0
        for _ in range(steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            s.eval_diff(x, v, j)
            e1.record(st)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        t = s.timing(reset=True)
        stats = s.stats()
    ms = tot / steps
    return {"config": name, "batch": B, "algo": {1: "eft", 2: "digits"}[stats["algo"]], "ms": ms,
            "products_per_s": stats["products"] / (ms * 1e-3),
            "frac": stats["fp64_ops_conv"] / (t["conv_ms"] / steps * 1e-3) / PEAK}


for name, Bs in (("dd", (1, 16, 256, 1024)), ("qd", (1, 4, 16))):
    for B in Bs:
        for algo in (mdps.MDPS_ALGO_AUTO, mdps.MDPS_ALGO_EFT):
            print(json.dumps(run(name, B, algo)), flush=True)
