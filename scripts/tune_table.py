"""Product-kernel launch geometry per (L, D): time every (F, P, NP) that fits on
the sweep cells and the configs, in one process per cell list
(mdps_test_force_geometry), and print the measured best next to the model's
choice.  Digits algorithm, complex systems; CUDA events around the product
launches (mdps_system_timing), L2 flushed between evaluations."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdinputs  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402

CELLS = sys.argv[1].split(",") if len(sys.argv) > 1 else (
    ["qd", "od", "deca"] + [f"sweep_d{d}_L{L}" for d in (15, 31, 63, 127) for L in (2, 3, 4, 5, 8, 10)])
# lane sets per job: real systems 1; complex 2 (part lanes) and 1 (the fused-parts kernel, L <= 5)
NPS = (1,) if os.environ.get("TUNE_REAL") == "1" else tuple(int(v) for v in os.environ.get("TUNE_NPS", "2,1,3").split(","))
GEOMS = [(0, 0, 0)] + [(f, p, q) for q in NPS for f in (1, 2, 4, 8) for p in (1, 2, 4, 8)]


def workload(c):
    if c.startswith("sweep"):
        _, d, L = c.split("_")
        return mdinputs.sweep_cell(int(d[1:]), int(L[1:]))
    return mdinputs.make_config(c)


def conv_ms(s, x, v, j, flush, reps):
    s.eval_diff(x, v, j)
    torch.cuda.synchronize()
    s.set_timing(True)
    s.timing(reset=True)
    for _ in range(reps):
        flush.zero_()
        s.eval_diff(x, v, j)
    t = s.timing(reset=True)
    s.set_timing(False)
    return t["conv_ms"] / reps


flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = []
REAL = os.environ.get("TUNE_REAL") == "1"  # the real-system kernel (mdps_options.real)
for c in CELLS:
    si = workload(c)
    if REAL:
        si = mdinputs.realify(si)
    with mdps.System.from_inputs(si, algo=mdps.MDPS_ALGO_DIGITS, real=REAL) as s:
        x = torch.from_numpy(si.x).cuda()
        v = torch.empty((si.n, 2, si.limbs, si.D), dtype=torch.float64, device="cuda")
        j = torch.empty((si.n, si.n, 2, si.limbs, si.D), dtype=torch.float64, device="cuda")
        reps = 3 if si.limbs * si.D <= 64 * 8 else 2
        res = {}
        for f, p, q in GEOMS:
            try:
                mdps.force_geometry(f, p, q)
                res[f"{f},{p},{q}"] = conv_ms(s, x, v, j, flush, reps)
            except Exception:
                pass
        mdps.force_geometry(0, 0, 0)
    best = min((k for k in res if k != "0,0,0"), key=lambda k: res[k])
    row = {"cell": c, "real": REAL, "L": si.limbs, "D": si.D, "default_ms": res.get("0,0,0"), "best": best,
           "best_ms": res[best], "gain": res.get("0,0,0", 0) / res[best], "all": res}
    out.append(row)
    print(json.dumps(row), flush=True)
json.dump(out, open(os.environ.get("TUNE_OUT", "gpurun_out/tune_table.json"), "w"), indent=1)
