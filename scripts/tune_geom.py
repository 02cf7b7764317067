"""Time the product kernel under forced geometries (MDPS_CONV_F / MDPS_CONV_P)."""
import json
import os
import subprocess
import sys

CASES = sys.argv[1].split(",") if len(sys.argv) > 1 else ["od", "qd", "sweep_d15_L2", "sweep_d127_L8"]
GEOMS = [(f, p) for f in (1, 2, 4, 8) for p in (1, 2, 4, 8, 16)]
CODE = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import scripts.sweep as sw, mdinputs
c = sys.argv[1]
si = mdinputs.sweep_cell(*map(int, [c.split("_")[1][1:], c.split("_")[2][1:]])) if c.startswith("sweep") else mdinputs.make_config(c)
r = sw.measure(si, steps=3, warmup=2)
print(json.dumps(r))
'''
for case in CASES:
    res = []
    for f, p in [(None, None)] + GEOMS:
        env = dict(os.environ)
        if f:
            env["MDPS_CONV_F"], env["MDPS_CONV_P"] = str(f), str(p)
        out = subprocess.run([sys.executable, "-c", CODE, case], env=env, capture_output=True, text=True, timeout=600)
        try:
            r = json.loads(out.stdout.strip().splitlines()[-1])
            res.append((f, p, r["conv_ms"], r["conv_frac_of_fp64_peak"]))
            print(case, f, p, round(r["conv_ms"], 3), round(r["conv_frac_of_fp64_peak"], 3), flush=True)
        except Exception:
            print(case, f, p, "failed", out.stderr.strip().splitlines()[-1:] if out.stderr else "", flush=True)
