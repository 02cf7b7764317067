"""profiles/r02_fp64_counts.json from the ncu counter runs of scripts/gpu_round3.sh:
executed FP64 instructions and DRAM bytes of one product launch per config
(gpurun_out/fp64_counts_{od,qd}.csv; the level's job count from the profiling
driver's own printout in gpurun_out/ncu_full_{cfg}.log) against the
algorithmic digit count W = jobs x D(D+1) S(S+1)."""
import ast
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
CFG = {"od": dict(D=64, L=8, S=21, level=8), "qd": dict(D=32, L=4, S=12, level=0)}
out = {"what": "executed FP64 instructions and DRAM bytes of one product launch (ncu --metrics "
               "smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum, dram__bytes_{read,write}.sum, "
               "--clock-control none; scripts/gpu_round3.sh) against the algorithmic digit count "
               "W = jobs x D(D+1) S(S+1) (DESIGN.md §7.1)", "launches": []}
for cfg, c in CFG.items():
    log = open(os.path.join(SRC, f"ncu_full_{cfg}.log")).read()
    levels = ast.literal_eval(re.search(r"levels: (\[[^\]]*\])", log).group(1))
    jobs = int(levels[c["level"]])
    m, kern = {}, ""
    for r in csv.reader(open(os.path.join(SRC, f"fp64_counts_{cfg}.csv"))):
        if len(r) > 14 and r[0].isdigit():
            scale = {"us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "Kbyte": 1e3, "Mbyte": 1e6,
                     "Gbyte": 1e9}.get(r[13], 1.0)  # -> ns, bytes
            m[r[12]] = float(r[14].replace(",", "")) * scale
            kern = r[4].split("(")[0].replace("void ", "")
    W = jobs * c["D"] * (c["D"] + 1) * c["S"] * (c["S"] + 1)
    dfma = m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
    dadd = m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
    dmul = m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
    out["launches"].append({
        "config": cfg, "kernel": kern, "level": c["level"], "jobs": jobs, "D": c["D"], "S": c["S"],
        "W_algorithmic_dfma": W, "dfma_executed": dfma, "dadd_executed": dadd, "dmul_executed": dmul,
        "dfma_over_W": dfma / W, "algorithmic_share_of_fp64": W / (dfma + dadd + dmul),
        "duration_ns": m["gpu__time_duration.sum"], "warp_inst": m["smsp__inst_executed.sum"],
        "dram_read_bytes": m["dram__bytes_read.sum"], "dram_write_bytes": m["dram__bytes_write.sum"],
        "operand_bytes_staged": jobs * 2 * 2 * c["S"] * c["D"] * 8})
json.dump(out, open(os.path.join(ROOT, "profiles", "r02_fp64_counts.json"), "w"), indent=1)
print(json.dumps(out["launches"], indent=1))
