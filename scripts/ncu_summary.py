"""Summarise an ncu report (raw page) into the numbers DESIGN/bench use."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__occupancy_limit_registers": "occ_limit_regs",
    "launch__occupancy_limit_shared_mem": "occ_limit_smem",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__inst_executed.sum": "warp_inst",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma_thread_inst",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd_thread_inst",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul_thread_inst",
    "smsp__sass_inst_executed_op_shared_ld.sum": "lds_inst",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefronts_pct",
    "smsp__sass_inst_executed_op_dfma.sum": "dfma_warp_inst",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def summarise(path):
    """path: an .ncu-rep (read with ncu -i) or its raw page already exported as CSV"""
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:60]}
        stalls = {}
        for h, u, v in zip(hdr, units, vals):
            if h in KEYS:
                try:
                    d[KEYS[h]] = float(v.replace(",", ""))
                except ValueError:
                    d[KEYS[h]] = v
                if KEYS[h] in ("dram_read", "dram_write") and u:
                    d[KEYS[h] + "_unit"] = u
                if KEYS[h] == "duration":
                    d["duration_unit"] = u
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(v))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        d["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
        res.append(d)
    return res


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(json.dumps({"report": p, "launches": summarise(p)}, indent=1))
