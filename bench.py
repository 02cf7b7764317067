#!/usr/bin/env python
"""bench.py — mdps_eval_diff throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config od]
                  [--impl mdps|reference] [--algo 0|1|2] [--no-cpu-baseline]

A step is one mdps_eval_diff of the whole workload (every product level and
the addition jobs) with the inputs resident in HBM.  Default workload:
BASELINE.json configs[2] (octo double: n = 64, 128 monomials of 8..16
variables, degree 63) — the configuration the north_star's >= 50% FP64
roofline target is quoted on.  Under torchrun each rank runs an independent
replica on its own GPU (the path needs no exchange: "replicas only",
DESIGN.md); time is the max over ranks.  --impl reference times the CPU
oracle (the reference arm of this tier) on a bounded sample of the same
workload; rank 0 only.

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import mdinputs  # noqa: E402

CONFIG_TEXT = {
    "dd": "BASELINE configs[0]: double double, n=8, 16 monomials x 3 vars, degree 15",
    "qd": "BASELINE configs[1]: quad double, n=32, 64 monomials x 4..8 vars, exponents {1,2}, degree 31",
    "od": "BASELINE configs[2]: octo double, n=64, 128 monomials x 8..16 vars, degree 63",
    "deca": "BASELINE configs[3]: deca double, n=128, 128 monomials x 16 vars, degree 63",
}
METRIC = "series products/s (mdps_eval_diff)"
TOL = {2: 1e-29, 3: 1e-45, 4: 1e-61, 5: 1e-77, 8: 1e-124, 10: 1e-156}

# PAPER.md:109-147 (Table 1): hardware double operations per md add and per
# md mul (the +, -, * columns summed; no division on this path)
TABLE1_ADD = {2: 8 + 12, 3: 13 + 22, 4: 35 + 54, 5: 44 + 78, 8: 95 + 174, 10: 139 + 258}
TABLE1_MUL = {2: 5 + 9 + 9, 3: 83 + 84 + 42, 4: 99 + 164 + 73, 5: 162 + 283 + 109, 8: 529 + 954 + 259,
              10: 952 + 1743 + 394}


def table1_ops_per_product(D: int, L: int) -> int:
    """The paper's cost of one truncated complex series product in hardware
    double operations: D(D+1)/2 complex md multiplications (4 md mul + 2 md
    add each, DESIGN R5) and D(D-1)/2 complex md additions (2 md add each),
    PAPER.md:233-239, priced with Table 1.  A reported
    context figure ("paper-equivalent" FP64 ops), not the kernel's own
    instruction count: the digit kernel does far fewer."""
    cmul = D * (D + 1) // 2
    cadd = D * (D - 1) // 2
    return cmul * (4 * TABLE1_MUL[L] + 2 * TABLE1_ADD[L]) + cadd * 2 * TABLE1_ADD[L]


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def workload(name: str):
    if name.startswith("sweep_"):
        _, d, L = name.split("_")
        return mdinputs.sweep_cell(int(d[1:]), int(L[1:]))
    return mdinputs.make_config(name)


def bench_config(si, name: str, world: int = 1, sharded: bool = False) -> dict:
    """The `config` object of the JSON line: identical for both arms (host-only
    facts about the workload; the GPU schedule's own figures go under
    `schedule`)."""
    from paper_2012_06607_b200 import shard
    return {"workload": CONFIG_TEXT.get(name, name), "name": name,
            "n": si.n, "monomials": si.M, "degree": si.degree, "limbs": si.limbs,
            "products_per_step": int(sum(shard.row_products(si.poly_ptr, si.mono_ptr, si.exps))),
            "parallelism": (f"rows sharded over {world} GPUs" if sharded else f"replicas x{world}")
            if world > 1 else "single GPU",
            "l2": "256 MiB buffer written between timed steps (L2 flushed)",
            "seed": mdinputs.CONFIGS[si.name].seed if si.name in mdinputs.CONFIGS else None,
            "input_sha256": si.sha256()[:16]}


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.dev)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        rows = []
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                rows.append(dict(sm=float(f[1]), smmax=float(f[2]), power=float(f[3]) if f[3] not in ("[N/A]", "") else 0.0,
                                 hw=f[5], hwth=f[6], swth=f[7], swpc=f[8]))
            except ValueError:
                continue
        if not rows:
            return None
        reasons = set()
        for r in rows:
            for key, name in (("hw", "hw_slowdown"), ("hwth", "hw_thermal_slowdown"),
                              ("swth", "sw_thermal_slowdown"), ("swpc", "sw_power_cap")):
                if r[key].lower().startswith("active"):
                    reasons.add(name)
        loaded = [r["sm"] for r in rows if r["power"] > 200.0] or [r["sm"] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r["smmax"] for r in rows),
                "reasons": sorted(reasons), "samples": len(rows),
                "power_w_max": max(r["power"] for r in rows)}


# ---------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def naive_products(si, entry) -> int:
    """series products the oracle computes for one output (naive, per
    monomial): the value multiplies c by every factor (sum of exponents), a
    Jacobian entry (i, j) one factor fewer for every monomial containing x_j."""
    i, j = entry
    tot = 0
    for r in range(si.poly_ptr[i], si.poly_ptr[i + 1]):
        vs = si.vars[si.mono_ptr[r]:si.mono_ptr[r + 1]]
        deg = int(si.exps[si.mono_ptr[r]:si.mono_ptr[r + 1]].sum())
        if j < 0:
            tot += deg
        elif j in vs:
            tot += deg - 1
    return tot


def row_entries_of(si, i):
    """the outputs of row i: its value and every structurally nonzero Jacobian entry."""
    cols = sorted({int(v) for r in range(si.poly_ptr[i], si.poly_ptr[i + 1])
                   for v in si.vars[si.mono_ptr[r]:si.mono_ptr[r + 1]]})
    return [(i, -1)] + [(i, j) for j in cols]


def row_entries(si, rows):
    """every output of rows 0..rows-1, largest first (the workers take them in
    this order)."""
    out = []
    for i in range(rows):
        out += row_entries_of(si, i)
    return sorted(out, key=lambda e: -naive_products(si, e))


def cpu_baseline(si, target_s: float = 15.0):
    """The oracle as it stands on a bounded, load-balanced sample of the same
    workload: ALL outputs (values and every nonzero Jacobian entry) of the
    first rows, as many rows as fit ~target_s seconds on every host core at
    the single-core rate measured first; workers claim outputs from a counter
    (the paper's job queue), largest first."""
    import oracle
    ncpu = os.cpu_count() or 1
    # single-core rate on one Jacobian entry of row 0
    probe = row_entries(si, 1)[-1]
    t0 = time.perf_counter()
    _, p1 = oracle.eval_entries(si, [probe], nthreads=1)
    rate1 = p1 / max(1e-9, time.perf_counter() - t0)
    n_rows = len(si.poly_ptr) - 1
    budget = target_s * rate1 * ncpu

    def row_cost(i):
        return sum(naive_products(si, e) for e in row_entries_of(si, i))

    rows, used = 1, row_cost(0)
    while rows < n_rows:
        c = row_cost(rows)
        if used + c > budget:
            break
        rows, used = rows + 1, used + c
    entries = row_entries(si, rows)
    cores = min(ncpu, len(entries))
    t0 = time.perf_counter()
    _, prods = oracle.eval_entries(si, entries, nthreads=cores)
    dt = time.perf_counter() - t0
    return {"value": prods / dt, "unit": "products/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(), "host_cpus": ncpu,
            "single_core_products_per_s": rate1,
            "sample": f"all {len(entries)} outputs of rows 0..{rows - 1} of {si.name} (values and every nonzero "
                      f"Jacobian entry), {prods} naive series products in {dt:.1f} s on {cores} threads",
            "seconds": dt}


def run_reference(args):
    """--impl reference: the CPU oracle, bounded sample per step (rank 0)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    si = workload(args.config)
    entries = mdinputs.first_entries(si, 1 + args.steps + args.warmup)[1:]  # one Jacobian entry per step
    cores = 1
    for e in entries[:args.warmup]:
        oracle.eval_entries(si, [e], nthreads=1)
    t0 = time.perf_counter()
    prods = 0
    for e in entries[args.warmup:args.warmup + args.steps]:
        _, p = oracle.eval_entries(si, [e], nthreads=1)
        prods += p
    dt = time.perf_counter() - t0
    value = prods / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "products/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / max(1, args.steps), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64 (exact superaccumulator)", "data": "synthetic",
            "config": bench_config(si, args.config, args.gpus),
            "cpu_baseline": {"value": value, "unit": "products/s", "cores": cores, "kind": "oracle",
                             "sample": f"one Jacobian entry of {si.name} per step (naive products)"},
            "e2e": {"value": value, "unit": "products/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
def max_over_ranks(value: float, dist=None, device="cpu") -> float:
    """The max of a per-rank time over all ranks (identity without a process group)."""
    if not dist:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_per_step: float, world: int, steps: int, ms: float) -> float:
    """Units per second of the whole job: every rank processes units_per_step
    per step (replicas, weak scaling); ms = the max over ranks."""
    return units_per_step * world * steps / (ms * 1e-3)


def bench_next(mdps, torch, sys_, si, x, vals, jac, flush, stream, peak_nominal, dist, args):
    """mdps_solve on the eval's own (J, -f) and mdps_newton_step from x."""
    steps = max(3, min(args.steps, 5))

    def timed(fn, prep=None):
        for _ in range(2):
            if prep:
                prep()
            fn()
        torch.cuda.synchronize()
        ms = []
        for _ in range(steps):
            if prep:
                prep()
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return max_over_ranks(sum(ms) / len(ms), dist, "cuda")

    with mdps.Solver(si.n, si.degree, si.limbs) as sol:
        sys_.eval_diff(x, vals, jac)
        rhs = -vals
        dx = torch.empty_like(vals)
        t_solve = timed(lambda: sol.solve(jac, rhs, dx))
        info = sol.stats()
        xw = torch.empty_like(x)
        t_newton = timed(lambda: sol.newton_step(sys_, xw), prep=lambda: xw.copy_(x))
        _, refine = sol.trace()
    achieved = info["fp64_ops"] / (t_solve * 1e-3)
    # the real path (mdps_options.real) on the same system with its imaginary
    # parts dropped: one product per term
    real = None
    try:
        sr = mdinputs.realify(si)
        with mdps.System.from_inputs(sr, real=True) as sysr:
            xr = torch.from_numpy(sr.x).cuda()
            vr, jr = torch.empty_like(vals), torch.empty_like(jac)
            t_real = timed(lambda: sysr.eval_diff(xr, vr, jr))
            str_ = sysr.stats()
        real = {"ms": t_real, "value": str_["products"] / (t_real * 1e-3), "unit": "products/s",
                "fp64_instr_per_s": str_["fp64_ops_total"] / (t_real * 1e-3),
                "input": "the same system with every imaginary limb 0 (mdps_options.real)"}
    except Exception as e:  # noqa: BLE001 - reported, not fatal
        real = {"error": str(e)}
    # the oracle's forward substitution on a bounded sample of the same solve:
    # the first coefficients (dx_0..dx_dc depend only on A_0..A_dc, b_0..b_dc)
    cpu = None
    if not args.no_cpu_baseline and (not dist or dist.get_rank() == 0):
        import oracle
        J, b = jac.cpu().numpy(), rhs.cpu().numpy()
        dc = {2: 15, 3: 12, 4: 10, 5: 8, 8: 5, 10: 3}[si.limbs]
        dc = min(dc, si.degree)
        cores = os.cpu_count() or 1
        t0 = time.perf_counter()
        oracle.toeplitz_solve(np.ascontiguousarray(J[..., :dc + 1]), np.ascontiguousarray(b[..., :dc + 1]),
                              nthreads=cores)
        dt = time.perf_counter() - t0
        n, D = si.n, dc + 1
        cfma = D * n * n + n * n * D * (D - 1) // 2 + n ** 3
        cpu = {"value": cfma / dt, "unit": "complex md multiply-adds/s", "cores": min(cores, n), "kind": "oracle",
               "sample": f"the same solve truncated at degree {dc} (n={n}), {dt:.1f} s"}
    return {
        "toeplitz_solve": {
            "ms": t_solve, "complex_md_fma": info["complex_fma"], "fp64_instr": info["fp64_ops"],
            "refine_steps": refine,
            "roofline": {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_nominal / 1e12,
                         "unit": "T FP64 instr/s", "frac": achieved / peak_nominal},
            "input": "the eval's own Jacobian and -f (one Newton step's linear system)",
            "value": info["complex_fma"] / (t_solve * 1e-3), "unit": "complex md multiply-adds/s",
            "cpu_baseline": cpu},
        "newton_step": {"ms": t_newton, "of_which_eval_ms": None,
                        "api": "mdps_newton_step (eval/diff + solve + update)"},
        "real_eval": real,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="od")
    ap.add_argument("--impl", default="mdps", choices=["mdps", "reference"])
    ap.add_argument("--algo", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--workspace-mb", type=int, default=0,
                    help="bound on the system's pool memory (mdps_options.workspace_mb; 0 = default)")
    ap.add_argument("--no-next", action="store_true", help="skip the solver / Newton-step measurements")
    ap.add_argument("--shard", default="replicas", choices=["replicas", "rows"],
                    help="N > 1: independent replicas (weak scaling, default) or one system's rows sharded (strong)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "mdps" else args.warmup

    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2012_06607_b200 as mdps
    from paper_2012_06607_b200 import build as mdps_build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if rank == 0:
        mdps_build.build()
    if dist:
        dist.barrier()
    mdps.lib()

    si = si_full = workload(args.config)
    sharded = args.shard == "rows" and world > 1
    if sharded:  # strong scaling: this rank evaluates its share of the rows
        import dataclasses
        from paper_2012_06607_b200 import shard
        costs = shard.row_products(si.poly_ptr, si.mono_ptr, si.exps)
        rows = shard.partition_rows(costs, world)[rank]
        pp, mp_, vv, ee, cc = shard.subsystem(si.poly_ptr, si.mono_ptr, si.vars, si.exps, si.coeffs, rows)
        si = dataclasses.replace(si, poly_ptr=pp, mono_ptr=mp_, vars=vv, exps=ee, coeffs=cc)
        full_products = sum(costs)
    n_rows = len(si.poly_ptr) - 1
    peaks = load_peaks()
    sys_ = mdps.System.from_inputs(si, algo=args.algo, workspace_mb=args.workspace_mb)
    st = sys_.stats()
    stream = torch.cuda.current_stream()
    x = torch.from_numpy(si.x).cuda()
    vals = torch.empty((n_rows, 2, si.limbs, si.D), dtype=torch.float64, device="cuda")
    jac = torch.empty((n_rows, si.n, 2, si.limbs, si.D), dtype=torch.float64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    fp64_peak_measured = mdps.fp64_peak(20000)

    for _ in range(args.warmup):
        sys_.eval_diff(x, vals, jac)
    torch.cuda.synchronize()

    sampler = ClockSampler(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ
                           else local_rank)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for s in range(args.steps):
        flush.zero_()                      # outside the timed events: L2 holds no inputs
        ev[s][0].record(stream)
        sys_.eval_diff(x, vals, jac)
        ev[s][1].record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = max_over_ranks(sum(step_ms), dist, "cuda")

    # a separate instrumented pass (the library records CUDA events around
    # every launch group on the caller's stream) for the per-kernel split and
    # the roofline of the dominant kernel; `value` above is timed without it
    sys_.set_timing(True)
    sys_.timing(reset=True)
    for s in range(args.steps):
        flush.zero_()
        sys_.eval_diff(x, vals, jac)
    torch.cuda.synchronize()
    sys_.set_timing(False)
    tim = sys_.timing(reset=True)
    products_per_step = st["products"]
    value = whole_job_rate(products_per_step, world, args.steps, ms)
    if sharded:  # the whole system's products once per step, over the slowest rank's time
        value = whole_job_rate(full_products, 1, args.steps, ms)
    fp64_per_s = whole_job_rate(st["fp64_ops_total"], world, args.steps, ms)

    # dominant kernel: the product jobs (all levels), live CUDA-event durations
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    peak_nominal = n_sm * 64 * sm_max * 1e6  # FP64 instr/s: 64 FP64 lanes per SM
    conv_launch_ms = tim["conv_ms"] / max(1, tim["conv_launches"])
    conv_ops_per_launch = st["fp64_ops_conv"] * args.steps / max(1, tim["conv_launches"])
    achieved = st["fp64_ops_conv"] * args.steps / (tim["conv_ms"] * 1e-3) if tim["conv_ms"] > 0 else 0.0
    roofline = {"bound": "alu", "achieved": achieved / 1e12, "peak": peak_nominal / 1e12,
                "unit": "T FP64 instr/s (DADD/DMUL/DFMA = 1)", "frac": achieved / peak_nominal,
                "traffic": None,
                "peak_measured_in_run": fp64_peak_measured / 1e12,
                "frac_of_measured": achieved / fp64_peak_measured if fp64_peak_measured > 0 else None,
                "kernel": "conv_dig_kernel" if st["algo"] == 2 else "conv_eft_kernel",
                "ops_per_launch": conv_ops_per_launch, "avg_launch_ms": conv_launch_ms,
                "share_of_step": tim["conv_ms"] / max(1e-9, tim["conv_ms"] + tim["accum_ms"] + tim["convert_ms"]),
                "timing": "separate instrumented pass of the same steps (CUDA events around each launch group)",
                "peak_source": f"{n_sm} SMs x 64 FP64 lanes x {sm_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
                # the same rate with an FMA counted as 2 FLOPs (every algorithmic
                # instruction of the digit kernel is a DFMA), against 2 x peak
                "fma_as_2_tflops": 2 * achieved / 1e12 if st["algo"] == 2 else None,
                "fma_as_2_peak_tflops": 2 * peak_nominal / 1e12,
                # compulsory bytes (x, coefficients, outputs once) per step over the step time
                "compulsory_gbs": st["compulsory_bytes"] / (ms / args.steps * 1e-3) / 1e9}
    # executed FP64 instructions per product (ncu hardware counters, one
    # launch, profiles/r02_fp64_counts.json) next to the algorithmic count W
    cprof = os.path.join(ROOT, "profiles", "r02_fp64_counts.json")
    if os.path.exists(cprof) and st["algo"] == 2:
        try:
            for c in json.load(open(cprof))["launches"]:
                if c["config"] == args.config:
                    roofline["executed_fp64_per_product_ncu"] = (c["dfma_executed"] + c["dadd_executed"] +
                                                                 c["dmul_executed"]) / c["jobs"]
                    roofline["algorithmic_fp64_per_product"] = c["W_algorithmic_dfma"] / c["jobs"]
        except Exception:
            pass
    tprof = os.path.join(ROOT, "profiles", f"traffic_{args.config}_algo{st['algo']}.json")
    if os.path.exists(tprof):
        try:
            tp = json.load(open(tprof))
            roofline["traffic"] = tp["dram_bytes_per_launch"]
            # DRAM bytes of one whole evaluation (every launch of the step, ncu)
            # next to its compulsory bytes (inputs, coefficients, outputs once)
            if "dram_bytes_per_step" in tp:
                roofline["traffic_per_step"] = tp["dram_bytes_per_step"]
                roofline["compulsory_bytes_per_step"] = st["compulsory_bytes"]
        except Exception:
            pass

    # end to end through the public C API with HOST buffers (pinned)
    e2e = None
    if not args.no_e2e:
        hx = torch.from_numpy(si.x).pin_memory()
        hv = torch.empty(tuple(vals.shape), dtype=torch.float64).pin_memory()
        hj = torch.empty(tuple(jac.shape), dtype=torch.float64).pin_memory()
        h = sys_.handle
        lib = mdps.lib()
        sh = stream.cuda_stream
        lib.mdps_eval_diff_host(h, hx.data_ptr(), hv.data_ptr(), hj.data_ptr(), sh)  # warm (allocates)
        e2e_steps = max(3, args.steps // 2)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            rc = lib.mdps_eval_diff_host(h, hx.data_ptr(), hv.data_ptr(), hj.data_ptr(), sh)
            if rc != 0:
                raise RuntimeError(mdps.mdps_last_error())
        e1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1), dist, "cuda")
        e2e = {"value": whole_job_rate(full_products, 1, e2e_steps, ems) if sharded else
               whole_job_rate(products_per_step, world, e2e_steps, ems), "unit": "products/s",
               "h2d_bytes_per_step": int(hx.numel() * 8), "d2h_bytes_per_step": int((hv.numel() + hj.numel()) * 8),
               "steps": e2e_steps, "ms_per_step": ems / e2e_steps, "api": "mdps_eval_diff_host (pinned host buffers)"}
        # the host-buffer outputs must equal the device path's outputs
        if not (torch.equal(hv, vals.cpu()) and torch.equal(hj, jac.cpu())):
            raise RuntimeError("e2e outputs differ from the device-path outputs")

    # the next rows of the hot path: the block Toeplitz solve of
    # this system's own Jacobian and f (J dx = -f), and whole Newton steps
    # (eval/diff + solve + update), device-timed like the eval
    nxt = None
    if not args.no_next and not sharded:
        nxt = bench_next(mdps, torch, sys_, si, x, vals, jac, flush, stream, peak_nominal, dist, args)
        nxt["newton_step"]["of_which_eval_ms"] = ms / args.steps

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(si)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "products/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "ms_median": statistics.median(step_ms), "ms_min": min(step_ms), "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(si_full, args.config, world, sharded),
            "schedule": {"algo": {1: "eft", 2: "digits"}[st["algo"]], "digits": st["digits"],
                         "products_per_step": products_per_step, "levels": st["levels"],
                         "order": {1: "levels", 2: "queue"}[st["schedule"]], "chunks": st["chunks"],
                         "workspace_bytes": st["workspace_bytes"], "pool_bytes": st["pool_bytes"]},
            "fp64_ops_per_s": fp64_per_s,
            "fp64_ops_per_step": st["fp64_ops_total"],
            "paper_equivalent": {
                "table1_fp64_ops_per_product": table1_ops_per_product(si.D, si.limbs),
                "table1_fp64_ops_per_s": value * table1_ops_per_product(si.D, si.limbs),
                "kernel_fp64_instr_per_product": st["fp64_ops_conv"] / max(1, products_per_step),
                "source": "PAPER.md:109-147 Table 1 (md add/mul in hardware double ops) x the product's "
                          "D(D+1)/2 complex md mul + D(D-1)/2 complex md add (PAPER.md:233-239); context only"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": st["launches"] * args.steps,
            "kernel_ms_per_step": {"conv": tim["conv_ms"] / args.steps, "accum": tim["accum_ms"] / args.steps,
                                   "convert": tim["convert_ms"] / args.steps},
            "clocks": clocks,
            "next_rows": nxt,
        }
        print(json.dumps(line), flush=True)
    sys_.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
