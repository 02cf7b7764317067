"""BASELINE config 4: the precision sweep (d x L) on one B200 — products/s,
FP64 instr/s and the product kernel's roofline fraction per cell, plus the
other configs.  Writes one JSON table (measurement only; not the bench line)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mdinputs  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402


def digits_for(L):
    """digits per part of the digit algorithm (kernels_dig.cuh digits_for)"""
    S = 2
    while (S - 2) * 23 < 53 * L + 8:
        S += 1
    return S


def measure(si, algo=0, steps=5, warmup=3):
    s = mdps.System.from_inputs(si, algo=algo)
    st = s.stats()
    x = torch.from_numpy(si.x).cuda()
    v = torch.empty((si.n, 2, si.limbs, si.D), dtype=torch.float64, device="cuda")
    j = torch.empty((si.n, si.n, 2, si.limbs, si.D), dtype=torch.float64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(warmup):
        s.eval_diff(x, v, j)
    torch.cuda.synchronize()
    s.set_timing(True)
    s.timing(reset=True)
    ms = 0.0
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s.eval_diff(x, v, j)
        b.record()
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    tim = s.timing(reset=True)
    s.close()
    peak = 148 * 64 * 1965e6
    ach = st["fp64_ops_conv"] * steps / (tim["conv_ms"] * 1e-3)
    return {"cell": si.name, "n": si.n, "degree": si.degree, "limbs": si.limbs, "algo": st["algo"],
            "digits": st["digits"], "products": st["products"], "ms_per_step": ms / steps,
            "products_per_s": st["products"] * steps / (ms * 1e-3),
            "fp64_instr_per_s": st["fp64_ops_total"] * steps / (ms * 1e-3),
            "conv_ms": tim["conv_ms"] / steps, "accum_ms": tim["accum_ms"] / steps,
            "conv_frac_of_fp64_peak": ach / peak, "launches": st["launches"],
            # one work count for every cell, whatever algorithm ran: the digit
            # method's D(D+1) S(S+1) DFMAs per complex product
            "frac_on_digit_count": st["products"] * si.D * (si.D + 1) * digits_for(si.limbs) *
            (digits_for(si.limbs) + 1) * steps / (tim["conv_ms"] * 1e-3) / peak}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    ap.add_argument("--eft", action="store_true", help="also time MDPS_ALGO_EFT")
    ap.add_argument("--l2-both", action="store_true", help="the L = 2 cells also under the algorithm AUTO does not pick")
    a = ap.parse_args()
    res = []
    for name in ("dd", "qd", "od", "deca"):
        res.append(measure(mdinputs.make_config(name)))
        if a.eft:
            res.append(measure(mdinputs.make_config(name), algo=1))
        print(json.dumps(res[-1]), flush=True)
    for d in mdinputs.SWEEP_DEGREES:
        for L in mdinputs.SWEEP_LIMBS:
            res.append(measure(mdinputs.sweep_cell(d, L)))
            print(json.dumps(res[-1]), flush=True)
            if a.l2_both and L == 2:
                other = mdps.MDPS_ALGO_DIGITS if res[-1]["algo"] == mdps.MDPS_ALGO_EFT else mdps.MDPS_ALGO_EFT
                r = measure(mdinputs.sweep_cell(d, L), algo=other)
                r["cell"] += "_other_algo"
                res.append(r)
                print(json.dumps(r), flush=True)
    json.dump(res, open(a.out, "w"), indent=1)
