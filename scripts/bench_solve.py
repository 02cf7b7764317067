"""Time mdps_solve (block Toeplitz forward substitution) on the configs'
shapes: CUDA events on the launching stream, L2 flushed between runs."""
import json
import sys

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import mdinputs  # noqa: E402
import paper_2012_06607_b200 as mdps  # noqa: E402


def measure(name, steps=5, warmup=2):
    t = mdinputs.toeplitz_config(name)
    s = mdps.Solver(t.n, t.degree, t.limbs)
    J, b = torch.from_numpy(t.jac).cuda(), torch.from_numpy(t.rhs).cuda()
    dx = torch.empty_like(b)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for _ in range(warmup):
        s.solve(J, b, dx)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    ms = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        s.solve(J, b, dx)
        e1.record(st)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    info = s.stats()
    best = min(ms)
    peak = 148 * 64 * 1.965e9
    out = {"config": name, "n": t.n, "degree": t.degree, "limbs": t.limbs, "ms": best, "ms_all": ms,
           "complex_fma": info["complex_fma"], "fp64_ops": info["fp64_ops"],
           "fp64_per_s": info["fp64_ops"] / (best * 1e-3), "frac": info["fp64_ops"] / (best * 1e-3) / peak,
           "grid_blocks": info["grid_blocks"]}
    s.close()
    return out




def trace(name):
    t = mdinputs.toeplitz_config(name)
    s = mdps.Solver(t.n, t.degree, t.limbs)
    J, b = torch.from_numpy(t.jac).cuda(), torch.from_numpy(t.rhs).cuda()
    s.solve(J, b)
    s.solve(J, b)
    tr, steps = s.trace()
    tr = [x for x in tr[:200] if x >= 0][:2 * t.D + 3 * 8 + 2]
    d = [round((tr[i + 1] - tr[i]) / 1e3, 1) for i in range(len(tr) - 1)]
    print(json.dumps({"config": name, "refine_steps": steps, "total_us": tr[-1] / 1e3,
                      "refine_us": d[:3 * steps], "loop_phase_us": d[3 * steps:3 * steps + 40]}), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    do_trace = "--trace" in args
    names = [a for a in args if not a.startswith("--")] or ["dd", "qd", "od", "deca"]
    for nm in names:
        print(json.dumps(measure(nm)), flush=True)
        if do_trace:
            trace(nm)
