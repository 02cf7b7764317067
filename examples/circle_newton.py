"""The paper's circle demo (arXiv 2012.06607, §3) through the public API.

    t - t^3/6 + t^5/120 - t^7/5040 - y = 0,   x^2 + y^2 - 1 = 0,

Newton's method on power series truncated at degree 8, started at x = 1,
y = 0: x(t) becomes the Taylor series of cos(t).  Run on a CUDA machine:

    python examples/circle_newton.py [limbs]
"""
import os
import sys
from fractions import Fraction

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2012_06607_b200 as mdps  # noqa: E402


def series(coefs, L, D):
    """a real md series [2][L][D] from exact rationals (greedy limbs)."""
    out = np.zeros((2, L, D))
    for k, c in enumerate(coefs):
        X = Fraction(c)
        for l in range(L):
            v = float(X)
            out[0, l, k] = v
            X -= Fraction(v)
    return out


def main(L=4, degree=8):
    D = degree + 1
    s = [0, 1, 0, Fraction(-1, 6), 0, Fraction(1, 120), 0, Fraction(-1, 5040)]
    # f0 = s(t) * 1 - 1 * y ;  f1 = x^2 + y^2 - 1     (variables x = 0, y = 1)
    poly_ptr = [0, 2, 5]
    mono_ptr = [0, 0, 1, 2, 3, 3]
    vars_, exps = [1, 0, 1], [1, 2, 2]
    coeffs = np.stack([series(s, L, D), series([-1], L, D), series([1], L, D), series([1], L, D),
                       series([-1], L, D)])
    x = torch.from_numpy(np.stack([series([1], L, D), series([0], L, D)])).cuda()
    with mdps.System(poly_ptr, mono_ptr, vars_, exps, coeffs, 2, degree, L) as system, \
            mdps.Solver(2, degree, L) as solver:
        steps, norm = solver.newton(system, x, max_iters=8, tol=1e-32)
    xs = x.cpu().numpy()
    print(f"{steps} Newton steps, last update norm {norm:.3e}, {L} limbs")
    print("x(t) =", " + ".join(f"({xs[0, 0, 0, k]:.15e}) t^{k}" for k in range(D) if xs[0, 0, 0, k] != 0))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
