"""Shared helpers for the GPU parity tests (tests only)."""
import os

import numpy as np

import mdinputs
import oracle

# BASELINE.json north_star: max|gpu - oracle| / max(|oracle|, 1) per output
# series (SURVEY §8(c) C2.9 reading), and C2.10's readings for L = 3, 5.
TOL = {2: 1e-29, 3: 1e-45, 4: 1e-61, 5: 1e-77, 8: 1e-124, 10: 1e-156}

NTHREADS = max(1, (os.cpu_count() or 1))


def structural_support(si):
    """boolean [n_polys][n]: does some monomial of f_i contain x_j?"""
    n_polys = len(si.poly_ptr) - 1
    sup = np.zeros((n_polys, si.n), dtype=bool)
    for i in range(n_polys):
        for r in range(si.poly_ptr[i], si.poly_ptr[i + 1]):
            sup[i, si.vars[si.mono_ptr[r]:si.mono_ptr[r + 1]]] = True
    return sup


def gpu_eval(si, algo=0, use_graph=False):
    import torch
    import paper_2012_06607_b200 as mdps
    with mdps.System.from_inputs(si, algo=algo, use_graph=use_graph) as sys_:
        x = torch.from_numpy(si.x).cuda()
        vals, jac = sys_.eval_diff(x)
        torch.cuda.synchronize()
        return vals.cpu().numpy(), jac.cpu().numpy(), sys_.stats()


def sample_entries(si, nvals, njac, seed=0, sup=None):
    """a few value rows and nonzero Jacobian entries, seeded."""
    rng = np.random.default_rng(seed)
    sup = structural_support(si) if sup is None else sup
    rows = rng.choice(si.n, size=min(nvals, si.n), replace=False)
    ent = [(int(i), -1) for i in rows]
    nz = np.argwhere(sup)
    pick = rng.choice(len(nz), size=min(njac, len(nz)), replace=False)
    ent += [(int(nz[p][0]), int(nz[p][1])) for p in pick]
    return ent


def check_against_oracle(si, vals, jac, entries, tol):
    """oracle computes `entries`; returns the max per-series error."""
    want, _ = oracle.eval_entries(si, entries, nthreads=NTHREADS)
    got = np.stack([vals[i] if j < 0 else jac[i, j] for i, j in entries])
    err = oracle.series_err(got, want)
    return float(err.max()), err


def euler_bound(x, jac, g, tol, g_tol=None):
    """Largest Euler residual |sum_j (x_j * J_ij)_k - g_ik| that outputs
    within the per-series tolerance can produce (R19): every
    Jacobian entry off by at most tol * max(max_k |J_ij,k|, 1) per
    coefficient, g by at most g_tol * max(max_k |g_ik|, 1):
        bound_ik = tol * sum_j max(|J_ij|_inf, 1) * sum_{q<=k} |x_j,q|
                   + g_tol * max(|g_i|_inf, 1),
    in float64 from the leading limbs (x 1.01 for their rounding)."""
    g_tol = tol if g_tol is None else g_tol
    ax = np.hypot(x[:, 0, 0, :], x[:, 1, 0, :])                      # [n][D]
    cx = np.cumsum(ax, axis=1)                                        # sum_{q<=k} |x_j,q|
    mj = np.maximum(np.hypot(jac[:, :, 0, 0, :], jac[:, :, 1, 0, :]).max(axis=2), 1.0)  # [rows][n]
    mg = np.maximum(np.hypot(g[:, 0, 0, :], g[:, 1, 0, :]).max(axis=1), 1.0)            # [rows]
    return 1.01 * (tol * (mj @ cx) + g_tol * mg[:, None])


def euler_check(si, vals, jac, tol, g=None, g_tol=None, nthreads=None):
    """Euler's identity on ALL rows of the GPU output: the exact residual
    (oracle.euler_residual) of every row and coefficient within euler_bound.
    g: the degree-weighted values (oracle.values_weighted), or None for a
    system homogeneous of degree m (every monomial m variables, exponent 1):
    then g = m * f from the GPU's own values (exact: m is a power of two here).
    Returns max(residual / bound)."""
    if g is None:
        degs = np.diff(si.mono_ptr)
        assert (degs == degs[0]).all() and (si.exps == 1).all() and degs[0] & (degs[0] - 1) == 0
        g = float(degs[0]) * vals
        g_tol = float(degs[0]) * tol
    res = oracle.euler_residual(si.x, jac, g, nthreads=nthreads or NTHREADS)
    bound = euler_bound(si.x, jac, g, tol, g_tol)
    ratio = res / bound
    assert (ratio <= 1.0).all(), (float(ratio.max()), np.unravel_index(int(ratio.argmax()), ratio.shape))
    return float(ratio.max())
