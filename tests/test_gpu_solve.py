"""CUDA parity of the block lower-triangular Toeplitz solver (libmdps.h
mdps_solve) against the CPU oracle's forward substitution.

Inputs: mdinputs.random_toeplitz / toeplitz_config (seeded unit-circle series
matrices, DESIGN.md input recipe).  Metric: the per-series error of
oracle.series_err (exact differences), tolerance TOL[L] of the north star
(reading R12).  The exactly solvable permutation case is compared
bit for bit, the pivot sequence against the oracle's.
"""
import numpy as np
import pytest

import mdinputs
import oracle
from tests.gpu_util import NTHREADS, TOL

pytestmark = pytest.mark.gpu
LEVELS = (2, 3, 4, 5, 8, 10)


@pytest.fixture(scope="module")
def mdps():
    import torch
    import paper_2012_06607_b200 as m
    assert torch.cuda.is_available()
    m.lib()
    return m


def cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_solve(mdps, t, jac=None):
    import torch
    jac = t.jac if jac is None else jac
    with mdps.Solver(t.n, t.degree, t.limbs) as s:
        dx = s.solve(cuda(jac), cuda(t.rhs))
        torch.cuda.synchronize()
        piv, sing = s.status()
        return dx.cpu().numpy(), piv, sing


@pytest.mark.parametrize("L", LEVELS)
@pytest.mark.parametrize("n,degree", [(1, 0), (1, 6), (2, 3), (3, 0), (5, 4), (7, 9)])
def test_small_random(mdps, n, degree, L):
    t = mdinputs.random_toeplitz(200 + 10 * n + degree, n, degree, L)
    dx, piv, sing = gpu_solve(mdps, t)
    want, wpiv = oracle.toeplitz_solve(t.jac, t.rhs, nthreads=NTHREADS)
    assert not sing
    assert np.array_equal(piv, wpiv)
    err = oracle.series_err(dx, want)
    assert err.max() <= TOL[L], err.max()


@pytest.mark.parametrize("L", (2, 5, 10))
def test_permutation_case_bitexact(mdps, L):
    """A_0 = P diag(+-2^e, +-i 2^e), A_i = 0: every operation is exact."""
    n, D = 5, 4
    rng = np.random.default_rng(3)
    sigma = [2, 0, 4, 1, 3]
    s = [(2.0 ** e, 0.0) if k % 2 == 0 else (0.0, -(2.0 ** e)) for k, e in enumerate([1, -3, 0, 5, -2])]
    jac = np.zeros((n, n, 2, L, D))
    for k in range(n):
        jac[sigma[k], k, 0, 0, 0], jac[sigma[k], k, 1, 0, 0] = s[k]
    rhs = np.zeros((n, 2, L, D))
    rhs[:, :, 0, :] = rng.integers(-50, 50, size=(n, 2, D)).astype(np.float64)
    t = mdinputs.ToeplitzInputs("perm", n, D - 1, L, jac, rhs)
    dx, piv, sing = gpu_solve(mdps, t)
    want, wpiv = oracle.toeplitz_solve(jac, rhs)
    assert np.array_equal(piv, wpiv)
    assert np.array_equal(dx, want)


@pytest.mark.parametrize("name", ["dd", "qd"])
def test_config_full(mdps, name):
    t = mdinputs.toeplitz_config(name)
    dx, piv, sing = gpu_solve(mdps, t)
    want, wpiv = oracle.toeplitz_solve(t.jac, t.rhs, nthreads=NTHREADS)
    assert np.array_equal(piv, wpiv)
    err = oracle.series_err(dx, want)
    assert err.max() <= TOL[t.limbs], err.max()


@pytest.mark.parametrize("name,degree", [("od", 15), ("deca", 5)])
def test_config_leading_coefficients(mdps, name, degree):
    """Full n and full degree on the GPU; the oracle solves the system
    truncated at `degree`, which fixes dx_0..dx_degree (truncation invariant,
    tests/test_oracle_solve.py)."""
    t = mdinputs.toeplitz_config(name)
    dx, piv, sing = gpu_solve(mdps, t)
    tt = t.truncate(degree)
    want, wpiv = oracle.toeplitz_solve(tt.jac, tt.rhs, nthreads=NTHREADS)
    assert np.array_equal(piv, wpiv)
    err = oracle.series_err(np.ascontiguousarray(dx[..., :degree + 1]), want)
    assert err.max() <= TOL[t.limbs], err.max()


@pytest.mark.parametrize("name", ["od", "deca"])
def test_config_residual_sampled_rows(mdps, name):
    """Full size: for two sampled rows p, sum_q J_pq * dx_q - b_p formed by the
    oracle at L+2 limbs is below TOL[L] times the largest product series."""
    t = mdinputs.toeplitz_config(name)
    dx, _, _ = gpu_solve(mdps, t)
    L, Lh = t.limbs, t.limbs + 2
    pad = lambda a: np.ascontiguousarray(np.pad(a, [(0, 0), (0, Lh - L), (0, 0)]))
    for p in (0, t.n - 1):
        acc = pad(-t.rhs[p])
        scale = 0.0
        for q in range(t.n):
            prod = oracle.series_mul(pad(t.jac[p, q]), pad(dx[q]))
            scale = max(scale, float(np.abs(prod[:, 0]).max()))
            acc = oracle.series_add(acc, prod)
        res = float(np.abs(acc[:, 0]).max())
        assert res <= TOL[L] * scale, (p, res / scale)


def test_deterministic(mdps):
    t = mdinputs.toeplitz_config("qd")
    a, _, _ = gpu_solve(mdps, t)
    b, _, _ = gpu_solve(mdps, t)
    assert np.array_equal(a, b)


def test_singular_flag(mdps):
    t = mdinputs.random_toeplitz(13, 3, 2, 2)
    jac = t.jac.copy()
    jac[:, 1, :, :, 0] = 0.0
    _, _, sing = gpu_solve(mdps, t, jac)
    assert sing


@pytest.mark.parametrize("L", LEVELS)
@pytest.mark.parametrize("N,n,degree", [(3, 2, 0), (5, 3, 4), (9, 4, 7), (12, 12, 3)])
def test_least_squares_small(mdps, N, n, degree, L):
    """N >= n: against the oracle's least-squares forward
    substitution (normal equations formed exactly, reading R18)."""
    import torch
    t = mdinputs.random_toeplitz_rect(500 + 7 * N + n + degree, N, n, degree, L)
    with mdps.Solver(n, degree, L, n_eqs=N) as s:
        dx = s.solve(cuda(t.jac), cuda(t.rhs))
        torch.cuda.synchronize()
        dx = dx.cpu().numpy()
    want = oracle.toeplitz_lstsq(t.jac, t.rhs, nthreads=NTHREADS)
    err = oracle.series_err(dx, want)
    assert err.max() <= TOL[L], err.max()


def test_least_squares_config_shape(mdps):
    """od-like limbs and degree, 2n x n."""
    import torch
    t = mdinputs.random_toeplitz_rect(77, 48, 24, 15, 8)
    with mdps.Solver(24, 15, 8, n_eqs=48) as s:
        dx = s.solve(cuda(t.jac), cuda(t.rhs))
        torch.cuda.synchronize()
        dx = dx.cpu().numpy()
    want = oracle.toeplitz_lstsq(t.jac, t.rhs, nthreads=NTHREADS)
    assert oracle.series_err(dx, want).max() <= TOL[8]


def _conditioned_toeplitz(kappa_exp, seed, L, n=4, degree=3):
    """A_0 = H1 diag(2, 1, .., 1, 10^-kappa_exp) H2 with rational Householder
    reflections H (exactly orthogonal), rounded to L limbs: kappa(A_0) ~
    2 10^kappa_exp; A_1.. and b from the seeded unit-circle generator."""
    import random
    from fractions import Fraction as Fr
    from tests.exact import greedy

    def householder(v):
        vv = sum(x * x for x in v)
        return [[(1 if i == j else 0) - 2 * v[i] * v[j] / vv for j in range(n)] for i in range(n)]

    def mm(A, B):
        return [[sum(A[i][k] * B[k][j] for k in range(n)) for j in range(n)] for i in range(n)]

    rng = random.Random(seed)
    H1 = householder([Fr(rng.randint(1, 9)) for _ in range(n)])
    H2 = householder([Fr(rng.randint(-9, 9) or 1) for _ in range(n)])
    d = [[Fr(0)] * n for _ in range(n)]
    for i in range(n):
        d[i][i] = Fr(1)
    d[0][0], d[n - 1][n - 1] = Fr(2), Fr(1, 10 ** kappa_exp)
    A0 = mm(mm(H1, d), H2)
    t = mdinputs.random_toeplitz(300 + seed, n, degree, L)
    jac = t.jac.copy()
    for p in range(n):
        for q in range(n):
            jac[p, q, 0, :, 0] = greedy(A0[p][q], L)
            jac[p, q, 1, :, 0] = 0.0
    return t, jac


@pytest.mark.parametrize("L", (2, 8))
@pytest.mark.parametrize("seed", (0, 1, 2))
def test_ill_conditioned_flags(mdps, L, seed):
    """kappa(A_0) ~ 1e12: the refinement converges (no flag) and dx matches
    the oracle's md LU within kappa x the md unit; kappa ~ 1e17: the double
    Gauss-Jordan seed has ||I - W A_0|| > 1, Newton-Schulz cannot converge,
    and the solve reports MDPS_SOLVE_NOT_CONVERGED (the
    paper's md LU has no such limit, so the limit is reported, not silent)."""
    import torch
    for kexp, must_flag in ((12, False), (17, True)):
        t, jac = _conditioned_toeplitz(kexp, seed, L)
        with mdps.Solver(t.n, t.degree, t.limbs) as s:
            dx = s.solve(cuda(jac), cuda(t.rhs))
            torch.cuda.synchronize()
            flags = s.flags()
            _, sing = s.status()
        assert not sing
        if must_flag:
            assert flags & mdps.MDPS_SOLVE_NOT_CONVERGED, (kexp, seed, flags)
        else:
            assert flags == 0, (kexp, seed, flags)
            want, _ = oracle.toeplitz_solve(jac, t.rhs, nthreads=NTHREADS)
            err = oracle.series_err(dx.cpu().numpy() if hasattr(dx, "cpu") else dx, want)
            assert err.max() <= 2.0 * 10.0 ** kexp * 4096 * 2.0 ** (-53 * L), err.max()
