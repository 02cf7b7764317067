"""CUDA parity: libmdps (through its C ABI) against the CPU oracle.

Every comparison forms the difference exactly (oracle.series_err) and uses
the per-series tolerance of BASELINE.json's north_star (tests/gpu_util.TOL).
Integer-valued cases are compared bit-exactly.
"""
import math
import random
from fractions import Fraction

import numpy as np
import pytest

import mdinputs
import oracle
from tests.exact import greedy, value
from tests.gpu_util import TOL, check_against_oracle, euler_check, gpu_eval, sample_entries, structural_support

pytestmark = pytest.mark.gpu
LEVELS = (2, 3, 4, 5, 8, 10)
ALGOS = (1, 2)  # MDPS_ALGO_EFT, MDPS_ALGO_DIGITS


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


@pytest.mark.parametrize("L", LEVELS)
def test_md_ops_device(mdps, L):
    """device md add/mul (md.cuh) vs exact rationals: error <= 8 u."""
    rng = random.Random(L)
    count = 64
    A = np.zeros((count, L))
    B = np.zeros((count, L))
    for c in range(count):
        A[c] = greedy(Fraction(rng.getrandbits(60 * L), 1 << (60 * L - 2)) - 2, L)
        B[c] = greedy(Fraction(rng.getrandbits(60 * L), 1 << (60 * L - 1)) - 1, L)
    for op in (0, 1):
        C = mdps.test_md_op(op, cuda(A), cuda(B)).cpu().numpy()
        for c in range(count):
            a, b = value(A[c]), value(B[c])
            ex = a + b if op == 0 else a * b
            assert abs(value(C[c]) - ex) <= Fraction(8, 2 ** (53 * L)) * max(abs(ex), Fraction(1, 2 ** 60))


@pytest.mark.parametrize("L", LEVELS)
def test_ex1_norm_on_device(mdps, L):
    """PAPER.md:82-95 on the device: sum |v_j|^2 = 64 for 64 unit complex entries."""
    from tests.test_oracle_md import unit_circle_md
    v = unit_circle_md(random.Random(640 + L), 64, L)
    s = mdps.test_norm2sq(cuda(v)).cpu().numpy()
    assert s[0] == 64.0
    assert abs(value(s) - 64) <= Fraction(64 * 8, 2 ** (53 * L))


@pytest.mark.parametrize("L", LEVELS)
def test_digits_roundtrip(mdps, L):
    """limbs -> 23-bit digit planes -> limbs preserves the value to the md unit."""
    si = mdinputs.random_system(7, 4, 2, (1, 2), (1,), 20, L)
    y = mdps.test_digits_roundtrip(cuda(si.x)).cpu().numpy()
    err = oracle.series_err(y, si.x)
    assert err.max() <= 4 * 2.0 ** (-53 * L)


@pytest.mark.parametrize("L", LEVELS)
@pytest.mark.parametrize("scale_exp", [-500, -160 * 3, -300, 300, 900])
def test_digits_roundtrip_extreme_magnitudes(mdps, L, scale_exp):
    """Tiny and huge md numbers (late Newton updates reach 2^-530 at L = 10):
    the digit split scales exactly, so no digit weight under/overflows; the
    round trip keeps every limb that is a normal double."""
    si = mdinputs.random_system(8, 4, 2, (1, 2), (1,), 9, L)
    x = si.x * 2.0 ** scale_exp            # exact power-of-two scaling
    y = mdps.test_digits_roundtrip(cuda(x)).cpu().numpy()
    assert np.isfinite(y).all()
    err = float(np.max(np.abs(y[:, :, 0] - x[:, :, 0]) / np.maximum(np.abs(x[:, :, 0]), 1e-300)))
    assert err <= 2.0 ** -52
    if scale_exp - 53 * L - 30 > -1074:   # the md precision floor is above the subnormals
        assert (oracle.series_err(y * 2.0 ** -scale_exp, si.x) <= 4 * 2.0 ** (-53 * L)).all()


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("L", LEVELS)
def test_series_product_grid(mdps, algo, L):
    """one product job per (D, L): D spans a single tile, odd D, the fold's
    middle thread, several warps and the maximum D."""
    for D in (1, 2, 9, 16, 17, 32, 64, 128):
        rng = mdinputs.SplitMix64(100 * L + D, "extra")
        count = 3
        x = mdinputs.unit_circle_series(rng, count, D, L, "random")
        y = mdinputs.unit_circle_series(rng, count, D, L, "random")
        z = mdps.test_series_mul(cuda(x), cuda(y), algo=algo).cpu().numpy()
        want = np.stack([oracle.series_mul(x[c], y[c]) for c in range(count)])
        err = oracle.series_err(z, want)
        assert err.max() <= TOL[L], (D, err)


@pytest.mark.parametrize("algo", ALGOS)
def test_series_product_edge_values(mdps, algo):
    """zeros, a zero leading coefficient, exact integers, mixed magnitudes."""
    L, D = 4, 12
    x = np.zeros((4, 2, L, D))
    y = np.zeros((4, 2, L, D))
    x[1, 0, 0, 3:] = 1.0                       # leading coefficients zero
    y[1, 1, 0, :] = np.arange(1, D + 1)
    x[2, 0, 0, :] = 2.0 ** np.arange(-40, -40 + 6 * D, 6)  # wide magnitude range
    x[2, 0, 1, :] = x[2, 0, 0, :] * 2.0 ** -60
    y[2, 0, 0, :] = 3.0
    x[3, 0, 0, 0] = 1.0
    y[3, 0, 0, :] = 1e-200                     # tiny values
    z = mdps.test_series_mul(cuda(x), cuda(y), algo=algo).cpu().numpy()
    want = np.stack([oracle.series_mul(x[c], y[c]) for c in range(4)])
    assert oracle.series_err(z, want).max() <= TOL[L]
    assert not z[0].any()
    assert np.array_equal(z[1], want[1])       # integer products are exact


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("m,L", [(3, 2), (8, 4), (16, 8), (16, 10)])
def test_exact_integer_case_bitexact(mdps, algo, m, L):
    """x_j = 1 + alpha_j t, c = 1: all results are integers < 2^53,
    so the GPU must be bit-exact; catches off-by-one cross-product indices."""
    from tests.test_oracle_evaldiff import const_series, esym, make_si
    D = m + 2
    alphas = list(range(1, m + 1))
    xs = [const_series([1, a], L, D) for a in alphas]
    si = make_si(m, [[[(j, 1) for j in range(m)]]] + [[] for _ in range(m - 1)],
                 [const_series([1], L, D)], xs, D - 1, L)
    vals, jac, _ = gpu_eval(si, algo)
    assert np.array_equal(vals[0], const_series([esym(alphas, k) for k in range(D)], L, D))
    for l in range(m):
        rest = alphas[:l] + alphas[l + 1:]
        assert np.array_equal(jac[0, l], const_series([esym(rest, k) for k in range(D)], L, D))
    assert not vals[1:].any() and not jac[1:].any()


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("L", (2, 4, 10))
def test_circle_system(mdps, algo, L):
    """f = (s(t) - y, x^2 + y^2 - 1) at (cos_8, sin_8)."""
    from tests.test_oracle_evaldiff import GOLD, const_series, make_si
    g = GOLD["circle"]
    d = g["degree"]
    D = d + 1
    s_coef = [Fraction(c) for c in g["s_coefficients"]]
    cos_coef = [Fraction(c) for c in g["cos_coefficients"]]
    polys = [[[], [(1, 1)]], [[(0, 2)], [(1, 2)], []]]
    coeffs = [const_series(s_coef, L, D), const_series([-1], L, D), const_series([1], L, D),
              const_series([1], L, D), const_series([-1], L, D)]
    x, y = const_series(cos_coef, L, D), const_series(s_coef, L, D)
    si = make_si(2, polys, coeffs, [x, y], d, L)
    vals, jac, _ = gpu_eval(si, algo)
    ov, oj, _ = oracle.eval_diff(si)
    assert oracle.series_err(vals, ov).max() <= TOL[L]
    assert oracle.series_err(jac, oj).max() <= TOL[L]
    assert not jac[0, 0].any()
    assert np.array_equal(jac[0, 1], const_series([-1], L, D))
    # J = [[0, -1], [2x, 2y]]: 2x is exact, the GPU's final limb rounding is faithful
    assert oracle.series_err(jac[1, 0], 2 * x) <= 4 * 2.0 ** (-53 * L)
    assert oracle.series_err(jac[1, 1], 2 * y) <= 4 * 2.0 ** (-53 * L)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("L", LEVELS)
def test_small_random_systems_full(mdps, algo, L):
    """every output of small systems: constants, m = 1, exponents 2 and 3,
    duplicate monomials allowed, degree spanning a ragged tail."""
    si = mdinputs.random_system(300 + L, n=5, monos=6, m_range=(0, 4), exps=(1, 2, 3), degree=18, limbs=L)
    vals, jac, _ = gpu_eval(si, algo)
    ov, oj, _ = oracle.eval_diff(si)
    assert oracle.series_err(vals, ov).max() <= TOL[L]
    assert oracle.series_err(jac, oj).max() <= TOL[L]
    sup = structural_support(si)
    assert not jac[~sup].any()


@pytest.mark.parametrize("algo", ALGOS)
def test_config_dd_full(mdps, algo):
    """BASELINE config 0 (dd), every output."""
    si = mdinputs.make_config("dd")
    vals, jac, st = gpu_eval(si, algo)
    ov, oj, _ = oracle.eval_diff(si)
    assert oracle.series_err(vals, ov).max() <= TOL[2]
    assert oracle.series_err(jac, oj).max() <= TOL[2]
    assert st["products"] == 128 * 3 * 2  # 3(m-1) per monomial, m = 3


@pytest.mark.parametrize("name,nv,nj", [("qd", 2, 6), ("od", 1, 4), ("deca", 1, 3)])
def test_config_sampled(mdps, name, nv, nj):
    """BASELINE configs 1-3 at full size in the launch configuration bench.py
    times: sampled outputs vs the oracle, all structural zeros exact, and
    bitwise run-to-run determinism."""
    si = mdinputs.make_config(name)
    vals, jac, st = gpu_eval(si, 0)
    sup = structural_support(si)
    assert not jac[~sup].any()
    assert np.isfinite(vals).all() and np.isfinite(jac).all()
    err, _ = check_against_oracle(si, vals, jac, sample_entries(si, nv, nj, seed=1, sup=sup), TOL[si.limbs])
    assert err <= TOL[si.limbs], err
    v2, j2, _ = gpu_eval(si, 0)
    assert np.array_equal(vals, v2) and np.array_equal(jac, j2)


@pytest.mark.parametrize("d", mdinputs.SWEEP_DEGREES)
def test_sweep_cells(mdps, d):
    """BASELINE config 4: the fixed system at d x L; one sampled Jacobian entry
    and (small cells) one value per cell against the oracle; EVERY output of
    every cell through Euler's identity on all 64 rows (all monomials have
    degree 8: sum_j x_j J_ij = 8 f_i, the residual formed exactly by the
    oracle, tests/gpu_util.euler_check)."""
    for L in mdinputs.SWEEP_LIMBS:
        si = mdinputs.sweep_cell(d, L)
        # the default (EFT for L = 2 below degree 63, digits otherwise) and, at
        # L <= 3, both algorithms explicitly
        for algo in ((0, 1, 2) if L <= 3 else (0,)):
            vals, jac, st = gpu_eval(si, algo)
            if algo == 0:
                assert st["algo"] == (1 if L == 2 and d < 63 else 2), (d, L, st["algo"])
            nv = 1 if d * L <= 63 * 4 else 0
            err, _ = check_against_oracle(si, vals, jac, sample_entries(si, nv, 1, seed=d + L), TOL[L])
            assert err <= TOL[L], (d, L, algo, err)
            euler_check(si, vals, jac, TOL[L])


def test_graph_and_stream_paths(mdps):
    """CUDA-graph replay and a non-default stream give bit-identical outputs."""
    import torch
    si = mdinputs.make_config("dd")
    v0, j0, _ = gpu_eval(si, 0)
    with mdps.System.from_inputs(si, use_graph=True) as s:
        x = torch.from_numpy(si.x).cuda()
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                v, j = s.eval_diff(x, stream=st)
        st.synchronize()
        assert np.array_equal(v.cpu().numpy(), v0) and np.array_equal(j.cpu().numpy(), j0)


def test_host_entry_point(mdps):
    si = mdinputs.make_config("dd")
    v0, j0, _ = gpu_eval(si, 0)
    with mdps.System.from_inputs(si) as s:
        v, j = s.eval_diff_host(si.x)
    assert np.array_equal(v, v0) and np.array_equal(j, j0)


@pytest.mark.parametrize("name,nv,nj,seed", [("od", 3, 13, 11), ("deca", 1, 15, 12)])
def test_config_wide_sample(mdps, name, nv, nj, seed):
    """A wider sample of the full-size od and deca outputs (16 each, another
    seed): one oracle worker per host core."""
    si = mdinputs.make_config(name)
    vals, jac, st = gpu_eval(si, 0)
    sup = structural_support(si)
    err, errs = check_against_oracle(si, vals, jac, sample_entries(si, nv, nj, seed=seed, sup=sup), TOL[si.limbs])
    assert err <= TOL[si.limbs], err
    # the error is far below the tolerance: report the margin in units of 2^-53L
    assert err <= 2.0 ** (-53 * si.limbs) * 4096
