"""CPU oracle for mdps_eval_diff — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  The product path
(paper_2012_06607_b200/) never imports it, and it shares no code with the
CUDA library.  The arithmetic lives in mdoracle.c (see its header for the
definitions it follows and the PAPER.md passages it cites); this module only
builds it and marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mdoracle.c")
_LIB = os.path.join(_HERE, "libmdoracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread", "-Wall"]
MAXL = 16


def build(force: bool = False) -> str:
    """Compile oracle/libmdoracle.so (gcc, no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        d, i32, ll = ctypes.c_double, ctypes.c_int, ctypes.c_longlong
        L.mdo_round.argtypes = [P(d), i32, i32, P(d)]
        for f in ("mdo_add", "mdo_mul", "mdo_div"):
            getattr(L, f).argtypes = [P(d), P(d), i32, P(d)]
        L.mdo_sqrt.argtypes = [P(d), i32, P(d)]
        L.mdo_norm2.argtypes = [P(d), i32, i32, P(d)]
        L.mdo_series_mul.argtypes = [P(d), P(d), i32, i32, P(d), P(ll)]
        L.mdo_series_add.argtypes = [P(d), P(d), i32, i32, P(d)]
        L.mdo_series_inv.argtypes = [P(d), i32, i32, P(d)]
        L.mdo_eval_entries.argtypes = [i32, i32, P(i32), P(i32), P(i32), P(i32), P(d), P(d), i32, i32,
                                       i32, P(i32), P(i32), P(d), i32, P(ll)]
        L.mdo_series_err.argtypes = [P(d), P(d), i32, i32, i32, P(d)]
        L.mdo_eval_values_weighted.argtypes = [i32, i32, P(i32), P(i32), P(i32), P(i32), P(d), P(d), i32, i32,
                                               i32, P(i32), P(d), P(d), i32, P(ll)]
        L.mdo_euler_residual.argtypes = [i32, i32, i32, i32, P(d), P(d), P(d), P(d), i32]
        L.mdo_toeplitz_solve.argtypes = [i32, i32, i32, P(d), P(d), P(d), P(i32), i32]
        L.mdo_toeplitz_normal.argtypes = [i32, i32, i32, i32, P(d), P(d), i32, P(d), P(d)]
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _check(rc: int, what: str):
    if rc != 0:
        raise ArithmeticError(f"oracle {what} failed (rc={rc})")


# ---- multiple-double numbers (real, L limbs) ------------------------------------
def md_round(values: Sequence[float], L: int) -> np.ndarray:
    """Greedy L-limb round-to-nearest of the exact sum of `values`."""
    v = _f64(values).ravel()
    out = np.zeros(L)
    _check(lib().mdo_round(_dp(v), v.size, L, _dp(out)), "round")
    return out


def _binop(name: str, a, b) -> np.ndarray:
    a, b = _f64(a), _f64(b)
    assert a.shape == b.shape and a.ndim == 1
    out = np.zeros_like(a)
    _check(getattr(lib(), name)(_dp(a), _dp(b), a.size, _dp(out)), name)
    return out


def md_add(a, b):
    return _binop("mdo_add", a, b)


def md_mul(a, b):
    return _binop("mdo_mul", a, b)


def md_div(a, b):
    return _binop("mdo_div", a, b)


def md_sqrt(a) -> np.ndarray:
    a = _f64(a)
    out = np.zeros_like(a)
    _check(lib().mdo_sqrt(_dp(a), a.size, _dp(out)), "sqrt")
    return out


def md_norm2(v) -> np.ndarray:
    """2-norm of a complex md vector v[count][2][L]."""
    v = _f64(v)
    count, two, L = v.shape
    assert two == 2
    out = np.zeros(L)
    _check(lib().mdo_norm2(_dp(v), count, L, _dp(out)), "norm2")
    return out


# ---- truncated power series [2][L][D] ------------------------------------------
def series_mul(x, y, counts: Optional[np.ndarray] = None) -> np.ndarray:
    x, y = _f64(x), _f64(y)
    _, L, D = x.shape
    z = np.zeros_like(x)
    cp = None
    if counts is not None:
        assert counts.dtype == np.int64 and counts.size >= 2
        cp = counts.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong))
    _check(lib().mdo_series_mul(_dp(x), _dp(y), D, L, _dp(z), cp), "series_mul")
    return z


def series_add(x, y) -> np.ndarray:
    """x + y for series [..., 2, L, D] (any leading shape)."""
    x, y = _f64(x), _f64(y)
    assert x.shape == y.shape
    _, L, D = x.shape[-3:]
    xf, yf = x.reshape(-1, 2, L, D), y.reshape(-1, 2, L, D)
    z = np.zeros_like(xf)
    for t in range(xf.shape[0]):
        zt = np.zeros((2, L, D))
        _check(lib().mdo_series_add(_dp(np.ascontiguousarray(xf[t])), _dp(np.ascontiguousarray(yf[t])),
                                    D, L, _dp(zt)), "series_add")
        z[t] = zt
    return z.reshape(x.shape)


def series_inv(x) -> np.ndarray:
    x = _f64(x)
    _, L, D = x.shape
    y = np.zeros_like(x)
    _check(lib().mdo_series_inv(_dp(x), D, L, _dp(y)), "series_inv")
    return y


# ---- eval/diff -------------------------------------------------------------------
def eval_entries(si, entries: Sequence[Tuple[int, int]], nthreads: Optional[int] = None,
                 limbs: Optional[int] = None) -> Tuple[np.ndarray, int]:
    """Oracle values (col < 0) and Jacobian entries (row, col) of system `si`
    (an mdinputs.SystemInputs).  Returns (out[n_entries][2][L][D], products).

    `limbs` > si.limbs evaluates the same inputs (zero-padded limbs) at a
    higher precision (the oracle's self-consistency pin)."""
    L = limbs or si.limbs
    coeffs, x = si.coeffs, si.x
    if L != si.limbs:
        assert L > si.limbs
        pad = [(0, 0), (0, 0), (0, L - si.limbs), (0, 0)]
        coeffs, x = np.pad(coeffs, pad), np.pad(x, pad)
    coeffs, x = _f64(coeffs), _f64(x)
    rows = _i32([e[0] for e in entries])
    cols = _i32([e[1] for e in entries])
    out = np.zeros((len(entries), 2, L, si.degree + 1))
    prods = ctypes.c_longlong(0)
    n_polys = int(si.poly_ptr.shape[0] - 1)
    nt = nthreads or os.cpu_count() or 1
    rc = lib().mdo_eval_entries(n_polys, si.n, _ip(_i32(si.poly_ptr)), _ip(_i32(si.mono_ptr)),
                                _ip(_i32(si.vars)), _ip(_i32(si.exps)), _dp(coeffs), _dp(x),
                                si.degree, L, len(entries), _ip(rows), _ip(cols), _dp(out), nt,
                                ctypes.byref(prods))
    _check(rc, "eval_entries")
    return out, int(prods.value)


def values_weighted(si, rows: Sequence[int], nthreads: Optional[int] = None):
    """(f, g) of the given rows from one set of monomial chains: f_i the
    value, g_i = sum_r deg(r) c_r x^{a_r} the degree-weighted value (Euler's
    identity: sum_j x_j J_ij = g_i).  Equal to eval_entries' (i, -1) and
    (i, -2) entries bit for bit."""
    L, D = si.limbs, si.degree + 1
    r = _i32(list(rows))
    f = np.zeros((len(r), 2, L, D))
    g = np.zeros((len(r), 2, L, D))
    prods = ctypes.c_longlong(0)
    n_polys = int(si.poly_ptr.shape[0] - 1)
    rc = lib().mdo_eval_values_weighted(n_polys, si.n, _ip(_i32(si.poly_ptr)), _ip(_i32(si.mono_ptr)),
                                        _ip(_i32(si.vars)), _ip(_i32(si.exps)), _dp(_f64(si.coeffs)), _dp(_f64(si.x)),
                                        si.degree, L, len(r), _ip(r), _dp(g), _dp(f),
                                        nthreads or os.cpu_count() or 1, ctypes.byref(prods))
    _check(rc, "values_weighted")
    return f, g


def eval_diff(si, nthreads: Optional[int] = None, limbs: Optional[int] = None):
    """Full naive evaluation: (values[n_polys][2][L][D], jac[n_polys][n][2][L][D], products)."""
    n_polys = int(si.poly_ptr.shape[0] - 1)
    entries = [(i, -1) for i in range(n_polys)] + [(i, j) for i in range(n_polys) for j in range(si.n)]
    out, prods = eval_entries(si, entries, nthreads, limbs)
    vals = out[:n_polys]
    jac = out[n_polys:].reshape((n_polys, si.n) + out.shape[1:])
    return vals, jac, prods


def series_err(a, b) -> np.ndarray:
    """Per-series error e_s = max_k |a-b| / max(max_k |b|, 1), differences exact.
    a, b: [..., 2, L, D]; returns an array of the leading shape."""
    a, b = _f64(a), _f64(b)
    assert a.shape == b.shape
    lead = a.shape[:-3]
    _, L, D = a.shape[-3:]
    count = int(np.prod(lead)) if lead else 1
    err = np.zeros(count)
    _check(lib().mdo_series_err(_dp(a), _dp(b), count, D, L, _dp(err)), "series_err")
    return err.reshape(lead)


def euler_residual(x, jac_rows, g, nthreads: Optional[int] = None) -> np.ndarray:
    """Exact Euler residual of Jacobian rows (mdoracle.c mdo_euler_residual):
    res[c][k] = |sum_j (x_j * J_cj)_k - g_ck|, the products truncated at t^D and
    every sum formed exactly, rounded once.  x [n][2][L][D], jac_rows
    [count][n][2][L][D], g [count][2][L][D] (g = deg * f for a system
    homogeneous of degree deg, else eval_entries' (i, -2) entries)."""
    x, jac_rows, g = _f64(x), _f64(jac_rows), _f64(g)
    n, _, L, D = x.shape
    count = jac_rows.shape[0]
    assert jac_rows.shape == (count, n, 2, L, D) and g.shape == (count, 2, L, D)
    res = np.zeros((count, D))
    _check(lib().mdo_euler_residual(count, n, D, L, _dp(x), _dp(jac_rows), _dp(g), _dp(res),
                                    nthreads or os.cpu_count() or 1), "euler_residual")
    return res


# ---- block lower-triangular Toeplitz forward substitution ------------------------
class SingularError(ArithmeticError):
    pass


def toeplitz_solve(jac, rhs, nthreads: Optional[int] = None, limbs: Optional[int] = None):
    """dx(t) with (A_0 + A_1 t + ...)(dx_0 + dx_1 t + ...) = b(t) mod t^D
    (PAPER.md:266-333): jac [n][n][2][L][D] (A_k = coefficient k), rhs
    [n][2][L][D].  Returns (dx [n][2][L][D], pivots [n]).  `limbs` > L solves
    the same inputs (zero-padded limbs) at a higher precision."""
    jac, rhs = _f64(jac), _f64(rhs)
    n, n2, two, L0, D = jac.shape
    assert n == n2 and two == 2 and rhs.shape == (n, 2, L0, D)
    L = limbs or L0
    if L != L0:
        assert L > L0
        jac = _f64(np.pad(jac, [(0, 0)] * 3 + [(0, L - L0), (0, 0)]))
        rhs = _f64(np.pad(rhs, [(0, 0)] * 2 + [(0, L - L0), (0, 0)]))
    dx = np.zeros((n, 2, L, D))
    piv = np.zeros(n, dtype=np.int32)
    nt = nthreads or os.cpu_count() or 1
    rc = lib().mdo_toeplitz_solve(n, D, L, _dp(jac), _dp(rhs), _dp(dx), _ip(piv), nt)
    if rc == -4:
        raise SingularError("A_0 is singular (zero pivot column)")
    _check(rc, "toeplitz_solve")
    return dx, piv


def toeplitz_lstsq(jac, rhs, nthreads: Optional[int] = None):
    """Least-squares forward substitution for N >= n equations:
    dx_j = argmin |A_0 dx_j - r_j|, r_j = b_j - sum_{i>=1} A_i dx_{j-i}, i.e. the
    square forward substitution of the normal equations A_0^H A(t) dx = A_0^H b
    (formed exactly, rounded to L+3 limbs, solved at L+3 limbs, dx rounded to L).
    jac [N][n][2][L][D], rhs [N][2][L][D] -> dx [n][2][L][D]."""
    jac, rhs = _f64(jac), _f64(rhs)
    N, n, two, L, D = jac.shape
    assert two == 2 and rhs.shape == (N, 2, L, D) and N >= n
    Lo = L + 3
    jt = np.zeros((n, n, 2, Lo, D))
    bt = np.zeros((n, 2, Lo, D))
    _check(lib().mdo_toeplitz_normal(N, n, D, L, _dp(jac), _dp(rhs), Lo, _dp(jt), _dp(bt)), "toeplitz_normal")
    dxo, _ = toeplitz_solve(jt, bt, nthreads)
    dx = np.zeros((n, 2, L, D))
    for q in range(n):
        for part in range(2):
            for k in range(D):
                dx[q, part, :, k] = md_round(dxo[q, part, :, k], L)
    return dx


# ---- Newton's method on power series ----------------------------------------------
def newton(si, steps: int, nthreads: Optional[int] = None):
    """`steps` Newton steps from si.x: at x_k, f and J by the
    plain definition (eval_diff), dx from J(t) dx(t) = -f(t) by forward
    substitution (toeplitz_solve), x_{k+1} = x_k + dx (series_add).
    Returns (x, update norms max_{q,k} |dx_{q,k}| of the leading limbs)."""
    x = _f64(si.x).copy()
    norms = []
    for _ in range(steps):
        vals, jac, _ = eval_diff(dataclasses.replace(si, x=x), nthreads)
        dx, _ = toeplitz_solve(jac, -vals, nthreads)
        x = series_add(x, dx)
        norms.append(float(np.max(np.hypot(dx[:, 0, 0, :], dx[:, 1, 0, :]))))
    return x, norms
