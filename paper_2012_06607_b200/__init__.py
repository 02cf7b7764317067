"""libmdps — B200-native evaluation and differentiation of a polynomial system
at a vector of truncated power series in complex multiple-double precision
(arXiv 2012.06607).  Thin Python binding of the C ABI in include/libmdps.h:
argument marshalling only; every step of the computation runs in the CUDA
kernels of libmdps.so (built in-tree by paper_2012_06607_b200/build.py).

There is no CPU fallback: if libmdps.so is missing or no CUDA device is
present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

__all__ = [
    "MDPS_OK", "MDPS_EINVAL", "MDPS_ENOMEM", "MDPS_ECUDA", "MDPS_ALGO_AUTO", "MDPS_ALGO_EFT",
    "MDPS_ALGO_DIGITS", "MDPS_SCHED_AUTO", "MDPS_SCHED_LEVELS", "MDPS_SCHED_QUEUE", "MdpsError", "lib", "library_path", "System",
    "mdps_system_create", "mdps_eval_diff", "mdps_eval_diff_host", "mdps_system_destroy",
    "mdps_last_error", "mdps_system_stats", "EXPORTED_SYMBOLS", "Solver",
]

MDPS_OK, MDPS_EINVAL, MDPS_ENOMEM, MDPS_ECUDA = 0, -1, -2, -3
MDPS_ALGO_AUTO, MDPS_ALGO_EFT, MDPS_ALGO_DIGITS = 0, 1, 2
MDPS_SCHED_AUTO, MDPS_SCHED_LEVELS, MDPS_SCHED_QUEUE = 0, 1, 2
MDPS_SOLVE_SINGULAR, MDPS_SOLVE_NOT_CONVERGED = 1, 2

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.path.join(_HERE, "libmdps.so")

# every extern "C" symbol declared in include/libmdps.h and include/mdps_test.h
EXPORTED_SYMBOLS = (
    "mdps_system_create", "mdps_system_create_ex", "mdps_eval_diff", "mdps_eval_diff_host",
    "mdps_system_destroy", "mdps_last_error", "mdps_system_stats", "mdps_system_level_jobs",
    "mdps_test_series_mul", "mdps_test_md_op", "mdps_test_norm2sq", "mdps_test_digits_roundtrip",
    "mdps_fp64_peak", "mdps_test_force_geometry", "mdps_test_set_pdl", "mdps_system_set_timing", "mdps_system_timing",
    "mdps_solver_create", "mdps_solve", "mdps_solver_status", "mdps_solver_stats", "mdps_solver_destroy",
    "mdps_solver_trace", "mdps_newton_step", "mdps_newton", "mdps_solver_create_ls", "mdps_test_queue_trace",
    "mdps_test_queue_config", "mdps_solver_flags", "mdps_test_plan", "mdps_test_balance",
)


class MdpsError(RuntimeError):
    pass


class _Supports(ctypes.Structure):
    _fields_ = [("n_polys", ctypes.c_int32), ("poly_ptr", ctypes.POINTER(ctypes.c_int32)),
                ("mono_ptr", ctypes.POINTER(ctypes.c_int32)), ("vars", ctypes.POINTER(ctypes.c_int32))]


class _Options(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int32), ("use_graph", ctypes.c_int32), ("real", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("schedule", ctypes.c_int32), ("workspace_mb", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = [("products", ctypes.c_int64), ("add_terms", ctypes.c_int64),
                ("fp64_ops_conv", ctypes.c_int64), ("fp64_ops_total", ctypes.c_int64),
                ("compulsory_bytes", ctypes.c_int64), ("levels", ctypes.c_int32),
                ("algo", ctypes.c_int32), ("digits", ctypes.c_int32), ("launches", ctypes.c_int32),
                ("workspace_bytes", ctypes.c_size_t), ("n", ctypes.c_int32), ("n_polys", ctypes.c_int32),
                ("degree", ctypes.c_int32), ("limbs", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("schedule", ctypes.c_int32), ("chunks", ctypes.c_int32), ("pool_bytes", ctypes.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class Timing(ctypes.Structure):
    _fields_ = [("conv_ms", ctypes.c_double), ("accum_ms", ctypes.c_double), ("convert_ms", ctypes.c_double),
                ("conv_launches", ctypes.c_int64), ("accum_launches", ctypes.c_int64),
                ("convert_launches", ctypes.c_int64), ("evals", ctypes.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


class SolverInfo(ctypes.Structure):
    _fields_ = [("complex_fma", ctypes.c_int64), ("fp64_ops", ctypes.c_int64), ("launches", ctypes.c_int32),
                ("grid_blocks", ctypes.c_int32), ("workspace_bytes", ctypes.c_size_t)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib: Optional[ctypes.CDLL] = None


def lib() -> ctypes.CDLL:
    """Load libmdps.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(library_path):
        raise MdpsError(f"{library_path} not built: run `python -m paper_2012_06607_b200.build` "
                        "or __graft_entry__.build()")
    L = ctypes.CDLL(library_path)
    P, vp = ctypes.POINTER, ctypes.c_void_p
    i32, i64 = ctypes.c_int32, ctypes.c_int64
    L.mdps_system_create.restype = vp
    L.mdps_system_create.argtypes = [P(_Supports), P(i32), P(ctypes.c_double), i32, i32, i32]
    L.mdps_system_create_ex.restype = vp
    L.mdps_system_create_ex.argtypes = [P(_Supports), P(i32), P(ctypes.c_double), i32, i32, i32, P(_Options)]
    L.mdps_eval_diff.argtypes = [vp, vp, vp, vp, vp]
    L.mdps_eval_diff_host.argtypes = [vp, vp, vp, vp, vp]
    L.mdps_system_destroy.argtypes = [vp]
    L.mdps_system_destroy.restype = None
    L.mdps_last_error.restype = ctypes.c_char_p
    L.mdps_system_stats.argtypes = [vp, P(Stats)]
    L.mdps_system_level_jobs.argtypes = [vp, P(i64), i32]
    L.mdps_test_series_mul.argtypes = [vp, vp, vp, i32, i32, i32, i32, vp]
    L.mdps_test_md_op.argtypes = [i32, vp, vp, vp, i32, i32, vp]
    L.mdps_test_norm2sq.argtypes = [vp, i32, i32, vp, vp]
    L.mdps_test_digits_roundtrip.argtypes = [vp, vp, i32, i32, i32, vp]
    L.mdps_fp64_peak.argtypes = [i64, P(ctypes.c_double), vp]
    L.mdps_test_force_geometry.argtypes = [i32, i32, i32]
    L.mdps_test_set_pdl.argtypes = [i32]
    L.mdps_system_set_timing.argtypes = [vp, i32]
    L.mdps_system_timing.argtypes = [vp, P(Timing), i32]
    L.mdps_solver_create.restype = vp
    L.mdps_solver_create.argtypes = [i32, i32, i32]
    L.mdps_solver_create_ls.restype = vp
    L.mdps_solver_create_ls.argtypes = [i32, i32, i32, i32]
    L.mdps_solve.argtypes = [vp, vp, vp, vp, vp]
    L.mdps_solver_status.argtypes = [vp, P(i32), P(i32)]
    L.mdps_solver_flags.argtypes = [vp, P(i32)]
    L.mdps_solver_stats.argtypes = [vp, P(SolverInfo)]
    L.mdps_solver_trace.argtypes = [vp, P(i64), i32, P(i32)]
    L.mdps_newton_step.argtypes = [vp, vp, vp, vp, vp, vp]
    L.mdps_newton.argtypes = [vp, vp, vp, i32, ctypes.c_double, P(ctypes.c_double), vp]
    L.mdps_test_queue_trace.argtypes = [vp, i32, P(i64), i32]
    L.mdps_test_queue_config.argtypes = [i32, i32]
    L.mdps_test_plan.argtypes = [P(_Supports), P(i32), i32, i32, i32, i32, i32, i32, i32, P(i64)]
    L.mdps_test_balance.argtypes = [P(_Supports), P(i32), i32, i64, P(i64), P(i64), i32, P(i64), P(i32)]
    L.mdps_solver_destroy.argtypes = [vp]
    L.mdps_solver_destroy.restype = None
    _lib = L
    return L


def mdps_last_error() -> str:
    return lib().mdps_last_error().decode()


def _check(rc: int, what: str):
    if rc != MDPS_OK:
        raise MdpsError(f"{what} failed (rc={rc}): {mdps_last_error()}")


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr_i32(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dptr(t, numel: Optional[int] = None, device: Optional[int] = None, name: str = "tensor") -> int:
    """device pointer of a torch CUDA float64 contiguous tensor; with `numel`
    and `device` given, its size and device are checked first (the C ABI only
    sees the pointer: a short buffer would be overrun by the kernels)."""
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise MdpsError(f"{name}: expected a contiguous float64 CUDA tensor")
    if numel is not None and t.numel() != numel:
        raise MdpsError(f"{name}: expected {numel} doubles, got {t.numel()} (shape {tuple(t.shape)})")
    if device is not None and t.device.index != device:
        raise MdpsError(f"{name}: on cuda:{t.device.index}, the object lives on cuda:{device}")
    return t.data_ptr()


def _hptr(a: np.ndarray, numel: int, name: str) -> int:
    """host pointer of a C-contiguous float64 numpy array of exactly `numel` doubles."""
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]):
        raise MdpsError(f"{name}: expected a C-contiguous float64 host array")
    if a.size != numel:
        raise MdpsError(f"{name}: expected {numel} doubles, got {a.size} (shape {a.shape})")
    return a.ctypes.data


def _current_device() -> int:
    import torch
    return torch.cuda.current_device()


def mdps_system_create(poly_ptr, mono_ptr, vars_, exponents, coefficients, n: int, degree: int,
                       limbs: int, algo: int = MDPS_ALGO_AUTO, use_graph: bool = False, real: bool = False,
                       batch: int = 1, schedule: int = MDPS_SCHED_AUTO, workspace_mb: int = 0) -> int:
    """Create a system; returns the opaque handle (int).  Host numpy inputs."""
    pp, mp, vv, ee = _i32(poly_ptr), _i32(mono_ptr), _i32(vars_), _i32(exponents)
    coeffs = np.ascontiguousarray(np.asarray(coefficients, dtype=np.float64))
    sup = _Supports(len(pp) - 1, _ptr_i32(pp), _ptr_i32(mp), _ptr_i32(vv))
    opts = _Options(algo, 1 if use_graph else 0, 1 if real else 0, int(batch), int(schedule), int(workspace_mb))
    h = lib().mdps_system_create_ex(ctypes.byref(sup), _ptr_i32(ee),
                                    coeffs.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                    n, degree, limbs, ctypes.byref(opts))
    if not h:
        raise MdpsError(f"mdps_system_create failed: {mdps_last_error()}")
    return h


def _sizes(handle: int):
    """(doubles of series_in, values_out, jacobian_out) of a system, from its stats."""
    st = mdps_system_stats(handle)
    return st["in_doubles"], st["values_doubles"], st["jacobian_doubles"]


def mdps_eval_diff(handle: int, series_in, values_out, jacobian_out, stream=None, device=None) -> None:
    """Asynchronous eval/diff on device tensors (libmdps.h); sizes and device checked."""
    nin, nval, njac = _sizes(handle)
    _check(lib().mdps_eval_diff(handle, _dptr(series_in, nin, device, "series_in"),
                                _dptr(values_out, nval, device, "values_out"),
                                _dptr(jacobian_out, njac, device, "jacobian_out"),
                                _stream_handle(stream)), "mdps_eval_diff")


def mdps_eval_diff_host(handle: int, series_in: np.ndarray, values_out: np.ndarray,
                        jacobian_out: np.ndarray, stream=None) -> None:
    """End-to-end eval/diff with HOST numpy buffers (synchronous); sizes checked."""
    nin, nval, njac = _sizes(handle)
    _check(lib().mdps_eval_diff_host(handle, _hptr(series_in, nin, "series_in"),
                                     _hptr(values_out, nval, "values_out"),
                                     _hptr(jacobian_out, njac, "jacobian_out"), _stream_handle(stream)),
           "mdps_eval_diff_host")


def mdps_system_destroy(handle: int) -> None:
    lib().mdps_system_destroy(handle)


def mdps_system_stats(handle: int) -> dict:
    st = Stats()
    _check(lib().mdps_system_stats(handle, ctypes.byref(st)), "mdps_system_stats")
    d = st.as_dict()
    ser = 2 * d["limbs"] * (d["degree"] + 1)
    d["in_doubles"] = d["batch"] * d["n"] * ser
    d["values_doubles"] = d["batch"] * d["n_polys"] * ser
    d["jacobian_doubles"] = d["batch"] * d["n_polys"] * d["n"] * ser
    return d


class System:
    """RAII wrapper: a polynomial system on the device (see libmdps.h)."""

    def __init__(self, poly_ptr, mono_ptr, vars_, exponents, coefficients, n, degree, limbs,
                 algo: int = MDPS_ALGO_AUTO, use_graph: bool = False, real: bool = False, batch: int = 1,
                 schedule: int = MDPS_SCHED_AUTO, workspace_mb: int = 0):
        self.n, self.degree, self.limbs = int(n), int(degree), int(limbs)
        self.n_polys = int(len(poly_ptr) - 1)
        self.batch = int(batch)
        self.handle = mdps_system_create(poly_ptr, mono_ptr, vars_, exponents, coefficients, n,
                                         degree, limbs, algo, use_graph, real, batch, schedule, workspace_mb)
        self.device = _current_device()  # the library allocated on the current device

    @classmethod
    def from_inputs(cls, si, algo: int = MDPS_ALGO_AUTO, use_graph: bool = False, real: bool = False,
                    batch: int = 1, schedule: int = MDPS_SCHED_AUTO, workspace_mb: int = 0) -> "System":
        """From an mdinputs.SystemInputs-like object (poly_ptr, mono_ptr, vars, exps, coeffs)."""
        return cls(si.poly_ptr, si.mono_ptr, si.vars, si.exps, si.coeffs, si.n, si.degree, si.limbs,
                   algo, use_graph, real, batch, schedule, workspace_mb)

    @property
    def series_shape(self):
        return (2, self.limbs, self.degree + 1)

    def eval_diff(self, series_in, values_out=None, jacobian_out=None, stream=None):
        import torch
        lead = (self.batch,) if self.batch > 1 else ()
        if values_out is None:
            values_out = torch.empty(lead + (self.n_polys,) + self.series_shape, dtype=torch.float64,
                                     device=series_in.device)
        if jacobian_out is None:
            jacobian_out = torch.empty(lead + (self.n_polys, self.n) + self.series_shape, dtype=torch.float64,
                                       device=series_in.device)
        mdps_eval_diff(self.handle, series_in, values_out, jacobian_out, stream, self.device)
        return values_out, jacobian_out

    def eval_diff_host(self, series_in: np.ndarray, stream=None):
        lead = (self.batch,) if self.batch > 1 else ()
        vals = np.empty(lead + (self.n_polys,) + self.series_shape)
        jac = np.empty(lead + (self.n_polys, self.n) + self.series_shape)
        mdps_eval_diff_host(self.handle, np.ascontiguousarray(series_in, dtype=np.float64), vals, jac, stream)
        return vals, jac

    def stats(self) -> dict:
        return mdps_system_stats(self.handle)

    def queue_trace(self, enable: Optional[bool] = None, read: bool = False):
        """Job-queue diagnostics (mdps_test_queue_trace): enable/disable the
        per-ticket trace; with read=True return [tickets][5] globaltimer ns
        (claimed, inputs ready, staged, computed, released) of the last evaluation."""
        L = lib()
        en = -1 if enable is None else (1 if enable else 0)
        if not read:
            n = L.mdps_test_queue_trace(self.handle, en, None, 0)
            if n < 0:
                raise MdpsError(mdps_last_error())
            return n
        n = L.mdps_test_queue_trace(self.handle, en, None, 0)
        if n < 0:
            raise MdpsError(mdps_last_error())
        buf = (ctypes.c_int64 * (5 * n))()
        n = L.mdps_test_queue_trace(self.handle, -1, buf, n)
        if n < 0:
            raise MdpsError(mdps_last_error())
        return np.array(buf[:5 * n], dtype=np.int64).reshape(n, 5)

    def level_jobs(self):
        buf = (ctypes.c_int64 * 4096)()
        n = lib().mdps_system_level_jobs(self.handle, buf, 4096)
        if n < 0:
            raise MdpsError(mdps_last_error())
        return list(buf[:n])

    def set_timing(self, enable: bool = True) -> None:
        _check(lib().mdps_system_set_timing(self.handle, 1 if enable else 0), "mdps_system_set_timing")

    def timing(self, reset: bool = True) -> dict:
        t = Timing()
        _check(lib().mdps_system_timing(self.handle, ctypes.byref(t), 1 if reset else 0), "mdps_system_timing")
        return t.as_dict()

    def close(self):
        if getattr(self, "handle", None):
            mdps_system_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Solver:
    """RAII wrapper of the block lower-triangular Toeplitz solver (libmdps.h):
    dx(t) with A(t) dx(t) = b(t) mod t^D, A(t) the n-by-n Jacobian series."""

    def __init__(self, n: int, degree: int, limbs: int, n_eqs: Optional[int] = None):
        self.n, self.degree, self.limbs = int(n), int(degree), int(limbs)
        self.n_eqs = int(n_eqs) if n_eqs is not None else self.n
        self.handle = lib().mdps_solver_create_ls(self.n_eqs, self.n, self.degree, self.limbs)
        if not self.handle:
            raise MdpsError(f"mdps_solver_create failed: {mdps_last_error()}")
        self.device = _current_device()

    def solve(self, jacobian, rhs, dx_out=None, stream=None):
        import torch
        if dx_out is None:
            dx_out = torch.empty((self.n, 2, self.limbs, self.degree + 1), dtype=torch.float64,
                                 device=rhs.device)
        ser = 2 * self.limbs * (self.degree + 1)
        _check(lib().mdps_solve(self.handle, _dptr(jacobian, self.n_eqs * self.n * ser, self.device, "jacobian"),
                                _dptr(rhs, self.n_eqs * ser, self.device, "rhs"),
                                _dptr(dx_out, self.n * ser, self.device, "dx_out"), _stream_handle(stream)),
               "mdps_solve")
        return dx_out

    def newton_step(self, system: "System", x, dx_out=None, norm_out=None, stream=None):
        """x <- x + dx with J dx = -f at x (asynchronous; device tensors)."""
        # sizes from the system (a system/solver shape mismatch is the library's to report)
        nx = system.n * 2 * system.limbs * (system.degree + 1)
        _check(lib().mdps_newton_step(system.handle, self.handle, _dptr(x, nx, system.device, "x"),
                                      _dptr(dx_out, nx, system.device, "dx_out") if dx_out is not None
                                      else None,
                                      _dptr(norm_out, 1, self.device, "norm_out") if norm_out is not None else None,
                                      _stream_handle(stream)),
               "mdps_newton_step")

    def newton(self, system: "System", x, max_iters: int, tol: float, stream=None):
        """Newton's method in place on x; returns (steps, last update norm)."""
        norm = ctypes.c_double(0.0)
        nx = system.n * 2 * system.limbs * (system.degree + 1)
        rc = lib().mdps_newton(system.handle, self.handle, _dptr(x, nx, system.device, "x"), int(max_iters), float(tol), ctypes.byref(norm),
                               _stream_handle(stream))
        if rc < 0:
            raise MdpsError(f"mdps_newton failed (rc={rc}): {mdps_last_error()}")
        return rc, norm.value

    def status(self):
        """(pivots [n] int32, singular bool) of the last solve (synchronises)."""
        piv = np.zeros(self.n, dtype=np.int32)
        sing = ctypes.c_int32(0)
        _check(lib().mdps_solver_status(self.handle, _ptr_i32(piv), ctypes.byref(sing)), "mdps_solver_status")
        return piv, bool(sing.value)

    def flags(self) -> int:
        """Outcome flags of the last solve (synchronises): MDPS_SOLVE_SINGULAR,
        MDPS_SOLVE_NOT_CONVERGED."""
        f = ctypes.c_int32(0)
        _check(lib().mdps_solver_flags(self.handle, ctypes.byref(f)), "mdps_solver_flags")
        return f.value

    def trace(self):
        """(barrier completion times in ns relative to the kernel start, refine steps)."""
        buf = (ctypes.c_int64 * 1024)()
        steps = ctypes.c_int32(0)
        cnt = lib().mdps_solver_trace(self.handle, buf, 1024, ctypes.byref(steps))
        if cnt < 0:
            raise MdpsError(mdps_last_error())
        t = list(buf[:cnt])
        return [x - t[0] for x in t], steps.value

    def stats(self) -> dict:
        st = SolverInfo()
        _check(lib().mdps_solver_stats(self.handle, ctypes.byref(st)), "mdps_solver_stats")
        return st.as_dict()

    def close(self):
        if getattr(self, "handle", None):
            lib().mdps_solver_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


# ---- diagnostic entry points (include/mdps_test.h) -----------------------------
def test_series_mul(x, y, algo: int = MDPS_ALGO_DIGITS, stream=None):
    """z[c] = x[c] * y[c] mod t^D for device tensors [count][2][L][D]."""
    import torch
    z = torch.empty_like(x)
    count, _, L, D = x.shape
    _check(lib().mdps_test_series_mul(_dptr(x), _dptr(y), _dptr(z), count, D - 1, L, algo,
                                      _stream_handle(stream)), "mdps_test_series_mul")
    return z


def test_md_op(op: int, a, b, stream=None):
    import torch
    c = torch.empty_like(a)
    count, L = a.shape
    _check(lib().mdps_test_md_op(op, _dptr(a), _dptr(b), _dptr(c), count, L, _stream_handle(stream)),
           "mdps_test_md_op")
    return c


def test_norm2sq(v, stream=None):
    import torch
    count, _, L = v.shape
    out = torch.empty(L, dtype=torch.float64, device=v.device)
    _check(lib().mdps_test_norm2sq(_dptr(v), count, L, _dptr(out), _stream_handle(stream)), "mdps_test_norm2sq")
    return out


def test_digits_roundtrip(x, stream=None):
    import torch
    y = torch.empty_like(x)
    count, _, L, D = x.shape
    _check(lib().mdps_test_digits_roundtrip(_dptr(x), _dptr(y), count, D - 1, L, _stream_handle(stream)),
           "mdps_test_digits_roundtrip")
    return y


def test_plan(si, eft: bool, batch: int = 1, chunks: int = 1, corrupt: int = 0):
    """Host-only schedule + memory-plan check (mdps_test_plan): returns
    (rc, {unplanned_bytes, planned_bytes, chunks, launches}, message)."""
    pp, mp, vv, ee = _i32(si.poly_ptr), _i32(si.mono_ptr), _i32(si.vars), _i32(si.exps)
    sup = _Supports(len(pp) - 1, _ptr_i32(pp), _ptr_i32(mp), _ptr_i32(vv))
    out = (ctypes.c_int64 * 4)()
    rc = lib().mdps_test_plan(ctypes.byref(sup), _ptr_i32(ee), si.n, si.degree, si.limbs, 1 if eft else 0, batch,
                              chunks, corrupt, out)
    return rc, dict(unplanned_bytes=out[0], planned_bytes=out[1], chunks=out[2], launches=out[3]), mdps_last_error()


def test_balance(si, min_jobs: int, max_levels: int = 256):
    """Host-only level balancing + checks (mdps_test_balance): returns
    (levels or rc < 0, before, after, moved, same_jobs, message)."""
    pp, mp, vv, ee = _i32(si.poly_ptr), _i32(si.mono_ptr), _i32(si.vars), _i32(si.exps)
    sup = _Supports(len(pp) - 1, _ptr_i32(pp), _ptr_i32(mp), _ptr_i32(vv))
    before, after = (ctypes.c_int64 * max_levels)(), (ctypes.c_int64 * max_levels)()
    moved, same = ctypes.c_int64(0), ctypes.c_int32(0)
    rc = lib().mdps_test_balance(ctypes.byref(sup), _ptr_i32(ee), si.n, min_jobs, before, after, max_levels,
                                 ctypes.byref(moved), ctypes.byref(same))
    nl = max(rc, 0)
    return rc, list(before[:nl]), list(after[:nl]), moved.value, same.value, mdps_last_error()


def queue_config(max_blocks: int = 0, lanes: int = 0) -> None:
    """Tuning only: job-queue grid cap and lanes per output pair for systems created afterwards."""
    _check(lib().mdps_test_queue_config(max_blocks, lanes), "mdps_test_queue_config")


def force_geometry(F: int = 0, P: int = 0, NP: int = 0) -> None:
    """Tuning only: force the digit product kernel's (F, P, NP); 0, 0, 0 = the default."""
    _check(lib().mdps_test_force_geometry(F, P, NP), "mdps_test_force_geometry")


def set_pdl(enable: bool = True, small_levels: bool = True, balance: bool = True) -> None:
    """Measurement only: programmatic dependent launch of the digit product levels, the wider
    launch geometry of levels below one wave, and (for systems created afterwards) the level
    balancing of the schedule (all default on)."""
    _check(lib().mdps_test_set_pdl((1 if enable else 0) | (0 if small_levels else 2) | (0 if balance else 4)),
           "mdps_test_set_pdl")


def fp64_peak(iters: int = 20000, stream=None) -> float:
    """Measured FP64 instructions/s (independent DFMA chains on every SM)."""
    out = ctypes.c_double(0.0)
    _check(lib().mdps_fp64_peak(iters, ctypes.byref(out), _stream_handle(stream)), "mdps_fp64_peak")
    return out.value
