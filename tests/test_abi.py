"""The C-ABI library builds for sm_100a, loads without a GPU, exports every
symbol include/*.h declares, and validates its arguments on the host
(create returns NULL with a message, no CUDA call is made)."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

import paper_2012_06607_b200 as mdps
from paper_2012_06607_b200 import build as mdps_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    mdps_build.build()
    return mdps.lib()


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b(mdps_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert {"mdps_system_create", "mdps_eval_diff", "mdps_system_destroy", "mdps_last_error"} <= names
    for name in names:
        assert hasattr(lib, name), name
    assert names == set(mdps.EXPORTED_SYMBOLS)


def test_sm100a_code_in_library(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", mdps.library_path],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _create(**kw):
    args = dict(poly_ptr=[0, 1, 1], mono_ptr=[0, 2], vars_=[0, 1], exponents=[1, 1],
                coefficients=np.zeros((1, 2, 2, 4)), n=2, degree=3, limbs=2)
    args.update(kw)
    return mdps.mdps_system_create(**args)


@pytest.mark.parametrize("kw,msg", [
    (dict(n=0), "n must be"),
    (dict(limbs=7), "limbs"),
    (dict(degree=-1), "degree"),
    (dict(poly_ptr=[0]), "n_polys"),
    (dict(poly_ptr=[0, 1, 0]), "non-decreasing"),
    (dict(mono_ptr=[0, 3], vars_=[0, 1, 1], exponents=[1, 1, 1]), "repeated"),
    (dict(vars_=[0, 2]), "out of range"),
    (dict(exponents=[1, 0]), "exponent"),
    (dict(algo=9), "algo"),
    (dict(degree=200, algo=2), "degree"),
])
def test_create_rejects_invalid_arguments(lib, kw, msg):
    with pytest.raises(mdps.MdpsError, match=msg):
        _create(**kw)


def test_null_handles_are_rejected(lib):
    assert lib.mdps_eval_diff(None, None, None, None, None) == mdps.MDPS_EINVAL
    assert "NULL" in mdps.mdps_last_error()
    assert lib.mdps_system_stats(None, None) == mdps.MDPS_EINVAL
    lib.mdps_system_destroy(None)  # no-op


def test_product_path_has_no_oracle_or_fallback():
    """the product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2012_06607_b200")
    for f in glob.glob(os.path.join(pkg, "**", "*"), recursive=True):
        if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
            src = open(f).read()
            assert "oracle" not in src.replace("CPU oracle (oracle/)", "").replace("oracle/)", ""), f


@pytest.mark.parametrize("n,degree,limbs", [(0, 3, 2), (129, 3, 2), (4, -1, 2), (4, 300, 2), (4, 3, 7)])
def test_solver_create_rejects_invalid_arguments(lib, n, degree, limbs):
    with pytest.raises(mdps.MdpsError, match="mdps_solver_create"):
        mdps.Solver(n, degree, limbs)


def test_solver_null_handles_are_rejected(lib):
    assert lib.mdps_solve(None, None, None, None, None) == mdps.MDPS_EINVAL
    assert lib.mdps_solver_status(None, None, None) == mdps.MDPS_EINVAL
    assert lib.mdps_solver_stats(None, None) == mdps.MDPS_EINVAL
    lib.mdps_solver_destroy(None)  # no-op
