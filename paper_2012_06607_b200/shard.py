"""Row sharding of a polynomial system over GPUs.

The polynomials (rows) of a system are independent: each needs all of x but
writes only its own value and Jacobian row ("one job is
concerned with one polynomial").  A system is split into row subsets
balanced by their product-job counts (longest-processing-time greedy); each
rank creates an mdps system with only its rows (N < n, libmdps.h) and the same
x, so no data moves between GPUs during an evaluation.  Host-side integer
work only (no arithmetic of the method).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def row_products(poly_ptr, mono_ptr, exps) -> List[int]:
    """Product jobs per row: 3(m-1) + w for m >= 2 variables, 1 + w for m = 1,
    0 for a constant, w = sum(a_l - 1) (the schedule's count)."""
    poly_ptr, mono_ptr, exps = (np.asarray(a, dtype=np.int64) for a in (poly_ptr, mono_ptr, exps))
    out = []
    for i in range(len(poly_ptr) - 1):
        c = 0
        for r in range(poly_ptr[i], poly_ptr[i + 1]):
            a, b = mono_ptr[r], mono_ptr[r + 1]
            m = int(b - a)
            w = int((exps[a:b] - 1).sum())
            c += 0 if m == 0 else (w + 1 if m == 1 else 3 * (m - 1) + w)
        out.append(c)
    return out


def partition_rows(costs: Sequence[int], parts: int) -> List[List[int]]:
    """Rows split into `parts` subsets: rows by decreasing cost (then index),
    each to the currently lightest subset (lowest index on ties).  Deterministic,
    every row exactly once; each subset sorted ascending."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-int(costs[i]), i))
    load = [0] * parts
    rows: List[List[int]] = [[] for _ in range(parts)]
    for i in order:
        p = min(range(parts), key=lambda q: (load[q], q))
        rows[p].append(i)
        load[p] += int(costs[i])
    return [sorted(r) for r in rows]


def subsystem(poly_ptr, mono_ptr, vars_, exps, coeffs, rows: Sequence[int]) -> Tuple[np.ndarray, ...]:
    """CSR arrays and coefficient series of the polynomials `rows` (same n
    variables): (poly_ptr, mono_ptr, vars, exps, coeffs)."""
    poly_ptr, mono_ptr = np.asarray(poly_ptr), np.asarray(mono_ptr)
    vars_, exps = np.asarray(vars_), np.asarray(exps)
    pp, mp, vv, ee, monos = [0], [0], [], [], []
    for i in rows:
        for r in range(int(poly_ptr[i]), int(poly_ptr[i + 1])):
            a, b = int(mono_ptr[r]), int(mono_ptr[r + 1])
            vv.extend(vars_[a:b].tolist())
            ee.extend(exps[a:b].tolist())
            mp.append(len(vv))
            monos.append(r)
        pp.append(len(mp) - 1)
    cc = np.ascontiguousarray(np.asarray(coeffs)[np.asarray(monos, dtype=np.int64)]) if monos else \
        np.zeros((0,) + np.asarray(coeffs).shape[1:])
    return (np.asarray(pp, np.int32), np.asarray(mp, np.int32), np.asarray(vv, np.int32),
            np.asarray(ee, np.int32), cc)
