"""Seeded synthetic inputs for mdps_eval_diff — shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no series products, no
multiple-double operations): it only draws random numbers and lays them out.
Both sides of every parity test consume exactly the arrays built here.

Recipe:

* Random streams: counter-based splitmix64, one stream per (seed, purpose),
  purposes "structure", "x" and "c".  BASELINE.json config i uses seed i+1.
* Structure (C2.11): per polynomial, `monos` monomials; each monomial has m
  distinct variables, m uniform on the config's inclusive range, drawn
  without replacement (partial Fisher-Yates) and sorted ascending; exponents
  uniform on the config's set.  A monomial equal (support and exponents) to an
  earlier one in the same polynomial is redrawn.
* Data (BASELINE.json configs; PAPER.md:82-85 for cos(theta)+i sin(theta)):
  every coefficient of every series (inputs x_j and monomial coefficients c_r)
  is cos(theta) + i sin(theta), theta = 2*pi*u, u from 53 random bits; the
  leading limb is the libm value.  Lower limbs (C2.12): "zero" -> 0;
  "random" -> limb_j = RN(r_j * 0.99 * ulpdown(limb_{j-1}) / 2), r_j uniform
  on [-1, 1), which is already a canonical (greedy round-to-nearest)
  non-overlapping expansion, so truncating it to fewer limbs equals rounding
  it to fewer limbs (the sweep relies on this).

Layout: series arrays are float64 [count][2][L][D] —
part (0 = re, 1 = im), limb (0 = most significant), coefficient k = 0..d.
"""
from __future__ import annotations

import dataclasses
import hashlib
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "CONFIGS", "SystemInputs", "SplitMix64", "make_config", "make_system",
    "sweep_cell", "unit_circle_series", "structure_from_monomials",
]

_MASK = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15
_PURPOSE = {"structure": 1, "x": 2, "c": 3, "extra": 4, "jac": 5, "rhs": 6}


def _mix64(z: int) -> int:
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9 & _MASK
    z = (z ^ (z >> 27)) * 0x94D049BB133111EB & _MASK
    return z ^ (z >> 31)


def _mix64_np(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


class SplitMix64:
    """Counter-based splitmix64 stream keyed by (seed, purpose).

    Output i is mix64(key + (i+1)*GAMMA); `take(n)` returns the next n outputs
    as uint64 (vectorised), `next()` one Python int.
    """

    def __init__(self, seed: int, purpose: str):
        self.key = _mix64((seed * 0x2545F4914F6CDD1D + _PURPOSE[purpose] * _GAMMA) & _MASK)
        self.counter = 0

    def next(self) -> int:
        self.counter += 1
        return _mix64((self.key + self.counter * _GAMMA) & _MASK)

    def take(self, n: int) -> np.ndarray:
        idx = np.arange(self.counter + 1, self.counter + 1 + n, dtype=np.uint64)
        self.counter += n
        with np.errstate(over="ignore"):
            z = np.uint64(self.key) + idx * np.uint64(_GAMMA)
        return _mix64_np(z)

    def below(self, bound: int) -> int:
        """Uniform integer in [0, bound) (multiply-shift, bias < 2^-56)."""
        return (self.next() * bound) >> 64

    def uniform53(self, n: int) -> np.ndarray:
        """n doubles u in [0, 1) from the top 53 bits of each output."""
        return (self.take(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    monos: int
    m_range: Tuple[int, int]
    exps: Tuple[int, ...]
    degree: int
    limbs: int
    lower: str          # "zero" | "random"
    seed: int


# BASELINE.json "configs" (0-based index i uses seed i+1).
CONFIGS = {
    "dd": Config("dd", 8, 16, (3, 3), (1,), 15, 2, "zero", 1),
    "qd": Config("qd", 32, 64, (4, 8), (1, 2), 31, 4, "random", 2),
    "od": Config("od", 64, 128, (8, 16), (1,), 63, 8, "random", 3),
    "deca": Config("deca", 128, 128, (16, 16), (1,), 63, 10, "random", 4),
    # the sweep's fixed system is generated once at its largest cell
    "sweep": Config("sweep", 64, 64, (8, 8), (1,), 127, 10, "random", 5),
}
SWEEP_DEGREES = (15, 31, 63, 127)
SWEEP_LIMBS = (2, 3, 4, 5, 8, 10)


@dataclasses.dataclass
class SystemInputs:
    """One eval/diff problem: structure (CSR), coefficients and the point x."""
    name: str
    n: int
    degree: int
    limbs: int
    poly_ptr: np.ndarray   # int32 [n+1]
    mono_ptr: np.ndarray   # int32 [M+1]
    vars: np.ndarray       # int32 [nnz]
    exps: np.ndarray       # int32 [nnz]
    coeffs: np.ndarray     # float64 [M][2][L][D]
    x: np.ndarray          # float64 [n][2][L][D]

    @property
    def D(self) -> int:
        return self.degree + 1

    @property
    def M(self) -> int:
        return int(self.mono_ptr.shape[0] - 1)

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (self.poly_ptr, self.mono_ptr, self.vars, self.exps, self.coeffs, self.x):
            h.update(np.ascontiguousarray(a).tobytes())
        h.update(f"{self.n},{self.degree},{self.limbs}".encode())
        return h.hexdigest()


def _lower_limbs(lead: np.ndarray, limbs: int, rule: str, rng: SplitMix64) -> np.ndarray:
    """Stack [.., limbs] of a canonical expansion whose leading limb is `lead`."""
    out = np.zeros(lead.shape + (limbs,), dtype=np.float64)
    out[..., 0] = lead
    if rule == "zero" or limbs == 1:
        return out
    assert rule == "random"
    prev = lead
    for j in range(1, limbs):
        r = rng.uniform53(prev.size).reshape(prev.shape) * 2.0 - 1.0
        a = np.abs(prev)
        ulpdown = a - np.nextafter(a, 0.0)
        limb = r * 0.99 * (ulpdown * 0.5)
        limb = np.where(a > 0, limb, 0.0)
        out[..., j] = limb
        prev = limb
    return out


def unit_circle_series(rng: SplitMix64, count: int, D: int, L: int, lower: str) -> np.ndarray:
    """`count` series of D coefficients cos(theta)+i sin(theta), L limbs each.

    Returns float64 [count][2][L][D].
    """
    theta = rng.uniform53(count * D).reshape(count, D) * (2.0 * math.pi)
    re = _lower_limbs(np.cos(theta), L, lower, rng)   # [count][D][L]
    im = _lower_limbs(np.sin(theta), L, lower, rng)
    out = np.stack([re, im], axis=1)                   # [count][2][D][L]
    return np.ascontiguousarray(out.transpose(0, 1, 3, 2))


def structure_from_monomials(n: int, polys: Sequence[Sequence[Sequence[Tuple[int, int]]]]):
    """CSR arrays from polys[i] = list of monomials, each a list of (var, exp)."""
    poly_ptr, mono_ptr, vars_, exps = [0], [0], [], []
    for poly in polys:
        for mono in poly:
            for v, a in mono:
                vars_.append(v)
                exps.append(a)
            mono_ptr.append(len(vars_))
        poly_ptr.append(len(mono_ptr) - 1)
    assert len(poly_ptr) == n + 1
    return (np.asarray(poly_ptr, np.int32), np.asarray(mono_ptr, np.int32),
            np.asarray(vars_, np.int32), np.asarray(exps, np.int32))


def _draw_structure(cfg: Config, rng: SplitMix64):
    polys = []
    lo, hi = cfg.m_range
    for _ in range(cfg.n):
        seen = set()
        poly = []
        while len(poly) < cfg.monos:
            m = lo + rng.below(hi - lo + 1)
            pool = list(range(cfg.n))
            for j in range(m):  # partial Fisher-Yates: m distinct variables
                r = j + rng.below(cfg.n - j)
                pool[j], pool[r] = pool[r], pool[j]
            support = sorted(pool[:m])
            mono = tuple((v, cfg.exps[rng.below(len(cfg.exps))]) for v in support)
            if mono in seen:      # C2.11: redraw a duplicate monomial
                continue
            seen.add(mono)
            poly.append(list(mono))
        polys.append(poly)
    return structure_from_monomials(cfg.n, polys)


_CACHE = {}


def make_config(name: str) -> SystemInputs:
    """The full BASELINE.json config `name` (dd, qd, od, deca, sweep@D=128,L=10)."""
    if name in _CACHE:
        return _CACHE[name]
    cfg = CONFIGS[name]
    si = make_system(cfg)
    _CACHE[name] = si
    return si


def make_system(cfg: Config) -> SystemInputs:
    poly_ptr, mono_ptr, vars_, exps = _draw_structure(cfg, SplitMix64(cfg.seed, "structure"))
    D = cfg.degree + 1
    M = len(mono_ptr) - 1
    coeffs = unit_circle_series(SplitMix64(cfg.seed, "c"), M, D, cfg.limbs, cfg.lower)
    x = unit_circle_series(SplitMix64(cfg.seed, "x"), cfg.n, D, cfg.limbs, cfg.lower)
    return SystemInputs(cfg.name, cfg.n, cfg.degree, cfg.limbs, poly_ptr, mono_ptr,
                        vars_, exps, coeffs, x)


def truncate(si: SystemInputs, degree: int, limbs: int, name: Optional[str] = None) -> SystemInputs:
    """Same system at a lower degree / fewer limbs (truncation == rounding, see above)."""
    assert degree <= si.degree and limbs <= si.limbs
    D = degree + 1
    return SystemInputs(name or f"{si.name}_d{degree}_L{limbs}", si.n, degree, limbs,
                        si.poly_ptr, si.mono_ptr, si.vars, si.exps,
                        np.ascontiguousarray(si.coeffs[:, :, :limbs, :D]),
                        np.ascontiguousarray(si.x[:, :, :limbs, :D]))


def realify(si: SystemInputs, name: Optional[str] = None) -> SystemInputs:
    """The same system with every imaginary limb set to 0 (a real system:
    coefficients cos(theta), inputs cos(theta) with their lower limbs)."""
    c, x = si.coeffs.copy(), si.x.copy()
    c[:, 1] = 0.0
    x[:, 1] = 0.0
    return dataclasses.replace(si, name=name or f"{si.name}_real", coeffs=c, x=x)


def sweep_cell(degree: int, limbs: int) -> SystemInputs:
    """One cell of config 4 (the precision sweep), derived from the fixed system."""
    assert degree in SWEEP_DEGREES and limbs in SWEEP_LIMBS
    return truncate(make_config("sweep"), degree, limbs, f"sweep_d{degree}_L{limbs}")


def subsystem(si: SystemInputs, rows: Sequence[int], name: Optional[str] = None) -> SystemInputs:
    """The polynomials `rows` of si (same variables and x), as a system with
    len(rows) polynomials — used to bound oracle work on sampled rows."""
    polys = []
    for i in rows:
        poly = []
        for r in range(si.poly_ptr[i], si.poly_ptr[i + 1]):
            a, b = si.mono_ptr[r], si.mono_ptr[r + 1]
            poly.append(list(zip(si.vars[a:b].tolist(), si.exps[a:b].tolist())))
        polys.append(poly)
    pp, mp, vv, ee = structure_from_monomials(len(rows), polys)
    monos = np.concatenate([np.arange(si.poly_ptr[i], si.poly_ptr[i + 1]) for i in rows]).astype(np.int64)
    return SystemInputs(name or f"{si.name}_rows", si.n, si.degree, si.limbs, pp, mp, vv, ee,
                        np.ascontiguousarray(si.coeffs[monos]), si.x)


def rect_system(seed: int, N: int, n: int, monos: int, m_range: Tuple[int, int], exps: Tuple[int, ...],
                degree: int, limbs: int, lower: str = "random") -> SystemInputs:
    """N polynomials in n variables (N != n allowed), same recipe as the configs."""
    rng = SplitMix64(seed, "structure")
    pp, mp, vv, ee = [0], [0], [], []
    lo, hi = m_range
    for _ in range(N):
        for _ in range(monos):
            m = min(n, lo + rng.below(hi - lo + 1))
            pool = list(range(n))
            for j in range(m):
                r = j + rng.below(n - j)
                pool[j], pool[r] = pool[r], pool[j]
            for v in sorted(pool[:m]):
                vv.append(v)
                ee.append(exps[rng.below(len(exps))])
            mp.append(len(vv))
        pp.append(len(mp) - 1)
    D = degree + 1
    M = len(mp) - 1
    coeffs = unit_circle_series(SplitMix64(seed, "c"), M, D, limbs, lower)
    x = unit_circle_series(SplitMix64(seed, "x"), n, D, limbs, lower)
    return SystemInputs(f"rect{seed}_{N}x{n}", n, degree, limbs, np.asarray(pp, np.int32), np.asarray(mp, np.int32),
                        np.asarray(vv, np.int32), np.asarray(ee, np.int32), coeffs, x)


def random_system(seed: int, n: int, monos: int, m_range: Tuple[int, int], exps: Tuple[int, ...],
                  degree: int, limbs: int, lower: str = "random") -> SystemInputs:
    """A small seeded random system in the same recipe (tests)."""
    cfg = Config(f"rand{seed}", n, monos, m_range, exps, degree, limbs, lower, seed)
    return make_system(cfg)


def first_entries(si: SystemInputs, count: int):
    """A deterministic bounded sample of outputs: (0, -1) = f_0, then the
    nonzero Jacobian entries of row 0, then of row 1, ... (`count` in all)."""
    out = [(0, -1)]
    n_polys = len(si.poly_ptr) - 1
    for i in range(n_polys):
        cols = sorted({int(v) for r in range(si.poly_ptr[i], si.poly_ptr[i + 1])
                       for v in si.vars[si.mono_ptr[r]:si.mono_ptr[r + 1]]})
        for j in cols:
            if len(out) >= count:
                return out
            out.append((i, j))
    return out[:count]


# ---------------------------------------------------------------------------
# Block lower-triangular Toeplitz systems (the linear solve of a Newton step,
# PAPER.md:266-333).  Recipe: a dense n-by-n matrix
# of series J and a right-hand side b(t), every coefficient of every series
# cos(theta) + i sin(theta) with the lower-limb rule of the config — the
# distribution of the configs' own data, at the configs' n, degree and limbs.
@dataclasses.dataclass
class ToeplitzInputs:
    name: str
    n: int
    degree: int
    limbs: int
    jac: np.ndarray   # float64 [n][n][2][L][D]
    rhs: np.ndarray   # float64 [n][2][L][D]

    @property
    def D(self) -> int:
        return self.degree + 1

    def truncate(self, degree: int) -> "ToeplitzInputs":
        D = degree + 1
        return ToeplitzInputs(f"{self.name}_d{degree}", self.n, degree, self.limbs,
                              np.ascontiguousarray(self.jac[..., :D]), np.ascontiguousarray(self.rhs[..., :D]))


def random_toeplitz(seed: int, n: int, degree: int, limbs: int, lower: str = "random",
                    name: Optional[str] = None) -> ToeplitzInputs:
    D = degree + 1
    jac = unit_circle_series(SplitMix64(seed, "jac"), n * n, D, limbs, lower).reshape(n, n, 2, limbs, D)
    rhs = unit_circle_series(SplitMix64(seed, "rhs"), n, D, limbs, lower)
    return ToeplitzInputs(name or f"toeplitz{seed}_n{n}_d{degree}_L{limbs}", n, degree, limbs,
                          np.ascontiguousarray(jac), rhs)


def random_toeplitz_rect(seed: int, N: int, n: int, degree: int, limbs: int, lower: str = "random",
                         name: Optional[str] = None) -> ToeplitzInputs:
    """N >= n equations (least squares): jac [N][n][2][L][D], rhs [N][2][L][D]."""
    D = degree + 1
    jac = unit_circle_series(SplitMix64(seed, "jac"), N * n, D, limbs, lower).reshape(N, n, 2, limbs, D)
    rhs = unit_circle_series(SplitMix64(seed, "rhs"), N, D, limbs, lower)
    return ToeplitzInputs(name or f"toeplitz{seed}_{N}x{n}_d{degree}_L{limbs}", n, degree, limbs,
                          np.ascontiguousarray(jac), rhs)


def toeplitz_config(name: str) -> ToeplitzInputs:
    """The solve that follows config `name`'s eval/diff: its n, degree, limbs,
    lower-limb rule and seed (sweep: its largest cell)."""
    key = ("toeplitz", name)
    if key not in _CACHE:
        cfg = CONFIGS[name]
        _CACHE[key] = random_toeplitz(cfg.seed, cfg.n, cfg.degree, cfg.limbs, cfg.lower, f"toeplitz_{name}")
    return _CACHE[key]
