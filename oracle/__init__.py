"""oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct float64 CPU reference ("oracle") for the
cascadic-multigrid Fiedler solver of Gandhi, arXiv 1602.04386.
The loops live in ``fiedler_oracle.c`` (single-threaded, -ffp-contract=off);
this module only marshals numpy arrays and walks Algorithm 3 level by level in
the paper's order.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the CUDA product path (``paper_1602_04386_b200``) and
never imports it.

Parity status: every public function here is pinned
by a ``-m "not gpu"`` test in ``tests/test_oracle_pins.py`` against closed
forms, dense linear algebra, hand traces or brute force.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fiedler_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

# Tags of the counter-based generator (reading R6).
TAG_MATCH = 0x6D61746368000000
TAG_COLOR = 0x636F6C6F72000000
MASK64 = (1 << 64) - 1


def build(force: bool = False) -> str:
    """Compile fiedler_oracle.c into liboracle.so (gcc, -O2, no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               "-ffp-contract=off", "-fno-fast-math",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, u64, i32, f64 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_double
        sig = {
            "orc_splitmix64": (u64, [u64]),
            "orc_rand_uniform": (None, [i64, u64, P]),
            "orc_randperm": (None, [i64, u64, i64, P]),
            "orc_degrees": (None, [i64, P, P, P, P]),
            "orc_laplacian_matvec": (None, [i64, P, P, P, P, P, P]),
            "orc_quadratic_form": (f64, [i64, P, P, P, P]),
            "orc_rayleigh": (f64, [i64, P, P, P, P]),
            "orc_deflate": (None, [i64, P]),
            "orc_normalize": (ctypes.c_int, [i64, P]),
            "orc_hec_sequential": (i64, [i64, P, P, P, P, P]),
            "orc_hec_parallel": (i64, [i64, P, P, P, u64, P, P]),
            "orc_galerkin": (i64, [i64, P, P, P, P, i64, P, P, P]),
            "orc_greedy_coloring": (i32, [i64, P, P, u64, P]),
            "orc_gs_solve": (i64, [i64, P, P, P, P, P, f64, i64]),
            "orc_gs_sweeps": (None, [i64, P, P, P, P, P, P, i64]),
            "orc_power_iterations": (ctypes.c_int, [i64, P, P, P, P, f64, P, i64, P]),
            "orc_prolongate": (None, [i64, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Graph:
    """Weighted adjacency W of G=(V,E,w) in CSR; L = D - W."""
    n: int
    rp: np.ndarray   # int64[n+1]
    ci: np.ndarray   # int32[nnz], ascending per row, no self loops
    w: np.ndarray    # float64[nnz], > 0, symmetric bit-for-bit

    @staticmethod
    def from_csr(n, rp, ci, w) -> "Graph":
        return Graph(int(n), np.ascontiguousarray(rp, dtype=np.int64),
                     np.ascontiguousarray(ci, dtype=np.int32),
                     np.ascontiguousarray(w, dtype=np.float64))

    @property
    def nnz(self) -> int:
        return int(self.rp[-1])

    def args(self):
        return (self.n, _p(self.rp), _p(self.ci), _p(self.w))


# ---------------------------------------------------------------- primitives

def splitmix64(x: int) -> int:
    return int(_L().orc_splitmix64(x & MASK64))


def salt_match(seed: int, level: int) -> int:
    return splitmix64((seed ^ (TAG_MATCH + level)) & MASK64)


def salt_color(seed: int, level: int) -> int:
    return splitmix64((seed ^ (TAG_COLOR + level)) & MASK64)


def rand_uniform(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    _L().orc_rand_uniform(n, seed & MASK64, _p(out))
    return out


def randperm(n: int, seed: int, level: int) -> np.ndarray:
    p = np.empty(n, dtype=np.int64)
    _L().orc_randperm(n, seed & MASK64, level, _p(p))
    return p


def degrees(g: Graph) -> np.ndarray:
    d = np.empty(g.n, dtype=np.float64)
    _L().orc_degrees(*g.args(), _p(d))
    return d


def laplacian_matvec(g: Graph, x: np.ndarray, d: Optional[np.ndarray] = None) -> np.ndarray:
    d = degrees(g) if d is None else d
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(g.n, dtype=np.float64)
    _L().orc_laplacian_matvec(*g.args(), _p(d), _p(x), _p(y))
    return y


def quadratic_form(g: Graph, x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(_L().orc_quadratic_form(*g.args(), _p(x)))


def rayleigh(g: Graph, x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return float(_L().orc_rayleigh(*g.args(), _p(x)))


def deflate(x: np.ndarray) -> np.ndarray:
    x = np.array(x, dtype=np.float64, copy=True)
    _L().orc_deflate(x.size, _p(x))
    return x


def normalize(x: np.ndarray) -> np.ndarray:
    x = np.array(x, dtype=np.float64, copy=True)
    if not _L().orc_normalize(x.size, _p(x)):
        raise ValueError("zero vector cannot be normalised")
    return x


def hec_sequential(g: Graph, p: np.ndarray):
    """Algorithm 1 verbatim with visiting order p (0-based). Returns (q, c)."""
    p = np.ascontiguousarray(p, dtype=np.int64)
    q = np.empty(g.n, dtype=np.int64)
    c = _L().orc_hec_sequential(*g.args(), _p(p), _p(q))
    return q, int(c)


def hec_parallel(g: Graph, salt: int):
    """Parallel-order heavy edge coarsening (reading R2). Returns (q, c, mate)."""
    q = np.empty(g.n, dtype=np.int64)
    mate = np.empty(g.n, dtype=np.int64)
    c = _L().orc_hec_parallel(*g.args(), salt & MASK64, _p(mate), _p(q))
    if c < 0:
        raise RuntimeError("orc_hec_parallel failed (%d)" % c)
    return q, int(c), mate


def galerkin(g: Graph, q: np.ndarray, c: int) -> Graph:
    """Coarse adjacency of I L I^T (Algorithm 3 line 5) with the R3 summation order."""
    q = np.ascontiguousarray(q, dtype=np.int64)
    crp = np.empty(c + 1, dtype=np.int64)
    cap = max(g.nnz, 1)
    cci = np.empty(cap, dtype=np.int32)
    cw = np.empty(cap, dtype=np.float64)
    nnz = _L().orc_galerkin(*g.args(), _p(q), c, _p(crp), _p(cci), _p(cw))
    if nnz < 0:
        raise MemoryError("orc_galerkin")
    return Graph(c, crp, cci[:nnz].copy(), cw[:nnz].copy())


def greedy_coloring(g: Graph, salt: int):
    color = np.empty(g.n, dtype=np.int32)
    ncol = _L().orc_greedy_coloring(g.n, _p(g.rp), _p(g.ci), salt & MASK64, _p(color))
    return color, int(ncol)


def color_order(color: np.ndarray) -> np.ndarray:
    """Sweep order of the multicolour Gauss-Seidel: by (colour, vertex index)."""
    return np.lexsort((np.arange(color.size), color)).astype(np.int64)


def gs_solve(n, rp, ci, a, b, x0, tol, N):
    """Algorithm 2 on a general CSR matrix (with diagonal). Returns (x, sweeps)."""
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    k = _L().orc_gs_solve(n, _p(rp), _p(ci), _p(a), _p(b), _p(x), float(tol), int(N))
    if k < 0:
        raise ZeroDivisionError("zero diagonal entry")
    return x, int(k)


def gs_sweeps(g: Graph, x: np.ndarray, sweeps: int, order: Optional[np.ndarray] = None,
              d: Optional[np.ndarray] = None) -> np.ndarray:
    d = degrees(g) if d is None else d
    order = np.arange(g.n, dtype=np.int64) if order is None else np.ascontiguousarray(order, dtype=np.int64)
    x = np.array(x, dtype=np.float64, copy=True)
    _L().orc_gs_sweeps(*g.args(), _p(d), _p(order), _p(x), int(sweeps))
    return x


def power_iterations(g: Graph, x: np.ndarray, iters: int, shift: float,
                     d: Optional[np.ndarray] = None) -> np.ndarray:
    d = degrees(g) if d is None else d
    x = np.array(x, dtype=np.float64, copy=True)
    work = np.empty(g.n, dtype=np.float64)
    if not _L().orc_power_iterations(*g.args(), _p(d), float(shift), _p(x), int(iters), _p(work)):
        raise ValueError("power iteration collapsed to the zero vector")
    return x


def prolongate(q: np.ndarray, yc: np.ndarray) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.int64)
    yc = np.ascontiguousarray(yc, dtype=np.float64)
    yf = np.empty(q.size, dtype=np.float64)
    _L().orc_prolongate(q.size, _p(q), _p(yc), _p(yf))
    return yf


def shift_of(d: np.ndarray) -> float:
    """Shift c of c I - L: Gershgorin bound 2 max_i d_i >= lambda_max (reading R8).
    On a 2-vertex level (K2) the bound is attained, 2 max d = lambda_max, and
    c I - L would map the only non-constant direction -- the Fiedler vector --
    to zero; there c = 3 max d (R8)."""
    if not d.size:
        return 0.0
    return (3.0 if d.size == 2 else 2.0) * float(d.max())


def sign_fix(v: np.ndarray) -> np.ndarray:
    """Make the first nonzero entry positive (north-star sign convention)."""
    nz = np.flatnonzero(v)
    if nz.size and v[nz[0]] < 0:
        return -v
    return v


# ---------------------------------------------------------------- Algorithm 3

@dataclass
class Config:
    coarsest_size: int = 25          # "While n_i > 25"
    max_levels: int = 50
    gs_sweeps: int = 2               # BASELINE.json configs: 2 sweeps per level
    power_iters: int = 10            # BASELINE.json configs: 10 power iterations per level
    coarsest_power_iters: Optional[int] = None   # None -> power_iters
    seed: int = 0
    mode: str = "parallel"           # "parallel" (GPU order) or "sequential" (paper order)
    stall_ratio: float = 0.95        # reading R9


@dataclass
class Level:
    g: Graph
    q: Optional[np.ndarray] = None         # fine -> coarse map to level+1
    c: int = 0
    mate: Optional[np.ndarray] = None
    d: Optional[np.ndarray] = None
    shift: float = 0.0
    color: Optional[np.ndarray] = None
    ncolors: int = 0
    order: Optional[np.ndarray] = None


def build_hierarchy(g: Graph, cfg: Config = Config()) -> List[Level]:
    """Algorithm 3 Step 1, Setup Phase."""
    levels = [Level(g)]
    while levels[-1].g.n > cfg.coarsest_size and len(levels) < cfg.max_levels:
        L = levels[-1]
        ell = len(levels) - 1
        if cfg.mode == "parallel":
            q, c, mate = hec_parallel(L.g, salt_match(cfg.seed, ell))
        elif cfg.mode == "sequential":
            q, c = hec_sequential(L.g, randperm(L.g.n, cfg.seed, ell))
            mate = None
        else:
            raise ValueError(cfg.mode)
        if c > cfg.stall_ratio * L.g.n or c < 2:     # stall guard / no 1-vertex level (R9)
            break
        L.q, L.c, L.mate = q, c, mate
        levels.append(Level(galerkin(L.g, q, c)))
    for ell, L in enumerate(levels):
        L.d = degrees(L.g)
        L.shift = shift_of(L.d)
        if cfg.mode == "parallel":
            L.color, L.ncolors = greedy_coloring(L.g, salt_color(cfg.seed, ell))
            L.order = color_order(L.color)
        else:
            L.order = np.arange(L.g.n, dtype=np.int64)
    return levels


@dataclass
class Result:
    vector: np.ndarray
    lambda2: float
    residual_norm: float
    levels: List[Level] = field(default_factory=list)


def smooth_level(L: Level, y: np.ndarray, cfg: Config) -> np.ndarray:
    """One cascadic level: GS(L^j, y) then the shifted power
    iteration, with deflation + normalisation (reading R5)."""
    y = gs_sweeps(L.g, y, cfg.gs_sweeps, L.order, L.d)
    y = normalize(deflate(y))
    return power_iterations(L.g, y, cfg.power_iters, L.shift, L.d)


def solve(g: Graph, cfg: Config = Config(), levels: Optional[List[Level]] = None) -> Result:
    """Algorithm 3 followed by the Rayleigh quotient."""
    if g.n < 2:
        raise ValueError("need n >= 2")
    levels = build_hierarchy(g, cfg) if levels is None else levels
    J = len(levels) - 1
    # Step 2 (reading R5): "A direct power iteration is used at this coarsest
    # level" from rand(n_J).
    LJ = levels[J]
    y = normalize(deflate(rand_uniform(LJ.g.n, cfg.seed)))
    kJ = cfg.power_iters if cfg.coarsest_power_iters is None else cfg.coarsest_power_iters
    y = power_iterations(LJ.g, y, kJ, LJ.shift, LJ.d)
    for j in range(J - 1, -1, -1):                                    # Step 3
        y = normalize(deflate(prolongate(levels[j].q, y)))
        y = smooth_level(levels[j], y, cfg)
    y = sign_fix(y)
    lam = rayleigh(g, y)
    r = laplacian_matvec(g, y, levels[0].d) - lam * y
    return Result(y, lam, float(np.sqrt(np.dot(r, r))), levels)
