"""graphgen -- seeded synthetic graph generators shared by the oracle side and
the GPU side (task rule 3: "only the seeded input generators serve both, from
a module of their own that holds none of the method's arithmetic").

Every generator returns a :class:`CSRGraph`: the weighted adjacency matrix W of
an undirected graph G=(V,E,w) in CSR with int64 row offsets,
int32 column indices sorted ascending within each row, float64 weights > 0,
no self loops, and w_ij == w_ji bit-for-bit.  Nothing here computes anything
of the paper's method (no Laplacian, coarsening, smoothing or eigen-work).

Recipes follow BASELINE.json "configs":
  * grid2d(m, ...)   -- m x m 4-neighbour lattice ("uniform square arrays")
  * grid3d(m, ...)   -- m^3 6-neighbour lattice
  * rmat(scale, ...) -- R-MAT power-law graph, symmetrised, largest component
  * small analytic families (path, cycle, star, complete) and random
    connected graphs for the oracle pins.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class CSRGraph:
    n: int
    rp: np.ndarray   # int64 [n+1]
    ci: np.ndarray   # int32 [nnz]
    w: np.ndarray    # float64 [nnz]
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.rp[-1])

    @property
    def num_edges(self) -> int:
        return self.nnz // 2


def csr_from_edges(n: int, u, v, w, name: str = "") -> CSRGraph:
    """Symmetric CSR from an undirected edge list with u != v and no duplicate
    pairs (callers dedupe).  Rows sorted by column."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    if u.size and (np.any(u == v) or u.min() < 0 or v.min() < 0 or max(u.max(), v.max()) >= n):
        raise ValueError("bad edge list")
    if np.any(~(w > 0)):
        raise ValueError("weights must be > 0")
    rows = np.concatenate([u, v])
    cols = np.concatenate([v, u])
    ww = np.concatenate([w, w])
    order = np.lexsort((cols, rows))
    rows, cols, ww = rows[order], cols[order], ww[order]
    if rows.size > 1:
        dup = (rows[1:] == rows[:-1]) & (cols[1:] == cols[:-1])
        if np.any(dup):
            raise ValueError("duplicate edges")
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    np.cumsum(rp, out=rp)
    return CSRGraph(n, rp, cols.astype(np.int32), ww, name)


def edges_of(g: CSRGraph):
    """Undirected edge list (u < v) of a CSRGraph."""
    rows = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.rp))
    cols = g.ci.astype(np.int64)
    keep = rows < cols
    return rows[keep], cols[keep], g.w[keep]


# ------------------------------------------------------------------ families

def path(n: int, weights=None) -> CSRGraph:
    u = np.arange(n - 1)
    w = np.ones(n - 1) if weights is None else np.asarray(weights, dtype=np.float64)
    return csr_from_edges(n, u, u + 1, w, "P%d" % n)


def cycle(n: int) -> CSRGraph:
    u = np.arange(n)
    v = (u + 1) % n
    return csr_from_edges(n, np.minimum(u, v), np.maximum(u, v), np.ones(n), "C%d" % n)


def star(n: int) -> CSRGraph:
    v = np.arange(1, n)
    return csr_from_edges(n, np.zeros(n - 1, dtype=np.int64), v, np.ones(n - 1), "S%d" % n)


def complete(n: int) -> CSRGraph:
    iu = np.triu_indices(n, 1)
    return csr_from_edges(n, iu[0], iu[1], np.ones(iu[0].size), "K%d" % n)


def random_connected(n: int, extra: int, seed: int, wlo: float = 0.0, whi: float = 1.0,
                     integer_weights: bool = False) -> CSRGraph:
    """Random spanning tree plus `extra` random chords, weights in (wlo, whi]
    (or small integers 1..4 when integer_weights, to exercise exact ties)."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    parents = np.array([perm[rng.integers(0, i)] for i in range(1, n)], dtype=np.int64)
    u = np.concatenate([perm[1:], rng.integers(0, n, extra)])
    v = np.concatenate([parents, rng.integers(0, n, extra)])
    keep = u != v
    a, b = np.minimum(u[keep], v[keep]), np.maximum(u[keep], v[keep])
    key = np.unique(a * n + b)
    a, b = key // n, key % n
    if integer_weights:
        w = rng.integers(1, 5, a.size).astype(np.float64)
    else:
        w = whi - (whi - wlo) * rng.random(a.size)
    return csr_from_edges(n, a, b, w, "rand%d_%d" % (n, seed))


def hub_graph(n: int, chords: int, hubs: int = 1, seed: int = 0) -> CSRGraph:
    """`hubs` hub vertices joined to every other vertex, plus `chords` random
    edges among the non-hub vertices; weights uniform (0, 1].  Exercises rows
    and aggregates far longer than a warp (power-law extremes)."""
    rng = np.random.default_rng(seed)
    us, vs = [], []
    for h in range(hubs):
        others = np.arange(hubs, n)
        us.append(np.full(others.size, h)); vs.append(others)
    a = rng.integers(hubs, n, chords)
    b = rng.integers(hubs, n, chords)
    us.append(a); vs.append(b)
    if hubs > 1:
        hh = np.triu_indices(hubs, 1)
        us.append(hh[0]); vs.append(hh[1])
    u = np.concatenate(us); v = np.concatenate(vs)
    keep = u != v
    lo, hi = np.minimum(u[keep], v[keep]), np.maximum(u[keep], v[keep])
    key = np.unique(lo * n + hi)
    lo, hi = key // n, key % n
    w = 1.0 - rng.random(lo.size)
    return csr_from_edges(n, lo, hi, w, "hub%d_%d" % (n, hubs))


def _grid_weights(rng, size, weights, lo, hi, mu, sigma):
    if weights == "unit":
        return np.ones(size)
    if weights == "uniform":
        return rng.uniform(lo, hi, size)
    if weights == "lognormal":
        return rng.lognormal(mu, sigma, size)
    raise ValueError(weights)


def grid2d(m: int, weights: str = "unit", seed: int = 0, lo: float = 0.5, hi: float = 1.5,
           mx: int = None) -> CSRGraph:
    """m x mx 4-neighbour lattice, vertex (r, c) -> r*mx + c (row-major).
    Edge weights: horizontal edges first (index r*(mx-1)+c), then vertical
    edges (index r*mx+c), drawn from numpy default_rng(seed)."""
    mx = m if mx is None else mx
    n = m * mx
    rng = np.random.default_rng(seed)
    wh = _grid_weights(rng, m * (mx - 1), weights, lo, hi, 0.0, 0.5).reshape(m, mx - 1)
    wv = _grid_weights(rng, (m - 1) * mx, weights, lo, hi, 0.0, 0.5).reshape(m - 1, mx)
    cols = np.empty((m, mx, 4), dtype=np.int32)
    ws = np.zeros((m, mx, 4), dtype=np.float64)
    mask = np.zeros((m, mx, 4), dtype=bool)
    idx = np.arange(n, dtype=np.int64).reshape(m, mx)
    # ascending neighbour order: up (v-mx), left (v-1), right (v+1), down (v+mx)
    cols[1:, :, 0] = idx[:-1, :]; ws[1:, :, 0] = wv; mask[1:, :, 0] = True
    cols[:, 1:, 1] = idx[:, :-1]; ws[:, 1:, 1] = wh; mask[:, 1:, 1] = True
    cols[:, :-1, 2] = idx[:, 1:]; ws[:, :-1, 2] = wh; mask[:, :-1, 2] = True
    cols[:-1, :, 3] = idx[1:, :]; ws[:-1, :, 3] = wv; mask[:-1, :, 3] = True
    deg = mask.sum(axis=2).reshape(-1)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=rp[1:])
    mflat = mask.reshape(-1)
    ci = cols.reshape(-1)[mflat]
    w = ws.reshape(-1)[mflat]
    del cols, ws, mask
    return CSRGraph(n, rp, ci, w, "grid2d_%dx%d_%s" % (m, mx, weights))


def grid3d(m: int, weights: str = "lognormal", seed: int = 0, mu: float = 0.0,
           sigma: float = 0.5, lo: float = 0.5, hi: float = 1.5) -> CSRGraph:
    """m^3 6-neighbour lattice, vertex (z, y, x) -> (z*m + y)*m + x.  Edge
    weights: x-edges, then y-edges, then z-edges, from default_rng(seed)."""
    n = m ** 3
    rng = np.random.default_rng(seed)
    wx = _grid_weights(rng, m * m * (m - 1), weights, lo, hi, mu, sigma).reshape(m, m, m - 1)
    wy = _grid_weights(rng, m * (m - 1) * m, weights, lo, hi, mu, sigma).reshape(m, m - 1, m)
    wz = _grid_weights(rng, (m - 1) * m * m, weights, lo, hi, mu, sigma).reshape(m - 1, m, m)
    idx = np.arange(n, dtype=np.int64).reshape(m, m, m)
    cols = np.empty((m, m, m, 6), dtype=np.int32)
    ws = np.zeros((m, m, m, 6), dtype=np.float64)
    mask = np.zeros((m, m, m, 6), dtype=bool)
    cols[1:, :, :, 0] = idx[:-1]; ws[1:, :, :, 0] = wz; mask[1:, :, :, 0] = True
    cols[:, 1:, :, 1] = idx[:, :-1]; ws[:, 1:, :, 1] = wy; mask[:, 1:, :, 1] = True
    cols[:, :, 1:, 2] = idx[:, :, :-1]; ws[:, :, 1:, 2] = wx; mask[:, :, 1:, 2] = True
    cols[:, :, :-1, 3] = idx[:, :, 1:]; ws[:, :, :-1, 3] = wx; mask[:, :, :-1, 3] = True
    cols[:, :-1, :, 4] = idx[:, 1:]; ws[:, :-1, :, 4] = wy; mask[:, :-1, :, 4] = True
    cols[:-1, :, :, 5] = idx[1:]; ws[:-1, :, :, 5] = wz; mask[:-1, :, :, 5] = True
    deg = mask.sum(axis=3).reshape(-1)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(deg, out=rp[1:])
    mflat = mask.reshape(-1)
    ci = cols.reshape(-1)[mflat]
    w = ws.reshape(-1)[mflat]
    del cols, ws, mask
    return CSRGraph(n, rp, ci, w, "grid3d_%d_%s" % (m, weights))


def rmat(scale: int, avg_degree: float = 16.0, abcd=(0.57, 0.19, 0.19, 0.05), seed: int = 0,
         largest_component: bool = True) -> CSRGraph:
    """R-MAT graph with 2^scale vertices and scale-independent quadrant
    probabilities abcd; n*avg_degree/2 sampled edges, symmetrised, self loops
    and duplicates removed, weights uniform(0,1], largest connected component
    kept (vertices relabelled preserving their original order)."""
    n = 1 << scale
    m = int(n * avg_degree / 2)
    rng = np.random.default_rng(seed)
    a, b, c, _ = abcd
    u = np.zeros(m, dtype=np.int64)
    v = np.zeros(m, dtype=np.int64)
    for bit in range(scale):
        r = rng.random(m)
        ubit = r >= a + b                       # quadrants c, d -> lower half (row bit 1)
        vbit = ((r >= a) & (r < a + b)) | (r >= a + b + c)
        u |= ubit.astype(np.int64) << bit
        v |= vbit.astype(np.int64) << bit
    keep = u != v
    lo, hi = np.minimum(u[keep], v[keep]), np.maximum(u[keep], v[keep])
    key = np.unique(lo * n + hi)
    lo, hi = key // n, key % n
    w = 1.0 - rng.random(lo.size)              # uniform (0, 1]
    if largest_component:
        import scipy.sparse as sp
        from scipy.sparse.csgraph import connected_components
        A = sp.coo_matrix((np.ones(lo.size), (lo, hi)), shape=(n, n))
        ncomp, lab = connected_components(A, directed=False)
        big = np.bincount(lab).argmax()
        keepv = lab == big
        newid = np.full(n, -1, dtype=np.int64)
        newid[keepv] = np.arange(int(keepv.sum()))
        ke = keepv[lo] & keepv[hi]
        lo, hi, w = newid[lo[ke]], newid[hi[ke]], w[ke]
        n = int(keepv.sum())
    return csr_from_edges(n, lo, hi, w, "rmat%d" % scale)


# BASELINE.json "configs" (index -> generator call)
def config(i: int, small: bool = False) -> CSRGraph:
    """The five BASELINE.json workloads.  `small=True` returns a down-scaled
    graph of the same recipe (used by the bounded CPU-baseline sample)."""
    if i == 0:
        return grid2d(32, "unit")
    if i == 1:
        return grid2d(256 if small else 1024, "uniform", seed=1)
    if i == 2:
        return rmat(14 if small else 20, 16.0, seed=2)
    if i == 3:
        return grid3d(40 if small else 256, "lognormal", seed=3)
    if i == 4:
        return grid2d(512 if small else 8192, "uniform", seed=4)
    raise ValueError(i)


CONFIG_NAMES = {
    0: "grid2d_32x32_unit",
    1: "grid2d_1024x1024_uniform[0.5,1.5]",
    2: "rmat20_deg16_(0.57,0.19,0.19,0.05)_lcc_uniform(0,1]",
    3: "grid3d_256^3_lognormal(0,0.5)",
    4: "grid2d_8192x8192_uniform[0.5,1.5]",
}
