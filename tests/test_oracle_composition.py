"""Pin of the oracle's COMPOSITION of Algorithm 3 at the north-star iteration
counts (2 Gauss-Seidel sweeps + 10 power iterations per level), where the
closed-form pins (thousands of iterations, any ordering converges) cannot see
a dropped step.

`dense_algorithm3` below is an independent transcription of Algorithm 3
 with the readings of DESIGN.md section 3, written with
dense numpy matrices and Python loops only -- it calls nothing in oracle/:

  Step 1: while n > coarsest: heaviest-first greedy
    matching in the (w, hash) order (R2) by sorting the edge list, unmatched
    vertices join their heaviest neighbour's aggregate,
    aggregates numbered by increasing leader; L^{l+1} = P L P^T as a dense
    product; greedy colouring by priority (R4); shift
    c = 2 max d, 3 max d on a 2-vertex level (R8).
  Step 2 (R5, R6): y = rand(n_J), deflate, normalise, k power
    steps y <- normalise(deflate((cI - L) y)).
  Step 3: y = P^T y, deflate, normalise; GS sweeps on
    L y = 0 in (colour, index) order (Algorithm 2 line 87 with b = 0);
    deflate, normalise; k power steps.
  Then sign (R10) and the Rayleigh quotient y^T L y / y^T y.

Weights are multiples of 1/8, so every coarse weight is exact in any
summation order and the dense product reproduces the R3 fold bit for bit
(the hierarchies then agree exactly, and only the solve arithmetic can
differ -- by rounding, far below 1e-13).  Negative controls: mutations of the
transcription (an iteration count off by one, Gauss-Seidel in lexicographic
instead of multicolour order, one level's smoothing skipped) must move the
result by more than 1e-10, which shows the pin can see them.  (Dropping one of
the deflations is NOT such a mutation: Gauss-Seidel on L y = 0 and c I - L are
linear and map the constant vector to a multiple of itself, and every step is
followed by a deflation, so the end result is the same in exact arithmetic.)
"""
import numpy as np
import pytest

import graphgen as gg

M64 = (1 << 64) - 1
TAG_MATCH = 0x6D61746368000000
TAG_COLOR = 0x636F6C6F72000000
TAG_RAND = 0x72616E6400000000


def sm64(x):
    z = (int(x) + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def dense_W(g):
    W = np.zeros((g.n, g.n))
    for i in range(g.n):
        for k in range(g.rp[i], g.rp[i + 1]):
            W[i, g.ci[k]] = g.w[k]
    return W


def ekey(salt, a, b, w):
    lo, hi = min(a, b), max(a, b)
    return (w, sm64(salt ^ ((lo << 32) | hi)))


def dense_hec(W, salt):
    n = W.shape[0]
    edges = [(ekey(salt, i, j, W[i, j]), i, j) for i in range(n) for j in range(i + 1, n) if W[i, j] > 0]
    edges.sort(reverse=True)
    mate = [-1] * n
    for _, i, j in edges:
        if mate[i] < 0 and mate[j] < 0:
            mate[i], mate[j] = j, i
    leader = list(range(n))
    for v in range(n):
        if mate[v] >= 0:
            leader[v] = min(v, mate[v])
        else:
            nb = [u for u in range(n) if W[v, u] > 0]
            if nb:
                m = max(nb, key=lambda u: ekey(salt, v, u, W[v, u]))
                leader[v] = min(m, mate[m])
    ids = {}
    for v in range(n):
        if leader[v] == v:
            ids[v] = len(ids)
    return np.array([ids[leader[v]] for v in range(n)]), len(ids)


def dense_colour_order(W, salt):
    n = W.shape[0]
    color = [-1] * n
    for v in sorted(range(n), key=lambda v: (sm64(salt ^ v), v), reverse=True):
        used = {color[u] for u in range(n) if W[v, u] > 0 and color[u] >= 0}
        c = 0
        while c in used:
            c += 1
        color[v] = c
    return sorted(range(n), key=lambda v: (color[v], v))


def dense_algorithm3(g, seed=0, gs=2, k=10, coarsest=25, mutate=None):
    # Step 1: setup phase
    Ws, Ps = [dense_W(g)], []
    while Ws[-1].shape[0] > coarsest and len(Ws) < 50:
        W = Ws[-1]
        ell = len(Ws) - 1
        q, c = dense_hec(W, sm64(seed ^ (TAG_MATCH + ell)))
        if c > 0.95 * W.shape[0] or c < 2:
            break
        P = np.zeros((c, W.shape[0]))
        P[q, np.arange(W.shape[0])] = 1.0
        L = np.diag(W.sum(1)) - W
        Lc = P @ L @ P.T
        Wc = -(Lc - np.diag(np.diag(Lc)))
        Ps.append(P)
        Ws.append(Wc)
    Ls = [np.diag(W.sum(1)) - W for W in Ws]
    orders = [dense_colour_order(W, sm64(seed ^ (TAG_COLOR + l))) for l, W in enumerate(Ws)]
    shifts = [(3.0 if W.shape[0] == 2 else 2.0) * W.sum(1).max() for W in Ws]

    def dn(y):
        y = y - y.mean()
        return y / np.linalg.norm(y)

    def power(l, y, its):
        for _ in range(its):
            y = dn(shifts[l] * y - Ls[l] @ y)
        return y

    def gs_sweeps(l, y, sweeps):
        W, d = Ws[l], Ws[l].sum(1)
        y = y.copy()
        for _ in range(sweeps):
            for i in orders[l]:
                y[i] = (W[i] @ y) / d[i]
        return y

    J = len(Ws) - 1
    s0 = sm64(seed ^ TAG_RAND)
    y = np.array([(sm64((s0 + i) & M64) >> 11) * 2.0 ** -53 for i in range(Ws[J].shape[0])])
    y = power(J, dn(y), k)
    for j in range(J - 1, -1, -1):
        y = dn(Ps[j].T @ y)
        if mutate == "skip_level1" and j == 1:
            continue
        if mutate == "lex_gs":
            orders[j] = list(range(Ws[j].shape[0]))
        y = gs_sweeps(j, y, gs - 1 if mutate == "one_gs" else gs)
        y = dn(y)
        y = power(j, y, k - 1 if mutate == "nine_pi" else k)
    nz = np.flatnonzero(y)
    if y[nz[0]] < 0:
        y = -y
    return y, float(y @ Ls[0] @ y / (y @ y)), J + 1


def eighths(g, seed):
    """Same graph, weights replaced by multiples of 1/8 in [1/8, 2] (symmetric)."""
    rng = np.random.default_rng(seed)
    u, v, _ = gg.edges_of(g)
    return gg.csr_from_edges(g.n, u, v, rng.integers(1, 17, u.size) / 8.0)


CASES = [("P4", gg.path(4), 2), ("C6", gg.cycle(6), 2), ("grid6x5", None, 3),
         ("grid6x5_eighths", "eighths", 3), ("grid12", gg.grid2d(12), 25),
         ("rand60_eighths", eighths(gg.random_connected(60, 70, 4), 4), 5)]


def _graph(name, g):
    if name.startswith("grid6x5"):
        m, k = 6, 5
        idx = np.arange(m * k).reshape(k, m)
        u = np.concatenate([idx[:, :-1].ravel(), idx[:-1, :].ravel()])
        v = np.concatenate([idx[:, 1:].ravel(), idx[1:, :].ravel()])
        base = gg.csr_from_edges(m * k, u, v, np.ones(u.size))
        return eighths(base, 7) if g == "eighths" else base
    return g


@pytest.mark.parametrize("name,g,coarsest", CASES, ids=[c[0] for c in CASES])
def test_oracle_solve_equals_dense_transcription(orc, name, g, coarsest):
    g = _graph(name, g)
    cfg = orc.Config(coarsest_size=coarsest)
    r = orc.solve(orc.Graph.from_csr(g.n, g.rp, g.ci, g.w), cfg)
    y, lam, nlev = dense_algorithm3(g, coarsest=coarsest)
    assert len(r.levels) == nlev
    assert abs(r.lambda2 - lam) <= 1e-13 * lam
    assert np.abs(r.vector - y).max() <= 1e-13
    if nlev > 2:
        for mut in ("one_gs", "nine_pi", "lex_gs", "skip_level1"):
            ym, lm, _ = dense_algorithm3(g, coarsest=coarsest, mutate=mut)
            assert np.abs(ym - r.vector).max() > 1e-10 or abs(lm - r.lambda2) > 1e-10 * lam, mut
