"""Pins of the oracle (task rule 3): every oracle function is checked against
something other than itself -- values the paper / its worked examples fix
(tests/golden/*.json, each with a citation), closed forms, dense linear
algebra (numpy), brute force and independent re-implementations in this file.
All CPU-only (`-m "not gpu"`)."""
import json
import math
import os

import numpy as np
import pytest

import graphgen as gg

GOLD = os.path.join(os.path.dirname(__file__), "golden")
M64 = (1 << 64) - 1


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def G(orc, g):
    return orc.Graph.from_csr(g.n, g.rp, g.ci, g.w)


def dense_laplacian(g):
    """Definition 2.1 written out densely from the edge list."""
    L = np.zeros((g.n, g.n))
    u, v, w = gg.edges_of(g)
    for a, b, x in zip(u, v, w):
        L[a, b] -= x
        L[b, a] -= x
        L[a, a] += x
        L[b, b] += x
    return L


def graph_from_edges(n, edges, one_based=False):
    e = np.array(edges, dtype=float).reshape(-1, 3)
    off = 1 if one_based else 0
    return gg.csr_from_edges(n, e[:, 0].astype(int) - off, e[:, 1].astype(int) - off, e[:, 2])


def py_splitmix64(x):
    x = int(x)
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


RANDOM_GRAPHS = [(n, extra, seed) for seed, (n, extra) in enumerate(
    [(12, 6), (30, 20), (57, 80), (100, 150), (150, 60), (200, 400)])]


# ------------------------------------------------------------ generator (R6)

def test_splitmix64_reference_vector(orc):
    gv = gold("splitmix64_seed0.json")
    gamma = int(gv["gamma"], 16)
    for k, h in enumerate(gv["outputs"]):
        assert orc.splitmix64((k * gamma) & M64) == int(h, 16)


def test_rand_uniform_matches_independent_formula(orc):
    seed = 12345
    u = orc.rand_uniform(64, seed)
    s0 = py_splitmix64(seed ^ 0x72616E6400000000)
    ref = np.array([(py_splitmix64((s0 + i) & M64) >> 11) * 2.0 ** -53 for i in range(64)])
    assert np.array_equal(u, ref)
    big = orc.rand_uniform(200000, 7)
    assert big.min() >= 0.0 and big.max() < 1.0 and abs(big.mean() - 0.5) < 5e-3


def test_randperm_is_permutation(orc):
    for n in [1, 2, 17, 1000]:
        p = orc.randperm(n, 3, 1)
        assert np.array_equal(np.sort(p), np.arange(n))


def test_randperm_hand_trace(orc):
    """Fisher-Yates traced by hand from SplitMix64 draws (golden/randperm_trace.json)."""
    gv = gold("randperm_trace.json")
    s0 = py_splitmix64(gv["seed"] ^ 0x7065726D00000000 ^ gv["level"])
    assert s0 == int(gv["s0"], 16)
    for st in gv["steps"]:
        r = py_splitmix64((s0 + st["i"]) & M64)
        assert r == int(st["r"], 16) and r % (st["i"] + 1) == st["j"]
    assert list(orc.randperm(gv["n"], gv["seed"], gv["level"])) == gv["perm"]


def test_randperm_is_uniform(orc):
    """Fisher-Yates draws every permutation of 4 items with probability 1/24.
    Sattolo's variant (j < i, the '% i' slip) draws only the 6 cyclic ones and
    an off-by-one range skews the counts: a chi-square test over 24000 seeds
    (23 degrees of freedom; 99.99 % quantile ~ 59) rejects both."""
    import itertools
    idx = {p: k for k, p in enumerate(itertools.permutations(range(4)))}
    counts = np.zeros(24)
    for seed in range(24000):
        counts[idx[tuple(int(x) for x in orc.randperm(4, seed, 0))]] += 1
    chi2 = float(((counts - 1000.0) ** 2 / 1000.0).sum())
    assert counts.min() > 0 and chi2 < 59.0, (chi2, counts)


# ------------------------------------------------------------ Definition 2.1

def test_laplacian_p3_and_k3(orc):
    p3 = G(orc, gg.path(3))
    cols = [orc.laplacian_matvec(p3, e) for e in np.eye(3)]
    assert np.array_equal(np.array(cols).T, np.array([[1, -1, 0], [-1, 2, -1], [0, -1, 1.0]]))
    assert np.array_equal(orc.laplacian_matvec(p3, np.array([1.0, 0, -1])), np.array([1.0, 0, -1]))
    k3 = G(orc, gg.complete(3))
    Lk = np.array([orc.laplacian_matvec(k3, e) for e in np.eye(3)]).T
    assert np.array_equal(np.diag(Lk), [2, 2, 2]) and np.all(Lk[~np.eye(3, dtype=bool)] == -1)


@pytest.mark.parametrize("n,extra,seed", RANDOM_GRAPHS)
def test_matvec_and_quadratic_form_vs_dense(orc, n, extra, seed):
    g = gg.random_connected(n, extra, seed)
    og = G(orc, g)
    L = dense_laplacian(g)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    assert np.allclose(orc.laplacian_matvec(og, x), L @ x, rtol=1e-13, atol=1e-12)
    assert abs(orc.laplacian_matvec(og, np.ones(n))).max() <= 1e-12 * L.diagonal().max()
    assert orc.quadratic_form(og, x) == pytest.approx(x @ L @ x, rel=1e-12)
    assert orc.rayleigh(og, x) == pytest.approx((x @ L @ x) / (x @ x), rel=1e-12)
    assert orc.rayleigh(og, x) >= 0.0
    assert orc.degrees(og) == pytest.approx(L.diagonal(), rel=1e-15)


def test_rayleigh_examples(orc):
    assert orc.rayleigh(G(orc, gg.path(3)), np.array([1.0, 0, -1])) == 1.0
    k4 = G(orc, gg.complete(4))
    v = np.array([3.0, -1, -1.5, -0.5])
    assert orc.rayleigh(k4, v) == pytest.approx(4.0, rel=1e-15)
    assert orc.rayleigh(k4, np.ones(4)) == 0.0


def test_deflate_normalize_examples(orc):
    assert np.array_equal(orc.deflate(np.array([1.0, 1, 1])), [0, 0, 0])
    assert np.array_equal(orc.deflate(np.array([2.0, 0, 1])), [1, -1, 0])
    assert np.array_equal(orc.normalize(np.array([0.0, 0, 2])), [0, 0, 1])
    assert np.allclose(orc.normalize(np.array([1.0, 1])), [2 ** -0.5] * 2, rtol=1e-15)
    with pytest.raises(ValueError):
        orc.normalize(np.zeros(3))
    assert np.array_equal(orc.sign_fix(np.array([0.0, -1, 2])), [0, 1, -2])


# ------------------------------------------------------------ Algorithm 1

def test_hec_sequential_hand_traces(orc):
    for case in gold("hec_hand_traces.json")["cases"]:
        g = G(orc, graph_from_edges(case["n"], case["edges"], one_based=True))
        q, c = orc.hec_sequential(g, np.array(case["p"]) - 1)
        assert c == case["c"], case["name"]
        assert list(q + 1) == case["q"], case["name"]


def brute_force_algorithm1(g, p):
    """Independent transcription of Algorithm 1 on the DENSE Laplacian:
    m = argmin of column p(i) (np.argmin returns the first minimum)."""
    L = dense_laplacian(g)
    q = np.zeros(g.n, dtype=int)
    c = 0
    for i in range(g.n):
        v = p[i]
        if q[v] == 0:
            m = int(np.argmin(L[:, v]))
            if q[m] == 0:
                c += 1
                q[m] = c
                q[v] = c
            else:
                q[v] = q[m]
    return q - 1, c


@pytest.mark.parametrize("n,extra,seed", RANDOM_GRAPHS[:4])
def test_hec_sequential_vs_dense_argmin(orc, n, extra, seed):
    for integer_weights in (False, True):
        g = gg.random_connected(n, extra, seed, integer_weights=integer_weights)
        p = orc.randperm(n, seed, 0)
        q, c = orc.hec_sequential(G(orc, g), p)
        qb, cb = brute_force_algorithm1(g, p)
        assert c == cb and np.array_equal(q, qb)
        assert c <= n - 1


def handshake_matching(g, salt):
    """Independent algorithm for the parallel-mode matching: iterated
    locally-dominant handshakes (each free vertex points at its heaviest free
    neighbour in the (w, hash) order; mutual pointers match).  For a strict
    edge order this equals the greedy heaviest-first matching (Preis 1999)."""
    def key(a, b, w):
        lo, hi = min(a, b), max(a, b)
        return (w, py_splitmix64(salt ^ ((lo << 32) | hi)))
    mate = [-1] * g.n
    while True:
        ptr = [-1] * g.n
        for v in range(g.n):
            if mate[v] != -1:
                continue
            best = None
            for k in range(g.rp[v], g.rp[v + 1]):
                u = int(g.ci[k])
                if mate[u] == -1:
                    kk = key(v, u, g.w[k])
                    if best is None or kk > best[0]:
                        best = (kk, u)
            if best is not None:
                ptr[v] = best[1]
        if all(p == -1 for p in ptr):
            return np.array(mate)
        for v in range(g.n):
            if ptr[v] != -1 and ptr[ptr[v]] == v:
                mate[v] = ptr[v]


@pytest.mark.parametrize("n,extra,seed", RANDOM_GRAPHS)
def test_hec_parallel_matching_equals_handshake(orc, n, extra, seed):
    for integer_weights in (False, True):
        g = gg.random_connected(n, extra, seed, integer_weights=integer_weights)
        salt = orc.salt_match(seed, 0)
        q, c, mate = orc.hec_parallel(G(orc, g), salt)
        assert np.array_equal(mate, handshake_matching(g, salt))
        # maximal: no edge with two free endpoints
        u, v, _ = gg.edges_of(g)
        assert not np.any((mate[u] == -1) & (mate[v] == -1))
        # matched pairs share an aggregate; leaders numbered in vertex order
        m = mate >= 0
        assert np.all(q[m] == q[mate[m]])
        # each aggregate holds exactly one matched pair; its leader min(u, mate u)
        # gives the aggregate id by increasing vertex order (prefix scan)
        lead = np.array([np.flatnonzero((q == a) & m).min() for a in range(c)])
        assert np.all(np.diff(lead) > 0)
        assert all(((q == a) & m).sum() == 2 for a in range(c))
        # unmatched vertices join their heaviest neighbour
        for x in np.flatnonzero(~m):
            nb = g.ci[g.rp[x]:g.rp[x + 1]]
            ws = g.w[g.rp[x]:g.rp[x + 1]]
            keys = [(ws[t], py_splitmix64(salt ^ ((min(int(x), int(nb[t])) << 32) | max(int(x), int(nb[t]))))) for t in range(nb.size)]
            best = max(range(nb.size), key=lambda t: keys[t])
            assert q[x] == q[nb[best]]
        assert c <= n // 2 + (n % 2)


def handshake_rounds(g, key):
    """Synchronous rounds of the locally-dominant handshake for edge order `key`."""
    mate = [-1] * g.n
    rounds = 0
    while True:
        ptr = [-1] * g.n
        for v in range(g.n):
            if mate[v] != -1:
                continue
            best = None
            for k in range(g.rp[v], g.rp[v + 1]):
                u = int(g.ci[k])
                if mate[u] == -1 and (best is None or key(v, u, g.w[k]) > best[0]):
                    best = (key(v, u, g.w[k]), u)
            if best is not None:
                ptr[v] = best[1]
        pairs = [v for v in range(g.n) if ptr[v] != -1 and ptr[ptr[v]] == v]
        if not pairs:
            return rounds
        for v in pairs:
            mate[v] = ptr[v]
        rounds += 1


def test_tie_rule_r2_depth(orc):
    """Why R2 breaks weight ties by splitmix64 of the index pair rather than by
    the plain index (R2): on unit-weight graphs (BASELINE config 0)
    an index order makes the greedy matching a chain -- the handshake needs
    ~1.5 m rounds on an m x m grid and n/2 on a path, i.e. no parallelism --
    whereas the hashed order (a fixed permutation of the index pairs, since
    splitmix64 is a bijection) needs a handful."""
    salt = orc.salt_match(0, 0)
    by_hash = lambda v, u, w: (w, py_splitmix64(salt ^ ((min(v, u) << 32) | max(v, u))))
    by_index = lambda v, u, w: (w, -min(v, u), -max(v, u))
    for m in (16, 32):
        g = gg.grid2d(m)
        assert handshake_rounds(g, by_index) >= 1.4 * m
        assert handshake_rounds(g, by_hash) <= 6
    p = gg.path(200)
    assert handshake_rounds(p, by_index) == 100 and handshake_rounds(p, by_hash) <= 6


def test_hec_parallel_p4(orc):
    g = G(orc, graph_from_edges(4, [[0, 1, 3.0], [1, 2, 1.0], [2, 3, 3.0]]))
    q, c, mate = orc.hec_parallel(g, orc.salt_match(0, 0))
    assert c == 2 and list(q) == [0, 0, 1, 1] and list(mate) == [1, 0, 3, 2]


# ------------------------------------------------------------ Galerkin

def test_galerkin_hand_cases(orc):
    for case in gold("galerkin_hand.json")["cases"]:
        g = G(orc, graph_from_edges(case["n"], case["edges"]))
        cg = orc.galerkin(g, np.array(case["q"]), case["c"])
        Lc = dense_laplacian(gg.CSRGraph(cg.n, cg.rp, cg.ci, cg.w))
        assert np.array_equal(Lc, np.array(case["coarse_laplacian"])), case["name"]


@pytest.mark.parametrize("n,extra,seed", RANDOM_GRAPHS)
def test_galerkin_equals_dense_triple_product(orc, n, extra, seed):
    g = gg.random_connected(n, extra, seed)
    og = G(orc, g)
    for q, c in (orc.hec_parallel(og, orc.salt_match(1, 0))[:2],
                 orc.hec_sequential(og, orc.randperm(n, 1, 0)),
                 (np.arange(n), n)):
        P = np.zeros((c, n))
        P[q, np.arange(n)] = 1.0
        ref = P @ dense_laplacian(g) @ P.T
        cg = orc.galerkin(og, q, c)
        cgg = gg.CSRGraph(cg.n, cg.rp, cg.ci, cg.w)
        Lc = dense_laplacian(cgg)
        assert np.allclose(Lc, ref, rtol=1e-12, atol=1e-12)
        # pattern: exactly the nonzero off-diagonal blocks
        assert np.array_equal((np.abs(ref) > 0) & ~np.eye(c, dtype=bool), (Lc != 0) & ~np.eye(c, dtype=bool))
        # Laplacian invariants: bit-exact symmetric weights, positive
        assert np.all(cg.w > 0)
        u, v, w = gg.edges_of(cgg)
        D = {(a, b): x for a, b, x in zip(np.repeat(np.arange(c), np.diff(cg.rp)), cg.ci, cg.w)}
        assert all(D[(b, a)] == x for (a, b), x in D.items())
        if c == n:
            assert np.array_equal(cg.rp, og.rp) and np.array_equal(cg.ci, og.ci) and np.array_equal(cg.w, og.w)


def test_galerkin_summation_order_r3(orc):
    """R3: coarse weights fold the crossing fine edges {i<j} left-to-right in
    (i, j) lexicographic order.  Fine vertices 0,1 -> a=0, 2,3 -> b=1 with
    cross edges (0,2)=1e16, (0,3)=1, (1,2)=1: the left fold (1e16 + 1) + 1 =
    1e16 exactly, whereas 1e16 + (1 + 1) = 1e16 + 2."""
    g = G(orc, graph_from_edges(4, [[0, 1, 1.0], [0, 2, 1e16], [0, 3, 1.0], [1, 2, 1.0], [2, 3, 1.0]]))
    cg = orc.galerkin(g, np.array([0, 0, 1, 1]), 2)
    assert cg.w[0] == 1e16 and cg.w[1] == 1e16
    assert (1e16 + 1.0) + 1.0 == 1e16 and 1e16 + 2.0 != 1e16


# ------------------------------------------------------------ colouring (R4)

@pytest.mark.parametrize("n,extra,seed", RANDOM_GRAPHS)
def test_coloring_is_the_greedy_priority_coloring(orc, n, extra, seed):
    g = gg.random_connected(n, extra, seed)
    salt = orc.salt_color(seed, 2)
    color, ncol = orc.greedy_coloring(G(orc, g), salt)
    pri = [(py_splitmix64(salt ^ v), v) for v in range(n)]
    for v in range(n):
        nb = g.ci[g.rp[v]:g.rp[v + 1]]
        assert np.all(color[nb] != color[v])
        higher = {int(color[u]) for u in nb if pri[u] > pri[v]}
        mex = 0
        while mex in higher:
            mex += 1
        assert color[v] == mex
    assert ncol == color.max() + 1


# ------------------------------------------------------------ Algorithm 2

def test_gauss_seidel_worked_example(orc):
    gv = gold("gauss_seidel_2x2.json")
    A = np.array(gv["A"])
    rp, ci, a = np.array([0, 2, 4]), np.array([0, 1, 0, 1]), A.reshape(-1)
    x1, k = orc.gs_solve(2, rp, ci, a, gv["b"], gv["x0"], 0.0, 1)
    assert list(x1) == gv["first_sweep"] and k == 1
    x, k = orc.gs_solve(2, rp, ci, a, gv["b"], gv["x0"], 1e-14, 200)
    assert np.allclose(x, gv["solution"], atol=1e-13) and k < 200
    x, k = orc.gs_solve(2, rp, ci, a, [0.0, 0.0], [0.0, 0.0], 1e-6, 50)
    assert np.array_equal(x, [0, 0]) and k == 1


@pytest.mark.parametrize("seed", range(10))
def test_gauss_seidel_converges_theorem_2_2(orc, seed):
    """Theorems 2.1/2.2: SPD diagonally dominant systems;
    energy-norm error nonincreasing per sweep, limit = dense solve."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(5, 50))
    B = rng.random((n, n)) * (rng.random((n, n)) < 0.3)
    A = -(B + B.T)
    np.fill_diagonal(A, 0)
    np.fill_diagonal(A, -A.sum(axis=1) + rng.random(n) + 0.1)
    b = rng.standard_normal(n)
    xs = np.linalg.solve(A, b)
    rp = np.arange(n + 1) * n
    ci = np.tile(np.arange(n), n)
    x = rng.standard_normal(n)
    err = lambda y: float((y - xs) @ A @ (y - xs))
    prev = err(x)
    for _ in range(30):
        x, _ = orc.gs_solve(n, rp, ci, A.reshape(-1), b, x, 0.0, 1)
        e = err(x)
        assert e <= prev * (1 + 1e-12) + 1e-300
        prev = e
    x, k = orc.gs_solve(n, rp, ci, A.reshape(-1), b, x, 1e-13, 5000)
    assert np.allclose(x, xs, atol=1e-10)


@pytest.mark.parametrize("n,extra,seed", RANDOM_GRAPHS)
def test_gs_sweep_equals_dense_triangular_solve(orc, n, extra, seed):
    """One in-place sweep on L x = 0 in visiting order pi is
    x' = -(D + L_low)^{-1} U x for the pi-permuted Laplacian (split of A)."""
    g = gg.random_connected(n, extra, seed)
    og = G(orc, g)
    L = dense_laplacian(g)
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    color, _ = orc.greedy_coloring(og, orc.salt_color(0, 0))
    for order in (np.arange(n), orc.color_order(color), rng.permutation(n)):
        A = L[np.ix_(order, order)]
        lowd = np.tril(A)
        up = np.triu(A, 1)
        ref = np.empty(n)
        ref[order] = np.linalg.solve(lowd, -up @ x[order])
        got = orc.gs_sweeps(og, x, 1, order)
        assert np.allclose(got, ref, rtol=1e-11, atol=1e-12)
    # the colour order is a valid multicolour order: same result as any
    # within-colour permutation (no same-colour neighbours)
    o1 = orc.color_order(color)
    o2 = np.lexsort((-np.arange(n), color))
    assert np.array_equal(orc.gs_sweeps(og, x, 2, o1), orc.gs_sweeps(og, x, 2, o2))


def test_gs_constant_is_fixed_point(orc):
    g = G(orc, gg.grid2d(6, "uniform", seed=3))
    y = orc.gs_sweeps(g, np.full(36, 0.7), 3)
    assert np.allclose(y, 0.7, rtol=1e-15)


# ------------------------------------------------------------ power iteration

@pytest.mark.parametrize("n,extra,seed", RANDOM_GRAPHS)
def test_power_step_equals_dense(orc, n, extra, seed):
    g = gg.random_connected(n, extra, seed)
    og = G(orc, g)
    L = dense_laplacian(g)
    c = orc.shift_of(orc.degrees(og))
    assert c >= np.linalg.eigvalsh(L).max()        # Gershgorin (R8)
    x = np.random.default_rng(seed).standard_normal(n)
    y = c * x - L @ x
    y -= y.mean()
    y /= np.linalg.norm(y)
    assert np.allclose(orc.power_iterations(og, x, 1, c), y, rtol=1e-12, atol=1e-14)


def test_prolongate_examples(orc):
    assert list(orc.prolongate(np.array([0, 0, 1, 1]), np.array([5.0, 7.0]))) == [5, 5, 7, 7]
    assert list(orc.prolongate(np.array([0, 0, 0]), np.array([5.0]))) == [5, 5, 5]
    y = np.array([1.0, 2, 3])
    assert np.array_equal(orc.prolongate(np.arange(3), y), y)


# ------------------------------------------------------------ Algorithm 3

def closed_form(kind, n):
    return {"path": 2 - 2 * math.cos(math.pi / n), "cycle": 2 - 2 * math.cos(2 * math.pi / n),
            "star": 1.0, "complete": float(n), "grid2d": 4 * math.sin(math.pi / (2 * n)) ** 2}[kind]


FAMILIES = [("path", 3, gg.path), ("path", 10, gg.path), ("path", 40, gg.path), ("cycle", 10, gg.cycle),
            ("cycle", 50, gg.cycle), ("star", 6, gg.star), ("star", 20, gg.star),
            ("complete", 4, gg.complete), ("complete", 8, gg.complete),
            ("grid2d", 5, lambda m: gg.grid2d(m)), ("grid2d", 8, lambda m: gg.grid2d(m))]


@pytest.mark.parametrize("kind,n,make", FAMILIES)
@pytest.mark.parametrize("mode", ["parallel", "sequential"])
def test_solve_closed_form_spectra(orc, kind, n, make, mode):
    """Run Algorithm 3 with enough power iterations to converge; the Rayleigh
    quotient must reach the closed-form lambda_2 (gold spectra_closed_forms)."""
    g = G(orc, make(n))
    cfg = orc.Config(mode=mode, power_iters=4000, gs_sweeps=2, seed=5)
    r = orc.solve(g, cfg)
    lam = closed_form(kind, n)
    assert r.lambda2 == pytest.approx(lam, rel=1e-8)
    assert np.linalg.norm(r.vector) == pytest.approx(1.0, rel=1e-14)
    assert abs(r.vector.sum()) < 1e-10
    # default iteration counts: Courant-Fischer lower bound and the
    # approximation quality of the cascadic method
    r2 = orc.solve(g, orc.Config(mode=mode))
    assert r2.lambda2 >= lam * (1 - 1e-12)


@pytest.mark.parametrize("n,extra,seed", RANDOM_GRAPHS)
def test_solve_vs_dense_eigensolver(orc, n, extra, seed):
    g = gg.random_connected(n, extra, seed, wlo=0.1)
    og = G(orc, g)
    ev, V = np.linalg.eigh(dense_laplacian(g))
    lam2, v2 = ev[1], V[:, 1]
    for mode in ("parallel", "sequential"):
        r = orc.solve(og, orc.Config(mode=mode))
        assert r.lambda2 >= lam2 - 1e-12                       # Courant-Fischer
        assert abs(r.vector @ np.ones(n)) < 1e-10 * n
        gap = (ev[2] - ev[1]) / ev[2]
        if gap > 0.3 and n <= 60:
            rc = orc.solve(og, orc.Config(mode=mode, power_iters=3000))
            assert rc.lambda2 == pytest.approx(lam2, rel=1e-9)
            assert 1 - abs(rc.vector @ v2) < 1e-9


def test_parallel_vs_sequential_end_results(orc):
    """North star: the parallel-order mode is checked against the paper's
    sequential order on end results."""
    for g in (gg.grid2d(30), gg.grid2d(24, "uniform", seed=2), gg.random_connected(200, 300, 9)):
        og = G(orc, g)
        lam_true = np.linalg.eigvalsh(dense_laplacian(g))[1]
        for it, tol in ((10, 1.0), (1000, 0.01)):
            rp = orc.solve(og, orc.Config(mode="parallel", power_iters=it))
            rs = orc.solve(og, orc.Config(mode="sequential", power_iters=it))
            for r in (rp, rs):
                assert lam_true * (1 - 1e-12) <= r.lambda2 <= lam_true * (1 + tol)
            assert rp.lambda2 == pytest.approx(rs.lambda2, rel=tol)


def test_hierarchy_invariants(orc):
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components
    for g in (gg.grid2d(100), gg.rmat(10, 8, seed=1), gg.grid3d(12, seed=2)):
        levels = orc.build_hierarchy(G(orc, g), orc.Config())
        sizes = [L.g.n for L in levels]
        assert all(b < a for a, b in zip(sizes, sizes[1:]))
        assert sizes[-1] <= 25
        for L in levels:
            A = sp.csr_matrix((L.g.w, L.g.ci, L.g.rp), shape=(L.g.n, L.g.n))
            assert (A != A.T).nnz == 0 and np.all(L.g.w > 0)
            assert connected_components(A, directed=False)[0] == 1
            assert L.shift >= 2 * L.d.max()


def test_solve_is_deterministic(orc):
    g = G(orc, gg.grid2d(40, "uniform", seed=1))
    a = orc.solve(g, orc.Config(seed=3))
    b = orc.solve(g, orc.Config(seed=3))
    assert np.array_equal(a.vector, b.vector) and a.lambda2 == b.lambda2
