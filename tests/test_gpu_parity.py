"""GPU parity tests: the CUDA path (through the C ABI) against the oracle, on
the same seeded inputs.  Bars:
  * hierarchy (matching, aggregate ids, coarse CSR pattern AND values, colours):
    bit-exact;
  * single operations from identical inputs: GS / power steps rel 1e-12,
    prolongation exact, Rayleigh quotient rel 1e-12;
  * full solve with identical iteration counts: |lambda_gpu - lambda_orc| /
    lambda_orc <= 1e-10 and 1 - |cos(v_gpu, v_orc)| <= 1e-10 (north star).
"""
import numpy as np
import pytest

import graphgen as gg

pytestmark = pytest.mark.gpu

LAM_TOL = 1e-10
COS_TOL = 1e-10


@pytest.fixture(scope="module")
def fd():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1602_04386_b200 as fd
    from paper_1602_04386_b200 import build
    build.build()
    return fd


def orc_graph(orc, g):
    return orc.Graph.from_csr(g.n, g.rp, g.ci, g.w)


def clique_with_tail(k, tail):
    """K_k (more than 64 colours) hanging off a long path: low average degree,
    so the thread-per-vertex kernels meet a > 64-colour neighbourhood."""
    iu = np.triu_indices(k, 1)
    u = np.r_[iu[0], np.arange(k - 1, k + tail - 1)]
    v = np.r_[iu[1], np.arange(k, k + tail)]
    w = 0.5 + (np.arange(u.size) % 7) / 7.0
    return gg.csr_from_edges(k + tail, u, v, w, "clique%d_tail%d" % (k, tail))


def unsorted_rows(g, seed):
    """Same graph with the entries of every CSR row in a seeded random order
    (violates the input contract: columns strictly increasing per row)."""
    rng = np.random.default_rng(seed)
    ci, w = g.ci.copy(), g.w.copy()
    for v in range(g.n):
        b, e = int(g.rp[v]), int(g.rp[v + 1])
        p = b + rng.permutation(e - b)
        ci[b:e], w[b:e] = g.ci[p], g.w[p]
    return gg.CSRGraph(g.n, g.rp.copy(), ci, w, g.name + "_unsorted")


SMALL = {
    "grid32_unit(config0)": lambda: gg.grid2d(32, "unit"),
    "grid50x37_uniform": lambda: gg.grid2d(50, "uniform", seed=7, mx=37),
    "grid3d_12_lognormal": lambda: gg.grid3d(12, "lognormal", seed=3),
    "rmat12": lambda: gg.rmat(12, 16.0, seed=5),
    "rand500_int_ties": lambda: gg.random_connected(500, 900, 11, integer_weights=True),
    "rand300": lambda: gg.random_connected(300, 1500, 12),
    "path100": lambda: gg.path(100),
    "star40": lambda: gg.star(40),
    # the byte colouring state holds degrees <= 126: the boundary and the int fallback
    "star127_deg126": lambda: gg.star(127),
    "star128_deg127": lambda: gg.star(128),
    "complete30": lambda: gg.complete(30),
    # dense small levels (average degree >= 64): the single-CTA colouring
    "complete100": lambda: gg.complete(100),
    "dense1500_deg120": lambda: gg.random_connected(1500, 90000, 21),
    # mid-size dense level (n > 12288, average degree >= 64): the cluster colouring
    "dense16k_deg70": lambda: gg.random_connected(16000, 560000, 22),
    # levels of >= 450 entries per row rank their long rows before the matching (k_rank_rows)
    "complete500": lambda: gg.complete(500),
    "dense3000_deg500": lambda: gg.random_connected(3000, 750000, 23),
    "hub3000_3hubs": lambda: gg.hub_graph(3000, 4000, hubs=3, seed=4),
    # a row of 4999 entries: five piece tiles of the row passes (hub rows > 1024 entries)
    "star5000": lambda: gg.star(5000),
    "clique70_tail2000": lambda: clique_with_tail(70, 2000),
    "tiny_p5": lambda: gg.path(5),
    "tiny_p3": lambda: gg.path(3),
    # K2: the Gershgorin shift 2 max d equals lambda_max = lambda_2 (R8: 3 max d there)
    "tiny_p2": lambda: gg.path(2, weights=[0.75]),
}


@pytest.mark.parametrize("name", sorted(SMALL))
def test_hierarchy_bit_exact(fd, orc, name):
    g = SMALL[name]()
    levels = orc.build_hierarchy(orc_graph(orc, g), orc.Config())
    h = fd.fiedler_create(g.n, g.nnz, g.rp, g.ci, g.w)
    try:
        assert fd.fiedler_num_levels(h) == len(levels)
        for ell, L in enumerate(levels):
            ex = fd.fiedler_level_export(h, ell)
            assert ex["n"] == L.g.n
            assert np.array_equal(ex["rp"], L.g.rp), (name, ell)
            assert np.array_equal(ex["ci"], L.g.ci), (name, ell)
            assert np.array_equal(ex["w"].view(np.uint64), L.g.w.view(np.uint64)), (name, ell)
            assert np.array_equal(ex["color"], L.color), (name, ell)
            if ell < len(levels) - 1:
                assert np.array_equal(ex["agg"], L.q), (name, ell)
                assert np.array_equal(ex["mate"], L.mate), (name, ell)
    finally:
        fd.fiedler_destroy(h)


@pytest.mark.parametrize("name", ["grid50x37_uniform", "grid3d_12_lognormal", "rand300"])
def test_hierarchy_full_sort_fallback(fd, orc, name, monkeypatch):
    """The Galerkin fallback of very large levels (full (B, lo, hi) sort of the
    class-0 rows), forced on small graphs: still bit-exact."""
    monkeypatch.setenv("FIEDLER_TEST_FULL_SORT", "1")
    test_hierarchy_bit_exact(fd, orc, name)


@pytest.mark.parametrize("name", ["grid32_unit(config0)", "grid3d_12_lognormal", "rmat12", "rand300",
                                  "hub3000_3hubs", "star5000"])
def test_single_ops_vs_oracle(fd, orc, name):
    g = SMALL[name]()
    levels = orc.build_hierarchy(orc_graph(orc, g), orc.Config())
    h = fd.fiedler_create(g.n, g.nnz, g.rp, g.ci, g.w)
    rng = np.random.default_rng(0)
    try:
        for ell, L in enumerate(levels):
            x = rng.standard_normal(L.g.n)
            # Gauss-Seidel sweeps in the multicolour order
            for sweeps in (1, 2):
                out = np.empty_like(x)
                fd.fiedler_level_apply(h, ell, fd.FIEDLER_OP_GS_SWEEPS, x, out, sweeps)
                ref = orc.gs_sweeps(L.g, x, sweeps, L.order, L.d)
                np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-13 * np.abs(ref).max())
            # power iteration on c I - L with deflation + normalisation
            for it in (1, 3):
                out = np.empty_like(x)
                fd.fiedler_level_apply(h, ell, fd.FIEDLER_OP_POWER, x, out, it)
                ref = orc.power_iterations(L.g, x, it, L.shift, L.d)
                np.testing.assert_allclose(out, ref, rtol=1e-11, atol=1e-13)
            # Rayleigh quotient
            lam, _ = fd.fiedler_level_apply(h, ell, fd.FIEDLER_OP_RAYLEIGH, x)
            assert lam == pytest.approx(orc.rayleigh(L.g, x), rel=1e-12)
            # prolongation from the next level (exact)
            if ell + 1 < len(levels):
                yc = rng.standard_normal(levels[ell + 1].g.n)
                out = np.empty(L.g.n)
                fd.fiedler_level_apply(h, ell, fd.FIEDLER_OP_PROLONG, yc, out)
                assert np.array_equal(out, orc.prolongate(L.q, yc))
    finally:
        fd.fiedler_destroy(h)


def test_gs_statistics_without_cancellation(fd):
    """The mean / deflated norm a GS pass reports (the lazy deflation and
    normalisation of R5) stay accurate when the vector is nearly constant,
    |mean| >> deflated norm: the sums are shifted (finish_stats), so
    Q - S^2/n does not cancel.  Reference: numpy two-pass on the returned vector."""
    g = gg.grid2d(64, "uniform", seed=4)
    h = fd.fiedler_create(g.n, g.nnz, g.rp, g.ci, g.w)
    try:
        x = 1.0e6 + 1.0e-3 * np.random.default_rng(3).standard_normal(g.n)
        out = np.empty_like(x)
        mu, sig = fd.fiedler_level_apply(h, 0, fd.FIEDLER_OP_GS_SWEEPS, x, out, 2)
    finally:
        fd.fiedler_destroy(h)
    ref_mu = out.mean()
    ref_sig = np.sqrt(((out - ref_mu) ** 2).sum())
    assert mu == pytest.approx(ref_mu, rel=1e-14)
    assert sig == pytest.approx(ref_sig, rel=1e-9)


def compare_solve(fd, orc, g, cfg_kw=None, device_input=False):
    cfg_kw = cfg_kw or {}
    ref = orc.solve(orc_graph(orc, g), orc.Config(**cfg_kw))
    opts = fd.fiedler_default_opts(**{k: v for k, v in cfg_kw.items()
                                      if k in ("gs_sweeps", "power_iters", "seed", "coarsest_size")})
    if device_input:
        import torch
        args = [torch.from_numpy(a).cuda() for a in (g.rp, g.ci, g.w)]
        vec = torch.empty(g.n, dtype=torch.float64, device="cuda")
    else:
        args = [g.rp, g.ci, g.w]
        vec = np.empty(g.n)
    info = fd.fiedler_info()
    h = fd.fiedler_create(g.n, g.nnz, *args, opts)
    try:
        lam = fd.fiedler_solve(h, vec, None, info)
    finally:
        fd.fiedler_destroy(h)
    v = vec.cpu().numpy() if device_input else vec
    assert info.num_levels == len(ref.levels)
    assert abs(lam - ref.lambda2) / ref.lambda2 <= LAM_TOL, (lam, ref.lambda2)
    cos = abs(float(v @ ref.vector)) / (np.linalg.norm(v) * np.linalg.norm(ref.vector))
    assert 1 - cos <= COS_TOL, 1 - cos
    assert np.linalg.norm(v) == pytest.approx(1.0, rel=1e-12)
    assert abs(v.sum()) <= 1e-9 * np.sqrt(g.n)
    nz = np.flatnonzero(v)
    assert v[nz[0]] > 0
    # the residual is a diagnostic from sqrt(||Lv||^2 - lambda^2 ||v||^2): absolute
    # accuracy ~ sqrt(eps) * lambda (cancellation when v is an exact eigenvector)
    assert info.residual_norm == pytest.approx(ref.residual_norm, rel=1e-6, abs=1e-7 * ref.lambda2)
    return lam, v, info


@pytest.mark.parametrize("name", sorted(SMALL))
def test_solve_parity_small(fd, orc, name):
    compare_solve(fd, orc, SMALL[name]())


def test_solve_parity_iteration_variants(fd, orc):
    g = gg.grid2d(40, "uniform", seed=2)
    for kw in ({"gs_sweeps": 0}, {"power_iters": 0}, {"gs_sweeps": 3, "power_iters": 25},
               {"seed": 12345}, {"coarsest_size": 100},
               {"coarsest_size": 2}):          # hierarchy down to a 2-vertex level (R8)
        compare_solve(fd, orc, g, kw)


def test_device_input_equals_host_input(fd, orc):
    g = gg.grid2d(64, "uniform", seed=9)
    lam_h, v_h, _ = compare_solve(fd, orc, g)
    lam_d, v_d, _ = compare_solve(fd, orc, g, device_input=True)
    assert lam_h == lam_d and np.array_equal(v_h, v_d)


def test_repeated_solves_bit_identical(fd):
    g = gg.rmat(13, 16.0, seed=1)
    s = fd.FiedlerSolver(g.n, g.rp, g.ci, g.w)
    a, b = np.empty(g.n), np.empty(g.n)
    la = s.solve(a)
    lb = s.solve(b)
    lc = s.solve(b, use_graph=0)
    s.close()
    assert la == lb == lc and np.array_equal(a, b)


@pytest.mark.parametrize("name,make", [
    ("grid256_uniform(config1_recipe)", lambda: gg.config(1, small=True)),
    ("rmat14(config2_recipe)", lambda: gg.config(2, small=True)),
    ("grid3d_40(config3_recipe)", lambda: gg.config(3, small=True)),
])
def test_solve_parity_medium(fd, orc, name, make):
    compare_solve(fd, orc, make())


def test_solve_parity_config1_full_size(fd, orc):
    """BASELINE configs[1] at full size (1024 x 1024, uniform weights):
    the oracle completes it in seconds, so every output is compared."""
    compare_solve(fd, orc, gg.config(1))


# ------------------------------------------------------------------ error paths

def test_rejects_disconnected(fd):
    a = gg.grid2d(8)
    b = gg.grid2d(5)
    u1, v1, w1 = gg.edges_of(a)
    u2, v2, w2 = gg.edges_of(b)
    g = gg.csr_from_edges(a.n + b.n, np.r_[u1, u2 + a.n], np.r_[v1, v2 + a.n], np.r_[w1, w2])
    with pytest.raises(fd.FiedlerError) as e:
        fd.fiedler_create(g.n, g.nnz, g.rp, g.ci, g.w)
    assert e.value.code == fd.FIEDLER_ERR_DISCONNECTED


def test_rejects_unsorted_rows(fd):
    # ascending rows are part of the contract (include/fiedler.h) and a
    # premise of the direct Galerkin path: validation must catch them
    g = unsorted_rows(gg.grid2d(12, "uniform", seed=9), 3)
    with pytest.raises(fd.FiedlerError) as e:
        fd.fiedler_create(g.n, g.nnz, g.rp, g.ci, g.w)
    assert e.value.code == fd.FIEDLER_ERR_GRAPH


def test_rejects_invalid_csr(fd):
    g = gg.grid2d(6, "uniform", seed=1)
    bad = g.w.copy(); bad[3] *= 1.0000001                     # asymmetric
    with pytest.raises(fd.FiedlerError) as e:
        fd.fiedler_create(g.n, g.nnz, g.rp, g.ci, bad)
    assert e.value.code == fd.FIEDLER_ERR_GRAPH
    bad = g.w.copy(); bad[0] = -1.0
    with pytest.raises(fd.FiedlerError):
        fd.fiedler_create(g.n, g.nnz, g.rp, g.ci, bad)
    ci = g.ci.copy(); ci[0], ci[1] = ci[1], ci[0]            # unsorted row
    with pytest.raises(fd.FiedlerError):
        fd.fiedler_create(g.n, g.nnz, g.rp, ci, g.w)
    rp = g.rp.copy(); rp[3] = rp[4] + 1                      # bad offsets
    with pytest.raises(fd.FiedlerError):
        fd.fiedler_create(g.n, g.nnz, rp, g.ci, g.w)
    with pytest.raises(fd.FiedlerError) as e:
        fd.fiedler_create(1, 0, np.zeros(2, np.int64), np.zeros(0, np.int32), np.zeros(0))
    assert e.value.code == fd.FIEDLER_ERR_ARG
