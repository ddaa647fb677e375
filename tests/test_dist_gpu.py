"""GPU tests of the partitioned solve (fiedler_dist_plan / fiedler_dist_op +
paper_1602_04386_b200/dist.py).  Several ranks run as threads of one process
on one GPU (ThreadComm): their kernels never wait on one another -- every
exchange is a host rendezvous after a device synchronisation."""
import numpy as np
import pytest

import graphgen as gg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fd():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1602_04386_b200 as fd
    from paper_1602_04386_b200 import build
    build.build()
    return fd


GRAPHS = {
    "grid64x45": lambda: gg.grid2d(64, "uniform", seed=3, mx=45),
    "rmat12": lambda: gg.rmat(12, 16.0, seed=5),
    "hub": lambda: gg.hub_graph(3000, 4000, hubs=3, seed=4),
    "grid3d_14": lambda: gg.grid3d(14, "lognormal", seed=2),
    "wcomplete300": lambda: _wcomplete(300, seed=7),   # 300 colours on level 0 (> 128)
}


def _wcomplete(n, seed):
    """Complete graph with random weights: every level needs as many colours as vertices."""
    rng = np.random.default_rng(seed)
    u, v = np.triu_indices(n, 1)
    return gg.csr_from_edges(n, u, v, rng.uniform(0.5, 1.5, u.size), "wcomplete%d" % n)


def _handle(fd, g):
    import torch
    args = [torch.from_numpy(a).cuda() for a in (g.rp, g.ci, g.w)]
    opts = fd.fiedler_default_opts(stream=torch.cuda.current_stream().cuda_stream)
    return fd.fiedler_create(g.n, g.nnz, *args, opts)


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_plans_match_reference(fd, orc, name):
    """Row bounds, halo counts and the halo lists themselves (recovered through
    HALO_PACK / HALO_UNPACK of index vectors) equal the reference plan."""
    import torch
    from dist_ref import ref_plan
    g = GRAPHS[name]()
    h = _handle(fd, g)
    try:
        levels = orc.build_hierarchy(orc.Graph.from_csr(g.n, g.rp, g.ci, g.w), orc.Config())
        for lev in (0, 1):
            L = levels[lev]
            for world in (2, 3):
                for rank in range(world):
                    info = fd.fiedler_dist_plan(h, lev, world, rank)
                    ref, sidx, ridx = ref_plan(L.g.rp, L.g.ci, L.ncolors, world, rank)
                    assert [info.row_bounds[k] for k in range(world + 1)] == ref.bounds
                    assert [info.send_count[k] for k in range(world)] == ref.send_count
                    assert [info.recv_count[k] for k in range(world)] == ref.recv_count
                    x = torch.arange(L.g.n, dtype=torch.float64, device="cuda")
                    sb = torch.zeros(max(ref.send_total, 1), dtype=torch.float64, device="cuda")
                    # the op runs on the handle's (non-blocking) stream: inputs made
                    # on torch's stream must be complete first
                    torch.cuda.synchronize()
                    fd.fiedler_dist_op(h, lev, fd.FIEDLER_DOP_HALO_PACK, 0, x=x, y=sb)
                    torch.cuda.synchronize()
                    assert np.array_equal(sb[:ref.send_total].cpu().numpy().astype(np.int64), sidx)
                    rb = torch.arange(max(ref.recv_total, 1), dtype=torch.float64, device="cuda")
                    y = torch.full((L.g.n,), -1.0, dtype=torch.float64, device="cuda")
                    torch.cuda.synchronize()
                    fd.fiedler_dist_op(h, lev, fd.FIEDLER_DOP_HALO_UNPACK, 0, x=rb, y=y)
                    torch.cuda.synchronize()
                    got = y.cpu().numpy()
                    pos = np.flatnonzero(got >= 0)
                    assert np.array_equal(pos[np.argsort(got[pos])], ridx)
    finally:
        fd.fiedler_destroy(h)


@pytest.mark.parametrize("name", sorted(GRAPHS))
def test_single_rank_equals_fiedler_solve(fd, orc, name):
    import torch
    from paper_1602_04386_b200.dist import LibOps, LocalComm, PartitionedSolver
    g = GRAPHS[name]()
    h = _handle(fd, g)
    try:
        vec = torch.empty(g.n, dtype=torch.float64, device="cuda")
        lam_ref = fd.fiedler_solve(h, vec)
        v, lam, _ = PartitionedSolver(LibOps(h, torch.device("cuda")), LocalComm()).solve()
        torch.cuda.synchronize()
        assert abs(lam - lam_ref) / lam_ref <= 1e-12
        a, b = v.cpu().numpy(), vec.cpu().numpy()
        assert 1 - abs(a @ b) / (np.linalg.norm(a) * np.linalg.norm(b)) <= 1e-12
        assert np.allclose(a, b, rtol=0, atol=1e-10)
    finally:
        fd.fiedler_destroy(h)


@pytest.mark.parametrize("name,world", [("grid64x45", 2), ("rmat12", 3), ("hub", 2), ("grid3d_14", 4)])
def test_multi_rank_threads_match_oracle(fd, orc, name, world):
    import torch
    from dist_ref import ThreadComm, run_threads
    from paper_1602_04386_b200.dist import LibOps, PartitionedSolver
    g = GRAPHS[name]()
    ref = orc.solve(orc.Graph.from_csr(g.n, g.rp, g.ci, g.w), orc.Config())

    def rank_fn(rank, shared):
        h = _handle(fd, g)
        try:
            solver = PartitionedSolver(LibOps(h, torch.device("cuda")),
                                       ThreadComm(shared, rank, world, sync_cuda=True), min_rows=1)
            v, lam, res = solver.solve()
            torch.cuda.synchronize()
            return v.cpu().numpy(), lam, sum(solver.part)
        finally:
            fd.fiedler_destroy(h)

    out = run_threads(world, rank_fn)
    for v, lam, nparts in out:
        assert nparts >= 1
        assert abs(lam - ref.lambda2) / ref.lambda2 <= 1e-10
        cos = abs(float(v @ ref.vector)) / (np.linalg.norm(v) * np.linalg.norm(ref.vector))
        assert 1 - cos <= 1e-10
        assert np.allclose(v, ref.vector, rtol=0, atol=1e-9)


# ------------------------------------------------------------------ partitioned setup
def _setup_graph(g):
    import torch
    from paper_1602_04386_b200.dist import SetupGraph
    return SetupGraph(g.n, g.nnz, torch.from_numpy(g.rp).cuda(), torch.from_numpy(g.ci).cuda(),
                      torch.from_numpy(g.w).cuda())


def _check_presets(pres, levels, n_expected):
    assert len(pres) == n_expected
    for ell, p in enumerate(pres):
        L, Ln = levels[ell], levels[ell + 1]
        assert np.array_equal(p.q.cpu().numpy(), L.q), ell
        assert np.array_equal(p.mate.cpu().numpy(), L.mate), ell
        assert np.array_equal(p.colour.cpu().numpy(), L.color), ell
        assert p.ncolors == L.ncolors
        assert p.nxt.n == Ln.g.n and p.nxt.nnz == Ln.g.nnz
        assert np.array_equal(p.nxt.rp.cpu().numpy(), Ln.g.rp)
        assert np.array_equal(p.nxt.ci[:p.nxt.nnz].cpu().numpy(), Ln.g.ci)
        assert np.array_equal(p.nxt.w[:p.nxt.nnz].cpu().numpy(), Ln.g.w)


@pytest.mark.parametrize("name,world", [("grid64x45", 2), ("rmat12", 3), ("hub", 2), ("grid3d_14", 4),
                                        ("wcomplete300", 3)])
def test_partitioned_setup_and_solve_threads_match_oracle(fd, orc, name, world):
    """Ranks as threads on one GPU: the partitioned setup (fiedler_pset_*) gives
    the oracle's hierarchy bit for bit on every rank; fiedler_create_preset on it
    exports the oracle's levels; the partitioned solve on that handle matches
    the oracle's Fiedler vector."""
    import torch
    from dist_ref import ThreadComm, run_threads
    from paper_1602_04386_b200.dist import (LibOps, LibSetupOps, PartitionedSetup, PartitionedSolver,
                                            create_from_presets)
    g = GRAPHS[name]()
    og = orc.Graph.from_csr(g.n, g.rp, g.ci, g.w)
    levels = orc.build_hierarchy(og, orc.Config())
    ref = orc.solve(og, orc.Config(), levels=levels)

    def rank_fn(rank, shared):
        comm = ThreadComm(shared, rank, world, sync_cuda=True)
        ops = LibSetupOps(torch.device("cuda"))
        sg = _setup_graph(g)
        torch.cuda.synchronize()
        ps = PartitionedSetup(ops, comm, min_rows=1)
        ps.match_lists = rank % 2 == 0      # both matching schedules (lists / all rows) on the ranks
        pres = ps.run(sg)
        torch.cuda.synchronize()
        _check_presets(pres, levels, len(levels) - 1)
        opts = fd.fiedler_default_opts(stream=ops.stream)
        h = create_from_presets(sg, pres, opts)
        try:
            for ell in range(len(levels)):
                ex = fd.fiedler_level_export(h, ell)
                L = levels[ell]
                assert np.array_equal(ex["rp"], L.g.rp) and np.array_equal(ex["ci"], L.g.ci)
                assert np.array_equal(ex["w"], L.g.w) and np.array_equal(ex["color"], L.color)
                if L.q is not None:
                    assert np.array_equal(ex["agg"], L.q) and np.array_equal(ex["mate"], L.mate)
            solver = PartitionedSolver(LibOps(h, torch.device("cuda")), comm, min_rows=1)
            v, lam, _ = solver.solve()
            torch.cuda.synchronize()
            return v.cpu().numpy(), lam, ps.bytes_sent
        finally:
            fd.fiedler_destroy(h)

    for v, lam, sent in run_threads(world, rank_fn):
        assert sent > 0
        assert abs(lam - ref.lambda2) / ref.lambda2 <= 1e-10
        cos = abs(float(v @ ref.vector)) / (np.linalg.norm(v) * np.linalg.norm(ref.vector))
        assert 1 - cos <= 1e-10


@pytest.mark.parametrize("name", ["grid64x45", "rmat12", "hub"])
def test_single_rank_setup_equals_fiedler_create(fd, orc, name):
    """World size 1 (LocalComm): the pset kernels alone rebuild fiedler_create's
    hierarchy; min_rows cuts the partitioned prefix at a middle level."""
    import torch
    from paper_1602_04386_b200.dist import LibSetupOps, LocalComm, PartitionedSetup, create_from_presets
    g = GRAPHS[name]()
    levels = orc.build_hierarchy(orc.Graph.from_csr(g.n, g.rp, g.ci, g.w), orc.Config())
    ops = LibSetupOps(torch.device("cuda"))
    sg = _setup_graph(g)
    torch.cuda.synchronize()
    cut = levels[min(2, len(levels) - 1)].g.n
    pres = PartitionedSetup(ops, LocalComm(), min_rows=cut).run(sg)
    torch.cuda.synchronize()
    _check_presets(pres, levels, sum(1 for L in levels[:-1] if L.g.n >= cut))
    h = create_from_presets(sg, pres, fd.fiedler_default_opts(stream=ops.stream))
    h2 = _handle(fd, g)
    try:
        assert fd.fiedler_num_levels(h) == fd.fiedler_num_levels(h2) == len(levels)
        for ell in range(len(levels)):
            a, b = fd.fiedler_level_export(h, ell), fd.fiedler_level_export(h2, ell)
            for k in ("rp", "ci", "w", "color"):
                assert np.array_equal(a[k], b[k]), (ell, k)
        v1 = torch.empty(g.n, dtype=torch.float64, device="cuda")
        v2 = torch.empty(g.n, dtype=torch.float64, device="cuda")
        l1, l2 = fd.fiedler_solve(h, v1), fd.fiedler_solve(h2, v2)
        assert l1 == l2 and torch.equal(v1, v2)
    finally:
        fd.fiedler_destroy(h)
        fd.fiedler_destroy(h2)


def test_own_stream_reused_per_thread(fd):
    """The Ops objects' stream for a NULL caller stream is one per device and
    host thread: torch's caching allocator pools freed blocks per stream, so a
    fresh stream per solve would reuse none of the previous solve's buffers."""
    import threading
    import torch
    from paper_1602_04386_b200.dist import _own_stream
    dev = torch.device("cuda", 0)
    a, b = _own_stream(dev, 0), _own_stream(dev, None)
    assert a is b and a.cuda_stream != 0
    other = []
    t = threading.Thread(target=lambda: other.append(_own_stream(dev, 0)))
    t.start()
    t.join()
    assert other[0] is not a
    ext = _own_stream(dev, a.cuda_stream)   # a caller's real stream is used as it is
    assert ext.cuda_stream == a.cuda_stream
