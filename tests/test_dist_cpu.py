"""CPU multi-process tests of the partitioned solve's host logic
(paper_1602_04386_b200/dist.py): world size 2 and 3 over gloo, the driver with
the reference operations of tests/dist_ref.py on the oracle's hierarchy.  The
end result must equal the oracle's single-process solve (north-star bars)."""
import os
import socket

import numpy as np
import pytest

import graphgen as gg




def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _graph(name):
    return {"grid": lambda: gg.grid2d(24, "uniform", seed=3, mx=17),
            "rand": lambda: gg.random_connected(300, 700, 5),
            "hub": lambda: gg.hub_graph(400, 500, hubs=2, seed=1),
            "unitgrid": lambda: gg.grid2d(20, "unit", seed=0, mx=13)}[name]()   # all weights tie (R2 hash order)


def _worker(rank, world, port, name, gs, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from dist_ref import RefOps
        from paper_1602_04386_b200.dist import PartitionedSolver, TorchComm
        g = _graph(name)
        og = oracle.Graph.from_csr(g.n, g.rp, g.ci, g.w)
        levels = oracle.build_hierarchy(og, oracle.Config())
        solver = PartitionedSolver(RefOps(levels), TorchComm(), min_rows=1)
        v, lam, res = solver.solve(gs_sweeps=gs)
        q.put((rank, v.numpy().copy(), lam, res, [p.row_begin for p in solver.plans],
               sum(solver.part)))
    finally:
        dist.destroy_process_group()


def _run(world, name, gs=2):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, gs, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get() for _ in range(world)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("world,name,gs", [(2, "grid", 2), (3, "rand", 2), (2, "hub", 2), (2, "grid", 0)])
def test_partitioned_driver_matches_oracle(orc, world, name, gs):
    g = _graph(name)
    ref = orc.solve(orc.Graph.from_csr(g.n, g.rp, g.ci, g.w), orc.Config(gs_sweeps=gs))
    res = _run(world, name, gs)
    for rank, v, lam, resid, row_begins, nparts in res:
        assert nparts >= 1, "no level was partitioned"
        assert abs(lam - ref.lambda2) / ref.lambda2 <= 1e-10
        cos = abs(float(v @ ref.vector)) / (np.linalg.norm(v) * np.linalg.norm(ref.vector))
        assert 1 - cos <= 1e-10
        assert np.allclose(v, ref.vector, rtol=0, atol=1e-9)     # sign convention R10 included
    # every rank returns the same vector and eigenvalue
    for r in res[1:]:
        assert np.array_equal(r[1], res[0][1]) and r[2] == res[0][2]


def test_ref_plan_halo_lists_are_consistent():
    """Rank p's send list to rank r equals rank r's recv list from rank p."""
    from dist_ref import ref_plan
    g = _graph("rand")
    for world in (2, 3, 5):
        plans = [ref_plan(g.rp, g.ci, 1, world, r) for r in range(world)]
        for r in range(world):
            pr, sr, rr = plans[r]
            assert pr.bounds[0] == 0 and pr.bounds[-1] == g.n
            assert all(a <= b for a, b in zip(pr.bounds, pr.bounds[1:]))
            roff = np.cumsum([0] + pr.recv_count)
            for p in range(world):
                pp, sp, _ = plans[p]
                soff = np.cumsum([0] + pp.send_count)
                assert np.array_equal(sp[soff[r]:soff[r + 1]], rr[roff[p]:roff[p + 1]])


def test_local_comm_single_rank(orc):
    """World size 1: the driver runs every level whole and equals the oracle."""
    from dist_ref import RefOps
    from paper_1602_04386_b200.dist import LocalComm, PartitionedSolver
    g = _graph("grid")
    og = orc.Graph.from_csr(g.n, g.rp, g.ci, g.w)
    ref = orc.solve(og, orc.Config())
    v, lam, _ = PartitionedSolver(RefOps(orc.build_hierarchy(og, orc.Config())), LocalComm()).solve()
    assert abs(lam - ref.lambda2) / ref.lambda2 <= 1e-10
    assert np.allclose(v.numpy(), ref.vector, rtol=0, atol=1e-9)


# ------------------------------------------------------------------ partitioned setup
def _setup_worker(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_ref import RefSetupOps
        from paper_1602_04386_b200.dist import PartitionedSetup, SetupGraph, TorchComm
        g = _graph(name)
        sg = SetupGraph(g.n, g.nnz, torch.from_numpy(g.rp), torch.from_numpy(g.ci), torch.from_numpy(g.w))
        ps = PartitionedSetup(RefSetupOps(), TorchComm(), min_rows=1)
        pres = ps.run(sg)
        q.put((rank, [(p.q[:p.q.numel()].numpy().copy(), p.mate.numpy().copy(), p.colour.numpy().copy(),
                       p.ncolors, p.nxt.rp.numpy().copy(), p.nxt.ci[:p.nxt.nnz].numpy().copy(),
                       p.nxt.w[:p.nxt.nnz].numpy().copy(), p.row_bounds) for p in pres], ps.bytes_sent))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "grid"), (3, "rand"), (2, "hub"), (3, "unitgrid")])
def test_partitioned_setup_matches_oracle_hierarchy(orc, world, name):
    """Every partitioned level's matching, aggregates, colouring and coarse
    level equal the oracle's hierarchy bit for bit, on every rank."""
    import torch.multiprocessing as mp
    g = _graph(name)
    levels = orc.build_hierarchy(orc.Graph.from_csr(g.n, g.rp, g.ci, g.w), orc.Config())
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_setup_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get() for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    for rank, pres, sent in out:
        assert len(pres) == len(levels) - 1, "every coarsened level is partitioned (min_rows=1)"
        assert sent > 0
        for ell, (qv, mate, col, ncol, rp, ci, w, bounds) in enumerate(pres):
            L, Ln = levels[ell], levels[ell + 1]
            assert len(set(bounds)) > 2 or L.g.n < world, "rows split across ranks"
            assert np.array_equal(qv, L.q) and np.array_equal(mate, L.mate)
            assert np.array_equal(col, L.color) and ncol == L.ncolors
            assert np.array_equal(rp, Ln.g.rp) and np.array_equal(ci, Ln.g.ci)
            assert np.array_equal(w, Ln.g.w)     # bit for bit (R3 summation order)
