#!/usr/bin/env python3
"""bench.py -- Fiedler solve throughput on B200 (driver contract).

One step = the whole hot path on one synthetic graph resident in HBM:
fiedler_create (Setup Phase: heavy-edge coarsening, prefix-scan numbering,
Galerkin products, colourings, solve layouts) + fiedler_solve (coarsest power
iteration, prolongation, multicolour Gauss-Seidel, shifted power iteration,
Rayleigh quotient) + fiedler_destroy, all through the C ABI.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Metric: fine-level Laplacian nonzeros (n + adjacency nnz) processed per second
by complete Fiedler solves, summed over ranks ("nnz/s", higher is better).
Default workload: BASELINE configs[4], the 8192 x 8192 grid quoted at
1/2/4/8 B200 (fits one GPU).  Prints ONE JSON line on rank 0.

The reference arm (--impl reference) times the oracle (oracle/, plain C,
single thread) on the host cores on a bounded sample of the same recipe.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import graphgen as gg  # noqa: E402

METRIC = "fiedler_solve_throughput (Fiedler solve time and SpMV/GS achieved HBM GB/s vs peak)"
UNIT = "nnz/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--kernel-reps", type=int, default=20)
    ap.add_argument("--sharded", action="store_true",
                    help="headline = the row-sharded step of one graph (default when --gpus > 1)")
    ap.add_argument("--partition-min-rows", type=int, default=1 << 20)
    ap.add_argument("--replicated-setup", action="store_true",
                    help="sharded step: fiedler_create on every rank instead of the partitioned setup")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks / throttle reasons during the timed region, sampled in-process
    through NVML (a light query every 100 ms; falls back to nvidia-smi)."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.stop_ev = threading.Event()
        self.t = None
        self.nvml = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.hdl = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:
            self.nvml = None
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nvml
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.hdl, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self.hdl, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.hdl)
                self.rows.append((sm, mx, rs))
            except Exception:
                pass
            self.stop_ev.wait(0.1)

    def stop(self):
        if self.nvml is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self.stop_ev.set()
        self.t.join(timeout=2)
        sm = [r[0] for r in self.rows]
        mx = [r[1] for r in self.rows]
        bits = [(name, getattr(self.nvml, attr, 0)) for name, attr in self.REASONS]
        reasons = sorted({name for r in self.rows for name, bit in bits if r[2] & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml"}


def cpu_sample_graph(config):
    """Bounded CPU sample of the same recipe (about 3-5 s of oracle work)."""
    if config in (1, 4):
        return gg.grid2d(1024, "uniform", seed=config), "grid2d 1024x1024 uniform[0.5,1.5] (same recipe, 1 solve)"
    if config == 2:
        return gg.rmat(17, 16.0, seed=2), "rmat scale 17 deg 16 lcc (same recipe, 1 solve)"
    if config == 3:
        return gg.grid3d(64, "lognormal", seed=3), "grid3d 64^3 lognormal(0,0.5) (same recipe, 1 solve)"
    return gg.grid2d(32, "unit"), "grid2d 32x32 unit (config 0 itself)"


def run_oracle_once(g):
    import oracle
    G = oracle.Graph.from_csr(g.n, g.rp, g.ci, g.w)
    t0 = time.perf_counter()
    r = oracle.solve(G, oracle.Config())
    dt = time.perf_counter() - t0
    return dt, r


def cpu_baseline(config, budget_s=10.0):
    """The oracle as it stands (single thread) on a bounded sample of the same
    recipe: whole solves repeated until ~budget_s of CPU work."""
    g, desc = cpu_sample_graph(config)
    tot, k = 0.0, 0
    while k == 0 or tot < budget_s:
        dt, _ = run_oracle_once(g)
        tot += dt
        k += 1
    return {"value": (g.n + g.nnz) * k / tot, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": desc.replace("1 solve", "%d solves" % k) + ", %.2f s wall" % tot}


def reference_arm(args, rank, world):
    """--impl reference: the oracle as it stands, on host cores, rank 0 only."""
    if rank != 0:
        return
    g, desc = cpu_sample_graph(args.config)
    for _ in range(max(args.warmup, 0)):
        run_oracle_once(g)
    times = []
    for _ in range(args.steps):
        dt, _ = run_oracle_once(g)
        times.append(dt)
    tot = sum(times)
    value = (g.n + g.nnz) * len(times) / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": gg.CONFIG_NAMES[args.config], "sample": desc},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def traffic_from_profiles():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except ValueError:
            return None
    return None


def phase_bytes(n, nnz, nc, nnzc):
    """Algorithmic bytes of the setup phases of one level:
    what a perfect kernel must move -- int32 CSR offsets / columns, f64 weights,
    int32 per-vertex outputs."""
    graph = 4 * (n + 1) + 12 * nnz          # rp, ci, w of the level
    pattern = 4 * (n + 1) + 4 * nnz         # rp, ci
    return {
        # read the graph; write mate, m (first pointer), aggregate id
        "match": graph + 12 * n,
        # read the fine graph and the aggregate ids; write the coarse CSR
        "galerkin": graph + 4 * n + (4 * (nc + 1) + 12 * nnzc if nc else 0),
        # read the pattern; write the colours
        "colour": pattern + 4 * n,
        # read the natural CSR and the colours; write the colour-permuted CSR, perm, inv
        "layout": 2 * graph + 12 * n,
    }


def setup_phase_rooflines(fd, n, nnz, rp, ci, w, opts, vec, peak):
    os.environ["FIEDLER_PHASE_TIMES"] = "1"
    try:
        info = fd.fiedler_info()
        hh = fd.fiedler_create(n, nnz, rp, ci, w, opts)
        fd.fiedler_solve(hh, vec, None, info)
        fd.fiedler_destroy(hh)
    finally:
        del os.environ["FIEDLER_PHASE_TIMES"]
    lv = info.levels()
    out = {"note": "device ms between CUDA events around each setup phase (one extra create with "
                   "FIEDLER_PHASE_TIMES=1, outside the timed region); the colouring runs on a second "
                   "stream, concurrently with the matching / Galerkin chain; algorithmic bytes: "
                   "DESIGN.md section 7", "setup_ms_this_create": info.setup_ms}
    tot = {k: 0.0 for k in ("match", "galerkin", "colour", "layout")}
    for i, L in enumerate(lv):
        for k in tot:
            tot[k] += L[k + "_ms"]
    out["all_levels_ms"] = tot
    L0 = lv[0]
    nc, nnzc = (lv[1]["n"], lv[1]["nnz"]) if len(lv) > 1 else (0, 0)
    by = phase_bytes(L0["n"], L0["nnz"], nc, nnzc)
    lvl0 = {}
    for k in tot:
        ms = L0[k + "_ms"]
        gbs = by[k] / (ms / 1e3) / 1e9 if ms > 0 else None
        lvl0[k] = {"ms": ms, "algorithmic_bytes": by[k], "GB/s": gbs,
                   "frac": (gbs / peak) if gbs else None}
    out["level0"] = lvl0
    return out


def sharded_step_timing(fd, g, rp, ci, w, dev, local, args, comm, dist):
    """The row-sharded step: fiedler_create (the setup,
    replicated on every rank) + the row-partitioned solve of ONE graph
    (paper_1602_04386_b200.dist, fine levels >= min_rows split across the
    ranks, NCCL halo exchange / all-reduce / all-gather).  Device time of every
    step between CUDA events on the stream everything runs on, max over ranks."""
    import torch
    from paper_1602_04386_b200.dist import (LibOps, LibSetupOps, PartitionedSetup, PartitionedSolver,
                                            SetupGraph, create_from_presets)
    stream = torch.cuda.current_stream(dev)
    opts = fd.fiedler_default_opts(device=local, validate=0, stream=stream.cuda_stream)
    info = {}
    sops = LibSetupOps(dev, stream=stream.cuda_stream)

    def create(rp, ci, w):
        """The setup: partitioned fine levels (fiedler_pset_*) + fiedler_create_preset,
        or (--replicated-setup) fiedler_create on every rank."""
        if args.replicated_setup:
            return fd.fiedler_create(g.n, g.nnz, rp, ci, w, opts)
        sg = SetupGraph(g.n, g.nnz, rp, ci, w)
        ps = PartitionedSetup(sops, comm, min_rows=args.partition_min_rows)
        pres = ps.run(sg)
        info.update(setup_levels_partitioned=len(pres), setup_bytes=ps.bytes_sent,
                    setup_rounds=[list(r) for r in ps.rounds])
        return create_from_presets(sg, pres, opts)

    def step():
        h = create(rp, ci, w)
        try:
            solver = PartitionedSolver(LibOps(h, dev, stream=stream.cuda_stream), comm,
                                       min_rows=args.partition_min_rows)
            _, lam, _ = solver.solve()
            info.update(lam=lam, levels_partitioned=int(sum(solver.part)),
                        halo_bytes=solver.halo_bytes_per_solve())
        finally:
            fd.fiedler_destroy(h)

    for _ in range(args.warmup):
        step()
    times = []
    ms0 = torch.cuda.memory_stats(dev)
    for _ in range(args.steps):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    tot = sum(times)
    ms1 = torch.cuda.memory_stats(dev)
    info["torch_allocator"] = {k: int(ms1.get(k, 0) - ms0.get(k, 0)) for k in
                               ("num_device_alloc", "num_device_free", "num_alloc_retries",
                                "reserved_bytes.all.current")}
    hb = float(info.get("halo_bytes", 0))
    sb = float(info.get("setup_bytes", 0))
    if dist:
        t = torch.tensor([tot, hb, sb], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot, hb, sb = float(t[0].item()), float(t[1].item()), float(t[2].item())
    ms = tot / args.steps
    return {"_create": create,
            "ms_per_step": ms, "step_ms": [round(t, 2) for t in times],
            "torch_allocator_in_timed_region": info.get("torch_allocator"), "lambda2": info.get("lam"), "levels_partitioned": info.get("levels_partitioned"),
            "setup": "replicated" if args.replicated_setup else "partitioned",
            "setup_levels_partitioned": info.get("setup_levels_partitioned", 0),
            "setup_rounds": info.get("setup_rounds"),
            "min_rows": args.partition_min_rows, "halo_bytes_per_step": hb + sb,
            "halo_bytes_solve": hb, "halo_bytes_setup": sb,
            "halo_GBps_effective": (hb + sb) / (ms / 1e3) / 1e9 if ms > 0 else None,
            "note": ("setup replicated on every rank" if args.replicated_setup else
                     "setup of the levels >= min_rows row-partitioned (fiedler_pset_*: matching / colouring "
                     "rounds with halo exchange, own coarse rows of the Galerkin product, all-gathered), "
                     "the coarser levels and the layouts by fiedler_create_preset on every rank") +
                    "; solve of one graph row-partitioned; "
                    "halo bytes = the most any rank sends per step (NCCL all-to-all / all-gather over NVLink); "
                    "GB/s = those bytes / the whole step time (a lower bound on the link rate)"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return

    import torch
    import paper_1602_04386_b200 as fd

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    g = gg.config(args.config)
    n, nnz = g.n, g.nnz
    nnz_L = n + nnz                      # Laplacian nonzeros incl. diagonal
    dev = torch.device("cuda", local)
    rp = torch.from_numpy(g.rp).to(dev)
    ci = torch.from_numpy(g.ci).to(dev)
    w = torch.from_numpy(g.w).to(dev)
    vec = torch.empty(n, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    opts = fd.fiedler_default_opts(device=local, validate=0, stream=stream.cuda_stream)
    # validate the input once (outside the timed region)
    h = fd.fiedler_create(n, nnz, rp, ci, w, fd.fiedler_default_opts(device=local, validate=1,
                                                                       stream=stream.cuda_stream))
    info = fd.fiedler_info()
    lam = fd.fiedler_solve(h, vec, None, info)
    fd.fiedler_destroy(h)
    l2_bytes = 126 * 2 ** 20
    big = (nnz * 12 + n * 12) > 2 * l2_bytes
    flush = None if big else torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev)

    def step():
        hh = fd.fiedler_create(n, nnz, rp, ci, w, opts)
        fd.fiedler_solve(hh, vec, None, info)
        fd.fiedler_destroy(hh)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    times = []
    launches = 0
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1.0)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        launches += info.launches + info.setup_launches
    ck = clocks.stop()
    tot_ms = sum(times)
    if dist:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    value = nnz_L * args.steps * world / (tot_ms / 1e3)
    setup_ms, solve_ms = info.setup_ms, info.solve_ms

    # ---- dominant-kernel roofline: level-0 power-iteration row pass (CUDA events)
    hh = fd.fiedler_create(n, nnz, rp, ci, w, opts)
    k_ms, k_bytes = fd.fiedler_level_time(hh, 0, fd.FIEDLER_OP_POWER, args.kernel_reps)
    gs_ms, gs_bytes = fd.fiedler_level_time(hh, 0, fd.FIEDLER_OP_GS_SWEEPS, args.kernel_reps)
    rq_ms, rq_bytes = fd.fiedler_level_time(hh, 0, fd.FIEDLER_OP_RAYLEIGH, args.kernel_reps)
    nlev = fd.fiedler_num_levels(hh)
    # the power step on the next levels (vectors and CSR smaller, still > L2 on config 4)
    pi_lv = {ell: fd.fiedler_level_time(hh, ell, fd.FIEDLER_OP_POWER, args.kernel_reps)
             for ell in (1, 2, 3) if ell < nlev - 1}
    fd.fiedler_destroy(hh)
    peak, peak_src = load_peaks()
    achieved = k_bytes / (k_ms / 1e3) / 1e9
    tr = traffic_from_profiles()
    traffic = None
    traffic_source = None
    if tr and tr.get("config") == args.config and tr.get("kernel_bytes_per_launch"):
        traffic = tr["kernel_bytes_per_launch"]
        traffic_source = tr.get("source")

    # algorithmic GB/s (the bytes a perfect kernel moves, per the DESIGN.md
    # formulas) and, where the committed ncu capture matches the config, the
    # measured DRAM GB/s (ncu bytes / this run's time)
    kernels = {"gs_sweep_level0": {"ms": gs_ms, "GB/s": gs_bytes / (gs_ms / 1e3) / 1e9,
                                   "frac": gs_bytes / (gs_ms / 1e3) / 1e9 / peak},
               "rayleigh_level0": {"ms": rq_ms, "GB/s": rq_bytes / (rq_ms / 1e3) / 1e9,
                                   "frac": rq_bytes / (rq_ms / 1e3) / 1e9 / peak}}
    for ell, (ms, by) in pi_lv.items():
        kernels["power_level%d" % ell] = {"ms": ms, "GB/s": by / (ms / 1e3) / 1e9,
                                          "frac": by / (ms / 1e3) / 1e9 / peak}
    if tr and tr.get("config") == args.config:
        for key, tkey, ms in (("gs_sweep_level0", "gs_sweep_dram_bytes", gs_ms),
                              ("rayleigh_level0", "rayleigh_dram_bytes", rq_ms)):
            if tr.get(tkey):
                kernels[key]["dram_GB/s"] = tr[tkey] / (ms / 1e3) / 1e9
                kernels[key]["dram_frac"] = tr[tkey] / (ms / 1e3) / 1e9 / peak
                kernels[key]["dram_bytes_source"] = tr.get("gs_rq_source")

    # ---- setup phases on the roofline: one extra create outside the timed
    # region with FIEDLER_PHASE_TIMES=1 (CUDA events around every phase of
    # every level, include/fiedler.h); algorithmic bytes per DESIGN.md section 7
    setup_kernels = setup_phase_rooflines(fd, n, nnz, rp, ci, w, opts, vec, peak)

    # ---- end to end through the public API with HOST buffers (pinned)
    prp = torch.from_numpy(g.rp).pin_memory()
    pci = torch.from_numpy(g.ci).pin_memory()
    pw = torch.from_numpy(g.w).pin_memory()
    pvec = torch.empty(n, dtype=torch.float64).pin_memory()
    eo = fd.fiedler_default_opts(device=local, validate=0, stream=stream.cuda_stream)

    def e2e_step():
        hh2 = fd.fiedler_create(n, nnz, prp, pci, pw, eo)
        fd.fiedler_solve(hh2, pvec, None, None)
        fd.fiedler_destroy(hh2)

    e2e_step()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        e2e_step()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = nnz_L * args.e2e_steps * world / e2e_s
    h2d = 8 * (n + 1) + 4 * nnz + 8 * nnz
    d2h = 8 * n + 8

    # ---- N > 1 (or --sharded): the headline is the row-sharded step of ONE
    # graph across the ranks (strong scaling); the
    # per-rank replica throughput measured above becomes a side field
    sharded = None
    if dist or args.sharded:
        from paper_1602_04386_b200.dist import LocalComm, TorchComm
        comm = TorchComm() if dist else LocalComm()
        sharded = sharded_step_timing(fd, g, rp, ci, w, dev, local, args, comm, dist)
        create_fn = sharded.pop("_create")
        # end to end: pinned host CSR in, Fiedler vector back to the host, wall clock, max over ranks
        from paper_1602_04386_b200.dist import LibOps, PartitionedSolver

        def e2e_sharded():
            if args.replicated_setup:
                hh2 = fd.fiedler_create(n, nnz, prp, pci, pw, eo)
            else:   # the partitioned setup works on device arrays: copy the host CSR in first
                drp, dci, dw = (x.to(dev, non_blocking=True) for x in (prp, pci, pw))
                hh2 = create_fn(drp, dci, dw)
            try:
                sv = PartitionedSolver(LibOps(hh2, dev, stream=stream.cuda_stream), comm,
                                       min_rows=args.partition_min_rows)
                vv, _, _ = sv.solve()
                pvec.copy_(vv)
            finally:
                fd.fiedler_destroy(hh2)
        e2e_sharded()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_sharded()
        torch.cuda.synchronize()
        es = time.perf_counter() - t0
        if dist:
            t = torch.tensor([es], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            es = float(t.item())
        sharded["e2e"] = {"value": nnz_L * args.e2e_steps / es, "unit": UNIT, "h2d_bytes_per_step": h2d,
                          "d2h_bytes_per_step": 8 * n}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": gg.CONFIG_NAMES[args.config], "n": n, "adjacency_nnz": nnz,
                       "laplacian_nnz": nnz_L, "levels": nlev, "gs_sweeps": 2, "power_iters": 10,
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": ("inputs larger than L2 (no flush)" if big else "L2 flushed between steps")},
            "solve_time_ms": tot_ms / args.steps, "setup_ms": setup_ms, "solve_ms": solve_ms,
            "lambda2": lam,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_source,
                         "kernel": "k_tilepass<OP_PI> level 0 (one power-iteration step)",
                         "algorithmic_bytes_per_launch": k_bytes, "launch_ms": k_ms,
                         "peak_source": peak_src},
            "kernels": kernels,
            "setup_kernels": setup_kernels,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": ck,
        }
        if sharded is not None:
            line["replicas"] = {"value": value, "ms_per_step": tot_ms / args.steps, "scaling": "weak",
                                "e2e": line["e2e"],
                                "note": "every rank solves its own copy of the graph (no communication)"}
            line["value"] = nnz_L * 1.0 / (sharded["ms_per_step"] / 1e3)
            line["ms_per_step"] = sharded["ms_per_step"]
            line["solve_time_ms"] = sharded["ms_per_step"]
            line["scaling"] = "strong"
            line["config"]["parallelism"] = "row-sharded fine levels over %d GPU(s), setup %s" % (
                world, "replicated" if args.replicated_setup else "partitioned")
            line["sharded"] = sharded
            line["e2e"] = sharded.pop("e2e")
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
