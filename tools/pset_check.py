"""Partitioned setup (one rank) + fiedler_create_preset + partitioned solve
on a BASELINE config, from pinned host arrays copied in, against
fiedler_create + fiedler_solve on the same graph (lambda_2, vector, levels):
python tools/pset_check.py CONFIG [MIN_ROWS] [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402
from paper_1602_04386_b200.dist import (LibOps, LibSetupOps, LocalComm, PartitionedSetup,  # noqa: E402
                                        PartitionedSolver, SetupGraph, create_from_presets)

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
min_rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = gg.config(cfg)
dev = torch.device("cuda")
stream = torch.cuda.current_stream(dev)
host = [torch.from_numpy(a).pin_memory() for a in (g.rp, g.ci, g.w)]
opts = fd.fiedler_default_opts(validate=0, stream=stream.cuda_stream)
ref_h = fd.fiedler_create(g.n, g.nnz, *[x.to(dev) for x in host], opts)
ref_v = torch.empty(g.n, dtype=torch.float64, device=dev)
ref_l = fd.fiedler_solve(ref_h, ref_v)
sops = LibSetupOps(dev, stream=stream.cuda_stream)
for rep in range(reps):
    drp, dci, dw = (x.to(dev, non_blocking=True) for x in host)
    sg = SetupGraph(g.n, g.nnz, drp, dci, dw)
    ps = PartitionedSetup(sops, LocalComm(), min_rows=min_rows)
    pres = ps.run(sg)
    torch.cuda.synchronize()
    print("rep", rep, "presets", len(pres), "rounds", ps.rounds, flush=True)
    h = create_from_presets(sg, pres, opts)
    torch.cuda.synchronize()
    for ell in range(len(pres) + 1):
        a, b = fd.fiedler_level_export(h, ell), fd.fiedler_level_export(ref_h, ell)
        for k in ("rp", "ci", "w", "color", "agg", "mate"):
            if ell == len(pres) and k in ("agg", "mate"):
                continue
            assert np.array_equal(a[k], b[k]), (rep, ell, k)
    print("rep", rep, "levels equal", flush=True)
    sv = PartitionedSolver(LibOps(h, dev, stream=stream.cuda_stream), LocalComm(), min_rows=min_rows)
    v, lam, _ = sv.solve()
    torch.cuda.synchronize()
    print("rep", rep, "lambda", lam, ref_l, "max|dv|", float((v - ref_v).abs().max()), flush=True)
    fd.fiedler_destroy(h)
fd.fiedler_destroy(ref_h)
print("ok")
