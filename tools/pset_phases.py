"""Phase times of the partitioned setup (dist.PartitionedSetup) on one GPU
(LocalComm: one rank owns every row), for a BASELINE config:
python tools/pset_phases.py CONFIG [MIN_ROWS]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402
from paper_1602_04386_b200.dist import (LibSetupOps, LocalComm, PartitionedSetup, SetupGraph,  # noqa: E402
                                        create_from_presets)

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
min_rows = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
g = gg.config(cfg)
dev = torch.device("cuda")
sg = SetupGraph(g.n, g.nnz, torch.from_numpy(g.rp).to(dev), torch.from_numpy(g.ci).to(dev),
                torch.from_numpy(g.w).to(dev))
ops = LibSetupOps(dev)
for rep in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    torch.cuda.synchronize()
    ps = PartitionedSetup(ops, LocalComm(), min_rows=min_rows)
    ps.phase_times = {}
    t0 = time.perf_counter()
    pres = ps.run(sg)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h = create_from_presets(sg, pres, fd.fiedler_default_opts(stream=ops.stream, validate=0))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    fd.fiedler_destroy(h)
    print(json.dumps({"config": cfg, "rep": rep, "pset_ms": (t1 - t0) * 1e3, "create_preset_ms": (t2 - t1) * 1e3,
                      "rounds": ps.rounds,
                      "phases": {k: {a: round(b, 2) for a, b in v.items()} for k, v in ps.phase_times.items()}}))
