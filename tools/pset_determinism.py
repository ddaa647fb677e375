"""Repeat the partitioned setup of a BASELINE config's level 0 (one rank) and
compare every result with the first repetition: python tools/pset_determinism.py CONFIG REPS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
from paper_1602_04386_b200.dist import LibSetupOps, LocalComm, PartitionedSetup, SetupGraph  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
g = gg.config(cfg)
dev = torch.device("cuda")
sg = SetupGraph(g.n, g.nnz, torch.from_numpy(g.rp).to(dev), torch.from_numpy(g.ci).to(dev),
                torch.from_numpy(g.w).to(dev))
ops = LibSetupOps(dev)
first = None
bad = 0
for rep in range(reps):
    ps = PartitionedSetup(ops, LocalComm(), min_rows=g.n)
    p = ps.run(sg)[0]
    torch.cuda.synchronize()
    cur = dict(mate=p.mate.clone(), q=p.q.clone(), colour=p.colour.clone(), rp=p.nxt.rp.clone(),
               ci=p.nxt.ci[:p.nxt.nnz].clone(), w=p.nxt.w[:p.nxt.nnz].clone())
    if first is None:
        first = cur
        print("rep 0 rounds", ps.rounds, flush=True)
        continue
    diff = {k: int((cur[k] != first[k]).sum()) if cur[k].shape == first[k].shape else -1 for k in cur}
    if any(diff.values()):
        bad += 1
        print("rep", rep, "rounds", ps.rounds, "DIFF", diff, flush=True)
print("reps", reps, "mismatching", bad)
