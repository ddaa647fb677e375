"""Device times of the setup phases per level (FIEDLER_PHASE_TIMES=1) of one
create + solve of a BASELINE config.  Usage: python tools/phase_times.py [config] [reps]"""
import os
import sys

os.environ["FIEDLER_PHASE_TIMES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = gg.config(cfg)
dev = torch.device("cuda", 0)
rp, ci, w = (torch.from_numpy(a).to(dev) for a in (g.rp, g.ci, g.w))
vec = torch.empty(g.n, dtype=torch.float64, device=dev)
for r in range(reps):
    info = fd.fiedler_info()
    h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, fd.fiedler_default_opts(validate=0))
    fd.fiedler_solve(h, vec, None, info)
    fd.fiedler_destroy(h)
tot = [0.0] * 4
print("config %d setup_ms %.2f solve_ms %.2f" % (cfg, info.setup_ms, info.solve_ms))
print("lvl        n        nnz  match_ms  galerkin_ms  colour_ms  layout_ms  rounds")
for i, L in enumerate(info.levels()):
    ph = (L["match_ms"], L["galerkin_ms"], L["colour_ms"], L["layout_ms"])
    tot = [a + b for a, b in zip(tot, ph)]
    print("%3d %9d %10d %9.3f %12.3f %10.3f %10.3f %7d" % ((i, L["n"], L["nnz"]) + ph + (L["match_rounds"],)))
print("sum %31.3f %12.3f %10.3f %10.3f" % tuple(tot))
