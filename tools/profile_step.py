"""One create + solve + destroy of a BASELINE config on cuda:0 (for ncu / nsys-less
launch lists).  Usage: python tools/profile_step.py [config] [--twice]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 4
g = gg.config(cfg)
dev = torch.device("cuda", 0)
rp, ci, w = (torch.from_numpy(a).to(dev) for a in (g.rp, g.ci, g.w))
vec = torch.empty(g.n, dtype=torch.float64, device=dev)
opts = fd.fiedler_default_opts(validate=0, use_graph=0)
for _ in range(2 if "--twice" in sys.argv else 1):
    info = fd.fiedler_info()
    h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, opts)
    lam = fd.fiedler_solve(h, vec, opts, info)
    fd.fiedler_destroy(h)
torch.cuda.synchronize()
print("config", cfg, "n", g.n, "lambda2", lam, "setup_ms", info.setup_ms, "solve_ms", info.solve_ms,
      "setup_launches", info.setup_launches, "launches", info.launches)
for i, L in enumerate(info.levels()):
    print(i, L)
