"""One create + solve + destroy of a BASELINE config on cuda:0 (for ncu launch
lists), with host wall-clock of each call.  Usage: python tools/profile_step.py [config] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = gg.config(cfg)
dev = torch.device("cuda", 0)
rp, ci, w = (torch.from_numpy(a).to(dev) for a in (g.rp, g.ci, g.w))
vec = torch.empty(g.n, dtype=torch.float64, device=dev)
opts = fd.fiedler_default_opts(validate=0, use_graph=0)
for r in range(reps):
    info = fd.fiedler_info()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, opts)
    t1 = time.perf_counter()
    lam = fd.fiedler_solve(h, vec, opts, info)
    t2 = time.perf_counter()
    fd.fiedler_destroy(h)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print("rep %d host ms: create %.2f solve %.2f destroy %.2f total %.2f" %
          (r, 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t3 - t0)))
print("config", cfg, "n", g.n, "lambda2", lam, "setup_ms", info.setup_ms, "solve_ms", info.solve_ms,
      "setup_launches", info.setup_launches, "launches", info.launches)
for i, L in enumerate(info.levels()):
    print(i, L)
