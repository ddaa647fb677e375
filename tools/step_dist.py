"""Distribution of bench-style step times (create + solve + destroy, CUDA
events on the caller's stream) over many reps: median, mean, outliers.
Usage: python tools/step_dist.py [config] [reps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
g = gg.config(cfg)
dev = torch.device("cuda", 0)
rp, ci, w = (torch.from_numpy(a).to(dev) for a in (g.rp, g.ci, g.w))
vec = torch.empty(g.n, dtype=torch.float64, device=dev)
stream = torch.cuda.current_stream(dev)
opts = fd.fiedler_default_opts(validate=0, stream=stream.cuda_stream)
ts, su, so = [], [], []
for r in range(reps + 3):
    info = fd.fiedler_info()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, opts)
    fd.fiedler_solve(h, vec, None, info)
    fd.fiedler_destroy(h)
    e1.record(stream)
    torch.cuda.synchronize()
    if r >= 3:
        ts.append(e0.elapsed_time(e1))
        su.append(info.setup_ms)
        so.append(info.solve_ms)
med = statistics.median(ts)
out = [(i, round(t, 1), round(a, 1), round(b, 1)) for i, (t, a, b) in enumerate(zip(ts, su, so)) if t > med + 3]
print("cfg %d reps %d median %.2f mean %.2f | setup median %.2f solve median %.2f | outliers (step, setup, solve): %s"
      % (cfg, reps, med, statistics.mean(ts), statistics.median(su), statistics.median(so), out))
