"""create + solve + destroy per step (as bench.py times it), solve with and
without CUDA-graph capture; CUDA events on the caller's stream.
Usage: python tools/graph_ab.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = gg.config(cfg)
dev = torch.device("cuda", 0)
rp, ci, w = (torch.from_numpy(a).to(dev) for a in (g.rp, g.ci, g.w))
vec = torch.empty(g.n, dtype=torch.float64, device=dev)
stream = torch.cuda.current_stream(dev)
for ug in (1, 0, 1, 0):
    opts = fd.fiedler_default_opts(validate=0, use_graph=ug, stream=stream.cuda_stream)
    ts = []
    for r in range(reps + 2):
        info = fd.fiedler_info()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, opts)
        fd.fiedler_solve(h, vec, None, info)
        fd.fiedler_destroy(h)
        e1.record(stream)
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    print("use_graph=%d step ms: mean %.2f min %.2f max %.2f | setup %.2f solve %.2f" %
          (ug, sum(ts) / len(ts), min(ts), max(ts), info.setup_ms, info.solve_ms))
