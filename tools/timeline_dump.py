"""Dump the GPU activity (kernels, memsets, copies: name, stream, start, duration
in us) of one warm fiedler_create of a BASELINE config, recorded with CUPTI via
torch.profiler.  Usage: python tools/timeline_dump.py [config] [out.json]"""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
what = sys.argv[2] if len(sys.argv) > 2 else "create"          # create | solve
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/timeline_%s_c%d.json" % (what, cfg)
g = gg.config(cfg)
dev = torch.device("cuda", 0)
rp, ci, w = (torch.from_numpy(a).to(dev) for a in (g.rp, g.ci, g.w))
opts = fd.fiedler_default_opts(validate=0, use_graph=0)
for _ in range(2):
    fd.fiedler_destroy(fd.fiedler_create(g.n, g.nnz, rp, ci, w, opts))
torch.cuda.synchronize()
if what in ("solve", "first_solve"):
    h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, opts)
    vec = torch.empty(g.n, dtype=torch.float64, device=dev)
    if what == "solve":     # a repeated solve (the first one also finishes the deferred level 0)
        fd.fiedler_solve(h, vec, opts, None)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fd.fiedler_solve(h, vec, opts, None)
        torch.cuda.synchronize()
else:
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, opts)
        torch.cuda.synchronize()
fd.fiedler_destroy(h)
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
rows = [(e["name"], e.get("tid"), float(e["ts"]), float(e.get("dur", 0)), e.get("cat"))
        for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
rows.sort(key=lambda r: r[2])
t0 = rows[0][2] if rows else 0.0
json.dump([(n, s, ts - t0, d, c) for n, s, ts, d, c in rows], open(out, "w"))
print("events", len(rows), "span_us", rows[-1][2] + rows[-1][3] - t0 if rows else 0)
