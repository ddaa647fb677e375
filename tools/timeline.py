"""GPU timeline of one fiedler_create + fiedler_solve (CUPTI kernel activity via
torch.profiler): real (concurrent, warm) kernel durations, per-stream busy time,
and the idle gaps of the device.  Usage: python tools/timeline.py [config] [warm_reps]"""
import json
import os
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = gg.config(cfg)
dev = torch.device("cuda", 0)
rp, ci, w = (torch.from_numpy(a).to(dev) for a in (g.rp, g.ci, g.w))
vec = torch.empty(g.n, dtype=torch.float64, device=dev)
opts = fd.fiedler_default_opts(validate=0, use_graph=0)


def once():
    h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, opts)
    fd.fiedler_solve(h, vec, opts, fd.fiedler_info())
    fd.fiedler_destroy(h)


for _ in range(warm):
    once()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    once()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
kern = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
kern.sort(key=lambda e: e["ts"])
t0 = kern[0]["ts"]
t1 = max(e["ts"] + e["dur"] for e in kern)
# union of busy intervals and the gaps between them
busy = 0.0
gaps = []
cur_s, cur_e = kern[0]["ts"], kern[0]["ts"] + kern[0]["dur"]
for e in kern[1:]:
    s, f = e["ts"], e["ts"] + e["dur"]
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, cur_e - t0, e["name"][:60]))
        cur_s, cur_e = s, f
    else:
        cur_e = max(cur_e, f)
busy += cur_e - cur_s
print("config %d: span %.1f us, busy %.1f us, idle %.1f us in %d gaps, %d activities" %
      (cfg, t1 - t0, busy, t1 - t0 - busy - 0, len(gaps), len(kern)))
per_stream = defaultdict(float)
for e in kern:
    per_stream[e.get("args", {}).get("stream", -1)] += e["dur"]
print("per-stream busy (us):", {k: round(v, 1) for k, v in per_stream.items()})
tot = defaultdict(lambda: [0.0, 0])
for e in kern:
    nm = e["name"].split("(")[0][:70]
    tot[nm][0] += e["dur"]
    tot[nm][1] += 1
print("%-72s %10s %6s" % ("kernel", "us", "count"))
for nm, (d, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:45]:
    print("%-72s %10.1f %6d" % (nm, d, c))
gaps.sort(reverse=True)
print("largest gaps (us, at us, next activity):")
for gp in gaps[:25]:
    print("  %8.1f %10.1f  %s" % gp)
hist = defaultdict(lambda: [0, 0.0])
for d, _, _ in gaps:
    b = "<5" if d < 5 else "<20" if d < 20 else "<100" if d < 100 else ">=100"
    hist[b][0] += 1
    hist[b][1] += d
print("gap histogram:", dict(hist))
# solve-phase split: first k_rand marks the start of the solve
rs = [e["ts"] for e in kern if e["name"].startswith("k_rand")]
if rs:
    print("setup span %.1f us, solve span %.1f us" % (rs[0] - t0, t1 - rs[0]))
