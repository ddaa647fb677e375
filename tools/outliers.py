"""Find what makes an occasional create slow: CUPTI kernel records over many
create+solve+destroy reps (torch.profiler), per-rep span, and for the slowest
rep the kernels / gaps that exceed the median rep.
Usage: python tools/outliers.py [config] [reps]"""
import json
import os
import sys
import tempfile
import time
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import graphgen as gg  # noqa: E402
import paper_1602_04386_b200 as fd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
g = gg.config(cfg)
dev = torch.device("cuda", 0)
rp, ci, w = (torch.from_numpy(a).to(dev) for a in (g.rp, g.ci, g.w))
vec = torch.empty(g.n, dtype=torch.float64, device=dev)
opts = fd.fiedler_default_opts(validate=0, use_graph=0)


def once():
    h = fd.fiedler_create(g.n, g.nnz, rp, ci, w, opts)
    fd.fiedler_solve(h, vec, opts, fd.fiedler_info())
    fd.fiedler_destroy(h)


for _ in range(2):
    once()
torch.cuda.synchronize()
host = []
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        t0 = time.perf_counter()
        once()
        torch.cuda.synchronize()
        host.append(1e3 * (time.perf_counter() - t0))
path = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
kern = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e],
              key=lambda e: e["ts"])
# reps split at the k_rp64_to_32 / first kernel of each create: use k_rand (solve start) as anchor
starts = [e["ts"] for e in kern if e["name"].startswith("fdl::k_member_count_deg")]
print("host ms per rep:", [round(x, 1) for x in host])
# group kernels into reps by the host-ordered sequence of k_rand (one per solve)
rand_ts = [e["ts"] for e in kern if "k_rand" in e["name"]]
bounds = [kern[0]["ts"]] + [t + 1 for t in rand_ts]
per = []
for r in range(len(rand_ts)):
    lo = bounds[r] if r == 0 else rand_ts[r - 1] + 1
    hi = rand_ts[r]
    ks = [e for e in kern if lo <= e["ts"] < hi]
    tot = defaultdict(float)
    for e in ks:
        tot[e["name"].split("(")[0][:60]] += e["dur"]
    span = (ks[-1]["ts"] + ks[-1]["dur"] - ks[0]["ts"]) if ks else 0
    per.append((span, tot, ks))
spans = [p[0] for p in per]
print("setup spans (us):", [round(x) for x in spans])
med = sorted(range(len(per)), key=lambda i: spans[i])[len(per) // 2]
worst = max(range(len(per)), key=lambda i: spans[i])
print("median rep", med, "worst rep", worst)
diff = []
for k in set(per[worst][1]) | set(per[med][1]):
    diff.append((per[worst][1].get(k, 0) - per[med][1].get(k, 0), k))
diff.sort(reverse=True)
for d, k in diff[:12]:
    print("  %+9.1f us  %s" % (d, k))
ks = per[worst][2]
gaps = []
for a, b in zip(ks, ks[1:]):
    gp = b["ts"] - (a["ts"] + a["dur"])
    if gp > 200:
        gaps.append((gp, a["name"][:50], b["name"][:50]))
gaps.sort(reverse=True)
print("gaps > 200 us in the worst rep:", [(round(x[0]), x[1], x[2]) for x in gaps[:8]])
