"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
with open(path) as f:
    lines = [ln for ln in f if not ln.startswith("==")]
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for row in csv.DictReader(lines):
    if row.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = row["Kernel Name"].split("(")[0]
    v = float(row["Metric Value"].replace(",", "")) * scale[row["Metric Unit"]]
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print("total %.1f us over %d launches" % (tot, sum(a[0] for a in agg.values())))
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print("%10.1f us %5.1f%% %6d  %s" % (t, 100 * t / tot, c, k))
