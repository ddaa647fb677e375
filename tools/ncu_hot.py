"""Hottest SASS lines (warp stall samples) of one kernel in an ncu report.
Usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
# first line is the kernel name; the rest is one CSV table (first kernel only)
body = []
for ln in lines[1:]:
    if ln.startswith('"Kernel Name"'):
        break
    body.append(ln)
r = list(csv.reader(io.StringIO("\n".join(body))))
h = r[0]
isrc = h.index("Source")
isamp = h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(x[isamp] or 0) for x in r[1:])
print("kernel:", lines[0][:150])
print("total samples", tot)
rows = sorted(r[1:], key=lambda x: -float(x[isamp] or 0))[:top]
for x in rows:
    print("%6.1f%%  %s" % (100 * float(x[isamp] or 0) / tot, x[isrc].strip()[:100]))
