"""Per-CUDA-source-line warp-stall samples of one kernel in an ncu report
(compiled with -lineinfo).  Usage: python tools/ncu_lines.py report kernel_regex [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre, "--launch-count", "1"], capture_output=True, text=True).stdout
samples, text = Counter(), {}
fname, hdr = "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 5 or not r[0].strip().isdigit():
        continue
    try:
        s = int(r[4] or 0)
    except ValueError:
        continue
    key = "%s:%s" % (fname, r[0])
    samples[key] += s
    text[key] = r[1].strip()[:100]
tot = sum(samples.values()) or 1
for k, s in samples.most_common(top):
    print("%6.2f%% %-22s %s" % (100.0 * s / tot, k, text[k]))
