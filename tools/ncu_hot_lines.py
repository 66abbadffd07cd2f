"""Warp-stall samples aggregated per CUDA source line (ncu --print-source cuda,sass).

    python tools/ncu_hot_lines.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
agg = collections.Counter()
text = {}
fname = None
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) != len(hdr) or not r[0].strip().isdigit():
        continue
    v = int(r[si]) if r[si].strip() else 0
    key = (fname, int(r[0]))
    agg[key] += v
    text[key] = r[1]
tot = sum(agg.values())
print("total samples", tot)
for (f, ln), v in agg.most_common(N):
    print(f"{100.0 * v / max(tot, 1):5.1f}% {f}:{ln:<5d} {text[(f, ln)].strip()[:100]}")
