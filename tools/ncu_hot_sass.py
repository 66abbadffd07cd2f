"""Top SASS lines by warp-stall samples for one kernel of an ncu report.

    python tools/ncu_hot_sass.py REPORT.ncu-rep KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 20
raw = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, row in enumerate(r) if "Warp Stall Sampling (All Samples)" in row)
h = r[hi]
si = h.index("Warp Stall Sampling (All Samples)")
rows = []
for x in r[hi + 1:]:
    if len(x) != len(h) or x[si] == h[si]:
        if rows:
            break  # first kernel instance only
        continue
    rows.append(x)
v = lambda x: int(x[si]) if x[si].strip() else 0  # noqa: E731
tot = sum(v(x) for x in rows)
print("total samples", tot, "instructions", len(rows))
top = sorted(range(len(rows)), key=lambda i: -v(rows[i]))[:N]
for i in sorted(top):
    print(f"{i:5d} {v(rows[i]):7d} {100.0 * v(rows[i]) / max(tot, 1):5.1f}%  {rows[i][1][:70]:70s} | prev: {rows[i - 1][1][:40]}")
