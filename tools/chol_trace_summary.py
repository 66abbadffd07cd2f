"""Summarise ABD_TRACE_CHOL lines ([abd chol] n=...) per 5-step bucket of the window."""
import re
import sys

import numpy as np

rows = []
for line in open(sys.argv[1]):
    d = dict(re.findall(r"(\w[\w+]*)=([\d.e+-]+)", line))
    if "coupled" not in d:
        continue
    rows.append((int(d["coupled"]), int(d["largest"]), int(d["levels"]), float(d["factor+solve_ms"]),
                 float(d["analysis_ms"]), int(d["cached"]), int(d["ctas"]), int(d["updates"])))
R = np.array(rows)
per = int(sys.argv[2]) if len(sys.argv) > 2 else 320
print(f"{len(R)} factorizations")
for i in range(0, len(R), per):
    seg = R[i:i + per]
    print(f"[{i:5d}] coupled {seg[:, 0].mean():6.0f} largest {seg[:, 1].max():5.0f} levels {seg[:, 2].max():3.0f} "
          f"factor+solve ms {seg[:, 3].mean():.3f} analysis ms {seg[:, 4].mean():.3f} cached {seg[:, 5].mean():.2f} "
          f"updates {seg[:, 7].mean():.0f} ctas {seg[:, 6].mean():.0f}")
print(f"total factor+solve ms {R[:, 3].sum():.1f}, analysis (host) ms {R[:, 4].sum():.1f}")
