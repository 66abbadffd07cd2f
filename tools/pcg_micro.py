"""PCG per-iteration latency probe on ill-conditioned 12x12-block BSR matrices."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2201_10022_b200 import _native  # noqa: E402


def make(n, nbr=8, seed=0):
    rng = np.random.default_rng(seed)
    keys = set()
    for i in range(n):
        for d in range(1, nbr // 2 + 1):
            j = (i + d) % n
            if j != i:
                keys.add((min(i, j), max(i, j)))
    keys = np.array(sorted(keys), dtype=np.int64).reshape(-1, 2)
    off = -np.broadcast_to(np.eye(12), (len(keys), 12, 12)) * (1.0 + 0.1 * rng.random((len(keys), 1, 1)))
    deg = np.zeros(n)
    np.add.at(deg, keys[:, 0], 1.1)
    np.add.at(deg, keys[:, 1], 1.1)
    diag = (deg[:, None, None] + 1e-3) * np.eye(12)
    return diag, keys, np.ascontiguousarray(off)


for n in [int(x) for x in (sys.argv[1:] or ["1000", "10000", "100000"])]:
    diag, keys, off = make(n)
    b = np.random.default_rng(1).normal(size=12 * n)
    res = {}
    for mi in (1, 3000):
        best = 1e9
        for rep in range(2):
            t0 = time.perf_counter()
            x, it, rel = _native.bsr_pcg(n, 12, diag, keys, off, b, 1e-10, mi)
            best = min(best, time.perf_counter() - t0)
        res[mi] = (best, it, rel)
    per = (res[3000][0] - res[1][0]) / max(1, res[3000][1] - res[1][1])
    print(f"n={n} nnzb={n + 2 * len(keys)} iters={res[3000][1]} rel={res[3000][2]:.2e} per-iteration {per * 1e6:.2f} us",
          flush=True)
