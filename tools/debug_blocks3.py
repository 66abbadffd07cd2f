import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
from paper_2201_10022_b200 import _native
from golden_io import oracle_bodies
from oracle import abd_oracle as O
g = dict(np.load("tests/golden/contact.npz"))
p = "twocube_"
ob = oracle_bodies(p, g)
d_hat, kappa, mu, _, _, dt = g[p + "params"]
X = O.all_world_points(ob, g[p + "q0"])
ra, d2, val, g12, H12, rp = O.contact_pair_terms("ee", ob, X, g[p + "c0_ee"], kappa, d_hat)
z, _, eps = O.gather("ee", ob, X, ra)
dyn2 = np.ones((len(ra), 2), dtype=np.uint8)
g12g, h12g, _, _ = _native.contact_pair_batch("ee", z, rp, eps, kappa, d_hat, dyn2, project=2)
bad = 0
for k in range(len(ra)):
    e = np.linalg.norm(h12g[k] - H12[k]) / np.linalg.norm(H12[k])
    eg = np.linalg.norm(g12g[k] - g12[k]) / np.linalg.norm(g12[k])
    if e > 1e-9 or eg > 1e-9:
        bad += 1
        print("H12 mismatch", k, e, eg)
print("stage2 bad", bad, flush=True)
_, _, g24, h24 = _native.contact_pair_batch("ee", z, rp, eps, kappa, d_hat, dyn2, project=0)
print("stage map ok", flush=True)
