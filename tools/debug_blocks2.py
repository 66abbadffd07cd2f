import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import paper_2201_10022_b200 as P  # noqa: E402
from paper_2201_10022_b200 import _native  # noqa: E402
from golden_io import oracle_bodies, unpack_meshes  # noqa: E402
from oracle import abd_oracle as O  # noqa: E402

g = dict(np.load("tests/golden/contact.npz"))
p = "twocube_"
ob = oracle_bodies(p, g)
d_hat, kappa, mu, _, _, dt = g[p + "params"]
q0 = g[p + "q0"]
X = O.all_world_points(ob, q0)
rows = g[p + "c0_ee"]
ra, d2, val, g12, H12, rp = O.contact_pair_terms("ee", ob, X, rows, kappa, d_hat)
z, _, eps = O.gather("ee", ob, X, ra)
# GPU batch pieces
d2g, gd, hd, reg, gam = _native.d2_derivatives("ee", z)
m, mg, mh = _native.mollifier(z, eps, True)
b0, b1, b2 = _native.barrier_batch(d2g, d_hat)
b0, b1, b2 = kappa * b0, kappa * b1, kappa * b2
for k in range(len(ra)):
    H = b2[k] * np.outer(gd[k], gd[k]) + b1[k] * hd[k]
    gg = b1[k] * gd[k]
    Hn = mh[k] * b0[k] + np.outer(mg[k], gg) + np.outer(gg, mg[k]) + m[k] * H
    e = np.linalg.norm(Hn - H12[k]) / np.linalg.norm(H12[k])
    if e > 1e-9:
        print("batch-combined mismatch", k, e)
print("eps", eps[:3])
bodies = [P.CollisionBody.from_mesh(P.SurfaceMesh(v, t, e_), dynamic=d) for v, t, e_, d in unpack_meshes(p, g)]
print("elen2 equal:", all(np.array_equal(a.edge_rest_len_sq, b.edge_rest_len_sq) for a, b in zip(bodies, ob)))
c = P.CandidateSet(np.zeros((0, 4), dtype=np.int64), ra, g[p + "c0_ov"])
blk = P.contact_gradient_hessian(bodies, q0, c, kappa, d_hat, project=False)
for k in range(len(ra)):
    J = O.pair_jacobian("ee", rp[k:k + 1])[0]
    ref = J.T @ H12[k] @ J
    eg = np.linalg.norm(blk.grad[k] - J.T @ g12[k]) / np.linalg.norm(J.T @ g12[k])
    e = np.linalg.norm(blk.hess[k] - ref) / np.linalg.norm(ref)
    if e > 1e-9 or eg > 1e-9:
        print("scene mismatch", k, "hess", e, "grad", eg, "mol", m[k], "region", reg[k])
# isolated pair kernel
zz = z
dyn2 = np.ones((len(ra), 2), dtype=np.uint8)
g12g, h12g, g24g, h24g = _native.contact_pair_batch("ee", zz, rp, eps, kappa, d_hat, dyn2, project=False)
for k in range(len(ra)):
    e = np.linalg.norm(h12g[k] - H12[k]) / np.linalg.norm(H12[k])
    J = O.pair_jacobian("ee", rp[k:k + 1])[0]
    ref = J.T @ H12[k] @ J
    e2 = np.linalg.norm(h24g[k] - ref) / np.linalg.norm(ref)
    e3 = np.linalg.norm(J.T @ h12g[k] @ J - ref) / np.linalg.norm(ref)
    if e > 1e-9 or e2 > 1e-9:
        print("pair-kernel", k, "H12 err", e, "H24 err", e2, "J^T H12gpu J err", e3)
