import sys
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests/golden")
import paper_2201_10022_b200 as P
from golden_io import unpack_meshes
g = dict(np.load("tests/golden/contact.npz"))
for tag in ["twocube", "floor"]:
    p = tag + "_"
    bodies = [P.CollisionBody.from_mesh(P.SurfaceMesh(v, t, e), dynamic=d) for v, t, e, d in unpack_meshes(p, g)]
    d_hat, kappa, mu, _, _, dt = g[p + "params"]
    q0 = g[p + "q0"]
    c = P.CandidateSet(g[p + "c0_vf"], g[p + "c0_ee"], g[p + "c0_ov"])
    fr = P.friction_precompute(bodies, q0, c, kappa, d_hat, mu)
    for k in range(min(4, len(fr))):
        qp = np.concatenate([q0[fr.body_a[k]], q0[fr.body_b[k]]])
        print(tag, k, "gpu off", fr.offset[k], "tmap.q", fr.tangent_map[k] @ qp, "ref off", g[p + "fr_off"][k],
              "ref tmap.q", g[p + "fr_tmap"][k] @ qp)
