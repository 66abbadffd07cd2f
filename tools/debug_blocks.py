import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests/golden")
import paper_2201_10022_b200 as P  # noqa: E402
from golden_io import unpack_meshes  # noqa: E402

g = dict(np.load("tests/golden/contact.npz"))
for tag in ["twocube", "aligned", "floor", "ico"]:
    p = tag + "_"
    bodies = [P.CollisionBody.from_mesh(P.SurfaceMesh(v, t, e), dynamic=d) for v, t, e, d in unpack_meshes(p, g)]
    d_hat, kappa, mu, _, _, dt = g[p + "params"]
    q0 = g[p + "q0"]
    nvf = len(g[p + "c0_vf"])
    for s, proj in (("U", False), ("P", True)):
        c = P.CandidateSet(g[p + "c0_vf"], g[p + "c0_ee"], g[p + "c0_ov"])
        blk = P.contact_gradient_hessian(bodies, q0, c, kappa, d_hat, project=proj)
        ref = g[p + f"blk{s}_h"]
        errs = [np.linalg.norm(blk.hess[k] - ref[k]) / np.linalg.norm(ref[k]) for k in range(len(ref))]
        errs = np.array(errs)
        bad = np.nonzero(errs > 1e-9)[0]
        print(tag, s, "n", len(errs), "bad", len(bad), "max", errs.max() if len(errs) else 0, "first bad", bad[:10],
              flush=True)
        if len(bad):
            k = bad[0]
            np.set_printoptions(precision=3, linewidth=200, suppress=True)
            print("gpu\n", blk.hess[k][:6, :6])
            print("ref\n", ref[k][:6, :6])
            print("eig gpu", np.linalg.eigvalsh(blk.hess[k])[-6:])
            print("eig ref", np.linalg.eigvalsh(ref[k])[-6:])
