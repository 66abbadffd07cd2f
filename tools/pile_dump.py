"""Dump the GPU path's step-local outputs on a pile checkpoint for offline comparison
with tests/golden/pile_step{N}.npz (the same quantities make_golden_pile.py stores).

    python tools/pile_dump.py 150 gpurun_out/pile_dump150.npz [--step]
"""
import sys
import warnings

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2201_10022_b200 as P  # noqa: E402
from paper_2201_10022_b200 import scenes  # noqa: E402
from pile_common import checkpoint, golden_path  # noqa: E402

step, out_path = int(sys.argv[1]), sys.argv[2]
spec = scenes.icosphere_pile(seed=0)
model, _, params = spec.build()
ck = checkpoint(step)
g = dict(np.load(golden_path(step)))
state = P.SimState(q=ck["q"].copy(), q_dot=ck["q_dot"].copy(), time=float(ck["time"]), step_index=int(ck["step"]))
q0 = state.q
out = {}
forces = model.forces(state.step_index, state.time + params.dt, q0)
out["qtilde"] = P.compute_q_tilde(model, state, params, forces)
c0 = P.broad_phase(model.bodies, q0, q0, params.d_hat)
out["c0_vf"], out["c0_ee"], out["c0_ov"] = c0.vf, c0.ee, c0.overlap_pairs
fr = P.friction_precompute(model.bodies, q0, c0, params.kappa_barrier, params.d_hat, params.mu)
out["fr_a"], out["fr_b"], out["fr_lam"], out["fr_tmap"], out["fr_off"] = (fr.body_a, fr.body_b, fr.lam,
                                                                           fr.tangent_map, fr.offset)
ref_fr = P.FrictionData(g["A_fr_a"], g["A_fr_b"], g["A_fr_lam"], params.mu, g["A_fr_tmap"], g["A_fr_off"],
                        np.zeros((len(g["A_fr_lam"]), 3, 2)))
for tag, frd in (("own", fr), ("ref", ref_fr)):
    ip = P.IncrementalPotentialState(q0, state.q_dot, g["A_qtilde"], frd, c0, model)
    grad, H = P.assemble(q0, ip, params)
    keys = np.array(sorted(H.off.keys()), dtype=np.int64).reshape(-1, 2)
    out[f"{tag}_grad"] = grad
    out[f"{tag}_off_keys"] = keys
    out[f"{tag}_off_blocks"] = np.array([H.off[tuple(k)] for k in keys]).reshape(-1, 12, 12)
    out[f"{tag}_diag"] = H.diag
    r = np.random.default_rng(int(g["r_seed"])).normal(size=grad.shape)
    out[f"{tag}_Hr"] = H.matvec(r)
    dx = P.solve_newton_system(H, grad)
    out[f"{tag}_dx"] = dx
    out[f"{tag}_res"] = np.array(np.linalg.norm(H.matvec(dx) + grad) / np.linalg.norm(grad))
dq = np.zeros_like(q0)
dq[model.dyn_indices] = g["A_dx"].reshape(-1, 12)
c1 = P.broad_phase(model.bodies, q0, q0 + dq, params.d_hat)
out["c1_vf"], out["c1_ee"], out["c1_ov"] = c1.vf, c1.ee, c1.overlap_pairs
out["alpha_max"] = np.array(P.step_filter(model.bodies, q0, dq, c1, slack=params.ccd_slack))
ip = P.IncrementalPotentialState(q0, state.q_dot, g["A_qtilde"], ref_fr, c1, model)
out["e0"] = np.array(P.ip_value(q0, ip, params))
a, e = P.line_search(q0, dq, ip, params)
out["alpha"], out["e"] = np.array(a), np.array(e)
if "--step" in sys.argv:
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        new, st = P.advance_step(model, state, params)
    out["B_q"], out["B_iterations"], out["B_energy_trace"] = new.q, np.array(st.iterations), np.array(st.energy_trace)
    out["B_min_distance"] = np.array(st.min_distance)
np.savez_compressed(out_path, **out)
print("wrote", out_path)
