"""Headline-config parity: the sm_100a path vs the REFERENCE on the 10k-body pile.

Inputs are the checkpointed states `bench_data/pile_step{150,100}.npz` (BASELINE
config 4, `scenes.icosphere_pile(seed=0)`, 10,001 bodies, 1.62 M vertices); the
expected values are the reference's own outputs on the same state
(`tests/golden/pile_step{N}.npz`, tests/golden/make_golden_pile.py).  Everything
goes through the public API (ctypes -> libabd_b200.so).  Tolerances (north_star):

* candidate rows (broad phase at (q, q) and at (q, q + dq_ref)): bit-exact;
* CCD bound alpha_max and the line-search step alpha: exact;
* q_tilde, friction lambdas, gradient / BSR blocks / H @ r, energies: <= 1e-9
  norm-relative; per 12-block, relative to the magnitude of the terms summed into
  the block (the fixture's A_*_scale: a body squeezed between contacts sums large
  opposing barrier terms, so its block norm alone understates the rounding scale);
* Newton direction: residual <= 1e-8 |g| (solve_refined's contract) and
  <= 1e-6 of the reference's direct solve;
* one full advance_step from the checkpoint: the same Newton iteration count and
  convergence flag, DOFs <= 1e-6 relative, energy trace <= 1e-6 relative per
  iteration, min distance > 0 and equal to the reference's within the DOF tolerance in
  length units (1e-6 x the largest position coordinate).
"""
import os
import warnings

import numpy as np
import pytest

from pile_common import assert_same_rows, block_rel, checkpoint, golden_path, load_golden, scaled_rel

pytestmark = pytest.mark.gpu

TOL = 1e-9
STEPS = [s for s in (150, 100) if os.path.exists(golden_path(s))]


@pytest.fixture(scope="module")
def pile_model():
    from paper_2201_10022_b200 import scenes

    spec = scenes.icosphere_pile(seed=0)
    return spec.build()


def _state(P, step):
    ck = checkpoint(step)
    return P.SimState(q=ck["q"].copy(), q_dot=ck["q_dot"].copy(), time=float(ck["time"]),
                      step_index=int(ck["step"]))


@pytest.mark.parametrize("step", STEPS)
def test_pile_newton_iteration_vs_reference(pile_model, step):
    import paper_2201_10022_b200 as P

    model, _, params = pile_model
    g = load_golden(step)
    state = _state(P, step)
    q0 = state.q
    forces = model.forces(state.step_index, state.time + params.dt, q0)
    qt = P.compute_q_tilde(model, state, params, forces)
    assert np.abs(qt - g["A_qtilde"]).max() <= 1e-12 * np.abs(g["A_qtilde"]).max()

    c0 = P.broad_phase(model.bodies, q0, q0, params.d_hat)
    assert_same_rows(c0.vf, g, "A_c0_vf")
    assert_same_rows(c0.ee, g, "A_c0_ee")
    assert_same_rows(c0.overlap_pairs, g, "A_c0_ov")

    fr = P.friction_precompute(model.bodies, q0, c0, params.kappa_barrier, params.d_hat, params.mu)
    assert np.array_equal(fr.body_a, g["A_fr_a"]) and np.array_equal(fr.body_b, g["A_fr_b"])
    assert block_rel(fr.lam, g["A_fr_lam"], 1e-300) <= TOL
    # tangent frames are defined up to an in-plane rotation: compare tmap^T tmap
    tt = np.einsum("nki,nkj->nij", fr.tangent_map, fr.tangent_map)
    tr = np.einsum("nki,nkj->nij", g["A_fr_tmap"], g["A_fr_tmap"])
    assert block_rel(tt, tr, 1e-300) <= 1e-12

    # the device's own lagged friction data feeds the assembly (the API's FrictionData
    # round trip re-packs tangent maps into basis x coefficients, a ~1e-10 change)
    ip = P.IncrementalPotentialState(q0, state.q_dot, g["A_qtilde"], fr, c0, model)
    grad, H = P.assemble(q0, ip, params)
    assert np.linalg.norm(grad - g["A_grad"]) <= TOL * np.linalg.norm(g["A_grad"])
    assert scaled_rel(grad.reshape(-1, 12), g["A_grad"].reshape(-1, 12), g["A_grad_scale"]) <= TOL
    keys = np.array(sorted(H.off.keys()), dtype=np.int64).reshape(-1, 2)
    assert np.array_equal(keys, g["A_off_keys"])
    ob = np.array([H.off[tuple(k)] for k in keys]).reshape(-1, 12, 12)
    assert scaled_rel(ob, g["A_off_blocks"], g["A_off_scale"]) <= TOL
    sel = g["A_diag_sel"]
    assert scaled_rel(H.diag[sel], g["A_diag_blocks"], g["A_diag_scale"][sel]) <= TOL
    fro = np.sqrt(np.einsum("nij,nij->n", H.diag, H.diag))
    assert (np.abs(fro - g["A_diag_fro"]) / g["A_diag_scale"]).max() <= TOL
    r = np.random.default_rng(int(g["r_seed"])).normal(size=grad.shape)
    hr_scale = np.linalg.norm(g["A_Hr"]) / np.sqrt(len(H.diag))
    assert block_rel(H.matvec(r).reshape(-1, 12), g["A_Hr"].reshape(-1, 12), hr_scale) <= TOL

    dx = P.solve_newton_system(H, grad)
    assert np.linalg.norm(H.matvec(dx) + grad) <= 1e-8 * np.linalg.norm(grad) * 1.0001
    assert np.abs(dx - g["A_dx"]).max() <= 1e-6 * np.abs(g["A_dx"]).max()

    # CCD and line search on the reference's direction (identical inputs)
    dq = np.zeros_like(q0)
    dq[model.dyn_indices] = g["A_dx"].reshape(-1, 12)
    c1 = P.broad_phase(model.bodies, q0, q0 + dq, params.d_hat)
    assert_same_rows(c1.vf, g, "A_c1_vf")
    assert_same_rows(c1.ee, g, "A_c1_ee")
    assert_same_rows(c1.overlap_pairs, g, "A_c1_ov")
    assert P.step_filter(model.bodies, q0, dq, c1, slack=params.ccd_slack) == float(g["A_alpha_max"])
    ip.candidates = c1
    e0 = P.ip_value(q0, ip, params)
    assert abs(e0 - float(g["A_e0"])) <= TOL * abs(float(g["A_e0"]))
    alpha, e = P.line_search(q0, dq, ip, params)
    assert alpha == float(g["A_alpha"])
    assert abs(e - float(g["A_e"])) <= TOL * abs(float(g["A_e"]))


@pytest.mark.parametrize("step", [s for s in STEPS if "B_iterations" in np.load(golden_path(s)).files])
def test_pile_advance_step_vs_reference(pile_model, step):
    import paper_2201_10022_b200 as P

    model, _, params = pile_model
    g = load_golden(step)
    state = _state(P, step)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        new, st = P.advance_step(model, state, params)
    ref_trace = g["B_energy_trace"]
    trace = np.asarray(st.energy_trace)
    n = min(len(trace), len(ref_trace))
    trace_err = np.abs(trace[:n] - ref_trace[:n]) / np.abs(ref_trace[:n])
    msg = (f"iterations {st.iterations} vs {int(g['B_iterations'])}; first trace error > 1e-6 at "
           f"{np.nonzero(trace_err > 1e-6)[0][:3]}")
    assert st.iterations == int(g["B_iterations"]), msg
    assert st.converged == bool(g["B_converged"])
    assert trace_err.max() <= 1e-6, msg
    qerr = np.abs(new.q - g["B_q"]).max() / np.abs(g["B_q"]).max()
    assert qerr <= 1e-6, qerr
    assert st.min_distance > 0
    # a distance moves with the positions: its tolerance is the DOF tolerance in length units
    assert abs(st.min_distance - float(g["B_min_distance"])) <= 1e-6 * np.abs(g["B_q"][:, :3]).max()
