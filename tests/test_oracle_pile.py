"""Pin the CPU oracle against the REFERENCE on the headline config (10k-body pile).

Step-local, at the checkpointed step-150 state: the oracle's broad phase at (q, q)
and at (q, q + dq_ref) must reproduce the reference's candidate rows bit for bit,
its CCD bound alpha_max must equal the reference's exactly, and its assembled
system (gradient, off-diagonal blocks, H @ r for the fixture's probe r) and
incremental potential must agree within 1e-9 (north_star tolerances).
"""
import os

import numpy as np
import pytest

from pile_common import assert_same_rows, block_rel, checkpoint, golden_path, load_golden, scaled_rel, oracle_pile_model

TOL = 1e-9

pytestmark = pytest.mark.skipif(not os.path.exists(golden_path(150)), reason="pile fixture not generated")


@pytest.fixture(scope="module")
def pile():
    from oracle import abd_oracle as O

    spec, model, prm, f = oracle_pile_model()
    g = load_golden(150)
    ck = checkpoint(150)
    q0, qd = ck["q"], ck["q_dot"]
    qt = O.q_tilde(model, q0, qd, f, prm.dt)
    c0 = O.broad_phase(model.bodies, q0, q0, prm.d_hat, workers=min(8, os.cpu_count() or 1))
    return O, model, prm, g, q0, qt, c0


def test_oracle_pile_broad_phase_and_ccd(pile):
    O, model, prm, g, q0, qt, c0 = pile
    assert_same_rows(c0.vf, g, "A_c0_vf")
    assert_same_rows(c0.ee, g, "A_c0_ee")
    assert_same_rows(c0.overlap_pairs, g, "A_c0_ov")
    dq = np.zeros_like(q0)
    dq[model.dyn] = g["A_dx"].reshape(-1, 12)
    c1 = O.broad_phase(model.bodies, q0, q0 + dq, prm.d_hat, workers=min(8, os.cpu_count() or 1))
    assert_same_rows(c1.vf, g, "A_c1_vf")
    assert_same_rows(c1.ee, g, "A_c1_ee")
    assert_same_rows(c1.overlap_pairs, g, "A_c1_ov")
    assert O.step_filter(model.bodies, q0, dq, c1.vf, c1.ee, prm.ccd_slack) == float(g["A_alpha_max"])


def test_oracle_pile_assembly(pile):
    O, model, prm, g, q0, qt, c0 = pile
    assert np.abs(qt - g["A_qtilde"]).max() <= 1e-12 * np.abs(g["A_qtilde"]).max()
    fr = O.friction_precompute(model.bodies, q0, c0.vf, c0.ee, prm.kappa_barrier, prm.d_hat, prm.mu)
    assert np.array_equal(fr.body_a, g["A_fr_a"]) and np.array_equal(fr.body_b, g["A_fr_b"])
    assert block_rel(fr.lam, g["A_fr_lam"], 1e-300) <= TOL
    assert block_rel(fr.tangent_map, g["A_fr_tmap"], 1e-300) <= TOL
    ip = O.OracleIP(qt, fr, c0)
    grad, D, off = O.assemble(model, q0, ip, prm)
    assert scaled_rel(grad.reshape(-1, 12), g["A_grad"].reshape(-1, 12), g["A_grad_scale"]) <= TOL
    keys = np.array(sorted(off.keys()), dtype=np.int64).reshape(-1, 2)
    assert np.array_equal(keys, g["A_off_keys"])
    ob = np.array([off[tuple(k)] for k in keys]).reshape(-1, 12, 12)
    assert scaled_rel(ob, g["A_off_blocks"], g["A_off_scale"]) <= TOL
    sel = g["A_diag_sel"]
    assert scaled_rel(D[sel], g["A_diag_blocks"], g["A_diag_scale"][sel]) <= TOL
    r = np.random.default_rng(int(g["r_seed"])).normal(size=grad.shape)
    Hr = O.bsr_matvec(D, off, r)
    hr_scale = np.linalg.norm(g["A_Hr"]) / np.sqrt(len(D))
    assert block_rel(Hr.reshape(-1, 12), g["A_Hr"].reshape(-1, 12), hr_scale) <= TOL
    # e0 in the fixture is evaluated with the candidate set at (q, q + dq)
    dq = np.zeros_like(q0)
    dq[model.dyn] = g["A_dx"].reshape(-1, 12)
    ip.cands = O.broad_phase(model.bodies, q0, q0 + dq, prm.d_hat, workers=min(8, os.cpu_count() or 1))
    assert abs(O.ip_value(model, q0, ip, prm) - float(g["A_e0"])) <= TOL * abs(float(g["A_e0"]))
    alpha, e, amax = O.line_search(model, q0, dq, ip, prm)
    assert alpha == float(g["A_alpha"])
    assert abs(e - float(g["A_e"])) <= TOL * abs(float(g["A_e"]))
    # the oracle's sparse direct solve meets the reference's residual contract on this system
    dx = O.solve_sparse(D, off, grad)
    res = O.bsr_matvec(D, off, dx) + grad
    assert np.linalg.norm(res) <= 1e-8 * np.linalg.norm(grad)
    assert np.abs(dx - g["A_dx"]).max() <= 1e-6 * np.abs(g["A_dx"]).max()
