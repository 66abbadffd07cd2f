"""Pin the CPU oracle (oracle/abd_oracle.py) against reference-generated goldens."""
import numpy as np
import pytest

from conftest import rel_err
from golden_io import oracle_bodies, unpack_meshes
from oracle import abd_oracle as O

TOL = 1e-9  # north-star relative tolerance for energies/gradients/Hessian blocks


def test_pt_closest_bitwise(golden):
    g = golden("kernels.npz")
    z = g["pt_z"]
    d2, reg, bary = O.pt_closest(z[:, 0], z[:, 1], z[:, 2], z[:, 3])
    assert np.array_equal(reg, g["pt_region"])
    assert np.array_equal(d2, g["pt_d2"])
    assert np.array_equal(bary, g["pt_bary"])


def test_ee_closest_bitwise(golden):
    g = golden("kernels.npz")
    z = g["ee_z"]
    d2, reg, s, t = O.ee_closest(z[:, 0], z[:, 1], z[:, 2], z[:, 3])
    assert np.array_equal(reg, g["ee_region"])
    assert np.array_equal(d2, g["ee_d2"])
    assert np.array_equal(s, g["ee_s"]) and np.array_equal(t, g["ee_t"])


@pytest.mark.parametrize("kind", ["vf", "ee"])
def test_d2_derivatives(golden, kind):
    g = golden("kernels.npz")
    d2, gr, h, reg, gam = O.d2_derivatives(kind, g[f"g{kind}_z"])
    assert np.array_equal(reg, g[f"g{kind}_region"])
    assert np.array_equal(d2, g[f"g{kind}_d2"])
    for k in range(len(d2)):
        assert rel_err(gr[k], g[f"g{kind}_grad"][k]) <= TOL
        assert rel_err(h[k], g[f"g{kind}_hess"][k]) <= TOL
    assert np.allclose(gam, g[f"g{kind}_gamma"], rtol=0, atol=1e-15)


def test_mollifier(golden):
    g = golden("kernels.npz")
    v, gr, h = O.ee_mollifier_derivs(g["mol_z"], g["mol_eps"])
    assert np.allclose(v, g["mol_val"], rtol=1e-12, atol=0)
    assert np.array_equal(O.ee_mollifier_value(g["mol_z"], g["mol_eps"]), g["mol_val2"])
    for k in range(len(v)):
        assert rel_err(gr[k], g["mol_grad"][k], tiny=1e-30) <= TOL or np.abs(g["mol_grad"][k]).max() == 0
        assert rel_err(h[k], g["mol_hess"][k], tiny=1e-30) <= TOL or np.abs(g["mol_hess"][k]).max() == 0


def test_barrier(golden):
    g = golden("kernels.npz")
    b0, b1, b2 = O.barrier_terms(g["bar_s"], float(g["bar_dhat"]))
    assert np.allclose(b0, g["bar_b0"], rtol=1e-13, atol=0)
    assert np.allclose(b1, g["bar_b1"], rtol=1e-13, atol=0)
    assert np.allclose(b2, g["bar_b2"], rtol=1e-13, atol=0)
    with pytest.raises(O.OracleBarrierDomainError):
        O.barrier_terms(np.array([0.0]), 1e-3)


def test_barrier_half_dhat_known_answer():
    d_hat = 1e-3
    b0, _, _ = O.barrier_terms(np.array([0.25 * d_hat ** 2]), d_hat)
    assert b0[0] == pytest.approx((d_hat ** 2 / 4) * np.log(2.0), rel=1e-12)


def test_ortho(golden):
    g = golden("kernels.npz")
    k = float(g["orth_k"])
    for i, q in enumerate(g["orth_q"]):
        assert O.ortho_energy(q, k) == pytest.approx(g["orth_e"][i], rel=1e-12, abs=1e-300)
        assert rel_err(O.ortho_gradient(q, k), g["orth_g"][i], tiny=1e-300) <= TOL or i == 0
        assert rel_err(O.ortho_hessian(q, k), g["orth_h"][i]) <= TOL
        assert rel_err(O.psd_clamp(O.ortho_hessian(q, k)), g["orth_hp"][i]) <= TOL
        assert O.ortho_error(q) == pytest.approx(g["orth_err"][i], rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("k", [2, 12, 24])
def test_psd(golden, k):
    g = golden("kernels.npz")
    out = O.psd_clamp(g[f"psd{k}_in"])
    for i in range(len(out)):
        assert rel_err(out[i], g[f"psd{k}_out"][i]) <= 1e-12


@pytest.mark.parametrize("kind", ["vf", "ee"])
def test_accd(golden, kind):
    g = golden("kernels.npz")
    t = O.accd(kind, g[f"ccd_{kind}_x"], g[f"ccd_{kind}_dx"], slack=0.1)
    assert np.array_equal(t, g[f"ccd_{kind}_t"])
    t3 = O.accd(kind, g[f"ccd_{kind}_x"], g[f"ccd_{kind}_dx"], slack=0.3, t_max=0.7)
    assert np.array_equal(t3, g[f"ccd_{kind}_t3"])


CASES = ["twocube", "aligned", "floor", "ico"]


def _case(golden, tag):
    g = golden("contact.npz")
    p = tag + "_"
    bodies = oracle_bodies(p, g)
    d_hat, kappa, mu, density, kappa_o, dt = g[p + "params"]
    return g, p, bodies, d_hat, kappa, mu, dt


@pytest.mark.parametrize("tag", CASES)
def test_broad_phase_exact(golden, tag):
    g, p, bodies, d_hat, *_ = _case(golden, tag)
    q0, dq = g[p + "q0"], g[p + "dq"]
    for nm, q1 in (("c0", q0), ("c1", q0 + dq)):
        c = O.broad_phase(bodies, q0, q1, d_hat)
        assert np.array_equal(c.vf, g[p + nm + "_vf"])
        assert np.array_equal(c.ee, g[p + nm + "_ee"])
        assert np.array_equal(c.overlap_pairs, g[p + nm + "_ov"])


@pytest.mark.parametrize("tag", CASES)
def test_contact_energy_and_blocks(golden, tag):
    g, p, bodies, d_hat, kappa, mu, dt = _case(golden, tag)
    q0 = g[p + "q0"]
    vf, ee = g[p + "c0_vf"], g[p + "c0_ee"]
    e = O.contact_energy(bodies, q0, vf, ee, kappa, d_hat)
    assert e == pytest.approx(float(g[p + "energy"]), rel=1e-12, abs=0)
    for s, proj in (("P", True), ("U", False)):
        blk = O.contact_blocks(bodies, q0, vf, ee, kappa, d_hat, project=proj)
        assert np.array_equal(blk.body_a, g[p + f"blk{s}_a"])
        assert np.array_equal(blk.body_b, g[p + f"blk{s}_b"])
        assert np.array_equal(blk.d_sq, g[p + f"blk{s}_d2"])
        for k in range(len(blk.body_a)):
            assert rel_err(blk.grad[k], g[p + f"blk{s}_g"][k]) <= TOL
            assert rel_err(blk.hess[k], g[p + f"blk{s}_h"][k]) <= TOL


@pytest.mark.parametrize("tag", CASES)
def test_friction(golden, tag):
    g, p, bodies, d_hat, kappa, mu, dt = _case(golden, tag)
    q0 = g[p + "q0"]
    fr = O.friction_precompute(bodies, q0, g[p + "c0_vf"], g[p + "c0_ee"], kappa, d_hat, mu)
    assert np.array_equal(fr.body_a, g[p + "fr_a"]) and np.array_equal(fr.body_b, g[p + "fr_b"])
    assert np.allclose(fr.lam, g[p + "fr_lam"], rtol=1e-12, atol=0)
    assert np.allclose(fr.tangent_map, g[p + "fr_tmap"], rtol=1e-12, atol=1e-15)
    assert np.allclose(fr.offset, g[p + "fr_off"], rtol=1e-11, atol=1e-13)
    qp = g[p + "qp"]
    assert O.friction_energy(qp, fr, dt, 1e-3) == pytest.approx(float(g[p + "fr_energy"]), rel=1e-11)
    dyn = np.array([b.dynamic for b in bodies])
    for s, proj in (("P", True), ("U", False)):
        fb = O.friction_blocks(qp, fr, dt, 1e-3, dyn, project=proj)
        for k in range(len(fr)):
            assert rel_err(fb.grad[k], g[p + f"frb{s}_g"][k], tiny=1e-300) <= 1e-8 or \
                np.abs(g[p + f"frb{s}_g"][k]).max() < 1e-14
            assert rel_err(fb.hess[k], g[p + f"frb{s}_h"][k]) <= TOL


@pytest.mark.parametrize("tag", CASES)
def test_step_filter_and_assembly(golden, tag):
    g, p, bodies, d_hat, kappa, mu, dt = _case(golden, tag)
    q0, dq = g[p + "q0"], g[p + "dq"]
    a = O.step_filter(bodies, q0, dq, g[p + "c1_vf"], g[p + "c1_ee"], 0.1)
    assert a == float(g[p + "alpha"])
    model = O.OracleModel(bodies, list(g[p + "masses"]), list(g[p + "stiff"]))
    fr = O.friction_precompute(bodies, q0, g[p + "c0_vf"], g[p + "c0_ee"], kappa, d_hat, mu)
    cands = O.OracleCandidates(g[p + "c0_vf"], g[p + "c0_ee"], g[p + "c0_ov"])
    ip = O.OracleIP(g[p + "qtilde"], fr, cands)
    prm = O.OracleParams(dt=dt, d_hat=d_hat, kappa_barrier=kappa, mu=mu)
    qp = g[p + "qp"]
    grad, diag, off = O.assemble(model, qp, ip, prm)
    assert rel_err(grad, g[p + "asm_g"]) <= TOL
    for s in range(len(diag)):
        assert rel_err(diag[s], g[p + "asm_diag"][s]) <= TOL
    keys = [tuple(k) for k in g[p + "asm_off_keys"]]
    assert sorted(off.keys()) == keys
    for k, blk in zip(keys, g[p + "asm_off_blocks"]):
        assert rel_err(off[k], blk, tiny=1e-300) <= TOL or np.abs(blk).max() == 0
    assert O.ip_value(model, qp, ip, prm) == pytest.approx(float(g[p + "ip"]), rel=1e-12)
    qt = O.q_tilde(model, q0, g[p + "qdot"], np.zeros_like(q0), dt)
    assert qt.shape == q0.shape
    dx = O.solve_dense(diag, off, grad)
    assert rel_err(dx, g[p + "solve_dx"]) <= 1e-7


def test_box_stack_trajectory(golden):
    """Oracle advance_step reproduces the reference's 100-step box stack."""
    g = golden("box_stack.npz")
    bodies = oracle_bodies("scene_", g)
    from paper_2201_10022_b200 import scenes
    spec = scenes.box_stack(seed=0)
    from paper_2201_10022_b200.body import mass_matrix
    masses, stiff = [], []
    for m, dyn in zip(spec.meshes, spec.dynamic):
        if dyn:
            gm, vol = mass_matrix(m, spec.density)
            masses.append(gm.matrix)
            stiff.append(spec.kappa_ortho * vol)
        else:
            masses.append(None)
            stiff.append(None)
    model = O.OracleModel(bodies, masses, stiff)
    prm = O.OracleParams(**{k: v for k, v in spec.params.items()})
    f = np.zeros((len(bodies), 12))
    for b in model.dyn:
        f[b, :3] = masses[b][0, 0] * np.array([0, 0, -9.8])
        f[b, 3:] = np.kron(np.array([0, 0, -9.8]), masses[b][0, 3:6])
    q, qd = g["q"][0].copy(), g["q_dot"][0].copy()
    steps = 25
    for s in range(steps):
        q, qd, st = O.advance_step(model, q, qd, f, prm, min_distance=(s % 5 == 4))
        ref = g["q"][s + 1]
        assert np.abs(q - ref).max() / np.abs(ref).max() <= 1e-6
        assert st.iterations == g["iterations"][s]


@pytest.mark.parametrize("name,steps", [("chainmail", 40), ("cube_drop", 35)])
def test_small_config_trajectories(golden, name, steps):
    """Oracle advance_step reproduces the reference on small configs 3 and 5
    (friction, kinematic walls / anchors, tori with mollified edge-edge contact)."""
    g = golden(name + ".npz")
    bodies = oracle_bodies("scene_", g)
    from paper_2201_10022_b200 import scenes
    from paper_2201_10022_b200.body import mass_matrix
    spec = (scenes.cube_drop(seed=0, n=2) if name == "cube_drop"
            else scenes.chainmail(seed=0, n_chains=2, links=3, chains_x=2))
    masses, stiff = [], []
    for m, dyn in zip(spec.meshes, spec.dynamic):
        if dyn:
            gm, vol = mass_matrix(m, spec.density)
            masses.append(gm.matrix)
            stiff.append(spec.kappa_ortho * vol)
        else:
            masses.append(None)
            stiff.append(None)
    model = O.OracleModel(bodies, masses, stiff)
    prm = O.OracleParams(**{k: v for k, v in spec.params.items()})
    f = np.zeros((len(bodies), 12))
    grav = np.array([0, 0, -9.8])
    for b in model.dyn:
        f[b, :3] = masses[b][0, 0] * grav
        f[b, 3:] = np.kron(grav, masses[b][0, 3:6])
    q, qd = g["q"][0].copy(), spec.q_dot0.copy()
    for s in range(steps):
        q, qd, st = O.advance_step(model, q, qd, f, prm, min_distance=False)
        ref = g["q"][s + 1]
        assert np.abs(q - ref).max() / np.abs(ref).max() <= 1e-6, (name, s)
        assert st.iterations == g["iterations"][s]


def test_oracle_intersection_audit_golden(golden):
    """Oracle restatement of the intersection audit against the reference's own verdicts."""
    g = golden("intersect.npz")
    assert np.array_equal(O.tri_intersect_batch(g["tri_a"], g["tri_b"]), g["tri_hit"])
    for c in range(2):
        bodies = oracle_bodies(f"s{c}_", g)
        pairs = O.intersecting_body_pairs(bodies, g[f"s{c}_q"])
        assert [list(p) for p in pairs] == g[f"s{c}_pairs"].tolist()
