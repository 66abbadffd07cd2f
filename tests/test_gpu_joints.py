"""Joint reduction on the GPU vs the REFERENCE.

The reduced Newton direction T (T^T H T)^-1 T^T (-g) runs on the device
(csrc/k_reduced.cu, solver.py:479-490); the reduction itself (constraints.py) is
host setup restated in paper_2201_10022_b200/constraints.py.  Fixtures:
tests/golden/joints.npz from tests/golden/make_golden_joints.py (the reference's
own constraint-test scenarios).  Tolerances: T and q_const identical to the
reference's; per step DOFs <= 1e-6 relative, the same Newton iteration counts,
and the reference tests' invariants (shared proxy entries bitwise equal, fixed
anchor entries bitwise constant, rotor points on their circles to 1e-6).
"""
import os
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(__file__), "golden", "joints.npz")


def _models():
    from paper_2201_10022_b200 import (BodyCoords, BodyMaterial, CollisionBody, SimState, StepParams, SystemModel,
                                       external_generalized_force, mass_matrix, torque_point_forces)
    from paper_2201_10022_b200 import constraints as rc
    from paper_2201_10022_b200.shapes import box_mesh, prism_mesh

    def model_of(meshes, kappa=1e11):
        bodies, gms, mats = [], [], []
        for m in meshes:
            gm, vol = mass_matrix(m, 1000.0)
            bodies.append(CollisionBody.from_mesh(m))
            gms.append(gm)
            mats.append(BodyMaterial(1000.0, kappa, vol))
        return SystemModel(bodies, gms, mats)

    def gravity(model):
        return lambda step, t, q: np.asarray([external_generalized_force(model.gmass[b], [0, 0, -9.8])
                                              for b in range(len(q))])

    out = {}
    ident = BodyCoords.identity().q
    # free proxy on a falling box
    m = model_of([box_mesh(0.4)])
    m.force_fn = gravity(m)
    q0 = np.tile(ident, (1, 1))
    m.reduction = rc.build_constrained_system([True], {0: rc.make_free_tet(size=0.5)}, q0)
    st = SimState(q=q0.copy(), q_dot=np.zeros((1, 12)))
    st.q_dot[0, :3] = [0.1, 0.2, 0.0]
    out["free"] = (m, st, StepParams(dt=0.01, newton_tol=1e-11), 10)
    # torqued rotor on an off-centre axis
    m = model_of([prism_mesh(8, radius=0.3, height=0.2, axis=2)])
    gm = m.gmass[0]
    m.force_fn = lambda step, t, q: np.asarray([external_generalized_force(
        gm, np.zeros(3), torque_point_forces([0, 0, 2.0], q[0, 3:].reshape(3, 3), arm_scale=0.2))])
    q0 = np.tile(ident, (1, 1))
    m.reduction = rc.build_constrained_system([True], {0: rc.make_axis_tet([0.1, 0.05, 0.0], [0, 0, 1.0],
                                                                             size=0.3)}, q0)
    out["rotor"] = (m, SimState(q=q0.copy(), q_dot=np.zeros((1, 12))), StepParams(dt=0.01, newton_tol=1e-6), 40)
    # hinged bars (+ an anchored spinning cube)
    for name, anchor in (("hinge", False), ("anchor", True)):
        bar = box_mesh([0.4, 0.1, 0.1])
        meshes = [bar, bar] + ([box_mesh(0.2)] if anchor else [])
        n = len(meshes)
        m = model_of(meshes, kappa=1e10)
        m.force_fn = gravity(m)
        q0 = np.tile(ident, (n, 1))
        q0[1, :3] = [0.42, 0.0, 0.0]
        if anchor:
            q0[2, :3] = [0.2, 0.6, 0.0]
        hw, d = np.array([0.21, 0.0, 0.0]), np.array([0.0, 1.0, 0.0])
        ta = rc.make_axis_tet(hw, d, size=0.1, fix_edge=False)
        tb = rc.make_axis_tet(hw - q0[1, :3], d, size=0.1, fix_edge=False)
        ta = rc.VirtualTet(ta.rest_vertices, ta.fixed_dof_mask | np.array([False] * 3 + [True] * 3 + [False] * 3
                                                                          + [True] * 3))
        tb = rc.VirtualTet(tb.rest_vertices, np.zeros(12, dtype=bool), shared_vertex_links=((1, 0, 1), (3, 0, 3)))
        red = rc.build_constrained_system([True] * n, {0: ta, 1: tb}, q0)
        if anchor:
            C, rhs = rc.axis_anchor_rows(2, n, [0.05, 0.0, 0.0], [0.0, 0.0, 1.0], q0[2], arm=0.1)
            red = rc.constrain_linear(red, C, rhs)
        m.reduction = red
        st = SimState(q=q0.copy(), q_dot=np.zeros((n, 12)))
        if anchor:
            w = 0.5
            st.q_dot[2, :3] = [0.0, -0.05 * w, 0.0]
            st.q_dot[2, 3:] = np.array([[0.0, -w, 0.0], [w, 0.0, 0.0], [0.0, 0.0, 0.0]]).reshape(9)
            st.q_dot = (red.T @ red.extract_u_rate(st.q_dot.reshape(-1))).reshape(n, 12)
        st.u = red.extract_u(st.q[m.dyn_indices].reshape(-1))
        out[name] = (m, st, StepParams(dt=0.01, newton_tol=1e-6), 20)
    return out


@pytest.fixture(scope="module")
def runs():
    import paper_2201_10022_b200 as P

    g = np.load(G)
    res = {}
    for name, (m, st, prm, steps) in _models().items():
        assert np.array_equal(m.reduction.T, g[f"{name}_T"]), name
        assert np.array_equal(m.reduction.q_const, g[f"{name}_qc"]), name
        assert np.array_equal(st.q, g[f"{name}_q0"]) and np.allclose(st.q_dot, g[f"{name}_qd0"], rtol=0, atol=1e-15)
        qs, us, its = [], [], []
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            for _ in range(steps):
                st, stats = P.advance_step(m, st, prm)
                qs.append(st.q.copy())
                us.append(st.u.copy())
                its.append(stats.iterations)
        res[name] = (m, np.array(qs), np.array(us), np.array(its))
    return g, res


@pytest.mark.parametrize("name", ["free", "rotor", "hinge", "anchor"])
def test_joint_trajectory_vs_reference(runs, name):
    g, res = runs
    m, qs, us, its = res[name]
    ref_q, ref_it = g[f"{name}_q"], g[f"{name}_iterations"]
    err = np.abs(qs - ref_q).max(axis=(1, 2)) / np.abs(ref_q).max(axis=(1, 2))
    assert err.max() <= 1e-6, (name, err.max(), int(np.argmax(err)))
    assert np.array_equal(its, ref_it), (name, its.tolist(), ref_it.tolist())


def test_hinge_shared_entries_bitwise(runs):
    """test_constraints.py:203-257: shared proxy vertices read identically, anchors constant."""
    _, res = runs
    for name in ("hinge", "anchor"):
        m, qs, us, _ = res[name]
        red = m.reduction
        for u in us:
            a, b = red.proxy_vertex_entries(0, u), red.proxy_vertex_entries(1, u)
            assert np.array_equal(a[3:6], b[3:6]) and np.array_equal(a[9:12], b[9:12])
            assert np.array_equal(a[3:6], red.entry_maps[0][1][3:6])


def test_rotor_stays_on_circles(runs):
    """test_constraints.py:156-200: points keep their distance to the axis and their height."""
    from paper_2201_10022_b200.shapes import prism_mesh

    _, res = runs
    _, qs, _, _ = res["rotor"]
    rest = prism_mesh(8, radius=0.3, height=0.2, axis=2).vertices
    ax = np.array([0.1, 0.05, 0.0])
    r0 = np.linalg.norm((rest - ax)[:, :2], axis=1)
    for q in qs:
        x = rest @ q[0, 3:].reshape(3, 3).T + q[0, :3] - ax
        assert np.abs(np.linalg.norm(x[:, :2], axis=1) - r0).max() < 1e-6
        assert np.abs(x[:, 2] - (rest[:, 2] - ax[2])).max() < 1e-6
    A = qs[-1, 0, 3:].reshape(3, 3)
    assert abs(np.arctan2(A[1, 0], A[0, 0])) > 1e-3


def test_free_proxy_matches_unconstrained(runs):
    """test_constraints.py:119-153: a free proxy is a similarity reparameterization."""
    import paper_2201_10022_b200 as P

    _, res = runs
    m, qs, _, _ = res["free"]
    m2 = P.SystemModel(m.bodies, m.gmass, m.materials, force_fn=m.force_fn)
    st = P.SimState(q=np.tile(P.BodyCoords.identity().q, (1, 1)), q_dot=np.zeros((1, 12)))
    st.q_dot[0, :3] = [0.1, 0.2, 0.0]
    for _ in range(10):
        st, _ = P.advance_step(m2, st, P.StepParams(dt=0.01, newton_tol=1e-11))
    assert np.allclose(st.q, qs[-1], rtol=0, atol=1e-12)
