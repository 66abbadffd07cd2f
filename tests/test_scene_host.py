"""Host-side scene logic (no GPU): JSON schema validation, OBJ I/O, CSV rows, joint
setup math -- the reference's scene / constraint tests that never touch the device
(pkg/tests/test_scene.py:59-65, :105-149, :217-234; test_constraints.py:29-117,
:260-275), plus the restated constraints checked against the reference's reduction
matrices (tests/golden/joints.npz)."""
import json
import os

import numpy as np
import pytest

from scene_files import write_mesh_obj


def test_obj_round_trip(tmp_path):
    from paper_2201_10022_b200.scene import read_obj
    from paper_2201_10022_b200.shapes import icosphere_mesh

    m = icosphere_mesh(0.7, 1, center=(0.3, -0.2, 0.5))
    write_mesh_obj(tmp_path / "ball.obj", m)
    back = read_obj(tmp_path / "ball.obj")
    assert np.array_equal(back.vertices, m.vertices) and np.array_equal(back.triangles, m.triangles)


def test_obj_rejects_polygons_and_empty(tmp_path):
    from paper_2201_10022_b200.scene import read_obj

    (tmp_path / "q.obj").write_text("v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\nf 1 2 3 4\n")
    with pytest.raises(ValueError, match="only triangle faces"):
        read_obj(tmp_path / "q.obj")
    (tmp_path / "e.obj").write_text("# nothing\n")
    with pytest.raises(ValueError, match="no triangle geometry"):
        read_obj(tmp_path / "e.obj")


def test_frame_writer_and_object_reader(tmp_path):
    from paper_2201_10022_b200.scene import read_obj_objects, write_obj_frame
    from paper_2201_10022_b200.shapes import box_mesh, prism_mesh

    a, b = box_mesh(1.0), prism_mesh(6, 0.5, 0.2)
    vb = b.vertices + [3.0, 1e-17, -2.5]
    write_obj_frame(tmp_path / "f.obj", ["a", "b"], [a.vertices, vb], [a.triangles, b.triangles])
    objs = read_obj_objects(tmp_path / "f.obj")
    assert [n for n, _, _ in objs] == ["a", "b"]
    assert np.array_equal(objs[0][1], a.vertices) and np.array_equal(objs[0][2], a.triangles)
    assert np.array_equal(objs[1][1], vb) and np.array_equal(objs[1][2], b.triangles)
    assert (tmp_path / "f.obj").read_text().splitlines()[1] == "v -0.5 -0.5 -0.5"


def test_schema_violations(tmp_path):
    from paper_2201_10022_b200.scene import SceneConfig
    from paper_2201_10022_b200.shapes import box_mesh

    write_mesh_obj(tmp_path / "cube.obj", box_mesh(1.0))
    bad = [({"bodies": []}, "at least one body"),
           ({"bodies": [{"name": "a", "mesh": "cube.obj"}, {"name": "a", "mesh": "cube.obj"}]}, "duplicate"),
           ({"bodies": [{"name": "a", "mesh": "cube.obj"}], "joints": [{"type": "warp", "body": "a"}]},
            "unknown joint"),
           ({"bodies": [{"name": "a", "mesh": "cube.obj"}], "forces": [{"body": "zz", "force": [0, 0, 1]}]},
            "unknown body"),
           ({"bodies": [{"name": "a", "mesh": "cube.obj", "velocity": [1, 2]}]}, "3 or 12"),
           ({"bodies": [{"name": "a", "mesh": "cube.obj"}, {"name": "b", "mesh": "cube.obj"}],
             "joints": [{"type": "hinge", "bodies": ["a"]}]}, "exactly two")]
    for raw, match in bad:
        with pytest.raises(ValueError, match=match):
            SceneConfig.from_dict(raw, base_dir=tmp_path)
    with pytest.raises(FileNotFoundError):
        SceneConfig.from_dict({"bodies": [{"name": "a", "mesh": "nope.obj"}]}, base_dir=tmp_path)
    (tmp_path / "broken.json").write_text("{")
    with pytest.raises(ValueError, match="invalid scene JSON"):
        SceneConfig.from_file(tmp_path / "broken.json")


def test_config_defaults_and_fields(tmp_path):
    from paper_2201_10022_b200.scene import SceneConfig
    from paper_2201_10022_b200.shapes import box_mesh

    write_mesh_obj(tmp_path / "cube.obj", box_mesh(1.0))
    raw = {"bodies": [{"name": "a", "mesh": "cube.obj", "velocity": [1, 2, 3]}],
           "forces": [{"body": "a", "type": "torque", "torque": [0, 0, 1], "start": 0.5}],
           "joints": [{"type": "axis", "body": "a", "point": [1, 0, 0]}], "params": {"dt": 0.02}}
    c = SceneConfig.from_dict(raw, base_dir=tmp_path)
    assert c.name == "scene" and np.array_equal(c.gravity, [0, 0, -9.8])
    b = c.bodies[0]
    assert b.density == 1000.0 and b.kappa_ortho == 1e11 and not b.kinematic
    assert np.array_equal(b.velocity, [1, 2, 3] + [0] * 9) and np.array_equal(b.linear, np.eye(3))
    assert c.forces[0].kind == "torque" and c.forces[0].end == np.inf and c.forces[0].start == 0.5
    assert c.joints[0].bodies == ["a"] and np.array_equal(c.joints[0].direction, [0, 0, 1])
    o = c.output
    assert (o.frame_interval, o.directory, o.audit, o.workers, o.seed) == (1, None, False, 1, 0)


def test_csv_row_format():
    from paper_2201_10022_b200.scene import STATS_HEADER, FrameStats

    fs = FrameStats(step=3, iterations=2, converged=True, min_distance=0.1, candidates=7, ip_value=-1.5,
                    max_ortho_error=2e-17, min_iterate_distance=np.inf, timings={"solve": 0.25, "total": 1.0})
    assert fs.csv_row() == "3,2,1,0.10000000000000001,7,-1.5,2.0000000000000001e-17,inf,0.000000,0.000000," \
                           "0.000000,0.250000,0.000000,0.000000,1.000000"
    assert len(STATS_HEADER.split(",")) == 15


def test_constraint_setup_matches_reference_matrices():
    """The restated reduction gives the reference's T and q_const exactly (joints.npz)."""
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "joints.npz"))
    from paper_2201_10022_b200 import BodyCoords
    from paper_2201_10022_b200 import constraints as rc

    q0 = np.tile(BodyCoords.identity().q, (1, 1))
    red = rc.build_constrained_system([True], {0: rc.make_free_tet(size=0.5)}, q0)
    assert np.array_equal(red.T, g["free_T"]) and np.array_equal(red.q_const, g["free_qc"])
    red = rc.build_constrained_system([True], {0: rc.make_axis_tet([0.1, 0.05, 0.0], [0, 0, 1.0], size=0.3)}, q0)
    assert np.array_equal(red.T, g["rotor_T"]) and np.array_equal(red.q_const, g["rotor_qc"])


def test_constraint_algebra():
    """test_constraints.py:29-117, :260-275: phi recovery, reparam map, degenerate / over-constrained."""
    from paper_2201_10022_b200 import BodyCoords
    from paper_2201_10022_b200 import constraints as rc

    rng = np.random.default_rng(0)
    Pb = rc.VirtualTet(rc.regular_tet_vertices(0.7) + rng.normal(size=(3, 4)) * 0.05).rest_vertices
    A = np.eye(3) + rng.normal(size=(3, 3)) * 0.2
    p = rng.normal(size=3)
    q = rc.phi(A @ Pb + p[:, None], Pb).q
    assert np.allclose(q, BodyCoords.from_parts(p, A).q, atol=1e-12)
    G = rc.reparam_map(Pb)
    P = rng.normal(size=(3, 4))
    assert np.allclose(G.apply(rc._vec(P)), rc.phi(P, Pb).q, atol=1e-12)
    with pytest.raises(ValueError, match="degenerate"):
        rc.VirtualTet(np.array([[0, 1, 0, 1], [0, 0, 1, 1], [0, 0, 0, 0]], dtype=float))
    with pytest.raises(ValueError, match="origin"):
        rc.make_axis_tet([0, 0, 1.0], [0, 0, 1.0])
    q0 = np.tile(BodyCoords.identity().q, (2, 1))
    with pytest.raises(ValueError):
        rc.build_constrained_system([True], {0: rc.VirtualTet(rc.regular_tet_vertices(1.0) + np.array([1.0, 0, 0])[:, None],
                                                              np.ones(12, dtype=bool))}, q0[:1])
    with pytest.raises(ValueError):
        rc.build_constrained_system([True, True], {0: rc.VirtualTet(rc.regular_tet_vertices(1.0),
                                                                    shared_vertex_links=((0, 1, 0),))}, q0)
    t = rc.make_axis_tet([0.3, 0.0, 0.0], [0, 0, 1.0], size=0.2)
    e = t.rest_vertices[:, 1] - t.rest_vertices[:, 3]
    assert np.allclose(np.cross(e, [0, 0, 1.0]), 0) and t.fixed_dof_mask[3:6].all() and t.fixed_dof_mask[9:].all()
