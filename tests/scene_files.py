"""Scene JSON + OBJ files for the scene-loader parity tests (tests/test_gpu_scene.py,
tests/test_scene_host.py) and their reference fixtures (tests/golden/make_golden_scene.py).

The files are written from procedural meshes, so the same scene is produced here and
when the reference generated the fixtures.  Scenarios follow the reference's own
scene tests (pkg/tests/test_scene.py: two cubes, a cube dropped on a kinematic floor)
plus joints and windowed loads, which the reference tests exercise only through
constraints.py: a hinged pair of bars (one on an axis) under a short torque window, and an axis-jointed
wheel with a point-force window and a seeded perturbation.
"""
from __future__ import annotations

import json
from pathlib import Path


def write_mesh_obj(path, mesh):
    lines = [f"v {v[0]:.17g} {v[1]:.17g} {v[2]:.17g}" for v in mesh.vertices]
    lines += [f"f {t[0] + 1} {t[1] + 1} {t[2] + 1}" for t in mesh.triangles]
    Path(path).write_text("\n".join(lines) + "\n", encoding="utf-8")


def write_scenes(d, shapes):
    """All scenes under directory d; `shapes` is a module with box_mesh / prism_mesh /
    icosphere_mesh (the reference's or ours -- they are vertex-for-vertex equal)."""
    d = Path(d)
    d.mkdir(parents=True, exist_ok=True)
    write_mesh_obj(d / "cube1.obj", shapes.box_mesh(1.0))
    write_mesh_obj(d / "cube04.obj", shapes.box_mesh(0.4))
    write_mesh_obj(d / "floor.obj", shapes.box_mesh([4.0, 4.0, 0.4]))
    write_mesh_obj(d / "bar.obj", shapes.box_mesh([0.4, 0.1, 0.1]))
    write_mesh_obj(d / "wheel.obj", shapes.prism_mesh(8, radius=0.3, height=0.1, axis=1))
    write_mesh_obj(d / "ball.obj", shapes.icosphere_mesh(0.15, 1))
    scenes = {
        "two_cubes": {
            "name": "two-cubes", "gravity": [0.0, 0.0, 0.0], "params": {"dt": 0.01},
            "output": {"frame_interval": 1, "seed": 0, "workers": 1},
            "bodies": [{"name": "a", "mesh": "cube1.obj", "density": 1000.0, "velocity": [0.2, 0, 0]},
                       {"name": "b", "mesh": "cube1.obj", "translation": [1.5, 0, 0]}],
        },
        "drop": {
            "name": "drop", "gravity": [0.0, 0.0, -9.8],
            "params": {"dt": 0.01, "d_hat": 1e-3, "kappa_barrier": 1e4},
            "output": {"frame_interval": 2, "seed": 0, "workers": 1},
            "bodies": [{"name": "floor", "mesh": "floor.obj", "kinematic": True},
                       {"name": "cube", "mesh": "cube04.obj", "translation": [0, 0, 0.5]},
                       {"name": "ball", "mesh": "ball.obj", "translation": [0.05, 0.02, 0.9],
                        "perturb_translation": 0.02}],
        },
        "hinge": {
            "name": "hinge", "gravity": [0.0, 0.0, -9.8], "params": {"dt": 0.01},
            "output": {"frame_interval": 1, "seed": 3, "workers": 2},
            "bodies": [{"name": "floor", "mesh": "floor.obj", "kinematic": True, "translation": [0, 0, -0.6]},
                       {"name": "bar_a", "mesh": "bar.obj", "kappa_ortho": 1e10},
                       {"name": "bar_b", "mesh": "bar.obj", "translation": [0.42, 0, 0], "kappa_ortho": 1e10}],
            "joints": [{"type": "hinge", "bodies": ["bar_a", "bar_b"], "point": [0.21, 0, 0],
                        "direction": [0, 1, 0]},
                       {"type": "axis", "body": "bar_a", "point": [-0.19, 0, 0], "direction": [0, 1, 0]}],
            "forces": [{"body": "bar_b", "type": "torque", "torque": [0, 0.05, 0], "start": 0.0, "end": 0.03}],
        },
        "wheel": {
            "name": "wheel", "gravity": [0.0, 0.0, -9.8], "params": {"dt": 0.01},
            "output": {"frame_interval": 1, "seed": 7, "workers": 1},
            "bodies": [{"name": "wheel", "mesh": "wheel.obj", "translation": [0, 0, 0.5]},
                       {"name": "floor", "mesh": "floor.obj", "kinematic": True, "translation": [0, 0, -0.2]},
                       {"name": "ball", "mesh": "ball.obj", "translation": [0.1, 0.0, 0.95],
                        "perturb_translation": 0.01}],
            "joints": [{"type": "axis", "body": "wheel", "point": [0, 0, 0.5], "direction": [0, 1, 0],
                        "size": 0.1}],
            "forces": [{"body": "wheel", "type": "point", "force": [0, 0, 30.0], "x_bar": [0.25, 0, 0],
                        "start": 0.02, "end": 0.08}],
        },
    }
    paths = {}
    for name, raw in scenes.items():
        p = d / f"{name}.json"
        p.write_text(json.dumps(raw), encoding="utf-8")
        paths[name] = p
    return paths


STEPS = {"two_cubes": 12, "drop": 30, "hinge": 10, "wheel": 16}
