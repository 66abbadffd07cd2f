"""Scene-loader / driver fixtures from the REFERENCE (scene.py:378-785).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_scene.py

For each scene of tests/scene_files.py: the loaded normalisation (scale, origin,
scene diameter), the initial q / q_dot (after the joint projection), the reduction
size, the stats.csv text of `run` (deterministic columns only), and every written
frame's vertices.  Nothing at test time reads /root/reference.
"""
from __future__ import annotations

import os
import sys
import tempfile
import warnings
from pathlib import Path

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

import stiffbody.shapes as rshapes  # noqa: E402
from stiffbody.scene import load_scene, read_obj_objects, run  # noqa: E402

from scene_files import STEPS, write_scenes  # noqa: E402


def main():
    out = {}
    with tempfile.TemporaryDirectory() as td:
        paths = write_scenes(td, rshapes)
        for name, path in paths.items():
            sc = load_scene(path)
            out[f"{name}_scale"] = np.array(sc.scale)
            out[f"{name}_origin"] = np.asarray(sc.origin)
            out[f"{name}_diameter"] = np.array(sc.scene_diameter)
            out[f"{name}_q0"] = sc.state.q.copy()
            out[f"{name}_qd0"] = sc.state.q_dot.copy()
            out[f"{name}_nu"] = np.array(-1 if sc.model.reduction is None else sc.model.reduction.n_unknowns)
            od = Path(td) / f"out_{name}"
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                stats, violations, nonconv = run(sc, STEPS[name], out_dir=od, audit=True)
            rows = (od / "stats.csv").read_text().strip().splitlines()
            out[f"{name}_csv_header"] = np.array(rows[0])
            out[f"{name}_csv_det"] = np.array([",".join(r.split(",")[:8]) for r in rows[1:]])
            out[f"{name}_violations"] = np.array(len(violations))
            frames = sorted(od.glob("frame_*.obj"))
            out[f"{name}_frame_names"] = np.array([f.name for f in frames])
            for f in frames:
                objs = read_obj_objects(f)
                out[f"{name}_{f.stem}"] = np.concatenate([v for _, v, _ in objs])
            out[f"{name}_objnames"] = np.array([n for n, _, _ in read_obj_objects(frames[0])])
            out[f"{name}_q_final"] = sc.state.q.copy()
            print(name, "steps", STEPS[name], "iterations", [s.iterations for s in stats], "frames", len(frames),
                  flush=True)
    path = os.path.join(HERE, "scenes.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)


if __name__ == "__main__":
    main()
