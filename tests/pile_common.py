"""Shared setup for the headline-config (10k-body pile) parity tests.

The fixtures `tests/golden/pile_step{N}.npz` come from the REFERENCE run on the
checkpointed state `bench_data/pile_step{N}.npz` (tests/golden/make_golden_pile.py).
"""
from __future__ import annotations

import hashlib
import os
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden_path(step):
    return os.path.join(GOLDEN, f"pile_step{step}.npz")


def load_golden(step):
    """The fixture, with the per-block term scales merged in when they were written to a
    side file (pile_step{N}_scales.npz) while stage B still owned the main file."""
    g = dict(np.load(golden_path(step)))
    side = golden_path(step).replace(".npz", "_scales.npz")
    if os.path.exists(side):
        for k, v in np.load(side).items():
            g.setdefault(k, v)
    return g


def scaled_rel(a, b, scale):
    """max over blocks of ||a - b|| / scale: `scale` is the magnitude of the terms summed
    into each block (A_*_scale in the fixture), so cancellation in a sum of large
    opposing contact terms does not inflate the comparison (SURVEY §8(c) comparator 2,
    norm-relative per block)."""
    a = np.asarray(a, dtype=float).reshape(len(b), -1)
    b = np.asarray(b, dtype=float).reshape(len(b), -1)
    e = np.linalg.norm(a - b, axis=1)
    scale = np.asarray(scale, dtype=float)
    if np.any(e[scale == 0] != 0):
        return np.inf
    return float((e[scale > 0] / scale[scale > 0]).max()) if np.any(scale > 0) else 0.0


def checkpoint(step):
    ck = np.load(os.path.join(ROOT, "bench_data", f"pile_step{step}.npz"))
    return {k: ck[k] for k in ck.files}


def rows_sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).tobytes()).hexdigest()


def assert_same_rows(ours, g, prefix):
    """Bit-exact candidate rows: count, SHA-256 of the int64 rows, and the rows."""
    ours = np.asarray(ours, dtype=np.int64)
    assert len(ours) == int(g[prefix + "_n"]), (prefix, len(ours), int(g[prefix + "_n"]))
    if rows_sha(ours) != str(g[prefix + "_sha"]):
        ref = g[prefix].astype(np.int64)
        bad = np.nonzero(np.any(ours != ref, axis=1))[0] if ours.shape == ref.shape else []
        raise AssertionError(f"{prefix}: rows differ (first mismatch at {bad[:5]})")


def block_rel(a, b, floor):
    """Per-block norm-relative error ||a - b|| / max(||b||, floor) (SURVEY §8(c) comparator 2)."""
    a = np.asarray(a, dtype=float).reshape(len(b), -1)
    b = np.asarray(b, dtype=float).reshape(len(b), -1)
    den = np.maximum(np.linalg.norm(b, axis=1), floor)
    return float((np.linalg.norm(a - b, axis=1) / den).max()) if len(b) else 0.0


def oracle_pile_model():
    """The oracle's model of BASELINE config 4 (scenes.icosphere_pile(seed=0))."""
    from oracle import abd_oracle as O
    from paper_2201_10022_b200 import scenes
    from paper_2201_10022_b200.body import mass_matrix

    spec = scenes.icosphere_pile(seed=0)
    bodies, masses, stiff = [], [], []
    for m, dyn in zip(spec.meshes, spec.dynamic):
        d = m.vertices[m.edges[:, 1]] - m.vertices[m.edges[:, 0]]
        bodies.append(SimpleNamespace(rest=m.vertices, triangles=m.triangles, edges=m.edges,
                                      edge_rest_len_sq=np.einsum("ij,ij->i", d, d), dynamic=bool(dyn)))
        if dyn:
            gm, vol = mass_matrix(m, spec.density)
            masses.append(gm.matrix)
            stiff.append(spec.kappa_ortho * vol)
        else:
            masses.append(None)
            stiff.append(None)
    model = O.OracleModel(bodies, masses, stiff)
    prm = O.OracleParams(**spec.params)
    f = np.zeros((len(bodies), 12))
    g = np.asarray(spec.gravity, dtype=float)
    for b in model.dyn:
        f[b, :3] = masses[b][0, 0] * g
        f[b, 3:] = np.kron(g, masses[b][0, 3:6])
    return spec, model, prm, f
