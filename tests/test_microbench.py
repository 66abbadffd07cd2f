"""BASELINE config 2 (kernel microbenchmark): synthetic pair geometry -> soup scene.

CPU: the soup layout reproduces every generated pair's rest points exactly and
its candidate rows follow the CandidateSet convention.  GPU: `assemble` over the
soup scene agrees with the oracle's `assemble` (solver.py:257-342) on the same
pairs, and the resident PCG meets the 1e-8 residual contract.
"""
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import rel_err
from oracle import abd_oracle as O
from paper_2201_10022_b200 import microbench as mb
from paper_2201_10022_b200 import scenes

TOL = 1e-9  # norm-relative, per BSR block (SURVEY §8(c) comparator 2)
ACC_TOL = 1e-9  # per entry, relative to the block scale of summed |contributions| (= the per-pair TOL)


def _small(seed=3, B=240, n=2500):
    d = scenes.microbench_pairs(seed=seed, n_bodies=B, n_vf=n, n_ee=n)
    return d, mb.soup_arrays(d)


def _soup_bodies(a, B):
    bodies = []
    for b in range(B):
        v0, v1 = a["v_off"][b], a["v_off"][b + 1]
        e0, e1 = a["e_off"][b], a["e_off"][b + 1]
        t0, t1 = a["t_off"][b], a["t_off"][b + 1]
        bodies.append(SimpleNamespace(rest=a["rest"][v0:v1], edges=a["edges"][e0:e1], triangles=a["tris"][t0:t1],
                                      edge_rest_len_sq=a["el2"][e0:e1], dynamic=True))
    return bodies


def test_soup_reproduces_pairs():
    d, a = _small()
    rest, vo, to, eo = a["rest"], a["v_off"], a["t_off"], a["e_off"]
    vf, ee = a["vf"], a["ee"]
    x0 = rest[vo[vf[:, 0]] + vf[:, 1]]
    tri = a["tris"][to[vf[:, 2]] + vf[:, 3]] + vo[vf[:, 2]][:, None]
    assert np.array_equal(np.concatenate([x0[:, None], rest[tri]], axis=1), d["vf"]["rest"][a["vf_perm"]])
    ea = a["edges"][eo[ee[:, 0]] + ee[:, 1]] + vo[ee[:, 0]][:, None]
    eb = a["edges"][eo[ee[:, 2]] + ee[:, 3]] + vo[ee[:, 2]][:, None]
    er = d["ee"]["rest"].copy()
    sw = d["ee"]["body_a"] > d["ee"]["body_b"]
    er[sw] = er[sw][:, [2, 3, 0, 1]]
    er = er[a["ee_perm"]]
    assert np.array_equal(np.concatenate([rest[ea], rest[eb]], axis=1), er)
    assert (ee[:, 0] < ee[:, 2]).all()
    # grouped by body pair (the runs of the fused assembly)
    for rows in (vf, ee):
        k = rows[:, 0] * (1 << 32) + rows[:, 2]
        assert (np.diff(k) >= 0).all()
    # every pair's body pair is a block of the Morton +-1..4 pattern
    ov = {tuple(r) for r in a["ov"]}
    for rows in (vf, ee):
        for i, j in zip(rows[:, 0], rows[:, 2]):
            assert (min(i, j), max(i, j)) in ov
    # pattern: 4 neighbours ahead of each body in Morton order
    B = len(d["q"])
    assert len(a["ov"]) == 4 * B - 10


def test_pairs_distances_in_range():
    d, a = _small(seed=5)
    bodies = _soup_bodies(a, len(d["q"]))
    X = O.all_world_points(bodies, d["q"])
    for kind, rows in (("vf", a["vf"]), ("ee", a["ee"])):
        z, _, _ = O.gather(kind, bodies, X, rows)
        d2 = O.pair_d2(kind, z)
        assert (d2 > 0).all() and (np.sqrt(d2) < d["d_hat"] * (1 + 1e-6)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("runs", ["0", "1"])
def test_microbench_assemble_and_pcg_vs_oracle(runs, monkeypatch):
    """runs=1: the fused run assembly (k_pair_runs: records stay in shared memory, one
    dense partial per run of one body pair), which config 2's 20M active pairs take."""
    monkeypatch.setenv("ABD_RUNS", runs)
    d, a = _small()
    B = len(d["q"])
    sysm = mb.PairSystem(d)
    n_off = sysm.assemble()
    grad, diag, keys, off = sysm.system()
    bodies = _soup_bodies(a, B)
    M1 = mb.unit_cube_mass()
    om = O.OracleModel(bodies, [M1] * B, [1e8] * B)
    prm = O.OracleParams(dt=0.01, d_hat=d["d_hat"], kappa_barrier=1e4)
    ip = O.OracleIP(sysm.q_tilde, O._empty_friction(0.0), O.OracleCandidates(a["vf"], a["ee"], a["ov"]))
    g_ref, diag_ref, off_ref = O.assemble(om, d["q"], ip, prm)
    assert n_off == len(off_ref)
    # the sums of thousands of stiff pair terms cancel: bound each entry's error by
    # ACC_TOL x the sum of the absolute contributions (a summation-order-free bound)
    blk = O.contact_blocks(bodies, d["q"], a["vf"], a["ee"], 1e4, d["d_hat"])
    g_abs = np.zeros((B, 12))
    h_abs = np.zeros((B, 12, 12))
    o_abs = {k: np.zeros((12, 12)) for k in off_ref}
    for k in range(len(blk.body_a)):
        i, j = int(blk.body_a[k]), int(blk.body_b[k])
        g_abs[i] += np.abs(blk.grad[k, :12])
        g_abs[j] += np.abs(blk.grad[k, 12:])
        h_abs[i] += np.abs(blk.hess[k, :12, :12])
        h_abs[j] += np.abs(blk.hess[k, 12:, 12:])
        up = np.abs(blk.hess[k, :12, 12:])
        o_abs[(min(i, j), max(i, j))] += up if i < j else up.T
    # per body block: the scale is the largest summed |contribution| in the block
    # (inertia and orthogonality terms included through |reference|)
    g_scale = (g_abs + np.abs(g_ref.reshape(B, 12))).max(axis=1, keepdims=True)
    h_scale = (h_abs + np.abs(diag_ref)).max(axis=(1, 2), keepdims=True)
    rg = np.abs(grad.reshape(B, 12) - g_ref.reshape(B, 12)) / g_scale
    rh = np.abs(diag - diag_ref) / h_scale
    assert rg.max() <= ACC_TOL, f"gradient: worst |err| / block scale = {rg.max():.3e} (body {rg.max(axis=1).argmax()})"
    assert rh.max() <= ACC_TOL, f"diagonal blocks: worst |err| / block scale = {rh.max():.3e}"
    assert rel_err(grad, g_ref) <= 1e-7
    assert sorted(tuple(k) for k in keys) == sorted(off_ref.keys())
    for k, blk_ in zip(keys, off):
        ref = off_ref[tuple(k)]
        sc = o_abs[tuple(k)].max() + np.abs(ref).max()
        assert np.abs(blk_ - ref).max() <= ACC_TOL * sc, f"off block {tuple(k)}"
    dx, iters, rel = sysm.solve(1e-8)
    assert iters > 0 and rel <= 1e-8
    r = O.bsr_matvec(diag_ref, off_ref, dx) + g_ref
    assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(g_ref) * 1.01
