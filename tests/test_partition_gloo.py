"""World-size-2 gloo tests (CPU) of the body-slab sharding logic.

The candidate set and energies come from the CPU oracle (checker); the code
under test is paper_2201_10022_b200.partition: slab ownership, halo bodies,
owned / counted pair selection and the rank-ordered scalar reduction.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_io import oracle_bodies
from oracle import abd_oracle as O
from paper_2201_10022_b200 import partition as PT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "contact.npz")))
    p = "ico_"
    bodies = oracle_bodies(p, g)
    q0, dq = g[p + "q0"], g[p + "dq"]
    d_hat, kappa = float(g[p + "params"][0]), float(g[p + "params"][1])
    return bodies, q0, dq, d_hat, kappa


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bodies, q0, dq, d_hat, kappa = _scene()
    full = O.broad_phase(bodies, q0, q0 + dq, d_hat)
    cent = q0[:, :3]  # the device cuts slabs on body positions p
    w = np.array([len(b.rest) + len(b.edges) + len(b.triangles) for b in bodies], dtype=float)
    owner = PT.slab_partition(cent, w, [b.dynamic for b in bodies], world)
    mine_vf = PT.owned_rows(full.vf, owner, rank)
    mine_ee = PT.owned_rows(full.ee, owner, rank)
    halo = PT.halo_bodies(full.overlap_pairs, owner, rank)
    # every body of an owned row is owned or halo (or replicated kinematic)
    for rows in (mine_vf, mine_ee):
        for b in np.unique(rows[:, [0, 2]]):
            assert owner[b] in (rank, -1) or b in set(halo.tolist())
    # union of owned rows == 1-GPU set (all_gather_object over gloo)
    got = [None] * world
    dist.all_gather_object(got, (mine_vf.tolist(), mine_ee.tolist()))
    uvf = PT.dedup_union([np.array(g_[0], dtype=np.int64).reshape(-1, 4) for g_ in got])
    uee = PT.dedup_union([np.array(g_[1], dtype=np.int64).reshape(-1, 4) for g_ in got])
    # energy: each rank adds its counted pairs; rank-ordered sum == global energy
    cvf = PT.counted_rows(full.vf, owner, rank)
    cee = PT.counted_rows(full.ee, owner, rank)
    e_part = O.contact_energy(bodies, q0, cvf, cee, kappa, d_hat)
    parts = [None] * world
    dist.all_gather_object(parts, e_part)
    total = PT.ordered_sum(parts)
    # the implemented split: body pairs by slab (disjoint sets, union = full set)
    pvf, pee = cvf, cee
    gp = [None] * world
    dist.all_gather_object(gp, (pvf.tolist(), pee.tolist(),
                                O.contact_energy(bodies, q0, pvf, pee, kappa, d_hat)))
    n_pvf = sum(len(x[0]) for x in gp)
    n_pee = sum(len(x[1]) for x in gp)
    uvf2 = PT.dedup_union([np.array(x[0], dtype=np.int64).reshape(-1, 4) for x in gp])
    uee2 = PT.dedup_union([np.array(x[1], dtype=np.int64).reshape(-1, 4) for x in gp])
    e_pairs = PT.ordered_sum([x[2] for x in gp])
    pair_ok = (n_pvf == len(full.vf) and n_pee == len(full.ee) and np.array_equal(uvf2, full.vf)
               and np.array_equal(uee2, full.ee))
    # global min CCD step: min over ranks of the evaluated rows' minima
    a_part = O.step_filter(bodies, q0, dq, pvf, pee, 0.1)
    t = torch.tensor([a_part], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if rank == 0:
        out.put((np.array_equal(uvf, full.vf), np.array_equal(uee, full.ee), total,
                 O.contact_energy(bodies, q0, full.vf, full.ee, kappa, d_hat), float(t.item()),
                 O.step_filter(bodies, q0, dq, full.vf, full.ee, 0.1), int((owner >= 0).sum()),
                 sorted(set(owner[owner >= 0].tolist())), pair_ok, e_pairs))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slab_sharding_gloo(world):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = out.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    vf_ok, ee_ok, total, ref, amin, aref, n_owned, parts, pair_ok, e_pairs = res
    assert vf_ok and ee_ok
    assert pair_ok  # slab-partitioned candidate sets are disjoint and complete
    assert e_pairs == pytest.approx(ref, rel=1e-12, abs=0)
    assert total == pytest.approx(ref, rel=1e-12, abs=0)
    assert amin == aref
    assert parts == list(range(world))


def test_slab_partition_balance():
    rng = np.random.default_rng(0)
    c = rng.uniform(0, 100, size=(1000, 3))
    c[:, 0] *= 3
    w = rng.integers(100, 1000, size=1000).astype(float)
    dyn = np.ones(1000, dtype=bool)
    dyn[:5] = False
    for n in (2, 4, 8):
        owner = PT.slab_partition(c, w, dyn, n)
        assert (owner[:5] == -1).all()
        loads = np.array([w[owner == k].sum() for k in range(n)])
        assert loads.max() <= 1.1 * loads.mean() + w.max()
        # contiguous slabs along x
        for k in range(n - 1):
            assert c[owner == k, 0].max() <= c[owner == k + 1, 0].min()
