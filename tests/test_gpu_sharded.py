"""Partitioned multi-rank Newton steps on one GPU.

Two ranks share the GPU and reduce through torch.distributed gloo
(`dist.attach_torch`); the per-pair work is split by overlap body pair.  The
ranks must stay bitwise identical to each other, take the same Newton
iterations as the single-rank step, and match the reference trajectory.
(The NCCL backend differs only in who carries the reductions.)
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _box_stack():
    from paper_2201_10022_b200 import scenes
    return scenes.box_stack(seed=0).build()


def _ico_pile():
    from paper_2201_10022_b200 import scenes
    return scenes.icosphere_pile(seed=0, nx=2, ny=2, nz=2, subdiv=1).build()


def _worker(rank, world, port, scene, steps, out):
    import warnings

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2201_10022_b200 as P
    from paper_2201_10022_b200 import dist as pdist

    warnings.simplefilter("ignore")
    model, state, params = _box_stack() if scene == "box" else _ico_pile()
    pdist.attach_torch(model)
    its, traj = [], []
    for _ in range(steps):
        state, st = P.advance_step(model, state, params)
        its.append(st.iterations)
        traj.append(state.q.copy())
    out.put((rank, np.array(traj), its))
    dist.barrier()
    dist.destroy_process_group()


def _run(scene, steps, world=2):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scene, steps, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, traj, its = out.get(timeout=600)
        res[r] = (traj, its)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def _single(scene, steps):
    import warnings

    import paper_2201_10022_b200 as P

    warnings.simplefilter("ignore")
    model, state, params = _box_stack() if scene == "box" else _ico_pile()
    its, traj = [], []
    for _ in range(steps):
        state, st = P.advance_step(model, state, params)
        its.append(st.iterations)
        traj.append(state.q.copy())
    return np.array(traj), its


@pytest.mark.parametrize("scene,steps", [("box", 30), ("ico", 25)])
def test_partitioned_two_ranks_match_single(scene, steps):
    res = _run(scene, steps)
    t0, i0 = res[0]
    t1, i1 = res[1]
    assert np.array_equal(t0, t1), "ranks must hold identical (replicated) state"
    assert i0 == i1
    ts, is_ = _single(scene, steps)
    assert i0 == is_
    for k in range(steps):
        scale = np.abs(ts[k]).max()
        assert np.abs(t0[k] - ts[k]).max() <= 1e-9 * scale, f"step {k}"
