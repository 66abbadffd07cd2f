"""Body-slab partitioned Newton steps on one GPU, vs the REFERENCE.

Two ranks share the GPU and reduce through torch.distributed gloo
(`dist.attach_torch`; NCCL differs only in who carries the reductions).  Each
rank evaluates the body pairs of its slab, the partial systems are all-reduced and
the Newton system is solved by the distributed slab PCG (csrc/k_chol.cu
slab_pcg).  Checked: the ranks hold bitwise-identical states; the device's slab
cut equals partition.slab_owner_of_q; the trajectories match the REFERENCE's
(tests/golden/box_stack.npz, ico_pile.npz) to 1e-6 relative per step with the
same Newton iteration counts, as the single-rank path does.
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
    return scenes.icosphere_pile(seed=3, nx=2, ny=2, nz=2, mu=0.5, subdiv=1).build()


def _worker(rank, world, port, scene, steps, out):
    import warnings

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2201_10022_b200 as P
    from paper_2201_10022_b200 import dist as pdist

    warnings.simplefilter("ignore")
    import ctypes as C

    from paper_2201_10022_b200 import _native
    from paper_2201_10022_b200 import partition as PT

    model, state, params = _box_stack() if scene == "box" else _ico_pile()
    pdist.attach_torch(model)
    its, traj = [], []
    owner_ok = True
    for _ in range(steps):
        q_before = state.q.copy()
        state, st = P.advance_step(model, state, params)
        its.append(st.iterations)
        traj.append(state.q.copy())
        own = np.zeros(len(model.bodies), dtype=np.int32)
        _native.check(_native.lib().abd_get_slab_owner(model.gpu_scene().ptr, own.ctypes.data, None))
        w = [len(b.rest) + len(b.edges) + len(b.triangles) for b in model.bodies]
        owner_ok &= bool(np.array_equal(own, PT.slab_owner_of_q(q_before, w, model.dynamic, world)))
    out.put((rank, np.array(traj), its, owner_ok))
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
        r, traj, its, owner_ok = out.get(timeout=600)
        res[r] = (traj, its, owner_ok)
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
def test_slab_partitioned_two_ranks_vs_reference(scene, steps):
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "box_stack.npz" if scene == "box" else "ico_pile.npz"))
    res = _run(scene, steps)
    t0, i0, ok0 = res[0]
    t1, i1, ok1 = res[1]
    assert np.array_equal(t0, t1), "ranks must hold identical (replicated) state"
    assert i0 == i1
    assert ok0 and ok1, "device slab cut differs from partition.slab_owner_of_q"
    assert i0 == [int(x) for x in g["iterations"][:steps]]
    for k in range(steps):
        ref = g["q"][k + 1]
        assert np.abs(t0[k] - ref).max() <= 1e-6 * np.abs(ref).max(), f"step {k}"
    ts, is_ = _single(scene, steps)
    assert is_ == i0
