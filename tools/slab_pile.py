"""Slab-partitioned steps of the 10k pile with W ranks sharing one GPU (gloo reductions):
distributed-PCG iteration counts per Newton iteration, and the state vs the 1-rank step.

    python tools/slab_pile.py [W] [STEPS] > gpurun_out/slab_pile.txt

Ranks on one GPU only validate the partitioned path (their kernels do not wait on one
another; the reductions go through the host); timings here are not scaling numbers.
"""
import os
import socket
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CKPT = os.path.join(ROOT, "bench_data", "pile_step150.npz")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _steps(world, rank, port, steps, out):
    import warnings

    warnings.simplefilter("ignore")
    import paper_2201_10022_b200 as P
    from paper_2201_10022_b200 import scenes

    if world > 1:
        import torch.distributed as dist

        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    model, _, params = scenes.icosphere_pile(seed=0).build()
    if world > 1:
        from paper_2201_10022_b200 import dist as pdist

        pdist.attach_torch(model)
    ck = np.load(CKPT)
    state = P.SimState(q=ck["q"].copy(), q_dot=ck["q_dot"].copy(), time=float(ck["time"]), step_index=int(ck["step"]))
    rows = []
    for _ in range(steps):
        t0 = time.perf_counter()
        state, st = P.advance_step(model, state, params)
        rows.append((st.iterations, st.pcg_iterations, time.perf_counter() - t0, st.min_distance))
    if out is not None:
        out.put((rank, state.q.copy(), rows))
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp

    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_steps, args=(world, r, port, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, qs, rows = q.get(timeout=1800)
        res[r] = (qs, rows)
    for p in procs:
        p.join(timeout=60)
    p1 = ctx.Process(target=_steps, args=(1, 0, 0, steps, q))
    p1.start()
    _, q1, rows1 = q.get(timeout=1800)
    p1.join(timeout=60)
    for r in range(world):
        qs, rows = res[r]
        print(f"rank {r}: (newton its, pcg its, s, min dist) per step {rows}")
        print(f"rank {r}: |q - q_1rank| / |q| = {np.abs(qs - q1).max() / np.abs(q1).max():.3e}")
    print(f"1 rank: {rows1}")
    for r in range(world):
        qs, rows = res[r]
        its = sum(x[0] for x in rows)
        pcg = sum(x[1] for x in rows)
        print(f"rank {r}: mean distributed-PCG iterations per Newton iteration {pcg / max(its, 1):.2f}")


if __name__ == "__main__":
    main()
