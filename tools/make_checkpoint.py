"""Run the 10k-body pile with the GPU solver and save (q, q_dot) at given steps.

    python tools/make_checkpoint.py 100 [more steps...]            (from step 0)
    python tools/make_checkpoint.py --from bench_data/pile_step150.npz 190 [--out DIR]

Writes {out}/pile_step{N}.npz (q, q_dot, step, seed, time); the bench starts its
timed window from the committed checkpoint (SimState is the complete
inter-step state, solver.py:131-147).
"""
import argparse
import os
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_2201_10022_b200 as P  # noqa: E402
from paper_2201_10022_b200 import scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("steps", type=int, nargs="+")
ap.add_argument("--from", dest="src", default=None)
ap.add_argument("--out", default=os.environ.get("ABD_CKPT_DIR", "bench_data"))
args = ap.parse_args()
targets = sorted(args.steps)
spec = scenes.icosphere_pile(seed=0)
model, state, params = spec.build()
if args.src:
    ck = np.load(args.src)
    state = P.SimState(q=ck["q"].copy(), q_dot=ck["q_dot"].copy(), time=float(ck["time"]), step_index=int(ck["step"]))
os.makedirs(args.out, exist_ok=True)
warnings.simplefilter("ignore")
t0 = time.time()
while state.step_index < max(targets):
    state, st = P.advance_step(model, state, params)
    if state.step_index in targets:
        path = f"{args.out}/pile_step{state.step_index}.npz"
        np.savez_compressed(path, q=state.q, q_dot=state.q_dot, step=state.step_index, seed=0, time=state.time)
        print(f"saved {path} after {time.time() - t0:.1f}s", flush=True)
