"""Run the 10k-body pile with the GPU solver and save (q, q_dot) at given steps.

    python tools/make_checkpoint.py 100 [more steps...]

Writes bench_data/pile_step{N}.npz (q, q_dot, step, seed); the bench starts its
timed window from the committed checkpoint (SimState is the complete
inter-step state, solver.py:131-147).
"""
import os
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_2201_10022_b200 as P  # noqa: E402
from paper_2201_10022_b200 import scenes  # noqa: E402

targets = sorted(int(x) for x in sys.argv[1:]) or [100]
spec = scenes.icosphere_pile(seed=0)
model, state, params = spec.build()
out_dir = os.environ.get("ABD_CKPT_DIR", "bench_data")
os.makedirs(out_dir, exist_ok=True)
warnings.simplefilter("ignore")
t0 = time.time()
for s in range(max(targets)):
    state, st = P.advance_step(model, state, params)
    if state.step_index in targets:
        path = f"{out_dir}/pile_step{state.step_index}.npz"
        np.savez_compressed(path, q=state.q, q_dot=state.q_dot, step=state.step_index, seed=0,
                            time=state.time)
        print(f"saved {path} after {time.time() - t0:.1f}s", flush=True)
