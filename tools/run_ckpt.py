"""Step the 10k pile from a committed checkpoint and print per-step Newton counts and
wall times (tool for Cholesky / latency studies; set ABD_* trace switches in the env).

    python tools/run_ckpt.py 190 STEPS [OUT.npz]
"""
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_2201_10022_b200 as P  # noqa: E402
from paper_2201_10022_b200 import scenes  # noqa: E402

step, nsteps = int(sys.argv[1]), int(sys.argv[2])
warnings.simplefilter("ignore")
model, state, params = scenes.icosphere_pile(seed=0).build()
ck = np.load(f"bench_data/pile_step{step}.npz")
state = P.SimState(q=ck["q"].copy(), q_dot=ck["q_dot"].copy(), time=float(ck["time"]), step_index=int(ck["step"]))
for i in range(nsteps):
    t0 = time.perf_counter()
    state, st = P.advance_step(model, state, params)
    print(f"step {state.step_index} its {st.iterations} wall {1e3 * (time.perf_counter() - t0):.1f} ms "
          f"min_d {st.min_distance:.3e}", flush=True)
if len(sys.argv) > 3:
    np.savez(sys.argv[3], q=state.q, q_dot=state.q_dot)
