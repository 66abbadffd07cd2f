"""Run K pile steps from a checkpoint with per-Newton-iteration tracing.

    ABD_TRACE_NEWTON=1 python tools/trace_step.py CKPT.npz K
"""
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_2201_10022_b200 as P  # noqa: E402
from paper_2201_10022_b200 import scenes  # noqa: E402

ck = np.load(sys.argv[1])
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
model, state, params = scenes.icosphere_pile(seed=int(ck["seed"])).build()
state.q = ck["q"].copy()
state.q_dot = ck["q_dot"].copy()
state.step_index = int(ck["step"])
state.time = float(ck["time"])
warnings.simplefilter("ignore")
for _ in range(K):
    t0 = time.time()
    state, st = P.advance_step(model, state, params)
    print(f"step {st.step} it={st.iterations} conv={st.converged} pcg={st.pcg_iterations} "
          f"mind={st.min_distance:.3e} wall={time.time() - t0:.3f}s "
          + " ".join(f"{k}={v * 1e3:.1f}ms" for k, v in st.timings.items()), file=sys.stderr, flush=True)
