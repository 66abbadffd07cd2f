"""Quick GPU probe: step the icosphere pile and print per-step stats."""
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_2201_10022_b200 as P  # noqa: E402
from paper_2201_10022_b200 import scenes  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 20
nz = int(sys.argv[2]) if len(sys.argv) > 2 else 25
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
t0 = time.time()
spec = scenes.icosphere_pile(nx=nx, ny=nx, nz=nz)
model, state, params = spec.build()
print(f"build {time.time() - t0:.1f}s bodies={len(model.bodies)}", flush=True)
warnings.simplefilter("ignore")
for s in range(steps):
    t = time.time()
    state, st = P.advance_step(model, state, params)
    tm = st.timings
    print(f"step {s} it={st.iterations} conv={st.converged} pcg={st.pcg_iterations} cand={st.candidates} "
          f"mind={st.min_distance:.3e} wall={time.time() - t:.3f}s "
          + " ".join(f"{k}={v * 1e3:.1f}ms" for k, v in tm.items()), flush=True)
