"""Per-step relative DOF error of a small BASELINE config against its reference golden.

    python tools/traj_err.py cube_drop|chainmail [linear_solver]
"""
import sys
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_2201_10022_b200 as P  # noqa: E402
from paper_2201_10022_b200 import scenes  # noqa: E402

name = sys.argv[1]
solver = sys.argv[2] if len(sys.argv) > 2 else "cholesky"
g = np.load(f"tests/golden/{name}.npz")
spec = scenes.cube_drop(seed=0, n=2) if name == "cube_drop" else scenes.chainmail(seed=0, n_chains=2, links=3,
                                                                                     chains_x=2)
model, state, params = spec.build()
params = P.StepParams(**{**params.__dict__, "linear_solver": solver})
warnings.simplefilter("ignore")
for s in range(len(g["iterations"])):
    state, st = P.advance_step(model, state, params)
    ref = g["q"][s + 1]
    err = np.abs(state.q - ref).max() / np.abs(ref).max()
    print(s, st.iterations, int(g["iterations"][s]), f"{err:.3e}", f"{st.min_distance:.3e}", flush=True)
