"""Dump the Newton system of a pile state for offline preconditioner studies.

    python tools/dump_system.py NX NZ STEPS OUT.npz

Runs the icosphere pile NX x NX x NZ for STEPS steps on the GPU, then saves the
BSR system (grad, diag blocks, upper off-diagonal keys/blocks) of the last
Newton iteration of the last step, plus q and the dynamic-body ids.
"""
import sys
import time
import warnings

import numpy as np

sys.path.insert(0, ".")
import paper_2201_10022_b200 as P  # noqa: E402
from paper_2201_10022_b200 import _native, scenes  # noqa: E402
import ctypes as C  # noqa: E402

nx, nz, steps, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
ckpt = sys.argv[5] if len(sys.argv) > 5 else None
keys_only = ckpt is not None
model, state, params = scenes.icosphere_pile(seed=0, nx=nx, ny=nx, nz=nz).build()
if ckpt:
    ck = np.load(ckpt)
    state.q, state.q_dot = ck["q"].copy(), ck["q_dot"].copy()
    state.step_index, state.time = int(ck["step"]), float(ck["time"])
warnings.simplefilter("ignore")
t0 = time.time()
for s in range(steps):
    state, st = P.advance_step(model, state, params)
    if s % 10 == 0 or s == steps - 1:
        print(f"step {st.step} it={st.iterations} pcg={st.pcg_iterations} wall={time.time() - t0:.1f}s", flush=True)
sc = model.gpu_scene()
L = _native.lib()
n = model.n_dyn
forces = model.forces(state.step_index, state.time + params.dt, state.q)
qt = P.solver.compute_q_tilde(model, state, params, forces)
n_off = C.c_int64(0)
_native.check(L.abd_assemble(sc.ptr, sc.q(state.q), sc.q(qt), float(params.dt), float(params.kappa_barrier),
                             float(params.d_hat), float(params.epsilon_v), C.byref(n_off)))
grad = np.empty(12 * n)
diag = np.empty((n, 12, 12))
keys = np.empty((n_off.value, 2), dtype=np.int64)
off = np.empty((n_off.value, 12, 12))
_native.check(L.abd_get_system(sc.ptr, grad, diag, keys, off))
nz_off = np.abs(off).reshape(len(off), -1).max(axis=1) > 0
if keys_only:
    np.savez_compressed(out, keys=keys, nz_off=nz_off, q=state.q, step=state.step_index)
else:
    np.savez_compressed(out, grad=grad, diag=diag, keys=keys, off=off, q=state.q, dyn=np.array(model.dyn_indices),
                        step=state.step_index)
print("saved", out, n, n_off.value, flush=True)
