"""GPU timeline of pile Newton steps through CUPTI (torch.profiler): kernel/memcpy
spans on the device, idle gaps between them and what precedes each gap.

    python tools/gpu_timeline.py [STEPS] [pile|boxstack|cubes|chainmail] [CKPT] > gpurun_out/timeline.txt
"""
import collections
import ctypes as C
import json
import os
import sys
import warnings

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_10022_b200 import _native, scenes  # noqa: E402
from paper_2201_10022_b200.solver import step_params_c  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1
WL = sys.argv[2] if len(sys.argv) > 2 else "pile"
torch.cuda.init()
torch.zeros(1, device="cuda")
spec = {"pile": scenes.icosphere_pile, "boxstack": scenes.box_stack, "cubes": scenes.cube_drop,
        "chainmail": scenes.chainmail}[WL](seed=0)
model, state, params = spec.build()
if WL == "pile":
    ck = np.load(sys.argv[3] if len(sys.argv) > 3 else os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench_data", "pile_step150.npz"))
    q, qd = ck["q"].copy(), ck["q_dot"].copy()
else:
    q, qd = state.q.copy(), state.q_dot.copy()
L = _native.lib()
sc = model.gpu_scene()
forces = np.ascontiguousarray(model.forces(0, 0.0, q))
_native.check(L.abd_set_state(sc.ptr, q.ctypes.data, qd.ctypes.data))
cp = step_params_c(params)
st = _native.StepStatsC()
warnings.simplefilter("ignore")
_native.check(L.abd_advance_step(sc.ptr, forces.ctypes.data, C.byref(cp), C.byref(st), None))
for _ in range(2):
    _native.check(L.abd_advance_step(sc.ptr, None, C.byref(cp), C.byref(st), None))
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(K):
        _native.check(L.abd_advance_step(sc.ptr, None, C.byref(cp), C.byref(st), None))
    torch.cuda.synchronize()
path = "/tmp/abd_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
t0, t1 = gpu[0]["ts"], gpu[-1]["ts"] + gpu[-1]["dur"]
busy = sum(e["dur"] for e in gpu)
print(f"steps={K} iters={st.iterations} span={t1 - t0:.0f}us busy={busy:.0f}us ({100 * busy / (t1 - t0):.1f}%) ops={len(gpu)}")
bycat = collections.Counter()
for e in gpu:
    bycat[e["cat"]] += e["dur"]
print("busy by category:", dict(bycat))
# true idle time: no op on any stream; each gap keyed by the op that ended last before
# it and the op that starts it
gaps = collections.defaultdict(lambda: [0, 0.0])
gap_tot = 0.0
end, last = gpu[0]["ts"] + gpu[0]["dur"], gpu[0]
for b in gpu[1:]:
    g = b["ts"] - end
    if g > 0:
        gap_tot += g
        key = last["name"].split("(")[0][:48] + " -> " + b["name"].split("(")[0][:48]
        gaps[key][0] += 1
        gaps[key][1] += g
    if b["ts"] + b["dur"] > end:
        end, last = b["ts"] + b["dur"], b
print(f"idle (no op on any stream) total {gap_tot:.0f}us")
for k, (n, g) in sorted(gaps.items(), key=lambda kv: -kv[1][1])[:45]:
    print(f"  {g:9.0f}us n={n:5d} avg={g / n:7.1f}us  {k}")
kt = collections.defaultdict(lambda: [0, 0.0])
for e in gpu:
    k = e["name"].split("(")[0][:60]
    kt[k][0] += 1
    kt[k][1] += e["dur"]
print("device time by op:")
for k, (n, d) in sorted(kt.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"  {d:9.0f}us n={n:5d} avg={d / n:7.1f}us  {k}")

# one Newton iteration in the middle of the last step: ops with stream, start, duration
if os.environ.get("ABD_TIMELINE_ITER"):
    ks = [i for i, e in enumerate(gpu) if e["name"].startswith("abd::k_chol_flow") or e["name"].startswith("abd::k_chol_sched")]
    if len(ks) > 3:
        a, b = ks[len(ks) // 2], ks[len(ks) // 2 + 1]
        t_a = gpu[a]["ts"]
        print("one iteration (us from the Cholesky launch; stream; duration):")
        for e in gpu[a:b + 1]:
            print(f"  {e['ts'] - t_a:8.1f} s{e.get('args', {}).get('stream', '?'):<3} {e['dur']:7.1f}  {e['name'].split('(')[0][:70]}")
