"""GPU timeline (CUPTI via torch.profiler) of one config-2 assembly: ops in start order with
stream, start and duration, and the idle gaps.

    python tools/micro_timeline.py [BODIES] [PAIRS] > gpurun_out/micro_timeline.txt
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2201_10022_b200 import microbench, scenes  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
npairs = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
torch.cuda.init()
torch.zeros(1, device="cuda")
sysm = microbench.PairSystem(scenes.microbench_pairs(seed=0, n_bodies=nb, n_vf=npairs, n_ee=npairs, d_lo_frac=0.0))
for _ in range(2):
    sysm.assemble()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sysm.assemble()
    torch.cuda.synchronize()
path = "/tmp/abd_micro_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
gpu = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
gpu.sort(key=lambda e: e["ts"])
t0 = gpu[0]["ts"]
t1 = max(e["ts"] + e["dur"] for e in gpu)
print(f"span {t1 - t0:.0f} us, busy {sum(e['dur'] for e in gpu):.0f} us, ops {len(gpu)}")
end = t0
for e in gpu:
    gap = e["ts"] - end
    print(f"{e['ts'] - t0:10.1f} s{e.get('args', {}).get('stream', '?'):<3} {e['dur']:10.1f} "
          f"{'gap %8.1f' % gap if gap > 20 else '            '}  {e['name'].split('(')[0][:70]}")
    end = max(end, e["ts"] + e["dur"])
