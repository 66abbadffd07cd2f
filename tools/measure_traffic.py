"""Measured DRAM traffic and executed FP64 flops per launch of the path's kernels
(bench.py roofline.traffic and the %FP64 figures).

    python tools/measure_traffic.py [--workload pile|chainmail|cubes|boxstack] [--steps 1]

Runs `bench.py` (one short window, no e2e / CPU legs) under

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none

restricted to the kernels behind the bench's instrumented groups, sums the DRAM bytes
and the executed DFMA / DADD / DMUL thread instructions and DMMA (m8n8k4 f64) warp
instructions of each group and divides by the group's launches as the bench counts them (one per
Newton iteration for K2/K3/K4/K5), and writes profiles/traffic_<workload>.json keyed
by the hash of the CUDA sources (bench.py ignores a capture of another source tree).
ncu replays each kernel with cold caches and serialised launches: the bytes are an
upper bound of what the live step moves (L2 reuse across kernels is lost).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GROUPS = {  # bench.Run.kernel_stats group (K2-K5) or SURVEY kernel (K1, K6) -> kernel name prefixes (csrc/)
    "k_chol": ("k_chol_sched", "k_chol_iso", "k_chol_apos", "k_chol_sched_init"),
    "k_pair_blocks": ("k_pair_blocks",),
    "k_ccd": ("k_ccd",),
    "k_prim_pairs": ("k_prim_pairs",),
    "k_body_terms": ("k_body_terms",),
    "k_energy_all": ("k_energy_all",),
}
METRICS = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
           "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "sm__inst_executed_pipe_tensor_subpipe_dmma.sum")
NCU = "/usr/local/cuda/bin/ncu"


def group_of(name):
    base = name.split("(")[0].split("<")[0].split("::")[-1].strip()
    base = base.replace("void ", "")
    for g, prefixes in GROUPS.items():
        if any(base == p or base.startswith(p) for p in prefixes):
            return g
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="pile")
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    import bench

    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    log = os.path.join(ROOT, "gpurun_out", f"traffic_{a.workload}.csv")
    out_json = os.path.join(ROOT, "gpurun_out", f"traffic_{a.workload}_bench.json")
    cmd = [NCU, "--metrics", ",".join(METRICS),
           "--clock-control", "none", "--csv", "--log-file", log,
           "-k", "regex:k_chol|k_pair_blocks|k_ccd|k_prim_pairs|k_body_terms|k_energy_all",
           sys.executable, os.path.join(ROOT, "bench.py"), "--workload", a.workload, "--steps", str(a.steps),
           "--warmup", "0", "--no-e2e", "--no-cpu", "--no-full-run"]
    if a.workload == "pile":
        cmd += ["--window-steps", str(a.steps)]
    with open(out_json, "w") as f:
        subprocess.run(cmd, check=True, stdout=f, cwd=ROOT)
    line = json.loads(open(out_json).read().strip().splitlines()[-1])
    kst = line["roofline"]["kernels"]
    rows = [r for r in csv.DictReader(io.StringIO("".join(l for l in open(log) if l.startswith('"'))))]
    acc = {}
    for r in rows:
        g = group_of(r["Kernel Name"])
        if g is None:
            continue
        d = acc.setdefault(g, {"read": 0.0, "write": 0.0, "ns": 0.0, "dfma": 0.0, "dadd": 0.0, "dmul": 0.0,
                               "dmma": 0.0, "kernels": set(), "ids": set()})
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        if r["Metric Name"] == "dram__bytes_read.sum":
            d["read"] += v * scale
        elif r["Metric Name"] == "dram__bytes_write.sum":
            d["write"] += v * scale
        elif r["Metric Name"] == "gpu__time_duration.sum":
            d["ns"] += v * scale
        else:
            for key in ("dfma", "dadd", "dmul", "dmma"):
                if f"_{key}" in r["Metric Name"]:
                    d[key] += v * (scale if unit not in ("byte", "Kbyte", "Mbyte", "Gbyte") else 1)
        d["kernels"].add(r["Kernel Name"].split("(")[0])
        d["ids"].add(r["ID"])
    peak = None
    try:
        peak = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
    except Exception:
        try:
            peak = json.load(open(os.path.join(ROOT, "gpurun_out", "fp64_peak.json")))
        except Exception:
            pass
    iters = line["config"]["window"]["newton_iters"] if a.workload == "pile" else None
    res = {}
    for g, d in acc.items():
        live = kst.get(g)
        n = (live or {}).get("launches") or iters or len(d["ids"])
        flops = 2.0 * d["dfma"] + d["dadd"] + d["dmul"] + 512.0 * d["dmma"]
        # FP64 rate: executed flops over the LIVE kernel time (bench CUDA events) when the
        # bench instruments the group, else over the ncu (cold, serialised) duration
        ms = (live["ms"] / live["launches"]) if live and live.get("launches") else d["ns"] / 1e6 / n
        tf = flops / n / (ms * 1e-3) / 1e12 if ms else None
        res.setdefault(g, {})["fp64"] = {
            "flops_per_launch": flops / n, "dfma": d["dfma"] / n, "dadd": d["dadd"] / n, "dmul": d["dmul"] / n,
            "dmma_warp_inst": d["dmma"] / n, "ms_per_launch": ms,
            "time_source": "bench CUDA events (live)" if live else "ncu gpu__time_duration (cold)",
            "achieved_tflops": tf,
            "peak_tflops": (peak or {}).get("dfma_tflops"),
            "frac_of_dfma_peak": tf / peak["dfma_tflops"] if (tf and peak) else None}
        res[g].update({"dram_bytes_per_launch": (d["read"] + d["write"]) / n if n else None,
                  "dram_read_per_launch": d["read"] / n if n else None,
                  "dram_write_per_launch": d["write"] / n if n else None,
                  "ncu_kernel_launches": len(d["ids"]), "bench_launches": n,
                  "algorithmic_bytes_per_launch": live["bytes"] / n if (live and n) else None,
                  "ncu_ms_per_launch": d["ns"] / 1e6 / n if n else None,
                  "kernels": sorted(d["kernels"])})
    out = {"workload": a.workload, "src_hash": bench.src_hash(), "command": " ".join(cmd[:12]) + " ...",
           "note": "ncu replay: cold caches, serialised launches; per launch = per bench group launch",
           "kernels": res}
    path = os.path.join(ROOT, "profiles", f"traffic_{a.workload}.json")
    for p in (path, os.path.join(ROOT, "gpurun_out", f"traffic_{a.workload}.json")):
        with open(p, "w") as f:
            json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
