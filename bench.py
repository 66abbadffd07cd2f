#!/usr/bin/env python
"""Benchmark: fp64 ABD Newton steps on the 10k-body icosphere pile (BASELINE config 4).

    python bench.py [--gpus N --steps K --warmup W --start S]
    python bench.py --impl reference ...        (CPU oracle arm)

A "step" is one implicit time step (`advance_step`: broad phase, friction
precompute, Newton loop with assembly / Cholesky / CCD / line search, stats).
By default the timed steps are [153, 163) from the committed step-150
checkpoint of the 200-step pile run (the late, contact-dense phase);
`--ckpt none --start S` times [S + W, S + W + K) from the seeded initial state.
`value` is measured on the device-resident C-ABI path; `e2e` repeats the same
window through the Python API (`advance_step`) with host numpy state (H2D q,
q_dot, forces and D2H q, q_dot every step).  Under torchrun (N > 1) the ranks
partition ONE pile (per-pair work split by overlap body pair, NCCL all-reduce
of the system, replicated solve): strong scaling, max-over-ranks device time.
Prints one JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": HBM_FALLBACK}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index=0):
        self.path = f"/tmp/abd_clocks_{os.getpid()}.csv"
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if len(r) > 5 + k and "Active" in r[5 + k]
                          and "Not" not in r[5 + k]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
def oracle_sample_rate(spec_kw, start_steps, budget_s, threads_note, threads=None):
    """Oracle advance_step steps/s on a 8x8x2 sub-pile (same generator), scaled to 10k bodies."""
    from oracle import abd_oracle as O
    from paper_2201_10022_b200 import scenes
    from paper_2201_10022_b200.body import mass_matrix

    spec = scenes.icosphere_pile(seed=0, nx=8, ny=8, nz=2, **spec_kw)
    from types import SimpleNamespace
    bodies, masses, stiff = [], [], []
    cache = {}
    for m, dyn in zip(spec.meshes, spec.dynamic):
        d = m.vertices[m.edges[:, 1]] - m.vertices[m.edges[:, 0]]
        bodies.append(SimpleNamespace(rest=m.vertices, triangles=m.triangles, edges=m.edges,
                                      edge_rest_len_sq=np.einsum("ij,ij->i", d, d), dynamic=bool(dyn)))
        if dyn:
            if id(m) not in cache:
                cache[id(m)] = mass_matrix(m, spec.density)
            gm, vol = cache[id(m)]
            masses.append(gm.matrix)
            stiff.append(spec.kappa_ortho * vol)
        else:
            masses.append(None)
            stiff.append(None)
    model = O.OracleModel(bodies, masses, stiff)
    prm = O.OracleParams(**spec.params)
    f = np.zeros((len(bodies), 12))
    g = np.array(spec.gravity)
    for b in model.dyn:
        f[b, :3] = masses[b][0, 0] * g
        f[b, 3:] = np.kron(g, masses[b][0, 3:6])
    q, qd = spec.q0.copy(), spec.q_dot0.copy()
    warnings.simplefilter("ignore")
    from threadpoolctl import threadpool_limits
    limiter = threadpool_limits(limits=threads) if threads else None
    for _ in range(start_steps):
        q, qd, _ = O.advance_step(model, q, qd, f, prm, min_distance=False)
    n = 0
    t0 = time.perf_counter()
    iters = 0
    while True:
        q, qd, st = O.advance_step(model, q, qd, f, prm, min_distance=True)
        n += 1
        iters += st.iterations
        el = time.perf_counter() - t0
        if el >= budget_s or n >= 200:
            break
    if limiter is not None:
        limiter.restore_original_limits()
    nb = int(model.dynamic.sum())
    scale = nb / 10000.0
    return {"rate_sample": n / el, "steps": n, "seconds": el, "iters": iters, "bodies": nb,
            "value": n / el * scale, "scale": scale, "note": threads_note}


def run_reference(args):
    """--impl reference: the oracle restatement of the reference path on the host CPU."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    r = oracle_sample_rate({}, args.warmup, args.steps * 4.0, f"numpy, {cores} host threads available")
    line = {
        "impl": "reference", "metric": "sim steps/s (10k-body icosphere pile, fp64 ABD)", "value": r["value"],
        "unit": "steps/s", "n_gpus": args.gpus, "steps": r["steps"], "warmup": args.warmup,
        "ms_per_step": 1e3 / r["value"] if r["value"] else None, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded procedural scene)",
        "config": {"workload": "icosphere_pile 20x20x25 (10,001 bodies, seed 0): CPU sample = 8x8x2 sub-pile "
                               "of the same generator, scaled linearly by body count",
                   "parallelism": f"cpu ({cores} host threads)"},
        "cpu_baseline": {"value": r["value"], "unit": "steps/s", "cores": cores, "kind": "port",
                         "sample": f"oracle/abd_oracle.py advance_step on a 8x8x2 sub-pile ({r['bodies']} "
                                   f"icospheres + ground, same generator) from step {args.warmup}, "
                                   f"{r['steps']} steps in {r['seconds']:.1f}s, x{r['scale']:.4f} linear "
                                   "body scaling to 10k (optimistic for the CPU)"},
        "e2e": {"value": r["value"], "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_micro(args):
    """--workload micro: BASELINE config 2 (SURVEY §8(d) kernel microbenchmark).

    One step = `assemble` (K1 + K3 + BSR reduction) over 10M VF + 10M EE synthetic
    pairs on 100k bodies, then the block-Jacobi PCG to 1e-8 relative residual.
    """
    from paper_2201_10022_b200 import _native, microbench, scenes

    t0 = time.perf_counter()
    data = scenes.microbench_pairs(seed=0, n_bodies=args.micro_bodies, n_vf=args.micro_pairs,
                                   n_ee=args.micro_pairs)
    sysm = microbench.PairSystem(data)
    setup_s = time.perf_counter() - t0
    L = _native.lib()
    sc = sysm.scene
    for _ in range(args.warmup):
        sysm.assemble()
        sysm.solve()
    _native.check(L.abd_kernel_stats_reset(sc.ptr))
    n_launch0 = _native.kernel_launches()
    asm_ms, sol_ms, iters, rels = [], [], [], []
    ms = C.c_double(0.0)
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            _native.check(L.abd_timer_start(sc.ptr))
            sysm.assemble()
            _native.check(L.abd_timer_stop(sc.ptr, C.byref(ms)))
            asm_ms.append(ms.value)
            _native.check(L.abd_timer_start(sc.ptr))
            _, it, rel = sysm.solve()
            _native.check(L.abd_timer_stop(sc.ptr, C.byref(ms)))
            sol_ms.append(ms.value)
            iters.append(it)
            rels.append(rel)
    launches = _native.kernel_launches() - n_launch0
    P_all = sysm.n_vf + sysm.n_ee
    B = sysm.B
    n_blk = B + 2 * sysm.n_off
    tot_ms = float(np.sum(asm_ms) + np.sum(sol_ms))
    kst = {}
    for which, name in ((0, "k_cg"), (1, "k_pair_blocks")):
        n_, t_, b_, u_ = C.c_int64(), C.c_double(), C.c_double(), C.c_int64()
        _native.check(L.abd_kernel_stats(sc.ptr, which, C.byref(n_), C.byref(t_), C.byref(b_), C.byref(u_)))
        kst[name] = {"launches": n_.value, "ms": t_.value, "bytes": b_.value, "units": u_.value}
    pk, pk_kind = peaks()
    hbm = float(pk.get("hbm_gbs", HBM_FALLBACK))
    # K4 per PCG iteration: 1152 (N_blk + B_d) + 13 x 96 B_d
    it_bytes = 1152.0 * (n_blk + B) + 13 * 96.0 * B
    it_ms = float(np.sum(sol_ms)) / max(1, int(np.sum(iters)))
    # K3 per call, pre-gathered form: 104 P_vf + 112 P_ee + 1152 N_blk + 192 B
    k3_bytes = 104.0 * sysm.n_vf + 112.0 * sysm.n_ee + 1152.0 * n_blk + 192.0 * B
    k3_ms = float(np.mean(asm_ms))
    cpu = None
    if not args.no_cpu:
        cpu = micro_cpu_rate(args.cpu_budget)
    line = {
        "metric": "microbench assemble + PCG time (100k bodies, 10M VF + 10M EE pairs, fp64)",
        "value": tot_ms / args.steps, "unit": "ms", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_ms / args.steps, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, scenes.microbench_pairs)",
        "config": {"workload": f"BASELINE config 2: {B} bodies, {sysm.n_vf} VF + {sysm.n_ee} EE pairs, "
                               f"Morton +-1..4 body graph ({sysm.n_off} off-diagonal blocks), all pairs active",
                   "assemble_ms": float(np.mean(asm_ms)), "pcg_ms": float(np.mean(sol_ms)),
                   "pcg_iters": iters, "pcg_rel_res": rels, "pcg_ms_per_iter": it_ms,
                   "pairs_per_s_assemble": P_all / (k3_ms * 1e-3), "setup_s": setup_s,
                   "l2": "inputs (~2 GB rest + 22 GB pair records) exceed L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": "K4 PCG iteration (k_cg) / K3 assemble",
                     "achieved": it_bytes / (it_ms * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": it_bytes / (it_ms * 1e-3) / 1e9 / hbm, "traffic": None,
                     "algorithmic_bytes_per_launch": it_bytes,
                     "bytes_model": "K4: 1152 (N_blk + B_d) + 13 x 96 B_d per PCG iteration",
                     "assemble": {"achieved": k3_bytes / (k3_ms * 1e-3) / 1e9, "bytes": k3_bytes,
                                  "frac": k3_bytes / (k3_ms * 1e-3) / 1e9 / hbm,
                                  "bytes_model": "K3 pre-gathered: 104 P_vf + 112 P_ee + 1152 N_blk + 192 B"},
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})", "kernels": kst},
        "cpu_baseline": cpu, "e2e": None, "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def micro_cpu_rate(budget_s):
    """Oracle per-pair pipeline (contact_blocks: distance, barrier, J^T H J, 24x24 PSD), pairs/s, 1 thread,
    on a sample drawn by the same generator (2,000 bodies, equal VF / EE counts)."""
    from types import SimpleNamespace

    from threadpoolctl import threadpool_limits

    from oracle import abd_oracle as O
    from paper_2201_10022_b200 import microbench, scenes
    lim = threadpool_limits(limits=1)
    n, el, seed = 0, 0.0, 1
    while el < budget_s:
        d = scenes.microbench_pairs(seed=seed, n_bodies=2000, n_vf=2000, n_ee=2000)
        a = microbench.soup_arrays(d)
        bodies = []
        for b in range(len(d["q"])):
            v0, v1 = a["v_off"][b], a["v_off"][b + 1]
            e0, e1 = a["e_off"][b], a["e_off"][b + 1]
            t0, t1 = a["t_off"][b], a["t_off"][b + 1]
            bodies.append(SimpleNamespace(rest=a["rest"][v0:v1], edges=a["edges"][e0:e1], triangles=a["tris"][t0:t1],
                                          edge_rest_len_sq=a["el2"][e0:e1], dynamic=True))
        ts = time.perf_counter()
        O.contact_blocks(bodies, d["q"], a["vf"], a["ee"], 1e4, d["d_hat"])
        el += time.perf_counter() - ts
        n += len(a["vf"]) + len(a["ee"])
        seed += 1
    lim.restore_original_limits()
    return {"value": n / el, "unit": "pairs/s", "cores": 1, "kind": "port",
            "sample": f"oracle/abd_oracle.py contact_blocks (distance, barrier, J^T H J, PSD projection) on {n} "
                      f"pairs of the config-2 generator (2,000-body draws, half VF, half EE) in {el:.1f}s; the GPU "
                      "rate to compare is config.pairs_per_s_assemble"}


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--start", type=int, default=0, help="untimed steps before warm-up (no checkpoint)")
    ap.add_argument("--ckpt", default=os.path.join(ROOT, "bench_data", "pile_step150.npz"),
                    help="start state (q, q_dot, step) of the 20x20x25 pile; 'none' = step 0")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nx", type=int, default=20)
    ap.add_argument("--nz", type=int, default=25)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--workload", default="pile", choices=["pile", "micro", "chainmail", "cubes", "boxstack"],
                    help="pile = BASELINE config 4 (headline); micro = config 2 kernel microbenchmark; "
                         "chainmail = config 5; cubes = config 3 (1000-cube drop); boxstack = config 1")
    ap.add_argument("--micro-bodies", type=int, default=100_000)
    ap.add_argument("--micro-pairs", type=int, default=10_000_000, help="VF pairs = EE pairs")
    args = ap.parse_args()
    if args.workload == "micro":
        if args.impl == "reference" or int(os.environ.get("RANK", "0")) != 0:
            return
        run_micro(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_mod
        torch.cuda.set_device(local)
        dist_mod.init_process_group("nccl")
        dist = dist_mod

    import paper_2201_10022_b200 as P
    from paper_2201_10022_b200 import _native, scenes
    from paper_2201_10022_b200.solver import step_params_c

    if args.workload == "pile":
        spec = scenes.icosphere_pile(seed=0, nx=args.nx, ny=args.nx, nz=args.nz)
    elif args.workload == "chainmail":
        spec = scenes.chainmail(seed=0)
    elif args.workload == "cubes":
        spec = scenes.cube_drop(seed=0)
    else:
        spec = scenes.box_stack(seed=0)
    model, state, params = spec.build()
    B = len(model.bodies)
    L = _native.lib()
    sc = model.gpu_scene()
    if world > 1:
        # one pile over all ranks: per-pair work split by overlap body pair, the system /
        # energies / CCD bound all-reduced over NCCL, the solve replicated (csrc/comm.cu)
        from paper_2201_10022_b200.dist import attach_nccl
        attach_nccl(model)
    step0, time0 = 0, 0.0
    use_ckpt = args.workload == "pile" and args.ckpt.lower() != "none" and (args.nx, args.nz) == (20, 25)
    if use_ckpt:
        ck = np.load(args.ckpt)
        assert int(ck["seed"]) == 0 and ck["q"].shape == state.q.shape
        state.q, state.q_dot = ck["q"].copy(), ck["q_dot"].copy()
        step0, time0 = int(ck["step"]), float(ck["time"])
        args.start = 0
    forces = np.ascontiguousarray(model.forces(step0, time0 + params.dt, state.q), dtype=np.float64)
    q = np.ascontiguousarray(state.q, dtype=np.float64)
    qd = np.ascontiguousarray(state.q_dot, dtype=np.float64)
    _native.check(L.abd_set_state(sc.ptr, q.ctypes.data, qd.ctypes.data))
    cp = step_params_c(params)
    st = _native.StepStatsC()
    warnings.simplefilter("ignore")

    def step(first=False):
        _native.check(L.abd_advance_step(sc.ptr, forces.ctypes.data if first else None, C.byref(cp), C.byref(st),
                                         None))
        return st.iterations

    step(first=True)
    for _ in range(args.start + args.warmup - 1):
        step()
    # snapshot the window's initial state for the e2e pass
    q_start = np.empty((B, 12))
    qd_start = np.empty((B, 12))
    _native.check(L.abd_get_state(sc.ptr, q_start.ctypes.data, qd_start.ctypes.data))

    def barrier():
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    _native.check(L.abd_kernel_stats_reset(sc.ptr))
    n_launch0 = _native.kernel_launches()
    barrier()
    iters = 0
    pcg_total = 0
    # small scenes (configs 1 and 3) fit in L2: flush it (write 512 MB) before every
    # timed step and time the steps one by one so the flush stays outside the sum
    flush = args.workload in ("cubes", "boxstack")
    fbuf = None
    if flush:
        import torch
        fbuf = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    ms = C.c_double(0.0)
    with ClockSampler(local) as clk:
        if flush:
            tot = 0.0
            for _ in range(args.steps):
                fbuf.fill_(1.0)
                torch.cuda.synchronize()
                _native.check(L.abd_timer_start(sc.ptr))
                iters += step()
                pcg_total += st.pcg_iters_total
                _native.check(L.abd_timer_stop(sc.ptr, C.byref(ms)))
                tot += ms.value
            ms.value = tot
        else:
            _native.check(L.abd_timer_start(sc.ptr))
            for _ in range(args.steps):
                iters += step()
                pcg_total += st.pcg_iters_total
            _native.check(L.abd_timer_stop(sc.ptr, C.byref(ms)))
    barrier()
    launches = _native.kernel_launches() - n_launch0
    elapsed_ms = max_over_ranks(ms.value)
    iters_all = max_over_ranks(float(iters))
    value = args.steps / (elapsed_ms * 1e-3)  # one partitioned pile: whole-job steps/s
    # per-kernel live stats (CUDA events on the scene stream, this rank); the roofline
    # is reported for the instrumented kernel with the largest share of the timed region
    names = {0: ("k_chol", "k_chol_factor + k_chol_solve (K4 sparse block Cholesky, one factor + solve "
                           "per Newton iteration; PCG iterations when linear_solver='pcg')",
                 "A blocks read + L written (1152 B each), 2x1152 B per update pair, L read twice by the "
                 "solve, 4 vectors of 96 B per body"),
             1: ("k_pair_blocks", "k_pair_blocks (K3 contact pair gradient/Hessian, VF + EE launches)",
                 "SURVEY 8(d) K3: 112 P_vf + 120 P_ee + 96 B + 1152 N_blk + 96 B_d"),
             2: ("k_ccd", "k_ccd (K5 additive CCD, VF + EE launches)", "SURVEY 8(d) K5: 112 (P_vf + P_ee) + 192 B"),
             3: ("k_prim_pairs", "k_prim_pairs (K2 broad phase primitive pairs)",
                 "SURVEY 8(d) K2: 24 V + 8 E + 12 T + 192 B + 16 (P_vf + P_ee)")}
    kst = {}
    for which, (name, _, _) in names.items():
        n_, t_, b_, u_ = C.c_int64(), C.c_double(), C.c_double(), C.c_int64()
        _native.check(L.abd_kernel_stats(sc.ptr, which, C.byref(n_), C.byref(t_), C.byref(b_), C.byref(u_)))
        kst[name] = {"launches": n_.value, "ms": t_.value, "bytes": b_.value, "units": u_.value,
                     "share_of_step": t_.value / elapsed_ms if elapsed_ms else None,
                     "achieved_gbs": (b_.value / (t_.value * 1e-3) / 1e9) if t_.value else None}
    top = max(names, key=lambda k: kst[names[k][0]]["ms"])
    tname, tdesc, tmodel = names[top]
    pk, pk_kind = peaks()
    hbm = float(pk.get("hbm_gbs", HBM_FALLBACK))
    pc = kst[tname]
    achieved = (pc["bytes"] / pc["launches"]) / (pc["ms"] / pc["launches"] * 1e-3) / 1e9 if pc["launches"] else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "dram_bytes_per_launch.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(tname)
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "kernel": tdesc, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm if hbm else None, "traffic": traffic,
                "algorithmic_bytes_per_launch": pc["bytes"] / pc["launches"] if pc["launches"] else None,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})", "bytes_model": tmodel,
                "share_of_step": pc["share_of_step"], "kernels": kst}

    # e2e through the public Python API with host numpy state
    e2e = None
    if not args.no_e2e:
        w0 = step0 + args.start + args.warmup
        state2 = P.SimState(q=q_start.copy(), q_dot=qd_start.copy(), time=w0 * params.dt, step_index=w0)
        barrier()
        _native.check(L.abd_timer_start(sc.ptr))
        for _ in range(args.steps):
            state2, _st = P.advance_step(model, state2, params)
        ms2 = C.c_double(0.0)
        _native.check(L.abd_timer_stop(sc.ptr, C.byref(ms2)))
        barrier()
        e_ms = max_over_ranks(ms2.value)
        e2e = {"value": args.steps / (e_ms * 1e-3), "unit": "steps/s",
               "h2d_bytes_per_step": 3 * 96 * B, "d2h_bytes_per_step": 2 * 96 * B,
               "path": "paper_2201_10022_b200.advance_step (Python API, host numpy q/q_dot/forces)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and args.workload == "pile":
        r = oracle_sample_rate({}, args.warmup, args.cpu_budget, "1 thread", threads=1)
        cpu = {"value": r["value"], "unit": "steps/s", "cores": 1, "kind": "port",
               "sample": f"oracle/abd_oracle.py advance_step on a 8x8x2 sub-pile ({r['bodies']} icospheres + "
                         f"ground, same generator) from step {args.warmup}: {r['steps']} steps in "
                         f"{r['seconds']:.1f}s ({r['rate_sample']:.3f} steps/s), x{r['scale']:.4f} linear body "
                         "scaling to the 10k pile (optimistic for the CPU)"}

    if rank == 0:
        metric = {"pile": "sim steps/s (10k-body icosphere pile, fp64 ABD)",
                  "chainmail": "sim steps/s (10k-link chainmail, fp64 ABD)",
                  "cubes": "sim steps/s (1000-cube drop, fp64 ABD)",
                  "boxstack": "sim steps/s (4-cube box stack, fp64 ABD)"}[args.workload]
        wl = (f"icosphere_pile {args.nx}x{args.nx}x{args.nz} ({B} bodies, seed 0)" if args.workload == "pile"
              else f"{spec.name} ({B} bodies, seed 0; BASELINE config "
                   f"{ {'chainmail': 5, 'cubes': 3, 'boxstack': 1}[args.workload]})")
        line = {
            "metric": metric, "value": value, "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded procedural scene)",
            "config": {"workload": f"{wl}, "
                                   f"steps [{step0 + args.start + args.warmup}, {step0 + args.start + args.warmup + args.steps})"
                                   + (f" from checkpoint {os.path.relpath(args.ckpt, ROOT)} (step {step0} of the "
                                      "200-step run; late, contact-dense phase)" if use_ckpt else ""),
                       "newton_iters": int(iters_all), "newton_it_per_s": iters_all / (elapsed_ms * 1e-3),
                       "pcg_iters": pcg_total,
                       "l2": ("L2 flushed (512 MB write) before every timed step; steps timed one by one"
                              if flush else "per-step working set exceeds L2 (rest+topology+vertex boxes "
                              "> 126 MB); no flush"),
                       "parallelism": (f"pair-partitioned over {world} GPUs (NCCL all-reduce of the system, "
                                       "replicated solve)") if world > 1 else "single"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
