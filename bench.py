#!/usr/bin/env python
"""Benchmark: fp64 ABD Newton steps on the 10k-body pile (BASELINE config 4).

    python bench.py [--gpus N --steps K --warmup W]
    python bench.py --impl reference ...        (the reference path on the host CPU)
    python bench.py --workload {micro,chainmail,cubes,boxstack} ...

A "step" is one implicit time step (`advance_step`: broad phase, friction
precompute, Newton loop with assembly / Cholesky / CCD / line search, stats).

Pile (headline).  The late, contact-dense window [150, 200) of the 200-step run
is stepped in full from the committed checkpoint `bench_data/pile_step150.npz`
(the GPU state after 150 steps; SimState is the complete inter-step state), each
step timed with CUDA events on the scene stream.  `value` = K / (sum of the K
step times), the K steps spread evenly over the 50-step window; `config` also
reports the whole window and the full 200-step run from step 0 (also timed step
by step).  `e2e` repeats the window through the public Python API with host
numpy state (H2D q, q_dot, forces and D2H q, q_dot inside every timed step).
`--gpus N` (N > 1) starts N ranks under torch.distributed.run when WORLD_SIZE is
unset; the ranks cut ONE pile into body slabs (strong scaling, max-over-ranks device
time; csrc/comm.cu, k_chol.cu slab_pcg).
Prints one JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import ctypes as C
import glob
import hashlib
import json
import os
import socket
import subprocess
import sys
import time
import warnings

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0
WINDOW = (150, 200)  # late window of the 200-step config-4 run
CKPT = os.path.join(ROOT, "bench_data", "pile_step150.npz")
METRICS = {"pile": "sim steps/s (10k-body icosphere pile, fp64 ABD)",
           "chainmail": "sim steps/s (10k-link chainmail, fp64 ABD)",
           "cubes": "sim steps/s (1000-cube drop, fp64 ABD)",
           "boxstack": "sim steps/s (4-cube box stack, fp64 ABD)"}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": HBM_FALLBACK}, "fallback"


def src_hash():
    """Digest of the CUDA sources the library is built from (keys measured ncu traffic)."""
    h = hashlib.sha256()
    files = sorted(glob.glob(os.path.join(ROOT, "paper_2201_10022_b200", "csrc", "*")))
    for p in files + [os.path.join(ROOT, "include", "abd_b200.h")]:
        with open(p, "rb") as f:
            h.update(os.path.basename(p).encode() + f.read())
    return h.hexdigest()[:16]


def measured_capture(workload):
    """ncu capture of this workload's kernels on THIS source tree (tools/measure_traffic.py
    writes profiles/traffic_<workload>.json with the src hash), or (None, why)."""
    path = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    try:
        d = json.load(open(path))
    except Exception:
        return None, "no capture"
    if d.get("src_hash") != src_hash():
        return None, f"capture {os.path.relpath(path, ROOT)} is for another source tree"
    return d, os.path.relpath(path, ROOT)


def measured_traffic(workload, kernel):
    """ncu DRAM bytes per launch of `kernel` on `workload`, if captured on this source tree."""
    d, src = measured_capture(workload)
    if d is None:
        return None, src
    k = d.get("kernels", {}).get(kernel)
    return (k.get("dram_bytes_per_launch") if k else None), src


def fp64_table(workload, kst):
    """Executed FP64 flops per launch (ncu: 2 DFMA + DADD + DMUL + 512 per DMMA m8n8k4) over the
    live per-launch time (bench CUDA events) for the instrumented kernels, over the ncu
    duration otherwise, against the DFMA peak measured by tools/ubench/dfma.cu."""
    d, src = measured_capture(workload)
    if d is None:
        return {"source": src}
    try:
        peak = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
    except Exception:
        peak = None
    out = {"source": src, "peak_tflops": (peak or {}).get("dfma_tflops"),
           "peak_source": "profiles/fp64_peak.json (tools/ubench/dfma.cu DFMA probe)" if peak else None}
    for g, k in d.get("kernels", {}).items():
        f = k.get("fp64") or {}
        flops = f.get("flops_per_launch")
        live = kst.get(g)
        ms = live["ms"] / live["launches"] if live and live.get("launches") else f.get("ms_per_launch")
        tf = flops / (ms * 1e-3) / 1e12 if (flops is not None and ms) else None
        out[g] = {"flops_per_launch": flops, "ms_per_launch": ms, "achieved_tflops": tf,
                  "frac": tf / out["peak_tflops"] if (tf is not None and out["peak_tflops"]) else None,
                  "time": "live" if live else "ncu (cold)"}
    return out


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


def spread(n, k):
    """k indices spread evenly over range(n) (all of them when k >= n)."""
    if k >= n:
        return list(range(n))
    return sorted({int((i + 0.5) * n / k) for i in range(k)})


# ---------------------------------------------------------------------------
# CPU legs: the oracle restatement of the reference path on the actual 10k pile
def _oracle_pile():
    from types import SimpleNamespace

    from oracle import abd_oracle as O
    from paper_2201_10022_b200 import scenes
    from paper_2201_10022_b200.body import mass_matrix

    spec = scenes.icosphere_pile(seed=0)
    bodies, masses, stiff = [], [], []
    for m, dyn in zip(spec.meshes, spec.dynamic):
        d = m.vertices[m.edges[:, 1]] - m.vertices[m.edges[:, 0]]
        bodies.append(SimpleNamespace(rest=m.vertices, triangles=m.triangles, edges=m.edges,
                                      edge_rest_len_sq=np.einsum("ij,ij->i", d, d), dynamic=bool(dyn)))
        if dyn:
            gm, vol = mass_matrix(m, spec.density)
            masses.append(gm.matrix)
            stiff.append(spec.kappa_ortho * vol)
        else:
            masses.append(None)
            stiff.append(None)
    model = O.OracleModel(bodies, masses, stiff)
    f = np.zeros((len(bodies), 12))
    g = np.asarray(spec.gravity, dtype=float)
    for b in model.dyn:
        f[b, :3] = masses[b][0, 0] * g
        f[b, 3:] = np.kron(g, masses[b][0, 3:6])
    return O, model, O.OracleParams(**spec.params), f


class OraclePileNewton:
    """The reference's Newton step (solver.py:493-628) restated by oracle/abd_oracle.py,
    run on the 10k pile from the step-150 checkpoint one Newton iteration at a time:
    setup = q_tilde + broad_phase(q, q) + friction_precompute; iteration = assemble +
    sparse direct solve (BlockCholesky's contract, solve_refined) + broad_phase(q, q + dq)
    + CCD-capped line search."""

    def __init__(self, workers):
        from threadpoolctl import threadpool_limits

        self.limiter = threadpool_limits(limits=workers)
        self.workers = workers
        self.O, self.model, self.prm, self.f = _oracle_pile()
        ck = np.load(CKPT)
        self.q0, self.qd = ck["q"].copy(), ck["q_dot"].copy()
        self.q = self.q0.copy()
        self.ip = None

    def setup(self):
        O, m, p = self.O, self.model, self.prm
        t0 = time.perf_counter()
        qt = O.q_tilde(m, self.q0, self.qd, self.f, p.dt)
        c = O.broad_phase(m.bodies, self.q0, self.q0, p.d_hat, workers=self.workers)
        fr = O.friction_precompute(m.bodies, self.q0, c.vf, c.ee, p.kappa_barrier, p.d_hat, p.mu)
        self.ip = O.OracleIP(qt, fr, c)
        self.q = self.q0.copy()
        return time.perf_counter() - t0

    def iteration(self):
        O, m, p = self.O, self.model, self.prm
        t0 = time.perf_counter()
        g, D, off = O.assemble(m, self.q, self.ip, p)
        dd = O.solve_sparse(D, off, g)
        if float(g @ dd) >= 0.0:
            dd = -g
        dq = np.zeros_like(self.q)
        dq[m.dyn] = dd.reshape(-1, 12)
        self.ip.cands = O.broad_phase(m.bodies, self.q, self.q + dq, p.d_hat, workers=self.workers)
        alpha, _, _ = O.line_search(m, self.q, dq, self.ip, p)
        self.q = self.q + alpha * dq
        return time.perf_counter() - t0

    def close(self):
        self.limiter.restore_original_limits()


def late_iters_per_step():
    """Newton iterations per late-window step: the reference's own count on its step from the
    checkpoint (tests/golden/pile_step150.npz, stage B) when present, else the cap (64)."""
    try:
        g = np.load(os.path.join(ROOT, "tests", "golden", "pile_step150.npz"))
        if "B_iterations" in g.files:
            return int(g["B_iterations"]), "reference advance_step from the step-150 checkpoint"
    except Exception:
        pass
    return 64, "max_newton_iters (every GPU step of the window hits it)"


def cpu_baseline_pile(n_iter=1):
    """Rank 0, N = 1: the oracle on ONE thread, setup + n_iter Newton iterations of the
    10k pile from the step-150 checkpoint (~20-30 s)."""
    r = OraclePileNewton(workers=1)
    try:
        t_setup = r.setup()
        t_it = [r.iteration() for _ in range(n_iter)]
    finally:
        r.close()
    its, src = late_iters_per_step()
    it_s = float(np.mean(t_it))
    step_s = t_setup + its * it_s
    return {"value": 1.0 / step_s, "unit": "steps/s", "cores": 1, "kind": "port",
            "newton_it_per_s": 1.0 / it_s,
            "sample": (f"oracle/abd_oracle.py on the 10k pile (config 4) at the step-150 checkpoint, 1 thread: "
                       f"step setup (q_tilde, broad phase, friction) {t_setup:.2f}s + {n_iter} Newton iteration(s) "
                       f"(assemble, sparse direct solve, broad phase, CCD line search) {it_s:.2f}s each; "
                       f"steps/s = 1 / (setup + {its} x iteration), {its} = {src}")}


def run_reference(args):
    """--impl reference: the reference path (oracle restatement; /root/reference is absent
    on the GPU box) on the host CPU with every host thread, on the headline pile."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    warnings.simplefilter("ignore")
    r = OraclePileNewton(workers=cores)
    try:
        t_setup = r.setup()
        for _ in range(max(0, args.warmup - 1)):
            r.iteration()
        t_it = [r.iteration() for _ in range(args.steps)]
    finally:
        r.close()
    its, src = late_iters_per_step()
    it_s = float(np.mean(t_it))
    value = 1.0 / (t_setup + its * it_s)
    sample = (f"oracle/abd_oracle.py on the 10k pile at the step-150 checkpoint with {cores} host threads "
              f"(broad phase over {cores} forked workers, BLAS threads {cores}): step setup {t_setup:.2f}s, "
              f"then {args.warmup - 1} warm-up + {args.steps} timed Newton iterations ({it_s:.2f}s mean; "
              f"assemble, sparse direct solve, broad phase, CCD line search); steps/s = 1 / (setup + {its} x "
              f"iteration), {its} = {src}")
    line = {
        "impl": "reference", "metric": METRICS["pile"], "value": value, "unit": "steps/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 / value, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded procedural scene)",
        "config": {"workload": "icosphere_pile 20x20x25 (10001 bodies, seed 0), late window from checkpoint "
                               "bench_data/pile_step150.npz", "newton_it_per_s": 1.0 / it_s,
                   "iteration_s": t_it, "setup_s": t_setup, "parallelism": f"cpu ({cores} host threads)"},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t0,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def run_micro(args):
    """--workload micro: BASELINE config 2 (SURVEY §8(d) kernel microbenchmark).

    One step = `assemble` (K1 + K3 + BSR reduction) over 10M VF + 10M EE synthetic
    pairs on 100k bodies with d ~ U(0, d_hat) (the stated config), then the block-Jacobi
    PCG to 1e-8 relative residual.  The PCG leg runs on a second instance drawn with
    d ~ U(0.1 d_hat, d_hat) (--micro-pcg-dlo): on the stated distribution no fp64
    block-Jacobi PCG reaches 1e-8 (Hessian blocks ~1e15 x the mass block).
    """
    from paper_2201_10022_b200 import _native, microbench, scenes

    t0 = time.perf_counter()

    def system(dlo):
        return microbench.PairSystem(scenes.microbench_pairs(seed=0, n_bodies=args.micro_bodies,
                                                             n_vf=args.micro_pairs, n_ee=args.micro_pairs,
                                                             d_lo_frac=dlo))

    sysm = system(args.micro_dlo)
    sysp = None
    if not args.micro_no_solve:
        sysp = sysm if args.micro_pcg_dlo == args.micro_dlo else system(args.micro_pcg_dlo)
    setup_s = time.perf_counter() - t0
    L = _native.lib()
    sc = sysm.scene
    for _ in range(args.warmup):
        sysm.assemble()
        if sysp is not None:
            if sysp is not sysm:
                sysp.assemble()
            sysp.solve()
    if sysp is not None and sysp is not sysm:
        _native.check(L.abd_kernel_stats_reset(sysp.scene.ptr))
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
            if sysp is None:
                continue
            if sysp is not sysm:
                sysp.assemble()  # its own system (untimed: the assembly leg is timed on the stated config)
            _native.check(L.abd_timer_start(sysp.scene.ptr))
            _, it, rel = sysp.solve()
            _native.check(L.abd_timer_stop(sysp.scene.ptr, C.byref(ms)))
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
        src = sysp.scene if (which == 0 and sysp is not None) else sc
        _native.check(L.abd_kernel_stats(src.ptr, which, C.byref(n_), C.byref(t_), C.byref(b_), C.byref(u_)))
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
        cpu = micro_cpu_rate(args.cpu_budget, args.micro_dlo)
    traffic, tsrc = measured_traffic("micro", "k_cg" if sol_ms else "k_pair_blocks")
    line = {
        "metric": "microbench assemble + PCG time (100k bodies, 10M VF + 10M EE pairs, fp64)",
        "value": tot_ms / args.steps, "unit": "ms", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_ms / args.steps, "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, scenes.microbench_pairs)",
        "config": {"workload": f"BASELINE config 2: {B} bodies, {sysm.n_vf} VF + {sysm.n_ee} EE pairs, "
                               f"d ~ U({args.micro_dlo} d_hat, d_hat) for the assembly, PCG on an instance with "
                               f"d ~ U({args.micro_pcg_dlo} d_hat, d_hat), Morton +-1..4 body graph "
                               f"({sysm.n_off} off-diagonal blocks), all pairs active",
                   "assemble_ms": float(np.mean(asm_ms)), "pcg_ms": float(np.mean(sol_ms)) if sol_ms else None,
                   "pcg_iters": iters, "pcg_rel_res": rels, "pcg_ms_per_iter": it_ms if sol_ms else None,
                   "pairs_per_s_assemble": P_all / (k3_ms * 1e-3), "setup_s": setup_s,
                   "l2": "inputs (~2 GB rest + 22 GB pair records) exceed L2; no flush"},
        "roofline": {"bound": "hbm", "kernel": "K4 PCG iteration (k_cg) / K3 assemble",
                     "achieved": it_bytes / (it_ms * 1e-3) / 1e9 if sol_ms else None, "peak": hbm, "unit": "GB/s",
                     "frac": it_bytes / (it_ms * 1e-3) / 1e9 / hbm if sol_ms else None, "traffic": traffic,
                     "traffic_source": tsrc, "algorithmic_bytes_per_launch": it_bytes,
                     "bytes_model": "K4: 1152 (N_blk + B_d) + 13 x 96 B_d per PCG iteration",
                     "assemble": {"achieved": k3_bytes / (k3_ms * 1e-3) / 1e9, "bytes": k3_bytes,
                                  "frac": k3_bytes / (k3_ms * 1e-3) / 1e9 / hbm,
                                  "bytes_model": "K3 pre-gathered: 104 P_vf + 112 P_ee + 1152 N_blk + 192 B"},
                     "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})", "kernels": kst},
        "cpu_baseline": cpu, "e2e": None, "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def micro_cpu_rate(budget_s, d_lo):
    """Oracle per-pair pipeline (contact_blocks: distance, barrier, J^T H J, 24x24 PSD), pairs/s, 1 thread,
    on a sample drawn by the same generator (2,000 bodies, equal VF / EE counts)."""
    from types import SimpleNamespace

    from threadpoolctl import threadpool_limits

    from oracle import abd_oracle as O
    from paper_2201_10022_b200 import microbench, scenes
    lim = threadpool_limits(limits=1)
    n, el, seed = 0, 0.0, 1
    while el < budget_s:
        d = scenes.microbench_pairs(seed=seed, n_bodies=2000, n_vf=2000, n_ee=2000, d_lo_frac=d_lo)
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
def maybe_spawn(args):
    """`--gpus N` with N > 1 and no launcher: re-exec under torch.distributed.run (one rank per
    GPU).  Under a launcher, WORLD_SIZE must equal --gpus."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is None:
        if args.gpus > 1:
            with socket.socket() as s:
                s.bind(("127.0.0.1", 0))
                port = s.getsockname()[1]
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
            os.execv(sys.executable, cmd)
        return
    if int(ws) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; launch with matching values")


class Run:
    """One scene on this rank's GPU, stepped through the device-resident C-ABI path
    (`abd_advance_step`) or the Python API, every step timed on the scene stream."""

    def __init__(self, args, dist):
        import paper_2201_10022_b200 as P
        from paper_2201_10022_b200 import _native, scenes
        from paper_2201_10022_b200.solver import step_params_c

        self.P, self.N, self.dist = P, _native, dist
        wl = args.workload
        self.spec = {"pile": lambda: scenes.icosphere_pile(seed=0, nx=args.nx, ny=args.nx, nz=args.nz),
                     "chainmail": lambda: scenes.chainmail(seed=0), "cubes": lambda: scenes.cube_drop(seed=0),
                     "boxstack": lambda: scenes.box_stack(seed=0)}[wl]()
        self.model, self.state0, self.params = self.spec.build()
        self.B = len(self.model.bodies)
        self.L = _native.lib()
        self.sc = self.model.gpu_scene()
        if dist is not None:
            # one pile over all ranks (csrc/comm.cu)
            from paper_2201_10022_b200.dist import attach_nccl
            attach_nccl(self.model)
        self.cp = step_params_c(self.params)
        self.st = _native.StepStatsC()
        self.forces = np.ascontiguousarray(self.model.forces(0, self.params.dt, self.state0.q), dtype=np.float64)
        self.first = True
        # small scenes (configs 1 and 3) fit in L2: flush it (write 512 MB) before every timed step
        self.flush = wl in ("cubes", "boxstack")
        self.fbuf = None
        if self.flush:
            import torch
            self.fbuf = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")

    def set_state(self, q, qd):
        q = np.ascontiguousarray(q, dtype=np.float64)
        qd = np.ascontiguousarray(qd, dtype=np.float64)
        self.N.check(self.L.abd_set_state(self.sc.ptr, q.ctypes.data, qd.ctypes.data))

    def get_state(self):
        q, qd = np.empty((self.B, 12)), np.empty((self.B, 12))
        self.N.check(self.L.abd_get_state(self.sc.ptr, q.ctypes.data, qd.ctypes.data))
        return q, qd

    def _flush(self):
        if self.flush:
            import torch
            self.fbuf.fill_(1.0)
            torch.cuda.synchronize()

    def device_steps(self, n):
        """n steps on the resident state; per-step (ms, Newton iterations)."""
        ms = C.c_double(0.0)
        out = []
        for _ in range(n):
            self._flush()
            self.N.check(self.L.abd_timer_start(self.sc.ptr))
            self.N.check(self.L.abd_advance_step(self.sc.ptr, self.forces.ctypes.data if self.first else None,
                                                 C.byref(self.cp), C.byref(self.st), None))
            self.N.check(self.L.abd_timer_stop(self.sc.ptr, C.byref(ms)))
            self.first = False
            out.append((ms.value, self.st.iterations))
        return out

    def api_steps(self, state, n):
        """n steps through the public Python API (host numpy state, copies in every step)."""
        ms = C.c_double(0.0)
        out = []
        for _ in range(n):
            self._flush()
            self.N.check(self.L.abd_timer_start(self.sc.ptr))
            state, st = self.P.advance_step(self.model, state, self.params)
            self.N.check(self.L.abd_timer_stop(self.sc.ptr, C.byref(ms)))
            out.append((ms.value, st.iterations))
        self.first = True  # advance_step uploaded its own forces
        return state, out

    def max_over_ranks(self, xs):
        if self.dist is None:
            return np.asarray(xs, dtype=float)
        import torch
        t = torch.tensor(np.asarray(xs, dtype=float), dtype=torch.float64, device="cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.cpu().numpy()

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def kernel_stats(self):
        names = {0: ("k_chol", "k_chol_factor + k_chol_solve (K4 sparse block Cholesky, one factor + solve "
                               "per Newton iteration)",
                     "A blocks read + L written (1152 B each), 2x1152 B per update pair, L read twice by the "
                     "solve, 4 vectors of 96 B per body"),
                 1: ("k_pair_blocks", "k_pair_blocks (K3 contact pair gradient/Hessian, VF + EE launches)",
                     "SURVEY 8(d) K3: 112 P_vf + 120 P_ee + 96 B + 1152 N_blk + 96 B_d"),
                 2: ("k_ccd", "k_ccd (K5 additive CCD, VF + EE launches)", "SURVEY 8(d) K5: 112 (P_vf + P_ee) + 192 B"),
                 3: ("k_prim_pairs", "k_prim_pairs (K2 broad phase primitive pairs)",
                     "SURVEY 8(d) K2: 24 V + 8 E + 12 T + 192 B + 16 (P_vf + P_ee)")}
        kst = {}
        for which, (name, desc, model) in names.items():
            n_, t_, b_, u_ = C.c_int64(), C.c_double(), C.c_double(), C.c_int64()
            self.N.check(self.L.abd_kernel_stats(self.sc.ptr, which, C.byref(n_), C.byref(t_), C.byref(b_),
                                                 C.byref(u_)))
            kst[name] = {"launches": n_.value, "ms": t_.value, "bytes": b_.value, "units": u_.value,
                         "desc": desc, "bytes_model": model}
        return kst


def rate(ms_list, iters=None):
    tot = float(np.sum(ms_list))
    d = {"steps": len(ms_list), "ms": tot, "steps_per_s": len(ms_list) / (tot * 1e-3) if tot else None}
    if iters is not None:
        d["newton_iters"] = int(np.sum(iters))
        d["newton_it_per_s"] = float(np.sum(iters)) / (tot * 1e-3) if tot else None
    return d


def run_scene(args):
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
    warnings.simplefilter("ignore")
    r = Run(args, dist)
    pile = args.workload == "pile" and (args.nx, args.nz) == (20, 25) and args.ckpt.lower() != "none"

    if pile:
        ck = np.load(args.ckpt)
        assert int(ck["seed"]) == 0 and ck["q"].shape == (r.B, 12)
        q_ck, qd_ck, step0 = ck["q"].copy(), ck["q_dot"].copy(), int(ck["step"])
        n_win = min(WINDOW[1] - step0, args.window_steps)
        r.forces = np.ascontiguousarray(r.model.forces(step0, (step0 + 1) * r.params.dt, q_ck), dtype=np.float64)
        # warm-up from the checkpoint, then back to it
        r.set_state(q_ck, qd_ck)
        r.device_steps(args.warmup)
        r.set_state(q_ck, qd_ck)
        q_start, qd_start = q_ck, qd_ck
    else:
        r.set_state(r.state0.q, r.state0.q_dot)
        r.device_steps(args.start + args.warmup)
        q_start, qd_start = r.get_state()
        step0 = args.start + args.warmup
        n_win = args.steps
    timed = spread(n_win, args.steps)

    # device-resident pass over the window; the K timed steps are spread over it
    r.N.check(r.L.abd_kernel_stats_reset(r.sc.ptr))
    n_launch0 = r.N.kernel_launches()
    r.barrier()
    with ClockSampler(local) as clk:
        per = r.device_steps(n_win)
    r.barrier()
    launches_window = r.N.kernel_launches() - n_launch0
    ms_all = r.max_over_ranks([p[0] for p in per])
    it_all = [p[1] for p in per]
    kst = r.kernel_stats()
    q_dev_end, _ = r.get_state()
    ms_t = ms_all[timed]
    it_t = [it_all[i] for i in timed]
    elapsed_ms = float(np.sum(ms_t))
    value = len(timed) / (elapsed_ms * 1e-3)
    launches = int(round(launches_window * len(timed) / max(1, n_win)))
    win_ms = float(np.sum(ms_all))

    # roofline: the instrumented kernel with the largest share of the window
    for k in kst.values():
        k["share_of_step"] = k["ms"] / win_ms if win_ms else None
        k["achieved_gbs"] = k["bytes"] / (k["ms"] * 1e-3) / 1e9 if k["ms"] else None
    top = max(kst, key=lambda k: kst[k]["ms"])
    pc = kst[top]
    pk, pk_kind = peaks()
    hbm = float(pk.get("hbm_gbs", HBM_FALLBACK))
    achieved = (pc["bytes"] / pc["launches"]) / (pc["ms"] / pc["launches"] * 1e-3) / 1e9 if pc["launches"] else 0.0
    traffic, tsrc = measured_traffic(args.workload, top)
    roofline = {"bound": "hbm", "kernel": pc["desc"], "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm if hbm else None, "traffic": traffic, "traffic_source": tsrc,
                "algorithmic_bytes_per_launch": pc["bytes"] / pc["launches"] if pc["launches"] else None,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({pk_kind})", "bytes_model": pc["bytes_model"],
                "share_of_step": pc["share_of_step"],
                "kernels": {k: {kk: vv for kk, vv in v.items() if kk not in ("desc", "bytes_model")}
                            for k, v in kst.items()},
                "measured_over": f"all {n_win} steps of the window",
                "fp64": fp64_table(args.workload, kst)}

    # e2e: the same window through the public Python API with host numpy state
    e2e = None
    if not args.no_e2e:
        state = r.P.SimState(q=q_start.copy(), q_dot=qd_start.copy(), time=step0 * r.params.dt, step_index=step0)
        r.barrier()
        state, per2 = r.api_steps(state, n_win)
        r.barrier()
        ms2 = r.max_over_ranks([p[0] for p in per2])
        e_ms = float(np.sum(ms2[timed]))
        e2e = {"value": len(timed) / (e_ms * 1e-3), "unit": "steps/s",
               "h2d_bytes_per_step": 3 * 96 * r.B, "d2h_bytes_per_step": 2 * 96 * r.B,
               "path": "paper_2201_10022_b200.advance_step (Python API, host numpy q/q_dot/forces)",
               "window": rate(ms2, [p[1] for p in per2]),
               "same_final_state_as_device_pass": bool(np.array_equal(state.q, q_dev_end))}

    # the full 200-step run from step 0 (pile), every step timed
    full = None
    if pile and not args.no_full_run:
        r.set_state(r.state0.q, r.state0.q_dot)
        r.forces = np.ascontiguousarray(r.model.forces(0, r.params.dt, r.state0.q), dtype=np.float64)
        r.first = True
        r.barrier()
        q150 = None
        perf = []
        for s in range(WINDOW[1]):
            perf += r.device_steps(1)
            if s + 1 == step0:
                q150, _ = r.get_state()
        r.barrier()
        msf = r.max_over_ranks([p[0] for p in perf])
        itf = [p[1] for p in perf]
        full = rate(msf, itf)
        full["early_0_50"] = rate(msf[:50], itf[:50])
        full["middle_50_150"] = rate(msf[50:150], itf[50:150])
        full["late_150_200"] = rate(msf[150:], itf[150:])
        full["checkpoint_rel_diff_at_step150"] = float(np.abs(q150 - q_ck).max() / np.abs(q_ck).max())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and pile:
        cpu = cpu_baseline_pile()

    if rank == 0:
        wl = (f"icosphere_pile {args.nx}x{args.nx}x{args.nz} ({r.B} bodies, seed 0)" if args.workload == "pile"
              else f"{r.spec.name} ({r.B} bodies, seed 0; BASELINE config "
                   f"{ {'chainmail': 5, 'cubes': 3, 'boxstack': 1}[args.workload]})")
        win = f"[{step0}, {step0 + n_win})"
        line = {
            "metric": METRICS[args.workload], "value": value, "unit": "steps/s",
            "n_gpus": world, "steps": len(timed), "warmup": args.warmup,
            "ms_per_step": elapsed_ms / len(timed), "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded procedural scene)",
            "config": {"workload": wl + (f", late window {win} of the 200-step run from checkpoint "
                                         f"{os.path.relpath(args.ckpt, ROOT)}" if pile else f", steps {win}"),
                       "timed_steps": [step0 + i for i in timed],
                       "newton_iters": int(np.sum(it_t)), "newton_it_per_s": float(np.sum(it_t)) / (elapsed_ms * 1e-3),
                       "window": rate(ms_all, it_all), "full_run": full,
                       "l2": ("L2 flushed (512 MB write) before every timed step" if r.flush else
                              "per-step working set exceeds L2 (rest+topology+vertex boxes > 126 MB); no flush"),
                       "parallelism": (f"body slabs over {world} GPUs: slab-owned pairs, NCCL all-reduce of the "
                                       "partial system, distributed PCG with slab-local Cholesky preconditioner")
                       if world > 1 else "single"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "gpu_launches_window": int(launches_window), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--start", type=int, default=0, help="untimed steps before warm-up (non-pile workloads)")
    ap.add_argument("--ckpt", default=CKPT, help="pile start state (q, q_dot, step); 'none' = from step 0")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nx", type=int, default=20)
    ap.add_argument("--nz", type=int, default=25)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-full-run", action="store_true")
    ap.add_argument("--window-steps", type=int, default=WINDOW[1] - WINDOW[0],
                    help="pile: steps of the late window stepped (default all 50); for experiments only")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--workload", default="pile", choices=["pile", "micro", "chainmail", "cubes", "boxstack"],
                    help="pile = BASELINE config 4 (headline); micro = config 2 kernel microbenchmark; "
                         "chainmail = config 5; cubes = config 3 (1000-cube drop); boxstack = config 1")
    ap.add_argument("--micro-bodies", type=int, default=100_000)
    ap.add_argument("--micro-pairs", type=int, default=10_000_000, help="VF pairs = EE pairs")
    ap.add_argument("--micro-dlo", type=float, default=0.0, help="assembly instance: d ~ U(dlo * d_hat, d_hat)")
    ap.add_argument("--micro-pcg-dlo", type=float, default=0.1, help="PCG instance: d ~ U(dlo * d_hat, d_hat)")
    ap.add_argument("--micro-no-solve", action="store_true")
    args = ap.parse_args()
    maybe_spawn(args)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.workload == "micro":
        if int(os.environ.get("RANK", "0")) == 0:
            run_micro(args)
        return
    run_scene(args)


if __name__ == "__main__":
    main()
