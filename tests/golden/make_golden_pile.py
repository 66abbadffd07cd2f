"""Step-local golden fixtures of the HEADLINE config (10k-body pile) from the REFERENCE.

Run in the build container (where /root/reference exists), in the background:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_pile.py [ckpt ...]

For each checkpoint `bench_data/pile_step{N}.npz` (the GPU state after N steps of
`scenes.icosphere_pile(seed=0)`; SimState is the complete inter-step state) this
imports `stiffbody` from /root/reference/pkg/src and evaluates, on the SAME q:

  stage A (one Newton iteration, step-local; solver.py:507-548):
    broad_phase(q, q)            -> counts + SHA-256 of the sorted vf/ee/overlap rows
                                    (+ the rows themselves as int32, compressed)
    friction_precompute(q)       -> body pairs, lambda, tangent maps, offsets
    assemble(q)                  -> gradient, H @ r for a seeded r, BSR pattern,
                                    off-diagonal blocks, 512 sampled diagonal blocks
    solve_newton_system          -> delta q
    broad_phase(q, q + dq)       -> counts + SHA-256 (+ rows)
    step_filter, ip_value(q), line_search -> alpha_max, e0, (alpha, e)
  stage B (solver.py:493-628): one full `advance_step` from the checkpoint, with ONE
    substitution: `solve_newton_system` (solver.py:345-348) is replaced by a SuperLU
    factorisation of the same assembled BSR with the same refinement contract
    (sparse.py:148-161: refine until |Hx + g| <= 1e-8 |g|, <= 3 corrections, residual by
    the reference's own BlockSparseMatrix.matvec).  The reference's natural-order
    BlockCholesky costs ~610 s per solve on this pile (O(n^2) python loop over column
    pairs, sparse.py:95-126; measured in stage A, A_t_solve), i.e. ~11 h for a 64-iteration
    step; both solves satisfy the same residual bound, so they differ at rounding level --
    iterations, converged, energy_trace, per-iteration alpha and candidate counts
    (recorded by wrapping the module's own line_search / broad_phase), final q,
    q_dot, min_distance, candidates, ip_value, max_ortho_error.

Results go to tests/golden/pile_step{N}.npz (stage A is written first, then
rewritten with stage B when it finishes).  Nothing at test time reads
/root/reference.  numpy's BLAS config and the CPU model are stored beside the data.
"""
from __future__ import annotations

import hashlib
import io
import os
import platform
import sys
import time
import warnings
from contextlib import redirect_stdout

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import stiffbody.ccd as rccd  # noqa: E402
import stiffbody.contact as rc  # noqa: E402
import stiffbody.solver as rs  # noqa: E402

from make_golden import ref_model  # noqa: E402
from paper_2201_10022_b200 import scenes  # noqa: E402

R_SEED = 777  # seed of the probe vector r in H @ r


def rows_sha(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int64).reshape(-1, a.shape[-1] if a.ndim > 1 else 1))
    return hashlib.sha256(a.tobytes()).hexdigest()


def put_cands(out, p, c):
    for nm, arr in (("vf", c.vf), ("ee", c.ee), ("ov", c.overlap_pairs)):
        arr = np.asarray(arr, dtype=np.int64)
        out[f"{p}{nm}_n"] = np.array(len(arr))
        out[f"{p}{nm}_sha"] = np.array(rows_sha(arr))
        out[f"{p}{nm}"] = arr.astype(np.int32)


def env_info(out):
    buf = io.StringIO()
    with redirect_stdout(buf):
        np.show_config()
    out["numpy_config"] = np.array(buf.getvalue())
    cpu = platform.processor()
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    out["cpu_model"] = np.array(cpu)
    out["numpy_version"] = np.array(np.__version__)


def save(path, out):
    tmp = path + ".tmp.npz"
    np.savez_compressed(tmp, **out)
    os.replace(tmp, path)
    print(f"wrote {path}: {os.path.getsize(path) / 1e6:.2f} MB", flush=True)


def stage_a(model, state, params, out):
    t0 = time.perf_counter()
    q0 = state.q.copy()
    forces = model.forces(state.step_index, state.time + params.dt, q0)
    q_tilde = rs.compute_q_tilde(model, state, params, forces)
    out["A_qtilde"] = q_tilde
    tic = time.perf_counter()
    c0 = rc.broad_phase(model.bodies, q0, q0, params.d_hat)
    out["A_t_broad"] = np.array(time.perf_counter() - tic)
    put_cands(out, "A_c0_", c0)
    print(f"  c0: vf {len(c0.vf)} ee {len(c0.ee)} ov {len(c0.overlap_pairs)} "
          f"({time.perf_counter() - t0:.1f}s)", flush=True)
    fr = rc.friction_precompute(model.bodies, q0, c0, params.kappa_barrier, params.d_hat, params.mu)
    out["A_fr_a"], out["A_fr_b"], out["A_fr_lam"] = fr.body_a, fr.body_b, fr.lam
    out["A_fr_tmap"], out["A_fr_off"] = fr.tangent_map, fr.offset
    ip = rs.IncrementalPotentialState(q0, state.q_dot.copy(), q_tilde, fr, c0, model)
    tic = time.perf_counter()
    g, H = rs.assemble(q0, ip, params)
    out["A_t_assemble"] = np.array(time.perf_counter() - tic)
    out["A_grad"] = g
    r = np.random.default_rng(R_SEED).normal(size=g.shape)
    out["A_Hr"] = H.matvec(r)
    keys = sorted(H.off.keys())
    out["A_off_keys"] = np.array(keys, dtype=np.int64).reshape(-1, 2)
    out["A_off_blocks"] = (np.array([H.off[k] for k in keys]).reshape(-1, 12, 12) if keys
                           else np.zeros((0, 12, 12)))
    nd = H.diag.shape[0]
    sel = np.sort(np.random.default_rng(R_SEED + 1).choice(nd, size=min(512, nd), replace=False))
    out["A_diag_sel"] = sel
    out["A_diag_blocks"] = H.diag[sel]
    out["A_diag_fro"] = np.sqrt(np.einsum("nij,nij->n", H.diag, H.diag))
    print(f"  assemble: {len(keys)} off blocks ({time.perf_counter() - t0:.1f}s)", flush=True)
    tic = time.perf_counter()
    dx = rs.solve_newton_system(H, g)
    out["A_t_solve"] = np.array(time.perf_counter() - tic)
    out["A_dx"] = dx
    dq = rs._expand_delta(model, dx)
    out["A_newton_dq_inf_over_dt"] = np.array(np.abs(dx).max() / params.dt)
    out["A_g_dot_dx"] = np.array(float(g @ dx))
    tic = time.perf_counter()
    c1 = rc.broad_phase(model.bodies, q0, q0 + dq, params.d_hat)
    out["A_t_broad1"] = np.array(time.perf_counter() - tic)
    put_cands(out, "A_c1_", c1)
    print(f"  c1: vf {len(c1.vf)} ee {len(c1.ee)} ({time.perf_counter() - t0:.1f}s)", flush=True)
    tic = time.perf_counter()
    out["A_alpha_max"] = np.array(rccd.step_filter(model.bodies, q0, dq, c1, slack=params.ccd_slack))
    out["A_t_ccd"] = np.array(time.perf_counter() - tic)
    ip.candidates = c1
    out["A_e0"] = np.array(rs.ip_value(q0, ip, params))
    alpha, e = rs.line_search(q0, dq, ip, params)
    out["A_alpha"], out["A_e"] = np.array(alpha), np.array(e)
    out["A_seconds"] = np.array(time.perf_counter() - t0)
    print(f"  alpha_max {float(out['A_alpha_max']):.6g} alpha {alpha:.6g} e0 {float(out['A_e0']):.10g} "
          f"e {e:.10g} ({time.perf_counter() - t0:.1f}s)", flush=True)


def stage_scales(model, state, params, out):
    """Per-block magnitude of the summed terms (the comparator's denominator for sums
    with cancellation): for each dynamic slot, |M(q - q~)| + dt^2 |grad V_perp| + sum over
    contact / friction pairs of |their 12-block gradient|; the same with Frobenius
    norms for the diagonal and off-diagonal Hessian blocks (solver.py:283-342)."""
    import stiffbody.body as rb

    q0 = state.q
    ck = dict(out)
    c0 = rc.CandidateSet(ck["A_c0_vf"].astype(np.int64), ck["A_c0_ee"].astype(np.int64),
                         ck["A_c0_ov"].astype(np.int64))
    slot = model.slot_of
    nd = model.n_dyn
    gs, ds = np.zeros(nd), np.zeros(nd)
    qt = ck["A_qtilde"]
    for b in model.dyn_indices:
        s = slot[int(b)]
        M = model.gmass[b].matrix
        gs[s] += np.linalg.norm(M @ (q0[b] - qt[b])) + params.dt ** 2 * np.linalg.norm(
            rb.ortho_gradient(q0[b], model.materials[b]))
        ds[s] += np.linalg.norm(M) + params.dt ** 2 * np.linalg.norm(
            rb.ortho_hessian(q0[b], model.materials[b], project_psd=True))
    keys = [tuple(k) for k in ck["A_off_keys"]]
    kidx = {k: i for i, k in enumerate(keys)}
    os_ = np.zeros(len(keys))
    fr = rc.FrictionData(ck["A_fr_a"], ck["A_fr_b"], ck["A_fr_lam"], params.mu, ck["A_fr_tmap"], ck["A_fr_off"],
                         np.zeros((len(ck["A_fr_lam"]), 3, 2)))
    parts = [rc.contact_gradient_hessian(model.bodies, q0, c0, params.kappa_barrier, params.d_hat),
             rc.friction_gradient_hessian(q0, fr, params.dt, params.epsilon_v, model.dynamic)]
    for blk in parts:
        for k in range(len(blk.body_a)):
            a, b = int(blk.body_a[k]), int(blk.body_b[k])
            sa, sb = slot.get(a), slot.get(b)
            if sa is not None:
                gs[sa] += np.linalg.norm(blk.grad[k, :12])
                ds[sa] += np.linalg.norm(blk.hess[k, :12, :12])
            if sb is not None:
                gs[sb] += np.linalg.norm(blk.grad[k, 12:])
                ds[sb] += np.linalg.norm(blk.hess[k, 12:, 12:])
            if sa is not None and sb is not None:
                os_[kidx[(min(sa, sb), max(sa, sb))]] += np.linalg.norm(blk.hess[k, :12, 12:])
    out["A_grad_scale"], out["A_diag_scale"], out["A_off_scale"] = gs, ds, os_
    print(f"  scales: grad median {np.median(gs):.4g}, off median {np.median(os_) if len(os_) else 0:.4g}",
          flush=True)


def fast_solve(H, g):
    """solve_newton_system's contract (solver.py:345-348, sparse.py:148-161) by SuperLU."""
    import scipy.sparse as sp
    from scipy.sparse.linalg import splu

    n = H.diag.shape[0]
    keys = list(H.off.keys())
    r = np.concatenate([np.arange(n)] + [np.array([k[0] for k in keys]), np.array([k[1] for k in keys])])
    c = np.concatenate([np.arange(n)] + [np.array([k[1] for k in keys]), np.array([k[0] for k in keys])])
    b = np.concatenate([H.diag, np.array([H.off[k] for k in keys]).reshape(-1, 12, 12),
                        np.array([H.off[k].T for k in keys]).reshape(-1, 12, 12)])
    ii = (12 * r[:, None, None] + np.arange(12)[None, :, None]).repeat(12, axis=2)
    jj = (12 * c[:, None, None] + np.arange(12)[None, None, :]).repeat(12, axis=1)
    A = sp.csc_matrix((b.reshape(-1), (ii.reshape(-1), jj.reshape(-1))), shape=(12 * n, 12 * n))
    lu = splu(A)
    rhs = -np.asarray(g, dtype=float)
    x = lu.solve(rhs)
    norm = np.linalg.norm(rhs)
    if norm == 0.0:
        return x
    for _ in range(3):
        res = rhs - H.matvec(x)
        if np.linalg.norm(res) <= 1e-8 * norm:
            break
        x = x + lu.solve(res)
    return x


def stage_b(model, state, params, out):
    alphas, ncand = [], []
    orig_ls, orig_bp, orig_solve = rs.line_search, rs.broad_phase, rs.solve_newton_system

    def ls(*a, **k):
        res = orig_ls(*a, **k)
        alphas.append(res[0])
        print(f"    it {len(alphas)}: alpha {res[0]:.6g} e {res[1]:.12g}", flush=True)
        return res

    def bp(*a, **k):
        c = orig_bp(*a, **k)
        ncand.append((len(c.vf), len(c.ee)))
        return c

    rs.line_search, rs.broad_phase, rs.solve_newton_system = ls, bp, fast_solve
    t0 = time.perf_counter()
    try:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            new, st = rs.advance_step(model, state, params)
    finally:
        rs.line_search, rs.broad_phase, rs.solve_newton_system = orig_ls, orig_bp, orig_solve
    out["B_seconds"] = np.array(time.perf_counter() - t0)
    out["B_q"], out["B_q_dot"] = new.q, new.q_dot
    out["B_iterations"], out["B_converged"] = np.array(st.iterations), np.array(st.converged)
    out["B_energy_trace"] = np.array(st.energy_trace)
    out["B_alphas"] = np.array(alphas)
    out["B_ncand"] = np.array(ncand).reshape(-1, 2)
    out["B_min_distance"], out["B_candidates"] = np.array(st.min_distance), np.array(st.candidates)
    out["B_ip_value"], out["B_max_ortho_error"] = np.array(st.ip_value), np.array(st.max_ortho_error)
    out["B_timings"] = np.array([st.timings.get(k, 0.0) for k in
                                 ("broad_phase", "narrow_phase", "assembly", "solve", "ccd", "line_search",
                                  "total")])
    print(f"  advance_step: {st.iterations} iterations, converged {st.converged}, "
          f"min_distance {st.min_distance:.6g} ({out['B_seconds']:.0f}s)", flush=True)


def main(steps):
    spec = scenes.icosphere_pile(seed=0)
    t0 = time.perf_counter()
    model = ref_model(spec.meshes, spec.dynamic, spec.density, spec.kappa_ortho)
    params = rs.StepParams(**spec.params)
    print(f"reference model: {len(model.bodies)} bodies ({time.perf_counter() - t0:.1f}s)", flush=True)
    for n in steps:
        ck = np.load(os.path.join(ROOT, "bench_data", f"pile_step{n}.npz"))
        state = rs.SimState(q=ck["q"].copy(), q_dot=ck["q_dot"].copy(), time=float(ck["time"]),
                            step_index=int(ck["step"]))
        path = os.path.join(HERE, f"pile_step{n}.npz")
        if os.path.exists(path):  # resume: keep a finished stage A
            out = dict(np.load(path))
        else:
            out = dict(step=np.array(int(ck["step"])), r_seed=np.array(R_SEED))
            env_info(out)
        print(f"checkpoint step {n}", flush=True)
        if "A_seconds" not in out:
            stage_a(model, state, params, out)
            save(path, out)
        if "A_grad_scale" not in out:
            stage_scales(model, state, params, out)
            if "--scales-side" in flags:  # another process still owns `path` (stage B running)
                save(path.replace(".npz", "_scales.npz"),
                     {k: out[k] for k in ("A_grad_scale", "A_diag_scale", "A_off_scale")})
                continue
            save(path, out)
        if "B_seconds" not in out and "--no-b" not in flags:
            stage_b(model, state, params, out)
            save(path, out)


if __name__ == "__main__":
    flags = {a for a in sys.argv[1:] if a.startswith("--")}
    main([int(a) for a in sys.argv[1:] if not a.startswith("--")] or [150, 100])
