/*
 * abd_b200.h — C ABI of the B200-native ABD (arXiv 2201.10022) Newton step.
 *
 * Plain pointers and sizes only: all arrays are C-contiguous HOST buffers
 * (float64 unless noted, int64 indices), copied to / from HBM by the
 * library.  Every entry returns an abd_status; on failure abd_last_error()
 * holds a message (thread-local) and abd_last_error_index() an index where
 * one applies (FactorizationError.block).
 *
 * Each entry names the reference interface it replaces
 * (file:line under /root/reference/pkg/src/stiffbody/).  The reference has
 * no FFI of its own; its drop-in surface is the Python API re-exported by
 * __init__.py:1-130, which paper_2201_10022_b200/*.py binds through ctypes
 * (INTEGRATION.md shows the stub a maintainer of the reference would add).
 */
#ifndef ABD_B200_H
#define ABD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum abd_status {
  ABD_OK = 0,
  ABD_ERR_ARG = 1,               /* ValueError / shape errors                          */
  ABD_ERR_CUDA = 2,              /* RuntimeError (CUDA failure)                        */
  ABD_ERR_BARRIER_DOMAIN = 3,    /* BarrierDomainError  contact.py:53-58               */
  ABD_ERR_CCD_DOMAIN = 4,        /* ValueError          ccd.py:81-82                   */
  ABD_ERR_FACTORIZATION = 5,     /* FactorizationError  sparse.py:17-25 (index=block)  */
  ABD_ERR_STEP_FAILURE = 6,      /* StepFailure         solver.py:69-74                */
  ABD_ERR_NO_DEVICE = 7,         /* no CUDA device / wrong architecture                */
  ABD_ERR_NOT_CONVERGED = 8      /* PCG hit its iteration cap                          */
};

enum abd_pair_kind { ABD_VF = 0, ABD_EE = 1 };

const char* abd_last_error(void);
int64_t abd_last_error_index(void);
/* device ordinal 0: SM count and compute capability (10.0 expected) */
int abd_device_info(int* sm_count, int* cc_major, int* cc_minor);
/* number of the library's own kernels launched since load (evidence counter) */
int64_t abd_kernel_launches(void);

/* ---------------- stateless batch kernels ------------------------------- */

/* point_triangle_closest  distance.py:86-150.  z: (n,4,3) rows (p, t0, t1, t2). */
int abd_pt_closest_batch(int64_t n, const double* z, double* d2, int32_t* region, double* bary);
/* edge_edge_closest  distance.py:167-204.  z: (n,4,3) rows (a0, a1, b0, b1). */
int abd_ee_closest_batch(int64_t n, const double* z, double* d2, int32_t* region, double* s, double* t);
/* pair_distance_gradients  distance.py:291-339.  grad (n,12), hess (n,12,12), gamma (n,4). */
int abd_pair_distance_gradients(int kind, int64_t n, const double* z, double* d2, double* grad,
                                double* hess, int32_t* region, double* gamma);
/* ee_mollifier / ee_mollifier_grad_hess  distance.py:207-225, :342-401 (grad, hess may be NULL). */
int abd_ee_mollifier_batch(int64_t n, const double* z, const double* eps_x, double* val, double* grad,
                           double* hess);
/* barrier, barrier_d1, barrier_d2  contact.py:87-121 (ABD_ERR_BARRIER_DOMAIN on d_sq <= 0). */
int abd_barrier_batch(int64_t n, const double* d_sq, double d_hat, double* b0, double* b1, double* b2);
/* ortho_energy / ortho_gradient / ortho_hessian  body.py:229-278 (q: (n,12)). */
int abd_ortho_batch(int64_t n, const double* q, const double* stiffness, int project, double* energy,
                    double* grad, double* hess);
/* project_psd  body.py:281-296, k <= 24. */
int abd_project_psd_batch(int64_t n, int k, const double* H, double* out);
/* accd_toi_batch  ccd.py:59-104.  x, dx: (n,4,3). */
int abd_accd_batch(int kind, int64_t n, const double* x, const double* dx, double slack, double t_max,
                   int max_iters, double* t);
/* per-pair contact terms on explicit points (contact.py:486-538 + :646-675 for one pair each):
 * z, rest (n,4,3) world / rest points, eps_x (n) (EE), dyn (n,2) uint8 side flags.
 * g12 (n,12), h12 (n,12,12) point-space barrier derivatives; g24 (n,24), h24 (n,24,24). */
int abd_contact_pair_batch(int kind, int64_t n, const double* z, const double* rest, const double* eps_x,
                           double kappa, double d_hat, const uint8_t* dyn, int project, double* g12, double* h12,
                           double* g24, double* h24);
/* friction_energy / friction_gradient_hessian  contact.py:815-853.
 * pairs: body ids (n), lam (n), tangent_map (n,2,24), offset (n,2); q: (n_bodies,12);
 * dynamic: (n_bodies) uint8.  energy may be NULL; grad24 (n,24)/hess24 (n,24,24) may be NULL. */
int abd_friction_batch(int64_t n, const int64_t* body_a, const int64_t* body_b, const double* lam, double mu,
                       const double* tangent_map, const double* offset, int n_bodies, const double* q,
                       const uint8_t* dynamic, double dt, double eps_v, int project, double* energy,
                       double* grad24, double* hess24);

/* symmetric block-sparse matrix (sparse.py:28-87): n diagonal blocks of bdim x bdim
 * (bdim <= 12), n_off upper blocks with keys (i < j) (n_off,2).  */
/* BlockSparseMatrix.matvec  sparse.py:77-84 */
int abd_bsr_matvec(int n, int bdim, const double* diag, int64_t n_off, const int64_t* keys,
                   const double* off, const double* x, double* y);
/* block-Jacobi PCG to ||A x - rhs|| <= rel_tol ||rhs||; replaces BlockCholesky.solve_refined
 * sparse.py:149-161 / solve_newton_system solver.py:345-348.  ABD_ERR_FACTORIZATION (index =
 * block) when a diagonal block is not SPD. */
int abd_bsr_pcg(int n, int bdim, const double* diag, int64_t n_off, const int64_t* keys, const double* off,
                const double* rhs, double rel_tol, int max_iters, double* x, int* iters, double* rel_res);
/* x = A^-1 rhs by the device sparse block Cholesky (minimum-degree order, elimination-tree
 * levels) with up to max_refine refinement steps until |A x - rhs| <= rel_tol |rhs|:
 * BlockCholesky(A).solve_refined (sparse.py:90-161).  rel_tol = 0, max_refine = 0 is the plain
 * BlockCholesky.solve (sparse.py:131-147).  Non-SPD pivot: ABD_ERR_FACTORIZATION, index = block. */
int abd_bsr_cholesky(int n, int bdim, const double* diag, int64_t n_off, const int64_t* keys, const double* off,
                     const double* rhs, double rel_tol, int max_refine, double* x, int* solves, double* rel_res);

/* ---------------- scene context (device-resident geometry) -------------- */

typedef struct abd_scene abd_scene;

/* SystemModel / CollisionBody arrays (solver.py:101-128, contact.py:128-146).
 * v_off/e_off/t_off: (n_bodies+1) prefix offsets; rest (V,3); edges (E,2) and tris (T,3)
 * hold per-body LOCAL vertex indices; edge_len_sq (E); dynamic (n_bodies);
 * mass (n_bodies,12,12) (ignored for kinematic); stiffness (n_bodies) = kappa*volume. */
abd_scene* abd_scene_create(int n_bodies, const int64_t* v_off, const int64_t* e_off, const int64_t* t_off,
                            const double* rest, const int64_t* edges, const int64_t* tris,
                            const double* edge_len_sq, const uint8_t* dynamic, const double* mass,
                            const double* stiffness);
void abd_scene_destroy(abd_scene* s);

/* broad_phase  contact.py:338-412 -> resident candidate set; counts out. */
int abd_broad_phase(abd_scene* s, const double* q0, const double* q1, double d_hat, int64_t* n_vf,
                    int64_t* n_ee, int64_t* n_ov);
/* copy the resident candidate set out: vf (n_vf,4), ee (n_ee,4), ov (n_ov,2) */
int abd_get_candidates(abd_scene* s, int64_t* vf, int64_t* ee, int64_t* ov);
/* upload a CandidateSet (contact.py:175-204) as the resident set */
int abd_set_candidates(abd_scene* s, int64_t n_vf, const int64_t* vf, int64_t n_ee, const int64_t* ee,
                       int64_t n_ov, const int64_t* ov);
/* contact_energy  contact.py:560-583 over the resident candidates */
int abd_contact_energy(abd_scene* s, const double* q, double kappa, double d_hat, double* energy);
/* candidate_min_distance_sq  contact.py:541-557 (returns +inf when empty) */
int abd_candidate_min_d2(abd_scene* s, const double* q, double* d2);
/* intersection audit: exact closed-triangle intersection (triangles_intersect_batch,
 * intersect.py:18-42); tri_a, tri_b (n,3,3); out[i] = 1 when they intersect */
int abd_tri_intersect_batch(int64_t n, const double* tri_a, const double* tri_b, uint8_t* out);
/* body pairs i < j whose surfaces intersect or one contains the other at q
 * (_intersecting_body_pairs, scene.py:652-698): pairs (cap,2) in canonical order,
 * n_pairs = total found (pairs beyond cap are not written) */
int abd_intersecting_pairs(abd_scene* s, const double* q, int64_t cap, int64_t* pairs, int64_t* n_pairs);
/* generation counters of the resident candidate and friction sets: bumped by every call
 * that rewrites them (abd_set_*, abd_broad_phase, abd_friction_precompute, abd_advance_step
 * and its stats broad phase).  Host-side caches of "what is resident" key on these. */
int abd_resident_generation(abd_scene* s, int64_t* cand_gen, int64_t* fric_gen);
/* global_min_distance  solver.py:396-473 (exact; pairs of two kinematic bodies are skipped
 * when skip_static_pairs != 0, the reference default) */
int abd_global_min_distance(abd_scene* s, const double* q, int skip_static_pairs, double* dist);
/* contact_gradient_hessian  contact.py:646-675 -> resident PairBlocks; n_active out */
int abd_contact_gradient_hessian(abd_scene* s, const double* q, double kappa, double d_hat, int project,
                                 int64_t* n_active);
/* copy resident PairBlocks out: grad (n,24), hess (n,24,24), d_sq (n) */
int abd_get_pair_blocks(abd_scene* s, int64_t* body_a, int64_t* body_b, double* grad, double* hess,
                        double* d_sq);
/* friction_precompute  contact.py:722-790 -> resident FrictionData; n out */
int abd_friction_precompute(abd_scene* s, const double* q_prev, double kappa, double d_hat, double mu,
                            int64_t* n);
int abd_get_friction(abd_scene* s, int64_t* body_a, int64_t* body_b, double* lam, double* tangent_map,
                     double* offset, double* basis);
int abd_set_friction(abd_scene* s, int64_t n, const int64_t* body_a, const int64_t* body_b, const double* lam,
                     double mu, const double* tangent_map, const double* offset);
/* step_filter  ccd.py:130-153 over the resident candidates */
int abd_step_filter(abd_scene* s, const double* q, const double* dq, double slack, double* alpha);

/* incremental-potential pieces over resident candidates + friction
 * (solver.py:179-205, :257-348).  q_tilde: (n_bodies,12). */
int abd_compute_q_tilde(abd_scene* s, const double* q, const double* q_dot, const double* forces, double dt,
                        double* q_tilde);
int abd_ip_value(abd_scene* s, const double* q, const double* q_tilde, double dt, double kappa, double d_hat,
                 double eps_v, double* value);
/* assemble  solver.py:257-342 -> resident gradient + BSR; n_off out */
int abd_assemble(abd_scene* s, const double* q, const double* q_tilde, double dt, double kappa, double d_hat,
                 double eps_v, int64_t* n_off);
/* copy the resident system out: grad (n_dyn*12), diag (n_dyn,12,12), keys (n_off,2), off (n_off,12,12) */
int abd_get_system(abd_scene* s, double* grad, double* diag, int64_t* off_keys, double* off_blocks);
/* solve the resident system H dx = -grad (block-Jacobi PCG) */
int abd_solve_resident(abd_scene* s, double rel_tol, int max_iters, double* dx, int* iters, double* rel_res);
/* dx = -H^-1 g of the resident system by the device sparse block Cholesky with refinement
 * (BlockCholesky(H).solve_refined(-g, rel_tol), sparse.py:90-161 / solver.py:345-348);
 * solves = triangular solves performed (1 + corrections, at most 3 corrections). */
int abd_solve_resident_cholesky(abd_scene* s, double rel_tol, double* dx, int* solves, double* rel_res);

/* advance_step  solver.py:493-628 with device-resident state. */
typedef struct abd_step_params {
  double dt, d_hat, kappa_barrier, mu, epsilon_v, newton_tol, ccd_slack, ccd_step_scale;
  double pcg_rel_tol;
  int max_newton_iters, friction_outer_iters, pcg_max_iters;
  int compute_min_distance; /* 1: StepStats.min_distance semantics (solver.py:604-611) */
  /* Newton linear solve: 0 = sparse block Cholesky + refinement (BlockCholesky.solve_refined,
   * sparse.py:90-161; the reference's solver), 1 = pipelined block-Jacobi PCG to pcg_rel_tol */
  int linear_solver;
  /* 1: StepStats.min_iterate_distance = min over the Newton iterates of
   * global_min_distance(q) (StepParams.audit_iterates, solver.py:577-580) */
  int audit_iterates;
} abd_step_params;

typedef struct abd_step_stats {
  int iterations, converged, nondescent_fallbacks;
  int pcg_iters_total;     /* PCG iterations, or triangular solves of the Cholesky path */
  int64_t candidates;      /* max candidate count over the step (StepStats.candidates) */
  double min_distance, ip_value, max_ortho_error, last_dq_over_dt;
  double min_iterate_distance; /* +inf unless audit_iterates */
  double t_broad, t_assemble, t_solve, t_ccd, t_line_search, t_total; /* ms, CUDA events */
} abd_step_stats;

/* per-kernel instrumentation accumulated by the driver (CUDA events on the scene stream):
 * which = 0: block-Jacobi PCG solve (k_pcg), 1: pair assembly (k_pair_blocks),
 * 2: CCD (k_ccd), 3: broad phase primitive pairs (k_prim_pairs).
 * launches, total device ms, total algorithmic bytes (SURVEY §8(d) per-unit figures). */
int abd_kernel_stats(abd_scene* s, int which, int64_t* launches, double* ms, double* bytes, int64_t* units);
int abd_kernel_stats_reset(abd_scene* s);
/* device timer on the scene stream: start records an event, stop syncs and returns ms */
int abd_timer_start(abd_scene* s);
int abd_timer_stop(abd_scene* s, double* ms);

/* ---------------- multi-GPU: one process per GPU ----------------
 * Body-slab partition, recut every step: dynamic bodies sorted by position along the
 * longest axis and cut into `world` slabs balanced by primitive count.  A body pair
 * belongs to the slab of its lower body (higher when the lower is kinematic): this
 * rank evaluates its primitive pairs, pair blocks, CCD queries and energies (halo
 * pairs across a slab face are evaluated once).  Partial systems are all-reduced;
 * the Newton system is solved by a distributed PCG over the slabs (slab-local
 * sparse Cholesky preconditioner, slab segments of the search direction exchanged,
 * dot products all-reduced); energies, CCD bound and error flags are all-reduced,
 * so every rank holds the same state.  A scene starts single-rank.  dtype: 0 f64,
 * 1 i32, 2 i64; op: 0 sum, 1 min, 2 max.  The callback receives a device pointer after
 * the scene stream has been synchronised and must complete the in-place reduction
 * before returning (0 = success). */
typedef int (*abd_allreduce_fn)(void* user, void* device_ptr, int64_t count, int dtype, int op);
int abd_nccl_unique_id(uint8_t* out128);
int abd_scene_set_comm_nccl(abd_scene* s, const uint8_t* id128, int rank, int world);
int abd_scene_set_comm_callback(abd_scene* s, int rank, int world, abd_allreduce_fn fn, void* user);
/* the current step's slab owner per body (-1 kinematic) and the cut axis (partition.py restates it) */
int abd_get_slab_owner(abd_scene* s, int32_t* owner, int32_t* axis);

int abd_set_state(abd_scene* s, const double* q, const double* q_dot);
/* World positions of every vertex (bodies concatenated, V x 3) at host q (n_bodies x 12), or at the
 * resident state when q is NULL: x = rest @ A^T + p with the reference's rounding
 * (contact.py:149-153 world_positions_all; scene.py:341-349 world_vertices for frames). */
int abd_world_vertices(abd_scene* s, const double* q, double* out);
/* Joint reduction q_dyn = T u + q_const (constraints.py:206-402, SystemModel.reduction,
 * solver.py:114): T row-major (12 n_dyn x n_unknowns), copied to the device; n_unknowns = 0
 * removes it.  With a reduction, abd_advance_step solves the Newton system through
 * T^T H T (solver.py:479-490, dense on the device) and falls back to T T^T (-g) on a
 * non-descent direction (solver.py:557-561).  Single-rank scenes only. */
int abd_set_reduction(abd_scene* s, int64_t n_unknowns, const double* T);
int abd_get_state(abd_scene* s, double* q, double* q_dot);
/* forces (n_bodies,12) host; NULL = reuse the last uploaded forces. energy_trace may be NULL
 * (else >= max_newton_iters*friction_outer_iters doubles). */
int abd_advance_step(abd_scene* s, const double* forces, const abd_step_params* p, abd_step_stats* st,
                     double* energy_trace);

#ifdef __cplusplus
}
#endif
#endif /* ABD_B200_H */
