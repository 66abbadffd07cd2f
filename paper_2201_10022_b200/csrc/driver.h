#pragma once
#include "abd_pair.cuh"
#include "kernels.h"

namespace abd {

// k_broad.cu
void broad_phase(Scene& s, const double* q0, const double* q1, double d_hat);
// k_solve.cu
void build_pattern(Scene& s, const int2* ov, int64_t n_ov, const int2* fb, int64_t n_f, bool from_cands = false);
void reduce_system(Scene& s, const double* diag0, const double* grad0, double* neg_out = nullptr);
int pcg_solve(Scene& s, const double* rhs, double* x, double rel_tol, int max_iters, double& rel_res);
// k_chol.cu: sparse block Cholesky + refinement; returns the number of triangular solves
int chol_solve(Scene& s, const double* rhs, double* x, double rel_tol, double& rel_res, int max_refine = 3);
void chol_begin(Scene& s, const double* rhs, double* x);
void launch_neg(cudaStream_t st, int64_t n, const double* a, double* b);  // b = -a
// the host analysis of the coupling structure copied out by mark_structure runs on a
// worker thread while the pair-block / reduction kernels are launched (post), or is
// discarded when the pattern changes (drop)
void chol_analysis_post(Scene& s);
void chol_analysis_drop(Scene& s);
void chol_verify_post(Scene& s);
int chol_finish(Scene& s, double rel_tol, double& rel_res, int max_refine, bool& changed);
void spmv(Scene& s, const double* x, double* y);
void load_bsr(Scene& s, int n, int bdim, const double* diag, int64_t n_off, const int64_t* keys, const double* off);
// k_reduced.cu: joint-reduced Newton direction (solver.py:479-490)
void set_reduction(Scene& s, int64_t nu, const double* T_host);
void reduced_solve(Scene& s, const double* neg_g, double* dx);
void reduced_project(Scene& s, const double* v, double* out);
// comm.cu
void comm_get_nccl_id(void* out128);
void comm_init_nccl(Scene& s, const void* id128, int rank, int world);
void comm_init_callback(Scene& s, int rank, int world, abd_allreduce_fn fn, void* user);
void comm_destroy(Scene& s);
void comm_allreduce(Scene& s, void* dptr, int64_t count, int dtype, int op);
int64_t comm_allgather_i64(Scene& s, const int64_t* local, int64_t n_local, DVec<int64_t>& out);
// body slabs of a multi-rank scene from the state q (device): owners per body / slot
void slab_partition(Scene& s, const double* q);
// zero the structure flags of pattern blocks not inside this rank's slab
void slab_mask_structure(Scene& s, int* flags);
// k_chol.cu: distributed PCG, slab-local sparse Cholesky preconditioner (multi-rank solve)
int slab_pcg(Scene& s, const double* b, double* x, double rel_tol, int max_iters, double& rel_res);
// k_stats.cu
double global_min_distance(Scene& s, const double* q, int skip_static = 1);
// the same value for the end-of-step stats; overwrites the resident candidate set
double global_min_distance_stats(Scene& s, const double* q);
// body pairs (i < j) whose closed surfaces intersect or contain one another (k_audit.cu)
std::vector<int2> intersecting_body_pairs(Scene& s, const double* q);
void world_vertices(Scene& s, const double* q, double* out);
// driver.cu
int64_t contact_blocks(Scene& s, const double* q, double kappa, double dh, int project, bool mark = false,
                       bool allow_runs = false);
void append_friction_blocks(Scene& s, const double* q, double dt, double eps_v, int project);
int64_t friction_precompute(Scene& s, const double* q, double kappa, double dh, double mu, DVec<double>* basis);
double contact_energy(Scene& s, const double* q, double kappa, double dh);
double friction_energy(Scene& s, const double* q, double dt, double eps_v);
double body_energy(Scene& s, const double* q, const double* qt, double dt);
double ip_value(Scene& s, const double* q, const double* qt, double dt, double kappa, double dh, double eps_v);
double step_filter(Scene& s, const double* q, const double* dq, double slack);
double candidate_min_d2(Scene& s, const double* q);
// neg_out: also write -gradient (12 n_dyn doubles; single rank only -- a partitioned system is summed afterwards)
void assemble(Scene& s, const double* q, const double* qt, double dt, double kappa, double dh, double eps_v,
              double* neg_out = nullptr);
void advance_step(Scene& s, const double* forces_host, const abd_step_params& P, abd_step_stats& st, double* trace);

}  // namespace abd
