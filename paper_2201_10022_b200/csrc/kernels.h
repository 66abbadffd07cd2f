// Host-side launchers of the sm_100a kernels (device pointers in/out).
#pragma once
#include "abd_math.cuh"
#include "scene.h"

#include <vector>

namespace abd {

void note_launch(const char* name);
void reduce_fixed_device(Scene& s, const double* partials, int n, double* out_dev);
void reduce_fixed_stream(cudaStream_t st, const double* partials, int n, double* out_dev);
void reduce_fixed_multi(cudaStream_t st, const double* partials, int n, int count, double* out_dev);

// plain-data view of the scene geometry passed to kernels by value
struct SceneView {
  const int* v_off;
  const int* e_off;
  const int* t_off;
  const double* rest;
  const int* edges;
  const int* tris;
  const double* elen2;
  const unsigned char* dyn;
  const int* slot;
  int B;
};
SceneView view(const Scene& s);

constexpr int FRIC_STRIDE = 51;  // tmap (48) | offset (2) | lam (1)
constexpr int RED_BLOCKS = 592;  // fixed grid for deterministic reductions (4 x 148)
constexpr int RED_THREADS = 256;

// ---- stateless batch launchers (k_batch.cu) ----
void launch_pt_closest(cudaStream_t st, int64_t n, const double* z, double* d2, int* region, double* bary);
void launch_ee_closest(cudaStream_t st, int64_t n, const double* z, double* d2, int* region, double* s,
                       double* t);
void launch_d2_derivs(cudaStream_t st, int kind, int64_t n, const double* z, double* d2, double* grad,
                      double* hess, int* region, double* gamma);
void launch_mollifier(cudaStream_t st, int64_t n, const double* z, const double* eps, double* val, double* grad,
                      double* hess);
void launch_barrier(cudaStream_t st, int64_t n, const double* s, double dh, double* b0, double* b1, double* b2,
                    int* err);
void launch_ortho(cudaStream_t st, int64_t n, const double* q, const double* k, int project, double* e,
                  double* g, double* h);
void launch_psd(cudaStream_t st, int64_t n, int k, const double* H, double* out);
void launch_accd(cudaStream_t st, int kind, int64_t n, const double* x, const double* dx, double slack,
                 double tmax, int max_iters, double* t, int* err);
void launch_contact_pairs(cudaStream_t st, int kind, int64_t n, const double* z, const double* xb, const double* eps,
                          double kappa, double dh, const unsigned char* dyn, int project, double* g12, double* h12,
                          double* g24, double* h24);
void launch_pblk_dense(cudaStream_t st, int64_t n, const double* pblk, double* dense);
void launch_friction(cudaStream_t st, int64_t n, const int2* bodies, const double* rec, double mu,
                     const double* q, const unsigned char* dyn, double dt, double eps_v, int project,
                     double* energy_partials, double* grad24, double* hess24, double* pblk_out);

// ---- scene narrow phase (k_narrow.cu) ----
// activity flags d^2 < d_hat^2 for the resident candidates of `kind`
// swept body boxes (union of vertex boxes inflated by h) into out (B x 6)
void launch_body_boxes(Scene& s, const double* q0, const double* q1, double h, double* out);
// intersection audit (k_audit.cu)
void launch_tri_intersect(cudaStream_t st, int64_t n, const double* ta, const double* tb, unsigned char* out);
void launch_pair_flags_both(Scene& s, const double* q, double dh2, int* flags, int* err);
void launch_mark_active_q(Scene& s, const double* q, double dh2, int* flags);
void launch_scatter_active(Scene& s, int64_t n, const int* flags, const int* pos, int* act);
void launch_pair_runs(Scene& s, const double* q, double kappa, double dh, int project, const int* act,
                      int64_t n_vf_act, int64_t total);
void launch_pair_blocks_act(Scene& s, int kind, const double* q, double kappa, double dh, int project,
                            const int* act, int64_t slot_off, int64_t count);
void launch_cand_min_d2(Scene& s, int kind, const double* q, unsigned long long* best_bits);
void launch_friction_pre(Scene& s, int kind, const double* q, double kappa, double dh, const int* flags,
                         const int* pos, int64_t base, double* basis_out);
// ACCD hot list (Scene::Work::hot_*): capacity and the iteration count that makes a query "slow"
constexpr int CCD_HOT_CAP = 64;
constexpr int CCD_SLOW_IT = 32;
struct HotCcd {
  const int4* rows;
  const int* kind;
  const double* t;
  const int* bad;
  const int* it;
  int n;
  int4* slow_rows;
  int* slow_kind;
  unsigned* slow_cnt;
  int slow_cap, slow_it;
};
void launch_ccd_hot(Scene& s, const double* q, const double* dq, double slack);
// K6 (body | contact VF | contact EE | friction partials, 4 x RED_BLOCKS) in one launch
void launch_energy_all(Scene& s, const double* q, const double* qt, double dt, double kappa, double dh,
                       double eps_v, double* red4, int* err);
void launch_ccd_both(Scene& s, const double* q, const double* dq, double slack, unsigned long long* tmin,
                     int* err, bool track = false);
// per-body inertia + orthogonality terms (K1): grad0/diag0 per dynamic slot, energy partials
void launch_body_terms(Scene& s, const double* q, const double* q_tilde, double dt, double* grad0,
                       double* diag0, double* energy_partials, int want_derivs);
void launch_q_tilde(Scene& s, const double* q, const double* q_dot, const double* f, double dt, double* qt);
void launch_axpy_q(Scene& s, const double* q, double alpha, const double* dq, double* out, int64_t n);

}  // namespace abd
