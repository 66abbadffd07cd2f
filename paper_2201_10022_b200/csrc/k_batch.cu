// Stateless batch kernels behind the per-function drop-in API
// (distance.py, contact.py barrier, body.py ortho/project_psd, ccd.py).
#include "abd_contact.cuh"
#include "abd_misc.cuh"
#include "abd_pblk.cuh"
#include "kernels.h"

namespace abd {

__device__ __forceinline__ void ldz(const double* z, int64_t i, V3* out) {
  for (int k = 0; k < 4; ++k) out[k] = ld3(z + i * 12 + 3 * k);
}

__global__ void k_pt_closest(int64_t n, const double* __restrict__ z, double* d2, int* region, double* bary) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 p[4];
  ldz(z, i, p);
  PTResult r = pt_closest(p[0], p[1], p[2], p[3]);
  d2[i] = r.d2;
  region[i] = r.region;
  bary[3 * i] = r.b0;
  bary[3 * i + 1] = r.b1;
  bary[3 * i + 2] = r.b2;
}

__global__ void k_ee_closest(int64_t n, const double* __restrict__ z, double* d2, int* region, double* s,
                             double* t) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 p[4];
  ldz(z, i, p);
  EEResult r = ee_closest(p[0], p[1], p[2], p[3]);
  d2[i] = r.d2;
  region[i] = r.region;
  s[i] = r.s;
  t[i] = r.t;
}

__global__ void k_d2_derivs(int kind, int64_t n, const double* __restrict__ z, double* d2, double* grad,
                            double* hess, int* region, double* gamma) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 p[4];
  ldz(z, i, p);
  Closest c = closest(kind, p);
  double g[12], H[144];
  d2_derivatives(kind, p, c, g, H);
  d2[i] = c.d2;
  region[i] = c.region;
  for (int k = 0; k < 4; ++k) gamma[4 * i + k] = c.gamma[k];
  for (int k = 0; k < 12; ++k) grad[12 * i + k] = g[k];
  for (int k = 0; k < 144; ++k) hess[144 * i + k] = H[k];
}

__global__ void k_mollifier(int64_t n, const double* __restrict__ z, const double* __restrict__ eps, double* val,
                            double* grad, double* hess) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 p[4];
  ldz(z, i, p);
  val[i] = mollifier_value(p, eps[i]);
  if (!grad) return;
  double g[12], H[144], v;
  if (!mollifier_derivs(p, eps[i], v, g, H)) {
    for (int k = 0; k < 12; ++k) g[k] = 0.0;
    for (int k = 0; k < 144; ++k) H[k] = 0.0;
  }
  for (int k = 0; k < 12; ++k) grad[12 * i + k] = g[k];
  for (int k = 0; k < 144; ++k) hess[144 * i + k] = H[k];
}

__global__ void k_barrier(int64_t n, const double* __restrict__ s, double dh, double* b0, double* b1, double* b2,
                          int* err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = s[i];
  if (!(v > 0.0)) atomicExch(err, 1);
  Barrier b = barrier_terms(v, dh);
  b0[i] = b.b0;
  b1[i] = b.b1;
  b2[i] = b.b2;
}

__global__ void k_ortho(int64_t n, const double* __restrict__ q, const double* __restrict__ k, int project,
                        double* e, double* g, double* h) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double qq[12], gg[12], H[144], V[144];
  for (int c = 0; c < 12; ++c) qq[c] = q[12 * i + c];
  e[i] = ortho_energy_dev(qq, k[i]);
  ortho_derivs_dev(qq, k[i], gg, H);
  (void)V;
  if (project) ortho_project_closed(qq, k[i], H);
  for (int c = 0; c < 12; ++c) g[12 * i + c] = gg[c];
  for (int c = 0; c < 144; ++c) h[144 * i + c] = H[c];
}

__global__ void k_psd(int64_t n, int k, const double* __restrict__ Hin, double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double A[24 * 24], V[24 * 24];
  for (int r = 0; r < k; ++r)
    for (int c = 0; c < k; ++c) A[r * 24 + c] = Hin[i * k * k + r * k + c];
  psd_project_jacobi<24>(A, V, k);
  for (int r = 0; r < k; ++r)
    for (int c = 0; c < k; ++c) out[i * k * k + r * k + c] = A[r * 24 + c];
}

__global__ void k_accd(int kind, int64_t n, const double* __restrict__ x, const double* __restrict__ dx,
                       double slack, double tmax, int max_iters, double* t, int* err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 xx[4], dd[4];
  ldz(x, i, xx);
  ldz(dx, i, dd);
  bool bad = false;
  t[i] = accd_query(kind, xx, dd, slack, tmax, max_iters, nullptr, bad);
  if (bad) atomicExch(err, 1);
}

// friction over explicit records: energy partials (fixed grid), blocks per pair
__global__ void k_friction(int64_t n, const int2* __restrict__ bodies, const double* __restrict__ rec, double mu,
                           const double* __restrict__ q, const unsigned char* __restrict__ dyn, double eh,
                           int project, double* partials, double* grad24, double* hess24, double* pblk) {
  __shared__ double sh[RED_THREADS];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int2 b = bodies[i];
    const double* r = rec + i * FRIC_STRIDE;
    FricEval e = friction_eval(r, q + 12 * b.x, q + 12 * b.y, eh);
    acc += mu * r[50] * e.f0;
    if (grad24 || pblk) {
      double g[24], haa[144], hbb[144], hab[144];
      friction_blocks_dev(r, e, mu, dyn[b.x] != 0, dyn[b.y] != 0, project != 0, g, haa, hbb, hab);
      if (grad24) {
        for (int c = 0; c < 24; ++c) grad24[i * 24 + c] = g[c];
        double* H = hess24 + i * 576;
        for (int rr = 0; rr < 12; ++rr)
          for (int cc = 0; cc < 12; ++cc) {
            H[rr * 24 + cc] = haa[rr * 12 + cc];
            H[(rr + 12) * 24 + cc + 12] = hbb[rr * 12 + cc];
            H[rr * 24 + cc + 12] = hab[rr * 12 + cc];
            H[(cc + 12) * 24 + rr] = hab[rr * 12 + cc];
          }
      }
      if (pblk) friction_compact_dev(r, e, mu, dyn[b.x] != 0, dyn[b.y] != 0, project != 0, pblk + i * PB_STRIDE);
    }
  }
  if (!partials) return;
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

// lean variants used by the Newton driver: energy-only partials, and pair blocks
// written straight into the PairBlocks records (no per-thread 24x24 staging)
__global__ void k_friction_energy(int64_t n, const int2* __restrict__ bodies, const double* __restrict__ rec,
                                  double mu, const double* __restrict__ q, double eh, double* partials) {
  __shared__ double sh[RED_THREADS];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int2 b = bodies[i];
    const double* r = rec + i * FRIC_STRIDE;
    FricEval e = friction_eval(r, q + 12 * b.x, q + 12 * b.y, eh);
    acc += mu * r[50] * e.f0;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

__global__ void k_friction_pblk(int64_t n, const int2* __restrict__ bodies, const double* __restrict__ rec,
                                double mu, const double* __restrict__ q, const unsigned char* __restrict__ dyn,
                                double eh, int project, double* pblk) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int2 b = bodies[i];
    const double* r = rec + i * FRIC_STRIDE;
    FricEval e = friction_eval(r, q + 12 * b.x, q + 12 * b.y, eh);
    friction_compact_dev(r, e, mu, dyn[b.x] != 0, dyn[b.y] != 0, project != 0, pblk + i * PB_STRIDE);
  }
}

// per-pair contact terms on explicit points (K3 arithmetic without the scene gather)
__global__ void __launch_bounds__(64) k_contact_pairs(int kind, int64_t n, const double* __restrict__ z,
                                                      const double* __restrict__ xb, const double* __restrict__ eps,
                                                      double kappa, double dh, const unsigned char* __restrict__ dyn,
                                                      int project, double* g12o, double* h12o, double* g24o,
                                                      double* h24o) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 p[4], r[4];
  ldz(z, i, p);
  ldz(xb, i, r);
  double blk[PB_DENSE];
  contact_pair_eval(kind, p, r, eps[i], kappa, dh, dyn[2 * i] != 0, dyn[2 * i + 1] != 0, project != 0, blk,
                    g12o + 12 * i, h12o + 144 * i);
  for (int k = 0; k < 24; ++k) g24o[24 * i + k] = blk[k];
  double* H = h24o + 576 * i;
  for (int rr = 0; rr < 12; ++rr)
    for (int cc = 0; cc < 12; ++cc) {
      H[rr * 24 + cc] = blk[24 + rr * 12 + cc];
      H[(rr + 12) * 24 + cc + 12] = blk[168 + rr * 12 + cc];
      H[rr * 24 + cc + 12] = blk[312 + rr * 12 + cc];
      H[(cc + 12) * 24 + rr] = blk[312 + rr * 12 + cc];
    }
}

// ---------------------------------------------------------------------------
#define GRID(n, b) dim3(grid_for((n), (b))), dim3(b), 0

void launch_contact_pairs(cudaStream_t st, int kind, int64_t n, const double* z, const double* xb, const double* eps,
                          double kappa, double dh, const unsigned char* dyn, int project, double* g12, double* h12,
                          double* g24, double* h24) {
  if (!n) return;
  k_contact_pairs<<<GRID(n, 64), st>>>(kind, n, z, xb, eps, kappa, dh, dyn, project, g12, h12, g24, h24);
  note_launch("k_contact_pairs");
}

void launch_pt_closest(cudaStream_t st, int64_t n, const double* z, double* d2, int* region, double* bary) {
  if (!n) return;
  k_pt_closest<<<GRID(n, 128), st>>>(n, z, d2, region, bary);
  note_launch("k_pt_closest");
}
void launch_ee_closest(cudaStream_t st, int64_t n, const double* z, double* d2, int* region, double* s,
                       double* t) {
  if (!n) return;
  k_ee_closest<<<GRID(n, 128), st>>>(n, z, d2, region, s, t);
  note_launch("k_ee_closest");
}
void launch_d2_derivs(cudaStream_t st, int kind, int64_t n, const double* z, double* d2, double* grad,
                      double* hess, int* region, double* gamma) {
  if (!n) return;
  k_d2_derivs<<<GRID(n, 64), st>>>(kind, n, z, d2, grad, hess, region, gamma);
  note_launch("k_d2_derivs");
}
void launch_mollifier(cudaStream_t st, int64_t n, const double* z, const double* eps, double* val, double* grad,
                      double* hess) {
  if (!n) return;
  k_mollifier<<<GRID(n, 64), st>>>(n, z, eps, val, grad, hess);
  note_launch("k_mollifier");
}
void launch_barrier(cudaStream_t st, int64_t n, const double* s, double dh, double* b0, double* b1, double* b2,
                    int* err) {
  if (!n) return;
  k_barrier<<<GRID(n, 128), st>>>(n, s, dh, b0, b1, b2, err);
  note_launch("k_barrier");
}
void launch_ortho(cudaStream_t st, int64_t n, const double* q, const double* k, int project, double* e, double* g,
                  double* h) {
  if (!n) return;
  k_ortho<<<GRID(n, 64), st>>>(n, q, k, project, e, g, h);
  note_launch("k_ortho");
}
void launch_psd(cudaStream_t st, int64_t n, int k, const double* H, double* out) {
  if (!n) return;
  k_psd<<<GRID(n, 32), st>>>(n, k, H, out);
  note_launch("k_psd");
}
void launch_accd(cudaStream_t st, int kind, int64_t n, const double* x, const double* dx, double slack, double tmax,
                 int max_iters, double* t, int* err) {
  if (!n) return;
  k_accd<<<GRID(n, 128), st>>>(kind, n, x, dx, slack, tmax, max_iters, t, err);
  note_launch("k_accd");
}
// compact pair records -> dense g24 | H_aa | H_bb | H_ab (readout / tests)
__global__ void k_pblk_dense(int64_t n, const double* __restrict__ pblk, double* dense) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n * PB_DENSE) return;
  const int64_t p = t / PB_DENSE;
  const int e = (int)(t % PB_DENSE);
  const double* rec = pblk + p * PB_STRIDE;
  double v;
  if (e < 24) {
    v = rec[e];
  } else {
    const int blk = (e - 24) / 144, idx = (e - 24) % 144, i = idx / 12, k = idx % 12;
    const int R = 12 * (blk == 1) + i, C = 12 * (blk >= 1) + k;
    v = pb_entry(rec, R, C);
  }
  dense[t] = v;
}

void launch_pblk_dense(cudaStream_t st, int64_t n, const double* pblk, double* dense) {
  if (n <= 0) return;
  k_pblk_dense<<<grid_for(n * PB_DENSE, 256), 256, 0, st>>>(n, pblk, dense);
  note_launch("k_pblk_dense");
}

void launch_friction(cudaStream_t st, int64_t n, const int2* bodies, const double* rec, double mu, const double* q,
                     const unsigned char* dyn, double dt, double eps_v, int project, double* partials,
                     double* grad24, double* hess24, double* pblk) {
  if (partials && !grad24 && !pblk) {
    k_friction_energy<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, bodies, rec, mu, q, eps_v * dt, partials);
    note_launch("k_friction_energy");
  } else if (pblk && !partials && !grad24) {
    k_friction_pblk<<<grid_for(n, 128), 128, 0, st>>>(n, bodies, rec, mu, q, dyn, eps_v * dt, project, pblk);
    note_launch("k_friction_pblk");
  } else {
    k_friction<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, bodies, rec, mu, q, dyn, eps_v * dt, project, partials,
                                                   grad24, hess24, pblk);
    note_launch("k_friction");
  }
}

}  // namespace abd
