// K4: block-Jacobi preconditioned CG on the resident symmetric BSR, replacing
// the reference's BlockCholesky.solve_refined (sparse.py:90-161, solver.py:
// 345-348) under the same contract ||A x - b|| <= rel_tol ||b||.
//
// One persistent cooperative launch per solve, pipelined CG (Ghysels &
// Vanroose 2014, preconditioned variant): per iteration ONE grid-wide sync
// carries both the dot products (r.u, w.u, r.r) and the SpMV input m = M w
// of every block row (m is double-buffered because neighbours read it while
// it is rewritten).
// Work mapping: one thread per scalar row; a CTA owns 16 whole block rows
// (192 threads) so the 12x12 block-Jacobi apply needs only __syncthreads.
// The SpMV row reads its 12x12 blocks as 6 double2 per block (the 12 threads
// of a block row read the block's 1152 contiguous bytes) and gathers the
// neighbour's 12 input values (L1-broadcast among those 12 threads).
// Every CTA reduces the per-CTA partials in the same fixed order after the
// grid sync (deterministic).  The recursive residual decides convergence;
// the true residual b - A x is then checked and CG restarts from x if needed.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "driver.h"

namespace cg = cooperative_groups;

namespace abd {

// R block rows per CTA (12 R threads); the solve picks R by problem size
template <int R>
struct CgShape {
  static constexpr int THREADS = 12 * R;
  static constexpr int WARPS = (THREADS + 31) / 32;
};

struct CgArgs {
  int n;
  const int* row_ptr;
  const int* col;
  const double* val;
  const double* pinv;
  const int* bad;
  const double* b;
  double* x;
  double *r, *u, *w, *m, *m2, *z, *q, *s, *p;
  double* part;  // 2 banks x 4 values x gridDim.x
  double rel_tol;
  int max_iters;
  int* out_iters;
  double* out_rel;
};

__device__ __forceinline__ double spmv_row(const CgArgs& a, int br, int rr, const double* __restrict__ v) {
  double acc0 = 0.0, acc1 = 0.0;
  const int k1 = a.row_ptr[br + 1];
  int k = a.row_ptr[br];
  for (; k + 1 < k1; k += 2) {
    const double2* b0 = reinterpret_cast<const double2*>(a.val + 144 * (int64_t)k + 12 * rr);
    const double2* b1 = b0 + 72;
    const double* x0 = v + 12 * (int64_t)__ldg(a.col + k);
    const double* x1 = v + 12 * (int64_t)__ldg(a.col + k + 1);
#pragma unroll
    for (int h = 0; h < 6; ++h) {
      double2 m0 = __ldg(b0 + h), m1 = __ldg(b1 + h);
      acc0 += m0.x * x0[2 * h] + m0.y * x0[2 * h + 1];
      acc1 += m1.x * x1[2 * h] + m1.y * x1[2 * h + 1];
    }
  }
  if (k < k1) {
    const double2* b0 = reinterpret_cast<const double2*>(a.val + 144 * (int64_t)k + 12 * rr);
    const double* x0 = v + 12 * (int64_t)__ldg(a.col + k);
#pragma unroll
    for (int h = 0; h < 6; ++h) {
      double2 m0 = __ldg(b0 + h);
      acc0 += m0.x * x0[2 * h] + m0.y * x0[2 * h + 1];
    }
  }
  return acc0 + acc1;
}

__device__ __forceinline__ double prec_row(const CgArgs& a, int br, int rr, const double* __restrict__ v) {
  const double2* P = reinterpret_cast<const double2*>(a.pinv + 144 * (int64_t)br + 12 * rr);
  const double* vv = v + 12 * (int64_t)br;
  double acc = 0.0;
#pragma unroll
  for (int h = 0; h < 6; ++h) {
    double2 pm = __ldg(P + h);
    acc += pm.x * vv[2 * h] + pm.y * vv[2 * h + 1];
  }
  return acc;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// per-CTA fixed-order sums of NV per-thread values -> part[v * gridDim.x + cta]
template <int NV, int CG_WARPS>
__device__ __forceinline__ void cta_partials(double (&v)[NV], double* sh, double* part) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) sh[k * CG_WARPS + wid] = v[k];
  __syncthreads();
  if (threadIdx.x < NV) {
    double t = 0.0;
#pragma unroll
    for (int wi = 0; wi < CG_WARPS; ++wi) t += sh[threadIdx.x * CG_WARPS + wi];
    part[threadIdx.x * gridDim.x + blockIdx.x] = t;
  }
}

// every CTA sums the per-CTA partials in the same fixed order
template <int NV, int CG_WARPS>
__device__ __forceinline__ void grid_totals(const double* part, double* sh, double (&out)[NV]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x)
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] += part[k * gridDim.x + i];
#pragma unroll
  for (int k = 0; k < NV; ++k) acc[k] = warp_sum(acc[k]);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) sh[128 + k * CG_WARPS + wid] = acc[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double t = 0.0;
#pragma unroll
    for (int wi = 0; wi < CG_WARPS; ++wi) t += sh[128 + k * CG_WARPS + wi];
    out[k] = t;
  }
}

template <int CG_ROWS>
__global__ void __launch_bounds__(CgShape<CG_ROWS>::THREADS) k_cg(CgArgs a) {
  constexpr int W = CgShape<CG_ROWS>::WARPS;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[256];
  if (*a.bad != 0x7fffffff) return;  // non-SPD preconditioner block: host raises
  const int lb = threadIdx.x / 12, rr = threadIdx.x % 12;
  const int groups = (a.n + CG_ROWS - 1) / CG_ROWS;
  double* bankA = a.part;
  double* bankB = a.part + 4 * gridDim.x;
  // ---- init: x = 0, r = b, |b|^2 ; then u = M r (block-row local)
  double v1[1] = {0.0};
  for (int g = blockIdx.x; g < groups; g += gridDim.x) {
    int br = g * CG_ROWS + lb;
    bool live = br < a.n;
    int64_t t = 12 * (int64_t)br + rr;
    if (live) {
      double bt = a.b[t];
      a.x[t] = 0.0;
      a.r[t] = bt;
      v1[0] += bt * bt;
    }
    __syncthreads();
    if (live) a.u[t] = prec_row(a, br, rr, a.r);
  }
  cta_partials<1, W>(v1, sh, bankA);
  grid.sync();
  double tb[1];
  grid_totals<1, W>(bankA, sh, tb);
  const double bnorm = sqrt(tb[0]);
  if (bnorm == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *a.out_iters = 0;
      *a.out_rel = 0.0;
    }
    return;
  }
  const double tol = a.rel_tol * bnorm;
  int it = 0;
  double rel = 1.0;
  for (int restart = 0; restart < 6; ++restart) {
    // ---- w = A u, m = M w, partials (r.u, w.u, r.r)
    double pv[3] = {0.0, 0.0, 0.0};
    for (int g = blockIdx.x; g < groups; g += gridDim.x) {
      int br = g * CG_ROWS + lb;
      bool live = br < a.n;
      int64_t t = 12 * (int64_t)br + rr;
      if (live) {
        double wt = spmv_row(a, br, rr, a.u);
        a.w[t] = wt;
        double rt = a.r[t], ut = a.u[t];
        pv[0] += rt * ut;
        pv[1] += wt * ut;
        pv[2] += rt * rt;
      }
      __syncthreads();
      if (live) a.m[t] = prec_row(a, br, rr, a.w);
    }
    cta_partials<3, W>(pv, sh, bankB);
    grid.sync();
    double* cur = bankB;
    double* nxt = bankA;
    double* mc = a.m;
    double* mn = a.m2;
    double gamma_old = 0.0, alpha_old = 1.0;
    bool first = true;
    while (true) {
      double tot[3];
      grid_totals<3, W>(cur, sh, tot);
      double gam = tot[0], del = tot[1], rn = sqrt(fmax(tot[2], 0.0));
      rel = rn / bnorm;
      if (rn <= tol) break;
      if (it >= a.max_iters || !(gam > 0.0)) break;
      double beta = first ? 0.0 : gam / gamma_old;
      double denom = first ? del : del - beta * gam / alpha_old;
      if (!(denom > 0.0)) break;  // breakdown: restart from the current x
      double alpha = gam / denom;
      double pv2[3] = {0.0, 0.0, 0.0};
      for (int g = blockIdx.x; g < groups; g += gridDim.x) {
        int br = g * CG_ROWS + lb;
        bool live = br < a.n;
        int64_t t = 12 * (int64_t)br + rr;
        if (live) {
          double nt = spmv_row(a, br, rr, mc);  // n = A m
          double zt = nt, qt = mc[t], st = a.w[t], pt = a.u[t];
          if (!first) {
            zt += beta * a.z[t];
            qt += beta * a.q[t];
            st += beta * a.s[t];
            pt += beta * a.p[t];
          }
          a.z[t] = zt;
          a.q[t] = qt;
          a.s[t] = st;
          a.p[t] = pt;
          a.x[t] += alpha * pt;
          double rt = a.r[t] - alpha * st;
          double ut = a.u[t] - alpha * qt;
          double wn = a.w[t] - alpha * zt;
          a.r[t] = rt;
          a.u[t] = ut;
          a.w[t] = wn;
          pv2[0] += rt * ut;
          pv2[1] += wn * ut;
          pv2[2] += rt * rt;
        }
        __syncthreads();  // the whole block row of w is written (same CTA)
        if (live) mn[t] = prec_row(a, br, rr, a.w);
      }
      cta_partials<3, W>(pv2, sh, nxt);
      grid.sync();
      ++it;
      gamma_old = gam;
      alpha_old = alpha;
      first = false;
      double* tmp = cur;
      cur = nxt;
      nxt = tmp;
      tmp = mc;
      mc = mn;
      mn = tmp;
    }
    // ---- true residual r = b - A x, u = M r, |r|^2
    grid.sync();
    double tv[1] = {0.0};
    for (int g = blockIdx.x; g < groups; g += gridDim.x) {
      int br = g * CG_ROWS + lb;
      bool live = br < a.n;
      int64_t t = 12 * (int64_t)br + rr;
      if (live) {
        double rt = a.b[t] - spmv_row(a, br, rr, a.x);
        a.r[t] = rt;
        tv[0] += rt * rt;
      }
      __syncthreads();
      if (live) a.u[t] = prec_row(a, br, rr, a.r);
    }
    cta_partials<1, W>(tv, sh, bankA);
    grid.sync();
    double tt[1];
    grid_totals<1, W>(bankA, sh, tt);
    rel = sqrt(tt[0]) / bnorm;
    if (sqrt(tt[0]) <= tol || it >= a.max_iters) break;
    grid.sync();  // bank reuse in the restart
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.out_iters = it;
    *a.out_rel = rel;
  }
}

// ---------------------------------------------------------------------------
// Register-resident variant for systems that fit one pass of the grid (one
// thread per scalar row for the whole solve): x, r, u, w, z, q, s, p and m
// live in registers, the CTA's 12x12 preconditioner blocks in shared memory;
// only m (read by neighbours' SpMV) and the per-CTA partials touch global
// memory per iteration.
constexpr int RES_ROWS = 80;  // 960 threads, one CTA per SM
constexpr int RES_THREADS = 12 * RES_ROWS;
constexpr int RES_WARPS = RES_THREADS / 32;

__global__ void __launch_bounds__(RES_THREADS, 1) k_cg_res(CgArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double dsm[];
  double* Psh = dsm;                       // RES_ROWS * 144
  double* vsh = dsm + RES_ROWS * 144;      // RES_ROWS * 12 (block-row exchange)
  double* sh = vsh + RES_ROWS * 12;        // 256 reduction scratch
  if (*a.bad != 0x7fffffff) return;
  const int lb = threadIdx.x / 12, rr = threadIdx.x % 12;
  // block rows dealt round-robin over CTAs: contact-heavy (long) rows are
  // spatially clustered in body order, this spreads them across SMs
  const int br = blockIdx.x + (int)gridDim.x * lb;
  const bool live = br < a.n;
  const int64_t t = 12 * (int64_t)br + rr;
  for (int e = threadIdx.x; e < RES_ROWS * 144; e += RES_THREADS) {
    int row = blockIdx.x + (int)gridDim.x * (e / 144);
    Psh[e] = row < a.n ? a.pinv[144 * (int64_t)row + e % 144] : 0.0;
  }
  auto prec = [&](double v) -> double {  // (P^-1 v)_row, v exchanged through smem
    __syncthreads();
    vsh[threadIdx.x] = v;
    __syncthreads();
    const double* P = Psh + 144 * lb + 12 * rr;
    const double* vv = vsh + 12 * lb;
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 12; ++c) acc += P[c] * vv[c];
    return acc;
  };
  double* bankA = a.part;
  double* bankB = a.part + 4 * gridDim.x;
  const double bt = live ? a.b[t] : 0.0;
  double x = 0.0, r = bt;
  double u = prec(r);
  if (live) a.u[t] = u;
  double v1[1] = {bt * bt};
  cta_partials<1, RES_WARPS>(v1, sh, bankA);
  grid.sync();
  double tb[1];
  grid_totals<1, RES_WARPS>(bankA, sh, tb);
  const double bnorm = sqrt(tb[0]);
  if (bnorm == 0.0) {
    if (live) a.x[t] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *a.out_iters = 0;
      *a.out_rel = 0.0;
    }
    return;
  }
  const double tol = a.rel_tol * bnorm;
  int it = 0;
  double rel = 1.0;
  double w = 0.0, m = 0.0, z = 0.0, q = 0.0, s = 0.0, p = 0.0;
  for (int restart = 0; restart < 6; ++restart) {
    // w = A u (u of neighbours from global), m = P^-1 w
    w = live ? spmv_row(a, br, rr, a.u) : 0.0;
    m = prec(w);
    double* mc = a.m;
    double* mn = a.m2;
    if (live) mc[t] = m;
    double pv[3] = {r * u, w * u, r * r};
    cta_partials<3, RES_WARPS>(pv, sh, bankB);
    grid.sync();
    double* cur = bankB;
    double* nxt = bankA;
    double gamma_old = 0.0, alpha_old = 1.0;
    bool first = true;
    while (true) {
      double tot[3];
      grid_totals<3, RES_WARPS>(cur, sh, tot);
      double gam = tot[0], del = tot[1], rn = sqrt(fmax(tot[2], 0.0));
      rel = rn / bnorm;
      if (rn <= tol) break;
      if (it >= a.max_iters || !(gam > 0.0)) break;
      double beta = first ? 0.0 : gam / gamma_old;
      double denom = first ? del : del - beta * gam / alpha_old;
      if (!(denom > 0.0)) break;
      double alpha = gam / denom;
      double nt = live ? spmv_row(a, br, rr, mc) : 0.0;  // n = A m
      z = nt + beta * z;
      q = m + beta * q;
      s = w + beta * s;
      p = u + beta * p;
      x += alpha * p;
      r -= alpha * s;
      u -= alpha * q;
      w -= alpha * z;
      m = prec(w);
      if (live) mn[t] = m;
      double pv2[3] = {r * u, w * u, r * r};
      cta_partials<3, RES_WARPS>(pv2, sh, nxt);
      grid.sync();
      ++it;
      gamma_old = gam;
      alpha_old = alpha;
      first = false;
      double* tmp = cur;
      cur = nxt;
      nxt = tmp;
      tmp = mc;
      mc = mn;
      mn = tmp;
    }
    // true residual r = b - A x
    if (live) a.x[t] = x;
    grid.sync();
    r = live ? bt - spmv_row(a, br, rr, a.x) : 0.0;
    u = prec(r);
    if (live) a.u[t] = u;
    double tv[1] = {r * r};
    cta_partials<1, RES_WARPS>(tv, sh, bankA);
    grid.sync();
    double tt[1];
    grid_totals<1, RES_WARPS>(bankA, sh, tt);
    rel = sqrt(tt[0]) / bnorm;
    if (sqrt(tt[0]) <= tol || it >= a.max_iters) break;
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.out_iters = it;
    *a.out_rel = rel;
  }
}

// ---------------------------------------------------------------------------
// Cluster block-Jacobi preconditioner.  The body-coupling graph of a contact
// step is mostly tiny connected components (isolated bodies, stacked pairs
// and short columns; see profiles/): block-Jacobi over single bodies leaves
// CG resolving every component's spectrum at once (~10^3 iterations).  Here
// each connected component of <= CL_SMALL bodies becomes ONE dense block
// (exact inverse: CG converges on it in one step) and larger components are
// cut into BFS-contiguous clusters of <= CL_BIG bodies.  Single-body
// clusters are exactly the 12x12 block-Jacobi of the north star.
constexpr int CL_MAX = 8;  // rows per cluster upper bound (dense size 96)

struct ClusterArgs {
  const int* slot_row;      // G * R: block row of each CTA slot (-1 = empty)
  const int* slot_base;     // G * R: CTA-local slot of the cluster's first row
  const int* slot_k;        // G * R: cluster size (rows)
  const long long* slot_off;  // G * R: offset of the cluster's (12K)^2 inverse
  const double* minv;
};

__global__ void __launch_bounds__(RES_THREADS, 1) k_cg_cluster(CgArgs a, ClusterArgs c) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double dsm[];
  double* vsh = dsm;                  // RES_ROWS * 12 (cluster exchange)
  double* sh = vsh + RES_ROWS * 12;   // 256 reduction scratch
  if (*a.bad != 0x7fffffff) return;
  const int lb = threadIdx.x / 12, rr = threadIdx.x % 12;
  const int slot = blockIdx.x * RES_ROWS + lb;
  const int br = c.slot_row[slot];
  const bool live = br >= 0;
  const int64_t t = 12 * (int64_t)(live ? br : 0) + rr;
  const int cbase = c.slot_base[slot];
  const int ck = c.slot_k[slot];
  const int dim = 12 * ck;
  const double* Mrow = c.minv + c.slot_off[slot] + (int64_t)(12 * (lb - cbase) + rr) * dim;
  auto prec = [&](double v) -> double {  // (M^-1 v)_row over the row's cluster
    __syncthreads();
    vsh[threadIdx.x] = v;
    __syncthreads();
    if (!live) return 0.0;
    const double* vv = vsh + 12 * cbase;
    double acc0 = 0.0, acc1 = 0.0;
    int j = 0;
    for (; j + 1 < dim; j += 2) {
      double2 mm = __ldg(reinterpret_cast<const double2*>(Mrow + j));
      acc0 += mm.x * vv[j];
      acc1 += mm.y * vv[j + 1];
    }
    if (j < dim) acc0 += Mrow[j] * vv[j];
    return acc0 + acc1;
  };
  double* bankA = a.part;
  double* bankB = a.part + 4 * gridDim.x;
  const double bt = live ? a.b[t] : 0.0;
  double x = 0.0, r = bt;
  double u = prec(r);
  if (live) a.u[t] = u;
  double v1[1] = {bt * bt};
  cta_partials<1, RES_WARPS>(v1, sh, bankA);
  grid.sync();
  double tb[1];
  grid_totals<1, RES_WARPS>(bankA, sh, tb);
  const double bnorm = sqrt(tb[0]);
  if (bnorm == 0.0) {
    if (live) a.x[t] = 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *a.out_iters = 0;
      *a.out_rel = 0.0;
    }
    return;
  }
  const double tol = a.rel_tol * bnorm;
  int it = 0;
  double rel = 1.0;
  double w = 0.0, m = 0.0, z = 0.0, q = 0.0, s = 0.0, p = 0.0;
  for (int restart = 0; restart < 6; ++restart) {
    w = live ? spmv_row(a, br, rr, a.u) : 0.0;
    m = prec(w);
    double* mc = a.m;
    double* mn = a.m2;
    if (live) mc[t] = m;
    double pv[3] = {r * u, w * u, r * r};
    cta_partials<3, RES_WARPS>(pv, sh, bankB);
    grid.sync();
    double* cur = bankB;
    double* nxt = bankA;
    double gamma_old = 0.0, alpha_old = 1.0;
    bool first = true;
    while (true) {
      double tot[3];
      grid_totals<3, RES_WARPS>(cur, sh, tot);
      double gam = tot[0], del = tot[1], rn = sqrt(fmax(tot[2], 0.0));
      rel = rn / bnorm;
      if (rn <= tol) break;
      if (it >= a.max_iters || !(gam > 0.0)) break;
      double beta = first ? 0.0 : gam / gamma_old;
      double denom = first ? del : del - beta * gam / alpha_old;
      if (!(denom > 0.0)) break;
      double alpha = gam / denom;
      double nt = live ? spmv_row(a, br, rr, mc) : 0.0;
      z = nt + beta * z;
      q = m + beta * q;
      s = w + beta * s;
      p = u + beta * p;
      x += alpha * p;
      r -= alpha * s;
      u -= alpha * q;
      w -= alpha * z;
      m = prec(w);
      if (live) mn[t] = m;
      double pv2[3] = {r * u, w * u, r * r};
      cta_partials<3, RES_WARPS>(pv2, sh, nxt);
      grid.sync();
      ++it;
      gamma_old = gam;
      alpha_old = alpha;
      first = false;
      double* tmp = cur;
      cur = nxt;
      nxt = tmp;
      tmp = mc;
      mc = mn;
      mn = tmp;
    }
    if (live) a.x[t] = x;
    grid.sync();
    r = live ? bt - spmv_row(a, br, rr, a.x) : 0.0;
    u = prec(r);
    if (live) a.u[t] = u;
    double tv[1] = {r * r};
    cta_partials<1, RES_WARPS>(tv, sh, bankA);
    grid.sync();
    double tt[1];
    grid_totals<1, RES_WARPS>(bankA, sh, tt);
    rel = sqrt(tt[0]) / bnorm;
    if (sqrt(tt[0]) <= tol || it >= a.max_iters) break;
    grid.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *a.out_iters = it;
    *a.out_rel = rel;
  }
}

// dense inverse of each cluster's diagonal block (one CTA of 96 threads per
// cluster): gather the cluster's BSR blocks, Cholesky with lane i owning row i,
// then lane j solves column j of the inverse.
__global__ void __launch_bounds__(96) k_cluster_inv(int ncl, const int* __restrict__ cl_off,
                                                    const int* __restrict__ cl_rows,
                                                    const long long* __restrict__ cl_minv, const int* __restrict__ row_ptr,
                                                    const int* __restrict__ col, const double* __restrict__ val,
                                                    double* minv, int* bad) {
  extern __shared__ double Ls[];  // dim x (dim + 1)
  const int cidx = blockIdx.x;
  if (cidx >= ncl) return;
  const int r0 = cl_off[cidx], K = cl_off[cidx + 1] - r0;
  const int dim = 12 * K, ld = dim + 1;
  for (int e = threadIdx.x; e < dim * ld; e += blockDim.x) Ls[e] = 0.0;
  __syncthreads();
  for (int i = 0; i < K; ++i) {
    int row = cl_rows[r0 + i];
    for (int k = row_ptr[row]; k < row_ptr[row + 1]; ++k) {
      int cc = col[k], j = -1;
      for (int q = 0; q < K; ++q)
        if (cl_rows[r0 + q] == cc) j = q;
      if (j < 0) continue;
      for (int e = threadIdx.x; e < 144; e += blockDim.x)
        Ls[(12 * i + e / 12) * ld + 12 * j + e % 12] = val[144 * (int64_t)k + e];
    }
  }
  __syncthreads();
  const int tid = threadIdx.x;
  bool ok = true;
  for (int j = 0; j < dim; ++j) {
    double d = Ls[j * ld + j];
    ok = ok && (d > 0.0);
    double sd = sqrt(fmax(d, 1e-300));
    __syncthreads();
    if (tid > j && tid < dim) Ls[tid * ld + j] /= sd;
    if (tid == j) Ls[j * ld + j] = sd;
    __syncthreads();
    if (tid > j && tid < dim) {
      double ltj = Ls[tid * ld + j];
      for (int k = j + 1; k <= tid; ++k) Ls[tid * ld + k] -= ltj * Ls[k * ld + j];
    }
    __syncthreads();
  }
  if (!ok) {
    if (tid == 0) atomicMin(bad, cl_rows[r0]);
    return;
  }
  if (tid >= dim) return;
  // column tid of L^-T L^-1, written row-major (symmetric)
  double* out = minv + cl_minv[cidx];
  double y[96];
  for (int i = 0; i < dim; ++i) {
    double v = (i == tid) ? 1.0 : 0.0;
    for (int k = 0; k < i; ++k) v -= Ls[i * ld + k] * y[k];
    y[i] = v / Ls[i * ld + i];
  }
  for (int i = dim - 1; i >= 0; --i) {
    double v = y[i];
    for (int k = i + 1; k < dim; ++k) v -= Ls[k * ld + i] * y[k];
    y[i] = v / Ls[i * ld + i];
  }
  for (int i = 0; i < dim; ++i) out[(int64_t)i * dim + tid] = y[i];
}

// host: components + clusters + CTA packing for the resident BSR; returns the
// number of CTAs (0 if the packing does not fit one cooperative wave)
static int build_clusters(Scene& s, int max_ctas, int ksmall, int kbig, int& ncl, int64_t& minv_total) {
  Bsr& H = s.H;
  int n = H.n;
  cudaStream_t st = s.stream;
  std::vector<int2> keys(H.n_off);
  H.upper_keys.download(keys.data(), H.n_off, st);
  SSYNC(st);
  std::vector<int> deg(n + 1, 0);
  for (auto& k : keys) {
    deg[k.x]++;
    deg[k.y]++;
  }
  std::vector<int> adj_off(n + 1, 0);
  for (int i = 0; i < n; ++i) adj_off[i + 1] = adj_off[i] + deg[i];
  std::vector<int> adj(adj_off[n]), fill(adj_off.begin(), adj_off.end() - 1);
  for (auto& k : keys) {
    adj[fill[k.x]++] = k.y;
    adj[fill[k.y]++] = k.x;
  }
  std::vector<int> seen(n, 0), comp, clust_off{0}, clust_rows;
  clust_rows.reserve(n);
  std::vector<int> queue;
  for (int s0 = 0; s0 < n; ++s0) {
    if (seen[s0]) continue;
    comp.clear();
    queue.clear();
    queue.push_back(s0);
    seen[s0] = 1;
    for (size_t h = 0; h < queue.size(); ++h) {
      int v = queue[h];
      comp.push_back(v);
      for (int e = adj_off[v]; e < adj_off[v + 1]; ++e)
        if (!seen[adj[e]]) {
          seen[adj[e]] = 1;
          queue.push_back(adj[e]);
        }
    }
    int kk = (int)comp.size() <= ksmall ? (int)comp.size() : kbig;  // BFS-contiguous chunks
    for (size_t b = 0; b < comp.size(); b += kk) {
      size_t e = std::min(comp.size(), b + kk);
      std::vector<int> chunk(comp.begin() + b, comp.begin() + e);
      std::sort(chunk.begin(), chunk.end());
      clust_rows.insert(clust_rows.end(), chunk.begin(), chunk.end());
      clust_off.push_back((int)clust_rows.size());
    }
  }
  ncl = (int)clust_off.size() - 1;
  // pack clusters into CTAs of RES_ROWS slots, round-robin for load balance
  int G = std::max(1, (n + RES_ROWS - 1) / RES_ROWS);
  std::vector<int> used;
  std::vector<int> cl_cta(ncl), cl_slot(ncl);
  for (;;) {
    if (G > max_ctas) return 0;
    used.assign(G, 0);
    bool fit = true;
    int cur = 0;
    for (int ci = 0; ci < ncl && fit; ++ci) {
      int K = clust_off[ci + 1] - clust_off[ci];
      int tries = 0;
      while (used[cur] + K > RES_ROWS && tries < G) {
        cur = (cur + 1) % G;
        ++tries;
      }
      if (used[cur] + K > RES_ROWS) {
        fit = false;
        break;
      }
      cl_cta[ci] = cur;
      cl_slot[ci] = used[cur];
      used[cur] += K;
      cur = (cur + 1) % G;
    }
    if (fit) break;
    ++G;
  }
  std::vector<int> slot_row(G * RES_ROWS, -1), slot_base(G * RES_ROWS, 0), slot_k(G * RES_ROWS, 1);
  std::vector<long long> slot_off(G * RES_ROWS, 0), cl_minv(ncl);
  long long off = 0;
  for (int ci = 0; ci < ncl; ++ci) {
    int K = clust_off[ci + 1] - clust_off[ci];
    cl_minv[ci] = off;
    for (int q = 0; q < K; ++q) {
      int sl = cl_cta[ci] * RES_ROWS + cl_slot[ci] + q;
      slot_row[sl] = clust_rows[clust_off[ci] + q];
      slot_base[sl] = cl_slot[ci];
      slot_k[sl] = K;
      slot_off[sl] = off;
    }
    off += (long long)(12 * K) * (12 * K);
  }
  minv_total = off;
  Scene::Work& w = s.w;
  w.cl_slot_row.upload(slot_row.data(), slot_row.size(), st);
  w.cl_slot_base.upload(slot_base.data(), slot_base.size(), st);
  w.cl_slot_k.upload(slot_k.data(), slot_k.size(), st);
  w.cl_slot_off.upload(slot_off.data(), slot_off.size(), st);
  w.cl_off.upload(clust_off.data(), clust_off.size(), st);
  w.cl_rows.upload(clust_rows.data(), clust_rows.size(), st);
  w.cl_minv.upload(cl_minv.data(), cl_minv.size(), st);
  return G;
}

void launch_jacobi_inv(Scene& s, int n, const int* diag_pos, const double* val, double* pinv, int* bad);

// solve H x = rhs on the resident BSR; returns iterations, rel residual
int pcg_solve(Scene& s, const double* rhs, double* x, double rel_tol, int max_iters, double& rel_res) {
  Bsr& H = s.H;
  cudaStream_t st = s.stream;
  int n = H.n;
  if (n == 0) {
    rel_res = 0.0;
    return 0;
  }
  int64_t N = 12 * (int64_t)n;
  Scene::Work& w = s.w;
  w.pinv.resize(144 * (int64_t)n);
  for (DVec<double>* v : {&w.r, &w.z, &w.p, &w.p2, &w.Ap, &w.cg_u, &w.cg_w, &w.cg_m, &w.cg_q}) v->resize(N);
  w.bad.resize(1);
  w.iters.resize(1);
  w.scal.resize(4);
  int big = 0x7fffffff;
  dev_set_i32(st, w.bad.p, big);
  launch_jacobi_inv(s, n, H.diag_pos.p, H.val.p, w.pinv.p, w.bad.p);
  // single-pass systems: register-resident solver
  const size_t res_smem = (size_t)(RES_ROWS * 144 + RES_ROWS * 12 + 256) * sizeof(double);
  static int res_bps = -1;
  if (res_bps < 0) {
    CK(cudaFuncSetAttribute((void*)k_cg_res, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&res_bps, k_cg_res, RES_THREADS, res_smem));
  }
  static const bool no_res = getenv("ABD_CG_NO_RES") != nullptr;
  int res_groups = (n + RES_ROWS - 1) / RES_ROWS;
  bool use_res = !no_res && res_bps >= 1 && res_groups <= res_bps * s.num_sms;
  // small systems: few fat CTAs (cheaper grid barrier); large: 16-row CTAs
  static int rows_env = -1;
  if (rows_env < 0) {
    const char* e = getenv("ABD_CG_ROWS");
    rows_env = e ? atoi(e) : 0;
  }
  int rows = rows_env ? rows_env : (n <= 80 * s.num_sms ? 80 : 16);
  void* kfun = rows == 80 ? (void*)k_cg<80> : (void*)k_cg<16>;
  int threads = 12 * (rows == 80 ? 80 : 16);
  static int bps[2] = {-1, -1};
  int& blocks_per_sm = bps[rows == 80 ? 1 : 0];
  if (blocks_per_sm < 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kfun, threads, 0));
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  int groups = (n + rows - 1) / rows;
  int grid = std::max(1, std::min(groups, blocks_per_sm * s.num_sms));
  w.part.resize(8 * (int64_t)std::max(grid, res_groups));
  CgArgs a;
  a.n = n;
  a.row_ptr = H.row_ptr.p;
  a.col = H.col.p;
  a.val = H.val.p;
  a.pinv = w.pinv.p;
  a.bad = w.bad.p;
  a.b = rhs;
  a.x = x;
  a.r = w.r.p;
  a.u = w.cg_u.p;
  a.w = w.cg_w.p;
  a.m = w.cg_m.p;
  a.m2 = w.p2.p;
  a.z = w.z.p;
  a.q = w.cg_q.p;
  a.s = w.Ap.p;
  a.p = w.p.p;
  a.part = w.part.p;
  a.rel_tol = rel_tol;
  a.max_iters = max_iters;
  a.out_iters = w.iters.p;
  a.out_rel = w.scal.p;
  void* args[] = {&a};
  static const bool no_cluster = getenv("ABD_CG_NO_CLUSTER") != nullptr;
  static const int ksmall = getenv("ABD_CL_SMALL") ? atoi(getenv("ABD_CL_SMALL")) : CL_MAX;
  static const int kbig = getenv("ABD_CL_BIG") ? atoi(getenv("ABD_CL_BIG")) : 4;
  static int cl_bps = -1;
  const size_t cl_smem = (size_t)(RES_ROWS * 12 + 256) * sizeof(double);
  if (cl_bps < 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cl_bps, k_cg_cluster, RES_THREADS, cl_smem));
    CK(cudaFuncSetAttribute((void*)k_cluster_inv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            96 * 97 * (int)sizeof(double)));
  }
  int G = 0, ncl = 0;
  int64_t minv_total = 0;
  if (use_res && !no_cluster && cl_bps >= 1)
    G = build_clusters(s, cl_bps * s.num_sms, std::min(ksmall, CL_MAX), std::min(kbig, CL_MAX), ncl, minv_total);
  if (G > 0) {
    w.minv.resize(std::max<int64_t>(minv_total, 1));
    w.part.resize(8 * (int64_t)std::max(grid, G));
    a.part = w.part.p;
    k_cluster_inv<<<ncl, 96, 96 * 97 * sizeof(double), st>>>(ncl, w.cl_off.p, w.cl_rows.p, w.cl_minv.p, H.row_ptr.p,
                                                            H.col.p, H.val.p, w.minv.p, w.bad.p);
    note_launch("k_cluster_inv");
    if (s.instrument) CK(cudaEventRecord(s.ev0, st));
    ClusterArgs ca{w.cl_slot_row.p, w.cl_slot_base.p, w.cl_slot_k.p, w.cl_slot_off.p, w.minv.p};
    void* cargs[] = {&a, &ca};
    grid = G;
    CK(cudaLaunchCooperativeKernel((void*)k_cg_cluster, dim3(G), dim3(RES_THREADS), cargs, cl_smem, st));
  } else if (use_res) {
    if (s.instrument) CK(cudaEventRecord(s.ev0, st));
    grid = res_groups;
    CK(cudaLaunchCooperativeKernel((void*)k_cg_res, dim3(grid), dim3(RES_THREADS), args, res_smem, st));
  } else {
    if (s.instrument) CK(cudaEventRecord(s.ev0, st));
    CK(cudaLaunchCooperativeKernel(kfun, dim3(grid), dim3(threads), args, 0, st));
  }
  note_launch("k_cg");
  if (s.instrument) CK(cudaEventRecord(s.ev1, st));
  int* hp = reinterpret_cast<int*>(s.h_pinned + 16);
  CK(cudaMemcpyAsync(hp, w.iters.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hp + 1, w.bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(s.h_pinned + 20, w.scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  SSYNC(st);
  int hit = hp[0];
  rel_res = s.h_pinned[20];
  if (hp[1] != big) throw Error(ABD_ERR_FACTORIZATION, "non-SPD diagonal block in block-Jacobi PCG", hp[1]);
  if (s.instrument) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, s.ev0, s.ev1));
    Scene::KStat& k = s.kstat[0];
    k.launches += 1;
    k.units += hit;
    k.ms += ms;
    // algorithmic bytes per iteration: BSR SpMV 1152 nnzb, preconditioner
    // (1152 n block-Jacobi, or 8 * sum k_c^2 * 144 for the dense cluster inverses), 13 vectors.
    const double prec_bytes = G > 0 ? 8.0 * (double)minv_total : 1152.0 * n;
    k.bytes += (double)hit * (1152.0 * (double)H.nnzb + prec_bytes + 13.0 * 96.0 * n);
    static const bool trace = getenv("ABD_TRACE_PCG") != nullptr;
    if (trace) {
      // connected components of the block graph (diagnostic)
      std::vector<int2> keys(H.n_off);
      H.upper_keys.download(keys.data(), H.n_off, st);
      SSYNC(st);
      std::vector<int> par(n);
      for (int i = 0; i < n; ++i) par[i] = i;
      auto find = [&](int v) {
        while (par[v] != v) v = par[v] = par[par[v]];
        return v;
      };
      for (auto& k : keys) par[find(k.x)] = find(k.y);
      std::vector<int> sz(n, 0);
      for (int i = 0; i < n; ++i) sz[find(i)]++;
      int ncomp = 0, big = 0, coupled = 0;
      for (int i = 0; i < n; ++i)
        if (sz[i]) {
          ++ncomp;
          big = std::max(big, sz[i]);
          if (sz[i] > 1) coupled += sz[i];
        }
      fprintf(stderr,
              "[abd pcg] n=%d nnzb=%lld grid=%d iters=%d ms=%.3f us/iter=%.2f rel=%.2e comps=%d largest=%d "
              "coupled=%d\n",
              n, (long long)H.nnzb, grid, hit, ms, hit ? 1e3 * ms / hit : 0.0, rel_res, ncomp, big, coupled);
    }
  }
  return hit;
}

}  // namespace abd
