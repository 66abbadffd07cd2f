// ACCD, orthogonality potential and friction evaluation device routines.
#pragma once
#include "abd_pair.cuh"

namespace abd {

// ---------------------------------------------------------------------------
// additive CCD conservative advancement for one query (ccd.py:59-104),
// reproducing numpy's arithmetic order bit-for-bit.  t_cut: early exit once
// t >= t_cut (t only grows, so a global minimum is unchanged).
ABD_D double accd_query(int kind, V3* x, const V3* dx, double slack, double tmax, int max_iters,
                        volatile const unsigned long long* t_cut_bits, bool& domain_err) {
  V3 mean;
  mean.x = xadd(xadd(xadd(dx[0].x, dx[1].x), dx[2].x), dx[3].x) / 4.0;
  mean.y = xadd(xadd(xadd(dx[0].y, dx[1].y), dx[2].y), dx[3].y) / 4.0;
  mean.z = xadd(xadd(xadd(dx[0].z, dx[1].z), dx[2].z), dx[3].z) / 4.0;
  V3 p[4];
  double nm[4];
  for (int k = 0; k < 4; ++k) {
    p[k] = xsub3(dx[k], mean);
    nm[k] = xnorm_seq(p[k]);
  }
  double lp;
  if (kind == KIND_VF) lp = xadd(nm[0], fmax(fmax(nm[1], nm[2]), nm[3]));
  else lp = xadd(fmax(nm[0], nm[1]), fmax(nm[2], nm[3]));
  double d0sq = pair_d2(kind, x);
  if (!(d0sq > 0.0)) {
    domain_err = true;
    return 0.0;
  }
  double d0 = sqrt(d0sq);
  double gap = xmul(slack, d0);
  if (!(lp > 0.0)) return tmax;
  double t = 0.0;
  double stall_eps = xmul(1e-12, d0);
  for (int it = 0; it < max_iters; ++it) {
    double d = sqrt(pair_d2(kind, x));
    double adv = xsub(d, gap);
    bool stalled = adv < stall_eps;
    double tl = stalled ? 0.0 : adv / lp;
    double tn = xadd(t, tl);
    bool reached = tn >= tmax;
    t = reached ? tmax : tn;
    if (stalled || reached) break;
    for (int k = 0; k < 4; ++k) x[k] = xadd3(x[k], xscale(tl, p[k]));
    if (t_cut_bits) {
      unsigned long long cb = *t_cut_bits;
      if (t >= __longlong_as_double((long long)cb)) break;
    }
  }
  return fmin(t, tmax);
}

// ---------------------------------------------------------------------------
// orthogonality potential (body.py:229-278): V = k (sum (G_ii-1)^2 + sum_{i!=j} G_ij^2)
ABD_D double ortho_energy_dev(const double* q, double k) {
  const double* A = q + 3;
  double G[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) G[i][j] = A[3 * i] * A[3 * j] + A[3 * i + 1] * A[3 * j + 1] + A[3 * i + 2] * A[3 * j + 2];
  double acc = 0.0;
  for (int i = 0; i < 3; ++i) acc += (G[i][i] - 1.0) * (G[i][i] - 1.0);
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (i != j) acc += G[i][j] * G[i][j];
  return k * acc;
}

// gradient (12, translation zero) and Hessian (12x12 row-major)
ABD_D void ortho_derivs_dev(const double* q, double k, double* g, double* H) {
  const double* A = q + 3;
  double G[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) G[i][j] = A[3 * i] * A[3 * j] + A[3 * i + 1] * A[3 * j + 1] + A[3 * i + 2] * A[3 * j + 2];
  double s = 4.0 * k;
  for (int c = 0; c < 3; ++c) g[c] = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;
      for (int j = 0; j < 3; ++j) acc += (G[i][j] - (i == j ? 1.0 : 0.0)) * A[3 * j + c];
      g[3 + 3 * i + c] = s * acc;
    }
  if (!H) return;
  double S[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) S[a][b] = A[a] * A[b] + A[3 + a] * A[3 + b] + A[6 + a] * A[6 + b];
  for (int r = 0; r < 144; ++r) H[r] = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
          double v;
          if (i == j) {
            double aa = A[3 * i + a] * A[3 * i + b];
            v = 2.0 * aa + (a == b ? G[i][i] - 1.0 : 0.0) + (S[a][b] - aa);
          } else {
            v = A[3 * j + a] * A[3 * i + b] + (a == b ? G[i][j] : 0.0);
          }
          H[(3 + 3 * i + a) * 12 + 3 + 3 * j + b] = s * v;
        }
}

// ---------------------------------------------------------------------------
// friction on one lagged pair (contact.py:805-853).  rec: tmap(48) off(2) lam(1)
struct FricEval {
  double u[2], y, f0, f1y, f1p;
};

ABD_D FricEval friction_eval(const double* rec, const double* qa, const double* qb, double eh) {
  FricEval e;
  for (int m = 0; m < 2; ++m) {
    double acc = 0.0;
    for (int c = 0; c < 12; ++c) acc += rec[m * 24 + c] * qa[c];
    for (int c = 0; c < 12; ++c) acc += rec[m * 24 + 12 + c] * qb[c];
    e.u[m] = acc - rec[48 + m];
  }
  e.y = sqrt(e.u[0] * e.u[0] + e.u[1] * e.u[1]);
  F0Terms t = f0_terms(e.y, eh);
  e.f0 = t.f0;
  e.f1y = t.f1y;
  e.f1p = t.f1p;
  return e;
}

// g24 and H24 (full 24x24 into out, row-major) with kinematic zeroing
ABD_D void friction_blocks_dev(const double* rec, const FricEval& e, double mu, bool dyn_a, bool dyn_b,
                               bool project, double* g24, double* haa, double* hbb, double* hab) {
  double sc = mu * rec[50];
  double gu0 = sc * e.f1y * e.u[0], gu1 = sc * e.f1y * e.u[1];
  double an = e.y > 0.0 ? (e.f1p - e.f1y) / (e.y * e.y) : 0.0;
  double h00 = sc * (e.f1y + an * e.u[0] * e.u[0]);
  double h01 = sc * (an * e.u[0] * e.u[1]);
  double h11 = sc * (e.f1y + an * e.u[1] * e.u[1]);
  if (project) psd_project_2x2(h00, h01, h11);
  const double* G0 = rec;
  const double* G1 = rec + 24;
  for (int c = 0; c < 24; ++c) {
    bool dc = c < 12 ? dyn_a : dyn_b;
    g24[c] = dc ? G0[c] * gu0 + G1[c] * gu1 : 0.0;
  }
  for (int r = 0; r < 24; ++r) {
    bool dr = r < 12 ? dyn_a : dyn_b;
    double t0 = h00 * G0[r] + h01 * G1[r];
    double t1 = h01 * G0[r] + h11 * G1[r];
    for (int c = 0; c < 24; ++c) {
      bool dc = c < 12 ? dyn_a : dyn_b;
      double v = (dr && dc && ((r < 12) == (c < 12) || (dyn_a && dyn_b))) ? t0 * G0[c] + t1 * G1[c] : 0.0;
      if (r < 12 && c < 12) haa[r * 12 + c] = v;
      else if (r >= 12 && c >= 12) hbb[(r - 12) * 12 + c - 12] = v;
      else if (r < 12 && c >= 12) hab[r * 12 + c - 12] = v;
    }
  }
}

}  // namespace abd
