// ACCD, orthogonality potential and friction evaluation device routines.
#pragma once
#include "abd_pair.cuh"

namespace abd {

// ---------------------------------------------------------------------------
// additive CCD conservative advancement for one query (ccd.py:59-104),
// reproducing numpy's arithmetic order bit-for-bit.  t_cut: early exit once
// t >= t_cut (t only grows, so a global minimum is unchanged).
ABD_D double accd_query(int kind, V3* x, const V3* dx, double slack, double tmax, int max_iters,
                        volatile const unsigned long long* t_cut_bits, bool& domain_err, int* it_out = nullptr) {
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
  int it = 0;
  for (; it < max_iters; ++it) {
    // the first iterate is x itself: reuse d0 (bitwise the same value)
    double d = it == 0 ? d0 : sqrt(pair_d2(kind, x));
    double adv = xsub(d, gap);
    bool stalled = adv < stall_eps;
    double tl = stalled ? 0.0 : adv / lp;
    double tn = xadd(t, tl);
    bool reached = tn >= tmax;
    t = reached ? tmax : tn;
    if (stalled || reached) break;
    for (int k = 0; k < 4; ++k) x[k] = xadd3(x[k], xscale(tl, p[k]));
    // early exit once this query can no longer lower the global minimum; the
    // shared bound lives in L2, so it is polled every 8 iterations (returning any
    // t >= the bound leaves the minimum unchanged)
    if (t_cut_bits && (it & 7) == 7) {
      unsigned long long cb = *t_cut_bits;
      if (t >= __longlong_as_double((long long)cb)) break;
    }
  }
  if (it_out) *it_out = it;
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

// symmetric 3x3 eigen-decomposition (cyclic Jacobi): S = V diag(w) V^T, columns V[:][i]
ABD_D void sym3_eig(double S[3][3], double w[3], double V[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) V[i][j] = i == j ? 1.0 : 0.0;
  double fro = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) fro += S[i][j] * S[i][j];
  for (int sweep = 0; sweep < 30 && fro > 0.0; ++sweep) {
    double off = S[0][1] * S[0][1] + S[0][2] * S[0][2] + S[1][2] * S[1][2];
    if (off <= 1e-36 * fro) break;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = p + 1; q < 3; ++q) {
        double apq = S[p][q];
        if (apq == 0.0) continue;
        double theta = (S[q][q] - S[p][p]) * rcp_fast(2.0 * apq);
        const double th2 = theta * theta + 1.0;
        double t = (theta >= 0.0 ? 1.0 : -1.0) * rcp_fast(fabs(theta) + th2 * rsqrt_fast(th2));
        double c = rsqrt_fast(t * t + 1.0), s = t * c, tau = s * rcp_fast(1.0 + c);
        S[p][p] -= t * apq;
        S[q][q] += t * apq;
        S[p][q] = S[q][p] = 0.0;
        int r = 3 - p - q;
        double g = S[r][p], h = S[r][q];
        S[r][p] = S[p][r] = g - s * (h + g * tau);
        S[r][q] = S[q][r] = h + s * (g - h * tau);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          double g2 = V[k][p], h2 = V[k][q];
          V[k][p] = g2 - s * (h2 + g2 * tau);
          V[k][q] = h2 + s * (g2 - h2 * tau);
        }
      }
  }
  w[0] = S[0][0];
  w[1] = S[1][1];
  w[2] = S[2][2];
}

// PSD projection of the orthogonality Hessian in closed form.  With
// A = U diag(s) V^T, the Hessian acts on dA = U X V^T as
//   H[X]_ij = 4k ((s_i^2 + s_j^2 - 1) X_ij + s_i s_j X_ji)
// so its 9 eigenpairs are 4k(3 s_i^2 - 1) on u_i v_i^T and
// 4k(s_i^2 + s_j^2 - 1 +- s_i s_j) on (u_i v_j^T +- u_j v_i^T)/sqrt2.
// proj(H) = H - sum_{lambda < 0} lambda vec(dA) vec(dA)^T  (equals the
// reference's eigh-clamp of body.py:281-296 applied at solver.py:292-294).
// singular values (descending) and vectors of the 3x3 A (u[i], v[i]: i-th pair)
ABD_D void ortho_svd3(const double* A, double s[3], double u[3][3], double v[3][3]) {
  double S[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) S[a][b] = A[a] * A[b] + A[3 + a] * A[3 + b] + A[6 + a] * A[6 + b];
  double w[3], V[3][3];
  sym3_eig(S, w, V);
  // order by descending singular value
  int o0 = 0, o1 = 1, o2 = 2;
  if (w[o0] < w[o1]) { int t = o0; o0 = o1; o1 = t; }
  if (w[o1] < w[o2]) { int t = o1; o1 = o2; o2 = t; }
  if (w[o0] < w[o1]) { int t = o0; o0 = o1; o1 = t; }
  int ord[3] = {o0, o1, o2};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    s[i] = sqrt(fmax(w[ord[i]], 0.0));
#pragma unroll
    for (int c = 0; c < 3; ++c) v[i][c] = V[c][ord[i]];
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
#pragma unroll
    for (int r = 0; r < 3; ++r) u[i][r] = A[3 * r] * v[i][0] + A[3 * r + 1] * v[i][1] + A[3 * r + 2] * v[i][2];
#pragma unroll
    for (int j = 0; j < i; ++j) {
      double d = u[i][0] * u[j][0] + u[i][1] * u[j][1] + u[i][2] * u[j][2];
#pragma unroll
      for (int r = 0; r < 3; ++r) u[i][r] -= d * u[j][r];
    }
    double nn = sqrt(u[i][0] * u[i][0] + u[i][1] * u[i][1] + u[i][2] * u[i][2]);
    if (nn > 1e-12 * (s[0] > 0.0 ? s[0] : 1.0)) {
#pragma unroll
      for (int r = 0; r < 3; ++r) u[i][r] /= nn;
    } else if (i == 2) {
      u[2][0] = u[0][1] * u[1][2] - u[0][2] * u[1][1];
      u[2][1] = u[0][2] * u[1][0] - u[0][0] * u[1][2];
      u[2][2] = u[0][0] * u[1][1] - u[0][1] * u[1][0];
    } else {
      // degenerate: any unit vector orthogonal to the previous ones
      double e[3] = {1.0, 0.0, 0.0};
      for (int tries = 0; tries < 3; ++tries) {
        e[0] = tries == 0; e[1] = tries == 1; e[2] = tries == 2;
        for (int j = 0; j < i; ++j) {
          double d = e[0] * u[j][0] + e[1] * u[j][1] + e[2] * u[j][2];
          for (int r = 0; r < 3; ++r) e[r] -= d * u[j][r];
        }
        double ne = sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
        if (ne > 0.5) {
          for (int r = 0; r < 3; ++r) u[i][r] = e[r] / ne;
          break;
        }
      }
    }
  }
}

ABD_D void ortho_project_closed(const double* q, double k, double* H) {
  const double* A = q + 3;  // A[r][c] = A[3 r + c]
  double s[3], v[3][3], u[3][3];  // v[i], u[i]: i-th singular vectors
  ortho_svd3(A, s, u, v);
  const double k4 = 4.0 * k;
  const double r2 = 0.70710678118654752440;
  // negative modes only
  for (int m = 0; m < 9; ++m) {
    int i, j;
    double sg;
    if (m < 3) { i = j = m; sg = 0.0; }
    else { int p = (m - 3) >> 1; i = p == 2 ? 1 : 0; j = p == 0 ? 1 : 2; sg = ((m - 3) & 1) ? -1.0 : 1.0; }
    double lam = (m < 3) ? k4 * (3.0 * s[i] * s[i] - 1.0) : k4 * (s[i] * s[i] + s[j] * s[j] - 1.0 + sg * s[i] * s[j]);
    if (!(lam < 0.0)) continue;
    double dA[9];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        dA[3 * r + c] = (m < 3) ? u[i][r] * v[i][c] : r2 * (u[i][r] * v[j][c] + sg * u[j][r] * v[i][c]);
    for (int a = 0; a < 9; ++a)
      for (int b = 0; b < 9; ++b) H[(3 + a) * 12 + 3 + b] -= lam * dA[a] * dA[b];
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
// compact friction record (abd_pblk.cuh type 2): g24 | 2 | G0 | G1 | h00 h01 h11
ABD_D void friction_compact_dev(const double* rec, const FricEval& e, double mu, bool dyn_a, bool dyn_b,
                                bool project, double* out) {
  double sc = mu * rec[50];
  double gu0 = sc * e.f1y * e.u[0], gu1 = sc * e.f1y * e.u[1];
  double an = e.y > 0.0 ? (e.f1p - e.f1y) / (e.y * e.y) : 0.0;
  double h00 = sc * (e.f1y + an * e.u[0] * e.u[0]);
  double h01 = sc * (an * e.u[0] * e.u[1]);
  double h11 = sc * (e.f1y + an * e.u[1] * e.u[1]);
  if (project) psd_project_2x2(h00, h01, h11);
  const double* G0 = rec;
  const double* G1 = rec + 24;
  out[24] = 2.0;
  for (int c = 0; c < 24; ++c) {
    bool dc = c < 12 ? dyn_a : dyn_b;
    out[c] = dc ? G0[c] * gu0 + G1[c] * gu1 : 0.0;
    out[25 + c] = dc ? G0[c] : 0.0;
    out[49 + c] = dc ? G1[c] : 0.0;
  }
  out[73] = h00;
  out[74] = h01;
  out[75] = h11;
}

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
