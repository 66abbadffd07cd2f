// Per-pair contact algebra (fp64): d^2 derivatives, EE mollifier, barrier
// chain rule, J^T H J through an orthonormal basis of J's row space, PSD
// projection, lagged friction.  One thread evaluates one pair.
//
// References (file:line under /root/reference/pkg/src/stiffbody/):
//   distance.py:238-339  envelope gradient + Schur-complement Hessian of d^2
//   distance.py:342-401  near-parallel EE mollifier derivatives
//   contact.py:486-538   barrier chain rule (VF / EE product rule)
//   contact.py:466-483   per-point Jacobian J = [I3 | I3 (x) xbar^T]
//   contact.py:619-675   J^T H J, 24x24 PSD projection, kinematic sub-block rule
//   contact.py:711-853   lagged friction precompute / energy / derivatives
#pragma once
#include "abd_math.cuh"

namespace abd {

enum { KIND_VF = 0, KIND_EE = 1 };

// side of stacked point k (VF: vertex | tri ; EE: edge a | edge b)
ABD_D int side_of(int kind, int k) { return kind == KIND_VF ? (k == 0 ? 0 : 1) : (k < 2 ? 0 : 1); }
ABD_D int side_begin(int kind, int s) { return s == 0 ? 0 : (kind == KIND_VF ? 1 : 2); }
ABD_D int side_count(int kind, int s) { return kind == KIND_VF ? (s == 0 ? 1 : 3) : 2; }

struct Closest {
  double d2;
  int region;
  double gamma[4];
};

ABD_D Closest closest(int kind, const V3* z) {
  Closest c;
  if (kind == KIND_VF) {
    PTResult r = pt_closest(z[0], z[1], z[2], z[3]);
    c.d2 = r.d2;
    c.region = r.region;
    c.gamma[0] = 1.0;
    c.gamma[1] = -r.b0;
    c.gamma[2] = -r.b1;
    c.gamma[3] = -r.b2;
  } else {
    EEResult r = ee_closest(z[0], z[1], z[2], z[3]);
    c.d2 = r.d2;
    c.region = r.region;
    c.gamma[0] = 1.0 - r.s;
    c.gamma[1] = r.s;
    c.gamma[2] = -(1.0 - r.t);
    c.gamma[3] = -r.t;
  }
  return c;
}

ABD_D double pair_d2(int kind, const V3* z) {
  return kind == KIND_VF ? pt_closest(z[0], z[1], z[2], z[3]).d2 : ee_closest(z[0], z[1], z[2], z[3]).d2;
}

// dgamma/dw tables (distance.py:252-270): D[i][m] for point i, free slot m
ABD_D void region_dirs(int kind, int region, double D[4][2]) {
  for (int i = 0; i < 4; ++i) D[i][0] = D[i][1] = 0.0;
  if (kind == KIND_VF) {
    if (region == 3 || region == 6) { D[1][0] = 1.0; D[2][0] = -1.0; }
    if (region == 4) { D[2][0] = 1.0; D[3][0] = -1.0; }
    if (region == 5) { D[1][0] = -1.0; D[3][0] = 1.0; }
    if (region == 6) { D[1][1] = 1.0; D[3][1] = -1.0; }
  } else {
    int fa = region / 3, fb = region % 3;
    int col = 0;
    if (fa == 2) { D[0][0] = -1.0; D[1][0] = 1.0; col = 1; }
    if (fb == 2) { D[2][col] = 1.0; D[3][col] = -1.0; }
  }
}

// d^2, grad (12) and Hessian (12x12, row-major) in stacked point coordinates
ABD_D void d2_derivatives(int kind, const V3* z, const Closest& c, double* g, double* H) {
  const double* gam = c.gamma;
  V3 r = gam[0] * z[0];
  r = r + gam[1] * z[1];
  r = r + gam[2] * z[2];
  r = r + gam[3] * z[3];
  for (int i = 0; i < 4; ++i) {
    g[3 * i + 0] = 2.0 * gam[i] * r.x;
    g[3 * i + 1] = 2.0 * gam[i] * r.y;
    g[3 * i + 2] = 2.0 * gam[i] * r.z;
  }
  double D[4][2];
  region_dirs(kind, c.region, D);
  V3 S[2];
  bool used[2];
  for (int m = 0; m < 2; ++m) {
    S[m] = D[0][m] * z[0] + D[1][m] * z[1] + D[2][m] * z[2] + D[3][m] * z[3];
    used[m] = (D[0][m] != 0.0) || (D[1][m] != 0.0) || (D[2][m] != 0.0) || (D[3][m] != 0.0);
  }
  double f00 = 2.0 * dot(S[0], S[0]) + (used[0] ? 0.0 : 1.0);
  double f11 = 2.0 * dot(S[1], S[1]) + (used[1] ? 0.0 : 1.0);
  double f01 = 2.0 * dot(S[0], S[1]);
  double det = f00 * f11 - f01 * f01;
  double i00 = f11 / det, i11 = f00 / det, i01 = -f01 / det;
  double F[12][2];
  for (int i = 0; i < 4; ++i)
    for (int k = 0; k < 3; ++k)
      for (int m = 0; m < 2; ++m) F[3 * i + k][m] = 2.0 * (D[i][m] * comp(r, k) + gam[i] * comp(S[m], k));
  for (int a = 0; a < 12; ++a) {
    double u0 = i00 * F[a][0] + i01 * F[a][1];
    double u1 = i01 * F[a][0] + i11 * F[a][1];
    for (int b = a; b < 12; ++b) {
      double fzz = ((a % 3) == (b % 3)) ? 2.0 * gam[a / 3] * gam[b / 3] : 0.0;
      double h = fzz - (u0 * F[b][0] + u1 * F[b][1]);
      H[a * 12 + b] = h;
      H[b * 12 + a] = h;
    }
  }
}

// near-parallel EE mollifier value (distance.py:207-225), numpy order for c
ABD_D double mollifier_value(const V3* z, double eps) {
  V3 u = xsub3(z[1], z[0]), v = xsub3(z[3], z[2]);
  V3 cr = xcross(u, v);
  double c = xdot(cr, cr);
  double ratio = eps > 0.0 ? c / eps : 1.0;
  return ratio >= 1.0 ? 1.0 : ratio * (2.0 - ratio);
}

// value, grad (12), Hessian (12x12) of the mollifier; returns false when the
// mollifier is inactive (value 1, zero derivatives) so callers can skip work
ABD_D bool mollifier_derivs(const V3* z, double eps, double& val, double* g, double* H) {
  V3 u = z[1] - z[0], v = z[3] - z[2];
  V3 cr = cross(u, v);
  double c = dot(cr, cr);
  double ratio = eps > 0.0 ? c / eps : 1.0;
  if (!(ratio < 1.0)) {
    val = 1.0;
    return false;
  }
  val = ratio * (2.0 - ratio);
  double e1 = 2.0 / eps * (1.0 - ratio);
  double e2 = -2.0 / (eps * eps);
  double uu = dot(u, u), vv = dot(v, v), uv = dot(u, v);
  V3 cu = 2.0 * (vv * u - uv * v);
  V3 cv = 2.0 * (uu * v - uv * u);
  double gc[12];
  for (int k = 0; k < 3; ++k) {
    gc[k] = -comp(cu, k);
    gc[3 + k] = comp(cu, k);
    gc[6 + k] = -comp(cv, k);
    gc[9 + k] = comp(cv, k);
  }
  // second derivatives of c wrt (u, v)
  double huu[3][3], hvv[3][3], huv[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double dij = (i == j) ? 1.0 : 0.0;
      huu[i][j] = 2.0 * (vv * dij - comp(v, i) * comp(v, j));
      hvv[i][j] = 2.0 * (uu * dij - comp(u, i) * comp(u, j));
      huv[i][j] = 4.0 * comp(u, i) * comp(v, j) - 2.0 * comp(v, i) * comp(u, j) - 2.0 * uv * dij;
    }
  const double sg[4] = {-1.0, 1.0, -1.0, 1.0};
  for (int a = 0; a < 12; ++a) {
    g[a] = e1 * gc[a];
    int pa = a / 3, ia = a % 3;
    for (int b = 0; b < 12; ++b) {
      int pb = b / 3, ib = b % 3;
      double blk;
      if (pa < 2 && pb < 2) blk = huu[ia][ib];
      else if (pa >= 2 && pb >= 2) blk = hvv[ia][ib];
      else if (pa < 2) blk = huv[ia][ib];
      else blk = huv[ib][ia];
      H[a * 12 + b] = e2 * gc[a] * gc[b] + e1 * sg[pa] * sg[pb] * blk;
    }
  }
  return true;
}

// Barrier (x kappa) chain rule into point space.  Returns value; fills g12,
// H12.  contact.py:512-537.
ABD_D double contact_point_terms(int kind, const V3* z, const Closest& c, double eps, double kappa,
                                 double dh, double* g, double* H, double* tmp_g, double* tmp_H) {
  d2_derivatives(kind, z, c, tmp_g, tmp_H);  // grad/hess of d^2
  Barrier b = barrier_terms(c.d2, dh);
  double b0 = kappa * b.b0, b1 = kappa * b.b1, b2 = kappa * b.b2;
  for (int a = 0; a < 12; ++a) {
    g[a] = b1 * tmp_g[a];
    for (int bb = 0; bb < 12; ++bb) H[a * 12 + bb] = b2 * tmp_g[a] * tmp_g[bb] + b1 * tmp_H[a * 12 + bb];
  }
  if (kind == KIND_VF) return b0;
  double mv;
  // reuse tmp buffers for mollifier derivatives
  bool on = mollifier_derivs(z, eps, mv, tmp_g, tmp_H);
  if (!on) return b0;  // m = 1, zero derivatives: H, g unchanged
  // H = mh*b0 + mg bg^T + bg mg^T + m * Hb ; g = mg*b0 + m*bg
  for (int a = 0; a < 12; ++a) {
    for (int bb = 0; bb < 12; ++bb)
      H[a * 12 + bb] = tmp_H[a * 12 + bb] * b0 + tmp_g[a] * g[bb] + g[a] * tmp_g[bb] + mv * H[a * 12 + bb];
  }
  for (int a = 0; a < 12; ++a) g[a] = tmp_g[a] * b0 + mv * g[a];
  return mv * b0;
}

// ---------------------------------------------------------------------------
// Orthonormal basis of one side's Jacobian row space.  Point k contributes
// w_k = (1, xbar_k) in the (j = 0: p_a, j = 1+c: A[a][c]) ordering, so for
// side s:  W_s (4 x n_s) = Q_s R_s  with Q_s orthonormal (CGS2).
struct SideBasis {
  double Q[3][4];  // Q[i][j]: column i, entry j
  double R[3][3];  // upper triangular R[i][k]
  int n;
};

ABD_D void side_basis(const V3* xb, int n, SideBasis& B) {
  B.n = n;
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) B.R[i][k] = 0.0;
  for (int k = 0; k < n; ++k) {
    double v[4] = {1.0, xb[k].x, xb[k].y, xb[k].z};
    double n0 = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3]);
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < k; ++i) {
        double c = B.Q[i][0] * v[0] + B.Q[i][1] * v[1] + B.Q[i][2] * v[2] + B.Q[i][3] * v[3];
        B.R[i][k] += c;
        for (int j = 0; j < 4; ++j) v[j] -= c * B.Q[i][j];
      }
    double nr = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3]);
    if (nr > 1e-14 * n0) {
      B.R[k][k] = nr;
      for (int j = 0; j < 4; ++j) B.Q[k][j] = v[j] / nr;
    } else {
      B.R[k][k] = 0.0;
      for (int j = 0; j < 4; ++j) B.Q[k][j] = 0.0;
    }
  }
}

// affine column of side-local (a, j): j = 0 -> a, j = 1 + c -> 3 + 3a + c
ABD_D int aff_col(int a, int j) { return j == 0 ? a : 3 + 3 * a + (j - 1); }

// Map point-space g12/H12 to the two bodies' 24 affine coordinates with the
// PSD projection and kinematic rule of contact.py:619-675:
//   M = R H R^T (12x12, mode space), P = proj(M) (dynamic sides only),
//   H24 = Q P Q^T, g24 = J^T g.
// Outputs: g24[24]; blocks haa/hbb/hab (12x12 row-major, hab = rows of a, cols of b).
ABD_D void map_to_bodies(int kind, const V3* xb, const double* g12, const double* H12, bool dyn_a,
                         bool dyn_b, bool project, double* M, double* V, double* g24, double* haa,
                         double* hbb, double* hab) {
  SideBasis SB[2];
  side_basis(xb + side_begin(kind, 0), side_count(kind, 0), SB[0]);
  side_basis(xb + side_begin(kind, 1), side_count(kind, 1), SB[1]);
  // gradient: g24[(s, a, j)] = sum_{k in s} w_k[j] g_k[a]
  for (int s = 0; s < 2; ++s) {
    bool dyn = s == 0 ? dyn_a : dyn_b;
    int k0 = side_begin(kind, s), nk = side_count(kind, s);
    for (int a = 0; a < 3; ++a)
      for (int j = 0; j < 4; ++j) {
        double acc = 0.0;
        if (dyn)
          for (int k = 0; k < nk; ++k) {
            double w = j == 0 ? 1.0 : comp(xb[k0 + k], j - 1);
            acc += w * g12[3 * (k0 + k) + a];
          }
        g24[12 * s + aff_col(a, j)] = acc;
      }
  }
  // M = R H R^T in mode ordering (3*mode + axis), zero for kinematic sides
  for (int ra = 0; ra < 12; ++ra) {
    int pa = ra / 3, ax = ra % 3, sa = side_of(kind, pa), ia = pa - side_begin(kind, sa);
    bool da = sa == 0 ? dyn_a : dyn_b;
    for (int rb = ra; rb < 12; ++rb) {
      int pb = rb / 3, bx = rb % 3, sb = side_of(kind, pb), ib = pb - side_begin(kind, sb);
      bool db = sb == 0 ? dyn_a : dyn_b;
      double acc = 0.0;
      if (da && db) {
        int ka0 = side_begin(kind, sa), kb0 = side_begin(kind, sb);
        for (int k = ia; k < SB[sa].n; ++k) {
          double rk = SB[sa].R[ia][k];
          if (rk == 0.0) continue;
          double inner = 0.0;
          for (int m = ib; m < SB[sb].n; ++m) inner += H12[(3 * (ka0 + k) + ax) * 12 + 3 * (kb0 + m) + bx] * SB[sb].R[ib][m];
          acc += rk * inner;
        }
      }
      M[ra * 12 + rb] = acc;
      M[rb * 12 + ra] = acc;
    }
  }
  if (project && dyn_a && dyn_b) {
    psd_project_jacobi<12>(M, V, 12);
  } else if (project && (dyn_a || dyn_b)) {
    // project only the dynamic side's sub-block (its rows are contiguous)
    int s = dyn_a ? 0 : 1;
    int off = 3 * side_begin(kind, s), nn = 3 * side_count(kind, s);
    double* sub = M + off * 12 + off;  // leading dimension 12
    psd_project_jacobi<12>(sub, V, nn);
  }
  // H24 blocks = Q P Q^T
  for (int s = 0; s < 2; ++s)
    for (int t = s; t < 2; ++t) {
      double* out = (s == 0 && t == 0) ? haa : ((s == 1 && t == 1) ? hbb : hab);
      int ms0 = side_begin(kind, s), mt0 = side_begin(kind, t);
      const SideBasis& A = SB[s];
      const SideBasis& Bb = SB[t];
      for (int a = 0; a < 3; ++a)
        for (int j = 0; j < 4; ++j) {
          int row = aff_col(a, j);
          for (int b = 0; b < 3; ++b)
            for (int l = 0; l < 4; ++l) {
              int col = aff_col(b, l);
              if (s == t && col < row) continue;
              double acc = 0.0;
              for (int i = 0; i < A.n; ++i) {
                double qi = A.Q[i][j];
                if (qi == 0.0) continue;
                double inner = 0.0;
                for (int m = 0; m < Bb.n; ++m) inner += M[(3 * (ms0 + i) + a) * 12 + 3 * (mt0 + m) + b] * Bb.Q[m][l];
                acc += qi * inner;
              }
              out[row * 12 + col] = acc;
              if (s == t) out[col * 12 + row] = acc;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// lagged friction: compact tangent map tmap[m][(s,a,j)] = T[a][m] * c_s[j],
// c_s = sum_{k in s} gamma_k w_k  (contact.py:766-769 restated)
struct FrictionPair {
  double T[3][2];
  double c[2][4];
  double off[2];
  double lam;
};

ABD_D double tmap_entry(const FrictionPair& f, int m, int col24) {
  int s = col24 / 12, r = col24 % 12;
  int a, j;
  if (r < 3) { a = r; j = 0; } else { a = (r - 3) / 3; j = 1 + (r - 3) % 3; }
  return f.T[a][m] * f.c[s][j];
}

// u = tmap . (q_a, q_b) - offset
ABD_D void friction_u(const FrictionPair& f, const double* qa, const double* qb, double u[2]) {
  for (int m = 0; m < 2; ++m) {
    double acc = 0.0;
    for (int col = 0; col < 24; ++col) acc += tmap_entry(f, m, col) * (col < 12 ? qa[col] : qb[col - 12]);
    u[m] = acc - f.off[m];
  }
}

struct F0Terms {
  double f0, f1y, f1p;
};

ABD_D F0Terms f0_terms(double y, double eh) {
  F0Terms t;
  if (y < eh) {
    t.f0 = y * y * (1.0 - y / (3.0 * eh)) / eh + eh / 3.0;
    t.f1y = 2.0 / eh - y / (eh * eh);
    t.f1p = 2.0 / eh - 2.0 * y / (eh * eh);
  } else {
    t.f0 = y;
    t.f1y = 1.0 / (y == 0.0 ? 1.0 : y);
    t.f1p = 0.0;
  }
  return t;
}

}  // namespace abd
