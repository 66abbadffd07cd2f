// K3 per-pair contact block, low-rank form (no 12x12 / 24x24 materialisation).
//
// The reference forms H12 (point space, contact.py:512-537), H24 = J^T H12 J
// (contact.py:668-670) and eigen-clamps the 24x24 (contact.py:619-643).
// Here, exactly in exact arithmetic (SURVEY §7 hard part 1):
//   * H12 = B C B^T with a small basis B:
//       unmollified pairs: B = [gamma(x)I3 | F_0 | F_1] (3 + #free-slot columns),
//         C = blockdiag(4 b2 r r^T + 2 b1 I3, -b1 W), W = f_ww^-1;
//       mollified EE pairs: B = [G | P_u | P_v] (9 columns, Kronecker form),
//         C = m C_bH + mollifier terms.
//   * J^T B is (side, j) (x) axis structured: J^T G = c (x) I3 with
//     c_s[j] = sum_{k in s} gamma_k w_k[j], w_k = (1, xbar_k).
//   * proj(J^T B C B^T J) = Q proj(R C R^T) Q^T with J^T B = Q R (thin QR),
//     so the eigen-clamp is 5x5 (or 9x9), not 24x24.
//   * a kinematic side is handled by zeroing its rows of J^T B first: the
//     projection then acts on the dynamic sub-block only (contact.py:631-642).
// 24-vector layout inside this file: idx = (4 s + j) * 3 + a ("sja");
// outputs are written in the reference's affine order (12 s + aff_col(a, j)).
#pragma once
#include "abd_pair.cuh"

namespace abd {

// cyclic Jacobi on a compile-time N x N symmetric matrix held in registers;
// overwrites a with V max(w, 0) V^T (clamp = true) or leaves a diagonalised
template <int N>
ABD_D void jacobi_psd_reg(double (&a)[N][N]) {
  double v[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) v[i][j] = (i == j) ? 1.0 : 0.0;
  double fro = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) fro += a[i][j] * a[i][j];
  if (fro == 0.0) return;
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int j = i + 1; j < N; ++j) off += a[i][j] * a[i][j];
    if (off <= 1e-32 * fro) break;
#pragma unroll
    for (int p = 0; p < N - 1; ++p) {
#pragma unroll
      for (int q = p + 1; q < N; ++q) {
        double apq = a[p][q];
        if (apq * apq > 1e-40 * fro) {
          // rotation with MUFU-seeded reciprocals (no IEEE div/sqrt sequences)
          double theta = (a[q][q] - a[p][p]) * rcp_fast(2.0 * apq);
          const double th2 = theta * theta + 1.0;
          const double sq = th2 * rsqrt_fast(th2);  // sqrt(theta^2 + 1)
          double t = (theta >= 0.0 ? 1.0 : -1.0) * rcp_fast(fabs(theta) + sq);
          double c = rsqrt_fast(t * t + 1.0);
          double s = t * c;
          double tau = s * rcp_fast(1.0 + c);
          a[p][p] -= t * apq;
          a[q][q] += t * apq;
          a[p][q] = 0.0;
          a[q][p] = 0.0;
#pragma unroll
          for (int r = 0; r < N; ++r) {
            if (r == p || r == q) continue;
            double g = a[r][p], h = a[r][q];
            double np_ = g - s * (h + g * tau);
            double nq_ = h + s * (g - h * tau);
            a[r][p] = np_;
            a[p][r] = np_;
            a[r][q] = nq_;
            a[q][r] = nq_;
          }
#pragma unroll
          for (int r = 0; r < N; ++r) {
            double g = v[r][p], h = v[r][q];
            v[r][p] = g - s * (h + g * tau);
            v[r][q] = h + s * (g - h * tau);
          }
        } else {
          a[p][q] = 0.0;
          a[q][p] = 0.0;
        }
      }
    }
  }
  double w[N];
#pragma unroll
  for (int i = 0; i < N; ++i) w[i] = fmax(a[i][i], 0.0);
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = i; j < N; ++j) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) acc += v[i][k] * w[k] * v[j][k];
      a[i][j] = acc;
      a[j][i] = acc;
    }
}

ABD_D int out_col(int sj, int a) {  // sja -> reference affine column (12 s + aff_col)
  int s = sj >> 2, j = sj & 3;
  return 12 * s + (j == 0 ? a : 3 + 3 * a + (j - 1));
}

// write symmetric 24x24 entry (row, col in affine order) into haa/hbb/hab blocks
ABD_D void put_h(double* haa, double* hbb, double* hab, int r, int c, double v) {
  if (r < 12 && c < 12) {
    haa[r * 12 + c] = v;
  } else if (r >= 12 && c >= 12) {
    hbb[(r - 12) * 12 + (c - 12)] = v;
  } else if (r < 12) {
    hab[r * 12 + (c - 12)] = v;
  } else {
    hab[c * 12 + (r - 12)] = v;
  }
}

struct PairEval {
  double d2, value;
};

// Full per-pair evaluation.  out: g24 (24) | haa (144) | hbb (144) | hab (144).
// h12/g12 (optional, may be null): point-space derivatives for testing.
// COMPACT: `out` receives a compact pair record (abd_pblk.cuh: g24 | type |
// low-rank factors) instead of the dense g24 | H_aa | H_bb | H_ab blocks.
// MOLL: 0 = either path, 1 = caller guarantees an unmollified pair (the 9-column
// code is compiled out), 2 = caller guarantees a mollified EE pair.
template <bool COMPACT = false, int MOLL = 0>
ABD_D PairEval contact_pair_eval(int kind, const V3* z, const V3* xb, double eps, double kappa, double dh,
                                 bool dyn_a, bool dyn_b, bool project, double* out, double* g12o = nullptr,
                                 double* h12o = nullptr) {
  Closest cl = closest(kind, z);
  Barrier bt = barrier_terms(cl.d2, dh);
  const double b0 = kappa * bt.b0, b1 = kappa * bt.b1, b2 = kappa * bt.b2;
  const double* gam = cl.gamma;
  V3 r = gam[0] * z[0];
  r = r + gam[1] * z[1];
  r = r + gam[2] * z[2];
  r = r + gam[3] * z[3];
  double D[4][2];
  region_dirs(kind, cl.region, D);
  V3 S[2];
  bool used[2];
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    S[m] = D[0][m] * z[0] + D[1][m] * z[1] + D[2][m] * z[2] + D[3][m] * z[3];
    used[m] = (D[0][m] != 0.0) || (D[1][m] != 0.0) || (D[2][m] != 0.0) || (D[3][m] != 0.0);
  }
  double f00 = 2.0 * dot(S[0], S[0]) + (used[0] ? 0.0 : 1.0);
  double f11 = 2.0 * dot(S[1], S[1]) + (used[1] ? 0.0 : 1.0);
  double f01 = 2.0 * dot(S[0], S[1]);
  double det = f00 * f11 - f01 * f01;
  double W[2][2] = {{f11 / det, -f01 / det}, {-f01 / det, f00 / det}};
  // affine-side vectors (8 = side * 4 + j), zero on kinematic sides
  double cv[8], dv[2][8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    cv[q] = 0.0;
    dv[0][q] = 0.0;
    dv[1][q] = 0.0;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int s = side_of(kind, k);
    bool dyn = s == 0 ? dyn_a : dyn_b;
    if (!dyn) continue;
    double w[4] = {1.0, xb[k].x, xb[k].y, xb[k].z};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      cv[4 * s + j] += gam[k] * w[j];
      dv[0][4 * s + j] += D[k][0] * w[j];
      dv[1][4 * s + j] += D[k][1] * w[j];
    }
  }
  // mollifier (EE only)
  double mv = 1.0;
  bool moll = false;
  double e1 = 0.0, e2 = 0.0;
  V3 u{0, 0, 0}, vv3{0, 0, 0};
  if (kind == KIND_EE) {
    u = z[1] - z[0];
    vv3 = z[3] - z[2];
    V3 cr = cross(u, vv3);
    double cc = dot(cr, cr);
    double ratio = eps > 0.0 ? cc / eps : 1.0;
    if (ratio < 1.0) {
      moll = true;
      mv = ratio * (2.0 - ratio);
      e1 = 2.0 / eps * (1.0 - ratio);
      e2 = -2.0 / (eps * eps);
    }
  }
  double* g24 = out;
  double* haa = out + 24;
  double* hbb = out + 24 + 144;
  double* hab = out + 24 + 288;
  PairEval res;
  res.d2 = cl.d2;
  if (MOLL == 1 || (MOLL == 0 && !moll)) {
    res.value = b0;
    // ---------------- 5-column path ----------------
    // g24 = 2 b1 c (x) r
#pragma unroll
    for (int sj = 0; sj < 8; ++sj)
#pragma unroll
      for (int a = 0; a < 3; ++a) g24[out_col(sj, a)] = 2.0 * b1 * cv[sj] * comp(r, a);
    double nc = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) nc += cv[q] * cv[q];
    nc = sqrt(nc);
    double ch[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) ch[q] = cv[q] / nc;
    // explicit F columns in J-space, orthogonalised against ch (x) I3
    double fq[2][24];
    double Rm[5][5];
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
      for (int j = 0; j < 5; ++j) Rm[i][j] = 0.0;
    Rm[0][0] = Rm[1][1] = Rm[2][2] = nc;
#pragma unroll
    for (int m = 0; m < 2; ++m) {
#pragma unroll
      for (int sj = 0; sj < 8; ++sj)
#pragma unroll
        for (int a = 0; a < 3; ++a)
          fq[m][sj * 3 + a] = used[m] ? 2.0 * (dv[m][sj] * comp(r, a) + cv[sj] * comp(S[m], a)) : 0.0;
#pragma unroll
      for (int pass = 0; pass < 2; ++pass)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          double t = 0.0;
#pragma unroll
          for (int sj = 0; sj < 8; ++sj) t += ch[sj] * fq[m][sj * 3 + a];
          Rm[a][3 + m] += t;
#pragma unroll
          for (int sj = 0; sj < 8; ++sj) fq[m][sj * 3 + a] -= t * ch[sj];
        }
    }
    // Gram-Schmidt between the two F residuals
    double n0 = 0.0;
#pragma unroll
    for (int q = 0; q < 24; ++q) n0 += fq[0][q] * fq[0][q];
    n0 = sqrt(n0);
    if (n0 > 0.0) {
#pragma unroll
      for (int q = 0; q < 24; ++q) fq[0][q] /= n0;
    }
    Rm[3][3] = n0;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < 24; ++q) t += fq[0][q] * fq[1][q];
      Rm[3][4] += t;
#pragma unroll
      for (int q = 0; q < 24; ++q) fq[1][q] -= t * fq[0][q];
    }
    double n1 = 0.0;
#pragma unroll
    for (int q = 0; q < 24; ++q) n1 += fq[1][q] * fq[1][q];
    n1 = sqrt(n1);
    if (n1 > 0.0) {
#pragma unroll
      for (int q = 0; q < 24; ++q) fq[1][q] /= n1;
    }
    Rm[4][4] = n1;
    // C5
    double C[5][5];
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
      for (int j = 0; j < 5; ++j) C[i][j] = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) C[a][b] = 4.0 * b2 * comp(r, a) * comp(r, b) + (a == b ? 2.0 * b1 : 0.0);
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int l = 0; l < 2; ++l) C[3 + m][3 + l] = (used[m] && used[l]) ? -b1 * W[m][l] : 0.0;
    // M = R C R^T
    double M[5][5];
#pragma unroll
    for (int i = 0; i < 5; ++i)
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          double inner = 0.0;
#pragma unroll
          for (int l = 0; l < 5; ++l) inner += C[k][l] * Rm[j][l];
          acc += Rm[i][k] * inner;
        }
        M[i][j] = acc;
      }
    if (project) jacobi_psd_reg<5>(M);
    if (COMPACT) {
      out[24] = 0.0;  // type: 5-column (ch (x) I3 | fq0 | fq1)
#pragma unroll
      for (int q = 0; q < 8; ++q) out[25 + q] = ch[q];
#pragma unroll
      for (int q = 0; q < 24; ++q) {
        out[33 + q] = fq[0][q];
        out[57 + q] = fq[1][q];
      }
#pragma unroll
      for (int i = 0; i < 5; ++i)
#pragma unroll
        for (int j = 0; j < 5; ++j) out[81 + 5 * i + j] = M[i][j];
      return res;
    }
    // H24 = Q M Q^T with Q = [ch (x) e_0..2 | fq0 | fq1]
    // U[(sj,a)][beta] = ch[sj] M[a][beta] + fq0[sja] M[3][beta] + fq1[sja] M[4][beta]
#pragma unroll
    for (int sj = 0; sj < 8; ++sj)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        int rho = sj * 3 + a;
        double U[5];
#pragma unroll
        for (int be = 0; be < 5; ++be)
          U[be] = ch[sj] * M[a][be] + fq[0][rho] * M[3][be] + fq[1][rho] * M[4][be];
        int rc = out_col(sj, a);
#pragma unroll
        for (int tl = 0; tl < 8; ++tl)
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            int sg = tl * 3 + b;
            if (sg < rho) continue;
            double h = U[b] * ch[tl] + U[3] * fq[0][sg] + U[4] * fq[1][sg];
            int cc = out_col(tl, b);
            put_h(haa, hbb, hab, rc, cc, h);
            put_h(haa, hbb, hab, cc, rc, h);
          }
      }
    if (g12o) {
      // point-space: g12 = 2 b1 gamma (x) r ; H12 = [G|F] C [G|F]^T (unprojected C)
      double Fp[2][12];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int a = 0; a < 3; ++a) Fp[m][3 * k + a] = used[m] ? 2.0 * (D[k][m] * comp(r, a) + gam[k] * comp(S[m], a)) : 0.0;
      for (int i = 0; i < 12; ++i) {
        g12o[i] = 2.0 * b1 * gam[i / 3] * comp(r, i % 3);
        for (int j = 0; j < 12; ++j) {
          double h = gam[i / 3] * gam[j / 3] * C[i % 3][j % 3];
          for (int m = 0; m < 2; ++m)
            for (int l = 0; l < 2; ++l) h += Fp[m][i] * C[3 + m][3 + l] * Fp[l][j];
          h12o[i * 12 + j] = h;
        }
      }
    }
    return res;
  }
  // ---------------- 9-column (mollified EE) path ----------------
  res.value = mv * b0;
  // X (8 x 3): columns c, du = (w1 - w0 | 0), dv = (0 | w3 - w2), zero kinematic rows
  double X[8][3];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    X[q][0] = cv[q];
    X[q][1] = 0.0;
    X[q][2] = 0.0;
  }
  if (dyn_a) {
    X[0][1] = 0.0;
    X[1][1] = xb[1].x - xb[0].x;
    X[2][1] = xb[1].y - xb[0].y;
    X[3][1] = xb[1].z - xb[0].z;
  }
  if (dyn_b) {
    X[4][2] = 0.0;
    X[5][2] = xb[3].x - xb[2].x;
    X[6][2] = xb[3].y - xb[2].y;
    X[7][2] = xb[3].z - xb[2].z;
  }
  // coordinates in [G | P_u | P_v]: F_m -> (2 S_m | 2 r [DS] | -2 r [DT])
  double Ft[2][9];
#pragma unroll
  for (int m = 0; m < 2; ++m) {
    bool isDS = used[m] && D[0][m] == -1.0 && D[1][m] == 1.0;
    bool isDT = used[m] && !isDS;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      Ft[m][a] = used[m] ? 2.0 * comp(S[m], a) : 0.0;
      Ft[m][3 + a] = isDS ? 2.0 * comp(r, a) : 0.0;
      Ft[m][6 + a] = isDT ? -2.0 * comp(r, a) : 0.0;
    }
  }
  double C[9][9];
#pragma unroll
  for (int i = 0; i < 9; ++i)
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      double h = 0.0;
      if (i < 3 && j < 3) h = 4.0 * b2 * comp(r, i) * comp(r, j) + (i == j ? 2.0 * b1 : 0.0);
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int l = 0; l < 2; ++l)
          if (used[m] && used[l]) h -= b1 * Ft[m][i] * W[m][l] * Ft[l][j];
      C[i][j] = mv * h;
    }
  // mollifier terms: P-block b0 (e2 cc6 cc6^T + e1 Hc6); cross e1 cc6 r'^T with r' = 2 b1 r
  double uu = dot(u, u), vv = dot(vv3, vv3), uvd = dot(u, vv3);
  V3 cu = 2.0 * (vv * u - uvd * vv3);
  V3 cvv = 2.0 * (uu * vv3 - uvd * u);
  double c6[6] = {cu.x, cu.y, cu.z, cvv.x, cvv.y, cvv.z};
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 6; ++j) {
      int ia = i % 3, ib = j % 3;
      double dij = ia == ib ? 1.0 : 0.0;
      double h6;
      if (i < 3 && j < 3) h6 = 2.0 * (vv * dij - comp(vv3, ia) * comp(vv3, ib));
      else if (i >= 3 && j >= 3) h6 = 2.0 * (uu * dij - comp(u, ia) * comp(u, ib));
      else if (i < 3) h6 = 4.0 * comp(u, ia) * comp(vv3, ib) - 2.0 * comp(vv3, ia) * comp(u, ib) - 2.0 * uvd * dij;
      else h6 = 4.0 * comp(u, ib) * comp(vv3, ia) - 2.0 * comp(vv3, ib) * comp(u, ia) - 2.0 * uvd * dij;
      C[3 + i][3 + j] += b0 * (e2 * c6[i] * c6[j] + e1 * h6);
    }
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double t = e1 * c6[i] * 2.0 * b1 * comp(r, a);
      C[3 + i][a] += t;
      C[a][3 + i] += t;
    }
  // gradient: coords (m r' | b0 e1 c6)
  double gc[9];
#pragma unroll
  for (int a = 0; a < 3; ++a) gc[a] = mv * 2.0 * b1 * comp(r, a);
#pragma unroll
  for (int i = 0; i < 6; ++i) gc[3 + i] = b0 * e1 * c6[i];
#pragma unroll
  for (int sj = 0; sj < 8; ++sj)
#pragma unroll
    for (int a = 0; a < 3; ++a)
      g24[out_col(sj, a)] = X[sj][0] * gc[a] + X[sj][1] * gc[3 + a] + X[sj][2] * gc[6 + a];
  if (g12o) {
    // point-space basis vectors of [G | P_u | P_v]
    for (int i = 0; i < 12; ++i) {
      int k = i / 3, a = i % 3;
      double bu = (k == 1 ? 1.0 : (k == 0 ? -1.0 : 0.0)), bv = (k == 3 ? 1.0 : (k == 2 ? -1.0 : 0.0));
      g12o[i] = gam[k] * gc[a] + bu * gc[3 + a] + bv * gc[6 + a];
      for (int j = 0; j < 12; ++j) {
        int kk = j / 3, b = j % 3;
        double cu_ = (kk == 1 ? 1.0 : (kk == 0 ? -1.0 : 0.0)), cv_ = (kk == 3 ? 1.0 : (kk == 2 ? -1.0 : 0.0));
        double wi[3] = {gam[k], bu, bv}, wj[3] = {gam[kk], cu_, cv_};
        double h = 0.0;
        for (int be = 0; be < 3; ++be)
          for (int ga = 0; ga < 3; ++ga) h += wi[be] * C[3 * be + a][3 * ga + b] * wj[ga];
        h12o[i * 12 + j] = h;
      }
    }
  }
  // thin QR of X (CGS2): X = Qx Rx
  double Qx[8][3], Rx[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) Rx[i][j] = 0.0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double col[8];
    double n0 = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      col[q] = X[q][k];
      n0 += col[q] * col[q];
    }
#pragma unroll
    for (int pass = 0; pass < 2; ++pass)
#pragma unroll
      for (int i = 0; i < k; ++i) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += Qx[q][i] * col[q];
        Rx[i][k] += t;
#pragma unroll
        for (int q = 0; q < 8; ++q) col[q] -= t * Qx[q][i];
      }
    double nr = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) nr += col[q] * col[q];
    nr = sqrt(nr);
    bool ok = nr > 1e-14 * sqrt(n0) && nr > 0.0;
    Rx[k][k] = ok ? nr : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) Qx[q][k] = ok ? col[q] / nr : 0.0;
  }
  // M9 = (Rx (x) I) C (Rx (x) I)^T
  double M[9][9];
#pragma unroll
  for (int be = 0; be < 3; ++be)
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int ga = 0; ga < 3; ++ga)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          double acc = 0.0;
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            double inner = 0.0;
#pragma unroll
            for (int q = 0; q < 3; ++q) inner += C[3 * p + a][3 * q + b] * Rx[ga][q];
            acc += Rx[be][p] * inner;
          }
          M[3 * be + a][3 * ga + b] = acc;
        }
  if (project) jacobi_psd_reg<9>(M);
  if (COMPACT) {
    out[24] = 1.0;  // type: 9-column Kronecker (Qx (x) I3)
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
      for (int k = 0; k < 3; ++k) out[25 + 3 * q + k] = Qx[q][k];
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
      for (int j = 0; j < 9; ++j) out[49 + 9 * i + j] = M[i][j];
    return res;
  }
  // H24[(sj,a),(tl,b)] = sum_{be,ga} Qx[sj][be] M[(be,a),(ga,b)] Qx[tl][ga]
#pragma unroll 1
  for (int sj = 0; sj < 8; ++sj)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int rho = sj * 3 + a;
      double U[9];
#pragma unroll
      for (int cidx = 0; cidx < 9; ++cidx)
        U[cidx] = Qx[sj][0] * M[a][cidx] + Qx[sj][1] * M[3 + a][cidx] + Qx[sj][2] * M[6 + a][cidx];
      int rc = out_col(sj, a);
#pragma unroll
      for (int tl = 0; tl < 8; ++tl)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          int sg = tl * 3 + b;
          if (sg < rho) continue;
          double h = U[b] * Qx[tl][0] + U[3 + b] * Qx[tl][1] + U[6 + b] * Qx[tl][2];
          int cc = out_col(tl, b);
          put_h(haa, hbb, hab, rc, cc, h);
          put_h(haa, hbb, hab, cc, rc, h);
        }
    }
  return res;
}

}  // namespace abd
