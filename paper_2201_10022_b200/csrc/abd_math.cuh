// Device math for the ABD Newton step (fp64, sm_100a).
//
// Two kinds of arithmetic live here:
//  * "exact-order" helpers (x*) that reproduce numpy's operation order and
//    rounding bit-for-bit (no FMA contraction: __dadd_rn/__dmul_rn are never
//    fused by ptxas).  Used wherever a value feeds a discrete decision that
//    must match the reference: world positions, closest-point
//    region cascades, the d^2 < d_hat^2 activity filter, ACCD.
//  * ordinary fp64 (FMA allowed) for derivative algebra, where parity is
//    the 1e-9 relative bar of the north star.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define ABD_HD __host__ __device__ __forceinline__
#define ABD_D __device__ __forceinline__

namespace abd {

// fast reciprocal / reciprocal square root for the small eigen-solvers (not on
// the bit-exact paths): MUFU seed + Newton steps, no libdevice slow-path call
// (whose register saves spill the callers' register-resident matrices)
ABD_D double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
ABD_D double rsqrt_fast(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-0.5 * x, r * r, 1.5);
  return r * fma(-0.5 * x, r * r, 1.5);
}

ABD_D double xadd(double a, double b) { return __dadd_rn(a, b); }
ABD_D double xsub(double a, double b) { return __dsub_rn(a, b); }
ABD_D double xmul(double a, double b) { return __dmul_rn(a, b); }

struct V3 {
  double x, y, z;
};

ABD_D V3 v3(double x, double y, double z) { return V3{x, y, z}; }
ABD_D V3 ld3(const double* p) { return V3{p[0], p[1], p[2]}; }
ABD_D void st3(double* p, V3 a) { p[0] = a.x; p[1] = a.y; p[2] = a.z; }
ABD_D V3 xsub3(V3 a, V3 b) { return V3{xsub(a.x, b.x), xsub(a.y, b.y), xsub(a.z, b.z)}; }
ABD_D V3 xadd3(V3 a, V3 b) { return V3{xadd(a.x, b.x), xadd(a.y, b.y), xadd(a.z, b.z)}; }
ABD_D V3 xscale(double s, V3 a) { return V3{xmul(s, a.x), xmul(s, a.y), xmul(s, a.z)}; }
// numpy einsum("...i,...i->...") over 3 terms on x86 SIMD: (x0*y0 + x2*y2) + x1*y1
ABD_D double xdot(V3 a, V3 b) {
  return xadd(xadd(xmul(a.x, b.x), xmul(a.z, b.z)), xmul(a.y, b.y));
}
// np.linalg.norm(axis=-1) of a 3-vector: sqrt((x0^2 + x1^2) + x2^2)
ABD_D double xnorm_seq(V3 a) {
  return sqrt(xadd(xadd(xmul(a.x, a.x), xmul(a.y, a.y)), xmul(a.z, a.z)));
}
// np.cross
ABD_D V3 xcross(V3 a, V3 b) {
  return V3{xsub(xmul(a.y, b.z), xmul(a.z, b.y)), xsub(xmul(a.z, b.x), xmul(a.x, b.z)),
            xsub(xmul(a.x, b.y), xmul(a.y, b.x))};
}

// plain (contractible) helpers for derivative algebra
ABD_D V3 operator+(V3 a, V3 b) { return V3{a.x + b.x, a.y + b.y, a.z + b.z}; }
ABD_D V3 operator-(V3 a, V3 b) { return V3{a.x - b.x, a.y - b.y, a.z - b.z}; }
ABD_D V3 operator*(double s, V3 a) { return V3{s * a.x, s * a.y, s * a.z}; }
ABD_D double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
ABD_D V3 cross(V3 a, V3 b) {
  return V3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
ABD_D double comp(V3 a, int i) { return i == 0 ? a.x : (i == 1 ? a.y : a.z); }

// World position of rest point xb under q = (p, A row-major), reproducing
// numpy's `rest @ A.T + p` bit-for-bit (OpenBLAS dgemm FMA chain, then a
// separate add, verified on 300k values).
ABD_D V3 world_pos(const double* q, V3 xb) {
  V3 r;
  r.x = xadd(fma(xb.z, q[5], fma(xb.y, q[4], xmul(xb.x, q[3]))), q[0]);
  r.y = xadd(fma(xb.z, q[8], fma(xb.y, q[7], xmul(xb.x, q[6]))), q[1]);
  r.z = xadd(fma(xb.z, q[11], fma(xb.y, q[10], xmul(xb.x, q[9]))), q[2]);
  return r;
}

// ---------------------------------------------------------------------------
// point-triangle closest point (reference distance.py:86-150), numpy order
struct PTResult {
  double d2;
  int region;  // 0,1,2 vertex; 3 edge01; 4 edge12; 5 edge20; 6 interior
  double b0, b1, b2;
};

ABD_D PTResult pt_closest(V3 p, V3 t0, V3 t1, V3 t2) {
  V3 ab = xsub3(t1, t0), ac = xsub3(t2, t0), ap = xsub3(p, t0);
  double d1 = xdot(ab, ap), d2 = xdot(ac, ap);
  V3 bp = xsub3(p, t1);
  double d3 = xdot(ab, bp), d4 = xdot(ac, bp);
  V3 cp = xsub3(p, t2);
  double d5 = xdot(ab, cp), d6 = xdot(ac, cp);
  double vc = xsub(xmul(d1, d4), xmul(d3, d2));
  double vb = xsub(xmul(d5, d2), xmul(d1, d6));
  double va = xsub(xmul(d3, d6), xmul(d5, d4));
  PTResult r;
  if (d1 <= 0.0 && d2 <= 0.0) {
    r.region = 0; r.b0 = 1.0; r.b1 = 0.0; r.b2 = 0.0;
  } else if (d3 >= 0.0 && d4 <= d3) {
    r.region = 1; r.b0 = 0.0; r.b1 = 1.0; r.b2 = 0.0;
  } else if (d6 >= 0.0 && d5 <= d6) {
    r.region = 2; r.b0 = 0.0; r.b1 = 0.0; r.b2 = 1.0;
  } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double v = (d1 != d3) ? d1 / xsub(d1, d3) : 0.0;
    r.region = 3; r.b0 = xsub(1.0, v); r.b1 = v; r.b2 = 0.0;
  } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double w = (d2 != d6) ? d2 / xsub(d2, d6) : 0.0;
    r.region = 5; r.b0 = xsub(1.0, w); r.b1 = 0.0; r.b2 = w;
  } else if (va <= 0.0 && xsub(d4, d3) >= 0.0 && xsub(d5, d6) >= 0.0) {
    double num = xsub(d4, d3);
    double den = xadd(num, xsub(d5, d6));
    double w = (den != 0.0) ? num / den : 0.0;
    r.region = 4; r.b0 = 0.0; r.b1 = xsub(1.0, w); r.b2 = w;
  } else {
    double tot = xadd(xadd(va, vb), vc);
    double v = (tot != 0.0) ? vb / tot : 0.0;
    double w = (tot != 0.0) ? vc / tot : 0.0;
    r.region = 6; r.b0 = xsub(xsub(1.0, v), w); r.b1 = v; r.b2 = w;
  }
  V3 c;
  c.x = xadd(xadd(xmul(r.b0, t0.x), xmul(r.b1, t1.x)), xmul(r.b2, t2.x));
  c.y = xadd(xadd(xmul(r.b0, t0.y), xmul(r.b1, t1.y)), xmul(r.b2, t2.y));
  c.z = xadd(xadd(xmul(r.b0, t0.z), xmul(r.b1, t1.z)), xmul(r.b2, t2.z));
  V3 d = xsub3(p, c);
  r.d2 = xdot(d, d);
  return r;
}

// ---------------------------------------------------------------------------
// segment-segment closest points (reference distance.py:167-204)
struct EEResult {
  double d2;
  int region;  // 3*feat_a + feat_b
  double s, t;
};

ABD_D double clip01(double x) { return fmin(fmax(x, 0.0), 1.0); }

ABD_D EEResult ee_closest(V3 a0, V3 a1, V3 b0, V3 b1) {
  V3 da = xsub3(a1, a0), db = xsub3(b1, b0), r = xsub3(a0, b0);
  double a = xdot(da, da), e = xdot(db, db), f = xdot(db, r), c = xdot(da, r), b = xdot(da, db);
  double denom = xsub(xmul(a, e), xmul(b, b));
  bool parallel = denom <= xmul(xmul(1e-12, a), e);
  double s;
  if (parallel) {
    s = 0.0;
  } else {
    s = clip01(xsub(xmul(b, f), xmul(c, e)) / (denom == 0.0 ? 1.0 : denom));
  }
  double t = xadd(xmul(b, s), f) / e;
  bool tlo = t <= 0.0, thi = t >= 1.0;
  t = clip01(t);
  if (tlo) s = clip01(-c / a);
  if (thi) s = clip01(xsub(b, c) / a);
  int fa = s <= 0.0 ? 0 : (s >= 1.0 ? 1 : 2);
  int fb = t <= 0.0 ? 0 : (t >= 1.0 ? 1 : 2);
  V3 pa = xadd3(a0, xscale(s, da));
  V3 pb = xadd3(b0, xscale(t, db));
  V3 d = xsub3(pa, pb);
  EEResult res;
  res.d2 = xdot(d, d);
  res.region = 3 * fa + fb;
  res.s = s;
  res.t = t;
  return res;
}

// ---------------------------------------------------------------------------
// clamped log barrier in s = d^2 (reference contact.py:87-121)
struct Barrier {
  double b0, b1, b2;
};

ABD_D Barrier barrier_terms(double s, double dh) {
  Barrier r{0.0, 0.0, 0.0};
  double d = sqrt(s);
  if (!(d < dh)) return r;
  double lg = log(d / dh);
  double g = d - dh;
  double bd = -2.0 * g * lg - g * g / d;
  double bdd = -2.0 * lg - 4.0 * g / d + (g * g) / (d * d);
  r.b0 = -(g * g) * lg;
  r.b1 = bd / (2.0 * d);
  r.b2 = bdd / (4.0 * s) - bd / (4.0 * s * d);
  return r;
}

// ---------------------------------------------------------------------------
// Symmetric eigen-clamp (PSD projection) by cyclic Jacobi.  `a` is n x n
// row-major with leading dimension LD, overwritten by V max(w,0) V^T.
// Work array v (LD*LD).  Converges to |a_pq| negligible against ||A||_F.
template <int LD>
ABD_D void psd_project_jacobi(double* a, double* v, int n) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) v[i * LD + j] = (i == j) ? 1.0 : 0.0;
  // symmetrise
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      double s = 0.5 * (a[i * LD + j] + a[j * LD + i]);
      a[i * LD + j] = s;
      a[j * LD + i] = s;
    }
  double fro = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) fro += a[i * LD + j] * a[i * LD + j];
  if (fro == 0.0) return;
  const double tol = 1e-34 * fro;  // (1e-17 ||A||_F)^2 on the off-diagonal mass
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) off += a[i * LD + j] * a[i * LD + j];
    if (off <= tol) break;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        double apq = a[p * LD + q];
        if (apq * apq <= 1e-40 * fro) {  // negligible: skip (keeps sweeps cheap)
          a[p * LD + q] = 0.0;
          a[q * LD + p] = 0.0;
          continue;
        }
        double app = a[p * LD + p], aqq = a[q * LD + q];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(t * t + 1.0);
        double s = t * c;
        double tau = s / (1.0 + c);
        a[p * LD + p] = app - t * apq;
        a[q * LD + q] = aqq + t * apq;
        a[p * LD + q] = 0.0;
        a[q * LD + p] = 0.0;
        for (int r = 0; r < n; ++r) {
          if (r == p || r == q) continue;
          double g = a[r * LD + p], h = a[r * LD + q];
          double np_ = g - s * (h + g * tau);
          double nq_ = h + s * (g - h * tau);
          a[r * LD + p] = np_;
          a[p * LD + r] = np_;
          a[r * LD + q] = nq_;
          a[q * LD + r] = nq_;
        }
        for (int r = 0; r < n; ++r) {
          double g = v[r * LD + p], h = v[r * LD + q];
          v[r * LD + p] = g - s * (h + g * tau);
          v[r * LD + q] = h + s * (g - h * tau);
        }
      }
    }
  }
  // reconstruct with clamped eigenvalues
  double w[LD];
  for (int i = 0; i < n; ++i) w[i] = fmax(a[i * LD + i], 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = i; j < n; ++j) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc += v[i * LD + k] * w[k] * v[j * LD + k];
      a[i * LD + j] = acc;
      a[j * LD + i] = acc;
    }
}

// 2x2 symmetric PSD projection in closed form
ABD_D void psd_project_2x2(double& a, double& b, double& d) {
  // [[a b][b d]]
  double tr = 0.5 * (a + d);
  double df = 0.5 * (a - d);
  double rad = sqrt(df * df + b * b);
  double l1 = tr + rad, l2 = tr - rad;
  if (l2 >= 0.0) return;
  if (l1 <= 0.0) {
    a = b = d = 0.0;
    return;
  }
  // eigenvector of l1
  double vx, vy;
  if (df >= 0.0) {
    vx = df + rad;
    vy = b;
  } else {
    vx = b;
    vy = rad - df;
  }
  double nn = vx * vx + vy * vy;
  if (nn == 0.0) {
    vx = 1.0;
    vy = 0.0;
    nn = 1.0;
  }
  double s = l1 / nn;
  a = s * vx * vx;
  b = s * vx * vy;
  d = s * vy * vy;
}

}  // namespace abd
