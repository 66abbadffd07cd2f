// Exact inter-body intersection audit: the reference's
// post-hoc check that a state is intersection-free.
//
//   triangle-triangle SAT            intersect.py:18-42   (triangles_intersect_batch)
//   body-pair audit with box pruning scene.py:652-698      (_intersecting_body_pairs)
//   ray-parity containment           scene.py:627-649      (_point_in_closed_mesh)
//
// Arithmetic follows the reference's numpy forms term by term (np.cross as
// products then differences, einsum dots summed left to right, no FMA), so the
// boolean results agree with the reference's on the same inputs.
#include <algorithm>
#include <vector>

#include "kernels.h"

namespace abd {

namespace {

struct D3 {
  double x, y, z;
};

__device__ __forceinline__ D3 sub3(D3 a, D3 b) { return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)}; }
// np.cross: (a1 b2 - a2 b1, a2 b0 - a0 b2, a0 b1 - a1 b0)
__device__ __forceinline__ D3 cross3(D3 a, D3 b) {
  return {__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)), __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
          __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
// einsum over k of a 3-vector product, left to right
__device__ __forceinline__ double dot3(D3 a, D3 b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}

constexpr double AXIS_EPS = 1e-30;  // intersect.py _AXIS_EPS

// closed triangles a, b intersect (touching counts): separating axes = two face
// normals, nine edge-edge crosses, six in-plane edge normals (intersect.py:21-42)
__device__ bool tri_intersect(const D3* a, const D3* b) {
  const D3 ea[3] = {sub3(a[1], a[0]), sub3(a[2], a[1]), sub3(a[0], a[2])};
  const D3 eb[3] = {sub3(b[1], b[0]), sub3(b[2], b[1]), sub3(b[0], b[2])};
  const D3 na = cross3(ea[0], ea[1]);
  const D3 nb = cross3(eb[0], eb[1]);
  for (int k = 0; k < 17; ++k) {
    D3 ax;
    if (k == 0) ax = na;
    else if (k == 1) ax = nb;
    else if (k < 11) ax = cross3(ea[(k - 2) / 3], eb[(k - 2) % 3]);
    else if (k < 14) ax = cross3(ea[k - 11], na);
    else ax = cross3(eb[k - 14], nb);
    if (dot3(ax, ax) <= AXIS_EPS) continue;  // degenerate axis
    double a0 = dot3(ax, a[0]), a1 = dot3(ax, a[1]), a2 = dot3(ax, a[2]);
    double b0 = dot3(ax, b[0]), b1 = dot3(ax, b[1]), b2 = dot3(ax, b[2]);
    const double mina = fmin(fmin(a0, a1), a2), maxa = fmax(fmax(a0, a1), a2);
    const double minb = fmin(fmin(b0, b1), b2), maxb = fmax(fmax(b0, b1), b2);
    if (mina > maxb || minb > maxa) return false;
  }
  return true;
}

__device__ __forceinline__ D3 ld(const double* p) { return {p[0], p[1], p[2]}; }

}  // namespace

__global__ void k_tri_intersect(int64_t n, const double* __restrict__ ta, const double* __restrict__ tb,
                                unsigned char* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  D3 a[3], b[3];
  for (int k = 0; k < 3; ++k) {
    a[k] = ld(ta + 9 * i + 3 * k);
    b[k] = ld(tb + 9 * i + 3 * k);
  }
  out[i] = tri_intersect(a, b) ? 1 : 0;
}

void launch_tri_intersect(cudaStream_t st, int64_t n, const double* ta, const double* tb, unsigned char* out) {
  if (n <= 0) return;
  k_tri_intersect<<<grid_for(n, 128), 128, 0, st>>>(n, ta, tb, out);
  note_launch("k_tri_intersect");
}

// world vertex positions (the reference's rest @ A^T + p, F2 FMA chain)
__global__ void k_world_vertices(int64_t V, const int* __restrict__ vert_body, const double* __restrict__ rest,
                                 const double* __restrict__ q, double* out) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= V) return;
  const V3 x = world_pos(q + 12 * (int64_t)vert_body[v], ld3(rest + 3 * v));
  out[3 * v] = x.x;
  out[3 * v + 1] = x.y;
  out[3 * v + 2] = x.z;
}

// world vertices of every body at q (device) into out (device, V x 3)
void world_vertices(Scene& s, const double* q, double* out) {
  if (!s.V) return;
  k_world_vertices<<<grid_for(s.V, 256), 256, 0, s.stream>>>(s.V, s.vert_body.p, s.rest.p, q, out);
  note_launch("k_world_vertices");
}

// all body pairs i < j whose vertex boxes overlap (closed), scene.py:660-668; the
// audit is not on the stepping path, so the O(B^2) box loop of the reference is
// kept (one thread per row i, pairs appended in any order, sorted on the host)
__global__ void k_audit_box_pairs(int B, const double* __restrict__ box, int64_t cap, int2* out,
                                  unsigned long long* cnt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const double* a = box + 6 * i;
  for (int j = i + 1; j < B; ++j) {
    const double* b = box + 6 * j;
    const bool ov = fmax(a[0], b[0]) <= fmin(a[3], b[3]) && fmax(a[1], b[1]) <= fmin(a[4], b[4]) &&
                    fmax(a[2], b[2]) <= fmin(a[5], b[5]);
    if (ov) {
      const unsigned long long at = atomicAdd(cnt, 1ull);
      if ((int64_t)at < cap) out[at] = make_int2(i, j);
    }
  }
}

namespace {
// ray-parity containment of point p in the closed mesh of triangles [t0, t1) of a
// body (scene.py:627-649): fixed skewed direction, hits with |a| > 1e-14, the
// barycentric window and t > 1e-12 counted; odd count = inside
__device__ bool point_in_mesh(D3 p, const double* __restrict__ X, const int* __restrict__ tris, int t0, int t1) {
  const D3 d = {0.5424426421, 0.7866258632, 0.2954766431};
  int hits = 0;
  for (int t = t0; t < t1; ++t) {
    const D3 v0 = ld(X + 3 * (int64_t)tris[3 * t]), v1 = ld(X + 3 * (int64_t)tris[3 * t + 1]),
             v2 = ld(X + 3 * (int64_t)tris[3 * t + 2]);
    const D3 e1 = sub3(v1, v0), e2 = sub3(v2, v0);
    const D3 h = cross3(d, e2);
    const double a = dot3(e1, h);
    if (!(fabs(a) > 1e-14)) continue;
    const double f = __ddiv_rn(1.0, a);
    const D3 s = sub3(p, v0);
    const double u = __dmul_rn(f, dot3(s, h));
    const D3 qv = cross3(s, e1);
    const double v = __dmul_rn(f, dot3(qv, d));
    const double tt = __dmul_rn(f, dot3(e2, qv));
    if (u >= 0.0 && u <= 1.0 && v >= 0.0 && __dadd_rn(u, v) <= 1.0 && tt > 1e-12) ++hits;
  }
  return hits & 1;
}
}  // namespace

// one CTA per box-overlapping body pair (scene.py:671-698): triangles of both
// bodies culled to the overlap box, every surviving pair with overlapping
// triangle boxes tested by SAT; no crossing -> ray-parity containment both ways
__global__ void __launch_bounds__(256) k_audit_pairs(int64_t n, const int2* __restrict__ pairs,
                                                     const double* __restrict__ box, const double* __restrict__ X,
                                                     const int* __restrict__ t_off, const int* __restrict__ tris,
                                                     const int* __restrict__ v_off, unsigned char* hit) {
  __shared__ int found;
  for (int64_t p = blockIdx.x; p < n; p += gridDim.x) {
    const int bi = pairs[p].x, bj = pairs[p].y;
    double lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
      lo[k] = fmax(box[6 * bi + k], box[6 * bj + k]);
      hi[k] = fmin(box[6 * bi + 3 + k], box[6 * bj + 3 + k]);
    }
    if (threadIdx.x == 0) found = 0;
    __syncthreads();
    const int ta0 = t_off[bi], na = t_off[bi + 1] - ta0;
    const int tb0 = t_off[bj], nb = t_off[bj + 1] - tb0;
    // (a, b) index pairs striped over the CTA; both triangle boxes must meet the
    // overlap box and each other (the reference's keep_a / keep_b / hit masks)
    for (int64_t w = threadIdx.x; w < (int64_t)na * nb && !found; w += blockDim.x) {
      const int ia = ta0 + (int)(w / nb), ib = tb0 + (int)(w % nb);
      D3 A[3], Bt[3];
      double alo[3], ahi[3], blo[3], bhi[3];
      for (int k = 0; k < 3; ++k) {
        A[k] = ld(X + 3 * (int64_t)tris[3 * ia + k]);
        Bt[k] = ld(X + 3 * (int64_t)tris[3 * ib + k]);
      }
      alo[0] = fmin(fmin(A[0].x, A[1].x), A[2].x);
      alo[1] = fmin(fmin(A[0].y, A[1].y), A[2].y);
      alo[2] = fmin(fmin(A[0].z, A[1].z), A[2].z);
      ahi[0] = fmax(fmax(A[0].x, A[1].x), A[2].x);
      ahi[1] = fmax(fmax(A[0].y, A[1].y), A[2].y);
      ahi[2] = fmax(fmax(A[0].z, A[1].z), A[2].z);
      blo[0] = fmin(fmin(Bt[0].x, Bt[1].x), Bt[2].x);
      blo[1] = fmin(fmin(Bt[0].y, Bt[1].y), Bt[2].y);
      blo[2] = fmin(fmin(Bt[0].z, Bt[1].z), Bt[2].z);
      bhi[0] = fmax(fmax(Bt[0].x, Bt[1].x), Bt[2].x);
      bhi[1] = fmax(fmax(Bt[0].y, Bt[1].y), Bt[2].y);
      bhi[2] = fmax(fmax(Bt[0].z, Bt[1].z), Bt[2].z);
      bool keep = true;
      for (int k = 0; k < 3; ++k)
        keep = keep && alo[k] <= hi[k] && ahi[k] >= lo[k] && blo[k] <= hi[k] && bhi[k] >= lo[k] &&
               alo[k] <= bhi[k] && blo[k] <= ahi[k];
      if (keep && tri_intersect(A, Bt)) found = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      bool h = found != 0;
      if (!h) {
        const D3 pa = ld(X + 3 * (int64_t)v_off[bi]), pb = ld(X + 3 * (int64_t)v_off[bj]);
        h = point_in_mesh(pa, X, tris, tb0, tb0 + nb) || point_in_mesh(pb, X, tris, ta0, ta0 + na);
      }
      hit[p] = h ? 1 : 0;
    }
    __syncthreads();
  }
}

// scene-level audit: world vertices, body boxes (no inflation), box-overlapping pairs,
// per-pair exact test.  Returns the offending pairs (i < j) in canonical order.
std::vector<int2> intersecting_body_pairs(Scene& s, const double* q) {
  cudaStream_t st = s.stream;
  Scene::Work& w = s.w;
  std::vector<int2> res;
  if (s.B < 2) return res;
  DVec<double> X, box;
  X.resize(3 * std::max<int64_t>(s.V, 1));
  box.resize(6 * (size_t)s.B);
  if (s.V) {
    k_world_vertices<<<grid_for(s.V, 256), 256, 0, st>>>(s.V, s.vert_body.p, s.rest.p, q, X.p);
    note_launch("k_world_vertices");
  }
  launch_body_boxes(s, q, q, 0.0, box.p);
  unsigned long long* cnt = w.ull.p + 15;
  DVec<int2> pairs;
  int64_t cap = 4 * (int64_t)s.B + 1024;
  unsigned long long hn = 0;
  for (int attempt = 0; attempt < 3; ++attempt) {
    pairs.resize(cap);
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    k_audit_box_pairs<<<grid_for(s.B, 128), 128, 0, st>>>(s.B, box.p, cap, pairs.p, cnt);
    note_launch("k_audit_box_pairs");
    CK(cudaMemcpyAsync(&hn, cnt, sizeof(hn), cudaMemcpyDeviceToHost, st));
    SSYNC(st);
    if ((int64_t)hn <= cap) break;
    cap = (int64_t)hn;
  }
  const int64_t n = (int64_t)hn;
  if (n == 0) return res;
  DVec<unsigned char> hit;
  hit.resize(n);
  k_audit_pairs<<<(int)std::min<int64_t>(n, 16 * (int64_t)s.num_sms), 256, 0, st>>>(
      n, pairs.p, box.p, X.p, s.t_off.p, s.tris.p, s.v_off.p, hit.p);
  note_launch("k_audit_pairs");
  std::vector<int2> hp(n);
  std::vector<unsigned char> hh(n);
  pairs.download(hp.data(), n, st);
  hit.download(hh.data(), n, st);
  SSYNC(st);
  for (int64_t k = 0; k < n; ++k)
    if (hh[k]) res.push_back(hp[k]);
  std::sort(res.begin(), res.end(), [](int2 a, int2 b) { return a.x != b.x ? a.x < b.x : a.y < b.y; });
  return res;
}

}  // namespace abd
