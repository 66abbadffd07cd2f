// K2 broad phase (contact.py:338-412), exact-set restatement:
// every kind-compatible inter-body primitive pair, in body pairs with >= 1
// dynamic body, whose closed d_hat/2-inflated start/end swept boxes overlap.
//
//  1. vertex boxes from the F2 world-position chain at q0 and q1
//  2. body boxes (warp min/max per body)
//  3. body-pair overlaps by sort-and-sweep along the widest axis
//  4. one CTA per overlapping body pair: cull primitives against the
//     overlap box into shared memory tiles, test culled tile pairs, emit
//     hits with warp-aggregated appends
//  5. canonical order by LSD radix sorts on (c0, c2, c1, c3)
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "kernels.h"

namespace abd {

__global__ void k_vertex_boxes(int64_t V, const int* __restrict__ vert_body, const double* __restrict__ rest,
                               const double* __restrict__ q0, const double* __restrict__ q1, double h,
                               double* __restrict__ vbox) {
  int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= V) return;
  int b = vert_body[v];
  V3 xb = ld3(rest + 3 * v);
  V3 a = world_pos(q0 + 12 * (int64_t)b, xb);
  V3 c = world_pos(q1 + 12 * (int64_t)b, xb);
  double* o = vbox + 6 * v;
  o[0] = xsub(fmin(a.x, c.x), h);
  o[1] = xsub(fmin(a.y, c.y), h);
  o[2] = xsub(fmin(a.z, c.z), h);
  o[3] = xadd(fmax(a.x, c.x), h);
  o[4] = xadd(fmax(a.y, c.y), h);
  o[5] = xadd(fmax(a.z, c.z), h);
}

// one warp per body
__global__ void k_body_boxes(int B, const int* __restrict__ v_off, const double* __restrict__ vbox,
                             double* __restrict__ bbox) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= B) return;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int v = v_off[w] + lane; v < v_off[w + 1]; v += 32) {
    const double* b = vbox + 6 * (int64_t)v;
    for (int k = 0; k < 3; ++k) {
      lo[k] = fmin(lo[k], b[k]);
      hi[k] = fmax(hi[k], b[3 + k]);
    }
  }
  for (int o = 16; o > 0; o >>= 1)
    for (int k = 0; k < 3; ++k) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  if (lane == 0)
    for (int k = 0; k < 3; ++k) {
      bbox[6 * w + k] = lo[k];
      bbox[6 * w + 3 + k] = hi[k];
    }
}

__device__ __forceinline__ uint64_t sortable_bits(double x) {
  uint64_t u = (uint64_t)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void k_sweep_keys(int B, const double* __restrict__ bbox, int axis, uint64_t* keys, int* vals) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  keys[b] = sortable_bits(bbox[6 * b + axis]);
  vals[b] = b;
}

__device__ __forceinline__ bool box_overlap(const double* a, const double* b) {
  return a[0] <= b[3] && b[0] <= a[3] && a[1] <= b[4] && b[1] <= a[4] && a[2] <= b[5] && b[2] <= a[5];
}

// count (fill == false) or emit (fill == true) overlapping pairs
__global__ void k_sweep(int B, const int* __restrict__ order, const double* __restrict__ bbox, int axis,
                        const unsigned char* __restrict__ dyn, int* counts, const int* __restrict__ offs,
                        int2* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  int bi = order[i];
  const double* a = bbox + 6 * bi;
  double hi = a[3 + axis];
  int cnt = 0;
  int base = offs ? offs[i] : 0;
  for (int j = i + 1; j < B; ++j) {
    int bj = order[j];
    const double* b = bbox + 6 * bj;
    if (b[axis] > hi) break;
    if (!(dyn[bi] || dyn[bj])) continue;
    if (!box_overlap(a, b)) continue;
    if (out) out[base + cnt] = make_int2(min(bi, bj), max(bi, bj));
    ++cnt;
  }
  if (counts) counts[i] = cnt;
}

__global__ void k_pair_keys(int64_t n, const int2* __restrict__ p, int bB, uint64_t* keys, int* vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = ((uint64_t)p[i].x << bB) | (uint64_t)p[i].y;
  vals[i] = (int)i;
}

template <class T>
__global__ void k_gather(int64_t n, const int* __restrict__ idx, const T* __restrict__ in, T* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[idx[i]];
}

// ---------------------------------------------------------------------------
// primitive boxes (kind 0 vertex, 1 edge, 2 triangle) from vertex boxes
struct PrimGeo {
  const double* vbox;
  const int* v_off;
  const int* e_off;
  const int* t_off;
  const int* edges;
  const int* tris;
};

__device__ __forceinline__ void prim_box(const PrimGeo& g, int kind, int body, int local, double* bx) {
  if (kind == 0) {
    const double* v = g.vbox + 6 * (int64_t)(g.v_off[body] + local);
    for (int k = 0; k < 6; ++k) bx[k] = v[k];
    return;
  }
  int nv = kind == 1 ? 2 : 3;
  const int* ids = kind == 1 ? g.edges + 2 * (int64_t)(g.e_off[body] + local) : g.tris + 3 * (int64_t)(g.t_off[body] + local);
  const double* v0 = g.vbox + 6 * (int64_t)ids[0];
  for (int k = 0; k < 6; ++k) bx[k] = v0[k];
  for (int m = 1; m < nv; ++m) {
    const double* vm = g.vbox + 6 * (int64_t)ids[m];
    for (int k = 0; k < 3; ++k) {
      bx[k] = fmin(bx[k], vm[k]);
      bx[3 + k] = fmax(bx[3 + k], vm[3 + k]);
    }
  }
}

__device__ __forceinline__ int prim_count(const PrimGeo& g, int kind, int body) {
  const int* o = kind == 0 ? g.v_off : (kind == 1 ? g.e_off : g.t_off);
  return o[body + 1] - o[body];
}

constexpr int BP_THREADS = 256;
constexpr int BP_TILE = 256;

// block-wide cull of primitives [start, start+TILE) of (kind, body) against the
// overlap box into shared lists; returns the culled count
__device__ int cull_tile(const PrimGeo& g, int kind, int body, int start, int count, const double* obox, int* ids,
                         double* boxes, int* warp_tot) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int local = start + threadIdx.x;
  bool keep = false;
  double bx[6];
  if (threadIdx.x < BP_TILE && local < count) {
    prim_box(g, kind, body, local, bx);
    keep = bx[0] <= obox[3] && obox[0] <= bx[3] && bx[1] <= obox[4] && obox[1] <= bx[4] && bx[2] <= obox[5] &&
           obox[2] <= bx[5];
  }
  unsigned m = __ballot_sync(0xffffffffu, keep);
  if (lane == 0) warp_tot[wid] = __popc(m);
  __syncthreads();
  int base = 0, total = 0;
  for (int w = 0; w < BP_THREADS / 32; ++w) {
    if (w < wid) base += warp_tot[w];
    total += warp_tot[w];
  }
  if (keep) {
    int at = base + __popc(m & ((1u << lane) - 1));
    ids[at] = local;
    for (int k = 0; k < 6; ++k) boxes[6 * at + k] = bx[k];
  }
  __syncthreads();
  return total;
}

// one CTA per overlapping body pair
__global__ void __launch_bounds__(BP_THREADS) k_prim_pairs(PrimGeo g, int64_t n_ov, const int2* __restrict__ ov,
                                                             const double* __restrict__ bbox,
                                                             unsigned long long* counters, int64_t cap_vf,
                                                             int64_t cap_ee, int4* out_vf, int4* out_ee) {
  __shared__ int ida[BP_TILE], idb[BP_TILE];
  __shared__ double bxa[6 * BP_TILE], bxb[6 * BP_TILE];
  __shared__ int warp_tot[BP_THREADS / 32];
  __shared__ double obox[6];
  for (int64_t pi = blockIdx.x; pi < n_ov; pi += gridDim.x) {
    int2 pr = ov[pi];
    int i = pr.x, j = pr.y;
    if (threadIdx.x < 3) {
      obox[threadIdx.x] = fmax(bbox[6 * i + threadIdx.x], bbox[6 * j + threadIdx.x]);
      obox[3 + threadIdx.x] = fmin(bbox[6 * i + 3 + threadIdx.x], bbox[6 * j + 3 + threadIdx.x]);
    }
    __syncthreads();
    // products: (vertex of i, tri of j) -> vf(i,.,j,.); (vertex of j, tri of i) -> vf(j,.,i,.); (edge i, edge j)
    for (int prod = 0; prod < 3; ++prod) {
      int ka = prod == 2 ? 1 : 0, kb = prod == 2 ? 1 : 2;
      int ba = prod == 1 ? j : i, bb = prod == 1 ? i : j;
      int na = prim_count(g, ka, ba), nb = prim_count(g, kb, bb);
      bool is_vf = prod < 2;
      for (int sa = 0; sa < na; sa += BP_TILE) {
        int ca = cull_tile(g, ka, ba, sa, na, obox, ida, bxa, warp_tot);
        if (ca == 0) continue;
        for (int sb = 0; sb < nb; sb += BP_TILE) {
          int cb = cull_tile(g, kb, bb, sb, nb, obox, idb, bxb, warp_tot);
          if (cb == 0) continue;
          int64_t tot = (int64_t)ca * cb;
          for (int64_t k0 = 0; k0 < tot; k0 += BP_THREADS) {
            int64_t k = k0 + threadIdx.x;
            bool hit = false;
            int x = 0, y = 0;
            if (k < tot) {
              x = (int)(k / cb);
              y = (int)(k % cb);
              hit = box_overlap(bxa + 6 * x, bxb + 6 * y);
            }
            unsigned m = __ballot_sync(0xffffffffu, hit);
            if (m) {
              int lane = threadIdx.x & 31;
              unsigned long long base = 0;
              if (lane == __ffs(m) - 1) base = atomicAdd(counters + (is_vf ? 0 : 1), (unsigned long long)__popc(m));
              base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
              if (hit) {
                unsigned long long at = base + __popc(m & ((1u << lane) - 1));
                if (is_vf) {
                  if ((int64_t)at < cap_vf) out_vf[at] = make_int4(ba, ida[x], bb, idb[y]);
                } else {
                  if ((int64_t)at < cap_ee) out_ee[at] = make_int4(ba, ida[x], bb, idb[y]);
                }
              }
            }
          }
          __syncthreads();
        }
      }
    }
    __syncthreads();
  }
}

// keys for canonical order (c0, c2, c1, c3): two LSD passes with stable sorts
__global__ void k_row_keys(int64_t n, const int4* __restrict__ rows, int pass, int w1, int w3, int wb,
                           const int* __restrict__ perm, uint64_t* keys, int* vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int src = perm ? perm[i] : (int)i;
  int4 r = rows[src];
  uint64_t k;
  if (pass == 0) k = ((uint64_t)r.y << w3) | (uint64_t)r.w;  // (c1, c3)
  else k = ((uint64_t)r.x << wb) | (uint64_t)r.z;            // (c0, c2)
  keys[i] = k;
  vals[i] = src;
  (void)w1;
}

// ---------------------------------------------------------------------------
static void sort_rows(Scene& s, DVec<int4>& rows, int64_t n, int w1, int w3) {
  if (n <= 1) return;
  int wb = bits_for(s.B - 1);
  s.tmp_l0.resize(n);
  s.tmp_l1.resize(n);
  s.tmp_i0.resize(n);
  s.tmp_i1.resize(n);
  uint64_t* k0 = (uint64_t*)s.tmp_l0.p;
  uint64_t* k1 = (uint64_t*)s.tmp_l1.p;
  bool alt = false;
  // pass 0: by (c1, c3)
  k_row_keys<<<grid_for(n, 256), 256, 0, s.stream>>>(n, rows.p, 0, w1, w3, wb, nullptr, k0, s.tmp_i0.p);
  note_launch("k_row_keys");
  sort_pairs_u64(s, k0, k1, s.tmp_i0.p, s.tmp_i1.p, n, w1 + w3, alt);
  int* perm = alt ? s.tmp_i1.p : s.tmp_i0.p;
  // pass 1: stable by (c0, c2) on the permuted rows
  s.tmp_i2.resize(n);
  s.tmp_i3.resize(n);
  k_row_keys<<<grid_for(n, 256), 256, 0, s.stream>>>(n, rows.p, 1, w1, w3, wb, perm, k0, s.tmp_i2.p);
  note_launch("k_row_keys");
  sort_pairs_u64(s, k0, k1, s.tmp_i2.p, s.tmp_i3.p, n, 2 * wb, alt);
  int* perm2 = alt ? s.tmp_i3.p : s.tmp_i2.p;
  DVec<int4> tmp;
  tmp.resize(n);
  k_gather<int4><<<grid_for(n, 256), 256, 0, s.stream>>>(n, perm2, rows.p, tmp.p);
  note_launch("k_gather");
  CK(cudaMemcpyAsync(rows.p, tmp.p, n * sizeof(int4), cudaMemcpyDeviceToDevice, s.stream));
  CK(cudaStreamSynchronize(s.stream));
}

void broad_phase(Scene& s, const double* q0, const double* q1, double d_hat) {
  cudaStream_t st = s.stream;
  double h = 0.5 * d_hat;
  Cands& c = s.cands;
  c.n_vf = c.n_ee = c.n_ov = 0;
  if (s.B < 2) return;
  s.vbox.resize(6 * s.V);
  s.bbox.resize(6 * s.B);
  k_vertex_boxes<<<grid_for(s.V, 256), 256, 0, st>>>(s.V, s.vert_body.p, s.rest.p, q0, q1, h, s.vbox.p);
  note_launch("k_vertex_boxes");
  k_body_boxes<<<grid_for((int64_t)s.B * 32, 256), 256, 0, st>>>(s.B, s.v_off.p, s.vbox.p, s.bbox.p);
  note_launch("k_body_boxes");
  // widest axis of the body-box lows (host side: B*6 doubles is small)
  std::vector<double> hb(6 * (size_t)s.B);
  s.bbox.download(hb.data(), hb.size(), st);
  CK(cudaStreamSynchronize(st));
  int axis = 0;
  double best = -1.0;
  for (int k = 0; k < 3; ++k) {
    double lo = INFINITY, hi = -INFINITY;
    for (int b = 0; b < s.B; ++b) {
      lo = fmin(lo, hb[6 * b + k]);
      hi = fmax(hi, hb[6 * b + k]);
    }
    if (hi - lo > best) {
      best = hi - lo;
      axis = k;
    }
  }
  // sort bodies along the axis
  s.tmp_l0.resize(s.B);
  s.tmp_l1.resize(s.B);
  s.tmp_i0.resize(s.B + 1);
  s.tmp_i1.resize(s.B + 1);
  k_sweep_keys<<<grid_for(s.B, 256), 256, 0, st>>>(s.B, s.bbox.p, axis, (uint64_t*)s.tmp_l0.p, s.tmp_i0.p);
  note_launch("k_sweep_keys");
  bool alt = false;
  sort_pairs_u64(s, (uint64_t*)s.tmp_l0.p, (uint64_t*)s.tmp_l1.p, s.tmp_i0.p, s.tmp_i1.p, s.B, 64, alt);
  DVec<int> order;
  order.resize(s.B);
  CK(cudaMemcpyAsync(order.p, alt ? s.tmp_i1.p : s.tmp_i0.p, s.B * sizeof(int), cudaMemcpyDeviceToDevice, st));
  DVec<int> cnt, off;
  cnt.resize(s.B + 1);
  off.resize(s.B + 1);
  CK(cudaMemsetAsync(cnt.p + s.B, 0, sizeof(int), st));
  k_sweep<<<grid_for(s.B, 128), 128, 0, st>>>(s.B, order.p, s.bbox.p, axis, s.dyn.p, cnt.p, nullptr, nullptr);
  note_launch("k_sweep");
  scan_exclusive_i32(s, cnt.p, off.p, s.B + 1);
  int n_ov = 0;
  CK(cudaMemcpyAsync(&n_ov, off.p + s.B, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  c.ov.resize(n_ov);
  c.n_ov = n_ov;
  if (n_ov == 0) return;
  k_sweep<<<grid_for(s.B, 128), 128, 0, st>>>(s.B, order.p, s.bbox.p, axis, s.dyn.p, nullptr, off.p, c.ov.p);
  note_launch("k_sweep");
  // canonical (i, j) order of overlap pairs
  {
    int bB = bits_for(s.B - 1);
    s.tmp_l0.resize(n_ov);
    s.tmp_l1.resize(n_ov);
    s.tmp_i0.resize(n_ov);
    s.tmp_i1.resize(n_ov);
    k_pair_keys<<<grid_for(n_ov, 256), 256, 0, st>>>(n_ov, c.ov.p, bB, (uint64_t*)s.tmp_l0.p, s.tmp_i0.p);
    note_launch("k_pair_keys");
    sort_pairs_u64(s, (uint64_t*)s.tmp_l0.p, (uint64_t*)s.tmp_l1.p, s.tmp_i0.p, s.tmp_i1.p, n_ov, 2 * bB, alt);
    DVec<int2> tmp;
    tmp.resize(n_ov);
    k_gather<int2><<<grid_for(n_ov, 256), 256, 0, st>>>(n_ov, alt ? s.tmp_i1.p : s.tmp_i0.p, c.ov.p, tmp.p);
    note_launch("k_gather");
    CK(cudaMemcpyAsync(c.ov.p, tmp.p, n_ov * sizeof(int2), cudaMemcpyDeviceToDevice, st));
  }
  // primitive pairs
  PrimGeo g{s.vbox.p, s.v_off.p, s.e_off.p, s.t_off.p, s.edges.p, s.tris.p};
  DVec<unsigned long long> counters;
  counters.resize(2);
  if (c.vf.cap < 1024) c.vf.resize(1024);
  if (c.ee.cap < 1024) c.ee.resize(1024);
  unsigned long long hc[2];
  for (int attempt = 0; attempt < 3; ++attempt) {
    CK(cudaMemsetAsync(counters.p, 0, 2 * sizeof(unsigned long long), st));
    int grid = (int)std::min<int64_t>(n_ov, (int64_t)s.num_sms * 8);
    k_prim_pairs<<<grid, BP_THREADS, 0, st>>>(g, n_ov, c.ov.p, s.bbox.p, counters.p, (int64_t)c.vf.cap,
                                              (int64_t)c.ee.cap, c.vf.p, c.ee.p);
    note_launch("k_prim_pairs");
    CK(cudaMemcpyAsync(hc, counters.p, sizeof(hc), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hc[0] <= c.vf.cap && hc[1] <= c.ee.cap) break;
    if (hc[0] > c.vf.cap) c.vf.resize(hc[0]);
    if (hc[1] > c.ee.cap) c.ee.resize(hc[1]);
  }
  c.n_vf = (int64_t)hc[0];
  c.n_ee = (int64_t)hc[1];
  c.vf.n = c.n_vf;
  c.ee.n = c.n_ee;
  sort_rows(s, c.vf, c.n_vf, bits_for(s.max_v - 1), bits_for(s.max_t - 1));
  sort_rows(s, c.ee, c.n_ee, bits_for(s.max_e - 1), bits_for(s.max_e - 1));
}

}  // namespace abd
