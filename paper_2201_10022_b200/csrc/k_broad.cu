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

// swept, inflated vertex box (contact.py:350-354) from the F2 world positions
__device__ __forceinline__ void vertex_box(const double* __restrict__ rest, int64_t v, const double* q0b,
                                           const double* q1b, double h, double* o) {
  V3 xb = ld3(rest + 3 * v);
  V3 a = world_pos(q0b, xb);
  V3 c = world_pos(q1b, xb);
  o[0] = xsub(fmin(a.x, c.x), h);
  o[1] = xsub(fmin(a.y, c.y), h);
  o[2] = xsub(fmin(a.z, c.z), h);
  o[3] = xadd(fmax(a.x, c.x), h);
  o[4] = xadd(fmax(a.y, c.y), h);
  o[5] = xadd(fmax(a.z, c.z), h);
}

// one warp per body: union of its swept vertex boxes (computed on the fly)
__global__ void k_body_boxes(int B, const int* __restrict__ v_off, const double* __restrict__ rest,
                             const double* __restrict__ q0, const double* __restrict__ q1, double h,
                             double* __restrict__ bbox) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= B) return;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int v = v_off[w] + lane; v < v_off[w + 1]; v += 32) {
    double b[6];
    vertex_box(rest, v, q0 + 12 * (int64_t)w, q1 + 12 * (int64_t)w, h, b);
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
  const double* rest;
  const double* q0;
  const double* q1;
  double h;
  const int* v_off;
  const int* e_off;
  const int* t_off;
  const int* edges;
  const int* tris;
};

// box of a vertex / edge / triangle = min/max of its swept vertex boxes (contact.py:222-229)
__device__ __forceinline__ void prim_box(const PrimGeo& g, int kind, int body, int local, double* bx) {
  const double* q0b = g.q0 + 12 * (int64_t)body;
  const double* q1b = g.q1 + 12 * (int64_t)body;
  if (kind == 0) {
    vertex_box(g.rest, g.v_off[body] + local, q0b, q1b, g.h, bx);
    return;
  }
  int nv = kind == 1 ? 2 : 3;
  const int* ids = kind == 1 ? g.edges + 2 * (int64_t)(g.e_off[body] + local) : g.tris + 3 * (int64_t)(g.t_off[body] + local);
  vertex_box(g.rest, ids[0], q0b, q1b, g.h, bx);
  for (int m = 1; m < nv; ++m) {
    double vm[6];
    vertex_box(g.rest, ids[m], q0b, q1b, g.h, vm);
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
  else if (pass == 1) k = ((uint64_t)r.x << wb) | (uint64_t)r.z;  // (c0, c2)
  else k = ((((((uint64_t)r.x << wb) | (uint64_t)r.z) << w1) | (uint64_t)r.y) << w3) | (uint64_t)r.w;  // all
  keys[i] = k;
  vals[i] = src;
  (void)w1;
}

// widest spread of body-box lows: 6 doubles (min/max per axis) via ordered atomics
__device__ __forceinline__ unsigned long long ord_bits(double x) {
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void k_axis_extent(int B, const double* __restrict__ bbox, unsigned long long* mm) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  for (int k = 0; k < 3; ++k) {
    unsigned long long o = ord_bits(bbox[6 * b + k]);
    atomicMin(mm + k, o);
    atomicMax(mm + 3 + k, o);
  }
}

__global__ void k_pick_axis(const unsigned long long* mm, int* axis) {
  double best = -1.0;
  int ax = 0;
  for (int k = 0; k < 3; ++k) {
    unsigned long long lo = mm[k], hi = mm[3 + k];
    auto dec = [](unsigned long long u) {
      u = (u & 0x8000000000000000ull) ? (u & 0x7fffffffffffffffull) : ~u;
      return __longlong_as_double((long long)u);
    };
    double ext = dec(hi) - dec(lo);
    if (ext > best) {
      best = ext;
      ax = k;
    }
  }
  *axis = ax;
}

__global__ void k_sweep_keys_dev(int B, const double* __restrict__ bbox, const int* __restrict__ axis, uint64_t* keys,
                                 int* vals) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  keys[b] = sortable_bits(bbox[6 * b + *axis]);
  vals[b] = b;
}

__global__ void k_sweep_dev(int B, const int* __restrict__ order, const double* __restrict__ bbox,
                            const int* __restrict__ axis_p, const unsigned char* __restrict__ dyn, int* counts,
                            const int* __restrict__ offs, int2* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  int axis = *axis_p;
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

// ---------------------------------------------------------------------------
// body-pair overlaps on a uniform grid.  Cell size = 90th percentile of the
// body-box extents; "small" bodies (extent <= cell) are binned by the cell of
// their box low corner and query the 3x3x3 cells that can hold an overlapping
// low corner; "large" bodies (ground slabs, walls) test every body directly.
// Only exact closed-box overlap tests decide membership, so the set equals the
// all-pairs test (contact.py:366-372) whatever the binning.
// extents as float bits (non-negative floats sort as unsigned ints); the cell
// size only steers the binning, never the overlap decision
__global__ void k_extent_keys(int B, const double* __restrict__ bbox, uint32_t* keys) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double* x = bbox + 6 * b;
  double e = fmax(fmax(x[3] - x[0], x[4] - x[1]), x[5] - x[2]);
  keys[b] = __float_as_uint((float)fmax(e, 0.0));
}

// 10 bits per axis (wraps every 1024 cells: collisions only add box tests)
__device__ __forceinline__ uint32_t cell_key(long long ix, long long iy, long long iz) {
  return (((uint32_t)ix & 1023u) << 20) | (((uint32_t)iy & 1023u) << 10) | ((uint32_t)iz & 1023u);
}

__global__ void k_cell_keys(int B, const double* __restrict__ bbox, const uint32_t* __restrict__ sorted_ext,
                            int pct_idx, uint32_t* keys, int* vals, double* cell_out) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  // cell = largest extent not above 4x the median (outliers such as ground slabs
  // and walls become "large"); next float up so every small body fits a cell
  uint32_t lim = __float_as_uint(4.0f * __uint_as_float(sorted_ext[(B - 1) / 2]));
  int lo = 0, hi = B;  // first index with key > lim
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (sorted_ext[mid] <= lim) lo = mid + 1;
    else hi = mid;
  }
  (void)pct_idx;
  double cell = (double)__uint_as_float(sorted_ext[max(lo - 1, 0)] + 1u);
  if (!(cell > 0.0)) cell = 1.0;
  if (b == 0) *cell_out = cell;
  const double* x = bbox + 6 * b;
  double e = fmax(fmax(x[3] - x[0], x[4] - x[1]), x[5] - x[2]);
  vals[b] = b;
  if (e > cell) {
    keys[b] = 0xffffffffu;  // large: not binned
    return;
  }
  keys[b] = cell_key((long long)floor(x[0] / cell), (long long)floor(x[1] / cell), (long long)floor(x[2] / cell));
}

__device__ __forceinline__ int lower_bound_u32(const uint32_t* a, int n, uint32_t k) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// one thread per body: emit (min, max) overlapping pairs exactly once
__global__ void k_grid_pairs(int B, const double* __restrict__ bbox, const unsigned char* __restrict__ dyn,
                             const uint32_t* __restrict__ skeys, const int* __restrict__ sbody, int n_small,
                             const double* __restrict__ cell_p, unsigned long long* count, int64_t cap, int2* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  const double cell = *cell_p;
  const double* a = bbox + 6 * i;
  double e = fmax(fmax(a[3] - a[0], a[4] - a[1]), a[5] - a[2]);
  auto emit = [&](int j) {
    if (!(dyn[i] || dyn[j])) return;
    if (!box_overlap(a, bbox + 6 * j)) return;
    unsigned long long at = atomicAdd(count, 1ull);
    if ((int64_t)at < cap) out[at] = make_int2(min(i, j), max(i, j));
  };
  // pairs involving a large body come from k_large_pairs
  if (e > cell) return;
  // an overlapping small body has lo_j in [lo_i - cell, hi_i]; floor(lo/cell) is
  // monotone in lo, and the 1e-9 margin absorbs the rounding of lo_i/cell - 1
  long long x0 = (long long)floor(a[0] / cell - 1.0 - 1e-9), x1 = (long long)floor(a[3] / cell);
  long long y0 = (long long)floor(a[1] / cell - 1.0 - 1e-9), y1 = (long long)floor(a[4] / cell);
  long long z0 = (long long)floor(a[2] / cell - 1.0 - 1e-9), z1 = (long long)floor(a[5] / cell);
  for (long long cx = x0; cx <= x1; ++cx)
    for (long long cy = y0; cy <= y1; ++cy)
      for (long long cz = z0; cz <= z1; ++cz) {
        uint32_t k = cell_key(cx, cy, cz);
        int p = lower_bound_u32(skeys, n_small, k);
        for (; p < n_small && skeys[p] == k; ++p) {
          int j = sbody[p];
          if (j > i) emit(j);  // small-small pairs once, from the lower index
        }
      }
}

// every (large body, body) pair: thread per body j over the few large bodies
// (the ~0-keyed tail of the sorted cell keys); large-large pairs once (j > i)
__global__ void k_large_pairs(int B, const double* __restrict__ bbox, const unsigned char* __restrict__ dyn,
                              const uint32_t* __restrict__ skeys, const int* __restrict__ sbody,
                              const double* __restrict__ cell_p, unsigned long long* count, int64_t cap, int2* out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= B) return;
  const double cell = *cell_p;
  int first = lower_bound_u32(skeys, B, 0xffffffffu);
  if (first >= B) return;
  const double* b = bbox + 6 * j;
  double ej = fmax(fmax(b[3] - b[0], b[4] - b[1]), b[5] - b[2]);
  bool j_large = ej > cell;
  for (int p = first; p < B; ++p) {
    int i = sbody[p];
    if (i == j || (j_large && j < i)) continue;
    if (!(dyn[i] || dyn[j])) continue;
    if (!box_overlap(bbox + 6 * i, b)) continue;
    unsigned long long at = atomicAdd(count, 1ull);
    if ((int64_t)at < cap) out[at] = make_int2(min(i, j), max(i, j));
  }
}

static void sort_rows(Scene& s, DVec<int4>& rows, int64_t n, int w1, int w3) {
  if (n <= 1) return;
  int wb = bits_for(s.B - 1);
  Scene::Work& w = s.w;
  w.k0.resize(n);
  w.k1.resize(n);
  w.va.resize(n);
  w.vb.resize(n);
  w.cnt.resize(n);
  w.off.resize(n);
  bool alt = false;
  if (2 * wb + w1 + w3 <= 64) {  // whole (c0, c2, c1, c3) key fits one 64-bit radix sort
    k_row_keys<<<grid_for(n, 256), 256, 0, s.stream>>>(n, rows.p, 2, w1, w3, wb, nullptr, w.k0.p, w.va.p);
    note_launch("k_row_keys");
    sort_pairs_u64(s, w.k0.p, w.k1.p, w.va.p, w.vb.p, n, 2 * wb + w1 + w3, alt);
    w.rows_tmp.resize(n);
    k_gather<int4><<<grid_for(n, 256), 256, 0, s.stream>>>(n, alt ? w.vb.p : w.va.p, rows.p, w.rows_tmp.p);
    note_launch("k_gather");
    CK(cudaMemcpyAsync(rows.p, w.rows_tmp.p, n * sizeof(int4), cudaMemcpyDeviceToDevice, s.stream));
    return;
  }
  // pass 0: by (c1, c3); pass 1: stable by (c0, c2) on the permuted rows (LSD)
  k_row_keys<<<grid_for(n, 256), 256, 0, s.stream>>>(n, rows.p, 0, w1, w3, wb, nullptr, w.k0.p, w.va.p);
  note_launch("k_row_keys");
  sort_pairs_u64(s, w.k0.p, w.k1.p, w.va.p, w.vb.p, n, w1 + w3, alt);
  int* perm = alt ? w.vb.p : w.va.p;
  k_row_keys<<<grid_for(n, 256), 256, 0, s.stream>>>(n, rows.p, 1, w1, w3, wb, perm, w.k0.p, w.cnt.p);
  note_launch("k_row_keys");
  sort_pairs_u64(s, w.k0.p, w.k1.p, w.cnt.p, w.off.p, n, 2 * wb, alt);
  int* perm2 = alt ? w.off.p : w.cnt.p;
  w.rows_tmp.resize(n);
  k_gather<int4><<<grid_for(n, 256), 256, 0, s.stream>>>(n, perm2, rows.p, w.rows_tmp.p);
  note_launch("k_gather");
  CK(cudaMemcpyAsync(rows.p, w.rows_tmp.p, n * sizeof(int4), cudaMemcpyDeviceToDevice, s.stream));
}

void broad_phase(Scene& s, const double* q0, const double* q1, double d_hat) {
  cudaStream_t st = s.stream;
  double h = 0.5 * d_hat;
  Cands& c = s.cands;
  Scene::Work& w = s.w;
  c.n_vf = c.n_ee = c.n_ov = 0;
  if (s.B < 2) return;
  s.bbox.resize(6 * s.B);
  k_body_boxes<<<grid_for((int64_t)s.B * 32, 256), 256, 0, st>>>(s.B, s.v_off.p, s.rest.p, q0, q1, h, s.bbox.p);
  note_launch("k_body_boxes");
  // body pairs on a uniform grid (cell = 90th-percentile body extent)
  bool alt = false;
  w.k0.resize(s.B);
  w.k1.resize(s.B);
  w.va.resize(s.B + 1);
  w.vb.resize(s.B + 1);
  w.ka.resize(s.B);
  w.kb.resize(s.B);
  uint32_t* ext_sorted = reinterpret_cast<uint32_t*>(w.e0.p);
  w.e0.resize(s.B);
  k_extent_keys<<<grid_for(s.B, 256), 256, 0, st>>>(s.B, s.bbox.p, w.ka.p);
  note_launch("k_extent_keys");
  ext_sorted = reinterpret_cast<uint32_t*>(w.e0.p);
  {
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, w.ka.p, ext_sorted, s.B, 0, 32, st));
    s.tmp_bytes.resize(bytes);
    CK(cub::DeviceRadixSort::SortKeys(s.tmp_bytes.p, bytes, w.ka.p, ext_sorted, s.B, 0, 32, st));
  }
  w.scal.resize(4);
  int pct = (int)((int64_t)(s.B - 1) * 9 / 10);
  k_cell_keys<<<grid_for(s.B, 256), 256, 0, st>>>(s.B, s.bbox.p, ext_sorted, pct, w.ka.p, w.va.p, w.scal.p);
  note_launch("k_cell_keys");
  sort_pairs_u32(s, w.ka.p, w.kb.p, w.va.p, w.vb.p, s.B, 32, alt);
  const uint32_t* skeys = alt ? w.kb.p : w.ka.p;
  const int* sbody = alt ? w.vb.p : w.va.p;
  int n_small = s.B;  // large bodies carry key ~0 and sort last; the lookups never match them
  unsigned long long* ovc = w.ull.p + 6;
  unsigned long long* hov = reinterpret_cast<unsigned long long*>(s.h_pinned);
  if (c.ov.cap < 256) c.ov.resize(256);
  for (int attempt = 0; attempt < 3; ++attempt) {
    CK(cudaMemsetAsync(ovc, 0, sizeof(unsigned long long), st));
    k_grid_pairs<<<grid_for(s.B, 128), 128, 0, st>>>(s.B, s.bbox.p, s.dyn.p, skeys, sbody, n_small, w.scal.p, ovc,
                                                     (int64_t)c.ov.cap, c.ov.p);
    note_launch("k_grid_pairs");
    k_large_pairs<<<grid_for(s.B, 128), 128, 0, st>>>(s.B, s.bbox.p, s.dyn.p, skeys, sbody, w.scal.p, ovc,
                                                      (int64_t)c.ov.cap, c.ov.p);
    note_launch("k_large_pairs");
    CK(cudaMemcpyAsync(hov, ovc, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (hov[0] <= c.ov.cap) break;
    c.ov.resize(hov[0]);
  }
  int n_ov = (int)hov[0];
  c.n_ov = n_ov;
  c.ov.n = n_ov;
  if (n_ov == 0) return;
  // canonical (i, j) order of overlap pairs
  {
    int bB = bits_for(s.B - 1);
    w.k0.resize(n_ov);
    w.k1.resize(n_ov);
    w.va.resize(n_ov);
    w.vb.resize(n_ov);
    k_pair_keys<<<grid_for(n_ov, 256), 256, 0, st>>>(n_ov, c.ov.p, bB, w.k0.p, w.va.p);
    note_launch("k_pair_keys");
    sort_pairs_u64(s, w.k0.p, w.k1.p, w.va.p, w.vb.p, n_ov, 2 * bB, alt);
    w.pairs_tmp.resize(n_ov);
    k_gather<int2><<<grid_for(n_ov, 256), 256, 0, st>>>(n_ov, alt ? w.vb.p : w.va.p, c.ov.p, w.pairs_tmp.p);
    note_launch("k_gather");
    CK(cudaMemcpyAsync(c.ov.p, w.pairs_tmp.p, n_ov * sizeof(int2), cudaMemcpyDeviceToDevice, st));
  }
  // primitive pairs
  PrimGeo g{s.rest.p, q0, q1, h, s.v_off.p, s.e_off.p, s.t_off.p, s.edges.p, s.tris.p};
  unsigned long long* counters = w.ull.p + 4;
  if (c.vf.cap < 1024) c.vf.resize(1024);
  if (c.ee.cap < 1024) c.ee.resize(1024);
  unsigned long long* hc = reinterpret_cast<unsigned long long*>(s.h_pinned);
  for (int attempt = 0; attempt < 3; ++attempt) {
    CK(cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), st));
    int grid = (int)std::min<int64_t>(n_ov, (int64_t)s.num_sms * 8);
    if (s.instrument) CK(cudaEventRecord(s.ev0, st));
    k_prim_pairs<<<grid, BP_THREADS, 0, st>>>(g, n_ov, c.ov.p, s.bbox.p, counters, (int64_t)c.vf.cap,
                                              (int64_t)c.ee.cap, c.vf.p, c.ee.p);
    note_launch("k_prim_pairs");
    if (s.instrument) CK(cudaEventRecord(s.ev1, st));
    CK(cudaMemcpyAsync(hc, counters, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (s.instrument) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, s.ev0, s.ev1));
      Scene::KStat& k = s.kstat[3];
      k.launches += 1;
      k.units += n_ov;
      k.ms += ms;
      // rest xyz, int32 edges/tris, q0+q1 per body, int4 candidate rows
      k.bytes += 24.0 * (double)s.V + 8.0 * (double)s.E + 12.0 * (double)s.T + 192.0 * (double)s.B +
                 16.0 * (double)(hc[0] + hc[1]);
    }
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
