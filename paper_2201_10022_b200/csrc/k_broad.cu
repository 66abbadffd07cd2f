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
#include <cstdlib>
#include <vector>

#include "kernels.h"

namespace abd {
void slab_partition(Scene& s, const double* q);  // comm.cu
}

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
                             double* __restrict__ bbox, const double* __restrict__ vl_box = nullptr,
                             int* viol = nullptr) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= B) return;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  // BB_UNROLL vertices per lane in flight: their rest loads issue together instead
  // of one DRAM round trip per vertex (min / max do not depend on the order)
  constexpr int BB_UNROLL = 4;
  const int v0 = v_off[w], v1 = v_off[w + 1];
  const double* q0b = q0 + 12 * (int64_t)w;
  const double* q1b = q1 + 12 * (int64_t)w;
  for (int base = v0 + lane; base < v1; base += 32 * BB_UNROLL) {
    V3 xb[BB_UNROLL];
#pragma unroll
    for (int u = 0; u < BB_UNROLL; ++u) {
      const int v = base + 32 * u;
      if (v < v1) xb[u] = ld3(rest + 3 * (int64_t)v);
    }
#pragma unroll
    for (int u = 0; u < BB_UNROLL; ++u) {
      if (base + 32 * u >= v1) break;
      const V3 a = world_pos(q0b, xb[u]);
      const V3 c = world_pos(q1b, xb[u]);
      lo[0] = fmin(lo[0], xsub(fmin(a.x, c.x), h));
      lo[1] = fmin(lo[1], xsub(fmin(a.y, c.y), h));
      lo[2] = fmin(lo[2], xsub(fmin(a.z, c.z), h));
      hi[0] = fmax(hi[0], xadd(fmax(a.x, c.x), h));
      hi[1] = fmax(hi[1], xadd(fmax(a.y, c.y), h));
      hi[2] = fmax(hi[2], xadd(fmax(a.z, c.z), h));
    }
  }
  for (int o = 16; o > 0; o >>= 1)
    for (int k = 0; k < 3; ++k) {
      lo[k] = fmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  if (lane == 0) {
    for (int k = 0; k < 3; ++k) {
      bbox[6 * w + k] = lo[k];
      bbox[6 * w + 3 + k] = hi[k];
    }
    // Verlet list: the box must still lie inside its inflated box (k_vl_contain's test)
    if (vl_box) {
      const double* y = vl_box + 6 * w;
      if (!(lo[0] >= y[0] && lo[1] >= y[1] && lo[2] >= y[2] && hi[0] <= y[3] && hi[1] <= y[4] && hi[2] <= y[5]))
        atomicExch(viol, 1);
    }
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

constexpr int BP_THREADS = 512;
constexpr int BP_TILE = 512;
constexpr int BP_VCAP = 256;  // vertex boxes cached in shared memory per body (else on the fly)

// primitive box from the body's cached vertex boxes (vb != nullptr) or recomputed
__device__ __forceinline__ void prim_box_c(const PrimGeo& g, int kind, int body, int local, const double* vb,
                                           double* bx) {
  if (vb == nullptr) {
    prim_box(g, kind, body, local, bx);
    return;
  }
  const int v0 = g.v_off[body];
  if (kind == 0) {
    const double* s = vb + 6 * local;
#pragma unroll
    for (int k = 0; k < 6; ++k) bx[k] = s[k];
    return;
  }
  const int nv = kind == 1 ? 2 : 3;
  const int* ids =
      kind == 1 ? g.edges + 2 * (int64_t)(g.e_off[body] + local) : g.tris + 3 * (int64_t)(g.t_off[body] + local);
  const double* s0 = vb + 6 * (ids[0] - v0);
#pragma unroll
  for (int k = 0; k < 6; ++k) bx[k] = s0[k];
  for (int m = 1; m < nv; ++m) {
    const double* sm = vb + 6 * (ids[m] - v0);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      bx[k] = fmin(bx[k], sm[k]);
      bx[3 + k] = fmax(bx[3 + k], sm[3 + k]);
    }
  }
}

// block-wide cull of primitives [start, start+TILE) of (kind, body) against the
// overlap box into shared lists; returns the culled count
__device__ int cull_tile(const PrimGeo& g, int kind, int body, int start, int count, const double* obox,
                         const double* vb, int* ids, double* boxes, int* warp_tot) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int local = start + threadIdx.x;
  bool keep = false;
  double bx[6];
  if (threadIdx.x < BP_TILE && local < count) {
    prim_box_c(g, kind, body, local, vb, bx);
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

constexpr size_t BP_SMEM = sizeof(double) * (2 * 6 * BP_VCAP + 2 * 6 * BP_TILE) + sizeof(int) * 2 * BP_TILE;

// one CTA per overlapping body pair; the vertex boxes of both bodies are computed
// once per pair into shared memory (edge / triangle boxes are their min/max)
__global__ void __launch_bounds__(BP_THREADS) k_prim_pairs(PrimGeo g, int64_t n_ov, const int2* __restrict__ ov,
                                                             const double* __restrict__ bbox,
                                                             unsigned long long* counters, int64_t cap_vf,
                                                             int64_t cap_ee, int4* out_vf, int4* out_ee) {
  extern __shared__ double bp_sm[];
  double* vbi = bp_sm;                      // BP_VCAP x 6
  double* vbj = vbi + 6 * BP_VCAP;          // BP_VCAP x 6
  double* bxa = vbj + 6 * BP_VCAP;          // BP_TILE x 6
  double* bxb = bxa + 6 * BP_TILE;          // BP_TILE x 6
  int* ida = reinterpret_cast<int*>(bxb + 6 * BP_TILE);
  int* idb = ida + BP_TILE;
  __shared__ int warp_tot[BP_THREADS / 32];
  __shared__ double obox[6];
  for (int64_t pi = blockIdx.x; pi < n_ov; pi += gridDim.x) {
    int2 pr = ov[pi];
    int i = pr.x, j = pr.y;
    if (threadIdx.x < 3) {
      obox[threadIdx.x] = fmax(bbox[6 * i + threadIdx.x], bbox[6 * j + threadIdx.x]);
      obox[3 + threadIdx.x] = fmin(bbox[6 * i + 3 + threadIdx.x], bbox[6 * j + 3 + threadIdx.x]);
    }
    const int nvi = prim_count(g, 0, i), nvj = prim_count(g, 0, j);
    const bool ci = nvi <= BP_VCAP, cj = nvj <= BP_VCAP;
    for (int t = threadIdx.x; t < 2 * BP_VCAP; t += BP_THREADS) {
      const int side = t / BP_VCAP, lv = t % BP_VCAP;
      const int body = side ? j : i;
      if ((side ? cj : ci) && lv < (side ? nvj : nvi)) {
        double* o = (side ? vbj : vbi) + 6 * lv;
        vertex_box(g.rest, g.v_off[body] + lv, g.q0 + 12 * (int64_t)body, g.q1 + 12 * (int64_t)body, g.h, o);
      }
    }
    __syncthreads();
    // products: (vertex of i, tri of j) -> vf(i,.,j,.); (vertex of j, tri of i) -> vf(j,.,i,.); (edge i, edge j)
    for (int prod = 0; prod < 3; ++prod) {
      int ka = prod == 2 ? 1 : 0, kb = prod == 2 ? 1 : 2;
      int ba = prod == 1 ? j : i, bb = prod == 1 ? i : j;
      const double* vba = (prod == 1 ? cj : ci) ? (prod == 1 ? vbj : vbi) : nullptr;
      const double* vbb = (prod == 1 ? ci : cj) ? (prod == 1 ? vbi : vbj) : nullptr;
      int na = prim_count(g, ka, ba), nb = prim_count(g, kb, bb);
      bool is_vf = prod < 2;
      for (int sa = 0; sa < na; sa += BP_TILE) {
        int ca = cull_tile(g, ka, ba, sa, na, obox, vba, ida, bxa, warp_tot);
        if (ca == 0) continue;
        for (int sb = 0; sb < nb; sb += BP_TILE) {
          int cb = cull_tile(g, kb, bb, sb, nb, obox, vbb, idb, bxb, warp_tot);
          if (cb == 0) continue;
          // each thread keeps one box of the larger side in registers and sweeps a
          // chunk of the other side (same smem address across the warp: broadcast)
          const bool a_thr = ca >= cb;
          const int nt = a_thr ? ca : cb, nl = a_thr ? cb : ca;
          const int G = nt >= BP_THREADS ? 1 : BP_THREADS / nt;
          const int Lc = (nl + G - 1) / G;
          const double* own_box = a_thr ? bxa : bxb;
          const double* oth_box = a_thr ? bxb : bxa;
          for (int base = 0; base < nt * G; base += BP_THREADS) {
            const int idx = base + threadIdx.x;
            const int own = idx % nt, chunk = idx / nt;
            const bool live = idx < nt * G;
            double ob[6];
#pragma unroll
            for (int k = 0; k < 6; ++k) ob[k] = live ? own_box[6 * own + k] : 0.0;
            const int y0 = chunk * Lc;
            for (int yy = 0; yy < Lc; ++yy) {
              const int y = y0 + yy;
              bool hit = false;
              if (live && y < nl) {
                const double* b2 = oth_box + 6 * y;
                hit = ob[0] <= b2[3] && b2[0] <= ob[3] && ob[1] <= b2[4] && b2[1] <= ob[4] && ob[2] <= b2[5] &&
                      b2[2] <= ob[5];
              }
              unsigned m = __ballot_sync(0xffffffffu, hit);
              if (m) {
                int lane = threadIdx.x & 31;
                unsigned long long base2 = 0;
                if (lane == __ffs(m) - 1)
                  base2 = atomicAdd(counters + (is_vf ? 0 : 1), (unsigned long long)__popc(m));
                base2 = __shfl_sync(0xffffffffu, base2, __ffs(m) - 1);
                if (hit) {
                  unsigned long long at = base2 + __popc(m & ((1u << lane) - 1));
                  const int x = a_thr ? own : y, yb = a_thr ? y : own;
                  if (is_vf) {
                    if ((int64_t)at < cap_vf) out_vf[at] = make_int4(ba, ida[x], bb, idb[yb]);
                  } else {
                    if ((int64_t)at < cap_ee) out_ee[at] = make_int4(ba, ida[x], bb, idb[yb]);
                  }
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

// ---------------------------------------------------------------------------
// k_prim_pairs2: one CTA per overlapping body pair, few barriers per pair.
//   1. per-pair metadata (offsets, counts, overlap box) and the vertex boxes of
//      both bodies into shared memory;
//   2. ONE pass culls all six primitive lists (verts/edges/tris of i and j)
//      against the overlap box into shared id lists (smem atomics; the final
//      canonical sort makes the output order deterministic);
//   3. per product (VF i->j, VF j->i, EE): the larger side stays in registers
//      (one box per thread), the other side's boxes are materialised once in
//      shared memory and swept with broadcast reads.
// Requires max_v <= P2_VCAP; larger meshes use k_prim_pairs.
constexpr int P2_THREADS = 256;
constexpr int P2_VCAP = 256;
constexpr int P2_HCAP = 1024;  // hits per (pair, product) sorted in shared memory

// box of a primitive from packed local vertex ids (8 bits each, P2_VCAP = 256); vertex
// boxes lie P2_VBS = 7 doubles apart in shared memory: the gathers of a half warp then
// fall into distinct banks for 16 consecutive vertices (6 doubles apart they share 8)
constexpr int P2_VBS = 7;
__device__ __forceinline__ void box_from_packed(int kind, unsigned pk, const double* vb, double* bx) {
  const double* s0 = vb + P2_VBS * (pk & 0xffu);
#pragma unroll
  for (int k = 0; k < 6; ++k) bx[k] = s0[k];
  const int nv = kind == 0 ? 1 : (kind == 1 ? 2 : 3);
  for (int m = 1; m < nv; ++m) {
    const double* sm = vb + P2_VBS * ((pk >> (8 * m)) & 0xffu);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      bx[k] = fmin(bx[k], sm[k]);
      bx[3 + k] = fmax(bx[3 + k], sm[3 + k]);
    }
  }
}

__device__ __forceinline__ void box_from_cache(const PrimGeo& g, int kind, int gid, int v0, const double* vb,
                                               double* bx) {
  if (kind == 0) {
    const double* s0 = vb + 6 * (gid - v0);
#pragma unroll
    for (int k = 0; k < 6; ++k) bx[k] = s0[k];
    return;
  }
  const int nv = kind == 1 ? 2 : 3;
  const int* ids = kind == 1 ? g.edges + 2 * (int64_t)gid : g.tris + 3 * (int64_t)gid;
  const double* s0 = vb + 6 * (ids[0] - v0);
#pragma unroll
  for (int k = 0; k < 6; ++k) bx[k] = s0[k];
  for (int m = 1; m < nv; ++m) {
    const double* sm = vb + 6 * (ids[m] - v0);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      bx[k] = fmin(bx[k], sm[k]);
      bx[3 + k] = fmax(bx[3 + k], sm[3 + k]);
    }
  }
}

// static primitive groups (Scene::grp_*), per kind
struct GrpGeo {
  const int* id[3];
  const unsigned* pk[3];
  const double* box[3];
  const int* off[3];
};

// conservative swept world box of a group's rest AABB (centre c, half extent e)
// under q0 and q1, inflated by h and a rounding margin: it contains the swept box of
// every primitive of the group, so culling against it only prunes
__device__ __forceinline__ void group_box(const double* __restrict__ gb, const double* __restrict__ q0b,
                                          const double* __restrict__ q1b, double h, double* o) {
  double lo[3], hi[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    lo[k] = INFINITY;
    hi[k] = -INFINITY;
  }
  for (int u = 0; u < 2; ++u) {
    const double* q = u ? q1b : q0b;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double a0 = q[3 + 3 * i], a1 = q[4 + 3 * i], a2 = q[5 + 3 * i];
      const double w = q[i] + a0 * gb[0] + a1 * gb[1] + a2 * gb[2];
      const double E = fabs(a0) * gb[3] + fabs(a1) * gb[4] + fabs(a2) * gb[5];
      const double m = 1e-12 * (1.0 + fabs(w) + E);
      lo[i] = fmin(lo[i], w - E - m);
      hi[i] = fmax(hi[i], w + E + m);
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o[k] = lo[k] - h;
    o[3 + k] = hi[k] + h;
  }
}

template <bool RUNS>
__global__ void __launch_bounds__(P2_THREADS, 3)
    k_prim_pairs2(PrimGeo g, GrpGeo gr, int use_groups, int64_t n_ov, const int2* __restrict__ ov,
                  const double* __restrict__ bbox, unsigned long long* counters, int64_t cap_vf, int64_t cap_ee,
                  int4* out_vf, int4* out_ee, int cap_list, int3 cap_k, int2* tab, int* unsorted,
                  int rank, const int* __restrict__ owner,
                  unsigned long long* work, const int* n_ov_dev) {
  if (n_ov_dev) n_ov = *n_ov_dev;  // deferred count (Verlet-list filter result, no host sync)
  const bool no_merge = (use_groups & 2) != 0;  // ABD_BP_NO_MERGE: every pair takes the per-product path (tests)
  use_groups &= 1;
  extern __shared__ double p2_sm[];
  double* vb = p2_sm;                        // [2][P2_VCAP][P2_VBS] vertex boxes of i and j
  double* obx = vb + 2 * P2_VBS * P2_VCAP;   // [cap_list][6] materialised boxes (one product at a time)
  // survivor lists (list l = 3 side + kind) with per-kind capacities cap_k = (V, E, T)
  const int ltot = 2 * (cap_k.x + cap_k.y + cap_k.z);
  int* lists = reinterpret_cast<int*>(obx + 6 * (size_t)cap_list);  // [ltot] local ids
  unsigned* lpk = reinterpret_cast<unsigned*>(lists + ltot);  // packed local vertex ids
  unsigned* hk = lpk + ltot;  // [P2_HCAP] hits of the current product
#define LOFF(l) ((l) / 3 * (cap_k.x + cap_k.y + cap_k.z) + ((l) % 3 > 0 ? cap_k.x : 0) + ((l) % 3 > 1 ? cap_k.y : 0))
  // runs: the survivors of one static group are contiguous in their list; run k of
  // list l covers [run_s, run_s + run_n) and carries a conservative float box of its
  // survivors, so a product only pairs runs whose boxes overlap
  __shared__ int nrun[6];
  __shared__ unsigned short run_s[6][32], run_n[6][32];
  __shared__ float run_b[6][32][6];
  __shared__ unsigned tmask[32];
  __shared__ int runs_ok;
  __shared__ int hcount;
  __shared__ unsigned long long hbase;
  __shared__ int meta[16];  // v0,e0,t0 (i) | v0,e0,t0 (j) | nv,ne,nt (i) | nv,ne,nt (j)
  __shared__ int lcount[6];
  __shared__ double obox[6];
  __shared__ int gfirst[6], gcount[6], ghits;
  __shared__ int hitg[256];
  // pairs are handed out dynamically (their costs vary by orders of magnitude);
  // multi-GPU (owner != null): this rank takes the overlap pairs of its slab -- the
  // slab of the lower body, or of the higher one when the lower is kinematic
  // (table rows of the other ranks' pairs stay 0)
  __shared__ long long next_k;
  __shared__ int pcnt[2];              // merged products: hits of products 0 and 1
  __shared__ unsigned long long hbase2;  // merged products: base of the EE chunk
  // thread 0 takes the following pair's index while the current pair is processed (the
  // atomic's round trip is off the per-pair chain)
  long long ahead = threadIdx.x == 0 ? (long long)atomicAdd(work, 1ull) : 0;
  for (;;) {
    if (threadIdx.x == 0) next_k = ahead;
    __syncthreads();
    const int64_t pi = next_k;
    if (pi >= n_ov) break;
    if (threadIdx.x == 0) ahead = (long long)atomicAdd(work, 1ull);
    const int2 pr = ov[pi];
    const int bi = pr.x, bj = pr.y;
    if (owner) {
      const int olo = owner[min(bi, bj)], ohi = owner[max(bi, bj)];
      if ((olo >= 0 ? olo : ohi) != rank) {
        __syncthreads();  // every thread has read next_k before thread 0 takes the next pair
        continue;
      }
    }
    if (threadIdx.x < 6) {
      const int side = threadIdx.x / 3, kind = threadIdx.x % 3;
      const int body = side ? bj : bi;
      const int* o = kind == 0 ? g.v_off : (kind == 1 ? g.e_off : g.t_off);
      const int a = o[body], b = o[body + 1];
      meta[3 * side + kind] = a;
      meta[6 + 3 * side + kind] = b - a;
      lcount[threadIdx.x] = 0;
      if (threadIdx.x == 0 && !use_groups) runs_ok = 0;  // (thread 64 writes it otherwise)
      if (threadIdx.x == 1) {  // merged products (hcount is dead: read before the last hbase barrier)
        hcount = 0;
        pcnt[0] = 0;
        pcnt[1] = 0;
      }
    } else if (threadIdx.x >= 32 && threadIdx.x < 35) {
      const int k = threadIdx.x - 32;
      obox[k] = fmax(bbox[6 * bi + k], bbox[6 * bj + k]);
      obox[3 + k] = fmin(bbox[6 * bi + 3 + k], bbox[6 * bj + 3 + k]);
    } else if (use_groups && threadIdx.x >= 64 && threadIdx.x < 70) {
      const int l = threadIdx.x - 64, side = l / 3, kind = l % 3;
      const int body = side ? bj : bi;
      const int a = gr.off[kind][body];
      gfirst[l] = a;
      gcount[l] = gr.off[kind][body + 1] - a;
      nrun[l] = 0;
      if (l == 0) {
        ghits = 0;
        runs_ok = RUNS ? 1 : 0;
      }
    }
    __syncthreads();
    // cull in two stages: (a) the static groups of 32 primitives of the six lists
    // against the overlap box (conservative swept boxes of their rest AABBs); (b) the
    // primitives of the surviving groups, one warp per group.  Stage (a) needs no vertex
    // box, so it shares one phase (one barrier) with the vertex boxes of both bodies: the
    // work items are the nv_i + nv_j vertices followed by the groups.
    const bool grouped = use_groups && gcount[0] + gcount[1] + gcount[2] + gcount[3] + gcount[4] + gcount[5] <= 256;
    {
      const int nvi = meta[6], nvj = meta[9];
      const int gt = grouped ? gcount[0] + gcount[1] + gcount[2] + gcount[3] + gcount[4] + gcount[5] : 0;
      for (int t = threadIdx.x; t < nvi + nvj + gt; t += P2_THREADS) {
        if (t < nvi + nvj) {
          const int side = t >= nvi, lv = side ? t - nvi : t;
          const int body = side ? bj : bi;
          vertex_box(g.rest, meta[3 * side] + lv, g.q0 + 12 * (int64_t)body, g.q1 + 12 * (int64_t)body, g.h,
                     vb + P2_VBS * (side * P2_VCAP + lv));
        } else {
          int l = 0, r = t - nvi - nvj;
          while (r >= gcount[l]) {
            r -= gcount[l];
            ++l;
          }
          const int side = l / 3, kind = l % 3, body = side ? bj : bi;
          double gb[6];
          group_box(gr.box[kind] + 6 * (int64_t)(gfirst[l] + r), g.q0 + 12 * (int64_t)body,
                    g.q1 + 12 * (int64_t)body, g.h, gb);
          const bool hit = gb[0] <= obox[3] && obox[0] <= gb[3] && gb[1] <= obox[4] && obox[1] <= gb[4] &&
                           gb[2] <= obox[5] && obox[2] <= gb[5];
          if (hit) hitg[atomicAdd(&ghits, 1)] = (l << 16) | r;
        }
      }
    }
    __syncthreads();
    if (grouped) {
      const int lane = threadIdx.x & 31;
      for (int u = threadIdx.x >> 5; u < ghits; u += P2_THREADS / 32) {
        const int l = hitg[u] >> 16, r = hitg[u] & 0xffff;
        const int side = l / 3, kind = l % 3;
        const int i = 32 * r + lane;
        bool keep = false;
        unsigned pk = 0;
        int id = 0;
        double bxs[6];
        if (i < meta[6 + l]) {
          const int64_t gi = (int64_t)meta[l] + i;  // prim offset of the body (grouped order)
          pk = gr.pk[kind][gi];
          id = gr.id[kind][gi];
          box_from_packed(kind, pk, vb + P2_VBS * side * P2_VCAP, bxs);
          keep = bxs[0] <= obox[3] && obox[0] <= bxs[3] && bxs[1] <= obox[4] && obox[1] <= bxs[4] &&
                 bxs[2] <= obox[5] && obox[2] <= bxs[5];
        }
        // the whole warp works on one group (one list): one shared-memory atomic per warp
        const unsigned m = __ballot_sync(0xffffffffu, keep);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(&lcount[l], __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
          const int at = base + __popc(m & ((1u << lane) - 1));
          lists[LOFF(l) + at] = id;
          lpk[LOFF(l) + at] = pk;
        }
        if (RUNS && m) {
          // the run's box: union of its survivors' boxes, rounded outward to float
          double lo0 = keep ? bxs[0] : INFINITY, lo1 = keep ? bxs[1] : INFINITY, lo2 = keep ? bxs[2] : INFINITY;
          double hi0 = keep ? bxs[3] : -INFINITY, hi1 = keep ? bxs[4] : -INFINITY, hi2 = keep ? bxs[5] : -INFINITY;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            lo0 = fmin(lo0, __shfl_xor_sync(0xffffffffu, lo0, o));
            lo1 = fmin(lo1, __shfl_xor_sync(0xffffffffu, lo1, o));
            lo2 = fmin(lo2, __shfl_xor_sync(0xffffffffu, lo2, o));
            hi0 = fmax(hi0, __shfl_xor_sync(0xffffffffu, hi0, o));
            hi1 = fmax(hi1, __shfl_xor_sync(0xffffffffu, hi1, o));
            hi2 = fmax(hi2, __shfl_xor_sync(0xffffffffu, hi2, o));
          }
          if (lane == 0) {
            const int k = atomicAdd(&nrun[l], 1);
            if (k < 32) {
              run_s[l][k] = (unsigned short)base;
              run_n[l][k] = (unsigned short)__popc(m);
              run_b[l][k][0] = __double2float_rd(lo0);
              run_b[l][k][1] = __double2float_rd(lo1);
              run_b[l][k][2] = __double2float_rd(lo2);
              run_b[l][k][3] = __double2float_ru(hi0);
              run_b[l][k][4] = __double2float_ru(hi1);
              run_b[l][k][5] = __double2float_ru(hi2);
            } else {
              runs_ok = 0;
            }
          }
        }
      }
    } else  // one cull pass over the six lists (list id = 3 * side + kind); topology is
    // prefetched 4 primitives per thread, survivors keep id + packed local vertex ids
    {
      if (threadIdx.x == 0) runs_ok = 0;  // no runs on this path
      const int tot = meta[6] + meta[7] + meta[8] + meta[9] + meta[10] + meta[11];
      for (int t0 = threadIdx.x; t0 < tot; t0 += 4 * P2_THREADS) {
        unsigned pk[4];
        int lst[4], loc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 + u * P2_THREADS;
          lst[u] = -1;
          loc[u] = 0;
          pk[u] = 0;
          if (t < tot) {
            int l = 0, r = t;
            while (r >= meta[6 + l]) {
              r -= meta[6 + l];
              ++l;
            }
            const int side = l / 3, kind = l % 3, v0 = meta[3 * side];
            lst[u] = l;
            loc[u] = r;
            if (kind == 0) {
              pk[u] = (unsigned)r;
            } else if (kind == 1) {
              const int2 e = *reinterpret_cast<const int2*>(g.edges + 2 * (int64_t)(meta[l] + r));
              pk[u] = (unsigned)(e.x - v0) | ((unsigned)(e.y - v0) << 8);
            } else {
              const int* tr = g.tris + 3 * (int64_t)(meta[l] + r);
              pk[u] = (unsigned)(tr[0] - v0) | ((unsigned)(tr[1] - v0) << 8) | ((unsigned)(tr[2] - v0) << 16);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (lst[u] < 0) continue;
          const int l = lst[u], side = l / 3, kind = l % 3;
          double bx[6];
          box_from_packed(kind, pk[u], vb + P2_VBS * side * P2_VCAP, bx);
          const bool keep = bx[0] <= obox[3] && obox[0] <= bx[3] && bx[1] <= obox[4] && obox[1] <= bx[4] &&
                            bx[2] <= obox[5] && obox[2] <= bx[5];
          if (keep) {
            const int at = atomicAdd(&lcount[l], 1);
            lists[LOFF(l) + at] = loc[u];
            lpk[LOFF(l) + at] = pk[u];
          }
        }
      }
    }
    __syncthreads();
    // products: (verts i, tris j) -> vf(i,.,j,.); (verts j, tris i) -> vf(j,.,i,.); (edges i, edges j)
    //
    // Small pairs (the pile's common case: ~120 survivors, ~1,500 box tests) take the three
    // products in ONE pass: every survivor's box is materialised once, the tests of the
    // three products are dealt to the threads as one flat range, the hits carry their
    // product in the key's top bits (so one sort gives the (product, prim_a, prim_b)
    // order), and one pair of global atomics reserves the VF and EE chunks: 3 barriers
    // and one atomic round trip per pair instead of 9 and 3.
    bool merged = false;
    {
      const int c0 = lcount[0], c1 = lcount[1], c2 = lcount[2], c3 = lcount[3], c4 = lcount[4], c5 = lcount[5];
      const int T0 = c0 * c5, T1 = c3 * c2, T2 = c1 * c4;  // (la, lb) = (0, 5), (3, 2), (1, 4)
      const int nbox = c0 + c1 + c2 + c3 + c4 + c5, TT = T0 + T1 + T2;
      const bool use_runs_any = RUNS && runs_ok != 0 && (T0 >= 4096 || T1 >= 4096 || T2 >= 4096);
      if (!no_merge && TT > 0 && TT <= 32 * P2_THREADS && nbox <= cap_list && !use_runs_any && cap_k.y <= 16384 &&
          cap_k.z <= 16384) {  // uniform
        const int o1 = c0, o2 = o1 + c1, o3 = o2 + c2, o4 = o3 + c3, o5 = o4 + c4;
        for (int t = threadIdx.x; t < nbox; t += P2_THREADS) {
          const int l = t < o1 ? 0 : (t < o2 ? 1 : (t < o3 ? 2 : (t < o4 ? 3 : (t < o5 ? 4 : 5))));
          const int ol = l == 0 ? 0 : (l == 1 ? o1 : (l == 2 ? o2 : (l == 3 ? o3 : (l == 4 ? o4 : o5))));
          box_from_packed(l % 3, lpk[LOFF(l) + (t - ol)], vb + P2_VBS * (l / 3) * P2_VCAP, obx + 6 * t);
        }
        __syncthreads();
        const int lane = threadIdx.x & 31;
        for (int base = 0; base < TT; base += P2_THREADS) {
          const int idx = base + threadIdx.x;
          bool hit = false;
          int pr_ = 0, a = 0, b = 0;
          if (idx < TT) {
            pr_ = idx < T0 ? 0 : (idx < T0 + T1 ? 1 : 2);
            const int loc = idx - (pr_ == 0 ? 0 : (pr_ == 1 ? T0 : T0 + T1));
            const int nb = pr_ == 0 ? c5 : (pr_ == 1 ? c2 : c4);
            a = loc / nb;
            b = loc - a * nb;
            const double2* A = reinterpret_cast<const double2*>(obx + 6 * ((pr_ == 0 ? 0 : (pr_ == 1 ? o3 : o1)) + a));
            const double2* B = reinterpret_cast<const double2*>(obx + 6 * ((pr_ == 0 ? o5 : (pr_ == 1 ? o2 : o4)) + b));
            const double2 a0 = A[0], a1 = A[1], a2 = A[2], b0 = B[0], b1 = B[1], b2 = B[2];
            hit = (a0.x <= b1.y) & (b0.x <= a1.y) & (a0.y <= b2.x) & (b0.y <= a2.x) & (a1.x <= b2.y) &
                  (b1.x <= a2.y);
          }
          const unsigned m = __ballot_sync(0xffffffffu, hit);
          if (m) {  // warp-uniform
            const unsigned m0 = __ballot_sync(0xffffffffu, hit && pr_ == 0);
            const unsigned m1 = __ballot_sync(0xffffffffu, hit && pr_ == 1);
            const int lead = __ffs(m) - 1;
            int at0 = 0;
            if (lane == lead) {
              at0 = atomicAdd(&hcount, __popc(m));
              if (m0) atomicAdd(&pcnt[0], __popc(m0));
              if (m1) atomicAdd(&pcnt[1], __popc(m1));
            }
            at0 = __shfl_sync(0xffffffffu, at0, lead);
            if (hit) {
              const int at = at0 + __popc(m & ((1u << lane) - 1));
              const int la = pr_ == 0 ? 0 : (pr_ == 1 ? 3 : 1), lb = pr_ == 0 ? 5 : (pr_ == 1 ? 2 : 4);
              const unsigned pa = (unsigned)lists[LOFF(la) + a], pb = (unsigned)lists[LOFF(lb) + b];
              if (at < P2_HCAP) hk[at] = ((unsigned)pr_ << 28) | (pa << 14) | pb;
            }
          }
        }
        __syncthreads();
        const int cnt = hcount;
        if (cnt <= P2_HCAP) {  // uniform
          merged = true;
          const int n0 = pcnt[0], n1 = pcnt[1], n01 = n0 + n1;
          if (threadIdx.x == 0) {
            const unsigned long long bv = n01 ? atomicAdd(counters + 0, (unsigned long long)n01) : 0ull;
            const unsigned long long be = cnt - n01 ? atomicAdd(counters + 1, (unsigned long long)(cnt - n01)) : 0ull;
            hbase = bv;
            hbase2 = be;
            tab[3 * pi + 0] = make_int2((int)bv, n0);
            tab[3 * pi + 1] = make_int2((int)bv + n0, n1);
            tab[3 * pi + 2] = make_int2((int)be, cnt - n01);
          }
          if (cnt > 256) {
            // larger chunks: bitonic sort in shared memory
            int P2 = 1;
            while (P2 < cnt) P2 <<= 1;
            for (int t = cnt + threadIdx.x; t < P2; t += P2_THREADS) hk[t] = 0xffffffffu;
            __syncthreads();
            for (int k = 2; k <= P2; k <<= 1)
              for (int jj = k >> 1; jj > 0; jj >>= 1) {
                for (int t = threadIdx.x; t < P2; t += P2_THREADS) {
                  const int u = t ^ jj;
                  if (u > t) {
                    const bool up = (t & k) == 0;
                    const unsigned x = hk[t], y = hk[u];
                    if ((x > y) == up) {
                      hk[t] = y;
                      hk[u] = x;
                    }
                  }
                }
                __syncthreads();
              }
          } else {
            __syncthreads();  // hbase / hbase2 visible
          }
          const unsigned long long bv = hbase, be = hbase2;
          for (int t = threadIdx.x; t < cnt; t += P2_THREADS) {
            const unsigned key = hk[t];
            int rank = t;
            if (cnt <= 256) {  // order by rank (unique keys): one pass of broadcast reads
              rank = 0;
              for (int u = 0; u < cnt; ++u) rank += hk[u] < key;
            }
            const int pq = (int)(key >> 28), pa = (int)((key >> 14) & 0x3fffu), pb = (int)(key & 0x3fffu);
            const int body_a = pq == 1 ? bj : bi, body_b = pq == 1 ? bi : bj;
            if (pq < 2) {
              const unsigned long long g2 = bv + (unsigned long long)rank;
              if ((int64_t)g2 < cap_vf) out_vf[g2] = make_int4(body_a, pa, body_b, pb);
            } else {
              const unsigned long long g2 = be + (unsigned long long)(rank - n01);
              if ((int64_t)g2 < cap_ee) out_ee[g2] = make_int4(body_a, pa, body_b, pb);
            }
          }
          // no barrier: hk, hbase, pcnt and hcount are rewritten only after the next pair's barriers
        } else {
          __syncthreads();  // every thread has read hcount before the per-product path resets it
        }
      }
    }
    if (!merged)
    for (int prod = 0; prod < 3; ++prod) {
      const int la = prod == 0 ? 0 : (prod == 1 ? 3 : 1);  // list of side a
      const int lb = prod == 0 ? 5 : (prod == 1 ? 2 : 4);  // list of side b
      const int ca = lcount[la], cb = lcount[lb];
      if (ca == 0 || cb == 0) {  // uniform across the CTA
        if (threadIdx.x == 0) tab[3 * pi + prod] = make_int2(0, 0);
        continue;
      }
      const int ka = la % 3, kb = lb % 3, sa = la / 3, sb = lb / 3;
      const bool a_thr = ca >= cb;  // thread side = a
      const int nt = a_thr ? ca : cb, nl = a_thr ? cb : ca;
      const int lt = a_thr ? la : lb, ll = a_thr ? lb : la;
      const int kt = a_thr ? ka : kb, kl = a_thr ? kb : ka;
      const int st_ = a_thr ? sa : sb, sl = a_thr ? sb : sa;
      // hcount of the previous product is dead here: every thread read it into cnt
      // before that product's hbase barrier, which thread 0 has passed
      if (threadIdx.x == 0) hcount = 0;
      // materialise the loop side's boxes
      for (int t = threadIdx.x; t < nl; t += P2_THREADS)
        box_from_packed(kl, lpk[LOFF(ll) + t], vb + P2_VBS * sl * P2_VCAP, obx + 6 * t);
      // run-pair mask: bit j of tmask[k] = run k of the thread side meets run j of the loop side
      // (only for large products: for small ones the plain warp-synchronous sweep wins)
      const bool use_runs = RUNS && runs_ok != 0 && nt * nl >= 4096;  // uniform
      const int nrt = use_runs ? min(nrun[lt], 32) : 0, nrl = use_runs ? min(nrun[ll], 32) : 1;
      if (RUNS && use_runs) {
        for (int t = threadIdx.x; t < 32; t += P2_THREADS) tmask[t] = 0u;
        __syncthreads();
        for (int t = threadIdx.x; t < nrt * nrl; t += P2_THREADS) {
          const int k = t / nrl, j = t % nrl;
          const float* A = run_b[lt][k];
          const float* B = run_b[ll][j];
          if (A[0] <= B[3] && B[0] <= A[3] && A[1] <= B[4] && B[1] <= A[4] && A[2] <= B[5] && B[2] <= A[5])
            atomicOr(&tmask[k], 1u << j);
        }
      }
      __syncthreads();
      const bool is_vf = prod < 2;
      const int body_a = prod == 1 ? bj : bi, body_b = prod == 1 ? bi : bj;
      const int G = nt >= P2_THREADS ? 1 : P2_THREADS / nt;
      const int Lc = (nl + G - 1) / G;
      // pass 0: hits into shared memory; pass 1 (only when they overflow P2_HCAP):
      // straight into the reserved chunk, which is then flagged for a global sort
      for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
          if (hcount <= P2_HCAP) break;  // uniform
          __syncthreads();
          if (threadIdx.x == 0) hcount = 0;
          __syncthreads();
        }
        if (RUNS && use_runs && pass == 0) {
          // filtered: each (own, chunk) thread walks only the loop-side runs its own
          // run's box meets; runs of disjoint boxes hold no overlapping primitive pair
          for (int base = 0; base < nt * G; base += P2_THREADS) {
            const int idx = base + threadIdx.x;
            if (idx >= nt * G) break;
            const int own = idx % nt, chunk = idx / nt;
            int kr = 0;  // the run holding own (runs are appended in any order)
            for (int k = 0; k < nrt; ++k)
              if (own >= run_s[lt][k] && own < run_s[lt][k] + run_n[lt][k]) kr = k;
            double ob[6];
            const int own_local = lists[LOFF(lt) + own];
            box_from_packed(kt, lpk[LOFF(lt) + own], vb + P2_VBS * st_ * P2_VCAP, ob);
            unsigned mk = tmask[kr];
            int cyc = 0;  // position in this thread's filtered sequence mod G (chunks take every G-th)
            while (mk) {
              const int j = __ffs(mk) - 1;
              mk &= mk - 1;
              const int y0 = run_s[ll][j], y1 = y0 + run_n[ll][j];
              for (int y = y0; y < y1; ++y) {
                const bool mine = cyc == chunk;
                if (++cyc == G) cyc = 0;
                if (!mine) continue;
                const double* b2 = obx + 6 * y;
                if (ob[0] <= b2[3] && b2[0] <= ob[3] && ob[1] <= b2[4] && b2[1] <= ob[4] && ob[2] <= b2[5] &&
                    b2[2] <= ob[5]) {
                  const int at = atomicAdd(&hcount, 1);
                  const int yl = lists[LOFF(ll) + y];
                  const int pa = a_thr ? own_local : yl, pb = a_thr ? yl : own_local;
                  if (at < P2_HCAP) hk[at] = ((unsigned)pa << 16) | (unsigned)pb;
                }
              }
            }
          }
        } else
        for (int base = 0; base < nt * G; base += P2_THREADS) {
          const int idx = base + threadIdx.x;
          const bool live = idx < nt * G;
          const int own = live ? idx % nt : 0, chunk = idx / nt;
          double ob[6];
          const int own_local = live ? lists[LOFF(lt) + own] : 0;
          if (live) box_from_packed(kt, lpk[LOFF(lt) + own], vb + P2_VBS * st_ * P2_VCAP, ob);
          const int y0 = chunk * Lc;
          for (int yy = 0; yy < Lc; ++yy) {
            const int y = y0 + yy;
            bool hit = false;
            if (live && y < nl) {
              // the box as three 16-byte broadcast loads: (lo0, lo1) (lo2, hi0) (hi1, hi2)
              const double2* b2 = reinterpret_cast<const double2*>(obx + 6 * y);
              const double2 u0 = b2[0], u1 = b2[1], u2 = b2[2];
              hit = (ob[0] <= u1.y) & (u0.x <= ob[3]) & (ob[1] <= u2.x) & (u0.y <= ob[4]) & (ob[2] <= u2.y) &
                    (u1.x <= ob[5]);
            }
            const unsigned m = __ballot_sync(0xffffffffu, hit);
            if (m) {
              const int lane = threadIdx.x & 31;
              int b0 = 0;
              if (lane == __ffs(m) - 1) b0 = atomicAdd(&hcount, __popc(m));
              b0 = __shfl_sync(0xffffffffu, b0, __ffs(m) - 1);
              if (hit) {
                const int at = b0 + __popc(m & ((1u << lane) - 1));
                const int yl = lists[LOFF(ll) + y];
                const int pa = a_thr ? own_local : yl, pb = a_thr ? yl : own_local;
                if (pass == 0) {
                  if (at < P2_HCAP) hk[at] = ((unsigned)pa << 16) | (unsigned)pb;
                } else {
                  const unsigned long long g2 = hbase + (unsigned long long)at;
                  if (is_vf) {
                    if ((int64_t)g2 < cap_vf) out_vf[g2] = make_int4(body_a, pa, body_b, pb);
                  } else {
                    if ((int64_t)g2 < cap_ee) out_ee[g2] = make_int4(body_a, pa, body_b, pb);
                  }
                }
              }
            }
          }
        }
        __syncthreads();
        if (pass == 0) {
          const int cnt = hcount;
          if (threadIdx.x == 0) {
            hbase = cnt ? atomicAdd(counters + (is_vf ? 0 : 1), (unsigned long long)cnt) : 0ull;
            tab[3 * pi + prod] = make_int2((int)hbase, cnt);
            if (cnt > P2_HCAP) atomicExch(unsorted, 1);
          }
          __syncthreads();  // hbase visible to the whole CTA
          if (cnt > 0 && cnt <= 256) {
            // deterministic in-chunk order by rank (keys are unique (prim_a, prim_b)):
            // one pass, broadcast smem reads, no barrier ladder
            const unsigned long long b0 = hbase;
            for (int t = threadIdx.x; t < cnt; t += P2_THREADS) {
              const unsigned key = hk[t];
              int rank = 0;
              for (int u = 0; u < cnt; ++u) rank += hk[u] < key;
              const unsigned long long g2 = b0 + (unsigned long long)rank;
              const int pa = (int)(key >> 16), pb = (int)(key & 0xffffu);
              if (is_vf) {
                if ((int64_t)g2 < cap_vf) out_vf[g2] = make_int4(body_a, pa, body_b, pb);
              } else {
                if ((int64_t)g2 < cap_ee) out_ee[g2] = make_int4(body_a, pa, body_b, pb);
              }
            }
          } else if (cnt > 256 && cnt <= P2_HCAP) {
            // larger chunks: bitonic sort in shared memory
            int P2 = 1;
            while (P2 < cnt) P2 <<= 1;
            for (int t = cnt + threadIdx.x; t < P2; t += P2_THREADS) hk[t] = 0xffffffffu;
            __syncthreads();
            for (int k = 2; k <= P2; k <<= 1)
              for (int jj = k >> 1; jj > 0; jj >>= 1) {
                for (int t = threadIdx.x; t < P2; t += P2_THREADS) {
                  const int u = t ^ jj;
                  if (u > t) {
                    const bool up = (t & k) == 0;
                    const unsigned a = hk[t], b = hk[u];
                    if ((a > b) == up) {
                      hk[t] = b;
                      hk[u] = a;
                    }
                  }
                }
                __syncthreads();
              }
            const unsigned long long b0 = hbase;
            for (int t = threadIdx.x; t < cnt; t += P2_THREADS) {
              const unsigned long long g2 = b0 + (unsigned long long)t;
              const int pa = (int)(hk[t] >> 16), pb = (int)(hk[t] & 0xffffu);
              if (is_vf) {
                if ((int64_t)g2 < cap_vf) out_vf[g2] = make_int4(body_a, pa, body_b, pb);
              } else {
                if ((int64_t)g2 < cap_ee) out_ee[g2] = make_int4(body_a, pa, body_b, pb);
              }
            }
          }
          // no barrier: the output only reads hk / hbase, which the next product
          // rewrites after its materialise barrier and hbase barrier respectively
        }
      }
    }
  }
}

__global__ void k_ov_in_pattern(int64_t n, const int2* __restrict__ ov, const int* __restrict__ slot, int64_t n_off,
                                const int2* __restrict__ keys, int* inside, const int* n_dev) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (n_dev) n = *n_dev;
  if (i >= n) return;
  const int sa = slot[ov[i].x], sb = slot[ov[i].y];
  if (sa < 0 || sb < 0 || sa == sb) return;  // no block for pairs with a kinematic body
  const int a = min(sa, sb), b = max(sa, sb);
  int64_t lo = 0, hi = n_off - 1;
  while (lo <= hi) {
    int64_t m = (lo + hi) >> 1;
    const int2 k = keys[m];
    if (k.x < a || (k.x == a && k.y < b)) lo = m + 1;
    else if (k.x == a && k.y == b) return;
    else hi = m - 1;
  }
  *inside = 0;
}

// Chunks to their final offsets in ONE launch (chunk counts, the two prefix sums and the
// two moves used to be nine launches of tiny kernels -- ~45 us of launch latency per broad
// phase).  A CTA owns CG_PAIRS consecutive body pairs: it sums the chunk counts of all
// pairs before its first one (the table is a few hundred KB in L2), scans its own pairs'
// counts, and its warps copy the chunks.  Offsets = the exclusive prefix sums in (pair,
// product) order, as before.
constexpr int CG_PAIRS = 32, CG_THREADS = 256;
__global__ void __launch_bounds__(CG_THREADS) k_chunk_gather(int n_ov, const int2* __restrict__ tab,
                                                             const int4* __restrict__ src_vf, int4* dst_vf,
                                                             const int4* __restrict__ src_ee, int4* dst_ee) {
  __shared__ int red_vf[CG_THREADS / 32], red_ee[CG_THREADS / 32];
  __shared__ int off_s[3 * CG_PAIRS];
  const int p0 = blockIdx.x * CG_PAIRS;
  const int np = min(CG_PAIRS, n_ov - p0);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // counts before this CTA's first pair
  int svf = 0, see = 0;
  for (int i = threadIdx.x; i < 3 * p0; i += CG_THREADS) {
    const int c = tab[i].y;
    if (i % 3 == 2) see += c;
    else svf += c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    svf += __shfl_xor_sync(0xffffffffu, svf, o);
    see += __shfl_xor_sync(0xffffffffu, see, o);
  }
  if (lane == 0) {
    red_vf[wid] = svf;
    red_ee[wid] = see;
  }
  __syncthreads();
  if (wid == 0) {
    // one warp: bases, then the exclusive scans over this CTA's pairs (lane = pair)
    int bvf = 0, bee = 0;
#pragma unroll
    for (int k = 0; k < CG_THREADS / 32; ++k) {
      bvf += red_vf[k];
      bee += red_ee[k];
    }
    const int c0 = lane < np ? tab[3 * (p0 + lane)].y : 0;
    const int c1 = lane < np ? tab[3 * (p0 + lane) + 1].y : 0;
    const int c2 = lane < np ? tab[3 * (p0 + lane) + 2].y : 0;
    int ivf = c0 + c1, iee = c2;  // inclusive scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, ivf, o), b = __shfl_up_sync(0xffffffffu, iee, o);
      if (lane >= o) {
        ivf += a;
        iee += b;
      }
    }
    off_s[3 * lane] = bvf + ivf - (c0 + c1);
    off_s[3 * lane + 1] = bvf + ivf - c1;
    off_s[3 * lane + 2] = bee + iee - c2;
  }
  __syncthreads();
  for (int ch = wid; ch < 3 * np; ch += CG_THREADS / 32) {
    const int2 e = tab[3 * p0 + ch];
    const int d = off_s[ch];
    if (ch % 3 == 2) {
      for (int k = lane; k < e.y; k += 32) dst_ee[d + k] = src_ee[e.x + k];
    } else {
      for (int k = lane; k < e.y; k += 32) dst_vf[d + k] = src_vf[e.x + k];
    }
  }
}

// chunk table -> per-list counts in (pair, product) order
__global__ void k_chunk_counts(int64_t n_ov, const int2* __restrict__ tab, int* cnt_vf, int* cnt_ee) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n_ov) return;
  cnt_vf[2 * p] = tab[3 * p].y;
  cnt_vf[2 * p + 1] = tab[3 * p + 1].y;
  cnt_ee[p] = tab[3 * p + 2].y;
}

// move every chunk to its final offset (warp per chunk)
__global__ void k_chunk_move(int64_t n_ov, const int2* __restrict__ tab, int prod_lo, int nprod,
                             const int* __restrict__ dst_off, const int4* __restrict__ src, int4* dst) {
  int64_t wgl = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (wgl >= n_ov * nprod) return;
  const int64_t p = wgl / nprod;
  const int pr = prod_lo + (int)(wgl % nprod);
  const int2 e = tab[3 * p + pr];
  const int d = dst_off[wgl];
  for (int k = lane; k < e.y; k += 32) dst[d + k] = src[e.x + k];
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

// 7 bits per axis (wraps every 128 cells: aliased cells only add exact box tests);
// "large" bodies get CELL_LARGE, so the keys fit 22 bits (3 radix passes)
constexpr uint32_t CELL_LARGE = 1u << 21;
constexpr int CELL_KEY_BITS = 22;
__device__ __forceinline__ uint32_t cell_key(long long ix, long long iy, long long iz) {
  return (((uint32_t)ix & 127u) << 14) | (((uint32_t)iy & 127u) << 7) | ((uint32_t)iz & 127u);
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
    keys[b] = CELL_LARGE;  // large: not binned
    return;
  }
  keys[b] = cell_key((long long)floor(x[0] / cell), (long long)floor(x[1] / cell), (long long)floor(x[2] / cell));
}

// cell size in one CTA: median of up to 2048 strided extent samples (bitonic
// sort in shared memory), then the largest extent <= 4x that median, next float
// up (outliers such as ground slabs and walls become "large").  The cell only
// steers the binning; overlap decisions are exact box tests.
__global__ void __launch_bounds__(1024) k_cell_size(int B, const uint32_t* __restrict__ ext, double* cell_out) {
  __shared__ uint32_t sk[2048];
  __shared__ uint32_t red[32];
  const int ns = min(B, 2048);
  for (int t = threadIdx.x; t < 2048; t += 1024)
    sk[t] = t < ns ? ext[(int64_t)t * B / ns] : 0xffffffffu;
  __syncthreads();
  for (int k = 2; k <= 2048; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < 2048; t += 1024) {
        int u = t ^ j;
        if (u > t) {
          bool up = (t & k) == 0;
          uint32_t a = sk[t], b = sk[u];
          if ((a > b) == up) {
            sk[t] = b;
            sk[u] = a;
          }
        }
      }
      __syncthreads();
    }
  const uint32_t lim = __float_as_uint(4.0f * __uint_as_float(sk[(ns - 1) / 2]));
  uint32_t best = 0;
  for (int b = threadIdx.x; b < B; b += 1024) {
    uint32_t e = ext[b];
    if (e <= lim && e > best) best = e;
  }
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = red[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (threadIdx.x == 0) {
      double cell = (double)__uint_as_float(best + 1u);
      if (!(cell > 0.0)) cell = 1.0;
      *cell_out = cell;
    }
  }
}

__global__ void k_cell_keys2(int B, const double* __restrict__ bbox, const double* __restrict__ cell_p,
                             uint32_t* keys, int* vals) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double cell = *cell_p;
  const double* x = bbox + 6 * b;
  double e = fmax(fmax(x[3] - x[0], x[4] - x[1]), x[5] - x[2]);
  vals[b] = b;
  if (e > cell) {
    keys[b] = CELL_LARGE;  // large: not binned
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

// one thread per (body, x column of cells): emit (min, max) overlapping pairs
// exactly once (an overlapping body's low corner lies in exactly one cell)
constexpr int GP_COLS = 4;  // x columns per body: floor(hi/c) - floor(lo/c - 1 - eps) <= 3 for extent <= c
__global__ void k_grid_pairs(int B, const double* __restrict__ bbox, const unsigned char* __restrict__ dyn,
                             const uint32_t* __restrict__ skeys, const int* __restrict__ sbody, int n_small,
                             const double* __restrict__ cell_p, unsigned long long* count, int64_t cap, int2* out) {
  const int64_t item = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (item >= (int64_t)B * GP_COLS) return;
  const int i = (int)(item / GP_COLS), dxc = (int)(item % GP_COLS);
  const double cell = *cell_p;
  const double* a = bbox + 6 * i;
  double e = fmax(fmax(a[3] - a[0], a[4] - a[1]), a[5] - a[2]);
  // pairs involving a large body come from k_large_pairs
  if (e > cell) return;
  // an overlapping small body has lo_j in [lo_i - cell, hi_i]; floor(lo/cell) is
  // monotone in lo, and the 1e-9 margin absorbs the rounding of lo_i/cell - 1
  long long x0 = (long long)floor(a[0] / cell - 1.0 - 1e-9), x1 = (long long)floor(a[3] / cell);
  long long y0 = (long long)floor(a[1] / cell - 1.0 - 1e-9), y1 = (long long)floor(a[4] / cell);
  long long z0 = (long long)floor(a[2] / cell - 1.0 - 1e-9), z1 = (long long)floor(a[5] / cell);
  const long long cx = x0 + dxc;
  const bool last = dxc == GP_COLS - 1;
  if (cx > x1) return;
  const long long cx_end = last ? x1 : cx;  // (never more than GP_COLS columns; kept exact)
  const unsigned char di = dyn[i];
  for (long long xx = cx; xx <= cx_end; ++xx)
    for (long long cy = y0; cy <= y1; ++cy) {
      // z is the fastest key field: one search per (x, y) column unless z wraps
      const uint32_t k0 = cell_key(xx, cy, z0), k1 = cell_key(xx, cy, z1);
      const bool contiguous = k1 - k0 == (uint32_t)(z1 - z0);
      for (long long cz = z0; cz <= (contiguous ? z0 : z1); ++cz) {
        const uint32_t lo = contiguous ? k0 : cell_key(xx, cy, cz), hi = contiguous ? k1 : lo;
        int p = lower_bound_u32(skeys, n_small, lo);
        for (; p < n_small && skeys[p] <= hi; ++p) {
          const int j = sbody[p];
          if (j <= i) continue;  // small-small pairs once, from the lower index
          if (!(di || dyn[j])) continue;
          if (!box_overlap(a, bbox + 6 * j)) continue;
          unsigned long long at = atomicAdd(count, 1ull);
          if ((int64_t)at < cap) out[at] = make_int2(i, j);
        }
      }
    }
}

// every (large body, body) pair: thread per body j over the few large bodies
// (the CELL_LARGE-keyed tail of the sorted cell keys); large-large pairs once (j > i)
__global__ void k_large_pairs(int B, const double* __restrict__ bbox, const unsigned char* __restrict__ dyn,
                              const uint32_t* __restrict__ skeys, const int* __restrict__ sbody,
                              const double* __restrict__ cell_p, unsigned long long* count, int64_t cap, int2* out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= B) return;
  const double cell = *cell_p;
  int first = lower_bound_u32(skeys, B, CELL_LARGE);
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

// inflated boxes of the body-pair superset: exact box +- frac x cell (cell from k_cell_size)
__global__ void k_inflate_boxes(int B, const double* __restrict__ bbox, const double* __restrict__ cell_p,
                                double frac, double* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double m = frac * *cell_p;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    out[6 * b + k] = bbox[6 * b + k] - m;
    out[6 * b + 3 + k] = bbox[6 * b + 3 + k] + m;
  }
}

void launch_body_boxes(Scene& s, const double* q0, const double* q1, double h, double* out) {
  if (s.B == 0) return;
  k_body_boxes<<<grid_for((int64_t)s.B * 32, 256), 256, 0, s.stream>>>(s.B, s.v_off.p, s.rest.p, q0, q1, h, out);
  note_launch("k_body_boxes");
}

// ---------------------------------------------------------------------------
// primitive Verlet list (Work::pvl_*)
// exact swept boxes of the candidate rows' primitives overlap? (contact.py:222-229 boxes)
__global__ void k_pvl_flags(PrimGeo g, int64_t n_vf, const int4* __restrict__ vf, int64_t n_ee,
                            const int4* __restrict__ ee, int* flags) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_vf + n_ee) return;
  const bool is_vf = i < n_vf;
  const int4 r = is_vf ? vf[i] : ee[i - n_vf];
  int va[3], vb2[3];
  int na, nb;
  if (is_vf) {
    va[0] = g.v_off[r.x] + r.y;
    na = 1;
    const int* t = g.tris + 3 * (int64_t)(g.t_off[r.z] + r.w);
    vb2[0] = t[0];
    vb2[1] = t[1];
    vb2[2] = t[2];
    nb = 3;
  } else {
    const int* ea = g.edges + 2 * (int64_t)(g.e_off[r.x] + r.y);
    const int* eb = g.edges + 2 * (int64_t)(g.e_off[r.z] + r.w);
    va[0] = ea[0];
    va[1] = ea[1];
    vb2[0] = eb[0];
    vb2[1] = eb[1];
    na = nb = 2;
  }
  double A[6], Bx[6], t6[6];
  for (int side = 0; side < 2; ++side) {
    const int body = side ? r.z : r.x;
    const int* vv = side ? vb2 : va;
    const int nv = side ? nb : na;
    double* o = side ? Bx : A;
    vertex_box(g.rest, vv[0], g.q0 + 12 * (int64_t)body, g.q1 + 12 * (int64_t)body, g.h, o);
    for (int m = 1; m < nv; ++m) {
      vertex_box(g.rest, vv[m], g.q0 + 12 * (int64_t)body, g.q1 + 12 * (int64_t)body, g.h, t6);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        o[k] = fmin(o[k], t6[k]);
        o[3 + k] = fmax(o[3 + k], t6[3 + k]);
      }
    }
  }
  flags[i] = A[0] <= Bx[3] && Bx[0] <= A[3] && A[1] <= Bx[4] && Bx[1] <= A[4] && A[2] <= Bx[5] && Bx[2] <= A[5];
}

// every body's current sweep [q0, q1] within half the margin of the build sweep
// [Q0, Q1]: for each end, its deviation e from the closest point of the segment
// bounds every vertex's displacement by sum_j |e_A,ij| R_j + |e_p,i| (R = max |rest|)
__global__ void k_pvl_check(int B, const double* __restrict__ q0, const double* __restrict__ q1,
                            const double* __restrict__ Q0, const double* __restrict__ Q1,
                            const double* __restrict__ rmax, double lim, int* viol) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double* P = Q0 + 12 * (int64_t)b;
  const double* Pe = Q1 + 12 * (int64_t)b;
  double d[12], dd = 0.0;
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    d[k] = Pe[k] - P[k];
    dd += d[k] * d[k];
  }
  bool bad = false;
  for (int u = 0; u < 2; ++u) {
    const double* x = (u ? q1 : q0) + 12 * (int64_t)b;
    double proj = 0.0;
#pragma unroll
    for (int k = 0; k < 12; ++k) proj += (x[k] - P[k]) * d[k];
    const double al = dd > 0.0 ? fmin(1.0, fmax(0.0, proj / dd)) : 0.0;
    double e[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) e[k] = x[k] - (P[k] + al * d[k]);
    for (int i = 0; i < 3; ++i) {
      const double bound = fabs(e[i]) + fabs(e[3 + 3 * i]) * rmax[3 * b] + fabs(e[4 + 3 * i]) * rmax[3 * b + 1] +
                           fabs(e[5 + 3 * i]) * rmax[3 * b + 2];
      if (!(bound <= lim)) bad = true;
    }
  }
  if (bad) atomicExch(viol, 1);
}

// primitive candidates of the body pairs ov (vertex boxes inflated by h, primitives
// culled against the body boxes bbox): rows into vf / ee in deterministic order
// (overlap pair, product, prim_a, prim_b), or canonical order when a chunk overflowed
static void prim_pairs_run(Scene& s, const double* q0, const double* q1, double h, const int2* ov, int& n_ov,
                           const double* bbox, DVec<int4>& vf, DVec<int4>& ee, int64_t& n_vf, int64_t& n_ee,
                           int* ov_same, bool& ov_same_h, const int* n_ov_dev = nullptr, int* viol_h = nullptr,
                           bool no_prezero = false) {
  // n_ov_dev: the pair count is on the device (n_ov is then only a capacity); it is
  // read back with the candidate counts, together with the Verlet-list violation flag
  const int n_cap = n_ov;
  cudaStream_t st = s.stream;
  Scene::Work& w = s.w;
  PrimGeo g{s.rest.p, q0, q1, h, s.v_off.p, s.e_off.p, s.t_off.p, s.edges.p, s.tris.p};
  unsigned long long* counters = w.ull.p + 4;
  int* unsorted = reinterpret_cast<int*>(w.ull.p + 8);
  bool chunked = false;
  if (vf.cap < 1024) vf.resize(1024);
  if (ee.cap < 1024) ee.resize(1024);
  unsigned long long* hc = reinterpret_cast<unsigned long long*>(s.h_pinned);
  for (int attempt = 0; attempt < 3; ++attempt) {
    // the counters, overflow flag and work queue start zeroed (broad_phase); retries re-zero
    if (attempt > 0 || no_prezero) CK(cudaMemsetAsync(counters, 0, 2 * sizeof(unsigned long long), st));
    static bool attr = false;
    const int cap_list = std::max(s.max_v, std::max(s.max_e, s.max_t));
    const int3 cap_k = make_int3(s.max_v, s.max_e, s.max_t);
    const size_t p2_smem = sizeof(double) * (2 * P2_VBS * P2_VCAP + 6 * (size_t)cap_list) +
                           2 * sizeof(int) * 2 * (size_t)(cap_k.x + cap_k.y + cap_k.z) + sizeof(unsigned) * P2_HCAP;
    const bool use2 = (s.max_v <= P2_VCAP && p2_smem <= 100 * 1024 && !getenv("ABD_BP_V1")) || s.comm.world > 1;
    if (s.comm.world > 1 && !(s.max_v <= P2_VCAP && p2_smem <= 100 * 1024))
      throw Error(ABD_ERR_ARG, "partitioned broad phase needs <= 256 vertices per body");
    if (!attr) {
      CK(cudaFuncSetAttribute((void*)k_prim_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BP_SMEM));
      CK(cudaFuncSetAttribute((void*)k_prim_pairs2<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      CK(cudaFuncSetAttribute((void*)k_prim_pairs2<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
      attr = true;
    }
    if (s.instrument) CK(cudaEventRecord(s.ev0, st));
    if (use2) {
      int grid = (int)std::max<int64_t>(1, std::min<int64_t>(n_cap, (int64_t)s.num_sms * 3));
      w.tab.resize(3 * (size_t)std::max(n_cap, 1));
      if (s.comm.world > 1) CK(cudaMemsetAsync(w.tab.p, 0, 3 * (size_t)n_cap * sizeof(int2), st));
      if (attempt > 0 || no_prezero) {
        CK(cudaMemsetAsync(unsorted, 0, sizeof(int), st));
        CK(cudaMemsetAsync(w.ull.p + 11, 0, sizeof(unsigned long long), st));
      }
      static const bool no_groups = getenv("ABD_BP_NO_GROUPS") != nullptr;
      GrpGeo gg{};
      for (int k = 0; k < 3; ++k) {
        gg.id[k] = s.grp_id[k].p;
        gg.pk[k] = s.grp_pk[k].p;
        gg.box[k] = s.grp_box[k].p;
        gg.off[k] = s.grp_off[k].p;
      }
      static const bool no_merge = getenv("ABD_BP_NO_MERGE") != nullptr;
      const int ug = (s.has_groups && !no_groups ? 1 : 0) | (no_merge ? 2 : 0);
      // run-pair filtering of the products pays for large meshes (tori: 960 edges +
      // triangles per body, products of thousands of pairs); for the pile's
      // icospheres (800) the plain sweep is faster
      static const int runs_env = getenv("ABD_BP_RUNS") ? atoi(getenv("ABD_BP_RUNS")) : -1;
      const int runs = runs_env >= 0 ? runs_env : (s.max_e + s.max_t > 800 ? 1 : 0);
      auto kfn = runs ? k_prim_pairs2<true> : k_prim_pairs2<false>;
      kfn<<<grid, P2_THREADS, p2_smem, st>>>(g, gg, ug, n_ov, ov, bbox, counters, (int64_t)vf.cap, (int64_t)ee.cap,
                                             vf.p, ee.p, cap_list, cap_k, w.tab.p, unsorted, s.comm.rank,
                                             s.comm.world > 1 ? s.slab_owner.p : nullptr, w.ull.p + 11, n_ov_dev);
    } else {
      int grid = (int)std::min<int64_t>(n_ov, (int64_t)s.num_sms);
      k_prim_pairs<<<grid, BP_THREADS, BP_SMEM, st>>>(g, n_ov, ov, bbox, counters, (int64_t)vf.cap,
                                                      (int64_t)ee.cap, vf.p, ee.p);
    }
    note_launch("k_prim_pairs");
    if (s.instrument) CK(cudaEventRecord(s.ev1, st));
    if (n_ov_dev)
      pack_to_host(st, hc, {{counters, 16, 0}, {unsorted, 4, 16}, {ov_same, 4, 24}, {n_ov_dev, 8, 32}});
    else
      pack_to_host(st, hc, {{counters, 16, 0}, {unsorted, 4, 16}, {ov_same, 4, 24}});
    SSYNC(st);
    ov_same_h = *reinterpret_cast<int*>(hc + 3) != 0;
    if (n_ov_dev) {
      n_ov = reinterpret_cast<const int*>(hc + 4)[0];
      if (viol_h) *viol_h = reinterpret_cast<const int*>(hc + 4)[1];
      if (viol_h && *viol_h) return;  // the caller rebuilds the Verlet list and starts over
    }
    chunked = use2 && *reinterpret_cast<int*>(hc + 2) == 0;
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
    if (hc[0] <= vf.cap && hc[1] <= ee.cap) break;
    if (hc[0] > vf.cap) vf.resize(hc[0]);
    if (hc[1] > ee.cap) ee.resize(hc[1]);
  }
  n_vf = (int64_t)hc[0];
  n_ee = (int64_t)hc[1];
  vf.n = n_vf;
  ee.n = n_ee;
  if (n_ov == 0) return;
  if (!chunked) {
    // canonical (c0, c2, c1, c3) order by radix sort
    sort_rows(s, vf, n_vf, bits_for(s.max_v - 1), bits_for(s.max_t - 1));
    sort_rows(s, ee, n_ee, bits_for(s.max_e - 1), bits_for(s.max_e - 1));
    return;
  }
  // Deterministic order without a global sort: (overlap pair, product, prim_a, prim_b).
  // Each (pair, product) chunk was sorted in shared memory; chunks move to their
  // prefix-sum offsets in pair order.  (abd_get_candidates returns the canonical order.)
  static const bool split = getenv("ABD_BP_CHUNK_SPLIT") != nullptr;  // the separate count / scan / move kernels
  if (!split) {
    w.rows_tmp.resize(std::max<int64_t>(n_vf, 1));
    w.rows_tmp2.resize(std::max<int64_t>(n_ee, 1));
    k_chunk_gather<<<(n_ov + CG_PAIRS - 1) / CG_PAIRS, CG_THREADS, 0, st>>>(n_ov, w.tab.p, vf.p, w.rows_tmp.p, ee.p,
                                                                          w.rows_tmp2.p);
    note_launch("k_chunk_gather");
    if (n_vf) {
      std::swap(vf.p, w.rows_tmp.p);
      std::swap(vf.cap, w.rows_tmp.cap);
      std::swap(vf.n, w.rows_tmp.n);
      vf.n = n_vf;
    }
    if (n_ee) {
      std::swap(ee.p, w.rows_tmp2.p);
      std::swap(ee.cap, w.rows_tmp2.cap);
      std::swap(ee.n, w.rows_tmp2.n);
      ee.n = n_ee;
    }
    return;
  }
  w.cnt.resize(2 * n_ov + 1);
  w.off.resize(2 * n_ov + 1);
  w.va.resize(n_ov + 1);
  w.vb.resize(n_ov + 1);
  k_chunk_counts<<<grid_for(n_ov, 256), 256, 0, st>>>(n_ov, w.tab.p, w.cnt.p, w.va.p);
  note_launch("k_chunk_counts");
  scan_exclusive_i32(s, w.cnt.p, w.off.p, 2 * n_ov);
  scan_exclusive_i32(s, w.va.p, w.vb.p, n_ov);
  w.rows_tmp.resize(std::max<int64_t>(n_vf, 1));
  if (n_vf) {
    k_chunk_move<<<grid_for(2 * n_ov * 32, 256), 256, 0, st>>>(n_ov, w.tab.p, 0, 2, w.off.p, vf.p, w.rows_tmp.p);
    note_launch("k_chunk_move");
    std::swap(vf.p, w.rows_tmp.p);
    std::swap(vf.cap, w.rows_tmp.cap);
    std::swap(vf.n, w.rows_tmp.n);
    vf.n = n_vf;
  }
  w.rows_tmp.resize(std::max<int64_t>(n_ee, 1));
  if (n_ee) {
    k_chunk_move<<<grid_for(n_ov * 32, 256), 256, 0, st>>>(n_ov, w.tab.p, 2, 1, w.vb.p, ee.p, w.rows_tmp.p);
    note_launch("k_chunk_move");
    std::swap(ee.p, w.rows_tmp.p);
    std::swap(ee.cap, w.rows_tmp.cap);
    std::swap(ee.n, w.rows_tmp.n);
    ee.n = n_ee;
  }
}

static void prim_stage(Scene& s, const double* q0, const double* q1, double h, int& n_ov, int* ov_same,
                       const int* n_ov_dev = nullptr, int* viol_h = nullptr) {
  cudaStream_t st = s.stream;
  Cands& c = s.cands;
  Scene::Work& w = s.w;
  // off by default: in the late pile the Newton sweeps move by centimetres per iteration,
  // so a margin that holds them makes the superset (and its rebuilds) costlier than
  // the exact broad phase (measured: 11.2 -> 8.6 steps/s at 1% of the cell)
  static const double pvl_frac = getenv("ABD_PVL_MARGIN") ? atof(getenv("ABD_PVL_MARGIN")) : 0.0;
  const bool use_pvl = pvl_frac > 0.0 && w.vl_valid && w.vl_cell > 0.0 && s.has_groups && !n_ov_dev;
  bool same = false;
  if (use_pvl) {
    PrimGeo g{s.rest.p, q0, q1, h, s.v_off.p, s.e_off.p, s.t_off.p, s.edges.p, s.tris.p};
    int* info = reinterpret_cast<int*>(w.ull.p + 14);  // {n_vf, n_ee, viol, -}
    for (int attempt = 0; attempt < 2; ++attempt) {
      const bool valid = w.pvl_valid && w.pvl_gen == w.vl_gen && w.pvl_h == h;
      if (!valid) {
        // rebuild: candidates of the whole body superset for margin-inflated boxes
        const double m = pvl_frac * w.vl_cell;
        bool dummy = false;
        int* no_same = reinterpret_cast<int*>(w.ull.p + 15);
        CK(cudaMemsetAsync(no_same, 0, sizeof(int), st));
        int n_sup = (int)w.vl_n;
        prim_pairs_run(s, q0, q1, h + m, w.vl_pairs.p, n_sup, w.vl_box.p, w.pvl_vf, w.pvl_ee, w.pvl_nvf,
                       w.pvl_nee, no_same, dummy, nullptr, nullptr, /*no_prezero=*/true);
        w.pvl_q0.resize(12 * (size_t)s.B);
        w.pvl_q1.resize(12 * (size_t)s.B);
        CK(cudaMemcpyAsync(w.pvl_q0.p, q0, 12 * (size_t)s.B * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(w.pvl_q1.p, q1, 12 * (size_t)s.B * sizeof(double), cudaMemcpyDeviceToDevice, st));
        w.pvl_m = m;
        w.pvl_h = h;
        w.pvl_gen = w.vl_gen;
        w.pvl_valid = true;
      }
      CK(cudaMemsetAsync(info, 0, 4 * sizeof(int), st));
      k_pvl_check<<<grid_for(s.B, 256), 256, 0, st>>>(s.B, q0, q1, w.pvl_q0.p, w.pvl_q1.p, s.body_rmax.p,
                                                      0.5 * w.pvl_m, info + 2);
      note_launch("k_pvl_check");
      const int64_t ns = w.pvl_nvf + w.pvl_nee;
      w.pvl_flags.resize(std::max<int64_t>(ns, 1));
      if (ns)
        k_pvl_flags<<<grid_for(ns, 128), 128, 0, st>>>(g, w.pvl_nvf, w.pvl_vf.p, w.pvl_nee, w.pvl_ee.p,
                                                       w.pvl_flags.p);
      note_launch("k_pvl_flags");
      if ((int64_t)c.vf.cap < std::max<int64_t>(w.pvl_nvf, 1024)) c.vf.resize(std::max<int64_t>(w.pvl_nvf, 1024));
      if ((int64_t)c.ee.cap < std::max<int64_t>(w.pvl_nee, 1024)) c.ee.resize(std::max<int64_t>(w.pvl_nee, 1024));
      size_t b1 = 0, b2 = 0;
      CK(cub::DeviceSelect::Flagged(nullptr, b1, w.pvl_vf.p, w.pvl_flags.p, c.vf.p, info, (int)w.pvl_nvf, st));
      CK(cub::DeviceSelect::Flagged(nullptr, b2, w.pvl_ee.p, w.pvl_flags.p + w.pvl_nvf, c.ee.p, info + 1,
                                    (int)w.pvl_nee, st));
      s.tmp_bytes.resize(std::max<size_t>(std::max(b1, b2), 16));
      if (w.pvl_nvf)
        CK(cub::DeviceSelect::Flagged(s.tmp_bytes.p, b1, w.pvl_vf.p, w.pvl_flags.p, c.vf.p, info, (int)w.pvl_nvf,
                                      st));
      if (w.pvl_nee)
        CK(cub::DeviceSelect::Flagged(s.tmp_bytes.p, b2, w.pvl_ee.p, w.pvl_flags.p + w.pvl_nvf, c.ee.p, info + 1,
                                      (int)w.pvl_nee, st));
      int* hi = reinterpret_cast<int*>(s.h_pinned);
      pack_to_host(st, hi, {{info, 16, 0}, {ov_same, 4, 16}});
      SSYNC(st);
      if (hi[2] && valid) {
        w.pvl_valid = false;  // a body left its margin: rebuild and filter again
        continue;
      }
      same = hi[4] != 0;
      c.n_vf = hi[0];
      c.n_ee = hi[1];
      c.vf.n = c.n_vf;
      c.ee.n = c.n_ee;
      c.ov_matches_pattern = same;
      return;
    }
  }
  prim_pairs_run(s, q0, q1, h, c.ov.p, n_ov, s.bbox.p, c.vf, c.ee, c.n_vf, c.n_ee, ov_same, same, n_ov_dev,
                 viol_h);
  c.ov_matches_pattern = same;
}

__global__ void k_vl_contain(int B, const double* __restrict__ bbox, const double* __restrict__ vl_box, int* viol) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double* x = bbox + 6 * b;
  const double* y = vl_box + 6 * b;
  if (!(x[0] >= y[0] && x[1] >= y[1] && x[2] >= y[2] && x[3] <= y[3] && x[4] <= y[4] && x[5] <= y[5]))
    atomicExch(viol, 1);
}

__global__ void k_vl_flags(int64_t n, const int2* __restrict__ sup, const double* __restrict__ bbox, int* flags,
                           int* set_one) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i == 0 && set_one) *set_one = 1;  // (the pattern check that follows clears it)
  if (i >= n) return;
  const int2 pr = sup[i];
  flags[i] = box_overlap(bbox + 6 * pr.x, bbox + 6 * pr.y);
}

// the Verlet-list filter over the whole GPU: containment flag, overlap flags and an
// ordered (stable) compaction into c.ov; info = {count, violation} on the device
static void vl_filter(Scene& s, int* info, bool zero_info, bool contain_done = false, int* set_one = nullptr) {
  cudaStream_t st = s.stream;
  Scene::Work& w = s.w;
  Cands& c = s.cands;
  if (zero_info) CK(cudaMemsetAsync(info, 0, 2 * sizeof(int), st));
  if (!contain_done) {  // (the deferred path folds the containment test into k_body_boxes)
    k_vl_contain<<<grid_for(s.B, 256), 256, 0, st>>>(s.B, s.bbox.p, w.vl_box.p, info + 1);
    note_launch("k_vl_contain");
  }
  if (w.vl_n == 0) return;
  w.flags.resize(w.vl_n);
  k_vl_flags<<<grid_for(w.vl_n, 256), 256, 0, st>>>(w.vl_n, w.vl_pairs.p, s.bbox.p, w.flags.p, set_one);
  note_launch("k_vl_flags");
  size_t bytes = 0;
  CK(cub::DeviceSelect::Flagged(nullptr, bytes, w.vl_pairs.p, w.flags.p, c.ov.p, info, (int)w.vl_n, st));
  s.tmp_bytes.resize(std::max<size_t>(bytes, 16));
  CK(cub::DeviceSelect::Flagged(s.tmp_bytes.p, bytes, w.vl_pairs.p, w.flags.p, c.ov.p, info, (int)w.vl_n, st));
}

void broad_phase(Scene& s, const double* q0, const double* q1, double d_hat) {
  cudaStream_t st = s.stream;
  if (s.comm.world > 1 && !s.slab_valid) slab_partition(s, q0);  // (advance_step re-cuts per step)
  double h = 0.5 * d_hat;
  Cands& c = s.cands;
  Scene::Work& w = s.w;
  c.n_vf = c.n_ee = c.n_ov = 0;
  c.gen += 1;
  // one memset for this broad phase's device scalars (w.ull[4..13]: pair / candidate
  // counters, overflow flag, work queue, pattern flag, Verlet-list info) and the
  // following line search's slow-query counter
  CK(cudaMemsetAsync(w.ull.p + 4, 0, 10 * sizeof(unsigned long long), st));
  if (s.B < 2) return;
  s.bbox.resize(6 * s.B);
  // body pairs: filter the superset with the exact boxes (one CTA, one sync); rebuild
  // the superset on the uniform grid when a box left its inflated box
  static const double vl_frac = getenv("ABD_VL_MARGIN") ? atof(getenv("ABD_VL_MARGIN")) : 0.05;
  // the superset serves the stepping broad phase (h = d_hat / 2); a call with another
  // inflation (the stats' distance search) runs the exact grid path and leaves it alone
  const bool use_vl = vl_frac > 0.0 && (w.vl_h < 0.0 || w.vl_h == h);
  int* vl_info = reinterpret_cast<int*>(w.ull.p + 13);
  int n_ov = 0;
  bool have = false;
  // the filtered count stays on the device and is read back with the primitive-pair
  // counts (one sync less); a containment violation then restarts the broad phase
  static const bool no_defer = getenv("ABD_VL_SYNC") != nullptr;
  const bool defer = use_vl && w.vl_valid && !no_defer && s.max_v <= P2_VCAP && !getenv("ABD_BP_V1");
  // (deferred path: the containment test rides in the body-box kernel; vl_info was zeroed above)
  k_body_boxes<<<grid_for((int64_t)s.B * 32, 256), 256, 0, st>>>(s.B, s.v_off.p, s.rest.p, q0, q1, h, s.bbox.p,
                                                                 defer ? w.vl_box.p : nullptr, vl_info + 1);
  note_launch("k_body_boxes");
  if (defer) {
    if ((int64_t)c.ov.cap < std::max<int64_t>(w.vl_n, 1)) c.ov.resize(std::max<int64_t>(w.vl_n, 1));
    int* ov_same = reinterpret_cast<int*>(w.ull.p + 9);  // zeroed with the broad phase's scalars
    const bool check_pat = w.pat_valid && s.H.n == s.n_dyn;
    vl_filter(s, vl_info, false, /*contain_done=*/true, check_pat && w.vl_n > 0 ? ov_same : nullptr);
    if (check_pat) {
      if (w.vl_n == 0) dev_set_i32(st, ov_same, 1);
      k_ov_in_pattern<<<grid_for(std::max<int64_t>(w.vl_n, 1), 256), 256, 0, st>>>(
          w.vl_n, c.ov.p, s.slot.p, s.H.n_off, s.H.upper_keys.p, ov_same, vl_info);
      note_launch("k_ov_in_pattern");
    }
    int n_cap = (int)w.vl_n;
    int viol = 0;
    prim_stage(s, q0, q1, h, n_cap, ov_same, vl_info, &viol);
    if (viol) {
      w.vl_valid = false;
      broad_phase(s, q0, q1, d_hat);
      return;
    }
    c.n_ov = n_cap;
    c.ov.n = n_cap;
    return;
  }
  if (use_vl && w.vl_valid) {
    if ((int64_t)c.ov.cap < std::max<int64_t>(w.vl_n, 1)) c.ov.resize(std::max<int64_t>(w.vl_n, 1));
    vl_filter(s, vl_info, true);
    int* hi = reinterpret_cast<int*>(s.h_pinned);
    pack_to_host(st, hi, {{vl_info, 8, 0}});
    SSYNC(st);
    if (hi[1] == 0) {
      n_ov = hi[0];
      have = true;
    }
  }
  if (!have) {
    // superset of pairs on a uniform grid (cell = largest extent <= 4x the median)
    bool alt = false;
    w.k0.resize(s.B);
    w.k1.resize(s.B);
    w.va.resize(s.B + 1);
    w.vb.resize(s.B + 1);
    w.ka.resize(s.B);
    w.kb.resize(s.B);
    w.scal.resize(4);
    const double* gbox = s.bbox.p;
    if (use_vl) {
      k_extent_keys<<<grid_for(s.B, 256), 256, 0, st>>>(s.B, s.bbox.p, w.ka.p);
      note_launch("k_extent_keys");
      k_cell_size<<<1, 1024, 0, st>>>(s.B, w.ka.p, w.scal.p);
      note_launch("k_cell_size");
      w.vl_box.resize(6 * s.B);
      k_inflate_boxes<<<grid_for(s.B, 256), 256, 0, st>>>(s.B, s.bbox.p, w.scal.p, vl_frac, w.vl_box.p);
      note_launch("k_inflate_boxes");
      gbox = w.vl_box.p;
    }
    k_extent_keys<<<grid_for(s.B, 256), 256, 0, st>>>(s.B, gbox, w.ka.p);
    note_launch("k_extent_keys");
    k_cell_size<<<1, 1024, 0, st>>>(s.B, w.ka.p, w.scal.p);
    note_launch("k_cell_size");
    k_cell_keys2<<<grid_for(s.B, 256), 256, 0, st>>>(s.B, gbox, w.scal.p, w.ka.p, w.va.p);
    note_launch("k_cell_keys");
    sort_pairs_u32(s, w.ka.p, w.kb.p, w.va.p, w.vb.p, s.B, CELL_KEY_BITS, alt);
    const uint32_t* skeys = alt ? w.kb.p : w.ka.p;
    const int* sbody = alt ? w.vb.p : w.va.p;
    int n_small = s.B;  // large bodies carry CELL_LARGE and sort last; the lookups never match them
    unsigned long long* ovc = w.ull.p + 6;
    unsigned long long* hov = reinterpret_cast<unsigned long long*>(s.h_pinned);
    DVec<int2>& dst = use_vl ? w.vl_pairs : c.ov;
    if (dst.cap < 256) dst.resize(256);
    for (int attempt = 0; attempt < 3; ++attempt) {
      CK(cudaMemsetAsync(ovc, 0, sizeof(unsigned long long), st));
      k_grid_pairs<<<grid_for((int64_t)s.B * GP_COLS, 128), 128, 0, st>>>(s.B, gbox, s.dyn.p, skeys, sbody, n_small,
                                                                          w.scal.p, ovc, (int64_t)dst.cap, dst.p);
      note_launch("k_grid_pairs");
      k_large_pairs<<<grid_for(s.B, 128), 128, 0, st>>>(s.B, gbox, s.dyn.p, skeys, sbody, w.scal.p, ovc,
                                                        (int64_t)dst.cap, dst.p);
      note_launch("k_large_pairs");
      CK(cudaMemcpyAsync(hov, ovc, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
      SSYNC(st);
      if (hov[0] <= dst.cap) break;
      dst.resize(hov[0]);
    }
    const int n_g = (int)hov[0];
    dst.n = n_g;
    // canonical (i, j) order
    if (n_g > 0) {
      int bB = bits_for(s.B - 1);
      w.k0.resize(n_g);
      w.k1.resize(n_g);
      w.va.resize(n_g);
      w.vb.resize(n_g);
      k_pair_keys<<<grid_for(n_g, 256), 256, 0, st>>>(n_g, dst.p, bB, w.k0.p, w.va.p);
      note_launch("k_pair_keys");
      sort_pairs_u64(s, w.k0.p, w.k1.p, w.va.p, w.vb.p, n_g, 2 * bB, alt);
      w.pairs_tmp.resize(n_g);
      k_gather<int2><<<grid_for(n_g, 256), 256, 0, st>>>(n_g, alt ? w.vb.p : w.va.p, dst.p, w.pairs_tmp.p);
      note_launch("k_gather");
      CK(cudaMemcpyAsync(dst.p, w.pairs_tmp.p, n_g * sizeof(int2), cudaMemcpyDeviceToDevice, st));
    }
    if (use_vl) {
      w.vl_n = n_g;
      w.vl_valid = true;
      w.vl_gen += 1;
      w.vl_h = h;
      if ((int64_t)c.ov.cap < std::max(n_g, 1)) c.ov.resize(std::max(n_g, 1));
      vl_filter(s, vl_info, true);
      int* hi = reinterpret_cast<int*>(s.h_pinned);
      pack_to_host(st, hi, {{vl_info, 8, 0}, {w.scal.p, 8, 8}});
      SSYNC(st);
      n_ov = hi[0];
      w.vl_cell = reinterpret_cast<const double*>(hi)[1];
    } else {
      n_ov = n_g;
    }
  }
  c.n_ov = n_ov;
  c.ov.n = n_ov;
  c.ov_matches_pattern = false;
  if (n_ov == 0) {
    c.ov_matches_pattern = w.pat_n_ov == 0;
    return;
  }
  // is every dynamic overlap pair already a block of the resident BSR pattern?
  // (read back with the primitive-pair counts below; build_pattern then keeps the
  // pattern -- extra blocks just hold zeros -- instead of re-sorting it)
  int* ov_same = reinterpret_cast<int*>(w.ull.p + 9);
  if (w.pat_valid && s.H.n == s.n_dyn) {
    const int one = 1;
    dev_set_i32(st, ov_same, one);
    k_ov_in_pattern<<<grid_for(n_ov, 256), 256, 0, st>>>(n_ov, c.ov.p, s.slot.p, s.H.n_off, s.H.upper_keys.p,
                                                         ov_same, nullptr);
    note_launch("k_ov_in_pattern");
  } else {
    CK(cudaMemsetAsync(ov_same, 0, sizeof(int), st));
  }
  prim_stage(s, q0, q1, h, n_ov, ov_same);
}

}  // namespace abd
