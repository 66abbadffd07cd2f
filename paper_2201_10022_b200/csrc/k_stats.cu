// Exact global minimum inter-body distance (solver.py:396-473): body pairs
// pruned by box gap against the exact distance of the closest-box pair, then
// exhaustive vertex-triangle / edge-edge evaluation per surviving pair.
#include <cmath>
#include <vector>

#include "abd_misc.cuh"
#include "driver.h"

namespace abd {

__global__ void k_body_boxes_q(int B, const int* __restrict__ v_off, const double* __restrict__ rest,
                               const double* __restrict__ q, double* bbox) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= B) return;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int v = v_off[w] + lane; v < v_off[w + 1]; v += 32) {
    V3 x = world_pos(q + 12 * (int64_t)w, ld3(rest + 3 * (int64_t)v));
    lo[0] = fmin(lo[0], x.x); lo[1] = fmin(lo[1], x.y); lo[2] = fmin(lo[2], x.z);
    hi[0] = fmax(hi[0], x.x); hi[1] = fmax(hi[1], x.y); hi[2] = fmax(hi[2], x.z);
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

__device__ __forceinline__ double box_gap(const double* a, const double* b) {
  double g2 = 0.0;
  for (int k = 0; k < 3; ++k) {
    double g = fmax(0.0, fmax(a[k] - b[3 + k], b[k] - a[3 + k]));
    g2 += g * g;
  }
  return sqrt(g2);
}

// pass 0: argmin gap (packed gap bits | pair index is not needed: we keep min gap
// and, separately, one pair achieving it); pass 1: list pairs with gap < bound
__global__ void k_pair_gaps(int B, const unsigned char* __restrict__ dyn, const double* __restrict__ bbox, double bound,
                            unsigned long long* min_gap, int2* list, int* count, int cap, int skip_static) {
  int64_t total = (int64_t)B * (B - 1) / 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    // invert t -> (i, j), i < j, row-major over the upper triangle
    int64_t i = (int64_t)((2.0 * B - 1 - sqrt((2.0 * B - 1) * (2.0 * B - 1) - 8.0 * (double)t)) / 2.0);
    if (i < 0) i = 0;
    while (i > 0 && i * (2 * (int64_t)B - i - 1) / 2 > t) --i;
    while ((i + 1) * (2 * (int64_t)B - i - 2) / 2 <= t) ++i;
    int64_t j = t - i * (2 * (int64_t)B - i - 1) / 2 + i + 1;
    if (skip_static && !(dyn[i] || dyn[j])) continue;
    double g = box_gap(bbox + 6 * i, bbox + 6 * j);
    if (min_gap) atomicMin(min_gap, (unsigned long long)__double_as_longlong(g));
    if (list && g < bound) {
      int at = atomicAdd(count, 1);
      if (at < cap) list[at] = make_int2((int)i, (int)j);
    }
  }
}

// one CTA per body pair: exact min d^2 over V_a x T_b, V_b x T_a, E_a x E_b
__global__ void k_pair_min_d2(SceneView sv, const int* __restrict__ vb_off_unused, const double* __restrict__ q,
                              const int2* __restrict__ list, int n, unsigned long long* best) {
  (void)vb_off_unused;
  __shared__ double sh[32];
  for (int pi = blockIdx.x; pi < n; pi += gridDim.x) {
    int2 pr = list[pi];
    double m = INFINITY;
    for (int dir = 0; dir < 2; ++dir) {
      int bv = dir == 0 ? pr.x : pr.y, bt = dir == 0 ? pr.y : pr.x;
      int nv = sv.v_off[bv + 1] - sv.v_off[bv], nt = sv.t_off[bt + 1] - sv.t_off[bt];
      int64_t tot = (int64_t)nv * nt;
      for (int64_t k = threadIdx.x; k < tot; k += blockDim.x) {
        int v = sv.v_off[bv] + (int)(k / nt);
        int t = sv.t_off[bt] + (int)(k % nt);
        V3 p = world_pos(q + 12 * (int64_t)bv, ld3(sv.rest + 3 * (int64_t)v));
        V3 a = world_pos(q + 12 * (int64_t)bt, ld3(sv.rest + 3 * (int64_t)sv.tris[3 * t]));
        V3 b = world_pos(q + 12 * (int64_t)bt, ld3(sv.rest + 3 * (int64_t)sv.tris[3 * t + 1]));
        V3 c = world_pos(q + 12 * (int64_t)bt, ld3(sv.rest + 3 * (int64_t)sv.tris[3 * t + 2]));
        m = fmin(m, pt_closest(p, a, b, c).d2);
      }
    }
    {
      int na = sv.e_off[pr.x + 1] - sv.e_off[pr.x], nb = sv.e_off[pr.y + 1] - sv.e_off[pr.y];
      int64_t tot = (int64_t)na * nb;
      for (int64_t k = threadIdx.x; k < tot; k += blockDim.x) {
        int ea = sv.e_off[pr.x] + (int)(k / nb), eb = sv.e_off[pr.y] + (int)(k % nb);
        V3 a0 = world_pos(q + 12 * (int64_t)pr.x, ld3(sv.rest + 3 * (int64_t)sv.edges[2 * ea]));
        V3 a1 = world_pos(q + 12 * (int64_t)pr.x, ld3(sv.rest + 3 * (int64_t)sv.edges[2 * ea + 1]));
        V3 b0 = world_pos(q + 12 * (int64_t)pr.y, ld3(sv.rest + 3 * (int64_t)sv.edges[2 * eb]));
        V3 b1 = world_pos(q + 12 * (int64_t)pr.y, ld3(sv.rest + 3 * (int64_t)sv.edges[2 * eb + 1]));
        m = fmin(m, ee_closest(a0, a1, b0, b1).d2);
      }
    }
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m < INFINITY) atomicMin(best, (unsigned long long)__double_as_longlong(m));
    __syncthreads();
  }
  (void)sh;
}

// Fast exact path for the end-of-step stats (the resident candidates are recomputed
// at the next step, so they may be overwritten): the broad phase at q with vertex
// boxes inflated by hp gives every primitive pair whose box gap is <= 2 hp; the
// minimum distance m over them is the global minimum whenever m <= 2 hp, because a
// closer pair would have a box gap < m and be a candidate.  hp grows 2x per attempt;
// after four the exhaustive search below decides.
double global_min_distance_stats(Scene& s, const double* q) {
  static const bool off = getenv("ABD_GMD_EXHAUSTIVE") != nullptr;
  if (!off && s.B >= 2 && s.has_groups) {
    // first inflation just covers the previous step's minimum (it changes slowly):
    // a tight candidate set, widened 2x per miss
    double hp = s.w.gmd_prev > 0.0 ? 0.55 * s.w.gmd_prev : 0.02 * (s.w.vl_cell > 0.0 ? s.w.vl_cell : 1.0);
    for (int attempt = 0; attempt < 4; ++attempt, hp *= 2.0) {
      broad_phase(s, q, q, 2.0 * hp);
      const double cm = candidate_min_d2(s, q);
      if (cm <= (2.0 * hp) * (2.0 * hp)) {
        s.w.gmd_prev = std::sqrt(cm);
        return s.w.gmd_prev;
      }
    }
  }
  return global_min_distance(s, q);
}

double global_min_distance(Scene& s, const double* q, int skip_static) {
  cudaStream_t st = s.stream;
  if (s.B < 2) return INFINITY;
  s.bbox.resize(6 * s.B);
  k_body_boxes_q<<<grid_for((int64_t)s.B * 32, 256), 256, 0, st>>>(s.B, s.v_off.p, s.rest.p, q, s.bbox.p);
  note_launch("k_body_boxes_q");
  DVec<unsigned long long> mg;
  mg.resize(1);
  unsigned long long inf = (unsigned long long)__builtin_bit_cast(long long, (double)INFINITY);
  dev_set_u64(st, mg.p, inf);
  int grid = s.num_sms * 8;
  k_pair_gaps<<<grid, 256, 0, st>>>(s.B, s.dyn.p, s.bbox.p, 0.0, mg.p, nullptr, nullptr, 0, skip_static);
  note_launch("k_pair_gaps");
  unsigned long long hg = 0;
  CK(cudaMemcpyAsync(&hg, mg.p, sizeof(hg), cudaMemcpyDeviceToHost, st));
  SSYNC(st);
  double gmin = __builtin_bit_cast(double, hg);
  if (!(gmin < INFINITY)) return INFINITY;
  // bound: exact distance over all pairs whose gap equals the minimum gap
  DVec<int2> list;
  DVec<int> cnt;
  cnt.resize(1);
  DVec<unsigned long long> best;
  best.resize(1);
  auto collect = [&](double bound) -> int {
    int cap = 1024;
    for (;;) {
      list.resize(cap);
      cnt.zero(st);
      k_pair_gaps<<<grid, 256, 0, st>>>(s.B, s.dyn.p, s.bbox.p, bound, nullptr, list.p, cnt.p, cap, skip_static);
      note_launch("k_pair_gaps");
      int hc = 0;
      CK(cudaMemcpyAsync(&hc, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      SSYNC(st);
      if (hc <= cap) return hc;
      cap = hc;
    }
  };
  auto exact = [&](int n) -> double {
    dev_set_u64(st, best.p, inf);
    if (n) {
      k_pair_min_d2<<<std::min(n, s.num_sms * 8), 256, 0, st>>>(view(s), nullptr, q, list.p, n, best.p);
      note_launch("k_pair_min_d2");
    }
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, best.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    SSYNC(st);
    return std::sqrt(__builtin_bit_cast(double, h));
  };
  int n0 = collect(std::nextafter(gmin, INFINITY));
  double ub = exact(n0);
  // every pair that could beat the bound
  int n1 = collect(ub);
  double d = exact(n1);
  return std::fmin(d, ub);
}

}  // namespace abd
