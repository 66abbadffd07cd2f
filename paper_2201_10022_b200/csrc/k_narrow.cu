// Scene narrow phase: activity filter, per-pair contact blocks (K3 first
// pass), contact energy (K6), friction precompute (K7), CCD (K5), per-body
// inertia + orthogonality terms (K1).
#include "abd_contact.cuh"
#include "abd_misc.cuh"
#include "abd_pblk.cuh"
#include "kernels.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace abd {

SceneView view(const Scene& s) {
  SceneView v;
  v.v_off = s.v_off.p;
  v.e_off = s.e_off.p;
  v.t_off = s.t_off.p;
  v.rest = s.rest.p;
  v.edges = s.edges.p;
  v.tris = s.tris.p;
  v.elen2 = s.elen2.p;
  v.dyn = s.dyn.p;
  v.slot = s.slot.p;
  v.B = s.B;
  return v;
}

// global vertex ids and owning bodies of a candidate's 4 stacked points
struct PairIds {
  int vid[4];
  int body[4];
  double eps;
};

__device__ __forceinline__ PairIds pair_ids(const SceneView& sv, int kind, int4 r) {
  PairIds p;
  if (kind == KIND_VF) {
    p.vid[0] = sv.v_off[r.x] + r.y;
    int t = sv.t_off[r.z] + r.w;
    p.vid[1] = sv.tris[3 * t];
    p.vid[2] = sv.tris[3 * t + 1];
    p.vid[3] = sv.tris[3 * t + 2];
    p.body[0] = r.x;
    p.body[1] = p.body[2] = p.body[3] = r.z;
    p.eps = 0.0;
  } else {
    int ea = sv.e_off[r.x] + r.y, eb = sv.e_off[r.z] + r.w;
    p.vid[0] = sv.edges[2 * ea];
    p.vid[1] = sv.edges[2 * ea + 1];
    p.vid[2] = sv.edges[2 * eb];
    p.vid[3] = sv.edges[2 * eb + 1];
    p.body[0] = p.body[1] = r.x;
    p.body[2] = p.body[3] = r.z;
    // DEFAULT_MOLLIFIER_SCALE * la * lb  (contact.py:462)
    p.eps = xmul(xmul(1e-3, sv.elen2[ea]), sv.elen2[eb]);
  }
  return p;
}

__device__ __forceinline__ void pair_points(const SceneView& sv, const PairIds& ids, const double* q, V3* z, V3* xb) {
  for (int k = 0; k < 4; ++k) {
    xb[k] = ld3(sv.rest + 3 * (int64_t)ids.vid[k]);
    z[k] = world_pos(q + 12 * (int64_t)ids.body[k], xb[k]);
  }
}

// activity flags over VF then EE candidates in one launch; flags[n] = 0 (the scan's tail)
__global__ void k_pair_flags_both(SceneView sv, int64_t n_vf, const int4* __restrict__ vf, int64_t n_ee,
                                  const int4* __restrict__ ee, const double* __restrict__ q, double dh2, int* flags,
                                  int* err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t n = n_vf + n_ee;
  if (i > n) return;
  if (i == n) {
    flags[n] = 0;
    return;
  }
  const int kind = i < n_vf ? KIND_VF : KIND_EE;
  PairIds ids = pair_ids(sv, kind, kind == KIND_VF ? vf[i] : ee[i - n_vf]);
  V3 z[4], xb[4];
  pair_points(sv, ids, q, z, xb);
  double d2 = pair_d2(kind, z);
  int on = d2 < dh2;
  flags[i] = on;
  if (on && !(d2 > 0.0)) atomicExch(err, 1);
}

void launch_pair_flags_both(Scene& s, const double* q, double dh2, int* flags, int* err) {
  const int64_t n = s.cands.n_vf + s.cands.n_ee;
  k_pair_flags_both<<<grid_for(n + 1, 128), 128, 0, s.stream>>>(view(s), s.cands.n_vf, s.cands.vf.p, s.cands.n_ee,
                                                                s.cands.ee.p, q, dh2, flags, err);
  note_launch("k_pair_flags");
}

// coupling structure at q (the line search's first trial, i.e. the next Newton
// iterate when it is accepted): pattern blocks of active candidates, marked by
// binary search in the sorted upper keys (as driver.cu k_mark_active_rows)
__global__ void k_mark_active_q(SceneView sv, int64_t n_vf, const int4* __restrict__ vf, int64_t n_ee,
                                const int4* __restrict__ ee, const double* __restrict__ q, double dh2,
                                const int* __restrict__ slot, int64_t n_off, const int2* __restrict__ keys,
                                int* flags) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_vf + n_ee) return;
  const int kind = i < n_vf ? KIND_VF : KIND_EE;
  const int4 r = kind == KIND_VF ? vf[i] : ee[i - n_vf];
  const int sa = slot[r.x], sb = slot[r.z];
  if (sa < 0 || sb < 0 || sa == sb) return;
  PairIds ids = pair_ids(sv, kind, r);
  V3 z[4], xb[4];
  pair_points(sv, ids, q, z, xb);
  if (!(pair_d2(kind, z) < dh2)) return;
  const int a = min(sa, sb), c = max(sa, sb);
  int64_t lo = 0, hi = n_off - 1;
  while (lo <= hi) {
    const int64_t m = (lo + hi) >> 1;
    const int2 k = keys[m];
    if (k.x < a || (k.x == a && k.y < c)) lo = m + 1;
    else if (k.x == a && k.y == c) {
      flags[m] = 1;
      return;
    } else hi = m - 1;
  }
}

void launch_mark_active_q(Scene& s, const double* q, double dh2, int* flags) {
  const int64_t n = s.cands.n_vf + s.cands.n_ee;
  if (!n || !s.H.n_off) return;
  k_mark_active_q<<<grid_for(n, 128), 128, 0, s.stream>>>(view(s), s.cands.n_vf, s.cands.vf.p, s.cands.n_ee,
                                                          s.cands.ee.p, q, dh2, s.slot.p, s.H.n_off,
                                                          s.H.upper_keys.p, flags);
  note_launch("k_mark_active_q");
}

// K3 first pass over the compacted active list (full warps instead of ~1/4 active
// lanes), one compact record per active pair (abd_pblk.cuh);
// specialised per kind so the VF kernel carries none of the mollified-EE state.
// EE pairs whose mollifier is active (near-parallel edges) are deferred to
// k_pair_blocks_moll, so the common EE pairs also run the lean 5-column kernel.
ABD_D bool ee_mollified(const V3* z, double eps) {
  V3 u = z[1] - z[0], v = z[3] - z[2];
  V3 cr = cross(u, v);
  double cc = dot(cr, cr);
  double ratio = eps > 0.0 ? cc / eps : 1.0;
  return ratio < 1.0;
}

template <int KIND>
__global__ void __launch_bounds__(64) k_pair_blocks_act(SceneView sv, int kind_unused, int64_t count,
                                                         const int* __restrict__ act, int64_t cand_off,
                                                         const int4* __restrict__ rows, const double* __restrict__ q,
                                                         double kappa, double dh, int project, int64_t slot_off,
                                                         int2* out_bodies, double* out_blk, double* out_d2,
                                                         int* moll_list, int* moll_count,
                                                         const unsigned char* __restrict__ moll_flag) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  (void)kind_unused;
  const int64_t slot = slot_off + t;
  const int64_t i = act[slot] - cand_off;
  int4 r = rows[i];
  PairIds ids = pair_ids(sv, KIND, r);
  V3 z[4], xb[4];
  pair_points(sv, ids, q, z, xb);
  out_bodies[slot] = make_int2(r.x, r.z);
  // mollified EE pairs belong to k_pair_blocks_moll: the predicate comes from
  // k_moll_classify's flag when it ran (evaluated once), else it is evaluated here
  if (KIND == KIND_EE && (moll_flag ? moll_flag[t] != 0 : ee_mollified(z, ids.eps))) {
    if (moll_list) moll_list[atomicAdd(moll_count, 1)] = (int)slot;
    return;
  }
  double* blk = out_blk + slot * PB_STRIDE;
  PairEval ev = contact_pair_eval<true, 1>(KIND, z, xb, ids.eps, kappa, dh, sv.dyn[r.x] != 0, sv.dyn[r.z] != 0,
                                           project != 0, blk);
  out_d2[slot] = ev.d2;
}

// ---------------------------------------------------------------------------
// Fused assembly of large active sets (config 2: millions of active pairs):
// records never round-trip HBM.  A warp takes a window of 32 consecutive active
// slots of one kind; each lane evaluates its pair into a compact record in shared
// memory (contact_pair_eval, as k_pair_blocks_act); the window's runs -- maximal
// lane ranges of one body pair -- are then summed, lane by lane in slot order, into
// dense run partials (aa | bb | ab blocks and both gradients in the reference's DOF
// order), which reduce_system adds to the BSR blocks as contributions of their own.
// Mollified EE pairs keep their 9-column record path (k_pair_blocks_moll).  Sums in
// fixed orders: deterministic.
constexpr int RUN_WARPS = 2;

__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int KIND>
__device__ __forceinline__ int2 run_pair(const int4* __restrict__ rows, const int* __restrict__ act, int64_t cand_off,
                                         int64_t slot_off, int64_t count, const unsigned char* __restrict__ moll_flag,
                                         int64_t t, bool& fused, int4& r) {
  fused = false;
  if (t >= count) return make_int2(-1, -1);
  r = rows[act[slot_off + t] - cand_off];
  fused = KIND == KIND_VF || !moll_flag || !moll_flag[t];
  return make_int2(r.x, r.z);
}

// lanes that start a run (fused, and a different body pair or a non-fused lane before)
__device__ __forceinline__ unsigned run_starts(bool fused, int2 bp, int lane) {
  const int px = __shfl_up_sync(0xffffffffu, bp.x, 1), py = __shfl_up_sync(0xffffffffu, bp.y, 1);
  const bool pf = __shfl_up_sync(0xffffffffu, fused ? 1 : 0, 1) != 0;
  const bool start = fused && (lane == 0 || !pf || px != bp.x || py != bp.y);
  return __ballot_sync(0xffffffffu, start);
}

template <int KIND>
__global__ void k_run_count(int64_t count, const int* __restrict__ act, int64_t cand_off,
                            const int4* __restrict__ rows, int64_t slot_off, const unsigned char* __restrict__ moll_flag,
                            int64_t n_win, int* wcount) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n_win) return;
  bool f;
  int4 r;
  const int2 bp = run_pair<KIND>(rows, act, cand_off, slot_off, count, moll_flag, 32 * w + lane, f, r);
  const unsigned m = run_starts(f, bp, lane);
  if (lane == 0) wcount[w] = __popc(m);
}

template <int KIND>
__global__ void __launch_bounds__(32 * RUN_WARPS) k_pair_runs(SceneView sv, int64_t count, const int* __restrict__ act,
                                                               int64_t cand_off, const int4* __restrict__ rows,
                                                               const double* __restrict__ q, double kappa, double dh,
                                                               int project, int64_t slot_off,
                                                               const unsigned char* __restrict__ moll_flag,
                                                               int64_t n_win, const int* __restrict__ wbase,
                                                               int2* out_bodies, double* out_d2, double* run_part,
                                                               int2* run_bodies) {
  extern __shared__ double run_sm[];  // [RUN_WARPS][32][PB_STRIDE]
  // run-sum read-out map: entry e of a run partial (aa | bb | ab, reference DOFs) ->
  // (rho, sigma) of the 24-space in which the run is summed, rho <= sigma
  __shared__ unsigned short emap[432];
  for (int e = threadIdx.x; e < 432; e += 32 * RUN_WARPS) {
    const int blk = e / 144, idx = e % 144, i = idx / 12, c = idx % 12;
    const int R = blk == 1 ? 12 + i : i, C = blk == 0 ? c : 12 + c;
    int rho = pb_rho(R / 12, R % 12), sg = pb_rho(C / 12, C % 12);
    if (sg < rho) {
      const int t = rho;
      rho = sg;
      sg = t;
    }
    emap[e] = (unsigned short)(rho * 32 + sg);
  }
  __syncthreads();
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * RUN_WARPS + wl;
  if (w >= n_win) return;
  double* recs = run_sm + (size_t)wl * 32 * PB_STRIDE;
  const int64_t t = 32 * w + lane;
  bool f;
  int4 r;
  const int2 bp = run_pair<KIND>(rows, act, cand_off, slot_off, count, moll_flag, t, f, r);
  if (t < count) {
    const int64_t slot = slot_off + t;
    out_bodies[slot] = f ? make_int2(-1, -1) : bp;  // folded pairs contribute through their run
    if (f) {
      PairIds ids = pair_ids(sv, KIND, r);
      V3 z[4], xb[4];
      pair_points(sv, ids, q, z, xb);
      PairEval ev = contact_pair_eval<true, 1>(KIND, z, xb, ids.eps, kappa, dh, sv.dyn[r.x] != 0, sv.dyn[r.z] != 0,
                                               project != 0, recs + (size_t)lane * PB_STRIDE);
      out_d2[slot] = ev.d2;
    }
  }
  const unsigned starts = run_starts(f, bp, lane);
  const unsigned fused = __ballot_sync(0xffffffffu, f);
  __syncwarp();
  const int base = wbase[w];
  unsigned rem = starts;
  // The run's Hessian sum_l Q_l M_l Q_l^T (fused pairs carry 5-column records) is
  // accumulated in the affine 24-space on the FP64 tensor core: per pair the fragments of
  // U = Q M (A operand) and Q (B operand) are formed from the record in shared memory --
  // lane (g, tq) holds row 8 t + g, column 4 kk + tq; columns 5..7 are zero padding --
  // and the six upper 8x8 tiles take two m8n8k4 steps each; pairs are added in lane
  // order (deterministic).  ~110 warp instructions per pair instead of ~430 for the
  // entry-by-entry expansion.
  const int g8 = lane >> 2, tq = lane & 3;
  for (int k = 0; rem; ++k) {
    const int l0 = __ffs(rem) - 1;
    rem &= rem - 1;
    // the run ends at the next start or the next non-fused lane
    const unsigned stop = (starts | ~fused) & ~((2u << l0) - 1u);
    const int l1 = stop ? __ffs(stop) - 1 : 32;
    double acc[6][2];
#pragma unroll
    for (int i = 0; i < 6; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int l = l0; l < l1; ++l) {
      const double* rec = recs + (size_t)l * PB_STRIDE;
      const double* ch = rec + 25;
      const double* f0 = rec + 33;
      const double* f1 = rec + 57;
      const double* M = rec + 81;
      double ua[3][2], wb[3][2];
#pragma unroll
      for (int tt = 0; tt < 3; ++tt) {
        const int rho = 8 * tt + g8, sj = rho / 3, a = rho - 3 * sj;
        const double c_ = ch[sj], p0 = f0[rho], p1 = f1[rho];
        ua[tt][0] = c_ * M[5 * a + tq] + p0 * M[15 + tq] + p1 * M[20 + tq];
        ua[tt][1] = tq == 0 ? c_ * M[5 * a + 4] + p0 * M[19] + p1 * M[24] : 0.0;
        wb[tt][0] = tq == 3 ? p0 : (a == tq ? c_ : 0.0);
        wb[tt][1] = tq == 0 ? p1 : 0.0;
      }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        dmma_f64(acc[0][0], acc[0][1], ua[0][kk], wb[0][kk]);
        dmma_f64(acc[1][0], acc[1][1], ua[0][kk], wb[1][kk]);
        dmma_f64(acc[2][0], acc[2][1], ua[0][kk], wb[2][kk]);
        dmma_f64(acc[3][0], acc[3][1], ua[1][kk], wb[1][kk]);
        dmma_f64(acc[4][0], acc[4][1], ua[1][kk], wb[2][kk]);
        dmma_f64(acc[5][0], acc[5][1], ua[2][kk], wb[2][kk]);
      }
    }
    // the 24 x 24 sum goes through the unused tails of records 0..23 (a 5-column record
    // ends at 106 of PB_STRIDE = 136 doubles): row rho in record rho
    __syncwarp();
    {
      constexpr int mi_of[6] = {0, 0, 0, 1, 1, 2}, ni_of[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        double* row = recs + (size_t)(8 * mi_of[i] + g8) * PB_STRIDE + 106 + 8 * ni_of[i] + 2 * tq;
        row[0] = acc[i][0];
        row[1] = acc[i][1];
      }
    }
    __syncwarp();
    double* out = run_part + (int64_t)(base + k) * RUN_STRIDE;
    for (int e = lane; e < RUN_STRIDE; e += 32) {
      double a = 0.0;
      if (e < 432) {
        const int m = emap[e];
        a = recs[(size_t)(m >> 5) * PB_STRIDE + 106 + (m & 31)];
      } else {
        for (int l = l0; l < l1; ++l) a += recs[(size_t)l * PB_STRIDE + (e - 432)];
      }
      out[e] = a;
    }
    const int bx = __shfl_sync(0xffffffffu, bp.x, l0), by = __shfl_sync(0xffffffffu, bp.y, l0);
    if (lane == 0) run_bodies[base + k] = make_int2(bx, by);
    __syncwarp();  // the next run rewrites the staging rows
  }
}

// the mollified active EE slots, listed ahead of the pair-block kernels so their
// (slower) 9-column records build on a side stream beside the plain EE pairs
__global__ void k_moll_classify(SceneView sv, int64_t count, const int* __restrict__ act, int64_t cand_off,
                                const int4* __restrict__ rows, const double* __restrict__ q, int64_t slot_off,
                                int* moll_list, int* moll_count, unsigned char* moll_flag) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= count) return;
  const int64_t slot = slot_off + t;
  int4 r = rows[act[slot] - cand_off];
  PairIds ids = pair_ids(sv, KIND_EE, r);
  V3 z[4], xb[4];
  pair_points(sv, ids, q, z, xb);
  const bool m = ee_mollified(z, ids.eps);
  moll_flag[t] = m ? 1 : 0;
  if (m) moll_list[atomicAdd(moll_count, 1)] = (int)slot;
}

// Warp-parallel PSD clamp of a symmetric 9x9 (padded to 10) in shared memory:
// parallel-ordered cyclic Jacobi (round-robin tournament, 5 disjoint rotations
// per round, 9 rounds per sweep), then M <- V max(w, 0) V^T.
__device__ void warp_psd9(double (*A)[11], double (*V)[11], double4* rot, int lane) {
  for (int e = lane; e < 110; e += 32) {
    const int i = e / 11, j = e % 11;
    if (j < 10) V[i][j] = (i == j) ? 1.0 : 0.0;
  }
  __syncwarp();
  double fro = 0.0;
  for (int e = lane; e < 81; e += 32) fro += A[e / 9][e % 9] * A[e / 9][e % 9];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  if (fro == 0.0) return;
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0;
    for (int e = lane; e < 81; e += 32) {
      const int i = e / 9, j = e % 9;
      if (j > i) off += A[i][j] * A[i][j];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(0xffffffffu, off, o);
    if (off <= 1e-32 * fro) break;
    for (int round = 0; round < 9; ++round) {
      // circle-method pairing: round r pairs (r, 9) and ((r + k) % 9, (r - k) % 9),
      // k = 1..4 -- every pair of 0..8 exactly once per sweep; 9 = zero padding
      if (lane < 5) {
        const int a = lane == 0 ? round : (round + lane) % 9;
        const int b = lane == 0 ? 9 : (round - lane + 9) % 9;
        const int p = min(a, b), q = max(a, b);
        double c = 1.0, sn = 0.0;
        const double apq = A[p][q];
        if (apq * apq > 1e-40 * fro) {
          const double theta = (A[q][q] - A[p][p]) * rcp_fast(2.0 * apq);
          const double th2 = theta * theta + 1.0;
          const double t = (theta >= 0.0 ? 1.0 : -1.0) * rcp_fast(fabs(theta) + th2 * rsqrt_fast(th2));
          c = rsqrt_fast(t * t + 1.0);
          sn = t * c;
        }
        rot[lane] = make_double4((double)p, (double)q, c, sn);
      }
      __syncwarp();
      // rows: B = J^T A (rows p, q of each rotation)
      for (int e = lane; e < 50; e += 32) {
        const int k = e / 10, j = e % 10;
        const double4 r = rot[k];
        const int p = (int)r.x, q = (int)r.y;
        const double ap = A[p][j], aq = A[q][j];
        A[p][j] = r.z * ap - r.w * aq;
        A[q][j] = r.w * ap + r.z * aq;
      }
      __syncwarp();
      // columns: A = B J, and V = V J
      for (int e = lane; e < 100; e += 32) {
        const int k = (e % 50) / 10, i = e % 10;
        const double4 r = rot[k];
        const int p = (int)r.x, q = (int)r.y;
        double (*X)[11] = e < 50 ? A : V;
        const double xp = X[i][p], xq = X[i][q];
        X[i][p] = r.z * xp - r.w * xq;
        X[i][q] = r.w * xp + r.z * xq;
      }
      __syncwarp();
    }
  }
  // M = V diag(max(w, 0)) V^T (w = diag A), written into A's upper triangle first
  double res[3];
  int n_res = 0;
  for (int e = lane; e < 81; e += 32) {
    const int i = e / 9, j = e % 9;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 9; ++k) acc += V[i][k] * fmax(A[k][k], 0.0) * V[j][k];
    res[n_res++] = acc;
  }
  __syncwarp();
  n_res = 0;
  for (int e = lane; e < 81; e += 32) A[e / 9][e % 9] = res[n_res++];
  __syncwarp();
}

// the deferred mollified EE pairs (9-column path), one warp per pair: lane 0
// builds the record with the unprojected 9x9 core, the warp clamps it
constexpr int MOLL_WARPS = 4;
__global__ void __launch_bounds__(32 * MOLL_WARPS) k_pair_blocks_moll(SceneView sv, const int* __restrict__ moll_list,
                                                                       const int* __restrict__ moll_count,
                                                                       const int* __restrict__ act, int64_t cand_off,
                                                                       const int4* __restrict__ rows,
                                                                       const double* __restrict__ q, double kappa,
                                                                       double dh, int project, double* out_blk,
                                                                       double* out_d2) {
  __shared__ double As[MOLL_WARPS][10][11], Vs[MOLL_WARPS][10][11];
  __shared__ double4 rots[MOLL_WARPS][5];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = *moll_count;
  for (int t = blockIdx.x * MOLL_WARPS + w; t < n; t += gridDim.x * MOLL_WARPS) {
    const int64_t slot = moll_list[t];
    double* blk = out_blk + slot * PB_STRIDE;
    if (lane == 0) {
      const int64_t i = act[slot] - cand_off;
      int4 r = rows[i];
      PairIds ids = pair_ids(sv, KIND_EE, r);
      V3 z[4], xb[4];
      pair_points(sv, ids, q, z, xb);
      PairEval ev = contact_pair_eval<true, 2>(KIND_EE, z, xb, ids.eps, kappa, dh, sv.dyn[r.x] != 0,
                                               sv.dyn[r.z] != 0, false, blk);
      out_d2[slot] = ev.d2;
    }
    __syncwarp();
    if (project) {
      double (*A)[11] = As[w];
      for (int e = lane; e < 110; e += 32) {
        const int i = e / 11, j = e % 11;
        if (j < 10) A[i][j] = (i < 9 && j < 9) ? blk[49 + 9 * i + j] : 0.0;
      }
      __syncwarp();
      warp_psd9(A, Vs[w], rots[w], lane);
      for (int e = lane; e < 81; e += 32) blk[49 + e] = A[e / 9][e % 9];
    }
    __syncwarp();
  }
}

__global__ void k_scatter_active(int64_t n, const int* __restrict__ flags, const int* __restrict__ pos, int* act) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && flags[i]) act[pos[i]] = (int)i;
}

__device__ __forceinline__ void contact_energy_part(const SceneView& sv, int kind, int64_t n,
                                                    const int4* __restrict__ rows, const double* __restrict__ q,
                                                    double kappa, double dh, double* partials, int* err, int bx,
                                                    int nbx) {
  __shared__ double sh[RED_THREADS];
  double acc = 0.0;
  double dh2 = dh * dh;
  for (int64_t i = bx * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)nbx * blockDim.x) {
    PairIds ids = pair_ids(sv, kind, rows[i]);
    V3 z[4], xb[4];
    pair_points(sv, ids, q, z, xb);
    double d2 = pair_d2(kind, z);
    if (!(d2 < dh2)) continue;
    if (!(d2 > 0.0)) atomicExch(err, 1);
    double b = kappa * barrier_terms(d2, dh).b0;
    if (kind == KIND_EE) b = mollifier_value(z, ids.eps) * b;
    acc += b;
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[bx] = sh[0];
}

__global__ void k_cand_min_d2(SceneView sv, int kind, int64_t n, const int4* __restrict__ rows,
                              const double* __restrict__ q, unsigned long long* best) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double d2 = INFINITY;
  if (i < n) {
    PairIds ids = pair_ids(sv, kind, rows[i]);
    V3 z[4], xb[4];
    pair_points(sv, ids, q, z, xb);
    d2 = pair_d2(kind, z);
  }
  for (int o = 16; o > 0; o >>= 1) d2 = fmin(d2, __shfl_xor_sync(0xffffffffu, d2, o));
  if ((threadIdx.x & 31) == 0 && d2 < INFINITY) atomicMin(best, (unsigned long long)__double_as_longlong(d2));
}

// K7: lagged friction records at q_prev for active candidates (contact.py:722-790)
__global__ void k_friction_pre(SceneView sv, int kind, int64_t n, const int4* __restrict__ rows,
                               const double* __restrict__ q, double kappa, double dh, const int* __restrict__ flags,
                               const int* __restrict__ pos, int64_t base, int2* out_bodies, double* out_rec,
                               double* out_basis) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || !flags[i]) return;
  int4 r = rows[i];
  PairIds ids = pair_ids(sv, kind, r);
  V3 z[4], xb[4];
  pair_points(sv, ids, q, z, xb);
  Closest c = closest(kind, z);
  double d = sqrt(c.d2);
  double lam = -kappa * 2.0 * d * barrier_terms(c.d2, dh).b1;
  if (kind == KIND_EE) lam = lam * mollifier_value(z, ids.eps);
  // r = einsum("ni,nik->nk", gamma, z): sequential order, no FMA (the tangent
  // helper axis below is picked by argmin |n|, so n must match numpy bitwise)
  V3 rr = xscale(c.gamma[0], z[0]);
  rr = xadd3(rr, xscale(c.gamma[1], z[1]));
  rr = xadd3(rr, xscale(c.gamma[2], z[2]));
  rr = xadd3(rr, xscale(c.gamma[3], z[3]));
  V3 nrm = V3{rr.x / d, rr.y / d, rr.z / d};
  double ax = fabs(nrm.x), ay = fabs(nrm.y), az = fabs(nrm.z);
  int pick = (ax <= ay && ax <= az) ? 0 : ((ay <= az) ? 1 : 2);
  V3 helper = V3{pick == 0 ? 1.0 : 0.0, pick == 1 ? 1.0 : 0.0, pick == 2 ? 1.0 : 0.0};
  V3 t1 = xcross(nrm, helper);
  double tn = xnorm_seq(t1);
  t1 = V3{t1.x / tn, t1.y / tn, t1.z / tn};
  V3 t2 = xcross(nrm, t1);
  double T[3][2] = {{t1.x, t2.x}, {t1.y, t2.y}, {t1.z, t2.z}};
  // c_s[j] = sum_{k in side s} gamma_k w_k[j]
  double cs[2][4];
  for (int s = 0; s < 2; ++s) {
    for (int j = 0; j < 4; ++j) cs[s][j] = 0.0;
    int k0 = side_begin(kind, s), nk = side_count(kind, s);
    for (int k = 0; k < nk; ++k) {
      double gk = c.gamma[k0 + k];
      cs[s][0] += gk;
      cs[s][1] += gk * xb[k0 + k].x;
      cs[s][2] += gk * xb[k0 + k].y;
      cs[s][3] += gk * xb[k0 + k].z;
    }
  }
  int64_t o = base + pos[i];
  double* rec = out_rec + o * FRIC_STRIDE;
  const double* qa = q + 12 * (int64_t)r.x;
  const double* qb = q + 12 * (int64_t)r.z;
  for (int m = 0; m < 2; ++m) {
    double off = 0.0;
    for (int col = 0; col < 24; ++col) {
      int s = col / 12, rem = col % 12;
      int a = rem < 3 ? rem : (rem - 3) / 3;
      int j = rem < 3 ? 0 : 1 + (rem - 3) % 3;
      double v = T[a][m] * cs[s][j];
      rec[m * 24 + col] = v;
      off += v * (s == 0 ? qa[rem] : qb[rem]);
    }
    rec[48 + m] = off;
  }
  rec[50] = lam;
  out_bodies[o] = make_int2(r.x, r.z);
  if (out_basis) {
    double* bs = out_basis + o * 6;
    for (int a = 0; a < 3; ++a) {
      bs[2 * a] = T[a][0];
      bs[2 * a + 1] = T[a][1];
    }
  }
}

// K5: ACCD over candidates with a global min (ccd.py:130-153), over both candidate lists in one launch (VF rows first, then EE): the
// heavy-tailed ACCD queries of the two kinds share one tail instead of two.
// Hot queries (rows of the hot list, already evaluated exactly by k_ccd_hot while
// the broad phase ran) take their precomputed t; queries that need >= slow_it
// iterations (hot ones included) form the next hot list.
__device__ __forceinline__ double ccd_row(const SceneView& sv, int kind, int4 row, const double* __restrict__ q,
                                          const double* __restrict__ dq, double slack,
                                          volatile const unsigned long long* cut, bool& bad, int& it) {
  PairIds ids = pair_ids(sv, kind, row);
  V3 x[4], xb[4], dx[4];
  pair_points(sv, ids, q, x, xb);
  for (int k = 0; k < 4; ++k) {
    int b = ids.body[k];
    dx[k] = sv.dyn[b] ? world_pos(dq + 12 * (int64_t)b, xb[k]) : V3{0.0, 0.0, 0.0};
  }
  return accd_query(kind, x, dx, slack, 1.0, 512, cut, bad, &it);
}

// one hot query per warp (lane 0): the queries' branch paths and iteration counts
// differ, so sharing a warp would serialise their divergent chains
__global__ void k_ccd_hot(SceneView sv, int n, const int4* __restrict__ rows, const int* __restrict__ kind,
                          const double* __restrict__ q, const double* __restrict__ dq, double slack, double* t_out,
                          int* bad_out, int* it_out) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n || (threadIdx.x & 31) != 0) return;
  bool bad = false;
  int it = 0;
  t_out[i] = ccd_row(sv, kind[i], rows[i], q, dq, slack, nullptr, bad, it);
  bad_out[i] = bad ? 1 : 0;
  it_out[i] = it;
}

__global__ void k_ccd_both(SceneView sv, int64_t n_vf, const int4* __restrict__ vf, int64_t n_ee,
                           const int4* __restrict__ ee, const double* __restrict__ q, const double* __restrict__ dq,
                           double slack, unsigned long long* tmin, int* err, HotCcd h) {
  __shared__ int4 hr[CCD_HOT_CAP];
  __shared__ int hk[CCD_HOT_CAP];
  for (int j = threadIdx.x; j < h.n; j += blockDim.x) {
    hr[j] = h.rows[j];
    hk[j] = h.kind[j];
  }
  __syncthreads();
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double t = INFINITY;
  if (i < n_vf + n_ee) {
    const int kind = i < n_vf ? KIND_VF : KIND_EE;
    const int4 r = kind == KIND_VF ? vf[i] : ee[i - n_vf];
    int hit = -1;
    for (int j = 0; j < h.n; ++j)
      if (hk[j] == kind && hr[j].x == r.x && hr[j].y == r.y && hr[j].z == r.z && hr[j].w == r.w) {
        hit = j;
        break;
      }
    int it = 0;
    if (hit >= 0) {
      t = h.t[hit];
      it = h.it[hit];
      if (h.bad[hit]) atomicExch(err, 1);
    } else {
      bool bad = false;
      t = ccd_row(sv, kind, r, q, dq, slack, tmin, bad, it);
      if (bad) atomicExch(err, 1);
    }
    if (h.slow_cap > 0 && it >= h.slow_it) {
      const unsigned at = atomicAdd(h.slow_cnt, 1u);
      if ((int)at < h.slow_cap) {
        h.slow_rows[at] = r;
        h.slow_kind[at] = kind;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) t = fmin(t, __shfl_xor_sync(0xffffffffu, t, o));
  if ((threadIdx.x & 31) == 0 && t < INFINITY) atomicMin(tmin, (unsigned long long)__double_as_longlong(t));
}

// diagnostic (ABD_CCD_STATS): per query iterations and t without the shared cut
__global__ void k_ccd_dbg(SceneView sv, int kind, int64_t n, const int4* __restrict__ rows,
                          const double* __restrict__ q, const double* __restrict__ dq, double slack, int* its,
                          double* ts) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  PairIds ids = pair_ids(sv, kind, rows[i]);
  V3 x[4], xb[4], dx[4];
  pair_points(sv, ids, q, x, xb);
  for (int k = 0; k < 4; ++k) {
    int b = ids.body[k];
    dx[k] = sv.dyn[b] ? world_pos(dq + 12 * (int64_t)b, xb[k]) : V3{0.0, 0.0, 0.0};
  }
  bool bad = false;
  int it = 0;
  ts[i] = accd_query(kind, x, dx, slack, 1.0, 512, nullptr, bad, &it);
  its[i] = it;
}

// K1: inertia + orthogonality per dynamic slot (solver.py:197-200, :283-296)
__global__ void k_body_terms(int n_dyn, const int* __restrict__ dyn_body, const double* __restrict__ mass,
                             const double* __restrict__ stiff, const double* __restrict__ q,
                             const double* __restrict__ qt, double dt, double* grad0, double* diag0,
                             double* partials, int want) {
  __shared__ double sh[RED_THREADS];
  double acc = 0.0;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_dyn; s += gridDim.x * blockDim.x) {
    int b = dyn_body[s];
    const double* M = mass + 144 * (int64_t)b;
    double qq[12], diff[12], Md[12];
    for (int c = 0; c < 12; ++c) {
      qq[c] = q[12 * (int64_t)b + c];
      diff[c] = qq[c] - qt[12 * (int64_t)b + c];
    }
    double quad = 0.0;
    for (int r = 0; r < 12; ++r) {
      double a = 0.0;
      for (int c = 0; c < 12; ++c) a += M[r * 12 + c] * diff[c];
      Md[r] = a;
      quad += diff[r] * a;
    }
    double dt2 = dt * dt;
    double k = stiff[b];
    acc += 0.5 * quad + dt2 * ortho_energy_dev(qq, k);
    if (!want) continue;
    double g[12], H[144];
    ortho_derivs_dev(qq, k, g, H);
    ortho_project_closed(qq, k, H);  // closed-form eigen-clamp via the 3x3 SVD of A
    for (int c = 0; c < 12; ++c) grad0[12 * (int64_t)s + c] = Md[c] + dt2 * g[c];
    for (int c = 0; c < 144; ++c) diag0[144 * (int64_t)s + c] = M[c] + dt2 * H[c];
  }
  if (!partials) return;
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

// K1 gradient + projected diagonal block, one warp per dynamic body: the 3x3 SVD
// of A is computed redundantly by the lanes, lanes 0..8 publish the negative
// modes of the closed-form projection (ortho_project_closed) in shared memory,
// and the 144 block entries are written coalesced (no per-thread 12x12 array)
constexpr int BT_WARPS = 8;
__global__ void __launch_bounds__(32 * BT_WARPS) k_body_derivs(int n_dyn, const int* __restrict__ dyn_body,
                                                               const double* __restrict__ mass,
                                                               const double* __restrict__ stiff,
                                                               const double* __restrict__ q,
                                                               const double* __restrict__ qt, double dt,
                                                               double* grad0, double* diag0) {
  __shared__ double modes[BT_WARPS][9][10];  // lambda (or 0 = inactive) | dA[9]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sidx = blockIdx.x * BT_WARPS + w;
  if (sidx >= n_dyn) return;
  const int b = dyn_body[sidx];
  const double* M = mass + 144 * (int64_t)b;
  const double* qb = q + 12 * (int64_t)b;
  double qq[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) qq[c] = qb[c];
  const double k = stiff[b];
  const double dt2 = dt * dt;
  const double* A = qq + 3;
  // closed-form eigenpairs (abd_misc.cuh ortho_project_closed), redundant per lane
  double S3[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) S3[a][c] = A[a] * A[c] + A[3 + a] * A[3 + c] + A[6 + a] * A[6 + c];
  if (lane == 0) {
    // all nine modes with compile-time indices (registers, no local memory)
    double sv[3], uu[3][3], vv[3][3];
    ortho_svd3(A, sv, uu, vv);
    const double k4 = 4.0 * k;
    const double r2 = 0.70710678118654752440;
#pragma unroll
    for (int m = 0; m < 9; ++m) {
      const int pp = m < 3 ? 0 : (m - 3) >> 1;
      const int i = m < 3 ? m : (pp == 2 ? 1 : 0);
      const int j = m < 3 ? m : (pp == 0 ? 1 : 2);
      const double sg = m < 3 ? 0.0 : (((m - 3) & 1) ? -1.0 : 1.0);
      const double lam = (m < 3) ? k4 * (3.0 * sv[i] * sv[i] - 1.0)
                                 : k4 * (sv[i] * sv[i] + sv[j] * sv[j] - 1.0 + sg * sv[i] * sv[j]);
      double* o = modes[w][m];
      o[0] = lam < 0.0 ? lam : 0.0;
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          o[1 + 3 * r + c] = (m < 3) ? uu[i][r] * vv[i][c] : r2 * (uu[i][r] * vv[j][c] + sg * uu[j][r] * vv[i][c]);
    }
  }
  __syncwarp();
  double G[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) G[i][j] = A[3 * i] * A[3 * j] + A[3 * i + 1] * A[3 * j + 1] + A[3 * i + 2] * A[3 * j + 2];
  const double s4 = 4.0 * k;
  double* D = diag0 + 144 * (int64_t)sidx;
  for (int e = lane; e < 144; e += 32) {
    const int r = e / 12, c = e % 12;
    double h = 0.0;
    if (r >= 3 && c >= 3) {
      const int i = (r - 3) / 3, a = (r - 3) % 3, j = (c - 3) / 3, bb = (c - 3) % 3;
      double v;
      if (i == j) {
        const double aa = A[3 * i + a] * A[3 * i + bb];
        v = 2.0 * aa + (a == bb ? G[i][i] - 1.0 : 0.0) + (S3[a][bb] - aa);
      } else {
        v = A[3 * j + a] * A[3 * i + bb] + (a == bb ? G[i][j] : 0.0);
      }
      h = s4 * v;
      for (int m = 0; m < 9; ++m) {
        const double lam = modes[w][m][0];
        if (lam < 0.0) h -= lam * modes[w][m][1 + (r - 3)] * modes[w][m][1 + (c - 3)];
      }
    }
    D[e] = M[e] + dt2 * h;
  }
  if (lane < 12) {
    double g[12];
    ortho_derivs_dev(qq, k, g, nullptr);
    const double* qtb = qt + 12 * (int64_t)b;
    double gr = 0.0;
#pragma unroll
    for (int c = 0; c < 12; ++c) gr += M[lane * 12 + c] * (qq[c] - qtb[c]);
    double gl = g[0];
#pragma unroll
    for (int c = 1; c < 12; ++c)
      if (c == lane) gl = g[c];
    grad0[12 * (int64_t)sidx + lane] = gr + dt2 * gl;
  }
}

// K1 energy only (line-search trials), one warp per dynamic slot: coalesced reads
// of the 12x12 mass block, fixed-order warp and block sums
__device__ __forceinline__ void body_energy_part(int n_dyn, const int* __restrict__ dyn_body,
                                                 const double* __restrict__ mass, const double* __restrict__ stiff,
                                                 const double* __restrict__ q, const double* __restrict__ qt,
                                                 double dt, double* partials, int bx, int nbx) {
  __shared__ double sh[RED_THREADS / 32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = nbx * (RED_THREADS / 32);
  double acc = 0.0;  // lane 0: this warp's bodies in slot order
  for (int sidx = bx * (RED_THREADS / 32) + w; sidx < n_dyn; sidx += nw) {
    const int b = dyn_body[sidx];
    const double* M = mass + 144 * (int64_t)b;
    const double* qb = q + 12 * (int64_t)b;
    const double* qtb = qt + 12 * (int64_t)b;
    double part = 0.0;
    for (int e = lane; e < 144; e += 32) {
      const int r = e / 12, c = e % 12;
      part += (qb[r] - qtb[r]) * M[e] * (qb[c] - qtb[c]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
    if (lane == 0) {
      double qq[12];
#pragma unroll
      for (int c = 0; c < 12; ++c) qq[c] = qb[c];
      acc += 0.5 * part + (dt * dt) * ortho_energy_dev(qq, stiff[b]);
    }
  }
  if (lane == 0) sh[w] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k2 = 0; k2 < RED_THREADS / 32; ++k2) t += sh[k2];
    partials[bx] = t;
  }
}

__global__ void __launch_bounds__(RED_THREADS) k_body_energy_w(int n_dyn, const int* __restrict__ dyn_body,
                                                               const double* __restrict__ mass,
                                                               const double* __restrict__ stiff,
                                                               const double* __restrict__ q,
                                                               const double* __restrict__ qt, double dt,
                                                               double* partials) {
  body_energy_part(n_dyn, dyn_body, mass, stiff, q, qt, dt, partials, blockIdx.x, gridDim.x);
}

// K6 in one launch: blocks [0, R) body terms, [R, 2R) contact VF, [2R, 3R) contact
// EE, [3R, 4R) friction (R = RED_BLOCKS).  Every part keeps its own fixed grid of R
// blocks, so the partials -- and their fixed-order sums -- are bitwise those of the
// separate kernels, while the parts run side by side.
struct EnergyArgs {
  SceneView sv;
  const double *q, *qt, *mass, *stiff;
  const int* dyn_body;
  int n_dyn, with_body;
  double dt, kappa, dh, mu, eh;
  int64_t n_vf, n_ee, n_f;
  const int4 *vf, *ee;
  const int2* fb;
  const double* frec;
  double* red4;
  int* err;
};

__global__ void __launch_bounds__(RED_THREADS) k_energy_all(EnergyArgs a) {
  const int part = blockIdx.x / RED_BLOCKS, bx = blockIdx.x % RED_BLOCKS;
  double* out = a.red4 + part * RED_BLOCKS;
  if (part == 0) {
    if (a.with_body) body_energy_part(a.n_dyn, a.dyn_body, a.mass, a.stiff, a.q, a.qt, a.dt, out, bx, RED_BLOCKS);
    else if (threadIdx.x == 0) out[bx] = 0.0;
  } else if (part < 3) {
    const int kind = part == 1 ? KIND_VF : KIND_EE;
    contact_energy_part(a.sv, kind, kind == KIND_VF ? a.n_vf : a.n_ee, kind == KIND_VF ? a.vf : a.ee, a.q, a.kappa,
                        a.dh, out, a.err, bx, RED_BLOCKS);
  } else {
    __shared__ double sh[RED_THREADS];
    double acc = 0.0;
    for (int64_t i = bx * (int64_t)blockDim.x + threadIdx.x; i < a.n_f; i += (int64_t)RED_BLOCKS * blockDim.x) {
      const int2 b = a.fb[i];
      const double* r = a.frec + i * FRIC_STRIDE;
      FricEval e = friction_eval(r, a.q + 12 * b.x, a.q + 12 * b.y, a.eh);
      acc += a.mu * r[50] * e.f0;
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[bx] = sh[0];
  }
}

void launch_energy_all(Scene& s, const double* q, const double* qt, double dt, double kappa, double dh,
                       double eps_v, double* red4, int* err) {
  EnergyArgs a;
  a.sv = view(s);
  a.q = q;
  a.qt = qt;
  a.mass = s.mass.p;
  a.stiff = s.stiff.p;
  a.dyn_body = s.dyn_body.p;
  a.n_dyn = s.n_dyn;
  a.with_body = s.comm.rank == 0 ? 1 : 0;
  a.dt = dt;
  a.kappa = kappa;
  a.dh = dh;
  a.mu = s.fric.mu;
  a.eh = eps_v * dt;
  a.n_vf = s.cands.n_vf;
  a.n_ee = s.cands.n_ee;
  a.n_f = s.fric.n;
  a.vf = s.cands.vf.p;
  a.ee = s.cands.ee.p;
  a.fb = s.fric.bodies.p;
  a.frec = s.fric.rec.p;
  a.red4 = red4;
  a.err = err;
  k_energy_all<<<4 * RED_BLOCKS, RED_THREADS, 0, s.stream>>>(a);
  note_launch("k_energy_all");
}

// K1 energy only (line-search trials): 0.5 dq^T M dq + dt^2 V_perp per dynamic slot
__global__ void k_body_energy(int n_dyn, const int* __restrict__ dyn_body, const double* __restrict__ mass,
                              const double* __restrict__ stiff, const double* __restrict__ q,
                              const double* __restrict__ qt, double dt, double* partials) {
  __shared__ double sh[RED_THREADS];
  double acc = 0.0;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_dyn; s += gridDim.x * blockDim.x) {
    int b = dyn_body[s];
    const double* M = mass + 144 * (int64_t)b;
    double qq[12], diff[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) {
      qq[c] = q[12 * (int64_t)b + c];
      diff[c] = qq[c] - qt[12 * (int64_t)b + c];
    }
    double quad = 0.0;
#pragma unroll
    for (int r = 0; r < 12; ++r) {
      double a = 0.0;
#pragma unroll
      for (int c = 0; c < 12; ++c) a += M[r * 12 + c] * diff[c];
      quad += diff[r] * a;
    }
    acc += 0.5 * quad + (dt * dt) * ortho_energy_dev(qq, stiff[b]);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

// q_tilde = q + dt qdot + dt^2 M^{-1} f (solver.py:179-190), Cholesky per body
__global__ void k_q_tilde(int B, const unsigned char* __restrict__ dyn, const double* __restrict__ mass,
                          const double* __restrict__ q, const double* __restrict__ qd, const double* __restrict__ f,
                          double dt, double* qt) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double* qb = q + 12 * (int64_t)b;
  if (!dyn[b]) {
    for (int c = 0; c < 12; ++c) qt[12 * (int64_t)b + c] = qb[c];
    return;
  }
  double L[144], y[12];
  const double* M = mass + 144 * (int64_t)b;
  for (int r = 0; r < 144; ++r) L[r] = M[r];
  for (int j = 0; j < 12; ++j) {
    double d = L[j * 12 + j];
    for (int k = 0; k < j; ++k) d -= L[j * 12 + k] * L[j * 12 + k];
    d = sqrt(d);
    L[j * 12 + j] = d;
    for (int i = j + 1; i < 12; ++i) {
      double v = L[i * 12 + j];
      for (int k = 0; k < j; ++k) v -= L[i * 12 + k] * L[j * 12 + k];
      L[i * 12 + j] = v / d;
    }
  }
  for (int i = 0; i < 12; ++i) {
    double v = f[12 * (int64_t)b + i];
    for (int k = 0; k < i; ++k) v -= L[i * 12 + k] * y[k];
    y[i] = v / L[i * 12 + i];
  }
  for (int i = 11; i >= 0; --i) {
    double v = y[i];
    for (int k = i + 1; k < 12; ++k) v -= L[k * 12 + i] * y[k];
    y[i] = v / L[i * 12 + i];
  }
  double dt2 = dt * dt;
  for (int c = 0; c < 12; ++c) qt[12 * (int64_t)b + c] = qb[c] + dt * qd[12 * (int64_t)b + c] + dt2 * y[c];
}

// trial = q + alpha * dq  (numpy: multiply then add, no FMA)
__global__ void k_axpy_q(int64_t n, const double* __restrict__ q, double alpha, const double* __restrict__ dq,
                         double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = xadd(q[i], xmul(alpha, dq[i]));
}

// ---------------------------------------------------------------------------
static const int4* rows_of(const Scene& s, int kind, int64_t& n) {
  n = kind == KIND_VF ? s.cands.n_vf : s.cands.n_ee;
  return kind == KIND_VF ? s.cands.vf.p : s.cands.ee.p;
}

void launch_scatter_active(Scene& s, int64_t n, const int* flags, const int* pos, int* act) {
  if (!n) return;
  k_scatter_active<<<grid_for(n, 256), 256, 0, s.stream>>>(n, flags, pos, act);
  note_launch("k_scatter_active");
}

void launch_pair_blocks_act(Scene& s, int kind, const double* q, double kappa, double dh, int project,
                            const int* act, int64_t slot_off, int64_t count) {
  if (count <= 0) return;
  int64_t n;
  const int4* rows = rows_of(s, kind, n);
  const int64_t cand_off = kind == KIND_VF ? 0 : s.cands.n_vf;
  int* moll_count = reinterpret_cast<int*>(s.w.ull.p + 10);
  if (kind == KIND_VF) {
    k_pair_blocks_act<KIND_VF><<<grid_for(count, 64), 64, 0, s.stream>>>(view(s), kind, count, act, cand_off, rows, q,
                                                                        kappa, dh, project, slot_off, s.pblk.bodies.p,
                                                                        s.pblk.blk.p, s.pblk.d2.p, nullptr, nullptr,
                                                                        nullptr);
  } else {
    s.w.moll.resize(std::max<int64_t>(count, 1));
    CK(cudaMemsetAsync(moll_count, 0, sizeof(int), s.stream));
    static const bool serial = getenv("ABD_MOLL_SERIAL") != nullptr;
    const int grid = (int)std::min<int64_t>(grid_for(count, MOLL_WARPS), 16 * (int64_t)s.num_sms);
    if (serial) {
      k_pair_blocks_act<KIND_EE><<<grid_for(count, 64), 64, 0, s.stream>>>(
          view(s), kind, count, act, cand_off, rows, q, kappa, dh, project, slot_off, s.pblk.bodies.p, s.pblk.blk.p,
          s.pblk.d2.p, s.w.moll.p, moll_count, nullptr);
      k_pair_blocks_moll<<<grid, 32 * MOLL_WARPS, 0, s.stream>>>(view(s), s.w.moll.p, moll_count, act, cand_off,
                                                                 rows, q, kappa, dh, project, s.pblk.blk.p,
                                                                 s.pblk.d2.p);
    } else {
      // list the mollified slots, build them on side3 while the plain EE pairs run here
      s.w.moll_flag.resize(std::max<int64_t>(count, 1));
      k_moll_classify<<<grid_for(count, 256), 256, 0, s.stream>>>(view(s), count, act, cand_off, rows, q, slot_off,
                                                                  s.w.moll.p, moll_count, s.w.moll_flag.p);
      note_launch("k_moll_classify");
      CK(cudaEventRecord(s.moll_fork_ev, s.stream));
      CK(cudaStreamWaitEvent(s.side3, s.moll_fork_ev, 0));
      k_pair_blocks_moll<<<grid, 32 * MOLL_WARPS, 0, s.side3>>>(view(s), s.w.moll.p, moll_count, act, cand_off,
                                                                rows, q, kappa, dh, project, s.pblk.blk.p,
                                                                s.pblk.d2.p);
      CK(cudaEventRecord(s.moll_ev, s.side3));
      k_pair_blocks_act<KIND_EE><<<grid_for(count, 64), 64, 0, s.stream>>>(
          view(s), kind, count, act, cand_off, rows, q, kappa, dh, project, slot_off, s.pblk.bodies.p, s.pblk.blk.p,
          s.pblk.d2.p, nullptr, nullptr, s.w.moll_flag.p);
      CK(cudaStreamWaitEvent(s.stream, s.moll_ev, 0));
    }
    note_launch("k_pair_blocks_moll");
  }
  note_launch("k_pair_blocks");
}

// Fused run assembly over all active contact pairs (VF slots [0, n_vf_act), EE after):
// counts the runs per window, scans them (one host read of the total), evaluates.
void launch_pair_runs(Scene& s, const double* q, double kappa, double dh, int project, const int* act,
                      int64_t n_vf_act, int64_t total) {
  cudaStream_t st = s.stream;
  const int64_t n_ee_act = total - n_vf_act;
  const int64_t win_vf = (n_vf_act + 31) / 32, win_ee = (n_ee_act + 31) / 32, nwin = win_vf + win_ee;
  PairBlockSet& pb = s.pblk;
  pb.run_wcount.resize(nwin + 1);
  pb.run_wbase.resize(nwin + 1);
  int* moll_count = reinterpret_cast<int*>(s.w.ull.p + 10);
  const int4* vf = s.cands.vf.p;
  const int4* ee = s.cands.ee.p;
  const int64_t cand_ee = s.cands.n_vf;
  const unsigned char* mflag = nullptr;
  if (n_ee_act > 0) {
    s.w.moll.resize(std::max<int64_t>(n_ee_act, 1));
    s.w.moll_flag.resize(std::max<int64_t>(n_ee_act, 1));
    CK(cudaMemsetAsync(moll_count, 0, sizeof(int), st));
    k_moll_classify<<<grid_for(n_ee_act, 256), 256, 0, st>>>(view(s), n_ee_act, act, cand_ee, ee, q, n_vf_act,
                                                              s.w.moll.p, moll_count, s.w.moll_flag.p);
    note_launch("k_moll_classify");
    mflag = s.w.moll_flag.p;
  }
  CK(cudaMemsetAsync(pb.run_wcount.p + nwin, 0, sizeof(int), st));
  if (win_vf) {
    k_run_count<KIND_VF><<<grid_for(32 * win_vf, 256), 256, 0, st>>>(n_vf_act, act, 0, vf, 0, nullptr, win_vf,
                                                                     pb.run_wcount.p);
    note_launch("k_run_count");
  }
  if (win_ee) {
    k_run_count<KIND_EE><<<grid_for(32 * win_ee, 256), 256, 0, st>>>(n_ee_act, act, cand_ee, ee, n_vf_act, mflag,
                                                                     win_ee, pb.run_wcount.p + win_vf);
    note_launch("k_run_count");
  }
  scan_exclusive_i32(s, pb.run_wcount.p, pb.run_wbase.p, nwin + 1);
  int hn = 0;
  CK(cudaMemcpyAsync(&hn, pb.run_wbase.p + nwin, sizeof(int), cudaMemcpyDeviceToHost, st));
  SSYNC(st);
  pb.n_runs = hn;
  pb.run_part.resize(std::max<int64_t>(hn, 1) * RUN_STRIDE);
  pb.run_bodies.resize(std::max(hn, 1));
  const size_t smem = (size_t)RUN_WARPS * 32 * PB_STRIDE * sizeof(double);
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_pair_runs<KIND_VF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_pair_runs<KIND_EE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  if (win_vf) {
    k_pair_runs<KIND_VF><<<grid_for(win_vf, RUN_WARPS), 32 * RUN_WARPS, smem, st>>>(
        view(s), n_vf_act, act, 0, vf, q, kappa, dh, project, 0, nullptr, win_vf, pb.run_wbase.p, pb.bodies.p,
        pb.d2.p, pb.run_part.p, pb.run_bodies.p);
    note_launch("k_pair_runs");
  }
  if (win_ee) {
    // the mollified EE pairs build their 9-column records beside the runs
    const int grid = (int)std::min<int64_t>(grid_for(n_ee_act, MOLL_WARPS), 16 * (int64_t)s.num_sms);
    CK(cudaEventRecord(s.moll_fork_ev, st));
    CK(cudaStreamWaitEvent(s.side3, s.moll_fork_ev, 0));
    k_pair_blocks_moll<<<grid, 32 * MOLL_WARPS, 0, s.side3>>>(view(s), s.w.moll.p, moll_count, act, cand_ee, ee, q,
                                                              kappa, dh, project, pb.blk.p, pb.d2.p);
    note_launch("k_pair_blocks_moll");
    CK(cudaEventRecord(s.moll_ev, s.side3));
    k_pair_runs<KIND_EE><<<grid_for(win_ee, RUN_WARPS), 32 * RUN_WARPS, smem, st>>>(
        view(s), n_ee_act, act, cand_ee, ee, q, kappa, dh, project, n_vf_act, mflag, win_ee,
        pb.run_wbase.p + win_vf, pb.bodies.p, pb.d2.p, pb.run_part.p, pb.run_bodies.p);
    note_launch("k_pair_runs");
    CK(cudaStreamWaitEvent(st, s.moll_ev, 0));
  }
}

void launch_cand_min_d2(Scene& s, int kind, const double* q, unsigned long long* best) {
  int64_t n;
  const int4* rows = rows_of(s, kind, n);
  if (!n) return;
  k_cand_min_d2<<<grid_for(n, 128), 128, 0, s.stream>>>(view(s), kind, n, rows, q, best);
  note_launch("k_cand_min_d2");
}

void launch_friction_pre(Scene& s, int kind, const double* q, double kappa, double dh, const int* flags,
                         const int* pos, int64_t base, double* basis_out) {
  int64_t n;
  const int4* rows = rows_of(s, kind, n);
  if (!n) return;
  k_friction_pre<<<grid_for(n, 128), 128, 0, s.stream>>>(view(s), kind, n, rows, q, kappa, dh, flags, pos, base,
                                                         s.fric.bodies.p, s.fric.rec.p, basis_out);
  note_launch("k_friction_pre");
}

void launch_ccd_hot(Scene& s, const double* q, const double* dq, double slack) {
  Scene::Work& w = s.w;
  w.hot_pending = false;
  static const bool off = getenv("ABD_CCD_NO_HOT") != nullptr;
  if (off || w.hot_n == 0) return;
  w.hot_t.resize(CCD_HOT_CAP);
  w.hot_bad.resize(CCD_HOT_CAP);
  w.hot_it.resize(CCD_HOT_CAP);
  CK(cudaEventRecord(s.hot_fork_ev, s.stream));
  CK(cudaStreamWaitEvent(s.side2, s.hot_fork_ev, 0));
  k_ccd_hot<<<w.hot_n, 32, 0, s.side2>>>(view(s), w.hot_n, w.hot_rows.p, w.hot_kind.p, q, dq, slack, w.hot_t.p,
                                         w.hot_bad.p, w.hot_it.p);
  note_launch("k_ccd_hot");
  CK(cudaEventRecord(s.hot_ev, s.side2));
  w.hot_pending = true;
}

void launch_ccd_both(Scene& s, const double* q, const double* dq, double slack, unsigned long long* tmin,
                     int* err, bool track) {
  const int64_t n = s.cands.n_vf + s.cands.n_ee;
  Scene::Work& w = s.w;
  HotCcd h{};
  if (track) {
    w.slow_rows.resize(CCD_HOT_CAP);
    w.slow_kind.resize(CCD_HOT_CAP);
    h.slow_rows = w.slow_rows.p;
    h.slow_kind = w.slow_kind.p;
    h.slow_cnt = reinterpret_cast<unsigned*>(w.ull.p + 12);
    h.slow_cap = CCD_HOT_CAP;
    h.slow_it = CCD_SLOW_IT;  // slow_cnt was zeroed with the broad phase's scalars
    if (w.hot_pending) {
      CK(cudaStreamWaitEvent(s.stream, s.hot_ev, 0));
      h.rows = w.hot_rows.p;
      h.kind = w.hot_kind.p;
      h.t = w.hot_t.p;
      h.bad = w.hot_bad.p;
      h.it = w.hot_it.p;
      h.n = w.hot_n;
    }
    w.hot_pending = false;
  }
  if (!n) return;
  k_ccd_both<<<grid_for(n, 128), 128, 0, s.stream>>>(view(s), s.cands.n_vf, s.cands.vf.p, s.cands.n_ee, s.cands.ee.p,
                                                    q, dq, slack, tmin, err, h);
  note_launch("k_ccd");
  static const bool stats = getenv("ABD_CCD_SLOW") != nullptr;
  if (stats) {
    // diagnostic: the slowest queries (iterations, t, row) of this call
    for (int kind = 0; kind < 2; ++kind) {
      int64_t nk;
      const int4* rows = rows_of(s, kind, nk);
      if (!nk) continue;
      DVec<int> its;
      DVec<double> ts;
      its.resize(nk);
      ts.resize(nk);
      k_ccd_dbg<<<grid_for(nk, 128), 128, 0, s.stream>>>(view(s), kind, nk, rows, q, dq, slack, its.p, ts.p);
      std::vector<int> hi(nk);
      std::vector<double> ht(nk);
      std::vector<int4> hr(nk);
      its.download(hi.data(), nk, s.stream);
      ts.download(ht.data(), nk, s.stream);
      CK(cudaMemcpyAsync(hr.data(), rows, nk * sizeof(int4), cudaMemcpyDeviceToHost, s.stream));
      SSYNC(s.stream);
      std::vector<int64_t> idx(nk);
      for (int64_t i = 0; i < nk; ++i) idx[i] = i;
      std::partial_sort(idx.begin(), idx.begin() + std::min<int64_t>(6, nk), idx.end(),
                        [&](int64_t a, int64_t b) { return hi[a] > hi[b]; });
      fprintf(stderr, "[ccd slow] kind=%d", kind);
      for (int64_t k = 0; k < std::min<int64_t>(6, nk); ++k) {
        const int4 r = hr[idx[k]];
        fprintf(stderr, " (%d,%d,%d,%d:it=%d,t=%.3e)", r.x, r.y, r.z, r.w, hi[idx[k]], ht[idx[k]]);
      }
      fprintf(stderr, "\n");
    }
  }
}

void launch_body_terms(Scene& s, const double* q, const double* qt, double dt, double* grad0, double* diag0,
                       double* partials, int want) {
  if (!want) {
    k_body_energy_w<<<RED_BLOCKS, RED_THREADS, 0, s.stream>>>(s.n_dyn, s.dyn_body.p, s.mass.p, s.stiff.p, q, qt, dt,
                                                              partials);
    note_launch("k_body_energy");
    return;
  }
  if (!partials && s.n_dyn) {
    k_body_derivs<<<grid_for(s.n_dyn, BT_WARPS), 32 * BT_WARPS, 0, s.stream>>>(s.n_dyn, s.dyn_body.p, s.mass.p,
                                                                               s.stiff.p, q, qt, dt, grad0, diag0);
    note_launch("k_body_derivs");
    return;
  }
  k_body_terms<<<RED_BLOCKS, RED_THREADS, 0, s.stream>>>(s.n_dyn, s.dyn_body.p, s.mass.p, s.stiff.p, q, qt, dt, grad0,
                                                         diag0, partials, want);
  note_launch("k_body_terms");
}

void launch_q_tilde(Scene& s, const double* q, const double* qd, const double* f, double dt, double* qt) {
  if (!s.B) return;
  k_q_tilde<<<grid_for(s.B, 64), 64, 0, s.stream>>>(s.B, s.dyn.p, s.mass.p, q, qd, f, dt, qt);
  note_launch("k_q_tilde");
}

void launch_axpy_q(Scene& s, const double* q, double alpha, const double* dq, double* out, int64_t n) {
  if (!n) return;
  k_axpy_q<<<grid_for(n, 256), 256, 0, s.stream>>>(n, q, alpha, dq, out);
  note_launch("k_axpy_q");
}

}  // namespace abd
