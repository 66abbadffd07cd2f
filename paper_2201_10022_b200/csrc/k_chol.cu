// K4 (direct): sparse block Cholesky with iterative refinement on the device,
// the reference's Newton linear solve BlockCholesky(A).solve_refined(-g,
// rel_tol=1e-8) (sparse.py:90-161, solver.py:345-348) restated for B200.
//
// Per Newton iteration:
//   * analysis (host, C++, on a worker thread overlapping the pair-block
//     kernels): the exactly-zero pattern blocks (overlapping body boxes without
//     an active contact) are dropped; the remaining block graph is ordered by
//     tree contraction (rake / compress) + minimum degree on the 2-core; the
//     symbolic factor (fill), the elimination tree and the task graph are packed
//     into one plan buffer.  A plan whose graph contains the new structure is
//     reused (extra blocks hold exact zeros).
//   * factor + solve (k_chol_sched): a persistent grid of warps runs node tasks
//     from one GPU-wide FIFO.  A node's column (D = A_jj - sum L_jk L_jk^T, 12x12
//     Cholesky, L_ij = (A_ij - sum L_ik L_jk^T) L_jj^-T) and its forward
//     substitution start when its elimination-tree children are done; its
//     backward substitution when its parent's is done.  Left-looking with a fixed
//     update order: deterministic, whatever the schedule.  The 12x12 pivots are
//     in-register Cholesky factors (shuffles, rsqrt per pivot).  Isolated nodes
//     (no coupling) are single factor + solve tasks.
//   * refinement solves reuse the factor and 1 / L_cc (same kernel, no factor).
//   * refinement exactly as solve_refined: r = b - A x over the resident BSR,
//     stop when |r| <= rel_tol |b|, at most 3 corrections.
// A failed pivot raises ABD_ERR_FACTORIZATION with the smallest failing
// dynamic slot (sparse.py:18-26 semantics).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <condition_variable>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <iterator>
#include <numeric>
#include <queue>
#include <vector>

#include "driver.h"

namespace abd {

constexpr int CH_THREADS = 128;
constexpr int CH_HW = CH_THREADS / 32;  // warps per CTA (one node per warp, lane t = row t)
constexpr int CH_MAX_GRID = 128;        // task-graph CTAs: the graph's width, not the GPU's

// Plan layout (one packed int buffer uploaded per analysis).  L holds the n
// diagonal blocks first (L_jj at index j), then the off-diagonal blocks.
// Scheduling: every node is a task; a node's factor column (and its forward
// substitution) may start once all its elimination-tree children are done (its
// column only reads L blocks of descendants), its backward substitution once its
// parent's is done.  Ready tasks go through one GPU-wide FIFO; every warp of a
// persistent grid pops, runs and pushes, so a component's levels spread over all
// SMs instead of one CTA (a settled pile couples ~2,300 bodies into one component
// whose elimination tree is ~60 levels deep).  Isolated nodes (no coupling) are
// independent factor + solve tasks handed out by a second counter.
struct CholView {
  int n, n_coupled, n_leaves, n_iso, n_tasks;  // factor-mode tasks: partials + off-diagonal blocks + n_coupled
  const int* leaves;    // coupled nodes with no elimination-tree child, deepest first
  const int* iso;       // isolated nodes
  const int* parent;    // elimination-tree parent (node id) or -1
  const int* nchild;    // elimination-tree child counts (initial dependency counters)
  const int* child_ptr; // n + 1: children of each node
  const int* child_idx;
  const int* col_ptr;   // n + 1: off-diagonal blocks of column j (index k -> L block n + k)
  const int* blk_row;   // per off block: row node i
  const int* blk_col;   // per off block: column node j
  const int* bsr_row;   // BSR row_ptr / col: A(i, j) found by binary search in row i (absent: fill)
  const int* bsr_col;
  int* apos;            // per off block: BSR position of A(i, j) or -1, filled by k_chol_apos
  const int* row_ptr;   // n + 1: range into row_blk (blocks L_jk, k eliminated before j)
  const int* row_blk;   // L block index
  const int* row_col;   // column node k of each row_blk entry
  const int* upd_ptr;   // per off block: range into upd
  const int2* upd;      // (L_ik, L_jk) block index pairs
  const int* diag_pos;  // BSR diagonal block positions
  const double* val;    // BSR values
  double* L;            // L blocks, 144 doubles each (row-major)
  double* dinv;         // n x 12: 1 / L_jj[c][c]
  int* bad;
  int* dep;             // n: remaining children (reset per launch)
  int* bleft;           // n: remaining off-diagonal block tasks of each column
  int* queue;           // task slots (item ids, see k_chol_sched); -1 = not yet pushed
  unsigned* ctr;        // [0] pop head, [1] push tail, [2] unused, [3] tasks done
  unsigned long long* trace;  // optional (ABD_CHOL_TRACE_TASKS): per popped slot (item, t_pop, t_start, t_end)
  // factor mode: the products of a heavy diagonal / block task are split into
  // partial tasks (fixed chunks, summed in chunk order by the finalizing warp)
  int n_part, n_init;   // partial tasks; initially ready partials (the leaves')
  const int* part_ptr;  // n + 1: partials of node j (its diagonal's, then its column blocks')
  const int4* part;     // per partial: (0 diagonal / 1 block, node / block, lo, hi) product range
  const int* dnp;       // n: diagonal partials of node j (1 = unsplit chol_diag)
  const int* bpart;     // per off block: its first partial
  const int* bnp;       // per off block: its partial count (>= 1)
  const int* init;      // n_init: partials of the leaves, deepest leaves first
  double* scratch;      // n_part x PART_STRIDE partial sums
  int* dleft;           // n: remaining diagonal partials
  int* bgate;           // per off block: remaining partials + 1 (the column's diagonal)
  // dataflow schedule (k_chol_flow): items in topological order, readiness by flags
  const int* fseq;      // n_coupled + nbo: per node in elimination order its diagonal (j), then its blocks (n + b)
  const int* eord;      // n_coupled: coupled nodes in elimination order
  int* flag;            // n + nbo: = epoch once L block (factor) / y_j (solve, index j) is final
  int* xflag;           // n: = epoch once x_j (backward substitution) is final
  int* sflag;           // n: = epoch once sbuf[k] (the parent block's update sum of column k) is final
  double* sbuf;         // n x 144: S_pk = A_pk - sum L_pi L_ki^T of each column's parent block p
};
constexpr int PART_STRIDE = 156;  // 12 x 13 (the forward-substitution column rides along)

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}


// position of block (r, c) in the sorted-column CSR, or -1
__device__ __forceinline__ int bsr_find(const int* __restrict__ row_ptr, const int* __restrict__ col, int r, int c) {
  int lo = row_ptr[r], hi = row_ptr[r + 1] - 1;
  while (lo <= hi) {
    const int m = (lo + hi) >> 1;
    const int cm = col[m];
    if (cm == c) return m;
    if (cm < c) lo = m + 1;
    else hi = m - 1;
  }
  return -1;
}

// full-warp shuffles: every lane of a warp runs the same node, so no partial-mask
// convergence checks are generated
__device__ __forceinline__ double hshfl(unsigned mask, double v, int src) { return __shfl_sync(mask, v, src); }

// 1/sqrt(x): MUFU.RSQ64H seed (rsqrt.approx.f64) + 2 Newton steps (>= 53 bits);
// no libdevice slow-path call, whose register saves would push the in-register
// factor onto the stack.  Pivots are never denormal (p > 0 checked, SPD blocks).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-0.5 * x, r * r, 1.5);
  r = r * fma(-0.5 * x, r * r, 1.5);
  return r;
}

// In-register 12x12 Cholesky on a warp: lane t < 12 holds row t of the
// symmetric matrix in d[]; on exit d[] is row t of L (zeros above the diagonal)
// and every lane holds rinv[c] = 1 / L_cc.  Division-free; the next pivot is
// formed by its owner lane right after the scaling and broadcast at once, so
// the trailing-update shuffles stay off the critical path (measured 5.2k ->
// 3.3k cycles per factor on B200, tools/ubench/chol12.cu).
__device__ __forceinline__ bool chol12(unsigned mask, int t, double d[12], double rinv[12]) {
  bool ok = true;
  double p = hshfl(mask, d[0], 0);
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    ok = ok && (p > 0.0);
    const double pp = p > 0.0 ? p : 1.0;
    const double r = rsqrt_nr(pp);
    rinv[c] = r;
    if (t == c) d[c] = pp * r;
    else if (t > c) d[c] *= r;
    double pn = 0.0;
    if (c < 11) pn = hshfl(mask, fma(-d[c], d[c], d[c + 1]), c + 1);
    // constant trip counts (k > c as a predicate) so both loops fully unroll and
    // d[] stays in registers
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      if (k > c) {
        const double lkc = hshfl(mask, d[c], k);
        if (t >= k) d[k] = fma(-d[c], lkc, d[k]);
      }
    }
    p = pn;
  }
#pragma unroll
  for (int c = 0; c < 12; ++c)
    if (c > t) d[c] = 0.0;
  return ok;
}

// lane t: acc <- row t of (L^-1 acc) for lower-triangular L whose row t is lrow
__device__ __forceinline__ double lower_solve12(unsigned mask, int t, double acc, const double lrow[12],
                                                const double rinv[12]) {
  double y = 0.0;
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    const double yc = hshfl(mask, acc, c) * rinv[c];
    if (t == c) y = yc;
    if (t > c) acc = fma(-lrow[c], yc, acc);
  }
  return y;
}

// lane t: row t of (L^-T acc); lcol = column t of L (lcol[c] = L[c][t])
__device__ __forceinline__ double upper_solve12(unsigned mask, int t, double acc, const double lcol[12],
                                                const double rinv[12]) {
  double x = 0.0;
#pragma unroll
  for (int c = 11; c >= 0; --c) {
    const double xc = hshfl(mask, acc, c) * rinv[c];
    if (t == c) x = xc;
    if (t < c) acc = fma(-lcol[c], xc, acc);
  }
  return x;
}

// BSR positions of the factor's off-diagonal source blocks, all nodes in parallel
// (takes the binary searches off the dependency-serial critical path)
__global__ void k_chol_apos(CholView v) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= v.n) return;
  for (int b = v.col_ptr[j]; b < v.col_ptr[j + 1]; ++b) v.apos[b] = bsr_find(v.bsr_row, v.bsr_col, v.blk_row[b], j);
}

// Data produced by other warps during the launch (L blocks, 1/L_cc, x) is read
// with ld.global.cg: L1 is not coherent across SMs, and a neighbouring node's
// entries may share a line that this SM cached before they were written.
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int atom_dec_acq_rel(int* p) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

// ---- per-warp operand pipeline: 12x12 blocks staged in shared memory by cp.async
// (L2-coherent .cg copies; NST stages in flight so the L2 round trips of
// consecutive block products overlap), products on the FP64 tensor core
// (mma.m8n8k4.f64: a 12x12x12 product = 2x2 output tiles x 3 k-steps, padded to
// 16x16; measured 327 vs 1509 cycles per product for the 12-lane FMA form,
// tools/ubench/chol_upd.cu).
constexpr int NST = 6;
struct WarpSmem {
  double stage[NST][2][144];  // two operand blocks per stage
  double vec[NST][12];        // y_k per stage (diagonal task)
  double pa[144];             // prefetched A block (A_jj / A_ij)
  double pl[144];             // prefetched L_jj (block task)
  double pv[12];              // prefetched b_j (diagonal task) / 1 / L_jj[c][c] (block task)
  double S[12][13];           // result rows (+ the forward-substitution column) / L_jj rows
  double dv[NST][12];         // 1 / L_kk[c][c] per stage (k_chol_flow: a child's parent block)
};

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_pipe() { asm volatile("cp.async.wait_group %0;" ::"n"(NST - 2) : "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// stage one 12x12 block (1152 B = 72 x 16 B) with the whole warp
__device__ __forceinline__ void stage_block(double* dst, const double* src, int lane) {
  for (int c = lane; c < 72; c += 32) cp16(dst + 2 * c, src + 2 * c);
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Warp-wide 12x12 products on m8n8k4 fragments.  Lane l holds A / B fragment
// entries (row 8 mi + (l >> 2), col 4 kk + (l & 3)) -- the same pattern for both
// operands, since B = M^T in col layout reads M row-major -- and accumulator
// entries (row 8 mi + (l >> 2), col 8 ni + 2 (l & 3) + e).  One accumulator set
// per k-step keeps the three MMAs of a tile independent.
struct Acc {
  double c[3][2][2][2];
};
__device__ __forceinline__ void acc_zero(Acc& a) {
#pragma unroll
  for (int i = 0; i < 24; ++i) (&a.c[0][0][0][0])[i] = 0.0;
}
// a -= X Y^T (X, Y 12x12 row-major in shared memory); ycol: optional 12-vector in
// column 12 of Y^T (the forward substitution's y_k rides along in the padding)
__device__ __forceinline__ void acc_sub_xyt(Acc& a, const double* X, const double* Y, const double* ycol, int lane) {
  const int r = lane >> 2, k4 = lane & 3;
#pragma unroll
  for (int kk = 0; kk < 3; ++kk) {
    double fa[2], fb[2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
      const bool in = 8 * mi + r < 12;
      fa[mi] = in ? -X[(8 * mi + r) * 12 + 4 * kk + k4] : 0.0;
      fb[mi] = in ? Y[(8 * mi + r) * 12 + 4 * kk + k4] : ((ycol && mi == 1 && r == 4) ? ycol[4 * kk + k4] : 0.0);
    }
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) dmma(a.c[kk][mi][ni][0], a.c[kk][mi][ni][1], fa[mi], fb[ni]);
  }
}
// out[r][c] = base[r][c] + acc (r, c < 12; column 12 = vbase[r] + acc when vbase)
__device__ __forceinline__ void acc_store(const Acc& a, const double* base, const double* vbase,
                                          double (*out)[13], int lane) {
  const int r = lane >> 2, c2 = 2 * (lane & 3);
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = 8 * mi + r, col = 8 * ni + c2 + e;
        const double s = a.c[0][mi][ni][e] + a.c[1][mi][ni][e] + a.c[2][mi][ni][e];
        if (row < 12 && col < 12) out[row][col] = (base ? base[row * 12 + col] : 0.0) + s;
        else if (row < 12 && col == 12 && vbase) out[row][12] = vbase[row] + s;
      }
}

// g[r][c] (12 x 13, row-major) = the accumulator (column 12: the ycol products)
__device__ __forceinline__ void acc_store_raw(const Acc& a, double* g, int lane) {
  const int r = lane >> 2, c2 = 2 * (lane & 3);
#pragma unroll
  for (int mi = 0; mi < 2; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = 8 * mi + r, col = 8 * ni + c2 + e;
        if (row < 12 && col < 13) g[row * 13 + col] = a.c[0][mi][ni][e] + a.c[1][mi][ni][e] + a.c[2][mi][ni][e];
      }
}

struct WarpSmem;
__device__ __forceinline__ void diag_finish(const CholView& v, int j, double* x, WarpSmem& sm);
__device__ __forceinline__ void block_finish(const CholView& v, int bb, WarpSmem& sm);

// Diagonal task of node j.  factor: D = A_jj - sum_k L_jk L_jk^T over the row list
// (fixed order), L_jj = chol(0.5 (D + D^T)), y_j = L_jj^-1 (b_j - sum_k L_jk y_k).
// !factor: y_j only, with the resident factor.
__device__ __forceinline__ void chol_diag(const CholView& v, int j, const double* __restrict__ b, double* x,
                                          bool factor, WarpSmem& sm) {
  const int t = threadIdx.x & 31, tt = t < 12 ? t : 0;
  const unsigned mask = 0xffffffffu;
  double d[12], rinv[12];
  const int e0 = v.row_ptr[j], U = v.row_ptr[j + 1] - e0;
  if (!factor) {  // refinement solve: y_j = L_jj^-1 (b_j - sum_k L_jk y_k), scalar
    double acc = b[12 * (int64_t)j + tt];
    for (int e = e0; e < e0 + U; ++e) {
      const double* Lk = v.L + 144 * (int64_t)v.row_blk[e] + 12 * tt;
      const double* yk = x + 12 * (int64_t)v.row_col[e];
      double s2 = 0.0;
#pragma unroll
      for (int m = 0; m < 12; ++m) s2 = fma(Lk[m], __ldcg(yk + m), s2);
      acc -= s2;
    }
    const double* Ld = v.L + 144 * (int64_t)j + 12 * tt;
    const double* di = v.dinv + 12 * (int64_t)j;
#pragma unroll
    for (int m = 0; m < 12; ++m) {
      d[m] = Ld[m];
      rinv[m] = di[m];
    }
    const double y = lower_solve12(mask, t, acc, d, rinv);
    if (t < 12) x[12 * (int64_t)j + t] = y;
    return;
  }
  // prefetch A_jj and b_j, then the row list's L_jk / y_k stages
  stage_block(sm.pa, v.val + 144 * (int64_t)v.diag_pos[j], t);
  if (t < 6) cp16(sm.pv + 2 * t, b + 12 * (int64_t)j + 2 * t);
  cp_commit();
  auto issue = [&](int u) {
    const int e = e0 + u;
    stage_block(sm.stage[u % NST][0], v.L + 144 * (int64_t)v.row_blk[e], t);
    if (t < 6) cp16(sm.vec[u % NST] + 2 * t, x + 12 * (int64_t)v.row_col[e] + 2 * t);
  };
  for (int p = 0; p < NST - 1; ++p) {
    if (p < U) issue(p);
    cp_commit();
  }
  Acc ac;
  acc_zero(ac);
  for (int u = 0; u < U; ++u) {
    cp_wait_pipe();
    __syncwarp(mask);
    const double* Lk = sm.stage[u % NST][0];
    acc_sub_xyt(ac, Lk, Lk, sm.vec[u % NST], t);
    __syncwarp(mask);
    if (u + NST - 1 < U) issue(u + NST - 1);
    cp_commit();
  }
  cp_wait_all();
  __syncwarp(mask);
  acc_store(ac, sm.pa, sm.pv, sm.S, t);
  __syncwarp(mask);
  diag_finish(v, j, x, sm);
}

// D (+ the right-hand side in column 12) in sm.S -> L_jj, 1 / L_jj[c][c], y_j
__device__ __forceinline__ void diag_finish(const CholView& v, int j, double* x, WarpSmem& sm) {
  const int t = threadIdx.x & 31, tt = t < 12 ? t : 0;
  const unsigned mask = 0xffffffffu;
  double d[12], rinv[12];
  double (*S)[13] = sm.S;
  // symmetrise (sparse.py:117: cholesky(0.5 (D + D^T)))
#pragma unroll
  for (int c = 0; c < 12; ++c) d[c] = 0.5 * (S[tt][c] + S[c][tt]);
  const double acc = S[tt][12];
  __syncwarp(mask);
  const bool ok = chol12(mask, t, d, rinv);
  if (!ok && t == 0) atomicMin(v.bad, j);
  if (t < 12) {
    double* Ld = v.L + 144 * (int64_t)j + 12 * t;
#pragma unroll
    for (int c = 0; c < 12; ++c) Ld[c] = d[c];
    double mine = rinv[0];
#pragma unroll
    for (int c = 1; c < 12; ++c)
      if (c == t) mine = rinv[c];
    v.dinv[12 * (int64_t)j + t] = mine;
  }
  const double y = lower_solve12(mask, t, acc, d, rinv);
  if (t < 12) x[12 * (int64_t)j + t] = y;
}

// Block task: L_ij = (A_ij - sum_u L_ik L_jk^T) L_jj^-T for one off-diagonal block of
// column j (its update pairs in fixed order), after j's diagonal task.
__device__ __forceinline__ void chol_block(const CholView& v, int bb, WarpSmem& sm) {
  const int t = threadIdx.x & 31, tt = t < 12 ? t : 0;
  const unsigned mask = 0xffffffffu;
  const int j = v.blk_col[bb];
  const int ap = v.apos[bb];
  // prefetch A_ij (absent: fill), L_jj and 1 / L_jj[c][c], then the update stages
  if (ap >= 0) stage_block(sm.pa, v.val + 144 * (int64_t)ap, t);
  stage_block(sm.pl, v.L + 144 * (int64_t)j, t);
  if (t < 6) cp16(sm.pv + 2 * t, v.dinv + 12 * (int64_t)j + 2 * t);
  cp_commit();
  const int u0 = v.upd_ptr[bb], U = v.upd_ptr[bb + 1] - u0;
  auto issue = [&](int u) {
    const int2 pq = v.upd[u0 + u];
    stage_block(sm.stage[u % NST][0], v.L + 144 * (int64_t)pq.x, t);  // L_ik
    stage_block(sm.stage[u % NST][1], v.L + 144 * (int64_t)pq.y, t);  // L_jk
  };
  for (int p = 0; p < NST - 1; ++p) {
    if (p < U) issue(p);
    cp_commit();
  }
  Acc ac;
  acc_zero(ac);
  for (int u = 0; u < U; ++u) {
    cp_wait_pipe();
    __syncwarp(mask);
    acc_sub_xyt(ac, sm.stage[u % NST][0], sm.stage[u % NST][1], nullptr, t);
    __syncwarp(mask);
    if (u + NST - 1 < U) issue(u + NST - 1);
    cp_commit();
  }
  cp_wait_all();
  __syncwarp(mask);
  acc_store(ac, ap >= 0 ? sm.pa : nullptr, nullptr, sm.S, t);
  __syncwarp(mask);
  block_finish(v, bb, sm);
}

// lane t: row t of X with X L_jj^T = B (forward substitution against the rows of
// L_jj); brow = row t of B (stride 1), Lj = L_jj rows, rinv = 1 / L_jj[c][c]
__device__ __forceinline__ void trsm_row(const double* brow, const double* Lj, const double* rv, double xr[12]) {
  double bt[12], rinv[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    bt[c] = brow[c];
    rinv[c] = rv[c];
  }
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    double s = bt[c];
#pragma unroll
    for (int m = 0; m < 12; ++m)
      if (m < c) s = fma(-Lj[12 * c + m], xr[m], s);
    xr[c] = s * rinv[c];
  }
}

// S = A_ij - sum (in sm.S), L_jj in sm.pl, 1 / L_jj[c][c] in sm.pv: L_ij = S L_jj^-T
__device__ __forceinline__ void block_finish(const CholView& v, int bb, WarpSmem& sm) {
  const int t = threadIdx.x & 31, tt = t < 12 ? t : 0;
  const unsigned mask = 0xffffffffu;
  double xr[12];
  trsm_row(sm.S[tt], sm.pl, sm.pv, xr);
  __syncwarp(mask);
  if (t < 12) {
    double* Lo = v.L + 144 * (int64_t)(v.n + bb) + 12 * t;
#pragma unroll
    for (int c = 0; c < 12; ++c) Lo[c] = xr[c];
  }
}

// Partial of a split diagonal task: -sum over row entries [lo, hi) of L_jk L_jk^T
// (and -sum L_jk y_k in column 12) into out (12 x 13).
__device__ __forceinline__ void chol_diag_part(const CholView& v, int lo, int hi, const double* x, double* out,
                                               WarpSmem& sm) {
  const int t = threadIdx.x & 31;
  const unsigned mask = 0xffffffffu;
  const int U = hi - lo;
  auto issue = [&](int u) {
    const int e = lo + u;
    stage_block(sm.stage[u % NST][0], v.L + 144 * (int64_t)v.row_blk[e], t);
    if (t < 6) cp16(sm.vec[u % NST] + 2 * t, x + 12 * (int64_t)v.row_col[e] + 2 * t);
  };
  for (int p = 0; p < NST - 1; ++p) {
    if (p < U) issue(p);
    cp_commit();
  }
  Acc ac;
  acc_zero(ac);
  for (int u = 0; u < U; ++u) {
    cp_wait_pipe();
    __syncwarp(mask);
    const double* Lk = sm.stage[u % NST][0];
    acc_sub_xyt(ac, Lk, Lk, sm.vec[u % NST], t);
    __syncwarp(mask);
    if (u + NST - 1 < U) issue(u + NST - 1);
    cp_commit();
  }
  cp_wait_all();
  __syncwarp(mask);
  acc_store_raw(ac, out, t);
}

// Partial of a split block task: -sum over update pairs [lo, hi) of L_ik L_jk^T into out.
__device__ __forceinline__ void chol_block_part(const CholView& v, int lo, int hi, double* out, WarpSmem& sm) {
  const int t = threadIdx.x & 31;
  const unsigned mask = 0xffffffffu;
  const int U = hi - lo;
  auto issue = [&](int u) {
    const int2 pq = v.upd[lo + u];
    stage_block(sm.stage[u % NST][0], v.L + 144 * (int64_t)pq.x, t);  // L_ik
    stage_block(sm.stage[u % NST][1], v.L + 144 * (int64_t)pq.y, t);  // L_jk
  };
  for (int p = 0; p < NST - 1; ++p) {
    if (p < U) issue(p);
    cp_commit();
  }
  Acc ac;
  acc_zero(ac);
  for (int u = 0; u < U; ++u) {
    cp_wait_pipe();
    __syncwarp(mask);
    acc_sub_xyt(ac, sm.stage[u % NST][0], sm.stage[u % NST][1], nullptr, t);
    __syncwarp(mask);
    if (u + NST - 1 < U) issue(u + NST - 1);
    cp_commit();
  }
  cp_wait_all();
  __syncwarp(mask);
  acc_store_raw(ac, out, t);
}

// sm.S (12 x 13) = base + the partials p0 .. p0 + np - 1 in order (written by other warps)
__device__ __forceinline__ void sum_partials(const CholView& v, const double* base, const double* vbase, int p0, int np,
                                             WarpSmem& sm) {
  const int t = threadIdx.x & 31;
  for (int e = t; e < PART_STRIDE; e += 32) {
    const int r = e / 13, c = e % 13;
    double a = c < 12 ? (base ? base[12 * r + c] : 0.0) : (vbase ? vbase[r] : 0.0);
    for (int q = 0; q < np; ++q) a += __ldcg(v.scratch + (int64_t)(p0 + q) * PART_STRIDE + e);
    sm.S[r][c] = a;
  }
  __syncwarp();
}

// The last partial of a split diagonal: D = A_jj + partials, b_j + partials -> diag_finish.
__device__ __forceinline__ void chol_diag_final(const CholView& v, int j, int p0, int np, const double* b, double* x,
                                                WarpSmem& sm) {
  sum_partials(v, v.val + 144 * (int64_t)v.diag_pos[j], b + 12 * (int64_t)j, p0, np, sm);
  diag_finish(v, j, x, sm);
}

// The last of a block's partials and its column's diagonal: S = A_ij + partials,
// L_ij = S L_jj^-T.
__device__ __forceinline__ void chol_block_final(const CholView& v, int bb, WarpSmem& sm) {
  const int t = threadIdx.x & 31;
  const int j = v.blk_col[bb];
  for (int e = t; e < 144; e += 32) sm.pl[e] = __ldcg(v.L + 144 * (int64_t)j + e);
  if (t < 12) sm.pv[t] = __ldcg(v.dinv + 12 * (int64_t)j + t);
  const int ap = v.apos[bb];
  sum_partials(v, ap >= 0 ? v.val + 144 * (int64_t)ap : nullptr, nullptr, v.bpart[bb], v.bnp[bb], sm);
  block_finish(v, bb, sm);
}

// Backward task of node j: x_j = L_jj^-T (y_j - sum_i L_ij^T x_i) over its column.
__device__ __forceinline__ void chol_backward(const CholView& v, int j, double* x, WarpSmem& sm) {
  const int t = threadIdx.x & 31, tt = t < 12 ? t : 0;
  const unsigned mask = 0xffffffffu;
  // L_jj, 1 / L_jj[c][c] and the column's blocks L_ij with x_i staged by cp.async
  // (all loads in flight together instead of one dependent L2 round trip per block)
  stage_block(sm.pl, v.L + 144 * (int64_t)j, t);
  if (t < 6) cp16(sm.pv + 2 * t, v.dinv + 12 * (int64_t)j + 2 * t);
  cp_commit();
  const int c0 = v.col_ptr[j], U = v.col_ptr[j + 1] - c0;
  auto issue = [&](int u) {
    const int bb = c0 + u;
    stage_block(sm.stage[u % NST][0], v.L + 144 * (int64_t)(v.n + bb), t);
    if (t < 6) cp16(sm.vec[u % NST] + 2 * t, x + 12 * (int64_t)v.blk_row[bb] + 2 * t);
  };
  for (int p = 0; p < NST - 1; ++p) {
    if (p < U) issue(p);
    cp_commit();
  }
  double acc = ldcg(x + 12 * (int64_t)j + tt);
  for (int u = 0; u < U; ++u) {
    cp_wait_pipe();
    __syncwarp(mask);
    const double* Lb = sm.stage[u % NST][0] + tt;  // column tt of L_ij
    const double* xi = sm.vec[u % NST];
    double s2 = 0.0;
#pragma unroll
    for (int r = 0; r < 12; ++r) s2 = fma(Lb[12 * r], xi[r], s2);
    acc -= s2;
    __syncwarp(mask);
    if (u + NST - 1 < U) issue(u + NST - 1);
    cp_commit();
  }
  cp_wait_all();
  __syncwarp(mask);
  double lcol[12], rinv[12];
#pragma unroll
  for (int m = 0; m < 12; ++m) {
    lcol[m] = sm.pl[12 * m + tt];
    rinv[m] = sm.pv[m];
  }
  const double xv = upper_solve12(mask, t, acc, lcol, rinv);
  __syncwarp(mask);
  if (t < 12) x[12 * (int64_t)j + t] = xv;
}

// Isolated node: factor (or reuse) L_jj and solve both triangles in one task.
__device__ __forceinline__ void chol_isolated(const CholView& v, int j, const double* __restrict__ b, double* x,
                                              bool factor, double (*S)[13]) {
  const int t = threadIdx.x & 31, tt = t < 12 ? t : 0;
  const unsigned mask = 0xffffffffu;
  double d[12], rinv[12];
  const double acc = b[12 * (int64_t)j + tt];
  if (factor) {
    const double* A = v.val + 144 * (int64_t)v.diag_pos[j] + 12 * tt;
#pragma unroll
    for (int c = 0; c < 12; ++c) d[c] = A[c];
    __syncwarp(mask);
    if (t < 12) {
#pragma unroll
      for (int c = 0; c < 12; ++c) S[t][c] = d[c];
    }
    __syncwarp(mask);
#pragma unroll
    for (int c = 0; c < 12; ++c) d[c] = 0.5 * (d[c] + S[c][tt]);
    const bool ok = chol12(mask, t, d, rinv);
    if (!ok && t == 0) atomicMin(v.bad, j);
    if (t < 12) {
      double* Ld = v.L + 144 * (int64_t)j + 12 * t;
#pragma unroll
      for (int c = 0; c < 12; ++c) Ld[c] = d[c];
      double mine = rinv[0];
#pragma unroll
      for (int c = 1; c < 12; ++c)
        if (c == t) mine = rinv[c];
      v.dinv[12 * (int64_t)j + t] = mine;
    }
  } else {
    const double* Ld = v.L + 144 * (int64_t)j + 12 * tt;
    const double* di = v.dinv + 12 * (int64_t)j;
#pragma unroll
    for (int m = 0; m < 12; ++m) {
      d[m] = Ld[m];
      rinv[m] = di[m];
    }
  }
  const double y = lower_solve12(mask, t, acc, d, rinv);
  // column t of L from the rows (transpose through shared memory)
  __syncwarp(mask);
  if (t < 12) {
#pragma unroll
    for (int c = 0; c < 12; ++c) S[t][c] = d[c];
  }
  __syncwarp(mask);
  double lcol[12];
#pragma unroll
  for (int c = 0; c < 12; ++c) lcol[c] = S[c][tt];
  const double xv = upper_solve12(mask, t, y, lcol, rinv);
  __syncwarp(mask);
  if (t < 12) x[12 * (int64_t)j + t] = xv;
}

__global__ void k_chol_sched_init(CholView v, int factor) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int nbo = v.col_ptr[v.n];
  if (i < v.n) {
    v.dep[i] = v.nchild[i];
    v.bleft[i] = v.col_ptr[i + 1] - v.col_ptr[i];
    if (factor) v.dleft[i] = v.dnp[i];
  }
  if (factor && i < nbo) v.bgate[i] = v.bnp[i] + 1;
  if (factor) {
    if (i < v.n_tasks) v.queue[i] = i < v.n_init ? v.init[i] : -1;
  } else if (i < 2 * v.n_coupled) {
    v.queue[i] = i < v.n_leaves ? v.leaves[i] : -1;
  }
  if (i < 4) v.ctr[i] = i == 1 ? (unsigned)(factor ? v.n_init : v.n_leaves) : 0u;
}

// Isolated nodes (no coupling): one independent factor + solve per warp.
__global__ void __launch_bounds__(CH_THREADS) k_chol_iso(CholView v, const double* __restrict__ b, double* x,
                                                         int factor) {
  __shared__ double Ss[CH_HW][12][13];
  const int hw = threadIdx.x >> 5;
  for (int i = blockIdx.x * CH_HW + hw; i < v.n_iso; i += gridDim.x * CH_HW)
    chol_isolated(v, v.iso[i], b, x, factor != 0, Ss[hw]);
}

__device__ __forceinline__ void push_task(const CholView& v, int item) {
  const unsigned slot = atomicAdd(v.ctr + 1, 1u);
  st_release(v.queue + slot, item);
}

__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// node j is complete (its column of L and y_j): the task that becomes ready -- the
// backward task at a root, or the parent's diagonal task once its last child is
// done -- or -1.  Lane 0 only, after the warp's writes are fenced.
__device__ __forceinline__ int node_ready(const CholView& v, int j) {
  const int p = v.parent[j];
  if (p < 0) return v.n + j;
  return atom_dec_acq_rel(v.dep + p) == 1 ? p : -1;
}

// push items [a, b) except the first, which is returned (the caller's continuation)
__device__ __forceinline__ int push_rest(const CholView& v, int a, int b) {
  if (b - a > 1) {
    const unsigned slot = atomicAdd(v.ctr + 1, (unsigned)(b - a - 1));
    for (int c = a + 1; c < b; ++c) st_release(v.queue + slot + (c - a - 1), c);
  }
  return b > a ? a : -1;
}

// factor mode: node j is complete; the parent's partials when it becomes ready (the
// first one returned, the others pushed), the backward task at a root, or -1
__device__ __forceinline__ int node_ready_f(const CholView& v, int j, int bwd0) {
  const int p = v.parent[j];
  if (p < 0) return bwd0 + j;
  if (atom_dec_acq_rel(v.dep + p) != 1) return -1;
  return push_rest(v, v.part_ptr[p], v.part_ptr[p + 1]);
}

// factor mode, whole warp: node j's diagonal is final; its unsplit column blocks and
// the split ones whose partials are all done become ready -- one lane per block, the
// first returned (warp-uniform), the others pushed with one slot reservation; no
// blocks: node done
__device__ __forceinline__ int diag_done_warp(const CholView& v, int j, int bwd0) {
  const int t = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const int c0 = v.col_ptr[j], c1 = v.col_ptr[j + 1];
  if (c1 == c0) {
    int r = -1;
    if (t == 0) r = node_ready_f(v, j, bwd0);
    return __shfl_sync(full, r, 0);
  }
  int first = -1;
  for (int base = c0; base < c1; base += 32) {
    const int c = base + t;
    bool ready = false;
    if (c < c1) ready = v.bnp[c] == 0 || atom_dec_acq_rel(v.bgate + c) == 1;
    unsigned m = __ballot_sync(full, ready);
    if (!m) continue;
    if (first < 0) {
      const int lead = __ffs(m) - 1;
      first = v.n_part + base + lead;
      m &= ~(1u << lead);
    }
    const int k = __popc(m);
    unsigned slot = 0;
    if (t == 0 && k) slot = atomicAdd(v.ctr + 1, (unsigned)k);
    slot = __shfl_sync(full, slot, 0);
    if ((m >> t) & 1u) st_release(v.queue + slot + __popc(m & ((1u << t) - 1u)), v.n_part + c);
  }
  return first;
}

// Persistent factor (+ forward / backward substitution) over the task FIFO of the
// coupled nodes.  Factor mode: items [0, P) are partial tasks (a diagonal's or a
// block's products in fixed chunks; an unsplit diagonal runs chol_diag whole), then
// [P, P + nbo) block finals, then backward tasks.  A node's partials are all
// released together when its last child completes, so a block's update sum runs
// beside its column's diagonal; the last of a split task's partials (by atomic
// count) sums them in chunk order and finishes it: deterministic, whatever the
// schedule.  Solve mode (refinement, preconditioner): j < n -> forward task of node
// j, n + j -> backward task.  A warp that makes
// a task ready runs one of them itself next (continuation: chains of the
// elimination tree never go through the FIFO) and pushes the others.  A warp that
// pops a slot not yet pushed polls it with backoff until it is filled or every
// task is done; every unpushed slot is produced by a warp that is running a task,
// so the grid cannot deadlock, whatever the residency.  The grid is sized to the
// task graph's width, not the GPU: idle pollers would only load L2.
__global__ void __launch_bounds__(CH_THREADS) k_chol_sched(CholView v, const double* __restrict__ b, double* x,
                                                           int factor) {
  extern __shared__ __align__(16) unsigned char ch_smem[];
  const int hw = threadIdx.x >> 5, t = threadIdx.x & 31;
  WarpSmem& sm = reinterpret_cast<WarpSmem*>(ch_smem)[hw];
  const unsigned mask = 0xffffffffu;
  const bool fac = factor != 0;
  const int total = fac ? v.n_tasks : 2 * v.n_coupled;
  const int nbo = v.col_ptr[v.n];
  const int bwd0 = fac ? v.n_part + nbo : v.n;  // first backward item
  constexpr int EXIT = -2;
  int next = -1;  // continuation task (warp-uniform)
  for (;;) {
    int item;
    unsigned long long t_pop = 0;
    if (next >= 0) {
      item = next;
      next = -1;
      fence_acq_rel();  // lane 0 acquired the dependency; order every lane's reads after it
    } else {
      int idx = 0;
      if (t == 0) idx = (int)atomicAdd(v.ctr, 1u);
      idx = __shfl_sync(mask, idx, 0);
      if (idx >= total) break;
      if (v.trace) t_pop = gtimer();
      item = -1;
      if (t == 0) {
        unsigned ns = 32;
        while ((item = ld_relaxed(v.queue + idx)) < 0) {
          if (ld_relaxed(reinterpret_cast<const int*>(v.ctr + 3)) >= total) {
            item = EXIT;
            break;
          }
          __nanosleep(ns);
          ns = min(2u * ns, 256u);
        }
      }
      item = __shfl_sync(mask, item, 0);
      if (item == EXIT) break;
      item = ld_acquire(v.queue + idx);  // every lane acquires the producer's writes
    }
    const unsigned long long t_start = v.trace ? gtimer() : 0;
    int info = 0;
    if (fac && item < v.n_part) {  // partial of a diagonal or block task
      const int4 pt = v.part[item];
      if (pt.x == 0) {
        const int j = pt.y;
        const int np = v.dnp[j];
        bool fin = true;
        if (np == 1) {
          chol_diag(v, j, b, x, true, sm);
        } else {
          chol_diag_part(v, pt.z, pt.w, x, v.scratch + (int64_t)item * PART_STRIDE, sm);
          fence_acq_rel();
          __syncwarp(mask);
          int last = 0;
          if (t == 0) last = atom_dec_acq_rel(v.dleft + j) == 1;
          fin = __shfl_sync(mask, last, 0) != 0;
          if (fin) {
            fence_acq_rel();
            chol_diag_final(v, j, v.part_ptr[j], np, b, x, sm);
          }
        }
        if (fin) {
          fence_acq_rel();
          __syncwarp(mask);
          next = diag_done_warp(v, j, bwd0);
        }
        info = pt.w - pt.z;
      } else {
        const int bb = pt.y;
        chol_block_part(v, pt.z, pt.w, v.scratch + (int64_t)item * PART_STRIDE, sm);
        fence_acq_rel();
        __syncwarp(mask);
        if (t == 0 && atom_dec_acq_rel(v.bgate + bb) == 1) next = v.n_part + bb;
        info = pt.w - pt.z;
      }
    } else if (fac && item < bwd0) {  // a block after its column's diagonal (and its partials, if split)
      const int bb = item - v.n_part;
      if (v.bnp[bb] == 0) chol_block(v, bb, sm);  // unsplit: its update sum and L_jj^-T here
      else chol_block_final(v, bb, sm);
      fence_acq_rel();
      __syncwarp(mask);
      if (t == 0) {
        const int j = v.blk_col[bb];
        if (atom_dec_acq_rel(v.bleft + j) == 1) next = node_ready_f(v, j, bwd0);
      }
    } else if (!fac && item < v.n) {  // diagonal task (solve mode: forward substitution only)
      const int j = item;
      chol_diag(v, j, b, x, fac, sm);
      fence_acq_rel();
      __syncwarp(mask);
      if (t == 0) {
        info = v.row_ptr[j + 1] - v.row_ptr[j];
        next = node_ready(v, j);
      }
    } else {  // backward task
      const int j = item - bwd0;
      chol_backward(v, j, x, sm);
      fence_acq_rel();
      __syncwarp(mask);
      if (t == 0) {
        const int c0 = v.child_ptr[j], c1 = v.child_ptr[j + 1];
        if (c1 - c0 > 1) {
          const unsigned slot = atomicAdd(v.ctr + 1, (unsigned)(c1 - c0 - 1));
          for (int c = c0 + 1; c < c1; ++c) st_release(v.queue + slot + (c - c0 - 1), bwd0 + v.child_idx[c]);
        }
        if (c1 > c0) next = bwd0 + v.child_idx[c0];
      }
    }
    if (t == 0) {
      const unsigned done = atomicAdd(v.ctr + 3, 1u);
      if (v.trace) {
        unsigned long long* o = v.trace + 4 * (int64_t)done;
        o[0] = (unsigned long long)(unsigned)item | ((unsigned long long)(unsigned)info << 32);
        o[1] = t_pop ? t_pop : t_start;
        o[2] = t_start;
        o[3] = gtimer();
      }
    }
    next = __shfl_sync(mask, next, 0);
  }
}

// ---- dataflow schedule: owner-computes with readiness flags --------------------
// Every L block (and every forward / backward substitution of a node) is one item;
// items are handed out in a topological order (elimination order: a node's
// diagonal, then its column blocks; then the backward substitutions in reverse
// order) by one atomic counter.  The warp that takes an item accumulates its update
// list in the plan's fixed order (so the result is bitwise that of the unsplit task
// graph, whatever the schedule), waiting on each operand's epoch flag as it comes:
// products whose operands are final are done while later ones are still being
// computed, so only the last update, the 12x12 pivot and the triangular solve of
// each level stay on the elimination tree's critical path (the FIFO task graph
// released a node's whole update sum only once its last child was done).  An item
// only waits on items earlier in the order, all of which are held by running warps:
// the least waiting item's operands are being produced, so the grid cannot
// deadlock, whatever its size or residency.  A wait longer than FLOW_TIMEOUT_NS
// (an inconsistent plan) raises a factorization error instead of hanging.
constexpr unsigned long long FLOW_TIMEOUT_NS = 2000000000ull;
constexpr unsigned FLOW_SLEEP_MAX = 64;  // poll back-off cap (ns): the flag hop is on the critical path

__device__ __forceinline__ void cp_wait_dyn(int k) {
  switch (k) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
  }
}

// lane 0 polls flags f0 (and f1 when >= 0) with acquire loads until both equal ep;
// the warp barrier then orders every lane's following loads and cp.async copies
// after the producer's writes.  false on timeout (raised as a factorization error).
__device__ __forceinline__ bool flow_wait(const CholView& v, const int* fl, int f0, int f1, int ep) {
  const int t = threadIdx.x & 31;
  int ok = 1;
  if (t == 0) {
    unsigned ns = 32;
    unsigned long long t0 = 0;
    while (ld_acquire(fl + f0) != ep || (f1 >= 0 && ld_acquire(fl + f1) != ep)) {
      const unsigned long long now = gtimer();
      if (!t0) t0 = now;
      else if (now - t0 > FLOW_TIMEOUT_NS) {
        ok = 0;
        atomicMin(v.bad, -1);
        break;
      }
      __nanosleep(ns);
      ns = min(2u * ns, FLOW_SLEEP_MAX);
    }
  }
  return __shfl_sync(0xffffffffu, ok, 0) != 0;
}

// every lane with `active` polls its flag fl[idx] (one L2 round trip per round for the
// whole warp) until all equal ep; then a warp barrier (as flow_wait)
__device__ __forceinline__ bool flow_wait_lanes(const CholView& v, const int* fl, bool active, int idx, int ep) {
  const unsigned mask = 0xffffffffu;
  bool done = !active;
  unsigned ns = 32;
  unsigned long long t0 = 0;
  for (;;) {
    if (!done) done = ld_acquire(fl + idx) == ep;
    if (__all_sync(mask, done)) break;
    const unsigned long long now = gtimer();
    if (!t0) t0 = now;
    else if (now - t0 > FLOW_TIMEOUT_NS) {
      if ((threadIdx.x & 31) == 0) atomicMin(v.bad, -1);
      __syncwarp(mask);
      return false;
    }
    __nanosleep(ns);
    ns = min(2u * ns, FLOW_SLEEP_MAX);
  }
  __syncwarp(mask);
  return true;
}

// every lane's writes, then the warp barrier, then lane 0's release store (cumulative:
// it publishes what the barrier ordered before it)
__device__ __forceinline__ void flow_release(int* p, int ep) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) st_release(p, ep);
}

// A list of U update items whose operands are L blocks a[u] (and b[u] when paired)
// read through a window of 32 items held one per lane: their operand indices and
// readiness are loaded together (one L2 round trip for 32 flags), so items whose
// operands are long final cost no per-item flag latency.
struct FlowWin {
  int base = 0, nready = 0;  // items [base, base + nready) known final
  int a = -1, b = -1, c = -1;  // this lane's item operands (c: y_k node for rows)
};

// refresh the window at item `from` of a row list (diagonal: L_jk, y_k) or an update
// list (block: L_ik, L_jk)
__device__ __forceinline__ void flow_window(const CholView& v, FlowWin& w, bool rows, int lo, int U, int from, int ep) {
  const int t = threadIdx.x & 31;
  const int u = from + t;
  bool rdy = true;
  w.a = w.b = w.c = -1;
  if (u < U) {
    if (rows) {
      w.a = v.row_blk[lo + u];
      w.c = v.row_col[lo + u];
      // L_jk of a child k (j = k's parent: the first block of column k) is this
      // diagonal's to finish: ready once k's diagonal and its update sum S_jk are
      w.b = w.a - v.n == v.col_ptr[w.c];
      rdy = w.b ? (ld_relaxed(v.sflag + w.c) == ep && ld_relaxed(v.flag + w.c) == ep)
                : ld_relaxed(v.flag + w.a) == ep;
    } else {
      const int2 pq = v.upd[lo + u];
      w.a = pq.x;
      w.b = pq.y;
      rdy = ld_relaxed(v.flag + pq.x) == ep && ld_relaxed(v.flag + pq.y) == ep;
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, rdy);
  w.base = from;
  w.nready = m == 0xffffffffu ? 32 : __ffs(~m) - 1;
  if (w.nready > 0) {
    // the relaxed reads above saw the producers' releases: the fence makes them
    // acquires, and the warp barrier orders every lane's copies after them
    fence_acq_rel();
    __syncwarp();
  }
}

// Accumulate the list in order into ac (subtracting products), staging operands by
// cp.async as they become final.  rows: X = Y = L_jk with y_k riding along.
__device__ __forceinline__ bool flow_accumulate(const CholView& v, Acc& ac, bool rows, int lo, int U, const double* x,
                                                int ep, WarpSmem& sm) {
  const int t = threadIdx.x & 31;
  const unsigned mask = 0xffffffffu;
  FlowWin w;
  int issued = 0;
  bool ok = true;
  unsigned fin = 0;  // stages holding a child's parent block to finish (bit = stage)
  auto issue = [&](int u) {
    const int src = u - w.base;
    const int a = __shfl_sync(mask, w.a, src);
    const int bb = __shfl_sync(mask, rows ? w.c : w.b, src);
    const int par = rows ? __shfl_sync(mask, w.b, src) : 0;
    const int sl = u % NST;
    if (par) {  // S_jk, L_kk, 1 / L_kk[c][c], y_k
      stage_block(sm.stage[sl][0], v.sbuf + 144 * (int64_t)bb, t);
      stage_block(sm.stage[sl][1], v.L + 144 * (int64_t)bb, t);
      if (t < 6) cp16(sm.dv[sl] + 2 * t, v.dinv + 12 * (int64_t)bb + 2 * t);
      fin |= 1u << sl;
    } else {
      fin &= ~(1u << sl);
      stage_block(sm.stage[sl][0], v.L + 144 * (int64_t)a, t);
      if (!rows) stage_block(sm.stage[sl][1], v.L + 144 * (int64_t)bb, t);
    }
    if (rows && t < 6) cp16(sm.vec[sl] + 2 * t, x + 12 * (int64_t)bb + 2 * t);
    cp_commit();
  };
  for (int u = 0; u < U; ++u) {
    while (issued <= u) {
      if (issued >= w.base + w.nready) {
        flow_window(v, w, rows, lo, U, issued, ep);
        if (w.nready == 0) {
          // block on this item's operands (the window now starts at it); the rest of
          // the window is polled again when reached
          const int a0 = __shfl_sync(mask, w.a, 0), b0 = __shfl_sync(mask, w.b, 0), c0 = __shfl_sync(mask, w.c, 0);
          const int f0 = rows ? (b0 ? (int)(v.sflag - v.flag) + c0 : a0) : a0;
          const int f1 = rows ? (b0 ? c0 : -1) : b0;
          ok = flow_wait(v, v.flag, f0, f1, ep) && ok;
          w.nready = 1;
        }
      }
      issue(issued++);
    }
    // issue ahead: within the window's ready run, and past a fully ready window into the
    // next one (loaded while the staged copies are in flight)
    while (issued < U && issued < u + NST) {
      if (issued >= w.base + w.nready) {
        if (w.nready < 32) break;
        flow_window(v, w, rows, lo, U, issued, ep);
        if (w.nready == 0) break;
      }
      issue(issued++);
    }
    cp_wait_dyn(issued - u - 1);
    __syncwarp(mask);
    if (rows && ((fin >> (u % NST)) & 1u)) {
      // a child's parent block: L_jk = S_jk L_kk^-T here (one flag hop and one block
      // staging fewer on the critical path than a block task), published for the
      // other updates and the backward substitution, then its product
      const int sl = u % NST;
      const int fb = v.row_blk[lo + u];
      double xr[12];
      trsm_row(sm.stage[sl][0] + 12 * (t < 12 ? t : 0), sm.stage[sl][1], sm.dv[sl], xr);
      __syncwarp(mask);
      if (t < 12) {
        double* Lo = v.L + 144 * (int64_t)fb + 12 * t;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          sm.stage[sl][0][12 * t + c] = xr[c];
          Lo[c] = xr[c];
        }
      }
      flow_release(v.flag + fb, ep);
      __syncwarp(mask);
    }
    if (rows) acc_sub_xyt(ac, sm.stage[u % NST][0], sm.stage[u % NST][0], sm.vec[u % NST], t);
    else acc_sub_xyt(ac, sm.stage[u % NST][0], sm.stage[u % NST][1], nullptr, t);
    __syncwarp(mask);
  }
  return ok;
}


// Persistent dataflow factor (+ forward and backward substitution); !factor: the two
// substitutions with the resident factor.  Items: factor: [0, m + nbo) fseq, then m
// backward substitutions in reverse elimination order; solve: [0, m) forward
// substitutions in elimination order, then the m backward ones.
__global__ void __launch_bounds__(CH_THREADS) k_chol_flow(CholView v, const double* __restrict__ b, double* x,
                                                          int factor, int ep) {
  extern __shared__ __align__(16) unsigned char ch_smem[];
  const int hw = threadIdx.x >> 5, t = threadIdx.x & 31, tt = t < 12 ? t : 0;
  WarpSmem& sm = reinterpret_cast<WarpSmem*>(ch_smem)[hw];
  const unsigned mask = 0xffffffffu;
  const bool fac = factor != 0;
  const int m = v.n_coupled;
  const int nbo = v.col_ptr[v.n];
  const int nf = fac ? m + nbo : m;
  const int total = nf + m;
  for (;;) {
    int idx = 0;
    if (t == 0) idx = (int)atomicAdd(v.ctr, 1u);
    idx = __shfl_sync(mask, idx, 0);
    if (idx >= total) break;
    const unsigned long long t_start = v.trace ? gtimer() : 0;
    unsigned long long t_rdy = 0;
    if (idx < nf) {
      const int code = fac ? v.fseq[idx] : v.eord[idx];
      if (code < v.n && fac) {  // diagonal of node j: D = A_jj - sum L_jk L_jk^T, L_jj, y_j
        const int j = code;
        const int e0 = v.row_ptr[j], U = v.row_ptr[j + 1] - e0;
        stage_block(sm.pa, v.val + 144 * (int64_t)v.diag_pos[j], t);
        if (t < 6) cp16(sm.pv + 2 * t, b + 12 * (int64_t)j + 2 * t);
        cp_commit();
        Acc ac;
        acc_zero(ac);
        flow_accumulate(v, ac, true, e0, U, x, ep, sm);
        if (v.trace) t_rdy = gtimer();
        cp_wait_all();
        __syncwarp(mask);
        acc_store(ac, sm.pa, sm.pv, sm.S, t);
        __syncwarp(mask);
        diag_finish(v, j, x, sm);
        flow_release(v.flag + j, ep);
      } else if (code < v.n) {  // solve mode: y_j = L_jj^-1 (b_j - sum_k L_jk y_k)
        const int j = code;
        const int e0 = v.row_ptr[j], U = v.row_ptr[j + 1] - e0;
        double acc = b[12 * (int64_t)j + tt];
        for (int e = e0; e < e0 + U; ++e) {
          const int k = v.row_col[e];
          flow_wait(v, v.flag, k, -1, ep);
          const double* Lk = v.L + 144 * (int64_t)v.row_blk[e] + 12 * tt;
          const double* yk = x + 12 * (int64_t)k;
          double s2 = 0.0;
#pragma unroll
          for (int q = 0; q < 12; ++q) s2 = fma(Lk[q], __ldcg(yk + q), s2);
          acc -= s2;
        }
        double d[12], rinv[12];
        const double* Ld = v.L + 144 * (int64_t)j + 12 * tt;
        const double* di = v.dinv + 12 * (int64_t)j;
#pragma unroll
        for (int q = 0; q < 12; ++q) {
          d[q] = Ld[q];
          rinv[q] = di[q];
        }
        const double y = lower_solve12(mask, t, acc, d, rinv);
        if (t < 12) x[12 * (int64_t)j + t] = y;
        flow_release(v.flag + j, ep);
      } else {  // block L_ij = (A_ij - sum L_ik L_jk^T) L_jj^-T
        const int bb = code - v.n;
        const int j = v.blk_col[bb];
        const int ap = v.apos[bb];
        if (ap >= 0) stage_block(sm.pa, v.val + 144 * (int64_t)ap, t);
        cp_commit();
        const int u0 = v.upd_ptr[bb], U = v.upd_ptr[bb + 1] - u0;
        Acc ac;
        acc_zero(ac);
        flow_accumulate(v, ac, false, u0, U, nullptr, ep, sm);
        if (bb == v.col_ptr[j]) {
          // j's parent block: publish S = A_pj - sum for the parent's diagonal, which
          // finishes L_pj itself
          cp_wait_all();
          __syncwarp(mask);
          acc_store(ac, ap >= 0 ? sm.pa : nullptr, nullptr, sm.S, t);
          __syncwarp(mask);
          if (t < 12) {
            double* So = v.sbuf + 144 * (int64_t)j + 12 * t;
#pragma unroll
            for (int c = 0; c < 12; ++c) So[c] = sm.S[t][c];
          }
          flow_release(v.sflag + j, ep);
          goto item_done;
        }
        flow_wait(v, v.flag, j, -1, ep);  // L_jj and 1 / L_jj[c][c]
        if (v.trace) t_rdy = gtimer();
        stage_block(sm.pl, v.L + 144 * (int64_t)j, t);
        if (t < 6) cp16(sm.pv + 2 * t, v.dinv + 12 * (int64_t)j + 2 * t);
        cp_commit();
        cp_wait_all();
        __syncwarp(mask);
        acc_store(ac, ap >= 0 ? sm.pa : nullptr, nullptr, sm.S, t);
        __syncwarp(mask);
        block_finish(v, bb, sm);
        flow_release(v.flag + v.n + bb, ep);
      }
    } else {  // backward substitution of node j: x_j = L_jj^-T (y_j - sum_i L_ij^T x_i)
      const int j = v.eord[m - 1 - (idx - nf)];
      const int c0 = v.col_ptr[j], U = v.col_ptr[j + 1] - c0;
      flow_wait(v, v.flag, j, -1, ep);  // y_j (and, factoring, L_jj)
      if (v.trace) t_rdy = gtimer();
      stage_block(sm.pl, v.L + 144 * (int64_t)j, t);
      if (t < 6) cp16(sm.pv + 2 * t, v.dinv + 12 * (int64_t)j + 2 * t);
      cp_commit();
      double acc = ldcg(x + 12 * (int64_t)j + tt);
      // the column in chunks of 2 NST blocks: blocks staged once final (factoring: long
      // before the ancestors' x), then the x_i polled together, summed in column order
      constexpr int BW = 2 * NST;
      for (int base = 0; base < U; base += BW) {
        const int cnt = min(BW, U - base);
        const bool mine = t < cnt;
        if (fac) flow_wait_lanes(v, v.flag, mine, v.n + c0 + base + (mine ? t : 0), ep);
        for (int l = 0; l < cnt; ++l) stage_block(sm.stage[l >> 1][l & 1], v.L + 144 * (int64_t)(v.n + c0 + base + l), t);
        cp_commit();
        const int i_l = mine ? v.blk_row[c0 + base + t] : 0;
        flow_wait_lanes(v, v.xflag, mine, i_l, ep);
        for (int e = t; e < 12 * cnt; e += 32) {
          const int l = e / 12, r = e - 12 * l;
          const int i = v.blk_row[c0 + base + l];
          sm.pa[e] = __ldcg(x + 12 * (int64_t)i + r);
        }
        cp_wait_all();
        __syncwarp(mask);
        for (int l = 0; l < cnt; ++l) {
          const double* Lb = sm.stage[l >> 1][l & 1] + tt;
          const double* xi = sm.pa + 12 * l;
          double s2 = 0.0;
#pragma unroll
          for (int r = 0; r < 12; ++r) s2 = fma(Lb[12 * r], xi[r], s2);
          acc -= s2;
        }
        __syncwarp(mask);
      }
      cp_wait_all();
      __syncwarp(mask);
      double lcol[12], rinv[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) {
        lcol[q] = sm.pl[12 * q + tt];
        rinv[q] = sm.pv[q];
      }
      const double xv = upper_solve12(mask, t, acc, lcol, rinv);
      __syncwarp(mask);
      if (t < 12) x[12 * (int64_t)j + t] = xv;
      flow_release(v.xflag + j, ep);
    }
  item_done:
    if (v.trace && t == 0) {
      const unsigned done = atomicAdd(v.ctr + 3, 1u);
      unsigned long long* o = v.trace + 4 * (int64_t)done;
      o[0] = (unsigned long long)(unsigned)idx;
      o[1] = t_start;
      o[2] = t_rdy ? t_rdy : t_start;
      o[3] = gtimer();
    }
  }
}

// nonzero flags of the upper off-diagonal pattern blocks
__global__ void k_block_nz(int64_t n_off, const int* __restrict__ upper_pos, const double* __restrict__ val,
                           int* flags) {
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= n_off) return;
  const double* B = val + 144 * (int64_t)upper_pos[w];
  bool nz = false;
  for (int e = lane; e < 144; e += 32) nz |= (B[e] != 0.0);
  unsigned any = __ballot_sync(0xffffffffu, nz);
  if (lane == 0) flags[w] = any ? 1 : 0;
}

// r = b - A x and the partial sums of r.r and b.b (fixed order)
__global__ void k_resid(int n, const int* __restrict__ row_ptr, const int* __restrict__ col,
                        const double* __restrict__ val, const double* __restrict__ x, const double* __restrict__ b,
                        double* r, double* part, unsigned long long* amax) {
  __shared__ double sr[RED_THREADS], sb[RED_THREADS];
  double ar = 0.0, ab = 0.0;
  if (amax) {
    // the Newton step's |x|_inf and b . x in the same launch (driver.cu reads them with the
    // residual: b = -g, so g . dx = -(b . x)); same grid-stride order as k_absmax_dot
    __shared__ double sd[RED_THREADS];
    const int64_t Nx = 12 * (int64_t)n;
    double m = 0.0, acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < Nx; i += (int64_t)gridDim.x * blockDim.x) {
      m = fmax(m, fabs(x[i]));
      acc += b[i] * x[i];
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(amax, (unsigned long long)__double_as_longlong(m));
    sd[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if (threadIdx.x < w) sd[threadIdx.x] += sd[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) part[2 * gridDim.x + blockIdx.x] = sd[0];
  }
  const int64_t N = 12 * (int64_t)n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    int br = (int)(t / 12), rr = (int)(t % 12);
    double acc = 0.0;
    for (int k = row_ptr[br]; k < row_ptr[br + 1]; ++k) {
      const double* blk = val + 144 * (int64_t)k + 12 * rr;
      const double* xv = x + 12 * (int64_t)col[k];
#pragma unroll
      for (int c = 0; c < 12; ++c) acc = fma(blk[c], xv[c], acc);
    }
    double ri = b[t] - acc;
    r[t] = ri;
    ar = fma(ri, ri, ar);
    ab = fma(b[t], b[t], ab);
  }
  sr[threadIdx.x] = ar;
  sb[threadIdx.x] = ab;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      sr[threadIdx.x] += sr[threadIdx.x + w];
      sb[threadIdx.x] += sb[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = sr[0];
    part[gridDim.x + blockIdx.x] = sb[0];
  }
}

__global__ void k_add_inplace(int64_t n, double* x, const double* d) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] += d[i];
}

// Sections of the packed plan buffer
enum { CH_LEAVES, CH_ISO, CH_PARENT, CH_NCHILD, CH_CHILDP, CH_CHILDI, CH_COLP, CH_BROW, CH_BCOL, CH_ROWP, CH_ROWB,
       CH_ROWC, CH_UPDP, CH_UPD, CH_PARTP, CH_PART, CH_DNP, CH_BPART, CH_BNP, CH_INIT, CH_FSEQ, CH_EORD, CH_NSEC };
// task splitting: a diagonal (row products) or block (update pairs) task with more
// than PART_MIN products is split into chunks of PART_CHUNK
constexpr int PART_MIN = 12, PART_CHUNK = 8;
// ABD_CHOL_FIFO: factor on the task-graph FIFO (k_chol_sched) instead of the dataflow
// schedule (k_chol_flow); only the FIFO needs the task-graph sections of the plan
static bool chol_fifo() {
  static const bool f = getenv("ABD_CHOL_FIFO") != nullptr;
  return f;
}

static CholView plan_view(Scene& s) {
  Scene::Work& w = s.w;
  const size_t* o = w.ch_cache.offs;
  const int* dp = w.ch_plan.p;
  const int n = s.H.n;
  const int m = (int)w.ch_cache.stats[1];
  const int nbo = (int)(w.ch_cache.stats[2] - n);
  const int n_part = (int)w.ch_cache.stats[8], n_init = (int)w.ch_cache.stats[9];
  CholView v{n,
             m,
             (int)w.ch_cache.stats[7],
             n - m,
             n_part + nbo + m,
             dp + o[CH_LEAVES],
             dp + o[CH_ISO],
             dp + o[CH_PARENT],
             dp + o[CH_NCHILD],
             dp + o[CH_CHILDP],
             dp + o[CH_CHILDI],
             dp + o[CH_COLP],
             dp + o[CH_BROW],
             dp + o[CH_BCOL],
             s.H.row_ptr.p,
             s.H.col.p,
             w.ch_apos.p,
             dp + o[CH_ROWP],
             dp + o[CH_ROWB],
             dp + o[CH_ROWC],
             dp + o[CH_UPDP],
             reinterpret_cast<const int2*>(dp + o[CH_UPD]),
             s.H.diag_pos.p,
             s.H.val.p,
             w.ch_L.p,
             w.ch_dinv.p,
             w.bad.p,
             w.ch_dep.p,
             w.ch_bleft.p,
             w.ch_queue.p,
             w.ch_ctr.p,
             nullptr};
  v.n_part = n_part;
  v.n_init = n_init;
  v.part_ptr = dp + o[CH_PARTP];
  v.part = reinterpret_cast<const int4*>(dp + o[CH_PART]);
  v.dnp = dp + o[CH_DNP];
  v.bpart = dp + o[CH_BPART];
  v.bnp = dp + o[CH_BNP];
  v.init = dp + o[CH_INIT];
  v.scratch = w.ch_scratch.p;
  v.dleft = w.ch_dleft.p;
  v.bgate = w.ch_bgate.p;
  v.fseq = dp + o[CH_FSEQ];
  v.eord = dp + o[CH_EORD];
  v.flag = w.ch_fl.p;
  v.xflag = w.ch_fl.p + n + nbo;
  v.sflag = w.ch_fl.p + 2 * n + nbo;
  v.sbuf = w.ch_sbuf.p;
  return v;
}

// ---------------------------------------------------------------------------
// host analysis
namespace {

struct Analysis {
  int n_cta = 0, n_coupled = 0;
  int64_t n_blk = 0, n_upd = 0, n_edges = 0;
  int max_level = 0, largest = 0;
  double ms_sync = 0, ms_order = 0, ms_plan = 0, ms_sub[6] = {};
  bool cached = false, order_reused = false;
  CholView view{};
};

// minimum-degree elimination on a (local) graph; colstruct[v] = neighbours
// still alive when v is eliminated (its L column structure), order = elimination order.
void min_degree_lists(int m, std::vector<std::vector<int>>& adj, std::vector<int>& order,
                      std::vector<std::vector<int>>& colstruct);

// Same elimination (repeatedly the live node of smallest (degree, id); its live
// neighbours become a clique) on adjacency bitsets: a neighbour update is W word
// ORs instead of a sorted-list merge.  Identical order and column structures to
// min_degree_lists; used while the core fits in a few hundred words per row.
void min_degree(int m, std::vector<std::vector<int>>& adj, std::vector<int>& order,
                std::vector<std::vector<int>>& colstruct) {
  const int W = (m + 63) / 64;
  if (m > 8192) {
    min_degree_lists(m, adj, order, colstruct);
    return;
  }
  order.clear();
  order.reserve(m);
  colstruct.assign(m, {});
  std::vector<uint64_t> bits((size_t)m * W, 0ull), nb(W);
  std::vector<int> deg(m);
  for (int v = 0; v < m; ++v) {
    uint64_t* r = bits.data() + (size_t)v * W;
    for (int a : adj[v]) r[a >> 6] |= 1ull << (a & 63);
    deg[v] = (int)adj[v].size();
  }
  std::vector<char> done(m, 0);
  typedef std::pair<int, int> DI;
  std::vector<DI> hv;
  hv.reserve(2 * m);
  for (int v = 0; v < m; ++v) hv.push_back({deg[v], v});
  std::priority_queue<DI, std::vector<DI>, std::greater<DI>> heap(std::greater<DI>(), std::move(hv));
  std::vector<int> list;
  while (!heap.empty()) {
    DI top = heap.top();
    heap.pop();
    const int v = top.second;
    if (done[v] || top.first != deg[v]) continue;
    done[v] = 1;
    order.push_back(v);
    const uint64_t* rv = bits.data() + (size_t)v * W;
    std::copy(rv, rv + W, nb.begin());
    list.clear();
    for (int w = 0; w < W; ++w)
      for (uint64_t x = nb[w]; x; x &= x - 1) list.push_back(64 * w + __builtin_ctzll(x));
    colstruct[v] = list;  // ascending ids, as the sorted lists
    for (int a : list) {
      uint64_t* ra = bits.data() + (size_t)a * W;
      int d = 0;
      for (int w = 0; w < W; ++w) {
        ra[w] |= nb[w];
        if (w == (a >> 6)) ra[w] &= ~(1ull << (a & 63));
        if (w == (v >> 6)) ra[w] &= ~(1ull << (v & 63));
        d += __builtin_popcountll(ra[w]);
      }
      deg[a] = d;
      heap.push({d, a});
    }
  }
}

void min_degree_lists(int m, std::vector<std::vector<int>>& adj, std::vector<int>& order,
                      std::vector<std::vector<int>>& colstruct) {
  order.clear();
  order.reserve(m);
  colstruct.assign(m, {});
  std::vector<char> done(m, 0);
  typedef std::pair<int, int> DI;
  std::vector<DI> hv;
  hv.reserve(2 * m);
  for (int v = 0; v < m; ++v) hv.push_back({(int)adj[v].size(), v});
  std::priority_queue<DI, std::vector<DI>, std::greater<DI>> heap(std::greater<DI>(), std::move(hv));
  std::vector<int> merged;
  while (!heap.empty()) {
    DI top = heap.top();
    heap.pop();
    int v = top.second;
    if (done[v] || top.first != (int)adj[v].size()) continue;
    done[v] = 1;
    order.push_back(v);
    std::vector<int>& nb = colstruct[v];
    nb.swap(adj[v]);
    for (int a : nb) {
      merged.clear();
      std::set_union(adj[a].begin(), adj[a].end(), nb.begin(), nb.end(), std::back_inserter(merged));
      std::vector<int>& out = adj[a];
      out.clear();
      for (int u : merged)
        if (u != a && u != v) out.push_back(u);
      heap.push({(int)out.size(), a});
    }
  }
}

constexpr double ORDER_REUSE_FILL = 1.05;  // factor blocks and update pairs, over the fresh order's

// Symbolic factorization of the local graph (adjacency adj_ptr / adj_idx, full
// degrees deg) under the cached global elimination order `gorder`, preceded by the
// nodes not in it (ascending local id).  Column structure of v = its later
// neighbours plus its elimination-tree children's structures minus v, sorted by
// position.  Fills order / pos / csp / csi as the fresh ordering does; false when the
// factor would exceed max_nnz off-diagonal blocks or max_upd update pairs.
bool symbolic_fixed_order(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj_idx,
                          const std::vector<int>& deg, const std::vector<int>& loc, const std::vector<int>& gorder,
                          int64_t max_nnz, int64_t max_upd, std::vector<int>* scratch, std::vector<int>& order,
                          std::vector<int>& pos, std::vector<int>& csp, std::vector<int>& csi) {
  int64_t upd = 0;
  std::vector<int>&seen = scratch[0], &mark = scratch[1], &head = scratch[2], &nxt = scratch[3], &st0 = scratch[4],
                  &len = scratch[5], &flat = scratch[6], &L = scratch[7];
  seen.assign(m, 0);
  order.clear();
  for (int g : gorder)
    if (loc[g] >= 0) seen[loc[g]] = 1;
  for (int v = 0; v < m; ++v)
    if (!seen[v]) order.push_back(v);
  for (int g : gorder)
    if (loc[g] >= 0) order.push_back(loc[g]);
  if ((int)order.size() != m) return false;
  pos.resize(m);
  for (int i = 0; i < m; ++i) pos[order[i]] = i;
  mark.assign(m, -1);
  head.assign(m, -1);
  nxt.assign(m, -1);
  st0.assign(m, 0);
  len.assign(m, 0);
  flat.clear();
  for (int i = 0; i < m; ++i) {
    const int v = order[i];
    L.clear();
    for (int e = adj_ptr[v]; e < adj_ptr[v] + deg[v]; ++e) {
      const int u = adj_idx[e];
      if (pos[u] > i && mark[u] != v) {
        mark[u] = v;
        L.push_back(u);
      }
    }
    for (int c = head[v]; c >= 0; c = nxt[c])
      for (int k = st0[c]; k < st0[c] + len[c]; ++k) {
        const int u = flat[k];
        if (u != v && mark[u] != v) {
          mark[u] = v;
          L.push_back(u);
        }
      }
    std::sort(L.begin(), L.end(), [&](int a, int b) { return pos[a] < pos[b]; });
    st0[v] = (int)flat.size();
    len[v] = (int)L.size();
    flat.insert(flat.end(), L.begin(), L.end());
    upd += (int64_t)L.size() * ((int64_t)L.size() - 1) / 2;  // update pairs of this column
    if ((int64_t)flat.size() > max_nnz || upd > max_upd) return false;
    if (!L.empty()) {
      nxt[v] = head[L[0]];
      head[L[0]] = v;
    }
  }
  csp.assign(m + 1, 0);
  for (int v = 0; v < m; ++v) csp[v + 1] = csp[v] + len[v];
  csi.resize(csp[m]);
  for (int v = 0; v < m; ++v) std::copy(flat.begin() + st0[v], flat.begin() + st0[v] + len[v], csi.begin() + csp[v]);
  return true;
}

double ms_since(std::chrono::steady_clock::time_point t) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
}

}  // namespace

static Analysis chol_analyze(Scene& s) {
  using clk = std::chrono::steady_clock;
  Bsr& H = s.H;
  Scene::Work& w = s.w;
  cudaStream_t st = s.main_stream;  // s.stream may be swapped to a side stream by the main thread
  const int n = H.n;
  const int64_t n_off = H.n_off;
  Analysis an;
  auto t0 = clk::now();
  // flags | keys (2 ints) per pattern block, one pinned staging buffer
  int* hm = w.h_meta.reserve(3 * (size_t)std::max<int64_t>(n_off, 1));
  int *flags = hm, *keys = hm + n_off;
  if (w.ch_pre) {
    // structure from the active pairs, already on its way to the host (assemble)
    w.ch_pre = false;
    HMARK();
    CK(cudaEventSynchronize(w.ch_pre_ev));
    HMARK();
  } else if (n_off) {
    w.ch_flags.resize(n_off);
    k_block_nz<<<grid_for(n_off * 32, 256), 256, 0, st>>>(n_off, H.upper_pos.p, H.val.p, w.ch_flags.p);
    note_launch("k_block_nz");
    CK(cudaMemcpyAsync(flags, w.ch_flags.p, n_off * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(keys, H.upper_keys.p, n_off * sizeof(int2), cudaMemcpyDeviceToHost, st));
    SSYNC(st);
  }
  an.ms_sync = ms_since(t0);
  t0 = clk::now();
  Scene::Work::CholCache& cc = w.ch_cache;
  // nonzero couplings (keys are sorted (i < j)); the cached plan is reused when
  // they are a subset of the cached graph (extra blocks then hold exact zeros)
  std::vector<uint64_t>& cur = w.ch_edges_cur;
  cur.clear();
  for (int64_t k = 0; k < n_off; ++k)
    if (flags[k]) cur.push_back(((uint64_t)(uint32_t)keys[2 * k] << 32) | (uint32_t)keys[2 * k + 1]);
  HMARK();
  if (cc.valid && cc.n == n && std::includes(cc.edges.begin(), cc.edges.end(), cur.begin(), cur.end())) {
    an.n_cta = (int)cc.stats[0];
    an.n_coupled = (int)cc.stats[1];
    an.n_blk = cc.stats[2];
    an.n_upd = cc.stats[3];
    an.n_edges = cc.stats[4];
    an.max_level = (int)cc.stats[5];
    an.largest = (int)cc.stats[6];
    an.view = plan_view(s);
    an.cached = true;
    ++cc.hits;
    return an;
  }
  ++cc.misses;
  // Build the plan for the union with the previously analysed graph of this step
  // (contacts come and go across Newton iterations; the union keeps later
  // iterations on the resident plan).  ch_cache.valid is reset per time step.
  static const bool no_union = getenv("ABD_CHOL_NO_UNION") != nullptr;
  if (cc.valid && cc.n == n && !no_union) {
    std::vector<uint64_t> un;
    un.reserve(cur.size() + cc.edges.size());
    std::set_union(cur.begin(), cur.end(), cc.edges.begin(), cc.edges.end(), std::back_inserter(un));
    cur.swap(un);
  }

  static const char* dump_graph = getenv("ABD_CHOL_DUMP_GRAPH");  // tools: coupling graph of the last analysis
  if (dump_graph) {
    if (FILE* f = fopen(dump_graph, "wb")) {
      const int64_t ne = (int64_t)cur.size();
      fwrite(&n, sizeof(int), 1, f);
      fwrite(&ne, sizeof(int64_t), 1, f);
      fwrite(cur.data(), sizeof(uint64_t), cur.size(), f);
      fclose(f);
    }
  }
  // coupled nodes (>= 1 nonzero coupling) get local ids in ascending node order;
  // host scratch persists across analyses (no allocations in the steady state)
  std::vector<int>&loc = w.hs_i[0], &glob = w.hs_i[1], &adj_ptr = w.hs_i[2], &adj_idx = w.hs_i[3],
                  &deg = w.hs_i[4], &live = w.hs_i[5], &live2 = w.hs_i[6], &sel = w.hs_i[7], &cs0 = w.hs_i[8],
                  &cs1 = w.hs_i[9], &order = w.hs_i[10], &pos = w.hs_i[11], &csp = w.hs_i[12], &csi = w.hs_i[13];
  std::vector<char>&gone = w.hs_c[0], &blocked = w.hs_c[1];
  const double ms_cur = ms_since(t0);
  loc.assign(n, -1);
  glob.clear();
  for (uint64_t e : cur) {
    loc[(int)(e >> 32)] = 0;
    loc[(int)(e & 0xffffffffu)] = 0;
    ++an.n_edges;
  }
  for (int v = 0; v < n; ++v)
    if (loc[v] == 0) {
      loc[v] = (int)glob.size();
      glob.push_back(v);
    }
  const int m = (int)glob.size();
  an.n_coupled = m;
  adj_ptr.assign(m + 1, 0);
  adj_idx.resize(2 * an.n_edges);
  for (uint64_t e : cur) {
    adj_ptr[loc[(int)(e >> 32)] + 1]++;
    adj_ptr[loc[(int)(e & 0xffffffffu)] + 1]++;
  }
  for (int v = 0; v < m; ++v) adj_ptr[v + 1] += adj_ptr[v];
  deg.assign(m, 0);
  for (uint64_t e : cur) {
    const int a2 = loc[(int)(e >> 32)], b2 = loc[(int)(e & 0xffffffffu)];
    adj_idx[adj_ptr[a2] + deg[a2]++] = b2;
    adj_idx[adj_ptr[b2] + deg[b2]++] = a2;
  }
  const double ms_adj = ms_since(t0);
  // Order reuse: a miss inside a step (the union graph grew by a few contacts)
  // keeps the step's fresh elimination order -- nodes new to the graph first -- and
  // redoes only the symbolic factorization, unless the fill grows by more than
  // ORDER_REUSE_FILL over the fresh order's, in factor blocks or update pairs (then
  // the graph is ordered afresh).
  static const bool no_reuse = getenv("ABD_CHOL_NO_ORDER_REUSE") != nullptr;
  int n_core = 0;
  bool reused = false;
  if (!no_reuse && cc.valid && cc.n == n && !cc.gorder.empty())
    reused = symbolic_fixed_order(m, adj_ptr, adj_idx, deg, loc, cc.gorder, (int64_t)(ORDER_REUSE_FILL * cc.fresh_nnz),
                                  (int64_t)(ORDER_REUSE_FILL * cc.fresh_upd), w.hs_i + 31, order, pos, csp, csi);
  if (!reused) {
    // Elimination order by tree contraction (contact graphs of piles are forests of
    // stacked chains): rounds of rake (every node of degree <= 1 at the start of the
    // round; no fill) and compress (an independent set of degree-2 nodes; the fill
    // edge joins the two neighbours), so a chain of L bodies is eliminated in
    // O(log L) elimination-tree levels instead of L / 2.  What remains (degree >= 3
    // everywhere) is ordered by minimum degree.  cs0/cs1 = the live neighbours of a
    // raked / compressed node when it is eliminated (its L column structure).
    // The live neighbour list of v is adj_idx[adj_ptr[v], adj_ptr[v] + deg[v]),
    // edited in place: rake and compress never raise a degree.
    order.clear();
    cs0.assign(m, -1);
    cs1.assign(m, -1);
    gone.assign(m, 0);
    blocked.assign(m, 0);
    live.resize(m);
    std::iota(live.begin(), live.end(), 0);
    static const bool no_compress = getenv("ABD_CHOL_NO_COMPRESS") != nullptr;
    auto drop = [&](int u, int x) {
      int* l = adj_idx.data() + adj_ptr[u];
      const int d = deg[u];
      for (int i = 0; i < d; ++i)
        if (l[i] == x) {
          l[i] = l[d - 1];
          deg[u] = d - 1;
          return;
        }
    };
    auto relink = [&](int u, int x, int y) {  // in u's list: x -> y, or drop x when y is already there
      int* l = adj_idx.data() + adj_ptr[u];
      const int d = deg[u];
      int ix = -1;
      bool has_y = false;
      for (int i = 0; i < d; ++i) {
        if (l[i] == x) ix = i;
        if (l[i] == y) has_y = true;
      }
      if (has_y) {
        l[ix] = l[d - 1];
        deg[u] = d - 1;
      } else {
        l[ix] = y;
      }
    };
    for (;;) {
      bool progress = false;
      sel.clear();
      for (int v : live)
        if (deg[v] <= 1) sel.push_back(v);
      for (int v : sel) {  // rake (a lone pair: the second end follows with no neighbour)
        if (gone[v]) continue;
        if (deg[v] == 1) {
          const int u = adj_idx[adj_ptr[v]];
          cs0[v] = u;
          drop(u, v);
        }
        deg[v] = 0;
        gone[v] = 1;
        order.push_back(v);
        progress = true;
      }
      if (!no_compress) {
        sel.clear();
        for (int v : live) blocked[v] = 0;
        for (int v : live)
          if (!gone[v] && !blocked[v] && deg[v] == 2) {
            const int* l = adj_idx.data() + adj_ptr[v];
            sel.push_back(v);
            blocked[v] = 1;
            blocked[l[0]] = 1;
            blocked[l[1]] = 1;
          }
        for (int v : sel) {  // compress: v's neighbours a, b become adjacent (fill)
          const int* l = adj_idx.data() + adj_ptr[v];
          const int a2 = l[0], b2 = l[1];
          cs0[v] = a2;
          cs1[v] = b2;
          relink(a2, v, b2);
          relink(b2, v, a2);
          deg[v] = 0;
          gone[v] = 1;
          order.push_back(v);
          progress = true;
        }
      }
      live2.clear();
      for (int v : live)
        if (!gone[v]) live2.push_back(v);
      live.swap(live2);
      if (!progress || live.empty()) break;
    }
    const double ms_contract = ms_since(t0);
    n_core = m - (int)order.size();
    std::vector<std::vector<int>> core_cs;
    std::vector<int> core_glob;
    if ((int)order.size() < m) {
      std::vector<int> core_id(m, -1);
      core_glob = live;
      const int mc = (int)core_glob.size();
      for (int c = 0; c < mc; ++c) core_id[core_glob[c]] = c;
      std::vector<std::vector<int>> cadj(mc);
      for (int c = 0; c < mc; ++c) {
        const int v = core_glob[c];
        for (int i = 0; i < deg[v]; ++i) cadj[c].push_back(core_id[adj_idx[adj_ptr[v] + i]]);
        std::sort(cadj[c].begin(), cadj[c].end());
      }
      std::vector<int> corder;
      min_degree(mc, cadj, corder, core_cs);
      for (int c : corder) order.push_back(core_glob[c]);
      for (auto& l : core_cs)
        for (int& x : l) x = core_glob[x];
    }
    const double ms_core = ms_since(t0);
    static const bool trace_ord = getenv("ABD_TRACE_CHOL") != nullptr;
    if (trace_ord)
      fprintf(stderr, "[abd chol order] m=%d core=%d cur_ms=%.3f adj_ms=%.3f contract_ms=%.3f core_ms=%.3f\n", m, n_core,
              ms_cur, ms_adj, ms_contract, ms_core);
    pos.resize(m);
    for (int i = 0; i < m; ++i) pos[order[i]] = i;
    csp.assign(m + 1, 0);
    for (int v = 0; v < m; ++v) csp[v + 1] = csp[v] + (cs0[v] >= 0) + (cs1[v] >= 0);
    for (size_t c = 0; c < core_glob.size(); ++c) csp[core_glob[c] + 1] = (int)core_cs[c].size();
    if (!core_glob.empty()) {  // recount: core nodes carry their min-degree column structures
      std::vector<int> cnt(m, 0);
      for (int v = 0; v < m; ++v) cnt[v] = (cs0[v] >= 0) + (cs1[v] >= 0);
      for (size_t c = 0; c < core_glob.size(); ++c) cnt[core_glob[c]] = (int)core_cs[c].size();
      csp[0] = 0;
      for (int v = 0; v < m; ++v) csp[v + 1] = csp[v] + cnt[v];
    }
    csi.resize(csp[m]);
    for (int v = 0; v < m; ++v) {
      int* o = csi.data() + csp[v];
      const int k = csp[v + 1] - csp[v];
      if (k == 1) {
        o[0] = cs0[v];
      } else if (k == 2 && cs1[v] >= 0) {
        const bool sw = pos[cs1[v]] < pos[cs0[v]];
        o[0] = sw ? cs1[v] : cs0[v];
        o[1] = sw ? cs0[v] : cs1[v];
      }
    }
    for (size_t c = 0; c < core_glob.size(); ++c) {
      std::vector<int>& l = core_cs[c];
      std::sort(l.begin(), l.end(), [&](int a2, int b2) { return pos[a2] < pos[b2]; });
      std::copy(l.begin(), l.end(), csi.begin() + csp[core_glob[c]]);
    }
    cc.gorder.resize(m);
    for (int i = 0; i < m; ++i) cc.gorder[i] = glob[order[i]];
    cc.fresh_nnz = csp[m];
    cc.fresh_upd = 0;
    for (int v = 0; v < m; ++v) {
      const int64_t k = csp[v + 1] - csp[v];
      cc.fresh_upd += k * (k - 1) / 2;
    }
  }
  an.order_reused = reused;
  an.ms_order = ms_since(t0);
  t0 = clk::now();

  // off-diagonal L blocks: column (local) v owns [col_off[v], col_off[v+1])
  const std::vector<int>& col_off = csp;
  const int nbo = csp[m];
  an.n_blk = n + (int64_t)nbo;
  an.ms_sub[0] = ms_since(t0);
  // row lists (local i): (k, off block) for k eliminated before i, in elimination order of k
  std::vector<int>&rcnt = w.hs_i[14], &rfill = w.hs_i[15], &r_k = w.hs_i[16], &r_b = w.hs_i[17],
                   &upd_ptr = w.hs_i[18], &upd = w.hs_i[19], &level = w.hs_i[20], &root = w.hs_i[21],
                   &csize = w.hs_i[22], &cdepth = w.hs_i[23], &comps = w.hs_i[24];
  rcnt.assign(m + 1, 0);
  for (int e = 0; e < nbo; ++e) rcnt[csi[e] + 1]++;
  for (int v = 0; v < m; ++v) rcnt[v + 1] += rcnt[v];
  rfill.assign(rcnt.begin(), rcnt.end() - 1);
  r_k.resize(nbo);
  r_b.resize(nbo);
  for (int k : order)
    for (int e = csp[k]; e < csp[k + 1]; ++e) {
      int i = csi[e];
      r_k[rfill[i]] = k;
      r_b[rfill[i]] = e;
      rfill[i]++;
    }
  an.ms_sub[1] = ms_since(t0);
  // update pairs for off block (i, j): k in rows(j) with i in cs[k], in elimination
  // order of k.  Every pair (j, i) of cs[k] (j before i) is one such update, so the
  // lists are built by walking each column's pairs once: O(#updates + sum |cs[j]|).
  upd_ptr.assign(nbo + 1, 0);
  std::vector<int>& ub = w.hs_i[29];
  ub.clear();
  // the later entries of cs[k] after j = csi[a2] are a subset of cs[j], both sorted by
  // elimination position: one merge walk finds their blocks in column j
  ub.reserve(4096);
  for (int k : order)
    for (int a2 = csp[k]; a2 < csp[k + 1]; ++a2) {
      const int j = csi[a2];
      int f = csp[j];
      for (int b2 = a2 + 1; b2 < csp[k + 1]; ++b2) {
        const int i = csi[b2];
        while (csi[f] != i) ++f;  // present by the fill property (f < csp[j + 1])
        ub.push_back(f);
        upd_ptr[f + 1]++;
      }
    }
  for (int b = 0; b < nbo; ++b) upd_ptr[b + 1] += upd_ptr[b];
  upd.resize(2 * (size_t)upd_ptr[nbo]);
  {
    std::vector<int>& fill = w.hs_i[30];
    fill.assign(upd_ptr.begin(), upd_ptr.end() - 1);
    size_t q = 0;
    for (int k : order)
      for (int a2 = csp[k]; a2 < csp[k + 1]; ++a2)
        for (int b2 = a2 + 1; b2 < csp[k + 1]; ++b2) {
          const int at = fill[ub[q++]]++;
          upd[2 * (size_t)at] = n + b2;      // L_ik
          upd[2 * (size_t)at + 1] = n + a2;  // L_jk
        }
  }
  an.n_upd = (int64_t)upd.size() / 2;
  an.ms_sub[2] = ms_since(t0);
  // elimination-tree levels and component roots (local)
  level.assign(m, 0);
  root.resize(m);
  for (int v : order)
    if (csp[v + 1] > csp[v]) level[csi[csp[v]]] = std::max(level[csi[csp[v]]], level[v] + 1);
  for (int q = m - 1; q >= 0; --q) {
    int v = order[q];
    root[v] = csp[v + 1] == csp[v] ? v : root[csi[csp[v]]];
  }
  csize.assign(m, 0);
  cdepth.assign(m, 0);
  comps.clear();
  for (int v = 0; v < m; ++v) {
    csize[root[v]]++;
    cdepth[root[v]] = std::max(cdepth[root[v]], level[v] + 1);
    an.max_level = std::max(an.max_level, level[v] + 1);
  }
  for (int v = 0; v < m; ++v)
    if (root[v] == v) comps.push_back(v);
  std::sort(comps.begin(), comps.end(),
            [&](int a, int b) { return csize[a] != csize[b] ? csize[a] > csize[b] : a < b; });
  an.largest = comps.empty() ? 0 : csize[comps[0]];
  static const bool trace_lv = getenv("ABD_TRACE_CHOL") != nullptr;
  if (trace_lv && !comps.empty()) {
    std::vector<int> h(cdepth[comps[0]], 0);
    for (int v = 0; v < m; ++v)
      if (root[v] == comps[0]) h[level[v]]++;
    fprintf(stderr, "[abd chol] largest component levels:");
    for (int x : h) fprintf(stderr, " %d", x);
    fprintf(stderr, "\n");
  }
  an.ms_sub[3] = ms_since(t0);
  an.ms_sub[4] = ms_since(t0);
  // task graph: elimination-tree parents, child lists, leaves (deepest first), isolated nodes
  std::vector<int>&par = w.hs_i[26], &dep = w.hs_i[27], &leaves = w.hs_i[28];
  const bool fifo = chol_fifo();
  static const bool trace_cp = getenv("ABD_TRACE_CHOL") != nullptr;
  leaves.clear();
  if (fifo || trace_cp) {
  par.assign(m, -1);
  for (int v = 0; v < m; ++v)
    if (csp[v + 1] > csp[v]) par[v] = csi[csp[v]];
  dep.assign(m, 0);
  for (int q = m - 1; q >= 0; --q) {
    const int v = order[q];
    dep[v] = par[v] < 0 ? 0 : dep[par[v]] + 1;
  }
  }
  std::vector<int>& nch = w.hs_i[25];
  if (fifo) {
    nch.assign(m, 0);
    for (int v = 0; v < m; ++v)
      if (par[v] >= 0) nch[par[v]]++;
    for (int v = 0; v < m; ++v)
      if (nch[v] == 0) leaves.push_back(v);
    std::sort(leaves.begin(), leaves.end(),
              [&](int a2, int b2) { return dep[a2] != dep[b2] ? dep[a2] > dep[b2] : glob[a2] < glob[b2]; });
  }
  const int n_leaves = (int)leaves.size();
  const int n_iso = n - m;
  an.n_cta = 0;  // set at launch
  if (trace_cp) {  // task costs in 12x12 block products: rows + sum over column blocks (1 + updates)
    std::vector<int64_t> cost(m, 0), cp(m, 0);
    int64_t tot = 0, maxc = 0, maxcp = 0;
    int maxcol = 0, maxrow = 0;
    for (int v : order) {
      int64_t c = rcnt[v + 1] - rcnt[v];
      for (int b2 = csp[v]; b2 < csp[v + 1]; ++b2) c += 1 + (upd_ptr[b2 + 1] - upd_ptr[b2]);
      cost[v] = c;
      cp[v] += c;
      if (par[v] >= 0) cp[par[v]] = std::max(cp[par[v]], cp[v]);
      tot += c;
      maxc = std::max(maxc, c);
      maxcp = std::max(maxcp, cp[v]);
      maxcol = std::max(maxcol, csp[v + 1] - csp[v]);
      maxrow = std::max(maxrow, rcnt[v + 1] - rcnt[v]);
    }
    fprintf(stderr, "[abd chol cp] m=%d core=%d leaves=%d total=%lld maxcost=%lld critpath=%lld maxcol=%d maxrow=%d\n",
            m, n_core, n_leaves, (long long)tot, (long long)maxc, (long long)maxcp, maxcol, maxrow);
  }
  // split factor tasks: a diagonal with R row products / a block with U update pairs
  // above PART_MIN becomes ceil(. / PART_CHUNK) partial tasks released with the node
  // (ABD_CHOL_NO_SPLIT: none).  An unsplit diagonal is one whole task; an unsplit
  // block (bnp = 0) runs whole after its diagonal, as without splitting.
  static const bool no_split = getenv("ABD_CHOL_NO_SPLIT") != nullptr;
  auto nparts = [&](int k) { return (!no_split && k > PART_MIN) ? (k + PART_CHUNK - 1) / PART_CHUNK : 1; };
  auto bparts = [&](int k) { const int q = nparts(k); return q > 1 ? q : 0; };
  int64_t n_part = 0, n_init = 0;
  if (fifo) {
    std::vector<int> per(m, 0);
    for (int v = 0; v < m; ++v) {
      per[v] = nparts(rcnt[v + 1] - rcnt[v]);
      for (int b2 = csp[v]; b2 < csp[v + 1]; ++b2) per[v] += bparts(upd_ptr[b2 + 1] - upd_ptr[b2]);
      n_part += per[v];
    }
    for (int v : leaves) n_init += per[v];
  }
  // packed plan: leaves | iso | parent | nchild | child_ptr | child_idx | col_ptr | blk_row |
  //              row_ptr | row_blk | row_col | upd_ptr | (pad) | upd pairs | part_ptr | (pad) |
  //              part (int4) | dnp | bpart | bnp | init
  size_t o[CH_NSEC + 1];
  o[0] = 0;
  const size_t nf = fifo ? (size_t)n : 0, mf = fifo ? (size_t)m : 0, bf = fifo ? (size_t)nbo : 0;
  const size_t len[CH_NSEC] = {(size_t)n_leaves, (size_t)n_iso, nf, nf, fifo ? nf + 1 : 0, mf,
                               (size_t)n + 1, (size_t)nbo, (size_t)nbo, (size_t)n + 1, (size_t)nbo, (size_t)nbo,
                               (size_t)nbo + 1, upd.size(), fifo ? nf + 1 : 0, 4 * (size_t)n_part, nf,
                               bf, bf, (size_t)n_init, (size_t)m + nbo, (size_t)m};
  for (int k = 0; k < CH_NSEC; ++k) {
    o[k + 1] = o[k] + len[k];
    if (k + 1 == CH_UPD) o[k + 1] += o[k + 1] & 1;          // int2 alignment of the update pairs
    if (k + 1 == CH_PART) o[k + 1] = (o[k + 1] + 3) & ~(size_t)3;  // int4 alignment of the partials
  }
  const size_t total = o[CH_NSEC] + 2;
  int* hp = w.h_plan.reserve(total);
  for (int i = 0; i < n_leaves; ++i) hp[o[CH_LEAVES] + i] = glob[leaves[i]];
  {
    int q = 0;
    for (int v = 0; v < n; ++v)
      if (loc[v] < 0) hp[o[CH_ISO] + q++] = v;
  }
  int* parent = hp + o[CH_PARENT];
  int* nchild = hp + o[CH_NCHILD];
  int* child_ptr = hp + o[CH_CHILDP];
  int* child_idx = hp + o[CH_CHILDI];
  if (fifo) {
    for (int v = 0; v < n; ++v) {
      const int l = loc[v];
      parent[v] = (l >= 0 && par[l] >= 0) ? glob[par[l]] : -1;
      nchild[v] = l >= 0 ? nch[l] : 0;
    }
    child_ptr[0] = 0;
    for (int v = 0; v < n; ++v) child_ptr[v + 1] = child_ptr[v] + nchild[v];
    std::vector<int> fill(child_ptr, child_ptr + n);
    for (int v = 0; v < n; ++v)  // children in ascending node order (deterministic)
      if (parent[v] >= 0) child_idx[fill[parent[v]]++] = v;
  }
  int* col_ptr = hp + o[CH_COLP];
  int* row_ptr = hp + o[CH_ROWP];
  {
    // per global node column/row ranges (empty for isolated nodes)
    int c = 0, r = 0;
    for (int v = 0; v < n; ++v) {
      col_ptr[v] = c;
      row_ptr[v] = r;
      int l = loc[v];
      if (l >= 0) {
        for (int b = csp[l]; b < csp[l + 1]; ++b) {  // b == c + q: locals follow global order
          hp[o[CH_BROW] + b] = glob[csi[b]];
          hp[o[CH_BCOL] + b] = v;
        }
        c += csp[l + 1] - csp[l];
        for (int e2 = rcnt[l]; e2 < rcnt[l + 1]; ++e2) {
          hp[o[CH_ROWB] + r] = r_b[e2] + n;
          hp[o[CH_ROWC] + r] = glob[r_k[e2]];
          ++r;
        }
      }
    }
    col_ptr[n] = c;
    row_ptr[n] = r;
  }
  if (fifo) {
    // partial tasks per global node: its diagonal's chunks of the row list, then each
    // column block's chunks of its update pairs (equal splits)
    int* partp = hp + o[CH_PARTP];
    int* part = hp + o[CH_PART];
    int* dnp = hp + o[CH_DNP];
    int* bpart = hp + o[CH_BPART];
    int* bnp = hp + o[CH_BNP];
    int pc = 0;
    for (int v = 0; v < n; ++v) {
      partp[v] = pc;
      dnp[v] = 0;
      if (loc[v] < 0) continue;
      const int r0 = row_ptr[v], R = row_ptr[v + 1] - r0;
      const int d = nparts(R);
      dnp[v] = d;
      for (int q = 0; q < d; ++q, ++pc) {
        part[4 * pc] = 0;
        part[4 * pc + 1] = v;
        part[4 * pc + 2] = r0 + (int)((int64_t)R * q / d);
        part[4 * pc + 3] = r0 + (int)((int64_t)R * (q + 1) / d);
      }
      for (int b = col_ptr[v]; b < col_ptr[v + 1]; ++b) {
        const int u0 = upd_ptr[b], U = upd_ptr[b + 1] - u0;
        const int nb = bparts(U);
        bpart[b] = pc;
        bnp[b] = nb;
        for (int q = 0; q < nb; ++q, ++pc) {
          part[4 * pc] = 1;
          part[4 * pc + 1] = b;
          part[4 * pc + 2] = u0 + (int)((int64_t)U * q / nb);
          part[4 * pc + 3] = u0 + (int)((int64_t)U * (q + 1) / nb);
        }
      }
    }
    partp[n] = pc;
    int* init = hp + o[CH_INIT];
    int k = 0;
    for (int i = 0; i < n_leaves; ++i) {
      const int g = glob[leaves[i]];
      for (int p2 = partp[g]; p2 < partp[g + 1]; ++p2) init[k++] = p2;
    }
  }
  {
    // dataflow order: per node in elimination order its diagonal, then its column blocks
    int* fseq = hp + o[CH_FSEQ];
    int* eord = hp + o[CH_EORD];
    int q = 0;
    for (int i = 0; i < m; ++i) {
      const int g = glob[order[i]];
      eord[i] = g;
      fseq[q++] = g;
      for (int b = col_ptr[g]; b < col_ptr[g + 1]; ++b) fseq[q++] = n + b;
    }
  }
  an.ms_sub[5] = ms_since(t0);
  std::copy(upd_ptr.begin(), upd_ptr.end(), hp + o[CH_UPDP]);
  std::copy(upd.begin(), upd.end(), hp + o[CH_UPD]);
  w.ch_plan.resize(total);
  // the plan goes up on the copy stream: every earlier use of the plan buffers has completed
  // (the analysis starts from structure flags this thread has host-synchronised on, which
  // the main stream produced after its last factorization), and the next factorization
  // waits on plan_ev (plan_wait)
  CK(cudaMemcpyAsync(w.ch_plan.p, hp, total * sizeof(int), cudaMemcpyHostToDevice, s.copy_stream));
  CK(cudaEventRecord(s.plan_ev, s.copy_stream));
  s.plan_pending = true;
  w.ch_L.resize(144 * std::max<int64_t>(an.n_blk, 1));
  w.ch_dinv.resize(12 * std::max<int64_t>(n, 1));
  w.ch_apos.resize(std::max<int64_t>(an.n_blk - n, 1));
  w.ch_dep.resize(std::max(n, 1));
  w.ch_bleft.resize(std::max(n, 1));
  w.ch_queue.resize(std::max<int64_t>(std::max<int64_t>(2 * m, n_part + nbo + m), 1));
  w.ch_ctr.resize(4);
  w.ch_dleft.resize(std::max(n, 1));
  w.ch_bgate.resize(std::max(nbo, 1));
  w.ch_scratch.resize(std::max<int64_t>(n_part, 1) * PART_STRIDE);
  {
    // epoch flags of k_chol_flow: zeroed when (re)allocated, never reset otherwise
    const size_t cap0 = w.ch_fl.cap;
    w.ch_fl.resize(3 * (size_t)n + nbo + 1);
    w.ch_sbuf.resize(144 * (size_t)std::max(n, 1));
    if (w.ch_fl.cap != cap0) CK(cudaMemsetAsync(w.ch_fl.p, 0, w.ch_fl.cap * sizeof(int), st));
  }
  cc.valid = true;
  cc.n = n;
  cc.n_off = n_off;
  cc.edges.swap(cur);
  const int64_t st10[10] = {an.n_cta, an.n_coupled, an.n_blk, an.n_upd, an.n_edges, an.max_level, an.largest,
                            n_leaves, n_part, n_init};
  std::copy(st10, st10 + 10, cc.stats);
  std::copy(o, o + CH_NSEC + 1, cc.offs);
  an.view = plan_view(s);
  an.ms_plan = ms_since(t0);
  static const bool trace_sub = getenv("ABD_TRACE_CHOL") != nullptr;
  if (trace_sub)
    fprintf(stderr, "[abd chol plan] cum ms: %.3f %.3f %.3f %.3f %.3f %.3f end %.3f (m=%d nbo=%d total=%zu)\n",
            an.ms_sub[0], an.ms_sub[1], an.ms_sub[2], an.ms_sub[3], an.ms_sub[4], an.ms_sub[5], an.ms_plan, m, nbo,
            total);
  return an;
}

// Direct solve of the resident system H x = rhs with refinement (sparse.py:149-161),
// split so the driver can fold the residual check into its own host sync:
//   chol_begin  : analysis + factor/solve + residual + async copies (no sync)
//   chol_finish : after a stream sync, pivot check, residual test, corrections
// one factor (+ both substitutions) or one pair of substitutions over the task FIFO;
// returns the grid size
// the stream that is about to use the plan waits for its upload
static void plan_wait(Scene& s, cudaStream_t st) {
  if (!s.plan_pending) return;
  CK(cudaStreamWaitEvent(st, s.plan_ev, 0));
  s.plan_pending = false;
}

static int launch_sched(Scene& s, const CholView& v, const double* b, double* x, bool factor) {
  cudaStream_t st = s.stream;
  static int bps = 0;
  const size_t smem = CH_HW * sizeof(WarpSmem);
  if (!bps) {
    CK(cudaFuncSetAttribute(k_chol_sched, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_chol_sched, CH_THREADS, smem));
    bps = std::max(bps, 1);
  }
  // dataflow schedule (k_chol_flow) by default; ABD_CHOL_FIFO: the task-graph FIFO
  const bool fifo = chol_fifo();
  static int bpf = 0;
  if (!fifo && !bpf) {
    CK(cudaFuncSetAttribute(k_chol_flow, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpf, k_chol_flow, CH_THREADS, smem));
    bpf = std::max(bpf, 1);
  }
  if (!fifo) CK(cudaMemsetAsync(v.ctr, 0, 4 * sizeof(unsigned), st));
  else {
    const int init_n = std::max(std::max(v.n, v.n_tasks), std::max(2 * v.n_coupled, v.n_tasks - v.n_part));
    k_chol_sched_init<<<grid_for(std::max(init_n, 4), 256), 256, 0, st>>>(v, factor ? 1 : 0);
    note_launch("k_chol_sched_init");
  }
  // isolated nodes on a side stream beside the task graph (joined before returning)
  if (v.n_iso > 0) {
    CK(cudaEventRecord(s.ch_fork_ev, st));
    CK(cudaStreamWaitEvent(s.side4, s.ch_fork_ev, 0));
    const int ig = (int)std::min<int64_t>((int64_t)s.num_sms * 4, (v.n_iso + CH_HW - 1) / CH_HW);
    k_chol_iso<<<ig, CH_THREADS, 0, s.side4>>>(v, b, x, factor ? 1 : 0);
    note_launch("k_chol_iso");
    CK(cudaEventRecord(s.ch_join_ev, s.side4));
  }
  // coupled task graph: about one warp per leaf (the widest front), at most what fits
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(std::min<int64_t>((int64_t)s.num_sms * bps, CH_MAX_GRID),
                           ((int64_t)std::max(v.n_leaves, 1) + CH_HW - 1) / CH_HW));
  static const char* trace_path = getenv("ABD_CHOL_TRACE_TASKS");  // tools: per-task timeline of factorizations
  static DVec<unsigned long long> tbuf;
  CholView vv = v;
  // trace slots: the FIFO's tasks, or the flow's items (diagonals, blocks, backward)
  const int n_trace = fifo ? v.n_tasks : v.n_tasks + v.n_coupled;
  if (trace_path && factor) {
    tbuf.resize(4 * (int64_t)std::max(n_trace, 1));
    tbuf.zero(st);
    vv.trace = tbuf.p;
  }
  if (v.n_coupled > 0 && !fifo) {
    // one warp per item up to what is resident (waiting warps hold their slots)
    const int nbo = v.n_tasks - v.n_part - v.n_coupled;
    const int64_t items = (factor ? (int64_t)nbo : 0) + 2 * (int64_t)v.n_coupled;
    const int fgrid = (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)s.num_sms * bpf, (items + CH_HW - 1) / CH_HW));
    Scene::Work& w = s.w;
    if (++w.ch_epoch <= 0) {  // wrapped: forget every flag
      CK(cudaMemsetAsync(w.ch_fl.p, 0, w.ch_fl.cap * sizeof(int), st));
      w.ch_epoch = 1;
    }
    k_chol_flow<<<fgrid, CH_THREADS, smem, st>>>(vv, b, x, factor ? 1 : 0, w.ch_epoch);
    note_launch(factor ? "k_chol_flow(factor)" : "k_chol_flow(solve)");
  } else if (v.n_coupled > 0) {
    k_chol_sched<<<grid, CH_THREADS, smem, st>>>(vv, b, x, factor ? 1 : 0);
    note_launch(factor ? "k_chol_sched(factor)" : "k_chol_sched(solve)");
  }
  if (trace_path && factor) {
    std::vector<unsigned long long> h(4 * (int64_t)std::max(n_trace, 1));
    tbuf.download(h.data(), h.size(), st);
    SSYNC(st);
    if (FILE* f = fopen(trace_path, "ab")) {
      const int hdr[6] = {v.n, v.n_coupled, n_trace, grid, fifo ? v.n_part : -1, v.n_tasks - v.n_part - v.n_coupled};
      fwrite(hdr, sizeof(int), 6, f);
      fwrite(h.data(), sizeof(unsigned long long), h.size(), f);
      if (!fifo) {  // the flow items' codes (fseq): diagonal j < n, block n + b
        const int nf = hdr[5] + v.n_coupled;
        std::vector<int> fs(std::max(nf, 1));
        CK(cudaMemcpy(fs.data(), v.fseq, nf * sizeof(int), cudaMemcpyDeviceToHost));
        fwrite(fs.data(), sizeof(int), nf, f);
      }
      fclose(f);
    }
  }
  if (v.n_iso > 0) CK(cudaStreamWaitEvent(st, s.ch_join_ev, 0));
  return grid;
}

// with_step (chol_begin): |x|_inf and rhs . x ride along -- one launch, one reduction and
// one pack for the residual check AND the Newton step's size / descent test (h_pinned[0] =
// |x|_inf bits, h_pinned[1] = rhs . x), which advance_step reads after its sync
static void launch_resid(Scene& s, const double* rhs, const double* x, bool with_step = false) {
  Scene::Work& w = s.w;
  cudaStream_t st = s.stream;
  unsigned long long* am = w.ull.p + 2;
  if (with_step) {
    w.part.resize(3 * RED_BLOCKS);
    CK(cudaMemsetAsync(am, 0, sizeof(unsigned long long), st));
  }
  k_resid<<<RED_BLOCKS, RED_THREADS, 0, st>>>(s.H.n, s.H.row_ptr.p, s.H.col.p, s.H.val.p, x, rhs, w.r.p, w.part.p,
                                              with_step ? am : nullptr);
  note_launch("k_resid");
  reduce_fixed_multi(st, w.part.p, RED_BLOCKS, with_step ? 3 : 2, w.scal.p + 4);
  if (with_step)
    pack_to_host(st, s.h_pinned, {{am, 8, 0}, {w.scal.p + 6, 8, 8}, {w.scal.p + 4, 16, 192}, {w.bad.p, 4, 224}});
  else
    pack_to_host(st, s.h_pinned + 24, {{w.scal.p + 4, 16, 0}, {w.bad.p, 4, 32}});
}

static void chol_verify_core(Scene& s, Analysis& an);

// ---------------------------------------------------------------------------
// analysis worker: one host thread per scene, one job at a time; a verify request
// (mark_structure after a speculative analysis) runs after the job, on the worker
namespace {
struct CholWorker {
  Scene* s = nullptr;
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  bool job = false, vreq = false, quit = false, has_result = false;
  Analysis result;
  std::exception_ptr err;
  explicit CholWorker(Scene* sc) : s(sc) {
    th = std::thread([this] { loop(); });
  }
  ~CholWorker() {
    {
      std::lock_guard<std::mutex> g(mu);
      quit = true;
    }
    cv.notify_all();
    th.join();
  }
  void loop() {
    for (;;) {
      std::unique_lock<std::mutex> lk(mu);
      cv.wait(lk, [this] { return job || vreq || quit; });
      if (quit) return;
      if (job) {
        lk.unlock();
        Analysis a;
        std::exception_ptr e;
        try {
          a = chol_analyze(*s);
        } catch (...) {
          e = std::current_exception();
        }
        lk.lock();
        result = a;
        err = e;
        has_result = true;
        job = false;
      } else {
        // the actual structure against the speculative plan (re-analysed on a miss)
        Analysis a = result;
        const bool run = has_result && !err;
        lk.unlock();
        std::exception_ptr e;
        if (run) {
          try {
            chol_verify_core(*s, a);
          } catch (...) {
            e = std::current_exception();
          }
        }
        lk.lock();
        if (run) {
          result = a;
          err = e;
        }
        vreq = false;
      }
      lk.unlock();
      cv.notify_all();
    }
  }
  void request_verify() {
    {
      std::lock_guard<std::mutex> g(mu);
      vreq = true;
    }
    cv.notify_all();
  }
  void post() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return !job && !vreq; });
    has_result = false;
    err = nullptr;
    job = true;
    lk.unlock();
    cv.notify_all();
  }
  // waits for the job in flight; true (and the analysis) when one was posted
  bool take(Analysis& out) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return !job && !vreq; });
    if (!has_result) return false;
    has_result = false;
    if (err) {
      std::exception_ptr e = err;
      err = nullptr;
      std::rethrow_exception(e);
    }
    out = result;
    return true;
  }
};

CholWorker* worker(Scene& s, bool create) {
  if (!s.chol_worker && create) s.chol_worker = std::make_shared<CholWorker>(&s);
  return static_cast<CholWorker*>(s.chol_worker.get());
}
}  // namespace

void chol_analysis_post(Scene& s) {
  static const bool off = getenv("ABD_CHOL_SYNC_ANALYSIS") != nullptr;
  if (off || s.H.n == 0) return;
  worker(s, true)->post();
}

void chol_analysis_drop(Scene& s) {
  CholWorker* wk = worker(s, false);
  Analysis a;
  if (wk) {
    try {
      wk->take(a);
    } catch (...) {
    }
  }
}

// An analysis posted at the first line-search trial (mark_structure_early) must cover
// the structure of the iterate actually accepted (copied out by mark_structure); a
// backtracked iterate whose couplings fall outside it is analysed again here.
static void chol_verify_early(Scene& s, Analysis& an) {
  Scene::Work& w = s.w;
  if (!w.ch_verify) return;
  w.ch_verify = false;
  chol_verify_core(s, an);
}

// hand the check to the worker (it runs after the speculative analysis, overlapping
// the pair blocks and the reduction); without a worker chol_begin does it
void chol_verify_post(Scene& s) {
  CholWorker* wk = worker(s, false);
  if (!wk) return;
  s.w.ch_verify = false;
  wk->request_verify();
}

static void chol_verify_core(Scene& s, Analysis& an) {
  Scene::Work& w = s.w;
  CK(cudaEventSynchronize(w.ch_act_ev));
  const int64_t n_off = s.H.n_off;
  const int* f2 = w.h_meta2.p;
  const int* keys = w.h_meta.p + n_off;
  const std::vector<uint64_t>& g = w.ch_cache.edges;
  bool covered = true;
  for (int64_t k = 0; k < n_off && covered; ++k)
    if (f2[k]) {
      const uint64_t e = ((uint64_t)(uint32_t)keys[2 * k] << 32) | (uint32_t)keys[2 * k + 1];
      covered = std::binary_search(g.begin(), g.end(), e);
    }
  if (covered) return;
  std::copy(f2, f2 + n_off, w.h_meta.p);
  w.ch_pre = true;
  an = chol_analyze(s);
}

void chol_begin(Scene& s, const double* rhs, double* x) {
  Bsr& H = s.H;
  Scene::Work& w = s.w;
  cudaStream_t st = s.stream;
  const int n = H.n;
  const int64_t N = 12 * (int64_t)n;
  Scene::Work::CholRun& run = w.ch_run;
  run = Scene::Work::CholRun{};
  if (n == 0) return;
  HMARK();
  auto th0 = std::chrono::steady_clock::now();
  w.bad.resize(1);
  Analysis an;
  CholWorker* wk = worker(s, false);
  if (!wk || !wk->take(an)) an = chol_analyze(s);
  chol_verify_early(s, an);
  HMARK();
  run.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count();
  run.active = true;
  run.rhs = rhs;
  run.x = x;
  run.n_cta = an.n_cta;
  run.stats[0] = an.n_edges;
  run.stats[1] = an.n_blk;
  run.stats[2] = an.n_upd;
  run.stats[3] = an.max_level;
  run.stats[4] = an.largest;
  run.stats[5] = an.n_coupled;
  run.stats[6] = an.cached ? 1 : (an.order_reused ? 2 : 0);  // 2: order reused
  run.ms3[0] = an.ms_sync;
  run.ms3[1] = an.ms_order;
  run.ms3[2] = an.ms_plan;
  CholView v = an.view;
  const int big = 0x7fffffff;
  dev_set_i32(st, w.bad.p, big);
  Scene::KStat& ks = s.kstat[0];
  if (s.instrument) {
    kstat_flush(s, 0);
    CK(cudaEventRecord(ks.e0, st));
  }
  plan_wait(s, st);
  k_chol_apos<<<grid_for(n, 128), 128, 0, st>>>(v);
  note_launch("k_chol_apos");
  run.n_cta = launch_sched(s, v, rhs, x, true);
  if (s.instrument) CK(cudaEventRecord(ks.e1, st));
  w.r.resize(N);
  w.z.resize(N);
  w.part.resize(3 * RED_BLOCKS);
  w.scal.resize(8);
  launch_resid(s, rhs, x, /*with_step=*/true);
}

int chol_finish(Scene& s, double rel_tol, double& rel_res, int max_refine, bool& changed) {
  Scene::Work& w = s.w;
  Scene::Work::CholRun& run = w.ch_run;
  cudaStream_t st = s.stream;
  changed = false;
  rel_res = 0.0;
  if (!run.active) return 0;
  run.active = false;
  const int n = s.H.n;
  const int64_t N = 12 * (int64_t)n;
  const int big = 0x7fffffff;
  double* hp = s.h_pinned + 24;
  int* hb = reinterpret_cast<int*>(s.h_pinned + 28);
  int solves = 1;
  for (int refine = 0;; ++refine) {
    if (refine > 0) SSYNC(st);
    if (*hb != big) throw Error(ABD_ERR_FACTORIZATION, "non-SPD pivot in the block Cholesky", *hb);
    const double rn = std::sqrt(hp[0]), bn = std::sqrt(hp[1]);
    rel_res = bn > 0.0 ? rn / bn : 0.0;
    if (bn == 0.0 || rn <= rel_tol * bn || refine >= max_refine) break;
    CholView v = plan_view(s);
    launch_sched(s, v, w.r.p, w.z.p, false);
    k_add_inplace<<<grid_for(N, 256), 256, 0, st>>>(N, run.x, w.z.p);
    note_launch("k_add_inplace");
    changed = true;
    ++solves;
    launch_resid(s, run.rhs, run.x);
  }
  if (s.instrument) {
    Scene::KStat& k = s.kstat[0];
    // algorithmic bytes of factor + one solve: A blocks read and L written once,
    // L_ik/L_jk read per update pair, L read twice by the solve, vectors.
    const double blk = 1152.0;
    k.pending = true;
    k.p_units = solves;
    k.p_bytes = blk * (double)run.stats[1] * 2.0 + blk * 2.0 * (double)run.stats[2] +
                blk * 2.0 * (double)run.stats[1] + 4.0 * 96.0 * n;
    static const bool trace = getenv("ABD_TRACE_CHOL") != nullptr;
    if (trace) {
      float ms = 0.f;
      CK(cudaEventSynchronize(k.e1));
      CK(cudaEventElapsedTime(&ms, k.e0, k.e1));
      fprintf(stderr,
              "[abd chol] n=%d edges=%lld L_blocks=%lld updates=%lld levels=%lld largest=%lld ctas=%d solves=%d "
              "rel=%.2e factor+solve_ms=%.3f analysis_ms=%.3f (sync %.3f order %.3f plan %.3f) coupled=%lld "
              "cached=%lld hits=%lld misses=%lld\n",
              n, (long long)run.stats[0], (long long)run.stats[1], (long long)run.stats[2], (long long)run.stats[3],
              (long long)run.stats[4], run.n_cta, solves, rel_res, ms, run.host_ms, run.ms3[0], run.ms3[1],
              run.ms3[2], (long long)run.stats[5], (long long)run.stats[6], (long long)w.ch_cache.hits,
              (long long)w.ch_cache.misses);
    }
  }
  return solves;
}

int chol_solve(Scene& s, const double* rhs, double* x, double rel_tol, double& rel_res, int max_refine) {
  chol_begin(s, rhs, x);
  SSYNC(s.stream);
  bool changed = false;
  return chol_finish(s, rel_tol, rel_res, max_refine, changed);
}

// ---------------------------------------------------------------------------
// Multi-rank solve: preconditioned CG on the all-reduced system,
// rows distributed by body slab.  Each rank owns the rows of its slab's dynamic
// slots; its preconditioner is the sparse Cholesky of its slab block (the
// analysis graph masked to in-slab couplings, slab_mask_structure; other slots
// are isolated nodes whose right-hand side is zero).  Per iteration: the search
// direction's slab segments are exchanged (all-reduce of vectors zero outside the
// owned rows = an all-gather, a superset of the SpMV halo), A p on the owned rows,
// and the dot products are all-reduced.  Converged when |b - A x| <= rel_tol |b|
// for the assembled x (solve_refined's contract, sparse.py:149-161), checked on the
// true residual.  p^T A p <= 0 raises ABD_ERR_FACTORIZATION (CG breakdown).
__global__ void k_own_copy(int64_t N, const int* __restrict__ own, const double* __restrict__ src, double* dst) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < N) dst[t] = own[t / 12] ? src[t] : 0.0;
}

// two owned-row dot products (a.b, c.d) as fixed-order partials [RED_BLOCKS][2]
__global__ void k_own_dots(int64_t N, const int* __restrict__ own, const double* __restrict__ a,
                           const double* __restrict__ b, const double* __restrict__ c, const double* __restrict__ d,
                           double* part) {
  __shared__ double s0[RED_THREADS], s1[RED_THREADS];
  double x0 = 0.0, x1 = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    if (own[t / 12]) {
      x0 = fma(a[t], b[t], x0);
      x1 = fma(c[t], d[t], x1);
    }
  s0[threadIdx.x] = x0;
  s1[threadIdx.x] = x1;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s0[threadIdx.x] += s0[threadIdx.x + w];
      s1[threadIdx.x] += s1[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s0[0];
    part[gridDim.x + blockIdx.x] = s1[0];
  }
}

// x += alpha p, r -= alpha q on the owned rows
__global__ void k_own_xr(int64_t N, const int* __restrict__ own, double alpha, const double* __restrict__ p,
                         const double* __restrict__ q, double* x, double* r) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= N || !own[t / 12]) return;
  x[t] = fma(alpha, p[t], x[t]);
  r[t] = fma(-alpha, q[t], r[t]);
}

// p = z + beta p on the owned rows, 0 elsewhere (ready for the segment exchange)
__global__ void k_own_p(int64_t N, const int* __restrict__ own, const double* __restrict__ z, double beta, double* p) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < N) p[t] = own[t / 12] ? fma(beta, p[t], z[t]) : 0.0;
}

int slab_pcg(Scene& s, const double* b, double* x, double rel_tol, int max_iters, double& rel_res) {
  Bsr& H = s.H;
  Scene::Work& w = s.w;
  cudaStream_t st = s.stream;
  const int n = H.n;
  const int64_t N = 12 * (int64_t)n;
  rel_res = 0.0;
  if (n == 0) return 0;
  if (!s.slab_valid) throw Error(ABD_ERR_ARG, "slab_pcg without a slab partition");
  const int* own = s.slab_own_slot.p;
  w.bad.resize(1);
  Analysis an;
  CholWorker* wk = worker(s, false);
  if (!wk || !wk->take(an)) an = chol_analyze(s);
  CholView v = an.view;
  const int big = 0x7fffffff;
  dev_set_i32(st, w.bad.p, big);
  w.r.resize(N);
  w.z.resize(N);
  w.p.resize(N);
  w.Ap.resize(N);
  w.part.resize(2 * RED_BLOCKS);
  w.scal.resize(8);
  double* hs = s.h_pinned + 48;  // scratch scalars (pinned; the line search uses [32, 43))
  int* hb = reinterpret_cast<int*>(s.h_pinned + 52);
  auto dots = [&](const double* a, const double* bb, const double* c, const double* d) {
    k_own_dots<<<RED_BLOCKS, RED_THREADS, 0, st>>>(N, own, a, bb, c, d, w.part.p);
    note_launch("k_own_dots");
    reduce_fixed_multi(st, w.part.p, RED_BLOCKS, 2, w.scal.p);
    comm_allreduce(s, w.scal.p, 2, 0, 0);
    pack_to_host(st, hs, {{w.scal.p, 16, 0}, {w.bad.p, 4, 32}});
    SSYNC(st);
    if (*hb != big) throw Error(ABD_ERR_FACTORIZATION, "non-SPD pivot in the slab block Cholesky", *hb);
  };
  Scene::KStat& ks = s.kstat[0];
  if (s.instrument) {
    kstat_flush(s, 0);
    CK(cudaEventRecord(ks.e0, st));
  }
  plan_wait(s, st);
  k_chol_apos<<<grid_for(n, 128), 128, 0, st>>>(v);
  note_launch("k_chol_apos");
  CK(cudaMemsetAsync(x, 0, N * sizeof(double), st));
  k_own_copy<<<grid_for(N, 256), 256, 0, st>>>(N, own, b, w.r.p);  // r = b (x = 0)
  note_launch("k_own_copy");
  launch_sched(s, v, w.r.p, w.z.p, true);  // factor the slab block, z = M^-1 r
  CK(cudaMemcpyAsync(w.p.p, w.z.p, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  dots(w.r.p, w.z.p, b, b);
  double rz = hs[0];
  const double bn = std::sqrt(hs[1] >= 0.0 ? hs[1] : 0.0);  // owned rows summed over ranks = |b|
  int it = 0;
  if (bn > 0.0) {
    for (int round = 0; round < 3; ++round) {
      for (; it < max_iters;) {
        comm_allreduce(s, w.p.p, N, 0, 0);  // slab segments of p on every rank
        spmv(s, w.p.p, w.Ap.p);
        dots(w.p.p, w.Ap.p, w.p.p, w.Ap.p);
        const double pq = hs[0];
        if (!(pq > 0.0)) throw Error(ABD_ERR_FACTORIZATION, "distributed PCG breakdown (p^T A p <= 0)");
        const double alpha = rz / pq;
        k_own_xr<<<grid_for(N, 256), 256, 0, st>>>(N, own, alpha, w.p.p, w.Ap.p, x, w.r.p);
        note_launch("k_own_xr");
        ++it;
        launch_sched(s, v, w.r.p, w.z.p, false);  // z = M^-1 r (slab triangular solves)
        dots(w.r.p, w.z.p, w.r.p, w.r.p);
        const double rz_new = hs[0];
        if (std::sqrt(std::max(hs[1], 0.0)) <= rel_tol * bn) break;
        k_own_p<<<grid_for(N, 256), 256, 0, st>>>(N, own, w.z.p, rz_new / rz, w.p.p);
        note_launch("k_own_p");
        rz = rz_new;
      }
      // the assembled x and its true residual (identical on every rank)
      CK(cudaMemcpyAsync(w.Ap.p, x, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
      comm_allreduce(s, w.Ap.p, N, 0, 0);
      launch_resid(s, b, w.Ap.p);
      SSYNC(st);
      const double rn = std::sqrt(s.h_pinned[24]), bt = std::sqrt(s.h_pinned[25]);
      rel_res = bt > 0.0 ? rn / bt : 0.0;
      if (rel_res <= rel_tol || it >= max_iters) break;
      // restart from the recursive residual's drift: r = b - A x on the owned rows
      k_own_copy<<<grid_for(N, 256), 256, 0, st>>>(N, own, w.r.p, w.r.p);
      launch_sched(s, v, w.r.p, w.z.p, false);
      CK(cudaMemcpyAsync(w.p.p, w.z.p, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
      dots(w.r.p, w.z.p, w.r.p, w.r.p);
      rz = hs[0];
    }
    CK(cudaMemcpyAsync(x, w.Ap.p, N * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  if (s.instrument) {
    CK(cudaEventRecord(ks.e1, st));
    ks.pending = true;
    ks.p_units = 1 + it;
    ks.p_bytes = 1152.0 * 2.0 * (double)an.n_blk + 1152.0 * 2.0 * (double)an.n_upd +
                 (double)(1 + it) * (1152.0 * 2.0 * (double)an.n_blk + 1152.0 * (double)H.nnzb);
  }
  return it;
}

}  // namespace abd
