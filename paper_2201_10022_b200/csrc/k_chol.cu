// K4 (direct): sparse block Cholesky with iterative refinement on the device,
// the reference's Newton linear solve BlockCholesky(A).solve_refined(-g,
// rel_tol=1e-8) (sparse.py:90-161, solver.py:345-348) restated for B200.
//
// Per Newton iteration:
//   * analysis (host, C++): the exactly-zero pattern blocks (overlapping body
//     boxes without an active contact) are dropped, the remaining block graph
//     is ordered by minimum degree, the symbolic factor (fill), elimination
//     tree and its levels are built, and connected components are packed onto
//     CTAs.  Contact graphs of piles are forests of short chains, so the fill
//     is ~0 and the tree height is tens of levels.
//   * factor + solve (k_chol_factor_solve): one CTA walks the levels of its components with
//     __syncthreads between levels; a warp (lane t = row t) owns one node:
//     D = A_jj - sum_k L_jk L_jk^T, 12x12 Cholesky, then L_ij = (A_ij -
//     sum_k L_ik L_jk^T) L_jj^-T for every block of the column.  Left-looking
//     with fixed update order: deterministic, no atomics.
//     The forward substitution of node j runs right after its factor; the
//     backward sweep follows in the same kernel (levels descending).  The
//     12x12 pivots are in-register Cholesky factors (shuffles, rsqrt per pivot).
//   * refinement solves (k_chol_solve) reuse the factor and 1 / L_cc.
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

constexpr int CH_THREADS = 384;
constexpr int CH_HW = CH_THREADS / 32;  // warps per CTA (one node per warp, lane t = row t)

// Plan layout (one packed int buffer uploaded per analysis).  L holds the n
// diagonal blocks first (L_jj at index j), then the off-diagonal blocks.
struct CholView {
  int n;
  const int* nodes;     // node ids, CTA-major then level-major (isolated nodes last)
  const int* lvl_ptr;   // per CTA: nlvl + 1 offsets into nodes (absolute)
  const int* cta_lvl;   // per CTA: start index into lvl_ptr
  const int* cta_nlvl;  // per CTA: number of levels
  const int* col_ptr;   // n + 1: off-diagonal blocks of column j (index k -> L block n + k)
  const int* blk_row;   // per off block: row node i
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
  long long* dbg;       // optional per-node phase clocks of CTA 0 (ABD_CHOL_CLOCK)
};


// full-warp shuffles: every lane of a warp runs the same node, so no partial-mask
// convergence checks are generated
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

// Factor + forward substitution (levels ascending), then backward substitution
// (levels descending), one CTA per group of components.  x receives y, then x.
// BSR positions of the factor's off-diagonal source blocks, all nodes in parallel
// (takes the binary searches off the level-serial critical path)
__global__ void k_chol_apos(CholView v) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= v.n) return;
  for (int b = v.col_ptr[j]; b < v.col_ptr[j + 1]; ++b) v.apos[b] = bsr_find(v.bsr_row, v.bsr_col, v.blk_row[b], j);
}

__global__ void __launch_bounds__(CH_THREADS) k_chol_factor_solve(CholView v, const double* __restrict__ b,
                                                                   double* x) {
  __shared__ double Ss[CH_HW][12][13];  // per warp: staged L_jk / symmetrisation / L_jj
  __shared__ double Ts[CH_HW][12][13];  // per warp: staged L_jk of update pairs
  const int hw = threadIdx.x >> 5, t = threadIdx.x & 31;
  const int tt = t < 12 ? t : 0;
  const unsigned mask = 0xffffffffu;
  double (*S)[13] = Ss[hw];
  double (*T)[13] = Ts[hw];
  const int c0 = v.cta_lvl[blockIdx.x], nl = v.cta_nlvl[blockIdx.x];
  for (int l = 0; l < nl; ++l) {
    const int lo = v.lvl_ptr[c0 + l], hi = v.lvl_ptr[c0 + l + 1];
    for (int idx = lo + hw; idx < hi; idx += CH_HW) {
      const int j = v.nodes[idx];
      long long ck0 = (v.dbg && blockIdx.x == 0) ? clock64() : 0;
      double d[12];
      {
        const double* A = v.val + 144 * (int64_t)v.diag_pos[j] + 12 * tt;
#pragma unroll
        for (int c = 0; c < 12; ++c) d[c] = A[c];
      }
      double acc = b[12 * (int64_t)j + tt];
      // D = A_jj - sum_k L_jk L_jk^T and b_j - sum_k L_jk y_k over the row list of j
      for (int e = v.row_ptr[j]; e < v.row_ptr[j + 1]; ++e) {
        const double* Lk = v.L + 144 * (int64_t)v.row_blk[e] + 12 * tt;
        const double* yk = x + 12 * (int64_t)v.row_col[e];
        double lr[12];
#pragma unroll
        for (int m = 0; m < 12; ++m) lr[m] = Lk[m];
        __syncwarp(mask);
        if (t < 12) {
#pragma unroll
          for (int m = 0; m < 12; ++m) S[t][m] = lr[m];
        }
        __syncwarp(mask);
        double s2 = 0.0;
#pragma unroll
        for (int m = 0; m < 12; ++m) s2 = fma(lr[m], yk[m], s2);
        acc -= s2;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          double s = 0.0;
#pragma unroll
          for (int m = 0; m < 12; ++m) s = fma(lr[m], S[c][m], s);
          d[c] -= s;
        }
      }
      // symmetrise (sparse.py:117: cholesky(0.5 (D + D^T)))
      __syncwarp(mask);
      if (t < 12) {
#pragma unroll
        for (int c = 0; c < 12; ++c) S[t][c] = d[c];
      }
      __syncwarp(mask);
#pragma unroll
      for (int c = 0; c < 12; ++c) d[c] = 0.5 * (d[c] + S[c][tt]);
      double rinv[12];
      long long ck1 = (v.dbg && blockIdx.x == 0) ? clock64() : 0;
      const bool ok = chol12(mask, t, d, rinv);
      long long ck2 = (v.dbg && blockIdx.x == 0) ? clock64() : 0;
      if (!ok && t == 0) atomicMin(v.bad, j);
      __syncwarp(mask);
      if (t < 12) {
        double* Ld = v.L + 144 * (int64_t)j + 12 * t;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          Ld[c] = d[c];
          S[t][c] = d[c];  // L_jj rows for the off-diagonal solves below
        }
        double mine = rinv[0];
#pragma unroll
        for (int c = 1; c < 12; ++c)
          if (c == t) mine = rinv[c];
        v.dinv[12 * (int64_t)j + t] = mine;
      }
      // forward substitution for node j
      const double y = lower_solve12(mask, t, acc, d, rinv);
      if (t < 12) x[12 * (int64_t)j + t] = y;
      __syncwarp(mask);
      long long ck3 = (v.dbg && blockIdx.x == 0) ? clock64() : 0;
      // off-diagonal blocks of column j: L_ij = (A_ij - sum L_ik L_jk^T) L_jj^-T
      for (int bb = v.col_ptr[j]; bb < v.col_ptr[j + 1]; ++bb) {
        double bt[12];
        const int ap = v.apos[bb];
        if (ap >= 0) {
          const double* A = v.val + 144 * (int64_t)ap + 12 * tt;
#pragma unroll
          for (int c = 0; c < 12; ++c) bt[c] = A[c];
        } else {
#pragma unroll
          for (int c = 0; c < 12; ++c) bt[c] = 0.0;
        }
        for (int u = v.upd_ptr[bb]; u < v.upd_ptr[bb + 1]; ++u) {
          const int2 pq = v.upd[u];
          const double* Li = v.L + 144 * (int64_t)pq.x + 12 * tt;  // row t of L_ik
          const double* Lj = v.L + 144 * (int64_t)pq.y + 12 * tt;  // row t of L_jk (staged)
          double lr[12];
#pragma unroll
          for (int m = 0; m < 12; ++m) lr[m] = Li[m];
          __syncwarp(mask);
          if (t < 12) {
#pragma unroll
            for (int m = 0; m < 12; ++m) T[t][m] = Lj[m];
          }
          __syncwarp(mask);
#pragma unroll
          for (int c = 0; c < 12; ++c) {
            double s = 0.0;
#pragma unroll
            for (int m = 0; m < 12; ++m) s = fma(lr[m], T[c][m], s);
            bt[c] -= s;
          }
        }
        // row t of X with X L_jj^T = B (forward substitution against L_jj rows)
        double xr[12];
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          double s = bt[c];
#pragma unroll
          for (int m = 0; m < 12; ++m)
            if (m < c) s = fma(-S[c][m], xr[m], s);
          xr[c] = s * rinv[c];
        }
        if (t < 12) {
          double* Lo = v.L + 144 * (int64_t)(v.n + bb) + 12 * t;
#pragma unroll
          for (int c = 0; c < 12; ++c) Lo[c] = xr[c];
        }
      }
      __syncwarp(mask);
      if (v.dbg && blockIdx.x == 0 && t == 0 && idx - v.lvl_ptr[c0] < 256) {
        long long* o = v.dbg + 8 * (idx - v.lvl_ptr[c0]);
        o[0] = j;
        o[1] = l;
        o[2] = ck0;
        o[3] = ck1;
        o[4] = ck2;
        o[5] = ck3;
        o[6] = clock64();
        o[7] = v.col_ptr[j + 1] - v.col_ptr[j];
      }
    }
    __syncthreads();
  }
  // backward: L^T x = y, levels descending
  for (int l = nl - 1; l >= 0; --l) {
    const int lo = v.lvl_ptr[c0 + l], hi = v.lvl_ptr[c0 + l + 1];
    for (int idx = lo + hw; idx < hi; idx += CH_HW) {
      const int j = v.nodes[idx];
      double acc = x[12 * (int64_t)j + tt];
      for (int bb = v.col_ptr[j]; bb < v.col_ptr[j + 1]; ++bb) {
        const double* Lb = v.L + 144 * (int64_t)(v.n + bb) + tt;  // column tt of L_ij
        const double* xi = x + 12 * (int64_t)v.blk_row[bb];
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < 12; ++r) s = fma(Lb[12 * r], xi[r], s);
        acc -= s;
      }
      double lcol[12], rinv[12];
      const double* Ld = v.L + 144 * (int64_t)j + tt;
      const double* di = v.dinv + 12 * (int64_t)j;
#pragma unroll
      for (int m = 0; m < 12; ++m) {
        lcol[m] = Ld[12 * m];
        rinv[m] = di[m];
      }
      const double xv = upper_solve12(mask, t, acc, lcol, rinv);
      __syncwarp(mask);
      if (t < 12) x[12 * (int64_t)j + t] = xv;
    }
    __syncthreads();
  }
}

// x = A^-1 b with the resident factor (refinement corrections)
__global__ void __launch_bounds__(CH_THREADS) k_chol_solve(CholView v, const double* __restrict__ b, double* x) {
  const int hw = threadIdx.x >> 5, t = threadIdx.x & 31;
  const unsigned mask = 0xffffffffu;
  const int c0 = v.cta_lvl[blockIdx.x], nl = v.cta_nlvl[blockIdx.x];
  const int tt = t < 12 ? t : 0;
  for (int l = 0; l < nl; ++l) {
    const int lo = v.lvl_ptr[c0 + l], hi = v.lvl_ptr[c0 + l + 1];
    for (int idx = lo + hw; idx < hi; idx += CH_HW) {
      const int j = v.nodes[idx];
      double acc = b[12 * (int64_t)j + tt];
      for (int e = v.row_ptr[j]; e < v.row_ptr[j + 1]; ++e) {
        const double* Lk = v.L + 144 * (int64_t)v.row_blk[e] + 12 * tt;
        const double* yk = x + 12 * (int64_t)v.row_col[e];
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < 12; ++m) s = fma(Lk[m], yk[m], s);
        acc -= s;
      }
      double lrow[12], rinv[12];
      const double* Ld = v.L + 144 * (int64_t)j + 12 * tt;
      const double* di = v.dinv + 12 * (int64_t)j;
#pragma unroll
      for (int m = 0; m < 12; ++m) {
        lrow[m] = Ld[m];
        rinv[m] = di[m];
      }
      const double y = lower_solve12(mask, t, acc, lrow, rinv);
      if (t < 12) x[12 * (int64_t)j + t] = y;
    }
    __syncthreads();
  }
  for (int l = nl - 1; l >= 0; --l) {
    const int lo = v.lvl_ptr[c0 + l], hi = v.lvl_ptr[c0 + l + 1];
    for (int idx = lo + hw; idx < hi; idx += CH_HW) {
      const int j = v.nodes[idx];
      double acc = x[12 * (int64_t)j + tt];
      for (int bb = v.col_ptr[j]; bb < v.col_ptr[j + 1]; ++bb) {
        const double* Lb = v.L + 144 * (int64_t)(v.n + bb) + tt;
        const double* xi = x + 12 * (int64_t)v.blk_row[bb];
        double s = 0.0;
#pragma unroll
        for (int r = 0; r < 12; ++r) s = fma(Lb[12 * r], xi[r], s);
        acc -= s;
      }
      double lcol[12], rinv[12];
      const double* Ld = v.L + 144 * (int64_t)j + tt;
      const double* di = v.dinv + 12 * (int64_t)j;
#pragma unroll
      for (int m = 0; m < 12; ++m) {
        lcol[m] = Ld[12 * m];
        rinv[m] = di[m];
      }
      const double xv = upper_solve12(mask, t, acc, lcol, rinv);
      __syncwarp(mask);
      if (t < 12) x[12 * (int64_t)j + t] = xv;
    }
    __syncthreads();
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
                        double* r, double* part) {
  __shared__ double sr[RED_THREADS], sb[RED_THREADS];
  double ar = 0.0, ab = 0.0;
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

// ---------------------------------------------------------------------------
// host analysis
namespace {

struct Analysis {
  int n_cta = 0, n_coupled = 0;
  int64_t n_blk = 0, n_upd = 0, n_edges = 0;
  int max_level = 0, largest = 0;
  double ms_sync = 0, ms_order = 0, ms_plan = 0, ms_sub[6] = {};
  bool cached = false;
  CholView view{};
};

// minimum-degree elimination on a (local) graph; colstruct[v] = neighbours
// still alive when v is eliminated (its L column structure), order = elimination order.
void min_degree(int m, std::vector<std::vector<int>>& adj, std::vector<int>& order,
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
  auto make_view = [&](const size_t* o) {
    const int* dp = w.ch_plan.p;
    return CholView{n,
                    dp + o[0],
                    dp + o[1],
                    dp + o[2],
                    dp + o[3],
                    dp + o[4],
                    dp + o[5],
                    H.row_ptr.p,
                    H.col.p,
                    w.ch_apos.p,
                    dp + o[7],
                    dp + o[8],
                    dp + o[9],
                    dp + o[10],
                    reinterpret_cast<const int2*>(dp + o[11]),
                    H.diag_pos.p,
                    H.val.p,
                    w.ch_L.p,
                    w.ch_dinv.p,
                    w.bad.p};
  };
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
    an.view = make_view(cc.offs);
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
  const int n_core = m - (int)order.size();
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
                   &csize = w.hs_i[22], &cdepth = w.hs_i[23], &comps = w.hs_i[24], &cta_of = w.hs_i[25],
                   &cta_nlvl = w.hs_i[26], &lcnt = w.hs_i[27], &fillp = w.hs_i[28];
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
  // update pairs for off block (i, j): k in rows(j) with i in cs[k]
  upd_ptr.assign(nbo + 1, 0);
  upd.clear();
  for (int j = 0; j < m; ++j)
    for (int b = csp[j]; b < csp[j + 1]; ++b) {
      const int i = csi[b];
      for (int e = rcnt[j]; e < rcnt[j + 1]; ++e) {
        const int k = r_k[e];
        for (int f = csp[k]; f < csp[k + 1]; ++f)
          if (csi[f] == i) {
            upd.push_back(n + f);
            upd.push_back(n + r_b[e]);
            break;
          }
      }
      upd_ptr[b + 1] = (int)(upd.size() / 2);
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
  // CTAs: components (largest first onto the least loaded), then isolated nodes
  const int n_iso = n - m;
  const int iso_per_cta = 4 * CH_HW;
  const int n_ccta = std::min((int)comps.size(), 2 * s.num_sms);
  const int n_icta = (n_iso + iso_per_cta - 1) / iso_per_cta;
  const int n_cta = std::max(1, n_ccta + n_icta);
  an.n_cta = n_cta;
  cta_of.assign(m, -1);
  cta_nlvl.assign(n_cta, 0);
  {
    typedef std::pair<int64_t, int> LI;
    std::priority_queue<LI, std::vector<LI>, std::greater<LI>> load;
    for (int c = 0; c < n_ccta; ++c) load.push({0, c});
    for (int r : comps) {
      LI top = load.top();
      load.pop();
      cta_of[r] = top.second;
      cta_nlvl[top.second] = std::max(cta_nlvl[top.second], cdepth[r]);
      top.first += (int64_t)csize[r] + 8 * (int64_t)cdepth[r];
      load.push(top);
    }
  }
  for (int c = n_ccta; c < n_cta; ++c) cta_nlvl[c] = (n_iso > 0) ? 1 : 0;

  an.ms_sub[4] = ms_since(t0);
  // packed plan: nodes | lvl_ptr | cta_lvl | cta_nlvl | col_ptr | blk_row | blk_apos | row_ptr |
  //              row_blk | row_col | upd_ptr | (pad) | upd pairs
  int n_lvl_entries = 0;
  for (int c = 0; c < n_cta; ++c) n_lvl_entries += cta_nlvl[c] + 1;
  size_t off_nodes = 0, off_lvl = off_nodes + n, off_ctal = off_lvl + n_lvl_entries, off_ctan = off_ctal + n_cta,
         off_colp = off_ctan + n_cta, off_brow = off_colp + n + 1, off_bapos = off_brow + nbo,
         off_rowp = off_bapos + nbo, off_rowb = off_rowp + n + 1, off_rowc = off_rowb + nbo,
         off_updp = off_rowc + nbo, off_upd = off_updp + nbo + 1;
  off_upd += off_upd & 1;  // int2 alignment
  const size_t total = off_upd + upd.size() + 2;
  int* hp = w.h_plan.reserve(total);
  int* nodes = hp + off_nodes;
  int* lvl_ptr = hp + off_lvl;
  int* cta_lvl = hp + off_ctal;
  int* cta_nl = hp + off_ctan;
  {
    // count nodes per (cta, level), then prefix offsets
    int e = 0;
    for (int c = 0; c < n_cta; ++c) {
      cta_lvl[c] = e;
      cta_nl[c] = cta_nlvl[c];
      e += cta_nlvl[c] + 1;
    }
    std::vector<int>& cnt = lcnt;
    cnt.assign(n_lvl_entries + 1, 0);
    for (int v = 0; v < m; ++v) cnt[cta_lvl[cta_of[root[v]]] + level[v]]++;
    int run = 0;
    for (int c = 0; c < n_ccta; ++c)
      for (int l = 0; l <= cta_nlvl[c]; ++l) {
        int ix = cta_lvl[c] + l;
        lvl_ptr[ix] = run;
        if (l < cta_nlvl[c]) run += cnt[ix];
      }
    fillp.assign(lvl_ptr, lvl_ptr + n_lvl_entries);
    for (int v = 0; v < m; ++v) nodes[fillp[cta_lvl[cta_of[root[v]]] + level[v]]++] = glob[v];
    // isolated nodes, iso_per_cta per CTA in node order
    int iso = m;
    for (int c = n_ccta; c < n_cta; ++c) {
      lvl_ptr[cta_lvl[c]] = iso;
      iso = std::min(n, iso + iso_per_cta);
      lvl_ptr[cta_lvl[c] + 1] = iso;
    }
    int q = m;
    for (int v = 0; v < n; ++v)
      if (loc[v] < 0) nodes[q++] = v;
  }
  int* col_ptr = hp + off_colp;
  int* row_ptr = hp + off_rowp;
  {
    // per global node column/row ranges (empty for isolated nodes)
    int c = 0, r = 0;
    for (int v = 0; v < n; ++v) {
      col_ptr[v] = c;
      row_ptr[v] = r;
      int l = loc[v];
      if (l >= 0) {
        for (int b = csp[l]; b < csp[l + 1]; ++b) {  // b == c + q: locals follow global order
          hp[off_brow + b] = glob[csi[b]];
        }
        c += csp[l + 1] - csp[l];
        for (int e2 = rcnt[l]; e2 < rcnt[l + 1]; ++e2) {
          hp[off_rowb + r] = r_b[e2] + n;
          hp[off_rowc + r] = glob[r_k[e2]];
          ++r;
        }
      }
    }
    col_ptr[n] = c;
    row_ptr[n] = r;
  }
  an.ms_sub[5] = ms_since(t0);
  std::copy(upd_ptr.begin(), upd_ptr.end(), hp + off_updp);
  std::copy(upd.begin(), upd.end(), hp + off_upd);
  w.ch_plan.resize(total);
  CK(cudaMemcpyAsync(w.ch_plan.p, hp, total * sizeof(int), cudaMemcpyHostToDevice, st));
  w.ch_L.resize(144 * std::max<int64_t>(an.n_blk, 1));
  w.ch_dinv.resize(12 * std::max<int64_t>(n, 1));
  w.ch_apos.resize(std::max<int64_t>(an.n_blk - n, 1));
  const size_t offs[13] = {off_nodes, off_lvl,  off_ctal, off_ctan, off_colp, off_brow, off_bapos,
                           off_rowp,  off_rowb, off_rowc, off_updp, off_upd,  total};
  an.view = make_view(offs);
  cc.valid = true;
  cc.n = n;
  cc.n_off = n_off;
  cc.edges.swap(cur);
  const int64_t st8[8] = {an.n_cta, an.n_coupled, an.n_blk, an.n_upd, an.n_edges, an.max_level, an.largest, 0};
  std::copy(st8, st8 + 8, cc.stats);
  std::copy(offs, offs + 13, cc.offs);
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
static CholView plan_view(Scene& s) {
  Scene::Work& w = s.w;
  const size_t* o = w.ch_cache.offs;
  const int* dp = w.ch_plan.p;
  return CholView{s.H.n,
                  dp + o[0],
                  dp + o[1],
                  dp + o[2],
                  dp + o[3],
                  dp + o[4],
                  dp + o[5],
                  s.H.row_ptr.p,
                  s.H.col.p,
                  w.ch_apos.p,
                  dp + o[7],
                  dp + o[8],
                  dp + o[9],
                  dp + o[10],
                  reinterpret_cast<const int2*>(dp + o[11]),
                  s.H.diag_pos.p,
                  s.H.val.p,
                  w.ch_L.p,
                  w.ch_dinv.p,
                  w.bad.p,
                  nullptr};
}

static void launch_resid(Scene& s, const double* rhs, const double* x) {
  Scene::Work& w = s.w;
  cudaStream_t st = s.stream;
  k_resid<<<RED_BLOCKS, RED_THREADS, 0, st>>>(s.H.n, s.H.row_ptr.p, s.H.col.p, s.H.val.p, x, rhs, w.r.p, w.part.p);
  note_launch("k_resid");
  reduce_fixed_multi(st, w.part.p, RED_BLOCKS, 2, w.scal.p + 4);
  pack_to_host(st, s.h_pinned + 24, {{w.scal.p + 4, 16, 0}, {w.bad.p, 4, 32}});
}

// ---------------------------------------------------------------------------
// analysis worker: one host thread per scene, one job at a time
namespace {
struct CholWorker {
  Scene* s = nullptr;
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  bool job = false, quit = false, has_result = false;
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
      cv.wait(lk, [this] { return job || quit; });
      if (quit) return;
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
      lk.unlock();
      cv.notify_all();
    }
  }
  void post() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return !job; });
    has_result = false;
    err = nullptr;
    job = true;
    lk.unlock();
    cv.notify_all();
  }
  // waits for the job in flight; true (and the analysis) when one was posted
  bool take(Analysis& out) {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return !job; });
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
  run.stats[6] = an.cached ? 1 : 0;
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
  static const bool clk_dbg = getenv("ABD_CHOL_CLOCK") != nullptr;
  static DVec<long long> dbgbuf;
  if (clk_dbg) {
    dbgbuf.resize(8 * 256);
    dbgbuf.zero(st);
    v.dbg = dbgbuf.p;
  }
  k_chol_apos<<<grid_for(n, 128), 128, 0, st>>>(v);
  note_launch("k_chol_apos");
  k_chol_factor_solve<<<an.n_cta, CH_THREADS, 0, st>>>(v, rhs, x);
  note_launch("k_chol_factor_solve");
  if (s.instrument) CK(cudaEventRecord(ks.e1, st));
  if (clk_dbg) {
    std::vector<long long> hb(8 * 256);
    dbgbuf.download(hb.data(), hb.size(), st);
    SSYNC(st);
    long long t0c = hb[2];
    fprintf(stderr, "[abd chol clock] node level start D_done chol_done fwd_done end n_off (cycles from first)\n");
    for (int q = 0; q < 256; ++q) {
      long long* o = &hb[8 * q];
      if (o[2] == 0) continue;
      fprintf(stderr, "  %6lld %3lld %8lld %6lld %6lld %6lld %6lld %lld\n", o[0], o[1], o[2] - t0c, o[3] - o[2],
              o[4] - o[3], o[5] - o[4], o[6] - o[5], o[7]);
    }
  }
  w.r.resize(N);
  w.z.resize(N);
  w.part.resize(2 * RED_BLOCKS);
  w.scal.resize(8);
  launch_resid(s, rhs, x);
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
    k_chol_solve<<<run.n_cta, CH_THREADS, 0, st>>>(v, w.r.p, w.z.p);
    note_launch("k_chol_solve");
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

}  // namespace abd
