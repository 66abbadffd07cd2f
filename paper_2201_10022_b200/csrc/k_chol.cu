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
//   * factor (k_chol_factor): one CTA walks the levels of its components with
//     __syncthreads between levels; a half-warp (lane t = row t) owns one node:
//     D = A_jj - sum_k L_jk L_jk^T, 12x12 Cholesky, then L_ij = (A_ij -
//     sum_k L_ik L_jk^T) L_jj^-T for every block of the column.  Left-looking
//     with fixed update order: deterministic, no atomics.
//   * solve (k_chol_solve): forward levels ascending, backward descending.
//   * refinement exactly as solve_refined: r = b - A x over the resident BSR,
//     stop when |r| <= rel_tol |b|, at most 3 corrections.
// A failed pivot raises ABD_ERR_FACTORIZATION with the smallest failing
// dynamic slot (sparse.py:18-26 semantics).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <iterator>
#include <numeric>
#include <queue>
#include <vector>

#include "driver.h"

namespace abd {

constexpr int CH_THREADS = 256;
constexpr int CH_HW = CH_THREADS / 16;  // half-warps per CTA

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
  const int* blk_apos;  // per off block: position of A(i, j) in the BSR (-1: fill)
  const int* row_ptr;   // n + 1: range into row_blk (blocks L_jk, k eliminated before j)
  const int* row_blk;   // L block index
  const int* row_col;   // column node k of each row_blk entry
  const int* upd_ptr;   // per off block: range into upd
  const int2* upd;      // (L_ik, L_jk) block index pairs
  const int* diag_pos;  // BSR diagonal block positions
  const double* val;    // BSR values
  double* L;            // L blocks, 144 doubles each (row-major)
  int* bad;
};

__device__ __forceinline__ unsigned half_mask(int half) { return 0xffffu << (16 * half); }

__global__ void __launch_bounds__(CH_THREADS) k_chol_factor(CholView v) {
  __shared__ double Ss[CH_HW][12][13];
  const int hw = threadIdx.x >> 4, t = threadIdx.x & 15, half = (threadIdx.x >> 4) & 1;
  const unsigned mask = half_mask(half);
  double (*S)[13] = Ss[hw];
  const int c0 = v.cta_lvl[blockIdx.x], nl = v.cta_nlvl[blockIdx.x];
  for (int l = 0; l < nl; ++l) {
    const int lo = v.lvl_ptr[c0 + l], hi = v.lvl_ptr[c0 + l + 1];
    for (int idx = lo + hw; idx < hi; idx += CH_HW) {
      const int j = v.nodes[idx];
      const int dblk = j;
      // D = A_jj - sum_k L_jk L_jk^T (row t), then symmetrised (sparse.py:117)
      double d[12];
      if (t < 12) {
        const double* A = v.val + 144 * (int64_t)v.diag_pos[j] + 12 * t;
#pragma unroll
        for (int c = 0; c < 12; ++c) d[c] = A[c];
        for (int e = v.row_ptr[j]; e < v.row_ptr[j + 1]; ++e) {
          const double* Lk = v.L + 144 * (int64_t)v.row_blk[e];
          double lr[12];
#pragma unroll
          for (int m = 0; m < 12; ++m) lr[m] = Lk[12 * t + m];
#pragma unroll
          for (int c = 0; c < 12; ++c) {
            double s = 0.0;
#pragma unroll
            for (int m = 0; m < 12; ++m) s = fma(lr[m], Lk[12 * c + m], s);
            d[c] -= s;
          }
        }
#pragma unroll
        for (int c = 0; c < 12; ++c) S[t][c] = d[c];
      }
      __syncwarp(mask);
      double e[12];
      if (t < 12) {
#pragma unroll
        for (int c = 0; c < 12; ++c) e[c] = S[c][t];
      }
      __syncwarp(mask);
      if (t < 12) {
#pragma unroll
        for (int c = 0; c < 12; ++c) S[t][c] = 0.5 * (d[c] + e[c]);
      }
      __syncwarp(mask);
      // right-looking 12x12 Cholesky, lane t owns row t
      bool ok = true;
      for (int c = 0; c < 12; ++c) {
        double p = S[c][c];
        ok = ok && (p > 0.0);
        double sp = sqrt(fmax(p, 1e-300));
        __syncwarp(mask);
        if (t > c && t < 12) S[t][c] /= sp;
        if (t == c) S[c][c] = sp;
        __syncwarp(mask);
        if (t > c && t < 12) {
          double ltc = S[t][c];
          for (int k = c + 1; k <= t; ++k) S[t][k] -= ltc * S[k][c];
        }
        __syncwarp(mask);
      }
      if (!ok && t == 0) atomicMin(v.bad, j);
      double lrow[12];
      if (t < 12) {
        double* Ld = v.L + 144 * (int64_t)dblk + 12 * t;
#pragma unroll
        for (int c = 0; c < 12; ++c) {
          lrow[c] = c <= t ? S[t][c] : 0.0;
          Ld[c] = lrow[c];
        }
      }
      // off-diagonal blocks of column j: L_ij = (A_ij - sum L_ik L_jk^T) L_jj^-T
      for (int b = v.col_ptr[j]; b < v.col_ptr[j + 1]; ++b) {
        const int blk = v.n + b;
        if (t < 12) {
          double bt[12];
          const int ap = v.blk_apos[b];
          if (ap >= 0) {
            const double* A = v.val + 144 * (int64_t)ap + 12 * t;
#pragma unroll
            for (int c = 0; c < 12; ++c) bt[c] = A[c];
          } else {
#pragma unroll
            for (int c = 0; c < 12; ++c) bt[c] = 0.0;
          }
          for (int u = v.upd_ptr[b]; u < v.upd_ptr[b + 1]; ++u) {
            const int2 pq = v.upd[u];
            const double* Li = v.L + 144 * (int64_t)pq.x;  // L_ik
            const double* Lj = v.L + 144 * (int64_t)pq.y;  // L_jk
            double lr[12];
#pragma unroll
            for (int m = 0; m < 12; ++m) lr[m] = Li[12 * t + m];
#pragma unroll
            for (int c = 0; c < 12; ++c) {
              double s = 0.0;
#pragma unroll
              for (int m = 0; m < 12; ++m) s = fma(lr[m], Lj[12 * c + m], s);
              bt[c] -= s;
            }
          }
          // row t of X with X L_jj^T = B: forward substitution against L_jj rows
          double x[12];
#pragma unroll
          for (int c = 0; c < 12; ++c) {
            double s = bt[c];
#pragma unroll
            for (int m = 0; m < c; ++m) s -= S[c][m] * x[m];
            x[c] = s / S[c][c];
          }
          double* Lo = v.L + 144 * (int64_t)blk + 12 * t;
#pragma unroll
          for (int c = 0; c < 12; ++c) Lo[c] = x[c];
        }
      }
      __syncwarp(mask);
    }
    __syncthreads();
  }
}

// x = A^-1 b via the factor (x may alias nothing; y is stored in x).
__global__ void __launch_bounds__(CH_THREADS) k_chol_solve(CholView v, const double* __restrict__ b, double* x) {
  const int hw = threadIdx.x >> 4, t = threadIdx.x & 15, half = (threadIdx.x >> 4) & 1;
  const unsigned mask = half_mask(half);
  const int c0 = v.cta_lvl[blockIdx.x], nl = v.cta_nlvl[blockIdx.x];
  const int tt = t < 12 ? t : 0;
  // forward: L y = b, levels ascending
  for (int l = 0; l < nl; ++l) {
    const int lo = v.lvl_ptr[c0 + l], hi = v.lvl_ptr[c0 + l + 1];
    for (int base = lo; base < hi; base += CH_HW) {
      const int idx = base + hw;
      const bool live = idx < hi;
      const int j = live ? v.nodes[idx] : 0;
      double acc = 0.0, lrow[12];
      if (live) {
        acc = b[12 * (int64_t)j + tt];
        for (int e = v.row_ptr[j]; e < v.row_ptr[j + 1]; ++e) {
          const double* Lk = v.L + 144 * (int64_t)v.row_blk[e] + 12 * tt;
          const double* yk = x + 12 * (int64_t)v.row_col[e];
          double s = 0.0;
#pragma unroll
          for (int m = 0; m < 12; ++m) s = fma(Lk[m], yk[m], s);
          acc -= s;
        }
        const double* Ld = v.L + 144 * (int64_t)j + 12 * tt;
#pragma unroll
        for (int m = 0; m < 12; ++m) lrow[m] = Ld[m];
      } else {
#pragma unroll
        for (int m = 0; m < 12; ++m) lrow[m] = (m == tt) ? 1.0 : 0.0;
      }
      double y = 0.0;
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        double dcc = __shfl_sync(mask, lrow[c], c, 16);
        double yc = __shfl_sync(mask, acc, c, 16) / dcc;
        if (t == c) y = yc;
        if (t > c) acc -= lrow[c] * yc;
      }
      if (live && t < 12) x[12 * (int64_t)j + t] = y;
    }
    __syncthreads();
  }
  // backward: L^T x = y, levels descending
  for (int l = nl - 1; l >= 0; --l) {
    const int lo = v.lvl_ptr[c0 + l], hi = v.lvl_ptr[c0 + l + 1];
    for (int base = lo; base < hi; base += CH_HW) {
      const int idx = base + hw;
      const bool live = idx < hi;
      const int j = live ? v.nodes[idx] : 0;
      double acc = 0.0, lcol[12];
      if (live) {
        acc = x[12 * (int64_t)j + tt];
        for (int bb = v.col_ptr[j]; bb < v.col_ptr[j + 1]; ++bb) {
          const double* Lb = v.L + 144 * (int64_t)(v.n + bb) + tt;  // column tt of L_ij
          const double* xi = x + 12 * (int64_t)v.blk_row[bb];
          double s = 0.0;
#pragma unroll
          for (int r = 0; r < 12; ++r) s = fma(Lb[12 * r], xi[r], s);
          acc -= s;
        }
        const double* Ld = v.L + 144 * (int64_t)j + tt;
#pragma unroll
        for (int m = 0; m < 12; ++m) lcol[m] = Ld[12 * m];  // L_jj[m][tt]
      } else {
#pragma unroll
        for (int m = 0; m < 12; ++m) lcol[m] = (m == tt) ? 1.0 : 0.0;
      }
      double xv = 0.0;
#pragma unroll
      for (int c = 11; c >= 0; --c) {
        double dcc = __shfl_sync(mask, lcol[c], c, 16);
        double xc = __shfl_sync(mask, acc, c, 16) / dcc;
        if (t == c) xv = xc;
        if (t < c) acc -= lcol[c] * xc;
      }
      __syncwarp(mask);
      if (live && t < 12) x[12 * (int64_t)j + t] = xv;
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
  double ms_sync = 0, ms_order = 0, ms_plan = 0;
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
  cudaStream_t st = s.stream;
  const int n = H.n;
  const int64_t n_off = H.n_off;
  Analysis an;
  auto t0 = clk::now();
  // flags | upper_pos | lower_pos | keys (2 ints) per pattern block, one pinned staging buffer
  int* hm = w.h_meta.reserve(5 * (size_t)std::max<int64_t>(n_off, 1));
  int *flags = hm, *upos = hm + n_off, *lpos = hm + 2 * n_off, *keys = hm + 3 * n_off;
  if (n_off) {
    w.ch_flags.resize(n_off);
    k_block_nz<<<grid_for(n_off * 32, 256), 256, 0, st>>>(n_off, H.upper_pos.p, H.val.p, w.ch_flags.p);
    note_launch("k_block_nz");
    CK(cudaMemcpyAsync(flags, w.ch_flags.p, n_off * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(upos, H.upper_pos.p, n_off * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(lpos, H.lower_pos.p, n_off * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(keys, H.upper_keys.p, n_off * sizeof(int2), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  an.ms_sync = ms_since(t0);
  t0 = clk::now();

  // coupled nodes (>= 1 nonzero coupling) get local ids in ascending node order
  std::vector<int> loc(n, -1), glob;
  for (int64_t k = 0; k < n_off; ++k)
    if (flags[k]) {
      loc[keys[2 * k]] = 0;
      loc[keys[2 * k + 1]] = 0;
      ++an.n_edges;
    }
  for (int v = 0; v < n; ++v)
    if (loc[v] == 0) {
      loc[v] = (int)glob.size();
      glob.push_back(v);
    }
  const int m = (int)glob.size();
  an.n_coupled = m;
  // adjacency in key order is already sorted per node (keys sorted by (i, j))
  std::vector<std::vector<int>> adj(m);
  for (int64_t k = 0; k < n_off; ++k)
    if (flags[k]) {
      int a = loc[keys[2 * k]], b = loc[keys[2 * k + 1]];
      adj[a].push_back(b);
      adj[b].push_back(a);
    }
  std::vector<int> order;
  std::vector<std::vector<int>> cs;
  min_degree(m, adj, order, cs);
  std::vector<int> pos(m);
  for (int i = 0; i < m; ++i) pos[order[i]] = i;
  for (auto& c : cs)
    if (c.size() > 1) std::sort(c.begin(), c.end(), [&](int a, int b) { return pos[a] < pos[b]; });
  an.ms_order = ms_since(t0);
  t0 = clk::now();

  auto apos_of = [&](int gi, int gj) -> int {  // BSR position of A(gi, gj) (nonzero coupling)
    int a = std::min(gi, gj), b = std::max(gi, gj);
    int64_t lo = 0, hi = n_off - 1;
    while (lo <= hi) {
      int64_t mm = (lo + hi) >> 1;
      int kx = keys[2 * mm], ky = keys[2 * mm + 1];
      if (kx < a || (kx == a && ky < b)) lo = mm + 1;
      else if (kx == a && ky == b) return flags[mm] ? (gi < gj ? upos[mm] : lpos[mm]) : -1;
      else hi = mm - 1;
    }
    return -1;
  };
  // off-diagonal L blocks: column (local) v owns [col_off[v], col_off[v+1])
  std::vector<int> col_off(m + 1, 0);
  for (int v = 0; v < m; ++v) col_off[v + 1] = col_off[v] + (int)cs[v].size();
  const int nbo = col_off[m];
  an.n_blk = n + (int64_t)nbo;
  // row lists (local i): (k, off block) for k eliminated before i, in elimination order of k
  std::vector<int> rcnt(m + 1, 0);
  for (int v = 0; v < m; ++v)
    for (int i : cs[v]) rcnt[i + 1]++;
  for (int v = 0; v < m; ++v) rcnt[v + 1] += rcnt[v];
  std::vector<int> rfill(rcnt.begin(), rcnt.end() - 1), r_k(nbo), r_b(nbo);
  for (int k : order)
    for (size_t q = 0; q < cs[k].size(); ++q) {
      int i = cs[k][q];
      r_k[rfill[i]] = k;
      r_b[rfill[i]] = col_off[k] + (int)q;
      rfill[i]++;
    }
  // update pairs for off block (i, j): k in rows(j) with i in cs[k]
  std::vector<int> upd_ptr(nbo + 1, 0), upd;
  for (int j = 0; j < m; ++j)
    for (size_t q = 0; q < cs[j].size(); ++q) {
      int b = col_off[j] + (int)q, i = cs[j][q];
      for (int e = rcnt[j]; e < rcnt[j + 1]; ++e) {
        const std::vector<int>& ck = cs[r_k[e]];
        auto it = std::find(ck.begin(), ck.end(), i);
        if (it != ck.end()) {
          upd.push_back(n + col_off[r_k[e]] + (int)(it - ck.begin()));
          upd.push_back(n + r_b[e]);
        }
      }
      upd_ptr[b + 1] = (int)(upd.size() / 2);
    }
  an.n_upd = (int64_t)upd.size() / 2;
  // elimination-tree levels and component roots (local)
  std::vector<int> level(m, 0), root(m);
  for (int v : order)
    if (!cs[v].empty()) level[cs[v][0]] = std::max(level[cs[v][0]], level[v] + 1);
  for (int q = m - 1; q >= 0; --q) {
    int v = order[q];
    root[v] = cs[v].empty() ? v : root[cs[v][0]];
  }
  std::vector<int> csize(m, 0), cdepth(m, 0), comps;
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
  // CTAs: components (largest first onto the least loaded), then isolated nodes
  const int n_iso = n - m;
  const int iso_per_cta = 4 * CH_HW;
  const int n_ccta = std::min((int)comps.size(), 2 * s.num_sms);
  const int n_icta = (n_iso + iso_per_cta - 1) / iso_per_cta;
  const int n_cta = std::max(1, n_ccta + n_icta);
  an.n_cta = n_cta;
  std::vector<int> cta_of(m, -1), cta_nlvl(n_cta, 0);
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
    std::vector<int> cnt(n_lvl_entries + 1, 0);
    for (int v = 0; v < m; ++v) cnt[cta_lvl[cta_of[root[v]]] + level[v]]++;
    int run = 0;
    for (int c = 0; c < n_ccta; ++c)
      for (int l = 0; l <= cta_nlvl[c]; ++l) {
        int ix = cta_lvl[c] + l;
        lvl_ptr[ix] = run;
        if (l < cta_nlvl[c]) run += cnt[ix];
      }
    std::vector<int> fillp(lvl_ptr, lvl_ptr + n_lvl_entries);
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
        for (size_t q = 0; q < cs[l].size(); ++q) {
          int b = col_off[l] + (int)q;  // == c + q since locals follow global order
          hp[off_brow + b] = glob[cs[l][q]];
          hp[off_bapos + b] = apos_of(glob[cs[l][q]], v);
        }
        c += (int)cs[l].size();
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
  std::copy(upd_ptr.begin(), upd_ptr.end(), hp + off_updp);
  std::copy(upd.begin(), upd.end(), hp + off_upd);
  w.ch_plan.resize(total);
  CK(cudaMemcpyAsync(w.ch_plan.p, hp, total * sizeof(int), cudaMemcpyHostToDevice, st));
  w.ch_L.resize(144 * std::max<int64_t>(an.n_blk, 1));
  const int* dp = w.ch_plan.p;
  an.view = CholView{n,
                     dp + off_nodes,
                     dp + off_lvl,
                     dp + off_ctal,
                     dp + off_ctan,
                     dp + off_colp,
                     dp + off_brow,
                     dp + off_bapos,
                     dp + off_rowp,
                     dp + off_rowb,
                     dp + off_rowc,
                     dp + off_updp,
                     reinterpret_cast<const int2*>(dp + off_upd),
                     H.diag_pos.p,
                     H.val.p,
                     w.ch_L.p,
                     w.bad.p};
  an.ms_plan = ms_since(t0);
  return an;
}

// Direct solve of the resident system H x = rhs with refinement (sparse.py:149-161).
// Returns the number of triangular solves (1 + corrections).
int chol_solve(Scene& s, const double* rhs, double* x, double rel_tol, double& rel_res, int max_refine) {
  Bsr& H = s.H;
  Scene::Work& w = s.w;
  cudaStream_t st = s.stream;
  const int n = H.n;
  const int64_t N = 12 * (int64_t)n;
  rel_res = 0.0;
  if (n == 0) return 0;
  auto th0 = std::chrono::steady_clock::now();
  w.bad.resize(1);
  Analysis an = chol_analyze(s);
  const double host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count();
  CholView v = an.view;
  const int big = 0x7fffffff;
  CK(cudaMemcpyAsync(w.bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  if (s.instrument) CK(cudaEventRecord(s.ev0, st));
  k_chol_factor<<<an.n_cta, CH_THREADS, 0, st>>>(v);
  note_launch("k_chol_factor");
  k_chol_solve<<<an.n_cta, CH_THREADS, 0, st>>>(v, rhs, x);
  note_launch("k_chol_solve");
  if (s.instrument) CK(cudaEventRecord(s.ev1, st));
  w.r.resize(N);
  w.z.resize(N);
  w.part.resize(2 * RED_BLOCKS);
  w.scal.resize(4);
  int solves = 1;
  double* hp = s.h_pinned + 24;
  int* hb = reinterpret_cast<int*>(s.h_pinned + 28);
  for (int refine = 0;; ++refine) {
    k_resid<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, H.row_ptr.p, H.col.p, H.val.p, x, rhs, w.r.p, w.part.p);
    note_launch("k_resid");
    reduce_fixed_multi(st, w.part.p, RED_BLOCKS, 2, w.scal.p);
    CK(cudaMemcpyAsync(hp, w.scal.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hb, w.bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*hb != big) throw Error(ABD_ERR_FACTORIZATION, "non-SPD pivot in the block Cholesky", *hb);
    const double rn = std::sqrt(hp[0]), bn = std::sqrt(hp[1]);
    rel_res = bn > 0.0 ? rn / bn : 0.0;
    if (bn == 0.0 || rn <= rel_tol * bn || refine >= max_refine) break;
    k_chol_solve<<<an.n_cta, CH_THREADS, 0, st>>>(v, w.r.p, w.z.p);
    note_launch("k_chol_solve");
    k_add_inplace<<<grid_for(N, 256), 256, 0, st>>>(N, x, w.z.p);
    note_launch("k_add_inplace");
    ++solves;
  }
  if (s.instrument) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, s.ev0, s.ev1));
    Scene::KStat& k = s.kstat[0];
    k.launches += 1;
    k.units += solves;
    k.ms += ms;
    // algorithmic bytes of factor + one solve: A blocks read and L written once,
    // L_ik/L_jk read per update pair, L read twice by the solve, vectors.
    const double blk = 1152.0;
    k.bytes += blk * (double)an.n_blk * 2.0 + blk * 2.0 * (double)an.n_upd + blk * 2.0 * (double)an.n_blk +
               4.0 * 96.0 * n;
    static const bool trace = getenv("ABD_TRACE_CHOL") != nullptr;
    if (trace)
      fprintf(stderr,
              "[abd chol] n=%d edges=%lld L_blocks=%lld updates=%lld levels=%d largest=%d ctas=%d solves=%d "
              "rel=%.2e factor+solve_ms=%.3f analysis_ms=%.3f (sync %.3f order %.3f plan %.3f) coupled=%d\n",
              n, (long long)an.n_edges, (long long)an.n_blk, (long long)an.n_upd, an.max_level, an.largest,
              an.n_cta, solves, rel_res, ms, host_ms, an.ms_sync, an.ms_order, an.ms_plan, an.n_coupled);
  }
  return solves;
}

}  // namespace abd
