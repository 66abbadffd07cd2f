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

struct CholView {
  const int* nodes;     // node ids, CTA-major then level-major
  const int* lvl_ptr;   // per CTA: nlvl + 1 offsets into nodes (absolute)
  const int* cta_lvl;   // per CTA: start index into lvl_ptr
  const int* cta_nlvl;  // per CTA: number of levels
  const int* diag_blk;  // per node: L block index of L_jj (column blocks follow)
  const int* col_cnt;   // per node: number of off-diagonal blocks in column j
  const int* blk_row;   // per L block: row node i (off-diagonal blocks)
  const int* blk_apos;  // per L block: position of A(i, j) in the BSR (-1: fill)
  const int* row_ptr;   // per node: range into row_blk (blocks L_jk, k before j)
  const int* row_blk;
  const int* row_col;   // column node k of each row_blk entry
  const int* upd_ptr;   // per L block: range into upd (pairs (L_ik, L_jk))
  const int2* upd;
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
      const int dblk = v.diag_blk[j];
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
      const int nb = v.col_cnt[j];
      for (int b = 1; b <= nb; ++b) {
        const int blk = dblk + b;
        if (t < 12) {
          double bt[12];
          const int ap = v.blk_apos[blk];
          if (ap >= 0) {
            const double* A = v.val + 144 * (int64_t)ap + 12 * t;
#pragma unroll
            for (int c = 0; c < 12; ++c) bt[c] = A[c];
          } else {
#pragma unroll
            for (int c = 0; c < 12; ++c) bt[c] = 0.0;
          }
          for (int u = v.upd_ptr[blk]; u < v.upd_ptr[blk + 1]; ++u) {
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
        const double* Ld = v.L + 144 * (int64_t)v.diag_blk[j] + 12 * tt;
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
        const int dblk = v.diag_blk[j];
        const int nb = v.col_cnt[j];
        for (int bb = 1; bb <= nb; ++bb) {
          const double* Lb = v.L + 144 * (int64_t)(dblk + bb) + tt;  // column tt of L_ij
          const double* xi = x + 12 * (int64_t)v.blk_row[dblk + bb];
          double s = 0.0;
#pragma unroll
          for (int r = 0; r < 12; ++r) s = fma(Lb[12 * r], xi[r], s);
          acc -= s;
        }
        const double* Ld = v.L + 144 * (int64_t)dblk + tt;
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
  int n_cta = 0;
  int64_t n_blk = 0, n_upd = 0, n_edges = 0;
  int max_level = 0, largest = 0;
};

// minimum-degree elimination on the block graph; returns struct(v) (later
// neighbours at elimination) per node and the elimination order.
void min_degree(int n, std::vector<std::vector<int>>& adj, std::vector<int>& order,
                std::vector<std::vector<int>>& colstruct) {
  order.clear();
  order.reserve(n);
  colstruct.assign(n, {});
  std::vector<char> done(n, 0);
  typedef std::pair<int, int> DI;
  std::priority_queue<DI, std::vector<DI>, std::greater<DI>> heap;
  for (int v = 0; v < n; ++v) {
    if (adj[v].empty()) {
      order.push_back(v);  // isolated: eliminated first, no structure
      done[v] = 1;
    } else {
      heap.push({(int)adj[v].size(), v});
    }
  }
  std::vector<int> merged;
  while (!heap.empty()) {
    DI top = heap.top();
    heap.pop();
    int v = top.second;
    if (done[v] || top.first != (int)adj[v].size()) continue;
    done[v] = 1;
    order.push_back(v);
    std::vector<int> nb = adj[v];  // sorted, alive neighbours
    colstruct[v] = nb;
    for (int a : nb) {
      // adj[a] = (adj[a] U nb) \ {a, v}
      merged.clear();
      std::set_union(adj[a].begin(), adj[a].end(), nb.begin(), nb.end(), std::back_inserter(merged));
      std::vector<int>& out = adj[a];
      out.clear();
      for (int u : merged)
        if (u != a && u != v) out.push_back(u);
      heap.push({(int)out.size(), a});
    }
    adj[v].clear();
  }
}

}  // namespace

static Analysis chol_analyze(Scene& s) {
  Bsr& H = s.H;
  Scene::Work& w = s.w;
  cudaStream_t st = s.stream;
  const int n = H.n;
  const int64_t n_off = H.n_off;
  Analysis an;
  std::vector<int> flags(n_off), upos(n_off), lpos(n_off), dpos(n);
  std::vector<int2> keys(n_off);
  if (n_off) {
    w.ch_flags.resize(n_off);
    k_block_nz<<<grid_for(n_off * 32, 256), 256, 0, st>>>(n_off, H.upper_pos.p, H.val.p, w.ch_flags.p);
    note_launch("k_block_nz");
    w.ch_flags.download(flags.data(), n_off, st);
    H.upper_pos.download(upos.data(), n_off, st);
    H.lower_pos.download(lpos.data(), n_off, st);
    H.upper_keys.download(keys.data(), n_off, st);
  }
  H.diag_pos.download(dpos.data(), n, st);
  CK(cudaStreamSynchronize(st));

  // graph of nonzero couplings (keys are (i < j) sorted)
  std::vector<std::vector<int>> adj(n);
  for (int64_t k = 0; k < n_off; ++k)
    if (flags[k]) {
      adj[keys[k].x].push_back(keys[k].y);
      adj[keys[k].y].push_back(keys[k].x);
      ++an.n_edges;
    }
  for (auto& a : adj) std::sort(a.begin(), a.end());
  // (row, col) -> BSR position of the original coupling, for L block sources
  auto apos_of = [&](int i, int j) -> int {
    int a = std::min(i, j), b = std::max(i, j);
    // binary search in the sorted upper keys
    int64_t lo = 0, hi = n_off - 1;
    while (lo <= hi) {
      int64_t m = (lo + hi) >> 1;
      int2 km = keys[m];
      if (km.x < a || (km.x == a && km.y < b)) lo = m + 1;
      else if (km.x == a && km.y == b) return flags[m] ? (i < j ? upos[m] : lpos[m]) : -1;
      else hi = m - 1;
    }
    return -1;
  };

  std::vector<int> order;
  std::vector<std::vector<int>> cs;
  min_degree(n, adj, order, cs);
  std::vector<int> pos(n);
  for (int i = 0; i < n; ++i) pos[order[i]] = i;
  for (auto& c : cs) std::sort(c.begin(), c.end(), [&](int a, int b) { return pos[a] < pos[b]; });

  // L blocks: per node the diagonal then its column structure
  std::vector<int> diag_blk(n), col_cnt(n);
  int64_t nb = 0;
  for (int j = 0; j < n; ++j) {
    diag_blk[j] = (int)nb;
    col_cnt[j] = (int)cs[j].size();
    nb += 1 + cs[j].size();
  }
  an.n_blk = nb;
  std::vector<int> blk_row(nb, -1), blk_apos(nb, -1);
  // row lists: for node i, blocks L_ik (k eliminated before i), ordered by pos[k]
  std::vector<std::vector<std::pair<int, int>>> rows(n);  // (k, blk)
  for (int k : order) {
    for (size_t q = 0; q < cs[k].size(); ++q) {
      int i = cs[k][q];
      int blk = diag_blk[k] + 1 + (int)q;
      blk_row[blk] = i;
      blk_apos[blk] = apos_of(i, k);
      rows[i].push_back({k, blk});
    }
  }
  std::vector<int> row_ptr(n + 1, 0), row_blk, row_col;
  for (int i = 0; i < n; ++i) {
    row_ptr[i + 1] = row_ptr[i] + (int)rows[i].size();
    for (auto& pr : rows[i]) {
      row_col.push_back(pr.first);
      row_blk.push_back(pr.second);
    }
  }
  // update lists for off-diagonal blocks (i, j): k in rows[j] with i in cs[k]
  std::vector<int> upd_ptr(nb + 1, 0);
  std::vector<int2> upd;
  for (int j = 0; j < n; ++j) {
    for (int bq = 0; bq <= col_cnt[j]; ++bq) {
      int blk = diag_blk[j] + bq;
      if (bq > 0) {
        int i = blk_row[blk];
        for (auto& pr : rows[j]) {
          int k = pr.first;
          const std::vector<int>& ck = cs[k];
          auto it = std::find(ck.begin(), ck.end(), i);
          if (it != ck.end()) upd.push_back(make_int2(diag_blk[k] + 1 + (int)(it - ck.begin()), pr.second));
        }
      }
      upd_ptr[blk + 1] = (int)upd.size();
    }
  }
  an.n_upd = (int64_t)upd.size();
  // elimination tree levels (height above the leaves) and component roots
  std::vector<int> level(n, 0), root(n);
  for (int v : order)
    if (!cs[v].empty()) {
      int p = cs[v][0];
      level[p] = std::max(level[p], level[v] + 1);
    }
  for (int q = n - 1; q >= 0; --q) {
    int v = order[q];
    root[v] = cs[v].empty() ? v : root[cs[v][0]];
  }
  // components -> CTAs (largest first onto the least loaded CTA)
  std::vector<int> csize(n, 0), cdepth(n, 0);
  for (int v = 0; v < n; ++v) {
    csize[root[v]]++;
    cdepth[root[v]] = std::max(cdepth[root[v]], level[v] + 1);
  }
  std::vector<int> comps;
  for (int v = 0; v < n; ++v)
    if (root[v] == v) comps.push_back(v);
  std::sort(comps.begin(), comps.end(), [&](int a, int b) {
    return csize[a] != csize[b] ? csize[a] > csize[b] : a < b;
  });
  an.largest = comps.empty() ? 0 : csize[comps[0]];
  const int n_cta = std::max(1, std::min((int)comps.size(), 4 * s.num_sms));
  an.n_cta = n_cta;
  std::vector<int> cta_of_root(n, -1);
  {
    typedef std::pair<int64_t, int> LI;
    std::priority_queue<LI, std::vector<LI>, std::greater<LI>> load;
    for (int c = 0; c < n_cta; ++c) load.push({0, c});
    for (int r : comps) {
      LI top = load.top();
      load.pop();
      cta_of_root[r] = top.second;
      // cost: nodes spread over the CTA's half-warps plus the level latency
      top.first += (int64_t)csize[r] + 8 * (int64_t)cdepth[r];
      load.push(top);
    }
  }
  std::vector<int> cta_nlvl(n_cta, 0);
  for (int v = 0; v < n; ++v) {
    int c = cta_of_root[root[v]];
    cta_nlvl[c] = std::max(cta_nlvl[c], level[v] + 1);
    an.max_level = std::max(an.max_level, level[v] + 1);
  }
  std::vector<int> cta_lvl(n_cta + 1, 0);
  for (int c = 0; c < n_cta; ++c) cta_lvl[c + 1] = cta_lvl[c] + cta_nlvl[c] + 1;
  std::vector<int> cnt(cta_lvl[n_cta], 0);
  for (int v = 0; v < n; ++v) cnt[cta_lvl[cta_of_root[root[v]]] + level[v]]++;
  std::vector<int> lvl_ptr(cta_lvl[n_cta], 0);
  {
    int run = 0;
    for (int c = 0; c < n_cta; ++c) {
      for (int l = 0; l <= cta_nlvl[c]; ++l) {
        int e = cta_lvl[c] + l;
        lvl_ptr[e] = run;
        if (l < cta_nlvl[c]) run += cnt[e];
      }
    }
  }
  std::vector<int> fillp(lvl_ptr), nodes(n);
  for (int v = 0; v < n; ++v) nodes[fillp[cta_lvl[cta_of_root[root[v]]] + level[v]]++] = v;

  auto up = [&](DVec<int>& d, const std::vector<int>& h) { d.upload(h.data(), std::max<size_t>(h.size(), 1), st); };
  up(w.ch_nodes, nodes);
  up(w.ch_lvl_ptr, lvl_ptr);
  up(w.ch_cta_lvl, cta_lvl);
  up(w.ch_cta_nlvl, cta_nlvl);
  up(w.ch_diag_blk, diag_blk);
  up(w.ch_col_cnt, col_cnt);
  up(w.ch_blk_row, blk_row);
  up(w.ch_blk_apos, blk_apos);
  up(w.ch_row_ptr, row_ptr);
  if (row_blk.empty()) row_blk.push_back(0), row_col.push_back(0);
  up(w.ch_row_blk, row_blk);
  up(w.ch_row_col, row_col);
  up(w.ch_upd_ptr, upd_ptr);
  if (upd.empty()) upd.push_back(make_int2(0, 0));
  w.ch_upd.upload(upd.data(), upd.size(), st);
  w.ch_L.resize(144 * std::max<int64_t>(nb, 1));
  return an;
}

static CholView chol_view(Scene& s) {
  Scene::Work& w = s.w;
  return CholView{w.ch_nodes.p,    w.ch_lvl_ptr.p, w.ch_cta_lvl.p, w.ch_cta_nlvl.p, w.ch_diag_blk.p,
                  w.ch_col_cnt.p,  w.ch_blk_row.p, w.ch_blk_apos.p, w.ch_row_ptr.p, w.ch_row_blk.p,
                  w.ch_row_col.p,  w.ch_upd_ptr.p, w.ch_upd.p,      s.H.diag_pos.p, s.H.val.p,
                  w.ch_L.p,        w.bad.p};
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
  Analysis an = chol_analyze(s);
  CholView v = chol_view(s);
  w.bad.resize(1);
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
              "rel=%.2e factor+solve_ms=%.3f\n",
              n, (long long)an.n_edges, (long long)an.n_blk, (long long)an.n_upd, an.max_level, an.largest,
              an.n_cta, solves, rel_res, ms);
  }
  return solves;
}

}  // namespace abd
