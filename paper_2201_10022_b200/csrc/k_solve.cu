// Assembly into a symmetric BSR (solver.py:257-342) and the block-Jacobi
// PCG (K4) that replaces BlockCholesky.solve_refined (sparse.py:90-161).
//
// Assembly is a deterministic segmented reduction: every per-pair local
// block (contact pairs in candidate order, then friction pairs) emits up to
// three contributions (diag a, diag b, upper (a,b)); a stable radix sort by
// target CSR position keeps pair order inside each target, and one warp per
// target block accumulates in that order on top of the K1 per-body terms —
// the same summation order as the reference's pair-major np.add.at.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace abd {

// ---------------------------------------------------------------------------
// sparsity pattern
__global__ void k_pattern_keys(int64_t n_ov, const int2* __restrict__ ov, int64_t n_f,
                               const int2* __restrict__ fb, const int* __restrict__ slot, int bS,
                               uint64_t* keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_ov + n_f) return;
  int2 p = i < n_ov ? ov[i] : fb[i - n_ov];
  int a = slot[p.x], b = slot[p.y];
  uint64_t k = ~0ull;
  if (a >= 0 && b >= 0 && a != b) k = ((uint64_t)min(a, b) << bS) | (uint64_t)max(a, b);
  keys[i] = k;
}

__global__ void k_row_counts(int n, int64_t n_off, const uint64_t* __restrict__ keys, int bS, int* cnt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) atomicAdd(cnt + i, 1);
  if (i < n_off) {
    uint64_t k = keys[i];
    atomicAdd(cnt + (int)(k >> bS), 1);
    atomicAdd(cnt + (int)(k & ((1ull << bS) - 1)), 1);
  }
}

// fill CSR columns: each row gets (lower cols ascending, diag, upper cols ascending)
// via per-row cursors after a global sort of (row, col) keys
__global__ void k_csr_entries(int n, int64_t n_off, const uint64_t* __restrict__ keys, int bS, uint64_t* ent) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) ent[i] = ((uint64_t)i << bS) | (uint64_t)i;
  if (i < n_off) {
    uint64_t k = keys[i];
    uint64_t r = k >> bS, c = k & ((1ull << bS) - 1);
    ent[n + 2 * i] = (r << bS) | c;
    ent[n + 2 * i + 1] = (c << bS) | r;
  }
}

__global__ void k_csr_cols(int64_t nnzb, const uint64_t* __restrict__ ent, int bS, int* col) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nnzb) col[i] = (int)(ent[i] & ((1ull << bS) - 1));
}

__device__ __forceinline__ int find_col(const int* __restrict__ row_ptr, const int* __restrict__ col, int r, int c) {
  int lo = row_ptr[r], hi = row_ptr[r + 1] - 1;
  while (lo <= hi) {
    int mid = (lo + hi) >> 1;
    int v = col[mid];
    if (v == c) return mid;
    if (v < c) lo = mid + 1;
    else hi = mid - 1;
  }
  return -1;
}

__global__ void k_csr_positions(int n, int64_t n_off, const uint64_t* __restrict__ keys, int bS,
                                const int* __restrict__ row_ptr, const int* __restrict__ col, int* diag_pos,
                                int* upper_pos, int* lower_pos, int2* upper_keys) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) diag_pos[i] = find_col(row_ptr, col, (int)i, (int)i);
  if (i < n_off) {
    uint64_t k = keys[i];
    int r = (int)(k >> bS), c = (int)(k & ((1ull << bS) - 1));
    upper_pos[i] = find_col(row_ptr, col, r, c);
    lower_pos[i] = find_col(row_ptr, col, c, r);
    upper_keys[i] = make_int2(r, c);
  }
}

// contributions: 3 per pair; key = target CSR position (or ~0 when absent)
// val = pair << 2 | which (0: haa/ga, 1: hbb/gb, 2: hab, 3: hab^T)
__global__ void k_contribs(int64_t np, const int2* __restrict__ bodies, const int* __restrict__ slot,
                           const int* __restrict__ diag_pos, int64_t n_off, const int2* __restrict__ upper_keys,
                           const int* __restrict__ upper_pos, uint32_t* keys, int* vals) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= np) return;
  int2 b = bodies[p];
  int sa = slot[b.x], sb = slot[b.y];
  uint32_t k0 = 0xffffffffu, k1 = 0xffffffffu, k2 = 0xffffffffu;
  int v2 = 0;
  if (sa >= 0) k0 = (uint32_t)diag_pos[sa];
  if (sb >= 0) k1 = (uint32_t)diag_pos[sb];
  if (sa >= 0 && sb >= 0 && sa != sb) {
    int lo = min(sa, sb), hi = max(sa, sb);
    // binary search the upper key list
    int64_t L = 0, R = n_off - 1, at = -1;
    while (L <= R) {
      int64_t m = (L + R) >> 1;
      int2 u = upper_keys[m];
      if (u.x == lo && u.y == hi) {
        at = m;
        break;
      }
      if (u.x < lo || (u.x == lo && u.y < hi)) L = m + 1;
      else R = m - 1;
    }
    if (at >= 0) {
      k2 = (uint32_t)upper_pos[at];
      v2 = sa < sb ? 2 : 3;
    }
  }
  keys[3 * p] = k0;
  vals[3 * p] = (int)(p << 2) | 0;
  keys[3 * p + 1] = k1;
  vals[3 * p + 1] = (int)(p << 2) | 1;
  keys[3 * p + 2] = k2;
  vals[3 * p + 2] = (int)(p << 2) | v2;
}

__global__ void k_seg_bounds(int64_t m, const uint32_t* __restrict__ keys, int64_t nnzb, int* start, int* end) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  uint32_t k = keys[i];
  if (k == 0xffffffffu) return;
  if (i == 0 || keys[i - 1] != k) start[k] = (int)i;
  if (i == m - 1 || keys[i + 1] != k) end[k] = (int)i + 1;
}

// one warp per CSR position that is a diagonal or an upper block
__global__ void k_reduce_blocks(int n, const int* __restrict__ row_ptr, const int* __restrict__ col,
                                const int* __restrict__ seg_start, const int* __restrict__ seg_end,
                                const int* __restrict__ cvals, const double* __restrict__ pblk,
                                const double* __restrict__ diag0, const double* __restrict__ grad0, double* val,
                                double* grad, const int* __restrict__ row_of) {
  int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nnzb = row_ptr[n];
  if (w >= nnzb) return;
  int r = row_of[w];
  int c = col[w];
  if (c < r) return;  // lower blocks are written by their upper twin
  bool is_diag = c == r;
  double acc[5];
  double gacc = 0.0;
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    int idx = lane + 32 * e;
    acc[e] = (is_diag && idx < 144) ? diag0[144 * (int64_t)r + idx] : 0.0;
  }
  if (is_diag && lane < 12) gacc = grad0[12 * (int64_t)r + lane];
  int s0 = seg_start[w], s1 = seg_end[w];
  for (int t = s0; t < s1; ++t) {
    int v = cvals[t];
    int64_t p = v >> 2;
    int which = v & 3;
    const double* blk = pblk + p * PB_STRIDE;
    const double* h = blk + 24 + 144 * (which == 0 ? 0 : (which == 1 ? 1 : 2));
#pragma unroll
    for (int e = 0; e < 5; ++e) {
      int idx = lane + 32 * e;
      if (idx < 144) {
        int src = which == 3 ? (idx % 12) * 12 + idx / 12 : idx;
        acc[e] += h[src];
      }
    }
    if (which < 2 && lane < 12) gacc += blk[12 * which + lane];
  }
  double* out = val + 144 * w;
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    int idx = lane + 32 * e;
    if (idx < 144) out[idx] = acc[e];
  }
  if (is_diag) {
    if (lane < 12) grad[12 * (int64_t)r + lane] = gacc;
  } else {
    int lw = find_col(row_ptr, col, c, r);
    double* o2 = val + 144 * (int64_t)lw;
#pragma unroll
    for (int e = 0; e < 5; ++e) {
      int idx = lane + 32 * e;
      if (idx < 144) o2[(idx % 12) * 12 + idx / 12] = acc[e];
    }
  }
}

__global__ void k_row_of(int n, const int* __restrict__ row_ptr, int* row_of) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k) row_of[k] = r;
}

// ---------------------------------------------------------------------------
// build pattern + CSR from overlap pairs and friction pairs (dyn-dyn only)
void build_pattern(Scene& s, const int2* ov, int64_t n_ov, const int2* fb, int64_t n_f) {
  Bsr& H = s.H;
  cudaStream_t st = s.stream;
  int n = s.n_dyn;
  H.n = n;
  int bS = bits_for(std::max(n - 1, 1));
  int64_t m = n_ov + n_f;
  DVec<uint64_t> k0, k1;
  k0.resize(std::max<int64_t>(m, 1));
  k1.resize(std::max<int64_t>(m, 1));
  int64_t n_off = 0;
  if (m > 0) {
    k_pattern_keys<<<grid_for(m, 256), 256, 0, st>>>(n_ov, ov, n_f, fb, s.slot.p, bS, k0.p);
    note_launch("k_pattern_keys");
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, k0.p, k1.p, (int)m, 0, 64, st));
    s.tmp_bytes.resize(bytes);
    CK(cub::DeviceRadixSort::SortKeys(s.tmp_bytes.p, bytes, k0.p, k1.p, (int)m, 0, 64, st));
    DVec<int> nsel;
    nsel.resize(1);
    bytes = 0;
    CK(cub::DeviceSelect::Unique(nullptr, bytes, k1.p, k0.p, nsel.p, (int)m, st));
    s.tmp_bytes.resize(bytes);
    CK(cub::DeviceSelect::Unique(s.tmp_bytes.p, bytes, k1.p, k0.p, nsel.p, (int)m, st));
    int hn = 0;
    CK(cudaMemcpyAsync(&hn, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // drop the ~0 sentinel (sorted last)
    uint64_t last = 0;
    if (hn > 0) {
      CK(cudaMemcpy(&last, k0.p + hn - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost));
      if (last == ~0ull) --hn;
    }
    n_off = hn;
  }
  H.n_off = n_off;
  H.nnzb = n + 2 * n_off;
  H.row_ptr.resize(n + 1);
  H.col.resize(std::max<int64_t>(H.nnzb, 1));
  H.val.resize(std::max<int64_t>(H.nnzb, 1) * 144);
  H.diag_pos.resize(std::max(n, 1));
  H.upper_keys.resize(std::max<int64_t>(n_off, 1));
  H.upper_pos.resize(std::max<int64_t>(n_off, 1));
  H.lower_pos.resize(std::max<int64_t>(n_off, 1));
  if (n == 0) return;
  DVec<int> cnt;
  cnt.resize(n + 1);
  cnt.zero(st);
  int64_t mx = std::max<int64_t>(n, n_off);
  k_row_counts<<<grid_for(mx, 256), 256, 0, st>>>(n, n_off, k0.p, bS, cnt.p);
  note_launch("k_row_counts");
  scan_exclusive_i32(s, cnt.p, H.row_ptr.p, n + 1);
  DVec<uint64_t> e0, e1;
  e0.resize(H.nnzb);
  e1.resize(H.nnzb);
  k_csr_entries<<<grid_for(mx, 256), 256, 0, st>>>(n, n_off, k0.p, bS, e0.p);
  note_launch("k_csr_entries");
  size_t bytes = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, e0.p, e1.p, (int)H.nnzb, 0, 2 * bS, st));
  s.tmp_bytes.resize(bytes);
  CK(cub::DeviceRadixSort::SortKeys(s.tmp_bytes.p, bytes, e0.p, e1.p, (int)H.nnzb, 0, 2 * bS, st));
  k_csr_cols<<<grid_for(H.nnzb, 256), 256, 0, st>>>(H.nnzb, e1.p, bS, H.col.p);
  note_launch("k_csr_cols");
  k_csr_positions<<<grid_for(mx, 256), 256, 0, st>>>(n, n_off, k0.p, bS, H.row_ptr.p, H.col.p, H.diag_pos.p,
                                                     H.upper_pos.p, H.lower_pos.p, H.upper_keys.p);
  note_launch("k_csr_positions");
}

// reduce resident pair blocks (s.pblk, n_pairs) + per-body diag0/grad0 into H, grad
void reduce_system(Scene& s, const double* diag0, const double* grad0) {
  Bsr& H = s.H;
  cudaStream_t st = s.stream;
  int n = H.n;
  if (n == 0) return;
  int64_t np = s.pblk.n;
  int64_t m = 3 * np;
  DVec<uint32_t> ka, kb;
  DVec<int> va, vb;
  ka.resize(std::max<int64_t>(m, 1));
  kb.resize(std::max<int64_t>(m, 1));
  va.resize(std::max<int64_t>(m, 1));
  vb.resize(std::max<int64_t>(m, 1));
  DVec<int> seg_s, seg_e, row_of;
  seg_s.resize(H.nnzb);
  seg_e.resize(H.nnzb);
  row_of.resize(H.nnzb);
  seg_s.zero(st);
  seg_e.zero(st);
  k_row_of<<<grid_for(n, 128), 128, 0, st>>>(n, H.row_ptr.p, row_of.p);
  note_launch("k_row_of");
  const int* cv = va.p;
  if (np > 0) {
    k_contribs<<<grid_for(np, 256), 256, 0, st>>>(np, s.pblk.bodies.p, s.slot.p, H.diag_pos.p, H.n_off,
                                                  H.upper_keys.p, H.upper_pos.p, ka.p, va.p);
    note_launch("k_contribs");
    cub::DoubleBuffer<uint32_t> dk(ka.p, kb.p);
    cub::DoubleBuffer<int> dv(va.p, vb.p);
    size_t bytes = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, (int)m, 0, 32, st));
    s.tmp_bytes.resize(bytes);
    CK(cub::DeviceRadixSort::SortPairs(s.tmp_bytes.p, bytes, dk, dv, (int)m, 0, 32, st));
    k_seg_bounds<<<grid_for(m, 256), 256, 0, st>>>(m, dk.Current(), H.nnzb, seg_s.p, seg_e.p);
    note_launch("k_seg_bounds");
    cv = dv.Current();
  }
  s.grad.resize(12 * (int64_t)n);
  k_reduce_blocks<<<grid_for(H.nnzb * 32, 256), 256, 0, st>>>(n, H.row_ptr.p, H.col.p, seg_s.p, seg_e.p, cv,
                                                              s.pblk.blk.p, diag0, grad0, H.val.p, s.grad.p,
                                                              row_of.p);
  note_launch("k_reduce_blocks");
  CK(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------------------
// block-Jacobi PCG
__global__ void k_jacobi_inv(int n, const int* __restrict__ diag_pos, const double* __restrict__ val, double* pinv,
                             int* bad) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double* D = val + 144 * (int64_t)diag_pos[r];
  double L[144];
  for (int i = 0; i < 12; ++i)
    for (int j = 0; j < 12; ++j) L[i * 12 + j] = 0.5 * (D[i * 12 + j] + D[j * 12 + i]);
  for (int j = 0; j < 12; ++j) {
    double d = L[j * 12 + j];
    for (int k = 0; k < j; ++k) d -= L[j * 12 + k] * L[j * 12 + k];
    if (!(d > 0.0)) {
      atomicMin(bad, r);
      return;
    }
    d = sqrt(d);
    L[j * 12 + j] = d;
    for (int i = j + 1; i < 12; ++i) {
      double v = L[i * 12 + j];
      for (int k = 0; k < j; ++k) v -= L[i * 12 + k] * L[j * 12 + k];
      L[i * 12 + j] = v / d;
    }
  }
  // inverse = L^-T L^-1, column by column
  double* P = pinv + 144 * (int64_t)r;
  for (int c = 0; c < 12; ++c) {
    double y[12];
    for (int i = 0; i < 12; ++i) {
      double v = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) v -= L[i * 12 + k] * y[k];
      y[i] = v / L[i * 12 + i];
    }
    for (int i = 11; i >= 0; --i) {
      double v = y[i];
      for (int k = i + 1; k < 12; ++k) v -= L[k * 12 + i] * y[k];
      y[i] = v / L[i * 12 + i];
    }
    for (int i = 0; i < 12; ++i) P[i * 12 + c] = y[i];
  }
}

struct PcgArgs {
  int n;
  const int* row_ptr;
  const int* col;
  const double* val;
  const double* pinv;
  const double* b;
  double* x;
  double* r;
  double* z;
  double* p;
  double* Ap;
  double* partials;  // 3 * gridDim.x
  double rel_tol;
  int max_iters;
  int* out_iters;
  double* out_rel;
};

__device__ __forceinline__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

// all blocks sum the per-block partials in the same fixed order
__device__ __forceinline__ double grid_total(const double* part, int stride_off, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v += part[3 * i + stride_off];
  return block_sum(v, sh);
}

// y = A x for scalar row t = 12 * block_row + rr
__device__ __forceinline__ double spmv_row(const PcgArgs& a, int br, int rr, const double* x) {
  double acc = 0.0;
  for (int k = a.row_ptr[br]; k < a.row_ptr[br + 1]; ++k) {
    const double* blk = a.val + 144 * (int64_t)k + 12 * rr;
    const double* xv = x + 12 * (int64_t)a.col[k];
#pragma unroll
    for (int c = 0; c < 12; ++c) acc += blk[c] * xv[c];
  }
  return acc;
}

__device__ __forceinline__ double prec_row(const PcgArgs& a, int br, int rr, const double* r) {
  const double* P = a.pinv + 144 * (int64_t)br + 12 * rr;
  const double* rv = r + 12 * (int64_t)br;
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 12; ++c) acc += P[c] * rv[c];
  return acc;
}

__global__ void k_pcg(PcgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[33];
  const int64_t N = 12 * (int64_t)a.n;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  // x = 0, r = b, |b|^2
  double bb = 0.0;
  for (int64_t t = tid; t < N; t += nth) {
    a.x[t] = 0.0;
    a.r[t] = a.b[t];
    bb += a.b[t] * a.b[t];
  }
  bb = block_sum(bb, sh);
  if (threadIdx.x == 0) a.partials[3 * blockIdx.x] = bb;
  grid.sync();
  double bnorm = sqrt(grid_total(a.partials, 0, sh));
  if (bnorm == 0.0) {
    if (tid == 0) {
      *a.out_iters = 0;
      *a.out_rel = 0.0;
    }
    return;
  }
  const double tol = a.rel_tol * bnorm;
  int it = 0;
  double rel = 1.0;
  bool done = false;
  for (int restart = 0; restart < 4 && !done; ++restart) {
    // z = P r, p = z, rz
    double rz = 0.0;
    for (int64_t t = tid; t < N; t += nth) {
      double zt = prec_row(a, (int)(t / 12), (int)(t % 12), a.r);
      a.z[t] = zt;
      a.p[t] = zt;
      rz += a.r[t] * zt;
    }
    rz = block_sum(rz, sh);
    grid.sync();  // partials slot 0 reuse after everyone read |b|
    if (threadIdx.x == 0) a.partials[3 * blockIdx.x + 1] = rz;
    grid.sync();
    rz = grid_total(a.partials, 1, sh);
    while (it < a.max_iters) {
      // Ap and p.Ap
      double pap = 0.0;
      for (int64_t t = tid; t < N; t += nth) {
        double v = spmv_row(a, (int)(t / 12), (int)(t % 12), a.p);
        a.Ap[t] = v;
        pap += a.p[t] * v;
      }
      pap = block_sum(pap, sh);
      if (threadIdx.x == 0) a.partials[3 * blockIdx.x] = pap;
      grid.sync();
      pap = grid_total(a.partials, 0, sh);
      double alpha = rz / pap;
      double rr = 0.0;
      for (int64_t t = tid; t < N; t += nth) {
        a.x[t] += alpha * a.p[t];
        double rt = a.r[t] - alpha * a.Ap[t];
        a.r[t] = rt;
        rr += rt * rt;
      }
      // z needs the full r of its own block row only (threads t..t+11 of a row may
      // live in different CTAs), so sync before applying the preconditioner
      rr = block_sum(rr, sh);
      if (threadIdx.x == 0) a.partials[3 * blockIdx.x + 2] = rr;
      grid.sync();
      double rn = sqrt(grid_total(a.partials, 2, sh));
      ++it;
      rel = rn / bnorm;
      if (rn <= tol || !(pap > 0.0)) break;
      double rz_new = 0.0;
      for (int64_t t = tid; t < N; t += nth) {
        double zt = prec_row(a, (int)(t / 12), (int)(t % 12), a.r);
        a.z[t] = zt;
        rz_new += a.r[t] * zt;
      }
      rz_new = block_sum(rz_new, sh);
      if (threadIdx.x == 0) a.partials[3 * blockIdx.x + 1] = rz_new;
      grid.sync();
      rz_new = grid_total(a.partials, 1, sh);
      double beta = rz_new / rz;
      rz = rz_new;
      for (int64_t t = tid; t < N; t += nth) a.p[t] = a.z[t] + beta * a.p[t];
      grid.sync();
    }
    // true residual r = b - A x
    grid.sync();
    double tr = 0.0;
    for (int64_t t = tid; t < N; t += nth) {
      double v = a.b[t] - spmv_row(a, (int)(t / 12), (int)(t % 12), a.x);
      a.r[t] = v;
      tr += v * v;
    }
    tr = block_sum(tr, sh);
    if (threadIdx.x == 0) a.partials[3 * blockIdx.x + 2] = tr;
    grid.sync();
    double trn = sqrt(grid_total(a.partials, 2, sh));
    rel = trn / bnorm;
    if (trn <= tol || it >= a.max_iters) done = true;
    grid.sync();
  }
  if (tid == 0) {
    *a.out_iters = it;
    *a.out_rel = rel;
  }
}

// solve H x = rhs on the resident BSR; returns iterations, rel residual
int pcg_solve(Scene& s, const double* rhs, double* x, double rel_tol, int max_iters, double& rel_res) {
  Bsr& H = s.H;
  cudaStream_t st = s.stream;
  int n = H.n;
  if (n == 0) {
    rel_res = 0.0;
    return 0;
  }
  int64_t N = 12 * (int64_t)n;
  DVec<double> pinv, r, z, p, Ap, part;
  pinv.resize(144 * (int64_t)n);
  r.resize(N);
  z.resize(N);
  p.resize(N);
  Ap.resize(N);
  DVec<int> bad, iters;
  DVec<double> rel;
  bad.resize(1);
  iters.resize(1);
  rel.resize(1);
  int big = 0x7fffffff;
  CK(cudaMemcpyAsync(bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  k_jacobi_inv<<<grid_for(n, 64), 64, 0, st>>>(n, H.diag_pos.p, H.val.p, pinv.p, bad.p);
  note_launch("k_jacobi_inv");
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hbad != big) throw Error(ABD_ERR_FACTORIZATION, "non-SPD diagonal block in block-Jacobi PCG", hbad);
  static int blocks_per_sm = -1;
  const int threads = 256;
  if (blocks_per_sm < 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_pcg, threads, 0));
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  int64_t want = grid_for(N, threads);
  int grid = (int)std::min<int64_t>(want, (int64_t)blocks_per_sm * s.num_sms);
  if (grid < 1) grid = 1;
  part.resize(3 * (int64_t)grid);
  PcgArgs a;
  a.n = n;
  a.row_ptr = H.row_ptr.p;
  a.col = H.col.p;
  a.val = H.val.p;
  a.pinv = pinv.p;
  a.b = rhs;
  a.x = x;
  a.r = r.p;
  a.z = z.p;
  a.p = p.p;
  a.Ap = Ap.p;
  a.partials = part.p;
  a.rel_tol = rel_tol;
  a.max_iters = max_iters;
  a.out_iters = iters.p;
  a.out_rel = rel.p;
  void* args[] = {&a};
  CK(cudaLaunchCooperativeKernel((void*)k_pcg, dim3(grid), dim3(threads), args, 0, st));
  note_launch("k_pcg");
  int hit = 0;
  CK(cudaMemcpyAsync(&hit, iters.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&rel_res, rel.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return hit;
}

// y = H x on the resident BSR (thread per scalar row)
__global__ void k_spmv(int n, const int* __restrict__ row_ptr, const int* __restrict__ col,
                       const double* __restrict__ val, const double* __restrict__ x, double* y) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 12 * (int64_t)n) return;
  int br = (int)(t / 12), rr = (int)(t % 12);
  double acc = 0.0;
  for (int k = row_ptr[br]; k < row_ptr[br + 1]; ++k) {
    const double* blk = val + 144 * (int64_t)k + 12 * rr;
    const double* xv = x + 12 * (int64_t)col[k];
    for (int c = 0; c < 12; ++c) acc += blk[c] * xv[c];
  }
  y[t] = acc;
}

void spmv(Scene& s, const double* x, double* y) {
  int64_t N = 12 * (int64_t)s.H.n;
  if (!N) return;
  k_spmv<<<grid_for(N, 256), 256, 0, s.stream>>>(s.H.n, s.H.row_ptr.p, s.H.col.p, s.H.val.p, x, y);
  note_launch("k_spmv");
}

}  // namespace abd

namespace abd {

// stateless BSR (sparse.py BlockSparseMatrix with block_dim <= 12, padded to 12)
__global__ void k_fill_bsr(int n, int bdim, const double* __restrict__ diag, int64_t n_off,
                           const int64_t* __restrict__ keys, const double* __restrict__ off,
                           const int* __restrict__ row_ptr, const int* __restrict__ col, double* val) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t nb = n + n_off;
  if (t >= nb * 144) return;
  int64_t b = t / 144;
  int e = (int)(t % 144), r = e / 12, c = e % 12;
  int bb = bdim * bdim;
  if (b < n) {
    double v = (r < bdim && c < bdim) ? diag[b * bb + r * bdim + c] : (r == c ? 1.0 : 0.0);
    val[144 * (int64_t)find_col(row_ptr, col, (int)b, (int)b) + e] = v;
  } else {
    int64_t k = b - n;
    int i = (int)keys[2 * k], j = (int)keys[2 * k + 1];
    double v = (r < bdim && c < bdim) ? off[k * bb + r * bdim + c] : 0.0;
    val[144 * (int64_t)find_col(row_ptr, col, i, j) + e] = v;
    val[144 * (int64_t)find_col(row_ptr, col, j, i) + c * 12 + r] = v;
  }
}

void load_bsr(Scene& s, int n, int bdim, const double* diag, int64_t n_off, const int64_t* keys, const double* off) {
  cudaStream_t st = s.stream;
  if (s.B != n) {
    s.B = n;
    s.n_dyn = n;
    std::vector<int> id(std::max(n, 1));
    for (int i = 0; i < n; ++i) id[i] = i;
    s.slot.upload(id.data(), std::max(n, 1), st);
    s.dyn_body.upload(id.data(), std::max(n, 1), st);
  }
  std::vector<int2> kv(std::max<int64_t>(n_off, 1));
  for (int64_t k = 0; k < n_off; ++k) {
    int i = (int)keys[2 * k], j = (int)keys[2 * k + 1];
    if (i == j || i < 0 || j < 0 || i >= n || j >= n) throw Error(ABD_ERR_ARG, "bad off-diagonal key");
    kv[k] = make_int2(i, j);
  }
  DVec<int2> dk;
  dk.upload(kv.data(), kv.size(), st);
  build_pattern(s, dk.p, n_off, nullptr, 0);
  if (n == 0) return;
  DVec<double> dd, doff;
  DVec<int64_t> dkeys;
  dd.upload(diag, (size_t)n * bdim * bdim, st);
  doff.upload(off, std::max<size_t>((size_t)n_off * bdim * bdim, 1), st);
  dkeys.upload(keys, std::max<size_t>(2 * (size_t)n_off, 1), st);
  int64_t tot = (n + n_off) * 144;
  k_fill_bsr<<<grid_for(tot, 256), 256, 0, st>>>(n, bdim, dd.p, n_off, dkeys.p, doff.p, s.H.row_ptr.p, s.H.col.p,
                                                s.H.val.p);
  note_launch("k_fill_bsr");
  CK(cudaStreamSynchronize(st));
}

}  // namespace abd
