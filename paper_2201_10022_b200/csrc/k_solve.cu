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

#include "driver.h"
#include "kernels.h"
#include "abd_pblk.cuh"

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
                           const int* __restrict__ upper_pos, uint32_t* keys, int* vals, int* cnt,
                           int64_t val_off = 0) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= np) return;
  int2 b = bodies[p];
  // (-1, -1): a pair folded into a run partial (k_pair_runs), no contribution of its own
  int sa = b.x >= 0 ? slot[b.x] : -1, sb = b.y >= 0 ? slot[b.y] : -1;
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
  const int64_t pv = p + val_off;  // run partials follow the records in value order
  keys[3 * p] = k0;
  vals[3 * p] = (int)(pv << 2) | 0;
  keys[3 * p + 1] = k1;
  vals[3 * p + 1] = (int)(pv << 2) | 1;
  keys[3 * p + 2] = k2;
  vals[3 * p + 2] = (int)(pv << 2) | v2;
  if (cnt) {
    if (k0 != 0xffffffffu) atomicAdd(cnt + k0, 1);
    if (k1 != 0xffffffffu) atomicAdd(cnt + k1, 1);
    if (k2 != 0xffffffffu) atomicAdd(cnt + k2, 1);
  }
}

// contributions into their block segments (unordered within a segment; the
// reduction orders each segment by value = pair-major, as the stable sort did)
__global__ void k_contrib_fill(int64_t m, const uint32_t* __restrict__ keys, const int* __restrict__ vals,
                               const int* __restrict__ seg, int* fill, int* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint32_t k = keys[i];
  if (k == 0xffffffffu) return;
  out[seg[k] + atomicAdd(fill + k, 1)] = vals[i];
}

__global__ void k_seg_bounds(int64_t m, const uint32_t* __restrict__ keys, int64_t nnzb, int* start, int* end) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  uint32_t k = keys[i];
  if (k == 0xffffffffu) return;
  if (i == 0 || keys[i - 1] != k) start[k] = (int)i;
  if (i == m - 1 || keys[i + 1] != k) end[k] = (int)i + 1;
}

// one warp per CSR position that is a diagonal or an upper block; each
// contribution's compact record (PB_STRIDE doubles) is staged in shared memory
// by one coalesced warp load (the next record prefetched into registers while the
// current one is evaluated), so the ~60 per-entry reads hit shared memory
constexpr int RB_WARPS = 8;
constexpr int RB_SPLIT = 4;  // warps per BSR block: the contributions are dealt round-robin
constexpr int RB_POS = RB_WARPS / RB_SPLIT;  // BSR blocks per CTA
constexpr int RB_PER_LANE = (PB_STRIDE + 31) / 32;
// RB_SPLIT warps per CSR position that is a diagonal or an upper block; warp s sums
// the contributions s, s + RB_SPLIT, ... of the block's segment (each record staged
// in shared memory by one coalesced warp load, the next one prefetched), then the
// partial blocks are added in warp order: a fixed, deterministic summation order
// with a quarter of the serial chain of one warp per block
__global__ void __launch_bounds__(32 * RB_WARPS) k_reduce_blocks(int n, const int* __restrict__ row_ptr,
                                                                 const int* __restrict__ col,
                                                                 const int* __restrict__ seg_start,
                                                                 const int* __restrict__ seg_end,
                                                                 const int* cvals,
                                                                 const double* __restrict__ pblk,
                                                                 const double* __restrict__ diag0,
                                                                 const double* __restrict__ grad0, double* val,
                                                                 double* grad, const int* __restrict__ row_of,
                                                                 int* sorted_out, int64_t n_rec,
                                                                 const double* __restrict__ run_part,
                                                                 double* neg_out) {
  __shared__ double srec[RB_WARPS][RB_PER_LANE * 32];
  __shared__ double part[RB_WARPS][160];
  __shared__ double gpart[RB_WARPS][12];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int split = wid % RB_SPLIT;
  const int64_t w = (int64_t)blockIdx.x * RB_POS + wid / RB_SPLIT;
  const int64_t nnzb = row_ptr[n];
  int r = 0, c = -1;
  if (w < nnzb) {
    r = row_of[w];
    c = col[w];
  }
  const bool active = w < nnzb && c >= r;  // lower blocks are written by their upper twin
  const bool is_diag = c == r;
  const int s0 = active ? seg_start[w] : 0, s1 = active ? seg_end[w] : 0;
  if (sorted_out && active && split == 0) {
    // rank sort of the segment by value (unique): pair-major order
    for (int i = s0 + lane; i < s1; i += 32) {
      const int vi = cvals[i];
      int rk = 0;
      for (int j = s0; j < s1; ++j) rk += cvals[j] < vi;
      sorted_out[s0 + rk] = vi;
    }
  }
  __syncthreads();
  const int* cv = sorted_out ? sorted_out : cvals;
  double acc[5];
  double gacc = 0.0;
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    int idx = lane + 32 * e;
    acc[e] = (active && split == 0 && is_diag && idx < 144) ? diag0[144 * (int64_t)r + idx] : 0.0;
  }
  if (active && split == 0 && is_diag && lane < 12) gacc = grad0[12 * (int64_t)r + lane];
  double* sr = srec[wid];
  double nxt[RB_PER_LANE];
  int vnext = 0;
  // contributions v >> 2 < n_rec are compact records (staged, next one prefetched);
  // the others are dense run partials (aa | bb | ab | ga | gb, RUN_STRIDE doubles)
  auto prefetch = [&](int v) {
    if ((int64_t)(v >> 2) >= n_rec) return;
    const double* blk = pblk + (int64_t)(v >> 2) * PB_STRIDE;
#pragma unroll
    for (int j = 0; j < RB_PER_LANE; ++j)
      if (lane + 32 * j < PB_STRIDE) nxt[j] = blk[lane + 32 * j];
  };
  if (s0 + split < s1) {
    vnext = cv[s0 + split];
    prefetch(vnext);
  }
  for (int t = s0 + split; t < s1; t += RB_SPLIT) {
    const int which = vnext & 3;
    const int64_t src = vnext >> 2;
    if (src >= n_rec) {  // dense run partial
      const double* P = run_part + (src - n_rec) * RUN_STRIDE;
      if (t + RB_SPLIT < s1) {
        vnext = cv[t + RB_SPLIT];
        prefetch(vnext);
      }
#pragma unroll
      for (int e = 0; e < 5; ++e) {
        int idx = lane + 32 * e;
        if (idx < 144) {
          const int i = idx / 12, k = idx % 12;
          acc[e] += which == 3 ? P[288 + 12 * k + i] : P[144 * which + idx];
        }
      }
      if (which < 2 && lane < 12) gacc += P[432 + 12 * which + lane];
      continue;
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < RB_PER_LANE; ++j)
      if (lane + 32 * j < PB_STRIDE) sr[lane + 32 * j] = nxt[j];
    __syncwarp();
    if (t + RB_SPLIT < s1) {
      vnext = cv[t + RB_SPLIT];
      prefetch(vnext);
    }
    // target entry (i, k) = H24(12 s_r + i, 12 s_c + k) for the aa / bb / ab blocks;
    // which 3 is the transposed ab block: H24(k, 12 + i)
#pragma unroll
    for (int e = 0; e < 5; ++e) {
      int idx = lane + 32 * e;
      if (idx < 144) {
        const int i = idx / 12, k = idx % 12;
        const int R = which == 3 ? k : 12 * (which == 1) + i;
        const int Cc = which == 3 ? 12 + i : 12 * (which >= 1) + k;
        acc[e] += pb_entry(sr, R, Cc);
      }
    }
    if (which < 2 && lane < 12) gacc += sr[12 * which + lane];
  }
#pragma unroll
  for (int e = 0; e < 5; ++e) part[wid][lane + 32 * e] = acc[e];
  if (lane < 12) gpart[wid][lane] = gacc;
  __syncthreads();
  if (!active || split != 0) return;
#pragma unroll
  for (int e = 0; e < 5; ++e)
    for (int sp = 1; sp < RB_SPLIT; ++sp) acc[e] += part[wid + sp][lane + 32 * e];
  if (lane < 12)
    for (int sp = 1; sp < RB_SPLIT; ++sp) gacc += gpart[wid + sp][lane];
  double* out = val + 144 * w;
#pragma unroll
  for (int e = 0; e < 5; ++e) {
    int idx = lane + 32 * e;
    if (idx < 144) out[idx] = acc[e];
  }
  if (is_diag) {
    if (lane < 12) {
      grad[12 * (int64_t)r + lane] = gacc;
      if (neg_out) neg_out[12 * (int64_t)r + lane] = -gacc;  // the Newton right-hand side (saves k_neg)
    }
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

__global__ void k_drop_sentinel(const uint64_t* keys, int* n) {
  int m = n[0];
  if (m > 0 && keys[m - 1] == ~0ull) n[0] = m - 1;
}

__global__ void k_row_of(int n, const int* __restrict__ row_ptr, int* row_of) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k) row_of[k] = r;
}

// ---------------------------------------------------------------------------
// build pattern + CSR from overlap pairs and friction pairs (dyn-dyn only)
void build_pattern(Scene& s, const int2* ov, int64_t n_ov, const int2* fb, int64_t n_f, bool from_cands) {
  Bsr& H = s.H;
  Scene::Work& wk = s.w;
  // overlap pairs all inside the resident pattern and the same friction set: the
  // pattern (row_ptr, col, positions) is reused -- no sorts, no host sync
  if (from_cands && wk.pat_valid && s.cands.ov_matches_pattern && wk.pat_n_f == n_f &&
      wk.pat_fric_gen == s.fric.gen && H.n == s.n_dyn)
    return;
  chol_analysis_drop(s);  // an analysis in flight belongs to the old pattern
  s.w.ch_pre = false;  // any structure copied out for the Cholesky belongs to the old pattern
  s.w.ch_early = false;
  s.w.ch_verify = false;
  wk.pat_valid = false;
  cudaStream_t st = s.stream;
  int n = s.n_dyn;
  H.n = n;
  int bS = bits_for(std::max(n - 1, 1));
  int64_t m = n_ov + n_f;
  DVec<uint64_t>& k0 = s.w.k0;
  DVec<uint64_t>& k1 = s.w.k1;
  k0.resize(std::max<int64_t>(m, 1));
  k1.resize(std::max<int64_t>(m, 1));
  int64_t n_off = 0;
  if (m > 0) {
    k_pattern_keys<<<grid_for(m, 256), 256, 0, st>>>(n_ov, ov, n_f, fb, s.slot.p, bS, k0.p);
    note_launch("k_pattern_keys");
    size_t bytes = 0;
    // valid keys use 2 bS bits; the ~0 sentinel's low bits are all ones so it sorts last
    CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, k0.p, k1.p, (int)m, 0, 2 * bS + 1, st));
    s.tmp_bytes.resize(bytes);
    CK(cub::DeviceRadixSort::SortKeys(s.tmp_bytes.p, bytes, k0.p, k1.p, (int)m, 0, 2 * bS + 1, st));
    DVec<int>& nsel = s.w.nsel;
    nsel.resize(2);
    bytes = 0;
    CK(cub::DeviceSelect::Unique(nullptr, bytes, k1.p, k0.p, nsel.p, (int)m, st));
    s.tmp_bytes.resize(bytes);
    CK(cub::DeviceSelect::Unique(s.tmp_bytes.p, bytes, k1.p, k0.p, nsel.p, (int)m, st));
    k_drop_sentinel<<<1, 1, 0, st>>>(k0.p, nsel.p);  // the ~0 sentinel sorts last
    note_launch("k_drop_sentinel");
    int hn = 0;
    CK(cudaMemcpyAsync(&hn, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    SSYNC(st);
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
  DVec<int>& cnt = s.w.cnt;
  cnt.resize(n + 1);
  cnt.zero(st);
  int64_t mx = std::max<int64_t>(n, n_off);
  k_row_counts<<<grid_for(mx, 256), 256, 0, st>>>(n, n_off, k0.p, bS, cnt.p);
  note_launch("k_row_counts");
  scan_exclusive_i32(s, cnt.p, H.row_ptr.p, n + 1);
  DVec<uint64_t>& e0 = s.w.e0;
  DVec<uint64_t>& e1 = s.w.e1;
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
  if (from_cands) {
    wk.pat_n_ov = n_ov;
    wk.pat_n_f = n_f;
    wk.pat_fric_gen = s.fric.gen;
    wk.pat_valid = true;
    s.cands.ov_matches_pattern = true;
  }
}

// reduce resident pair blocks (s.pblk, n_pairs) + per-body diag0/grad0 into H, grad
void reduce_system(Scene& s, const double* diag0, const double* grad0, double* neg_out) {
  Bsr& H = s.H;
  cudaStream_t st = s.stream;
  int n = H.n;
  if (n == 0) return;
  int64_t np = s.pblk.n;
  const int64_t nr = s.pblk.n_runs;  // dense run partials (k_pair_runs), after the records
  int64_t m = 3 * (np + nr);
  DVec<uint32_t>& ka = s.w.ka;
  DVec<uint32_t>& kb = s.w.kb;
  DVec<int>& va = s.w.va;
  DVec<int>& vb = s.w.vb;
  ka.resize(std::max<int64_t>(m, 1));
  kb.resize(std::max<int64_t>(m, 1));
  va.resize(std::max<int64_t>(m, 1));
  vb.resize(std::max<int64_t>(m, 1));
  DVec<int>& seg_s = s.w.seg_s;
  DVec<int>& seg_e = s.w.seg_e;
  DVec<int>& row_of = s.w.row_of;
  static const bool sort_path = getenv("ABD_CONTRIB_SORT") != nullptr;
  seg_s.resize(H.nnzb + 1);
  seg_e.resize(H.nnzb + 1);
  row_of.resize(H.nnzb);
  k_row_of<<<grid_for(n, 128), 128, 0, st>>>(n, H.row_ptr.p, row_of.p);
  note_launch("k_row_of");
  const int* cv = va.p;
  const int* sb = seg_s.p;
  const int* se = seg_e.p;
  int* sorted_out = nullptr;
  if (sort_path || np + nr == 0) {
    seg_s.zero(st);
    seg_e.zero(st);
  }
  if (nr > 0 && sort_path) throw Error(ABD_ERR_ARG, "ABD_CONTRIB_SORT does not take run partials");
  if (np > 0 && sort_path) {
    k_contribs<<<grid_for(np, 256), 256, 0, st>>>(np, s.pblk.bodies.p, s.slot.p, H.diag_pos.p, H.n_off,
                                                  H.upper_keys.p, H.upper_pos.p, ka.p, va.p, nullptr);
    note_launch("k_contribs");
    int kb_bits = bits_for(H.nnzb) + 1;  // the 0xffffffff "absent" key still sorts last
    if (kb_bits > 32) kb_bits = 32;
    bool alt = false;
    sort_pairs_u32(s, ka.p, kb.p, va.p, vb.p, m, kb_bits, alt);
    k_seg_bounds<<<grid_for(m, 256), 256, 0, st>>>(m, alt ? kb.p : ka.p, H.nnzb, seg_s.p, seg_e.p);
    note_launch("k_seg_bounds");
    cv = alt ? vb.p : va.p;
  } else if (np + nr > 0) {
    // counting placement: per-block counts, exclusive scan (segment starts), fill;
    // the reduction rank-sorts each (short) segment
    DVec<int>& cnt = s.w.cnt;
    cnt.resize(H.nnzb + 1);
    cnt.zero(st);
    if (np > 0) {
      k_contribs<<<grid_for(np, 256), 256, 0, st>>>(np, s.pblk.bodies.p, s.slot.p, H.diag_pos.p, H.n_off,
                                                    H.upper_keys.p, H.upper_pos.p, ka.p, va.p, cnt.p);
      note_launch("k_contribs");
    }
    if (nr > 0) {
      k_contribs<<<grid_for(nr, 256), 256, 0, st>>>(nr, s.pblk.run_bodies.p, s.slot.p, H.diag_pos.p, H.n_off,
                                                    H.upper_keys.p, H.upper_pos.p, ka.p + 3 * np, va.p + 3 * np,
                                                    cnt.p, np);
      note_launch("k_contribs");
    }
    scan_exclusive_i32(s, cnt.p, seg_s.p, H.nnzb + 1);
    cnt.zero(st);
    k_contrib_fill<<<grid_for(m, 256), 256, 0, st>>>(m, ka.p, va.p, seg_s.p, cnt.p, vb.p);
    note_launch("k_contrib_fill");
    cv = vb.p;
    sorted_out = va.p;  // keys/vals of the contributions are dead after the fill
    sb = seg_s.p;
    se = seg_s.p + 1;
  }
  s.grad.resize(12 * (int64_t)n);
  k_reduce_blocks<<<grid_for(H.nnzb, RB_POS), 32 * RB_WARPS, 0, st>>>(n, H.row_ptr.p, H.col.p, sb, se, cv,
                                                              s.pblk.blk.p, diag0, grad0, H.val.p, s.grad.p,
                                                              row_of.p, sorted_out, np, s.pblk.run_part.p, neg_out);
  note_launch("k_reduce_blocks");
}


}  // namespace abd
