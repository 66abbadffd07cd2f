// Block-Jacobi preconditioner setup for K4 (the PCG itself is k_cg.cu), the
// standalone BSR SpMV (BlockSparseMatrix.matvec, sparse.py:77-84) and the
// stateless BSR loader used by the sparse.py drop-in.
#include <algorithm>
#include <vector>

#include "driver.h"

namespace abd {

// block-Jacobi preconditioner: inverse of each 12x12 diagonal block.  16 lanes
// per block (two blocks per warp): right-looking Cholesky with lane t owning
// row t in shared memory, then lane t solves column t of the inverse.
constexpr int JI_BLOCKS = 8;  // blocks per CTA (128 threads)
__global__ void __launch_bounds__(128) k_jacobi_inv(int n, const int* __restrict__ diag_pos,
                                                     const double* __restrict__ val, double* pinv, int* bad) {
  __shared__ double Ls[JI_BLOCKS][12][13];
  const int lb = threadIdx.x >> 4, t = threadIdx.x & 15;
  const int r = blockIdx.x * JI_BLOCKS + lb;
  const bool live = r < n;
  double (*L)[13] = Ls[lb];
  if (live && t < 12) {
    const double* D = val + 144 * (int64_t)diag_pos[r];
    for (int j = 0; j < 12; ++j) L[t][j] = 0.5 * (D[t * 12 + j] + D[j * 12 + t]);
  }
  __syncwarp();
  bool ok = true;
  for (int j = 0; j < 12; ++j) {
    double d = live ? L[j][j] : 1.0;
    ok = ok && (d > 0.0);
    double sd = sqrt(fmax(d, 1e-300));
    __syncwarp();
    if (live && t > j && t < 12) L[t][j] /= sd;
    if (live && t == j) L[j][j] = sd;
    __syncwarp();
    if (live && t > j && t < 12) {
      double ltj = L[t][j];
      for (int k = j + 1; k <= t; ++k) L[t][k] -= ltj * L[k][j];
    }
    __syncwarp();
  }
  if (!live) return;
  if (!ok) {
    if (t == 0) atomicMin(bad, r);
    return;
  }
  if (t >= 12) return;
  // column t of L^-T L^-1
  double y[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    double v = (i == t) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) v -= L[i][k] * y[k];
    y[i] = v / L[i][i];
  }
#pragma unroll
  for (int i = 11; i >= 0; --i) {
    double v = y[i];
#pragma unroll
    for (int k = i + 1; k < 12; ++k) v -= L[k][i] * y[k];
    y[i] = v / L[i][i];
  }
  double* P = pinv + 144 * (int64_t)r;
#pragma unroll
  for (int i = 0; i < 12; ++i) P[i * 12 + t] = y[i];
}


void launch_jacobi_inv(Scene& s, int n, const int* diag_pos, const double* val, double* pinv, int* bad) {
  k_jacobi_inv<<<grid_for(n, JI_BLOCKS), 128, 0, s.stream>>>(n, diag_pos, val, pinv, bad);
  note_launch("k_jacobi_inv");
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

// ---------------------------------------------------------------------------
// stateless BSR (sparse.py BlockSparseMatrix with block_dim <= 12, padded to 12)
__device__ __forceinline__ int find_col2(const int* __restrict__ row_ptr, const int* __restrict__ col, int r, int c) {
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
    val[144 * (int64_t)find_col2(row_ptr, col, (int)b, (int)b) + e] = v;
  } else {
    int64_t k = b - n;
    int i = (int)keys[2 * k], j = (int)keys[2 * k + 1];
    double v = (r < bdim && c < bdim) ? off[k * bb + r * bdim + c] : 0.0;
    val[144 * (int64_t)find_col2(row_ptr, col, i, j) + e] = v;
    val[144 * (int64_t)find_col2(row_ptr, col, j, i) + c * 12 + r] = v;
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
  s.w.pairs_tmp.upload(kv.data(), kv.size(), st);
  build_pattern(s, s.w.pairs_tmp.p, n_off, nullptr, 0);
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
  SSYNC(st);
}

}  // namespace abd
