// K4: block-Jacobi PCG on the resident symmetric BSR (replaces the reference's
// BlockCholesky.solve_refined, sparse.py:90-161, to the same ||Ax-b|| <=
// rel_tol ||b|| contract).
//
// One persistent cooperative launch per solve.  Each CTA owns whole block
// rows (16 block rows x 12 scalar rows = 192 threads), so the 12x12
// block-Jacobi apply needs only __syncthreads, and an iteration costs two
// grid-wide reductions:
//   phase A: p_new = z + beta p_old fused into the SpMV gather (double-
//            buffered p), Ap = A p_new, partial p_new.Ap        -> grid sync
//   phase B: x += alpha p, r -= alpha Ap, z = P^-1 r,
//            partials r.z and r.r                              -> grid sync
// Dot products are reduced in a fixed order by every CTA (deterministic).
// On convergence of the recursive residual the true residual b - A x is
// checked and CG restarts from x if it fails.
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "driver.h"

namespace cg = cooperative_groups;

namespace abd {

constexpr int PCG_ROWS = 16;               // block rows per CTA
constexpr int PCG_THREADS = PCG_ROWS * 12;  // 192

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

struct PcgArgs {
  int n;
  const int* row_ptr;
  const int* col;
  const double* val;
  const double* pinv;
  const int* bad;
  const double* b;
  double* x;
  double* r;
  double* z;
  double* pa;
  double* pb;
  double* Ap;
  double* part;  // 4 * gridDim.x: two alternating (A | B) banks of 2 values per CTA
  double rel_tol;
  int max_iters;
  int* out_iters;
  double* out_rel;
};

__device__ __forceinline__ double cta_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < PCG_THREADS / 32; ++w) t += sh[w];
  return t;
}

// every CTA reduces the per-CTA partials in the same fixed order
__device__ __forceinline__ double grid_total(const double* part, int which, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v += part[2 * i + which];
  return cta_sum(v, sh);
}

__device__ __forceinline__ void cta_sum2(double& a, double& b, double* sh) {
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    sh[wid] = a;
    sh[8 + wid] = b;
  }
  __syncthreads();
  double ta = 0.0, tb = 0.0;
#pragma unroll
  for (int w = 0; w < PCG_THREADS / 32; ++w) {
    ta += sh[w];
    tb += sh[8 + w];
  }
  a = ta;
  b = tb;
}

__device__ __forceinline__ void grid_total2(const double* part, double& a, double& b, double* sh) {
  double va = 0.0, vb = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
    va += part[2 * i];
    vb += part[2 * i + 1];
  }
  cta_sum2(va, vb, sh);
  a = va;
  b = vb;
}

// row (br, rr) of A (z + beta p_old); beta == 0 reads only z
__device__ __forceinline__ double spmv_fused(const PcgArgs& a, int br, int rr, const double* __restrict__ zv,
                                             const double* __restrict__ po, double beta) {
  double acc = 0.0;
  int k1 = a.row_ptr[br + 1];
  for (int k = a.row_ptr[br]; k < k1; ++k) {
    const double2* blk = reinterpret_cast<const double2*>(a.val + 144 * (int64_t)k + 12 * rr);
    int c = a.col[k];
    const double* zc = zv + 12 * (int64_t)c;
    const double* pc = po + 12 * (int64_t)c;
#pragma unroll
    for (int h = 0; h < 6; ++h) {
      double2 m = __ldg(blk + h);
      acc += m.x * (zc[2 * h] + beta * pc[2 * h]) + m.y * (zc[2 * h + 1] + beta * pc[2 * h + 1]);
    }
  }
  return acc;
}

__device__ __forceinline__ double spmv_plain(const PcgArgs& a, int br, int rr, const double* __restrict__ xv) {
  double acc = 0.0;
  int k1 = a.row_ptr[br + 1];
  for (int k = a.row_ptr[br]; k < k1; ++k) {
    const double2* blk = reinterpret_cast<const double2*>(a.val + 144 * (int64_t)k + 12 * rr);
    const double* xc = xv + 12 * (int64_t)a.col[k];
#pragma unroll
    for (int h = 0; h < 6; ++h) {
      double2 m = __ldg(blk + h);
      acc += m.x * xc[2 * h] + m.y * xc[2 * h + 1];
    }
  }
  return acc;
}

__device__ __forceinline__ double prec_row(const PcgArgs& a, int br, int rr, const double* __restrict__ r) {
  const double2* P = reinterpret_cast<const double2*>(a.pinv + 144 * (int64_t)br + 12 * rr);
  const double* rv = r + 12 * (int64_t)br;
  double acc = 0.0;
#pragma unroll
  for (int h = 0; h < 6; ++h) {
    double2 m = __ldg(P + h);
    acc += m.x * rv[2 * h] + m.y * rv[2 * h + 1];
  }
  return acc;
}

__global__ void __launch_bounds__(PCG_THREADS) k_pcg(PcgArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double sh[16];
  if (*a.bad != 0x7fffffff) return;  // non-SPD preconditioner block: host raises
  const int lb = threadIdx.x / 12, rr = threadIdx.x % 12;
  const int groups = (a.n + PCG_ROWS - 1) / PCG_ROWS;
  // x = 0, r = b, p = 0
  double bb = 0.0;
  for (int g = blockIdx.x; g < groups; g += gridDim.x) {
    int br = g * PCG_ROWS + lb;
    if (br >= a.n) continue;
    int64_t t = 12 * (int64_t)br + rr;
    a.x[t] = 0.0;
    double bt = a.b[t];
    a.r[t] = bt;
    a.pa[t] = 0.0;
    bb += bt * bt;
  }
  double dummy = 0.0;
  cta_sum2(bb, dummy, sh);
  double* partA = a.part;
  double* partB = a.part + 2 * gridDim.x;
  if (threadIdx.x == 0) {
    partA[2 * blockIdx.x] = bb;
    partA[2 * blockIdx.x + 1] = 0.0;
  }
  grid.sync();
  double bn2, d2_;
  grid_total2(partA, bn2, d2_, sh);
  const double bnorm = sqrt(bn2);
  if (bnorm == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *a.out_iters = 0;
      *a.out_rel = 0.0;
    }
    return;
  }
  const double tol = a.rel_tol * bnorm;
  double* po = a.pa;
  double* pn = a.pb;
  int it = 0;
  double rel = 1.0;
  for (int restart = 0; restart < 4; ++restart) {
    // z = P^-1 r (CTA-local block rows), rz
    double rz = 0.0;
    for (int g = blockIdx.x; g < groups; g += gridDim.x) {
      int br = g * PCG_ROWS + lb;
      if (br >= a.n) continue;
      int64_t t = 12 * (int64_t)br + rr;
      double zt = prec_row(a, br, rr, a.r);
      a.z[t] = zt;
      rz += a.r[t] * zt;
    }
    double rr0 = 0.0;
    cta_sum2(rz, rr0, sh);
    if (threadIdx.x == 0) {
      partB[2 * blockIdx.x] = rz;
      partB[2 * blockIdx.x + 1] = 0.0;
    }
    grid.sync();
    grid_total2(partB, rz, rr0, sh);
    double beta = 0.0;
    bool conv = false;
    while (it < a.max_iters) {
      // phase A: p_new = z + beta p_old ; Ap = A p_new
      double pap = 0.0;
      for (int g = blockIdx.x; g < groups; g += gridDim.x) {
        int br = g * PCG_ROWS + lb;
        if (br >= a.n) continue;
        int64_t t = 12 * (int64_t)br + rr;
        double v = spmv_fused(a, br, rr, a.z, po, beta);
        double pt = a.z[t] + beta * po[t];
        pn[t] = pt;
        a.Ap[t] = v;
        pap += pt * v;
      }
      double zero = 0.0;
      cta_sum2(pap, zero, sh);
      if (threadIdx.x == 0) {
        partA[2 * blockIdx.x] = pap;
        partA[2 * blockIdx.x + 1] = 0.0;
      }
      grid.sync();
      grid_total2(partA, pap, zero, sh);
      double alpha = rz / pap;
      // phase B
      double rzn = 0.0, rrn = 0.0;
      for (int g = blockIdx.x; g < groups; g += gridDim.x) {
        int br = g * PCG_ROWS + lb;
        bool live = br < a.n;
        int64_t t = 12 * (int64_t)br + rr;
        if (live) {
          a.x[t] += alpha * pn[t];
          double rt = a.r[t] - alpha * a.Ap[t];
          a.r[t] = rt;
          rrn += rt * rt;
        }
        __syncthreads();  // whole block row of r written (same CTA)
        if (live) {
          double zt = prec_row(a, br, rr, a.r);
          a.z[t] = zt;
          rzn += a.r[t] * zt;
        }
      }
      cta_sum2(rzn, rrn, sh);
      if (threadIdx.x == 0) {
        partB[2 * blockIdx.x] = rzn;
        partB[2 * blockIdx.x + 1] = rrn;
      }
      grid.sync();
      grid_total2(partB, rzn, rrn, sh);
      ++it;
      double rn = sqrt(rrn);
      rel = rn / bnorm;
      double* tmp = po;
      po = pn;
      pn = tmp;
      if (rn <= tol || !(pap > 0.0)) {
        conv = rn <= tol;
        break;
      }
      beta = rzn / rz;
      rz = rzn;
    }
    // true residual r = b - A x
    grid.sync();
    double tr = 0.0;
    for (int g = blockIdx.x; g < groups; g += gridDim.x) {
      int br = g * PCG_ROWS + lb;
      if (br >= a.n) continue;
      int64_t t = 12 * (int64_t)br + rr;
      double v = a.b[t] - spmv_plain(a, br, rr, a.x);
      a.r[t] = v;
      tr += v * v;
    }
    double z0 = 0.0;
    cta_sum2(tr, z0, sh);
    if (threadIdx.x == 0) {
      partA[2 * blockIdx.x] = tr;
      partA[2 * blockIdx.x + 1] = 0.0;
    }
    grid.sync();
    grid_total2(partA, tr, z0, sh);
    rel = sqrt(tr) / bnorm;
    (void)conv;
    if (sqrt(tr) <= tol || it >= a.max_iters) break;
    // restart: reset p
    for (int g = blockIdx.x; g < groups; g += gridDim.x) {
      int br = g * PCG_ROWS + lb;
      if (br >= a.n) continue;
      po[12 * (int64_t)br + rr] = 0.0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
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
  Scene::Work& w = s.w;
  w.pinv.resize(144 * (int64_t)n);
  w.r.resize(N);
  w.z.resize(N);
  w.p.resize(N);
  w.p2.resize(N);
  w.Ap.resize(N);
  w.bad.resize(1);
  w.iters.resize(1);
  w.scal.resize(4);
  int big = 0x7fffffff;
  CK(cudaMemcpyAsync(w.bad.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
  k_jacobi_inv<<<grid_for(n, JI_BLOCKS), 128, 0, st>>>(n, H.diag_pos.p, H.val.p, w.pinv.p, w.bad.p);
  note_launch("k_jacobi_inv");
  static int blocks_per_sm = -1;
  if (blocks_per_sm < 0) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_pcg, PCG_THREADS, 0));
    if (blocks_per_sm < 1) blocks_per_sm = 1;
  }
  int groups = (n + PCG_ROWS - 1) / PCG_ROWS;
  int grid = std::max(1, std::min(groups, blocks_per_sm * s.num_sms));
  w.part.resize(4 * (int64_t)grid);
  PcgArgs a;
  a.n = n;
  a.row_ptr = H.row_ptr.p;
  a.col = H.col.p;
  a.val = H.val.p;
  a.pinv = w.pinv.p;
  a.bad = w.bad.p;
  a.b = rhs;
  a.x = x;
  a.r = w.r.p;
  a.z = w.z.p;
  a.pa = w.p.p;
  a.pb = w.p2.p;
  a.Ap = w.Ap.p;
  a.part = w.part.p;
  a.rel_tol = rel_tol;
  a.max_iters = max_iters;
  a.out_iters = w.iters.p;
  a.out_rel = w.scal.p;
  void* args[] = {&a};
  if (s.instrument) CK(cudaEventRecord(s.ev0, st));
  CK(cudaLaunchCooperativeKernel((void*)k_pcg, dim3(grid), dim3(PCG_THREADS), args, 0, st));
  note_launch("k_pcg");
  if (s.instrument) CK(cudaEventRecord(s.ev1, st));
  int hit = 0, hbad = 0;
  CK(cudaMemcpyAsync(&hit, w.iters.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&rel_res, w.scal.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&hbad, w.bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hbad != big) throw Error(ABD_ERR_FACTORIZATION, "non-SPD diagonal block in block-Jacobi PCG", hbad);
  if (s.instrument) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, s.ev0, s.ev1));
    Scene::KStat& k = s.kstat[0];
    k.launches += 1;
    k.units += hit;
    k.ms += ms;
    // algorithmic bytes per iteration: 1152 (nnzb + n) + 13 * 96 * n
    k.bytes += (double)hit * (1152.0 * (double)(H.nnzb + n) + 13.0 * 96.0 * n);
  }
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
  CK(cudaStreamSynchronize(st));
}

}  // namespace abd
