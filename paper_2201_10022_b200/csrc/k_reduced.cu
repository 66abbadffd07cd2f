// Joint-reduced Newton direction on the device (solver.py:479-490): with the
// embedding q_dyn = T u + q_const of constraints.py (T dense, 12 n_dyn x n_u,
// uploaded once per model by abd_set_reduction),
//     H_u = T^T H T,  g_u = T^T g,  L L^T = 0.5 (H_u + H_u^T),  du = -L^-T L^-1 g_u,
//     dx = T du,
// and the non-descent fallback dx = T (T^T (-g)) (solver.py:557-561).  Joint
// scenes are small (tens of bodies, n_u <= a few thousand): W = H T is a BSR x
// dense product, T^T W a dense product, and the dense Cholesky / triangular solves
// run right-looking in one CTA over an L2-resident matrix.  A non-positive pivot
// raises ABD_ERR_FACTORIZATION (numpy's cholesky raises LinAlgError there).
#include "driver.h"

namespace abd {

// W[r][c] = sum_k sum_m H(br, col_k)[rr][m] T[12 col_k + m][c]   (r = 12 br + rr)
__global__ void k_red_ht(int n, const int* __restrict__ row_ptr, const int* __restrict__ col,
                         const double* __restrict__ val, int64_t nu, const double* __restrict__ T, double* W) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (c >= nu || r >= 12 * n) return;
  const int br = r / 12, rr = r % 12;
  double acc = 0.0;
  for (int k = row_ptr[br]; k < row_ptr[br + 1]; ++k) {
    const double* h = val + 144 * (int64_t)k + 12 * rr;
    const double* t = T + (int64_t)12 * col[k] * nu + c;
#pragma unroll
    for (int m = 0; m < 12; ++m) acc = fma(h[m], t[m * nu], acc);
  }
  W[(int64_t)r * nu + c] = acc;
}

// X[a][b] = sum_r T[r][a] W[r][b]
__global__ void k_red_tw(int64_t rows, int64_t nu, const double* __restrict__ T, const double* __restrict__ W,
                         double* X) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t a = blockIdx.y;
  if (b >= nu || a >= nu) return;
  double acc = 0.0;
  for (int64_t r = 0; r < rows; ++r) acc = fma(T[r * nu + a], W[r * nu + b], acc);
  X[a * nu + b] = acc;
}

// A = 0.5 (X + X^T)
__global__ void k_red_sym(int64_t nu, const double* __restrict__ X, double* A) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nu * nu) return;
  const int64_t a = i / nu, b = i % nu;
  A[i] = 0.5 * (X[a * nu + b] + X[b * nu + a]);
}

// y[a] = sign * sum_r T[r][a] v[r]
__global__ void k_red_tt(int64_t rows, int64_t nu, const double* __restrict__ T, const double* __restrict__ v,
                         double sign, double* y) {
  const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (a >= nu) return;
  double acc = 0.0;
  for (int64_t r = 0; r < rows; ++r) acc = fma(T[r * nu + a], v[r], acc);
  y[a] = sign * acc;
}

// x[r] = sum_a T[r][a] u[a]
__global__ void k_red_t(int64_t rows, int64_t nu, const double* __restrict__ T, const double* __restrict__ u,
                        double* x) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double acc = 0.0;
  for (int64_t a = 0; a < nu; ++a) acc = fma(T[r * nu + a], u[a], acc);
  x[r] = acc;
}

// In-place lower Cholesky of A (nu x nu, row-major), then L y = b, L^T x = y with
// x = du written to out (b = -g_u); one CTA, right-looking.  bad = first failing pivot + 1.
__global__ void __launch_bounds__(1024) k_red_chol_solve(int64_t nu, double* A, const double* __restrict__ b,
                                                         double* out, int* bad) {
  __shared__ double piv;
  __shared__ int fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) fail = 0;
  __syncthreads();
  for (int64_t k = 0; k < nu; ++k) {
    if (tid == 0) {
      const double d = A[k * nu + k];
      if (!(d > 0.0)) {
        fail = (int)k + 1;
        piv = 1.0;
      } else {
        piv = sqrt(d);
      }
      A[k * nu + k] = piv;
    }
    __syncthreads();
    if (fail) break;
    const double p = piv;
    for (int64_t i = k + 1 + tid; i < nu; i += nt) A[i * nu + k] /= p;
    __syncthreads();
    // trailing lower triangle: rows i > k, columns k < j <= i
    const int64_t m = nu - k - 1;
    const int64_t tri = m * (m + 1) / 2;
    for (int64_t e = tid; e < tri; e += nt) {
      // e -> (ii, jj) with 0 <= jj <= ii < m, row-major over the triangle
      int64_t ii = (int64_t)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
      while (ii * (ii + 1) / 2 > e) --ii;
      while ((ii + 1) * (ii + 2) / 2 <= e) ++ii;
      const int64_t jj = e - ii * (ii + 1) / 2;
      const int64_t i = k + 1 + ii, j = k + 1 + jj;
      A[i * nu + j] = fma(-A[i * nu + k], A[j * nu + k], A[i * nu + j]);
    }
    __syncthreads();
  }
  if (fail) {
    if (tid == 0) *bad = fail;
    return;
  }
  // forward: L y = b (y in out)
  for (int64_t i = tid; i < nu; i += nt) out[i] = b[i];
  __syncthreads();
  for (int64_t k = 0; k < nu; ++k) {
    if (tid == 0) out[k] = out[k] / A[k * nu + k];
    __syncthreads();
    const double yk = out[k];
    for (int64_t i = k + 1 + tid; i < nu; i += nt) out[i] = fma(-A[i * nu + k], yk, out[i]);
    __syncthreads();
  }
  // backward: L^T x = y
  for (int64_t k = nu - 1; k >= 0; --k) {
    if (tid == 0) out[k] = out[k] / A[k * nu + k];
    __syncthreads();
    const double xk = out[k];
    for (int64_t i = tid; i < k; i += nt) out[i] = fma(-A[k * nu + i], xk, out[i]);
    __syncthreads();
  }
}

void set_reduction(Scene& s, int64_t nu, const double* T_host) {
  if (nu < 0) throw Error(ABD_ERR_ARG, "negative reduced unknown count");
  s.red_nu = nu;
  if (nu == 0) return;
  if (s.comm.world > 1) throw Error(ABD_ERR_ARG, "joint reduction is single-rank");
  if (12 * (int64_t)s.n_dyn > 65535 || nu > 65535)
    throw Error(ABD_ERR_ARG, "joint reduction supports at most 5461 dynamic bodies and 65535 unknowns");
  s.red_T.upload(T_host, (size_t)12 * s.n_dyn * nu, s.stream);
  SSYNC(s.stream);
}

// dx = T du with H_u du = -T^T g (neg_g = -g); throws ABD_ERR_FACTORIZATION
void reduced_solve(Scene& s, const double* neg_g, double* dx) {
  const int64_t nu = s.red_nu, rows = 12 * (int64_t)s.n_dyn;
  cudaStream_t st = s.stream;
  s.red_W.resize(rows * nu);
  s.red_X.resize(nu * nu);
  s.red_A.resize(nu * nu);
  s.red_v.resize(2 * nu);
  s.w.err.resize(2);
  s.w.err.zero(st);
  const int TB = 128;
  dim3 g1((unsigned)((nu + TB - 1) / TB), (unsigned)rows);
  k_red_ht<<<g1, TB, 0, st>>>(s.n_dyn, s.H.row_ptr.p, s.H.col.p, s.H.val.p, nu, s.red_T.p, s.red_W.p);
  note_launch("k_red_ht");
  dim3 g2((unsigned)((nu + TB - 1) / TB), (unsigned)nu);
  k_red_tw<<<g2, TB, 0, st>>>(rows, nu, s.red_T.p, s.red_W.p, s.red_X.p);
  note_launch("k_red_tw");
  k_red_sym<<<grid_for(nu * nu, 256), 256, 0, st>>>(nu, s.red_X.p, s.red_A.p);
  note_launch("k_red_sym");
  // b = T^T (-g) = -g_u
  k_red_tt<<<grid_for(nu, TB), TB, 0, st>>>(rows, nu, s.red_T.p, neg_g, 1.0, s.red_v.p);
  note_launch("k_red_tt");
  k_red_chol_solve<<<1, 1024, 0, st>>>(nu, s.red_A.p, s.red_v.p, s.red_v.p + nu, s.w.err.p);
  note_launch("k_red_chol_solve");
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, s.w.err.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  SSYNC(st);
  if (bad)
    throw Error(ABD_ERR_FACTORIZATION, "reduced Newton matrix T^T H T is not positive definite (pivot " +
                                           std::to_string(bad - 1) + ")", (bad - 1) / 12);
  k_red_t<<<grid_for(rows, TB), TB, 0, st>>>(rows, nu, s.red_T.p, s.red_v.p + nu, dx);
  note_launch("k_red_t");
}

// out = T (T^T v)
void reduced_project(Scene& s, const double* v, double* out) {
  const int64_t nu = s.red_nu, rows = 12 * (int64_t)s.n_dyn;
  s.red_v.resize(2 * nu);
  k_red_tt<<<grid_for(nu, 128), 128, 0, s.stream>>>(rows, nu, s.red_T.p, v, 1.0, s.red_v.p);
  note_launch("k_red_tt");
  k_red_t<<<grid_for(rows, 128), 128, 0, s.stream>>>(rows, nu, s.red_T.p, s.red_v.p, out);
  note_launch("k_red_t");
}

}  // namespace abd
