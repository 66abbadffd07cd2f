// Cycle counts of 12x12 in-register Cholesky variants on one warp (lane t = row t).
#include <cstdio>
__device__ __forceinline__ double hshfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double rsqrt_nr(double x) {
  if (!(x > 1e-36 && x < 1e36)) return 1.0 / sqrt(x);
  double r = (double)rsqrtf((float)x);
  r = r * fma(-0.5 * x, r * r, 1.5);
  r = r * fma(-0.5 * x, r * r, 1.5);
  r = r * fma(-0.5 * x, r * r, 1.5);
  return r;
}
__device__ __forceinline__ double rsqrt_hw(double x) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = r * fma(-0.5 * x, r * r, 1.5);
  r = r * fma(-0.5 * x, r * r, 1.5);
  return r;
}
template <int V>
__device__ __forceinline__ bool chol12(int t, double d[12], double rinv[12]) {
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    const double p = hshfl(d[c], c);
    ok = ok && (p > 0.0);
    const double pp = p > 0.0 ? p : 1.0;
    const double r = V == 0 ? rsqrt_nr(pp) : rsqrt_hw(pp);
    rinv[c] = r;
    if (t == c) d[c] = pp * r;
    else if (t > c) d[c] *= r;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      if (k > c) {
        const double lkc = hshfl(d[c], k);
        if (t >= k) d[k] = fma(-d[c], lkc, d[k]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 12; ++c)
    if (c > t) d[c] = 0.0;
  return ok;
}
// variant 3: the next pivot is computed by its owner lane right after scaling and
// broadcast at once, so the trailing-update shuffles leave the critical path
__device__ __forceinline__ bool chol12_fast(int t, double d[12], double rinv[12]) {
  bool ok = true;
  double p = hshfl(d[0], 0);
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    ok = ok && (p > 0.0);
    const double pp = p > 0.0 ? p : 1.0;
    const double r = rsqrt_hw(pp);
    rinv[c] = r;
    if (t == c) d[c] = pp * r;
    else if (t > c) d[c] *= r;
    double pn = 0.0;
    if (c < 11) pn = hshfl(fma(-d[c], d[c], d[c + 1]), c + 1);
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      if (k > c) {
        const double lkc = hshfl(d[c], k);
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

// variant 2: column c broadcast through shared memory
__device__ __forceinline__ bool chol12_smem(int t, double d[12], double rinv[12], double* col) {
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 12; ++c) {
    if (t == c) col[12] = d[c];
    __syncwarp();
    const double p = col[12];
    ok = ok && (p > 0.0);
    const double pp = p > 0.0 ? p : 1.0;
    const double r = rsqrt_hw(pp);
    rinv[c] = r;
    if (t == c) d[c] = pp * r;
    else if (t > c) d[c] *= r;
    if (t < 12) col[t] = d[c];
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 12; ++k)
      if (k > c && t >= k) d[k] = fma(-d[c], col[k], d[k]);
    __syncwarp();
  }
#pragma unroll
  for (int c = 0; c < 12; ++c)
    if (c > t) d[c] = 0.0;
  return ok;
}
__global__ void k(double* out, long long* cyc, int variant) {
  __shared__ double col[16];
  const int t = threadIdx.x & 31;
  double d[12], r[12];
  long long tot = 0;
  double acc = 0.0;
  for (int rep = 0; rep < 64; ++rep) {
#pragma unroll
    for (int c = 0; c < 12; ++c) d[c] = (t == c ? 20.0 + rep : 0.0) + 1.0 / (1.0 + t + c);
    __syncwarp();
    long long t0 = clock64();
    bool ok;
    if (variant == 0) ok = chol12<0>(t, d, r);
    else if (variant == 1) ok = chol12<1>(t, d, r);
    else if (variant == 2) ok = chol12_smem(t, d, r, col);
    else ok = chol12_fast(t, d, r);
    __syncwarp();
    long long t1 = clock64();
    tot += t1 - t0;
    acc += ok ? d[t % 12] : 0.0;
  }
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[variant] = tot / 64;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 32 * 8);
  cudaMallocManaged(&c, 4 * 8);
  double h[4][32];
  for (int v = 0; v < 4; ++v) {
    k<<<1, 32>>>(o, c, v);
    k<<<1, 32>>>(o, c, v);
    cudaMemcpy(h[v], o, 32 * 8, cudaMemcpyDeviceToHost);
  }
  cudaDeviceSynchronize();
  printf("chol12 cycles: shfl+rsqrt_nr %lld, shfl+rsqrt.approx %lld, smem+rsqrt.approx %lld, early-pivot %lld\n", c[0],
         c[1], c[2], c[3]);
  double md = 0;
  for (int v = 1; v < 4; ++v)
    for (int i = 0; i < 12; ++i) md = fmax(md, fabs(h[v][i] - h[0][i]) / fabs(h[0][i]));
  printf("max rel diff vs variant 0: %.3e\n", md);
  return 0;
}
