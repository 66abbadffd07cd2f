// Dependent-chain latency probes (cycles per op): DFMA, DMUL, SHFL(double), rsqrt_nr.
#include <cstdio>
__device__ __forceinline__ double rsqrt_nr(double x) {
  double r = (double)rsqrtf((float)x);
  r = r * fma(-0.5 * x, r * r, 1.5);
  r = r * fma(-0.5 * x, r * r, 1.5);
  r = r * fma(-0.5 * x, r * r, 1.5);
  return r;
}
__global__ void k(double* out, long long* cyc, double seed) {
  double a = seed + threadIdx.x, b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  for (int i = 0; i < 1024; ++i) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31);
  long long t2 = clock64();
  for (int i = 0; i < 256; ++i) a = rsqrt_nr(a) + 1.0;
  long long t3 = clock64();
  float f = (float)a;
  for (int i = 0; i < 1024; ++i) f = fmaf(f, 1.0000001f, 1e-9f);
  long long t4 = clock64();
  out[threadIdx.x] = a + f;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
  }
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 32 * 8);
  cudaMallocManaged(&c, 4 * 8);
  k<<<1, 32>>>(o, c, 1.0);
  k<<<1, 32>>>(o, c, 1.0);
  cudaDeviceSynchronize();
  printf("DFMA dep latency %.1f cyc, SHFL(double) %.1f cyc, rsqrt_nr+add %.1f cyc, FFMA %.1f cyc\n", c[0] / 1024.0,
         c[1] / 1024.0, c[2] / 256.0, c[3] / 1024.0);
  return 0;
}
