// FP64 peak probe for the %FP64 roofline of the FP64-bound kernels (K1, K3, K5):
// DFMA throughput (8 independent FMA chains per thread, all SMs, enough warps to
// hide the pipe latency) and DMMA throughput (mma.sync.m8n8k4.f64, the FP64 tensor
// core path the Cholesky block products use).  Prints one JSON line.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench/dfma tools/ubench/dfma.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_dfma(double* out, double a, double b) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;  // never true; keeps the chains live
}

__global__ void k_dmma(double* out, double a) {
  double d[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i][0] = d[i][1] = 0.0;
  double fa = a * (threadIdx.x + 1), fb = a * 0.5;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[i][0]), "+d"(d[i][1])
                   : "d"(fa), "d"(fb));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  double best_fma = 0, best_mma = 0;
  int best_fma_cfg = 0, best_mma_cfg = 0;
  for (int per_sm : {4, 8, 16}) {
    for (int rep = 0; rep < 3; ++rep) {
      const int grid = sms * per_sm, block = 256;
      k_dfma<<<grid, block>>>(out, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      k_dfma<<<grid, block>>>(out, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 8 * ITERS * (double)grid * block;
      const double tf = flops / (ms * 1e-3) / 1e12;
      if (tf > best_fma) best_fma = tf, best_fma_cfg = per_sm;
    }
    for (int rep = 0; rep < 3; ++rep) {
      const int grid = sms * per_sm, block = 128;
      k_dmma<<<grid, block>>>(out, 1e-3);
      cudaEventRecord(e0);
      k_dmma<<<grid, block>>>(out, 1e-3);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      // one m8n8k4 = 8*8*4 FMAs = 512 flop per warp
      const double flops = 512.0 * 4 * ITERS * (double)grid * (block / 32);
      const double tf = flops / (ms * 1e-3) / 1e12;
      if (tf > best_mma) best_mma = tf, best_mma_cfg = per_sm;
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f, \"dfma_tflops\": %.3f, \"dfma_ctas_per_sm\": %d, "
         "\"dmma_tflops\": %.3f, \"dmma_ctas_per_sm\": %d, \"error\": \"%s\"}\n",
         p.name, sms, clk_khz / 1e3, best_fma, best_fma_cfg, best_mma, best_mma_cfg, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
