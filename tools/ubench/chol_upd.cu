// Micro-benchmark: one warp accumulating U block products bt -= L_ik L_jk^T (12x12)
// from L2-resident blocks, as in the Cholesky block task (k_chol.cu).  Variants:
//   0: cp.async.cg 3-stage pipeline into shared memory (the k_chol.cu scheme)
//   1: ld.global.cg straight into registers, no pipeline
//   2: ld.global (L1-cached) straight into registers
// Prints cycles per update for 1 warp and for many concurrent warps.
#include <cstdio>
#include <cuda_runtime.h>


__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int NST> __device__ __forceinline__ void cp_wait_pipe() { asm volatile("cp.async.wait_group %0;" ::"n"(NST - 2) : "memory"); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE, int NST>
__global__ void k_upd(const double* L, const int2* pairs, int U, double* out, long long* cyc) {
  __shared__ __align__(16) double st[2][NST][2][144];
  const int t = threadIdx.x & 31, hw = threadIdx.x >> 5, tt = t < 12 ? t : 0;
  double bt[12];
  for (int c = 0; c < 12; ++c) bt[c] = 0.0;
  const int2* pr = pairs + (blockIdx.x * 2 + hw) * U;
  long long t0 = clock64();
  if (MODE == 4 || MODE == 5) {
    double acc[2][2][2] = {};
    auto issue = [&](int u) {
      const double* a = L + 144 * (long long)pr[u].x;
      const double* b = L + 144 * (long long)pr[u].y;
      for (int c = t; c < 72; c += 32) {
        cp16(st[hw][u % NST][0] + 2 * c, a + 2 * c);
        cp16(st[hw][u % NST][1] + 2 * c, b + 2 * c);
      }
    };
    if (MODE == 5) {
      for (int c = t; c < 2 * 144; c += 32) (&st[hw][0][0][0])[c] = L[c];
      __syncwarp();
    } else {
      for (int p = 0; p < NST - 1; ++p) {
        if (p < U) issue(p);
        cp_commit();
      }
    }
    const int r = t >> 2, k4 = t & 3;
    for (int u = 0; u < U; ++u) {
      if (MODE == 4) {
        cp_wait_pipe<NST>();
        __syncwarp();
      }
      const double* Li = st[hw][MODE == 4 ? u % NST : 0][0];
      const double* Lj = st[hw][MODE == 4 ? u % NST : 0][1];
      double fa[2][3], fb[2][3];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const bool ok = 8 * mi + r < 12;
          fa[mi][kk] = ok ? -Li[(8 * mi + r) * 12 + 4 * kk + k4] : 0.0;
          fb[mi][kk] = ok ? Lj[(8 * mi + r) * 12 + 4 * kk + k4] : 0.0;
        }
#pragma unroll
      for (int kk = 0; kk < 3; ++kk)
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], fa[mi][kk], fb[ni][kk]);
      if (MODE == 4) {
        __syncwarp();
        if (u + NST - 1 < U) issue(u + NST - 1);
        cp_commit();
      }
    }
    for (int c = 0; c < 8; ++c) bt[c % 12] += (&acc[0][0][0])[c];
  } else if (MODE == 3) {
    for (int c = t; c < 2 * 144; c += 32) (&st[hw][0][0][0])[c] = L[c];
    __syncwarp();
    for (int u = 0; u < U; ++u) {
      const double* Li = st[hw][0][0];
      const double* Lj = st[hw][0][1];
      double lr[12];
      for (int m = 0; m < 12; ++m) lr[m] = Li[12 * tt + m] + u;
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < 12; ++m) s = fma(lr[m], Lj[12 * c + m], s);
        bt[c] -= s;
      }
    }
  } else if (MODE == 0) {
    auto issue = [&](int u) {
      const double* a = L + 144 * (long long)pr[u].x;
      const double* b = L + 144 * (long long)pr[u].y;
      for (int c = t; c < 72; c += 32) {
        cp16(st[hw][u % NST][0] + 2 * c, a + 2 * c);
        cp16(st[hw][u % NST][1] + 2 * c, b + 2 * c);
      }
    };
    for (int p = 0; p < NST - 1; ++p) {
      if (p < U) issue(p);
      cp_commit();
    }
    for (int u = 0; u < U; ++u) {
      cp_wait_pipe<NST>();
      __syncwarp();
      const double* Li = st[hw][u % NST][0];
      const double* Lj = st[hw][u % NST][1];
      double lr[12];
      for (int m = 0; m < 12; ++m) lr[m] = Li[12 * tt + m];
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < 12; ++m) s = fma(lr[m], Lj[12 * c + m], s);
        bt[c] -= s;
      }
      __syncwarp();
      if (u + NST - 1 < U) issue(u + NST - 1);
      cp_commit();
    }
  } else {
    for (int u = 0; u < U; ++u) {
      const double* a = L + 144 * (long long)pr[u].x + 12 * tt;
      const double* b = L + 144 * (long long)pr[u].y;
      double lr[12];
      for (int m = 0; m < 12; ++m) lr[m] = MODE == 1 ? __ldcg(a + m) : a[m];
#pragma unroll
      for (int c = 0; c < 12; ++c) {
        double s = 0.0;
#pragma unroll
        for (int m = 0; m < 12; ++m) s = fma(lr[m], MODE == 1 ? __ldcg(b + 12 * c + m) : b[12 * c + m], s);
        bt[c] -= s;
      }
    }
  }
  long long t1 = clock64();
  double acc = 0;
  for (int c = 0; c < 12; ++c) acc += bt[c];
  out[blockIdx.x * 64 + threadIdx.x] = acc;
  if (t == 0) cyc[blockIdx.x * 2 + hw] = t1 - t0;
}

int main() {
  const int NB = 16000, U = 64, maxw = 592 * 4;
  double* L;
  int2* pairs;
  double* out;
  long long* cyc;
  cudaMalloc(&L, 144LL * NB * 8);
  cudaMemset(L, 0, 144LL * NB * 8);
  int2* hp = new int2[(size_t)maxw * U];
  unsigned s = 1;
  for (int i = 0; i < maxw * U; ++i) {
    s = s * 1664525u + 1013904223u;
    int a = s % NB;
    s = s * 1664525u + 1013904223u;
    hp[i] = make_int2(a, s % NB);
  }
  cudaMalloc(&pairs, sizeof(int2) * maxw * U);
  cudaMemcpy(pairs, hp, sizeof(int2) * maxw * U, cudaMemcpyHostToDevice);
  cudaMalloc(&out, 8LL * 592 * 128);
  cudaMalloc(&cyc, 8LL * maxw);
  long long* hc = new long long[maxw];
  auto run = [&](const char* name, auto kern, int blocks) {
    for (int rep = 0; rep < 3; ++rep) kern<<<blocks, blocks == 1 ? 32 : 64, 0>>>(L, pairs, U, out, cyc);
    cudaDeviceSynchronize();
    int nw = blocks == 1 ? 1 : blocks * 2;
    cudaMemcpy(hc, cyc, 8 * nw, cudaMemcpyDeviceToHost);
    double m = 0;
    for (int i = 0; i < nw; ++i) m += hc[i];
    printf("%-22s warps %5d: %.0f cycles/update\n", name, nw, m / nw / U);
  };
  for (int blocks : {1, 148}) {
    run("cp.async NST=3", k_upd<0, 3>, blocks);
    run("cp.async NST=4", k_upd<0, 4>, blocks);
    run("cp.async NST=6", k_upd<0, 6>, blocks);
    run("ld.cg regs", k_upd<1, 3>, blocks);
    run("ld L1 regs", k_upd<2, 3>, blocks);
    run("compute only (smem)", k_upd<3, 3>, blocks);
    run("DMMA cp.async NST=3", k_upd<4, 3>, blocks);
    run("DMMA cp.async NST=4", k_upd<4, 4>, blocks);
    run("DMMA compute only", k_upd<5, 3>, blocks);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
