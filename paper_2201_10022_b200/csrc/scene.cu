// Scene lifetime, cub wrappers, deterministic reductions.
#include <cub/cub.cuh>

#include <atomic>
#include <cstdio>

#include "kernels.h"
#include "scene.h"

namespace abd {

std::atomic<int64_t> g_launches{0};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Error(ABD_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

void note_launch(const char* name) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Error(ABD_ERR_CUDA, std::string("launch ") + name + ": " + cudaGetErrorString(e));
}

int bits_for(int64_t maxval) {
  int b = 0;
  while (b < 63 && (int64_t(1) << b) <= maxval) ++b;
  return b < 1 ? 1 : b;
}

Scene::Scene() {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  CK(cudaMallocHost(&h_pinned, 64 * sizeof(double)));
  CK(cudaEventCreate(&ev0));
  CK(cudaEventCreate(&ev1));
  CK(cudaEventCreate(&tev0));
  CK(cudaEventCreate(&tev1));
  for (auto& k : kstat) {
    CK(cudaEventCreate(&k.e0));
    CK(cudaEventCreate(&k.e1));
  }
  w.ull.resize(16);
}

Scene::~Scene() {
  if (stream) cudaStreamDestroy(stream);
  if (h_pinned) cudaFreeHost(h_pinned);
  for (cudaEvent_t e : {ev0, ev1, tev0, tev1})
    if (e) cudaEventDestroy(e);
  if (w.ch_pre_ev) cudaEventDestroy(w.ch_pre_ev);
  for (auto& k : kstat) {
    if (k.e0) cudaEventDestroy(k.e0);
    if (k.e1) cudaEventDestroy(k.e1);
  }
}

void scan_exclusive_i32(Scene& s, const int* in, int* out, int64_t n) {
  if (n == 0) return;
  size_t bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, s.stream));
  s.tmp_bytes.resize(bytes);
  CK(cub::DeviceScan::ExclusiveSum(s.tmp_bytes.p, bytes, in, out, (int)n, s.stream));
}

void sort_pairs_u64(Scene& s, uint64_t* keys, uint64_t* keys_alt, int* vals, int* vals_alt, int64_t n,
                    int end_bit, bool& result_in_alt) {
  result_in_alt = false;
  if (n <= 1) return;
  cub::DoubleBuffer<uint64_t> k(keys, keys_alt);
  cub::DoubleBuffer<int> v(vals, vals_alt);
  size_t bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, (int)n, 0, end_bit, s.stream));
  s.tmp_bytes.resize(bytes);
  CK(cub::DeviceRadixSort::SortPairs(s.tmp_bytes.p, bytes, k, v, (int)n, 0, end_bit, s.stream));
  result_in_alt = (k.Current() == keys_alt);
}

void sort_pairs_u32(Scene& s, uint32_t* keys, uint32_t* keys_alt, int* vals, int* vals_alt, int64_t n, int end_bit,
                    bool& result_in_alt) {
  result_in_alt = false;
  if (n <= 1) return;
  cub::DoubleBuffer<uint32_t> k(keys, keys_alt);
  cub::DoubleBuffer<int> v(vals, vals_alt);
  size_t bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k, v, (int)n, 0, end_bit, s.stream));
  s.tmp_bytes.resize(bytes);
  CK(cub::DeviceRadixSort::SortPairs(s.tmp_bytes.p, bytes, k, v, (int)n, 0, end_bit, s.stream));
  result_in_alt = (k.Current() == keys_alt);
}

// fixed-order tree reduction of a partials array (one CTA, deterministic)
__global__ void k_reduce_fixed(const double* __restrict__ in, int n, double* __restrict__ out) {
  __shared__ double sh[1024];
  in += (int64_t)blockIdx.x * n;  // one CTA per partials array
  out += blockIdx.x;
  double acc = 0.0;
  // each thread sums a contiguous strided slice in index order
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += in[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

void kstat_flush(Scene& s, int which) {
  Scene::KStat& k = s.kstat[which];
  if (!k.pending) return;
  float ms = 0.f;
  CK(cudaEventSynchronize(k.e1));
  CK(cudaEventElapsedTime(&ms, k.e0, k.e1));
  k.launches += 1;
  k.units += k.p_units;
  k.ms += ms;
  k.bytes += k.p_bytes;
  k.pending = false;
}

void reduce_fixed_stream(cudaStream_t st, const double* partials, int n, double* out_dev) {
  if (n == 0) {
    CK(cudaMemsetAsync(out_dev, 0, sizeof(double), st));
    return;
  }
  k_reduce_fixed<<<1, 1024, 0, st>>>(partials, n, out_dev);
  note_launch("k_reduce_fixed");
}

void reduce_fixed_device(Scene& s, const double* partials, int n, double* out_dev) {
  reduce_fixed_stream(s.stream, partials, n, out_dev);
}

// `count` consecutive partial arrays of length n -> count sums (deterministic)
void reduce_fixed_multi(cudaStream_t st, const double* partials, int n, int count, double* out_dev) {
  k_reduce_fixed<<<count, 1024, 0, st>>>(partials, n, out_dev);
  note_launch("k_reduce_fixed");
}

double reduce_sum_det(Scene& s, const double* partials, int n) {
  s.tmp_d3.resize(1);
  reduce_fixed_device(s, partials, n, s.tmp_d3.p);
  CK(cudaMemcpyAsync(s.h_pinned, s.tmp_d3.p, sizeof(double), cudaMemcpyDeviceToHost, s.stream));
  CK(cudaStreamSynchronize(s.stream));
  return s.h_pinned[0];
}

}  // namespace abd
