// Scene lifetime, cub wrappers, deterministic reductions.
#include <cub/cub.cuh>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

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
  // the main stream carries the critical path: its pending CTAs are dispatched ahead of the
  // side streams' (a 4-wave side kernel launched first -- k_body_derivs -- otherwise holds up
  // the activity scan behind it for ~40 us per Newton iteration)
  int prio_least = 0, prio_greatest = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
  CK(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, prio_greatest));
  main_stream = stream;
  CK(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, prio_least));
  CK(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming));
  CK(cudaStreamCreateWithPriority(&side2, cudaStreamNonBlocking, prio_least));
  CK(cudaStreamCreateWithPriority(&side3, cudaStreamNonBlocking, prio_least));
  CK(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&plan_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&moll_fork_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&moll_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&hot_fork_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&hot_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&pb_fork_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&pb_ev, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&side4, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ch_fork_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ch_join_ev, cudaEventDisableTiming));
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
  chol_worker.reset();  // joins the analysis thread before any buffer it uses goes away
  if (stream) cudaStreamDestroy(stream);
  if (side) cudaStreamDestroy(side);
  if (fork_ev) cudaEventDestroy(fork_ev);
  if (join_ev) cudaEventDestroy(join_ev);
  if (side2) cudaStreamDestroy(side2);
  if (side3) cudaStreamDestroy(side3);
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (plan_ev) cudaEventDestroy(plan_ev);
  if (moll_fork_ev) cudaEventDestroy(moll_fork_ev);
  if (moll_ev) cudaEventDestroy(moll_ev);
  if (hot_fork_ev) cudaEventDestroy(hot_fork_ev);
  if (hot_ev) cudaEventDestroy(hot_ev);
  if (pb_fork_ev) cudaEventDestroy(pb_fork_ev);
  if (pb_ev) cudaEventDestroy(pb_ev);
  if (side4) cudaStreamDestroy(side4);
  if (ch_fork_ev) cudaEventDestroy(ch_fork_ev);
  if (ch_join_ev) cudaEventDestroy(ch_join_ev);
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

// Small sorts (n <= 16384 keys of <= 32 bits): one CTA, cub::BlockRadixSort, one
// launch instead of the device sort's memset + histogram + scan + onesweep passes.
// Stable (padding sorts after every real key), so the result equals the device sort's.
constexpr int BS_THREADS = 1024, BS_ITEMS = 16, BS_CAP = BS_THREADS * BS_ITEMS;
typedef cub::BlockRadixSort<uint32_t, BS_THREADS, BS_ITEMS, int, 6> BlockSortU32;
static_assert(sizeof(BlockSortU32::TempStorage) <= 200 * 1024, "block sort smem");

template <class K>
__global__ void __launch_bounds__(BS_THREADS) k_block_sort(const K* __restrict__ kin, const int* __restrict__ vin,
                                                           K* kout, int* vout, int n, int end_bit) {
  extern __shared__ __align__(16) unsigned char bs_smem[];
  auto& temp = *reinterpret_cast<typename BlockSortU32::TempStorage*>(bs_smem);
  uint32_t k[BS_ITEMS];
  int v[BS_ITEMS];
#pragma unroll
  for (int i = 0; i < BS_ITEMS; ++i) {
    const int idx = threadIdx.x * BS_ITEMS + i;  // blocked: input order preserved
    k[i] = idx < n ? (uint32_t)kin[idx] : 0xffffffffu;
    v[i] = idx < n ? vin[idx] : -1;
  }
  BlockSortU32(temp).SortBlockedToStriped(k, v, 0, end_bit);
#pragma unroll
  for (int i = 0; i < BS_ITEMS; ++i) {
    const int idx = i * BS_THREADS + threadIdx.x;
    if (idx < n) {
      kout[idx] = (K)k[i];
      vout[idx] = v[i];
    }
  }
}

template <class K>
static bool block_sort(Scene& s, K* keys, K* keys_alt, int* vals, int* vals_alt, int64_t n, int end_bit) {
  static const bool off = getenv("ABD_NO_BLOCK_SORT") != nullptr;
  if (off || n > BS_CAP || end_bit > 32) return false;
  static bool attr = false;
  const int smem = (int)sizeof(typename BlockSortU32::TempStorage);
  if (!attr) {
    CK(cudaFuncSetAttribute((void*)k_block_sort<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute((void*)k_block_sort<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  k_block_sort<K><<<1, BS_THREADS, smem, s.stream>>>(keys, vals, keys_alt, vals_alt, (int)n, end_bit);
  note_launch("k_block_sort");
  return true;
}

void sort_pairs_u64(Scene& s, uint64_t* keys, uint64_t* keys_alt, int* vals, int* vals_alt, int64_t n,
                    int end_bit, bool& result_in_alt) {
  result_in_alt = false;
  if (n <= 1) return;
  if (block_sort(s, keys, keys_alt, vals, vals_alt, n, end_bit)) {
    result_in_alt = true;
    return;
  }
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
  if (block_sort(s, keys, keys_alt, vals, vals_alt, n, end_bit)) {
    result_in_alt = true;
    return;
  }
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

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }
__global__ void k_set_i32(int* p, int v) { *p = v; }
__global__ void k_set_i64(int64_t* p, int64_t v) { *p = v; }

void dev_set_u64(cudaStream_t st, unsigned long long* p, unsigned long long v) {
  k_set_u64<<<1, 1, 0, st>>>(p, v);
  note_launch("k_set");
}
void dev_set_i32(cudaStream_t st, int* p, int v) {
  k_set_i32<<<1, 1, 0, st>>>(p, v);
  note_launch("k_set");
}
void dev_set_i64(cudaStream_t st, int64_t* p, int64_t v) {
  k_set_i64<<<1, 1, 0, st>>>(p, v);
  note_launch("k_set");
}

struct PackArgs {
  const int* src[8];
  int words[8];
  int off[8];
  int n;
  int* dst;
};
__global__ void k_pack(PackArgs a) {
  for (int i = 0; i < a.n; ++i)
    for (int w = threadIdx.x; w < a.words[i]; w += blockDim.x) a.dst[a.off[i] + w] = a.src[i][w];
}

void pack_to_host(cudaStream_t st, void* host_dst, std::initializer_list<PackItem> items) {
  PackArgs a{};
  a.dst = reinterpret_cast<int*>(host_dst);
  for (const PackItem& it : items) {
    if (a.n == 8) throw Error(ABD_ERR_ARG, "pack_to_host: more than 8 items");
    a.src[a.n] = reinterpret_cast<const int*>(it.src);
    a.words[a.n] = it.bytes / 4;
    a.off[a.n] = it.dst_off / 4;
    ++a.n;
  }
  k_pack<<<1, 32, 0, st>>>(a);
  note_launch("k_pack");
}

static const bool g_prof_on = getenv("ABD_HOST_PROF") != nullptr;
struct ProfSite {
  int64_t n = 0;
  double host_ms = 0.0, blocked_ms = 0.0;
};
static std::map<std::string, ProfSite> g_sites;
static std::mutex g_prof_mu;
static std::chrono::steady_clock::time_point g_last;
static bool g_last_set = false;

void host_sync(cudaStream_t st, const char* site) {
  if (!g_prof_on) {
    CK(cudaStreamSynchronize(st));
    return;
  }
  using clk = std::chrono::steady_clock;
  auto t0 = clk::now();
  CK(cudaStreamSynchronize(st));
  auto t1 = clk::now();
  std::lock_guard<std::mutex> g(g_prof_mu);
  const char* base = strrchr(site, '/');
  ProfSite& p = g_sites[base ? base + 1 : site];
  p.n += 1;
  if (g_last_set) p.host_ms += std::chrono::duration<double, std::milli>(t0 - g_last).count();
  p.blocked_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
  g_last = t1;
  g_last_set = true;
}

void host_mark(const char* site) {
  if (!g_prof_on) return;
  auto t = std::chrono::steady_clock::now();
  std::lock_guard<std::mutex> g(g_prof_mu);
  const char* base = strrchr(site, '/');
  ProfSite& p = g_sites[std::string("mark ") + (base ? base + 1 : site)];
  p.n += 1;
  if (g_last_set) p.host_ms += std::chrono::duration<double, std::milli>(t - g_last).count();
  g_last = t;
  g_last_set = true;
}

void host_prof_reset() {
  g_sites.clear();
  g_last_set = false;
}

void host_prof_dump() {
  if (!g_prof_on) return;
  double h = 0.0, b = 0.0;
  int64_t n = 0;
  for (auto& kv : g_sites) {
    fprintf(stderr, "[host_prof] %-22s n=%7lld host=%9.2fms blocked=%9.2fms\n", kv.first.c_str(),
            (long long)kv.second.n, kv.second.host_ms, kv.second.blocked_ms);
    h += kv.second.host_ms;
    b += kv.second.blocked_ms;
    n += kv.second.n;
  }
  fprintf(stderr, "[host_prof] total syncs=%lld host=%.2fms blocked=%.2fms\n", (long long)n, h, b);
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
  SSYNC(s.stream);
  return s.h_pinned[0];
}

}  // namespace abd
