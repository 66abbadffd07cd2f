// Multi-GPU collectives and the body-slab partition of the Newton step.
//
// One process per GPU.  Each step the dynamic bodies are cut into W slabs along
// the longest axis of their positions, balanced by primitive count
// (slab_partition; partition.py restates it for the CPU tests).  A body pair
// belongs to the slab owning its lower body (its higher one when the lower is
// kinematic), so pairs across a slab face are halo pairs of exactly one rank:
// its primitive pairs, pair blocks, CCD queries and contact / friction energies.
// The assembled system is all-reduced so every rank holds complete rows; the
// Newton system is solved by a distributed PCG (k_chol.cu slab_pcg) whose
// preconditioner is each rank's sparse Cholesky of its own slab block, with the
// search vector's slab segments exchanged and its dot products all-reduced.
// Scalars (energies, CCD bound, flags) are all-reduced; every rank takes the same
// decisions and holds the same state.
//
// Backends: NCCL loaded at run time (whichever libnccl.so.2 the process already
// uses, e.g. torch's), or a host callback (tests drive it with torch.distributed
// gloo ranks sharing one GPU).  Reductions are enqueued on the scene stream.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>
#include <mutex>

#include "driver.h"

namespace abd {

namespace {

// minimal NCCL ABI (nccl.h types, resolved with dlsym)
typedef struct {
  char internal[128];
} NcclId;
typedef void* NcclComm;
enum { kNcclInt32 = 2, kNcclInt64 = 4, kNcclFloat64 = 8 };
enum { kNcclSum = 0, kNcclMax = 2, kNcclMin = 3 };
typedef int (*FnGetId)(NcclId*);
typedef int (*FnInit)(NcclComm*, int, NcclId, int);
typedef int (*FnAllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*FnDestroy)(NcclComm);
typedef const char* (*FnErr)(int);

struct NcclLib {
  void* h = nullptr;
  FnGetId get_id = nullptr;
  FnInit init = nullptr;
  FnAllReduce all_reduce = nullptr;
  FnDestroy destroy = nullptr;
  FnErr err = nullptr;
};

NcclLib& nccl() {
  static NcclLib lib;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      lib.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (lib.h) break;
    }
    if (!lib.h) return;
    lib.get_id = (FnGetId)dlsym(lib.h, "ncclGetUniqueId");
    lib.init = (FnInit)dlsym(lib.h, "ncclCommInitRank");
    lib.all_reduce = (FnAllReduce)dlsym(lib.h, "ncclAllReduce");
    lib.destroy = (FnDestroy)dlsym(lib.h, "ncclCommDestroy");
    lib.err = (FnErr)dlsym(lib.h, "ncclGetErrorString");
  });
  if (!lib.h || !lib.get_id || !lib.init || !lib.all_reduce)
    throw Error(ABD_ERR_ARG, "NCCL (libnccl.so.2) is not available in this process");
  return lib;
}

void nccl_check(int r, const char* what) {
  if (r != 0) {
    const char* m = nccl().err ? nccl().err(r) : "?";
    throw Error(ABD_ERR_CUDA, std::string("NCCL ") + what + " failed: " + m);
  }
}

}  // namespace

void comm_get_nccl_id(void* out128) {
  NcclId id;
  nccl_check(nccl().get_id(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

void comm_init_nccl(Scene& s, const void* id128, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(ABD_ERR_ARG, "bad rank / world size");
  comm_destroy(s);
  if (world > 1) {
    NcclId id;
    std::memcpy(&id, id128, sizeof(id));
    NcclComm c = nullptr;
    nccl_check(nccl().init(&c, world, id, rank), "ncclCommInitRank");
    s.comm.nccl = c;
    s.comm.kind = 1;
  }
  s.comm.rank = rank;
  s.comm.world = world;
}

void comm_init_callback(Scene& s, int rank, int world, abd_allreduce_fn fn, void* user) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(ABD_ERR_ARG, "bad rank / world size");
  if (world > 1 && !fn) throw Error(ABD_ERR_ARG, "callback required for world > 1");
  comm_destroy(s);
  s.comm.rank = rank;
  s.comm.world = world;
  s.comm.kind = world > 1 ? 2 : 0;
  s.comm.cb = fn;
  s.comm.user = user;
}

void comm_destroy(Scene& s) {
  if (s.comm.kind == 1 && s.comm.nccl) {
    NcclLib& l = nccl();
    if (l.destroy) l.destroy(s.comm.nccl);
  }
  s.comm = Comm{};
}

// dtype: 0 = f64, 1 = i32, 2 = i64; op: 0 = sum, 1 = min, 2 = max
void comm_allreduce(Scene& s, void* dptr, int64_t count, int dtype, int op) {
  if (s.comm.world <= 1 || count <= 0) return;
  if (s.comm.kind == 1) {
    const int nd = dtype == 0 ? kNcclFloat64 : (dtype == 1 ? kNcclInt32 : kNcclInt64);
    const int no = op == 0 ? kNcclSum : (op == 1 ? kNcclMin : kNcclMax);
    nccl_check(nccl().all_reduce(dptr, dptr, (size_t)count, nd, no, s.comm.nccl, s.stream), "ncclAllReduce");
    return;
  }
  SSYNC(s.stream);
  int rc = s.comm.cb(s.comm.user, dptr, count, dtype, op);
  if (rc != 0) throw Error(ABD_ERR_CUDA, "collective callback failed");
}

// kernels for the partitioned step
__global__ void k_scatter_slot(int64_t n, const int64_t* __restrict__ src, int64_t* dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}

// all ranks' variable-length int64 lists -> one list on every rank (allreduce-sum of
// rank slots: works with any allreduce-only backend); returns the total count
int64_t comm_allgather_i64(Scene& s, const int64_t* local, int64_t n_local, DVec<int64_t>& out) {
  const int W = s.comm.world;
  if (W <= 1) {
    out.resize(std::max<int64_t>(n_local, 1));
    if (n_local) CK(cudaMemcpyAsync(out.p, local, n_local * sizeof(int64_t), cudaMemcpyDeviceToDevice, s.stream));
    return n_local;
  }
  // counts
  DVec<int64_t>& cnt = s.w.comm_cnt;
  cnt.resize(W);
  cnt.zero(s.stream);
  dev_set_i64(s.stream, cnt.p + s.comm.rank, n_local);
  comm_allreduce(s, cnt.p, W, 2, 0);
  std::vector<int64_t> hc(W);
  cnt.download(hc.data(), W, s.stream);
  SSYNC(s.stream);
  int64_t mx = 0, tot = 0;
  for (int64_t c : hc) mx = std::max(mx, c), tot += c;
  DVec<int64_t>& buf = s.w.comm_buf;
  buf.resize(std::max<int64_t>(W * mx, 1));
  buf.zero(s.stream);
  if (n_local)
    CK(cudaMemcpyAsync(buf.p + s.comm.rank * mx, local, n_local * sizeof(int64_t), cudaMemcpyDeviceToDevice,
                       s.stream));
  comm_allreduce(s, buf.p, W * mx, 2, 0);
  out.resize(std::max<int64_t>(tot, 1));
  int64_t at = 0;
  for (int r = 0; r < W; ++r) {
    if (hc[r])
      CK(cudaMemcpyAsync(out.p + at, buf.p + r * mx, hc[r] * sizeof(int64_t), cudaMemcpyDeviceToDevice, s.stream));
    at += hc[r];
  }
  return tot;
}

// Slabs: dynamic bodies sorted by (p[axis], id), axis = longest extent of their
// positions; slab k takes the bodies whose primitive-weight midpoint falls in
// [k/W, (k+1)/W) of the total: owner = floor((2 cum - w) W / (2 total)) in integers.
void slab_partition(Scene& s, const double* q) {
  const int W = s.comm.world, B = s.B;
  s.slab_valid = false;
  if (W <= 1) return;
  if ((int)s.h_prim_w.size() != B) {
    std::vector<int> vo(B + 1), eo(B + 1), to(B + 1);
    s.v_off.download(vo.data(), B + 1, s.stream);
    s.e_off.download(eo.data(), B + 1, s.stream);
    s.t_off.download(to.data(), B + 1, s.stream);
    SSYNC(s.stream);
    s.h_prim_w.resize(B);
    for (int b = 0; b < B; ++b) s.h_prim_w[b] = (vo[b + 1] - vo[b]) + (eo[b + 1] - eo[b]) + (to[b + 1] - to[b]);
  }
  std::vector<double> hq(12 * (size_t)B);
  CK(cudaMemcpyAsync(hq.data(), q, hq.size() * sizeof(double), cudaMemcpyDeviceToHost, s.stream));
  SSYNC(s.stream);
  std::vector<int> idx;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int b = 0; b < B; ++b)
    if (s.h_dyn[b]) {
      idx.push_back(b);
      for (int k = 0; k < 3; ++k) lo[k] = std::min(lo[k], hq[12 * (size_t)b + k]), hi[k] = std::max(hi[k], hq[12 * (size_t)b + k]);
    }
  int axis = 0;
  for (int k = 1; k < 3; ++k)
    if (hi[k] - lo[k] > hi[axis] - lo[axis]) axis = k;
  std::sort(idx.begin(), idx.end(), [&](int a, int b) {
    const double pa = hq[12 * (size_t)a + axis], pb = hq[12 * (size_t)b + axis];
    return pa != pb ? pa < pb : a < b;
  });
  int64_t total = 0;
  for (int b : idx) total += s.h_prim_w[b];
  s.h_slab_owner.assign(B, -1);
  int64_t cum = 0;
  for (int b : idx) {
    const int64_t w = s.h_prim_w[b];
    cum += w;
    s.h_slab_owner[b] = total > 0 ? (int)std::min<int64_t>((2 * cum - w) * W / (2 * total), W - 1) : 0;
  }
  std::vector<int> own_slot(std::max(s.n_dyn, 1), 0);
  for (int k = 0; k < s.n_dyn; ++k) own_slot[k] = s.h_slab_owner[s.h_dyn_body[k]] == s.comm.rank ? 1 : 0;
  s.slab_owner.upload(s.h_slab_owner.data(), B, s.stream);
  s.slab_own_slot.upload(own_slot.data(), std::max(s.n_dyn, 1), s.stream);
  s.slab_axis = axis;
  s.slab_valid = true;
}

__global__ void k_slab_mask(int64_t n_off, const int2* __restrict__ keys, const int* __restrict__ own, int* flags) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_off) return;
  const int2 k = keys[i];
  if (!own[k.x] || !own[k.y]) flags[i] = 0;
}

void slab_mask_structure(Scene& s, int* flags) {
  if (!s.slab_valid || s.H.n_off == 0) return;
  k_slab_mask<<<grid_for(s.H.n_off, 256), 256, 0, s.stream>>>(s.H.n_off, s.H.upper_keys.p, s.slab_own_slot.p, flags);
  note_launch("k_slab_mask");
}

}  // namespace abd
