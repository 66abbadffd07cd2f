// Device-resident scene context: geometry SoA, per-step state, work buffers.
// Host-side C++ (no torch types); see DESIGN.md "Data layout in HBM".
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <initializer_list>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/abd_b200.h"

namespace abd {

// ---------------------------------------------------------------------------
// errors: C++ exceptions inside the library, mapped to status codes at the
// C-ABI boundary (capi.cu) together with a thread-local message.
struct Error : std::runtime_error {
  int code;
  int64_t index;
  Error(int c, const std::string& m, int64_t idx = -1) : std::runtime_error(m), code(c), index(idx) {}
};

void cuda_check(cudaError_t e, const char* what);
#define CK(x) ::abd::cuda_check((x), #x)

// stream sync through one choke point: with ABD_HOST_PROF set, the host time
// since the previous sync (issue + host work) and the time blocked in the sync
// are accumulated per call site and printed by host_prof_dump()
void host_sync(cudaStream_t st, const char* site);
// store one scalar on the device in stream order (a kernel argument: no pageable
// host->device copy, which may serialise with the stream)
void dev_set_u64(cudaStream_t st, unsigned long long* p, unsigned long long v);
void dev_set_i32(cudaStream_t st, int* p, int v);
void dev_set_i64(cudaStream_t st, int64_t* p, int64_t v);
// gather small device scalars into pinned host memory with ONE kernel (the
// kernel stores straight into the UVA-mapped pinned buffer): replaces a
// series of tiny cudaMemcpyAsync D2H copies before a host sync.
// bytes and dst_off are multiples of 4.
struct PackItem {
  const void* src;
  int bytes;
  int dst_off;
};
void pack_to_host(cudaStream_t st, void* host_dst, std::initializer_list<PackItem> items);
void host_prof_dump();
void host_prof_reset();
#define ABD_STR2(x) #x
#define ABD_STR(x) ABD_STR2(x)
#define SSYNC(st) ::abd::host_sync((st), __FILE__ ":" ABD_STR(__LINE__))
void host_mark(const char* site);  // host time since the previous sync / mark (ABD_HOST_PROF)
#define HMARK() ::abd::host_mark(__FILE__ ":" ABD_STR(__LINE__))

// growable device vector (never shrinks; contents undefined after grow)
template <class T>
struct DVec {
  T* p = nullptr;
  size_t n = 0, cap = 0;
  DVec() = default;
  DVec(const DVec&) = delete;
  DVec& operator=(const DVec&) = delete;
  ~DVec() {
    if (p) cudaFree(p);
  }
  void resize(size_t m) {
    if (m > cap) {
      // 2x headroom: workspaces grow in a handful of steps and then stay put
      // (cudaFree synchronises the device, so steady-state regrowth would stall)
      if (p) CK(cudaFree(p));
      size_t c = 2 * m + 16;
      CK(cudaMalloc(&p, c * sizeof(T)));
      cap = c;
    }
    n = m;
  }
  void upload(const T* h, size_t m, cudaStream_t s) {
    resize(m);
    if (m) CK(cudaMemcpyAsync(p, h, m * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void download(T* h, size_t m, cudaStream_t s) const {
    if (m) CK(cudaMemcpyAsync(h, p, m * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
  void zero(cudaStream_t s) {
    if (n) CK(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
};

// growable pinned host buffer (never shrinks)
template <class T>
struct HostPinned {
  T* p = nullptr;
  size_t cap = 0;
  HostPinned() = default;
  HostPinned(const HostPinned&) = delete;
  HostPinned& operator=(const HostPinned&) = delete;
  ~HostPinned() {
    if (p) cudaFreeHost(p);
  }
  T* reserve(size_t m) {
    if (m > cap) {
      if (p) CK(cudaFreeHost(p));
      size_t c = 2 * m + 64;
      CK(cudaMallocHost(&p, c * sizeof(T)));
      cap = c;
    }
    return p;
  }
};

struct Cands {
  DVec<int4> vf, ee;  // (body_a, prim_a, body_b, prim_b) in canonical order
  DVec<int2> ov;      // overlapping body pairs (i < j)
  int64_t n_vf = 0, n_ee = 0, n_ov = 0;
  bool ov_matches_pattern = false;  // ov equals the overlap list of the resident BSR pattern
  int64_t gen = 0;                  // bumped whenever the resident candidate set is rewritten
};

// lagged friction records (compact form of contact.py:687-708)
struct FrictionSet {
  DVec<int2> bodies;      // (body_a, body_b)
  DVec<double> rec;       // 17 doubles per pair: T(6) c(8) off(2) lam(1)
  int64_t n = 0;
  int64_t n_pattern = 0;  // all ranks' pairs (multi-GPU BSR pattern)
  int64_t gen = 0;        // bumped whenever the friction set changes
  double mu = 0.0;
};

// per-active-pair records (PairBlocks restated): compact g24 | type | low-rank
// factors (abd_pblk.cuh); PB_DENSE = g24 | haa | hbb | hab for dense readout
constexpr int PB_STRIDE = 136;
constexpr int PB_DENSE = 24 + 3 * 144;
constexpr int RUN_STRIDE = 456;  // run partial: aa 144 | bb 144 | ab 144 | ga 12 | gb 12 (reference DOFs)

struct PairBlockSet {
  DVec<int2> bodies;  // (-1, -1) for pairs folded into a run partial
  DVec<double> blk;  // PB_STRIDE per pair
  DVec<double> d2;
  int64_t n = 0;
  // fused assembly of large active sets (k_pair_runs): per run of consecutive active
  // pairs of one body pair (within a 32-pair window) its summed blocks and gradients
  DVec<int2> run_bodies;
  DVec<double> run_part;  // RUN_STRIDE per run
  DVec<int> run_wcount, run_wbase;
  int64_t n_runs = 0;
};

// symmetric BSR over dynamic slots, stored in full (both triangles) CSR
struct Bsr {
  int n = 0;                 // block rows
  int64_t nnzb = 0;          // stored blocks (diag + 2 * n_off)
  int64_t n_off = 0;         // upper off-diagonal blocks
  DVec<int> row_ptr;         // n + 1
  DVec<int> col;             // nnzb
  DVec<double> val;          // nnzb * 144
  DVec<int> diag_pos;        // n: position of the diagonal block
  DVec<int2> upper_keys;     // n_off (i < j) sorted
  DVec<int> upper_pos;       // position of (i,j)
  DVec<int> lower_pos;       // position of (j,i)
};

struct Stats;  // driver statistics (driver.cu)

// multi-GPU communicator (comm.cu): kind 0 = single process, 1 = NCCL, 2 = host callback
struct Comm {
  int rank = 0, world = 1, kind = 0;
  void* nccl = nullptr;
  abd_allreduce_fn cb = nullptr;
  void* user = nullptr;
};

struct Scene {
  int B = 0, n_dyn = 0;
  // host-side readout permutations into the reference's record order (capi.cu)
  std::vector<int64_t> pblk_order, fric_order;
  int64_t fric_order_gen = -1;
  int64_t V = 0, E = 0, T = 0;
  int max_v = 0, max_e = 0, max_t = 0;  // per-body primitive maxima (sort key widths)
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;            // forked work that overlaps the main stream (event-joined)
  cudaStream_t main_stream = nullptr;     // == stream, never swapped (used by the analysis worker thread)
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  cudaStream_t side2 = nullptr;  // early ACCD of the hot queries (overlaps the broad phase)
  cudaEvent_t hot_fork_ev = nullptr, hot_ev = nullptr;
  cudaEvent_t pb_fork_ev = nullptr, pb_ev = nullptr;  // VF pair blocks on side2
  cudaStream_t side3 = nullptr;  // mollified EE pair blocks beside the plain EE pairs
  // Cholesky plan uploads (issued by the analysis worker): on their own stream, so the copy
  // does not queue between the main stream's kernels; chol_begin waits on plan_ev
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t plan_ev = nullptr;
  bool plan_pending = false;
  cudaStream_t side4 = nullptr;  // Cholesky: isolated nodes beside the coupled task graph
  cudaEvent_t ch_fork_ev = nullptr, ch_join_ev = nullptr;
  cudaEvent_t moll_fork_ev = nullptr, moll_ev = nullptr;
  int num_sms = 148;

  // geometry (immutable after create)
  DVec<int> v_off, e_off, t_off;  // B + 1
  DVec<double> rest;              // V * 3
  DVec<int> edges;                // E * 2 (global vertex ids)
  DVec<int> tris;                 // T * 3 (global vertex ids)
  // static primitive groups for the broad phase cull (bodies with <= 256 vertices):
  // per kind (0 vertex, 1 edge, 2 triangle) the body's primitives in rest-space
  // Morton order, in groups of 32: local ids, packed local vertex ids (8 bits each),
  // per-group rest AABB (centre, half extent) and per-body group offsets
  bool has_groups = false;
  DVec<int> grp_id[3];
  DVec<unsigned> grp_pk[3];
  DVec<double> grp_box[3];
  DVec<int> grp_off[3];  // B + 1
  DVec<double> elen2;             // E
  DVec<int> vert_body, edge_body, tri_body;
  DVec<unsigned char> dyn;        // B
  DVec<int> slot;                 // B (dynamic slot or -1)
  DVec<int> dyn_body;             // n_dyn
  DVec<double> mass;              // B * 144 (full 12x12, zero for kinematic)
  DVec<double> stiff;             // B
  std::vector<int> h_slot, h_dyn_body;
  std::vector<unsigned char> h_dyn;

  // state
  DVec<double> q, q0, q_dot, q_tilde, dq, q_trial, forces;

  // broad / narrow phase
  Cands cands;
  FrictionSet fric;
  PairBlockSet pblk;

  // assembly / solve
  Bsr H;
  DVec<double> grad, dx;  // n_dyn * 12

  // scratch
  DVec<unsigned char> tmp_bytes;
  DVec<int> tmp_i0, tmp_i1, tmp_i2, tmp_i3;
  DVec<int64_t> tmp_l0, tmp_l1, tmp_l2, tmp_l3;
  DVec<double> tmp_d0, tmp_d1, tmp_d2, tmp_d3;
  DVec<double> red;  // reduction partials
  double* h_pinned = nullptr;  // small pinned staging for scalars
  DVec<double> vbox;  // V * 6 vertex boxes (broad phase)
  DVec<double> bbox;  // B * 6 body boxes
  DVec<double> body_rmax;  // B * 3: max |rest coordinate| per axis (primitive Verlet-list bound)

  // persistent workspaces (grown, never shrunk: no cudaMalloc in steady state)
  struct Work {
    // host scratch of the Cholesky analysis (reused: no allocations in the steady state)
    std::vector<int> hs_i[40];
    // ACCD hot list: the slowest queries (>= CCD_SLOW_IT iterations) of the previous
    // line search, re-evaluated right after the solve on side2 while the broad phase runs
    DVec<int4> hot_rows, slow_rows;
    DVec<int> hot_kind, slow_kind, hot_bad, hot_it;
    DVec<double> hot_t;
    int hot_n = 0;
    bool hot_pending = false;
    std::vector<char> hs_c[2];
    DVec<int64_t> comm_cnt, comm_buf, fric_keys, fric_keys_all;  // multi-GPU scratch
    DVec<int> act;      // compacted active candidate indices (VF then EE)
    DVec<int> moll;     // active EE slots with an active mollifier (deferred 9-column path)
    DVec<unsigned char> moll_flag;  // per active EE slot: mollified (k_moll_classify, read by k_pair_blocks_act)
    int64_t n_act_vf = 0;
    DVec<int> flags, pos, err, order, cnt, off, seg_s, seg_e, row_of, nsel, bad, iters;
    DVec<uint64_t> k0, k1, e0, e1;
    DVec<uint32_t> ka, kb;
    DVec<int> va, vb;
    DVec<int4> rows_tmp, rows_tmp2;
    DVec<int2> tab;  // broad phase (pair, product) -> (chunk start, count)
    // overlap list / friction generation of the resident BSR pattern (build_pattern reuse)
    DVec<int2> pat_ov;
    int64_t pat_n_ov = -1, pat_n_f = -1, pat_fric_gen = -1;
    bool pat_valid = false;
    DVec<int2> pairs_tmp;
    // body-pair superset ("Verlet list"): canonical (i, j) pairs whose boxes inflated
    // by a margin overlap; each broad phase filters it with the exact swept boxes and
    // rebuilds it only when a body's box leaves its inflated box
    DVec<double> vl_box;
    DVec<int2> vl_pairs;
    int64_t vl_n = 0;
    bool vl_valid = false;
    int vl_gen = 0;
    double vl_cell = 0.0;
    double vl_h = -1.0;  // vertex-box inflation the superset was built for
    double gmd_prev = 0.0;  // last end-of-step global minimum distance (first inflation guess)
    // primitive-pair superset ("primitive Verlet list"): the candidate rows of the body
    // superset for vertex boxes inflated by pvl_m, built for the sweep [pvl_q0, pvl_q1];
    // valid while every body stays within pvl_m / 2 of that sweep (k_pvl_check)
    DVec<int4> pvl_vf, pvl_ee;
    int64_t pvl_nvf = 0, pvl_nee = 0;
    DVec<double> pvl_q0, pvl_q1;
    DVec<int> pvl_flags;
    double pvl_m = 0.0, pvl_h = -1.0;
    int pvl_gen = -1;
    bool pvl_valid = false;
    DVec<unsigned long long> ull;   // small atomics scratch (8 slots)
    DVec<double> grad0, diag0, neg, pinv, r, z, p, p2, Ap, part, scal, basis;
    DVec<double> lsred, lsscal;  // merged CCD + e0 + first-trial line-search reductions
    DVec<int> lserr;
    DVec<double> cg_u, cg_w, cg_m, cg_q;
    // cluster block-Jacobi preconditioner (k_cg.cu)
    DVec<int> cl_slot_row, cl_slot_base, cl_slot_k, cl_off, cl_rows;
    DVec<long long> cl_slot_off, cl_minv;
    DVec<double> minv;
    // sparse block Cholesky plan (one packed int buffer) and factor (k_chol.cu)
    DVec<int> ch_flags, ch_plan, ch_apos, ch_dep, ch_bleft, ch_queue, ch_dleft, ch_bgate;
    DVec<double> ch_scratch;  // partial sums of split factor tasks
    DVec<unsigned> ch_ctr;
    DVec<int> ch_fl;   // k_chol_flow readiness flags (L blocks, x, parent-block sums)
    DVec<double> ch_sbuf;  // k_chol_flow parent-block update sums (n x 144)
    int ch_epoch = 0;  // k_chol_flow launches so far (the flag value of the next one is + 1)
    DVec<double> ch_L, ch_dinv;
    HostPinned<int> h_plan, h_meta;
    // last analysed pattern (nonzero flags + keys) and its plan: Newton iterations
    // whose coupling pattern is unchanged reuse the resident plan
    struct CholCache {
      bool valid = false;
      int n = 0;
      int64_t n_off = 0;
      std::vector<uint64_t> edges;  // (i << 32 | j) nonzero couplings the plan was built for
      int64_t stats[12] = {};
      size_t offs[32] = {};
      int64_t hits = 0, misses = 0;
      std::vector<int> gorder;  // elimination order (global ids) of the step's last fresh ordering
      int64_t fresh_nnz = 0;    // its off-diagonal factor blocks
      int64_t fresh_upd = 0;    // and update pairs
    } ch_cache;
    std::vector<uint64_t> ch_edges_cur;
    // structure flags + keys copied out by assemble() (event-ordered); consumed once
    bool ch_pre = false;
    // the next iteration's structure was marked at the accepted line-search trial
    // and its analysis posted early (mark_structure then has nothing to do)
    bool ch_early = false;
    cudaEvent_t ch_pre_ev = nullptr;
    // actual structure of an iteration whose analysis was posted early (at the first
    // line-search trial): checked against the plan in chol_begin
    DVec<int> ch_flags2;
    HostPinned<int> h_meta2;
    cudaEvent_t ch_act_ev = nullptr;
    bool ch_verify = false;
    DVec<double> q_pred;       // speculated next iterate (q + alpha_prev dq)
    double alpha_prev = 1.0;   // the last accepted line-search step
    // an in-flight chol_begin awaiting chol_finish
    struct CholRun {
      bool active = false;
      const double* rhs = nullptr;
      double* x = nullptr;
      int n_cta = 0;
      int64_t stats[8] = {};
      double host_ms = 0.0, ms3[3] = {};
    } ch_run;
  } w;

  Comm comm;
  // body-slab partition of a multi-rank scene (comm.cu slab_partition, once per step):
  // owner rank per body (-1 kinematic), owned flag per dynamic slot
  DVec<int> slab_owner, slab_own_slot;
  std::vector<int> h_slab_owner, h_prim_w;
  int slab_axis = 0;
  bool slab_valid = false;

  // joint reduction q_dyn = T u + q_const (constraints.py): dense T (12 n_dyn x red_nu),
  // red_nu = 0 without joints; workspaces of the reduced solve (k_reduced.cu)
  int64_t red_nu = 0;
  DVec<double> red_T, red_W, red_X, red_A, red_v;

  // per-kernel instrumentation (CUDA events on `stream`)
  struct KStat {
    int64_t launches = 0, units = 0;
    double ms = 0.0, bytes = 0.0;
    // lazily resolved timing of the last launch (its own event pair, no extra sync)
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    bool pending = false;
    int64_t p_units = 0;
    double p_bytes = 0.0;
  } kstat[4];
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, tev0 = nullptr, tev1 = nullptr;
  bool instrument = true;

  // host worker thread of the Cholesky analysis (k_chol.cu); stopped first on destruction
  std::shared_ptr<void> chol_worker;
  Scene();
  ~Scene();
};

// ---------------------------------------------------------------------------
// cub wrappers (scene.cu)
void scan_exclusive_i32(Scene& s, const int* in, int* out, int64_t n);
void sort_pairs_u64(Scene& s, uint64_t* keys, uint64_t* keys_alt, int* vals, int* vals_alt, int64_t n,
                    int end_bit, bool& result_in_alt);
void sort_pairs_u32(Scene& s, uint32_t* keys, uint32_t* keys_alt, int* vals, int* vals_alt, int64_t n, int end_bit,
                    bool& result_in_alt);
double reduce_sum_det(Scene& s, const double* partials, int n);  // deterministic
void kstat_flush(Scene& s, int which);  // resolve a pending lazily-timed launch

inline int grid_for(int64_t n, int block) { return (int)((n + block - 1) / block); }
int bits_for(int64_t maxval);

}  // namespace abd
