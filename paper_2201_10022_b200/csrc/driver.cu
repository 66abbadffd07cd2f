// Scene-level operations and the Newton driver (solver.py:179-628) with
// device-resident state.  Per Newton iteration only a handful of scalars
// cross to the host (candidate counts, |dq|_inf and g.dq, alpha_max, one
// energy per line-search trial); all buffers are persistent workspaces.
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <vector>

#include "driver.h"

namespace abd {

// ---------------------------------------------------------------------------
// small helper kernels
__global__ void k_absmax_dot(int64_t n, const double* __restrict__ x, const double* __restrict__ g,
                             unsigned long long* amax, double* partials) {
  __shared__ double sh[RED_THREADS];
  double m = 0.0, acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    m = fmax(m, fabs(x[i]));
    acc += g[i] * x[i];
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(amax, (unsigned long long)__double_as_longlong(m));
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

// trial q + alpha0 dq with alpha0 from the device CCD minimum (solver.py:375-376):
// alpha_max = min(1, t_min); alpha0 = 1 if alpha_max >= 1 else min(1, scale alpha_max)
__global__ void k_alpha_trial(int64_t n, const double* __restrict__ q, const double* __restrict__ dq,
                              const unsigned long long* __restrict__ tmin, double scale, double* out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double amax = fmin(1.0, __longlong_as_double((long long)*tmin));
  const double alpha = amax >= 1.0 ? 1.0 : fmin(1.0, scale * amax);
  out[i] = xadd(q[i], xmul(alpha, dq[i]));
}

// dq over all bodies: sign * dx for dynamic bodies, 0 for static ones (no memset)
__global__ void k_expand_dq(int B, const int* __restrict__ slot, const double* __restrict__ dx, double sign,
                            double* dq) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 12 * (int64_t)B) return;
  const int k = slot[t / 12];
  dq[t] = k >= 0 ? sign * dx[12 * (int64_t)k + t % 12] : 0.0;
}

__global__ void k_qdot(int B, const unsigned char* __restrict__ dyn, const double* __restrict__ q,
                       const double* __restrict__ q0, double dt, double* qd) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 12 * (int64_t)B) return;
  int b = (int)(t / 12);
  qd[t] = dyn[b] ? (q[t] - q0[t]) / dt : 0.0;
}

__global__ void k_neg(int64_t n, const double* __restrict__ a, double* b) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = -a[i];
}

void launch_neg(cudaStream_t st, int64_t n, const double* a, double* b) {
  if (n <= 0) return;
  k_neg<<<grid_for(n, 256), 256, 0, st>>>(n, a, b);
  note_launch("k_neg");
}

// per dynamic body ||A A^T - I||_F (ortho_error, body.py:216-220), max via bits
__global__ void k_ortho_err(int n_dyn, const int* __restrict__ dyn_body, const double* __restrict__ q,
                            unsigned long long* out) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  double e = 0.0;
  if (s < n_dyn) {
    const double* A = q + 12 * (int64_t)dyn_body[s] + 3;
    double acc = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double g = A[3 * i] * A[3 * j] + A[3 * i + 1] * A[3 * j + 1] + A[3 * i + 2] * A[3 * j + 2] - (i == j ? 1.0 : 0.0);
        acc += g * g;
      }
    e = sqrt(acc);
  }
  for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(e));
}

// ---------------------------------------------------------------------------
static double bits_to_d(unsigned long long b) { return __builtin_bit_cast(double, b); }
static unsigned long long d_to_bits(double d) { return (unsigned long long)__builtin_bit_cast(long long, d); }

// per-kernel event timing on the scene stream, resolved lazily (kstat_flush) at
// the next use of the same slot or when the stats are read: no extra host sync
struct EventTimer {
  Scene& s;
  int which;
  bool on;
  EventTimer(Scene& sc, int w) : s(sc), which(w), on(sc.instrument) {
    if (!on) return;
    kstat_flush(s, which);
    CK(cudaEventRecord(s.kstat[which].e0, s.stream));
  }
  void done(int64_t units, double bytes) {
    if (!on) return;
    Scene::KStat& k = s.kstat[which];
    k.pending = true;
    k.p_units = units;
    k.p_bytes = bytes;
  }
  void stop() {
    if (on) CK(cudaEventRecord(s.kstat[which].e1, s.stream));
  }
};

static void mark_structure(Scene& s);
static void mark_structure_early(Scene& s, const double* q, double dh, bool on_main = false);

// flags + exclusive scan of candidate activity (d^2 < d_hat^2) into s.w.flags/pos;
// returns the active count (one host sync, also checks the barrier domain)
static int active_scan(Scene& s, const double* q, double dh) {
  int64_t n_vf = s.cands.n_vf, n_ee = s.cands.n_ee;
  int64_t n = n_vf + n_ee;
  Scene::Work& w = s.w;
  w.flags.resize(n + 1);
  w.pos.resize(n + 1);
  w.err.resize(2);
  w.err.zero(s.stream);
  double dh2 = dh * dh;
  launch_pair_flags_both(s, q, dh2, w.flags.p, w.err.p);
  scan_exclusive_i32(s, w.flags.p, w.pos.p, n + 1);
  // compacted active list: act[pos[i]] = i (VF slots first, then EE)
  w.act.resize(n + 1);
  launch_scatter_active(s, n, w.flags.p, w.pos.p, w.act.p);
  comm_allreduce(s, w.err.p, 1, 1, 2);  // a domain error on any rank stops every rank
  int* hp = reinterpret_cast<int*>(s.h_pinned);
  pack_to_host(s.stream, hp, {{w.pos.p + n, 4, 0}, {w.err.p, 4, 4}, {w.pos.p + n_vf, 4, 8}});
  SSYNC(s.stream);
  if (hp[1]) throw Error(ABD_ERR_BARRIER_DOMAIN, "barrier evaluated at non-positive squared distance "
                                                 "(intersection reached; CCD filtering must prevent this)");
  w.n_act_vf = hp[2];
  return hp[0];
}

// active sets at least this large take the fused run assembly (k_pair_runs) when the
// caller reduces into the system (assemble); ABD_RUNS=0/1 forces it off / on
static bool use_runs(int64_t total) {
  const char* e = getenv("ABD_RUNS");  // read per call: tests switch it inside one process
  return e ? atoi(e) != 0 : total >= (int64_t)1 << 20;
}

int64_t contact_blocks(Scene& s, const double* q, double kappa, double dh, int project, bool mark, bool allow_runs) {
  int64_t n_vf = s.cands.n_vf;
  int total = active_scan(s, q, dh);
  if (mark) mark_structure(s);
  s.pblk.bodies.resize(std::max(total, 1));
  s.pblk.blk.resize((int64_t)std::max(total, 1) * PB_STRIDE);
  s.pblk.d2.resize(std::max(total, 1));
  s.pblk.n = total;
  s.pblk.n_runs = 0;
  EventTimer tm(s, 1);
  (void)n_vf;
  if (allow_runs && total > 0 && use_runs(total)) {
    launch_pair_runs(s, q, kappa, dh, project, s.w.act.p, s.w.n_act_vf, total);
    tm.stop();
    // records stay on chip: candidate record + rest points read, one run partial written per run
    tm.done(total, 112.0 * (double)(s.cands.n_vf + s.cands.n_ee) + 8.0 * (double)s.cands.n_ee +
                       8.0 * RUN_STRIDE * (double)s.pblk.n_runs);
    return total;
  }
  // VF pairs on side2 beside the EE pairs (+ mollified EE) on the main stream
  const bool fork_vf = s.w.n_act_vf > 0 && total - s.w.n_act_vf > 0;
  if (fork_vf) {
    CK(cudaEventRecord(s.pb_fork_ev, s.stream));
    CK(cudaStreamWaitEvent(s.side2, s.pb_fork_ev, 0));
    std::swap(s.stream, s.side2);
  }
  launch_pair_blocks_act(s, KIND_VF, q, kappa, dh, project, s.w.act.p, 0, s.w.n_act_vf);
  if (fork_vf) {
    std::swap(s.stream, s.side2);
    CK(cudaEventRecord(s.pb_ev, s.side2));
  }
  launch_pair_blocks_act(s, KIND_EE, q, kappa, dh, project, s.w.act.p, s.w.n_act_vf, total - s.w.n_act_vf);
  if (fork_vf) CK(cudaStreamWaitEvent(s.stream, s.pb_ev, 0));
  tm.stop();
  // algorithmic bytes (scene form): candidate record 16 B + 4 rest points 96 B
  // (+ eps 8 B for EE) per candidate, one compact PB_STRIDE record written per active pair
  double bytes = 112.0 * (double)(s.cands.n_vf + s.cands.n_ee) + 8.0 * (double)s.cands.n_ee +
                 8.0 * PB_STRIDE * (double)total;
  tm.done(total, bytes);
  return total;
}

// append friction blocks of the resident friction set after the contact blocks
void append_friction_blocks(Scene& s, const double* q, double dt, double eps_v, int project) {
  int64_t nc = s.pblk.n, nf = s.fric.n;
  if (nf == 0) return;
  int64_t tot = nc + nf;
  if ((size_t)tot > s.pblk.bodies.cap || (size_t)tot * PB_STRIDE > s.pblk.blk.cap || (size_t)tot > s.pblk.d2.cap) {
    DVec<int2> b2;
    DVec<double> k2, d2;
    b2.resize(tot);
    k2.resize(tot * PB_STRIDE);
    d2.resize(tot);
    if (nc) {
      CK(cudaMemcpyAsync(b2.p, s.pblk.bodies.p, nc * sizeof(int2), cudaMemcpyDeviceToDevice, s.stream));
      CK(cudaMemcpyAsync(k2.p, s.pblk.blk.p, nc * PB_STRIDE * sizeof(double), cudaMemcpyDeviceToDevice, s.stream));
      CK(cudaMemcpyAsync(d2.p, s.pblk.d2.p, nc * sizeof(double), cudaMemcpyDeviceToDevice, s.stream));
    }
    SSYNC(s.stream);
    std::swap(s.pblk.bodies.p, b2.p);
    std::swap(s.pblk.bodies.cap, b2.cap);
    std::swap(s.pblk.blk.p, k2.p);
    std::swap(s.pblk.blk.cap, k2.cap);
    std::swap(s.pblk.d2.p, d2.p);
    std::swap(s.pblk.d2.cap, d2.cap);
  }
  s.pblk.bodies.n = tot;
  CK(cudaMemcpyAsync(s.pblk.bodies.p + nc, s.fric.bodies.p, nf * sizeof(int2), cudaMemcpyDeviceToDevice, s.stream));
  launch_friction(s.stream, nf, s.fric.bodies.p, s.fric.rec.p, s.fric.mu, q, s.dyn.p, dt, eps_v, project, nullptr,
                  nullptr, nullptr, s.pblk.blk.p + nc * PB_STRIDE);
  s.pblk.n = tot;
}

int64_t friction_precompute(Scene& s, const double* q, double kappa, double dh, double mu, DVec<double>* basis) {
  if (mu < 0) throw Error(ABD_ERR_ARG, "friction coefficient must be >= 0");
  int64_t n_vf = s.cands.n_vf;
  s.fric.mu = mu;
  int total = active_scan(s, q, dh);
  s.fric.n = total;
  s.fric.gen += 1;
  s.fric.bodies.resize(std::max(total, 1));
  s.fric.rec.resize((int64_t)std::max(total, 1) * FRIC_STRIDE);
  double* bp = nullptr;
  if (basis) {
    basis->resize((int64_t)std::max(total, 1) * 6);
    bp = basis->p;
  }
  launch_friction_pre(s, KIND_VF, q, kappa, dh, s.w.flags.p, s.w.pos.p, 0, bp);
  launch_friction_pre(s, KIND_EE, q, kappa, dh, s.w.flags.p + n_vf, s.w.pos.p + n_vf, 0, bp);
  if (s.comm.world > 1) {
    // every rank's friction body pairs enter the (replicated) BSR pattern
    static_assert(sizeof(int2) == sizeof(int64_t), "int2 packs into int64");
    s.fric.n_pattern = comm_allgather_i64(s, reinterpret_cast<const int64_t*>(s.fric.bodies.p), total,
                                          s.w.fric_keys_all);
  }
  return total;
}

// friction pairs entering the BSR pattern (all ranks' pairs when partitioned)
static const int2* fric_pattern(Scene& s, int64_t& n) {
  if (s.comm.world > 1) {
    n = s.fric.n_pattern;
    return reinterpret_cast<const int2*>(s.w.fric_keys_all.p);
  }
  n = s.fric.n;
  return s.fric.bodies.p;
}

// energy pieces as 4 fixed-order sums: body | contact VF | contact EE | friction
static void energy_terms(Scene& s, const double* q, const double* qt, double dt, double kappa, double dh,
                         double eps_v, double out[4]) {
  s.red.resize(4 * RED_BLOCKS);
  s.w.err.resize(2);
  s.w.err.zero(s.stream);
  s.w.scal.resize(4);
  launch_energy_all(s, q, qt, dt, kappa, dh, eps_v, s.red.p, s.w.err.p);
  reduce_fixed_multi(s.stream, s.red.p, RED_BLOCKS, 4, s.w.scal.p);
  comm_allreduce(s, s.w.scal.p, 4, 0, 0);
  comm_allreduce(s, s.w.err.p, 1, 1, 2);
  int* he = reinterpret_cast<int*>(s.h_pinned + 8);
  pack_to_host(s.stream, s.h_pinned, {{s.w.scal.p, 32, 0}, {s.w.err.p, 4, 64}});
  SSYNC(s.stream);
  if (he[0]) throw Error(ABD_ERR_BARRIER_DOMAIN, "barrier evaluated at non-positive squared distance "
                                                 "(intersection reached; CCD filtering must prevent this)");
  for (int k = 0; k < 4; ++k) out[k] = s.h_pinned[k];
}

double contact_energy(Scene& s, const double* q, double kappa, double dh) {
  double e[4];
  int64_t nf = s.fric.n;
  s.fric.n = 0;  // contact only
  try {
    energy_terms(s, q, q, 1.0, kappa, dh, 0.0, e);
  } catch (...) {
    s.fric.n = nf;
    throw;
  }
  s.fric.n = nf;
  return (0.0 + e[1]) + e[2];
}

double friction_energy(Scene& s, const double* q, double dt, double eps_v) {
  if (s.fric.n == 0) return 0.0;
  s.red.resize(RED_BLOCKS);
  launch_friction(s.stream, s.fric.n, s.fric.bodies.p, s.fric.rec.p, s.fric.mu, q, s.dyn.p, dt, eps_v, 0, s.red.p,
                  nullptr, nullptr, nullptr);
  return reduce_sum_det(s, s.red.p, RED_BLOCKS);
}

double body_energy(Scene& s, const double* q, const double* qt, double dt) {
  s.red.resize(RED_BLOCKS);
  launch_body_terms(s, q, qt, dt, nullptr, nullptr, s.red.p, 0);
  return reduce_sum_det(s, s.red.p, RED_BLOCKS);
}

// ip_value (solver.py:193-205): ((sum_b body_b) + ((0 + E_vf) + E_ee)) + E_f
double ip_value(Scene& s, const double* q, const double* qt, double dt, double kappa, double dh, double eps_v) {
  double e[4];
  energy_terms(s, q, qt, dt, kappa, dh, eps_v, e);
  double total = e[0];
  total += (0.0 + e[1]) + e[2];
  total += e[3];
  return total;
}

// energy pieces launched without a host sync: partials into red4 (4 x RED_BLOCKS),
// fixed-order sums into scal4[0..3], barrier-domain flag into err
static void launch_energy(Scene& s, const double* q, const double* qt, double dt, double kappa, double dh,
                          double eps_v, double* red4, double* scal4, int* err) {
  launch_energy_all(s, q, qt, dt, kappa, dh, eps_v, red4, err);
  reduce_fixed_multi(s.stream, red4, RED_BLOCKS, 4, scal4);
}

static double ip_combine(const double* e) {  // ((body + ((0 + vf) + ee)) + fric), solver.py:193-205
  double total = e[0];
  total += (0.0 + e[1]) + e[2];
  total += e[3];
  return total;
}

// CCD step bound, e0 = ip_value(q) and the first trial energy in ONE host sync
// (ccd.py:130-153, solver.py:358-393); returns alpha_max, alpha0, e0, e(alpha0)
struct LsFirst {
  double amax, alpha, e0, e, ccd_ms;
};
static LsFirst line_search_first(Scene& s, const abd_step_params& P, int64_t NB) {
  cudaStream_t st = s.stream;
  Scene::Work& w = s.w;
  unsigned long long* tmin = w.ull.p;
  w.lsred.resize(8 * RED_BLOCKS);
  w.lsscal.resize(8);
  w.lserr.resize(2);
  w.lserr.zero(st);
  unsigned long long one = d_to_bits(1.0);
  dev_set_u64(st, tmin, one);
  // e0 = ip_value(q) on the side stream, overlapping the CCD (whose runtime is a
  // heavy tail of a few long ACCD queries)
  CK(cudaEventRecord(s.fork_ev, st));
  CK(cudaStreamWaitEvent(s.side, s.fork_ev, 0));
  std::swap(s.stream, s.side);
  launch_energy(s, s.q.p, s.q_tilde.p, P.dt, P.kappa_barrier, P.d_hat, P.epsilon_v, w.lsred.p, w.lsscal.p,
                w.lserr.p + 1);
  std::swap(s.stream, s.side);
  CK(cudaEventRecord(s.join_ev, s.side));
  EventTimer tm(s, 2);
  launch_ccd_both(s, s.q.p, s.dq.p, P.ccd_slack, tmin, w.lserr.p, /*track=*/true);
  tm.stop();
  // partitioned: the global CCD bound (t >= 0: min of the bit patterns == min of the
  // values) before the trial point, so every rank evaluates its pairs at the same q_trial
  comm_allreduce(s, tmin, 1, 0, 1);
  CK(cudaStreamWaitEvent(st, s.join_ev, 0));
  k_alpha_trial<<<grid_for(NB, 256), 256, 0, st>>>(NB, s.q.p, s.dq.p, tmin, P.ccd_step_scale, s.q_trial.p);
  note_launch("k_alpha_trial");
  launch_energy(s, s.q_trial.p, s.q_tilde.p, P.dt, P.kappa_barrier, P.d_hat, P.epsilon_v,
                w.lsred.p + 4 * RED_BLOCKS, w.lsscal.p + 4, w.lserr.p + 1);
  // partitioned: energies and error flags over all ranks
  comm_allreduce(s, w.lsscal.p, 8, 0, 0);
  comm_allreduce(s, w.lserr.p, 2, 1, 2);
  double* hp = s.h_pinned + 32;
  pack_to_host(st, hp, {{tmin, 8, 0}, {w.lsscal.p, 64, 8}, {w.lserr.p, 8, 72}, {w.ull.p + 12, 4, 80}});
  SSYNC(st);
  {
    // this line search's slow queries are the next iteration's hot list
    const int n_slow = std::max(0, std::min<int>(*reinterpret_cast<const int*>(hp + 10), CCD_HOT_CAP));
    w.hot_rows.resize(CCD_HOT_CAP);
    w.hot_kind.resize(CCD_HOT_CAP);
    if (n_slow > 0) {
      CK(cudaMemcpyAsync(w.hot_rows.p, w.slow_rows.p, n_slow * sizeof(int4), cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(w.hot_kind.p, w.slow_kind.p, n_slow * sizeof(int), cudaMemcpyDeviceToDevice, st));
    }
    w.hot_n = n_slow;
  }
  const int* he = reinterpret_cast<const int*>(hp + 9);
  if (he[0]) throw Error(ABD_ERR_CCD_DOMAIN, "CCD query issued at non-positive initial distance");
  if (he[1]) throw Error(ABD_ERR_BARRIER_DOMAIN, "barrier evaluated at non-positive squared distance "
                                                 "(intersection reached; CCD filtering must prevent this)");
  int64_t nq = s.cands.n_vf + s.cands.n_ee;
  LsFirst r;
  r.ccd_ms = 0.0;
  if (s.instrument) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, s.kstat[2].e0, s.kstat[2].e1));
    r.ccd_ms = ms;
  }
  tm.done(nq, 112.0 * (double)nq + 192.0 * s.B);
  r.amax = std::fmin(1.0, bits_to_d(*reinterpret_cast<const unsigned long long*>(hp)));
  r.alpha = r.amax >= 1.0 ? 1.0 : std::fmin(1.0, P.ccd_step_scale * r.amax);
  r.e0 = ip_combine(hp + 1);
  r.e = ip_combine(hp + 5);
  // accepted first trial: the next iteration's coupling structure is that of q_trial;
  // when the next assemble keeps the BSR pattern (its overlap pairs are already in
  // it -- decided by this iteration's broad phase), mark it now and start the
  // analysis while the next iteration's activity scan, pair blocks and reduction run
  static const bool no_early = getenv("ABD_CHOL_NO_EARLY") != nullptr;
  const bool keeps_pattern = w.pat_valid && s.cands.ov_matches_pattern && s.H.n == s.n_dyn &&
                             w.pat_fric_gen == s.fric.gen && w.pat_n_f == s.fric.n;
  // also when the trial is rejected (speculation): the backtracked iterate's structure
  // is usually inside the union with the cached graph; chol_begin verifies it.  Unlike
  // the accepted-trial case this can change the plan (and rounding): ABD_CHOL_NO_SPECULATE
  static const bool no_spec = getenv("ABD_CHOL_NO_SPECULATE") != nullptr;
  if (!no_early && P.linear_solver != 1 && s.red_nu == 0 && s.n_dyn > 0 && s.comm.world == 1 && keeps_pattern &&
      (r.e < r.e0 || !no_spec) && !w.ch_early)
    mark_structure_early(s, s.q_trial.p, P.d_hat);
  return r;
}

double step_filter(Scene& s, const double* q, const double* dq, double slack) {
  unsigned long long* tmin = s.w.ull.p;
  s.w.err.resize(2);
  s.w.err.zero(s.stream);
  unsigned long long one = d_to_bits(1.0);
  dev_set_u64(s.stream, tmin, one);
  EventTimer tm(s, 2);
  launch_ccd_both(s, q, dq, slack, tmin, s.w.err.p);
  tm.stop();
  comm_allreduce(s, tmin, 1, 0, 1);
  comm_allreduce(s, s.w.err.p, 1, 1, 2);
  unsigned long long* hb = reinterpret_cast<unsigned long long*>(s.h_pinned);
  CK(cudaMemcpyAsync(hb, tmin, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s.stream));
  int* he = reinterpret_cast<int*>(s.h_pinned + 2);
  CK(cudaMemcpyAsync(he, s.w.err.p, sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  SSYNC(s.stream);
  if (he[0]) throw Error(ABD_ERR_CCD_DOMAIN, "CCD query issued at non-positive initial distance");
  int64_t nq = s.cands.n_vf + s.cands.n_ee;
  tm.done(nq, 112.0 * (double)nq + 192.0 * s.B);
  return std::fmin(1.0, bits_to_d(hb[0]));
}

double candidate_min_d2(Scene& s, const double* q) {
  unsigned long long* best = s.w.ull.p + 1;
  unsigned long long inf = d_to_bits(INFINITY);
  dev_set_u64(s.stream, best, inf);
  launch_cand_min_d2(s, KIND_VF, q, best);
  launch_cand_min_d2(s, KIND_EE, q, best);
  comm_allreduce(s, best, 1, 0, 1);  // d2 >= 0 (inf when empty): bit order == value order
  unsigned long long* hb = reinterpret_cast<unsigned long long*>(s.h_pinned);
  CK(cudaMemcpyAsync(hb, best, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s.stream));
  SSYNC(s.stream);
  return bits_to_d(hb[0]);
}

// coupling structure for the Cholesky analysis: pattern blocks touched by an
// active contact or a friction pair between two dynamic bodies (a superset of
// the nonzero blocks), marked by binary search in the sorted upper keys
__global__ void k_mark_active(int64_t n, const int2* __restrict__ bodies, const int* __restrict__ slot,
                              int64_t n_off, const int2* __restrict__ keys, int* flags) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int2 b = bodies[i];
  int sa = slot[b.x], sb = slot[b.y];
  if (sa < 0 || sb < 0 || sa == sb) return;
  int a = min(sa, sb), c = max(sa, sb);
  int64_t lo = 0, hi = n_off - 1;
  while (lo <= hi) {
    int64_t m = (lo + hi) >> 1;
    int2 k = keys[m];
    if (k.x < a || (k.x == a && k.y < c)) lo = m + 1;
    else if (k.x == a && k.y == c) {
      flags[m] = 1;
      return;
    } else hi = m - 1;
  }
}

__global__ void k_mark_active_rows(int64_t n, const int4* __restrict__ rows, const int* __restrict__ act,
                                   const int* __restrict__ slot, int64_t n_off, const int2* __restrict__ keys,
                                   int* flags) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || !act[i]) return;
  int4 r = rows[i];
  int sa = slot[r.x], sb = slot[r.z];
  if (sa < 0 || sb < 0 || sa == sb) return;
  int a = min(sa, sb), c = max(sa, sb);
  int64_t lo = 0, hi = n_off - 1;
  while (lo <= hi) {
    int64_t m = (lo + hi) >> 1;
    int2 k = keys[m];
    if (k.x < a || (k.x == a && k.y < c)) lo = m + 1;
    else if (k.x == a && k.y == c) {
      flags[m] = 1;
      return;
    } else hi = m - 1;
  }
}

// structure flags (active contact candidates + friction pairs) copied to the host
// right after the activity scan, so the host analysis overlaps the pair blocks
// structure at the accepted first trial q_trial (== the next iterate): marked on the
// side stream, flags only (the pattern -- and the upper keys already on the host --
// is kept, see line_search_first), then the analysis job is posted
static void mark_structure_early(Scene& s, const double* q, double dh, bool on_main) {
  Scene::Work& w = s.w;
  const int64_t n_off = s.H.n_off;
  if (!on_main) {
    CK(cudaEventRecord(s.fork_ev, s.stream));
    CK(cudaStreamWaitEvent(s.side, s.fork_ev, 0));
    std::swap(s.stream, s.side);
  }
  w.ch_flags.resize(std::max<int64_t>(n_off, 1));
  if (n_off) {
    w.ch_flags.zero(s.stream);
    launch_mark_active_q(s, q, dh * dh, w.ch_flags.p);
    if (s.fric.n) {
      k_mark_active<<<grid_for(s.fric.n, 256), 256, 0, s.stream>>>(s.fric.n, s.fric.bodies.p, s.slot.p, n_off,
                                                                   s.H.upper_keys.p, w.ch_flags.p);
      note_launch("k_mark_active");
    }
    int* hm = w.h_meta.reserve(3 * (size_t)n_off);
    CK(cudaMemcpyAsync(hm, w.ch_flags.p, n_off * sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  }
  if (!w.ch_pre_ev) CK(cudaEventCreateWithFlags(&w.ch_pre_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(w.ch_pre_ev, s.stream));
  if (!on_main) std::swap(s.stream, s.side);
  w.ch_pre = true;
  w.ch_early = true;
  chol_analysis_post(s);
}

// structure flags of the active candidates (activity flags w.flags) and friction pairs
static void mark_active_flags(Scene& s, int* flags) {
  const int64_t n_off = s.H.n_off;
  CK(cudaMemsetAsync(flags, 0, n_off * sizeof(int), s.stream));
  const int64_t n_vf = s.cands.n_vf, n_ee = s.cands.n_ee;
  if (n_vf)
    k_mark_active_rows<<<grid_for(n_vf, 256), 256, 0, s.stream>>>(n_vf, s.cands.vf.p, s.w.flags.p, s.slot.p, n_off,
                                                                  s.H.upper_keys.p, flags);
  if (n_ee)
    k_mark_active_rows<<<grid_for(n_ee, 256), 256, 0, s.stream>>>(n_ee, s.cands.ee.p, s.w.flags.p + n_vf, s.slot.p,
                                                                  n_off, s.H.upper_keys.p, flags);
  note_launch("k_mark_active_rows");
  if (s.fric.n) {
    k_mark_active<<<grid_for(s.fric.n, 256), 256, 0, s.stream>>>(s.fric.n, s.fric.bodies.p, s.slot.p, n_off,
                                                                 s.H.upper_keys.p, flags);
    note_launch("k_mark_active");
  }
}

static void mark_structure(Scene& s) {
  Scene::Work& w = s.w;
  if (w.ch_early) {
    // the analysis posted at the first line-search trial is in flight; the actual
    // structure goes to the host beside it, and chol_begin checks that the plan covers
    // it (a rejected trial's structure may not) before factoring
    w.ch_early = false;
    const int64_t n_off = s.H.n_off;
    if (n_off) {
      w.ch_flags2.resize(n_off);
      mark_active_flags(s, w.ch_flags2.p);
      int* hm2 = w.h_meta2.reserve((size_t)n_off);
      CK(cudaMemcpyAsync(hm2, w.ch_flags2.p, n_off * sizeof(int), cudaMemcpyDeviceToHost, s.stream));
    }
    if (!w.ch_act_ev) CK(cudaEventCreateWithFlags(&w.ch_act_ev, cudaEventDisableTiming));
    CK(cudaEventRecord(w.ch_act_ev, s.stream));
    w.ch_verify = true;
    chol_verify_post(s);  // the worker checks (and re-analyses) beside the pair blocks
    return;
  }
  const int64_t n_off = s.H.n_off;
  w.ch_flags.resize(std::max<int64_t>(n_off, 1));
  if (n_off) {
    mark_active_flags(s, w.ch_flags.p);
    comm_allreduce(s, w.ch_flags.p, n_off, 1, 2);  // union of the ranks' couplings
    slab_mask_structure(s, w.ch_flags.p);          // multi-rank: this slab's block only
    int* hm = w.h_meta.reserve(3 * (size_t)n_off);
    CK(cudaMemcpyAsync(hm, w.ch_flags.p, n_off * sizeof(int), cudaMemcpyDeviceToHost, s.stream));
    CK(cudaMemcpyAsync(hm + n_off, s.H.upper_keys.p, n_off * sizeof(int2), cudaMemcpyDeviceToHost, s.stream));
  }
  if (!w.ch_pre_ev) CK(cudaEventCreateWithFlags(&w.ch_pre_ev, cudaEventDisableTiming));
  CK(cudaEventRecord(w.ch_pre_ev, s.stream));
  w.ch_pre = true;
  chol_analysis_post(s);
}

void assemble(Scene& s, const double* q, const double* qt, double dt, double kappa, double dh, double eps_v,
              double* neg_out) {
  int n = s.n_dyn;
  s.w.grad0.resize(std::max(12 * n, 1));
  s.w.diag0.resize(std::max(144 * n, 1));
  // body terms enter once (rank 0); pair terms are split across ranks
  // body terms on the side stream: only the reduction consumes them, so the
  // activity-scan sync below does not wait for them
  bool body_forked = false;
  if (s.comm.rank == 0) {
    CK(cudaEventRecord(s.fork_ev, s.stream));
    CK(cudaStreamWaitEvent(s.side, s.fork_ev, 0));
    std::swap(s.stream, s.side);
    launch_body_terms(s, q, qt, dt, s.w.grad0.p, s.w.diag0.p, nullptr, 1);
    std::swap(s.stream, s.side);
    CK(cudaEventRecord(s.join_ev, s.side));
    body_forked = true;
  } else {
    s.w.grad0.zero(s.stream);
    s.w.diag0.zero(s.stream);
  }
  // the pattern depends only on the overlap and friction pairs: build it first so
  // the Cholesky analysis inputs can be copied out while the values are reduced
  int64_t nfp = 0;
  const int2* fp = fric_pattern(s, nfp);
  build_pattern(s, s.cands.ov.p, s.cands.n_ov, fp, nfp, /*from_cands=*/true);
  HMARK();
  contact_blocks(s, q, kappa, dh, 1, /*mark=*/s.red_nu == 0, /*allow_runs=*/true);
  HMARK();
  append_friction_blocks(s, q, dt, eps_v, 1);
  if (body_forked) CK(cudaStreamWaitEvent(s.stream, s.join_ev, 0));
  reduce_system(s, s.w.diag0.p, s.w.grad0.p, s.comm.world > 1 ? nullptr : neg_out);
  HMARK();
  if (s.comm.world > 1) {
    // the replicated system: sum of the ranks' partial assemblies
    comm_allreduce(s, s.H.val.p, 144 * s.H.nnzb, 0, 0);
    comm_allreduce(s, s.grad.p, 12 * (int64_t)n, 0, 0);
  }
}

// ---------------------------------------------------------------------------
void advance_step(Scene& s, const double* forces_host, const abd_step_params& P, abd_step_stats& st,
                  double* trace) {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  auto t_start = clk::now();
  static const bool trace_newton = getenv("ABD_TRACE_NEWTON") != nullptr;
  st = abd_step_stats{};
  st.min_iterate_distance = INFINITY;
  cudaStream_t stream = s.stream;
  int64_t NB = 12 * (int64_t)s.B;
  int64_t ND = 12 * (int64_t)s.n_dyn;
  if (forces_host) s.forces.upload(forces_host, NB, stream);
  else if (s.forces.n != (size_t)NB) {
    s.forces.resize(NB);
    s.forces.zero(stream);
  }
  s.w.ch_cache.valid = false;  // Cholesky plans are reused within a step only
  s.w.pat_valid = false;       // and so is the (superset) BSR pattern
  s.q0.resize(NB);
  s.q_tilde.resize(NB);
  s.dq.resize(NB);
  s.q_trial.resize(NB);
  s.dx.resize(std::max<int64_t>(ND, 1));
  s.w.neg.resize(std::max<int64_t>(ND, 1));
  s.red.resize(4 * RED_BLOCKS);
  CK(cudaMemcpyAsync(s.q0.p, s.q.p, NB * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  launch_q_tilde(s, s.q0.p, s.q_dot.p, s.forces.p, P.dt, s.q_tilde.p);
  if (s.comm.world > 1) slab_partition(s, s.q.p);  // body slabs for this step (comm.cu)

  auto t0 = clk::now();
  broad_phase(s, s.q.p, s.q.p, P.d_hat);
  st.t_broad += ms(t0, clk::now());
  friction_precompute(s, s.q.p, P.kappa_barrier, P.d_hat, P.mu, nullptr);
  int64_t max_c = s.cands.n_vf + s.cands.n_ee;
  double last_dq = 0.0;
  int n_trace = 0;
  int outer_n = std::max(1, P.friction_outer_iters);
  for (int outer = 0; outer < outer_n; ++outer) {
    if (outer > 0) {
      t0 = clk::now();
      broad_phase(s, s.q.p, s.q.p, P.d_hat);
      st.t_broad += ms(t0, clk::now());
      friction_precompute(s, s.q.p, P.kappa_barrier, P.d_hat, P.mu, nullptr);
    }
    bool converged = false;
    for (int it = 0; it < P.max_newton_iters; ++it) {
      t0 = clk::now();
      // single rank with every dynamic body a row: the reduction writes -g as well
      const bool fuse_neg = s.comm.world == 1 && ND > 0;
      assemble(s, s.q.p, s.q_tilde.p, P.dt, P.kappa_barrier, P.d_hat, P.epsilon_v, fuse_neg ? s.w.neg.p : nullptr);
      st.t_assemble += ms(t0, clk::now());
      t0 = clk::now();
      double amax = 0.0, gd = 0.0, rel = 0.0;
      int pcg_it = 0;
      if (ND) {
        if (!(fuse_neg && s.H.n == s.n_dyn)) {
          k_neg<<<grid_for(ND, 256), 256, 0, stream>>>(ND, s.grad.p, s.w.neg.p);
          note_launch("k_neg");
        }
        const bool reduced = s.red_nu > 0;  // joints: dense T^T H T (k_reduced.cu)
        // multi-rank: distributed PCG over the slabs, slab-local Cholesky preconditioner
        const bool slab = !reduced && P.linear_solver != 1 && s.comm.world > 1;
        const bool chol = !reduced && !slab && P.linear_solver != 1;
        if (reduced) reduced_solve(s, s.w.neg.p, s.dx.p);
        else if (slab) pcg_it = slab_pcg(s, s.w.neg.p, s.dx.p, P.pcg_rel_tol, P.pcg_max_iters, rel);
        else if (chol) chol_begin(s, s.w.neg.p, s.dx.p);
        else pcg_it = pcg_solve(s, s.w.neg.p, s.dx.p, P.pcg_rel_tol, P.pcg_max_iters, rel);
        HMARK();
        // |dx|_inf and g.dx in one pass; the Cholesky residual check shares the host sync
        auto absmax_dot = [&]() {
          unsigned long long* am = s.w.ull.p + 2;
          CK(cudaMemsetAsync(am, 0, sizeof(unsigned long long), stream));
          k_absmax_dot<<<RED_BLOCKS, RED_THREADS, 0, stream>>>(ND, s.dx.p, s.grad.p, am, s.red.p);
          note_launch("k_absmax_dot");
          s.w.scal.resize(8);
          reduce_fixed_stream(stream, s.red.p, RED_BLOCKS, s.w.scal.p);
          pack_to_host(stream, s.h_pinned, {{am, 8, 0}, {s.w.scal.p, 8, 8}});
          SSYNC(stream);
        };
        if (chol) {
          // chol_begin's residual launch carried |dx|_inf and rhs . dx (rhs = -g) along
          SSYNC(stream);
          s.h_pinned[1] = -s.h_pinned[1];
        } else {
          absmax_dot();
        }
        if (chol) {
          bool changed = false;
          pcg_it = chol_finish(s, P.pcg_rel_tol, rel, 3, changed);
          if (changed) absmax_dot();
        }
        st.pcg_iters_total += pcg_it;
        amax = bits_to_d(*reinterpret_cast<unsigned long long*>(s.h_pinned));
        gd = s.h_pinned[1];
      }
      st.t_solve += ms(t0, clk::now());
      last_dq = amax / P.dt;
      if (ND == 0 || amax / P.dt < P.newton_tol) {
        converged = true;
        break;
      }
      double sign = 1.0;
      const double* dsrc = s.dx.p;
      if (gd >= 0.0) {
        st.nondescent_fallbacks += 1;
        if (s.red_nu > 0) {  // T (T^T (-g)) (solver.py:560-561)
          reduced_project(s, s.w.neg.p, s.dx.p);
        } else {
          dsrc = s.grad.p;
          sign = -1.0;
        }
      }
      k_expand_dq<<<grid_for(NB, 256), 256, 0, stream>>>(s.B, s.slot.p, dsrc, sign, s.dq.p);
      note_launch("k_expand_dq");
      // speculative analysis of the next iterate's structure, q + alpha_prev dq over the
      // current candidates, so the host analysis overlaps this iteration's broad phase,
      // CCD and line search (chol_begin verifies that the plan covers the structure
      // actually reached, and re-analyses otherwise); ABD_CHOL_NO_SPEC_SOLVE disables
      static const bool no_spec_solve = getenv("ABD_CHOL_NO_SPEC_SOLVE") != nullptr ||
                                         getenv("ABD_CHOL_NO_SPECULATE") != nullptr ||
                                         getenv("ABD_CHOL_NO_EARLY") != nullptr;
      if (!no_spec_solve && P.linear_solver != 1 && s.red_nu == 0 && s.comm.world == 1 && s.w.pat_valid &&
          s.H.n == s.n_dyn && s.H.n_off > 0 && !s.w.ch_early) {
        s.w.q_pred.resize(NB);
        launch_axpy_q(s, s.q.p, s.w.alpha_prev, s.dq.p, s.w.q_pred.p, NB);
        mark_structure_early(s, s.w.q_pred.p, P.d_hat, /*on_main=*/true);
      }
      // the previous line search's slowest ACCD queries start now on side2 (exact,
      // without the shared cut) and overlap the broad phase
      launch_ccd_hot(s, s.q.p, s.dq.p, P.ccd_slack);
      // candidates over the proposed interval [q, q + dq]
      t0 = clk::now();
      launch_axpy_q(s, s.q.p, 1.0, s.dq.p, s.q_trial.p, NB);  // q + dq (exact add)
      HMARK();
      broad_phase(s, s.q.p, s.q_trial.p, P.d_hat);
      st.t_broad += ms(t0, clk::now());
      max_c = std::max<int64_t>(max_c, s.cands.n_vf + s.cands.n_ee);
      // line search (solver.py:358-393)
      auto tls = clk::now();
      LsFirst lf = line_search_first(s, P, NB);
      st.t_ccd += lf.ccd_ms;
      const double amax_ccd = lf.amax, e0 = lf.e0;
      double alpha = lf.alpha, e = lf.e;
      while (!(e < e0)) {
        alpha *= 0.5;
        if (alpha < 1e-12) throw Error(ABD_ERR_STEP_FAILURE, "line search underflow (no descent below alpha = 1e-12)");
        launch_axpy_q(s, s.q.p, alpha, s.dq.p, s.q_trial.p, NB);
        e = ip_value(s, s.q_trial.p, s.q_tilde.p, P.dt, P.kappa_barrier, P.d_hat, P.epsilon_v);
      }
      CK(cudaMemcpyAsync(s.q.p, s.q_trial.p, NB * sizeof(double), cudaMemcpyDeviceToDevice, stream));
      s.w.alpha_prev = alpha;
      if (trace_newton) {
        std::vector<double> hq(NB), hd(NB);
        CK(cudaMemcpyAsync(hq.data(), s.q.p, NB * sizeof(double), cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(hd.data(), s.dq.p, NB * sizeof(double), cudaMemcpyDeviceToHost, stream));
        SSYNC(stream);
        double cq = 0.0, cd = 0.0;
        for (int64_t i = 0; i < NB; ++i) cq += hq[i] * (1.0 + 1e-3 * (double)(i % 97)), cd += hd[i] * (1.0 + 1e-3 * (double)(i % 89));
        fprintf(stderr, "newton it=%d dq/dt=%.3e gd=%.3e pcg=%d rel=%.2e ccd=%.3e alpha=%.3e e0=%.10e de=%.3e ncand=%lld "
                "sum_q=%.17g sum_dq=%.17g\n",
                it, amax / P.dt, gd, pcg_it, rel, amax_ccd, alpha, e0, e - e0,
                (long long)(s.cands.n_vf + s.cands.n_ee), cq, cd);
      }
      st.t_line_search += ms(tls, clk::now());
      if (trace) trace[n_trace] = e;
      ++n_trace;
      st.iterations += 1;
      if (P.audit_iterates) st.min_iterate_distance = std::fmin(st.min_iterate_distance, global_min_distance(s, s.q.p));
    }
    st.converged = converged ? 1 : 0;
  }
  st.last_dq_over_dt = last_dq;
  st.candidates = max_c;
  // an early analysis posted for an iteration that did not come belongs to no
  // structure a later call may assemble: discard it
  if (s.w.ch_early) {
    chol_analysis_drop(s);
    s.w.ch_early = false;
    s.w.ch_pre = false;
  }
  s.w.ch_verify = false;
  k_qdot<<<grid_for(NB, 256), 256, 0, stream>>>(s.B, s.dyn.p, s.q.p, s.q0.p, P.dt, s.q_dot.p);
  note_launch("k_qdot");
  // stats (solver.py:604-627)
  st.ip_value = ip_value(s, s.q.p, s.q_tilde.p, P.dt, P.kappa_barrier, P.d_hat, P.epsilon_v);
  st.min_distance = NAN;
  if (P.compute_min_distance) {
    double cm = candidate_min_d2(s, s.q.p);
    if (cm < P.d_hat * P.d_hat) st.min_distance = std::sqrt(cm);
    else st.min_distance = global_min_distance_stats(s, s.q.p);
  }
  {
    unsigned long long* m = s.w.ull.p + 3;
    CK(cudaMemsetAsync(m, 0, sizeof(unsigned long long), stream));
    if (s.n_dyn) {
      k_ortho_err<<<grid_for(s.n_dyn, 256), 256, 0, stream>>>(s.n_dyn, s.dyn_body.p, s.q.p, m);
      note_launch("k_ortho_err");
    }
    unsigned long long* hb = reinterpret_cast<unsigned long long*>(s.h_pinned);
    CK(cudaMemcpyAsync(hb, m, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
    SSYNC(stream);
    st.max_ortho_error = bits_to_d(hb[0]);
  }
  st.t_total = ms(t_start, clk::now());
}

}  // namespace abd
