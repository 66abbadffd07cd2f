// Scene-level operations and the Newton driver (solver.py:179-628) with
// device-resident state; only scalars (alpha, energies, |dq|, g.dq) cross
// to the host per iteration.
#include <chrono>
#include <cmath>
#include <vector>

#include "driver.h"

namespace abd {

// ---------------------------------------------------------------------------
// small helper kernels
__global__ void k_absmax(int64_t n, const double* __restrict__ x, unsigned long long* out) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_dot_partials(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                               double* partials) {
  __shared__ double sh[RED_THREADS];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += a[i] * b[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partials[blockIdx.x] = sh[0];
}

__global__ void k_expand_dq(int n_dyn, const int* __restrict__ dyn_body, const double* __restrict__ dx, double sign,
                            double* dq) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= 12 * (int64_t)n_dyn) return;
  int s = (int)(t / 12), c = (int)(t % 12);
  dq[12 * (int64_t)dyn_body[s] + c] = sign * dx[t];
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
static double absmax(Scene& s, const double* x, int64_t n) {
  DVec<unsigned long long> m;
  m.resize(1);
  m.zero(s.stream);
  if (n) {
    k_absmax<<<RED_BLOCKS, RED_THREADS, 0, s.stream>>>(n, x, m.p);
    note_launch("k_absmax");
  }
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, m.p, sizeof(h), cudaMemcpyDeviceToHost, s.stream));
  CK(cudaStreamSynchronize(s.stream));
  return __builtin_bit_cast(double, h);
}

static double dot_det(Scene& s, const double* a, const double* b, int64_t n) {
  s.red.resize(RED_BLOCKS);
  k_dot_partials<<<RED_BLOCKS, RED_THREADS, 0, s.stream>>>(n, a, b, s.red.p);
  note_launch("k_dot_partials");
  return reduce_sum_det(s, s.red.p, RED_BLOCKS);
}

static void check_err_flag(Scene& s, DVec<int>& err, int code, const char* msg) {
  int h = 0;
  CK(cudaMemcpyAsync(&h, err.p, sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  CK(cudaStreamSynchronize(s.stream));
  if (h) throw Error(code, msg);
}

// ---------------------------------------------------------------------------
int64_t contact_blocks(Scene& s, const double* q, double kappa, double dh, int project) {
  int64_t n_vf = s.cands.n_vf, n_ee = s.cands.n_ee;
  int64_t n = n_vf + n_ee;
  DVec<int> flags, pos, err;
  flags.resize(n + 1);
  pos.resize(n + 1);
  err.resize(1);
  err.zero(s.stream);
  double dh2 = dh * dh;
  launch_pair_flags(s, KIND_VF, q, dh2, flags.p, err.p);
  launch_pair_flags(s, KIND_EE, q, dh2, flags.p + n_vf, err.p);
  CK(cudaMemsetAsync(flags.p + n, 0, sizeof(int), s.stream));
  scan_exclusive_i32(s, flags.p, pos.p, n + 1);
  int total = 0, n_vf_act = 0;
  CK(cudaMemcpyAsync(&total, pos.p + n, sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  CK(cudaMemcpyAsync(&n_vf_act, pos.p + n_vf, sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  check_err_flag(s, err, ABD_ERR_BARRIER_DOMAIN,
                 "barrier evaluated at non-positive squared distance (intersection reached)");
  s.pblk.bodies.resize(std::max(total, 1));
  s.pblk.blk.resize((int64_t)std::max(total, 1) * PB_STRIDE);
  s.pblk.d2.resize(std::max(total, 1));
  s.pblk.n = total;
  launch_pair_blocks(s, KIND_VF, q, kappa, dh, project, flags.p, pos.p, 0, err.p);
  launch_pair_blocks(s, KIND_EE, q, kappa, dh, project, flags.p + n_vf, pos.p + n_vf, 0, err.p);
  CK(cudaStreamSynchronize(s.stream));
  (void)n_vf_act;
  return total;
}

// append friction blocks of the resident friction set after n_c contact blocks
void append_friction_blocks(Scene& s, const double* q, double dt, double eps_v, int project) {
  int64_t nc = s.pblk.n, nf = s.fric.n;
  if (nf == 0) return;
  // grow keeping the contact part
  int64_t tot = nc + nf;
  if ((size_t)tot > s.pblk.bodies.cap || (size_t)tot * PB_STRIDE > s.pblk.blk.cap) {
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
    CK(cudaStreamSynchronize(s.stream));
    std::swap(s.pblk.bodies.p, b2.p);
    std::swap(s.pblk.bodies.cap, b2.cap);
    std::swap(s.pblk.blk.p, k2.p);
    std::swap(s.pblk.blk.cap, k2.cap);
    std::swap(s.pblk.d2.p, d2.p);
    std::swap(s.pblk.d2.cap, d2.cap);
  }
  CK(cudaMemcpyAsync(s.pblk.bodies.p + nc, s.fric.bodies.p, nf * sizeof(int2), cudaMemcpyDeviceToDevice, s.stream));
  launch_friction(s.stream, nf, s.fric.bodies.p, s.fric.rec.p, s.fric.mu, q, s.dyn.p, dt, eps_v, project, nullptr,
                  nullptr, nullptr, s.pblk.blk.p + nc * PB_STRIDE);
  s.pblk.n = tot;
}

int64_t friction_precompute(Scene& s, const double* q, double kappa, double dh, double mu, DVec<double>* basis) {
  if (mu < 0) throw Error(ABD_ERR_ARG, "friction coefficient must be >= 0");
  int64_t n_vf = s.cands.n_vf, n_ee = s.cands.n_ee;
  int64_t n = n_vf + n_ee;
  s.fric.mu = mu;
  DVec<int> flags, pos, err;
  flags.resize(n + 1);
  pos.resize(n + 1);
  err.resize(1);
  err.zero(s.stream);
  double dh2 = dh * dh;
  launch_pair_flags(s, KIND_VF, q, dh2, flags.p, err.p);
  launch_pair_flags(s, KIND_EE, q, dh2, flags.p + n_vf, err.p);
  CK(cudaMemsetAsync(flags.p + n, 0, sizeof(int), s.stream));
  scan_exclusive_i32(s, flags.p, pos.p, n + 1);
  int total = 0;
  CK(cudaMemcpyAsync(&total, pos.p + n, sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  check_err_flag(s, err, ABD_ERR_BARRIER_DOMAIN, "barrier evaluated at non-positive squared distance");
  s.fric.n = total;
  s.fric.bodies.resize(std::max(total, 1));
  s.fric.rec.resize((int64_t)std::max(total, 1) * FRIC_STRIDE);
  double* bp = nullptr;
  if (basis) {
    basis->resize((int64_t)std::max(total, 1) * 6);
    bp = basis->p;
  }
  launch_friction_pre(s, KIND_VF, q, kappa, dh, flags.p, pos.p, 0, bp);
  launch_friction_pre(s, KIND_EE, q, kappa, dh, flags.p + n_vf, pos.p + n_vf, 0, bp);
  CK(cudaStreamSynchronize(s.stream));
  return total;
}

double contact_energy(Scene& s, const double* q, double kappa, double dh) {
  DVec<int> err;
  err.resize(1);
  err.zero(s.stream);
  s.red.resize(2 * RED_BLOCKS);
  launch_contact_energy(s, KIND_VF, q, kappa, dh, s.red.p, err.p);
  launch_contact_energy(s, KIND_EE, q, kappa, dh, s.red.p + RED_BLOCKS, err.p);
  check_err_flag(s, err, ABD_ERR_BARRIER_DOMAIN,
                 "barrier evaluated at non-positive squared distance (intersection reached)");
  double vf = reduce_sum_det(s, s.red.p, RED_BLOCKS);
  double ee = reduce_sum_det(s, s.red.p + RED_BLOCKS, RED_BLOCKS);
  return (0.0 + vf) + ee;
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

double ip_value(Scene& s, const double* q, const double* qt, double dt, double kappa, double dh, double eps_v) {
  double e = body_energy(s, q, qt, dt);
  e += contact_energy(s, q, kappa, dh);
  e += friction_energy(s, q, dt, eps_v);
  return e;
}

double step_filter(Scene& s, const double* q, const double* dq, double slack) {
  DVec<unsigned long long> tmin;
  DVec<int> err;
  tmin.resize(1);
  err.resize(1);
  err.zero(s.stream);
  unsigned long long one = (unsigned long long)__builtin_bit_cast(long long, 1.0);
  CK(cudaMemcpyAsync(tmin.p, &one, sizeof(one), cudaMemcpyHostToDevice, s.stream));
  launch_ccd(s, KIND_VF, q, dq, slack, tmin.p, err.p);
  launch_ccd(s, KIND_EE, q, dq, slack, tmin.p, err.p);
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, tmin.p, sizeof(h), cudaMemcpyDeviceToHost, s.stream));
  check_err_flag(s, err, ABD_ERR_CCD_DOMAIN, "CCD query issued at non-positive initial distance");
  return std::fmin(1.0, __builtin_bit_cast(double, h));
}

double candidate_min_d2(Scene& s, const double* q) {
  DVec<unsigned long long> best;
  best.resize(1);
  unsigned long long inf = (unsigned long long)__builtin_bit_cast(long long, (double)INFINITY);
  CK(cudaMemcpyAsync(best.p, &inf, sizeof(inf), cudaMemcpyHostToDevice, s.stream));
  launch_cand_min_d2(s, KIND_VF, q, best.p);
  launch_cand_min_d2(s, KIND_EE, q, best.p);
  unsigned long long h = 0;
  CK(cudaMemcpyAsync(&h, best.p, sizeof(h), cudaMemcpyDeviceToHost, s.stream));
  CK(cudaStreamSynchronize(s.stream));
  return __builtin_bit_cast(double, h);
}

void assemble(Scene& s, const double* q, const double* qt, double dt, double kappa, double dh, double eps_v) {
  int n = s.n_dyn;
  DVec<double> grad0, diag0;
  grad0.resize(std::max(12 * n, 1));
  diag0.resize(std::max(144 * n, 1));
  launch_body_terms(s, q, qt, dt, grad0.p, diag0.p, nullptr, 1);
  contact_blocks(s, q, kappa, dh, 1);
  append_friction_blocks(s, q, dt, eps_v, 1);
  build_pattern(s, s.cands.ov.p, s.cands.n_ov, s.fric.bodies.p, s.fric.n);
  reduce_system(s, diag0.p, grad0.p);
}

// ---------------------------------------------------------------------------
void advance_step(Scene& s, const double* forces_host, const abd_step_params& P, abd_step_stats& st,
                  double* trace) {
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  auto t_start = clk::now();
  st = abd_step_stats{};
  cudaStream_t stream = s.stream;
  int64_t NB = 12 * (int64_t)s.B;
  int64_t ND = 12 * (int64_t)s.n_dyn;
  if (forces_host) s.forces.upload(forces_host, NB, stream);
  else if (s.forces.n != (size_t)NB) {
    s.forces.resize(NB);
    s.forces.zero(stream);
  }
  s.q0.resize(NB);
  s.q_tilde.resize(NB);
  s.dq.resize(NB);
  s.q_trial.resize(NB);
  s.dx.resize(std::max<int64_t>(ND, 1));
  CK(cudaMemcpyAsync(s.q0.p, s.q.p, NB * sizeof(double), cudaMemcpyDeviceToDevice, stream));
  launch_q_tilde(s, s.q0.p, s.q_dot.p, s.forces.p, P.dt, s.q_tilde.p);

  auto t0 = clk::now();
  broad_phase(s, s.q.p, s.q.p, P.d_hat);
  st.t_broad += ms(t0, clk::now());
  friction_precompute(s, s.q.p, P.kappa_barrier, P.d_hat, P.mu, nullptr);
  int64_t max_c = s.cands.n_vf + s.cands.n_ee;
  DVec<double> neg;
  neg.resize(std::max<int64_t>(ND, 1));
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
      assemble(s, s.q.p, s.q_tilde.p, P.dt, P.kappa_barrier, P.d_hat, P.epsilon_v);
      st.t_assemble += ms(t0, clk::now());
      t0 = clk::now();
      if (ND) {
        k_neg<<<grid_for(ND, 256), 256, 0, stream>>>(ND, s.grad.p, neg.p);
        note_launch("k_neg");
        double rel = 0.0;
        int its = 0;
        try {
          its = pcg_solve(s, neg.p, s.dx.p, P.pcg_rel_tol, P.pcg_max_iters, rel);
        } catch (Error& e) {
          throw;
        }
        st.pcg_iters_total += its;
      }
      st.t_solve += ms(t0, clk::now());
      double amax = ND ? absmax(s, s.dx.p, ND) : 0.0;
      last_dq = amax / P.dt;
      if (ND == 0 || amax / P.dt < P.newton_tol) {
        converged = true;
        break;
      }
      double gd = dot_det(s, s.grad.p, s.dx.p, ND);
      double sign = 1.0;
      const double* dsrc = s.dx.p;
      if (gd >= 0.0) {
        st.nondescent_fallbacks += 1;
        dsrc = s.grad.p;
        sign = -1.0;
      }
      s.dq.zero(stream);
      k_expand_dq<<<grid_for(ND, 256), 256, 0, stream>>>(s.n_dyn, s.dyn_body.p, dsrc, sign, s.dq.p);
      note_launch("k_expand_dq");
      // candidates over the proposed interval
      t0 = clk::now();
      launch_axpy_q(s, s.q.p, 1.0, s.dq.p, s.q_trial.p, NB);  // q + dq (alpha = 1: exact add)
      broad_phase(s, s.q.p, s.q_trial.p, P.d_hat);
      st.t_broad += ms(t0, clk::now());
      max_c = std::max<int64_t>(max_c, s.cands.n_vf + s.cands.n_ee);
      // line search (solver.py:358-393)
      auto tls = clk::now();
      t0 = clk::now();
      double amax_ccd = step_filter(s, s.q.p, s.dq.p, P.ccd_slack);
      st.t_ccd += ms(t0, clk::now());
      double alpha = amax_ccd >= 1.0 ? 1.0 : std::fmin(1.0, P.ccd_step_scale * amax_ccd);
      double e0 = ip_value(s, s.q.p, s.q_tilde.p, P.dt, P.kappa_barrier, P.d_hat, P.epsilon_v);
      double e = 0.0;
      while (true) {
        launch_axpy_q(s, s.q.p, alpha, s.dq.p, s.q_trial.p, NB);
        e = ip_value(s, s.q_trial.p, s.q_tilde.p, P.dt, P.kappa_barrier, P.d_hat, P.epsilon_v);
        if (e < e0) break;
        alpha *= 0.5;
        if (alpha < 1e-12) {
          throw Error(ABD_ERR_STEP_FAILURE, "line search underflow (no descent below alpha = 1e-12)");
        }
      }
      CK(cudaMemcpyAsync(s.q.p, s.q_trial.p, NB * sizeof(double), cudaMemcpyDeviceToDevice, stream));
      st.t_line_search += ms(tls, clk::now());
      if (trace) trace[n_trace] = e;
      ++n_trace;
      st.iterations += 1;
    }
    st.converged = converged ? 1 : 0;
  }
  st.last_dq_over_dt = last_dq;
  st.candidates = max_c;
  // q_dot
  k_qdot<<<grid_for(NB, 256), 256, 0, stream>>>(s.B, s.dyn.p, s.q.p, s.q0.p, P.dt, s.q_dot.p);
  note_launch("k_qdot");
  // stats (solver.py:604-627)
  st.min_distance = NAN;
  if (P.compute_min_distance) {
    double cm = candidate_min_d2(s, s.q.p);
    if (cm < P.d_hat * P.d_hat) st.min_distance = std::sqrt(cm);
    else st.min_distance = global_min_distance(s, s.q.p);
  }
  st.ip_value = ip_value(s, s.q.p, s.q_tilde.p, P.dt, P.kappa_barrier, P.d_hat, P.epsilon_v);
  {
    DVec<unsigned long long> m;
    m.resize(1);
    m.zero(stream);
    if (s.n_dyn) {
      k_ortho_err<<<grid_for(s.n_dyn, 256), 256, 0, stream>>>(s.n_dyn, s.dyn_body.p, s.q.p, m.p);
      note_launch("k_ortho_err");
    }
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, m.p, sizeof(h), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    st.max_ortho_error = __builtin_bit_cast(double, h);
  }
  st.t_total = ms(t_start, clk::now());
}

}  // namespace abd
