// extern "C" boundary (include/abd_b200.h): host buffers in, host buffers
// out; exceptions mapped to abd_status + thread-local message.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "driver.h"

using namespace abd;

namespace abd {
extern std::atomic<int64_t> g_launches;
}

struct abd_scene {
  Scene s;
};

static thread_local std::string t_err;
static thread_local int64_t t_err_idx = -1;

template <class F>
static int guard(F&& f) {
  try {
    f();
    return ABD_OK;
  } catch (Error& e) {
    t_err = e.what();
    t_err_idx = e.index;
    return e.code;
  } catch (std::exception& e) {
    t_err = e.what();
    t_err_idx = -1;
    return ABD_ERR_CUDA;
  }
}

static void ensure_device() {
  static int ok = -1;
  if (ok == 1) return;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw Error(ABD_ERR_NO_DEVICE, "no CUDA device visible (the sm_100a kernels need a B200)");
  }
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  if (p.major != 10) throw Error(ABD_ERR_NO_DEVICE, "device is not sm_100 (Blackwell B200 required)");
  size_t cur = 0;
  CK(cudaDeviceGetLimit(&cur, cudaLimitStackSize));
  if (cur < 16384) CK(cudaDeviceSetLimit(cudaLimitStackSize, 16384));
  ok = 1;
}

// RAII device staging buffer
template <class T>
struct Dev {
  DVec<T> v;
  cudaStream_t st;
  explicit Dev(cudaStream_t s) : st(s) {}
  T* up(const T* h, size_t n) {
    v.upload(h, std::max<size_t>(n, 0), st);
    if (!n) v.resize(1);
    return v.p;
  }
  T* alloc(size_t n) {
    v.resize(std::max<size_t>(n, 1));
    return v.p;
  }
  void down(T* h, size_t n) {
    if (h && n) v.download(h, n, st);
  }
};

static cudaStream_t g_stream() {
  static cudaStream_t s = nullptr;
  if (!s) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

static void sync(cudaStream_t s) { CK(cudaStreamSynchronize(s)); }

static void check_flag(Dev<int>& f, cudaStream_t st, int code, const char* msg) {
  int h = 0;
  f.down(&h, 1);
  sync(st);
  if (h) throw Error(code, msg);
}

extern "C" {

const char* abd_last_error(void) { return t_err.c_str(); }
int64_t abd_last_error_index(void) { return t_err_idx; }
int64_t abd_kernel_launches(void) { return g_launches.load(); }

int abd_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  return guard([&] {
    ensure_device();
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (cc_major) *cc_major = p.major;
    if (cc_minor) *cc_minor = p.minor;
  });
}

int abd_pt_closest_batch(int64_t n, const double* z, double* d2, int32_t* region, double* bary) {
  return guard([&] {
    ensure_device();
    cudaStream_t st = g_stream();
    Dev<double> dz(st), dd(st), db(st);
    Dev<int> dr(st);
    launch_pt_closest(st, n, dz.up(z, 12 * n), dd.alloc(n), dr.alloc(n), db.alloc(3 * n));
    dd.down(d2, n);
    dr.down(region, n);
    db.down(bary, 3 * n);
    sync(st);
  });
}

int abd_ee_closest_batch(int64_t n, const double* z, double* d2, int32_t* region, double* s, double* t) {
  return guard([&] {
    ensure_device();
    cudaStream_t st = g_stream();
    Dev<double> dz(st), dd(st), ds(st), dt(st);
    Dev<int> dr(st);
    launch_ee_closest(st, n, dz.up(z, 12 * n), dd.alloc(n), dr.alloc(n), ds.alloc(n), dt.alloc(n));
    dd.down(d2, n);
    dr.down(region, n);
    ds.down(s, n);
    dt.down(t, n);
    sync(st);
  });
}

int abd_pair_distance_gradients(int kind, int64_t n, const double* z, double* d2, double* grad, double* hess,
                                int32_t* region, double* gamma) {
  return guard([&] {
    ensure_device();
    if (kind != ABD_VF && kind != ABD_EE) throw Error(ABD_ERR_ARG, "unknown pair kind");
    cudaStream_t st = g_stream();
    Dev<double> dz(st), dd(st), dg(st), dh(st), dga(st);
    Dev<int> dr(st);
    launch_d2_derivs(st, kind, n, dz.up(z, 12 * n), dd.alloc(n), dg.alloc(12 * n), dh.alloc(144 * n), dr.alloc(n),
                     dga.alloc(4 * n));
    dd.down(d2, n);
    dg.down(grad, 12 * n);
    dh.down(hess, 144 * n);
    dr.down(region, n);
    dga.down(gamma, 4 * n);
    sync(st);
  });
}

int abd_ee_mollifier_batch(int64_t n, const double* z, const double* eps_x, double* val, double* grad, double* hess) {
  return guard([&] {
    ensure_device();
    cudaStream_t st = g_stream();
    Dev<double> dz(st), de(st), dv(st), dg(st), dh(st);
    bool full = grad && hess;
    launch_mollifier(st, n, dz.up(z, 12 * n), de.up(eps_x, n), dv.alloc(n), full ? dg.alloc(12 * n) : nullptr,
                     full ? dh.alloc(144 * n) : nullptr);
    dv.down(val, n);
    if (full) {
      dg.down(grad, 12 * n);
      dh.down(hess, 144 * n);
    }
    sync(st);
  });
}

int abd_barrier_batch(int64_t n, const double* d_sq, double d_hat, double* b0, double* b1, double* b2) {
  return guard([&] {
    ensure_device();
    cudaStream_t st = g_stream();
    Dev<double> ds(st), o0(st), o1(st), o2(st);
    Dev<int> err(st);
    err.alloc(1);
    err.v.zero(st);
    launch_barrier(st, n, ds.up(d_sq, n), d_hat, o0.alloc(n), o1.alloc(n), o2.alloc(n), err.v.p);
    check_flag(err, st, ABD_ERR_BARRIER_DOMAIN,
               "barrier evaluated at non-positive squared distance (intersection reached; CCD filtering must "
               "prevent this)");
    o0.down(b0, n);
    o1.down(b1, n);
    o2.down(b2, n);
    sync(st);
  });
}

int abd_ortho_batch(int64_t n, const double* q, const double* stiffness, int project, double* energy, double* grad,
                    double* hess) {
  return guard([&] {
    ensure_device();
    cudaStream_t st = g_stream();
    Dev<double> dq(st), dk(st), de(st), dg(st), dh(st);
    launch_ortho(st, n, dq.up(q, 12 * n), dk.up(stiffness, n), project, de.alloc(n), dg.alloc(12 * n),
                 dh.alloc(144 * n));
    de.down(energy, n);
    dg.down(grad, 12 * n);
    dh.down(hess, 144 * n);
    sync(st);
  });
}

int abd_project_psd_batch(int64_t n, int k, const double* H, double* out) {
  return guard([&] {
    ensure_device();
    if (k < 1 || k > 24) throw Error(ABD_ERR_ARG, "project_psd supports 1 <= k <= 24");
    cudaStream_t st = g_stream();
    Dev<double> di(st), dout(st);
    launch_psd(st, n, k, di.up(H, (size_t)n * k * k), dout.alloc((size_t)n * k * k));
    dout.down(out, (size_t)n * k * k);
    sync(st);
  });
}

int abd_accd_batch(int kind, int64_t n, const double* x, const double* dx, double slack, double t_max, int max_iters,
                   double* t) {
  return guard([&] {
    ensure_device();
    cudaStream_t st = g_stream();
    Dev<double> dxv(st), ddx(st), dt(st);
    Dev<int> err(st);
    err.alloc(1);
    err.v.zero(st);
    launch_accd(st, kind, n, dxv.up(x, 12 * n), ddx.up(dx, 12 * n), slack, t_max, max_iters, dt.alloc(n), err.v.p);
    check_flag(err, st, ABD_ERR_CCD_DOMAIN, "CCD query issued at non-positive initial distance");
    dt.down(t, n);
    sync(st);
  });
}

int abd_contact_pair_batch(int kind, int64_t n, const double* z, const double* rest, const double* eps_x,
                           double kappa, double d_hat, const uint8_t* dyn, int project, double* g12, double* h12,
                           double* g24, double* h24) {
  return guard([&] {
    ensure_device();
    cudaStream_t st = g_stream();
    Dev<double> dz(st), dr(st), de(st), o1(st), o2(st), o3(st), o4(st);
    Dev<unsigned char> dd(st);
    launch_contact_pairs(st, kind, n, dz.up(z, 12 * n), dr.up(rest, 12 * n), de.up(eps_x, n), kappa, d_hat,
                         dd.up(dyn, 2 * n), project, o1.alloc(12 * n), o2.alloc(144 * n), o3.alloc(24 * n),
                         o4.alloc(576 * n));
    o1.down(g12, 12 * n);
    o2.down(h12, 144 * n);
    o3.down(g24, 24 * n);
    o4.down(h24, 576 * n);
    sync(st);
  });
}

static void pack_friction(int64_t n, const int64_t* ba, const int64_t* bb, const double* lam, const double* tmap,
                          const double* off, std::vector<int2>& hb, std::vector<double>& hr) {
  hb.resize(std::max<int64_t>(n, 1));
  hr.resize(std::max<int64_t>(n, 1) * FRIC_STRIDE);
  for (int64_t i = 0; i < n; ++i) {
    hb[i] = make_int2((int)ba[i], (int)bb[i]);
    std::memcpy(&hr[i * FRIC_STRIDE], tmap + 48 * i, 48 * sizeof(double));
    hr[i * FRIC_STRIDE + 48] = off[2 * i];
    hr[i * FRIC_STRIDE + 49] = off[2 * i + 1];
    hr[i * FRIC_STRIDE + 50] = lam[i];
  }
}

int abd_friction_batch(int64_t n, const int64_t* body_a, const int64_t* body_b, const double* lam, double mu,
                       const double* tangent_map, const double* offset, int n_bodies, const double* q,
                       const uint8_t* dynamic, double dt, double eps_v, int project, double* energy, double* grad24,
                       double* hess24) {
  return guard([&] {
    ensure_device();
    cudaStream_t st = g_stream();
    std::vector<int2> hb;
    std::vector<double> hr;
    pack_friction(n, body_a, body_b, lam, tangent_map, offset, hb, hr);
    Dev<int2> db(st);
    Dev<double> dr(st), dq(st), part(st), dg(st), dh(st);
    Dev<unsigned char> dd(st);
    db.up(hb.data(), hb.size());
    dr.up(hr.data(), hr.size());
    dq.up(q, 12 * (size_t)n_bodies);
    dd.up(dynamic, n_bodies);
    bool want = grad24 && hess24;
    launch_friction(st, n, db.v.p, dr.v.p, mu, dq.v.p, dd.v.p, dt, eps_v, project, part.alloc(RED_BLOCKS),
                    want ? dg.alloc(24 * n) : nullptr, want ? dh.alloc(576 * n) : nullptr, nullptr);
    if (energy) {
      Dev<double> one(st);
      one.alloc(1);
      reduce_fixed_stream(st, part.v.p, RED_BLOCKS, one.v.p);  // deterministic fixed-order sum
      one.down(energy, 1);
    }
    if (want) {
      dg.down(grad24, 24 * n);
      dh.down(hess24, 576 * n);
    }
    sync(st);
  });
}

static Scene& bsr_scene() {
  static thread_local Scene* s = nullptr;
  if (!s) s = new Scene();
  return *s;
}

static void pad_vec(int n, int bdim, const double* in, std::vector<double>& out) {
  out.assign(12 * (size_t)n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < bdim; ++c) out[12 * (size_t)i + c] = in[(size_t)bdim * i + c];
}

int abd_bsr_matvec(int n, int bdim, const double* diag, int64_t n_off, const int64_t* keys, const double* off,
                   const double* x, double* y) {
  return guard([&] {
    ensure_device();
    if (bdim < 1 || bdim > 12) throw Error(ABD_ERR_ARG, "block_dim must be in [1, 12]");
    Scene& s = bsr_scene();
    load_bsr(s, n, bdim, diag, n_off, keys, off);
    std::vector<double> xp;
    pad_vec(n, bdim, x, xp);
    DVec<double> dx, dy;
    dx.upload(xp.data(), xp.size(), s.stream);
    dy.resize(std::max<size_t>(xp.size(), 1));
    spmv(s, dx.p, dy.p);
    std::vector<double> yp(xp.size());
    dy.download(yp.data(), yp.size(), s.stream);
    sync(s.stream);
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < bdim; ++c) y[(size_t)bdim * i + c] = yp[12 * (size_t)i + c];
  });
}

int abd_bsr_pcg(int n, int bdim, const double* diag, int64_t n_off, const int64_t* keys, const double* off,
                const double* rhs, double rel_tol, int max_iters, double* x, int* iters, double* rel_res) {
  return guard([&] {
    ensure_device();
    if (bdim < 1 || bdim > 12) throw Error(ABD_ERR_ARG, "block_dim must be in [1, 12]");
    Scene& s = bsr_scene();
    load_bsr(s, n, bdim, diag, n_off, keys, off);
    std::vector<double> bp;
    pad_vec(n, bdim, rhs, bp);
    DVec<double> db, dx;
    db.upload(bp.data(), bp.size(), s.stream);
    dx.resize(std::max<size_t>(bp.size(), 1));
    double rel = 0.0;
    int it = pcg_solve(s, db.p, dx.p, rel_tol, max_iters, rel);
    std::vector<double> xp(bp.size());
    dx.download(xp.data(), xp.size(), s.stream);
    sync(s.stream);
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < bdim; ++c) x[(size_t)bdim * i + c] = xp[12 * (size_t)i + c];
    if (iters) *iters = it;
    if (rel_res) *rel_res = rel;
  });
}

int abd_bsr_cholesky(int n, int bdim, const double* diag, int64_t n_off, const int64_t* keys, const double* off,
                     const double* rhs, double rel_tol, int max_refine, double* x, int* solves, double* rel_res) {
  return guard([&] {
    ensure_device();
    if (bdim < 1 || bdim > 12) throw Error(ABD_ERR_ARG, "block_dim must be in [1, 12]");
    if (max_refine < 0) throw Error(ABD_ERR_ARG, "max_refine < 0");
    Scene& s = bsr_scene();
    load_bsr(s, n, bdim, diag, n_off, keys, off);
    std::vector<double> bp;
    pad_vec(n, bdim, rhs, bp);
    DVec<double> db, dx;
    db.upload(bp.data(), bp.size(), s.stream);
    dx.resize(std::max<size_t>(bp.size(), 1));
    double rel = 0.0;
    int ns = chol_solve(s, db.p, dx.p, rel_tol, rel, max_refine);
    std::vector<double> xp(bp.size());
    dx.download(xp.data(), xp.size(), s.stream);
    sync(s.stream);
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < bdim; ++c) x[(size_t)bdim * i + c] = xp[12 * (size_t)i + c];
    if (solves) *solves = ns;
    if (rel_res) *rel_res = rel;
  });
}

// ---------------------------------------------------------------------------
// static primitive groups of the broad-phase cull (see Scene::grp_*): per body and
// kind, primitives sorted by the Morton code of their rest centroid, 32 per group,
// with the rest AABB of each group's vertices
static void build_prim_groups(Scene& s, int B, const std::vector<int>& vo, const std::vector<int>& eo,
                              const std::vector<int>& to, const double* rest, const std::vector<int>& ge,
                              const std::vector<int>& gt) {
  s.has_groups = s.max_v <= 256;
  if (!s.has_groups) return;
  const std::vector<int>* offs[3] = {&vo, &eo, &to};
  for (int kind = 0; kind < 3; ++kind) {
    const std::vector<int>& off = *offs[kind];
    const int n_all = off[B];
    std::vector<int> gid(n_all);
    std::vector<unsigned> gpk(n_all);
    std::vector<int> goff(B + 1, 0);
    std::vector<double> gbox;
    std::vector<std::pair<uint32_t, int>> key;
    for (int b = 0; b < B; ++b) {
      const int v0 = vo[b], np = off[b + 1] - off[b];
      double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
      for (int v = vo[b]; v < vo[b + 1]; ++v)
        for (int k = 0; k < 3; ++k) {
          lo[k] = std::min(lo[k], rest[3 * (int64_t)v + k]);
          hi[k] = std::max(hi[k], rest[3 * (int64_t)v + k]);
        }
      auto verts = [&](int i, int* out) {
        const int g = off[b] + i;
        if (kind == 0) { out[0] = v0 + i; return 1; }
        if (kind == 1) { out[0] = ge[2 * g]; out[1] = ge[2 * g + 1]; return 2; }
        out[0] = gt[3 * g]; out[1] = gt[3 * g + 1]; out[2] = gt[3 * g + 2];
        return 3;
      };
      key.clear();
      for (int i = 0; i < np; ++i) {
        int vs[3];
        const int nv = verts(i, vs);
        uint32_t code = 0;
        int cell[3];
        for (int k = 0; k < 3; ++k) {
          double c = 0.0;
          for (int m = 0; m < nv; ++m) c += rest[3 * (int64_t)vs[m] + k];
          c /= nv;
          const double ext = hi[k] - lo[k];
          int q = ext > 0 ? (int)((c - lo[k]) / ext * 1023.0) : 0;
          cell[k] = std::min(1023, std::max(0, q));
        }
        for (int bit = 9; bit >= 0; --bit)
          for (int k = 0; k < 3; ++k) code = (code << 1) | ((cell[k] >> bit) & 1);
        key.push_back({code, i});
      }
      std::sort(key.begin(), key.end());
      for (int i = 0; i < np; ++i) {
        const int loc = key[i].second;
        int vs[3];
        const int nv = verts(loc, vs);
        unsigned pk = 0;
        for (int m = 0; m < nv; ++m) pk |= (unsigned)(vs[m] - v0) << (8 * m);
        gid[off[b] + i] = loc;
        gpk[off[b] + i] = pk;
      }
      const int ng = (np + 31) / 32;
      goff[b + 1] = goff[b] + ng;
      for (int g = 0; g < ng; ++g) {
        double glo[3] = {1e300, 1e300, 1e300}, ghi[3] = {-1e300, -1e300, -1e300};
        for (int i = 32 * g; i < std::min(np, 32 * g + 32); ++i) {
          int vs[3];
          const int nv = verts(key[i].second, vs);
          for (int m = 0; m < nv; ++m)
            for (int k = 0; k < 3; ++k) {
              glo[k] = std::min(glo[k], rest[3 * (int64_t)vs[m] + k]);
              ghi[k] = std::max(ghi[k], rest[3 * (int64_t)vs[m] + k]);
            }
        }
        for (int k = 0; k < 3; ++k) gbox.push_back(0.5 * (glo[k] + ghi[k]));
        for (int k = 0; k < 3; ++k) gbox.push_back(0.5 * (ghi[k] - glo[k]) * (1.0 + 1e-12) + 1e-300);
      }
    }
    s.grp_id[kind].upload(gid.data(), n_all, s.stream);
    s.grp_pk[kind].upload(gpk.data(), n_all, s.stream);
    s.grp_off[kind].upload(goff.data(), B + 1, s.stream);
    s.grp_box[kind].upload(gbox.data(), gbox.size(), s.stream);
  }
}

abd_scene* abd_scene_create(int n_bodies, const int64_t* v_off, const int64_t* e_off, const int64_t* t_off,
                            const double* rest, const int64_t* edges, const int64_t* tris, const double* edge_len_sq,
                            const uint8_t* dynamic, const double* mass, const double* stiffness) {
  abd_scene* out = nullptr;
  int rc = guard([&] {
    ensure_device();
    if (n_bodies < 0) throw Error(ABD_ERR_ARG, "n_bodies < 0");
    auto* h = new abd_scene();
    Scene& s = h->s;
    int B = n_bodies;
    s.B = B;
    s.V = v_off[B];
    s.E = e_off[B];
    s.T = t_off[B];
    if (s.V >= (1ll << 31) || s.E >= (1ll << 31) || s.T >= (1ll << 31)) throw Error(ABD_ERR_ARG, "scene too large");
    std::vector<int> vo(B + 1), eo(B + 1), to(B + 1), vb(s.V), eb(s.E), tb(s.T);
    std::vector<int> ge(2 * s.E), gt(3 * s.T);
    for (int b = 0; b <= B; ++b) {
      vo[b] = (int)v_off[b];
      eo[b] = (int)e_off[b];
      to[b] = (int)t_off[b];
    }
    for (int b = 0; b < B; ++b) {
      s.max_v = std::max(s.max_v, vo[b + 1] - vo[b]);
      s.max_e = std::max(s.max_e, eo[b + 1] - eo[b]);
      s.max_t = std::max(s.max_t, to[b + 1] - to[b]);
      for (int v = vo[b]; v < vo[b + 1]; ++v) vb[v] = b;
      for (int e = eo[b]; e < eo[b + 1]; ++e) {
        eb[e] = b;
        for (int k = 0; k < 2; ++k) {
          int64_t lv = edges[2 * e + k];
          if (lv < 0 || lv >= vo[b + 1] - vo[b]) throw Error(ABD_ERR_ARG, "edge index out of range");
          ge[2 * e + k] = vo[b] + (int)lv;
        }
      }
      for (int t = to[b]; t < to[b + 1]; ++t) {
        tb[t] = b;
        for (int k = 0; k < 3; ++k) {
          int64_t lv = tris[3 * t + k];
          if (lv < 0 || lv >= vo[b + 1] - vo[b]) throw Error(ABD_ERR_ARG, "triangle index out of range");
          gt[3 * t + k] = vo[b] + (int)lv;
        }
      }
    }
    cudaStream_t st = s.stream;
    build_prim_groups(s, B, vo, eo, to, rest, ge, gt);
    s.v_off.upload(vo.data(), B + 1, st);
    s.e_off.upload(eo.data(), B + 1, st);
    s.t_off.upload(to.data(), B + 1, st);
    s.rest.upload(rest, 3 * s.V, st);
    s.edges.upload(ge.data(), 2 * s.E, st);
    s.tris.upload(gt.data(), 3 * s.T, st);
    s.elen2.upload(edge_len_sq, s.E, st);
    s.vert_body.upload(vb.data(), s.V, st);
    s.edge_body.upload(eb.data(), s.E, st);
    s.tri_body.upload(tb.data(), s.T, st);
    {
      std::vector<double> rm(3 * (size_t)B, 0.0);
      for (int b = 0; b < B; ++b)
        for (int v = vo[b]; v < vo[b + 1]; ++v)
          for (int k = 0; k < 3; ++k) rm[3 * b + k] = std::max(rm[3 * b + k], std::fabs(rest[3 * (int64_t)v + k]));
      s.body_rmax.upload(rm.data(), 3 * (size_t)B, st);
    }
    s.h_dyn.assign(dynamic, dynamic + B);
    s.dyn.upload(s.h_dyn.data(), B, st);
    s.h_slot.assign(B, -1);
    s.h_dyn_body.clear();
    for (int b = 0; b < B; ++b)
      if (dynamic[b]) {
        s.h_slot[b] = (int)s.h_dyn_body.size();
        s.h_dyn_body.push_back(b);
      }
    s.n_dyn = (int)s.h_dyn_body.size();
    s.slot.upload(s.h_slot.data(), B, st);
    s.dyn_body.upload(s.h_dyn_body.data(), std::max(s.n_dyn, 0), st);
    if (s.n_dyn == 0) s.dyn_body.resize(1);
    s.mass.upload(mass, 144 * (size_t)B, st);
    s.stiff.upload(stiffness, B, st);
    s.q.resize(12 * (size_t)B);
    s.q.zero(st);
    s.q_dot.resize(12 * (size_t)B);
    s.q_dot.zero(st);
    CK(cudaStreamSynchronize(st));
    out = h;
  });
  (void)rc;
  return out;
}

void abd_scene_destroy(abd_scene* s) {
  if (!s) return;
  try {
    comm_destroy(s->s);
  } catch (...) {
  }
  delete s;
}

#define SC(h) Scene& s = (h)->s

int abd_broad_phase(abd_scene* h, const double* q0, const double* q1, double d_hat, int64_t* n_vf, int64_t* n_ee,
                    int64_t* n_ov) {
  return guard([&] {
    SC(h);
    s.q.upload(q0, 12 * (size_t)s.B, s.stream);
    s.q_trial.upload(q1, 12 * (size_t)s.B, s.stream);
    broad_phase(s, s.q.p, s.q_trial.p, d_hat);
    sync(s.stream);
    *n_vf = s.cands.n_vf;
    *n_ee = s.cands.n_ee;
    *n_ov = s.cands.n_ov;
  });
}

int abd_get_candidates(abd_scene* h, int64_t* vf, int64_t* ee, int64_t* ov) {
  return guard([&] {
    SC(h);
    std::vector<int4> a(s.cands.n_vf), b(s.cands.n_ee);
    std::vector<int2> c(s.cands.n_ov);
    s.cands.vf.download(a.data(), a.size(), s.stream);
    s.cands.ee.download(b.data(), b.size(), s.stream);
    s.cands.ov.download(c.data(), c.size(), s.stream);
    sync(s.stream);
    // the device keeps a deterministic per-overlap-pair order; the API returns the
    // reference's canonical (c0, c2, c1, c3) order (contact.py:404)
    auto canon = [](const int4& p, const int4& q) {
      if (p.x != q.x) return p.x < q.x;
      if (p.z != q.z) return p.z < q.z;
      if (p.y != q.y) return p.y < q.y;
      return p.w < q.w;
    };
    std::sort(a.begin(), a.end(), canon);
    std::sort(b.begin(), b.end(), canon);
    for (size_t i = 0; i < a.size(); ++i) {
      vf[4 * i] = a[i].x; vf[4 * i + 1] = a[i].y; vf[4 * i + 2] = a[i].z; vf[4 * i + 3] = a[i].w;
    }
    for (size_t i = 0; i < b.size(); ++i) {
      ee[4 * i] = b[i].x; ee[4 * i + 1] = b[i].y; ee[4 * i + 2] = b[i].z; ee[4 * i + 3] = b[i].w;
    }
    for (size_t i = 0; i < c.size(); ++i) {
      ov[2 * i] = c[i].x;
      ov[2 * i + 1] = c[i].y;
    }
  });
}

int abd_set_candidates(abd_scene* h, int64_t n_vf, const int64_t* vf, int64_t n_ee, const int64_t* ee, int64_t n_ov,
                       const int64_t* ov) {
  return guard([&] {
    SC(h);
    std::vector<int4> a(n_vf), b(n_ee);
    std::vector<int2> c(n_ov);
    for (int64_t i = 0; i < n_vf; ++i) a[i] = make_int4((int)vf[4 * i], (int)vf[4 * i + 1], (int)vf[4 * i + 2], (int)vf[4 * i + 3]);
    for (int64_t i = 0; i < n_ee; ++i) b[i] = make_int4((int)ee[4 * i], (int)ee[4 * i + 1], (int)ee[4 * i + 2], (int)ee[4 * i + 3]);
    for (int64_t i = 0; i < n_ov; ++i) c[i] = make_int2((int)ov[2 * i], (int)ov[2 * i + 1]);
    s.cands.vf.upload(a.data(), n_vf, s.stream);
    s.cands.ee.upload(b.data(), n_ee, s.stream);
    s.cands.ov.upload(c.data(), n_ov, s.stream);
    s.cands.n_vf = n_vf;
    s.cands.n_ee = n_ee;
    s.cands.n_ov = n_ov;
    s.cands.gen += 1;
    sync(s.stream);
  });
}

static const double* up_q(Scene& s, DVec<double>& buf, const double* q) {
  buf.upload(q, 12 * (size_t)s.B, s.stream);
  return buf.p;
}

int abd_contact_energy(abd_scene* h, const double* q, double kappa, double d_hat, double* energy) {
  return guard([&] {
    SC(h);
    *energy = contact_energy(s, up_q(s, s.q_trial, q), kappa, d_hat);
  });
}

int abd_candidate_min_d2(abd_scene* h, const double* q, double* d2) {
  return guard([&] {
    SC(h);
    *d2 = candidate_min_d2(s, up_q(s, s.q_trial, q));
  });
}

int abd_tri_intersect_batch(int64_t n, const double* tri_a, const double* tri_b, uint8_t* out) {
  return guard([&] {
    ensure_device();
    if (n < 0) throw Error(ABD_ERR_ARG, "n < 0");
    if (n == 0) return;
    cudaStream_t st = g_stream();
    Dev<double> da(st), db(st);
    Dev<unsigned char> dout(st);
    launch_tri_intersect(st, n, da.up(tri_a, 9 * n), db.up(tri_b, 9 * n), dout.alloc(n));
    dout.down(out, n);
    sync(st);
  });
}

int abd_intersecting_pairs(abd_scene* h, const double* q, int64_t cap, int64_t* pairs, int64_t* n_pairs) {
  return guard([&] {
    SC(h);
    std::vector<int2> r = intersecting_body_pairs(s, up_q(s, s.q_trial, q));
    *n_pairs = (int64_t)r.size();
    for (int64_t k = 0; k < std::min<int64_t>(cap, (int64_t)r.size()); ++k) {
      pairs[2 * k] = r[k].x;
      pairs[2 * k + 1] = r[k].y;
    }
  });
}

int abd_world_vertices(abd_scene* h, const double* q, double* out) {
  return guard([&] {
    SC(h);
    const double* qd = q ? up_q(s, s.q_trial, q) : s.q.p;
    DVec<double>& X = s.w.basis;  // scratch
    X.resize(3 * std::max<int64_t>(s.V, 1));
    world_vertices(s, qd, X.p);
    if (s.V) X.download(out, 3 * (size_t)s.V, s.stream);
    sync(s.stream);
  });
}

static std::vector<int64_t> canonical_record_order(Scene& s, int64_t total);

int abd_resident_generation(abd_scene* h, int64_t* cand_gen, int64_t* fric_gen) {
  return guard([&] {
    SC(h);
    *cand_gen = s.cands.gen;
    *fric_gen = s.fric.gen;
  });
}

int abd_global_min_distance(abd_scene* h, const double* q, int skip_static_pairs, double* dist) {
  return guard([&] {
    SC(h);
    *dist = global_min_distance(s, up_q(s, s.q_trial, q), skip_static_pairs ? 1 : 0);
  });
}

int abd_contact_gradient_hessian(abd_scene* h, const double* q, double kappa, double d_hat, int project,
                                 int64_t* n_active) {
  return guard([&] {
    SC(h);
    *n_active = contact_blocks(s, up_q(s, s.q_trial, q), kappa, d_hat, project);
    s.pblk_order = canonical_record_order(s, *n_active);
  });
}

// The device keeps active pair records in its own candidate order (per overlap pair);
// the reference lists them as the active VF rows in canonical (c0, c2, c1, c3) order,
// then the active EE rows (contact.py:646-675, :722-790).  Right after an active scan,
// w.act[p] is the candidate slot of record p (VF slots first): the permutation that
// reads the records out in the reference's order.
static std::vector<int64_t> canonical_record_order(Scene& s, int64_t total) {
  std::vector<int64_t> perm(total);
  if (total <= 0) return perm;
  std::vector<int> act(total);
  std::vector<int4> vf(s.cands.n_vf), ee(s.cands.n_ee);
  CK(cudaMemcpyAsync(act.data(), s.w.act.p, total * sizeof(int), cudaMemcpyDeviceToHost, s.stream));
  s.cands.vf.download(vf.data(), vf.size(), s.stream);
  s.cands.ee.download(ee.data(), ee.size(), s.stream);
  sync(s.stream);
  const int64_t n_vf = s.cands.n_vf;
  auto row = [&](int64_t p) -> const int4& { return act[p] < n_vf ? vf[act[p]] : ee[act[p] - n_vf]; };
  for (int64_t p = 0; p < total; ++p) perm[p] = p;
  std::sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) {
    const bool ka = act[a] >= n_vf, kb = act[b] >= n_vf;
    if (ka != kb) return kb;
    const int4 &p = row(a), &q = row(b);
    if (p.x != q.x) return p.x < q.x;
    if (p.z != q.z) return p.z < q.z;
    if (p.y != q.y) return p.y < q.y;
    return p.w < q.w;
  });
  return perm;
}

int abd_get_pair_blocks(abd_scene* h, int64_t* body_a, int64_t* body_b, double* grad, double* hess, double* d_sq) {
  return guard([&] {
    SC(h);
    int64_t n = s.pblk.n;
    std::vector<int2> b(n);
    std::vector<double> blk((size_t)n * PB_DENSE), d2(n);
    s.pblk.bodies.download(b.data(), n, s.stream);
    // compact records -> dense g24 | H_aa | H_bb | H_ab for readout
    DVec<double> dense;
    dense.resize(std::max<size_t>((size_t)n * PB_DENSE, 1));
    launch_pblk_dense(s.stream, n, s.pblk.blk.p, dense.p);
    dense.download(blk.data(), (size_t)n * PB_DENSE, s.stream);
    s.pblk.d2.download(d2.data(), n, s.stream);
    sync(s.stream);
    const bool ordered = (int64_t)s.pblk_order.size() == n;
    for (int64_t k = 0; k < n; ++k) {
      const int64_t i = k;
      const int64_t src = ordered ? s.pblk_order[k] : k;
      if (body_a) body_a[i] = b[src].x;
      if (body_b) body_b[i] = b[src].y;
      if (d_sq) d_sq[i] = d2[src];
      const double* o = &blk[(size_t)src * PB_DENSE];
      if (grad) std::memcpy(grad + 24 * i, o, 24 * sizeof(double));
      if (hess) {
        double* H = hess + 576 * i;
        for (int r = 0; r < 12; ++r)
          for (int c = 0; c < 12; ++c) {
            H[r * 24 + c] = o[24 + r * 12 + c];
            H[(r + 12) * 24 + c + 12] = o[24 + 144 + r * 12 + c];
            H[r * 24 + c + 12] = o[24 + 288 + r * 12 + c];
            H[(c + 12) * 24 + r] = o[24 + 288 + r * 12 + c];
          }
      }
    }
  });
}

int abd_friction_precompute(abd_scene* h, const double* q_prev, double kappa, double d_hat, double mu, int64_t* n) {
  return guard([&] {
    SC(h);
    static thread_local DVec<double>* basis = nullptr;
    if (!basis) basis = new DVec<double>();
    *n = friction_precompute(s, up_q(s, s.q_trial, q_prev), kappa, d_hat, mu, basis);
    s.fric_order = canonical_record_order(s, *n);
    s.fric_order_gen = s.fric.gen;
    s.red.resize(std::max<int64_t>(*n, 1) * 6);
    CK(cudaMemcpyAsync(s.red.p, basis->p, std::max<int64_t>(*n, 1) * 6 * sizeof(double), cudaMemcpyDeviceToDevice,
                       s.stream));
    sync(s.stream);
  });
}

int abd_get_friction(abd_scene* h, int64_t* body_a, int64_t* body_b, double* lam, double* tangent_map, double* offset,
                     double* basis) {
  return guard([&] {
    SC(h);
    int64_t n = s.fric.n;
    std::vector<int2> b(n);
    std::vector<double> rec((size_t)n * FRIC_STRIDE), bs((size_t)n * 6);
    s.fric.bodies.download(b.data(), n, s.stream);
    s.fric.rec.download(rec.data(), (size_t)n * FRIC_STRIDE, s.stream);
    if (basis && n) CK(cudaMemcpyAsync(bs.data(), s.red.p, n * 6 * sizeof(double), cudaMemcpyDeviceToHost, s.stream));
    sync(s.stream);
    // reference order when this set came from abd_friction_precompute (else device order)
    const bool ordered = s.fric_order_gen == s.fric.gen && (int64_t)s.fric_order.size() == n;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t k = ordered ? s.fric_order[i] : i;
      body_a[i] = b[k].x;
      body_b[i] = b[k].y;
      const double* r = &rec[(size_t)k * FRIC_STRIDE];
      std::memcpy(tangent_map + 48 * i, r, 48 * sizeof(double));
      offset[2 * i] = r[48];
      offset[2 * i + 1] = r[49];
      lam[i] = r[50];
      if (basis) std::memcpy(basis + 6 * i, &bs[6 * k], 6 * sizeof(double));
    }
  });
}

int abd_set_friction(abd_scene* h, int64_t n, const int64_t* body_a, const int64_t* body_b, const double* lam, double mu,
                     const double* tangent_map, const double* offset) {
  return guard([&] {
    SC(h);
    std::vector<int2> hb;
    std::vector<double> hr;
    pack_friction(n, body_a, body_b, lam, tangent_map, offset, hb, hr);
    s.fric.bodies.upload(hb.data(), hb.size(), s.stream);
    s.fric.rec.upload(hr.data(), hr.size(), s.stream);
    s.fric.n = n;
    s.fric.gen += 1;
    s.fric.mu = mu;
    sync(s.stream);
  });
}

int abd_step_filter(abd_scene* h, const double* q, const double* dq, double slack, double* alpha) {
  return guard([&] {
    SC(h);
    const double* dqq = up_q(s, s.q_trial, q);
    s.dq.upload(dq, 12 * (size_t)s.B, s.stream);
    *alpha = step_filter(s, dqq, s.dq.p, slack);
  });
}

int abd_compute_q_tilde(abd_scene* h, const double* q, const double* q_dot, const double* forces, double dt,
                        double* q_tilde) {
  return guard([&] {
    SC(h);
    size_t NB = 12 * (size_t)s.B;
    DVec<double> a, b, c, o;
    a.upload(q, NB, s.stream);
    b.upload(q_dot, NB, s.stream);
    c.upload(forces, NB, s.stream);
    o.resize(NB);
    launch_q_tilde(s, a.p, b.p, c.p, dt, o.p);
    o.download(q_tilde, NB, s.stream);
    sync(s.stream);
  });
}

int abd_ip_value(abd_scene* h, const double* q, const double* q_tilde, double dt, double kappa, double d_hat,
                 double eps_v, double* value) {
  return guard([&] {
    SC(h);
    s.q_tilde.upload(q_tilde, 12 * (size_t)s.B, s.stream);
    *value = ip_value(s, up_q(s, s.q_trial, q), s.q_tilde.p, dt, kappa, d_hat, eps_v);
  });
}

int abd_assemble(abd_scene* h, const double* q, const double* q_tilde, double dt, double kappa, double d_hat,
                 double eps_v, int64_t* n_off) {
  return guard([&] {
    SC(h);
    s.q_tilde.upload(q_tilde, 12 * (size_t)s.B, s.stream);
    assemble(s, up_q(s, s.q_trial, q), s.q_tilde.p, dt, kappa, d_hat, eps_v);
    *n_off = s.H.n_off;
  });
}

int abd_get_system(abd_scene* h, double* grad, double* diag, int64_t* off_keys, double* off_blocks) {
  return guard([&] {
    SC(h);
    Bsr& H = s.H;
    int n = H.n;
    std::vector<double> val((size_t)H.nnzb * 144);
    std::vector<int> dpos(n), upos(H.n_off);
    std::vector<int2> keys(H.n_off);
    H.val.download(val.data(), val.size(), s.stream);
    H.diag_pos.download(dpos.data(), n, s.stream);
    H.upper_pos.download(upos.data(), H.n_off, s.stream);
    H.upper_keys.download(keys.data(), H.n_off, s.stream);
    if (grad) s.grad.download(grad, 12 * (size_t)n, s.stream);
    sync(s.stream);
    for (int i = 0; i < n; ++i)
      if (diag) std::memcpy(diag + 144 * (size_t)i, &val[144 * (size_t)dpos[i]], 144 * sizeof(double));
    for (int64_t k = 0; k < H.n_off; ++k) {
      if (off_keys) {
        off_keys[2 * k] = keys[k].x;
        off_keys[2 * k + 1] = keys[k].y;
      }
      if (off_blocks) std::memcpy(off_blocks + 144 * k, &val[144 * (size_t)upos[k]], 144 * sizeof(double));
    }
  });
}

int abd_solve_resident(abd_scene* h, double rel_tol, int max_iters, double* dx, int* iters, double* rel_res) {
  return guard([&] {
    SC(h);
    const int64_t N = 12 * (int64_t)s.H.n;
    // -g and x stay on the device (the scene's persistent Newton workspaces)
    s.w.neg.resize(std::max<int64_t>(N, 1));
    s.dx.resize(std::max<int64_t>(N, 1));
    launch_neg(s.stream, N, s.grad.p, s.w.neg.p);
    double rel = 0.0;
    int it = pcg_solve(s, s.w.neg.p, s.dx.p, rel_tol, max_iters, rel);
    s.dx.download(dx, N, s.stream);
    sync(s.stream);
    if (iters) *iters = it;
    if (rel_res) *rel_res = rel;
  });
}

int abd_solve_resident_cholesky(abd_scene* h, double rel_tol, double* dx, int* solves, double* rel_res) {
  return guard([&] {
    SC(h);
    const int64_t N = 12 * (int64_t)s.H.n;
    s.w.neg.resize(std::max<int64_t>(N, 1));
    s.dx.resize(std::max<int64_t>(N, 1));
    launch_neg(s.stream, N, s.grad.p, s.w.neg.p);
    double rel = 0.0;
    int ns = chol_solve(s, s.w.neg.p, s.dx.p, rel_tol, rel);
    s.dx.download(dx, N, s.stream);
    sync(s.stream);
    if (solves) *solves = ns;
    if (rel_res) *rel_res = rel;
  });
}

int abd_kernel_stats(abd_scene* h, int which, int64_t* launches, double* ms, double* bytes, int64_t* units) {
  return guard([&] {
    SC(h);
    if (which < 0 || which > 3) throw Error(ABD_ERR_ARG, "kernel stats index out of range");
    kstat_flush(s, which);
    Scene::KStat& k = s.kstat[which];
    if (launches) *launches = k.launches;
    if (ms) *ms = k.ms;
    if (bytes) *bytes = k.bytes;
    if (units) *units = k.units;
  });
}

int abd_kernel_stats_reset(abd_scene* h) {
  return guard([&] {
    SC(h);
    for (auto& k : s.kstat) {
      k.launches = k.units = 0;
      k.ms = k.bytes = 0.0;
      k.pending = false;
    }
  });
}

int abd_timer_start(abd_scene* h) {
  return guard([&] {
    SC(h);
    CK(cudaStreamSynchronize(s.stream));
    host_prof_reset();
    CK(cudaEventRecord(s.tev0, s.stream));
  });
}

int abd_timer_stop(abd_scene* h, double* ms) {
  return guard([&] {
    SC(h);
    CK(cudaEventRecord(s.tev1, s.stream));
    CK(cudaEventSynchronize(s.tev1));
    host_prof_dump();
    float m = 0.f;
    CK(cudaEventElapsedTime(&m, s.tev0, s.tev1));
    *ms = m;
  });
}

int abd_nccl_unique_id(uint8_t* out128) {
  return guard([&] {
    ensure_device();
    comm_get_nccl_id(out128);
  });
}

int abd_scene_set_comm_nccl(abd_scene* h, const uint8_t* id128, int rank, int world) {
  return guard([&] {
    SC(h);
    comm_init_nccl(s, id128, rank, world);
  });
}

int abd_scene_set_comm_callback(abd_scene* h, int rank, int world, abd_allreduce_fn fn, void* user) {
  return guard([&] {
    SC(h);
    comm_init_callback(s, rank, world, fn, user);
  });
}

int abd_set_state(abd_scene* h, const double* q, const double* q_dot) {
  return guard([&] {
    SC(h);
    if (q) s.q.upload(q, 12 * (size_t)s.B, s.stream);
    if (q_dot) s.q_dot.upload(q_dot, 12 * (size_t)s.B, s.stream);
    sync(s.stream);
  });
}

int abd_get_state(abd_scene* h, double* q, double* q_dot) {
  return guard([&] {
    SC(h);
    if (q) s.q.download(q, 12 * (size_t)s.B, s.stream);
    if (q_dot) s.q_dot.download(q_dot, 12 * (size_t)s.B, s.stream);
    sync(s.stream);
  });
}

int abd_get_slab_owner(abd_scene* h, int32_t* owner, int32_t* axis) {
  return guard([&] {
    SC(h);
    if (!s.slab_valid) throw Error(ABD_ERR_ARG, "no slab partition (single-rank scene or no step yet)");
    for (int b = 0; b < s.B; ++b) owner[b] = s.h_slab_owner[b];
    if (axis) *axis = s.slab_axis;
  });
}

int abd_set_reduction(abd_scene* h, int64_t n_unknowns, const double* T) {
  return guard([&] {
    SC(h);
    if (n_unknowns > 0 && !T) throw Error(ABD_ERR_ARG, "null reduction matrix");
    set_reduction(s, n_unknowns, T);
  });
}

int abd_advance_step(abd_scene* h, const double* forces, const abd_step_params* p, abd_step_stats* st,
                     double* energy_trace) {
  return guard([&] {
    SC(h);
    advance_step(s, forces, *p, *st, energy_trace);
  });
}

}  // extern "C"
