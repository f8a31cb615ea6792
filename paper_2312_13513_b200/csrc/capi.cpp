// capi.cpp -- the C ABI of include/rc.h: argument checks, table building and
// stage dispatch.  Host code only; kernels live in thermo.cu, transport.cu and
// mlp_sm100.cu.  Citations: PAPER.md:114 (§2, DNN), PAPER.md:135 (§3.1, Thermo),
// PAPER.md:180-181 (§3.2, SoA layout, coefficient tables); DESIGN.md readings.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "rc_internal.h"

static thread_local char g_err[512] = "";
static thread_local int64_t g_launches = 0;

int rc_fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}
void rc_count_launch(int n) { g_launches += n; }

int rc_sm_count() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> g(mu);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cache[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 1;
    cache[dev] = n;
  }
  return cache[dev];
}

int rc_resident_blocks(const void *kernel, int threads, size_t smem) {
  struct Key { const void *k; int t; size_t s; int dev; int v; };
  static std::mutex mu;
  static std::vector<Key> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> g(mu);
    for (const Key &e : cache)
      if (e.k == kernel && e.t == threads && e.s == smem && e.dev == dev) return e.v;
  }
  if (smem > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem) != cudaSuccess || per < 1) per = 1;
  const int v = per * rc_sm_count();
  std::lock_guard<std::mutex> g(mu);
  cache.push_back(Key{kernel, threads, smem, dev, v});
  return v;
}
void rc_reset_launches() { g_launches = 0; }

// ---------------------------------------------------------------------------
// per-stage profiling
// ---------------------------------------------------------------------------
namespace {
struct ProfRec {
  int stage;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;      // recorded, not yet read
std::vector<cudaEvent_t> g_pool;  // free events
cudaEvent_t prof_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

ProfScope::ProfScope(int st, cudaStream_t str) : stage(st), s(str), slot(-1) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on) return;
  ProfRec r{st, prof_event(), prof_event()};
  cudaEventRecord(r.a, s);
  slot = (int)g_prof.size();
  g_prof.push_back(r);
}
ProfScope::~ProfScope() {
  if (slot < 0) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  cudaEventRecord(g_prof[slot].b, s);
}

extern "C" int rc_profile_enable(int on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = on != 0;
  return RC_OK;
}

extern "C" int rc_profile_read(double *ms, int64_t *launches, int reset) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (ms) for (int i = 0; i < RC_STAGE_COUNT; ++i) ms[i] = 0.0;
  if (launches) for (int i = 0; i < RC_STAGE_COUNT; ++i) launches[i] = 0;
  for (auto &r : g_prof) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) return rc_fail(RC_ECUDA, "rc_profile_read: event sync failed");
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (r.stage >= 0 && r.stage < RC_STAGE_COUNT) {
      if (ms) ms[r.stage] += t;
      if (launches) launches[r.stage] += 1;
    }
  }
  if (reset) {
    for (auto &r : g_prof) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
    g_prof.clear();
  }
  return RC_OK;
}

extern "C" int rc_overlap_read(int64_t *out, int reset) {
  if (!out) return rc_fail(RC_EINVAL, "rc_overlap_read: NULL out");
  long long v[3];
  const int r = l2_overlap_read(v, reset);
  if (r) return r;
  for (int i = 0; i < 3; ++i) out[i] = v[i];
  return RC_OK;
}

extern "C" int rc_profile_timeline(int32_t *stage, double *t0, double *t1, int max) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (max > 0 && (!stage || !t0 || !t1)) return rc_fail(RC_EINVAL, "rc_profile_timeline: NULL arrays");
  if (g_prof.empty()) return 0;
  for (auto &r : g_prof)
    if (cudaEventSynchronize(r.b) != cudaSuccess) return rc_fail(RC_ECUDA, "rc_profile_timeline: event sync failed");
  const cudaEvent_t origin = g_prof.front().a;
  const int n = (int)g_prof.size();
  for (int i = 0; i < n && i < max; ++i) {
    float a = 0.f, b = 0.f;
    if (cudaEventElapsedTime(&a, origin, g_prof[i].a) != cudaSuccess ||
        cudaEventElapsedTime(&b, origin, g_prof[i].b) != cudaSuccess)
      return rc_fail(RC_ECUDA, "rc_profile_timeline: elapsed time");
    stage[i] = g_prof[i].stage;
    t0[i] = a;
    t1[i] = b;
  }
  return n;
}

extern "C" const char *rc_last_error(void) { return g_err; }
extern "C" const char *rc_version(void) { return "rc-b200 0.1 (sm_100a)"; }
extern "C" int64_t rc_last_launch_count(void) { return g_launches; }

// ---------------------------------------------------------------------------
// mechanism
// ---------------------------------------------------------------------------
static int invert_small(std::vector<double> &G, int n) {  // in-place Gauss-Jordan, partial pivoting
  std::vector<double> I(n * n, 0.0);
  for (int i = 0; i < n; ++i) I[i * n + i] = 1.0;
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(G[r * n + c]) > std::fabs(G[piv * n + c])) piv = r;
    if (G[piv * n + c] == 0.0) return -1;
    for (int q = 0; q < n; ++q) {
      std::swap(G[c * n + q], G[piv * n + q]);
      std::swap(I[c * n + q], I[piv * n + q]);
    }
    double d = G[c * n + c];
    for (int q = 0; q < n; ++q) { G[c * n + q] /= d; I[c * n + q] /= d; }
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      double f = G[r * n + c];
      for (int q = 0; q < n; ++q) { G[r * n + q] -= f * G[c * n + q]; I[r * n + q] -= f * I[c * n + q]; }
    }
  }
  G = I;
  return 0;
}

extern "C" int rc_mech_create(const rc_mech_desc *d, rc_mech **out) {
  rc_reset_launches();
  if (!d || !out) return rc_fail(RC_EINVAL, "rc_mech_create: NULL argument");
  *out = nullptr;
  const int ns = d->ns, ne = d->ne;
  if (ns < 1 || ns > RC_MAX_NS || ne < 1 || ne > RC_MAX_NE)
    return rc_fail(RC_EINVAL, "rc_mech_create: ns=%d ne=%d out of range", ns, ne);
  if (!d->W_elem || !d->atoms || !d->nasa_lo || !d->nasa_hi || !d->T_lo || !d->T_mid || !d->T_hi || !d->visc ||
      !d->cond || !d->diff || !d->inert)
    return rc_fail(RC_EINVAL, "rc_mech_create: NULL table pointer");
  rc_mech *m = new rc_mech();
  m->ns = ns;
  m->ne = ne;
  cudaGetDevice(&m->device);
  m->W.assign(ns, 0.0);
  for (int k = 0; k < ns; ++k) {
    for (int e = 0; e < ne; ++e) m->W[k] += d->atoms[e * ns + k] * d->W_elem[e];
    if (!(m->W[k] > 0.0)) { delete m; return rc_fail(RC_EINVAL, "species %d has non-positive molar mass", k); }
    if (!(d->T_lo[k] < d->T_mid[k] && d->T_mid[k] < d->T_hi[k])) {
      delete m;
      return rc_fail(RC_EINVAL, "species %d: need T_lo < T_mid < T_hi", k);
    }
  }
  m->inert.assign(d->inert, d->inert + ns);
  m->nasa_lo.assign(d->nasa_lo, d->nasa_lo + 7 * ns);
  m->nasa_hi.assign(d->nasa_hi, d->nasa_hi + 7 * ns);
  m->T_mid.assign(d->T_mid, d->T_mid + ns);
  m->Tmin = d->T_lo[0];
  m->Tmax = d->T_hi[0];
  m->uniform_tmid = true;
  for (int k = 1; k < ns; ++k) {
    m->Tmin = std::fmin(m->Tmin, d->T_lo[k]);
    m->Tmax = std::fmax(m->Tmax, d->T_hi[k]);
    if (d->T_mid[k] != d->T_mid[0]) m->uniform_tmid = false;
  }
  // thermo segment: per-range h coefficients pre-scaled by R/W_k and 1/j so that
  // h = T(c1 + T(c2 + T(c3 + T(c4 + T c5)))) + c6 and cp = c1 + T(2c2 + T(3c3 + ...))
  auto &th = m->thermo_host;
  th.assign(ThermoSeg::size(ns), 0.0);
  th[0] = m->Tmin; th[1] = m->Tmax; th[2] = d->T_mid[0]; th[3] = m->uniform_tmid ? 1.0 : 0.0;
  for (int k = 0; k < ns; ++k) {
    double r = RC_RU / m->W[k];
    for (int j = 0; j < 5; ++j) {
      th[ThermoSeg::hlo(ns) + 6 * k + j] = r * d->nasa_lo[7 * k + j] / (j + 1);
      th[ThermoSeg::hhi(ns) + 6 * k + j] = r * d->nasa_hi[7 * k + j] / (j + 1);
    }
    th[ThermoSeg::hlo(ns) + 6 * k + 5] = r * d->nasa_lo[7 * k + 5];
    th[ThermoSeg::hhi(ns) + 6 * k + 5] = r * d->nasa_hi[7 * k + 5];
    th[ThermoSeg::invW(ns) + k] = 1.0 / m->W[k];
    th[ThermoSeg::tmid(ns) + k] = d->T_mid[k];
  }
  // transport segment: fits (diff rows padded to 6) + the factorised Wilke matrices (rc_internal.h)
  auto &tr = m->transport_host;
  tr.assign(TransportSeg::size(ns), 0.0);
  const int np = ns * (ns + 1) / 2;
  std::memcpy(&tr[TransportSeg::visc(ns)], d->visc, sizeof(double) * 5 * ns);
  std::memcpy(&tr[TransportSeg::cond(ns)], d->cond, sizeof(double) * 5 * ns);
  for (int q = 0; q < np; ++q)
    for (int j = 0; j < 5; ++j) tr[TransportSeg::diff(ns) + 6 * q + j] = d->diff[5 * q + j];
  const int nse = TransportSeg::nse(ns);
  for (int k = 0; k < ns; ++k) {
    tr[TransportSeg::W(ns) + k] = m->W[k];
    tr[TransportSeg::invW(ns) + k] = 1.0 / m->W[k];
    for (int j = 0; j < ns; ++j) {
      const double c1 = std::sqrt(std::sqrt(m->W[j] / m->W[k])), c2 = 1.0 / std::sqrt(8.0 * (1.0 + m->W[k] / m->W[j]));
      tr[TransportSeg::M(ns, 0) + k * nse + j] = c2;
      tr[TransportSeg::M(ns, 1) + k * nse + j] = 2.0 * c2 * c1;
      tr[TransportSeg::M(ns, 2) + k * nse + j] = c2 * c1 * c1;
    }
  }
  // element projection P = I - E^T (E E^T)^-1 E, E_ek = a_ek A_e / W_k (R6)
  std::vector<double> E(ne * ns), G(ne * ne, 0.0);
  for (int e = 0; e < ne; ++e)
    for (int k = 0; k < ns; ++k) E[e * ns + k] = d->atoms[e * ns + k] * d->W_elem[e] / m->W[k];
  for (int a = 0; a < ne; ++a)
    for (int b = 0; b < ne; ++b)
      for (int k = 0; k < ns; ++k) G[a * ne + b] += E[a * ns + k] * E[b * ns + k];
  if (invert_small(G, ne) != 0) { delete m; return rc_fail(RC_EINVAL, "singular E E^T (element matrix rank-deficient)"); }
  m->P.assign(ns * ns, 0.0);
  for (int k = 0; k < ns; ++k)
    for (int j = 0; j < ns; ++j) {
      double s = 0.0;
      for (int a = 0; a < ne; ++a)
        for (int b = 0; b < ne; ++b) s += E[a * ns + k] * G[a * ne + b] * E[b * ns + j];
      m->P[k * ns + j] = (k == j ? 1.0 : 0.0) - s;
    }
  // the same projection in factored form for the chemistry epilogue: F = G E, P = I - E^T F
  std::vector<double> EF(2 * ne * ns, 0.0);
  for (int a = 0; a < ne; ++a)
    for (int k = 0; k < ns; ++k) {
      double f = 0.0;
      for (int b = 0; b < ne; ++b) f += G[a * ne + b] * E[b * ns + k];
      EF[a * ns + k] = f;
      EF[(ne + a) * ns + k] = E[a * ns + k];
    }
  m->EF_host = EF;
  if (cudaMalloc(&m->d_EF, EF.size() * 8) != cudaSuccess ||
      cudaMemcpy(m->d_EF, EF.data(), EF.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
    rc_mech_destroy(m);
    return rc_fail(RC_ENOMEM, "rc_mech_create: cudaMalloc failed");
  }
  if (cudaMalloc(&m->d_thermo, th.size() * 8) != cudaSuccess ||
      cudaMalloc(&m->d_transport, tr.size() * 8) != cudaSuccess ||
      cudaMalloc(&m->d_P, (size_t)((ns * ns + 1) & ~1) * 8) != cudaSuccess ||  // padded: 16-byte bulk copies
      cudaMemset(m->d_P, 0, (size_t)((ns * ns + 1) & ~1) * 8) != cudaSuccess) {
    rc_mech_destroy(m);
    return rc_fail(RC_ENOMEM, "rc_mech_create: cudaMalloc failed");
  }
  if (cudaMemcpy(m->d_thermo, th.data(), th.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(m->d_transport, tr.data(), tr.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(m->d_P, m->P.data(), ns * ns * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
    rc_mech_destroy(m);
    return rc_fail(RC_ECUDA, "rc_mech_create: upload failed");
  }
  *out = m;
  return RC_OK;
}

extern "C" void rc_mech_destroy(rc_mech *m) {
  if (!m) return;
  cudaFree(m->d_thermo);
  cudaFree(m->d_transport);
  cudaFree(m->d_P);
  cudaFree(m->d_EF);
  delete m;
}

extern "C" int rc_mech_ns(const rc_mech *m) { return m ? m->ns : 0; }

// ---------------------------------------------------------------------------
// MLP bundle
// ---------------------------------------------------------------------------
extern "C" int rc_mlp_create(const rc_mech *m, const rc_mlp_desc *d, rc_mlp **out) {
  rc_reset_launches();
  if (!m || !d || !out) return rc_fail(RC_EINVAL, "rc_mlp_create: NULL argument");
  *out = nullptr;
  if (!d->species_of_net || !d->params || !d->x_mean || !d->x_std || !d->y_mean || !d->y_std)
    return rc_fail(RC_EINVAL, "rc_mlp_create: NULL array");
  if (d->n_nets < 1 || d->n_nets > m->ns) return rc_fail(RC_EINVAL, "rc_mlp_create: n_nets=%d", d->n_nets);
  const int h1 = d->hidden[0], h2 = d->hidden[1], h3 = d->hidden[2];
  if (h1 < 64 || h2 < 16 || h3 < 16 || h1 % 64 || h2 % 16 || h3 % 16 || h1 > 4096 || h2 > 4096 || h3 > 4096)
    return rc_fail(RC_EUNSUPPORTED, "rc_mlp_create: hidden (%d,%d,%d) must be multiples of (64,16,16)", h1, h2, h3);
  if (d->precision != RC_BF16 && d->precision != RC_TF32 && d->precision != RC_TF32X3)
    return rc_fail(RC_EINVAL, "rc_mlp_create: unknown precision %d", d->precision);
  if (d->flags & ~(RC_MLP_LAYERWISE | RC_MLP_SHARED | RC_MLP_SERIAL)) return rc_fail(RC_EINVAL, "rc_mlp_create: unknown flags 0x%x", d->flags);
  if ((d->flags & RC_MLP_SHARED) && d->precision == RC_TF32X3)
    return rc_fail(RC_EUNSUPPORTED, "rc_mlp_create: RC_MLP_SHARED runs in RC_BF16 or RC_TF32");
  if (!(d->lambda_bc > 0.0) || !(d->dt > 0.0)) return rc_fail(RC_EINVAL, "rc_mlp_create: lambda and dt must be > 0");
  double inv = 1.0 / d->lambda_bc;
  int invi = (int)std::lround(inv);
  if (std::fabs(inv - invi) > 1e-9 * inv || invi < 1 || invi > 16)
    return rc_fail(RC_EUNSUPPORTED, "rc_mlp_create: 1/lambda_bc must be an integer in [1,16]");
  const int d_in = m->ns + 2;
  if (d_in + 2 > 32)  // z row: d_in inputs + two bias columns, padded to 16 or 32
    return rc_fail(RC_EUNSUPPORTED, "rc_mlp_create: d_in=%d too large for the layer-1 tile (ns <= 28)", d_in);
  for (int i = 0; i < d->n_nets; ++i) {
    int s = d->species_of_net[i];
    if (s < 0 || s >= m->ns) return rc_fail(RC_EINVAL, "species_of_net[%d]=%d out of range", i, s);
    for (int k = 0; k < d_in; ++k)
      if (!(d->x_std[k] > 0.0)) return rc_fail(RC_EINVAL, "x_std[%d] must be > 0", k);
  }
  rc_mlp *n = new rc_mlp();
  n->n_nets = d->n_nets;
  n->gnets = (d->flags & RC_MLP_SHARED) ? 1 : d->n_nets;
  n->d_in = d_in;
  n->h1 = h1; n->h2 = h2; n->h3 = h3;
  n->precision = d->precision;
  n->flags = d->flags;
  n->ns = m->ns;
  n->lambda_bc = d->lambda_bc;
  n->inv_lambda = invi;
  n->dt = d->dt;
  n->kpad1 = d_in + 2 <= 16 ? 16 : 32;  // z row: d_in inputs, two constant-1 bias columns, zero padding
  n->species_of_net.assign(d->species_of_net, d->species_of_net + d->n_nets);
  n->species_identity = true;
  for (int i = 0; i < d->n_nets; ++i) n->species_identity &= d->species_of_net[i] == i;
  cudaGetDevice(&n->device);
  int rc = mlp_upload(n, d);
  if (rc != RC_OK) { rc_mlp_destroy(n); return rc; }
  *out = n;
  return RC_OK;
}

extern "C" void rc_mlp_destroy(rc_mlp *n) {
  if (!n) return;
  void *ptrs[] = {n->d_W1, n->d_W2, n->d_W3, n->d_W1lo, n->d_W2lo, n->d_W3lo, n->d_b1, n->d_b2, n->d_b3, n->d_w4, n->d_b4,
                  n->d_b2k, n->d_b3k, n->d_xmean, n->d_xinvstd, n->d_ymean, n->d_ystd, n->d_species};
  for (void *p : ptrs) cudaFree(p);
  delete n;
}

// ---------------------------------------------------------------------------
// cells
// ---------------------------------------------------------------------------
static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

static int check_cells(const rc_mech *m, const rc_cells *c, CellsDev &o) {
  if (!m || !c) return rc_fail(RC_EINVAL, "NULL mech or cells");
  if (c->n < 0 || c->ld < c->n || (c->ld & 1)) return rc_fail(RC_EINVAL, "need 0 <= n <= ld and ld even (n=%lld ld=%lld)",
                                                            (long long)c->n, (long long)c->ld);
  if (c->mode != RC_MODE_H && c->mode != RC_MODE_T) return rc_fail(RC_EINVAL, "mode must be RC_MODE_H or RC_MODE_T");
  if (!c->T || !c->p || !c->Y) return rc_fail(RC_EINVAL, "T, p and Y are required");
  if (c->mode == RC_MODE_H && !c->h) return rc_fail(RC_EINVAL, "h-mode needs h");
  const void *ptrs[] = {c->h, c->T, c->p, c->Y, c->cp, c->rho, c->mu, c->lambda, c->D, c->wdot, c->qdot, c->o, c->tau_mix};
  for (const void *p : ptrs)
    if (p && !aligned16(p)) return rc_fail(RC_EALIGN, "cell arrays must be 16-byte aligned");
  if (((uintptr_t)c->red & 7u) || ((uintptr_t)c->diag & 7u))  // 64-bit atomics only
    return rc_fail(RC_EALIGN, "red / diag must be 8-byte aligned");
  o = CellsDev{c->n, c->ld, c->mode, c->h, c->T, c->p, c->Y, c->cp, c->rho, c->mu, c->lambda, c->D, c->wdot,
               c->qdot, c->o, c->red, c->diag, c->tau_mix};
  return RC_OK;
}

extern "C" int rc_thermo(const rc_mech *m, const rc_cells *c, void *stream) {
  rc_reset_launches();
  CellsDev d;
  int rc = check_cells(m, c, d);
  if (rc) return rc;
  return launch_thermo(m, d, (cudaStream_t)stream);
}

extern "C" int rc_transport(const rc_mech *m, const rc_cells *c, void *stream) {
  rc_reset_launches();
  CellsDev d;
  int rc = check_cells(m, c, d);
  if (rc) return rc;
  if (!c->mu && !c->lambda && !c->D) return RC_OK;
  return launch_transport(m, d, (cudaStream_t)stream);
}

static int chem_checks(const rc_mech *m, const rc_mlp *n, const rc_cells *c, CellsDev &d, void *ws, size_t ws_bytes) {
  int rc = check_cells(m, c, d);
  if (rc) return rc;
  if (!n) return rc_fail(RC_EINVAL, "NULL mlp");
  if (n->ns != m->ns) return rc_fail(RC_EINVAL, "mlp built for ns=%d, mech has ns=%d", n->ns, m->ns);
  if (!c->wdot) return rc_fail(RC_EINVAL, "chemistry needs wdot");
  if (!c->rho) return rc_fail(RC_EINVAL, "chemistry needs rho (from rc_thermo)");
  if (!(std::fabs(c->dt - n->dt) <= 1e-12 * n->dt))
    return rc_fail(RC_EDTMISMATCH, "cells.dt=%g differs from the bundle's training dt=%g", c->dt, n->dt);
  if (c->n > 0 && (!ws || ((uintptr_t)ws & 255u)))
    return rc_fail(RC_EINVAL, "workspace must be non-NULL and 256-byte aligned");
  size_t need = chem_workspace_min_bytes(n, c->n);  // z of every cell + the smallest legal chunk
  if (c->n > 0 && ws_bytes < need) return rc_fail(RC_EINVAL, "workspace too small: %zu < %zu", ws_bytes, need);
  return RC_OK;
}

extern "C" int rc_chem(const rc_mech *m, const rc_mlp *n, const rc_cells *c, void *ws, size_t ws_bytes, void *stream) {
  rc_reset_launches();
  CellsDev d;
  int rc = chem_checks(m, n, c, d, ws, ws_bytes);
  if (rc) return rc;
  return launch_chem(m, n, d, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" size_t rc_workspace_bytes(const rc_mech *m, const rc_mlp *n, int64_t ncells) {
  if (!m || !n || ncells < 0) return 0;
  return chem_workspace_bytes(m, n, ncells);
}

extern "C" int rc_step(const rc_mech *m, const rc_mlp *n, const rc_cells *c, void *ws, size_t ws_bytes, void *stream) {
  rc_reset_launches();
  CellsDev d;
  int rc = n ? chem_checks(m, n, c, d, ws, ws_bytes) : check_cells(m, c, d);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  if (c->red) RC_CUDA_TRY(cudaMemsetAsync(c->red, 0, 2 * sizeof(double), s));
  if (c->diag) RC_CUDA_TRY(cudaMemsetAsync(c->diag, 0, RC_DIAG_COUNT * sizeof(int64_t), s));
  int64_t total = 0;
  if ((rc = launch_thermo(m, d, s))) return rc;
  total += rc_last_launch_count();
  if (c->mu || c->lambda || c->D) {
    rc_reset_launches();
    if ((rc = launch_transport(m, d, s))) return rc;
    total += rc_last_launch_count();
  }
  if (n) {
    rc_reset_launches();
    if ((rc = launch_chem(m, n, d, ws, ws_bytes, s))) return rc;
    total += rc_last_launch_count();
  }
  rc_reset_launches();
  rc_count_launch((int)total);
  return RC_OK;
}

extern "C" int rc_combine_reductions(const double *red_parts, const int64_t *diag_parts, int k, double *red,
                                     int64_t *diag, void *stream) {
  if (k < 1 || !red_parts || !red) return rc_fail(RC_EINVAL, "rc_combine_reductions: bad arguments");
  rc_reset_launches();
  return launch_combine_reductions(red_parts, diag_parts, k, red, diag, static_cast<cudaStream_t>(stream));
}

extern "C" int rc_partition(int64_t n_global, int rank, int world, int64_t *begin, int64_t *end) {
  if (!begin || !end || world < 1 || rank < 0 || rank >= world || n_global < 0)
    return rc_fail(RC_EINVAL, "rc_partition: bad arguments");
  auto bound = [&](int r) -> int64_t {
    if (r >= world) return n_global;
    __int128 b = (__int128)n_global * r / world;
    return (int64_t)(b / 128 * 128);
  };
  *begin = bound(rank);
  *end = bound(rank + 1);
  return RC_OK;
}

// ---------------------------------------------------------------------------
// detailed kinetics (NEXT-3): table building lives in kinetics.cu (kin_build)
// ---------------------------------------------------------------------------
int kin_build(const rc_mech *m, const rc_kin_desc *d, rc_kin *k);

extern "C" int rc_kin_create(const rc_mech *m, const rc_kin_desc *d, rc_kin **out) {
  rc_reset_launches();
  if (!m || !d || !out) return rc_fail(RC_EINVAL, "rc_kin_create: NULL argument");
  *out = nullptr;
  if (d->nr < 1 || d->nr > 256) return rc_fail(RC_EINVAL, "rc_kin_create: nr=%d out of range", d->nr);
  if (!d->nu_f || !d->nu_r || !d->type || !d->reversible || !d->A || !d->b || !d->Ea || !d->eff || !d->A0 ||
      !d->b0 || !d->Ea0 || !d->troe)
    return rc_fail(RC_EINVAL, "rc_kin_create: NULL array");
  rc_kin *k = new rc_kin();
  int rc = kin_build(m, d, k);
  if (rc != RC_OK) { rc_kin_destroy(k); return rc; }
  *out = k;
  return RC_OK;
}

extern "C" void rc_kin_destroy(rc_kin *k) {
  if (!k) return;
  cudaFree(k->d_tab);
  cudaFree(k->d_qpart);
  delete k;
}

extern "C" int rc_kinetics(const rc_mech *m, const rc_kin *k, const rc_cells *c, void *stream) {
  rc_reset_launches();
  CellsDev d;
  int rc = check_cells(m, c, d);
  if (rc) return rc;
  if (!k) return rc_fail(RC_EINVAL, "NULL kinetics handle");
  if (k->ns != m->ns) return rc_fail(RC_EINVAL, "kinetics built for ns=%d, mech has ns=%d", k->ns, m->ns);
  if (!c->wdot) return rc_fail(RC_EINVAL, "rc_kinetics needs wdot");
  return launch_kinetics(m, k, d, (cudaStream_t)stream);
}
