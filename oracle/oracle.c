/* oracle.c -- plain fp64 CPU oracle for the cell-local reactive update.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Written from the paper and the
 * build's readings of it, never from the CUDA path:
 *   PAPER.md:114 (§2)   per-species GELU MLPs 1600/800/400, inputs T, p, Y
 *   PAPER.md:135 (§3.1) "Newton's method and high-order temperature polynomials"
 *   PAPER.md:112 (§2)   transport "via the Cantera interface"
 *   SURVEY.md §8(c) steps 1-10 and DESIGN.md readings R1-R16 fill in what the
 *   paper leaves unstated (Box-Cox, Wilke/Mathur, mixture-averaged D, element
 *   projection, dt).
 * Every quantity is IEEE fp64; every sum runs in index order; compile with
 * -ffp-contract=off so no multiply-add is fused behind the reader's back.
 *
 * Parity status of each function is pinned in tests/test_oracle_*.py:
 *   thermo (cp, h, W, rho, Newton)  pinned: closed forms, finite differences,
 *                                   round trip, single-species reduction
 *   transport mixing rules          pinned: pure-species limits, binary closed
 *                                   forms, Wilke symmetry, Blanc trace limit
 *   transport fit coefficients      parity unpinned against real data (no
 *                                   Cantera): self-consistency + handbook sanity
 *   GELU / MLP                      pinned: erf values, torch float64 forward,
 *                                   hand-computable nets
 *   Box-Cox / projection / sources  pinned: inverse(forward) identity, P^2=P,
 *                                   E P = 0, zero-output identity, sum wdot = 0
 *   whole chemistry vs the paper's trained DNN: parity unpinned (no weights)
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <sched.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

/* ------------------------------------------------------------------ */
/* step 1 -- mixture molar mass W = 1 / sum_k Y_k / W_k                 */
/* ------------------------------------------------------------------ */
static double species_W(const orc_mech *m, int k) {
  /* W_k = sum_e a_ek A_e (keeps sum_e E_ek = 1 exact) */
  double w = 0.0;
  for (int e = 0; e < m->ne; ++e) w += (double)m->atoms[e * m->ns + k] * m->W_elem[e];
  return w;
}

double orc_mix_W(const orc_mech *m, const double *Y) {
  double s = 0.0;
  for (int k = 0; k < m->ns; ++k) s += Y[k] / species_W(m, k);
  return 1.0 / s;
}

/* ------------------------------------------------------------------ */
/* step 2 -- NASA-7 per species; range T <= T_mid -> low (reading R9)   */
/* ------------------------------------------------------------------ */
static const double *nasa_coeffs(const orc_mech *m, int k, double T) {
  return (T <= m->T_mid[k]) ? &m->nasa_lo[7 * k] : &m->nasa_hi[7 * k];
}

double orc_species_cp(const orc_mech *m, int k, double T) {
  const double *a = nasa_coeffs(m, k, T);
  /* cp_k = (R_u/W_k)(a1 + a2 T + a3 T^2 + a4 T^3 + a5 T^4) */
  double cpR = a[0] + a[1] * T + a[2] * T * T + a[3] * T * T * T + a[4] * T * T * T * T;
  return ORC_RU / species_W(m, k) * cpR;
}

double orc_species_h(const orc_mech *m, int k, double T) {
  const double *a = nasa_coeffs(m, k, T);
  /* h_k = (R_u/W_k)(a1 T + a2 T^2/2 + a3 T^3/3 + a4 T^4/4 + a5 T^5/5 + a6) */
  double hR = a[0] * T + a[1] * T * T / 2.0 + a[2] * T * T * T / 3.0 + a[3] * T * T * T * T / 4.0 +
              a[4] * T * T * T * T * T / 5.0 + a[5];
  return ORC_RU / species_W(m, k) * hR;
}

double orc_mix_h(const orc_mech *m, const double *Y, double T) {
  double h = 0.0;
  for (int k = 0; k < m->ns; ++k) h += Y[k] * orc_species_h(m, k, T);
  return h;
}

double orc_mix_cp(const orc_mech *m, const double *Y, double T) {
  double cp = 0.0;
  for (int k = 0; k < m->ns; ++k) cp += Y[k] * orc_species_cp(m, k, T);
  return cp;
}

/* ------------------------------------------------------------------ */
/* step 3 -- Newton h -> T with clamp, then bisection fallback (R8)     */
/* ------------------------------------------------------------------ */
double orc_T_from_h(const orc_mech *m, const double *Y, double h, double T_guess, int *flags, int *iters) {
  double Tmin = m->T_lo[0], Tmax = m->T_hi[0];
  for (int k = 1; k < m->ns; ++k) {
    if (m->T_lo[k] < Tmin) Tmin = m->T_lo[k];
    if (m->T_hi[k] > Tmax) Tmax = m->T_hi[k];
  }
  double T = T_guess;
  if (T < Tmin) T = Tmin;
  if (T > Tmax) T = Tmax;
  int clamp_hits = 0;
  for (int it = 1; it <= 50; ++it) {
    double dT = (h - orc_mix_h(m, Y, T)) / orc_mix_cp(m, Y, T);
    double Tn = T + dT;
    int clamped = 0;
    if (Tn < Tmin) { Tn = Tmin; clamped = 1; }
    if (Tn > Tmax) { Tn = Tmax; clamped = 1; }
    clamp_hits = clamped ? clamp_hits + 1 : 0;
    if (clamp_hits >= 2) break;
    if (!clamped && fabs(Tn - T) <= 1e-10 * Tn) {
      if (iters) *iters = it;
      return Tn;
    }
    T = Tn;
    if (it == 50 && flags) *flags |= 2;
  }
  /* bisection on [Tmin, Tmax]; h(T) is increasing because cp > 0 */
  if (flags) *flags |= 1;
  double lo = Tmin, hi = Tmax;
  int n = 0;
  while (hi - lo > 1e-10 * (0.5 * (lo + hi))) {
    double mid = 0.5 * (lo + hi);
    if (orc_mix_h(m, Y, mid) < h) lo = mid; else hi = mid;
    ++n;
  }
  if (iters) *iters = 50 + n;
  return 0.5 * (lo + hi);
}

/* ------------------------------------------------------------------ */
/* step 5 -- transport: fits, Wilke, Mathur, mixture-averaged (R10, R11)*/
/* ------------------------------------------------------------------ */
static double poly_lnT(const double *c, double L) {
  /* c0 + c1 L + c2 L^2 + c3 L^3 + c4 L^4 */
  return c[0] + c[1] * L + c[2] * L * L + c[3] * L * L * L + c[4] * L * L * L * L;
}

double orc_species_mu(const orc_mech *m, int k, double T) {
  double r = pow(T, 0.25) * poly_lnT(&m->visc[5 * k], log(T));
  return r * r; /* mu_k = (T^(1/4) P_k(ln T))^2 */
}

double orc_species_lambda(const orc_mech *m, int k, double T) {
  return sqrt(T) * poly_lnT(&m->cond[5 * k], log(T)); /* lambda_k = sqrt(T) Q_k(ln T) */
}

double orc_binary_D(const orc_mech *m, int j, int k, double T, double p) {
  int a = j < k ? j : k, b = j < k ? k : j; /* symmetric, packed a <= b */
  const double *c = &m->diff[5 * (b * (b + 1) / 2 + a)];
  return pow(T, 1.5) * poly_lnT(c, log(T)) / p; /* D_jk = T^(3/2) R_jk(ln T) / p */
}

void orc_transport_cell(const orc_mech *m, double T, double p, const double *Y,
                        double *mu_out, double *lambda_out, double *D_out) {
  int ns = m->ns;
  double Wbar = orc_mix_W(m, Y);
  double Xp[64], mu[64], lam[64];
  for (int k = 0; k < ns; ++k) {
    double X = Y[k] * Wbar / species_W(m, k);
    Xp[k] = X > 0.0 ? X : 0.0; /* X+ = max(X, 0) */
    mu[k] = orc_species_mu(m, k, T);
    lam[k] = orc_species_lambda(m, k, T);
  }
  /* Wilke: mu = sum_k X_k mu_k / sum_j X_j Phi_kj,
     Phi_kj = [1 + sqrt(mu_k/mu_j) (W_j/W_k)^(1/4)]^2 / sqrt(8 (1 + W_k/W_j)) */
  double mix_mu = 0.0;
  for (int k = 0; k < ns; ++k) {
    double den = 0.0;
    for (int j = 0; j < ns; ++j) {
      double Wk = species_W(m, k), Wj = species_W(m, j);
      double t = 1.0 + sqrt(mu[k] / mu[j]) * pow(Wj / Wk, 0.25);
      double phi = t * t / sqrt(8.0 * (1.0 + Wk / Wj));
      den += Xp[j] * phi;
    }
    if (den > 0.0) mix_mu += Xp[k] * mu[k] / den;
  }
  /* Mathur: lambda = 1/2 (sum X_k lambda_k + 1 / sum X_k / lambda_k) */
  double s1 = 0.0, s2 = 0.0;
  for (int k = 0; k < ns; ++k) {
    s1 += Xp[k] * lam[k];
    s2 += Xp[k] / lam[k];
  }
  if (mu_out) *mu_out = mix_mu;
  if (lambda_out) *lambda_out = 0.5 * (s1 + 1.0 / s2);
  if (D_out) {
    /* D_k = (sum_{j!=k} X_j W_j) / (Wbar+ * sum_{j!=k} X_j / D_jk);  D_kk if the sum is 0 */
    double Wp = 0.0;
    for (int j = 0; j < ns; ++j) Wp += Xp[j] * species_W(m, j);
    for (int k = 0; k < ns; ++k) {
      double S = 0.0, num = 0.0;
      for (int j = 0; j < ns; ++j) {
        if (j == k) continue;
        S += Xp[j] / orc_binary_D(m, j, k, T, p);
        num += Xp[j] * species_W(m, j);
      }
      D_out[k] = (S == 0.0) ? orc_binary_D(m, k, k, T, p) : num / (Wp * S);
    }
  }
}

/* ------------------------------------------------------------------ */
/* steps 6-7 -- Box-Cox prologue, exact-erf GELU MLP (R3, R4, R5)       */
/* ------------------------------------------------------------------ */
double orc_gelu(double x) { return 0.5 * x * (1.0 + erf(x / sqrt(2.0))); }

void orc_prologue_cell(const orc_mech *m, const orc_mlp *n, double T, double p, const double *Y,
                       double *z, double *b) {
  double x[66];
  x[0] = T;
  x[1] = p;
  for (int k = 0; k < m->ns; ++k) {
    double Yh = Y[k] > 0.0 ? Y[k] : 0.0;            /* Y^ = max(Y, 0) */
    b[k] = pow(Yh, n->lambda_bc);                   /* b_k = Y^^lambda */
    x[2 + k] = (b[k] - 1.0) / n->lambda_bc;         /* BCT_k = (b_k - 1)/lambda */
  }
  for (int i = 0; i < n->d_in; ++i) z[i] = (x[i] - n->x_mean[i]) / n->x_std[i];
}

/* parameters of one net (one-net-per-species bundles) or of the single shared net */
static int64_t net_param_count(const orc_mlp *n) {
  int64_t d = n->d_in, h1 = n->hidden[0], h2 = n->hidden[1], h3 = n->hidden[2];
  int64_t nout = n->shared ? n->n_nets : 1;
  return h1 * d + h1 + h2 * h1 + h2 + h3 * h2 + h3 + nout * h3 + nout;
}

/* output layer of net `net`: row W4[net] and b4[net] of the shared net, or the net's own W4, b4 */
static void output_layer(const orc_mlp *n, int net, const double **W4, const double **b4) {
  int64_t d = n->d_in, h1 = n->hidden[0], h2 = n->hidden[1], h3 = n->hidden[2];
  const double *P = n->params + (n->shared ? 0 : (int64_t)net * net_param_count(n));
  const double *W4all = P + h1 * d + h1 + h2 * h1 + h2 + h3 * h2 + h3;
  int64_t nout = n->shared ? n->n_nets : 1;
  *W4 = W4all + (n->shared ? (int64_t)net * h3 : 0);
  *b4 = W4all + nout * h3 + (n->shared ? net : 0);
}

/* out[j] = b[j] + sum_{k=0}^{in-1} W[j][k] x[k], sum in index order k = 0, 1, ... */
static void dense_ref(const double *W, const double *bias, int in, int out, const double *x, double *y) {
  for (int j = 0; j < out; ++j) {
    double acc = 0.0;
    for (int k = 0; k < in; ++k) acc += W[(int64_t)j * in + k] * x[k];
    y[j] = acc + bias[j];
  }
}

double orc_mlp_forward(const orc_mlp *n, int net, const double *z) {
  int d = n->d_in, h1 = n->hidden[0], h2 = n->hidden[1], h3 = n->hidden[2];
  const double *P = n->params + (n->shared ? 0 : (int64_t)net * net_param_count(n));
  const double *W1 = P, *b1 = W1 + (int64_t)h1 * d, *W2 = b1 + h1, *b2 = W2 + (int64_t)h2 * h1;
  const double *W3 = b2 + h2, *b3 = W3 + (int64_t)h3 * h2, *W4, *b4;
  output_layer(n, net, &W4, &b4);
  double *a1 = malloc(sizeof(double) * (h1 + h2 + h3));
  double *a2 = a1 + h1, *a3 = a2 + h2, o;
  dense_ref(W1, b1, d, h1, z, a1);
  for (int j = 0; j < h1; ++j) a1[j] = orc_gelu(a1[j]);
  dense_ref(W2, b2, h1, h2, a1, a2);
  for (int j = 0; j < h2; ++j) a2[j] = orc_gelu(a2[j]);
  dense_ref(W3, b3, h2, h3, a2, a3);
  for (int j = 0; j < h3; ++j) a3[j] = orc_gelu(a3[j]);
  dense_ref(W4, b4, h3, 1, a3, &o);
  free(a1);
  return o;
}

/* Same arithmetic as dense_ref (each y[j] = (sum_k W[j][k] x[k] in k order) + b[j]),
 * evaluated with the k loop outside so the compiler can run several j at once.
 * Wt is W transposed ([in][out]); no sum is reassociated. */
static void dense_t(const double *Wt, const double *bias, int in, int out, const double *x, double *y) {
  for (int j = 0; j < out; ++j) y[j] = 0.0;
  for (int k = 0; k < in; ++k) {
    const double xk = x[k];
    const double *w = Wt + (int64_t)k * out;
    for (int j = 0; j < out; ++j) y[j] += w[j] * xk;
  }
  for (int j = 0; j < out; ++j) y[j] += bias[j];
}

/* ------------------------------------------------------------------ */
/* step 9 -- element projection P = I - E^T (E E^T)^-1 E (R6)           */
/* ------------------------------------------------------------------ */
int orc_projection(const orc_mech *m, double *P) {
  int ns = m->ns, ne = m->ne;
  double E[8 * 64], G[8 * 16];
  for (int e = 0; e < ne; ++e)
    for (int k = 0; k < ns; ++k) E[e * ns + k] = m->atoms[e * ns + k] * m->W_elem[e] / species_W(m, k);
  /* G = [E E^T | I], Gauss-Jordan with partial pivoting -> [I | (E E^T)^-1] */
  int w = 2 * ne;
  for (int a = 0; a < ne; ++a)
    for (int b = 0; b < ne; ++b) {
      double s = 0.0;
      for (int k = 0; k < ns; ++k) s += E[a * ns + k] * E[b * ns + k];
      G[a * w + b] = s;
      G[a * w + ne + b] = (a == b) ? 1.0 : 0.0;
    }
  for (int c = 0; c < ne; ++c) {
    int piv = c;
    for (int r = c + 1; r < ne; ++r)
      if (fabs(G[r * w + c]) > fabs(G[piv * w + c])) piv = r;
    if (G[piv * w + c] == 0.0) return -1;
    if (piv != c)
      for (int q = 0; q < w; ++q) { double t = G[c * w + q]; G[c * w + q] = G[piv * w + q]; G[piv * w + q] = t; }
    double d = G[c * w + c];
    for (int q = 0; q < w; ++q) G[c * w + q] /= d;
    for (int r = 0; r < ne; ++r) {
      if (r == c) continue;
      double f = G[r * w + c];
      for (int q = 0; q < w; ++q) G[r * w + q] -= f * G[c * w + q];
    }
  }
  /* P_kj = delta_kj - sum_a sum_b E_ak Ginv_ab E_bj */
  for (int k = 0; k < ns; ++k)
    for (int j = 0; j < ns; ++j) {
      double s = 0.0;
      for (int a = 0; a < ne; ++a)
        for (int b = 0; b < ne; ++b) s += E[a * ns + k] * G[a * w + ne + b] * E[b * ns + j];
      P[k * ns + j] = (k == j ? 1.0 : 0.0) - s;
    }
  return 0;
}

/* ------------------------------------------------------------------ */
/* whole field                                                          */
/* ------------------------------------------------------------------ */
/* step 11, LES partially-stirred reactor (PAPER.md:112 names PaSR for the SGS turbulence-chemistry
 * interaction; its equations are not in the paper, reading R19):
 *   C+_k = rho max(Y_k, 0) / W_k,  1/tau_c = (1/2 sum_k |wdot_k| / W_k) / sum_k C+_k,
 *   kappa = tau_c / (tau_c + tau_mix), and kappa = 1 if sum_k |wdot_k| = 0. */
double orc_pasr_kappa(const orc_mech *m, double rho, const double *Y, const double *wdot, double tau_mix) {
  double conc = 0.0, act = 0.0;
  for (int k = 0; k < m->ns; ++k) {
    double W = species_W(m, k);
    conc += rho * (Y[k] > 0.0 ? Y[k] : 0.0) / W;
    act += fabs(wdot[k]) / W;
  }
  if (act == 0.0) return 1.0;
  double tau_c = conc / (0.5 * act);
  return tau_c / (tau_c + tau_mix);
}

typedef struct {
  const orc_mech *m;
  const orc_mlp *n;
  orc_cells *c;
  const double *P;
  double **Wt;      /* per net: transposed W1, W2, W3 */
  int64_t c0, c1;
  int64_t diag[5];
} job_t;

static int ncpu(void) {
  cpu_set_t s;
  if (sched_getaffinity(0, sizeof s, &s) == 0) return CPU_COUNT(&s);
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static void *run_cells(void *arg) {
  job_t *J = (job_t *)arg;
  const orc_mech *m = J->m;
  const orc_mlp *n = J->n;
  orc_cells *c = J->c;
  int ns = m->ns;
  int64_t ld = c->ld;
  double Y[64], D[64], z[66], b[64], dY[64], dYp[64];
  int h1 = n ? n->hidden[0] : 0, h2 = n ? n->hidden[1] : 0, h3 = n ? n->hidden[2] : 0;
  double *act = n ? malloc(sizeof(double) * (h1 + h2 + h3)) : NULL;
  for (int64_t i = J->c0; i < J->c1; ++i) {
    int negin = 0;
    for (int k = 0; k < ns; ++k) {
      Y[k] = c->Y[k * ld + i];
      if (Y[k] < 0.0) negin = 1;
    }
    J->diag[3] += negin;
    /* steps 3-4: thermo */
    double T;
    if (c->mode == 0) {
      int flags = 0;
      T = orc_T_from_h(m, Y, c->h[i], c->T[i], &flags, NULL);
      if (flags & 1) J->diag[0]++;
      if (flags & 2) J->diag[1]++;
      c->T[i] = T;
    } else {
      T = c->T[i];
      if (c->h) c->h[i] = orc_mix_h(m, Y, T);
    }
    double p = c->p[i];
    double cp = orc_mix_cp(m, Y, T);
    double rho = p * orc_mix_W(m, Y) / (ORC_RU * T);
    if (c->cp) c->cp[i] = cp;
    if (c->rho) c->rho[i] = rho;
    int bad = !isfinite(T) || !isfinite(cp) || !isfinite(rho);
    /* step 5: transport */
    if (c->mu || c->lambda || c->D) {
      double mu, lam;
      orc_transport_cell(m, T, p, Y, &mu, &lam, D);
      if (c->mu) c->mu[i] = mu;
      if (c->lambda) c->lambda[i] = lam;
      if (c->D)
        for (int k = 0; k < ns; ++k) c->D[k * ld + i] = D[k];
      bad |= !isfinite(mu) || !isfinite(lam);
    }
    /* steps 6-10: chemistry */
    if (n && c->wdot) {
      orc_prologue_cell(m, n, T, p, Y, z, b);
      for (int k = 0; k < ns; ++k) dY[k] = 0.0;
      for (int net = 0; net < n->n_nets; ++net) {
        /* hidden layers of this net (of the shared net: once per cell) */
        int g = n->shared ? 0 : net;
        double *a1 = act, *a2 = act + h1, *a3 = a2 + h2, o;
        if (!n->shared || net == 0) {
          const double *const *Wt = (const double *const *)&J->Wt[3 * g];
          const double *Pn = n->params + (int64_t)g * net_param_count(n);
          int d = n->d_in;
          const double *b1 = Pn + (int64_t)h1 * d, *b2 = b1 + h1 + (int64_t)h2 * h1;
          const double *b3 = b2 + h2 + (int64_t)h3 * h2;
          dense_t(Wt[0], b1, d, h1, z, a1);
          for (int j = 0; j < h1; ++j) a1[j] = orc_gelu(a1[j]);
          dense_t(Wt[1], b2, h1, h2, a1, a2);
          for (int j = 0; j < h2; ++j) a2[j] = orc_gelu(a2[j]);
          dense_t(Wt[2], b3, h2, h3, a2, a3);
          for (int j = 0; j < h3; ++j) a3[j] = orc_gelu(a3[j]);
        }
        const double *W4, *b4;
        output_layer(n, net, &W4, &b4);
        dense_ref(W4, b4, h3, 1, a3, &o);
        if (c->o) c->o[net * ld + i] = o;
        /* step 8: inverse Box-Cox */
        int s = n->species_of_net[net];
        double Delta = o * n->y_std[net] + n->y_mean[net];
        double a = b[s] + n->lambda_bc * Delta;
        double Ystar = a > 0.0 ? pow(a, 1.0 / n->lambda_bc) : 0.0;
        double Yh = Y[s] > 0.0 ? Y[s] : 0.0;
        dY[s] = Ystar - Yh;
      }
      /* step 9: projection */
      int negout = 0;
      for (int k = 0; k < ns; ++k) {
        double s = 0.0;
        for (int j = 0; j < ns; ++j) s += J->P[k * ns + j] * dY[j];
        dYp[k] = s;
        double Yh = Y[k] > 0.0 ? Y[k] : 0.0;
        if (Yh + s < 0.0) negout = 1;
      }
      J->diag[4] += negout;
      /* step 10: sources */
      double w[64];
      for (int k = 0; k < ns; ++k) w[k] = rho * dYp[k] / n->dt;
      /* step 11 (LES): PaSR scaling of the laminar sources */
      if (c->tau_mix) {
        double kappa = orc_pasr_kappa(m, rho, Y, w, c->tau_mix[i]);
        for (int k = 0; k < ns; ++k) w[k] = kappa * w[k];
      }
      double q = 0.0;
      for (int k = 0; k < ns; ++k) {
        c->wdot[k * ld + i] = w[k];
        q -= orc_species_h(m, k, T) * w[k];
        bad |= !isfinite(w[k]);
      }
      if (c->qdot) c->qdot[i] = q;
      bad |= !isfinite(q);
    }
    J->diag[2] += bad;
  }
  free(act);
  return NULL;
}

int orc_step(const orc_mech *m, const orc_mlp *n, orc_cells *c, int nthreads) {
  if (!m || !c || m->ns <= 0 || m->ns > 64 || m->ne <= 0 || m->ne > 8 || c->n < 0 || c->ld < c->n) return -1;
  if (n && (n->d_in != m->ns + 2 || n->n_nets <= 0)) return -1;
  double P[64 * 64];
  if (orc_projection(m, P) != 0) return -2;
  double **Wt = NULL;
  if (n && c->wdot) {
    /* transposed copies of W1..W3 for dense_t (layout only, no arithmetic) */
    Wt = calloc((size_t)3 * n->n_nets, sizeof(double *));
    int dims[4] = {n->d_in, n->hidden[0], n->hidden[1], n->hidden[2]};
    for (int net = 0; net < (n->shared ? 1 : n->n_nets); ++net) {
      const double *W = n->params + (int64_t)net * net_param_count(n);
      for (int l = 0; l < 3; ++l) {
        int in = dims[l], out = dims[l + 1];
        double *t = malloc(sizeof(double) * (size_t)in * out);
        for (int j = 0; j < out; ++j)
          for (int k = 0; k < in; ++k) t[(int64_t)k * out + j] = W[(int64_t)j * in + k];
        Wt[3 * net + l] = t;
        W += (int64_t)in * out + out; /* skip W_l and b_l */
      }
    }
  }
  int nt = nthreads > 0 ? nthreads : ncpu();
  if (nt > c->n) nt = c->n > 0 ? (int)c->n : 1;
  job_t *jobs = calloc((size_t)nt, sizeof(job_t));
  pthread_t *th = calloc((size_t)nt, sizeof(pthread_t));
  for (int t = 0; t < nt; ++t) {
    jobs[t].m = m; jobs[t].n = n; jobs[t].c = c; jobs[t].P = P; jobs[t].Wt = Wt;
    jobs[t].c0 = c->n * t / nt;
    jobs[t].c1 = c->n * (t + 1) / nt;
    pthread_create(&th[t], NULL, run_cells, &jobs[t]);
  }
  for (int k = 0; k < 5; ++k) c->diag[k] = 0;
  for (int t = 0; t < nt; ++t) {
    pthread_join(th[t], NULL);
    for (int k = 0; k < 5; ++k) c->diag[k] += jobs[t].diag[k];
  }
  free(jobs);
  free(th);
  if (Wt) {
    for (int i = 0; i < 3 * n->n_nets; ++i) free(Wt[i]); /* unused slots are NULL */
    free(Wt);
  }
  /* step a6: T_max and Neumaier-compensated sum of qdot (V_c = 1), cell order */
  double Tmax = -INFINITY, s = 0.0, comp = 0.0;
  for (int64_t i = 0; i < c->n; ++i) {
    if (c->T[i] > Tmax) Tmax = c->T[i];
    if (c->qdot && n && c->wdot) {
      double v = c->qdot[i], t = s + v;
      comp += (fabs(s) >= fabs(v)) ? (s - t) + v : (v - t) + s;
      s = t;
    }
  }
  c->red[0] = Tmax;
  c->red[1] = s + comp;
  return 0;
}


/* ====================================================================== detailed kinetics (NEXT-3)
 * Mass-action law (textbook; the CVODE path's right-hand side), R21:
 *   C_k = rho Y_k / W_k                                   [kmol/m^3]
 *   k_f = A T^b exp(-Ea / (R_u T))
 *   three-body: q *= [M],  [M] = sum_k eff_k C_k
 *   falloff: Pr = k0 [M] / k_inf, k_f = k_inf Pr / (1 + Pr) F, F = 1 (Lindemann) or Troe:
 *     Fcent = (1 - a) exp(-T/T3) + a exp(-T/T1) + exp(-T2/T)   (T3, T1, T2 = Troe's T***, T*, T**)
 *     c = -0.4 - 0.67 log10 Fcent, n = 0.75 - 1.27 log10 Fcent, d = 0.14
 *     log10 F = log10 Fcent / (1 + ((log10 Pr + c) / (n - d (log10 Pr + c)))^2)
 *   K_c = exp(-sum_k nu_k g_k) (p0 / (R_u T))^(sum_k nu_k),  nu = nu_r - nu_f, p0 = 101325 Pa
 *   q = k_f (prod_k C_k^nu_f - prod_k C_k^nu_r / K_c)
 *   wdot_k = W_k sum_r nu_rk q_r,   qdot = -sum_k h_k wdot_k  */
#define ORC_P0 101325.0

double orc_species_g(const orc_mech *m, int k, double T) {
  const double *a = nasa_coeffs(m, k, T);
  /* h/RT = a1 + a2 T/2 + a3 T^2/3 + a4 T^3/4 + a5 T^4/5 + a6/T
   * s/R  = a1 ln T + a2 T + a3 T^2/2 + a4 T^3/3 + a5 T^4/4 + a7 */
  double hRT = a[0] + a[1] * T / 2.0 + a[2] * T * T / 3.0 + a[3] * T * T * T / 4.0 + a[4] * T * T * T * T / 5.0 + a[5] / T;
  double sR = a[0] * log(T) + a[1] * T + a[2] * T * T / 2.0 + a[3] * T * T * T / 3.0 + a[4] * T * T * T * T / 4.0 + a[6];
  return hRT - sR;
}

double orc_rate_constant(const orc_kin *kin, int r, double T, double M) {
  double kinf = kin->A[r] * pow(T, kin->b[r]) * exp(-kin->Ea[r] / (ORC_RU * T));
  if (kin->type[r] != 2) return kinf;
  double k0 = kin->A0[r] * pow(T, kin->b0[r]) * exp(-kin->Ea0[r] / (ORC_RU * T));
  double Pr = k0 * M / kinf;
  double F = 1.0;
  const double *tr = kin->troe + 4 * r;
  if (tr[0] >= 0.0) {
    double Fcent = (1.0 - tr[0]) * exp(-T / tr[1]) + tr[0] * exp(-T / tr[2]) + exp(-tr[3] / T);
    double lF = log10(Fcent);
    double c = -0.4 - 0.67 * lF, n = 0.75 - 1.27 * lF, d = 0.14;
    double x = (log10(Pr) + c) / (n - d * (log10(Pr) + c));
    F = pow(10.0, lF / (1.0 + x * x));
  }
  return kinf * (Pr / (1.0 + Pr)) * F;
}

void orc_kinetics_cell(const orc_mech *m, const orc_kin *kin, double T, double p, const double *Y, double *wdot,
                       double *qnet, double *scale) {
  int ns = m->ns;
  double C[64], g[64];
  double rho = p * orc_mix_W(m, Y) / (ORC_RU * T);
  for (int k = 0; k < ns; ++k) {
    C[k] = rho * Y[k] / species_W(m, k);
    g[k] = orc_species_g(m, k, T);
    wdot[k] = 0.0;
    if (scale) scale[k] = 0.0;
  }
  for (int r = 0; r < kin->nr; ++r) {
    const int32_t *nf = kin->nu_f + (int64_t)r * ns, *nr = kin->nu_r + (int64_t)r * ns;
    double M = 0.0;
    for (int k = 0; k < ns; ++k) M += kin->eff[(int64_t)r * ns + k] * C[k];
    double kf = orc_rate_constant(kin, r, T, M);
    double fwd = kf, rev = 0.0;
    for (int k = 0; k < ns; ++k)
      for (int j = 0; j < nf[k]; ++j) fwd *= C[k];
    if (kin->reversible[r]) {
      double sg = 0.0;
      int dnu = 0;
      for (int k = 0; k < ns; ++k) {
        sg += (nr[k] - nf[k]) * g[k];
        dnu += nr[k] - nf[k];
      }
      double Kc = exp(-sg) * pow(ORC_P0 / (ORC_RU * T), dnu);
      rev = kf / Kc;
      for (int k = 0; k < ns; ++k)
        for (int j = 0; j < nr[k]; ++j) rev *= C[k];
    }
    if (kin->type[r] == 1) {
      fwd *= M;
      rev *= M;
    }
    double q = fwd - rev;
    if (qnet) qnet[r] = q;
    for (int k = 0; k < ns; ++k) {
      int nu = nr[k] - nf[k];
      if (nu) wdot[k] += nu * q;
      if (scale && (nf[k] || nr[k])) scale[k] += (nf[k] + nr[k]) * (fabs(fwd) + fabs(rev));
    }
  }
  for (int k = 0; k < ns; ++k) {
    wdot[k] *= species_W(m, k);
    if (scale) scale[k] *= species_W(m, k);
  }
}

typedef struct {
  const orc_mech *m;
  const orc_kin *kin;
  orc_cells *c;
  double *wscale;
  int64_t c0, c1;
  int64_t bad;
} kjob_t;

static void *run_kin(void *arg) {
  kjob_t *J = (kjob_t *)arg;
  const orc_mech *m = J->m;
  orc_cells *c = J->c;
  int ns = m->ns;
  int64_t ld = c->ld;
  double Y[64], w[64], sc[64];
  for (int64_t i = J->c0; i < J->c1; ++i) {
    for (int k = 0; k < ns; ++k) Y[k] = c->Y[k * ld + i];
    double T = c->T[i], p = c->p[i];
    orc_kinetics_cell(m, J->kin, T, p, Y, w, NULL, sc);
    if (c->tau_mix) {
      double rho = p * orc_mix_W(m, Y) / (ORC_RU * T);
      double kappa = orc_pasr_kappa(m, rho, Y, w, c->tau_mix[i]);
      for (int k = 0; k < ns; ++k) w[k] = kappa * w[k];
    }
    double q = 0.0;
    int bad = 0;
    for (int k = 0; k < ns; ++k) {
      c->wdot[k * ld + i] = w[k];
      if (J->wscale) J->wscale[k * ld + i] = sc[k];
      q -= orc_species_h(m, k, T) * w[k];
      bad |= !isfinite(w[k]);
    }
    if (c->qdot) c->qdot[i] = q;
    J->bad += bad | !isfinite(q);
  }
  return NULL;
}

int orc_kinetics(const orc_mech *m, const orc_kin *kin, orc_cells *c, double *wscale, int nthreads) {
  if (!m || !kin || !c || !c->wdot || m->ns <= 0 || m->ns > 64 || c->n < 0 || c->ld < c->n) return -1;
  int nt = nthreads > 0 ? nthreads : ncpu();
  if (nt > c->n) nt = c->n > 0 ? (int)c->n : 1;
  kjob_t *jobs = calloc((size_t)nt, sizeof(kjob_t));
  pthread_t *th = calloc((size_t)nt, sizeof(pthread_t));
  for (int t = 0; t < nt; ++t) {
    jobs[t].m = m; jobs[t].kin = kin; jobs[t].c = c; jobs[t].wscale = wscale;
    jobs[t].c0 = c->n * t / nt;
    jobs[t].c1 = c->n * (t + 1) / nt;
    pthread_create(&th[t], NULL, run_kin, &jobs[t]);
  }
  for (int k = 0; k < 5; ++k) c->diag[k] = 0;
  for (int t = 0; t < nt; ++t) {
    pthread_join(th[t], NULL);
    c->diag[2] += jobs[t].bad;
  }
  free(jobs);
  free(th);
  double Tmax = -INFINITY, s = 0.0, comp = 0.0;
  for (int64_t i = 0; i < c->n; ++i) {
    if (c->T[i] > Tmax) Tmax = c->T[i];
    if (c->qdot) {
      double v = c->qdot[i], t = s + v;
      comp += (fabs(s) >= fabs(v)) ? (s - t) + v : (v - t) + s;
      s = t;
    }
  }
  c->red[0] = Tmax;
  c->red[1] = s + comp;
  return 0;
}


/* ====================================================================== Laplacian assembly (NEXT-1)
 * PAPER.md Algorithm 1: for every face, gamma_f <- interpolation(w, gamma_c) (w = 1/2 on the uniform
 * mesh), upper, lower <- gamma_f delta_f S_f (delta_f = 1/|d_f|, S_f the face area), then the diagonal
 * accumulates -upper at the owner and -lower at the neighbour.  Written face by face in face order. */
void orc_laplacian_gamma(int ns, int64_t n, const double *rho, const double *D, const double *lambda,
                         const double *cp, double *gamma) {
  for (int k = 0; k < ns; ++k)
    for (int64_t c = 0; c < n; ++c) gamma[k * n + c] = rho[c] * D[k * n + c];
  for (int64_t c = 0; c < n; ++c) gamma[(int64_t)ns * n + c] = lambda[c] / cp[c];
}

void orc_laplacian(const orc_mesh *m, int nsys, const double *gamma, const double *halo_lo, const double *halo_hi,
                   double *upper, double *diag) {
  int64_t nx = m->nx, ny = m->ny, nz = m->nz, N = nx * ny * nz, plane = nx * ny;
  double SdX = m->dy * m->dz / m->dx, SdY = m->dx * m->dz / m->dy, SdZ = m->dx * m->dy / m->dz;
  for (int s = 0; s < nsys; ++s) {
    const double *g = gamma + (int64_t)s * N;
    double *up = upper + (int64_t)s * 3 * N, *dg = diag + (int64_t)s * N;
    for (int64_t c = 0; c < N; ++c) dg[c] = 0.0;
    for (int d = 0; d < 3; ++d)
      for (int64_t c = 0; c < N; ++c) {
        int64_t i = c % nx, j = (c / nx) % ny, k = c / plane;
        int64_t nb;               /* neighbour cell, -1: in the halo plane above */
        double gN, SdD = d == 0 ? SdX : d == 1 ? SdY : SdZ;
        if (d == 0) nb = (i + 1 == nx ? 0 : i + 1) + nx * (j + ny * k);
        else if (d == 1) nb = i + nx * ((j + 1 == ny ? 0 : j + 1) + ny * k);
        else nb = (k + 1 < nz) ? c + plane : (halo_hi ? -1 : c + plane - N);
        gN = nb >= 0 ? g[nb] : halo_hi[(int64_t)s * plane + (c - (nz - 1) * plane)];
        double gf = 0.5 * (g[c] + gN);       /* interpolation(w = 1/2) */
        double a = gf * SdD;                 /* gamma_f delta_f S_f */
        up[(int64_t)d * N + c] = a;
        dg[c] -= a;                          /* diag[owner] -= upper */
        if (nb >= 0) dg[nb] -= a;            /* diag[neighbour] -= lower (lower = upper) */
      }
    if (halo_lo) /* faces from the plane below the slab onto plane 0 (owned by the rank below) */
      for (int64_t c = 0; c < plane; ++c) {
        double gf = 0.5 * (halo_lo[(int64_t)s * plane + c] + g[c]);
        dg[c] -= gf * SdZ;
      }
  }
}

void orc_ldu_matvec(const orc_mesh *m, const double *upper, const double *diag, const double *x, double *y) {
  int64_t nx = m->nx, ny = m->ny, nz = m->nz, N = nx * ny * nz, plane = nx * ny;
  for (int64_t c = 0; c < N; ++c) y[c] = diag[c] * x[c];
  for (int d = 0; d < 3; ++d)
    for (int64_t c = 0; c < N; ++c) {
      int64_t i = c % nx, j = (c / nx) % ny, k = c / plane, nb;
      if (d == 0) nb = (i + 1 == nx ? 0 : i + 1) + nx * (j + ny * k);
      else if (d == 1) nb = i + nx * ((j + 1 == ny ? 0 : j + 1) + ny * k);
      else nb = (k + 1 < nz) ? c + plane : c + plane - N;
      double a = upper[(int64_t)d * N + c];
      y[c] += a * x[nb];   /* upper: row owner, column neighbour */
      y[nb] += a * x[c];   /* lower: row neighbour, column owner */
    }
}
