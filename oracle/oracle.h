/* oracle.h -- plain, slow, fp64 CPU oracle for the cell-local reactive update
 * of arXiv 2312.13513 (thermo Newton + transport + DNN chemistry).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path in
 * paper_2312_13513_b200/ and neither side includes the other.
 *
 * Every function follows SURVEY.md §8(c) steps 1-10 (the build's reading of
 * PAPER.md §2 line 114 and §3.1) in that order, in IEEE fp64, scalar,
 * with sums in index order.  Cells are independent; threads split the cell
 * range only (no arithmetic is reordered by threading).
 *
 * Layout: per-cell fields are component-major (SoA): field[k*ld + c].
 */
#ifndef RC_ORACLE_H
#define RC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_RU 8314.46261815324 /* J/kmol/K, reading R12 */

typedef struct {
  int32_t ns, ne;
  const double *W_elem;   /* [ne] kg/kmol */
  const int32_t *atoms;   /* [ne][ns] */
  const double *nasa_lo;  /* [ns][7] */
  const double *nasa_hi;  /* [ns][7] */
  const double *T_lo, *T_mid, *T_hi; /* [ns] */
  const double *visc;     /* [ns][5]  sqrt(mu_k)/T^(1/4) in powers of ln T */
  const double *cond;     /* [ns][5]  lambda_k/sqrt(T) */
  const double *diff;     /* [ns(ns+1)/2][5] D_jk p/T^(3/2), packed j<=k at k(k+1)/2+j */
  const uint8_t *inert;   /* [ns] */
} orc_mech;

typedef struct {
  int32_t n_nets, d_in;       /* d_in = ns + 2 */
  int32_t hidden[3];          /* (1600, 800, 400) paper; (64, 32, 16) C1 */
  const int32_t *species_of_net; /* [n_nets] */
  const double *params;       /* per net, concatenated: W1[h1][d_in] b1[h1] W2[h2][h1] b2[h2]
                                 W3[h3][h2] b3[h3] W4[1][h3] b4[1] (row-major [out][in]) */
  const double *x_mean, *x_std; /* [d_in] */
  const double *y_mean, *y_std; /* [n_nets] */
  double lambda_bc, dt;
  int32_t shared;             /* 0: one net per species (reading R1);
                                 1: ONE shared net d_in -> h1 -> h2 -> h3 -> n_nets (SURVEY §8(f) NEXT-2,
                                 reading R20): params = W1 b1 W2 b2 W3 b3 W4[n_nets][h3] b4[n_nets] */
} orc_mlp;

/* ---- per-species / per-cell primitives (exposed for the pin tests) ---- */
double orc_species_cp(const orc_mech *m, int k, double T); /* J/kg/K, step 2 */
double orc_species_h(const orc_mech *m, int k, double T);  /* J/kg,   step 2 */
double orc_mix_W(const orc_mech *m, const double *Y);      /* kg/kmol, step 1 */
double orc_mix_h(const orc_mech *m, const double *Y, double T);
double orc_mix_cp(const orc_mech *m, const double *Y, double T);
/* step 3: returns T; *flags |= 1 bisection used, 2 max-iterations hit */
double orc_T_from_h(const orc_mech *m, const double *Y, double h, double T_guess, int *flags, int *iters);
/* step 5, one cell: X^+ based Wilke mu, Mathur lambda, mixture-averaged D[ns] */
void orc_transport_cell(const orc_mech *m, double T, double p, const double *Y,
                        double *mu, double *lambda, double *D);
double orc_species_mu(const orc_mech *m, int k, double T);
double orc_species_lambda(const orc_mech *m, int k, double T);
double orc_binary_D(const orc_mech *m, int j, int k, double T, double p);
double orc_gelu(double x); /* step 7, exact erf */
/* step 7 for one input row z[d_in]: returns o of net i */
double orc_mlp_forward(const orc_mlp *n, int net, const double *z);
/* step 9: P = I - E^T (E E^T)^-1 E, E_ek = a_ek A_e / W_k; writes P[ns][ns]; returns 0 ok */
int orc_projection(const orc_mech *m, double *P);
/* step 6 for one cell: z[d_in] and b[ns] = max(Y,0)^lambda */
void orc_prologue_cell(const orc_mech *m, const orc_mlp *n, double T, double p, const double *Y,
                       double *z, double *b);

/* step 11 (LES only, reading R19): PaSR fraction kappa = tau_c / (tau_c + tau_mix) of a cell
 * from its laminar sources wdot[ns], density and mass fractions, with the chemical time
 * tau_c = sum_k rho max(Y_k,0)/W_k / (1/2 sum_k |wdot_k|/W_k); kappa = 1 when wdot = 0 */
double orc_pasr_kappa(const orc_mech *m, double rho, const double *Y, const double *wdot, double tau_mix);

/* ---- detailed kinetics (reading R21): the CVODE path's right-hand
 * side ("CVODE on CPU"), mass-action law with Arrhenius rates, reverse rates from the
 * equilibrium constant of the NASA-7 tables, third-body and Lindemann/Troe falloff forms ---- */
typedef struct {
  int32_t nr;
  const int32_t *nu_f, *nu_r;   /* [nr][ns] reactant / product stoichiometric coefficients */
  const int32_t *type;          /* [nr] 0 elementary, 1 three-body (+M), 2 falloff (+M) */
  const int32_t *reversible;    /* [nr] */
  const double *A, *b, *Ea;     /* [nr] k = A T^b exp(-Ea / (R_u T)); SI (kmol, m^3, s, J/kmol) */
  const double *eff;            /* [nr][ns] third-body efficiencies */
  const double *A0, *b0, *Ea0;  /* [nr] falloff low-pressure limit k0 */
  const double *troe;           /* [nr][4] a, T3, T1, T2 (Troe's T***, T*, T**); a < 0: Lindemann (F = 1) */
} orc_kin;

/* g_k = h_k/(R_u T) - s_k/R_u (molar, dimensionless) of species k at T (NASA-7) */
double orc_species_g(const orc_mech *m, int k, double T);
/* forward rate constant of reaction r at T with third-body concentration M (falloff blending) */
double orc_rate_constant(const orc_kin *kin, int r, double T, double M);
/* one cell: wdot[ns] (kg/m^3/s); qnet[nr] rates of progress (kmol/m^3/s, may be NULL);
 * scale[ns] = W_k sum_r |nu_rk| (|q_f,r| + |q_r,r|), the gross rates (may be NULL) */
void orc_kinetics_cell(const orc_mech *m, const orc_kin *kin, double T, double p, const double *Y, double *wdot,
                       double *qnet, double *scale);

/* ---- downstream consumer (reading R22): implicit Laplacian
 * assembly of PAPER.md Algorithm 1 (lines 137-158) on a periodic Cartesian mesh, ldu storage
 * (PAPER.md:160-167), ldu -> CSR.  Cells c = i + nx (j + ny k); face (d, c) joins cell c
 * and its +d neighbour (d = x, y, z; periodic wrap, or the halo plane above the slab in z). ---- */
typedef struct {
  int32_t nx, ny, nz;   /* cells; nz = planes of this slab */
  double dx, dy, dz;    /* m */
} orc_mesh;
/* Laplacian coefficients from the property outputs: gamma[k] = rho D_k (species k < ns),
 * gamma[ns] = lambda / cp (energy); gamma [ns+1][n] */
void orc_laplacian_gamma(int ns, int64_t n, const double *rho, const double *D, const double *lambda,
                         const double *cp, double *gamma);
/* Algorithm 1 for nsys systems: gamma_f = (gamma_P + gamma_N)/2 (linear interpolation, uniform mesh),
 * upper[f] = lower[f] = gamma_f |S_f| / |d_f|, diag[P] -= upper[f], diag[N] -= lower[f], faces in
 * order f = d N + c.  halo_lo / halo_hi [nsys][nx ny]: gamma of the planes below / above the slab
 * (NULL: periodic in z within the slab).  upper [nsys][3 N], diag [nsys][N]. */
void orc_laplacian(const orc_mesh *m, int nsys, const double *gamma, const double *halo_lo, const double *halo_hi,
                   double *upper, double *diag);
/* y = A x for one system in ldu form (periodic slab), x [N], y [N] */
void orc_ldu_matvec(const orc_mesh *m, const double *upper, const double *diag, const double *x, double *y);

/* ---- whole-field entry points (SoA, host arrays) ---- */
typedef struct {
  int64_t n, ld;
  int32_t mode;        /* 0 = h-mode (Newton, T in = guess), 1 = T-mode (T in = value, h out) */
  double *h, *T;
  const double *p, *Y;
  double *cp, *rho, *mu, *lambda, *D; /* D [ns][ld] */
  double *o;           /* [n_nets][ld] raw net outputs (may be NULL) */
  double *wdot;        /* [ns][ld] */
  double *qdot;        /* [ld] */
  double red[2];       /* out: max T, sum qdot (Neumaier) */
  int64_t diag[5];     /* out: newton_bisect, newton_maxit, nonfinite, negY_in, negY_out */
  const double *tau_mix; /* [ld] LES PaSR subgrid mixing time (NULL = laminar), step 11 */
} orc_cells;

/* a1 (+cp, rho); a2 if mu/lambda/D non-NULL; a3-a5 if mlp != NULL and wdot != NULL; a6 reductions.
 * nthreads <= 0 -> all online cores.  Returns 0 on success, <0 on bad arguments. */
int orc_step(const orc_mech *m, const orc_mlp *n, orc_cells *c, int nthreads);

/* detailed-kinetics sources of every cell at the given T (T-mode values), p, Y: wdot, qdot (PaSR
 * scaled if c->tau_mix), red = {max T, sum qdot}; wscale [ns][ld] (may be NULL) = the gross rates
 * W_k sum_r |nu_rk| (|q_f| + |q_r|) of each cell (the parity scale of wdot).  Returns 0 ok. */
int orc_kinetics(const orc_mech *m, const orc_kin *kin, orc_cells *c, double *wscale, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
