/* rc.h -- C ABI of the B200-native cell-local reactive update (arXiv 2312.13513).
 *
 * The paper's GPU solver computes, per finite-volume cell, thermophysical and
 * transport properties "with Newton's method and high-order temperature
 * polynomials" (§3.1, class Thermo) and the chemical source term
 * by "individual neural networks ... for each component, excluding inert
 * gases", hidden layers 1600/800/400, GELU, inputs "temperature, pressure and
 * mass fractions", output "the rate of change for a given species"
 * (§2, class DNNInference).  This library is that update behind
 * a plain C interface: mechanism tables plus component-major (SoA) cell arrays
 * in, properties and source terms out ("coalesced the same
 * components of fields").  The paper leaves Box-Cox, the mixing rules, the
 * element projection and dt unstated; DESIGN.md lists the readings (R1-R16).
 *
 * Conventions for every call:
 *  - Return value: RC_OK (0) or a negative RC_E* code.  rc_last_error() returns
 *    a thread-local message for the last failure on the calling thread.
 *  - Argument checks happen before any launch; a failing call launches nothing.
 *  - Work is enqueued on the caller's stream; no call synchronises the device,
 *    allocates device memory (except *_create), or copies to the host.
 *  - Handles (rc_mech, rc_mlp) are immutable after create, device-resident on
 *    the device current at create time, and safe to share across streams and
 *    host threads.  Cell arrays and workspace are BORROWED: they must stay
 *    valid until the enqueued work completes.
 *  - Per-cell numerical anomalies never fail a call; they are counted in
 *    rc_cells.diag (SPEC.md:420 precedent: count, don't abort).
 *  - No cross-GPU reduction happens inside the library: multi-GPU callers
 *    all-reduce rc_cells.red / diag themselves (NCCL via torch.distributed).
 *  - Units: SI with kmol (J/kg, J/kg/K, kg/m^3, Pa, K, Pa s, W/m/K, m^2/s,
 *    kg/m^3/s, W/m^3).  h is absolute (formation-inclusive) enthalpy.
 */
#ifndef RC_H
#define RC_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* only the rc_* entry points are exported */
#endif

enum {
  RC_OK = 0,
  RC_EINVAL = -1,        /* bad argument: NULL, size, stride, alignment, range */
  RC_ENOMEM = -2,        /* device allocation failed (create calls only) */
  RC_ECUDA = -3,         /* a CUDA runtime/driver call or launch failed */
  RC_EALIGN = -4,        /* pointer not 16-byte aligned or ld not a multiple of 2 */
  RC_EUNSUPPORTED = -5,  /* shape the kernels do not implement (see each call) */
  RC_EDTMISMATCH = -6    /* rc_cells.dt != the bundle's training dt */
};

enum { RC_MODE_H = 0, RC_MODE_T = 1 };               /* rc_cells.mode */
enum { RC_BF16 = 0, RC_TF32 = 1, RC_TF32X3 = 2 };     /* rc_mlp_desc.precision */
enum { RC_MLP_LAYERWISE = 1, RC_MLP_SHARED = 2, RC_MLP_SERIAL = 4 };     /* rc_mlp_desc.flags */

/* Diagnostic counters in rc_cells.diag[] (int64, accumulated with atomics). */
enum {
  RC_DIAG_NEWTON_BISECT = 0,  /* cells whose Newton fell back to bisection */
  RC_DIAG_NEWTON_MAXIT = 1,   /* ... of which because 50 iterations were reached */
  RC_DIAG_NONFINITE = 2,      /* (cell, stage) pairs with a non-finite output */
  RC_DIAG_NEGY_IN = 3,        /* cells with some input Y_k < 0 (counted by thermo) */
  RC_DIAG_NEGY_OUT = 4,       /* cells with some max(Y_k,0) + dY_k < 0 after projection */
  RC_DIAG_COUNT = 5
};

typedef struct rc_mech rc_mech; /* opaque: device-resident species tables */
typedef struct rc_mlp rc_mlp;   /* opaque: device-resident MLP bundle */

/* ---------------------------------------------------------------------------
 * Mechanism tables (HOST pointers; copied at create; caller may free after).
 * Limits: 1 <= ns <= 32 (kernels specialise ns = 9 and ns = 20; others run a
 * generic path), 1 <= ne <= 8.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t ns, ne;                 /* species, elements */
  const double *W_elem;           /* [ne] atomic weights, kg/kmol; W_k = sum_e atoms[e][k] W_elem[e] */
  const int32_t *atoms;           /* [ne][ns] atom counts a_ek */
  const double *nasa_lo;          /* [ns][7] NASA-7 a1..a7, T_lo <= T <= T_mid */
  const double *nasa_hi;          /* [ns][7] NASA-7 a1..a7, T_mid <  T <= T_hi */
  const double *T_lo, *T_mid, *T_hi; /* [ns] K */
  const double *visc;             /* [ns][5]  sqrt(mu_k)/T^(1/4) = sum_n c_n (ln T)^n */
  const double *cond;             /* [ns][5]  lambda_k/sqrt(T)   = sum_n c_n (ln T)^n */
  const double *diff;             /* [ns(ns+1)/2][5] D_jk p/T^(3/2) = sum_n c_n (ln T)^n, packed j<=k at k(k+1)/2+j */
  const uint8_t *inert;           /* [ns] 1 = no net predicts this species ("excluding inert gases") */
} rc_mech_desc;

/* Builds, on the current device: molar masses, per-range mixture-NASA
 * coefficient rows, Wilke constants (W_j/W_k)^(1/4) and 1/sqrt(8(1+W_k/W_j)),
 * and the element projection P = I - E^T (E E^T)^-1 E with E_ek = a_ek A_e/W_k
 * (reading R6).  Errors: RC_EINVAL (NULL/range, singular E E^T),
 * RC_ENOMEM, RC_ECUDA. */
int rc_mech_create(const rc_mech_desc *desc, rc_mech **out);
void rc_mech_destroy(rc_mech *m);
int rc_mech_ns(const rc_mech *m);

/* ---------------------------------------------------------------------------
 * MLP bundle (HOST pointers, fp64; converted at create).  One net per
 * non-inert species, d_in = ns + 2 inputs [T, p, BCT(Y_1..ns)], hidden widths
 * hidden[0..2], 1 output.  Row-major [out][in] weights.
 * Kernels require hidden[1] % 16 == 0 and
 * hidden[2] % 16 == 0 (hidden[0] % 64 == 0 for the fused layer-1/2 kernel), and ns <= 28 (else RC_EUNSUPPORTED).
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t n_nets;                 /* = number of non-inert species */
  int32_t hidden[3];              /* (1600, 800, 400) in the paper */
  const int32_t *species_of_net;  /* [n_nets] species index predicted by net i */
  const double *params;           /* [n_nets][P] per net: W1[h1][d_in] b1[h1] W2[h2][h1] b2[h2]
                                     W3[h3][h2] b3[h3] W4[1][h3] b4[1] */
  const double *x_mean, *x_std;   /* [d_in] input z-score (R4) */
  const double *y_mean, *y_std;   /* [n_nets] output de-normalisation (R2) */
  double lambda_bc;               /* Box-Cox lambda (R3; 0.1) -- must satisfy 1/lambda integer <= 16 */
  double dt;                      /* training dt of the bundle, s (R7) */
  int32_t precision;              /* RC_BF16: bf16 operands and activations, fp32 accumulate, tanh-form
                                     GELU (north_star gate 2e-2 on o);
                                     RC_TF32: tf32-rounded fp32 operands and activations, fp32
                                     accumulate, exact-erf GELU (gate 1e-3 on o);
                                     RC_TF32X3: fp32-accurate GEMMs as three tf32 MMAs per product
                                     (a_hi b_hi + a_lo b_hi + a_hi b_lo), activations kept as tf32
                                     hi/lo pairs, exact-erf GELU (gate 1e-3 on o and wdot) */
  int32_t flags;                  /* bitwise OR of
                                     RC_MLP_LAYERWISE: run layers 1 and 2 as separate kernels (h1
                                     through the workspace) even where the fused layer-1/2 kernel
                                     applies -- the comparison path; results agree to rounding;
                                     RC_MLP_SHARED: ONE shared net with n_nets outputs instead of one
                                     net per species (reading R20:
                                     the Table-1-consistent reading of PAPER.md:114/210); params is
                                     then one block W1 b1 W2 b2 W3 b3 W4[n_nets][h3] b4[n_nets] and
                                     output i predicts species_of_net[i].  RC_BF16 or RC_TF32 only;
                                     RC_MLP_SERIAL: run every MLP kernel on the caller's stream, in
                                     chunk order.  By default, where the fused layer-1/2 kernel runs,
                                     layer 3 of a chunk runs partly
                                     beside the fused kernel of the next chunk on the SMs that
                                     kernel's 4-CTA clusters leave idle, on a library-owned
                                     auxiliary stream (one per host thread and device) forked from
                                     and joined back into the caller's stream by events inside the
                                     call (so stream capture works); DESIGN.md 6.4.  Results are
                                     bitwise identical either way. */
} rc_mlp_desc;

int rc_mlp_create(const rc_mech *m, const rc_mlp_desc *desc, rc_mlp **out);
void rc_mlp_destroy(rc_mlp *n);

/* ---------------------------------------------------------------------------
 * Cell state: caller-owned DEVICE arrays, component-major (field[k*ld + c]).
 * Every array pointer 16-byte aligned (red / diag: 8-byte); ld >= n and ld even.  Output pointers may be
 * NULL to skip that output (the stage still runs if any of its outputs is
 * requested).  Inputs are never written except T (h-mode: in = guess, out =
 * converged) and h (T-mode: out).
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t n, ld;
  int32_t mode;                   /* RC_MODE_H: Newton from h (T in = guess); RC_MODE_T: h = h(T) */
  double *h;                      /* [ld]  J/kg */
  double *T;                      /* [ld]  K */
  const double *p;                /* [ld]  Pa */
  const double *Y;                /* [ns][ld] mass fractions (may hold tiny negatives) */
  double *cp, *rho;               /* [ld] (a1) */
  double *mu, *lambda;            /* [ld] Wilke viscosity, Mathur conductivity (a2) */
  double *D;                      /* [ns][ld] mixture-averaged diffusivities (a2) */
  double *wdot;                   /* [ns][ld] species source terms rho dY_k / dt (a5) */
  double *qdot;                   /* [ld] heat release -sum_k h_k(T) wdot_k (a5) */
  float *o;                       /* [n_nets][ld] raw net outputs (optional, parity/debug) */
  double dt;                      /* must equal the bundle's dt when chemistry runs */
  double *red;                    /* [2] device: red[0] = max over cells of T (atomic max,
                                     caller/rc_step zeroes), red[1] = sum qdot (written by chem) */
  int64_t *diag;                  /* [RC_DIAG_COUNT] device counters (atomic adds), may be NULL */
  const double *tau_mix;          /* [ld] s, optional (NULL = laminar / quasi-DNS).  LES partially-stirred
                                     reactor ("the partially-stirred reactor (PaSR) model
                                     ... to account for the SGS turbulence-chemistry interaction"; its
                                     equations are not in the paper -- DESIGN.md reading R19): the
                                     subgrid mixing time of each cell (from the caller's SGS model).
                                     rc_chem then scales wdot and qdot of the cell by
                                     kappa = tau_c / (tau_c + tau_mix), with the chemical time
                                     tau_c = sum_k C+_k / (1/2 sum_k |wdot_k| / W_k),
                                     C+_k = rho max(Y_k, 0) / W_k, from the cell's unscaled wdot
                                     (kappa = 1 where wdot = 0).  tau_mix >= 0. */
} rc_cells;

/* Workspace bytes rc_chem / rc_step use for n cells: the layer-1 input rows and the raw net outputs
 * of all n cells (32 + 4 n_nets B per cell in bf16) plus the activations of one cell chunk and
 * partial sums.  A smaller workspace (down to the 256-cell-chunk minimum) runs with smaller chunks.
 * Alignment 256 B. */
size_t rc_workspace_bytes(const rc_mech *m, const rc_mlp *n, int64_t ncells);

/* a1: Newton h -> T (h-mode) or h(T) (T-mode); cp, rho.
 * Newton: T <- clamp(T + (h* - h(T))/cp(T), min T_lo, max T_hi), stop after an
 * unclamped update with |dT| <= 1e-10 T; 50 iterations or two consecutive
 * clamps -> bisection to width 1e-10 T (R8). */
int rc_thermo(const rc_mech *m, const rc_cells *c, void *stream);

/* a2: Wilke viscosity, Mathur conductivity, mixture-averaged D_k with
 * X+ = max(X, 0) and the D_kk pure-species fallback (R10, R11).  Reads T as
 * stored (run after rc_thermo). */
int rc_transport(const rc_mech *m, const rc_cells *c, void *stream);

/* a3-a5: Box-Cox prologue, per-species MLP on the tensor cores, inverse
 * Box-Cox, element projection, wdot, qdot; red[1] = sum qdot.  Reads T and rho
 * as stored (run after rc_thermo).  Errors: RC_EDTMISMATCH, RC_EINVAL
 * (workspace too small / NULL wdot), RC_ECUDA. */
int rc_chem(const rc_mech *m, const rc_mlp *n, const rc_cells *c, void *ws, size_t ws_bytes, void *stream);

/* a1 + a2 + a3-a5 in order on one stream; zeroes red and diag first. */
int rc_step(const rc_mech *m, const rc_mlp *n, const rc_cells *c, void *ws, size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * Downstream consumer (reading R22): implicit Laplacian assembly of
 * PAPER.md Algorithm 1 (lines 137-158) for the ns species equations and the energy equation with the
 * coefficients this path produces -- gamma = rho D_k (system k < ns), lambda / cp (system ns) -- on a
 * periodic Cartesian mesh of uniform spacing, or on a z-slab of one (multi-GPU block).
 * Cells c = i + nx (j + ny k); face f = d n + c (d = x, y, z) joins cell c and its +d
 * neighbour (periodic wrap in x, y; in z the wrap or, with halos, the plane above the slab).
 *   gamma_f = (gamma_P + gamma_N) / 2 (linear interpolation, uniform mesh: w = 1/2)
 *   upper[f] = lower[f] = gamma_f |S_f| / |d_f|;  diag[P] -= upper[f], diag[N] -= lower[f]
 * ldu storage: the matrix is symmetric, so lower = upper is not stored.
 * ------------------------------------------------------------------------- */
typedef struct {
  int32_t nx, ny, nz;             /* cells per direction (nz: planes of this block) */
  double dx, dy, dz;              /* uniform spacing, m */
} rc_mesh;
enum { RC_LAP_GATHER = 0, RC_LAP_ATOMIC = 1 };  /* one thread per cell, diagonal gathered (deterministic) |
                                                   one thread per face, diagonal by atomicAdd (Algorithm 1) */
/* c: n = nx ny nz cells with rho, lambda, cp, D (device, as rc_step left them).  halo_lo / halo_hi:
 * both NULL (periodic in z) or device [(ns + 3)][nx ny] planes (rho, lambda, cp, D_0..D_{ns-1}) of the
 * cells below plane 0 / above plane nz-1 (rc_pack_planes of the neighbouring ranks).  Out (device,
 * 8-byte aligned): upper [ns+1][3 n], diag [ns+1][n].  Errors: RC_EINVAL, RC_EALIGN, RC_ECUDA. */
int rc_laplacian(const rc_mech *m, const rc_mesh *mesh, const rc_cells *c, const double *halo_lo,
                 const double *halo_hi, double *upper, double *diag, int mode, void *stream);
/* ldu -> CSR of nsys systems of a periodic block: row_ptr [n+1] (int64), col [7 n]
 * (int32, ascending per row), val [nsys][7 n].  Needs nx, ny, nz >= 3 (else RC_EUNSUPPORTED). */
int rc_ldu_to_csr(const rc_mesh *mesh, int nsys, const double *upper, const double *diag, int64_t *row_ptr,
                  int32_t *col, double *val, void *stream);
/* The bottom and top planes of this block's rho, lambda, cp, D -> bottom / top [(ns + 3)][nx ny]
 * (device; either may be NULL): what the neighbouring ranks receive as their halos. */
int rc_pack_planes(const rc_mech *m, const rc_mesh *mesh, const rc_cells *c, double *bottom, double *top,
                   void *stream);

/* ---------------------------------------------------------------------------
 * Detailed kinetics (reading R21): the right-hand side the paper's
 * CVODE option integrates ("CVODE ... on CPU or DNN on GPU"; the 9-species /
 * 12-reaction H2 mechanism of PAPER.md:231) -- an alternative source term to the DNN, per cell:
 *   C_k = rho Y_k / W_k with rho = p W / (R_u T);  k = A T^b exp(-Ea / (R_u T))
 *   three-body: q *= [M], [M] = sum_k eff_k C_k;  falloff: k = k_inf Pr / (1 + Pr) F,
 *   Pr = k0 [M] / k_inf, F = 1 (Lindemann, troe[0] < 0) or Troe with
 *   Fcent = (1 - a) exp(-T/T3) + a exp(-T/T1) + exp(-T2/T), troe = {a, T3, T1, T2}
 *   K_c = exp(-sum_k nu_k g_k) (p0 / (R_u T))^(sum_k nu_k), g_k = h_k/(R_u T) - s_k/R_u (NASA-7 a1..a7),
 *   p0 = 101325 Pa, nu = nu_r - nu_f;  q = k (prod C^nu_f - prod C^nu_r / K_c) (reverse term only if
 *   reversible);  wdot_k = W_k sum_r nu_rk q_r;  qdot = -sum_k h_k(T) wdot_k.
 * HOST pointers, SI units (kmol, m^3, s, J/kmol), copied at create.  At most 3 reactant and 3 product
 * molecules per reaction (RC_EUNSUPPORTED otherwise).
 * ------------------------------------------------------------------------- */
typedef struct rc_kin rc_kin;
enum { RC_RX_ELEMENTARY = 0, RC_RX_THREE_BODY = 1, RC_RX_FALLOFF = 2 };
typedef struct {
  int32_t nr;                     /* reactions */
  const int32_t *nu_f, *nu_r;     /* [nr][ns] stoichiometric coefficients of reactants / products */
  const int32_t *type;            /* [nr] RC_RX_* */
  const int32_t *reversible;      /* [nr] 0 / 1 */
  const double *A, *b, *Ea;       /* [nr] (high-pressure limit for falloff) */
  const double *eff;              /* [nr][ns] third-body efficiencies (three-body and falloff) */
  const double *A0, *b0, *Ea0;    /* [nr] low-pressure limit (falloff) */
  const double *troe;             /* [nr][4] a, T3, T1, T2 (falloff); a < 0: Lindemann */
} rc_kin_desc;
int rc_kin_create(const rc_mech *m, const rc_kin_desc *desc, rc_kin **out);
void rc_kin_destroy(rc_kin *k);
/* wdot, qdot of every cell from T (as stored: run after rc_thermo), p, Y; PaSR-scaled if tau_mix;
 * red[1] = sum qdot (deterministic; one rc_kinetics in flight per handle), diag nonfinite counted.
 * Errors: RC_EINVAL (NULL wdot), RC_EALIGN, RC_ECUDA. */
int rc_kinetics(const rc_mech *m, const rc_kin *k, const rc_cells *c, void *stream);

/* Step a6 on one device for a step run as k sub-batches (e.g. to overlap the host
 * copies of one batch with the compute of another, each rc_step writing its own
 * red/diag): red = {max_i red_parts[i][0], sum_i red_parts[i][1]} (sum in index
 * order, Neumaier-compensated), diag[j] = sum_i diag_parts[i][j].  Device
 * pointers: red_parts [k][2] fp64, diag_parts [k][RC_DIAG_COUNT] int64 (NULL
 * with diag NULL skips the counters); asynchronous on `stream`.
 * Errors: RC_EINVAL (k < 1, NULL red/red_parts), RC_ECUDA. */
int rc_combine_reductions(const double *red_parts, const int64_t *diag_parts, int k, double *red, int64_t *diag,
                          void *stream);

/* Multi-GPU block partition: rank r of world G gets
 * [begin, end) with boundaries floor(r N / G) rounded down to 128 cells (the
 * MLP tile) except end = N for the last rank.  Pure host function. */
int rc_partition(int64_t n_global, int rank, int world, int64_t *begin, int64_t *end);

/* ---------------------------------------------------------------------------
 * Per-stage device timing (SURVEY.md §5 "CUDA events per stage").  When
 * enabled, every launch is bracketed by CUDA events on the caller's stream
 * (a few microseconds of overhead per launch).  rc_profile_read waits for the
 * recorded events, returns the summed milliseconds and launch counts per
 * stage since the last reset, and optionally resets.  Process-global.
 * ------------------------------------------------------------------------- */
enum {
  RC_STAGE_THERMO = 0, RC_STAGE_TRANSPORT = 1, RC_STAGE_PROLOGUE = 2, RC_STAGE_L1 = 3, RC_STAGE_L2 = 4,
  RC_STAGE_L3 = 5, RC_STAGE_EPILOGUE = 6, RC_STAGE_FINALIZE = 7,
  RC_STAGE_L12 = 8,  /* fused layers 1+2 (bf16 at the paper widths; replaces L1 and L2) */
  RC_STAGE_L4 = 9,   /* layer 4 of the shared net (RC_MLP_SHARED) */
  RC_STAGE_KINETICS = 10, /* detailed kinetics (rc_kinetics) */
  RC_STAGE_LAPLACIAN = 11, /* Laplacian assembly (rc_laplacian) */
  RC_STAGE_CSR = 12,      /* ldu -> CSR (rc_ldu_to_csr) */
  RC_STAGE_L3_FILL = 13,  /* layer-3 launches on the auxiliary stream, beside the fused kernel */
  RC_STAGE_COUNT = 14
};
int rc_profile_enable(int on);
int rc_profile_read(double *ms /* [RC_STAGE_COUNT] */, int64_t *launches /* [RC_STAGE_COUNT] */, int reset);
/* The recorded launches one by one, in record order (call before rc_profile_read resets them): stage[i]
 * and the start / end of launch i in ms relative to the first recorded start (CUDA events, so
 * launches on different streams share one time axis -- the layer-3 side launches next to the fused
 * kernel show as intersecting intervals).  Fills at most `max` entries; returns the number recorded
 * (>= 0) or an error status (RC_EINVAL: NULL arrays with max > 0; RC_ECUDA). */
int rc_profile_timeline(int32_t *stage, double *t_start_ms, double *t_end_ms, int max);
/* Layer-3 overlap counters since the last reset (process-global, current device; synchronous):
 * out[0] = layer-3 tiles (256 cells x one pass of one net) run by the launches beside the fused
 * kernel, out[1] = CTA pairs of those launches that found the fused kernel not yet resident after
 * 50 us and did nothing, out[2] = CTA pairs that ran.  Errors: RC_EINVAL (NULL out), RC_ECUDA. */
int rc_overlap_read(int64_t *out /* [3] */, int reset);

/* Number of kernel launches the last rc_* call on this thread enqueued. */
int64_t rc_last_launch_count(void);

const char *rc_last_error(void);
const char *rc_version(void);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* RC_H */
