// kinetics.cu -- detailed-kinetics source term (reading R21): the
// right-hand side of the paper's CVODE option ("CVODE ... on CPU or DNN on GPU") for the
// 9-species / 12-reaction H2 mechanism of its quasi-DNS runs, as an alternative to the
// DNN chemistry on the same cells.  Mass-action law with Arrhenius rates, three-body and
// Lindemann/Troe falloff forms, reverse rates from the equilibrium constant of the mechanism's NASA-7
// tables (include/rc.h rc_kinetics states the formulas).
//
// FP64-bound (two exp per reaction, a handful more per falloff reaction).  Cells stream through the
// TMA tile ring of stream.cuh (rows T, p, Y_k); per cell one thread.  The reaction loop is driven by
// a table in shared memory, so species are indexed at run time: each thread keeps its cell's
// concentrations C_k, Gibbs functions g_k and the accumulating molar rates in its own column of a
// per-CTA shared-memory scratch ([ns][TILE], conflict-free), and reads the reaction records as
// broadcasts.
#include <cmath>
#include <cstring>

#include "ptx.cuh"
#include "rc_internal.h"
#include "stream.cuh"

namespace {

// KinSeg: the device table (doubles)
//   [0] nr  [1] ns
//   G   [ns][2][8] per species and NASA range: g = c0 + c1 ln T + T (c2 + T (c3 + T (c4 + T c5))) + c6 / T
//   TM  [nse]      T_mid per species (T <= T_mid: low range)
//   W   [nse], IW [nse]
//   REC [nr][48]   per reaction (see kin_build)
//   EFF [nr][nse]  third-body efficiencies
struct KinSeg {
  static int nse(int ns) { return (ns + 1) & ~1; }
  __host__ __device__ static int G(int) { return 4; }
  __host__ __device__ static int TM(int ns) { return 4 + 16 * ns; }
  __host__ __device__ static int W(int ns) { return TM(ns) + ((ns + 1) & ~1); }
  __host__ __device__ static int IW(int ns) { return W(ns) + ((ns + 1) & ~1); }
  __host__ __device__ static int REC(int ns) { return IW(ns) + ((ns + 1) & ~1); }
  __host__ __device__ static int EFF(int ns, int nr) { return REC(ns) + 48 * nr; }
  // IREC [nr][24] int32 (12 doubles per reaction): type, reversible, sum nu, then the species of the
  // reactant / product slots and of the nonzero-nu pairs as scratch-column offsets k * KIN_TILE
  // (-1: empty), then the pair nu
  __host__ __device__ static int IREC(int ns, int nr) { return (EFF(ns, nr) + nr * ((ns + 1) & ~1) + 1) & ~1; }
  __host__ __device__ static int size(int ns, int nr) { return IREC(ns, nr) + 12 * nr; }
};
enum { I_TYPE = 0, I_REV = 1, I_DNU = 2, I_REAC = 3, I_PROD = 6, I_PSP = 9, I_PNU = 15, I_N = 24 };
enum {
  R_LNA = 0, R_B = 1, R_ER = 2, R_TYPE = 3, R_REV = 4, R_DNU = 5, R_REAC = 6, R_PROD = 9, R_PSP = 12, R_PNU = 18,
  R_LNA0 = 24, R_B0 = 25, R_ER0 = 26, R_TA = 27, R_IT3 = 28, R_IT1 = 29, R_T2 = 30
};

constexpr int KIN_TILE = 128;
constexpr int KIN_THREADS = KIN_TILE + 32;  // + the producer warp (stream.cuh run_ws)
constexpr int KIN_QPART = 1024;
constexpr double KIN_P0 = 101325.0;

template <int NS>
__global__ void __launch_bounds__(KIN_THREADS) kinetics_kernel(const double *__restrict__ tab, int ns_rt, int nr,
                                                               const double *__restrict__ thermo, CellsDev c,
                                                               double *qpart, int stages) {
  constexpr int CAP = NS ? NS : RC_MAX_NS;
  constexpr int UR = NS ? NS : 1;
  const int ns = NS ? NS : ns_rt;
  extern __shared__ __align__(16) double ks[];
  __shared__ __align__(8) uint64_t bars[1 + 16];
  __shared__ double red_s[KIN_THREADS / 32];
  const int ksz = KinSeg::size(ns, nr), tsz = ThermoSeg::size(ns);
  double *sT = ks + ksz;                       // thermo segment (mass-based h_k for qdot)
  double *scr = sT + tsz;                      // scratch: C [ns][TILE], g [ns][TILE], rate [ns][TILE]
  double *sC = scr, *sG = scr + ns * KIN_TILE, *sR = scr + 2 * ns * KIN_TILE;
  const rcs::Ring<KIN_TILE> ring{reinterpret_cast<uint8_t *>(scr + 3 * ns * KIN_TILE), bars + 1, 2 + ns, 0, stages};
  if (threadIdx.x == 0) {
    rcx::mbar_init(&bars[0], 1);
    ring.init(KIN_TILE / 32);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    rcx::mbar_arrive_expect_tx(&bars[0], (uint32_t)(ksz + tsz) * 8u);
    rcx::bulk_g2s(ks, tab, (uint32_t)ksz * 8u, &bars[0]);
    rcx::bulk_g2s(sT, thermo, (uint32_t)tsz * 8u, &bars[0]);
  }
  auto src8 = [&](int r) -> const double * { return r == 0 ? c.T : r == 1 ? c.p : c.Y + (size_t)(r - 2) * c.ld; };
  auto src4 = [&](int) -> const float * { return nullptr; };
  rcx::mbar_wait(&bars[0], 0);
  const double *G = ks + KinSeg::G(ns), *TM = ks + KinSeg::TM(ns), *W = ks + KinSeg::W(ns);
  const double *IW = ks + KinSeg::IW(ns), *REC = ks + KinSeg::REC(ns), *EFF = ks + KinSeg::EFF(ns, nr);
  const int *IREC = reinterpret_cast<const int *>(ks + KinSeg::IREC(ns, nr));
  const int nse = (ns + 1) & ~1;
  const double *hlo = sT + ThermoSeg::hlo(ns), *hhi = sT + ThermoSeg::hhi(ns);

  double qsum = 0.0;
  int n_bad = 0;
  // the stage is read once, into the per-thread scratch columns, and released before the reaction
  // loop (stream.cuh run_ws_release): the ring needs only one or two stages, so four CTAs fit per SM
  ring.run_ws_release(c.n, src8, src4, [&](int st, int64_t tile, int j, auto &&release) {
    const int64_t i = tile * KIN_TILE + j;
    const bool valid = i < c.n;  // lanes past the end stay until the release
    const double *S8 = ring.row8(st, 0) + j;
    const double T = valid ? S8[0] : 1000.0, p = valid ? S8[KIN_TILE] : KIN_P0;
    const double lnT = log(T), invT = 1.0 / T;
    double sW = 0.0, conc = 0.0;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        const double y = valid ? S8[(2 + k) * KIN_TILE] : 0.0;
        sW = fma(y, IW[k], sW);
        conc = fma(y > 0.0 ? y : 0.0, IW[k], conc);  // PaSR: sum_k C+_k / rho
      }
    const double rho = p / (RC_RU * T * sW);
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        sC[k * KIN_TILE + j] = rho * (valid ? S8[(2 + k) * KIN_TILE] : 0.0) * IW[k];
        const double *a = G + 16 * k + (T <= TM[k] ? 0 : 8);
        sG[k * KIN_TILE + j] = fma(a[1], lnT, a[0]) + T * fma(T, fma(T, fma(T, a[5], a[4]), a[3]), a[2]) + a[6] * invT;
        sR[k * KIN_TILE + j] = 0.0;
      }
    release();
    if (!valid) return;
    const double lnp0RT = log(KIN_P0 / RC_RU) - lnT;
    // Reactions in blocks of KB: the Arrhenius and equilibrium exponents of the block first, then
    // their 2 KB exponentials as independent straight-line code (the exp chains overlap; one reaction
    // at a time left the FP64 pipe waiting on each chain), then the per-reaction rest (third body,
    // falloff, concentration products) and the rate updates.  k_r = k_f / K_c is formed as
    // exp(ln k_f + sum nu g - dnu ln(p0/RT)) (one exponential instead of exp(ln k_f) exp(...)).
    // per-thread scratch columns: sC / sG / sR + q * KIN_TILE + j (q = species offset from IREC)
    const double *cC = sC + j, *cG = sG + j;
    double *cR = sR + j;
    constexpr int KB = 4;
#pragma unroll 1
    for (int r0 = 0; r0 < nr; r0 += KB) {
      double ef[KB], er[KB];
#pragma unroll
      for (int q = 0; q < KB; ++q) {  // exponents (a reaction past nr: both exponentials 0)
        const int r = r0 + q < nr ? r0 + q : nr - 1;
        const double *R = REC + 48 * r;
        const int *I = IREC + I_N * r;
        const double lnk = R[R_LNA] + R[R_B] * lnT - R[R_ER] * invT;
        double sg = 0.0;
#pragma unroll
        for (int u = 0; u < 6; ++u) {
          const int o = I[I_PSP + u];
          if (o >= 0) sg = fma((double)I[I_PNU + u], cG[o], sg);
        }
        const bool live = r0 + q < nr;
        ef[q] = live ? lnk : -INFINITY;
        er[q] = live && I[I_REV] ? lnk + (sg - (double)I[I_DNU] * lnp0RT) : -INFINITY;
      }
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        ef[q] = exp(ef[q]);
        er[q] = exp(er[q]);
      }
#pragma unroll
      for (int q = 0; q < KB; ++q) {
        const int r = r0 + q;
        if (r >= nr) break;
        const double *R = REC + 48 * r;
        const int *I = IREC + I_N * r;
        const int type = I[I_TYPE];
        double fwd = ef[q], rev = er[q], M = 0.0;
        if (type >= 1)
          for (int k = 0; k < ns; ++k) M = fma(EFF[r * nse + k], cC[k * KIN_TILE], M);
        if (type == 2) {  // falloff: k = k_inf Pr / (1 + Pr) F (the same factor on k_r = k_f / K_c)
          const double lnk = R[R_LNA] + R[R_B] * lnT - R[R_ER] * invT;
          const double Pr = exp(R[R_LNA0] + R[R_B0] * lnT - R[R_ER0] * invT - lnk) * M;
          double F = 1.0;
          if (R[R_TA] >= 0.0) {  // Troe
            const double a = R[R_TA];
            const double Fc = (1.0 - a) * exp(-T * R[R_IT3]) + a * exp(-T * R[R_IT1]) + exp(-R[R_T2] * invT);
            const double lF = log10(Fc), cc = -0.4 - 0.67 * lF, nn = 0.75 - 1.27 * lF;
            const double lp = log10(Pr) + cc, x = lp / (nn - 0.14 * lp);
            F = exp10(lF / (1.0 + x * x));
          }
          const double fac = Pr / (1.0 + Pr) * F;
          fwd *= fac;
          rev *= fac;
        }
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int o = I[I_REAC + u];
          if (o >= 0) fwd *= cC[o];
        }
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int o = I[I_PROD + u];
          if (o >= 0) rev *= cC[o];
        }
        if (type == 1) {
          fwd *= M;
          rev *= M;
        }
        const double qn = fwd - rev;
#pragma unroll
        for (int u = 0; u < 6; ++u) {
          const int o = I[I_PSP + u];
          if (o >= 0) cR[o] = fma((double)I[I_PNU + u], qn, cR[o]);
        }
      }
    }
    // wdot_k = W_k sum_r nu_rk q_r; LES: PaSR factor (rc.h tau_mix, R19); qdot
    double scale = 1.0;
    if (c.tau_mix) {
      double act = 0.0;
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k < ns) act += fabs(W[k] * sR[k * KIN_TILE + j]) * IW[k];
      const double r = act > 0.0 ? 0.5 * act / (rho * conc) : 0.0;
      scale = 1.0 / fma(c.tau_mix[i], r, 1.0);
    }
    double qd = 0.0;
    bool bad = false;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        const double w = scale * (W[k] * sR[k * KIN_TILE + j]);
        c.wdot[k * c.ld + i] = w;
        const double *h = (T <= TM[k]) ? hlo + 6 * k : hhi + 6 * k;
        const double hk = fma(T, fma(T, fma(T, fma(T, fma(T, h[4], h[3]), h[2]), h[1]), h[0]), h[5]);
        qd = fma(-hk, w, qd);
        bad |= !isfinite(w);
      }
    if (c.qdot) c.qdot[i] = qd;
    bad |= !isfinite(qd);
    qsum += qd;
    n_bad += bad;
  });
  if (c.diag) {
    const unsigned v = __reduce_add_sync(0xffffffffu, (unsigned)n_bad);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd((unsigned long long *)(c.diag + RC_DIAG_NONFINITE), v);
  }
  for (int o = 16; o; o >>= 1) qsum += __shfl_xor_sync(0xffffffffu, qsum, o);
  if ((threadIdx.x & 31) == 0) red_s[threadIdx.x >> 5] = qsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < KIN_THREADS / 32; ++w) t += red_s[w];
    qpart[blockIdx.x] = t;
  }
}

template <int NS>
int launch_kinetics_t(const rc_mech *m, const rc_kin *k, const CellsDev &c, cudaStream_t s) {
  const int ns = m->ns, stages = 1;
  const size_t smem = (size_t)(KinSeg::size(ns, k->nr) + ThermoSeg::size(ns) + 3 * ns * KIN_TILE) * 8 +
                      rcs::Ring<KIN_TILE>::smem_bytes(2 + ns, 0, stages);
  const int64_t ntiles = (c.n + KIN_TILE - 1) / KIN_TILE;
  int64_t grid = rc_resident_blocks((const void *)kinetics_kernel<NS>, KIN_THREADS, smem);
  if (grid > ntiles) grid = ntiles;
  if (grid > KIN_QPART) grid = KIN_QPART;
  RC_CUDA_TRY(cudaMemsetAsync(k->d_qpart, 0, KIN_QPART * sizeof(double), s));
  {
    ProfScope prof(RC_STAGE_KINETICS, s);
    kinetics_kernel<NS><<<(unsigned)grid, KIN_THREADS, smem, s>>>(k->d_tab, ns, k->nr, m->d_thermo, c, k->d_qpart, stages);
    RC_LAUNCH_CHECK();
  }
  if (c.red) return launch_qdot_finalize(k->d_qpart, KIN_QPART, c.red, s);
  return RC_OK;
}

}  // namespace

int launch_kinetics(const rc_mech *m, const rc_kin *k, const CellsDev &c, cudaStream_t s) {
  if (c.n == 0) return RC_OK;
  if (m->ns == 9) return launch_kinetics_t<9>(m, k, c, s);
  if (m->ns == 20) return launch_kinetics_t<20>(m, k, c, s);
  return launch_kinetics_t<0>(m, k, c, s);
}

// Host: the device table from the mechanism (NASA-7 a1..a7 -> Gibbs-function coefficients, molar
// masses) and the reaction description (SI).  g = h/(R T) - s/R = a1 (1 - ln T) - a2 T/2 - a3 T^2/6
// - a4 T^3/12 - a5 T^4/20 + a6/T - a7.
int kin_build(const rc_mech *m, const rc_kin_desc *d, rc_kin *k) {
  const int ns = m->ns, nr = d->nr, nse = (ns + 1) & ~1;
  std::vector<double> t(KinSeg::size(ns, nr), 0.0);
  t[0] = nr;
  t[1] = ns;
  for (int sp = 0; sp < ns; ++sp) {
    for (int rg = 0; rg < 2; ++rg) {
      const double *a = (rg ? m->nasa_hi.data() : m->nasa_lo.data()) + 7 * sp;
      double *g = &t[KinSeg::G(ns) + 16 * sp + 8 * rg];
      g[0] = a[0] - a[6];
      g[1] = -a[0];
      g[2] = -a[1] / 2.0;
      g[3] = -a[2] / 6.0;
      g[4] = -a[3] / 12.0;
      g[5] = -a[4] / 20.0;
      g[6] = a[5];
    }
    t[KinSeg::TM(ns) + sp] = m->T_mid[sp];
    t[KinSeg::W(ns) + sp] = m->W[sp];
    t[KinSeg::IW(ns) + sp] = 1.0 / m->W[sp];
  }
  for (int r = 0; r < nr; ++r) {
    double *R = &t[KinSeg::REC(ns) + 48 * r];
    const int32_t *nf = d->nu_f + (size_t)r * ns, *nb = d->nu_r + (size_t)r * ns;
    const int type = d->type[r];
    if (type < RC_RX_ELEMENTARY || type > RC_RX_FALLOFF) return rc_fail(RC_EINVAL, "reaction %d: unknown type %d", r, type);
    if (!(d->A[r] >= 0.0)) return rc_fail(RC_EINVAL, "reaction %d: A < 0", r);
    R[R_LNA] = d->A[r] > 0.0 ? std::log(d->A[r]) : -INFINITY;
    R[R_B] = d->b[r];
    R[R_ER] = d->Ea[r] / RC_RU;
    R[R_TYPE] = type;
    R[R_REV] = d->reversible[r] ? 1.0 : 0.0;
    for (int q = 0; q < 3; ++q) R[R_REAC + q] = R[R_PROD + q] = -1.0;
    for (int q = 0; q < 6; ++q) { R[R_PSP + q] = -1.0; R[R_PNU + q] = 0.0; }
    int nre = 0, npr = 0, npair = 0, dnu = 0;
    for (int sp = 0; sp < ns; ++sp) {
      if (nf[sp] < 0 || nb[sp] < 0) return rc_fail(RC_EINVAL, "reaction %d: negative stoichiometry", r);
      for (int q = 0; q < nf[sp]; ++q) {
        if (nre == 3) return rc_fail(RC_EUNSUPPORTED, "reaction %d: more than 3 reactant molecules", r);
        R[R_REAC + nre++] = sp;
      }
      for (int q = 0; q < nb[sp]; ++q) {
        if (npr == 3) return rc_fail(RC_EUNSUPPORTED, "reaction %d: more than 3 product molecules", r);
        R[R_PROD + npr++] = sp;
      }
      const int nu = nb[sp] - nf[sp];
      if (nu) {
        R[R_PSP + npair] = sp;
        R[R_PNU + npair++] = nu;
      }
      dnu += nu;
    }
    if (nre == 0) return rc_fail(RC_EINVAL, "reaction %d has no reactants", r);
    R[R_DNU] = dnu;
    if (type == RC_RX_FALLOFF) {
      if (!(d->A0[r] > 0.0)) return rc_fail(RC_EINVAL, "reaction %d: falloff needs A0 > 0", r);
      const double *tr = d->troe + 4 * (size_t)r;
      R[R_LNA0] = std::log(d->A0[r]);
      R[R_B0] = d->b0[r];
      R[R_ER0] = d->Ea0[r] / RC_RU;
      R[R_TA] = tr[0];
      R[R_IT3] = tr[0] >= 0.0 ? 1.0 / tr[1] : 0.0;
      R[R_IT1] = tr[0] >= 0.0 ? 1.0 / tr[2] : 0.0;
      R[R_T2] = tr[3];
    }
    for (int sp = 0; sp < ns; ++sp) t[KinSeg::EFF(ns, nr) + r * nse + sp] = d->eff[(size_t)r * ns + sp];
    int32_t I[I_N] = {0};  // copied into the table's bytes below (the table is one device buffer)
    I[I_TYPE] = type;
    I[I_REV] = d->reversible[r] ? 1 : 0;
    I[I_DNU] = dnu;
    for (int q = 0; q < 3; ++q) {
      I[I_REAC + q] = R[R_REAC + q] >= 0 ? (int)R[R_REAC + q] * KIN_TILE : -1;
      I[I_PROD + q] = R[R_PROD + q] >= 0 ? (int)R[R_PROD + q] * KIN_TILE : -1;
    }
    for (int q = 0; q < 6; ++q) {
      I[I_PSP + q] = R[R_PSP + q] >= 0 ? (int)R[R_PSP + q] * KIN_TILE : -1;
      I[I_PNU + q] = (int)R[R_PNU + q];
    }
    std::memcpy(reinterpret_cast<char *>(t.data() + KinSeg::IREC(ns, nr)) + sizeof(I) * r, I, sizeof(I));
  }
  k->nr = nr;
  k->ns = ns;
  cudaGetDevice(&k->device);
  k->tab_doubles = t.size();
  if (cudaMalloc(&k->d_tab, t.size() * 8) != cudaSuccess || cudaMalloc(&k->d_qpart, KIN_QPART * 8) != cudaSuccess)
    return rc_fail(RC_ENOMEM, "rc_kin_create: cudaMalloc failed");
  if (cudaMemcpy(k->d_tab, t.data(), t.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
    return rc_fail(RC_ECUDA, "rc_kin_create: upload failed");
  return RC_OK;
}
