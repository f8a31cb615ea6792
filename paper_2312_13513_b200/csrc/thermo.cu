// thermo.cu -- path step a1: enthalpy -> temperature Newton inversion on NASA-7
// polynomials, then cp and rho (§3.1 "Newton's method and
// high-order temperature polynomials"; R8, R9).
//
// HBM-bound design: component-major fp64 (h, T, p, Y_k) in,
// 96 B/cell for the H2 set, 24 B/cell out.  A persistent grid streams 128-cell
// tiles through a ring of shared-memory stages filled by one bulk-TMA copy per
// SoA row (stream.cuh), so 2-3 tiles per CTA are always in flight while one
// thread per cell runs the Newton iteration from shared memory.  The species
// table is staged once per CTA with one bulk copy.  To keep the per-iteration
// cost independent of ns the mass-fraction-weighted NASA coefficients of the
// mixture are formed once per range (12 ns DFMA), so each Newton iteration is
// two Horner polynomials and a reciprocal instead of a loop over species
// ("computation consolidation").
#include <type_traits>

#include "ptx.cuh"
#include "rc_internal.h"
#include "stream.cuh"

namespace {

// 16-byte shared load kept in program order (see the mixture-coefficient loop)
__device__ __forceinline__ double2 lds_f64x2(const double *p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(rcx::smem_u32(p)));
  return v;
}

__device__ __forceinline__ double lds_f64(const double *p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(rcx::smem_u32(p)));
  return v;
}

__device__ __forceinline__ void warp_count_add(int64_t *dst, int v) {
  unsigned s = __reduce_add_sync(0xffffffffu, (unsigned)v);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd((unsigned long long *)dst, (unsigned long long)s);
}

__device__ __forceinline__ void warp_max_T(double *dst, double T) {
  double v = (T > 0.0 && T < 1e300) ? T : 0.0;
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0 && v > 0.0)
    atomicMax((unsigned long long *)dst, (unsigned long long)__double_as_longlong(v));
}

// cells per stage = consumer threads per CTA (+ the producer warp, stream.cuh run_ws): 256 for the
// H2 set; 128 otherwise, where a 256-cell stage of 3 + Ns fp64 rows (47 KB at Ns = 20) leaves one
// CTA (8 consumer warps) per SM
template <int NS> constexpr int thermo_tile() { return NS == 9 ? 256 : 128; }

template <int NS, bool UNIFORM>
__global__ void __launch_bounds__(thermo_tile<NS>() + 32, 3) thermo_kernel(const double *__restrict__ tab, int ns_rt, CellsDev c, int stages) {
  constexpr int THERMO_TILE = thermo_tile<NS>();
  extern __shared__ __align__(16) double s_tab[];
  __shared__ __align__(8) uint64_t bars[1 + 16];
  const int ns = NS ? NS : ns_rt;
  const int tsz = ThermoSeg::size(ns);
  const bool hmode = c.mode == RC_MODE_H;
  // stage rows (fp64): T, p, Y_0..Y_{ns-1}, then h (h-mode only)
  const rcs::Ring<THERMO_TILE> ring{reinterpret_cast<uint8_t *>(s_tab + tsz), bars + 1, 2 + ns + (hmode ? 1 : 0), 0, stages};
  if (threadIdx.x == 0) {
    rcx::mbar_init(&bars[0], 1);
    ring.init(THERMO_TILE / 32);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    rcx::mbar_arrive_expect_tx(&bars[0], (uint32_t)tsz * 8u);
    rcx::bulk_g2s(s_tab, tab, (uint32_t)tsz * 8u, &bars[0]);
  }
  auto src8 = [&](int r) -> const double * {
    return r == 0 ? c.T : r == 1 ? c.p : r < 2 + ns ? c.Y + (size_t)(r - 2) * c.ld : c.h;
  };
  auto src4 = [&](int) -> const float * { return nullptr; };
  rcx::mbar_wait(&bars[0], 0);

  const double Tmin = s_tab[0], Tmax = s_tab[1], Tmid = s_tab[2];
  const double *hlo = s_tab + ThermoSeg::hlo(ns), *hhi = s_tab + ThermoSeg::hhi(ns);
  const double *invW = s_tab + ThermoSeg::invW(ns), *tmid = s_tab + ThermoSeg::tmid(ns);
  constexpr int CAP = NS ? NS : RC_MAX_NS;
  constexpr int UR = NS ? NS : 1;
  constexpr int UR1 = NS ? (NS > 10 ? 5 : NS) : 1;  // the mixture pass: a partial unroll for Ns = 20 (no spill)

  int n_bisect = 0, n_maxit = 0, n_neg = 0, n_bad = 0;
  double Tloc_max = 0.0;
  ring.run_ws(c.n, src8, src4, [&](int st, int64_t tile, int j) {
    const int64_t i = tile * THERMO_TILE + j;
    if (i >= c.n) return;
    const double *S8 = ring.row8(st, 0) + j;  // fp64 row q of this cell: S8[q * THERMO_TILE]
    // mixture NASA coefficients per range and 1/W = sum Y_k / W_k.  The table is read with
    // volatile shared loads next to their use: a fully unrolled loop would otherwise hoist the
    // whole coefficient table into registers.
    bool neg = false;
    const double p = S8[THERMO_TILE];
    double T = S8[0], hT, cpT;
    double rho;
    if constexpr (UNIFORM) {
      // One T_mid for every species: the mixture polynomial of ONE range, a[6] = sum_k Y_k a_k,
      // formed for the range T lies in and re-formed only when an iterate crosses T_mid (a cell
      // rarely does): 6 ns instead of 12 ns DFMA and no per-evaluation range selects.
      double sW = 0.0, a[6];
      bool lo_rng = false;
      auto mix = [&](bool lo, auto unroll) {
        const double *tb = lo ? hlo : hhi;
#pragma unroll
        for (int q = 0; q < 6; ++q) a[q] = 0.0;
        auto term = [&](int k) {
          const double yk = lds_f64(S8 + (2 + k) * THERMO_TILE);  // re-read: no Ns registers held
#pragma unroll
          for (int q = 0; q < 6; q += 2) {
            const double2 v = lds_f64x2(tb + 6 * k + q);
            a[q] = fma(yk, v.x, a[q]);
            a[q + 1] = fma(yk, v.y, a[q + 1]);
          }
          return yk;
        };
        if constexpr (decltype(unroll)::value) {  // first pass: also 1/W and the negative-Y count
#pragma unroll UR1
          for (int k = 0; k < CAP; ++k)
            if (k < ns) {
              const double yk = term(k);
              neg |= yk < 0.0;
              sW = fma(yk, invW[k], sW);
            }
        } else {  // an iterate crossed T_mid: rare, kept small
#pragma unroll 1
          for (int k = 0; k < ns; ++k) term(k);
        }
        lo_rng = lo;
      };
      auto eval = [&](double T, double &h, double &cp) {
        if ((T <= Tmid) != lo_rng) mix(T <= Tmid, std::false_type{});
        // Estrin form (dependency depth 3 instead of 5: the Newton iteration is a latency chain)
        const double T2 = T * T;
        h = fma(T2 * T2, fma(T, a[4], a[3]), fma(T2, fma(T, a[2], a[1]), fma(T, a[0], a[5])));
        cp = fma(T2 * T2, 5.0 * a[4], fma(T2, fma(T, 4.0 * a[3], 3.0 * a[2]), fma(T, 2.0 * a[1], a[0])));
      };
      if (hmode) {
        const double hs = S8[(2 + ns) * THERMO_TILE];
        T = fmin(fmax(T, Tmin), Tmax);
        mix(T <= Tmid, std::true_type{});
        int clamp_hits = 0;
        bool done = false, fresh = false;
#pragma unroll 1
        for (int it = 1; it <= 50; ++it) {
          eval(T, hT, cpT);
          double Tn = T + (hs - hT) * rcx::rcp_f64_fast(cpT);
          bool clamped = false;
          if (Tn < Tmin) { Tn = Tmin; clamped = true; }
          if (Tn > Tmax) { Tn = Tmax; clamped = true; }
          clamp_hits = clamped ? clamp_hits + 1 : 0;
          if (clamp_hits >= 2) break;
          if (!clamped && fabs(Tn - T) <= 1e-10 * Tn) {
            // cp(T) stands for cp(Tn) when the last step is below 1e-13 T (relative change of cp
            // <= (T cp'/cp) 1e-13 < 1e-13; DESIGN.md §6 thermo): the usual case, quadratic convergence
            fresh = fabs(Tn - T) <= 1e-13 * Tn && (Tn <= Tmid) == (T <= Tmid);
            T = Tn;
            done = true;
            break;
          }
          T = Tn;
          if (it == 50) ++n_maxit;
        }
        if (!done) {  // bisection on [Tmin, Tmax]; h increasing since cp > 0
          ++n_bisect;
          double lo = Tmin, hi = Tmax;
#pragma unroll 1
          while (hi - lo > 1e-10 * (0.5 * (lo + hi))) {
            double mid = 0.5 * (lo + hi), hm, cm;
            eval(mid, hm, cm);
            if (hm < hs) lo = mid; else hi = mid;
          }
          T = 0.5 * (lo + hi);
        }
        c.T[i] = T;
        if (!fresh) eval(T, hT, cpT);
      } else {
        mix(T <= Tmid, std::true_type{});
        eval(T, hT, cpT);
        if (c.h) c.h[i] = hT;
      }
      rho = p * rcx::rcp_f64_fast(RC_RU * T * sW);
    } else {  // per-species ranges (T_mid differs between species)
      double Y[CAP];
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k < ns) {
          Y[k] = S8[(2 + k) * THERMO_TILE];
          neg |= Y[k] < 0.0;
        }
      double sW = 0.0;
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k < ns) sW = fma(Y[k], invW[k], sW);
      auto eval = [&](double T, double &h, double &cp) {
        h = 0.0;
        cp = 0.0;
#pragma unroll UR
        for (int k = 0; k < CAP; ++k)
          if (k < ns) {
            const double *a = (T <= tmid[k]) ? hlo + 6 * k : hhi + 6 * k;
            double hk = fma(T, fma(T, fma(T, fma(T, fma(T, a[4], a[3]), a[2]), a[1]), a[0]), a[5]);
            double ck = fma(T, fma(T, fma(T, fma(T, 5.0 * a[4], 4.0 * a[3]), 3.0 * a[2]), 2.0 * a[1]), a[0]);
            h = fma(Y[k], hk, h);
            cp = fma(Y[k], ck, cp);
          }
      };
      if (hmode) {
        const double hs = S8[(2 + ns) * THERMO_TILE];
        T = fmin(fmax(T, Tmin), Tmax);
        int clamp_hits = 0;
        bool done = false;
#pragma unroll 1
        for (int it = 1; it <= 50; ++it) {
          eval(T, hT, cpT);
          double Tn = T + (hs - hT) * rcx::rcp_f64_fast(cpT);
          bool clamped = false;
          if (Tn < Tmin) { Tn = Tmin; clamped = true; }
          if (Tn > Tmax) { Tn = Tmax; clamped = true; }
          clamp_hits = clamped ? clamp_hits + 1 : 0;
          if (clamp_hits >= 2) break;
          if (!clamped && fabs(Tn - T) <= 1e-10 * Tn) { T = Tn; done = true; break; }
          T = Tn;
          if (it == 50) ++n_maxit;
        }
        if (!done) {
          ++n_bisect;
          double lo = Tmin, hi = Tmax;
#pragma unroll 1
          while (hi - lo > 1e-10 * (0.5 * (lo + hi))) {
            double mid = 0.5 * (lo + hi), hm, cm;
            eval(mid, hm, cm);
            if (hm < hs) lo = mid; else hi = mid;
          }
          T = 0.5 * (lo + hi);
        }
        c.T[i] = T;
      }
      eval(T, hT, cpT);
      if (!hmode && c.h) c.h[i] = hT;
      rho = p / (RC_RU * T * sW);
    }
    if (c.cp) c.cp[i] = cpT;
    if (c.rho) c.rho[i] = rho;
    n_neg += neg;
    n_bad += !(isfinite(T) && isfinite(cpT) && isfinite(rho));
    Tloc_max = fmax(Tloc_max, (T > 0.0 && T < 1e300) ? T : 0.0);
  });
  if (c.diag) {
    warp_count_add(c.diag + RC_DIAG_NEWTON_BISECT, n_bisect);
    warp_count_add(c.diag + RC_DIAG_NEWTON_MAXIT, n_maxit);
    warp_count_add(c.diag + RC_DIAG_NEGY_IN, n_neg);
    warp_count_add(c.diag + RC_DIAG_NONFINITE, n_bad);
  }
  if (c.red) warp_max_T(c.red, Tloc_max);
}

template <int NS, bool U>
int launch_thermo_t(const rc_mech *m, const CellsDev &c, cudaStream_t s) {
  const int rows = 2 + m->ns + (c.mode == RC_MODE_H ? 1 : 0);
  // 3 stages: two tiles in flight per CTA behind the one being computed
  const int stages = 3;
  constexpr int THERMO_TILE = thermo_tile<NS>(), THERMO_THREADS = THERMO_TILE + 32;
  const size_t smem = (size_t)ThermoSeg::size(m->ns) * 8 + rcs::Ring<THERMO_TILE>::smem_bytes(rows, 0, stages);
  const int64_t ntiles = (c.n + THERMO_TILE - 1) / THERMO_TILE;
  int64_t grid = rc_resident_blocks((const void *)thermo_kernel<NS, U>, THERMO_THREADS, smem);
  if (grid > ntiles) grid = ntiles;
  thermo_kernel<NS, U><<<(unsigned)grid, THERMO_THREADS, smem, s>>>(m->d_thermo, m->ns, c, stages);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

}  // namespace

int launch_thermo(const rc_mech *m, const CellsDev &c, cudaStream_t s) {
  if (c.n == 0) return RC_OK;
  const bool u = m->uniform_tmid;
  ProfScope prof(RC_STAGE_THERMO, s);
  if (m->ns == 9 && u) return launch_thermo_t<9, true>(m, c, s);
  if (m->ns == 20 && u) return launch_thermo_t<20, true>(m, c, s);
  if (u) return launch_thermo_t<0, true>(m, c, s);
  return launch_thermo_t<0, false>(m, c, s);
}
