// thermo.cu -- path step a1: enthalpy -> temperature Newton inversion on NASA-7
// polynomials, then cp and rho (§3.1 "Newton's method and
// high-order temperature polynomials"; R8, R9).
//
// HBM-bound design: one thread per cell, component-major
// coalesced fp64 loads of (h, T, p, Y_k) -> 96 B/cell in, 24 B/cell out for the
// H2 set.  The species table is staged once per CTA into shared memory with a
// single bulk-TMA copy.  To keep the per-iteration cost independent of ns the
// mass-fraction-weighted NASA coefficients of the mixture are formed once per
// range (12 ns DFMA), so each Newton iteration is two Horner polynomials and a
// division instead of a loop over species ("computation consolidation",
// PAPER.md:180).
#include "ptx.cuh"
#include "rc_internal.h"

namespace {

// 16-byte shared load kept in program order (see the mixture-coefficient loop)
__device__ __forceinline__ double2 lds_f64x2(const double *p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(rcx::smem_u32(p)));
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

template <int NS, bool UNIFORM>
__global__ void __launch_bounds__(256, 4) thermo_kernel(const double *__restrict__ tab, int ns_rt, CellsDev c) {
  extern __shared__ __align__(16) double s_tab[];
  __shared__ __align__(8) uint64_t bar;
  const int ns = NS ? NS : ns_rt;
  const uint32_t bytes = (uint32_t)ThermoSeg::size(ns) * 8u;
  if (threadIdx.x == 0) {
    rcx::mbar_init(&bar, 1);
    rcx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    rcx::mbar_arrive_expect_tx(&bar, bytes);
    rcx::bulk_g2s(s_tab, tab, bytes, &bar);
  }
  rcx::mbar_wait(&bar, 0);

  const double Tmin = s_tab[0], Tmax = s_tab[1], Tmid = s_tab[2];
  const double *hlo = s_tab + ThermoSeg::hlo(ns), *hhi = s_tab + ThermoSeg::hhi(ns);
  const double *invW = s_tab + ThermoSeg::invW(ns), *tmid = s_tab + ThermoSeg::tmid(ns);
  constexpr int CAP = NS ? NS : RC_MAX_NS;
  constexpr int UR = NS ? NS : 1;

  int n_bisect = 0, n_maxit = 0, n_neg = 0, n_bad = 0;
  double Tloc_max = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (int64_t)gridDim.x * blockDim.x) {
    // mixture NASA coefficients per range and 1/W = sum Y_k / W_k.  All Y loads are issued
    // up front; the table is read with volatile shared loads next to their use, because a
    // fully unrolled loop would otherwise hoist the whole coefficient table into registers.
    double Y[CAP];
    bool neg = false;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        Y[k] = c.Y[k * c.ld + i];
        neg |= Y[k] < 0.0;
      }
    double Hl[6] = {0, 0, 0, 0, 0, 0}, Hh[6] = {0, 0, 0, 0, 0, 0}, sW = 0.0;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
#pragma unroll
        for (int j = 0; j < 6; j += 2) {
          const double2 lo = lds_f64x2(hlo + 6 * k + j), hi = lds_f64x2(hhi + 6 * k + j);
          Hl[j] = fma(Y[k], lo.x, Hl[j]);
          Hl[j + 1] = fma(Y[k], lo.y, Hl[j + 1]);
          Hh[j] = fma(Y[k], hi.x, Hh[j]);
          Hh[j + 1] = fma(Y[k], hi.y, Hh[j + 1]);
        }
        sW = fma(Y[k], invW[k], sW);
      }
    const double p = c.p[i];
    auto eval = [&](double T, double &h, double &cp) {
      if constexpr (UNIFORM) {
        const bool lo = T <= Tmid;
        double a0 = lo ? Hl[0] : Hh[0], a1 = lo ? Hl[1] : Hh[1], a2 = lo ? Hl[2] : Hh[2];
        double a3 = lo ? Hl[3] : Hh[3], a4 = lo ? Hl[4] : Hh[4], a5 = lo ? Hl[5] : Hh[5];
        h = fma(T, fma(T, fma(T, fma(T, fma(T, a4, a3), a2), a1), a0), a5);
        cp = fma(T, fma(T, fma(T, fma(T, 5.0 * a4, 4.0 * a3), 3.0 * a2), 2.0 * a1), a0);
      } else {  // per-species ranges (T_mid differs between species)
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
      }
    };
    double T = c.T[i], hT, cpT;
    if (c.mode == RC_MODE_H) {
      const double hs = c.h[i];
      T = fmin(fmax(T, Tmin), Tmax);
      int clamp_hits = 0;
      bool done = false;
#pragma unroll 1
      for (int it = 1; it <= 50; ++it) {
        eval(T, hT, cpT);
        double Tn = T + (hs - hT) * rcx::rcp_f64(cpT);
        bool clamped = false;
        if (Tn < Tmin) { Tn = Tmin; clamped = true; }
        if (Tn > Tmax) { Tn = Tmax; clamped = true; }
        clamp_hits = clamped ? clamp_hits + 1 : 0;
        if (clamp_hits >= 2) break;
        if (!clamped && fabs(Tn - T) <= 1e-10 * Tn) { T = Tn; done = true; break; }
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
    }
    eval(T, hT, cpT);
    if (c.mode == RC_MODE_T && c.h) c.h[i] = hT;
    const double rho = p / (RC_RU * T * sW);
    if (c.cp) c.cp[i] = cpT;
    if (c.rho) c.rho[i] = rho;
    n_neg += neg;
    n_bad += !(isfinite(T) && isfinite(cpT) && isfinite(rho));
    Tloc_max = fmax(Tloc_max, (T > 0.0 && T < 1e300) ? T : 0.0);
  }
  if (c.diag) {
    warp_count_add(c.diag + RC_DIAG_NEWTON_BISECT, n_bisect);
    warp_count_add(c.diag + RC_DIAG_NEWTON_MAXIT, n_maxit);
    warp_count_add(c.diag + RC_DIAG_NEGY_IN, n_neg);
    warp_count_add(c.diag + RC_DIAG_NONFINITE, n_bad);
  }
  if (c.red) warp_max_T(c.red, Tloc_max);
}

}  // namespace

int launch_thermo(const rc_mech *m, const CellsDev &c, cudaStream_t s) {
  if (c.n == 0) return RC_OK;
  const int threads = 256;
  int64_t blocks = (c.n + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const size_t smem = (size_t)ThermoSeg::size(m->ns) * 8;
  const bool u = m->uniform_tmid;
  ProfScope prof(RC_STAGE_THERMO, s);
  if (m->ns == 9 && u)
    thermo_kernel<9, true><<<(unsigned)blocks, threads, smem, s>>>(m->d_thermo, m->ns, c);
  else if (m->ns == 20 && u)
    thermo_kernel<20, true><<<(unsigned)blocks, threads, smem, s>>>(m->d_thermo, m->ns, c);
  else if (u)
    thermo_kernel<0, true><<<(unsigned)blocks, threads, smem, s>>>(m->d_thermo, m->ns, c);
  else
    thermo_kernel<0, false><<<(unsigned)blocks, threads, smem, s>>>(m->d_thermo, m->ns, c);
  RC_LAUNCH_CHECK();
  return RC_OK;
}
