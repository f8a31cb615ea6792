// transport.cu -- path step a2: Wilke mixture viscosity, Mathur conductivity and
// mixture-averaged species diffusivities from per-species polynomial fits in
// ln T ("molecular transport models ... via the Cantera
// interface", "high-order temperature polynomials"; SURVEY.md
// §8(c) step 5; R10, R11).
//
// FP64-pipe-bound: the Ns^2 Wilke sums and the Ns(Ns+1)/2
// binary-diffusion fits dominate.  One thread per cell, cells streamed through a
// ring of shared-memory stages by bulk-TMA copies of the SoA rows (stream.cuh);
// the coefficient table is staged once per CTA and read as shared-memory
// broadcasts, two doubles per 16-byte load.
//
// Operation count, "computation consolidation":
//  - sqrt(mu_k) = s_k = T^(1/4) P_k(ln T), T^(1/4) = sqrt(sqrt(T));
//  - Wilke: with u_j = X_j / s_j and v_j = u_j / s_j the denominator
//    sum_j X_j [1 + (s_k/s_j) c1_kj]^2 c2_kj expands exactly into
//    A_k + s_k (B_k + s_k C_k), A = M0 X, B = M1 u, C = M2 v (rc_internal.h
//    TransportSeg): three FMAs per (k, j) pair, all terms positive (no
//    cancellation against the oracle's direct form);
//  - mixture-averaged D_k: 1/R_jk(ln T) once per pair j < k, used for S_k and
//    S_j; the numerator sum_{j != k} X_j W_j as prefix + suffix sums (no
//    1 - Y_k cancellation, R11).
#include <cstring>

#include "ptx.cuh"
#include "rc_internal.h"
#include "stream.cuh"

namespace {

// Shared-memory table reads kept in program order: with the species loops fully
// unrolled the compiler would otherwise hoist the whole coefficient table into
// registers (255 registers and spills for 20 species).
__device__ __forceinline__ double lds(const double *p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(rcx::smem_u32(p)));
  return v;
}
__device__ __forceinline__ double2 lds2(const double *p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(rcx::smem_u32(p)));
  return v;
}
__device__ __forceinline__ double poly5(const double *c, double L) {
  return fma(L, fma(L, fma(L, fma(L, lds(c + 4), lds(c + 3)), lds(c + 2)), lds(c + 1)), lds(c));
}
// 16-byte aligned 6-slot fit row (diff): three 16-byte loads
__device__ __forceinline__ double poly5a(const double *c, double L) {
  const double2 a = lds2(c), b = lds2(c + 2), d = lds2(c + 4);
  return fma(L, fma(L, fma(L, fma(L, d.x, b.y), b.x), a.y), a.x);
}

constexpr int TR_TILE = 128;

// The coefficient table of a compiled mechanism size travels as a kernel parameter (constant bank):
// with the species loops fully unrolled every coefficient is a compile-time offset, so the DFMAs take
// it as a constant-bank operand -- no shared-memory load per coefficient (~40% of the kernel's
// instructions were such loads) and no per-CTA table staging.  The generic size stages it in smem.
// (Ns = 9 only: at Ns = 20 the 21.6 KB table as uniform-register operands made the kernel larger and
// spill, and the one-thread kernel there is bound by its FP64 issue anyway)
template <int NS> constexpr bool tr_param() { return NS == 9; }
template <int NS>
struct TrParam {
  double v[tr_param<NS>() ? TransportSeg::size(NS) : 2];
};

template <int NS>
__global__ void __launch_bounds__(TR_TILE, NS == 9 ? 4 : NS == 20 ? 2 : 1)
    transport_kernel(const double *__restrict__ tab, const __grid_constant__ TrParam<NS> P, int ns_rt, CellsDev c,
                     int stages) {
  extern __shared__ __align__(16) double s_tab[];
  __shared__ __align__(8) uint64_t bars[1 + 8];
  const int ns = NS ? NS : ns_rt;
  constexpr bool PT = tr_param<NS>();
  const int tsz = PT ? 0 : TransportSeg::size(ns);
  const rcs::Ring<TR_TILE> ring{reinterpret_cast<uint8_t *>(s_tab + tsz), bars + 1, 2 + ns, 0, stages};
  if (threadIdx.x == 0) {
    rcx::mbar_init(&bars[0], 1);
    ring.init();
  }
  __syncthreads();
  if (!PT && threadIdx.x == 0) {
    rcx::mbar_arrive_expect_tx(&bars[0], (uint32_t)tsz * 8u);
    rcx::bulk_g2s(s_tab, tab, (uint32_t)tsz * 8u, &bars[0]);
  }
  auto src8 = [&](int r) -> const double * { return r == 0 ? c.T : r == 1 ? c.p : c.Y + (size_t)(r - 2) * c.ld; };
  auto src4 = [&](int) -> const float * { return nullptr; };
  if (!PT) rcx::mbar_wait(&bars[0], 0);
  const int nse = TransportSeg::nse(ns);
  // table entry i: a constant-bank operand (NS > 0) or an ordered shared-memory load (generic)
  auto tv = [&](int i) -> double {
    if constexpr (PT) return P.v[i];
    else return lds(s_tab + i);
  };
  auto poly5t = [&](int o, double L) {
    return fma(L, fma(L, fma(L, fma(L, tv(o + 4), tv(o + 3)), tv(o + 2)), tv(o + 1)), tv(o));
  };
  const int VISC = TransportSeg::visc(ns), COND = TransportSeg::cond(ns), DIFF = TransportSeg::diff(ns);
  const int WO = TransportSeg::W(ns), IWO = TransportSeg::invW(ns);
  const int M0 = TransportSeg::M(ns, 0), M1 = TransportSeg::M(ns, 1), M2 = TransportSeg::M(ns, 2);
  constexpr int CAP = NS ? NS : RC_MAX_NS;
  constexpr int UR = NS ? NS : 1;
  constexpr int CAPE = (CAP + 1) & ~1;

  int n_bad = 0;
  ring.run(c.n, src8, src4, [&](int st, int64_t tile) {
    const int jt = threadIdx.x;
    const int64_t i = tile * TR_TILE + jt;
    if (i >= c.n) return;
    const double *S8 = ring.row8(st, 0) + jt;  // fp64 row q of this cell: S8[q * TR_TILE]
    const double T = S8[0], p = S8[TR_TILE];
    double X[CAPE], s[CAP], u[CAPE], v[CAPE];
    double sW = 0.0;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        X[k] = S8[(2 + k) * TR_TILE];
        sW = fma(X[k], tv(IWO + k), sW);
      }
    if (ns & 1) X[ns] = u[ns] = v[ns] = 0.0;  // pad slot: M rows are zero there
    const double Wbar = rcx::rcp_f64_fast(sW);
    const double L = log(T), sT = sqrt(T), qT = sqrt(sT), T15 = T * sT, pT = p / T15;
    double s1 = 0.0, s2 = 0.0, Wp = 0.0;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        const double x = X[k] * Wbar * tv(IWO + k);
        X[k] = x > 0.0 ? x : 0.0;                 // X+ = max(X, 0)
        s[k] = qT * poly5t(VISC + 5 * k, L);      // sqrt(mu_k)
        const double rs = rcx::rcp_f64_fast(s[k]);
        u[k] = X[k] * rs;
        v[k] = u[k] * rs;
        const double lam = sT * poly5t(COND + 5 * k, L);
        s1 = fma(X[k], lam, s1);
        s2 = fma(X[k], rcx::rcp_f64_fast(lam), s2);
        Wp = fma(X[k], tv(WO + k), Wp);
      }
    // Wilke: mu = sum_k X_k s_k^2 / (A_k + s_k (B_k + s_k C_k))
    double mu = 0.0;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        double A = 0.0, B = 0.0, C = 0.0;
#pragma unroll
        for (int j = 0; j < CAPE; j += 2)
          if (j < ns) {
            if constexpr (PT) {
              A = fma(tv(M0 + k * nse + j), X[j], A);
              B = fma(tv(M1 + k * nse + j), u[j], B);
              C = fma(tv(M2 + k * nse + j), v[j], C);
              A = fma(tv(M0 + k * nse + j + 1), X[j + 1], A);
              B = fma(tv(M1 + k * nse + j + 1), u[j + 1], B);
              C = fma(tv(M2 + k * nse + j + 1), v[j + 1], C);
            } else {
              const double2 m0 = lds2(s_tab + M0 + k * nse + j), m1 = lds2(s_tab + M1 + k * nse + j),
                            m2 = lds2(s_tab + M2 + k * nse + j);
              A = fma(m0.x, X[j], A);
              B = fma(m1.x, u[j], B);
              C = fma(m2.x, v[j], C);
              A = fma(m0.y, X[j + 1], A);
              B = fma(m1.y, u[j + 1], B);
              C = fma(m2.y, v[j + 1], C);
            }
          }
        const double den = fma(s[k], fma(s[k], C, B), A);
        if (den > 0.0) mu = fma(X[k] * (s[k] * s[k]), rcx::rcp_f64_fast(den), mu);
      }
    if (c.mu) c.mu[i] = mu;
    const double lam = 0.5 * (s1 + rcx::rcp_f64_fast(s2));
    if (c.lambda) c.lambda[i] = lam;
    bool bad = !(isfinite(mu) && isfinite(lam));
    if (c.D) {
      // S_k = sum_{j != k} X_j / R_jk(L) (the p / T^1.5 factor is applied once per species)
      double S[CAP];
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k < ns) S[k] = 0.0;
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k < ns) {
#pragma unroll UR
          for (int j = 0; j < CAP; ++j)
            if (j < k) {
              const int o = DIFF + 6 * (k * (k + 1) / 2 + j);
              const double iR = rcx::rcp_f64_fast(PT ? poly5t(o, L) : poly5a(s_tab + o, L));
              S[k] = fma(X[j], iR, S[k]);
              S[j] = fma(X[k], iR, S[j]);
            }
        }
      // numerators sum_{j != k} X_j W_j = prefix_k + suffix_k; reuse u as the prefix array
      double acc = 0.0;
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k < ns) {
          u[k] = acc;
          acc = fma(X[k], tv(WO + k), acc);
        }
      acc = 0.0;
#pragma unroll UR
      for (int k = CAP - 1; k >= 0; --k)
        if (k < ns) {
          const double num = u[k] + acc;
          acc = fma(X[k], tv(WO + k), acc);
          const int o = DIFF + 6 * (k * (k + 1) / 2 + k);
          const double Dk = (S[k] == 0.0) ? (PT ? poly5t(o, L) : poly5a(s_tab + o, L)) * rcx::rcp_f64_fast(pT)
                                          : num * rcx::rcp_f64_fast(Wp * pT * S[k]);
          c.D[k * c.ld + i] = Dk;
          bad |= !isfinite(Dk);
        }
    }
    n_bad += bad;
  });
  if (c.diag) {
    unsigned v = __reduce_add_sync(0xffffffffu, (unsigned)n_bad);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd((unsigned long long *)(c.diag + RC_DIAG_NONFINITE), v);
  }
}

template <int NS>
int launch_transport_t(const rc_mech *m, const CellsDev &c, cudaStream_t s) {
  const int stages = 3;
  const size_t smem = (size_t)(tr_param<NS>() ? 0 : TransportSeg::size(m->ns)) * 8 + rcs::Ring<TR_TILE>::smem_bytes(2 + m->ns, 0, stages);
  const int64_t ntiles = (c.n + TR_TILE - 1) / TR_TILE;
  int64_t grid = rc_resident_blocks((const void *)transport_kernel<NS>, TR_TILE, smem);
  if (grid > ntiles) grid = ntiles;
  TrParam<NS> P;
  if (tr_param<NS>()) std::memcpy(P.v, m->transport_host.data(), sizeof(P.v));
  transport_kernel<NS><<<(unsigned)grid, TR_TILE, smem, s>>>(m->d_transport, P, m->ns, c, stages);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

}  // namespace

int launch_transport(const rc_mech *m, const CellsDev &c, cudaStream_t s) {
  if (c.n == 0) return RC_OK;
  ProfScope prof(RC_STAGE_TRANSPORT, s);
  if (m->ns == 9) return launch_transport_t<9>(m, c, s);
  if (m->ns == 20) return launch_transport_t<20>(m, c, s);
  return launch_transport_t<0>(m, c, s);
}
