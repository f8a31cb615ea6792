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

template <int NS>
__global__ void __launch_bounds__(TR_TILE, NS == 9 ? 3 : NS == 20 ? 2 : 1)
    transport_kernel(const double *__restrict__ tab, int ns_rt, CellsDev c, int stages) {
  extern __shared__ __align__(16) double s_tab[];
  __shared__ __align__(8) uint64_t bars[1 + 8];
  const int ns = NS ? NS : ns_rt;
  const int tsz = TransportSeg::size(ns);
  const rcs::Ring<TR_TILE> ring{reinterpret_cast<uint8_t *>(s_tab + tsz), bars + 1, 2 + ns, 0, stages};
  if (threadIdx.x == 0) {
    rcx::mbar_init(&bars[0], 1);
    ring.init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    rcx::mbar_arrive_expect_tx(&bars[0], (uint32_t)tsz * 8u);
    rcx::bulk_g2s(s_tab, tab, (uint32_t)tsz * 8u, &bars[0]);
  }
  auto src8 = [&](int r) -> const double * { return r == 0 ? c.T : r == 1 ? c.p : c.Y + (size_t)(r - 2) * c.ld; };
  auto src4 = [&](int) -> const float * { return nullptr; };
  rcx::mbar_wait(&bars[0], 0);
  const int nse = TransportSeg::nse(ns);
  const double *visc = s_tab + TransportSeg::visc(ns), *cond = s_tab + TransportSeg::cond(ns);
  const double *diff = s_tab + TransportSeg::diff(ns), *W = s_tab + TransportSeg::W(ns);
  const double *invW = s_tab + TransportSeg::invW(ns);
  const double *M0 = s_tab + TransportSeg::M(ns, 0), *M1 = s_tab + TransportSeg::M(ns, 1),
               *M2 = s_tab + TransportSeg::M(ns, 2);
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
        sW = fma(X[k], invW[k], sW);
      }
    if (ns & 1) X[ns] = u[ns] = v[ns] = 0.0;  // pad slot: M rows are zero there
    const double Wbar = rcx::rcp_f64_fast(sW);
    const double L = log(T), sT = sqrt(T), qT = sqrt(sT), T15 = T * sT, pT = p / T15;
    double s1 = 0.0, s2 = 0.0, Wp = 0.0;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        const double x = X[k] * Wbar * invW[k];
        X[k] = x > 0.0 ? x : 0.0;                 // X+ = max(X, 0)
        s[k] = qT * poly5(visc + 5 * k, L);       // sqrt(mu_k)
        const double rs = rcx::rcp_f64_fast(s[k]);
        u[k] = X[k] * rs;
        v[k] = u[k] * rs;
        const double lam = sT * poly5(cond + 5 * k, L);
        s1 = fma(X[k], lam, s1);
        s2 = fma(X[k], rcx::rcp_f64_fast(lam), s2);
        Wp = fma(X[k], W[k], Wp);
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
            const double2 m0 = lds2(M0 + k * nse + j), m1 = lds2(M1 + k * nse + j), m2 = lds2(M2 + k * nse + j);
            A = fma(m0.x, X[j], A);
            B = fma(m1.x, u[j], B);
            C = fma(m2.x, v[j], C);
            A = fma(m0.y, X[j + 1], A);
            B = fma(m1.y, u[j + 1], B);
            C = fma(m2.y, v[j + 1], C);
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
              const double iR = rcx::rcp_f64_fast(poly5a(diff + 6 * (k * (k + 1) / 2 + j), L));
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
          acc = fma(X[k], W[k], acc);
        }
      acc = 0.0;
#pragma unroll UR
      for (int k = CAP - 1; k >= 0; --k)
        if (k < ns) {
          const double num = u[k] + acc;
          acc = fma(X[k], W[k], acc);
          const double Dk = (S[k] == 0.0) ? poly5a(diff + 6 * (k * (k + 1) / 2 + k), L) * rcx::rcp_f64_fast(pT)
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

// ---------------------------------------------------------------------------------------------
// Warp-cooperative variant for large mechanisms (north_star: "warp-level reductions for the Ns^2
// Wilke mixing sums"; "shared memory for mass and mole fractions"): L = 4 lanes per
// cell, lane q owns species k = q, q + 4, ...  Per-species quantities are computed by their owner;
// the Wilke sums A_k, B_k, C_k run over all j with X_j, u_j, v_j broadcast from the owner lane by
// shuffles; binary pairs j < k are evaluated once by the owner of k, which also accumulates the
// partner's S_j in a per-lane partial that is reduced over the 4 lanes at the end; the cell sums
// (1/W, s1, s2, W+, mu) are reduced over the lanes with two xor-shuffles.  The per-thread state is a
// quarter of the one-thread-per-cell kernel's (which needs ~255 registers and spills at Ns = 20).
constexpr int TRC_TILE = 64;  // cells per stage; 4 lanes each

__device__ __forceinline__ double quad_sum(double v) {  // sum over the 4 lanes of a cell
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

template <int NS>
__global__ void __launch_bounds__(TRC_TILE * 4, 2) transport_coop_kernel(const double *__restrict__ tab, CellsDev c, int stages) {
  constexpr int L = 4, SPL = (NS + L - 1) / L;
  extern __shared__ __align__(16) double s_tab[];
  __shared__ __align__(8) uint64_t bars[1 + 8];
  const int tsz = TransportSeg::size(NS);
  const rcs::Ring<TRC_TILE> ring{reinterpret_cast<uint8_t *>(s_tab + tsz), bars + 1, 2 + NS, 0, stages};
  if (threadIdx.x == 0) {
    rcx::mbar_init(&bars[0], 1);
    ring.init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    rcx::mbar_arrive_expect_tx(&bars[0], (uint32_t)tsz * 8u);
    rcx::bulk_g2s(s_tab, tab, (uint32_t)tsz * 8u, &bars[0]);
  }
  auto src8 = [&](int r) -> const double * { return r == 0 ? c.T : r == 1 ? c.p : c.Y + (size_t)(r - 2) * c.ld; };
  auto src4 = [&](int) -> const float * { return nullptr; };
  rcx::mbar_wait(&bars[0], 0);
  constexpr int nse = (NS + 1) & ~1;
  const double *visc = s_tab + TransportSeg::visc(NS), *cond = s_tab + TransportSeg::cond(NS);
  const double *diff = s_tab + TransportSeg::diff(NS), *W = s_tab + TransportSeg::W(NS);
  const double *invW = s_tab + TransportSeg::invW(NS);
  const double *M0 = s_tab + TransportSeg::M(NS, 0), *M1 = s_tab + TransportSeg::M(NS, 1),
               *M2 = s_tab + TransportSeg::M(NS, 2);
  const int lane = threadIdx.x & 31, q = lane & 3, base = lane & ~3;
  const int cell = threadIdx.x >> 2;
  int n_bad = 0;
  ring.run(c.n, src8, src4, [&](int st, int64_t tile) {
    const int64_t i = tile * TRC_TILE + cell;
    const bool valid = i < c.n;                          // every lane takes part in the shuffles
    const double *S8 = ring.row8(st, 0) + cell;
    const double T = valid ? S8[0] : 300.0, p = valid ? S8[TRC_TILE] : 1e5;
    double X[SPL], s[SPL], u[SPL], v[SPL];
    double sW = 0.0;
#pragma unroll
    for (int a = 0; a < SPL; ++a) {
      const int k = q + L * a;
      X[a] = (k < NS && valid) ? S8[(2 + k) * TRC_TILE] : 0.0;
      if (k < NS) sW = fma(X[a], invW[k], sW);
    }
    sW = quad_sum(sW);
    const double Wbar = rcx::rcp_f64_fast(sW > 0.0 ? sW : 1.0);
    const double Lg = log(T), sT = sqrt(T), qT = sqrt(sT), T15 = T * sT, pT = p / T15;
    double s1 = 0.0, s2 = 0.0, Wp = 0.0;
#pragma unroll
    for (int a = 0; a < SPL; ++a) {
      const int k = q + L * a;
      if (k < NS) {
        const double x = X[a] * Wbar * invW[k];
        X[a] = x > 0.0 ? x : 0.0;                        // X+ = max(X, 0)
        s[a] = qT * poly5(visc + 5 * k, Lg);             // sqrt(mu_k)
        const double rs = rcx::rcp_f64_fast(s[a]);
        u[a] = X[a] * rs;
        v[a] = u[a] * rs;
        const double lam = sT * poly5(cond + 5 * k, Lg);
        s1 = fma(X[a], lam, s1);
        s2 = fma(X[a], rcx::rcp_f64_fast(lam), s2);
        Wp = fma(X[a], W[k], Wp);
      } else {
        s[a] = 1.0;
        u[a] = v[a] = 0.0;
      }
    }
    s1 = quad_sum(s1);
    s2 = quad_sum(s2);
    Wp = quad_sum(Wp);
    // Wilke sums and the D_k numerators sum_{j != k} X_j W_j, j broadcast from its owner lane
    double A[SPL], B[SPL], C[SPL], num[SPL];
#pragma unroll
    for (int a = 0; a < SPL; ++a) A[a] = B[a] = C[a] = num[a] = 0.0;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      const int src = base | (j % L);
      const double xj = __shfl_sync(0xffffffffu, X[j / L], src), uj = __shfl_sync(0xffffffffu, u[j / L], src),
                   vj = __shfl_sync(0xffffffffu, v[j / L], src);
#pragma unroll
      for (int a = 0; a < SPL; ++a) {
        const int k = q + L * a;
        if (k < NS) {
          A[a] = fma(lds(M0 + k * nse + j), xj, A[a]);
          B[a] = fma(lds(M1 + k * nse + j), uj, B[a]);
          C[a] = fma(lds(M2 + k * nse + j), vj, C[a]);
          if (j != k) num[a] = fma(xj, W[j], num[a]);
        }
      }
    }
    double mu = 0.0;
#pragma unroll
    for (int a = 0; a < SPL; ++a) {
      const int k = q + L * a;
      if (k < NS) {
        const double den = fma(s[a], fma(s[a], C[a], B[a]), A[a]);
        if (den > 0.0) mu = fma(X[a] * (s[a] * s[a]), rcx::rcp_f64_fast(den), mu);
      }
    }
    mu = quad_sum(mu);
    const double lam = 0.5 * (s1 + rcx::rcp_f64_fast(s2));
    bool bad = !(isfinite(mu) && isfinite(lam));
    if (valid && q == 0) {
      if (c.mu) c.mu[i] = mu;
      if (c.lambda) c.lambda[i] = lam;
    }
    if (c.D) {
      // pairs j < k by the owner of k: S_k (own) and the partner's share S_j in a per-lane partial
      double S[SPL], Sp[NS];
#pragma unroll
      for (int a = 0; a < SPL; ++a) S[a] = 0.0;
#pragma unroll
      for (int j = 0; j < NS; ++j) Sp[j] = 0.0;
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const double xj = __shfl_sync(0xffffffffu, X[j / L], base | (j % L));
#pragma unroll
        for (int a = 0; a < SPL; ++a) {
          const int k = q + L * a;
          if (k < NS && j < k) {
            const double iR = rcx::rcp_f64_fast(poly5a(diff + 6 * (k * (k + 1) / 2 + j), Lg));
            S[a] = fma(xj, iR, S[a]);
            Sp[j] = fma(X[a], iR, Sp[j]);
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NS; ++j) {
        const double tot = quad_sum(Sp[j]);
        if (q == j % L) S[j / L] += tot;
      }
#pragma unroll
      for (int a = 0; a < SPL; ++a) {
        const int k = q + L * a;
        if (k < NS) {
          const double Dk = (S[a] == 0.0) ? poly5a(diff + 6 * (k * (k + 1) / 2 + k), Lg) * rcx::rcp_f64_fast(pT)
                                          : num[a] * rcx::rcp_f64_fast(Wp * pT * S[a]);
          if (valid) c.D[k * c.ld + i] = Dk;
          bad |= !isfinite(Dk);
        }
      }
    }
    if (valid && q == 0) n_bad += bad;
  });
  if (c.diag) {
    unsigned v = __reduce_add_sync(0xffffffffu, (unsigned)n_bad);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd((unsigned long long *)(c.diag + RC_DIAG_NONFINITE), v);
  }
}

template <int NS>
int launch_transport_coop(const rc_mech *m, const CellsDev &c, cudaStream_t s) {
  const int stages = 3;
  const size_t smem = (size_t)TransportSeg::size(m->ns) * 8 + rcs::Ring<TRC_TILE>::smem_bytes(2 + m->ns, 0, stages);
  const int64_t ntiles = (c.n + TRC_TILE - 1) / TRC_TILE;
  int64_t grid = rc_resident_blocks((const void *)transport_coop_kernel<NS>, TRC_TILE * 4, smem);
  if (grid > ntiles) grid = ntiles;
  transport_coop_kernel<NS><<<(unsigned)grid, TRC_TILE * 4, smem, s>>>(m->d_transport, c, stages);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

template <int NS>
int launch_transport_t(const rc_mech *m, const CellsDev &c, cudaStream_t s) {
  const int stages = 3;
  const size_t smem = (size_t)TransportSeg::size(m->ns) * 8 + rcs::Ring<TR_TILE>::smem_bytes(2 + m->ns, 0, stages);
  const int64_t ntiles = (c.n + TR_TILE - 1) / TR_TILE;
  int64_t grid = rc_resident_blocks((const void *)transport_kernel<NS>, TR_TILE, smem);
  if (grid > ntiles) grid = ntiles;
  transport_kernel<NS><<<(unsigned)grid, TR_TILE, smem, s>>>(m->d_transport, m->ns, c, stages);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

}  // namespace

int launch_transport(const rc_mech *m, const CellsDev &c, cudaStream_t s) {
  if (c.n == 0) return RC_OK;
  ProfScope prof(RC_STAGE_TRANSPORT, s);
  if (m->ns == 9) return launch_transport_t<9>(m, c, s);
  if (m->ns == 20) return launch_transport_coop<20>(m, c, s);
  return launch_transport_t<0>(m, c, s);
}
