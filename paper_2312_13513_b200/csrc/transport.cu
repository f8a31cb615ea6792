// transport.cu -- path step a2: Wilke mixture viscosity, Mathur conductivity and
// mixture-averaged species diffusivities from per-species polynomial fits in
// ln T ("molecular transport models ... via the Cantera
// interface", "high-order temperature polynomials"; SURVEY.md
// §8(c) step 5; R10, R11).
//
// FP64-pipe-bound: the Ns^2 Wilke sums and the Ns(Ns+1)/2 binary-diffusion
// fits dominate.  One thread per cell; the coefficient table
// (fits + precomputed Wilke constants (W_j/W_k)^(1/4), 1/sqrt(8(1+W_k/W_j)))
// is staged into shared memory with one bulk-TMA copy and read as broadcasts.
// "Computation consolidation": sqrt(mu_k/mu_j) = s_k / s_j with
// s_k = T^(1/4) P_k(ln T) (so mu_k = s_k^2), and T^(1/4) = sqrt(sqrt(T)).
#include "ptx.cuh"
#include "rc_internal.h"

namespace {

// Shared-memory table reads kept in program order: with the species loops fully
// unrolled the compiler would otherwise hoist the whole coefficient table into
// registers (255 registers and spills for 20 species).
__device__ __forceinline__ double lds(const double *p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(rcx::smem_u32(p)));
  return v;
}
__device__ __forceinline__ double poly5(const double *c, double L) {
  return fma(L, fma(L, fma(L, fma(L, lds(c + 4), lds(c + 3)), lds(c + 2)), lds(c + 1)), lds(c));
}

template <int NS>
__global__ void __launch_bounds__(128, NS == 9 ? 4 : 1) transport_kernel(const double *__restrict__ tab, int ns_rt, CellsDev c) {
  extern __shared__ __align__(16) double s_tab[];
  __shared__ __align__(8) uint64_t bar;
  const int ns = NS ? NS : ns_rt;
  const uint32_t bytes = (uint32_t)TransportSeg::size(ns) * 8u;
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
  const double *visc = s_tab + TransportSeg::visc(ns), *cond = s_tab + TransportSeg::cond(ns);
  const double *diff = s_tab + TransportSeg::diff(ns), *W = s_tab + TransportSeg::W(ns);
  const double *invW = s_tab + TransportSeg::invW(ns), *c1 = s_tab + TransportSeg::c1(ns);
  const double *c2 = s_tab + TransportSeg::c2(ns);
  constexpr int CAP = NS ? NS : RC_MAX_NS;
  constexpr int UR = NS ? NS : 1;

  int n_bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.n; i += (int64_t)gridDim.x * blockDim.x) {
    const double T = c.T[i], p = c.p[i];
    double X[CAP], s[CAP], rs[CAP], S[CAP];
    double sW = 0.0;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        X[k] = c.Y[k * c.ld + i];
        sW = fma(X[k], invW[k], sW);
      }
    const double Wbar = rcx::rcp_f64(sW);
    const double L = log(T), sT = sqrt(T), qT = sqrt(sT), T15 = T * sT, pT = p / T15;
    double s1 = 0.0, s2 = 0.0, Wp = 0.0;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        double x = X[k] * Wbar * invW[k];
        X[k] = x > 0.0 ? x : 0.0;                 // X+ = max(X, 0)
        s[k] = qT * poly5(visc + 5 * k, L);       // sqrt(mu_k)
        rs[k] = rcx::rcp_f64(s[k]);
        double lam = sT * poly5(cond + 5 * k, L);
        s1 = fma(X[k], lam, s1);
        s2 = fma(X[k], rcx::rcp_f64(lam), s2);
        Wp = fma(X[k], W[k], Wp);
        S[k] = 0.0;
      }
    // Wilke: mu = sum_k X_k mu_k / sum_j X_j Phi_kj
    double mu = 0.0;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        double den = 0.0;
#pragma unroll UR
        for (int j = 0; j < CAP; ++j)
          if (j < ns) {
            double t = fma(s[k] * rs[j], lds(c1 + k * ns + j), 1.0);
            den = fma(X[j], t * t * lds(c2 + k * ns + j), den);
          }
        if (den > 0.0) mu += X[k] * (s[k] * s[k]) * rcx::rcp_f64(den);
      }
    // mixture-averaged diffusion: S_k = sum_{j != k} X_j / D_jk, 1/D_jk = p / (T^1.5 R_jk(L))
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
#pragma unroll UR
        for (int j = 0; j < CAP; ++j)
          if (j < k) {
            double iD = pT * rcx::rcp_f64(poly5(diff + 5 * (k * (k + 1) / 2 + j), L));
            S[k] = fma(X[j], iD, S[k]);
            S[j] = fma(X[k], iD, S[j]);
          }
      }
    if (c.mu) c.mu[i] = mu;
    const double lam = 0.5 * (s1 + rcx::rcp_f64(s2));
    if (c.lambda) c.lambda[i] = lam;
    bool bad = !(isfinite(mu) && isfinite(lam));
    if (c.D) {
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k < ns) {
          double num = 0.0;  // sum_{j != k} X_j W_j (stable numerator, R11)
#pragma unroll UR
          for (int j = 0; j < CAP; ++j)
            if (j < ns && j != k) num = fma(X[j], W[j], num);
          double Dk = (S[k] == 0.0) ? poly5(diff + 5 * (k * (k + 1) / 2 + k), L) * rcx::rcp_f64(pT)
                                    : num * rcx::rcp_f64(Wp * S[k]);
          c.D[k * c.ld + i] = Dk;
          bad |= !isfinite(Dk);
        }
    }
    n_bad += bad;
  }
  if (c.diag) {
    unsigned v = __reduce_add_sync(0xffffffffu, (unsigned)n_bad);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd((unsigned long long *)(c.diag + RC_DIAG_NONFINITE), v);
  }
}

}  // namespace

int launch_transport(const rc_mech *m, const CellsDev &c, cudaStream_t s) {
  if (c.n == 0) return RC_OK;
  const int threads = 128;
  int64_t blocks = (c.n + threads - 1) / threads;
  if (blocks > 148 * 32) blocks = 148 * 32;
  const size_t smem = (size_t)TransportSeg::size(m->ns) * 8;
  ProfScope prof(RC_STAGE_TRANSPORT, s);
  if (m->ns == 9)
    transport_kernel<9><<<(unsigned)blocks, threads, smem, s>>>(m->d_transport, m->ns, c);
  else if (m->ns == 20) {
    cudaFuncSetAttribute(transport_kernel<20>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    transport_kernel<20><<<(unsigned)blocks, threads, smem, s>>>(m->d_transport, m->ns, c);
  } else {
    cudaFuncSetAttribute(transport_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    transport_kernel<0><<<(unsigned)blocks, threads, smem, s>>>(m->d_transport, m->ns, c);
  }
  RC_LAUNCH_CHECK();
  return RC_OK;
}
