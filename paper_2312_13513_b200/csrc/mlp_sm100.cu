// mlp_sm100.cu -- path steps a3-a5: the DNN chemistry step on the 5th-generation
// tensor cores (§2: "individual neural networks ... for each
// component, excluding inert gases ... three hidden layers comprising 1600,
// 800, and 400 perceptrons ... GELU"; inputs T, p, Y; output the species'
// rate of change).  Box-Cox / z-score prologue, the per-species MLPs as
// tcgen05 GEMMs with TMEM accumulators and fused bias+GELU epilogues, and an
// fp64 epilogue doing the inverse Box-Cox, element projection, wdot and qdot
// (R1-R7, R13).
//
// Kernel structure (per chunk of `cap` cells, all nets batched in one launch):
//   prologue      T,p,Y (fp64 SoA) -> z [cap][kz] bf16 (K-major A operand, two 1-columns for b1)
//   l1_kernel     h1 = GELU(z W1^T)                  [nets][cap][h1] bf16   (mlp_l1_sm100.cu)
//   l2_pair       h2 = GELU(h1 W2^T + b2)            [nets][cap][h2] bf16   (mlp_l2_sm100.cu)
//   l3_kernel     o_part = GELU(h2 W3^T + b3) . w4   (layer 4 folded into the epilogue)
//   chem_epilogue o = b4 + sum(o_part) -> dY -> P dY -> wdot, qdot, sum qdot partials
// The layer-3 GEMM is a persistent, warp-specialised kernel: one warp issues
// TMA loads into a multi-stage shared-memory ring (128-byte swizzle), one
// issues tcgen05.mma (M=128, N=BN, K=16) into a double-buffered TMEM
// accumulator, sixteen drain TMEM with tcgen05.ld, add b3, apply GELU and
// reduce against w4.
#include <cuda_bf16.h>

#include <cmath>
#include <cstring>
#include <mutex>

#include "mlp_common.cuh"
#include "mlp_internal.h"
#include "ptx.cuh"
#include "rc_internal.h"


namespace {

constexpr int BM = 128;       // UMMA M (one CTA, cta_group::1)
constexpr int BK = 64;        // K elements per pipeline stage (128 B of bf16 = one swizzle row)
constexpr int GEMM_NEPI = 16;                      // epilogue warps: 4 per TMEM lane quadrant
constexpr int GEMM_THREADS = 32 * GEMM_NEPI + 64;  // + TMA producer warp + MMA issuer warp
constexpr int MAX_CAP = 32768;     // cells per chunk (activation working set)
constexpr int QPART_BLOCKS = 148 * 4;

using rcm::bf_hi;
using rcm::bf_lo;
using rcm::cvt_bf16x2;
using rcm::desc_sw;
using rcm::gelu_bf16x2;

struct GemmArgs {
  int m_tiles, n_tiles, nets, k_blocks, a_shared, N, cap, stages;
  const float *bias;   // [nets][N] or nullptr (bias folded into the MMA)
  const float *w4;     // MODE 1: [nets][N]
  float *opart;        // MODE 1: [nets][n_tiles*4][cap]
};

// Persistent warp-specialised tcgen05 GEMM, M = 128 per CTA, N tile BN
// (runtime-narrower last tile), K chunks of 64, double-buffered TMEM
// accumulator so the epilogue of tile i overlaps the MMAs of tile i+1.
// opart = GELU(A B^T + bias) . w4 per row and column quarter (layer 3 with
// layer 4 folded in).
template <int BN, int KB = BK>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    l3_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, GemmArgs g) {
  static_assert(KB == 16 || KB == 32 || KB == 64, "K atom: 32/64/128-byte swizzle rows");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = rcx::smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  constexpr uint32_t A_BYTES = BM * KB * 2, B_BYTES = BN * KB * 2;
  constexpr int W_TMA = GEMM_NEPI, W_MMA = GEMM_NEPI + 1;
  const int S = g.stages;
  uint8_t *sA = smem, *sB = smem + S * A_BYTES;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + S * B_BYTES);
  uint64_t *empty = full + S, *tfull = empty + S, *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
  constexpr uint32_t TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == W_TMA && lane == 0) {
    rcx::prefetch_tmap(&mapA);
    rcx::prefetch_tmap(&mapB);
    for (int s = 0; s < S; ++s) {
      rcx::mbar_init(&full[s], 1);
      rcx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      rcx::mbar_init(&tfull[a], 1);
      rcx::mbar_init(&tempty[a], GEMM_NEPI);
    }
    rcx::fence_mbar_init();
  }
  if (warp == W_MMA) rcx::tmem_alloc(tmem_slot, TMEM_COLS);
  rcx::tc_fence_before();
  __syncthreads();
  rcx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total = g.m_tiles * g.n_tiles * g.nets;

  if (warp == W_TMA) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int n_blk = tile % g.n_tiles, rest = tile / g.n_tiles;
        const int m_blk = rest % g.m_tiles, net = rest / g.m_tiles;
        for (int kb = 0; kb < g.k_blocks; ++kb) {
          rcx::mbar_wait(&empty[stage], phase ^ 1);
          rcx::mbar_arrive_expect_tx(&full[stage], A_BYTES + B_BYTES);
          rcx::tma_load_3d(sA + stage * A_BYTES, &mapA, &full[stage], kb * KB, m_blk * BM, g.a_shared ? 0 : net);
          rcx::tma_load_3d(sB + stage * B_BYTES, &mapB, &full[stage], kb * KB, n_blk * BN, net);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == W_MMA) {
    if (lane == 0) {  // ---------------- MMA issuer (single thread)
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
        const int n_blk = tile % g.n_tiles;
        const int n_eff = min(BN, g.N - n_blk * BN);  // ragged last tile: multiple of 16
        const uint32_t idesc = rcx::make_idesc(1u, BM, (uint32_t)n_eff);
        const int as = it & 1;
        const uint32_t aphase = (it >> 1) & 1;
        rcx::mbar_wait(&tempty[as], aphase ^ 1);
        rcx::tc_fence_after();
        const uint32_t d = tmem_base + as * BN;
        for (int kb = 0; kb < g.k_blocks; ++kb) {
          rcx::mbar_wait(&full[stage], phase);
          rcx::tc_fence_after();
          const uint64_t ad = desc_sw<KB * 2>(sA + stage * A_BYTES);
          const uint64_t bd = desc_sw<KB * 2>(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < KB / 16; ++k)
            rcx::mma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          rcx::mma_commit(&empty[stage]);
          if (++stage == S) { stage = 0; phase ^= 1; }
        }
        rcx::mma_commit(&tfull[as]);
      }
    }
  } else {  // ---------------- epilogue warps 0..15: four per TMEM lane quadrant, each a quarter of the columns
    const int q = warp & 3;     // TMEM lane quadrant this warp may access
    const int sub = warp >> 2;  // column quarter 0..3
    constexpr int MAXC = (BN / 16 + 3) / 4;  // 16-column chunks per warp (<= 4 for BN <= 256)
    int it = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      const int n_blk = tile % g.n_tiles, rest = tile / g.n_tiles;
      const int m_blk = rest % g.m_tiles, net = rest / g.m_tiles;
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const int NCH = min(BN, g.N - n_blk * BN) / 16;
      const int ch_lo = (NCH * sub) / 4, nch = (NCH * (sub + 1)) / 4 - ch_lo;  // warp-uniform
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + as * BN + ch_lo * 16;
      rcx::mbar_wait(&tfull[as], aphase);
      rcx::tc_fence_after();
      // all of this warp's accumulator columns -> registers, one wait, release the TMEM buffer.
      // Always MAXC chunks (branch-free, so the GELU chains of all chunks interleave); chunks past
      // this warp's range read valid but unused TMEM columns and are never stored.
      uint32_t v[MAXC][16];
#pragma unroll
      for (int c = 0; c < MAXC; ++c) rcx::tmem_ld16(tbase + c * 16, v[c]);
      rcx::tmem_ld_wait();
      rcx::tc_fence_before();
      __syncwarp();
      if (lane == 0) rcx::mbar_arrive(&tempty[as]);
      const size_t col0 = (size_t)net * g.N + n_blk * BN + ch_lo * 16;
      {
        // GELU(acc + b3) . w4 over this warp's columns (layer 4 folded into layer 3)
        float dot = 0.f;
#pragma unroll
        for (int c = 0; c < MAXC; ++c) {
          // chunks past this warp's range contribute with weight 0
          const bool on = c < nch;
          const float4 *bb = reinterpret_cast<const float4 *>(g.bias + col0 + (on ? c * 16 : 0));
          const float4 *ww = reinterpret_cast<const float4 *>(g.w4 + col0 + (on ? c * 16 : 0));
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 b = __ldg(bb + j);
            float4 w = __ldg(ww + j);
            if (!on) w = make_float4(0.f, 0.f, 0.f, 0.f);
#ifdef L3_BF16_GELU
            const uint32_t p0 = gelu_bf16x2(cvt_bf16x2(__uint_as_float(v[c][4 * j]) + b.x, __uint_as_float(v[c][4 * j + 1]) + b.y));
            const uint32_t p1 = gelu_bf16x2(cvt_bf16x2(__uint_as_float(v[c][4 * j + 2]) + b.z, __uint_as_float(v[c][4 * j + 3]) + b.w));
            dot = fmaf(bf_lo(p0), w.x, dot);
            dot = fmaf(bf_hi(p0), w.y, dot);
            dot = fmaf(bf_lo(p1), w.z, dot);
            dot = fmaf(bf_hi(p1), w.w, dot);
#else
            // h3 never leaves the SM: GELU and the layer-4 dot stay in fp32
            dot = fmaf(rcm::gelu_f32(__uint_as_float(v[c][4 * j]) + b.x), w.x, dot);
            dot = fmaf(rcm::gelu_f32(__uint_as_float(v[c][4 * j + 1]) + b.y), w.y, dot);
            dot = fmaf(rcm::gelu_f32(__uint_as_float(v[c][4 * j + 2]) + b.z), w.z, dot);
            dot = fmaf(rcm::gelu_f32(__uint_as_float(v[c][4 * j + 3]) + b.w), w.w, dot);
#endif
          }
        }
        g.opart[((size_t)net * g.n_tiles * 4 + n_blk * 4 + sub) * g.cap + m_blk * BM + q * 32 + lane] = dot;
      }
    }
  }
  __syncthreads();
  if (warp == W_MMA) {
    rcx::tc_fence_after();
    rcx::tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

// ------------------------------------------------------------------ prologue (a3)
struct ProArgs {
  int64_t c0;       // first global cell of the chunk
  int rows, rows_pad, d_in, ns, kz;
  float lambda, inv_lambda;
  const float *xmean, *xinvstd;
  __nv_bfloat16 *z;  // [cap][kz]: z-scored inputs, then two 1.0 columns (b1 hi/lo), then zeros
};

__global__ void __launch_bounds__(256) prologue_kernel(ProArgs a, CellsDev c) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.rows_pad) return;
  float x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = 0.f;
  if (r < a.rows) {
    const int64_t i = a.c0 + r;
    x[0] = ((float)c.T[i] - a.xmean[0]) * a.xinvstd[0];
    x[1] = ((float)c.p[i] - a.xmean[1]) * a.xinvstd[1];
#pragma unroll
    for (int k = 0; k < 30; ++k)
      if (k < a.ns) {
        float y = (float)c.Y[k * c.ld + i];
        y = y > 0.f ? y : 0.f;                                       // Y^ = max(Y, 0)
        float b = y > 0.f ? exp2f(a.lambda * log2f(y)) : 0.f;        // Y^^lambda
        x[2 + k] = ((b - 1.f) * a.inv_lambda - a.xmean[2 + k]) * a.xinvstd[2 + k];  // Box-Cox, z-score
      }
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j == a.d_in || j == a.d_in + 1) x[j] = 1.f;
  }
  uint4 *dst = reinterpret_cast<uint4 *>(a.z + (size_t)r * a.kz);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q * 8 >= a.kz) break;
    uint32_t pk[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __nv_bfloat162 b2 = __floats2bfloat162_rn(x[8 * q + 2 * j], x[8 * q + 2 * j + 1]);
      pk[j] = *reinterpret_cast<uint32_t *>(&b2);
    }
    dst[q] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
  }
}

// ------------------------------------------------------------------ epilogue (a5)
struct EpiArgs {
  int64_t c0;
  int rows, cap, n_nets, nparts, inv_lambda, ns;
  double lambda, inv_dt;
  const float *opart, *b4;
  const double *ymean, *ystd, *P, *thermo;
  const int *species;
  double *qpart;  // [gridDim.x], accumulated across chunks in stream order
};

__device__ __forceinline__ double ipow(double a, int e) {
  double r = 1.0, b = a;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

template <int NS>
__global__ void __launch_bounds__(256) chem_epilogue_kernel(EpiArgs a, CellsDev c) {
  constexpr int CAP = NS ? NS : RC_MAX_NS;
  constexpr int UR = NS ? NS : 1;
  const int ns = NS ? NS : a.ns;
  extern __shared__ __align__(16) double s_tab[];  // thermo segment, then P
  __shared__ __align__(8) uint64_t bar;
  __shared__ double red_s[8];
  const uint32_t tb = (uint32_t)ThermoSeg::size(ns) * 8u, pb = (uint32_t)(((ns * ns + 1) & ~1) * 8);
  double *sP = s_tab + ThermoSeg::size(ns);
  if (threadIdx.x == 0) {
    rcx::mbar_init(&bar, 1);
    rcx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    rcx::mbar_arrive_expect_tx(&bar, tb + pb);
    rcx::bulk_g2s(s_tab, a.thermo, tb, &bar);
    rcx::bulk_g2s(sP, a.P, pb, &bar);
  }
  rcx::mbar_wait(&bar, 0);
  const double *hlo = s_tab + ThermoSeg::hlo(ns), *hhi = s_tab + ThermoSeg::hhi(ns), *tmid = s_tab + ThermoSeg::tmid(ns);

  double qsum = 0.0;
  int n_negout = 0, n_bad = 0;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < a.rows; r += gridDim.x * blockDim.x) {
    const int64_t i = a.c0 + r;
    const double T = c.T[i], rho = c.rho[i];
    double Yh[CAP], dY[CAP];
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        double y = c.Y[k * c.ld + i];
        Yh[k] = y > 0.0 ? y : 0.0;
        dY[k] = 0.0;
      }
    for (int net = 0; net < a.n_nets; ++net) {
      float of = a.b4[net];
      const float *op = a.opart + (size_t)net * a.nparts * a.cap + r;
      for (int p = 0; p < a.nparts; ++p) of += op[(size_t)p * a.cap];
      if (c.o) c.o[net * c.ld + i] = of;
      const int s = a.species[net];
      double ys = 0.0;
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k == s) ys = Yh[k];
      const double b = pow(ys, a.lambda);                         // b_s = Y^_s^lambda
      const double ap = b + a.lambda * ((double)of * a.ystd[net] + a.ymean[net]);
      const double ystar = ap > 0.0 ? ipow(ap, a.inv_lambda) : 0.0;  // inverse Box-Cox
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k == s) dY[k] = ystar - ys;
    }
    // element projection dY <- P dY (fp64), sources
    double q = 0.0;
    bool neg = false, bad = false;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        double v = 0.0;
#pragma unroll UR
        for (int j = 0; j < CAP; ++j)
          if (j < ns) v = fma(sP[k * ns + j], dY[j], v);
        neg |= (Yh[k] + v) < 0.0;
        const double w = rho * v * a.inv_dt;
        c.wdot[k * c.ld + i] = w;
        const double *h = (T <= tmid[k]) ? hlo + 6 * k : hhi + 6 * k;
        const double hk = fma(T, fma(T, fma(T, fma(T, fma(T, h[4], h[3]), h[2]), h[1]), h[0]), h[5]);
        q = fma(-hk, w, q);
        bad |= !isfinite(w);
      }
    if (c.qdot) c.qdot[i] = q;
    bad |= !isfinite(q);
    qsum += q;
    n_negout += neg;
    n_bad += bad;
  }
  if (c.diag) {
    unsigned v1 = __reduce_add_sync(0xffffffffu, (unsigned)n_negout);
    unsigned v2 = __reduce_add_sync(0xffffffffu, (unsigned)n_bad);
    if ((threadIdx.x & 31) == 0) {
      if (v1) atomicAdd((unsigned long long *)(c.diag + RC_DIAG_NEGY_OUT), v1);
      if (v2) atomicAdd((unsigned long long *)(c.diag + RC_DIAG_NONFINITE), v2);
    }
  }
  // fixed-order block sum of qdot -> qpart[block] (deterministic)
  for (int o = 16; o; o >>= 1) qsum += __shfl_xor_sync(0xffffffffu, qsum, o);
  if ((threadIdx.x & 31) == 0) red_s[threadIdx.x >> 5] = qsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red_s[w];
    a.qpart[blockIdx.x] += t;
  }
}

__global__ void qdot_finalize_kernel(const double *qpart, int n, double *out) {
  // one warp, Neumaier-compensated, fixed order
  __shared__ double ss[32], sc[32];
  double s = 0.0, comp = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) {
    double v = qpart[i], t = s + v;
    comp += (fabs(s) >= fabs(v)) ? (s - t) + v : (v - t) + s;
    s = t;
  }
  ss[threadIdx.x] = s;
  sc[threadIdx.x] = comp;
  __syncwarp();
  if (threadIdx.x == 0) {
    double S = 0.0, C = 0.0;
    for (int w = 0; w < 32; ++w) {
      double v = ss[w], t = S + v;
      C += (fabs(S) >= fabs(v)) ? (S - t) + v : (v - t) + S;
      S = t;
      C += sc[w];
    }
    out[1] = S + C;
  }
}

// ------------------------------------------------------------------ host helpers
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 3D bf16 map over [d2][d1][d0] (d0 contiguous), box {box0, box1, 1}; the swizzle
// width equals the box row (box0 * 2 bytes: 32, 64 or 128)
int make_map(CUtensorMap *m, const void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t box1,
             uint32_t box0 = BK) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return rc_fail(RC_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 2, d0 * d1 * 2};
  cuuint32_t box[3] = {box0, box1, 1};
  const CUtensorMapSwizzle sw = box0 * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : box0 * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return rc_fail(RC_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return RC_OK;
}

// N-tile width: split N into ceil(N/208) near-equal tiles rounded up to 16
// (the UMMA N granularity); the last tile may be narrower (runtime N in the
// instruction descriptor, TMA zero-fills the rows past N).  Wide tiles keep the
// shared-memory operand traffic per MMA under the 128 B/clk SMEM port.
int pick_bn(int N) {
  if (N % 16) return 0;
  const int nt = (N + 207) / 208;
  int bn = ((N + nt - 1) / nt + 15) / 16 * 16;
  const int c[] = {16, 32, 48, 64, 96, 128, 160, 208};
  for (int b : c)
    if (b >= bn) return b;
  return 0;
}
int n_tiles_of(int N) { return (N + pick_bn(N) - 1) / pick_bn(N); }

}  // namespace
int mlp_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}
namespace {
int num_sms() { return mlp_num_sms(); }

template <int BN>
int launch_l3_t(const CUtensorMap &A, const CUtensorMap &B, GemmArgs g, cudaStream_t s) {
  const size_t stage_bytes = (size_t)BM * BK * 2 + (size_t)BN * BK * 2;
  const size_t fixed = 1024 + 256;
  int stages = (int)((232448 - fixed) / stage_bytes);
  if (stages > 8) stages = 8;
  g.stages = stages;
  const size_t smem = fixed + stages * stage_bytes;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(l3_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    attr_set = true;
  }
  const int total = g.m_tiles * g.n_tiles * g.nets;
  int grid = total < num_sms() ? total : num_sms();
  ProfScope prof(RC_STAGE_L3, s);
  l3_kernel<BN><<<grid, GEMM_THREADS, smem, s>>>(A, B, g);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

// layer 3 (+ layer 4 folded into its epilogue)
int launch_l3(int BN, const CUtensorMap &A, const CUtensorMap &B, const GemmArgs &g, cudaStream_t s) {
#define RC_GEMM_CASE(bn) \
  case bn:               \
    return launch_l3_t<bn>(A, B, g, s);
  switch (BN) {
    RC_GEMM_CASE(16)
    RC_GEMM_CASE(32)
    RC_GEMM_CASE(48)
    RC_GEMM_CASE(64)
    RC_GEMM_CASE(96)
    RC_GEMM_CASE(128)
    RC_GEMM_CASE(160)
    RC_GEMM_CASE(208)
    default:
      return rc_fail(RC_EUNSUPPORTED, "no layer-3 GEMM tile for BN=%d", BN);
  }
#undef RC_GEMM_CASE
}

struct WsLayout {
  size_t z, h1, h2, opart, qpart, total;
  int cap;
};

WsLayout ws_layout(const rc_mlp *n, int cap) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  WsLayout L;
  L.cap = cap;
  size_t o = 0;
  L.qpart = o; o = al(o + QPART_BLOCKS * 8);
  L.z = o; o = al(o + (size_t)cap * n->kpad1 * 2);
  L.h1 = o; o = al(o + (size_t)n->n_nets * cap * n->h1 * 2);
  L.h2 = o; o = al(o + (size_t)n->n_nets * cap * n->h2 * 2);
  const int np3 = 4 * n_tiles_of(n->h3);
  L.opart = o; o = al(o + (size_t)n->n_nets * np3 * cap * 4);
  L.total = o;
  return L;
}

uint16_t f2bf(float f) {  // round-to-nearest-even float -> bf16 bits
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)(u >> 16);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

}  // namespace

size_t chem_workspace_bytes(const rc_mech *, const rc_mlp *n, int64_t ncells) {
  int64_t cap = (ncells + 255) / 256 * 256;  // chunks of CTA-pair (256-row) tiles
  if (cap > MAX_CAP) cap = MAX_CAP;
  if (cap < 256) cap = 256;
  return ws_layout(n, (int)cap).total;
}

int mlp_upload(rc_mlp *n, const rc_mlp_desc *d) {
  if (n->precision != RC_BF16) return rc_fail(RC_EUNSUPPORTED, "TF32 MLP variant not built yet");
  if (n->h1 % 64 || !l2_pass_width(n->h2) || !pick_bn(n->h3))
    return rc_fail(RC_EUNSUPPORTED, "hidden widths (%d,%d,%d) not supported by the fused kernels", n->h1, n->h2, n->h3);
  const int nets = n->n_nets, din = n->d_in, h1 = n->h1, h2 = n->h2, h3 = n->h3, kp = n->kpad1;
  const size_t P = (size_t)h1 * din + h1 + (size_t)h2 * h1 + h2 + (size_t)h3 * h2 + h3 + h3 + 1;
  std::vector<uint16_t> W1((size_t)nets * h1 * kp, 0), W2((size_t)nets * h2 * h1), W3((size_t)nets * h3 * h2);
  std::vector<float> b1((size_t)nets * h1), b2((size_t)nets * h2), b3((size_t)nets * h3), w4((size_t)nets * h3), b4(nets);
  for (int i = 0; i < nets; ++i) {
    const double *p = d->params + i * P;
    const double *pb1 = p + (size_t)h1 * din;
    for (int r = 0; r < h1; ++r) {
      // W1 is stored halved (exact in bf16): the layer-1 epilogue evaluates GELU(2y) from y = x/2
      for (int k = 0; k < din; ++k) W1[((size_t)i * h1 + r) * kp + k] = f2bf(0.5f * (float)p[(size_t)r * din + k]);
      // b1 folded into the layer-1 MMA: z carries 1.0 in columns din and din+1
      const uint16_t hi = f2bf(0.5f * (float)pb1[r]);
      uint32_t hb = (uint32_t)hi << 16;
      float hf;
      std::memcpy(&hf, &hb, 4);
      W1[((size_t)i * h1 + r) * kp + din] = hi;
      W1[((size_t)i * h1 + r) * kp + din + 1] = f2bf((float)(0.5 * pb1[r] - (double)hf));
      b1[(size_t)i * h1 + r] = (float)pb1[r];
    }
    p += (size_t)h1 * din + h1;
    for (size_t e = 0; e < (size_t)h2 * h1; ++e) W2[(size_t)i * h2 * h1 + e] = f2bf((float)p[e]);
    p += (size_t)h2 * h1;
    for (int r = 0; r < h2; ++r) b2[(size_t)i * h2 + r] = (float)p[r];
    p += h2;
    for (size_t e = 0; e < (size_t)h3 * h2; ++e) W3[(size_t)i * h3 * h2 + e] = f2bf((float)p[e]);
    p += (size_t)h3 * h2;
    for (int r = 0; r < h3; ++r) b3[(size_t)i * h3 + r] = (float)p[r];
    p += h3;
    for (int r = 0; r < h3; ++r) w4[(size_t)i * h3 + r] = (float)p[r];
    p += h3;
    b4[i] = (float)p[0];
  }
  std::vector<float> xm(din), xi(din);
  for (int k = 0; k < din; ++k) {
    xm[k] = (float)d->x_mean[k];
    xi[k] = (float)(1.0 / d->x_std[k]);
  }
  auto up = [](void **dst, const void *src, size_t bytes) -> bool {
    return cudaMalloc(dst, bytes) == cudaSuccess && cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  bool ok = up(&n->d_W1, W1.data(), W1.size() * 2) && up(&n->d_W2, W2.data(), W2.size() * 2) &&
            up(&n->d_W3, W3.data(), W3.size() * 2) && up((void **)&n->d_b1, b1.data(), b1.size() * 4) &&
            up((void **)&n->d_b2, b2.data(), b2.size() * 4) && up((void **)&n->d_b3, b3.data(), b3.size() * 4) &&
            up((void **)&n->d_w4, w4.data(), w4.size() * 4) && up((void **)&n->d_b4, b4.data(), b4.size() * 4) &&
            up((void **)&n->d_xmean, xm.data(), xm.size() * 4) && up((void **)&n->d_xinvstd, xi.data(), xi.size() * 4) &&
            up((void **)&n->d_ymean, d->y_mean, nets * 8) && up((void **)&n->d_ystd, d->y_std, nets * 8) &&
            up((void **)&n->d_species, d->species_of_net, nets * 4);
  if (!ok) return rc_fail(RC_ENOMEM, "rc_mlp_create: device upload failed");
  return RC_OK;
}

int launch_chem(const rc_mech *m, const rc_mlp *n, const CellsDev &c, void *ws, size_t ws_bytes, cudaStream_t s) {
  if (c.n == 0) return RC_OK;
  // chunk capacity: largest multiple of 128 (<= MAX_CAP, <= n rounded up) whose layout fits the workspace
  int cap = (int)std::min<int64_t>((c.n + 255) / 256 * 256, MAX_CAP);
  while (cap > 256 && ws_layout(n, cap).total > ws_bytes) cap -= 256;
  WsLayout L = ws_layout(n, cap);
  if (L.total > ws_bytes) return rc_fail(RC_EINVAL, "workspace too small (%zu < %zu)", ws_bytes, L.total);
  uint8_t *w = static_cast<uint8_t *>(ws);
  auto *z = reinterpret_cast<__nv_bfloat16 *>(w + L.z);
  auto *h1 = reinterpret_cast<__nv_bfloat16 *>(w + L.h1);
  auto *h2 = reinterpret_cast<__nv_bfloat16 *>(w + L.h2);
  auto *opart = reinterpret_cast<float *>(w + L.opart);
  auto *qpart = reinterpret_cast<double *>(w + L.qpart);
  const int nets = n->n_nets;
  const int bn1 = l1_tile_n(), bn3 = pick_bn(n->h3), NP = l2_pass_width(n->h2), KZ = n->kpad1;
  const int P1 = NP > 256 ? 256 : NP, P2 = NP - P1;
  CUtensorMap mz, mh1, mh1st, mh2, mh2st, mw1, mw2a, mw2b, mw3;
  int rc;
  if ((rc = make_map(&mz, z, KZ, cap, 1, BM, KZ)) || (rc = make_map(&mw1, n->d_W1, KZ, n->h1, nets, l1_box_rows(), KZ)) ||
      (rc = make_map(&mh1, h1, n->h1, cap, nets, BM)) || (rc = make_map(&mh1st, h1, n->h1, cap, nets, 32)) ||
      (rc = make_map(&mw2a, n->d_W2, n->h1, n->h2, nets, P1 / 2)) ||
      (rc = make_map(&mw2b, n->d_W2, n->h1, n->h2, nets, P2 > 0 ? P2 / 2 : P1 / 2)) ||
      (rc = make_map(&mh2, h2, n->h2, cap, nets, BM)) || (rc = make_map(&mh2st, h2, n->h2, cap, nets, 32, 16)) ||
      (rc = make_map(&mw3, n->d_W3, n->h2, n->h3, nets, bn3)))
    return rc;
  RC_CUDA_TRY(cudaMemsetAsync(qpart, 0, QPART_BLOCKS * 8, s));
  int64_t launches = 1;
  for (int64_t c0 = 0; c0 < c.n; c0 += cap) {
    const int rows = (int)std::min<int64_t>(cap, c.n - c0);
    const int mt = (rows + 2 * BM - 1) / (2 * BM) * 2;  // even: CTA pairs of 128-row tiles
    ProArgs pa{c0, rows, mt * BM, n->d_in, n->ns, KZ, (float)n->lambda_bc, (float)(1.0 / n->lambda_bc), n->d_xmean,
               n->d_xinvstd, z};
    {
      ProfScope prof(RC_STAGE_PROLOGUE, s);
      prologue_kernel<<<(mt * BM + 255) / 256, 256, 0, s>>>(pa, c);
      RC_LAUNCH_CHECK();
    }
    // layer 1: h1 = GELU(z W1^T) (b1 folded into z's constant-1 columns)
    L1Args g1{mt, (n->h1 + bn1 - 1) / bn1, nets, n->h1, 0, cap, h1};
    if ((rc = launch_l1(KZ, mz, mw1, mh1st, g1, s))) return rc;
    // layer 2: h2 = GELU(h1 W2^T + b2), CTA-pair GEMM
    L2Args la{mt, n->h2 / NP, nets, n->h1 / 64, n->h2, 0, n->d_b2};
    if ((rc = launch_l2_pair(NP, mh1, mw2a, mw2b, mh2st, la, s))) return rc;
    GemmArgs g3{mt, n_tiles_of(n->h3), nets, (n->h2 + BK - 1) / BK, 0, n->h3, cap, 0, n->d_b3, n->d_w4, opart};
    if ((rc = launch_l3(bn3, mh2, mw3, g3, s))) return rc;
    EpiArgs ea{c0, rows, cap, nets, 4 * n_tiles_of(n->h3), n->inv_lambda, n->ns, n->lambda_bc, 1.0 / n->dt, opart,
               n->d_b4, n->d_ymean, n->d_ystd, m->d_P, m->d_thermo, n->d_species, qpart};
    const size_t esm = (size_t)ThermoSeg::size(m->ns) * 8 + (size_t)((m->ns * m->ns + 1) & ~1) * 8;
    int eblocks = (rows + 255) / 256;
    if (eblocks > QPART_BLOCKS) eblocks = QPART_BLOCKS;
    ProfScope prof(RC_STAGE_EPILOGUE, s);
    if (m->ns == 9)
      chem_epilogue_kernel<9><<<eblocks, 256, esm, s>>>(ea, c);
    else if (m->ns == 20)
      chem_epilogue_kernel<20><<<eblocks, 256, esm, s>>>(ea, c);
    else
      chem_epilogue_kernel<0><<<eblocks, 256, esm, s>>>(ea, c);
    RC_LAUNCH_CHECK();
    launches += 5;
  }
  if (c.red) {
    ProfScope prof(RC_STAGE_FINALIZE, s);
    qdot_finalize_kernel<<<1, 32, 0, s>>>(qpart, QPART_BLOCKS, c.red);
    RC_LAUNCH_CHECK();
  }
  (void)launches;
  return RC_OK;
}
