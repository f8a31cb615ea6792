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
//   l2_pair<dot>  o_part = GELU(h2 W3^T + b3) . w4   (layer 3, layer 4 folded into the epilogue)
//   chem_epilogue o = b4 + sum(o_part) -> dY -> P dY -> wdot, qdot, sum qdot partials
// The GEMMs are persistent warp-specialised tcgen05 kernels (TMA producer warp,
// single-thread MMA issuer, sixteen TMEM-draining epilogue warps); this file
// holds the prologue, the fp64 chem epilogue, the weight upload and the driver.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "mlp_common.cuh"
#include "mlp_internal.h"
#include "ptx.cuh"
#include "rc_internal.h"
#include "stream.cuh"


namespace {

constexpr int BM = 128;       // UMMA M (one CTA, cta_group::1)
// cells per chunk (the activation working set: h2 = 12.8 KB per cell for the paper MLP in bf16 on
// the fused path, 3.4 GB at 262144 cells; the layer-wise path adds h1).  Larger chunks amortise the
// per-chunk launches and persistent-grid tails: 262144 measured +1.5% over 131072 on C2
// (tools/capsweep.sh); 524288 no further gain
// (tools/capsweep.sh varies it through the workspace size: the chunk is the largest that fits)
constexpr int MAX_CAP = 262144;
constexpr int QPART_BLOCKS = 1024;  // q-dot block partials (>= the epilogue's resident grid)


// ------------------------------------------------------------------ prologue (a3)
struct ProArgs {
  int64_t c0;       // first global cell of the chunk
  int rows, rows_pad, d_in, ns, kz;
  float lambda, inv_lambda;
  const float *xmean, *xinvstd;
  void *z;  // [cap][kz] bf16 (or tf32-rounded fp32): z-scored inputs, two 1.0 columns (b1 hi/lo), zeros
  int tf32;         // 0 bf16, 1 tf32, 2 tf32 hi at z and tf32 lo at z + lo_off
  int64_t lo_off;   // elements
  float xm[32], xs[32];  // z-score constants (d_in <= 30) as kernel-parameter (constant-bank) operands
};

// cells per stage = consumer threads (+ the producer warp, stream.cuh run_ws).  256-cell tiles for
// the H2 set (3 CTAs/SM with 3 stages); 128 for larger mechanisms, where a 256-cell stage of 2 + Ns
// fp64 rows (45 KB at Ns = 20) would leave one CTA (8 consumer warps) per SM
template <int TILE> constexpr int pro_threads() { return TILE + 32; }

// one z row (d_in transformed inputs, two 1.0 bias columns, zeros) -> bf16 or tf32 (hi[, lo])
__device__ __forceinline__ void store_z_row(const ProArgs &a, int64_t r, const float (&x)[32]) {
  if (a.tf32) {
    float4 *dst = reinterpret_cast<float4 *>(static_cast<float *>(a.z) + (size_t)r * a.kz);
    float4 *lo = reinterpret_cast<float4 *>(static_cast<float *>(a.z) + a.lo_off + (size_t)r * a.kz);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q * 4 >= a.kz) break;
      const float4 h = make_float4(rcm::tf32_rn(x[4 * q]), rcm::tf32_rn(x[4 * q + 1]), rcm::tf32_rn(x[4 * q + 2]),
                                   rcm::tf32_rn(x[4 * q + 3]));
      dst[q] = h;
      if (a.tf32 == 2)
        lo[q] = make_float4(rcm::tf32_rn(x[4 * q] - h.x), rcm::tf32_rn(x[4 * q + 1] - h.y),
                            rcm::tf32_rn(x[4 * q + 2] - h.z), rcm::tf32_rn(x[4 * q + 3] - h.w));
    }
    return;
  }
  uint4 *dst = reinterpret_cast<uint4 *>(static_cast<__nv_bfloat16 *>(a.z) + (size_t)r * a.kz);
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

// a3 for every cell of the call: T, p, Y streamed through the TMA tile ring (stream.cuh), one
// thread per cell writes its z row; rows [rows, rows_pad) of the 256-row tiles are zero.
// NS > 0: the species count of a compiled mechanism (loops without runtime bounds); 0: generic
template <int PRO_TILE, int NS>
__global__ void __launch_bounds__(pro_threads<PRO_TILE>()) prologue_kernel(const __grid_constant__ ProArgs a, CellsDev c,
                                                                          int stages) {
  constexpr int PRO_THREADS = pro_threads<PRO_TILE>();
  constexpr int CAP = NS ? NS : 30;
  const int ns = NS ? NS : a.ns;
  extern __shared__ __align__(16) uint8_t pro_smem[];
  __shared__ __align__(8) uint64_t bars[16];
  const rcs::Ring<PRO_TILE> ring{pro_smem, bars, 2 + ns, 0, stages};
  if (threadIdx.x == 0) ring.init(PRO_TILE / 32);
  __syncthreads();
  const float *s_xm = a.xm, *s_xs = a.xs;
  auto src8 = [&](int r) -> const double * {
    return (r == 0 ? c.T : r == 1 ? c.p : c.Y + (size_t)(r - 2) * c.ld) + a.c0;
  };
  auto src4 = [&](int) -> const float * { return nullptr; };
  ring.run_ws(a.rows, src8, src4, [&](int st, int64_t tile, int jt) {
    const int64_t r = tile * PRO_TILE + jt;
    if (r >= a.rows) return;
    const double *S8 = ring.row8(st, 0) + jt;  // fp64 row q of this cell: S8[q * PRO_TILE]
    float x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = 0.f;
    x[0] = ((float)S8[0] - s_xm[0]) * s_xs[0];
    x[1] = ((float)S8[PRO_TILE] - s_xm[1]) * s_xs[1];
#pragma unroll
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        float y = (float)S8[(2 + k) * PRO_TILE];
        y = y > 0.f ? y : 0.f;                                       // Y^ = max(Y, 0)
        // Y^^lambda with the MUFU lg2/ex2 (relative error ~1e-7, far below the bf16/tf32 rounding of z);
        // Y^ = 0: lg2 = -inf, ex2(-inf) = 0 (lambda > 0), so no branch
        float l2, b;
        asm("lg2.approx.f32 %0, %1;" : "=f"(l2) : "f"(y));
        asm("ex2.approx.f32 %0, %1;" : "=f"(b) : "f"(a.lambda * l2));
        x[2 + k] = ((b - 1.f) * a.inv_lambda - s_xm[2 + k]) * s_xs[2 + k];  // Box-Cox, z-score
      }
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j == a.d_in || j == a.d_in + 1) x[j] = 1.f;
    store_z_row(a, r, x);
  });
  float x0[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x0[j] = 0.f;
  for (int64_t r = a.rows + (int64_t)blockIdx.x * PRO_THREADS + threadIdx.x; r < a.rows_pad; r += (int64_t)gridDim.x * PRO_THREADS)
    store_z_row(a, r, x0);
}

// ------------------------------------------------------------------ layer 4 of the shared net (NEXT-2)
// RC_MLP_SHARED (R20): o[out][r] = h3[r] . W4[out] for the n_out outputs of the one shared
// net (b4 is added by the epilogue, as for the per-species nets).  h3 = GELU(h2 W3^T + b3) was
// stored by the layer-3 GEMM ([cap][h3], bf16 or tf32-rounded fp32).  CUDA cores (2 h3 n_out FLOP
// per cell is ~1% of the shared net's GEMM work), HBM-bound on the h3 read: one warp per row, lane
// l owning the 8-column chunks l and l + 32 of the row (coalesced 16-byte loads of the contiguous
// row), with its W4 slice (8 outputs x 16 columns) held in registers for all the warp's rows; the
// 8 per-lane partial dots are combined by a 9-shuffle reduce-scatter (lane 4o holds output o).
// Outputs beyond 8 run as further passes of 8.
template <bool TF32> constexpr int l4_warps() { return TF32 ? 2 : 4; }  // per CTA; each streams its own 16-row blocks
constexpr int L4_MAXO = 32;      // outputs (multiple of 8 after padding)

// m16n8k16 bf16 (or m16n8k8 tf32) warp MMA, fp32 accumulate
template <bool TF32>
__device__ __forceinline__ void mma16n8(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (TF32)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  else
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Layer 4 of the shared net on the warp-level tensor-core MMA: o[16 rows][8 outputs] tiles,
// K = h3 in atoms of 16 (bf16) / 8 (tf32).  W4 enters as an exact hi + lo pair of operand-type
// values (two MMAs per atom), so the weights keep fp32 accuracy; h3 is the operand-type value the
// layer-3 GEMM stored.  Each warp double-buffers its own 16-row blocks of h3 (one bulk copy each).
template <bool TF32>
__global__ void __launch_bounds__(32 * l4_warps<TF32>()) l4_kernel(const void *__restrict__ h3, const float *__restrict__ w4,
                                                           float *__restrict__ o, int rows, int h3n, int nout, int cap) {
  constexpr int EB = TF32 ? 4 : 2, KA = TF32 ? 8 : 16, L4_WARPS = l4_warps<TF32>();
  extern __shared__ __align__(128) uint8_t l4s[];
  __shared__ __align__(8) uint64_t full[L4_WARPS][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nt = (nout + 7) / 8;                       // 8-output n tiles
  const uint32_t row_bytes = (uint32_t)h3n * EB, blk = 16 * row_bytes;
  // W4 hi / lo as [n][k] operand values (32-bit words: bf16 pairs or tf32)
  uint32_t *wh = reinterpret_cast<uint32_t *>(l4s);
  const int wwords = nt * 8 * h3n * EB / 4;
  uint32_t *wl = wh + wwords;
  uint8_t *abuf = reinterpret_cast<uint8_t *>(wl + wwords) + warp * 2 * blk;
  for (int e = threadIdx.x; e < nt * 8 * h3n; e += blockDim.x) {
    const int n = e / h3n, k = e % h3n;
    const float w = n < nout ? w4[(size_t)n * h3n + k] : 0.f;
    if constexpr (TF32) {
      const float hi = rcm::tf32_rn(w);
      reinterpret_cast<float *>(wh)[e] = hi;
      reinterpret_cast<float *>(wl)[e] = rcm::tf32_rn(w - hi);
    } else {
      const __nv_bfloat16 hi = __float2bfloat16_rn(w);
      reinterpret_cast<__nv_bfloat16 *>(wh)[e] = hi;
      reinterpret_cast<__nv_bfloat16 *>(wl)[e] = __float2bfloat16_rn(w - __bfloat162float(hi));
    }
  }
  if (lane == 0) {
    rcx::mbar_init(&full[warp][0], 1);
    rcx::mbar_init(&full[warp][1], 1);
    rcx::fence_mbar_init();
  }
  __syncthreads();
  const int nblk = (rows + 15) / 16, wstride = gridDim.x * L4_WARPS;
  auto issue = [&](int b, int slot) {
    const int nr = rows - b * 16 < 16 ? rows - b * 16 : 16;
    rcx::mbar_arrive_expect_tx(&full[warp][slot], nr * row_bytes);
    rcx::bulk_g2s(abuf + slot * blk, static_cast<const uint8_t *>(h3) + (size_t)b * blk, nr * row_bytes, &full[warp][slot]);
  };
  int it = 0;
  const int b0 = blockIdx.x * L4_WARPS + warp;
  if (lane == 0 && b0 < nblk) issue(b0, 0);
  for (int b = b0; b < nblk; b += wstride, ++it) {
    const int slot = it & 1;
    if (lane == 0 && b + wstride < nblk) issue(b + wstride, slot ^ 1);  // the other buffer is free (read last round)
    rcx::mbar_wait(&full[warp][slot], (uint32_t)(it >> 1) & 1u);
    const uint8_t *A = abuf + slot * blk;
    const int nr = rows - b * 16 < 16 ? rows - b * 16 : 16;
    for (int n0 = 0; n0 < nt; ++n0) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f}, acl[4] = {0.f, 0.f, 0.f, 0.f};  // hi and lo chains
      for (int k0 = 0; k0 < h3n; k0 += KA) {
        uint32_t af[4];
        // A fragment (row-major 16 x KA): a0 (g, c), a1 (g + 8, c), a2 (g, c + KA/2), a3 (g + 8, c + KA/2)
        const int c = TF32 ? k0 + t : k0 + 2 * t;
        const int ga = g < nr ? g : 0, gb = g + 8 < nr ? g + 8 : 0;  // rows past the block end: any valid row
        af[0] = *reinterpret_cast<const uint32_t *>(A + ga * row_bytes + c * EB);
        af[1] = *reinterpret_cast<const uint32_t *>(A + gb * row_bytes + c * EB);
        af[2] = *reinterpret_cast<const uint32_t *>(A + ga * row_bytes + (c + KA / 2) * EB);
        af[3] = *reinterpret_cast<const uint32_t *>(A + gb * row_bytes + (c + KA / 2) * EB);
        // B fragment (col-major KA x 8 = W4 [n][k]): b0 (k = c, n = g), b1 (k = c + KA/2, n = g)
        const int wi = ((n0 * 8 + g) * h3n + c) * EB / 4, wj = ((n0 * 8 + g) * h3n + c + KA / 2) * EB / 4;
        mma16n8<TF32>(acc, af, wh[wi], wh[wj]);
        mma16n8<TF32>(acl, af, wl[wi], wl[wj]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] += acl[e];
      // D fragment: d0, d1 (row g, outputs 2t, 2t+1), d2, d3 (row g + 8)
      const int r0 = b * 16 + g, r1 = r0 + 8, q0 = n0 * 8 + 2 * t;
      if (g < nr) {
        if (q0 < nout) o[(size_t)q0 * cap + r0] = acc[0];
        if (q0 + 1 < nout) o[(size_t)(q0 + 1) * cap + r0] = acc[1];
      }
      if (g + 8 < nr) {
        if (q0 < nout) o[(size_t)q0 * cap + r1] = acc[2];
        if (q0 + 1 < nout) o[(size_t)(q0 + 1) * cap + r1] = acc[3];
      }
    }
    __syncwarp();  // every lane has read this buffer before it is refilled (two rounds later)
  }
}

// ------------------------------------------------------------------ epilogue (a5)
struct EpiArgs {
  int64_t c0;
  int rows, cap, n_nets, passes, inv_lambda, ns;
  double lambda, inv_dt;
  const float *opart, *b4;     // raw net outputs [nets][passes][cap] (column quarters summed by layer 3)
  const double *ymean, *ystd, *P, *thermo;
  const int *species;
  const double *EF;  // [2][ne][ns]: F = (E E^T)^-1 E, then E (the factored P = I - E^T F)
  int ne;
  double *qpart;  // [gridDim.x], accumulated across chunks in stream order
  double binom[17];  // C(n, m), m = 0..n, n = inv_lambda <= 16 (factorised inverse Box-Cox)
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

// Inverse Box-Cox increment: dY = Y* - Y^ with Y* = a^n,
// a = b + lambda Delta, b = Y^^lambda, n = 1/lambda.  In exact arithmetic
// dY = Y^ ((1 + u)^n - 1) with u = lambda Delta / b (and Y* = 0, dY = -Y^ when a <= 0, i.e.
// u <= -1), and (1 + u)^n - 1 = sum_{m=1..n} C(n, m) u^m by Horner: the relative error of dY
// is that of u, i.e. of b, with no cancellation between Y* and Y^ (the "factorised" dY of
// SURVEY.md §8(a) a5).  1/b = Y^^(-lambda): fp32 MUFU seed (~1e-7) + one division-free fp64
// Newton step on Y^ r^n = 1 (error x (n+1)/2 squared: ~5e-14).  Tiny Y^ (fp32 seed out of range) and a
// non-integer or large 1/lambda take the direct pow() form.
// the general form: Y^ = 0 (b = 0), Y^ below the fp32 seed's range, or 1/lambda not 10
__device__ __noinline__ double inv_boxcox_dy_general(double ys, double delta, const EpiArgs &a) {
  const int n = a.inv_lambda;
  const double ld = a.lambda * delta;
  if (!(ys > 0.0)) return ld > 0.0 ? (n > 0 ? ipow(ld, n) : pow(ld, 1.0 / a.lambda)) : 0.0;  // b = 0
  if (n <= 0 || n > 16 || ys < 1e-30) {
    const double b = pow(ys, a.lambda), ap = b + ld;
    return (ap > 0.0 ? pow(ap, 1.0 / a.lambda) : 0.0) - ys;
  }
  double b = (double)exp2f((float)a.lambda * log2f((float)ys));
  b = fma(ys * rcx::rcp_f64(ipow(b, n - 1)) - b, a.lambda, b);
  const double u = ld * rcx::rcp_f64(b);
  if (u <= -1.0) return -ys;
  double g = 0.0;
  for (int m = n; m >= 1; --m) g = fma(g, u, a.binom[m]);
  return ys * (g * u);
}

// lambda_BC = 0.1 (R3, n = 10) with Y^ >= 1e-30: MUFU seed, one Newton step, 9-FMA Horner
__device__ __forceinline__ double inv_boxcox_dy(double ys, double delta, const EpiArgs &a) {
  if (a.inv_lambda != 10 || !(ys >= 1e-30)) return inv_boxcox_dy_general(ys, delta, a);
  // r = 1/b = Y^^(-lambda): MUFU seed, then one Newton step on Y^ r^10 = 1 (no division:
  // r <- r + r (1 - Y^ r^10) / 10), relative error ~(11/2) 1e-14; u = lambda Delta r
  float l2, e2;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"((float)ys));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e2) : "f"(-0.1f * l2));
  double r = (double)e2;
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  r = fma(0.1 * r, fma(-ys, r8 * r2, 1.0), r);
  const double u = (a.lambda * delta) * r;
  constexpr double C10[10] = {10.0, 45.0, 120.0, 210.0, 252.0, 210.0, 120.0, 45.0, 10.0, 1.0};
  double g = C10[9];
#pragma unroll
  for (int m = 8; m >= 0; --m) g = fma(g, u, C10[m]);
  return u <= -1.0 ? -ys : ys * (g * u);
}

// the factored path's per-mechanism constants as a kernel parameter: with the species loops unrolled
// each is a compile-time offset into the constant bank, a DFMA operand with no shared-memory load
constexpr int EPI_KN = 20, EPI_KE = 4;
struct EpiConst {
  double F[EPI_KE][EPI_KN];  // F = (E E^T)^-1 E, column of net i's species (= i)
  double E[EPI_KE][EPI_KN];  // E, column k
  double ym[EPI_KN], ys[EPI_KN];
  float b4[EPI_KN];
};

// inverse Box-Cox increment with lambda = 1/10 for Y^ >= 1e-30 (the fast branch of inv_boxcox_dy,
// checked once per cell by the caller)
__device__ __forceinline__ double inv_boxcox_dy10(double ys, double delta, double lambda) {
  float l2, e2;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"((float)ys));
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e2) : "f"(-0.1f * l2));
  double r = (double)e2;
  const double r2 = r * r, r4 = r2 * r2, r8 = r4 * r4;
  r = fma(0.1 * r, fma(-ys, r8 * r2, 1.0), r);
  const double u = (lambda * delta) * r;
  constexpr double C10[10] = {10.0, 45.0, 120.0, 210.0, 252.0, 210.0, 120.0, 45.0, 10.0, 1.0};
  double g = C10[9];
#pragma unroll
  for (int m = 8; m >= 0; --m) g = fma(g, u, C10[m]);
  return u <= -1.0 ? -ys : ys * (g * u);
}

__device__ __forceinline__ double2 lds2_epi(const double *p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(rcx::smem_u32(p)));
  return v;
}

// cells per stage = consumer threads (+ the producer warp, stream.cuh run_ws): 256 (two CTAs of
// eight consumer warps per SM) unless the Ns = 20 register/shared footprint needs 128
template <int NS> constexpr int epi_tile() { return NS == 20 ? 128 : 256; }
// Ns = 20: two stages (one tile in flight per CTA while one is computed) and three CTAs per SM: the
// per-cell chain (19 inverse transforms) is latency-bound at the two CTAs three stages allow
template <int NS> constexpr int epi_stages() { return NS == 20 ? 2 : 3; }
template <int NS> constexpr int epi_min_ctas() { return NS == 0 ? 1 : NS == 20 ? 3 : 2; }

// NE > 0: net `net` predicts species `net` for the first Ns - 1 species (the inert species last),
// layer 3 ran in one pass (h3 = 400, the paper width), 1/lambda = 10, the mechanism has one T_mid and
// NE elements (all checked at launch); the projection is then applied in factored form, v = dY - E^T (F dY), with F dY
// accumulated per net (NE FMAs instead of Ns) and dY kept in registers (the net loop is fully
// unrolled, so dY_net has a static register).  NE == 0: the outer product with the columns of P.
template <int NS, int NE>
__global__ void __launch_bounds__(epi_tile<NS>() + 32, epi_min_ctas<NS>())
    chem_epilogue_kernel(EpiArgs a, CellsDev c, int stages, const __grid_constant__ EpiConst K) {
  constexpr int EPI_TILE = epi_tile<NS>(), EPI_THREADS = EPI_TILE + 32;
  constexpr int CAP = NS ? NS : RC_MAX_NS;
  constexpr int UR = NS ? NS : 1;
  constexpr int NETUNR = 2;  // partial unroll: the fully unrolled net loop overflowed the instruction cache
  const int ns = NS ? NS : a.ns;
  const int nn = a.n_nets;
  extern __shared__ __align__(16) double s_tab[];  // thermo segment | P | P columns by net | species | ring
  __shared__ __align__(8) uint64_t bars[1 + 16];
  __shared__ double red_s[EPI_THREADS / 32];
  const int nse = (ns + 1) & ~1;
  // P columns by net [nn][nse] | species [32 ints] | b4, y_mean, y_std [nn] each (no global loads per cell)
  // NE > 0: [nn][NE] F columns by net, then [ns][NE] E columns, in the Pn slot
  const int tsz = ThermoSeg::size(ns), psz = (ns * ns + 1) & ~1,
            pnsz = (NE ? ((nn + ns) * NE + 1) & ~1 : nn * nse) + 16 + ((3 * nn + 1) & ~1);
  double *sP = s_tab + tsz, *sPn = sP + psz;
  const int pnt = NE ? ((nn + ns) * NE + 1) & ~1 : nn * nse;
  int *sSpec = reinterpret_cast<int *>(sPn + pnt);
  double *sB4 = sPn + pnt + 16, *sYM = sB4 + nn, *sYS = sYM + nn;
  const rcs::Ring<EPI_TILE, epi_stages<NS>()> ring{reinterpret_cast<uint8_t *>(sPn + pnsz), bars + 1, 2 + ns, nn * a.passes, stages};
  if (threadIdx.x == 0) {
    rcx::mbar_init(&bars[0], 1);
    ring.init(EPI_TILE / 32);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    rcx::mbar_arrive_expect_tx(&bars[0], (uint32_t)(tsz + psz) * 8u);
    rcx::bulk_g2s(s_tab, a.thermo, (uint32_t)tsz * 8u, &bars[0]);
    rcx::bulk_g2s(sP, a.P, (uint32_t)psz * 8u, &bars[0]);
  }
  // stage rows: fp64 T, rho, Y_0..Y_{ns-1} of the chunk's cells; fp32 raw outputs per (net, pass)
  auto src8 = [&](int r) -> const double * {
    return (r == 0 ? c.T : r == 1 ? c.rho : c.Y + (size_t)(r - 2) * c.ld) + a.c0;
  };
  auto src4 = [&](int r) -> const float * { return a.opart + (size_t)r * a.cap; };
  rcx::mbar_wait(&bars[0], 0);
  const double *hlo = s_tab + ThermoSeg::hlo(ns), *hhi = s_tab + ThermoSeg::hhi(ns), *tmid = s_tab + ThermoSeg::tmid(ns);
  const double *invW = s_tab + ThermoSeg::invW(ns);
  // the columns of P gathered by net and stored contiguously: Pn[net][k] = P[k][species[net]]
  // (the other columns multiply dY = 0), padded to an even length for 16-byte loads
  if constexpr (NE > 0) {
    for (int e = threadIdx.x; e < (nn + ns) * NE; e += blockDim.x) {
      const int r = e / NE, q = e % NE;  // r < nn: F column of net r's species (= r); else E column r - nn
      sPn[e] = r < nn ? a.EF[q * ns + r] : a.EF[(NE + q) * ns + (r - nn)];
    }
  } else {
    for (int e = threadIdx.x; e < nn * nse; e += blockDim.x) {
      const int net = e / nse, k = e % nse;
      sPn[e] = k < ns ? sP[k * ns + a.species[net]] : 0.0;
    }
  }
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    sSpec[e] = a.species[e];
    reinterpret_cast<float *>(sB4)[e] = a.b4[e];  // fp32, as the net output it is added to
    sYM[e] = a.ymean[e];
    sYS[e] = a.ystd[e];
  }
  __syncthreads();

  double qsum = 0.0;
  int n_negout = 0, n_bad = 0;
  ring.run_ws(a.rows, src8, src4, [&](int st, int64_t tile, int jt) {
    const int r = (int)(tile * EPI_TILE) + jt;
    if (r >= a.rows) return;
    const int64_t i = a.c0 + r;
    const double *S8 = ring.row8(st, 0) + jt;  // fp64 row q of this cell: S8[q * EPI_TILE]
    const float *S4 = ring.row4(st, 0) + jt;
    const double T = S8[0], rho = S8[EPI_TILE];
    // net loop: dY of net's species (inverse Box-Cox), accumulated straight into the projection
    // v = P dY as an outer product with column `species[net]` of P (species without a net
    // contribute 0); the loop stays rolled for large mechanisms (instruction-cache footprint)
    auto net_out = [&](int net) {  // raw output o of the net (layer 3's passes summed), b4 added
      float o = reinterpret_cast<const float *>(sB4)[net] + S4[net * a.passes * EPI_TILE];
#pragma unroll 1
      for (int ps = 1; ps < a.passes; ++ps) o += S4[(net * a.passes + ps) * EPI_TILE];
      if (c.o) c.o[net * c.ld + i] = o;
      return o;
    };
    double v[CAP];
    if constexpr (NE > 0) {
      // 1/lambda = 10 (checked at launch): Y^ >= 1e-30 takes the check-free inverse transform, a
      // smaller or zero Y^ the general one (per net: zero mass fractions are common in the air
      // and fuel streams); the constants come from K
      // nets = species - 1, the inert species last (checked at launch): no runtime net bound
      constexpr int NN = NE > 0 ? CAP - 1 : 0;
#pragma unroll
      for (int net = 0; net < CAP; ++net) {
        v[net] = 0.0;
        if (net < NN) {  // one layer-3 pass (checked at launch)
          const float o = K.b4[net] + S4[net * EPI_TILE];
          const double y = S8[(2 + net) * EPI_TILE], delta = (double)o * K.ys[net] + K.ym[net];
          if (y >= 1e-30) {
            v[net] = inv_boxcox_dy10(y, delta, a.lambda);
          } else if (!(y > 0.0)) {  // Y^ = 0 (b = 0): dY = (lambda Delta)^10 if positive (as the general form)
            const double l = a.lambda * delta, l2 = l * l, l4 = l2 * l2;
            v[net] = l > 0.0 ? l2 * (l4 * l4) : 0.0;
          } else {
            v[net] = inv_boxcox_dy_general(y, delta, a);
          }
        }
      }
      if (c.o) {  // the raw net outputs (a diagnostic output), outside the net loop
        float *op = c.o + i;
#pragma unroll
        for (int net = 0; net < NN; ++net, op += c.ld) *op = K.b4[net] + S4[net * EPI_TILE];
      }
      double w[NE];
#pragma unroll
      for (int e = 0; e < NE; ++e) {  // F dY
        w[e] = 0.0;
#pragma unroll
        for (int net = 0; net < NN; ++net) w[e] = fma(K.F[e][net], v[net], w[e]);
      }
#pragma unroll
      for (int k = 0; k < CAP; ++k) {  // v = dY - E^T (F dY)
        double t = 0.0;
#pragma unroll
        for (int e = 0; e < NE; ++e) t = fma(K.E[e][k], w[e], t);
        v[k] -= t;
      }
    } else {
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k < ns) v[k] = 0.0;
#pragma unroll NETUNR
      for (int net = 0; net < nn; ++net) {
        const float o = net_out(net);
        const double y = S8[(2 + sSpec[net]) * EPI_TILE];
        const double dy = inv_boxcox_dy(y > 0.0 ? y : 0.0, (double)o * sYS[net] + sYM[net], a);
        const double *pc = sPn + net * nse;  // column species[net] of P, contiguous in k
#pragma unroll UR
        for (int k = 0; k < CAP; k += 2)
          if (k < ns) {
            const double2 pp = lds2_epi(pc + k);
            v[k] = fma(pp.x, dy, v[k]);
            if (k + 1 < ns) v[k + 1] = fma(pp.y, dy, v[k + 1]);
          }
      }
    }
    // sources; LES: PaSR factor kappa = tau_c / (tau_c + tau_mix) = 1 / (1 + tau_mix / tau_c) with
    // 1 / tau_c = (1/2 sum_k |wdot_k| / W_k) / sum_k C+_k (rc.h tau_mix, R19)
    double scale = rho * a.inv_dt;
    if (c.tau_mix) {
      double act = 0.0, conc = 0.0;
#pragma unroll UR
      for (int k = 0; k < CAP; ++k)
        if (k < ns) {
          const double y = S8[(2 + k) * EPI_TILE];
          act = fma(fabs(v[k]), invW[k], act);
          conc = fma(y > 0.0 ? y : 0.0, invW[k], conc);
        }
      // 1/tau_c = (rho/dt) (1/2) act / (rho conc); kappa = 1 when nothing reacts
      const double r = act > 0.0 ? 0.5 * act * a.inv_dt / conc : 0.0;
      scale *= rcx::rcp_f64(fma(c.tau_mix[i], r, 1.0));
    }
    double q = 0.0;
    bool neg = false, bad = false;
    double *wp = c.wdot + i;
#pragma unroll UR
    for (int k = 0; k < CAP; ++k)
      if (k < ns) {
        const double y = S8[(2 + k) * EPI_TILE];
        neg |= ((y > 0.0 ? y : 0.0) + v[k]) < 0.0;
        const double w = scale * v[k];
        *wp = w;
        wp += c.ld;
        // NE > 0 runs only for a mechanism with one T_mid (checked at launch): one range per cell
        const double *h = NE > 0 ? (T <= s_tab[2] ? hlo : hhi) + 6 * k : (T <= tmid[k]) ? hlo + 6 * k : hhi + 6 * k;
        const double hk = fma(T, fma(T, fma(T, fma(T, fma(T, h[4], h[3]), h[2]), h[1]), h[0]), h[5]);
        q = fma(-hk, w, q);
        // (NE > 0: a non-finite w_k makes q non-finite -- inf or NaN times the finite h_k, or NaN
        // from 0 x inf -- so the test of q below counts the cell)
        if constexpr (NE == 0) bad |= !isfinite(w);
      }
    if (c.qdot) c.qdot[i] = q;
    bad |= !isfinite(q);
    qsum += q;
    n_negout += neg;
    n_bad += bad;
  });
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

// step a6 over k sub-batch reductions (rc_combine_reductions): one thread, index order
__global__ void combine_reductions_kernel(const double *rp, const int64_t *dp, int k, double *red, int64_t *diag) {
  double mx = 0.0, S = 0.0, C = 0.0;
  for (int i = 0; i < k; ++i) {
    mx = fmax(mx, rp[2 * i]);
    const double v = rp[2 * i + 1], t = S + v;
    C += (fabs(S) >= fabs(v)) ? (S - t) + v : (v - t) + S;
    S = t;
  }
  red[0] = mx;
  red[1] = S + C;
  if (diag && dp)
    for (int j = 0; j < RC_DIAG_COUNT; ++j) {
      int64_t a = 0;
      for (int i = 0; i < k; ++i) a += dp[i * RC_DIAG_COUNT + j];
      diag[j] = a;
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

// 3D map over [d2][d1][d0] (d0 contiguous) of bf16 (esize 2) or fp32 (esize 4) elements,
// box {box0, box1, 1}; the swizzle width equals the box row (box0 * esize bytes: 32, 64 or 128)
int make_map(CUtensorMap *m, const void *base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t box1, uint32_t box0,
             int esize) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return rc_fail(RC_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * esize, d0 * d1 * esize};
  cuuint32_t box[3] = {box0, box1, 1};
  const uint32_t rowb = box0 * esize;
  const CUtensorMapSwizzle sw = rowb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : rowb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                   const_cast<void *>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return rc_fail(RC_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return RC_OK;
}

// W1 [nets][h1][KZ] bf16 as 5D {KZ, 32 rows, 4 groups, h1/128 chunk pairs, nets}: row
// 128 cp + 32 q4 + i.  One box at q4 = 2 pair + rank = the 32 rows a CTA of the fused
// layer-1/2 cluster needs of each of its pair's chunks (c = 2 cp + pair).  The last chunk
// pair may reach 64 rows past the net (zero-padded after the last net, see mlp_upload).
int make_map_w1_groups(CUtensorMap *m, const void *W1, int KZ, int h1, int nets) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return rc_fail(RC_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t row = (cuuint64_t)KZ * 2;
  const cuuint64_t cps = (cuuint64_t)(h1 / 64 + 1) / 2;
  cuuint64_t dims[5] = {(cuuint64_t)KZ, 32, 4, cps, (cuuint64_t)nets};
  cuuint64_t strides[4] = {row, 32 * row, 128 * row, (cuuint64_t)h1 * row};
  cuuint32_t box[5] = {(cuuint32_t)KZ, 32, 1, (cuuint32_t)cps, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const CUtensorMapSwizzle sw = KZ * 2 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void *>(W1), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return rc_fail(RC_ECUDA, "cuTensorMapEncodeTiled (W1 groups) failed (%d)", (int)r);
  return RC_OK;
}

}  // namespace
int mlp_num_sms() { return rc_sm_count(); }
namespace {

struct WsLayout {
  size_t z, h1, h2, h2b, h3, opart, qpart, sched, total;
  int cap;
  int64_t nchunks;
};

// z (the layer-1 A operand) is held for all `ncells` cells (one prologue launch per call; 32 B per
// cell in bf16), the activations and partial outputs for one chunk of `cap` cells
// the fused layer-1/2 kernel runs (bf16, widths it holds, not RC_MLP_LAYERWISE): no h1 buffer
bool fused_path(const rc_mlp *n) {
  return (n->precision == RC_BF16 || n->precision == RC_TF32) &&
         l12_supported(n->h1, n->h2, n->kpad1, n->precision == RC_TF32) && !(n->flags & RC_MLP_LAYERWISE);
}
// layer 3 of chunk j - 1 overlapped with the fused layer-1/2 kernel of chunk j: a
// second h2 buffer and per-chunk tile counters; RC_MLP_SERIAL keeps the one-stream order.  The
// shared net's layer 4 follows both layer-3 launches of its chunk on the caller's stream.
bool overlap_path(const rc_mlp *n) {
  return fused_path(n) && !(n->flags & RC_MLP_SERIAL);
}

WsLayout ws_layout(const rc_mlp *n, int cap, int64_t ncells) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  WsLayout L;
  L.cap = cap;
  size_t o = 0;
  L.qpart = o; o = al(o + QPART_BLOCKS * 8);
  // activation element bytes (RC_TF32X3 keeps a tf32 hi and a tf32 lo array of each)
  const size_t eb = n->precision == RC_BF16 ? 2 : 4, nc = n->precision == RC_TF32X3 ? 2 : 1;
  const size_t zrows = (size_t)((ncells + 255) / 256 * 256);
  L.z = o; o = al(o + nc * zrows * n->kpad1 * eb);
  L.h1 = o; o = al(o + (fused_path(n) ? 0 : nc * (size_t)n->gnets * cap * n->h1 * eb));
  L.h2 = o; o = al(o + nc * (size_t)n->gnets * cap * n->h2 * eb);
  L.nchunks = (ncells + cap - 1) / cap;
  const bool ov = overlap_path(n) && L.nchunks >= 2;
  L.h2b = o; o = al(o + (ov ? (size_t)n->gnets * cap * n->h2 * eb : 0));  // h2 of the odd chunks
  L.sched = o; o = al(o + (ov ? (size_t)L.nchunks * 2 * 4 : 0));         // tile counters, cluster counts
  const bool shared = (n->flags & RC_MLP_SHARED) != 0;
  L.h3 = o; o = al(o + (shared ? (size_t)cap * n->h3 * eb : 0));  // shared net: h3 for the layer-4 kernel
  const int np3 = shared ? 1 : n->h3 / l2_pass_width(n->h3);  // raw outputs per row: one per layer-3 pass
  // raw outputs of EVERY cell of the call (like z): the chemistry epilogue runs once over all cells
  L.opart = o; o = al(o + (size_t)n->n_nets * np3 * zrows * 4);
  L.total = o;
  return L;
}

float f2tf32(float f) {  // round-to-nearest (ties away, as cvt.rna.tf32.f32) float -> tf32 value
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & ~0x1FFFu;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

uint16_t f2bf(float f) {  // round-to-nearest-even float -> bf16 bits
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)(u >> 16);
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

}  // namespace

int launch_qdot_finalize(const double *qpart, int n, double *red, cudaStream_t s) {
  ProfScope prof(RC_STAGE_FINALIZE, s);
  qdot_finalize_kernel<<<1, 32, 0, s>>>(qpart, n, red);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

int launch_combine_reductions(const double *rp, const int64_t *dp, int k, double *red, int64_t *diag, cudaStream_t s) {
  ProfScope prof(RC_STAGE_FINALIZE, s);
  combine_reductions_kernel<<<1, 1, 0, s>>>(rp, dp, k, red, diag);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

// The auxiliary stream of the layer-3 overlap and its events, one set per host thread (a thread
// enqueues its calls in order, so reusing them across calls never orders one call after a record of
// another): `go` marks the point where the fused kernel of chunk j is enqueued, fill[j % 2] the end of
// chunk j's filler launch.
struct AuxStreams {
  cudaStream_t s2 = nullptr;
  cudaEvent_t go = nullptr, fill[2] = {nullptr, nullptr};
};
constexpr int AUX_MAX_DEVICES = 64;
// one set per (host thread, device), created on first use and kept for the thread's lifetime (a
// thread that alternates between devices reuses each device's set)
AuxStreams *aux_streams() {
  thread_local AuxStreams per_dev[AUX_MAX_DEVICES];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= AUX_MAX_DEVICES) return nullptr;
  AuxStreams &a = per_dev[dev];
  if (!a.s2) {
    AuxStreams b;
    if (cudaStreamCreateWithFlags(&b.s2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&b.go, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&b.fill[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&b.fill[1], cudaEventDisableTiming) != cudaSuccess)
      return nullptr;
    a = b;
  }
  return &a;
}

int cap_limit(const rc_mlp *n) { return n->precision == RC_TF32X3 ? std::min(MAX_CAP, 32768) : MAX_CAP; }

size_t chem_workspace_min_bytes(const rc_mlp *n, int64_t ncells) { return ws_layout(n, 256, ncells).total; }

// chunk capacity for a call of ncells cells: chunks of CTA-pair (256-row) tiles, at most cap_limit;
// with the layer-3 overlap a call that would be one chunk runs as two halves (from OVERLAP_SPLIT_MIN
// cells), so layer 3 of the first half runs beside the fused kernel of the second
constexpr int64_t OVERLAP_SPLIT_MIN = 65536;
int chunk_cap(const rc_mlp *n, int64_t ncells) {
  int64_t cap = (ncells + 255) / 256 * 256;
  if (cap > cap_limit(n)) cap = cap_limit(n);
  if (overlap_path(n) && ncells >= OVERLAP_SPLIT_MIN && ncells <= cap) cap = ((ncells + 1) / 2 + 255) / 256 * 256;
  if (cap < 256) cap = 256;
  return (int)cap;
}

size_t chem_workspace_bytes(const rc_mech *, const rc_mlp *n, int64_t ncells) {
  return ws_layout(n, chunk_cap(n, ncells), ncells).total;
}

int mlp_upload(rc_mlp *n, const rc_mlp_desc *d) {
  if (n->h1 % 64 || !l2_pass_width(n->h2) || !l2_pass_width(n->h3))
    return rc_fail(RC_EUNSUPPORTED, "hidden widths (%d,%d,%d) not supported by the MLP kernels", n->h1, n->h2, n->h3);
  const bool tf32 = n->precision != RC_BF16, x3 = n->precision == RC_TF32X3;
  // hidden layers: one block per GEMM net (shared: one); output layer: one row per output
  const int nets = n->gnets, nout = n->n_nets, din = n->d_in, h1 = n->h1, h2 = n->h2, h3 = n->h3, kp = n->kpad1;
  const bool shared = (n->flags & RC_MLP_SHARED) != 0;
  const size_t P = (size_t)h1 * din + h1 + (size_t)h2 * h1 + h2 + (size_t)h3 * h2 + h3 + (shared ? (size_t)nout : 1) * (h3 + 1);
  // weights, K-major [net][out][in]: bf16 (RNE) or tf32-rounded fp32
  // W1 gets 64 zero rows after the last net: the fused layer-1/2 kernel's W1 box of the last
  // chunk pair can reach past the last net when h1 / 64 is odd
  std::vector<uint16_t> W1((size_t)nets * h1 * kp + 64 * (size_t)kp, 0), W2((size_t)nets * h2 * h1),
      W3((size_t)nets * h3 * h2);
  std::vector<float> F1, F2, F3;
  std::vector<float> L1v, L2v, L3v;  // RC_TF32X3: tf32 residuals W - W_hi
  if (tf32) {
    F1.assign((size_t)nets * h1 * kp, 0.f);
    F2.resize((size_t)nets * h2 * h1);
    F3.resize((size_t)nets * h3 * h2);
  }
  if (x3) {
    L1v.assign((size_t)nets * h1 * kp, 0.f);
    L2v.resize((size_t)nets * h2 * h1);
    L3v.resize((size_t)nets * h3 * h2);
  }
  auto split = [&](double w, float &hi, float *lo) {  // hi = tf32(w); lo = tf32(w - hi) (X3 only)
    hi = f2tf32((float)w);
    if (lo) *lo = f2tf32((float)(w - (double)hi));
  };
  // b2, b3 as an extra K = 16 operand of the layer-2/3 MMAs (the A side is a tile of ones):
  // column 0 = bf16(b), column 1 = bf16(b - bf16(b)), so the accumulator starts at b to ~2^-17
  std::vector<uint16_t> B2k(tf32 ? 0 : (size_t)nets * h2 * 16, 0), B3k(tf32 ? 0 : (size_t)nets * h3 * 16, 0);
  // TF32 (fused layer-1/2 kernel): b2 as a K = 8 tf32 operand, (tf32(b), tf32(b - tf32(b)), 0...)
  std::vector<float> B2f(tf32 && !x3 ? (size_t)nets * h2 * 8 : 0, 0.f);
  auto bias_operand = [](double b, uint16_t *row) {
    const uint16_t hi = f2bf((float)b);
    uint32_t hb = (uint32_t)hi << 16;
    float hf;
    std::memcpy(&hf, &hb, 4);
    row[0] = hi;
    row[1] = f2bf((float)(b - (double)hf));
  };
  std::vector<float> b1((size_t)nets * h1), b2((size_t)nets * h2), b3((size_t)nets * h3), w4((size_t)nout * h3), b4(nout);
  for (int i = 0; i < nets; ++i) {
    const double *p = d->params + i * P;
    const double *pb1 = p + (size_t)h1 * din;
    for (int r = 0; r < h1; ++r) {
      const size_t row = ((size_t)i * h1 + r) * kp;
      if (tf32) {
        for (int k = 0; k < din; ++k) split(p[(size_t)r * din + k], F1[row + k], x3 ? &L1v[row + k] : nullptr);
        // b1 folded into the layer-1 MMA as tf32 hi + lo parts (z carries 1.0 in columns din, din+1);
        // X3 also keeps the residual of the lo part
        const float hi = f2tf32((float)pb1[r]);
        F1[row + din] = hi;
        split(pb1[r] - (double)hi, F1[row + din + 1], x3 ? &L1v[row + din + 1] : nullptr);
      } else {
        // W1 is stored halved (exact in bf16): the layer-1 epilogue evaluates GELU(2y) from y = x/2
        for (int k = 0; k < din; ++k) W1[row + k] = f2bf(0.5f * (float)p[(size_t)r * din + k]);
        // b1 folded into the layer-1 MMA: z carries 1.0 in columns din and din+1
        const uint16_t hi = f2bf(0.5f * (float)pb1[r]);
        uint32_t hb = (uint32_t)hi << 16;
        float hf;
        std::memcpy(&hf, &hb, 4);
        W1[row + din] = hi;
        W1[row + din + 1] = f2bf((float)(0.5 * pb1[r] - (double)hf));
      }
      b1[(size_t)i * h1 + r] = (float)pb1[r];
    }
    p += (size_t)h1 * din + h1;
    for (size_t e = 0; e < (size_t)h2 * h1; ++e) {
      if (tf32) split(p[e], F2[(size_t)i * h2 * h1 + e], x3 ? &L2v[(size_t)i * h2 * h1 + e] : nullptr);
      else W2[(size_t)i * h2 * h1 + e] = f2bf((float)p[e]);
    }
    p += (size_t)h2 * h1;
    for (int r = 0; r < h2; ++r) {
      b2[(size_t)i * h2 + r] = (float)p[r];
      if (!tf32) bias_operand(p[r], &B2k[((size_t)i * h2 + r) * 16]);
      if (tf32 && !x3) {
        const float hi = f2tf32((float)p[r]);
        B2f[((size_t)i * h2 + r) * 8] = hi;
        B2f[((size_t)i * h2 + r) * 8 + 1] = f2tf32((float)(p[r] - (double)hi));
      }
    }
    p += h2;
    for (size_t e = 0; e < (size_t)h3 * h2; ++e) {
      if (tf32) split(p[e], F3[(size_t)i * h3 * h2 + e], x3 ? &L3v[(size_t)i * h3 * h2 + e] : nullptr);
      else W3[(size_t)i * h3 * h2 + e] = f2bf((float)p[e]);
    }
    p += (size_t)h3 * h2;
    for (int r = 0; r < h3; ++r) {
      b3[(size_t)i * h3 + r] = (float)p[r];
      if (!tf32) bias_operand(p[r], &B3k[((size_t)i * h3 + r) * 16]);
    }
    p += h3;
    if (shared) {  // W4 [nout][h3], b4 [nout] of the one shared net
      for (size_t e = 0; e < (size_t)nout * h3; ++e) w4[e] = (float)p[e];
      for (int o = 0; o < nout; ++o) b4[o] = (float)p[(size_t)nout * h3 + o];
    } else {
      for (int r = 0; r < h3; ++r) w4[(size_t)i * h3 + r] = (float)p[r];
      b4[i] = (float)p[h3];
    }
  }
  std::vector<float> xm(din), xi(din);
  for (int k = 0; k < din; ++k) {
    xm[k] = (float)d->x_mean[k];
    xi[k] = (float)(1.0 / d->x_std[k]);
  }
  auto up = [](void **dst, const void *src, size_t bytes) -> bool {
    return cudaMalloc(dst, bytes) == cudaSuccess && cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  bool ok = (tf32 ? up(&n->d_W1, F1.data(), F1.size() * 4) && up(&n->d_W2, F2.data(), F2.size() * 4) &&
                        up(&n->d_W3, F3.data(), F3.size() * 4)
                   : up(&n->d_W1, W1.data(), W1.size() * 2) && up(&n->d_W2, W2.data(), W2.size() * 2) &&
                        up(&n->d_W3, W3.data(), W3.size() * 2)) &&
            up((void **)&n->d_b1, b1.data(), b1.size() * 4) &&
            up((void **)&n->d_b2, b2.data(), b2.size() * 4) && up((void **)&n->d_b3, b3.data(), b3.size() * 4) &&
            up((void **)&n->d_w4, w4.data(), w4.size() * 4) && up((void **)&n->d_b4, b4.data(), b4.size() * 4) &&
            up((void **)&n->d_xmean, xm.data(), xm.size() * 4) && up((void **)&n->d_xinvstd, xi.data(), xi.size() * 4) &&
            up((void **)&n->d_ymean, d->y_mean, nout * 8) && up((void **)&n->d_ystd, d->y_std, nout * 8) &&
            up((void **)&n->d_species, d->species_of_net, nout * 4);
  n->b4_host = b4;
  n->xmean_host = xm;
  n->xinvstd_host = xi;
  n->ymean_host.assign(d->y_mean, d->y_mean + nout);
  n->ystd_host.assign(d->y_std, d->y_std + nout);
  if (ok && !tf32) ok = up(&n->d_b2k, B2k.data(), B2k.size() * 2) && up(&n->d_b3k, B3k.data(), B3k.size() * 2);
  if (ok && tf32 && !x3) ok = up(&n->d_b2k, B2f.data(), B2f.size() * 4);
  if (ok && x3)
    ok = up(&n->d_W1lo, L1v.data(), L1v.size() * 4) && up(&n->d_W2lo, L2v.data(), L2v.size() * 4) &&
         up(&n->d_W3lo, L3v.data(), L3v.size() * 4);
  if (!ok) return rc_fail(RC_ENOMEM, "rc_mlp_create: device upload failed");
  return RC_OK;
}

namespace {
double binom(int n, int m) {
  double r = 1.0;
  for (int q = 1; q <= m; ++q) r = r * (n - m + q) / q;
  return r;
}

template <int NS, int NE>
int launch_epilogue_t(const rc_mech *m, const rc_mlp *n, const EpiArgs &ea, const CellsDev &c, cudaStream_t s) {
  const int ns = m->ns, nn = ea.n_nets;
  const int stages = epi_stages<NS>();
  const int pn = NE ? ((nn + ns) * NE + 1) & ~1 : nn * ((ns + 1) & ~1);
  const size_t smem = (size_t)(ThermoSeg::size(ns) + ((ns * ns + 1) & ~1) + pn + 16 + ((3 * nn + 1) & ~1)) * 8 +
                      rcs::Ring<epi_tile<NS>()>::smem_bytes(2 + ns, nn * ea.passes, stages);
  constexpr int EPI_TILE = epi_tile<NS>(), EPI_THREADS = EPI_TILE + 32;
  const int64_t ntiles = (ea.rows + EPI_TILE - 1) / EPI_TILE;
  int64_t grid = rc_resident_blocks((const void *)chem_epilogue_kernel<NS, NE>, EPI_THREADS, smem);
  if (grid > ntiles) grid = ntiles;
  if (grid > QPART_BLOCKS) grid = QPART_BLOCKS;
  EpiConst K{};
  if (NE > 0) {  // (launch_epilogue checked n_nets <= EPI_KN, ne <= EPI_KE, ns <= EPI_KN)
    for (int e = 0; e < m->ne; ++e)
      for (int k = 0; k < ns; ++k) {
        K.E[e][k] = m->EF_host[(m->ne + e) * ns + k];
        if (k < nn) K.F[e][k] = m->EF_host[e * ns + k];
      }
    for (int q = 0; q < nn; ++q) {
      K.b4[q] = n->b4_host[q];
      K.ym[q] = n->ymean_host[q];
      K.ys[q] = n->ystd_host[q];
    }
  }
  ProfScope prof(RC_STAGE_EPILOGUE, s);
  chem_epilogue_kernel<NS, NE><<<(unsigned)grid, EPI_THREADS, smem, s>>>(ea, c, stages, K);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

int launch_l4(const rc_mlp *n, const void *h3, float *o, int rows, int cap, bool tf32, cudaStream_t s) {
  if (n->n_nets > L4_MAXO || n->h3 % 16) return rc_fail(RC_EUNSUPPORTED, "shared net: layer 4 needs <= 32 outputs, h3 % 16 == 0");
  ProfScope prof(RC_STAGE_L4, s);
  const int EB = tf32 ? 4 : 2, nt = (n->n_nets + 7) / 8, W = tf32 ? l4_warps<true>() : l4_warps<false>();
  const size_t smem = 2 * (size_t)nt * 8 * n->h3 * EB + (size_t)W * 2 * 16 * n->h3 * EB;
  if (smem > 227 * 1024) return rc_fail(RC_EUNSUPPORTED, "shared net: layer-4 shared memory (%zu B)", smem);
  const void *k = tf32 ? (const void *)l4_kernel<true> : (const void *)l4_kernel<false>;
  int64_t grid = rc_resident_blocks(k, 32 * W, smem);
  const int64_t want = ((rows + 15) / 16 + W - 1) / W;
  if (grid > want) grid = want;
  if (tf32) l4_kernel<true><<<(unsigned)grid, 32 * W, smem, s>>>(h3, n->d_w4, o, rows, n->h3, n->n_nets, cap);
  else l4_kernel<false><<<(unsigned)grid, 32 * W, smem, s>>>(h3, n->d_w4, o, rows, n->h3, n->n_nets, cap);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

int launch_epilogue(const rc_mech *m, const rc_mlp *n, const EpiArgs &ea, const CellsDev &c, cudaStream_t s) {
  // factored projection when net i predicts species i (checked at rc_mlp_create) and the element
  // count has an instance
  const bool ident = n->species_identity && ea.passes == 1 && m->uniform_tmid && n->inv_lambda == 10 &&
                     n->n_nets == m->ns - 1 && n->n_nets <= EPI_KN;
  if (m->ns == 9) return ident && m->ne == 3 ? launch_epilogue_t<9, 3>(m, n, ea, c, s) : launch_epilogue_t<9, 0>(m, n, ea, c, s);
  if (m->ns == 20) return ident && m->ne == 4 ? launch_epilogue_t<20, 4>(m, n, ea, c, s) : launch_epilogue_t<20, 0>(m, n, ea, c, s);
  return launch_epilogue_t<0, 0>(m, n, ea, c, s);
}
}  // namespace

int launch_chem(const rc_mech *m, const rc_mlp *n, const CellsDev &c, void *ws, size_t ws_bytes, cudaStream_t s) {
  if (c.n == 0) return RC_OK;
  // chunk capacity: largest multiple of 128 (<= MAX_CAP, <= n rounded up) whose layout fits the workspace
  int cap = chunk_cap(n, c.n);
  while (cap > 256 && ws_layout(n, cap, c.n).total > ws_bytes) cap -= 256;
  WsLayout L = ws_layout(n, cap, c.n);
  if (L.total > ws_bytes) return rc_fail(RC_EINVAL, "workspace too small (%zu < %zu)", ws_bytes, L.total);
  uint8_t *w = static_cast<uint8_t *>(ws);
  const int prec = n->precision == RC_BF16 ? 0 : n->precision == RC_TF32 ? 1 : 2;
  const bool tf32 = prec != 0, x3 = prec == 2;
  const int EB = tf32 ? 4 : 2;
  const int RB = x3 ? 64 : 128, KC = RB / EB;  // element bytes; K elements per swizzled operand row
  const int KATOM = tf32 ? 8 : 16;  // K elements per MMA (32 bytes)
  const int nets = n->gnets, nout = n->n_nets;  // GEMM nets (shared: 1), raw outputs per cell
  const bool shared = (n->flags & RC_MLP_SHARED) != 0;
  // activations: hi copy at the start of each region, X3's lo copy right after it
  uint8_t *z = w + L.z, *h1 = w + L.h1, *h2 = w + L.h2;
  const bool overlap = overlap_path(n) && L.nchunks >= 2;
  const int64_t zrows = (c.n + 255) / 256 * 256;  // z holds every cell of the call
  const size_t zlo = (size_t)zrows * n->kpad1 * EB, h1lo = (size_t)nets * cap * n->h1 * EB,
               h2lo = (size_t)nets * cap * n->h2 * EB;
  auto *opart = reinterpret_cast<float *>(w + L.opart);
  auto *qpart = reinterpret_cast<double *>(w + L.qpart);
  const int bn1 = l1_tile_n(), NP = l2_pass_width(n->h2), NP3 = l2_pass_width(n->h3), KZ = n->kpad1;
  const int P1 = NP > 256 ? 256 : NP, P2 = NP - P1;
  const int Q1 = NP3 > 256 ? 256 : NP3, Q2 = NP3 - Q1;
  // layer 1: {z, W1, h1 store (32-row boxes of one 128-byte row), z lo, W1 lo, h1 lo store}
  // layers 2/3: {A, B piece 1, B piece 2, h2 store (32 x 16 boxes), lo copies of the same}
  CUtensorMap m1[6], m2[10], m3[10];
  const int sbox = 128 / EB;  // h1 store box width: one 128-byte row
  int rc;
  for (int part = 0; part < (x3 ? 2 : 1); ++part) {
    const size_t oz = part ? zlo : 0, o1 = part ? h1lo : 0, o2 = part ? h2lo : 0;
    const void *W1 = part ? n->d_W1lo : n->d_W1, *W2 = part ? n->d_W2lo : n->d_W2, *W3 = part ? n->d_W3lo : n->d_W3;
    CUtensorMap *a1 = m1 + 3 * part, *a2 = m2 + 4 * part, *a3 = m3 + 4 * part;
    if ((rc = make_map(&a1[0], z + oz, KZ, cap, 1, BM, KZ, EB)) ||
        (rc = make_map(&a1[1], W1, KZ, n->h1, nets, l1_box_rows(), KZ, EB)) ||
        (rc = make_map(&a1[2], h1 + o1, n->h1, cap, nets, 32, sbox, EB)) ||
        (rc = make_map(&a2[0], h1 + o1, n->h1, cap, nets, BM, KC, EB)) ||
        (rc = make_map(&a2[1], W2, n->h1, n->h2, nets, P1 / 2, KC, EB)) ||
        (rc = make_map(&a2[2], W2, n->h1, n->h2, nets, P2 > 0 ? P2 / 2 : P1 / 2, KC, EB)) ||
        (rc = make_map(&a2[3], h2 + o2, n->h2, cap, nets, 32, 16, EB)) ||
        (rc = make_map(&a3[0], h2 + o2, n->h2, cap, nets, BM, KC, EB)) ||
        (rc = make_map(&a3[1], W3, n->h2, n->h3, nets, Q1 / 2, KC, EB)) ||
        (rc = make_map(&a3[2], W3, n->h2, n->h3, nets, Q2 > 0 ? Q2 / 2 : Q1 / 2, KC, EB)))
      return rc;
    if (shared) {  // layer 3 stores h3 = GELU(h2 W3^T + b3) for the layer-4 kernel
      if ((rc = make_map(&a3[3], w + L.h3, n->h3, cap, 1, 32, 16, EB))) return rc;
    } else {
      a3[3] = a2[3];  // unused by the dot epilogue
    }
  }
  // fused layers 1+2 (bf16, paper widths); RC_MLP_LAYERWISE forces the layer-wise path (comparisons)
  const bool fused = fused_path(n);
  CUtensorMap m12[7];
  // (TF32: 32-element K chunks, 16 W1 rows per CTA and chunk, b2 as a K = 8 fp32 operand)
  const int BKK = tf32 ? 8 : 16;
  if (fused && ((rc = make_map(&m12[0], z, KZ, cap, 1, BM, KZ, EB)) ||
                (rc = tf32 ? make_map(&m12[1], n->d_W1, KZ, n->h1, nets, 16, KZ, EB)       // per-chunk W1 ring
                      : KZ == 32 ? make_map(&m12[1], n->d_W1, KZ, n->h1, nets, 32, KZ, EB)
                                 : make_map_w1_groups(&m12[1], n->d_W1, KZ, n->h1, nets)) ||
                (rc = make_map(&m12[2], n->d_W2, n->h1, n->h2, nets, 128, KC, EB)) ||
                (rc = make_map(&m12[3], n->d_W2, n->h1, n->h2, nets, 72, KC, EB)) ||
                (rc = make_map(&m12[4], h2, n->h2, cap, nets, 32, 16, EB)) ||
                (rc = make_map(&m12[5], n->d_b2k, BKK, n->h2, nets, 128, BKK, EB)) ||
                (rc = make_map(&m12[6], n->d_b2k, BKK, n->h2, nets, 72, BKK, EB))))
    return rc;
  if (!x3) {  // the lo slots are never read: any valid map
    for (int k = 0; k < 3; ++k) m1[3 + k] = m1[k];
    for (int k = 0; k < 4; ++k) m2[4 + k] = m2[k], m3[4 + k] = m3[k];
  }
  // bf16: bias operand tiles of layers 2 and 3 (K = 16, 32-byte rows); unused (any valid map) otherwise
  if (!tf32) {
    if ((rc = make_map(&m2[8], n->d_b2k, 16, n->h2, nets, P1 / 2, 16, 2)) ||
        (rc = make_map(&m2[9], n->d_b2k, 16, n->h2, nets, P2 > 0 ? P2 / 2 : P1 / 2, 16, 2)) ||
        (rc = make_map(&m3[8], n->d_b3k, 16, n->h3, nets, Q1 / 2, 16, 2)) ||
        (rc = make_map(&m3[9], n->d_b3k, 16, n->h3, nets, Q2 > 0 ? Q2 / 2 : Q1 / 2, 16, 2)))
      return rc;
  } else {
    m2[8] = m2[9] = m2[0];
    m3[8] = m3[9] = m3[0];
  }
  // overlap: the odd chunks' h2 buffer (fused kernel's store map, layer 3's A map; never X3)
  CUtensorMap m12b[7], m3b[10];
  AuxStreams *aux = nullptr;
  int *sched = reinterpret_cast<int *>(w + L.sched);  // [nchunks] layer-3 tile counters | [nchunks] resident clusters
  if (overlap) {
    for (int k = 0; k < 7; ++k) m12b[k] = m12[k];
    for (int k = 0; k < 10; ++k) m3b[k] = m3[k];
    if ((rc = make_map(&m12b[4], w + L.h2b, n->h2, cap, nets, 32, 16, EB)) ||
        (rc = make_map(&m3b[0], w + L.h2b, n->h2, cap, nets, BM, KC, EB)))
      return rc;
    m3b[4] = m3b[0];
    if (!(aux = aux_streams())) return rc_fail(RC_ECUDA, "layer-3 overlap: auxiliary stream");
    RC_CUDA_TRY(cudaMemsetAsync(sched, 0, (size_t)L.nchunks * 2 * 4, s));
  }
  RC_CUDA_TRY(cudaMemsetAsync(qpart, 0, QPART_BLOCKS * 8, s));
  int64_t launches = 1;
  {  // a3 for every cell of the call in one launch (HBM-bound: per-chunk launches were tail-dominated)
    ProArgs pa{0, (int)c.n, (int)zrows, n->d_in, n->ns, KZ, (float)n->lambda_bc, (float)(1.0 / n->lambda_bc),
               n->d_xmean, n->d_xinvstd, z, prec, (int64_t)(zlo / EB), {}, {}};
    for (int k = 0; k < n->d_in && k < 32; ++k) pa.xm[k] = n->xmean_host[k], pa.xs[k] = n->xinvstd_host[k];
    ProfScope prof(RC_STAGE_PROLOGUE, s);
    auto launch_pro = [&](auto tile_c, auto ns_c) {
      constexpr int TILE = decltype(tile_c)::value, NS = decltype(ns_c)::value;
      const int pstages = 3;
      const size_t psmem = rcs::Ring<TILE>::smem_bytes(2 + n->ns, 0, pstages);
      int64_t pgrid = rc_resident_blocks((const void *)prologue_kernel<TILE, NS>, pro_threads<TILE>(), psmem);
      const int64_t ptiles = (c.n + TILE - 1) / TILE;
      if (pgrid > ptiles) pgrid = ptiles;
      if (pgrid < 1) pgrid = 1;  // n == 0 cannot reach here; padding rows only would need one CTA
      prologue_kernel<TILE, NS><<<(unsigned)pgrid, pro_threads<TILE>(), psmem, s>>>(pa, c, pstages);
    };
    using I = std::integral_constant<int, 0>;
    if (n->ns == 9)
      launch_pro(std::integral_constant<int, 256>{}, std::integral_constant<int, 9>{});
    else if (n->ns == 20)
      launch_pro(std::integral_constant<int, 128>{}, std::integral_constant<int, 20>{});
    else if (n->ns <= 12)
      launch_pro(std::integral_constant<int, 256>{}, I{});
    else
      launch_pro(std::integral_constant<int, 128>{}, I{});
    RC_LAUNCH_CHECK();
  }
  // overlap: layer 3 of chunk j - 1 is launched after the fused kernel of chunk j, in two launches
  // sharing one tile counter: a filler on the auxiliary stream that runs on the SMs the fused
  // kernel's 4-CTA clusters leave idle (it takes tiles only once every cluster is resident), and
  // the main launch on `s` once the fused kernel is done.  h2 alternates between two buffers.
  int fill_pairs = 0;
  L2Args pend{};
  bool have_pend = false;
  float *pend_oc = nullptr;  // shared net: the pending chunk's raw-output rows and row count (layer 4)
  int pend_rows = 0;
  int j = 0;
  for (int64_t c0 = 0; c0 < c.n; c0 += cap, ++j) {
    const int rows = (int)std::min<int64_t>(cap, c.n - c0);
    const int mt = (rows + 2 * BM - 1) / (2 * BM) * 2;  // even: CTA pairs of 128-row tiles
    if (c0 > 0) {  // this chunk's rows of z: re-point the layer-1 A operand maps
      const int zr = (int)std::min<int64_t>(cap, zrows - c0);
      uint8_t *zc = z + (size_t)c0 * KZ * EB;
      if ((rc = make_map(&m1[0], zc, KZ, zr, 1, BM, KZ, EB))) return rc;
      if (x3 && (rc = make_map(&m1[3], zc + zlo, KZ, zr, 1, BM, KZ, EB))) return rc;
      if (!x3) m1[3] = m1[0];
      if (fused && (rc = make_map(&m12[0], zc, KZ, zr, 1, BM, KZ, EB))) return rc;
    }
    const bool odd = overlap && (j & 1);
    if (odd) m12b[0] = m12[0];
    int ncl12 = 0;
    if (fused) {
      if (overlap && j >= 2 && fill_pairs > 0)  // this chunk's h2 buffer: chunk j - 2's filler is done with it
        RC_CUDA_TRY(cudaStreamWaitEvent(s, aux->fill[j & 1], 0));
      if (overlap && j >= 1) RC_CUDA_TRY(cudaEventRecord(aux->go, s));  // chunk j - 1's h2 is complete here
      // layers 1+2 in one kernel: h1 stays on chip; clusters of two CTA pairs share h1 chunks
      L12Args g12{mt, nets, n->h1 / (tf32 ? 32 : 64), n->h2, 0, n->d_b2};
      if (overlap) g12.started = sched + L.nchunks + j;
      if ((rc = launch_l12(KZ, tf32, odd ? m12b : m12, g12, s, &ncl12))) return rc;
      if (overlap && j == 0) fill_pairs = (rc_sm_count() - 4 * ncl12) / 2;
    } else {
      // layer 1: h1 = GELU(z W1^T) (b1 folded into z's constant-1 columns)
      L1Args g1{mt, (n->h1 + bn1 - 1) / bn1, nets, n->h1, 0, cap};
      if ((rc = launch_l1(KZ, prec, m1, g1, s))) return rc;
      // layer 2: h2 = GELU(h1 W2^T + b2), CTA-pair GEMM
      L2Args la{mt, n->h2 / NP, nets, (n->h1 + KC - 1) / KC, n->h2, 0, n->d_b2, nullptr, nullptr, cap, (n->h1 % KC) / KATOM};
      if ((rc = launch_l2_pair(NP, prec, m2, la, s))) return rc;
    }
    // layer 3 + folded layer 4: the same CTA-pair GEMM with the dot epilogue (K = h2, zero-filled to KC);
    // the raw outputs land in the all-cells array o [nets][passes][zrows] at this chunk's rows
    float *oc = opart + c0;
    if (overlap) {
      if (have_pend) {  // layer 3 of chunk j - 1 (h2 buffer (j - 1) % 2)
        const CUtensorMap *mp3 = (j - 1) & 1 ? m3b : m3;
        if (fill_pairs > 0) {
          RC_CUDA_TRY(cudaStreamWaitEvent(aux->s2, aux->go, 0));
          L2Args f = pend;
          f.gate = sched + L.nchunks + j;
          f.gate_target = ncl12;
          f.gate_ns = 50000;  // 50 us: a cluster of the fused kernel this launch kept out starts that late
          f.prof_stage = RC_STAGE_L3_FILL;
          if ((rc = launch_l2_pair(NP3, prec, mp3, f, aux->s2, fill_pairs))) return rc;
          RC_CUDA_TRY(cudaEventRecord(aux->fill[(j - 1) & 1], aux->s2));
        }
        if ((rc = launch_l2_pair(NP3, prec, mp3, pend, s))) return rc;
        if (shared) {  // layer 4 of chunk j - 1 once h3 is complete (both layer-3 launches)
          if (fill_pairs > 0) RC_CUDA_TRY(cudaStreamWaitEvent(s, aux->fill[(j - 1) & 1], 0));
          if ((rc = launch_l4(n, w + L.h3, pend_oc, pend_rows, (int)zrows, tf32, s))) return rc;
        }
      }
      if (shared) {  // layer 3 as a plain GELU layer into h3 (one buffer: layer 4 of a chunk runs
                     // before the next fused kernel, whose side launch writes h3 next)
        pend = L2Args{mt, n->h3 / NP3, 1, (n->h2 + KC - 1) / KC, n->h3, 0, n->d_b3, nullptr, nullptr, cap, (n->h2 % KC) / KATOM};
        pend.prof_stage = RC_STAGE_L3;
      } else {
        pend = L2Args{mt, n->h3 / NP3, nets, (n->h2 + KC - 1) / KC, n->h3, 0, n->d_b3, n->d_w4, oc, (int)zrows, (n->h2 % KC) / KATOM};
      }
      pend.tile_ctr = sched + j;
      pend_oc = oc;
      pend_rows = rows;
      have_pend = true;
    } else if (!shared) {
      L2Args l3{mt, n->h3 / NP3, nets, (n->h2 + KC - 1) / KC, n->h3, 0, n->d_b3, n->d_w4, oc, (int)zrows, (n->h2 % KC) / KATOM};
      if ((rc = launch_l2_pair(NP3, prec, m3, l3, s))) return rc;
    } else {
      // shared net (NEXT-2): layer 3 as a plain GELU layer into h3, then the n_out-wide layer 4
      L2Args l3{mt, n->h3 / NP3, 1, (n->h2 + KC - 1) / KC, n->h3, 0, n->d_b3, nullptr, nullptr, cap, (n->h2 % KC) / KATOM};
      l3.prof_stage = RC_STAGE_L3;
      if ((rc = launch_l2_pair(NP3, prec, m3, l3, s))) return rc;
      if ((rc = launch_l4(n, w + L.h3, oc, rows, (int)zrows, tf32, s))) return rc;
    }
    launches += 4;
  }
  if (overlap) {  // the last chunk's layer 3 (nothing left to overlap it with), then join the fillers
    if ((rc = launch_l2_pair(NP3, prec, (j - 1) & 1 ? m3b : m3, pend, s))) return rc;
    if (fill_pairs > 0) RC_CUDA_TRY(cudaStreamWaitEvent(s, aux->fill[j & 1], 0));
    if (shared && (rc = launch_l4(n, w + L.h3, pend_oc, pend_rows, (int)zrows, tf32, s))) return rc;
  }
  {  // a5 once over every cell of the call (one streaming pass, like the prologue)
    EpiArgs ea{0, (int)c.n, (int)zrows, nout, shared ? 1 : n->h3 / NP3, n->inv_lambda, n->ns, n->lambda_bc, 1.0 / n->dt,
               opart, n->d_b4, n->d_ymean, n->d_ystd, m->d_P, m->d_thermo, n->d_species, m->d_EF, m->ne, qpart, {}};
    for (int q = 0; q <= 16; ++q) ea.binom[q] = q <= n->inv_lambda ? binom(n->inv_lambda, q) : 0.0;
    if ((rc = launch_epilogue(m, n, ea, c, s))) return rc;
  }
  if (c.red) {
    ProfScope prof(RC_STAGE_FINALIZE, s);
    qdot_finalize_kernel<<<1, 32, 0, s>>>(qpart, QPART_BLOCKS, c.red);
    RC_LAUNCH_CHECK();
  }
  (void)launches;
  return RC_OK;
}
