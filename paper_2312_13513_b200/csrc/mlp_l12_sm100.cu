// mlp_l12_sm100.cu -- layers 1 and 2 of the per-species MLP fused in one
// persistent tcgen05 kernel (hidden layers 1600 and 800, GELU).
//
//   h2[:, pass] = GELU( GELU(z W1^T + b1) W2[pass]^T + b2 )
//
// The 1600-wide first hidden layer never leaves the SM: for each 64-column
// chunk c of h1 the MMA warp computes acc1 = z W1[c]^T (M=128, N=64, K=16 or
// 32; b1 is folded into the MMA through two constant-1 columns of z carrying
// b1 split into bf16 hi + lo), eight epilogue warps drain acc1 from TMEM,
// apply GELU, round to bf16 and write the chunk into a shared-memory ring in
// the 128-byte-swizzled K-major layout the tensor core reads, and the MMA warp
// then accumulates acc2 += h1[c] W2[pass, c]^T (N = NP split into <=256-wide
// MMAs).  At the end of the tile the same warps apply b2 + GELU to acc2 and
// store h2 (bf16).
// This removes the h1 round trip through HBM (3.2 KB per cell per net) and
// hides layer-1's GELU work under layer-2's tensor-core time.
//
// TMEM (512 columns): acc2 at [0, NP), acc1 at [448, 512).
// Warps: 0 TMA producer, 1 MMA issuer, 2-9 epilogue (layer-1 GELU producers
// during the tile, acc2 drain at its end; two warps per TMEM lane quadrant).
#include <cuda_bf16.h>

#include "mlp_internal.h"
#include "ptx.cuh"

namespace {

constexpr int L12_THREADS = 320;
constexpr int C1 = 64;          // h1 chunk width (one 128-byte swizzle row of bf16)
constexpr int A2_SLOTS = 3;     // h1-chunk ring depth
constexpr int ACC1_COL = 448;   // TMEM column of acc1

__device__ __forceinline__ float gelu_f(float x) {
  float u = x * fmaf(0.0356774081f, x * x, 0.7978845608f);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  float hx = 0.5f * x;
  return fmaf(hx, t, hx);
}

// debug timeline: dbg[(role * 8 + it) * 64 + c] = globaltimer, CTA 0, first 8 tiles, 64 chunks
__device__ __forceinline__ void dbg_rec(unsigned long long *d, int role, int it, int c) {
  if (d && blockIdx.x == 0 && it < 8 && c < 64) d[(role * 8 + it) * 64 + c] = rcx::global_ns();
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&v);
}

// UMMA K-major descriptor for a 32/64/128-byte swizzled tile (8-row atoms)
template <int ROW_BYTES>
__device__ __forceinline__ uint64_t desc_sw(const void *smem) {
  constexpr uint64_t layout = ROW_BYTES == 128 ? 2 : ROW_BYTES == 64 ? 4 : 6;
  uint64_t d = (uint64_t)((rcx::smem_u32(smem) & 0x3FFFF) >> 4);
  d |= (uint64_t)((8 * ROW_BYTES) >> 4) << 32;  // SBO: 8 rows
  d |= (uint64_t)1 << 46;
  d |= layout << 61;
  return d;
}

template <int NP, int KZ>
__global__ void __launch_bounds__(L12_THREADS, 1)
    l12_kernel(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapW1,
               const __grid_constant__ CUtensorMap mapW2, L12Args a) {
  static_assert(NP % 16 == 0 && NP <= ACC1_COL, "pass width");
  static_assert(KZ == 16 || KZ == 32, "layer-1 K");
  constexpr int P1 = NP > 256 ? 256 : NP, P2 = NP - P1;   // MMA pieces of the pass (N <= 256 each)
  constexpr int W2_BOX = NP > 256 ? NP / 2 : NP;          // TMA box rows (<= 256)
  constexpr uint32_t Z_BYTES = 128 * KZ * 2, W1_BYTES = C1 * KZ * 2, W2_BYTES = NP * C1 * 2;
  constexpr uint32_t STAGE_BYTES = W2_BYTES + W1_BYTES;
  constexpr uint32_t A2_BYTES = 128 * C1 * 2;
  static_assert(W2_BYTES % 1024 == 0 && (W2_BOX * 128) % 1024 == 0, "swizzle atoms");

  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = rcx::smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  const int S = a.stages;
  uint8_t *sW = smem;                                  // S x [W2 chunk | W1 chunk]
  uint8_t *sA2 = sW + S * STAGE_BYTES;                 // A2_SLOTS x 16 KB
  uint8_t *sZ = sA2 + A2_SLOTS * A2_BYTES;             // 2 x Z tile
  float *sB2 = reinterpret_cast<float *>(sZ + 2 * Z_BYTES);   // 2 x b2 slice of the tile's pass (NP floats)
  uint64_t *bar = reinterpret_cast<uint64_t *>(sB2 + 2 * NP);
  uint64_t *full = bar, *empty = full + S, *zfull = empty + S, *zempty = zfull + 2;
  uint64_t *a1full = zempty + 2, *a1empty = a1full + 1, *a2full = a1empty + 1, *a2empty = a2full + A2_SLOTS;
  uint64_t *c2full = a2empty + A2_SLOTS, *c2empty = c2full + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(c2empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    rcx::prefetch_tmap(&mapZ);
    rcx::prefetch_tmap(&mapW1);
    rcx::prefetch_tmap(&mapW2);
    for (int s = 0; s < S; ++s) { rcx::mbar_init(&full[s], 1); rcx::mbar_init(&empty[s], 1); }
    for (int z = 0; z < 2; ++z) { rcx::mbar_init(&zfull[z], 1); rcx::mbar_init(&zempty[z], 1); }
    rcx::mbar_init(a1full, 1);
    rcx::mbar_init(a1empty, 8);
    for (int r = 0; r < A2_SLOTS; ++r) { rcx::mbar_init(&a2full[r], 8); rcx::mbar_init(&a2empty[r], 1); }
    rcx::mbar_init(c2full, 1);
    rcx::mbar_init(c2empty, 8);
    rcx::fence_mbar_init();
  }
  if (warp == 1) rcx::tmem_alloc(tmem_slot, 512);
  rcx::tc_fence_before();
  __syncthreads();
  rcx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int C = a.chunks;
  const int total = a.nets * a.m_tiles * a.passes;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
        const int pass = tile % a.passes, rest = tile / a.passes;
        const int m_blk = rest % a.m_tiles, net = rest / a.m_tiles;
        const int zb = it & 1;
        rcx::mbar_wait(&zempty[zb], ((it >> 1) & 1) ^ 1);
        rcx::mbar_arrive_expect_tx(&zfull[zb], Z_BYTES + NP * 4);
        rcx::tma_load_3d(sZ + zb * Z_BYTES, &mapZ, &zfull[zb], 0, m_blk * 128, 0);
        rcx::bulk_g2s(sB2 + zb * NP, a.b2 + (size_t)net * a.h2 + pass * NP, NP * 4, &zfull[zb]);
        for (int c = 0; c < C; ++c) {
          rcx::mbar_wait(&empty[s], ph ^ 1);
          rcx::mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
          uint8_t *st = sW + s * STAGE_BYTES;
          rcx::tma_load_3d(st + W2_BYTES, &mapW1, &full[s], 0, c * C1, net);
          rcx::tma_load_3d(st, &mapW2, &full[s], c * C1, pass * NP, net);
          if (NP > 256) rcx::tma_load_3d(st + W2_BOX * 128, &mapW2, &full[s], c * C1, pass * NP + W2_BOX, net);
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      constexpr uint32_t id1 = rcx::make_idesc(1u, 128, C1);
      constexpr uint32_t idp1 = rcx::make_idesc(1u, 128, P1);
      constexpr uint32_t idp2 = rcx::make_idesc(1u, 128, P2 > 0 ? P2 : 16);
      const uint32_t acc1 = tmem + ACC1_COL, acc2 = tmem;
      int s = 0;
      uint32_t ph = 0;
      uint32_t n_l1 = 0, n_a2 = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
        const int zb = it & 1;
        rcx::mbar_wait(&zfull[zb], (it >> 1) & 1);
        const uint64_t dz = desc_sw<KZ * 2>(sZ + zb * Z_BYTES);
        // acc1 = z W1[chunk]^T for the chunk whose weights sit in W stage `stage`
        auto issue_l1 = [&](int stage) {
          rcx::mbar_wait(a1empty, (n_l1 & 1) ^ 1);
          rcx::tc_fence_after();
          const uint64_t dw = desc_sw<KZ * 2>(sW + stage * STAGE_BYTES + W2_BYTES);
#pragma unroll
          for (int k = 0; k < KZ / 16; ++k) rcx::mma_bf16(acc1, dz + 2 * k, dw + 2 * k, id1, k != 0);
          rcx::mma_commit(a1full);
          ++n_l1;
        };
        rcx::mbar_wait(&full[s], ph);  // chunk 0's W stage
        rcx::tc_fence_after();
        issue_l1(s);
        for (int c = 0; c < C; ++c) {
          int s_n = s + 1;
          uint32_t ph_n = ph;
          if (s_n == S) { s_n = 0; ph_n ^= 1; }
          if (c + 1 < C) {  // next chunk's layer-1 MMA runs ahead of this chunk's layer-2 MMAs
            rcx::mbar_wait(&full[s_n], ph_n);
            issue_l1(s_n);
          }
          if (c == 0) rcx::mbar_wait(c2empty, (it & 1) ^ 1);
          const int slot = n_a2 % A2_SLOTS;
          dbg_rec(a.dbg, 0, it, c);
          rcx::mbar_wait(&a2full[slot], (n_a2 / A2_SLOTS) & 1);
          dbg_rec(a.dbg, 1, it, c);
          rcx::tc_fence_after();
          const uint64_t da = desc_sw<128>(sA2 + slot * A2_BYTES);
          const uint64_t db = desc_sw<128>(sW + s * STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < C1 / 16; ++k) {
            rcx::mma_bf16(acc2, da + 2 * k, db + 2 * k, idp1, (c | k) != 0);
            if (P2 > 0)
              rcx::mma_bf16(acc2 + P1, da + 2 * k, db + (uint64_t)((P1 * 128) >> 4) + 2 * k, idp2, (c | k) != 0);
          }
          rcx::mma_commit(&a2empty[slot]);
          rcx::mma_commit(&empty[s]);
          ++n_a2;
          s = s_n;
          ph = ph_n;
        }
        rcx::mma_commit(c2full);
        rcx::mma_commit(&zempty[zb]);
      }
    }
  } else {  // ------------------------------------------------------ epilogue warps 2-9
    // Two warps per TMEM lane quadrant q (rows 32q..32q+31); `half` picks the
    // column half each one handles.  Per chunk: layer-1 GELU -> A2 ring; per
    // tile: b2 + GELU of acc2 -> h2.
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t tq = (uint32_t)(q * 32) << 16;
    constexpr int NCH = NP / 16, CH0 = (NCH + 1) / 2;   // acc2 16-column chunks: [0,CH0) half 0, [CH0,NCH) half 1
    uint32_t n1 = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      const int pass = tile % a.passes, rest = tile / a.passes;
      const int m_blk = rest % a.m_tiles, net = rest / a.m_tiles;
      for (int c = 0; c < C; ++c, ++n1) {
        rcx::mbar_wait(a1full, n1 & 1);
        if (warp == 2 && lane == 0) dbg_rec(a.dbg, 2, it, c);
        rcx::tc_fence_after();
        uint32_t v[32];
        tmem_ld32(tmem + ACC1_COL + tq + half * 32, v);
        rcx::tmem_ld_wait();
        rcx::tc_fence_before();
        __syncwarp();
        if (lane == 0) rcx::mbar_arrive(a1empty);
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) pk[j] = pack_bf16(gelu_f(__uint_as_float(v[2 * j])), gelu_f(__uint_as_float(v[2 * j + 1])));
        const int slot = n1 % A2_SLOTS;
        rcx::mbar_wait(&a2empty[slot], ((n1 / A2_SLOTS) & 1) ^ 1);
        uint8_t *dst = sA2 + slot * A2_BYTES + row * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          *reinterpret_cast<uint4 *>(dst + (((half * 4 + j) ^ (row & 7)) << 4)) =
              make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) rcx::mbar_arrive(&a2full[slot]);
        if (warp == 2 && lane == 0) dbg_rec(a.dbg, 3, it, c);
      }
      // ---- drain acc2 of this tile
      rcx::mbar_wait(c2full, it & 1);
      if (warp == 2 && lane == 0) dbg_rec(a.dbg, 4, it, 0);
      rcx::tc_fence_after();
      const float *b2 = sB2 + (it & 1) * NP;
      __nv_bfloat16 *out = a.h2out + ((size_t)net * a.cap + m_blk * 128 + row) * a.h2 + pass * NP;
      const int ch_lo = half ? CH0 : 0, ch_hi = half ? NCH : CH0;
      for (int cc = ch_lo; cc < ch_hi; cc += 2) {
        uint32_t v[32];
        const bool two = cc + 1 < ch_hi;
        if (two)
          tmem_ld32(tmem + tq + cc * 16, v);
        else
          rcx::tmem_ld16(tmem + tq + cc * 16, *reinterpret_cast<uint32_t(*)[16]>(v));
        rcx::tmem_ld_wait();
        if (cc + 2 >= ch_hi) {  // this warp's last acc2 columns are in registers: release acc2
          rcx::tc_fence_before();
          __syncwarp();
          if (lane == 0) rcx::mbar_arrive(c2empty);
        }
        const int nv = two ? 32 : 16;
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (2 * j < nv)
            pk[j] = pack_bf16(gelu_f(__uint_as_float(v[2 * j]) + b2[cc * 16 + 2 * j]),
                              gelu_f(__uint_as_float(v[2 * j + 1]) + b2[cc * 16 + 2 * j + 1]));
        uint4 *d = reinterpret_cast<uint4 *>(out + cc * 16);
        d[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        d[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        if (two) {
          d[2] = make_uint4(pk[8], pk[9], pk[10], pk[11]);
          d[3] = make_uint4(pk[12], pk[13], pk[14], pk[15]);
        }
      }
      if (warp == 2 && lane == 0) dbg_rec(a.dbg, 4, it, 1);
    }
  }
  __syncthreads();
  if (warp == 1) {
    rcx::tc_fence_after();
    rcx::tmem_dealloc(tmem, 512);
  }
}

template <int NP, int KZ>
int launch_l12_t(const CUtensorMap &Z, const CUtensorMap &W1, const CUtensorMap &W2, L12Args a, cudaStream_t s) {
  constexpr size_t Z_BYTES = 128 * KZ * 2, STAGE = NP * C1 * 2 + C1 * KZ * 2, A2 = 128 * C1 * 2;
  const size_t fixed = 1024 + A2_SLOTS * A2 + 2 * Z_BYTES + 2 * NP * 4 + 256;
  int stages = (int)((232448 - fixed) / STAGE);
  if (stages > 6) stages = 6;
  if (stages < 2) return rc_fail(RC_EUNSUPPORTED, "fused L1/L2: pass width %d does not fit shared memory", NP);
  a.stages = stages;
  const size_t smem = fixed + stages * STAGE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(l12_kernel<NP, KZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    attr = true;
  }
  const int total = a.nets * a.m_tiles * a.passes;
  const int grid = total < mlp_num_sms() ? total : mlp_num_sms();
  l12_kernel<NP, KZ><<<grid, L12_THREADS, smem, s>>>(Z, W1, W2, a);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

}  // namespace

// pass width: the widest NP <= 448 (TMEM) that divides h2 into equal passes
int l12_pass_width(int h2) {
  for (int p = 1; p <= h2 / 16; ++p)
    if (h2 % p == 0 && (h2 / p) % 16 == 0 && h2 / p <= 400 && (h2 / p <= 256 || (h2 / p / 2) % 8 == 0)) return h2 / p;
  return 0;
}

int launch_l12(int NP, int KZ, const CUtensorMap &Z, const CUtensorMap &W1, const CUtensorMap &W2, const L12Args &a,
               cudaStream_t s) {
  ProfScope prof(RC_STAGE_L2, s);
#define RC_L12(np)                                                              \
  if (NP == np) return KZ == 16 ? launch_l12_t<np, 16>(Z, W1, W2, a, s) : launch_l12_t<np, 32>(Z, W1, W2, a, s);
  RC_L12(400)
  RC_L12(256)
  RC_L12(208)
  RC_L12(128)
  RC_L12(64)
  RC_L12(32)
  RC_L12(16)
#undef RC_L12
  return rc_fail(RC_EUNSUPPORTED, "fused L1/L2: no instance for pass width %d", NP);
}
