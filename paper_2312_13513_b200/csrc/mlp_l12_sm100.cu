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
// Warps: 0 TMA producer, 1 MMA issuer, 2-17 epilogue (layer-1 GELU producers
// during the tile, acc2 drain at its end; four warps per TMEM lane quadrant).
#include <cuda_bf16.h>

#include "mlp_internal.h"
#include "ptx.cuh"

namespace {

constexpr int NEPI = 16;                  // epilogue warps: 4 per TMEM lane quadrant
constexpr int L12_THREADS = 64 + 32 * NEPI;
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
  if (d && blockIdx.x == 0 && it < 8 && c < 64) d[(role * 8 + it) * 64 + c] = clock64();
}

// GELU on two bf16 values at once (tanh form, packed bf16x2 FMA pipe + one MUFU
// op per pair): 0.5 x (1 + tanh(x (c0 + c1 x^2))), c0 = sqrt(2/pi), c1 = 0.044715 c0.
// The result is rounded to bf16 anyway before it feeds the next tensor-core
// layer; the packed arithmetic adds ~2^-9 relative error per op (DESIGN.md,
// MLP numerics) and halves the epilogue's FMA-pipe and MUFU time.
__device__ __forceinline__ uint32_t gelu_bf16x2(uint32_t x) {
  const uint32_t c0 = 0x3F4C3F4Cu;   // bf16(0.7978846) x2
  const uint32_t c1 = 0x3D123D12u;   // bf16(0.0356774) x2
  const uint32_t hf = 0x3F003F00u;   // 0.5 x2
  uint32_t xx, t, u, th, hx, r;
  asm("mul.rn.bf16x2 %0, %1, %1;" : "=r"(xx) : "r"(x));
  asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(t) : "r"(xx), "r"(c1), "r"(c0));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(u) : "r"(t), "r"(x));
  asm("tanh.approx.bf16x2 %0, %1;" : "=r"(th) : "r"(u));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(hx) : "r"(x), "r"(hf));
  asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(hx), "r"(th), "r"(hx));
  return r;
}
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// TMA tensor store shared -> global (bulk-group completion)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, const void *src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(rcx::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

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

// ---------------------------------------------------------------------------
// CTA-pair version (cta_group::2, M = 256): the even CTA of each cluster issues
// M=256 MMAs whose A rows are split 128/128 between the two CTAs and whose B
// operand (W1 / W2 chunk) is split by N, so every SM stages only half of each
// weight chunk -- half the TMA write and operand-read shared-memory traffic of
// the single-CTA kernel, which was shared-memory-bandwidth bound.
//   B split: piece 1 (N = P1 <= 256) rows [0,P1/2) in CTA 0, [P1/2,P1) in CTA 1;
//            piece 2 (N = P2) rows P1 + [0,P2/2) in CTA 0, P1 + [P2/2,P2) in CTA 1.
// Barriers owned by the even CTA: full / zfull (both CTAs' TMA bytes),
// a1empty / a2full / c2empty (16 warp arrivals, 8 per CTA).  Barriers the
// MMA commits to (empty, zempty, a1full, a2empty, c2full) are multicast to both.
// ---------------------------------------------------------------------------
template <int NP, int KZ>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(L12_THREADS, 1)
    l12_pair_kernel(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapW1,
                    const __grid_constant__ CUtensorMap mapW2a, const __grid_constant__ CUtensorMap mapW2b,
                    const __grid_constant__ CUtensorMap mapH2, L12Args a) {
  static_assert(NP % 16 == 0 && NP <= ACC1_COL, "pass width");
  constexpr int P1 = NP > 256 ? 256 : NP, P2 = NP - P1;
  constexpr int H1 = P1 / 2, H2 = P2 / 2;                 // B rows per CTA of each piece
  static_assert(H1 % 8 == 0 && H2 % 8 == 0, "8-row swizzle atoms");
  constexpr uint32_t Z_BYTES = 128 * KZ * 2, W1_BYTES = (C1 / 2) * KZ * 2, W2_BYTES = (NP / 2) * C1 * 2;
  constexpr uint32_t STAGE_BYTES = W2_BYTES + W1_BYTES;
  constexpr uint32_t A2_BYTES = 128 * C1 * 2;
  static_assert(STAGE_BYTES % 1024 == 0 || (W2_BYTES % 1024 == 0), "alignment");

  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = rcx::smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  const int S = a.stages;
  constexpr uint32_t STAGE_AL = (STAGE_BYTES + 1023u) & ~1023u;
  uint8_t *sW = smem;
  uint8_t *sA2 = sW + S * STAGE_AL;
  uint8_t *sZ = sA2 + A2_SLOTS * A2_BYTES;
  uint8_t *sST = sZ + 2 * Z_BYTES;                    // NEPI warps x 2 x [32 rows x 16 cols] bf16 store staging
  float *sB2 = reinterpret_cast<float *>(sST + NEPI * 2 * 1024);
  uint64_t *bar = reinterpret_cast<uint64_t *>(sB2 + 2 * NP);
  uint64_t *full = bar, *empty = full + S, *zfull = empty + S, *zempty = zfull + 2;
  uint64_t *a1full = zempty + 2, *a1empty = a1full + 2, *a2full = a1empty + 1, *a2empty = a2full + A2_SLOTS;
  uint64_t *c2full = a2empty + A2_SLOTS, *c2empty = c2full + 1, *bfull = c2empty + 1, *bempty = bfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bempty + 2);

  // warp roles: 0..NEPI-1 epilogue, NEPI TMA producer, NEPI+1 MMA issuer (the
  // scheduler favours higher warp ids, so the two latency-critical single-thread
  // roles get the highest ids)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int W_TMA = NEPI, W_MMA = NEPI + 1;
  const uint32_t rank = rcx::cluster_rank();
  const bool leader = rank == 0;
  if (warp == W_TMA && lane == 0) {
    rcx::prefetch_tmap(&mapZ);
    rcx::prefetch_tmap(&mapW1);
    rcx::prefetch_tmap(&mapW2a);
    if (P2 > 0) rcx::prefetch_tmap(&mapW2b);
    rcx::prefetch_tmap(&mapH2);
    for (int s = 0; s < S; ++s) { rcx::mbar_init(&full[s], 2); rcx::mbar_init(&empty[s], 1); }
    for (int z = 0; z < 2; ++z) {
      rcx::mbar_init(&zfull[z], 2);
      rcx::mbar_init(&zempty[z], 1);
      rcx::mbar_init(&bfull[z], 1);
      rcx::mbar_init(&bempty[z], NEPI);
    }
    rcx::mbar_init(&a1full[0], 1);
    rcx::mbar_init(&a1full[1], 1);
    rcx::mbar_init(a1empty, NEPI);          // one epilogue group (NEPI/2 warps) x 2 CTAs per h1 chunk
    for (int r = 0; r < A2_SLOTS; ++r) { rcx::mbar_init(&a2full[r], NEPI); rcx::mbar_init(&a2empty[r], 1); }
    rcx::mbar_init(c2full, 1);
    rcx::mbar_init(c2empty, 2 * NEPI);
    rcx::fence_mbar_init();
  }
  if (warp == W_MMA) rcx::tmem_alloc_pair(tmem_slot, 512);
  rcx::tc_fence_before();
  rcx::cluster_sync();
  rcx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int C = a.chunks;
  const int pairs = a.m_tiles / 2;
  const int total = a.nets * pairs * a.passes;
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == W_TMA) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer (both CTAs)
      const uint32_t full0 = rcx::map_cta(full, 0), zfull0 = rcx::map_cta(zfull, 0);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int tile = cl; tile < total; tile += ncl, ++it) {
        const int pass = tile % a.passes, rest = tile / a.passes;
        const int mp = rest % pairs, net = rest / pairs;
        const int zb = it & 1;
        rcx::mbar_wait(&zempty[zb], ((it >> 1) & 1) ^ 1);
        rcx::mbar_arrive_expect_tx_cluster(zfull0 + zb * 8, Z_BYTES);
        rcx::tma_load_3d_pair(sZ + zb * Z_BYTES, &mapZ, &zfull[zb], 0, mp * 256 + rank * 128, 0);
        rcx::mbar_wait(&bempty[zb], ((it >> 1) & 1) ^ 1);   // b2 slice for this CTA's drain
        rcx::mbar_arrive_expect_tx(&bfull[zb], NP * 4);
        rcx::bulk_g2s(sB2 + zb * NP, a.b2 + (size_t)net * a.h2 + pass * NP, NP * 4, &bfull[zb]);
        for (int c = 0; c < C; ++c) {
          if (a.flags & 2) break;  // diagnostic: weights stay whatever the stages hold
          rcx::mbar_wait(&empty[s], ph ^ 1);
          rcx::mbar_arrive_expect_tx_cluster(full0 + s * 8, STAGE_BYTES);
          uint8_t *st = sW + s * STAGE_AL;
          rcx::tma_load_3d_pair(st + W2_BYTES, &mapW1, &full[s], 0, c * C1 + rank * (C1 / 2), net);
          rcx::tma_load_3d_pair(st, &mapW2a, &full[s], c * C1, pass * NP + rank * H1, net);
          if (P2 > 0) rcx::tma_load_3d_pair(st + H1 * 128, &mapW2b, &full[s], c * C1, pass * NP + P1 + rank * H2, net);
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == W_MMA) {
    if (lane == 0 && leader) {  // ------------------------------------- MMA issuer (even CTA)
      // The tensor pipe accepts roughly one MMA ahead of execution, so every
      // barrier wait / commit of this thread is placed between layer-2 MMAs
      // (where the thread would block on issue anyway), and layer-1 MMAs run
      // two chunks ahead of the layer-2 MMAs that consume their output, giving
      // the epilogue ~1.5 chunks of latency budget per h1 chunk.
      constexpr uint32_t id1 = rcx::make_idesc(1u, 256, C1);
      constexpr uint32_t idp1 = rcx::make_idesc(1u, 256, P1);
      constexpr uint32_t idp2 = rcx::make_idesc(1u, 256, P2 > 0 ? P2 : 16);
      const uint32_t acc1 = tmem + ACC1_COL, acc2 = tmem;
      uint32_t n_l1 = 0, n_a2 = 0, g0 = 0;  // global counters: layer-1 MMAs, A2 chunks, W stages
      int it = 0;
      for (int tile = cl; tile < total; tile += ncl, ++it, g0 += C) {
        const int zb = it & 1;
        rcx::mbar_wait(&zfull[zb], (it >> 1) & 1);
        const uint64_t dz = desc_sw<KZ * 2>(sZ + zb * Z_BYTES);
        auto stage_of = [&](int j) { return (int)((g0 + j) % S); };
        auto phase_of = [&](int j) { return (uint32_t)(((g0 + j) / S) & 1); };
        auto issue_l1 = [&](int j) {  // acc1 = z W1[chunk j]^T ; the chunk's W stage must be full
          rcx::mbar_wait(a1empty, (n_l1 & 1) ^ 1);
          rcx::tc_fence_after();
          const uint64_t dw = desc_sw<KZ * 2>(sW + stage_of(j) * STAGE_AL + W2_BYTES);
#pragma unroll
          for (int k = 0; k < KZ / 16; ++k) rcx::mma_bf16_pair(acc1, dz + 2 * k, dw + 2 * k, id1, k != 0);
          rcx::mma_commit_pair(&a1full[n_l1 & 1]);   // h1 chunk n goes to epilogue group n % 2
          ++n_l1;
        };
        rcx::mbar_wait(&full[stage_of(0)], phase_of(0));
        issue_l1(0);
        if (C > 1) {
          if (!(a.flags & 2)) rcx::mbar_wait(&full[stage_of(1)], phase_of(1));
          issue_l1(1);
        }
        rcx::mbar_wait(c2empty, (it & 1) ^ 1);  // previous tile's acc2 drained
        for (int c = 0; c < C; ++c) {
          const int slot = n_a2 % A2_SLOTS;
          const int sc = stage_of(c);
          dbg_rec(a.dbg, 0, it, c);
          if (!(a.flags & 1)) rcx::mbar_wait(&a2full[slot], (n_a2 / A2_SLOTS) & 1);
          dbg_rec(a.dbg, 1, it, c);
          rcx::tc_fence_after();
          const uint64_t da = desc_sw<128>(sA2 + slot * A2_BYTES);
          const uint64_t db = desc_sw<128>(sW + sc * STAGE_AL);
#pragma unroll
          for (int k = 0; k < C1 / 16; ++k) {
            rcx::mma_bf16_pair(acc2, da + 2 * k, db + 2 * k, idp1, (c | k) != 0);
            if (P2 > 0)
              rcx::mma_bf16_pair(acc2 + P1, da + 2 * k, db + (uint64_t)((H1 * 128) >> 4) + 2 * k, idp2, (c | k) != 0);
            if (k == 0 && c + 2 < C && !(a.flags & 2)) rcx::mbar_wait(&full[stage_of(c + 2)], phase_of(c + 2));
            if (k == 1 && c + 2 < C) issue_l1(c + 2);
          }
          rcx::mma_commit_pair(&a2empty[slot]);
          rcx::mma_commit_pair(&empty[sc]);
          ++n_a2;
        }
        rcx::mma_commit_pair(c2full);
        rcx::mma_commit_pair(&zempty[zb]);
      }
    }
  } else {  // ------------------------------------------------------ epilogue warps 0..NEPI-1 (both CTAs)
    // Two groups of NEPI/2 warps ping-pong over the h1 chunks (global chunk n
    // -> group n % 2), so each chunk's GELU has ~1.5 chunk periods of latency
    // budget; inside a group two warps per TMEM lane quadrant q take 32 of the
    // 64 columns each.  In the drain all NEPI warps (four per quadrant) split
    // the NP acc2 columns.
    const int q = warp & 3, sub = warp >> 2;
    const int grp = warp >> 3, half = (warp >> 2) & 1;
    const int row = q * 32 + lane;
    const uint32_t tq = (uint32_t)(q * 32) << 16;
    constexpr int NCH = NP / 16;
    const int ch_lo = (NCH * sub) / 4, ch_hi = (NCH * (sub + 1)) / 4;
    const uint32_t a1empty0 = rcx::map_cta(a1empty, 0), a2full0 = rcx::map_cta(a2full, 0);
    const uint32_t c2empty0 = rcx::map_cta(c2empty, 0);
    uint8_t *stg_base = sST + warp * 2 * 1024;
    uint32_t nst = 0, g0 = 0;
    int it = 0;
    for (int tile = cl; tile < total; tile += ncl, ++it, g0 += C) {
      const int pass = tile % a.passes, rest = tile / a.passes;
      const int mp = rest % pairs, net = rest / pairs;
      for (int c = (int)((grp + 2 - (g0 & 1)) & 1); c < C; c += 2) {
        const uint32_t n = g0 + c;                       // global h1 chunk index, n % 2 == grp
        rcx::mbar_wait(&a1full[grp], (n >> 1) & 1);
        if (leader && warp == 0 && lane == 0) dbg_rec(a.dbg, 2, it, c);
        rcx::tc_fence_after();
        uint32_t v[32];
        tmem_ld32(tmem + ACC1_COL + tq + half * 32, v);
        rcx::tmem_ld_wait();
        rcx::tc_fence_before();
        __syncwarp();
        if (lane == 0) rcx::mbar_arrive_cluster(a1empty0);
        uint32_t pk[16];
        if (a.flags & 4) {  // diagnostic: no GELU math
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = cvt_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) pk[j] = gelu_bf16x2(cvt_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1])));
        }
        const int slot = n % A2_SLOTS;
        rcx::mbar_wait(&a2empty[slot], ((n / A2_SLOTS) & 1) ^ 1);
        uint8_t *dst = sA2 + slot * A2_BYTES + row * 128;
        if (!(a.flags & 16)) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4 *>(dst + (((half * 4 + j) ^ (row & 7)) << 4)) =
                make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
        if (!(a.flags & 8)) fence_async_smem();
        __syncwarp();
        if (lane == 0) rcx::mbar_arrive_cluster(a2full0 + slot * 8);
        if (leader && warp == 0 && lane == 0) dbg_rec(a.dbg, 3, it, c);
      }
      // ---- drain acc2 of this tile (this CTA's 128 rows), b2 + GELU -> h2 via TMA stores
      rcx::mbar_wait(c2full, it & 1);
      rcx::mbar_wait(&bfull[it & 1], (it >> 1) & 1);
      if (leader && warp == 0 && lane == 0) dbg_rec(a.dbg, 4, it, 0);
      rcx::tc_fence_after();
      const float *b2 = sB2 + (it & 1) * NP;
      const int grow = mp * 256 + rank * 128 + q * 32;   // first global row of this warp's 32 rows
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
          if (lane == 0) rcx::mbar_arrive_cluster(c2empty0);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1 && !two) break;
          const int col = (cc + h) * 16;
          const float4 *bb = reinterpret_cast<const float4 *>(b2 + col);
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float4 b = bb[j];
            pk[2 * j] = gelu_bf16x2(cvt_bf16x2(__uint_as_float(v[16 * h + 4 * j]) + b.x,
                                               __uint_as_float(v[16 * h + 4 * j + 1]) + b.y));
            pk[2 * j + 1] = gelu_bf16x2(cvt_bf16x2(__uint_as_float(v[16 * h + 4 * j + 2]) + b.z,
                                                   __uint_as_float(v[16 * h + 4 * j + 3]) + b.w));
          }
          // staging buffer (alternates per store): [32 rows][32 B], 32-byte TMA swizzle
          uint8_t *stg = stg_base + (nst & 1) * 1024;
          if (lane == 0) bulk_wait_read<1>();       // the store that last used this buffer has read it
          __syncwarp();
          *reinterpret_cast<uint4 *>(stg + lane * 32 + ((0 ^ ((lane >> 2) & 1)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          *reinterpret_cast<uint4 *>(stg + lane * 32 + ((1 ^ ((lane >> 2) & 1)) << 4)) = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&mapH2, stg, pass * NP + col, grow, net);
            bulk_commit();
          }
          ++nst;
        }
      }
      __syncwarp();
      if (lane == 0) rcx::mbar_arrive(&bempty[it & 1]);
      if (leader && warp == 0 && lane == 0) dbg_rec(a.dbg, 4, it, 1);
    }
    if (lane == 0) bulk_wait_all();  // h2 stores complete before the CTA's shared memory goes away
    __syncwarp();
  }
  rcx::tc_fence_before();
  rcx::cluster_sync();
  if (warp == W_MMA) {
    rcx::tc_fence_after();
    rcx::tmem_dealloc_pair(tmem, 512);
  }
}

template <int NP, int KZ>
int launch_l12_pair_t(const CUtensorMap &Z, const CUtensorMap &W1, const CUtensorMap &W2a, const CUtensorMap &W2b,
                      const CUtensorMap &H2, L12Args a, cudaStream_t s) {
  constexpr size_t Z_BYTES = 128 * KZ * 2, A2 = 128 * C1 * 2;
  constexpr size_t STAGE = (((NP / 2) * C1 * 2 + (C1 / 2) * KZ * 2) + 1023) & ~(size_t)1023;
  const size_t fixed = 1024 + A2_SLOTS * A2 + 2 * Z_BYTES + NEPI * 2 * 1024 + 2 * NP * 4 + 512;
  int stages = (int)((232448 - fixed) / STAGE);
  if (stages > 8) stages = 8;
  if (stages < 2) return rc_fail(RC_EUNSUPPORTED, "fused L1/L2 (pair): pass width %d does not fit", NP);
  a.stages = stages;
  const size_t smem = fixed + stages * STAGE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(l12_pair_kernel<NP, KZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    attr = true;
  }
  const int total = a.nets * (a.m_tiles / 2) * a.passes;
  int clusters = mlp_num_sms() / 2;
  if (clusters > total) clusters = total;
  l12_pair_kernel<NP, KZ><<<2 * clusters, L12_THREADS, smem, s>>>(Z, W1, W2a, W2b, H2, a);
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

int launch_l12_pair(int NP, int KZ, const CUtensorMap &Z, const CUtensorMap &W1, const CUtensorMap &W2a,
                    const CUtensorMap &W2b, const CUtensorMap &H2, const L12Args &a, cudaStream_t s) {
  ProfScope prof(RC_STAGE_L2, s);
#define RC_L12P(np)                                                                                     \
  if (NP == np)                                                                                         \
    return KZ == 16 ? launch_l12_pair_t<np, 16>(Z, W1, W2a, W2b, H2, a, s)                             \
                    : launch_l12_pair_t<np, 32>(Z, W1, W2a, W2b, H2, a, s);
  RC_L12P(400)
  RC_L12P(256)
  RC_L12P(208)
  RC_L12P(128)
  RC_L12P(64)
  RC_L12P(32)
#undef RC_L12P
  return rc_fail(RC_EUNSUPPORTED, "fused L1/L2 (pair): no instance for pass width %d", NP);
}

