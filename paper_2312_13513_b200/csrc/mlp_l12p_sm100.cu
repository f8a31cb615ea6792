// mlp_l12p_sm100.cu -- layers 1 and 2 of the per-species MLP fused on one CTA pair
// (inputs -> 1600 -> 800, GELU), bf16, h1 never leaves shared memory:
//
//   h2[:, pass] = GELU( GELU(z W1^T) W2[pass]^T + b2[pass] )   (W1 stored halved, b1 folded)
//
// The four-CTA kernel (mlp_l12_sm100.cu) shares each h1 chunk between two pairs (one per layer-2
// pass of 400 outputs), but a cluster of four must sit inside one GPC and only 33 of them fit
// (132 of 148 SMs).  Here a tile is (row block of 256 cells, net, pass) and one CTA pair computes
// every h1 chunk it needs itself: the layer-1 work (K = 16) is 1% of the layer-2 MMAs, and the
// h1 GELU doubles (per CTA and 64-column chunk 8192 MUFU ops against ~1000 clk of layer-2 MMAs).
// Clusters of two fit on all 148 SMs, there is no DSMEM exchange and no cross-pair barrier.
//
// One MMA thread issues both layers in one stream, layer 1 two chunks ahead of layer 2:
//
//   queue order: ... L2(c-2) L1(c+1) | L2(c-1) L1(c+2) | L2(c) L1(c+3) ...
//   iteration c: wait a1empty (producers loaded acc1 of chunk c+1), issue L1(c+2); wait ready(c)
//   (slot c produced, W2 stage c loaded), issue L2(c)
//
// so L1(c+2) executes as soon as L2(c-1) is done and the producers have two chunk periods to turn
// it into slot c+2 (TMEM holds one 64-column layer-1 accumulator next to the 400 of layer 2; the
// producers load it long before the next layer-1 MMA overwrites it).  Stage s of chunk g holds
// W2(g) and the W1 rows of chunk g+2 (the layer-1 B operand, 32 rows x KZ per CTA), so one
// barrier per chunk covers both layers; the first two chunks' W1 rows have their own buffers.
// Every mbarrier wait costs the issuing thread ~70-140 clk even when the phase is complete.
//
// Warps: 0..7 h1 producers (TMEM -> GELU -> A slot), 8..15 acc2 drain (as in mlp_l12_sm100.cu:
// b2 folded into the MMAs, two-piece release, GELU + TMA stores under the next tile's MMAs),
// 16 TMA producer, 17 MMA issuer (even CTA), 18 slot forwarder, 19 idle.
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "mlp_common.cuh"
#include "mlp_internal.h"

namespace {

constexpr int NEPI = 16, NPROD = 8, NDRAIN = NEPI - NPROD;
constexpr int W_TMA = NEPI, W_MMA = NEPI + 1, W_FWD = NEPI + 2;
constexpr int LP_THREADS = 32 * (NEPI + 4);
constexpr int NP = 400, P1 = 256, P2 = 144, H1 = P1 / 2, H2 = P2 / 2;  // pass width and its two MMA pieces
constexpr uint32_t SLOT = 128 * 128;      // [128 rows][64 bf16] h1 chunk, 128-byte swizzle (16 KB)
constexpr uint32_t W2T = (NP / 2) * 128;  // W2 chunk tile of one CTA: 200 rows x 128 B (25.6 KB)
constexpr uint32_t TMEM_ACC1 = 448;       // acc2 uses [0, 400)
constexpr uint32_t BK_BYTES = (NP / 2) * 32, BK_AL = 7168;  // b2 as a K = 16 operand: 200 rows x 32 B

using rcm::cvt_bf16x2;
using rcm::gelu_bf16x2;

#ifdef L12TRACE  // timing experiment: clock64 stamps of pair 0, first 64 chunks (tools/l12ptrace.py)
__device__ long long g_l12ptrace[2][4][64][4];  // [cta rank][role: 0 MMA, 1 producer warp 0, 2 drain warp 8][chunk|tile][event]
#define TRP(role, ch, ev)                                                                      \
  do {                                                                                         \
    if (blockIdx.x < 2 && (ch) < 64 && lane == 0) g_l12ptrace[blockIdx.x & 1][role][ch][ev] = clock64(); \
  } while (0)
#else
#define TRP(role, ch, ev) \
  do {                    \
  } while (0)
#endif

template <int KZ, int R>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(LP_THREADS, 1)
    l12p_kernel(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapW1,
                const __grid_constant__ CUtensorMap mapW2a, const __grid_constant__ CUtensorMap mapW2b,
                const __grid_constant__ CUtensorMap mapOut, const __grid_constant__ CUtensorMap mapBa,
                const __grid_constant__ CUtensorMap mapBb, L12Args a) {
  constexpr uint32_t Z_BYTES = 128 * KZ * 2, Z_AL = (Z_BYTES + 1023u) & ~1023u;
  constexpr uint32_t W1_CH = 32 * KZ * 2;                         // W1 rows of one chunk, this CTA
  constexpr uint32_t STAGE = (W2T + W1_CH + 1023u) & ~1023u;      // [W2 tile | W1 rows of chunk g+2]
  static_assert(NP == 400 && P1 == 256, "drain split below assumes 25 column groups, 16 in piece 1");

  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = rcx::smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  uint8_t *sW = smem;                           // R x stage
  uint8_t *sA = sW + R * STAGE;                 // R x SLOT
  uint8_t *sZ = sA + R * SLOT;                  // 2 x z tile
  uint8_t *sW1 = sZ + 2 * Z_AL;                 // W1 rows of chunks 0 and 1 (1 KB each, 2 KB at KZ = 32)
  uint8_t *sST = sW1 + 2 * W1_CH;               // 8 drain warps x 2 x 1 KB h2 staging
  uint8_t *sBK = sST + NDRAIN * 2 * 1024;       // 2 x b2 operand tile (with the z tile of the same buffer)
  uint8_t *sOnes = sBK + 2 * BK_AL;             // 128 rows x 16 bf16 ones: the A side of the b2 MMA
  uint64_t *bar = reinterpret_cast<uint64_t *>(sOnes + 4096);
  // ready[s] (leader): stage s loaded in both CTAs (2 TMA arrivals + bytes) and slot s written in
  //   both CTAs (2 forwarder arrivals).  own[s]: the 8 local producers wrote slot s.  freed[s]: the
  //   layer-2 MMAs of the chunk in stage/slot s completed (both CTAs).
  uint64_t *ready = bar, *freed = ready + R, *own = freed + R, *zfull = own + R, *zempty = zfull + 2,
           *a1full = zempty + 2, *a1empty = a1full + 1, *c2full = a1empty + 1, *c2empty = c2full + 1,
           *c2emptyB = c2empty + 1, *w1full = c2emptyB + 1;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(w1full + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = rcx::cluster_rank();  // rank in the pair
  if (warp == W_TMA && lane == 0) {
    rcx::prefetch_tmap(&mapZ);
    rcx::prefetch_tmap(&mapW1);
    rcx::prefetch_tmap(&mapW2a);
    rcx::prefetch_tmap(&mapW2b);
    rcx::prefetch_tmap(&mapOut);
    rcx::prefetch_tmap(&mapBa);
    rcx::prefetch_tmap(&mapBb);
    for (int r = 0; r < R; ++r) {
      rcx::mbar_init(&ready[r], 4);
      rcx::mbar_init(&freed[r], 1);
      rcx::mbar_init(&own[r], NPROD);
    }
    for (int z = 0; z < 2; ++z) {
      rcx::mbar_init(&zfull[z], 2);
      rcx::mbar_init(&zempty[z], 1);
    }
    rcx::mbar_init(a1full, 1);
    rcx::mbar_init(a1empty, 2 * NPROD);
    rcx::mbar_init(c2full, 1);
    rcx::mbar_init(c2empty, 2 * NDRAIN);   // piece 1: the drain warps of both CTAs
    rcx::mbar_init(c2emptyB, 2 * NDRAIN);  // piece 2
    for (int r = 0; r < 2; ++r) rcx::mbar_init(&w1full[r], 2);
    rcx::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < 1024; i += LP_THREADS) reinterpret_cast<uint32_t *>(sOnes)[i] = 0x3F803F80u;
  rcm::fence_async_smem();  // the ones tile is read by the tensor core (async proxy)
  if (warp == W_MMA) rcx::tmem_alloc_pair(tmem_slot, 512);
  rcx::tc_fence_before();
  rcx::cluster_sync();
  rcx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int C = a.chunks;  // 64-column h1 chunks (K chunks of layer 2)
  const int pairs = a.m_tiles / 2;
  const int total = a.nets * pairs * 2;  // (net, row block, pass)
  const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int ntiles = cl < total ? (total - 1 - cl) / ncl + 1 : 0;
  const uint32_t nchunks = (uint32_t)ntiles * C;
  // tile it of this pair -> (net, row block, pass)
  auto tile_of = [&](int it, int &net, int &mp, int &pass) {
    const int t = cl + it * ncl;
    pass = t & 1;
    mp = (t >> 1) % pairs;
    net = (t >> 1) / pairs;
  };

  if (warp >= NEPI) {
    rcx::setmaxnreg_dec<48>();
    if (warp == W_TMA && lane == 0) {  // ---------------------------------------- TMA producer (both CTAs)
      const uint32_t ready0 = rcx::map_cta(ready, 0), zfull0 = rcx::map_cta(zfull, 0);
      // z tile and b2 operand tile of tile it (pair TMA, counted on the leader's zfull)
      auto load_zb = [&](int it) {
        int net, mp, pass;
        tile_of(it, net, mp, pass);
        const int zb = it & 1;
        rcx::mbar_wait_sleep(&zempty[zb], ((it >> 1) & 1) ^ 1);
        rcx::mbar_arrive_expect_tx_cluster(zfull0 + zb * 8, Z_BYTES + BK_BYTES);
        rcx::tma_load_3d_pair(sZ + zb * Z_AL, &mapZ, &zfull[zb], 0, mp * 256 + (int)rank * 128, 0);
        rcx::tma_load_3d_pair(sBK + zb * BK_AL, &mapBa, &zfull[zb], 0, pass * NP + (int)rank * H1, net);
        rcx::tma_load_3d_pair(sBK + zb * BK_AL + H1 * 32, &mapBb, &zfull[zb], 0, pass * NP + P1 + (int)rank * H2, net);
      };
      // W1 rows of chunk g (global): rows c*64 + 32 rank .. + 32 of its net (B of the M = 256, N = 64 MMA)
      auto w1_rows = [&](uint32_t g, int &row, int &net) {
        int mp, pass;
        tile_of((int)(g / C), net, mp, pass);
        row = (int)(g % C) * 64 + (int)rank * 32;
      };
      if (ntiles > 0) {
        load_zb(0);
        for (uint32_t g = 0; g < 2 && g < nchunks; ++g) {
          int row, net;
          w1_rows(g, row, net);
          rcx::mbar_arrive_expect_tx_cluster(rcx::map_cta(&w1full[g], 0), W1_CH);
          rcx::tma_load_3d_pair(sW1 + g * W1_CH, &mapW1, &w1full[g], 0, row, net);
        }
      }
      for (uint32_t g = 0; g < nchunks; ++g) {
        const int it = (int)(g / C), c = (int)(g % C);
        int net, mp, pass;
        tile_of(it, net, mp, pass);
        const int s = (int)(g % R);
        const bool w1 = g + 2 < nchunks;
        rcx::mbar_wait_sleep(&freed[s], ((g / R) & 1) ^ 1);
        rcx::mbar_arrive_expect_tx_cluster(ready0 + s * 8, W2T + (w1 ? W1_CH : 0));
        uint8_t *st = sW + s * STAGE;
        rcx::tma_load_3d_pair(st, &mapW2a, &ready[s], c * 64, pass * NP + (int)rank * H1, net);
        rcx::tma_load_3d_pair(st + H1 * 128, &mapW2b, &ready[s], c * 64, pass * NP + P1 + (int)rank * H2, net);
        if (w1) {
          int row, wnet;
          w1_rows(g + 2, row, wnet);
          rcx::tma_load_3d_pair(st + W2T, &mapW1, &ready[s], 0, row, wnet);
        }
        if (c == C / 2 && it + 1 < ntiles) load_zb(it + 1);
      }
    } else if (warp == W_MMA && rank == 0) {  // ------ MMA issuer (even CTA; converged warp, elected lane issues)
      constexpr uint32_t id1 = rcx::make_idesc(1u, 256, 64);
      constexpr uint32_t idp1 = rcx::make_idesc(1u, 256, P1), idp2 = rcx::make_idesc(1u, 256, P2);
      // layer 1 of chunk g (tile it, chunk c of the tile): acc1 = z(tile) W1(chunk)^T
      auto issue_l1 = [&](uint32_t g, int it, int c, const uint8_t *w1) {
        const int zb = it & 1;
        TRP(3, g, 0);
        if (c == 0) rcx::mbar_wait(&zfull[zb], (it >> 1) & 1);
        TRP(3, g, 1);
        rcx::mbar_wait(a1empty, (g & 1) ^ 1);  // producers loaded acc1 of chunk g-1
        TRP(3, g, 2);
        rcx::tc_fence_after();
        const uint64_t dz = rcm::desc_sw<KZ * 2>(sZ + zb * Z_AL), dw = rcm::desc_sw<KZ * 2>(w1);
        if (rcx::elect_one()) {
#pragma unroll
          for (int k = 0; k < KZ / 16; ++k) rcx::mma_bf16_pair(tmem + TMEM_ACC1, dz + 2 * k, dw + 2 * k, id1, k != 0);
          rcx::mma_commit_pair(a1full);
          // the z / b2 buffer of a tile is released after its last layer-1 MMA (the b2 MMA, issued at
          // the tile's first layer-2 chunk, precedes it in this thread's order when C >= 3)
          if (c == C - 1) rcx::mma_commit_pair(&zempty[zb]);
        }
        __syncwarp();
        TRP(3, g, 3);
      };
      for (uint32_t g = 0; g < 2 && g < nchunks; ++g) {
        rcx::mbar_wait(&w1full[g], 0);
        issue_l1(g, (int)(g / C), (int)(g % C), sW1 + g * W1_CH);
      }
      int it = 0, c = 0, it2 = (int)(2 / C), c2 = (int)(2 % C);  // (it, c) of chunk g and of chunk g + 2
      for (uint32_t g = 0; g < nchunks; ++g) {
        const int s = (int)(g % R);
        TRP(0, g, 0);
        rcx::mbar_wait(&ready[s], (g / R) & 1);  // slot g produced; W2(g) and W1(g+2) loaded
        TRP(0, g, 1);
        rcx::tc_fence_after();
        uint8_t *A = sA + s * SLOT, *B = sW + s * STAGE;
        if (g + 2 < nchunks) issue_l1(g + 2, it2, c2, B + W2T);
        TRP(0, g, 2);
        const uint64_t da = rcm::desc_sw<128>(A), db = rcm::desc_sw<128>(B);
        if (c == 0) {
          // first chunk of a tile: the accumulator starts at b2 (ones x b2 operand); piece 1 restarts
          // as soon as the drain copied it out, then the pieces are interleaved again
          const int zb = it & 1;
          const uint64_t d1 = rcm::desc_sw<32>(sOnes), dbk = rcm::desc_sw<32>(sBK + zb * BK_AL);
          rcx::mbar_wait_sleep(c2empty, (it & 1) ^ 1);
          rcx::tc_fence_after();
          if (rcx::elect_one()) {
            rcx::mma_bf16_pair(tmem, d1, dbk, idp1, 0);
            rcx::mma_bf16_pair(tmem, da, db, idp1, 1);
          }
          __syncwarp();
          rcx::mbar_wait(c2emptyB, (it & 1) ^ 1);
          rcx::tc_fence_after();
          if (rcx::elect_one()) {
            rcx::mma_bf16_pair(tmem + P1, d1, dbk + ((H1 * 32) >> 4), idp2, 0);
            rcx::mma_bf16_pair(tmem + P1, da, db + ((H1 * 128) >> 4), idp2, 1);
#pragma unroll
            for (int k = 1; k < 4; ++k) {
              rcx::mma_bf16_pair(tmem, da + 2 * k, db + 2 * k, idp1, 1);
              rcx::mma_bf16_pair(tmem + P1, da + 2 * k, db + ((H1 * 128) >> 4) + 2 * k, idp2, 1);
            }
          }
          __syncwarp();
        } else {
          if (rcx::elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // K16 steps: 32-byte atoms along the 128-byte rows
              rcx::mma_bf16_pair(tmem, da + 2 * k, db + 2 * k, idp1, 1);
              rcx::mma_bf16_pair(tmem + P1, da + 2 * k, db + ((H1 * 128) >> 4) + 2 * k, idp2, 1);
            }
          }
          __syncwarp();
        }
        if (rcx::elect_one()) {
          rcx::mma_commit_pair(&freed[s]);
          if (c == C - 1) rcx::mma_commit_pair(c2full);
        }
        __syncwarp();
        TRP(0, g, 3);
        if (++c == C) c = 0, ++it;
        if (++c2 == C) c2 = 0, ++it2;
      }
    } else if (warp == W_FWD && lane == 0) {  // ------------ slot s written here -> the leader's ready[s]
      const uint32_t ready0 = rcx::map_cta(ready, 0);
      for (uint32_t g = 0; g < nchunks; ++g) {
        const int s = (int)(g % R);
        rcx::mbar_wait(&own[s], (g / R) & 1);
        rcx::mbar_arrive_cluster(ready0 + s * 8);
      }
    }
  } else if (warp < NPROD) {  // -------------------------------------------- h1 producers, warps 0..7
    rcx::setmaxnreg_dec<72>();
    const int q = warp & 3, ph = (warp >> 2) & 1;  // ph: 32-column half of the 64-column chunk
    const uint32_t tq = (uint32_t)(q * 32) << 16;
    const uint32_t a1empty0 = rcx::map_cta(a1empty, 0);
    const int row = q * 32 + lane;
    for (uint32_t g = 0; g < nchunks; ++g) {
      if (warp == 0) TRP(1, g, 0);
      rcx::mbar_wait(a1full, g & 1);
      if (warp == 0) TRP(1, g, 1);
      rcx::tc_fence_after();
      uint32_t v[2][16];
      rcx::tmem_ld16(tmem + tq + TMEM_ACC1 + ph * 32, v[0]);
      rcx::tmem_ld16(tmem + tq + TMEM_ACC1 + ph * 32 + 16, v[1]);
      rcx::tmem_ld_wait();
      rcx::tc_fence_before();
      __syncwarp();
      if (lane == 0) rcx::mbar_arrive_cluster(a1empty0);
      uint32_t pk[2][8];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          pk[h][j] = rcm::gelu_half_bf16x2(cvt_bf16x2(__uint_as_float(v[h][2 * j]), __uint_as_float(v[h][2 * j + 1])));
      const int s = (int)(g % R);
      rcx::mbar_wait(&freed[s], ((g / R) & 1) ^ 1);  // the layer-2 MMAs of chunk g - R are done with the slot
      if (warp == 0) TRP(1, g, 2);
      // columns [32 ph, 32 ph + 32) of the chunk = 16-byte units 4 ph .. 4 ph + 3 of the 128-byte row
      uint8_t *r = sA + s * SLOT + row * 128;
      const int x = row & 7;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        *reinterpret_cast<uint4 *>(r + (((4 * ph + u) ^ x) << 4)) =
            make_uint4(pk[u >> 1][4 * (u & 1)], pk[u >> 1][4 * (u & 1) + 1], pk[u >> 1][4 * (u & 1) + 2],
                       pk[u >> 1][4 * (u & 1) + 3]);
      rcm::fence_async_smem();
      __syncwarp();
      if (lane == 0) rcx::mbar_arrive(&own[s]);
      if (warp == 0) TRP(1, g, 3);
    }
  } else {  // ------------------------------------------------------ acc2 drain, warps 8..15
    rcx::setmaxnreg_inc<144>();
    // two warps per TMEM lane quadrant; warp half hh drains column groups (16 columns) 8hh..8hh+7
    // of piece 1 and then 16..20 (hh = 0) or 21..24 (hh = 1) of piece 2, released separately
    const int w = warp - NPROD, q = w & 3, hh = w >> 2;
    const uint32_t tq = (uint32_t)(q * 32) << 16;
    const int nch = 13 - hh;
    auto grp = [&](int c) { return c < 8 ? 8 * hh + c : 16 + 5 * hh + (c - 8); };
    const uint32_t c2empty0 = rcx::map_cta(c2empty, 0), c2emptyB0 = rcx::map_cta(c2emptyB, 0);
    uint8_t *stg_base = sST + w * 2 * 1024;  // two 1 KB TMA-store staging buffers per warp
    uint32_t nst = 0;
    for (int it = 0; it < ntiles; ++it) {
      int net, mp, pass;
      tile_of(it, net, mp, pass);
      rcx::mbar_wait_sleep(c2full, it & 1);
      if (warp == 8) TRP(2, it, 0);
      rcx::tc_fence_after();
      const int grow = mp * 256 + (int)rank * 128 + q * 32;
      uint32_t pk[13][8];
      auto cvt = [&](const uint32_t *v, int c, int n) {  // n groups from v (b2 already included)
#pragma unroll
        for (int h = 0; h < n; ++h)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            pk[c + h][j] = cvt_bf16x2(__uint_as_float(v[16 * h + 2 * j]), __uint_as_float(v[16 * h + 2 * j + 1]));
      };
#pragma unroll
      for (int c = 0; c < 8; c += 4) {  // piece 1: two rounds of two 32-column loads in flight
        uint32_t v[64];
        rcm::tmem_ld32(tmem + tq + grp(c) * 16, *reinterpret_cast<uint32_t(*)[32]>(v));
        rcm::tmem_ld32(tmem + tq + grp(c + 2) * 16, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        rcx::tmem_ld_wait();
        cvt(v, c, 4);
      }
      rcx::tc_fence_before();
      __syncwarp();
      if (lane == 0) rcx::mbar_arrive_cluster(c2empty0);
#pragma unroll
      for (int c = 8; c < 12; c += 2) {  // piece 2: groups 8..11, then group 12 (hh = 0)
        uint32_t v[32];
        rcm::tmem_ld32(tmem + tq + grp(c) * 16, v);
        rcx::tmem_ld_wait();
        cvt(v, c, 2);
      }
      if (hh == 0) {
        uint32_t v[16];
        rcx::tmem_ld16(tmem + tq + grp(12) * 16, v);
        rcx::tmem_ld_wait();
        cvt(v, 12, 1);
      }
      rcx::tc_fence_before();
      __syncwarp();
      if (lane == 0) rcx::mbar_arrive_cluster(c2emptyB0);
      if (warp == 8) TRP(2, it, 1);
      // phase 2: GELU and TMA stores (32 rows x 16 columns per store) under the next tile's MMAs
#pragma unroll
      for (int c = 0; c < 13; ++c) {
        if (c < nch) {
          uint32_t gg[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) gg[j] = gelu_bf16x2(pk[c][j]);
          uint8_t *stg = stg_base + (nst & 1) * 1024;
          if (lane == 0) rcm::bulk_wait_read1();
          __syncwarp();
          const int sw = (lane >> 2) & 1;
          *reinterpret_cast<uint4 *>(stg + lane * 32 + (sw << 4)) = make_uint4(gg[0], gg[1], gg[2], gg[3]);
          *reinterpret_cast<uint4 *>(stg + lane * 32 + ((sw ^ 1) << 4)) = make_uint4(gg[4], gg[5], gg[6], gg[7]);
          rcm::fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            rcm::tma_store_3d(&mapOut, stg, pass * NP + grp(c) * 16, grow, net);
            rcm::bulk_commit();
          }
          ++nst;
        }
      }
    }
    if (lane == 0) rcm::bulk_wait_all();
    __syncwarp();
  }
  rcx::tc_fence_before();
  rcx::cluster_sync();
  if (warp == W_MMA) {
    rcx::tc_fence_after();
    rcx::tmem_dealloc_pair(tmem, 512);
  }
}

template <int KZ>
int launch_t(const CUtensorMap *M, L12Args a, cudaStream_t s) {
  constexpr int R = KZ == 16 ? 4 : 3;
  constexpr size_t Z_AL = ((size_t)128 * KZ * 2 + 1023) & ~(size_t)1023;
  constexpr size_t W1_CH = (size_t)32 * KZ * 2;
  constexpr size_t STAGE = ((size_t)W2T + W1_CH + 1023) & ~(size_t)1023;
  const size_t smem = 1024 + R * (SLOT + STAGE) + 2 * Z_AL + 2 * W1_CH + NDRAIN * 2 * 1024 +
                      2 * BK_AL + 4096 + 1024;
  if (smem > 232448) return rc_fail(RC_EUNSUPPORTED, "pair-local fused layer-1/2 kernel: shared memory");
  a.stages = R;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(l12p_kernel<KZ, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    attr = true;
  }
  static int resident = 0;  // CTA pairs that fit at once (a persistent grid must not need a second wave)
  if (!resident) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (mlp_num_sms() / 2));
    cfg.blockDim = dim3(LP_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&resident, l12p_kernel<KZ, R>, &cfg) != cudaSuccess || resident <= 0)
      resident = mlp_num_sms() / 2;
    if (getenv("RC_VERBOSE")) fprintf(stderr, "pair-local fused layer-1/2 kernel: %d resident CTA pairs\n", resident);
  }
  const int total = a.nets * (a.m_tiles / 2) * 2;
  int clusters = resident;
  if (clusters > total) clusters = total;
  l12p_kernel<KZ, R><<<2 * clusters, LP_THREADS, smem, s>>>(M[0], M[1], M[2], M[3], M[4], M[5], M[6], a);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

}  // namespace

#ifdef L12TRACE
extern "C" __attribute__((visibility("default"))) int rc_debug_l12ptrace(void *host) {
  return (int)cudaMemcpyFromSymbol(host, g_l12ptrace, sizeof(g_l12ptrace));
}
#endif

int launch_l12p(int KZ, const CUtensorMap *maps, const L12Args &a, cudaStream_t s) {
  ProfScope prof(RC_STAGE_L12, s);
  if (KZ == 16) return launch_t<16>(maps, a, s);
  if (KZ == 32) return launch_t<32>(maps, a, s);
  return rc_fail(RC_EUNSUPPORTED, "pair-local fused layer-1/2 kernel: K = %d", KZ);
}
