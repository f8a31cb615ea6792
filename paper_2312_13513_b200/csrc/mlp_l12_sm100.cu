// mlp_l12_sm100.cu -- layers 1 and 2 of the per-species MLP fused (PAPER.md:114:
// inputs -> 1600 -> 800, GELU), bf16, so the 1600-wide h1 never goes to HBM:
//
//   h2 = GELU( GELU(z W1^T) W2^T + b2 )      (W1 stored halved, b1 folded, as in layer 1)
//
// A cluster of four CTAs = two CTA pairs owns a 256-cell row block.  Pair p computes the
// layer-2 outputs of pass p (400 of the 800 columns) with the cta_group::2 GEMM of the layer-2
// kernel (M = 256, N = 256 + 144, K chunks of 64).  Both pairs need every 64-column chunk of h1
// for all 256 rows, so the pairs take turns: chunk c is produced by pair c % 2 (a cta_group::2
// M = 256, N = 64, K = KZ layer-1 MMA into a 64-column TMEM accumulator; eight producer warps per
// CTA apply GELU and write the 128 x 64 bf16 chunk, 128-byte swizzled, into the CTA's A slot) and
// a copier thread sends it with one 16 KB DSMEM bulk copy into the same slot of the CTA with the
// same rows in the other pair.  Per CTA and chunk period this costs on average 4096 GELUs (256
// clk of MUFU) against ~900 clk of layer-2 MMA, instead of a separate layer-1 pass writing and
// then re-reading 3.2 KB of h1 per cell and net.  DESIGN.md 6.1 has the measured timeline.
//
// Barriers (per CTA; "leader" = even CTA of a pair, which issues the MMAs):
//   ready[R]        chunk g's W2 stage and A slot g % R complete (leader: both CTAs' W2 bytes,
//                   the slot's writer (own copier or incoming copy bytes), the odd forwarder)
//   freed[R]        both pairs' layer-2 MMAs of the chunk done (commit multicast to all four CTAs)
//   own[R]          the 8 local producer warps wrote this pair's chunk
//   zfull/zempty[2] z tile + b2 operand tile of a tile (pair TMA; prefetched half a tile ahead)
//   a1full/a1empty  layer-1 accumulator (commit -> pair; 16 producer warps of the pair)
//   w1full/w1empty  this CTA's W1 rows of a net
//   c2full, c2empty/c2emptyB  layer-2 accumulator, released in two pieces by the drain warps
// Warps: 0..7 h1 producers, 8..15 acc2 drain, 16 TMA producer, 17 layer-2 MMA issuer,
// 18 chunk copier, 19 layer-1 MMA issuer (even CTA) / slot forwarder (odd CTA).
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "mlp_common.cuh"
#include "mlp_internal.h"

namespace {

constexpr int NEPI = 16, NPROD = 8;
// W_AUX: the layer-1 MMA issuer in the even CTA of a pair, the slot forwarder in the odd one
constexpr int W_TMA = NEPI, W_MMA = NEPI + 1, W_CPY = NEPI + 2, W_AUX = NEPI + 3;
constexpr int L12_THREADS = 32 * (NEPI + 4);
constexpr int NA1 = 1;                        // layer-1 accumulator (64 TMEM columns)
constexpr int NP = 400, P1 = 256, P2 = 144, H1 = P1 / 2, H2 = P2 / 2;  // pass width and its two MMA pieces
constexpr uint32_t SLOT = 128 * 128;         // [128 rows][64 bf16] h1 chunk, 128-byte swizzle (16 KB)
constexpr uint32_t W2T = (NP / 2) * 128;      // W2 chunk tile of one CTA: 200 rows x 128 B (25.6 KB)
constexpr uint32_t TMEM_ACC1 = 448;          // acc2 uses [0, 400)

using rcm::cvt_bf16x2;

#ifdef L12TRACE  // timing experiment: clock64 stamps of cluster 0, first 64 chunks (tools/l12trace.py)
// [cta rank][role: 0 MMA, 1 producer warp 0, 2 forwarder, 3 drain (by tile), 4 layer-1 issuer, 5 TMA (by tile)][chunk][event]
__device__ long long g_l12trace[4][6][64][4];
#define TR(role, ch, ev)                                                                              \
  do {                                                                                                \
    if (blockIdx.x < 4 && (ch) < 64 && lane == 0) g_l12trace[blockIdx.x & 3][role][ch][ev] = clock64(); \
  } while (0)
#else
#define TR(role, ch, ev) \
  do {                   \
  } while (0)
#endif

// R = ring depth: chunk g uses W2 stage and A slot g % R, so one barrier per chunk tells the
// layer-2 issuer that both operands are in place (every wait between MMAs costs a tensor-pipe bubble)
// TF: the TF32 mode (RC_TF32): fp32 (tf32-rounded) operands, kind::tf32 MMAs, a 128-byte operand row
// holds 32 elements, so a chunk is 32 h1 columns (K = 32 of layer 2, the same 4 MMA K atoms of 32
// bytes); erf-form GELU in fp32 with one tf32 rounding; b2 enters as a K = 8 (hi, lo) tf32 operand.
template <int KZ, int R, bool TF>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(L12_THREADS, 1)
    l12_kernel(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapW1,
               const __grid_constant__ CUtensorMap mapW2a, const __grid_constant__ CUtensorMap mapW2b,
               const __grid_constant__ CUtensorMap mapOut, const __grid_constant__ CUtensorMap mapBa,
               const __grid_constant__ CUtensorMap mapBb, L12Args a) {
  constexpr int EB = TF ? 4 : 2;                  // operand element bytes
  constexpr int CW = TF ? 32 : 64;                // h1 columns per chunk: one 128-byte operand row
  constexpr uint32_t FMT = rcm::Elem<TF>::FMT;
  constexpr int KATOM = rcm::Elem<TF>::KATOM;
  constexpr uint32_t Z_BYTES = 128 * KZ * EB, W1_CH = (CW / 2) * KZ * EB;  // W1: CW/2 rows per CTA and chunk
  // KZ = 16 (bf16): this CTA's W1 rows of all its pair's chunks of a net (13 KB, one 5D box per net);
  // KZ = 32 (CH4) and TF32: a 4-deep ring of per-chunk W1 rows (8 KB instead of 26 KB, so the W2/A
  // ring stays 4 deep)
  constexpr bool W1RING = KZ == 32 || TF;
  constexpr uint32_t STGB = TF ? 2048 : 1024;     // h2 store staging buffer: 32 rows x 16 columns
  constexpr int NSTG = TF ? 1 : 2;                // staging buffers per drain warp
  constexpr int RW = 4;
  constexpr uint32_t STAGE_BYTES = W2T;                             // TMA bytes per CTA
  constexpr uint32_t BK_BYTES = (NP / 2) * 32, BK_AL = 7168;        // b2 as a K = 16 operand: 200 rows x 32 B
  constexpr uint32_t STAGE = (W2T + 1023u) & ~1023u;                // layout size
  static_assert(NP == 400 && P1 == 256, "drain split below assumes 25 column groups, 16 in piece 1");

  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = rcx::smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  constexpr int S = R;
  uint8_t *sW = smem;                        // R x W2 chunk tile
  uint8_t *sA = sW + S * STAGE;              // R x SLOT
  uint8_t *sZ = sA + R * SLOT;               // 2 x Z_BYTES
  uint8_t *sW1 = sZ + 2 * ((Z_BYTES + 1023u) & ~1023u);  // this CTA's W1 rows of its pair's chunks of the net
  uint8_t *sST = sW1 + (W1RING ? RW * W1_CH : ((((a.chunks + 1) / 2) * W1_CH + 1023u) & ~1023u));  // drain h2 staging
  uint8_t *sBK = sST + (NEPI - NPROD) * NSTG * STGB;  // 2 x b2 operand tile (with the z tile of the same buffer)
  uint8_t *sOnes = sBK + 2 * BK_AL;                // 128 rows x 16 bf16 ones: the A side of the b2 MMA
  uint64_t *bar = reinterpret_cast<uint64_t *>(sOnes + 4096);
  // ready[i]: leader = both operands of chunk i in both CTAs (its slot: own copier or incoming copy;
  //   the odd forwarder; W2 TMA of both CTAs); odd CTA = its slot.  own[i]: the local producers wrote
  //   slot i (chunks of this pair).  freed[i]: both pairs consumed chunk i's slot and stage.
  uint64_t *ready = bar, *freed = ready + R, *zfull = freed + R, *zempty = zfull + 2, *a1full = zempty + 2,
           *a1empty = a1full + NA1, *own = a1empty + NA1, *c2full = own + R, *c2empty = c2full + 1,
           *c2emptyB = c2empty + 1, *w1full = c2emptyB + 1, *w1empty = w1full + RW;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(w1empty + RW);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = rcx::cluster_rank();
  const int pr = (int)(rank >> 1), prank = (int)(rank & 1);  // pair (= layer-2 pass), rank in the pair
  const uint32_t lead = rank & ~1u, partner = rank ^ 2u;
  const uint16_t pair_mask = (uint16_t)(3u << (2 * pr));
  if (warp == W_TMA && lane == 0) {
    rcx::prefetch_tmap(&mapZ);
    rcx::prefetch_tmap(&mapW1);
    rcx::prefetch_tmap(&mapW2a);
    rcx::prefetch_tmap(&mapW2b);
    rcx::prefetch_tmap(&mapOut);
    rcx::prefetch_tmap(&mapBa);
    rcx::prefetch_tmap(&mapBb);
    for (int r = 0; r < R; ++r) {
      rcx::mbar_init(&ready[r], prank == 0 ? 4 : 1);
      rcx::mbar_init(&freed[r], 2);
      rcx::mbar_init(&own[r], NPROD);
    }
    for (int j = 0; j < RW; ++j) {
      rcx::mbar_init(&w1full[j], 2);
      rcx::mbar_init(&w1empty[j], 1);
    }
    for (int z = 0; z < 2; ++z) {
      rcx::mbar_init(&zfull[z], 2);
      rcx::mbar_init(&zempty[z], 1);
    }
    for (int z = 0; z < NA1; ++z) {
      rcx::mbar_init(&a1full[z], 1);
      rcx::mbar_init(&a1empty[z], 2 * NPROD);
    }
    rcx::mbar_init(c2full, 1);
    rcx::mbar_init(c2empty, 2 * (NEPI - NPROD));  // piece 1: the drain warps of both CTAs
    rcx::mbar_init(c2emptyB, 2 * (NEPI - NPROD));  // piece 2
    rcx::fence_mbar_init();
  }
  // the ones tile: 128 rows x 32 bytes of 1.0 (bf16 pairs or fp32)
  for (int i = threadIdx.x; i < 1024; i += L12_THREADS) reinterpret_cast<uint32_t *>(sOnes)[i] = TF ? 0x3F800000u : 0x3F803F80u;
  rcm::fence_async_smem();  // the ones tile is read by the tensor core (async proxy)
  if (warp == W_MMA) rcx::tmem_alloc_pair(tmem_slot, 512);
  rcx::tc_fence_before();
  rcx::cluster_sync();
  rcx::tc_fence_after();
  // this cluster is resident: count it for the layer-3 filler's gate
  if (a.started && rank == 0 && threadIdx.x == 0) rcx::red_release_gpu_add(a.started, 1);
  const uint32_t tmem = *tmem_slot;
  const int C = a.chunks;  // CW-column h1 chunks (K chunks of layer 2)
  const int pairs = a.m_tiles / 2;
  const int total = a.nets * pairs;
  const int cl = blockIdx.x >> 2, ncl = gridDim.x >> 2;

  // Registers are rebalanced by warpgroup: the single-thread roles (warps 16..19) give registers
  // to the 16 epilogue warps (96 per thread at launch -> 48 / 104).
  if (warp >= NEPI) {
  rcx::setmaxnreg_dec<48>();
  if (warp == W_TMA) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer (all CTAs)
      const uint32_t ready0 = rcx::map_cta(ready, lead), zfull0 = rcx::map_cta(zfull, lead);
      const uint32_t w1full0 = rcx::map_cta(w1full, lead);
      uint32_t g = 0, nw = 0;
      int it = 0, cur_net = -1;
      // z tile and b2 operand tile of the it-th tile: issued half-way through the previous tile, so
      // the layer-1 MMAs of a tile's first chunks never wait for them at the tile transition
      auto load_zb = [&](int tile, int it) {
        const int zb = it & 1, net = tile / pairs;
        TR(5, it, 0);
        rcx::mbar_wait_sleep(&zempty[zb], ((it >> 1) & 1) ^ 1);
        rcx::mbar_arrive_expect_tx_cluster(zfull0 + zb * 8, Z_BYTES + BK_BYTES);
        rcx::tma_load_3d_pair(sZ + zb * ((Z_BYTES + 1023u) & ~1023u), &mapZ, &zfull[zb], 0,
                              (tile % pairs) * 256 + prank * 128, 0);
        rcx::tma_load_3d_pair(sBK + zb * BK_AL, &mapBa, &zfull[zb], 0, pr * NP + prank * H1, net);
        rcx::tma_load_3d_pair(sBK + zb * BK_AL + H1 * 32, &mapBb, &zfull[zb], 0, pr * NP + P1 + prank * H2, net);
        TR(5, it, 1);
      };
      if (cl < total) load_zb(cl, 0);
      // W1RING: this CTA's rows of the pair's own chunks (c % 2 == pr), loaded up to 6 global chunks
      // ahead of the W2 stream (the ring entry of own chunk k is released by its layer-1 MMA)
      const uint32_t nchunks = (uint32_t)(cl < total ? (total - 1 - cl) / ncl + 1 : 0) * C;
      uint32_t wg = (uint32_t)pr, nwr = 0;  // next own chunk (global index), own W1 loads issued
      auto load_w1_upto = [&](uint32_t gmax) {
        for (; wg <= gmax && wg < nchunks; ++nwr) {
          const int wt = cl + (int)(wg / C) * ncl, wc = (int)(wg % C);
          const int j = (int)(nwr % RW);
          rcx::mbar_wait_sleep(&w1empty[j], ((nwr / RW) & 1) ^ 1);
          rcx::mbar_arrive_expect_tx_cluster(w1full0 + j * 8, W1_CH);
          rcx::tma_load_3d_pair(sW1 + j * W1_CH, &mapW1, &w1full[j], 0, wc * CW + prank * (CW / 2), wt / pairs);
          // next own chunk: c + 2 in the tile, else the first own chunk of the next tile
          wg = (wc + 2 < C) ? wg + 2 : (wg / C + 1) * C + (uint32_t)pr;
        }
      };
      for (int tile = cl; tile < total; tile += ncl, ++it) {
        const int net = tile / pairs;
        if (!W1RING && net != cur_net) {  // this CTA's W1 rows of all chunks of the new net (one 5D box)
          rcx::mbar_wait_sleep(w1empty, (nw & 1) ^ 1);
          rcx::mbar_arrive_expect_tx_cluster(w1full0, ((C + 1) / 2) * W1_CH);
          rcx::tma_load_5d_pair(sW1, &mapW1, w1full, 0, 0, pr * 2 + prank, 0, net);  // rows c*64 + 32 prank, c%2 == pr
          cur_net = net;
          ++nw;
        }
        for (int c = 0; c < C; ++c, ++g) {
          const int s = (int)(g % S);
          if (W1RING) load_w1_upto(g + 6);
          rcx::mbar_wait_sleep(&freed[s], ((g / S) & 1) ^ 1);
          rcx::mbar_arrive_expect_tx_cluster(ready0 + s * 8, STAGE_BYTES);
          uint8_t *st = sW + s * STAGE;
          rcx::tma_load_3d_pair(st, &mapW2a, &ready[s], c * CW, pr * NP + prank * H1, net);
          rcx::tma_load_3d_pair(st + H1 * 128, &mapW2b, &ready[s], c * CW, pr * NP + P1 + prank * H2, net);
          if (c == C / 2 && tile + ncl < total) load_zb(tile + ncl, it + 1);
        }
      }
    }
  } else if (warp == W_AUX && prank == 0) {
    {  // ------------------------------ layer-1 MMA issuer (pair leaders; converged warp, elected lane issues)
      // Runs ahead of the layer-2 issuer by up to NA1 chunks (the layer-1 accumulators), so the
      // GELU + DSMEM exchange of a half-chunk overlaps several layer-2 chunk periods.
      constexpr uint32_t id1 = rcx::make_idesc(FMT, 256, CW);
      uint32_t g = 0, nw = 0;
      int it = 0, cur_net = -1;
      for (int tile = cl; tile < total; tile += ncl, ++it) {
        const int zb = it & 1, net = tile / pairs;
        if (!W1RING && net != cur_net) {
          if (cur_net >= 0 && rcx::elect_one()) rcx::mma_commit_pair_mask(w1empty, pair_mask);  // previous net's W1 done
          __syncwarp();
          rcx::mbar_wait(w1full, nw & 1);
          cur_net = net;
          ++nw;
        }
        TR(4, it * C, 0);
        rcx::mbar_wait_sleep(&zfull[zb], (it >> 1) & 1);
        TR(4, it * C, 1);
        const uint64_t dz = rcm::desc_sw<KZ * EB>(sZ + zb * ((Z_BYTES + 1023u) & ~1023u));
        for (int c = pr; c < C; c += 2, ++g) {  // g counts this pair's chunks
          const uint32_t b = g % NA1;
          TR(4, it * C + c, 2);
          rcx::mbar_wait(&a1empty[b], ((g / NA1) & 1) ^ 1);
          TR(4, it * C + c, 3);
          const int j = (int)(g % RW);  // W1RING entry of this own chunk (g counts own chunks)
          if (W1RING) rcx::mbar_wait(&w1full[j], (g / RW) & 1);
          rcx::tc_fence_after();
          const uint64_t dw = rcm::desc_sw<KZ * EB>(W1RING ? sW1 + j * W1_CH : sW1 + (c >> 1) * W1_CH);
          if (rcx::elect_one()) {
#pragma unroll
            for (int k = 0; k < KZ / KATOM; ++k)
              rcm::mma_pair<TF>(tmem + TMEM_ACC1 + b * 64, dz + 2 * k, dw + 2 * k, id1, k != 0);
            rcx::mma_commit_pair_mask(&a1full[b], pair_mask);
            if (W1RING) rcx::mma_commit_pair_mask(&w1empty[j], pair_mask);
          }
          __syncwarp();
        }
        if (rcx::elect_one()) rcx::mma_commit_pair_mask(&zempty[zb], pair_mask);
        __syncwarp();
      }
    }
  } else if (warp == W_MMA) {
    if (prank == 0) {  // ------------------------------------------------ layer-2 MMA issuer (pair leaders)
      // the whole warp runs the loop converged; one elected lane issues (descriptors stay uniform)
      constexpr uint32_t idp1 = rcx::make_idesc(FMT, 256, P1), idp2 = rcx::make_idesc(FMT, 256, P2);
      uint32_t G = 0;
      int it = 0;
      for (int tile = cl; tile < total; tile += ncl, ++it, G += C) {
        for (int c = 0; c < C; ++c) {
          const uint32_t g = G + c;
          const int s = (int)(g % R), slot = s;
          TR(0, g, 0);
          rcx::mbar_wait(&ready[s], (g / R) & 1);  // W2 stage and h1 chunk, both CTAs of the pair
          TR(0, g, 1);
          rcx::tc_fence_after();
          const uint64_t da = rcm::desc_sw<128>(sA + slot * SLOT), db = rcm::desc_sw<128>(sW + s * STAGE);
          if (c == 0) {
            // first chunk of a tile: the accumulator starts at b2 (one K = 16 MMA of a ones tile
            // against the b2 operand tile), and the drain releases it in two pieces, so the
            // piece-1 MMAs (columns [0, 256)) run while piece 2 is still being copied out
            // (one accumulator chain advances ~220 clk per MMA: after the first two piece-1 MMAs
            // the pieces are interleaved again, as in the main loop)
            const int zb = it & 1;
            rcx::mbar_wait(&zfull[zb], (it >> 1) & 1);
            const uint64_t d1 = rcm::desc_sw<32>(sOnes), dbk = rcm::desc_sw<32>(sBK + zb * BK_AL);
            rcx::mbar_wait_sleep(c2empty, (it & 1) ^ 1);
            rcx::tc_fence_after();
            if (rcx::elect_one()) {
              rcm::mma_pair<TF>(tmem, d1, dbk, idp1, 0);
              rcm::mma_pair<TF>(tmem, da, db, idp1, 1);
            }
            __syncwarp();
            rcx::mbar_wait(c2emptyB, (it & 1) ^ 1);
            rcx::tc_fence_after();
            if (rcx::elect_one()) {
              rcm::mma_pair<TF>(tmem + P1, d1, dbk + ((H1 * 32) >> 4), idp2, 0);
              rcm::mma_pair<TF>(tmem + P1, da, db + ((H1 * 128) >> 4), idp2, 1);
#pragma unroll
              for (int k = 1; k < 4; ++k) {
                rcm::mma_pair<TF>(tmem, da + 2 * k, db + 2 * k, idp1, 1);
                rcm::mma_pair<TF>(tmem + P1, da + 2 * k, db + ((H1 * 128) >> 4) + 2 * k, idp2, 1);
              }
              rcx::mma_commit_pair_mask(&freed[s], (uint16_t)0xF);
            }
            __syncwarp();
            TR(0, g, 2);
            continue;
          }
          if (rcx::elect_one()) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // K atoms: 32-byte steps along the 128-byte rows
              rcm::mma_pair<TF>(tmem, da + 2 * k, db + 2 * k, idp1, 1);
              rcm::mma_pair<TF>(tmem + P1, da + 2 * k, db + ((H1 * 128) >> 4) + 2 * k, idp2, 1);
            }
            rcx::mma_commit_pair_mask(&freed[s], (uint16_t)0xF);  // all four CTAs wait for both pairs
          }
          __syncwarp();
          TR(0, g, 2);
        }
        if (rcx::elect_one()) rcx::mma_commit_pair_mask(c2full, pair_mask);
        __syncwarp();
      }
    }
  } else if (warp == W_CPY) {
    if (lane == 0) {  // ------------------------------- this pair's chunks: slot ready here, copy to the other pair
      uint32_t g = 0, my = 0;
      for (int tile = cl; tile < total; tile += ncl)
        for (int c = 0; c < C; ++c, ++g) {
          if ((c & 1) != pr) continue;
          const int slot = (int)(g % R);
          // own[] is indexed by this pair's chunk count (the pair skips every other chunk)
          rcx::mbar_wait_sleep(&own[my % R], (my / R) & 1);  // the local producers wrote the chunk
          ++my;
          rcx::mbar_arrive(&ready[slot]);
          uint8_t *src = sA + slot * SLOT;
          const uint32_t dst_bar = rcx::map_cta(&ready[slot], partner);
          rcx::mbar_arrive_expect_tx_cluster(dst_bar, SLOT);
          rcx::bulk_s2s_cluster(rcx::map_cta(src, partner), src, SLOT, dst_bar);
        }
    }
  } else if (warp == W_AUX) {
    if (lane == 0) {  // ---------------------------------- odd CTA: both halves in place -> leader
      const uint32_t ready_lead = rcx::map_cta(ready, lead);
      uint32_t g = 0;
      for (int tile = cl; tile < total; tile += ncl)
        for (int c = 0; c < C; ++c, ++g) {
          const int slot = (int)(g % R);
          const uint32_t par = (g / R) & 1;
          TR(2, g, 0);
          rcx::mbar_wait_sleep(&ready[slot], par);  // the chunk is in this CTA's slot
          TR(2, g, 2);
          rcx::mbar_arrive_cluster(ready_lead + slot * 8);
        }
    }
  }
  } else if (warp < NPROD) {  // ---------------------------------------- h1 producers, warps 0..7
    rcx::setmaxnreg_dec<72>();
    const int q = warp & 3, ph = (warp >> 2) & 1;  // ph: 32-column half of the 64-column chunk
    const uint32_t tq = (uint32_t)(q * 32) << 16;
    const uint32_t a1empty0 = rcx::map_cta(a1empty, lead);
    const int row = q * 32 + lane;
    const int ntiles = cl < total ? (total - 1 - cl) / ncl + 1 : 0;
    const uint32_t nchunks = (uint32_t)ntiles * C;
    uint32_t lg = 0;  // this pair's chunks produced so far (layer-1 accumulator phase, own[] ring)
    for (uint32_t g = 0; g < nchunks; ++g) {  // this CTA's tiles in order, C chunks each
      if ((int)((g % C) & 1) != pr) continue;  // the other pair's chunk
      const uint32_t b = lg % NA1, my = lg;
      if (warp == 0) TR(1, g, 0);
      rcx::mbar_wait_sleep(&a1full[b], (lg / NA1) & 1);
      if (warp == 0) TR(1, g, 1);
      rcx::tc_fence_after();
      uint8_t *r = sA + (g % R) * SLOT + row * 128;
      const int x = row & 7;
      if constexpr (TF) {  // 16 fp32 columns per warp: GELU, one tf32 rounding
        uint32_t v[16];
        rcx::tmem_ld16(tmem + tq + TMEM_ACC1 + b * 64 + ph * 16, v);
        rcx::tmem_ld_wait();
        rcx::tc_fence_before();
        __syncwarp();
        if (lane == 0) rcx::mbar_arrive_cluster(a1empty0 + b * 8);
        ++lg;
        float y[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) y[j] = rcm::tf32_rn(rcm::gelu_erf_f32(__uint_as_float(v[j])));
        const int slot = (int)(g % R);
        rcx::mbar_wait_sleep(&freed[slot], ((g / R) & 1) ^ 1);  // both pairs are done with the slot
        // columns [16 ph, 16 ph + 16) of the chunk = 16-byte units 4 ph .. 4 ph + 3 of the 128-byte row
#pragma unroll
        for (int u = 0; u < 4; ++u)
          *reinterpret_cast<float4 *>(r + (((4 * ph + u) ^ x) << 4)) = make_float4(y[4 * u], y[4 * u + 1], y[4 * u + 2], y[4 * u + 3]);
      } else {
        uint32_t v[2][16];
        rcx::tmem_ld16(tmem + tq + TMEM_ACC1 + b * 64 + ph * 32, v[0]);
        rcx::tmem_ld16(tmem + tq + TMEM_ACC1 + b * 64 + ph * 32 + 16, v[1]);
        rcx::tmem_ld_wait();
        rcx::tc_fence_before();
        __syncwarp();
        if (lane == 0) rcx::mbar_arrive_cluster(a1empty0 + b * 8);
        ++lg;
        uint32_t pk[2][8];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            pk[h][j] = rcm::gelu_half_f16x2_bf16x2(rcm::cvt_f16x2(__uint_as_float(v[h][2 * j]), __uint_as_float(v[h][2 * j + 1])));
        const int slot = (int)(g % R);
        rcx::mbar_wait_sleep(&freed[slot], ((g / R) & 1) ^ 1);  // both pairs are done with the slot
        if (warp == 0) TR(1, g, 2);
        // columns [32 ph, 32 ph + 32) of the chunk = 16-byte units 4 ph .. 4 ph + 3 of the 128-byte row
#pragma unroll
        for (int u = 0; u < 4; ++u)
          *reinterpret_cast<uint4 *>(r + (((4 * ph + u) ^ x) << 4)) =
              make_uint4(pk[u >> 1][4 * (u & 1)], pk[u >> 1][4 * (u & 1) + 1], pk[u >> 1][4 * (u & 1) + 2],
                         pk[u >> 1][4 * (u & 1) + 3]);
      }
      rcm::fence_async_smem();
      __syncwarp();
      if (lane == 0) rcx::mbar_arrive(&own[my % R]);
      if (warp == 0) TR(1, g, 3);
    }
  } else {  // ------------------------------------------------------ acc2 drain, warps 8..15
    rcx::setmaxnreg_inc<144>();
    // Two warps per TMEM lane quadrant; warp half hh drains column groups (16 columns) 8hh..8hh+7
    // of piece 1 (the N = 256 MMA, columns [0, 256)) and then 16..20 (hh = 0) or 21..24 (hh = 1)
    // of piece 2.  Each piece is released as soon as it is copied out (c2empty / c2emptyB), so the
    // MMA issuer restarts piece 1 of the next tile while piece 2 is still being copied.  The
    // producers never drain: h1 production runs straight through the tile transition.
    const int w = warp - NPROD, q = w & 3, hh = w >> 2;
    const uint32_t tq = (uint32_t)(q * 32) << 16;
    const int nch = 13 - hh;
    auto grp = [&](int c) { return c < 8 ? 8 * hh + c : 16 + 5 * hh + (c - 8); };
    const uint32_t c2empty0 = rcx::map_cta(c2empty, lead), c2emptyB0 = rcx::map_cta(c2emptyB, lead);
    uint8_t *stg_base = sST + w * NSTG * STGB;  // TMA-store staging: two 1 KB buffers (bf16), one 2 KB (tf32)
    uint32_t nst = 0;
    const int ntiles = cl < total ? (total - 1 - cl) / ncl + 1 : 0;
    for (int it = 0; it < ntiles; ++it) {
      const int tile = cl + it * ncl;
      const int mp = tile % pairs, net = tile / pairs;
      rcx::mbar_wait_sleep(c2full, it & 1);
      if (warp == 8) TR(3, it, 0);
      rcx::tc_fence_after();
      const int grow = mp * 256 + prank * 128 + q * 32;
      if constexpr (TF) {
        // fp32 accumulators (b2 included by the MMA): GELU and one tf32 rounding per group of 16
        // columns straight from TMEM; piece 1 is released after its second half is loaded, piece 2
        // as soon as it is loaded (the values wait in registers)
        uint8_t *stg = stg_base;
        auto gelu_store = [&](const uint32_t *v, int c) {
          float gg[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) gg[j] = rcm::tf32_rn(rcm::gelu_erf_f32(__uint_as_float(v[j])));
          if (lane == 0) rcm::bulk_wait_read0();  // the previous store has read the staging buffer
          __syncwarp();
          const int xx = (lane >> 1) & 3;  // [32 rows][64 B] staging, 64-byte TMA swizzle
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<float4 *>(stg + lane * 64 + ((u ^ xx) << 4)) =
                make_float4(gg[4 * u], gg[4 * u + 1], gg[4 * u + 2], gg[4 * u + 3]);
          rcm::fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            rcm::tma_store_3d(&mapOut, stg, pr * NP + grp(c) * 16, grow, net);
            rcm::bulk_commit();
          }
        };
        {
          uint32_t v[64];
          rcm::tmem_ld32(tmem + tq + grp(0) * 16, *reinterpret_cast<uint32_t(*)[32]>(v));
          rcm::tmem_ld32(tmem + tq + grp(2) * 16, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
          rcx::tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < 4; ++c) gelu_store(v + 16 * c, c);
        }
        {
          uint32_t v[64];
          rcm::tmem_ld32(tmem + tq + grp(4) * 16, *reinterpret_cast<uint32_t(*)[32]>(v));
          rcm::tmem_ld32(tmem + tq + grp(6) * 16, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
          rcx::tmem_ld_wait();
          rcx::tc_fence_before();
          __syncwarp();
          if (lane == 0) rcx::mbar_arrive_cluster(c2empty0);
#pragma unroll
          for (int c = 0; c < 4; ++c) gelu_store(v + 16 * c, 4 + c);
        }
        {
          uint32_t v[80];
          rcm::tmem_ld32(tmem + tq + grp(8) * 16, *reinterpret_cast<uint32_t(*)[32]>(v));
          rcm::tmem_ld32(tmem + tq + grp(10) * 16, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
          if (hh == 0) rcx::tmem_ld16(tmem + tq + grp(12) * 16, *reinterpret_cast<uint32_t(*)[16]>(v + 64));
          rcx::tmem_ld_wait();
          rcx::tc_fence_before();
          __syncwarp();
          if (lane == 0) rcx::mbar_arrive_cluster(c2emptyB0);
          if (warp == 8) TR(3, it, 1);
#pragma unroll
          for (int c = 0; c < 5; ++c)
            if (c < nch - 8) gelu_store(v + 16 * c, 8 + c);
        }
      } else {
      uint32_t pk[13][8];
      // accumulator columns (n groups from v, b2 already included) -> bf16 pairs
      auto cvt = [&](const uint32_t *v, int c, int n) {
#pragma unroll
        for (int h = 0; h < n; ++h)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            pk[c + h][j] = rcm::cvt_f16x2(__uint_as_float(v[16 * h + 2 * j]), __uint_as_float(v[16 * h + 2 * j + 1]));
      };
      // piece 1: two rounds of two 32-column loads in flight
#pragma unroll
      for (int c = 0; c < 8; c += 4) {
        uint32_t v[64];
        rcm::tmem_ld32(tmem + tq + grp(c) * 16, *reinterpret_cast<uint32_t(*)[32]>(v));
        rcm::tmem_ld32(tmem + tq + grp(c + 2) * 16, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
        rcx::tmem_ld_wait();
        cvt(v, c, 4);
      }
      rcx::tc_fence_before();
      __syncwarp();
      if (lane == 0) rcx::mbar_arrive_cluster(c2empty0);
      // piece 2: groups 8..11 (32-column loads), then group 12 (hh = 0 only)
#pragma unroll
      for (int c = 8; c < 12; c += 2) {
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
      if (warp == 8) TR(3, it, 1);
      // phase 2: GELU and TMA stores (32 rows x 16 columns per store) under the next tile's MMAs
#pragma unroll
      for (int c = 0; c < 13; ++c) {
        if (c < nch) {
          uint32_t gg[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) gg[j] = rcm::gelu_f16x2_bf16x2(pk[c][j]);
          uint8_t *stg = stg_base + (nst & 1) * 1024;
          if (lane == 0) rcm::bulk_wait_read1();
          __syncwarp();
          const int sw = (lane >> 2) & 1;
          *reinterpret_cast<uint4 *>(stg + lane * 32 + (sw << 4)) = make_uint4(gg[0], gg[1], gg[2], gg[3]);
          *reinterpret_cast<uint4 *>(stg + lane * 32 + ((sw ^ 1) << 4)) = make_uint4(gg[4], gg[5], gg[6], gg[7]);
          rcm::fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            rcm::tma_store_3d(&mapOut, stg, pr * NP + grp(c) * 16, grow, net);
            rcm::bulk_commit();
          }
          ++nst;
        }
      }
      }
      if (warp == 8) TR(3, it, 2);
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

constexpr int L12_RING = 4;  // W2 stage / h1 slot ring depth
// dynamic shared memory of the fused kernel; KZ = 16 bf16 keeps the W1 rows of a whole net (grows with h1)
size_t l12_smem(int KZ, int chunks, bool tf, int R = L12_RING) {
  const size_t EB = tf ? 4 : 2, CW = tf ? 32 : 64;
  const size_t Z_AL = ((size_t)128 * KZ * EB + 1023) & ~(size_t)1023;
  const size_t STAGE = ((size_t)W2T + 1023) & ~(size_t)1023;
  const size_t W1_CH = CW / 2 * KZ * EB;
  const size_t w1 = (KZ == 32 || tf) ? 4 * W1_CH : (((size_t)(chunks + 1) / 2) * W1_CH + 1023) & ~(size_t)1023;
  const size_t stg = (NEPI - NPROD) * (tf ? 1 * 2048 : 2 * 1024);
  return 1024 + R * (SLOT + STAGE) + 2 * Z_AL + w1 + stg + 2 * 7168 + 4096 + 1024;
}
constexpr size_t L12_SMEM_MAX = 232448;

// ring depth: 4, except TF32 with the 32-wide z rows of CH4 (3: the fp32 z tiles take the room)
template <int KZ, bool TF> constexpr int l12_ring() { return TF && KZ == 32 ? 3 : L12_RING; }

template <int KZ, bool TF>
int launch_t(const CUtensorMap *M, L12Args a, cudaStream_t s, int *nclusters) {
  constexpr int R = l12_ring<KZ, TF>();
  const size_t smem = l12_smem(KZ, a.chunks, TF, R);
  if (smem > L12_SMEM_MAX) return rc_fail(RC_EUNSUPPORTED, "fused layer-1/2 kernel: shared memory");
  a.stages = R;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(l12_kernel<KZ, R, TF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L12_SMEM_MAX);
    attr = true;
  }
  // persistent grid: only as many clusters of four as can be resident at once (a 4-CTA cluster
  // must fit in one GPC, so fewer than 148 / 4 are; a second wave would serialise their tiles)
  static int resident = 0;
  if (!resident) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(4 * (mlp_num_sms() / 4));
    cfg.blockDim = dim3(L12_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 4;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&resident, l12_kernel<KZ, R, TF>, &cfg) != cudaSuccess || resident <= 0)
      resident = mlp_num_sms() / 4;
  }
  const int total = a.nets * (a.m_tiles / 2);
  int clusters = resident;
  if (clusters > total) clusters = total;
  if (nclusters) *nclusters = clusters;
  l12_kernel<KZ, R, TF><<<4 * clusters, L12_THREADS, smem, s>>>(M[0], M[1], M[2], M[3], M[4], M[5], M[6], a);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

}  // namespace

// decided at create / workspace-sizing time (mlp_sm100.cu fused_path), so a shape the fused kernel
// cannot hold (e.g. KZ = 16 with h1 >= 2496: the whole-net W1 rows outgrow shared memory) takes the
// layer-wise path from the start instead of failing after the prologue launch.  TF32 with KZ = 32
// (CH4) runs a 3-deep W2/A ring: its fp32 z tiles take the room of the fourth stage.
bool l12_supported(int h1, int h2, int kz, bool tf) {
  const int cw = tf ? 32 : 64, R = tf && kz == 32 ? 3 : L12_RING;
  return h1 % 64 == 0 && h1 >= 128 && h2 == 2 * NP && (kz == 16 || kz == 32) && l12_smem(kz, h1 / cw, tf, R) <= L12_SMEM_MAX;
}

#ifdef L12TRACE
extern "C" __attribute__((visibility("default"))) int rc_debug_l12trace(void *host) {
  return (int)cudaMemcpyFromSymbol(host, g_l12trace, sizeof(g_l12trace));
}
#endif

int launch_l12(int KZ, bool tf, const CUtensorMap *maps, const L12Args &a, cudaStream_t s, int *clusters) {
  ProfScope prof(RC_STAGE_L12, s);
  if (tf) {
    if (KZ == 16) return launch_t<16, true>(maps, a, s, clusters);
    if (KZ == 32) return launch_t<32, true>(maps, a, s, clusters);
    return rc_fail(RC_EUNSUPPORTED, "fused layer-1/2 kernel (tf32): K = %d", KZ);
  }
  if (KZ == 16) return launch_t<16, false>(maps, a, s, clusters);
  if (KZ == 32) return launch_t<32, false>(maps, a, s, clusters);
  return rc_fail(RC_EUNSUPPORTED, "fused layer-1/2 kernel: K = %d", KZ);
}
