// mlp_l2_sm100.cu -- layer 2 of the per-species MLP (1600 -> 800,
// GELU) as a persistent CTA-pair tcgen05 GEMM:
//
//   h2[:, pass] = GELU( h1 W2[pass]^T + b2 )        (bf16 in, fp32 accumulate, bf16 out)
//
// Each CTA pair (cluster of 2) owns a 256-cell x NP tile (NP = 400: one of two
// passes over the 800 outputs).  The even CTA issues M=256 cta_group::2 MMAs
// whose A rows (h1, loaded by TMA) are split 128/128 between the two CTAs and
// whose B operand (a 64-wide K chunk of W2[pass]) is split by N, so each SM
// stages half of every weight chunk.  The NP outputs are two MMA pieces
// (N = 256 + 144) that alternate in the instruction stream: back-to-back MMAs
// into one accumulator stall on the accumulator dependency, alternating two
// accumulators runs at the nominal rate (tools/microbench/mma_rate.cu).
// The only barrier the MMA thread waits on per K chunk is the TMA "full"
// barrier (extra waits between MMAs cost ~70 clk of tensor-pipe bubble each).
// Sixteen epilogue warps (four per TMEM lane quadrant) drain acc2: b2 + GELU
// (packed bf16x2, tanh form) -> swizzled smem staging -> TMA bulk tensor store.
//
// Warps: 0..15 epilogue, 16 TMA producer, 17 MMA issuer (the scheduler favours
// higher warp ids, so the single-thread roles get the highest ids).
//
// DOT = true runs layer 3 (800 -> 400) with layer 4 folded in: the epilogue
// computes GELU(acc + b3) . w4 in fp32 over each warp's columns and writes one
// partial per (row, column quarter); the chem epilogue sums the four.
//
// The accumulator is drained in two phases: each warp first copies all its
// columns out of TMEM as 16-bit (acc + bias) pairs (no MUFU work, ~1 K clk)
// and releases it, then applies GELU and stores while the next tile's MMAs run
// (tools/l2trace.py: releasing after the GELU of all but the last columns kept
// the tensor pipe idle ~7 K of ~27 K clk per layer-2 tile).  Overlapping the drain with the next
// tile's MMAs (piece 2 trailing piece 1 by D chunks) measured slower: an MMA
// chain into one accumulator runs at one K16 step per ~220 clk whatever N
// (tools/microbench/mma_rate.cu), so the full rate needs ~400+ accumulator
// columns in flight, which leaves no TMEM to drain from.
#include <cuda_bf16.h>

#include "mlp_common.cuh"
#include "mlp_internal.h"

namespace {

constexpr int NEPI = 16;
constexpr int L2_THREADS = 32 * NEPI + 64;
// K chunk = one swizzled operand row: 128 B = 64 bf16 or 32 fp32 (tf32) elements; 64 B = 16 fp32
// for tf32x3, whose stages hold a hi and a lo copy of each operand
template <int PREC>
constexpr int row_bytes() { return PREC == 2 ? 64 : 128; }
template <int PREC>
constexpr int kc() { return row_bytes<PREC>() / rcm::Elem<(PREC != 0)>::BYTES; }
// store staging per warp: [32 rows][16 cols] = 1 KB bf16 / 2 KB fp32, two slots
template <bool TF32>
constexpr uint32_t stg_bytes() { return 32 * 16 * rcm::Elem<TF32>::BYTES; }

using rcm::bulk_commit;
using rcm::bulk_wait_all;
using rcm::bulk_wait_read1;
using rcm::cvt_bf16x2;
using rcm::fence_async_smem;
using rcm::tma_store_3d;
using rcm::tmem_ld32;
// Both layers park their pre-activations as f16 pairs (rcm::cvt_f16x2, .satfinite range guard)
// between the TMEM copy-out and the GELU: layer 2 then runs the f16x2 GELU with one bf16
// rounding, layer 3 widens to fp32 for the GELU + w4 dot.
using rcm::cvt_f16x2;
__device__ __forceinline__ float2 f16x2_to_f2(uint32_t v) {
  float lo, hi;
  asm("{\n\t.reg .f16 l, h;\n\tmov.b32 {l, h}, %2;\n\tcvt.f32.f16 %0, l;\n\tcvt.f32.f16 %1, h;\n}"
      : "=f"(lo), "=f"(hi) : "r"(v));
  return make_float2(lo, hi);
}

// tile queue: the pair leader's TMA thread decides the pair's next tile (static
// schedule, or an atomic counter shared with other launches) and publishes it into both CTAs.
// Readers per slot: rank 0's MMA warp and rank 1's TMA thread; each CTA's TMA thread hands the tile
// to its epilogue warps with the tile's bias slice (sTile[zb], published by the bfull barrier), so the
// register-bound epilogue warps carry no queue state.
// The leader publishes TQ_AHEAD tiles past the one its TMA thread loads, so rank 1's TMA thread never
// waits for a tile index at a tile boundary (publishing at the boundary cost ~1 us per tile).
constexpr int TQD = 8, TQ_READERS = 2, TQ_AHEAD = 1;
// [0] tiles run by filler launches, [1] filler pairs that gave up at the gate, [2] filler pairs that ran
__device__ unsigned long long g_l2_overlap[3];

#ifdef L2TRACE  // timing experiment: per-tile clock64 stamps of cluster 0 (tools/l2trace.py)
constexpr int TR_TILES = 40;
__device__ long long g_l2trace[2][20][TR_TILES][4];  // [DOT][warp][tile][event]
#define TRACE(w, it, k)                                                                                  \
  do {                                                                                                   \
    if (blockIdx.x == 0 && (it) < TR_TILES && lane == 0) g_l2trace[DOT ? 1 : 0][w][it][k] = clock64(); \
  } while (0)
#else
#define TRACE(w, it, k) \
  do {                  \
  } while (0)
#endif

template <int NP, bool DOT, int PREC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(L2_THREADS, 1)
    l2_pair_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapBa,
                   const __grid_constant__ CUtensorMap mapBb, const __grid_constant__ CUtensorMap mapOut,
                   const __grid_constant__ CUtensorMap mapAlo, const __grid_constant__ CUtensorMap mapBalo,
                   const __grid_constant__ CUtensorMap mapBblo, const __grid_constant__ CUtensorMap mapOutlo,
                   const __grid_constant__ CUtensorMap mapKa, const __grid_constant__ CUtensorMap mapKb, L2Args a) {
  static_assert(NP % 16 == 0 && NP <= 512, "pass width");
  constexpr int P1 = NP > 256 ? 256 : NP, P2 = NP - P1;
  constexpr int H1 = P1 / 2, H2 = P2 / 2;  // B rows per CTA of each piece
  static_assert(H1 % 8 == 0 && H2 % 8 == 0, "8-row swizzle atoms");
  constexpr bool TF32 = rcm::Prec<PREC>::TF32, X3 = rcm::Prec<PREC>::X3;
  constexpr int NOP = rcm::Prec<PREC>::NOP;
  using E = rcm::Elem<TF32>;
  constexpr int RB = row_bytes<PREC>(), KC = kc<PREC>();
  constexpr uint32_t STG = stg_bytes<TF32>();
  constexpr uint32_t A_BYTES = 128 * RB, B_BYTES = (NP / 2) * RB;  // one copy; X3 stages hold hi and lo
  constexpr uint32_t STAGE = (NOP * (A_BYTES + B_BYTES) + 1023u) & ~1023u;  // [A hi | A lo | B hi | B lo]
  constexpr int W_TMA = NEPI, W_MMA = NEPI + 1;
  // bf16: the bias is folded into the MMAs (one K = 16 MMA per piece of a ones tile against the
  // (b_hi, b_lo, 0...) operand tile at the start of a tile), so the drain only converts; tf32/X3
  // add the fp32 bias in the epilogue
  constexpr bool BFOLD = !TF32;
  constexpr uint32_t BK_BYTES = (NP / 2) * 32, BK_AL = ((NP / 2) * 32 + 1023u) & ~1023u;
  constexpr int P1G = P1 / 16, P2G = P2 / 16;  // 16-column groups of the two accumulator pieces

  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = rcx::smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  const int S = a.stages;
  uint8_t *sW = smem;                                   // S x [A tile | B half]
  uint8_t *sST = sW + S * STAGE;                        // NEPI x 2 x 1 KB store staging
  float *sB2 = reinterpret_cast<float *>(sST + NEPI * 2 * STG);  // 2 x [b | w4 (DOT)] slices
  constexpr int VEC = DOT ? 2 * NP : NP;
  uint8_t *sBK = reinterpret_cast<uint8_t *>(sB2) + ((2 * VEC * 4 + 1023u) & ~1023u);  // BFOLD: 2 x b operand tile
  uint8_t *sOnes = sBK + (BFOLD ? 2 * BK_AL : 0);                                   // BFOLD: 128 x 16 bf16 ones
  uint64_t *bar = reinterpret_cast<uint64_t *>(sOnes + (BFOLD ? 4096 : 0));
  uint64_t *full = bar, *empty = full + S, *c2full = empty + S, *c2empty = c2full + 1, *c2emptyB = c2empty + 1,
           *bfull = c2emptyB + 1, *bempty = bfull + 2, *bkfull = bempty + 2, *bkempty = bkfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bkempty + 2);
  uint64_t *tqfull = bkempty + 3, *tqempty = tqfull + TQD;  // (bkempty + 2 holds the TMEM address)
  int *tq = reinterpret_cast<int *>(tqempty + TQD);
  int *sTile = tq + TQD;  // [2]: the tile of bias slice zb, for the epilogue warps

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = rcx::cluster_rank();
  const bool leader = rank == 0;
  if (warp == W_TMA && lane == 0) {
    rcx::prefetch_tmap(&mapA);
    rcx::prefetch_tmap(&mapBa);
    if (P2 > 0) rcx::prefetch_tmap(&mapBb);
    if (!DOT) rcx::prefetch_tmap(&mapOut);
    if (X3) {
      rcx::prefetch_tmap(&mapAlo);
      rcx::prefetch_tmap(&mapBalo);
      if (P2 > 0) rcx::prefetch_tmap(&mapBblo);
      if (!DOT) rcx::prefetch_tmap(&mapOutlo);
    }
    if (BFOLD) {
      rcx::prefetch_tmap(&mapKa);
      if (P2 > 0) rcx::prefetch_tmap(&mapKb);
    }
    for (int s = 0; s < S; ++s) { rcx::mbar_init(&full[s], 2); rcx::mbar_init(&empty[s], 1); }
    rcx::mbar_init(c2full, 1);
    rcx::mbar_init(c2empty, 2 * NEPI);   // piece 1 (columns [0, P1)) copied out, both CTAs
    rcx::mbar_init(c2emptyB, 2 * NEPI);  // piece 2
    for (int z = 0; z < 2; ++z) {
      rcx::mbar_init(&bfull[z], 1);
      rcx::mbar_init(&bempty[z], NEPI);
      rcx::mbar_init(&bkfull[z], 2);
      rcx::mbar_init(&bkempty[z], 1);
    }
    for (int d = 0; d < TQD; ++d) {
      rcx::mbar_init(&tqfull[d], 1);
      rcx::mbar_init(&tqempty[d], TQ_READERS);  // used in the leader only
    }
    rcx::fence_mbar_init();
  }
  if (BFOLD) {
    for (int i = threadIdx.x; i < 1024; i += L2_THREADS) reinterpret_cast<uint32_t *>(sOnes)[i] = 0x3F803F80u;
    fence_async_smem();  // read by the tensor core (async proxy)
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
  const uint32_t tqempty0 = rcx::map_cta(tqempty, 0);
  // reader side: the pair's it-th tile (>= total: none left); `warp_reader`: the whole warp reads,
  // then one lane reports the slot read.  Rank 0's slot is written by its own TMA thread (ordinary
  // arrive); rank 1's arrives by st.async with completion (4 tx bytes) on rank 1's tqfull, so an
  // ordinary wait orders it and the leader's TMA thread issues no release fence (a cluster-scope
  // release there waited for the thread's outstanding TMA loads: layer 3 lost 5%).  The read-done
  // arrivals order nothing: a slot is rewritten only TQD tiles later.
  auto tq_take = [&](int it, bool warp_reader) -> int {
    const int d = it % TQD;
    rcx::mbar_wait(&tqfull[d], (uint32_t)(it / TQD) & 1);
    const int t = rcx::ld_shared_s32(&tq[d]);
    if (warp_reader) __syncwarp();
    if (!warp_reader || lane == 0) {
      if (leader) rcx::mbar_arrive(&tqempty[d]);
      else rcx::mbar_arrive_relaxed_cluster(tqempty0 + d * 8);
    }
    return t;
  };

  if (warp == W_TMA) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer (both CTAs)
      const uint32_t full0 = rcx::map_cta(full, 0);
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      // leader: the next tile, decided a tile ahead (the counter's atomic latency hides behind a
      // tile's loads).  A filler waits at the gate first and takes nothing if it stays closed.
      int t_next = cl, n_done = 0, pub = 0;
      bool pub_end = false;
      if (leader && a.tile_ctr) {
        bool go = true;
        if (a.gate) {
          const uint64_t t0 = rcx::global_ns();
          while (rcx::ld_acquire_gpu(a.gate) < a.gate_target)
            if (rcx::global_ns() - t0 > a.gate_ns) {
              go = false;
              break;
            }
          atomicAdd(&g_l2_overlap[go ? 2 : 1], 1ull);
        }
        t_next = go ? atomicAdd(a.tile_ctr, 1) : total;
      }
      for (;; ++it) {
        int tile;
        if (leader) {  // publish up to TQ_AHEAD tiles ahead into both CTAs' queue slots
          for (; pub <= it + TQ_AHEAD && !pub_end; ++pub) {
            const int tp = t_next < total ? t_next : total, d = pub % TQD;
            rcx::mbar_wait(&tqempty[d], ((uint32_t)(pub / TQD) & 1) ^ 1);
            *reinterpret_cast<volatile int *>(&tq[d]) = tp;
            rcx::mbar_arrive(&tqfull[d]);
            const uint32_t rbar = rcx::map_cta(&tqfull[d], 1);
            rcx::mbar_arrive_expect_tx_relaxed_cluster(rbar, 4);
            rcx::st_async_u32(rcx::map_cta(&tq[d], 1), (uint32_t)tp, rbar);
            if (tp >= total) pub_end = true;
            else t_next = a.tile_ctr ? atomicAdd(a.tile_ctr, 1) : tp + ncl;
          }
          // (slot it is not rewritten before this read: that needs pub = it + TQD)
          tile = *reinterpret_cast<volatile int *>(&tq[it % TQD]);
          if (tile < total) ++n_done;
        } else {
          tile = tq_take(it, false);
        }
        const int zb = it & 1;
        rcx::mbar_wait_sleep(&bempty[zb], ((it >> 1) & 1) ^ 1);  // b2 slice for this CTA's drain
        *reinterpret_cast<volatile int *>(&sTile[zb]) = tile;
        if (tile >= total) {  // tell the epilogue warps: no more tiles
          rcx::mbar_arrive(&bfull[zb]);
          break;
        }
        const int pass = tile % a.passes, rest = tile / a.passes;
        const int mp = rest % pairs, net = rest / pairs;
        rcx::mbar_arrive_expect_tx(&bfull[zb], VEC * 4);
        rcx::bulk_g2s(sB2 + zb * VEC, a.bias + (size_t)net * a.N + pass * NP, NP * 4, &bfull[zb]);
        if (DOT) rcx::bulk_g2s(sB2 + zb * VEC + NP, a.w4 + (size_t)net * a.N + pass * NP, NP * 4, &bfull[zb]);
        if (BFOLD) {  // this CTA's rows of the bias operand tile, completion on the leader's barrier
          rcx::mbar_wait_sleep(&bkempty[zb], ((it >> 1) & 1) ^ 1);
          rcx::mbar_arrive_expect_tx_cluster(rcx::map_cta(&bkfull[zb], 0), BK_BYTES);
          rcx::tma_load_3d_pair(sBK + zb * BK_AL, &mapKa, &bkfull[zb], 0, pass * NP + rank * H1, net);
          if (P2 > 0) rcx::tma_load_3d_pair(sBK + zb * BK_AL + H1 * 32, &mapKb, &bkfull[zb], 0, pass * NP + P1 + rank * H2, net);
        }
        for (int c = 0; c < C; ++c) {
          rcx::mbar_wait_sleep(&empty[s], ph ^ 1);
          rcx::mbar_arrive_expect_tx_cluster(full0 + s * 8, NOP * (A_BYTES + B_BYTES));
          uint8_t *st = sW + s * STAGE;
          uint8_t *sb = st + NOP * A_BYTES;
          rcx::tma_load_3d_pair(st, &mapA, &full[s], c * KC, mp * 256 + rank * 128, net);
          rcx::tma_load_3d_pair(sb, &mapBa, &full[s], c * KC, pass * NP + rank * H1, net);
          if (P2 > 0)
            rcx::tma_load_3d_pair(sb + H1 * RB, &mapBb, &full[s], c * KC, pass * NP + P1 + rank * H2, net);
          if (X3) {
            rcx::tma_load_3d_pair(st + A_BYTES, &mapAlo, &full[s], c * KC, mp * 256 + rank * 128, net);
            rcx::tma_load_3d_pair(sb + B_BYTES, &mapBalo, &full[s], c * KC, pass * NP + rank * H1, net);
            if (P2 > 0)
              rcx::tma_load_3d_pair(sb + B_BYTES + H1 * RB, &mapBblo, &full[s], c * KC, pass * NP + P1 + rank * H2, net);
          }
          if (++s == S) { s = 0; ph ^= 1; }
        }
      }
      if (leader && a.gate && n_done) atomicAdd(&g_l2_overlap[0], (unsigned long long)n_done);
    }
  } else if (warp == W_MMA) {
    if (leader) {  // ------------- MMA issuer (even CTA; converged warp, one elected lane issues)
      constexpr uint32_t idp1 = rcx::make_idesc(E::FMT, 256, P1);
      constexpr uint32_t idp2 = rcx::make_idesc(E::FMT, 256, P2 > 0 ? P2 : 16);
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0;; ++it) {
        if (tq_take(it, true) >= total) break;
        TRACE(W_MMA, it, 0);
        if (!BFOLD) {
          rcx::mbar_wait(c2empty, (it & 1) ^ 1);  // previous tile drained
          rcx::mbar_wait(c2emptyB, (it & 1) ^ 1);
        }
        TRACE(W_MMA, it, 1);
        rcx::tc_fence_after();
        for (int c = 0; c < C; ++c) {
          rcx::mbar_wait(&full[s], ph);
          rcx::tc_fence_after();
          const uint64_t da = rcm::desc_sw<RB>(sW + s * STAGE);
          const uint64_t db = rcm::desc_sw<RB>(sW + s * STAGE + NOP * A_BYTES);
          constexpr uint64_t ALO = A_BYTES >> 4, BLO = B_BYTES >> 4, BP2 = (H1 * RB) >> 4;
          // the last K chunk may be partial (K = 800: 32 of 64); its zero-filled atoms are skipped
          const int nk = (c == C - 1 && a.ktail) ? a.ktail : KC / E::KATOM;
          if (BFOLD && c == 0) {
            // the accumulator starts at the bias (ones x b operand); piece 1 restarts as soon as the
            // drain has copied it out, piece 2 (c2emptyB) follows
            const int zb = it & 1;
            rcx::mbar_wait(&bkfull[zb], (it >> 1) & 1);
            const uint64_t d1 = rcm::desc_sw<32>(sOnes), dk = rcm::desc_sw<32>(sBK + zb * BK_AL);
            // (the tensor pipe runs one accumulator chain at ~220 clk per MMA: after the first two
            // piece-1 MMAs the pieces are interleaved again, as in the main loop)
            rcx::mbar_wait(c2empty, (it & 1) ^ 1);
            rcx::tc_fence_after();
            if (rcx::elect_one()) {
              rcm::mma_pair<false>(tmem, d1, dk, idp1, 0);
              rcm::mma_pair<false>(tmem, da, db, idp1, 1);
            }
            __syncwarp();
            if (P2 > 0) {
              rcx::mbar_wait(c2emptyB, (it & 1) ^ 1);
              rcx::tc_fence_after();
            }
            if (rcx::elect_one()) {
              if (P2 > 0) {
                rcm::mma_pair<false>(tmem + P1, d1, dk + ((H1 * 32) >> 4), idp2, 0);
                rcm::mma_pair<false>(tmem + P1, da, db + BP2, idp2, 1);
              }
#pragma unroll
              for (int k = 1; k < KC / E::KATOM; ++k) {
                if (k >= nk) break;
                rcm::mma_pair<false>(tmem, da + 2 * k, db + 2 * k, idp1, 1);
                if (P2 > 0) rcm::mma_pair<false>(tmem + P1, da + 2 * k, db + BP2 + 2 * k, idp2, 1);
              }
              rcx::mma_commit_pair(&empty[s]);
              rcx::mma_commit_pair(&bkempty[zb]);
            }
            __syncwarp();
            if (++s == S) { s = 0; ph ^= 1; }
            continue;
          }
          // (the full-chunk loop is kept free of the tail test: a per-MMA branch slows the issue)
          if (rcx::elect_one()) {
          if (nk == KC / E::KATOM) {
#pragma unroll
          for (int k = 0; k < KC / E::KATOM; ++k) {  // 32-byte K atoms: descriptor start += 2
            const uint32_t acc = BFOLD || (c | k) != 0;
            rcm::mma_pair<TF32>(tmem, da + 2 * k, db + 2 * k, idp1, acc);
            if (P2 > 0) rcm::mma_pair<TF32>(tmem + P1, da + 2 * k, db + BP2 + 2 * k, idp2, acc);
            if (X3) {  // + a_lo b_hi + a_hi b_lo
              rcm::mma_pair<TF32>(tmem, da + ALO + 2 * k, db + 2 * k, idp1, 1);
              if (P2 > 0) rcm::mma_pair<TF32>(tmem + P1, da + ALO + 2 * k, db + BP2 + 2 * k, idp2, 1);
              rcm::mma_pair<TF32>(tmem, da + 2 * k, db + BLO + 2 * k, idp1, 1);
              if (P2 > 0) rcm::mma_pair<TF32>(tmem + P1, da + 2 * k, db + BLO + BP2 + 2 * k, idp2, 1);
            }
          }
          } else {
#pragma unroll
          for (int k = 0; k < KC / E::KATOM; ++k) {  // 32-byte K atoms: descriptor start += 2
            if (k >= nk) break;  // partial last chunk (uniform branch, once per tile)
            const uint32_t acc = BFOLD || (c | k) != 0;
            rcm::mma_pair<TF32>(tmem, da + 2 * k, db + 2 * k, idp1, acc);
            if (P2 > 0) rcm::mma_pair<TF32>(tmem + P1, da + 2 * k, db + BP2 + 2 * k, idp2, acc);
            if (X3) {  // + a_lo b_hi + a_hi b_lo
              rcm::mma_pair<TF32>(tmem, da + ALO + 2 * k, db + 2 * k, idp1, 1);
              if (P2 > 0) rcm::mma_pair<TF32>(tmem + P1, da + ALO + 2 * k, db + BP2 + 2 * k, idp2, 1);
              rcm::mma_pair<TF32>(tmem, da + 2 * k, db + BLO + 2 * k, idp1, 1);
              if (P2 > 0) rcm::mma_pair<TF32>(tmem + P1, da + 2 * k, db + BLO + BP2 + 2 * k, idp2, 1);
            }
          }
          }
          rcx::mma_commit_pair(&empty[s]);
          }
          __syncwarp();
          if (++s == S) { s = 0; ph ^= 1; }
        }
        if (rcx::elect_one()) rcx::mma_commit_pair(c2full);
        __syncwarp();
        TRACE(W_MMA, it, 2);
      }
    }
  } else {  // ------------------------------------------------------ epilogue warps 0..15 (both CTAs)
    const int q = warp & 3, sub = warp >> 2;
    const uint32_t tq = (uint32_t)(q * 32) << 16;
    constexpr int NCH = NP / 16;
    const int ch_lo = (NCH * sub) / 4, ch_hi = (NCH * (sub + 1)) / 4;
    const uint32_t c2empty0 = rcx::map_cta(c2empty, 0), c2emptyB0 = rcx::map_cta(c2emptyB, 0);
    // bf16: this warp's groups of piece 1 and of piece 2 (released separately)
    const int g1lo = P1G * sub / 4, n1 = P1G * (sub + 1) / 4 - g1lo;
    const int g2lo = P1G + P2G * sub / 4, n2 = P1G + P2G * (sub + 1) / 4 - g2lo;
    uint8_t *stg_base = sST + warp * 2 * STG;
    // layer 3 (DOT): the four warps of a lane quadrant (q, q+4, q+8, q+12) each hold the dot over one
    // column quarter of their 32 rows; they meet at named barrier 1+q and warp sub 0 stores the row
    // sums ((p0 + p1) + p2) + p3 (fixed order), so the epilogue reads one fp32 per net and row
    // instead of four.  The reduction buffer [2 tile parities][4][128] floats lives in the store
    // staging, which the dot epilogue does not use; the barrier of tile t+1 orders sub 0's reads
    // of parity (t & 1) before any write of tile t+2.
    auto emit_o = [&](float dot, int it_, int net_, int pass_, int grow_) {
      float *red = reinterpret_cast<float *>(sST) + (it_ & 1) * 512;
      red[sub * 128 + q * 32 + lane] = dot;
      asm volatile("bar.sync %0, 128;" ::"r"(1 + q) : "memory");
      if (sub == 0) {
        const float *r = red + q * 32 + lane;
        a.opart[(size_t)(net_ * a.passes + pass_) * a.cap + grow_ + lane] = ((r[0] + r[128]) + r[256]) + r[384];
      }
    };
    uint32_t nst = 0;
    for (int it = 0;; ++it) {
      rcx::mbar_wait_sleep(&bfull[it & 1], (it >> 1) & 1);  // this tile's bias slice and index
      const int tile = *reinterpret_cast<volatile int *>(&sTile[it & 1]);
      if (tile >= total) break;
      const int pass = tile % a.passes, rest = tile / a.passes;
      const int mp = rest % pairs, net = rest / pairs;
      TRACE(warp, it, 0);
#ifdef L2_EPI_SPIN
      rcx::mbar_wait(c2full, it & 1);
#else
      rcx::mbar_wait_sleep(c2full, it & 1);  // parked for the whole mainloop: leave issue slots and power to the rest
#endif
      TRACE(warp, it, 1);
      rcx::tc_fence_after();
      const float *b2 = sB2 + (it & 1) * VEC;
      const int grow = mp * 256 + rank * 128 + q * 32;  // first global row of this warp's 32 rows
      if constexpr (TF32) {
        // fp32 accumulators chunk pair by chunk pair; the accumulator is released after the last load
        float dot = 0.f;
        if (ch_lo == ch_hi) {
          rcx::tc_fence_before();
          __syncwarp();
          if (lane == 0) rcx::mbar_arrive_cluster(c2empty0), rcx::mbar_arrive_cluster(c2emptyB0);
        }
        for (int cc = ch_lo; cc < ch_hi; cc += 2) {
          uint32_t v[32];
          const bool two = cc + 1 < ch_hi;
          if (two)
            tmem_ld32(tmem + tq + cc * 16, v);
          else
            rcx::tmem_ld16(tmem + tq + cc * 16, *reinterpret_cast<uint32_t(*)[16]>(v));
          rcx::tmem_ld_wait();
          if (cc + 2 >= ch_hi) {
            rcx::tc_fence_before();
            __syncwarp();
            if (lane == 0) rcx::mbar_arrive_cluster(c2empty0), rcx::mbar_arrive_cluster(c2emptyB0);
            TRACE(warp, it, 2);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !two) break;
            const int col = (cc + h) * 16;
            const float4 *bb = reinterpret_cast<const float4 *>(b2 + col);
            if constexpr (DOT) {  // layer 3: exact GELU(acc + b3) . w4
              const float4 *ww = reinterpret_cast<const float4 *>(b2 + NP + col);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 b = bb[j], w = ww[j];
                dot = fmaf(rcm::gelu_erf_f32(__uint_as_float(v[16 * h + 4 * j]) + b.x), w.x, dot);
                dot = fmaf(rcm::gelu_erf_f32(__uint_as_float(v[16 * h + 4 * j + 1]) + b.y), w.y, dot);
                dot = fmaf(rcm::gelu_erf_f32(__uint_as_float(v[16 * h + 4 * j + 2]) + b.z), w.z, dot);
                dot = fmaf(rcm::gelu_erf_f32(__uint_as_float(v[16 * h + 4 * j + 3]) + b.w), w.w, dot);
              }
            } else {  // layer 2: tf32-rounded exact GELU -> [32 rows][64 B] staging (64-byte swizzle) -> TMA store
              float y[16];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 b = bb[j];
                y[4 * j] = rcm::gelu_erf_f32(__uint_as_float(v[16 * h + 4 * j]) + b.x);
                y[4 * j + 1] = rcm::gelu_erf_f32(__uint_as_float(v[16 * h + 4 * j + 1]) + b.y);
                y[4 * j + 2] = rcm::gelu_erf_f32(__uint_as_float(v[16 * h + 4 * j + 2]) + b.z);
                y[4 * j + 3] = rcm::gelu_erf_f32(__uint_as_float(v[16 * h + 4 * j + 3]) + b.w);
              }
#pragma unroll
              for (int part = 0; part < NOP; ++part) {  // hi (= tf32(y)); X3: then lo (= tf32(y - hi))
                float g[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) g[j] = part == 0 ? rcm::tf32_rn(y[j]) : rcm::tf32_rn(y[j] - rcm::tf32_rn(y[j]));
                uint8_t *stg = stg_base + (nst & 1) * STG;
                if (lane == 0) bulk_wait_read1();
                __syncwarp();
                const int x = (lane >> 1) & 3;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  *reinterpret_cast<float4 *>(stg + lane * 64 + ((u ^ x) << 4)) =
                      make_float4(g[4 * u], g[4 * u + 1], g[4 * u + 2], g[4 * u + 3]);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                  tma_store_3d(part == 0 ? &mapOut : &mapOutlo, stg, pass * NP + col, grow, net);
                  bulk_commit();
                }
                ++nst;
              }
            }
          }
        }
        if constexpr (DOT) emit_o(dot, it, net, pass, grow);
      } else {
        // Phase A (no MUFU): every accumulator column of this warp (bias included by the MMA) ->
        // registers as 16-bit pairs: bf16 for layer 2 (the GELU input), f16 for the fp32 layer-3
        // GELU.  Piece 1 is released first (its MMAs of the next tile restart), then piece 2, so
        // the next tile's MMAs run under phase B.
        constexpr int MAX1 = (P1G + 3) / 4, MAX2 = P2G > 0 ? (P2G + 3) / 4 : 1;
        uint32_t pk1[MAX1][8], pk2[MAX2][8];
        auto copy = [&](auto &pk, int glo, int n) {  // n groups from glo, two loads in flight at a time
          constexpr int M = sizeof(pk) / sizeof(pk[0]);
#pragma unroll
          for (int i0 = 0; i0 < M; i0 += 2) {
            uint32_t v[2][16];
#pragma unroll
            for (int i = 0; i < 2; ++i)
              if (i0 + i < M && i0 + i < n) rcx::tmem_ld16(tmem + tq + (glo + i0 + i) * 16, v[i]);
            rcx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 2; ++i)
              if (i0 + i < M)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  const float x0 = __uint_as_float(v[i][2 * j]), x1 = __uint_as_float(v[i][2 * j + 1]);
                  pk[i0 + i][j] = cvt_f16x2(x0, x1);
                }
          }
        };
        copy(pk1, g1lo, n1);
        rcx::tc_fence_before();
        __syncwarp();
        if (lane == 0) rcx::mbar_arrive_cluster(c2empty0);
        copy(pk2, g2lo, n2);
        rcx::tc_fence_before();
        __syncwarp();
        if (lane == 0) rcx::mbar_arrive_cluster(c2emptyB0);
        TRACE(warp, it, 2);
        // Phase B: GELU (MUFU) and the layer's output path
        if constexpr (DOT) {  // layer 3: GELU(acc + b3) . w4 in fp32
          const float *w4s = b2 + NP;
          float dot = 0.f;
  #pragma unroll
          for (int c = 0; c < MAX1 + MAX2; ++c) {
            if (c < MAX1 ? c < n1 : c - MAX1 < n2) {
              const uint32_t *p = c < MAX1 ? pk1[c] : pk2[c - MAX1];
              const int gc = c < MAX1 ? g1lo + c : g2lo + c - MAX1;
              const float4 *ww = reinterpret_cast<const float4 *>(w4s + gc * 16);
  #pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 w = ww[j];
                const float2 a01 = f16x2_to_f2(p[2 * j]), a23 = f16x2_to_f2(p[2 * j + 1]);
                dot = fmaf(rcm::gelu_f32(a01.x), w.x, dot);
                dot = fmaf(rcm::gelu_f32(a01.y), w.y, dot);
                dot = fmaf(rcm::gelu_f32(a23.x), w.z, dot);
                dot = fmaf(rcm::gelu_f32(a23.y), w.w, dot);
              }
            }
          }
          emit_o(dot, it, net, pass, grow);
        } else {  // layer 2: bf16 GELU -> [32 rows][32 B] staging (32-byte TMA swizzle) -> TMA store
  #pragma unroll
          for (int c = 0; c < MAX1 + MAX2; ++c) {
            if (c < MAX1 ? c < n1 : c - MAX1 < n2) {
              const uint32_t *p = c < MAX1 ? pk1[c] : pk2[c - MAX1];
              const int gc = c < MAX1 ? g1lo + c : g2lo + c - MAX1;
              uint32_t g[8];
  #pragma unroll
              for (int j = 0; j < 8; ++j) g[j] = rcm::gelu_f16x2_bf16x2(p[j]);
              uint8_t *stg = stg_base + (nst & 1) * 1024;
              if (lane == 0) bulk_wait_read1();  // the store that last used this buffer has read it
              __syncwarp();
              const int sw = (lane >> 2) & 1;
              *reinterpret_cast<uint4 *>(stg + lane * 32 + (sw << 4)) = make_uint4(g[0], g[1], g[2], g[3]);
              *reinterpret_cast<uint4 *>(stg + lane * 32 + ((sw ^ 1) << 4)) = make_uint4(g[4], g[5], g[6], g[7]);
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(&mapOut, stg, pass * NP + gc * 16, grow, net);
                bulk_commit();
              }
              ++nst;
            }
          }
        }
      }
      __syncwarp();
      TRACE(warp, it, 3);
      if (lane == 0) rcx::mbar_arrive(&bempty[it & 1]);
    }
    if (!DOT && lane == 0) bulk_wait_all();
    __syncwarp();
  }
  rcx::tc_fence_before();
  rcx::cluster_sync();
  if (warp == W_MMA) {
    rcx::tc_fence_after();
    rcx::tmem_dealloc_pair(tmem, 512);
  }
}

template <int NP, bool DOT, int PREC>
int launch_l2_pair_t(const CUtensorMap *M, L2Args a, cudaStream_t s, int pairs) {
  constexpr int RB = row_bytes<PREC>();
  constexpr size_t STAGE = (rcm::Prec<PREC>::NOP * (128 * RB + (NP / 2) * RB) + 1023) & ~(size_t)1023;
  constexpr size_t BK = PREC == 0 ? 2 * ((((size_t)NP / 2) * 32 + 1023) & ~(size_t)1023) + 4096 : 0;  // b operand + ones
  const size_t fixed = 1024 + NEPI * 2 * stg_bytes<(PREC != 0)>() + ((2 * (DOT ? 2 : 1) * NP * 4 + 1023) & ~(size_t)1023) + BK + 512;
  int stages = (int)((232448 - fixed) / STAGE);
  if (stages > 8) stages = 8;
  if (stages < 2) return rc_fail(RC_EUNSUPPORTED, "layer-2 GEMM: pass width %d does not fit", NP);
  a.stages = stages;
  const size_t smem = fixed + stages * STAGE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(l2_pair_kernel<NP, DOT, PREC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    attr = true;
  }
  static int resident = 0;  // CTA pairs that fit at once (a persistent grid must not need a second wave)
  if (!resident) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * (mlp_num_sms() / 2));
    cfg.blockDim = dim3(L2_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&resident, l2_pair_kernel<NP, DOT, PREC>, &cfg) != cudaSuccess || resident <= 0)
      resident = mlp_num_sms() / 2;
  }
  const int total = a.nets * (a.m_tiles / 2) * a.passes;
  int clusters = pairs > 0 ? pairs : resident;
  if (clusters > total) clusters = total;
  l2_pair_kernel<NP, DOT, PREC><<<2 * clusters, L2_THREADS, smem, s>>>(M[0], M[1], M[2], M[3], M[4], M[5], M[6], M[7], M[8], M[9], a);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

}  // namespace

#ifdef L2TRACE
extern "C" __attribute__((visibility("default"))) int rc_debug_l2trace(void *host) {
  return (int)cudaMemcpyFromSymbol(host, g_l2trace, sizeof(g_l2trace));
}
#endif

// pass width: the widest instantiated NP (TMEM: one pass accumulator of <= 400 columns) that
// divides h into equal passes; every multiple of 16 has one (16 itself), so any hidden[1] /
// hidden[2] that rc_mlp_create accepts runs (tests/test_capi.py sweeps create + launch widths)
int l2_pass_width(int h) {
  static const int inst[] = {400, 256, 208, 128, 64, 32, 16};  // the RC_L2P instances below
  if (h <= 0 || h % 16) return 0;
  for (int np : inst)
    if (h % np == 0) return np;
  return 0;
}

int l2_overlap_read(long long *out, int reset) {
  unsigned long long v[3];
  if (cudaMemcpyFromSymbol(v, g_l2_overlap, sizeof(v)) != cudaSuccess) return rc_fail(RC_ECUDA, "rc_overlap_read");
  for (int i = 0; i < 3; ++i) out[i] = (long long)v[i];
  if (reset) {
    const unsigned long long z[3] = {0, 0, 0};
    if (cudaMemcpyToSymbol(g_l2_overlap, z, sizeof(z)) != cudaSuccess) return rc_fail(RC_ECUDA, "rc_overlap_read");
  }
  return RC_OK;
}

int launch_l2_pair(int NP, int prec, const CUtensorMap *maps, const L2Args &a, cudaStream_t s, int pairs) {
  ProfScope prof(a.prof_stage >= 0 ? a.prof_stage : a.w4 ? RC_STAGE_L3 : RC_STAGE_L2, s);
#define RC_L2P_PREC(np, dot)                                                                                \
  return prec == 0 ? launch_l2_pair_t<np, dot, 0>(maps, a, s, pairs)                                        \
                   : prec == 1 ? launch_l2_pair_t<np, dot, 1>(maps, a, s, pairs) : launch_l2_pair_t<np, dot, 2>(maps, a, s, pairs);
#define RC_L2P(np)                     \
  if (NP == np) {                      \
    if (a.w4) RC_L2P_PREC(np, true)    \
    else RC_L2P_PREC(np, false)        \
  }
  RC_L2P(400)
  RC_L2P(256)
  RC_L2P(208)
  RC_L2P(128)
  RC_L2P(64)
  RC_L2P(32)
  RC_L2P(16)
#undef RC_L2P
#undef RC_L2P_PREC
  return rc_fail(RC_EUNSUPPORTED, "layer-2 GEMM: no instance for pass width %d", NP);
}
