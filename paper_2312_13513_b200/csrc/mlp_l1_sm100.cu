// mlp_l1_sm100.cu -- layer 1 of the per-species MLP (inputs ->
// 1600, GELU) as a persistent tcgen05 GEMM with K = 16 (or 32):
//
//   h1 = GELU( z W1^T )     z = [z-scored Box-Cox inputs | 1 | 1 | 0...] (bf16),
//                           W1 carries b1 as bf16 hi/lo parts in the two 1-columns.
//
// K is tiny, so the kernel is bound by its epilogue: one MUFU tanh per output
// (16 per clock per SM) and the 2-byte-per-output h1 write to HBM (~5.6 TB/s for
// this tile pattern, tools/microbench/store2d_bw.cu), which are about equal here.
//  * W1 is stored halved (exact in bf16), so the accumulator holds x/2 and the
//    GELU needs one multiply fewer (rcm::gelu_half_bf16x2, bit-identical).
//  * 128 x 256 tiles, two TMEM accumulators; sixteen epilogue warps = four TMEM
//    lane quadrants x four 64-column blocks.  Each warp copies its 32 x 64 block
//    to registers, releases the accumulator, applies GELU, writes the block into
//    one of its two 128-byte-swizzled 4 KB staging slots and stores it with one
//    TMA bulk tensor store; the only cross-warp coupling is the accumulator release.
//  Measured alternatives (tools/l1trace.py, tools/l1var.sh, profiles/): 1 KB stores
//  capped the store path at ~3.5 TB/s; a per-tile named barrier across the warps,
//  one store-issuing thread fed through mbarriers, and coalesced STG stores from
//  the warps were all slower.
// TF32 precision mode (RC_TF32): fp32 z/W1 (tf32-rounded) with kind::tf32 MMAs,
// exact-erf GELU in fp32, fp32 h1 rounded to tf32; each warp's 32 x 64 block is
// staged as two 32 x 32 fp32 swizzled blocks (one 8 KB slot per warp).
// RC_TF32X3: z, W1 and h1 as tf32 hi/lo pairs, three MMAs per K atom
// (z_hi W_hi + z_lo W_hi + z_hi W_lo); h1 hi and lo are stored one after the other.
// Warps: 0..15 epilogue, 16 TMA producer, 17 MMA issuer.
#include <cuda_bf16.h>

#include "mlp_common.cuh"
#include "mlp_internal.h"

namespace {

constexpr int BM = 128, BN = 256;
constexpr int NEPI = 16;
constexpr int W_TMA = NEPI, W_MMA = NEPI + 1;
constexpr int L1_THREADS = 32 * (NEPI + 2);
// per-warp staging: [32 rows][64 cols] = 4 KB bf16 (2 slots) or 8 KB fp32 (1 slot)
template <bool TF32>
struct L1Stg {
  static constexpr uint32_t SLOT = 32 * 64 * (TF32 ? 4 : 2);
  static constexpr int NSLOT = TF32 ? 1 : 2;
};
#ifdef L1TRACE  // timing experiment: per-tile clock64 stamps of CTA 0 (tools/l1trace.py)
constexpr int TR_TILES = 96;
__device__ long long g_l1trace[24][TR_TILES][8];
#define TRACE(w, it, k)                                                                    \
  do {                                                                                     \
    if (blockIdx.x == 0 && (it) < TR_TILES && lane == 0) g_l1trace[w][it][k] = clock64(); \
  } while (0)
#else
#define TRACE(w, it, k) \
  do {                  \
  } while (0)
#endif

#ifndef L1_SLEEP_MASK  // which roles park while waiting: 1 producer, 2 MMA, 8 epilogue
#define L1_SLEEP_MASK 3
#endif
template <int ROLE>
__device__ __forceinline__ void wait(uint64_t *bar, uint32_t phase) {
  if (L1_SLEEP_MASK & ROLE)
    rcx::mbar_wait_sleep(bar, phase);
  else
    rcx::mbar_wait(bar, phase);
}

template <int KZ, int PREC>
__global__ void __launch_bounds__(L1_THREADS, 1)
    l1_kernel(const __grid_constant__ CUtensorMap mapZ, const __grid_constant__ CUtensorMap mapW,
              const __grid_constant__ CUtensorMap mapOut, const __grid_constant__ CUtensorMap mapZlo,
              const __grid_constant__ CUtensorMap mapWlo, const __grid_constant__ CUtensorMap mapOutlo, L1Args a) {
  static_assert(KZ == 16 || KZ == 32, "z row of 16 or 32 elements");
  constexpr bool TF32 = rcm::Prec<PREC>::TF32, X3 = rcm::Prec<PREC>::X3;
  constexpr int NOP = rcm::Prec<PREC>::NOP;
  using E = rcm::Elem<TF32>;
  constexpr int ROWB = KZ * E::BYTES;  // 32, 64 or 128-byte swizzled operand rows
  constexpr uint32_t SLOT = L1Stg<TF32>::SLOT;
  constexpr int NSLOT = L1Stg<TF32>::NSLOT;
  constexpr uint32_t A_BYTES = BM * ROWB, B_BYTES = BN * ROWB;
  constexpr uint32_t STAGE = (NOP * (A_BYTES + B_BYTES) + 1023u) & ~1023u;  // [A hi | A lo | B hi | B lo]
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base_u32 = rcx::smem_u32(smem_raw);
  uint8_t *smem = smem_raw + (((base_u32 + 1023u) & ~1023u) - base_u32);
  const int S = a.stages;
  uint8_t *sST = smem;                       // NEPI x NSLOT x SLOT
  uint8_t *sW = sST + NEPI * NSLOT * SLOT;   // S x [z tile | W1 tile]
  uint64_t *full = reinterpret_cast<uint64_t *>(sW + S * STAGE);
  uint64_t *empty = full + S, *tfull = empty + S, *tempty = tfull + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == W_TMA && lane == 0) {
    rcx::prefetch_tmap(&mapZ);
    rcx::prefetch_tmap(&mapW);
    rcx::prefetch_tmap(&mapOut);
    if (X3) {
      rcx::prefetch_tmap(&mapZlo);
      rcx::prefetch_tmap(&mapWlo);
      rcx::prefetch_tmap(&mapOutlo);
    }
    for (int s = 0; s < S; ++s) {
      rcx::mbar_init(&full[s], 1);
      rcx::mbar_init(&empty[s], 1);
    }
    for (int z = 0; z < 2; ++z) {
      rcx::mbar_init(&tfull[z], 1);
      rcx::mbar_init(&tempty[z], TF32 ? NEPI : NEPI / 2);  // bf16: one warp group per accumulator
    }
    rcx::fence_mbar_init();
  }
  if (warp == W_MMA) rcx::tmem_alloc(tmem_slot, 512);
  rcx::tc_fence_before();
  __syncthreads();
  rcx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = a.m_tiles * a.n_tiles * a.nets;

  if (warp == W_TMA) {
    if (lane == 0) {  // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int nb = tile % a.n_tiles, rest = tile / a.n_tiles;
        const int mb = rest % a.m_tiles, net = rest / a.m_tiles;
        wait<1>(&empty[s], ph ^ 1);
        rcx::mbar_arrive_expect_tx(&full[s], NOP * (A_BYTES + B_BYTES));
        uint8_t *st = sW + s * STAGE;
        rcx::tma_load_3d(st, &mapZ, &full[s], 0, mb * BM, 0);
        if (X3) rcx::tma_load_3d(st + A_BYTES, &mapZlo, &full[s], 0, mb * BM, 0);
        rcx::tma_load_3d(st + NOP * A_BYTES, &mapW, &full[s], 0, nb * BN, net);
        if (X3) rcx::tma_load_3d(st + NOP * A_BYTES + B_BYTES, &mapWlo, &full[s], 0, nb * BN, net);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == W_MMA) {
    if (lane == 0) {  // ---------------- MMA issuer
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
        const int nb = tile % a.n_tiles;
        const int n_eff = min(BN, a.N - nb * BN);  // multiple of 64
        const uint32_t idesc = rcx::make_idesc(E::FMT, BM, (uint32_t)n_eff);
        const int as = it & 1;
        TRACE(W_MMA, it, 0);
        wait<2>(&tempty[as], ((it >> 1) & 1) ^ 1);
        TRACE(W_MMA, it, 1);
        wait<2>(&full[s], ph);
        TRACE(W_MMA, it, 2);
        rcx::tc_fence_after();
        const uint64_t ad = rcm::desc_sw<ROWB>(sW + s * STAGE);
        const uint64_t bd = rcm::desc_sw<ROWB>(sW + s * STAGE + NOP * A_BYTES);
        constexpr uint64_t ALO = A_BYTES >> 4, BLO = B_BYTES >> 4;  // descriptor offsets of the lo copies
#pragma unroll
        for (int k = 0; k < KZ / E::KATOM; ++k) {  // one 32-byte K atom per MMA: descriptor start += 2
          rcm::mma_cta<TF32>(tmem + as * BN, ad + 2 * k, bd + 2 * k, idesc, k != 0);
          if (X3) {
            rcm::mma_cta<TF32>(tmem + as * BN, ad + ALO + 2 * k, bd + 2 * k, idesc, 1);
            rcm::mma_cta<TF32>(tmem + as * BN, ad + 2 * k, bd + BLO + 2 * k, idesc, 1);
          }
        }
        rcx::mma_commit(&empty[s]);
        rcx::mma_commit(&tfull[as]);
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if constexpr (!TF32) {
    // ---------------- bf16 epilogue: two groups of eight warps take alternate tiles (group g drains
    // accumulator g), so one group's TMA-store phase overlaps the other's GELU phase instead of all
    // sixteen warps of an SM sub-partition pausing the MUFU pipe together.  In a group, warp
    // (q, hb) converts rows q*32.. and columns hb*128.. as two 64-column blocks; it releases the
    // accumulator after loading its second block.
    const int g = warp >> 3, q = warp & 3, hb = (warp >> 2) & 1;
    uint8_t *stg0 = sST + warp * NSLOT * SLOT;
    int it = 0, nst = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      if ((it & 1) != g) continue;
      const int nb = tile % a.n_tiles, rest = tile / a.n_tiles;
      const int mb = rest % a.m_tiles, net = rest / a.m_tiles;
      const int n_eff = min(BN, a.N - nb * BN);
      const int nblk = max(0, min(2, (n_eff - hb * 128) / 64));  // this warp's 64-column blocks: 0..2
      wait<8>(&tfull[g], (it >> 1) & 1);
      rcx::tc_fence_after();
      if (nblk == 0) {
        rcx::tc_fence_before();
        __syncwarp();
        if (lane == 0) rcx::mbar_arrive(&tempty[g]);
        continue;
      }
#pragma unroll 1
      for (int j = 0; j < nblk; ++j) {
        uint32_t v[4][16];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + g * BN + hb * 128 + j * 64;
#pragma unroll
        for (int c = 0; c < 4; ++c) rcx::tmem_ld16(ta + c * 16, v[c]);
        rcx::tmem_ld_wait();
        if (j == nblk - 1) {  // all of this warp's columns are out of TMEM
          rcx::tc_fence_before();
          __syncwarp();
          if (lane == 0) rcx::mbar_arrive(&tempty[g]);
        }
        uint8_t *stg = stg0 + (nst & 1) * SLOT;
        if (lane == 0) rcm::bulk_wait_read1();  // the store that last used this slot has read it
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            pk[k] = rcm::gelu_half_f16x2_bf16x2(rcm::cvt_f16x2(__uint_as_float(v[c][2 * k]), __uint_as_float(v[c][2 * k + 1])));
          rcm::stage_sw128(stg, lane, 2 * c, pk);
        }
        rcm::fence_async_smem();
        __syncwarp();
        if (lane == 0) {
          rcm::tma_store_3d(&mapOut, stg, nb * BN + hb * 128 + j * 64, mb * BM + q * 32, net);
          rcm::bulk_commit();
        }
        ++nst;
      }
    }
    if (lane == 0) rcm::bulk_wait_all();
    __syncwarp();
  } else {  // ---------------- TF32 epilogue, warps 0..15: 32 rows (lane quadrant q) x 64 columns (block sub)
    const int q = warp & 3, sub = warp >> 2;
    uint8_t *stg0 = sST + warp * NSLOT * SLOT;
    int it = 0, nst = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      const int nb = tile % a.n_tiles, rest = tile / a.n_tiles;
      const int mb = rest % a.m_tiles, net = rest / a.m_tiles;
      const bool mine = sub * 64 < a.N - nb * BN;  // warp-uniform: this column block exists
      const int as = it & 1;
      TRACE(warp, it, 0);
      wait<8>(&tfull[as], (it >> 1) & 1);
      TRACE(warp, it, 1);
      rcx::tc_fence_after();
      uint32_t v[4][16];
      if (mine) {
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + as * BN + sub * 64;
#pragma unroll
        for (int c = 0; c < 4; ++c) rcx::tmem_ld16(ta + c * 16, v[c]);
        rcx::tmem_ld_wait();
      }
      rcx::tc_fence_before();
      __syncwarp();
      if (lane == 0) rcx::mbar_arrive(&tempty[as]);
      TRACE(warp, it, 2);
      if (!mine) continue;
      uint8_t *stg = stg0 + (nst % NSLOT) * SLOT;
      if (lane == 0) {  // the store that last used this slot has read it
        if constexpr (NSLOT == 2) rcm::bulk_wait_read1(); else rcm::bulk_wait_read0();
      }
      __syncwarp();
      if constexpr (TF32) {
        // exact GELU in fp32, tf32-rounded (X3: hi now, lo after the hi stores have read the slot);
        // [32 rows][32 fp32] blocks, 128-byte swizzle
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float g[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) g[j] = rcm::tf32_rn(rcm::gelu_erf_f32(__uint_as_float(v[c][j])));
          uint8_t *r = stg + (c >> 1) * 4096 + lane * 128;
          const int x = lane & 7, u0 = (c & 1) * 4;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            *reinterpret_cast<float4 *>(r + (((u0 + u) ^ x) << 4)) = make_float4(g[4 * u], g[4 * u + 1], g[4 * u + 2], g[4 * u + 3]);
        }
        if constexpr (X3) {
          rcm::fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            rcm::tma_store_3d(&mapOut, stg, nb * BN + sub * 64, mb * BM + q * 32, net);
            rcm::tma_store_3d(&mapOut, stg + 4096, nb * BN + sub * 64 + 32, mb * BM + q * 32, net);
            rcm::bulk_commit();
            rcm::bulk_wait_read0();
          }
          __syncwarp();
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float g[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float y = rcm::gelu_erf_f32(__uint_as_float(v[c][j]));
              g[j] = rcm::tf32_rn(y - rcm::tf32_rn(y));
            }
            uint8_t *r = stg + (c >> 1) * 4096 + lane * 128;
            const int x = lane & 7, u0 = (c & 1) * 4;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              *reinterpret_cast<float4 *>(r + (((u0 + u) ^ x) << 4)) = make_float4(g[4 * u], g[4 * u + 1], g[4 * u + 2], g[4 * u + 3]);
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t pk[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            pk[j] = rcm::gelu_half_f16x2_bf16x2(rcm::cvt_f16x2(__uint_as_float(v[c][2 * j]), __uint_as_float(v[c][2 * j + 1])));
          rcm::stage_sw128(stg, lane, 2 * c, pk);
        }
      }
      rcm::fence_async_smem();
      __syncwarp();
      TRACE(warp, it, 3);
      if (lane == 0) {
        if constexpr (TF32) {
          const CUtensorMap *mo = X3 ? &mapOutlo : &mapOut;  // X3: the hi half was stored above
          rcm::tma_store_3d(mo, stg, nb * BN + sub * 64, mb * BM + q * 32, net);
          rcm::tma_store_3d(mo, stg + 4096, nb * BN + sub * 64 + 32, mb * BM + q * 32, net);
        } else {
          rcm::tma_store_3d(&mapOut, stg, nb * BN + sub * 64, mb * BM + q * 32, net);
        }
        rcm::bulk_commit();
      }
      ++nst;
    }
    if (lane == 0) rcm::bulk_wait_all();
    __syncwarp();
  }
  __syncthreads();
  if (warp == W_MMA) {
    rcx::tc_fence_after();
    rcx::tmem_dealloc(tmem, 512);
  }
}

template <int KZ, int PREC>
int launch_t(const CUtensorMap *M, L1Args a, cudaStream_t s) {
  constexpr bool TF32 = PREC != 0;
  constexpr int EB = rcm::Elem<TF32>::BYTES;
  constexpr size_t STAGE = (rcm::Prec<PREC>::NOP * (BM * KZ * EB + BN * KZ * EB) + 1023) & ~(size_t)1023;
  const size_t fixed = 1024 + NEPI * L1Stg<TF32>::NSLOT * L1Stg<TF32>::SLOT + 256;
  int stages = (int)((232448 - fixed) / STAGE);
  if (stages > 8) stages = 8;
  a.stages = stages;
  const size_t smem = fixed + stages * STAGE;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(l1_kernel<KZ, PREC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    attr = true;
  }
  const int total = a.m_tiles * a.n_tiles * a.nets;
  const int grid = total < mlp_num_sms() ? total : mlp_num_sms();
  l1_kernel<KZ, PREC><<<grid, L1_THREADS, smem, s>>>(M[0], M[1], M[2], M[3], M[4], M[5], a);
  RC_LAUNCH_CHECK();
  return RC_OK;
}

}  // namespace

int l1_tile_n() { return BN; }
int l1_box_rows() { return BN; }

#ifdef L1TRACE
extern "C" __attribute__((visibility("default"))) int rc_debug_l1trace(void *host) {
  return (int)cudaMemcpyFromSymbol(host, g_l1trace, sizeof(g_l1trace));
}
#endif

int launch_l1(int KZ, int prec, const CUtensorMap *maps, const L1Args &a, cudaStream_t s) {
  ProfScope prof(RC_STAGE_L1, s);
  if (a.N % 64) return rc_fail(RC_EUNSUPPORTED, "layer-1 GEMM: h1 = %d is not a multiple of 64", a.N);
#define RC_L1(kz)                                                                                      \
  if (KZ == kz)                                                                                        \
    return prec == 0 ? launch_t<kz, 0>(maps, a, s) : prec == 1 ? launch_t<kz, 1>(maps, a, s) : launch_t<kz, 2>(maps, a, s);
  RC_L1(16)
  RC_L1(32)
#undef RC_L1
  return rc_fail(RC_EUNSUPPORTED, "layer-1 GEMM: no instance for K = %d", KZ);
}
