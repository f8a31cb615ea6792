// mlp_internal.h -- shared declarations of the MLP kernels (mlp_sm100.cu, mlp_l2_sm100.cu)
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "rc_internal.h"

int mlp_num_sms();

// layer 1 (mlp_l1_sm100.cu): h1 = GELU(z W1^T), 128 x 256 tiles (W1 boxes of l1_box_rows() rows),
// h1 TMA-stored through `Out` (128-byte-swizzled 32-row boxes: 64 bf16 or 32 fp32 columns) into
// [nets][cap][N]; bf16 (W1 stored halved) or tf32 (fp32 storage, tf32-rounded) precision
struct L1Args {
  int m_tiles, n_tiles, nets, N, stages, cap;
};
int l1_tile_n();
int l1_box_rows();
// maps: {z, W1, h1 store, z lo, W1 lo, h1 lo store} (the lo maps are used by precision 2 only)
int launch_l1(int KZ, int prec, const CUtensorMap *maps, const L1Args &a, cudaStream_t s);
int l2_pass_width(int h2);

struct L2Args {
  int m_tiles, passes, nets, chunks, N, stages;
  const float *bias;       // [nets][N]
  const float *w4;         // layer-3 mode (nullptr: layer 2): [nets][N], layer 4 folded into the epilogue
  float *opart;            // layer-3 mode: [nets][passes][cap] dots (column quarters summed in-kernel)
  int cap;
  int ktail;               // MMA K atoms in the last K chunk when K is not a multiple of it (0: full chunk)
  int prof_stage = -1;     // rc_profile stage (-1: L3 with w4, else L2)
  // Dynamic tile schedule (layer 3 overlapped with the fused layer-1/2 kernel): the
  // CTA pairs take tiles from *tile_ctr (zeroed before the first launch that shares it); nullptr:
  // the static schedule cl, cl + ncl, ...
  int *tile_ctr = nullptr;
  // Filler launch (runs beside the fused layer-1/2 kernel on the SMs its 4-CTA clusters leave
  // idle): take tiles only once *gate >= gate_target (every cluster of that kernel is resident,
  // so this launch holds no SM the kernel needs); after gate_ns without that, do nothing.
  const int *gate = nullptr;
  int gate_target = 0;
  unsigned gate_ns = 0;
};
// fused layers 1+2 (mlp_l12_sm100.cu, bf16, h2 = 800): clusters of two CTA pairs share h1 chunks
// maps: {z (KZ x 128 rows), W1 (KZ x 16 rows), W2 piece 1 (32 x 128 rows), W2 piece 2 (32 x 72 rows),
//        h2 store (16 x 32), b2 as K = 16 operand piece 1 (16 x 128 rows), piece 2 (16 x 72 rows)}
struct L12Args {
  int m_tiles, nets, chunks, N, stages;
  const float *bias;  // b2 [nets][N]
  int *started = nullptr;  // += 1 per cluster once it is resident (the layer-3 filler's gate)
};
bool l12_supported(int h1, int h2, int kz, bool tf32);
// *clusters (optional) = the 4-CTA clusters launched
int launch_l12(int KZ, bool tf32, const CUtensorMap *maps, const L12Args &a, cudaStream_t s, int *clusters = nullptr);

// maps: {A, B piece 1, B piece 2, out store, A lo, B1 lo, B2 lo, out lo store, bias operand piece 1,
//        bias operand piece 2} (lo: precision 2 only; bias operand tiles: bf16 only)
// pairs (optional): CTA pairs to launch (default: as many as are resident at once)
int launch_l2_pair(int NP, int prec, const CUtensorMap *maps, const L2Args &a, cudaStream_t s, int pairs = 0);
