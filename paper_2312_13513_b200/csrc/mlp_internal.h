// mlp_internal.h -- shared declarations of the MLP kernels (mlp_sm100.cu, mlp_l12_sm100.cu)
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "rc_internal.h"

struct L12Args {
  int m_tiles, passes, nets, chunks, h2, cap, stages;
  const float *b2;         // [nets][h2]
  __nv_bfloat16 *h2out;    // [nets][cap][h2]
  unsigned long long *dbg; // optional event timeline of CTA 0 (developer tool)
  int flags;               // developer diagnostics (0 in production): bit0 skip a2full, bit1 skip weight loads
};

int mlp_num_sms();
int l12_pass_width(int h2);
int launch_l12_pair(int NP, int KZ, const CUtensorMap &Z, const CUtensorMap &W1, const CUtensorMap &W2a,
                    const CUtensorMap &W2b, const CUtensorMap &H2, const L12Args &a, cudaStream_t s);
