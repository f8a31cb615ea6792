// Raw tcgen05.mma issue/execute rate on B200 for the shapes the fused MLP uses.
// Each CTA (or CTA pair) loops MMAs on garbage smem operands with no other work;
// reports achieved dense TFLOP/s for the whole GPU.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2312_13513_b200/csrc/ptx.cuh"

template <int ROWB>
__device__ __forceinline__ uint64_t dsw(const void *p) {
  constexpr uint64_t layout = ROWB == 128 ? 2 : ROWB == 64 ? 4 : 6;
  uint64_t d = (uint64_t)((rcx::smem_u32(p) & 0x3FFFF) >> 4);
  d |= (uint64_t)((8 * ROWB) >> 4) << 32; d |= (uint64_t)1 << 46; d |= layout << 61; return d;
}

// mode 0: cta_group::1, M=128, N=n1 (+ n2 second MMA); mode 1: cta_group::2 M=256
template <int PAIR>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, int n1, int n2, unsigned long long *out, int l1) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *base = sm + ((1024 - (rcx::smem_u32(sm) & 1023)) & 1023);
  const int warp = threadIdx.x >> 5;
  uint32_t rank = PAIR ? rcx::cluster_rank() : 0;
  if (threadIdx.x == 0) { rcx::mbar_init(&bar, 1); rcx::fence_mbar_init(); }
  if (warp == 0) { if (PAIR) rcx::tmem_alloc_pair(&slot, 512); else rcx::tmem_alloc(&slot, 512); }
  rcx::tc_fence_before();
  if (PAIR) rcx::cluster_sync(); else __syncthreads();
  rcx::tc_fence_after();
  uint32_t tm = slot;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t M = PAIR ? 256 : 128;
    uint32_t id1 = rcx::make_idesc(1, M, n1), id2 = rcx::make_idesc(1, M, n2 > 0 ? n2 : 16);
    uint64_t da = dsw<128>(base), db = dsw<128>(base + 32768);
    if (l1 == 64) { da = dsw<64>(base); db = dsw<64>(base + 32768); }  // 64-byte swizzle operands
    unsigned long long t0 = clock64();
    const uint32_t idl1 = rcx::make_idesc(1, M, 64);
    uint64_t dz = dsw<128>(base + 65536), dw1 = dsw<128>(base + 98304);
    __shared__ uint64_t done_bar, cbar[4];
    rcx::mbar_init(&done_bar, 1); for (int b = 0; b < 4; ++b) rcx::mbar_init(&cbar[b], 1);
    rcx::fence_mbar_init();
    rcx::mbar_arrive(&done_bar);            // phase 0 complete: try_wait(parity 0) returns true forever after
    for (int i = 0; i < iters; ++i) {
      // sync-overhead emulation between K64 steps: l1 >= 10 -> (l1 - 10) try_waits on a completed barrier,
      // l1 >= 20 -> (l1 - 20) commits, l1 >= 30 -> waits+commits interleaved between MMAs
      if (l1 >= 10 && l1 < 20) for (int w = 0; w < l1 - 10; ++w) rcx::mbar_wait(&done_bar, 0);
      if (l1 >= 20 && l1 < 30) for (int w = 0; w < l1 - 20; ++w) { if (PAIR) rcx::mma_commit_pair(&cbar[w & 3]); else rcx::mma_commit(&cbar[w & 3]); }
      if (l1 == 1) {  // layer-1 MMA (N=64, K=16) into its own accumulator before the layer-2 chunk
        if (PAIR) rcx::mma_bf16_pair(tm + 448, dz, dw1, idl1, 1); else rcx::mma_bf16(tm + 448, dz, dw1, idl1, 1);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (l1 >= 30 && k < l1 - 30) { rcx::mbar_wait(&done_bar, 0); if (PAIR) rcx::mma_commit_pair(&cbar[k]); else rcx::mma_commit(&cbar[k]); }
        if (l1 == 2 && k == 1) {  // layer-1 MMA issued between the layer-2 K16 steps
          if (PAIR) rcx::mma_bf16_pair(tm + 448, dz, dw1, idl1, 1); else rcx::mma_bf16(tm + 448, dz, dw1, idl1, 1);
        }
        if (PAIR) {
          rcx::mma_bf16_pair(tm, da + 2 * k, db + 2 * k, id1, 1);
          if (n2) rcx::mma_bf16_pair(tm + n1, da + 2 * k, db + 2048 + 2 * k, id2, 1);
        } else {
          rcx::mma_bf16(tm, da + 2 * k, db + 2 * k, id1, 1);
          if (n2) rcx::mma_bf16(tm + n1, da + 2 * k, db + 2048 + 2 * k, id2, 1);
        }
      }
    }
    if (PAIR) rcx::mma_commit_pair(&bar); else rcx::mma_commit(&bar);
    rcx::mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  if (PAIR) { rcx::tc_fence_before(); rcx::cluster_sync(); }
  else { rcx::tc_fence_before(); __syncthreads(); }
  if (PAIR && rank == 1 && threadIdx.x == 0) {}  // peer just waits
  if (warp == 0) { rcx::tc_fence_after(); if (PAIR) rcx::tmem_dealloc_pair(tm, 512); else rcx::tmem_dealloc(tm, 512); }
}

int main() {
  unsigned long long *d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_loop<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(mma_loop<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct C { int pair, n1, n2, l1; } cs[] = {{1, 256, 144, 0}, {1, 256, 144, 64}, {1, 256, 144, 11}, {1, 256, 144, 21}};
  for (auto c : cs) {
    int iters = 2000;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = c.pair ? 2 : 1;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (c.pair) cudaLaunchKernelEx(&cfg, mma_loop<1>, iters, c.n1, c.n2, d, c.l1);
      else cudaLaunchKernelEx(&cfg, mma_loop<0>, iters, c.n1, c.n2, d, c.l1);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    double M = c.pair ? 256 : 128, ctas = c.pair ? 74 : 148;
    double flops = 2.0 * M * (c.n1 + c.n2) * 64 * iters * ctas;
    cudaError_t e = cudaGetLastError();
    printf("pair=%d N=%d+%d l1=%d : %.1f TFLOP/s (L2 flops only), %.1f clk per K64-step (cta0), err=%s\n", c.pair, c.n1, c.n2, c.l1, flops / ms / 1e9,
           (double)cyc / iters, cudaGetErrorString(e));
  }
  return 0;
}
