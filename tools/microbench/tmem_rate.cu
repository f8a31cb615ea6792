// TMEM read throughput on B200 (tcgen05.ld 32x32b.x16, 16 warps = 4 per lane quadrant),
// alone and interleaved with the packed-bf16x2 GELU of the layer-1 epilogue.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2312_13513_b200/csrc tmem_rate.cu -o tmem_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

__device__ __forceinline__ uint32_t gelu2(uint32_t x) {
  const uint32_t c0 = 0x3F4C3F4Cu, c1 = 0x3D123D12u, hf = 0x3F003F00u; uint32_t xx, t, u, th, hx, r;
  asm("mul.rn.bf16x2 %0, %1, %1;" : "=r"(xx) : "r"(x)); asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(t) : "r"(xx), "r"(c1), "r"(c0));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(u) : "r"(t), "r"(x)); asm("tanh.approx.bf16x2 %0, %1;" : "=r"(th) : "r"(u));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(hx) : "r"(x), "r"(hf)); asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(hx), "r"(th), "r"(hx));
  return r;
}

template <int MODE, int NC>
__global__ void __launch_bounds__(512, 1) k(int iters, uint32_t *out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) rcx::tmem_alloc(&slot, 512);
  rcx::tc_fence_before();
  __syncthreads();
  rcx::tc_fence_after();
  const uint32_t tb = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * NC * 16;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t v[NC][16];
    if (MODE != 2) {
#pragma unroll
      for (int c = 0; c < NC; ++c) rcx::tmem_ld16(tb + c * 16, v[c]);
      rcx::tmem_ld_wait();
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < 16; ++j) v[c][j] = __float_as_uint(0.01f * (it + c + j) + threadIdx.x * 1e-3f);
    }
    if (MODE == 0) {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < 16; ++j) acc ^= v[c][j];
    } else {
#pragma unroll
      for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          uint32_t p;
          asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(__uint_as_float(v[c][2 * j + 1])), "f"(__uint_as_float(v[c][2 * j])));
          acc ^= gelu2(p);
        }
    }
  }
  if (acc == 0x12345678) out[0] = acc;
  rcx::tc_fence_before();
  __syncthreads();
  if (warp == 0) rcx::tmem_dealloc(slot, 512);
}

int main() {
  uint32_t *d; cudaMalloc(&d, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *names[] = {"tmem ld only", "tmem ld + cvt + gelu", "gelu only (register data)"};
  for (int m = 0; m < 3; ++m) {
    const int iters = 20000; dim3 g(148), b(512);
    auto launch = [&]() { if (m == 0) k<0, 4><<<g, b>>>(iters, d); else if (m == 1) k<1, 4><<<g, b>>>(iters, d); else k<2, 4><<<g, b>>>(iters, d); };
    launch(); cudaError_t e = cudaDeviceSynchronize(); if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double elems = 4.0 * 16 * 32 * 16 * (double)iters * g.x;  // fp32 accumulator elements read per launch
    printf("%-28s %8.1f Gelem/s = %6.2f elem/clk/SM (%.1f B/clk/SM) @%.2f GHz\n", names[m], elems / ms / 1e6,
           elems / ms / 1e6 / 148 / (clk / 1e6), 4 * elems / ms / 1e6 / 148 / (clk / 1e6), clk / 1e6);
  }
  return 0;
}
