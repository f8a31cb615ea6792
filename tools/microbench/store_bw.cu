// HBM write bandwidth on B200 by store path (per-SM staging -> global):
//   stg   : every warp writes 16-byte coalesced STG.128 (4 full 128-B lines per instruction)
//   bulk1 : one thread per CTA issues cp.async.bulk (smem -> global) of CHUNK bytes, D groups in flight
//   bulkw : every warp's lane 0 issues its own cp.async.bulk of CHUNK bytes, 2 in flight per warp
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 store_bw.cu -o store_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512) k_stg(uint4 *out, size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) out[i] = v;
}

template <int CHUNK, int D>
__global__ void __launch_bounds__(512) k_bulk1(uint8_t *out, size_t bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < CHUNK * D / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nchunks = bytes / CHUNK;
  int k = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * CHUNK),
                 "r"(smem_u32(sm + (k % D) * CHUNK)), "r"(CHUNK)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(D - 1) : "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int CHUNK>
__global__ void __launch_bounds__(512) k_bulkw(uint8_t *out, size_t bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint8_t *mine = sm + warp * 2 * CHUNK;
  for (int i = lane; i < 2 * CHUNK / 4; i += 32) reinterpret_cast<uint32_t *>(mine)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane != 0) return;
  const size_t nchunks = bytes / CHUNK;
  int k = 0;
  for (size_t c = (size_t)blockIdx.x * nw + warp; c < nchunks; c += (size_t)gridDim.x * nw, ++k) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * CHUNK),
                 "r"(smem_u32(mine + (k & 1) * CHUNK)), "r"(CHUNK)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = (size_t)1 << 31;  // 2 GiB
  uint8_t *d;
  cudaMalloc(&d, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  auto run = [&](const char *name, auto launch) {
    launch();
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = 5.0 * bytes / (ms * 1e-3) / 1e9;
    printf("%-34s %8.1f GB/s  (%5.1f B/clk/SM @ %.2f GHz)\n", name, gbs, gbs * 1e9 / 148 / (clk * 1e3), clk / 1e6);
  };
  run("stg 512 thr x 148", [&] { k_stg<<<148, 512>>>(reinterpret_cast<uint4 *>(d), bytes / 16); });
  run("stg 512 thr x 296", [&] { k_stg<<<296, 512>>>(reinterpret_cast<uint4 *>(d), bytes / 16); });
#define B1(C, D)                                                                                   \
  cudaFuncSetAttribute(k_bulk1<C, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);   \
  run("bulk1 chunk " #C " depth " #D, [&] { k_bulk1<C, D><<<148, 32, C * D>>>(d, bytes); });
  B1(4096, 2) B1(4096, 6) B1(4096, 16) B1(4096, 32) B1(16384, 4) B1(16384, 8) B1(32768, 4)
#define BW(C, W)                                                                                    \
  cudaFuncSetAttribute(k_bulkw<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);       \
  run("bulkw chunk " #C " warps " #W, [&] { k_bulkw<C><<<148, 32 * W, 2 * C * W>>>(d, bytes); });
  BW(1024, 16) BW(4096, 16) BW(4096, 8) BW(8192, 8)
  return 0;
}
