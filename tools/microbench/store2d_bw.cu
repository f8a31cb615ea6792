// HBM write bandwidth of 2D TMA tensor stores in the layer-1 pattern:
// h1 [nets=8][cap=32768][1600] bf16, tiles of 128 rows x 256 cols (last 64) in
// round-robin over 148 CTAs, each tile written as 16 boxes of 64 cols x 32 rows
// (128-byte swizzle), either by one issuing thread (depth D) or by 16 warps.
// Also: the same tile sweep with plain coalesced STG.128 (4 rows x 128 B per instr).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 store2d_bw.cu -o store2d_bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int NETS = 8, CAP = 32768, N = 1600, BM = 128, BN = 256;
constexpr int MT = CAP / BM, NT = (N + BN - 1) / BN;

__device__ __forceinline__ void st3d(const CUtensorMap *m, const void *src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

template <int D>
__global__ void k_one(const __grid_constant__ CUtensorMap map) {
  extern __shared__ __align__(1024) uint8_t sm[];
  for (int i = threadIdx.x; i < 4096 * D / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i * 2654435761u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  int k = 0;
  for (int t = blockIdx.x; t < NETS * MT * NT; t += gridDim.x) {
    const int nb = t % NT, mb = (t / NT) % MT, net = t / (NT * MT);
    for (int w = 0; w < 16; ++w) {
      const int q = w & 3, sub = w >> 2;
      if (nb * BN + sub * 64 >= N) continue;
      st3d(&map, sm + (k % D) * 4096, nb * BN + sub * 64, mb * BM + q * 32, net);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(D - 1) : "memory");
      ++k;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_warps(const __grid_constant__ CUtensorMap map) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = warp & 3, sub = warp >> 2;
  uint8_t *mine = sm + warp * 8192;
  for (int i = lane; i < 2048; i += 32) reinterpret_cast<uint32_t *>(mine)[i] = i * 2654435761u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane != 0) return;
  int k = 0;
  for (int t = blockIdx.x; t < NETS * MT * NT; t += gridDim.x) {
    const int nb = t % NT, mb = (t / NT) % MT, net = t / (NT * MT);
    if (nb * BN + sub * 64 >= N) continue;
    st3d(&map, mine + (k & 1) * 4096, nb * BN + sub * 64, mb * BM + q * 32, net);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    ++k;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_stg(uint16_t *h1) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = warp & 3, sub = warp >> 2;
  const uint4 v = make_uint4(lane, warp, 7, 9);
  for (int t = blockIdx.x; t < NETS * MT * NT; t += gridDim.x) {
    const int nb = t % NT, mb = (t / NT) % MT, net = t / (NT * MT);
    if (nb * BN + sub * 64 >= N) continue;
    uint16_t *g = h1 + ((size_t)net * CAP + (size_t)mb * BM + q * 32) * N + nb * BN + sub * 64;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int r = 4 * k + (lane >> 3);
      *reinterpret_cast<uint4 *>(g + (size_t)r * N + (lane & 7) * 8) = v;
    }
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const size_t bytes = (size_t)NETS * CAP * N * 2;
  uint16_t *d;
  cudaMalloc(&d, bytes);
  void *p = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<EncodeTiledFn>(p);
  CUtensorMap map;
  cuuint64_t dims[3] = {N, CAP, NETS}, strides[2] = {N * 2, (cuuint64_t)N * CAP * 2};
  cuuint32_t box[3] = {64, 32, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) { printf("encode failed %d\n", (int)r); return 1; }
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
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double gbs = 5.0 * bytes / (ms * 1e-3) / 1e9;
    printf("%-30s %7.1f us/launch %8.1f GB/s (%5.1f B/clk/SM)\n", name, ms * 1e3 / 5, gbs, gbs * 1e9 / 148 / (clk * 1e3));
  };
#define ONE(D)                                                                               \
  cudaFuncSetAttribute(k_one<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 * D);     \
  run("tma2d one thread depth " #D, [&] { k_one<D><<<148, 128, 4096 * D>>>(map); });
  ONE(2) ONE(6) ONE(16) ONE(32)
  cudaFuncSetAttribute(k_warps, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 8192);
  run("tma2d 16 warps x 2", [&] { k_warps<<<148, 512, 16 * 8192>>>(map); });
  run("stg tile sweep 16 warps", [&] { k_stg<<<148, 512>>>(d); });
  run("stg tile sweep 16 warps x2 CTA", [&] { k_stg<<<296, 512>>>(d); });
  return 0;
}
