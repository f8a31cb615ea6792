// fp64_lat.cu -- dependent-issue latency of DFMA / DMUL / MUFU.RCP64H + Newton, and the FP64 pipe
// throughput per SM vs independent chains per warp and warps per SM (the cell-local fp64 kernels are
// latency chains: Newton, Horner, exp).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat(double *out, long long *cyc, int n) {
  double x = out[threadIdx.x], a = 1.0000001, b = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CH>
__global__ void thr(double *out, int n) {
  double x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = out[threadIdx.x] + c;
  const double a = 1.0000001, b = 1e-9;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double *d; long long *c;
  cudaMalloc(&d, 1 << 26); cudaMalloc(&c, 8);
  cudaMemset(d, 0, 1 << 26);
  const int n = 4096;
  lat<<<1, 32>>>(d, c, n);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("{\"dfma_dependent_latency_clk\": %.2f", (double)h / n);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int warps : {4, 8, 16, 32}) {
    for (int ch : {1, 2, 4, 8}) {
      auto run = [&](auto k) {
        k<<<sms, warps * 32>>>(d, n);
        cudaEventRecord(e0);
        k<<<sms, warps * 32>>>(d, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)sms * warps * 32 * n * ch;
        printf(", \"w%d_ch%d_dfma_per_clk_per_sm\": %.1f", warps, ch, ops / (ms * 1e-3) / sms / (clk * 1e3));
      };
      if (ch == 1) run(thr<1>); else if (ch == 2) run(thr<2>); else if (ch == 4) run(thr<4>); else run(thr<8>);
    }
  }
  printf("}\n");
  return 0;
}
