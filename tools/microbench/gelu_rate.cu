// Throughput of the GELU building blocks on B200: tanh.approx.{f32,bf16x2},
// fma.rn.bf16x2, and the full packed-bf16x2 GELU vs the fp32 one.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t tanh2(uint32_t x) { uint32_t r; asm volatile("tanh.approx.bf16x2 %0, %1;" : "=r"(r) : "r"(x)); return r; }
__device__ __forceinline__ uint32_t tanh2h(uint32_t x) { uint32_t r; asm volatile("tanh.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x)); return r; }
__device__ __forceinline__ uint32_t ex2h(uint32_t x) { uint32_t r; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x)); return r; }
__device__ __forceinline__ float tanh1(float x) { float r; asm volatile("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ uint32_t fma2(uint32_t a, uint32_t b, uint32_t c) { uint32_t r; asm volatile("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r; }
__device__ __forceinline__ uint32_t gelu2(uint32_t x) {
  const uint32_t c0 = 0x3F4C3F4Cu, c1 = 0x3D123D12u, hf = 0x3F003F00u; uint32_t xx, t, u, th, hx, r;
  asm("mul.rn.bf16x2 %0, %1, %1;" : "=r"(xx) : "r"(x)); asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(t) : "r"(xx), "r"(c1), "r"(c0));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(u) : "r"(t), "r"(x)); asm("tanh.approx.bf16x2 %0, %1;" : "=r"(th) : "r"(u));
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(hx) : "r"(x), "r"(hf)); asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(hx), "r"(th), "r"(hx));
  return r;
}
__device__ __forceinline__ float gelu1(float x) { float u = x * fmaf(0.0356774081f, x * x, 0.7978845608f); float hx = 0.5f * x; return fmaf(hx, tanh1(u), hx); }

template <int MODE>
__global__ void k(int iters, uint32_t *out) {
  uint32_t v[8]; float f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { v[i] = 0x3E003E00u + threadIdx.x + i; f[i] = 0.1f * i + threadIdx.x * 1e-4f; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) v[i] = tanh2(v[i]);
      if (MODE == 1) f[i] = tanh1(f[i]);
      if (MODE == 2) v[i] = fma2(v[i], 0x3F803F80u, 0x00010001u);
      if (MODE == 3) v[i] = gelu2(v[i]);
      if (MODE == 4) f[i] = gelu1(f[i]);
      if (MODE == 5) {  // fp32 accumulator pair -> cvt.rn.bf16x2 -> packed GELU (the epilogue's per-pair work)
        uint32_t p; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(f[i]), "f"(f[(i + 1) & 7]));
        p = gelu2(p); f[i] = __uint_as_float(p) * 1e-3f + f[i];
      }
      if (MODE == 7) v[i] = tanh2h(v[i]);
      if (MODE == 8) v[i] = ex2h(v[i]);
      if (MODE == 9) {  // RNE to bf16 on the FMA pipe (Veltkamp split, s = 2^16 + 1) + PRMT pack
        const float a = f[i], b = f[(i + 1) & 7];
        const float ta = a * 65537.0f, tb = b * 65537.0f;
        const float ha = ta - (ta - a), hb = tb - (tb - b);
        uint32_t p; asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(p) : "r"(__float_as_uint(ha)), "r"(__float_as_uint(hb)));
        f[i] = __uint_as_float(p) + f[i];
      }
      if (MODE == 10) {  // one cvt.rn.bf16x2 + one tanh.approx.f32 per pair: do they share a pipe?
        uint32_t p; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(f[i]), "f"(f[(i + 1) & 7]));
        f[i] = __uint_as_float(p) + tanh1(f[i]);
      }
      if (MODE == 6) { uint32_t p; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(f[i]), "f"(f[(i + 1) & 7])); f[i] = __uint_as_float(p) + f[i]; }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= v[i] ^ __float_as_uint(f[i]);
  if (s == 0x12345678) out[0] = s;
}
int main() {
  uint32_t *d; cudaMalloc(&d, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *names[] = {"tanh.approx.bf16x2 (elements)", "tanh.approx.f32", "fma.rn.bf16x2 (elements)", "gelu bf16x2 (elements)", "gelu f32", "cvt+gelu bf16x2 (elements)", "cvt.rn.bf16x2.f32 (elements)", "tanh.approx.f16x2 (elements)", "ex2.approx.f16x2 (elements)", "veltkamp rne + prmt (elements)", "cvt pair + tanh.f32 (pairs)"};
  for (int warps : {16}) {
    for (int m = 0; m < 11; ++m) {
      int iters = 4096; dim3 g(148), b(32 * warps);
      auto launch = [&]() { switch (m) { case 0: k<0><<<g, b>>>(iters, d); break; case 1: k<1><<<g, b>>>(iters, d); break;
        case 2: k<2><<<g, b>>>(iters, d); break; case 3: k<3><<<g, b>>>(iters, d); break; case 4: k<4><<<g, b>>>(iters, d); break; case 5: k<5><<<g, b>>>(iters, d); break; case 6: k<6><<<g, b>>>(iters, d); break; case 7: k<7><<<g, b>>>(iters, d); break; case 8: k<8><<<g, b>>>(iters, d); break; case 9: k<9><<<g, b>>>(iters, d); break; case 10: k<10><<<g, b>>>(iters, d); break; } };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double elems = 8.0 * iters * g.x * b.x * ((m == 0 || m == 2 || m == 3 || m == 5 || m == 6 || m == 7 || m == 8 || m == 9) ? 2 : 1);
      printf("warps/SM=%2d %-32s %8.1f Gelem/s = %6.1f elem/clk/SM @1.9GHz\n", warps, names[m], elems / ms / 1e6, elems / ms / 1e6 / 148 / 1.9);
    }
  }
  return 0;
}
