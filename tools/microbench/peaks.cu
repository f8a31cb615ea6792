// Microbenchmarks for the B200 roofline denominators this build needs but
// MEASURED_PEAKS.json lacks: FP64 DFMA rate, FP32 FFMA rate, MUFU tanh rate,
// L2-resident read bandwidth, HBM read bandwidth.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template<int CH>
__global__ void dfma_k(double* out, int iters, double a, double b){
  double x[CH];
  #pragma unroll
  for(int i=0;i<CH;i++) x[i]=threadIdx.x*1e-3+i;
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int i=0;i<CH;i++) x[i]=fma(x[i],a,b);
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<CH;i++) s+=x[i];
  if(s==1234.5) out[0]=s;
}
template<int CH>
__global__ void ffma_k(float* out, int iters, float a, float b){
  float x[CH];
  #pragma unroll
  for(int i=0;i<CH;i++) x[i]=threadIdx.x*1e-3f+i;
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int i=0;i<CH;i++) x[i]=fmaf(x[i],a,b);
  }
  float s=0;
  #pragma unroll
  for(int i=0;i<CH;i++) s+=x[i];
  if(s==1234.5f) out[0]=s;
}
template<int CH>
__global__ void tanh_k(float* out, int iters){
  float x[CH];
  #pragma unroll
  for(int i=0;i<CH;i++) x[i]=threadIdx.x*1e-3f+i*0.01f;
  for(int it=0;it<iters;it++){
    #pragma unroll
    for(int i=0;i<CH;i++){ float y; asm volatile("tanh.approx.f32 %0, %1;":"=f"(y):"f"(x[i])); x[i]=y; }
  }
  float s=0;
  #pragma unroll
  for(int i=0;i<CH;i++) s+=x[i];
  if(s==1234.5f) out[0]=s;
}
__global__ void read_k(const int4* __restrict__ p, size_t n, int reps, int* out){
  int acc=0;
  for(int r=0;r<reps;r++)
    for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n;i+=(size_t)gridDim.x*blockDim.x){
      int4 v=__ldcg(p+i); acc^=v.x^v.y^v.z^v.w;
    }
  if(acc==0x7fffffff) out[0]=acc;
}
int main(){
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr,0));
  int sms=pr.multiProcessorCount;
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double *dd; float* fd; int* id; CK(cudaMalloc(&dd,64)); CK(cudaMalloc(&fd,64)); CK(cudaMalloc(&id,64));
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu, \"clock_khz\": %d",sms,pr.l2CacheSize,pr.sharedMemPerMultiprocessor,pr.clockRate);
  // DFMA
  { int it=4096; dim3 g(sms*8), b(256);
    dfma_k<8><<<g,b>>>(dd,16,1.0000001,1e-9); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dfma_k<8><<<g,b>>>(dd,it,1.0000001,1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); double fl=2.0*8*it*(double)g.x*b.x; printf(", \"fp64_fma_tflops\": %.3f",fl/ms/1e9); }
  { int it=8192; dim3 g(sms*8), b(256);
    ffma_k<16><<<g,b>>>(fd,16,1.0000001f,1e-9f); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); ffma_k<16><<<g,b>>>(fd,it,1.0000001f,1e-9f); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); double fl=2.0*16*it*(double)g.x*b.x; printf(", \"fp32_fma_tflops\": %.3f",fl/ms/1e9); }
  { int it=4096; dim3 g(sms*8), b(256);
    tanh_k<8><<<g,b>>>(fd,16); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); tanh_k<8><<<g,b>>>(fd,it); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); double n=8.0*it*(double)g.x*b.x; printf(", \"tanh_approx_gops\": %.1f",n/ms/1e6); }
  for(size_t mb: {32ul, 64ul, 96ul}){
    size_t bytes=mb<<20; int4* p; CK(cudaMalloc(&p,bytes)); CK(cudaMemset(p,1,bytes));
    size_t n=bytes/16; int reps=20;
    read_k<<<sms*4,512>>>(p,n,2,id); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); read_k<<<sms*4,512>>>(p,n,reps,id); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf(", \"l2_read_gbs_%zuMB\": %.1f",mb,(double)bytes*reps/ms/1e6);
    cudaFree(p);
  }
  { size_t bytes=4ul<<30; int4* p; CK(cudaMalloc(&p,bytes)); CK(cudaMemset(p,1,bytes));
    size_t n=bytes/16;
    read_k<<<sms*4,512>>>(p,n,1,id); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); read_k<<<sms*4,512>>>(p,n,3,id); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf(", \"hbm_read_gbs\": %.1f",(double)bytes*3/ms/1e6); cudaFree(p); }
  printf("}\n");
  return 0;
}
