// FP64 peak microbenchmarks on B200 (sm_100a): DFMA pipe, DMMA (mma.sync m8n8k4 f64)
// and a plain HBM copy.  Written to fix the roofline denominators for the FP64
// kernels, which MEASURED_PEAKS.json does not cover.  Timed with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int ILP>
__global__ void __launch_bounds__(256) dfma_kernel(double* out, double a, double b, int iters){
  double acc[ILP];
  #pragma unroll
  for(int i=0;i<ILP;i++) acc[i]=threadIdx.x*1e-3+i;
  for(int it=0; it<iters; it++){
    #pragma unroll
    for(int i=0;i<ILP;i++) acc[i]=fma(acc[i],a,b);
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<ILP;i++) s+=acc[i];
  if(s==12345.0) out[0]=s;
}

template<int ILP>
__global__ void __launch_bounds__(256) dmma_kernel(double* out, int iters){
  double acc[ILP][2];
  double x = threadIdx.x*1e-3, y = 1.0 - threadIdx.x*1e-4;
  #pragma unroll
  for(int i=0;i<ILP;i++){acc[i][0]=0;acc[i][1]=0;}
  for(int it=0; it<iters; it++){
    #pragma unroll
    for(int i=0;i<ILP;i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]),"+d"(acc[i][1]) : "d"(x),"d"(y));
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<ILP;i++) s+=acc[i][0]+acc[i][1];
  if(s==12345.0) out[0]=s;
}

__global__ void copy_kernel(const double4* __restrict__ a, double4* __restrict__ b, size_t n){
  size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x*blockDim.x;
  for(; i<n; i+=st) b[i]=a[i];
}

int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%zu", p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin);
  double* out; CK(cudaMalloc(&out,64));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms=p.multiProcessorCount; float ms;
  // DFMA
  { int iters=20000; dim3 g(sms*8), b(256);
    dfma_kernel<8><<<g,b>>>(out,1.0000001,1e-9,100); CK(cudaDeviceSynchronize());
    float best=1e30; for(int r=0;r<5;r++){cudaEventRecord(e0); dfma_kernel<8><<<g,b>>>(out,1.0000001,1e-9,iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    double flops=2.0*8*iters*(double)g.x*b.x; printf(",\"dfma_tflops\":%.2f",flops/best/1e9); }
  // DMMA m8n8k4
  { int iters=20000; dim3 g(sms*8), b(256);
    dmma_kernel<4><<<g,b>>>(out,100); CK(cudaDeviceSynchronize());
    float best=1e30; for(int r=0;r<5;r++){cudaEventRecord(e0); dmma_kernel<4><<<g,b>>>(out,iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    double flops=2.0*256*4*(double)iters*(g.x*b.x/32); printf(",\"dmma_m8n8k4_tflops\":%.2f",flops/best/1e9); }
  // HBM copy 4 GiB total (2 GiB read + 2 GiB write)
  { size_t bytes=(size_t)2<<30; double4 *a,*bb; CK(cudaMalloc(&a,bytes)); CK(cudaMalloc(&bb,bytes)); cudaMemset(a,0,bytes);
    size_t n=bytes/sizeof(double4); copy_kernel<<<sms*16,256>>>(a,bb,n); CK(cudaDeviceSynchronize());
    float best=1e30; for(int r=0;r<10;r++){cudaEventRecord(e0); copy_kernel<<<sms*16,256>>>(a,bb,n); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
    printf(",\"copy_gbs\":%.1f", 2.0*bytes/best/1e6); cudaFree(a); cudaFree(bb);}
  printf("}\n");
  return 0;
}
