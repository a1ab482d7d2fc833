// Do DMMA (tensor FP64) and DFMA (FP64 ALU) run concurrently on B200?  Mixed-instruction throughput.
#include <cstdio>
#include <cuda_runtime.h>
template<int NM, int NF>
__global__ void __launch_bounds__(256) mix_kernel(double* out, int iters){
  double acc[4][2]; double f[8];
  double x = threadIdx.x*1e-3, y = 1.0 - threadIdx.x*1e-4;
  #pragma unroll
  for(int i=0;i<4;i++){acc[i][0]=0;acc[i][1]=0;}
  #pragma unroll
  for(int i=0;i<8;i++) f[i]=i*0.1;
  for(int it=0; it<iters; it++){
    #pragma unroll
    for(int i=0;i<NM;i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]),"+d"(acc[i][1]) : "d"(x),"d"(y));
    #pragma unroll
    for(int j=0;j<NF;j++){
      #pragma unroll
      for(int i=0;i<8;i++) f[i]=fma(f[i],1.0000001,1e-9);
    }
  }
  double s=0;
  #pragma unroll
  for(int i=0;i<4;i++) s+=acc[i][0]+acc[i][1];
  #pragma unroll
  for(int i=0;i<8;i++) s+=f[i];
  if(s==12345.0) out[0]=s;
}
template<int NM,int NF> void run(double* out, int sms){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters=20000; dim3 g(sms*8), b(256);
  mix_kernel<NM,NF><<<g,b>>>(out,100); cudaDeviceSynchronize();
  float best=1e30, ms;
  for(int r=0;r<5;r++){cudaEventRecord(e0); mix_kernel<NM,NF><<<g,b>>>(out,iters); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1); if(ms<best)best=ms;}
  double warps = (double)g.x*b.x/32;
  double fm = 2.0*256*NM*(double)iters*warps, ff = 2.0*8*NF*32.0*iters*warps;
  printf("NM=%d NF=%d: %.2f ms  dmma %.2f TF  dfma %.2f TF  total %.2f TF\n", NM, NF, best, fm/best/1e9, ff/best/1e9, (fm+ff)/best/1e9);
}
int main(){ double* out; cudaMalloc(&out,64); int sms=148;
  run<4,0>(out,sms); run<0,8>(out,sms); run<4,4>(out,sms); run<4,8>(out,sms); run<2,8>(out,sms); run<4,2>(out,sms); return 0; }
