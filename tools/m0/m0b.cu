// M0b: FP64 tensor-core (DMMA m8n8k4) throughput, co-issue with DFMA, smem fp64 atomics.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template<int DM, int DF>
__global__ void mix_kernel(double* out, int iters, double a, double b) {
  double acc[8][2]; for (int k=0;k<8;k++){acc[k][0]=threadIdx.x; acc[k][1]=k;}
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<iters;i++){
#pragma unroll
    for(int k=0;k<DM;k++) dmma(acc[k&7], a+k, b);
#pragma unroll
    for(int k=0;k<DF;k++){ x0=fma(x0,a,b); x1=fma(x1,a,b); x2=fma(x2,a,b); x3=fma(x3,a,b);
      x4=fma(x4,a,b); x5=fma(x5,a,b); x6=fma(x6,a,b); x7=fma(x7,a,b);}
  }
  double s=x0+x1+x2+x3+x4+x5+x6+x7; for(int k=0;k<8;k++) s+=acc[k][0]+acc[k][1];
  if (s==1.2345) out[0]=s;
}
__global__ void smem_atomic(double* out, int iters, int spread) {
  __shared__ double buf[4096];
  for (int i=threadIdx.x;i<4096;i+=blockDim.x) buf[i]=0;
  __syncthreads();
  int base = (threadIdx.x*spread) & 4095;
  for (int i=0;i<iters;i++){ atomicAdd(&buf[(base + i*7) & 4095], 1.0); }
  __syncthreads();
  if (threadIdx.x==0) out[blockIdx.x]=buf[0];
}
__global__ void smem_rmw(double* out, int iters) {
  __shared__ double buf[4096];
  for (int i=threadIdx.x;i<4096;i+=blockDim.x) buf[i]=0;
  __syncthreads();
  int base = threadIdx.x;
  for (int i=0;i<iters;i++){ double* p=&buf[(base + i*256) & 4095]; *p += 1.0; }
  __syncthreads();
  if (threadIdx.x==0) out[blockIdx.x]=buf[0];
}
template<int DM,int DF> int run(const char* name, int sms, double* out){
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int iters=2048, blocks=sms*4, threads=256;
  mix_kernel<DM,DF><<<blocks,threads>>>(out,16,1.0,1e-9);
  cudaEventRecord(e0); mix_kernel<DM,DF><<<blocks,threads>>>(out,iters,0.999999,1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms,e0,e1);
  double warps=(double)blocks*threads/32;
  double mma_fl=2.0*256*DM*iters*warps, fma_fl=2.0*8*DF*iters*(double)blocks*threads;
  printf("%s: %.3f ms  DMMA %.2f TF  DFMA %.2f TF  total %.2f TF\n", name, ms, mma_fl/ms/1e9, fma_fl/ms/1e9, (mma_fl+fma_fl)/ms/1e9);
  return 0;
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0)); int sms=p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out,sms*64*8));
  for(int r=0;r<2;r++){
    run<8,0>("dmma only     ", sms, out);
    run<0,8>("dfma only     ", sms, out);
    run<8,8>("dmma8+dfma8   ", sms, out);
    run<4,8>("dmma4+dfma8   ", sms, out);
    run<8,4>("dmma8+dfma4   ", sms, out);
  }
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int spread: {1, 33}) {
    int iters=4096, blocks=sms*4, threads=256;
    cudaEventRecord(e0); smem_atomic<<<blocks,threads>>>(out,iters,spread); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    printf("smem fp64 atomicAdd spread %d: %.1f Gop/s\n", spread, (double)iters*blocks*threads/ms/1e6);
  }
  {
    int iters=4096, blocks=sms*4, threads=256;
    cudaEventRecord(e0); smem_rmw<<<blocks,threads>>>(out,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    printf("smem fp64 plain RMW: %.1f Gop/s\n", (double)iters*blocks*threads/ms/1e6);
  }
  return 0;
}
