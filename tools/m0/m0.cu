// M0 microbenchmarks: FP64 FMA peak, fp64 RED throughput, HBM write/copy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0=threadIdx.x, x1=x0+1, x2=x0+2, x3=x0+3, x4=x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i=0;i<iters;i++){
#pragma unroll
    for(int k=0;k<8;k++){ x0=fma(x0,a,b); x1=fma(x1,a,b); x2=fma(x2,a,b); x3=fma(x3,a,b);
      x4=fma(x4,a,b); x5=fma(x5,a,b); x6=fma(x6,a,b); x7=fma(x7,a,b);}
  }
  double s=x0+x1+x2+x3+x4+x5+x6+x7; if (s==1.2345) out[0]=s;
}
__device__ __forceinline__ uint64_t hash64(uint64_t x){ x^=x>>33; x*=0xff51afd7ed558ccdULL; x^=x>>33; x*=0xc4ceb9fe1a85ec53ULL; x^=x>>33; return x;}
__global__ void red_random(double* v, uint64_t n, uint64_t nops, int seed){
  uint64_t tid=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x, stride=(uint64_t)gridDim.x*blockDim.x;
  for(uint64_t i=tid;i<nops;i+=stride){ uint64_t j=hash64(i*2654435761ULL+seed)%n; atomicAdd(v+j,1.0);}
}
// each warp hits a run of 32 consecutive doubles at a random base (like a CSR row segment)
__global__ void red_segment(double* v, uint64_t n, uint64_t nops, int seg){
  uint64_t tid=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x, stride=(uint64_t)gridDim.x*blockDim.x;
  for(uint64_t i=tid;i<nops;i+=stride){ uint64_t grp=i/seg; uint64_t base=hash64(grp)%(n-seg); atomicAdd(v+base+(i%seg),1.0);}
}
__global__ void red_stream(double* v, uint64_t n, uint64_t nops){
  uint64_t tid=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x, stride=(uint64_t)gridDim.x*blockDim.x;
  for(uint64_t i=tid;i<nops;i+=stride){ atomicAdd(v+(i%n),1.0);}
}
__global__ void rmw_stream(double* v, uint64_t n){
  uint64_t tid=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x, stride=(uint64_t)gridDim.x*blockDim.x;
  for(uint64_t i=tid;i<n;i+=stride){ v[i]+=1.0;}
}
__global__ void write_stream(double* v, uint64_t n){
  uint64_t tid=blockIdx.x*(uint64_t)blockDim.x+threadIdx.x, stride=(uint64_t)gridDim.x*blockDim.x;
  for(uint64_t i=tid;i<n;i+=stride){ v[i]=1.0;}
}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("gpu %s sms %d cc %d.%d l2 %d MB\n", p.name, p.multiProcessorCount, p.major,p.minor, p.l2CacheSize>>20);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double* out; CK(cudaMalloc(&out,8));
  int sms=p.multiProcessorCount;
  for(int rep=0;rep<2;rep++){
    int iters=4096; int blocks=sms*8, threads=256;
    cudaEventRecord(e0); dfma_kernel<<<blocks,threads>>>(out,iters,0.999999,1e-7); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    double flops=2.0*64*iters*(double)blocks*threads;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops/ms/1e9, ms);
  }
  uint64_t n=(uint64_t)4<<27; // 512M doubles = 4 GB
  double* v; CK(cudaMalloc(&v,n*8)); CK(cudaMemset(v,0,n*8));
  for(int rep=0;rep<2;rep++){
    cudaEventRecord(e0); CK(cudaMemsetAsync(v,0,n*8)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("memset 4GB: %.1f GB/s\n", n*8/ms/1e6);
    cudaEventRecord(e0); write_stream<<<sms*16,256>>>(v,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("write kernel 4GB: %.1f GB/s\n", n*8/ms/1e6);
    cudaEventRecord(e0); rmw_stream<<<sms*16,256>>>(v,n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("rmw kernel 4GB: %.1f GB/s (r+w)\n", 2*n*8/ms/1e6);
    uint64_t nops=n; 
    cudaEventRecord(e0); red_stream<<<sms*16,256>>>(v,n,nops); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("RED coalesced-stream 4GB: %.2f Gop/s, %.1f GB/s eff(r+w)\n", nops/ms/1e6, 2*n*8/ms/1e6);
    nops=n/4;
    cudaEventRecord(e0); red_random<<<sms*16,256>>>(v,n,nops,rep); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("RED random over 4GB: %.2f Gop/s\n", nops/ms/1e6);
    uint64_t nsmall=(uint64_t)1<<23; // 64 MB L2 resident
    cudaEventRecord(e0); red_random<<<sms*16,256>>>(v,nsmall,nops,rep); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
    printf("RED random over 64MB (L2): %.2f Gop/s\n", nops/ms/1e6);
    for(int seg: {3,8,9,27}){
      cudaEventRecord(e0); red_segment<<<sms*16,256>>>(v,n,nops,seg); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms,e0,e1);
      printf("RED segments of %d over 4GB: %.2f Gop/s\n", seg, nops/ms/1e6);
    }
  }
  return 0;
}
