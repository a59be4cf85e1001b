// Lean shared-atomic throughput probe: precomputed per-thread LCG, 32 features x 256 bins
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int NF=32, NB = NF*256;
template<int NAT, int BINMASK>
__global__ void __launch_bounds__(512) kern(unsigned* out, int iters){
  extern __shared__ uint32_t sm[];
  for(int i=threadIdx.x;i<NAT*NB;i+=blockDim.x) sm[i]=0; __syncthreads();
  uint32_t r = (blockIdx.x*1024+threadIdx.x)*2654435761u + 12345u;
  uint32_t foff = (threadIdx.x & 31)*256;
  #pragma unroll 4
  for(int it=0; it<iters; ++it){
    r = r*1664525u + 1013904223u;
    uint32_t bin = foff + ((r>>24) & BINMASK);
    foff = (foff + 256) & (NB-1);
    #pragma unroll
    for(int a=0;a<NAT;++a) atomicAdd(&sm[a*NB+bin], r);
  }
  __syncthreads();
  unsigned s=0; for(int i=threadIdx.x;i<NAT*NB;i+=blockDim.x) s+=sm[i];
  atomicAdd(out, s);
}
template<int NAT,int BM> void run(){
  unsigned* out; cudaMalloc(&out, 8); int smem=NAT*NB*4;
  cudaFuncSetAttribute(kern<NAT,BM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int occ=0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern<NAT,BM>, 512, smem);
  int grid=148*occ, iters=8192;
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  kern<NAT,BM><<<grid,512,smem>>>(out,iters); cudaDeviceSynchronize();
  cudaEventRecord(a); kern<NAT,BM><<<grid,512,smem>>>(out,iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b);
  double lanes=(double)grid*512*iters*NAT;
  printf("NAT=%d binmask=%3d occ=%d %.3f ms  ATOMS lanes/clk/SM @1.965GHz = %.2f  updates(=lanes/NAT)/clk/SM=%.2f\n",NAT,BM,occ,ms,lanes/(ms*1e-3)/148/1.965e9, lanes/NAT/(ms*1e-3)/148/1.965e9);
}
int main(){ run<1,255>(); run<2,255>(); run<4,255>(); run<1,31>(); run<2,31>(); run<1,3>(); run<2,3>(); run<1,0>(); return 0; }
