// shared atomics: random banks vs lane-private banks (32 copies) vs 16 copies
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template<int MODE>
__global__ void __launch_bounds__(512) kern(unsigned* out, int iters){
  extern __shared__ uint32_t sm[];
  const int words = 2*768*32;  // 768 bins x 32 copies x 2 channels = 196 KB
  for(int i=threadIdx.x;i<words;i+=blockDim.x) sm[i]=0; __syncthreads();
  uint32_t r = (blockIdx.x*1024+threadIdx.x)*2654435761u + 12345u;
  const uint32_t lane = threadIdx.x & 31;
  #pragma unroll 4
  for(int it=0; it<iters; ++it){
    r = r*1664525u + 1013904223u;
    uint32_t bin = (r>>22) % 768;
    uint32_t a;
    if (MODE==0) a = bin;                 // one copy, random bank
    else if (MODE==1) a = bin*32 + lane;  // 32 copies: lane-private bank
    else a = bin*16 + (lane&15);          // 16 copies
    atomicAdd(&sm[a], r);
    atomicAdd(&sm[a + 768*32], r>>3);
  }
  __syncthreads();
  unsigned s=0; for(int i=threadIdx.x;i<words;i+=blockDim.x) s+=sm[i];
  atomicAdd(out, s);
}
template<int M> void run(const char* nm){
  unsigned* out; cudaMalloc(&out, 8); int smem=2*768*32*4;
  cudaFuncSetAttribute(kern<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int occ=0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern<M>, 512, smem);
  int grid=148*occ, iters=16384;
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  kern<M><<<grid,512,smem>>>(out,iters); cudaDeviceSynchronize();
  cudaEventRecord(a); kern<M><<<grid,512,smem>>>(out,iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b);
  double lanes=(double)grid*512*iters*2;
  printf("%-28s occ=%d %.3f ms  ATOMS lanes/clk/SM @1.965GHz = %.2f  (g,h) updates/clk/SM = %.2f\n",nm,occ,ms,lanes/(ms*1e-3)/148/1.965e9, lanes/2/(ms*1e-3)/148/1.965e9);
}
int main(){ run<0>("random bank (1 copy)"); run<1>("lane-private (32 copies)"); run<2>("16 copies"); return 0; }
