// Microbenchmark: shared-memory histogram update throughput on B200 (random bins, 28 features x 256 bins)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }
constexpr int NB = 28*256;
template<int MODE>
__global__ void __launch_bounds__(512) kern(unsigned long long* out, int iters, int nbins_feat){
  extern __shared__ uint32_t sm[];
  uint32_t* h32 = sm; unsigned long long* h64 = (unsigned long long*)sm;
  int words = (MODE==0)? 2*NB : (MODE==1? NB : (MODE==2? 2*NB: 4*NB));
  for(int i=threadIdx.x;i<words;i+=blockDim.x) sm[i]=0; __syncthreads();
  uint32_t seed = hsh(blockIdx.x*1024+threadIdx.x);
  for(int it=0; it<iters; ++it){
    uint32_t r = hsh(seed + it*0x9e3779b9u);
    int f = (threadIdx.x + it) % 28;               // lanes spread over features (row-per-lane style)
    int bin = f*256 + (r % nbins_feat);
    int g = (int)(r>>8) & 0x7fff;
    if(MODE==0){ atomicAdd(&h32[bin], (uint32_t)g); atomicAdd(&h32[NB+bin], (uint32_t)(r&0xff)); }
    else if(MODE==1){ atomicAdd(&h32[bin], (uint32_t)g); }
    else if(MODE==2){ atomicAdd(&h64[bin], (unsigned long long)g); }
    else { atomicAdd(&h64[bin], (unsigned long long)g); atomicAdd(&h64[NB+bin], (unsigned long long)r); }
  }
  __syncthreads();
  unsigned long long s=0; for(int i=threadIdx.x;i<words;i+=blockDim.x) s+=sm[i];
  atomicAdd(out, s);
}
template<int MODE> void run(int smem, const char* name, int nbf){
  unsigned long long* out; cudaMalloc(&out, 8);
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int occ=0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern<MODE>, 512, smem);
  int grid = 148*occ; int iters = 4096;
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  kern<MODE><<<grid,512,smem>>>(out, iters, nbf); cudaDeviceSynchronize();
  cudaEventRecord(a); kern<MODE><<<grid,512,smem>>>(out, iters, nbf); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b);
  double upd = (double)grid*512*iters; int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-28s bins/feat=%3d occ=%d  %.3f ms  %.1f Gupd/s  %.2f upd/clk/SM(@%.0fMHz)  err=%s\n", name, nbf, occ, ms, upd/ms/1e6, upd/(ms*1e-3)/148/(clk*1e3), clk/1e3, cudaGetErrorString(cudaGetLastError()));
}
int main(){
  for(int nbf : {256, 32, 4}){
  run<0>(2*NB*4, "2x ATOMS.ADD.32 (g,h)", nbf);
  run<1>(NB*4, "1x ATOMS.ADD.32 (packed)", nbf);
  run<2>(NB*8, "1x atomicAdd u64 (CAS)", nbf);
  run<3>(2*NB*8, "2x atomicAdd u64 (CAS)", nbf);
  }
  return 0;
}
