// Same-address global atomicAdd (with return) throughput under contention: the reservation
// pattern of the record level pass (one atomic per warp-chunk on a parent's cursor).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(unsigned long long *ctr, int n_addr, int iters, unsigned long long *sink) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    unsigned long long acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (lane == 0) acc += atomicAdd(ctr + ((gw + i) % n_addr) * 16, 37ull);
        __syncwarp();
    }
    if (lane == 0 && acc == 1) sink[0] = acc;
}
int main() {
    unsigned long long *ctr, *sink;
    cudaMalloc(&ctr, 1 << 20); cudaMalloc(&sink, 8);
    cudaMemset(ctr, 0, 1 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int n_addr : {1, 2, 16, 64}) {
        for (int blocks : {296, 592}) {
            const int iters = 64;
            k<<<blocks, 512>>>(ctr, n_addr, iters, sink);
            cudaEventRecord(a);
            k<<<blocks, 512>>>(ctr, n_addr, iters, sink);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)blocks * 16 * iters;
            printf("addresses=%3d warps=%6d atomics=%9.0f  %.3f ms  %.2f Gatomics/s (%.1f ns per atomic per address)\n",
                   n_addr, blocks * 16, ops, ms, ops / ms / 1e6, ms * 1e6 / (ops / n_addr));
        }
    }
    return 0;
}
