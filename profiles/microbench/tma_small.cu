// Throughput of many small cp.async.bulk copies (one 32-byte row per lane, random rows) into
// shared memory: could TMA do the row gathers of the level histogram pass?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int BYTES>
__global__ void __launch_bounds__(512) k(const char *__restrict__ src, long long nrows, int iters, unsigned seed,
                                         unsigned long long *sink) {
    __shared__ __align__(128) char buf[16][2][32 * BYTES > 1024 ? 1024 : 32 * BYTES];
    __shared__ uint64_t bar[16][2];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[w][0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[w][1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    unsigned x = seed ^ (blockIdx.x * 7919u + threadIdx.x * 104729u);
    unsigned ph[2] = {0, 0};
    unsigned long long acc = 0;
    for (int i = 0; i < iters; ++i) {
        const int b = i & 1;
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[w][b])), "r"(32 * BYTES) : "memory");
        __syncwarp();
        x = x * 1664525u + 1013904223u;
        const long long r = (long long)(x % (unsigned)nrows);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(&buf[w][b][lane * BYTES])),
                     "l"(src + r * BYTES), "r"(BYTES), "r"(su(&bar[w][b])) : "memory");
        if (i > 0) {
            const int pb = b ^ 1;
            asm volatile("{\n\t.reg .pred p;\nW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n}" ::"r"(su(&bar[w][pb])), "r"(ph[pb] & 1u) : "memory");
            ph[pb]++;
            acc += buf[w][pb][lane * BYTES];
        }
    }
    const int pb = (iters - 1) & 1;
    asm volatile("{\n\t.reg .pred p;\nW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n}" ::"r"(su(&bar[w][pb])), "r"(ph[pb] & 1u) : "memory");
    if (acc == 12345) sink[0] = acc;
}
int main() {
    const long long nrows = 11000000;
    char *src; unsigned long long *sink;
    cudaMalloc(&src, nrows * 48); cudaMalloc(&sink, 8); cudaMemset(src, 1, nrows * 48);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int bytes : {16, 32}) {
        for (int grid : {148, 296}) {
            const int iters = 400;
            auto run = [&]() {
                if (bytes == 16) k<16><<<grid, 512>>>(src, nrows, iters, 1u, sink);
                else if (bytes == 32) k<32><<<grid, 512>>>(src, nrows, iters, 1u, sink);
                
            };
            run();
            cudaEventRecord(a); run(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double ops = (double)grid * 512 * iters;
            printf("bytes=%d grid=%d: %.3f ms, %.2f G copies/s, %.2f copies/clk/SM @1.965GHz, %.0f GB/s useful  err=%s\n", bytes, grid, ms,
                   ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.965e9, ops * bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
