// tree_common.cuh -- definitions shared by the tree-construction translation units
// (tree.cu: Algorithm 1 driver, evaluation, loss-guided steps; records.cu: the depth-wise
// level pass over physically partitioned row records).
#pragma once

#include "gbm_internal.cuh"

namespace gbm {

struct NodeDev {
    long long Tg, Th;        // node totals over all ranks (fixed point)
    long long start, count;  // this rank's segment in the level's ridx buffer
    int state;               // GBM_NODE_ABSENT / SPLIT / LEAF
    int f, b, dl;            // split (state == SPLIT)
    int build_left;          // which child's histogram is built at the next level
    int pad;
};

constexpr int PT = 2048;         // partition tile (rows): 16 warps x 128 rows
constexpr int WROWS = PT / 16;   // rows per warp per tile
constexpr int P_THREADS = 256;   // partition kernels: 8 warps x 4 ballot words
constexpr int H_THREADS = 512;   // histogram / fused kernels
#ifndef GBM_PH_UNR
#define GBM_PH_UNR 4
#endif
#ifndef GBM_PH_TPS  // tiles per step of the fused level kernel's byte path (1 or 2)
#define GBM_PH_TPS 2
#endif
#ifndef GBM_PH_MINB
#define GBM_PH_MINB 3
#endif
#ifndef GBM_HR_MINB  // root histogram kernel: 2 resident blocks (Bosch root 1.65 vs 1.86 ms at 3)
#define GBM_HR_MINB 2
#endif
constexpr int PH_UNR = GBM_PH_UNR;    // rows in flight per lane in the fused level kernel's byte path
// resident blocks the fused level kernel is compiled for: the byte path runs best with the
// register room of 2 blocks (Higgs 1.86 vs 1.97 ms/round, Epsilon 5.09 vs 5.18), the generic path
// with the occupancy of 3 (Bosch 4.73 vs 5.04)
constexpr int PH_MINB = GBM_PH_MINB;
constexpr int PH_MINB_BYTE = 2;
constexpr int RUN_MAX = 16;      // tiles per fused work item: chosen per tree (flush amortisation
                                 // vs. enough items for every resident block)
constexpr int MAX_CHUNK = 65535; // rows per flush (exactness bound above)

// ============================================================== bank-column histograms (shared)
struct ColGroup {
    int f_lo, f_hi;  // features [f_lo, f_hi), Fg <= 32
};

constexpr int COLB_STRIDE = 256 * 32;

template <bool WIDE>
__device__ __forceinline__ void col_add_b(int *hs, int word, int2 q) {
    if (WIDE) {
        atomicAdd(hs + word, q.x & 0x7fff);
        atomicAdd(hs + COLB_STRIDE + word, q.y & 0x7fff);
        atomicAdd(hs + 2 * COLB_STRIDE + word, q.x >> 15);
        atomicAdd(hs + 3 * COLB_STRIDE + word, q.y >> 15);
    } else {
        atomicAdd(hs + word, q.x);
        atomicAdd(hs + COLB_STRIDE + word, q.y);
    }
}

template <bool WIDE>
__device__ void col_flush(const int *hs, int cstride, const ColGroup &cg, const int32_t *__restrict__ cut_ptr,
                          unsigned long long *dst /* slot base */) {
    const int Fg = cg.f_hi - cg.f_lo, R = 32 / Fg;
    // a thread's words all sit in one bank column (blockDim is a multiple of 32): its feature and
    // bin range are fixed, and its bins only grow -- look them up once, stop at the last bin
    const int col = threadIdx.x & 31;
    if (col >= R * Fg) return;
    const int f = cg.f_lo + col % Fg;
    const int c0 = __ldg(cut_ptr + f), nb = __ldg(cut_ptr + f + 1) - c0;
    for (int w = threadIdx.x; w < cstride; w += blockDim.x) {
        const int b = w >> 5;
        if (b >= nb) break;
        long long G, H;
        if (WIDE) {
            G = (long long)hs[2 * cstride + w] * 32768 + (long long)(unsigned)hs[w];
            H = (long long)hs[3 * cstride + w] * 32768 + (long long)(unsigned)hs[cstride + w];
        } else {
            G = hs[w];
            H = hs[cstride + w];
        }
        if (G) atomicAdd(dst + 2ll * (c0 + b), (unsigned long long)G);
        if (H) atomicAdd(dst + 2ll * (c0 + b) + 1, (unsigned long long)H);
    }
}

// ---- TMA bulk copies (cp.async.bulk, global -> shared, completion on an mbarrier)
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }


__device__ __forceinline__ int find_parent(const int *__restrict__ tile_base, int n_par, int t) {
    int lo = 0, hi = n_par - 1;  // largest j with tile_base[j] <= t
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(tile_base + mid) <= t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// Dynamic work distribution: the block claims the next item from counter[0]; n_items[0] items.
__device__ __forceinline__ int claim_item(int *counter) {
    __shared__ int s_item;
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(counter, 1);
    __syncthreads();
    return s_item;
}


// ---- records.cu: the depth-wise level pass over physically partitioned row records
struct RecLaunch {
    NodeDev *nodes;
    int first, n_par;                 // the level's parents (heap ids)
    const int *tile_base;             // device plan of the split parents' 2048-row items
    int items_hint;                   // upper bound on the items (grid size)
    const uint32_t *in_rows;          // [pos][RW] row words (level 1: the canonical packed matrix)
    const int2 *in_q;                 // [pos] gradient pairs (level 1: qpair)
    unsigned long long in_rows_bytes, in_q_bytes;  // readable extents of the two inputs
    uint32_t *out_rows;               // null on the last histogram level
    int2 *out_q;
    unsigned long long *cursor;       // [node][2]
    const int32_t *cut_ptr;
    int F, B, RW;                     // RW: words per packed row (record rows: rec_row_words(RW))
    int RW_in;                        // words per input row: RW at level 1, rec_row_words(RW) after
    bool wide;
    unsigned long long *hist;         // [n_par][TB][2] built-child histograms
    long long TB;
    unsigned long long *rows_ctr;
    int bits_parent_row, bits_built_row;
};
size_t rec_smem_bytes(bool wide);
int rec_row_words(int rw);  // record row width: RW rounded up to 1, 2, 4 or 8 words
int rec_level_launch(gbm_ctx *ctx, const RecLaunch &L, cudaStream_t s);
int rec_seg_launch(gbm_ctx *ctx, NodeDev *nodes, int first, int n_par, unsigned long long *cursor, cudaStream_t s);
int rec_root_launch(gbm_ctx *ctx, unsigned long long *cursor, long long n, cudaStream_t s);

// ---- root_ct.cu: the root histogram fed by TMA tensor tiles of the feature-major symbols
struct RootCtLaunch {
    const uint8_t *colsym;            // [F][n] (null: not available)
    const int2 *qpair;
    long long n;
    int F, bits;
    bool wide;
    const int32_t *cut_ptr;
    unsigned long long *hist, *totals, *rows_ctr;
};
int root_ct_launch(gbm_ctx *ctx, const RootCtLaunch &L, cudaStream_t s);  // 1 launched, 0 n/a, < 0 error

}  // namespace gbm
