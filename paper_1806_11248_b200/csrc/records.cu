// records.cu -- the depth-wise level pass of Algorithm 1 over physically partitioned row records:
// RepartitionInstances + BuildPartialHistograms of the smaller child, fused (SURVEY §8a
// a5 + a6), for narrow byte-symbol matrices (8-bit symbols, <= 32 features, word-aligned rows:
// the Higgs- and Airline-shaped workloads).
//
// Why records.  The index-based level pass (tree.cu part_hist_kernel) gathers, per level, the
// split symbol of every parent row (1 byte out of a 32-byte sector) and the packed row + qpair of
// every row of the built child (28 + 8 bytes out of 2-3 sectors) through a row-index list; at the
// deeper levels the rows of a node are spread over the whole matrix, and ncu measured 2.3-6x the
// algorithmic DRAM bytes (profiles/r01_ncu_hist_summary.md).  Here every level streams its
// parents' rows instead: each rank keeps a copy of its rows -- the packed row words and the
// row's fixed-point gradient pair, a "record" -- grouped by node, and the level pass moves every
// parent row into its child's segment while it accumulates the smaller child's rows.  Level 1
// reads the canonical packed matrix and qpair (identity order); level l >= 2 reads the records
// level l - 1 wrote.  Reads are TMA bulk copies (cp.async.bulk) of 32-row batches into per-warp
// shared-memory buffers, writes are coalesced stores, and the histogram is the conflict-free
// bank-column layout of the staged root (lane f owns bank f: word = bin * 32 + lane).
//
// Work item = one 2048-row tile of one split parent's segment; each block takes a contiguous
// range of items (the shared histogram is flushed only when the parent changes).  Per item:
//   phase A  every warp stages its 32-row batches, decides left/right from the staged split
//            byte (R6/R7: sym <= b, the sentinel goes the learned default direction), keeps the
//            ballot, and adds the rows of the built child (R17) into the shared histogram;
//   reserve  one warp scans the 64 batches' left/right counts; the block reserves its rows in
//            the children's segments with one atomic per child on the parent's cursors: the
//            left child fills the parent's segment from the front, the right child from the back,
//            so the two meet exactly at start + n_left with no counting pass;
//   phase B  every warp re-stages its batches (from L2) and stores them at their positions.
// The order of rows inside a child segment depends on which block reserved first; nothing
// observable does (histograms are exact int64 sums, the row -> leaf map is written by the final
// row-order walk), so results are identical for every order (R28).
#include "tree_common.cuh"

namespace gbm {

constexpr int REC_THREADS = 512;
constexpr int REC_NW = REC_THREADS / 32;
constexpr int REC_ROWS = 1024;    // rows per work item: two 32-row batches per warp
constexpr int REC_BPI = REC_ROWS / 32;  // 32-row batches per item
constexpr int REC_WMAX = 8;       // words per row: <= 32 byte features
static_assert(REC_BPI == 2 * REC_NW && 2 * REC_ROWS == PT, "two batches per warp, two items per plan tile");

struct RecStage {                 // one staging buffer of a warp (TMA destination, 16-B aligned)
    uint32_t w[32 * REC_WMAX + 4];  // 32 rows (+ the 16-byte alignment head)
    int2 q[32 + 2];                 // their pairs (+ head)
};
static_assert(sizeof(RecStage) % 16 == 0, "staging buffers must stay 16-byte aligned");

struct RecArgs {
    const NodeDev *nodes;
    int first, n_par;                 // parents: heap ids first .. first + n_par - 1
    const int *tile_base;             // plan (split parents only): items of parent j
    const uint32_t *in_rows;          // [pos][RW] words
    const int2 *in_q;                 // [pos]
    unsigned long long in_rows_bytes, in_q_bytes;  // readable extents (TMA bounds)
    uint32_t *out_rows;               // null: last histogram level (no partition output)
    int2 *out_q;
    unsigned long long *cursor;       // [node][2]: left (grows), right (shrinks)
    const int32_t *cut_ptr;
    int F, B;
    unsigned long long *hist;         // [n_par][TB][2]
    long long TB;
    unsigned long long *rows_ctr;     // profiling: algorithmic bits
    int bits_parent_row, bits_built_row;
    int tma;                          // bulk copies allowed (16-byte aligned bases)
};

// conflict-free bank-column updates by 32-bit shared address (this lane's column base + bin*128)
__device__ __forceinline__ void red_s32(unsigned addr, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
template <bool WIDE>
__device__ __forceinline__ void col_red(unsigned addr, int2 q) {
    if (WIDE) {
        red_s32(addr, q.x & 0x7fff);
        red_s32(addr + 4 * COLB_STRIDE, q.y & 0x7fff);
        red_s32(addr + 8 * COLB_STRIDE, q.x >> 15);
        red_s32(addr + 12 * COLB_STRIDE, q.y >> 15);
    } else {
        red_s32(addr, q.x);
        red_s32(addr + 4 * COLB_STRIDE, q.y);
    }
}

// One work item: rows [s0, s0 + nv) of parent j's segment (nv <= REC_ROWS).  Uniform per block.
struct RecItem {
    int j;             // parent slot (-1: none)
    long long s0;
    int nv;
    int tma;           // every batch of the item may be fetched by TMA
    int head_r, head_q;  // bytes from the 16-byte aligned base to row s0 (same for every batch)
};

template <int RB>
__device__ __forceinline__ RecItem rec_item(const RecArgs &a, int it) {
    RecItem x;
    const int tile = it >> 1;
    x.j = find_parent(a.tile_base, a.n_par, tile);
    const NodeDev *nd = a.nodes + a.first + x.j;
    const long long st = nd->start, cnt = nd->count;
    x.s0 = st + (long long)(tile - a.tile_base[x.j]) * PT + (it & 1) * REC_ROWS;
    x.nv = (int)max(0ll, min((long long)REC_ROWS, st + cnt - x.s0));
    const unsigned long long r0 = (unsigned long long)x.s0 * RB, q0 = (unsigned long long)x.s0 * 8;
    x.head_r = (int)(r0 & 15);
    x.head_q = (int)(q0 & 15);
    const unsigned long long re = (r0 + (unsigned long long)x.nv * RB + 15) & ~15ull;
    const unsigned long long qe = (q0 + (unsigned long long)x.nv * 8 + 15) & ~15ull;
    x.tma = a.tma && re <= a.in_rows_bytes && qe <= a.in_q_bytes;
    return x;
}

// Stage batch b (32 rows) of item x into the warp's buffer: lane 0 issues two TMA bulk copies
// (rows, pairs) completing on bar, or every lane copies with plain loads when the item may not
// use TMA (the tail of an odd-length canonical qpair).
template <int RWI>
__device__ __forceinline__ void rec_stage(const RecArgs &a, const RecItem &x, int b, RecStage *st, uint64_t *bar) {
    constexpr int RB = RWI * 4;
    const int lane = threadIdx.x & 31;
    const int nrows = min(32, x.nv - 32 * b);
    if (x.tma) {
        if (lane == 0) {
            const char *rsrc = reinterpret_cast<const char *>(a.in_rows) + (x.s0 * RB - x.head_r) + b * (32 * RB);
            const char *qsrc = reinterpret_cast<const char *>(a.in_q) + (x.s0 * 8 - x.head_q) + b * 256;
            const unsigned rbytes = (unsigned)(x.head_r + nrows * RB + 15) & ~15u;
            const unsigned qbytes = (unsigned)(x.head_q + nrows * 8 + 15) & ~15u;
            fence_proxy_async();  // this buffer's earlier generic accesses precede the async writes
            mbar_arrive_expect_tx(bar, rbytes + qbytes);
            bulk_g2s(st->w, rsrc, rbytes, bar);
            bulk_g2s(st->q, qsrc, qbytes, bar);
        }
    } else {
        const long long pos = x.s0 + 32 * b;
        const uint32_t *src = a.in_rows + pos * RWI;
        for (int i = lane; i < nrows * RWI; i += 32) st->w[i] = __ldg(src + i);
        if (lane < nrows) st->q[lane] = __ldg(a.in_q + pos + lane);
        __syncwarp();
    }
}

// RWI: words per input row (level 1: the packed matrix's stride; later levels RWP), RWP: words per
// record row written (RWI rounded up to 1, 2, 4 or 8: whole 16-byte units for the copies).
//
// Per item of <= 1024 rows every warp holds two 32-row batches in its two staging buffers:
//   phase A  (each batch) decide every row's side from its split byte; permute the batch in place
//            into [rows of the built child | the others] (rows and pairs, stable); add the built
//            rows into the bank-column histogram;
//   reserve  one warp scans the 32 batches' counts; the block takes its rows of each child from
//            the parent's two cursors (left grows from the segment's front, right from its back);
//   phase B  (each batch) store the two contiguous runs at their positions, then fetch the next
//            item's batch into the freed buffer (the loads overlap the rest of this item).
template <bool WIDE, int RWI, int RWP, bool OUT>
__global__ void __launch_bounds__(REC_THREADS, WIDE ? 1 : 2) rec_level_kernel(RecArgs a) {
    extern __shared__ __align__(16) int smem[];
    constexpr int CH = WIDE ? 4 : 2;
    constexpr int RB = RWI * 4;  // staged row pitch in bytes
    int *hs = smem;  // [CH][COLB_STRIDE] bank-column histogram of the current parent's built child
    RecStage *stage = reinterpret_cast<RecStage *>(smem + CH * COLB_STRIDE);  // [REC_NW][2]
    __shared__ uint64_t s_bar[2 * REC_NW];
    __shared__ int s_nl[REC_BPI], s_nb[REC_BPI];  // per batch: left rows, built rows
    __shared__ int s_loff[REC_BPI], s_roff[REC_BPI];
    __shared__ long long s_baseL, s_baseR;
    __shared__ __align__(16) unsigned char s_order[REC_NW][2][32];  // per batch: built rows, then the rest
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t ltm = (1u << lane) - 1u;
    uint64_t *bar = s_bar + 2 * wid;
    RecStage *buf = stage + 2 * wid;
    if (lane == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    unsigned phbits = 0;  // parity of the next completion of each buffer's barrier
    const ColGroup cg{0, a.F};
    const int F = a.F, R = 32 / F;  // R copies of every feature column per warp (R rows per step)
    const int copy = lane / F, fcol = lane - copy * F;
    const bool lane_on = copy < R;
    const unsigned hb = smem_u32(hs) + 4u * lane;  // this lane's bank column
    const int n_items = 2 * a.tile_base[a.n_par];
    const int i0 = (int)((long long)blockIdx.x * n_items / gridDim.x);
    const int i1 = (int)((long long)(blockIdx.x + 1) * n_items / gridDim.x);
    for (int i = threadIdx.x; i < CH * COLB_STRIDE; i += REC_THREADS) hs[i] = 0;
    // the first item's two batches
    int it = i0;
    RecItem x = it < i1 ? rec_item<RB>(a, it) : RecItem{-1, 0, 0, 0, 0, 0};
    for (int m = 0; m < 2; ++m)
        if (it < i1 && 32 * (wid + REC_NW * m) < x.nv) rec_stage<RWI>(a, x, wid + REC_NW * m, buf + m, bar + m);
    __syncthreads();
    int cur_j = -1;
    for (; it < i1; ++it) {
        const RecItem nx = it + 1 < i1 ? rec_item<RB>(a, it + 1) : RecItem{-1, 0, 0, 0, 0, 0};
        if (x.nv > 0 && x.j != cur_j) {
            if (cur_j >= 0) {  // flush the previous parent's built child, restart from zero
                __syncthreads();
                col_flush<WIDE>(hs, COLB_STRIDE, cg, a.cut_ptr, a.hist + (long long)cur_j * a.TB * 2);
                __syncthreads();
                for (int i = threadIdx.x; i < CH * COLB_STRIDE; i += REC_THREADS) hs[i] = 0;
                __syncthreads();
            }
            cur_j = x.j;
        }
        const NodeDev nd = a.nodes[a.first + x.j];
        const int fs = nd.f, bs = nd.b;
        const bool dl = nd.dl != 0, build_left = nd.build_left != 0;
        const int k = a.first + x.j;
        unsigned built = 0;
        // ---------------- phase A
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            const int b = wid + REC_NW * m;
            const int nrows = min(32, x.nv - 32 * b);
            if (nrows > 0) {
            if (x.tma) {
                mbar_wait(bar + m, (phbits >> m) & 1u);
                phbits ^= 1u << m;
            }
            uint8_t *sb = reinterpret_cast<uint8_t *>(buf[m].w) + x.head_r;
            int2 *sq = reinterpret_cast<int2 *>(reinterpret_cast<char *>(buf[m].q) + x.head_q);
            bool left = false;
            if (lane < nrows) {
                const int sy = sb[lane * RB + fs];
                left = sy == a.B ? dl : sy <= bs;
            }
            const uint32_t vmask = nrows == 32 ? 0xffffffffu : ((1u << nrows) - 1u);
            const uint32_t lmask = __ballot_sync(0xffffffffu, left) & vmask;
            const uint32_t bmask = build_left ? lmask : (vmask & ~lmask), omask = vmask & ~bmask;
            const int nbr = __popc(bmask);
            built += nbr;
            if (lane == 0) {
                s_nl[b] = __popc(lmask);
                s_nb[b] = nbr;
            }
            // the batch's order: built rows first, then the others (each ascending); the histogram
            // walks the first nbr entries, phase B stores the two runs in this order
            unsigned char *ord = s_order[wid][m];
            if (lane < nrows) ord[((bmask >> lane) & 1u) ? __popc(bmask & ltm) : nbr + __popc(omask & ltm)] = (unsigned char)lane;
            __syncwarp();
            if (lane_on) {  // R rows per step: lane = copy * F + feature
                const uint8_t *sp = sb + fcol;
                if (R == 1) {
                    int c = 0;
                    for (; c + 4 <= nbr; c += 4) {  // four rows in flight per lane
                        const uint32_t o4 = *reinterpret_cast<const uint32_t *>(ord + c);
                        int sy[4];
                        int2 q[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int r = (o4 >> (8 * u)) & 255u;
                            sy[u] = sp[r * RB];
                            q[u] = sq[r];
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) col_red<WIDE>(hb + ((unsigned)sy[u] << 7), q[u]);
                    }
                    for (; c < nbr; ++c) {
                        const int r = ord[c];
                        col_red<WIDE>(hb + ((unsigned)sp[r * RB] << 7), sq[r]);
                    }
                } else {
                    for (int c = copy; c < nbr; c += R) {
                        const int r = ord[c];
                        col_red<WIDE>(hb + ((unsigned)sp[r * RB] << 7), sq[r]);
                    }
                }
            }
            __syncwarp();
            }
            if (!OUT && nx.j >= 0 && 32 * b < nx.nv) rec_stage<RWI>(a, nx, b, buf + m, bar + m);  // buffer free
        }
        if (a.rows_ctr && lane == 0)  // `built` is warp-uniform (ballot counts)
            atomicAdd(a.rows_ctr, (wid == 0 ? (unsigned long long)x.nv * a.bits_parent_row : 0ull) +
                                      (unsigned long long)built * a.bits_built_row);
        if (!OUT) {
            x = nx;
            continue;
        }
        __syncthreads();
        // ---------------- reserve: the item's left / right rows in the children's segments
        if (wid == 0) {
            const int nvb = max(0, min(32, x.nv - 32 * lane));
            const int nl = nvb > 0 ? s_nl[lane] : 0, nr = nvb - nl;
            int xl = nl, xr = nr;
            for (int o = 1; o < 32; o <<= 1) {
                const int yl = __shfl_up_sync(0xffffffffu, xl, o), yr = __shfl_up_sync(0xffffffffu, xr, o);
                if (lane >= o) {
                    xl += yl;
                    xr += yr;
                }
            }
            s_loff[lane] = xl - nl;
            s_roff[lane] = xr - nr;
            if (lane == 31) {
                s_baseL = (long long)atomicAdd(a.cursor + 2 * k, (unsigned long long)xl);
                s_baseR = (long long)atomicAdd(a.cursor + 2 * k + 1, (unsigned long long)(-(long long)xr)) - xr;
            }
        }
        __syncthreads();
        const long long baseL = s_baseL, baseR = s_baseR;
        // ---------------- phase B: the two runs of every batch to their children's segments
#pragma unroll
        for (int m = 0; m < 2; ++m) {
            const int b = wid + REC_NW * m;
            const int nrows = min(32, x.nv - 32 * b);
            if (nrows > 0) {
                const uint32_t *sw = reinterpret_cast<const uint32_t *>(reinterpret_cast<const char *>(buf[m].w) + x.head_r);
                const int2 *sq = reinterpret_cast<const int2 *>(reinterpret_cast<const char *>(buf[m].q) + x.head_q);
                const int nbr = s_nb[b];
                const unsigned char *ord = s_order[wid][m];
                const long long dL = baseL + s_loff[b], dR = baseR + s_roff[b];
                // destinations: run position c -> build child dB + c, or the other child dO + (c - nbr)
                const long long dB = build_left ? dL : dR, dO = (build_left ? dR : dL) - nbr;
                if (lane < nrows) a.out_q[(lane < nbr ? dB : dO) + lane] = sq[ord[lane]];
                if constexpr (RWI == RWP && RWP >= 4) {  // 16-byte units
                    constexpr int U = RWP / 4;
                    uint4 *o4 = reinterpret_cast<uint4 *>(a.out_rows);
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int t = lane + 32 * u, c = t / U, part = t - c * U;
                        if (c < nrows)
                            o4[((c < nbr ? dB : dO) + c) * U + part] = reinterpret_cast<const uint4 *>(sw)[ord[c] * U + part];
                    }
                } else if constexpr (RWI == RWP) {  // 1 or 2 words
                    if (lane < nrows) {
                        const long long d = ((lane < nbr ? dB : dO) + lane) * RWP;
                        const int r = ord[lane];
#pragma unroll
                        for (int w = 0; w < RWP; ++w) a.out_rows[d + w] = sw[r * RWP + w];
                    }
                } else {  // level 1: the packed rows padded to RWP words
#pragma unroll
                    for (int u = 0; u < RWP; ++u) {
                        const int t = lane + 32 * u, c = t / RWP, w = t - c * RWP;
                        if (c < nrows)
                            a.out_rows[((c < nbr ? dB : dO) + c) * RWP + w] = w < RWI ? sw[ord[c] * RWI + w] : 0u;
                    }
                }
            }
            __syncwarp();
            if (nx.j >= 0 && 32 * b < nx.nv) rec_stage<RWI>(a, nx, b, buf + m, bar + m);  // buffer free
        }
        x = nx;
    }
    __syncthreads();
    if (cur_j >= 0) col_flush<WIDE>(hs, COLB_STRIDE, cg, a.cut_ptr, a.hist + (long long)cur_j * a.TB * 2);
}

// After the level pass: the children's segments from the parents' cursors, and the children's
// own cursors for the next level (left fills from the front, right from the back).
__global__ void __launch_bounds__(1024) rec_seg_kernel(NodeDev *__restrict__ nodes, int first, int n_par,
                                                       unsigned long long *__restrict__ cursor) {
    for (int j = threadIdx.x; j < n_par; j += blockDim.x) {
        const int k = first + j;
        const NodeDev nd = nodes[k];
        NodeDev *Lc = nodes + 2 * k + 1, *Rc = nodes + 2 * k + 2;
        if (nd.state != GBM_NODE_SPLIT) {
            Lc->start = Lc->count = 0;
            Rc->start = Rc->count = 0;
            Lc->state = Rc->state = GBM_NODE_ABSENT;
            continue;
        }
        const long long nl = (long long)cursor[2 * k] - nd.start;
        Lc->start = nd.start;
        Lc->count = nl;
        Rc->start = nd.start + nl;
        Rc->count = nd.count - nl;
        cursor[2 * (2 * k + 1)] = nd.start;
        cursor[2 * (2 * k + 1) + 1] = nd.start + nl;
        cursor[2 * (2 * k + 2)] = nd.start + nl;
        cursor[2 * (2 * k + 2) + 1] = nd.start + nd.count;
    }
}

__global__ void rec_root_kernel(unsigned long long *cursor, long long n) {
    cursor[0] = 0;
    cursor[1] = (unsigned long long)n;
}

// ------------------------------------------------------------------ host side
size_t rec_smem_bytes(bool wide) {
    return (size_t)(wide ? 4 : 2) * COLB_STRIDE * 4 + 2 * REC_NW * sizeof(RecStage);
}

template <bool W, int RWI, int RWP, bool OUT>
static int rec_launch_t(gbm_ctx *ctx, const RecArgs &a, int n_items_hint, cudaStream_t s) {
    const size_t sm = rec_smem_bytes(W);
    auto kern = rec_level_kernel<W, RWI, RWP, OUT>;
    GBM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int occ = 0;
    GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, REC_THREADS, sm));
    if (occ < 1) return fail(GBM_E_ARG, "record level kernel cannot be resident");
    const int grid = std::max(1, std::min(occ * ctx->sm_count, n_items_hint));
    kern<<<grid, REC_THREADS, sm, s>>>(a);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

int rec_row_words(int rw) { return rw <= 1 ? 1 : rw <= 2 ? 2 : rw <= 4 ? 4 : 8; }

template <bool W, bool OUT>
static int rec_launch_rw(gbm_ctx *ctx, const RecArgs &a, int RWI, int RWP, int hint, cudaStream_t s) {
    if (RWP != rec_row_words(RWI) && RWP != RWI) return fail(GBM_E_ARG, "record row widths");
    switch (RWI) {
        case 1: return rec_launch_t<W, 1, 1, OUT>(ctx, a, hint, s);
        case 2: return rec_launch_t<W, 2, 2, OUT>(ctx, a, hint, s);
        case 3: return rec_launch_t<W, 3, 4, OUT>(ctx, a, hint, s);
        case 4: return rec_launch_t<W, 4, 4, OUT>(ctx, a, hint, s);
        case 5: return rec_launch_t<W, 5, 8, OUT>(ctx, a, hint, s);
        case 6: return rec_launch_t<W, 6, 8, OUT>(ctx, a, hint, s);
        case 7: return rec_launch_t<W, 7, 8, OUT>(ctx, a, hint, s);
        case 8: return rec_launch_t<W, 8, 8, OUT>(ctx, a, hint, s);
        default: return fail(GBM_E_ARG, "record rows hold 1..8 words");
    }
}

int rec_level_launch(gbm_ctx *ctx, const RecLaunch &L, cudaStream_t s) {
    RecArgs a = {};
    a.nodes = L.nodes;
    a.first = L.first;
    a.n_par = L.n_par;
    a.tile_base = L.tile_base;
    a.in_rows = L.in_rows;
    a.in_q = L.in_q;
    a.in_rows_bytes = L.in_rows_bytes;
    a.in_q_bytes = L.in_q_bytes;
    a.out_rows = L.out_rows;
    a.out_q = L.out_q;
    a.cursor = L.cursor;
    a.cut_ptr = L.cut_ptr;
    a.F = L.F;
    a.B = L.B;
    a.hist = L.hist;
    a.TB = L.TB;
    a.rows_ctr = L.rows_ctr;
    a.bits_parent_row = L.bits_parent_row;
    a.bits_built_row = L.bits_built_row;
    a.tma = (reinterpret_cast<uintptr_t>(L.in_rows) % 16 == 0 && reinterpret_cast<uintptr_t>(L.in_q) % 16 == 0 &&
             ctx->stage_tma) ? 1 : 0;
    const bool out = L.out_rows != nullptr;
    const int RWP = rec_row_words(L.RW);
    if (L.wide) return out ? rec_launch_rw<true, true>(ctx, a, L.RW_in, RWP, L.items_hint, s)
                           : rec_launch_rw<true, false>(ctx, a, L.RW_in, RWP, L.items_hint, s);
    return out ? rec_launch_rw<false, true>(ctx, a, L.RW_in, RWP, L.items_hint, s)
               : rec_launch_rw<false, false>(ctx, a, L.RW_in, RWP, L.items_hint, s);
}

int rec_seg_launch(gbm_ctx *, NodeDev *nodes, int first, int n_par, unsigned long long *cursor, cudaStream_t s) {
    rec_seg_kernel<<<1, 1024, 0, s>>>(nodes, first, n_par, cursor);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

int rec_root_launch(gbm_ctx *, unsigned long long *cursor, long long n, cudaStream_t s) {
    rec_root_kernel<<<1, 1, 0, s>>>(cursor, n);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

}  // namespace gbm
