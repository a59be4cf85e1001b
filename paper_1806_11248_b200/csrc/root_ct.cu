// root_ct.cu -- InitRoot's histogram fed by TMA tensor tiles of the
// feature-major symbol copy.
//
// The staged root (tree.cu hist_cs_range_kernel) copies 32 whole packed rows per warp and lane f
// reads byte f of each row: one LDS.U8 and one LDS.64 (the pair) per row besides the two ATOMS,
// which keeps the L1/TEX data pipe at ~83 % (profiles/r02_ncu_hist_summary.md).  Here every warp
// fetches a [features x 32 rows] byte tile of the feature-major copy colsym[F][n] with one
// cp.async.bulk.tensor.2d (the tensor map is built on the host per launch), plus the 32 rows'
// pairs with one bulk copy, so lane f holds its feature's 32 symbols after two 16-byte loads
// (8 registers) and extracts them with shifts; the pairs come two rows per 16-byte broadcast load.
// Per row and feature that leaves the two conflict-free ATOMS (word = bin * 32 + lane) and half
// a shared load.  Rows stream once (n * F bytes + 8 n), the histogram is the bank-column layout
// flushed into int64 (exact).  Requirements: 8-bit symbols with the colsym copy, n a multiple of
// 16 (the tensor map's row pitch), groups of <= 32 features with 32 / Fg in {1, 2, 4}.
#include <cudaTypedefs.h>

#include "tree_common.cuh"

namespace gbm {


template <int TR>
struct __align__(128) CtBuf {  // one staging buffer of a warp (tensor-copy destination)
    uint8_t sym[32][TR];       // [feature of the group][row of the batch]
    int2 q[TR];
};

struct CtArgs {
    const int2 *qpair;
    long long n;
    int F, ng, fbox;           // features, groups, features per tensor box
    long long chunk;           // rows per work item (a multiple of 32)
    const int32_t *cut_ptr;
    unsigned long long *hist;    // [TB][2]
    unsigned long long *totals;  // [2] or null
    unsigned long long *rows_ctr;
};

__device__ __forceinline__ void tensor_g2s(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void red_s32(unsigned addr, int v) {
    asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

template <bool WIDE>
__device__ __forceinline__ void col_red2(unsigned addr, int qx, int qy) {
    if (WIDE) {
        red_s32(addr, qx & 0x7fff);
        red_s32(addr + 4 * COLB_STRIDE, qy & 0x7fff);
        red_s32(addr + 8 * COLB_STRIDE, qx >> 15);
        red_s32(addr + 12 * COLB_STRIDE, qy >> 15);
    } else {
        red_s32(addr, qx);
        red_s32(addr + 4 * COLB_STRIDE, qy);
    }
}

// R rows per accumulate step: lane = copy * Fg + feature, copy c takes rows c, c + R, ...
// TR rows per tensor tile (32, 64 or 128): each feature's piece of a tile is TR contiguous bytes.
template <bool WIDE, int R, int NW, int NS, int TR>
__global__ void __launch_bounds__(NW * 32, WIDE ? 1 : 2) hist_ct_root_kernel(const __grid_constant__ CUtensorMap map,
                                                                            CtArgs a) {
    extern __shared__ __align__(128) int smem[];
    constexpr int CH = WIDE ? 4 : 2;
    using CtBuf = gbm::CtBuf<TR>;
    CtBuf *stage = reinterpret_cast<CtBuf *>(smem + CH * COLB_STRIDE);  // [NW][NS]
    __shared__ uint64_t s_bar[NS * NW];
    __shared__ long long s_red[2 * NW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t *bar = s_bar + NS * wid;
    CtBuf *buf = stage + NS * wid;
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < NS; ++i) mbar_init(bar + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    unsigned phbits = 0;
    unsigned seq = 0;
    const unsigned hb = smem_u32(smem) + 4u * lane;
    long long tg = 0, th = 0;
    const long long n_chunks = (a.n + a.chunk - 1) / a.chunk;
    const long long n_items = n_chunks * a.ng;
    for (long long it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int g = (int)(it % a.ng);
        const long long start = (it / a.ng) * a.chunk;
        const long long end = min(a.n, start + a.chunk);
        const int f_lo = (int)((long long)a.F * g / a.ng), f_hi = (int)((long long)a.F * (g + 1) / a.ng);
        const int Fg = f_hi - f_lo;
        const int c = lane / Fg, f = lane - c * Fg;
        const bool on = c < R;
        const bool tot = a.totals && g == 0;
        for (int i = threadIdx.x; i < CH * COLB_STRIDE; i += NW * 32) smem[i] = 0;
        if (a.rows_ctr && g == 0 && threadIdx.x == 0) atomicAdd(a.rows_ctr, (unsigned long long)(end - start));
        __syncthreads();
        // this warp's 32-row batches b0 = start + 32 (wid + NW m) < end; the last one of the
        // matrix may hold 16 rows (n is a multiple of 16): the tensor copy zero-fills the rows past
        // n, the pair copy takes 16 rows and the rest of the pairs are zeroed (adds of 0)
        const long long b_first = start + (long long)TR * wid;
        const int nb = b_first < end ? (int)((end - b_first - 1) / ((long long)TR * NW)) + 1 : 0;
        auto issue = [&](int m, unsigned cb) {
            const long long b0 = b_first + (long long)TR * NW * m;
            const int rows = (int)min((long long)TR, end - b0);
            if (rows < TR) {
                for (int i = lane; i < TR; i += 32)
                    if (i >= rows) buf[cb].q[i] = make_int2(0, 0);
                __syncwarp();
            }
            if (lane == 0) {
                fence_proxy_async();
                mbar_arrive_expect_tx(bar + cb, (unsigned)TR * a.fbox + 8u * rows);
                tensor_g2s(buf[cb].sym, &map, (int)b0, f_lo, bar + cb);
                bulk_g2s(buf[cb].q, a.qpair + b0, 8u * rows, bar + cb);
            }
        };
        // NS-deep pipeline: batch m lands in buffer (seq0 + m) % NS, NS - 1 batches in flight
        const unsigned seq0 = seq;
#pragma unroll
        for (int m = 0; m < NS - 1; ++m)
            if (m < nb) issue(m, (seq0 + m) % NS);
        for (int m = 0; m < nb; ++m) {
            const unsigned cb = seq % NS;
            if (m + NS - 1 < nb) issue(m + NS - 1, (seq + NS - 1) % NS);
            mbar_wait(bar + cb, (phbits >> cb) & 1u);
            phbits ^= 1u << cb;
            const CtBuf &st = buf[cb];
#pragma unroll 1
            for (int sb = 0; sb < TR; sb += 32)  // 32-row sub-batches of the tile
            if (on) {
                const uint4 v0 = *reinterpret_cast<const uint4 *>(&st.sym[f][sb]);
                const uint4 v1 = *reinterpret_cast<const uint4 *>(&st.sym[f][sb + 16]);
                const uint32_t w[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                const int4 *q2 = reinterpret_cast<const int4 *>(st.q + sb);
#pragma unroll
                for (int mm = 0; mm < 32 / R; mm += 2) {  // rows R mm + c and R (mm + 1) + c
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int m2 = mm + h;
                        const int sh = 8 * ((R * m2 + c) & 3);
                        const int sy = (w[(R * m2) >> 2] >> sh) & 255;  // (R m2 + c) >> 2 == (R m2) >> 2 for c < R <= 4
                        int qx, qy;
                        if (R == 1) {
                            const int4 qq = q2[m2 >> 1];
                            qx = (m2 & 1) ? qq.z : qq.x;
                            qy = (m2 & 1) ? qq.w : qq.y;
                        } else {
                            const int2 qq = st.q[sb + R * m2 + c];
                            qx = qq.x;
                            qy = qq.y;
                        }
                        col_red2<WIDE>(hb + ((unsigned)sy << 7), qx, qy);
                    }
                }
            }
            if (tot) {
#pragma unroll
                for (int i = lane; i < TR; i += 32) {
                    const int2 qq = st.q[i];
                    tg += qq.x;
                    th += qq.y;
                }
            }
            __syncwarp();
            ++seq;
        }
        if (tot) {
            for (int o = 16; o > 0; o >>= 1) {
                tg += __shfl_xor_sync(0xffffffffu, tg, o);
                th += __shfl_xor_sync(0xffffffffu, th, o);
            }
            if (lane == 0) {
                s_red[2 * wid] = tg;
                s_red[2 * wid + 1] = th;
            }
            tg = th = 0;
        }
        __syncthreads();
        if (tot && threadIdx.x == 0) {
            long long x = 0, y = 0;
            for (int i = 0; i < NW; ++i) {
                x += s_red[2 * i];
                y += s_red[2 * i + 1];
            }
            atomicAdd(a.totals, (unsigned long long)x);
            atomicAdd(a.totals + 1, (unsigned long long)y);
        }
        col_flush<WIDE>(smem, COLB_STRIDE, ColGroup{f_lo, f_hi}, a.cut_ptr, a.hist);
        __syncthreads();
    }
}

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        else
            cudaGetLastError();
    }
    return fn;
}

template <bool W, int R, int NW, int NS, int TR>
static int ct_launch_t(gbm_ctx *ctx, const CUtensorMap &map, const CtArgs &a, long long n_items, cudaStream_t s) {
    const size_t sm = (size_t)(W ? 4 : 2) * COLB_STRIDE * 4 + (size_t)NS * NW * sizeof(CtBuf<TR>);
    auto kern = hist_ct_root_kernel<W, R, NW, NS, TR>;
    GBM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    int occ = 0;
    GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, sm));
    if (occ < 1) return fail(GBM_E_ARG, "tensor-fed root kernel cannot be resident");
    const int grid = (int)std::max<long long>(1, std::min<long long>(n_items, (long long)occ * ctx->sm_count));
    kern<<<grid, NW * 32, sm, s>>>(map, a);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

template <bool W, int R>
static int ct_launch_cfg(gbm_ctx *ctx, const CUtensorMap &map, const CtArgs &a, long long n_items, int cfg,
                         cudaStream_t s) {
    switch (cfg) {  // (warps per block, pipeline depth, rows per tile)
        case 3: return ct_launch_t<W, R, 12, 3, 32>(ctx, map, a, n_items, s);
        case 4: return ct_launch_t<W, R, 8, 4, 32>(ctx, map, a, n_items, s);
        case 5: return ct_launch_t<W, R, 8, 2, 64>(ctx, map, a, n_items, s);
        case 6: return ct_launch_t<W, R, 16, 2, 64>(ctx, map, a, n_items, s);
        case 7: return ct_launch_t<W, R, 16, 2, 128>(ctx, map, a, n_items, s);
        default: return ct_launch_t<W, R, 16, 2, 32>(ctx, map, a, n_items, s);
    }
}

// 1: launched; 0: does not apply (the caller uses the staged / compact root); < 0: error
int root_ct_launch(gbm_ctx *ctx, const RootCtLaunch &L, cudaStream_t s) {
    if (!L.colsym || L.bits != 8 || L.n < 32 || L.n % 16 != 0 || L.n > INT_MAX || L.F < 8 || ctx->root_ct == 1 ||
        reinterpret_cast<uintptr_t>(L.colsym) % 16 != 0 || reinterpret_cast<uintptr_t>(L.qpair) % 16 != 0)
        return 0;
    const int ng = (L.F + 31) / 32;
    const int fmin = L.F / ng, fmax = (L.F + ng - 1) / ng;
    const int R = 32 / fmax;
    if ((R != 1 && R != 2 && R != 4) || 32 / fmin != R) return 0;  // every group the same copy count
    // measured (profiles/r02/root_tensor_ab.txt): faster with several feature groups (Epsilon root
    // 0.58 vs 0.76 ms) or several rows per step (Airline, 13 features: 1.29 vs 1.66 ms) at 32-row
    // tiles; for one group of 17..32 features the 28 scattered 32-byte pieces of a 32-row tile
    // arrive too late (Higgs: 0.31 vs 0.28 ms staged, ncu long-scoreboard 5.6 vs 1.5), 64-row
    // tiles with 16 warps x 2 stages (one block per SM) win (0.262 vs 0.285 ms)
    int cfg = ctx->root_ct;  // 2 (default shape), 3-7: the measured pipeline shapes / tile rows
    if (cfg == 0) cfg = (ng == 1 && R == 1) ? 6 : 2;  // (wide accumulators too: Higgs P = 30 root 0.744 -> 0.302 ms)
    if (cfg == 1) return 0;
    PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
    if (!enc) return 0;
    CUtensorMap map;
    const cuuint64_t dims[2] = {(cuuint64_t)L.n, (cuuint64_t)L.F};
    const cuuint64_t strides[1] = {(cuuint64_t)L.n};
    const int TR = cfg == 7 ? 128 : (cfg == 5 || cfg == 6) ? 64 : 32;
    {  // the shape's shared memory (histogram channels + staging buffers) must fit one block
        const int NWS[8] = {0, 0, 32, 36, 32, 16, 32, 32};  // warps x stages per shape
        const size_t sm = (size_t)(L.wide ? 4 : 2) * COLB_STRIDE * 4 + (size_t)NWS[cfg] * (32 * TR + 8 * TR);
        if (sm + 1024 > ctx->smem_optin) return 0;  // (wide accumulators at 128-row tiles)
    }
    const cuuint32_t box[2] = {(cuuint32_t)TR, (cuuint32_t)fmax};
    const cuuint32_t estr[2] = {1u, 1u};
    if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t *>(L.colsym), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return 0;
    CtArgs a = {};
    a.qpair = L.qpair;
    a.n = L.n;
    a.F = L.F;
    a.ng = ng;
    a.fbox = fmax;
    a.cut_ptr = L.cut_ptr;
    a.hist = L.hist;
    a.totals = L.totals;
    // items: one per resident block for one feature group (every item zeroes and flushes the whole
    // bank-column histogram), two per block with several groups (Epsilon root 0.586 vs 0.686 at
    // one: wave quantisation) -- both capped by the exactness bound below
    const long long blocks = (long long)(L.wide || cfg == 6 || cfg == 7 ? 1 : 2) * ctx->sm_count;
    // exactness: a copy's int32 bank column takes at most MAX_CHUNK rows per flush (|q| <= 2^15),
    // so an item holds at most cap rows; whole waves of items over the resident blocks
    const long long cap = (long long)MAX_CHUNK * R / TR * TR;
    long long waves = ng == 1 ? 1 : 2;
    while ((L.n * ng + waves * blocks - 1) / (waves * blocks) > cap) ++waves;
    const long long per = waves * blocks;  // items wanted
    a.chunk = std::min<long long>(cap, std::max<long long>((long long)TR * 16,
                                                           ((L.n * ng + per - 1) / per + TR - 1) / TR * TR));
    const long long n_items = (L.n + a.chunk - 1) / a.chunk * ng;
    int slot = -1;
    a.rows_ctr = prof_rows_slot(ctx, &slot);  // algorithmic bytes: n (F b / 8 + 8), SURVEY §8(d)
    ProfScope ps(ctx, PC_HIST_ROOT, s, 0.0, slot, (double)L.F + 8.0);
    int rc;
    if (L.wide) rc = R == 1 ? ct_launch_cfg<true, 1>(ctx, map, a, n_items, cfg, s)
                            : R == 2 ? ct_launch_cfg<true, 2>(ctx, map, a, n_items, cfg, s)
                                     : ct_launch_cfg<true, 4>(ctx, map, a, n_items, cfg, s);
    else rc = R == 1 ? ct_launch_cfg<false, 1>(ctx, map, a, n_items, cfg, s)
                     : R == 2 ? ct_launch_cfg<false, 2>(ctx, map, a, n_items, cfg, s)
                              : ct_launch_cfg<false, 4>(ctx, map, a, n_items, cfg, s);
    return rc == GBM_OK ? 1 : rc;
}

}  // namespace gbm
