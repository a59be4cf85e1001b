// tree.cu -- §2.3 decision-tree construction (Algorithm 1) on sm_100a.
//
// The tree is grown level-synchronously (R15): each depth is one pass of a fixed launch
// sequence, and one NCCL allreduce per level carries the histograms of all of that level's
// built children.  For level l = 1..D-1 (parents = the nodes of depth l-1):
//
//   plan         1 block: tile plan of the parents (1024-row tiles of their ridx segments) and
//                the work items of the fused kernel (runs of RUN tiles x feature groups).
//   part_hist    RepartitionInstances + BuildPartialHistograms, fused (north star, SURVEY §8a
//                a5+a6): per tile the split symbol of every row (warp-ballot flag words, the
//                tile's left count), then the rows falling into the parent's smaller child
//                (R17) are accumulated into a privatised shared-memory histogram; flushed once
//                per work item into the parent's int64 slot.  Leaf parents write row_leaf.
//   part_scan    1 block per parent: exclusive scan of its tiles' left counts (stable order)
//                -> the children's ridx segments.
//   part_scatter stable scatter of the row ids into the children's segments (flags + ridx only).
//   allreduce    AllReduceHistograms: ncclAllReduce(int64, sum) over the level's built slots.
//   eval_feat    one warp per (node, feature): sibling = parent - built child (exact int64),
//                prefix scan over the feature's bins, both default directions, XGBoost gain in
//                the op order of R8, best candidate of the feature.
//   eval_final   1 block per node: canonical argmax over features -> split record / leaf.
//
// Shared-memory accumulators (R14): 32-bit ATOMS.ADD is native on sm_100 while 64-bit shared
// atomics compile to a CAS loop, so bins are int32 and flushed into int64 global histograms
// after at most 65535 rows.  With grad_bits P <= 15 each |q| <= 2^15 and a bin's sum stays below
// 65535 * 2^15 < 2^31 ("narrow", 2 ATOMS per update).  With 15 < P <= 30, q = hi*2^15 + lo with
// 0 <= lo < 2^15, |hi| <= 2^15, both accumulated ("wide", 4 ATOMS per update).
#include <algorithm>
#include <climits>
#include <vector>

#include "tree_common.cuh"

namespace gbm {

// Loss-guided growth (R25-R27).  A node evaluated with a positive-gain split that may still be
// expanded is OPEN until the step kernel selects it (then SPLIT) -- internal state only.
constexpr int NODE_OPEN = 3;
struct LgNode {        // per node, loss-guided only
    double gain;       // best split gain (OPEN nodes)
    long long Lg, Lh;  // left child totals of that split
    int depth;
    int hslot;         // histogram pool slot (nodes that may be expanded)
    int buf;           // ridx buffer holding the node's rows: 0 / 1, -1 = identity (root)
    int pad;
};
struct StepDev {       // the expansion of the current step, written by lg_select_kernel
    int k;             // parent (-1: nothing left to expand -- every later launch is a no-op)
    int c;             // its left child (2j+1); right = c + 1
    int in_buf, out_buf;
    int run_tiles;     // tiles per work item of the fused kernel, sized to the parent
    int pad;
};

struct TreeDev {
    int8_t *kind;
    int32_t *feature, *bin;
    float *threshold;
    int8_t *default_left;
    double *gain, *weight;
    long long *sum_qg, *sum_qh;
    int32_t *left_child;  // optional for depth-wise trees
};

struct Group {
    int u_lo, u_hi;      // units [u_lo, u_hi) of a row (a unit = S consecutive features)
    int bin_lo, bin_hi;  // global bins of the group's features
};

struct FeatBest {  // best candidate of one (node, feature)
    double gain;
    long long idx;  // canonical candidate order: (global bin)*2 + (dl ? 0 : 1); LLONG_MAX = none
    long long Lg, Lh;
};

// what the finishing block already knows about a node (skips a second node_source round trip)
struct NodeKnown {
    int state;  // 0 unknown, 1 present with totals Tg, Th, 2 absent
    long long Tg, Th;
};

constexpr int E_THREADS = 256;   // evaluation kernels
constexpr int DUMMY_BINS = 32;   // scratch bins: padding features of the byte path (symbol 0)
// Replicated bins of low-cardinality features (fused level kernel, byte path): lanes of different
// row slots that hit the same bin of a feature with few bins serialise on one address; with R
// copies (row slot r adds into copy r mod R) they hit R different words.  Copies 1..R-1 live in
// REP_CAP words after the scratch bins of each channel and are folded into copy 0 before the flush.
constexpr int REP_CAP = 512;     // replica words per channel
constexpr int REP_F = 128;       // groups of more features are not replicated
constexpr int REP_NB = 128;      // R * bins <= REP_NB, R <= 8 and R <= rows per pass
__host__ __device__ __forceinline__ int rep_log2(int nb, int rpp) {
    int r = 1, l = 0;
    while (2 * r <= rpp && 2 * r <= 8 && 2 * r * nb <= REP_NB) {
        r *= 2;
        ++l;
    }
    return l;
}

struct EvalParams {
    double eta, lambda, gamma, mcw;
    int max_depth;
    int screen;  // 1: exact evaluation only of candidates that pass the approximate screen
};

// ============================================================== shared-memory histogram
// Layout per channel: [bins of the group (nb)][DUMMY_BINS scratch], channels at stride hstride.
// narrow: channel 0 = g, 1 = h;  wide: 0 = g_lo, 1 = h_lo, 2 = g_hi, 3 = h_hi.
struct SmemHist {
    int *base;
    int nb, hstride;
};

template <bool WIDE>
__device__ __forceinline__ void hist_add(int *hs, int hstride, int bin, int2 q) {
    if (WIDE) {
        atomicAdd(hs + bin, q.x & 0x7fff);
        atomicAdd(hs + hstride + bin, q.y & 0x7fff);
        atomicAdd(hs + 2 * hstride + bin, q.x >> 15);
        atomicAdd(hs + 3 * hstride + bin, q.y >> 15);
    } else {
        atomicAdd(hs + bin, q.x);
        atomicAdd(hs + hstride + bin, q.y);
    }
}

template <bool WIDE>
__device__ void smem_zero(const SmemHist &h) {
    const int n = (WIDE ? 4 : 2) * h.hstride;
    for (int i = threadIdx.x; i < n; i += blockDim.x) h.base[i] = 0;
}

// flush the group's bins into the int64 slot (global atomics: several items share a slot)
template <bool WIDE>
__device__ void smem_flush(const SmemHist &h, unsigned long long *dst /* slot + 2*bin_lo */) {
    for (int b = threadIdx.x; b < h.nb; b += blockDim.x) {
        long long G, H;
        if (WIDE) {
            G = (long long)h.base[2 * h.hstride + b] * 32768 + (long long)(unsigned)h.base[b];
            H = (long long)h.base[3 * h.hstride + b] * 32768 + (long long)(unsigned)h.base[h.hstride + b];
        } else {
            G = h.base[b];
            H = h.base[h.hstride + b];
        }
        if (G) atomicAdd(dst + 2 * b, (unsigned long long)G);
        if (H) atomicAdd(dst + 2 * b + 1, (unsigned long long)H);
    }
}

// Per-thread setup of the byte path: thread -> (row lane r0, word w of the group); the bin
// offsets of its 4 features live in registers (padding features -> the scratch bins).
struct ByteLane {
    int r0, rstep, w;  // r0 < 0: thread idle
    int off[4];
    unsigned agg;      // symbol slots (bit j) warp-aggregated: some lane's feature has few bins
};

// Features with at most this many bins are warp-aggregated.  0 = off: measured on B200,
// __match_any_sync costs far more than the same-address ATOMS replays it removes (Higgs root
// 0.33 -> 2.14 ms, Airline root 0.65 -> 7.6 ms with 64), so the path is kept but disabled.
constexpr int AGG_MAX_BINS = 0;

// Adds the 4 byte symbols of word wd with pair q.  Slots flagged in agg go through
// __match_any_sync + __reduce_add_sync first, so the lanes that hit the same bin of a
// low-cardinality feature (same-address ATOMS serialise) issue a single atomic (north star:
// "warp-aggregated updates").  Called by all 32 lanes (warp-uniform control flow).
template <bool WIDE, bool SENT>
__device__ __forceinline__ void byte_word_add(const SmemHist &h, const int (&off)[4], unsigned agg, uint32_t wd,
                                              int2 q, bool valid, int B) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int sy = (wd >> (8 * j)) & 255;
        const bool ok = valid && (!SENT || sy != B);
        const int bin = off[j] + sy;
        if (!WIDE && ((agg >> j) & 1u)) {
            const unsigned peers = __match_any_sync(0xffffffffu, ok ? bin : -1 - lane);
            const int gs = __reduce_add_sync(peers, ok ? q.x : 0);
            const int hs = __reduce_add_sync(peers, ok ? q.y : 0);
            if (ok && lane == __ffs(peers) - 1) {
                atomicAdd(h.base + bin, gs);
                atomicAdd(h.base + h.hstride + bin, hs);
            }
        } else if (ok) {
            hist_add<WIDE>(h.base, h.hstride, bin, q);
        }
    }
}

__device__ __forceinline__ ByteLane byte_lane(const QM &qm, const Group &grp, const int *s_off, int nb) {
    ByteLane L;
    const int Ug = grp.u_hi - grp.u_lo;
    const int rb = H_THREADS / Ug;
    L.rstep = rb;
    L.r0 = (int)threadIdx.x < rb * Ug ? (int)threadIdx.x / Ug : -1;
    const int wr = L.r0 < 0 ? 0 : (int)threadIdx.x - L.r0 * Ug;
    L.w = grp.u_lo + wr;
    const int f_lo = grp.u_lo * 4;
    unsigned lc = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        int f = L.w * 4 + j;
        const bool real = L.r0 >= 0 && f < qm.F;
        L.off[j] = real ? s_off[f - f_lo] : nb + (int)(threadIdx.x & 31);  // padding: a scratch bin per lane
        if (real && s_off[f - f_lo + 1] - s_off[f - f_lo] <= AGG_MAX_BINS) lc |= 1u << j;
    }
    L.agg = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (__any_sync(0xffffffffu, (lc >> j) & 1u)) L.agg |= 1u << j;
    return L;
}

// Accumulate rows [0, nrows) of a row source.  BYTE: 8-bit symbols, rows word-aligned.
// SENT: the sentinel fits in the symbol width (missing values possible) -> skip it.
template <bool WIDE, bool BYTE, bool SENT, class RowFn>
__device__ __forceinline__ void accumulate(const QM &qm, const Group &grp, const int *s_off,
                                           const SmemHist &h, const int2 *__restrict__ qpair, RowFn rowf,
                                           int nrows, const ByteLane &L, long long *tg, long long *th,
                                           bool totals) {
    if (BYTE) {
        totals = totals && L.r0 >= 0 && L.w == grp.u_lo;  // each row's pair counted once
        const long long sw = qm.stride >> 5;                // words per row
        for (int rb = 0; rb < nrows; rb += 4 * L.rstep) {   // warp-uniform; four rows in flight
            uint32_t wd[4];
            int2 qq[4];
            bool ok[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int r = rb + L.r0 + i * L.rstep;
                ok[i] = L.r0 >= 0 && r < nrows;
                const uint32_t ra = rowf(ok[i] ? r : 0);
                wd[i] = __ldg(qm.P + ra * sw + L.w);
                qq[i] = __ldg(qpair + ra);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (totals && ok[i]) {
                    *tg += qq[i].x;
                    *th += qq[i].y;
                }
                byte_word_add<WIDE, SENT>(h, L.off, L.agg, wd[i], qq[i], ok[i], qm.B);
            }
        }
    } else {
        // generic widths / layouts: thread -> (row, unit) over the flattened range
        const int Ug = grp.u_hi - grp.u_lo;
        const uint32_t magic = 0xffffffffu / (uint32_t)Ug + 1u;
        const uint32_t total = (uint32_t)nrows * (uint32_t)Ug;
        const int f_lo = grp.u_lo * qm.S;
        const uint32_t mask = (1u << qm.bits) - 1u;
        for (uint32_t j0 = threadIdx.x; j0 < total; j0 += 4 * H_THREADS) {  // four (row, unit) in flight
            uint32_t win[4];
            int2 q[4];
            int f0[4], ns[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t j = j0 + i * H_THREADS;
                const bool ok = j < total;
                const uint32_t r = Ug == 1 ? j : fast_div(j, magic);
                const int u = grp.u_lo + (int)(j - r * (uint32_t)Ug);
                const uint32_t row = rowf(ok ? (int)r : 0);
                q[i] = __ldg(qpair + row);
                if (totals && ok && u == grp.u_lo) {
                    *tg += q[i].x;
                    *th += q[i].y;
                }
                f0[i] = ok ? u * qm.S : f_lo;
                ns[i] = ok ? min(qm.S, qm.F - f0[i]) : 0;
                win[i] = get_bits(qm.P, (long long)row * qm.stride + (long long)f0[i] * qm.bits, max(ns[i], 1) * qm.bits);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
                for (int jj = 0; jj < ns[i]; ++jj) {
                    const int s = (int)((win[i] >> (jj * qm.bits)) & mask);
                    if (s == qm.B) continue;  // missing: mass recovered as total - sum (R7)
                    hist_add<WIDE>(h.base, h.hstride, s_off[f0[i] + jj - f_lo] + s, q[i]);
                }
        }
    }
}

__device__ __forceinline__ void load_group(const QM &qm, const Group &grp, const int32_t *__restrict__ cut_ptr,
                                           int *s_off) {
    const int f_lo = grp.u_lo * qm.S, f_hi = min(grp.u_hi * qm.S, qm.F);
    for (int f = f_lo + threadIdx.x; f <= f_hi; f += blockDim.x) s_off[f - f_lo] = __ldg(cut_ptr + f) - grp.bin_lo;
}

__device__ __forceinline__ void block_totals(long long tg, long long th, long long *red, unsigned long long *out) {
    for (int o = 16; o > 0; o >>= 1) {
        tg += __shfl_xor_sync(0xffffffffu, tg, o);
        th += __shfl_xor_sync(0xffffffffu, th, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[2 * w] = tg;
        red[2 * w + 1] = th;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long a = 0, b = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            a += red[2 * i];
            b += red[2 * i + 1];
        }
        atomicAdd(out + 0, (unsigned long long)a);
        atomicAdd(out + 1, (unsigned long long)b);
    }
}

// ============================================================== range histogram (root, entry)
struct RangeArgs {
    QM qm;
    const int2 *qpair;
    const uint32_t *ridx;        // null = identity rows
    long long n_sel;             // rows
    int chunk, n_groups;
    const Group *groups;
    const int32_t *cut_ptr;
    unsigned long long *hist;    // [TB][2] (one slot)
    unsigned long long *totals;  // [2] or null
    unsigned long long *rows_ctr;
    int hstride;
};

template <bool WIDE, bool BYTE, bool SENT>
__global__ void __launch_bounds__(H_THREADS, GBM_HR_MINB) hist_range_kernel(RangeArgs a) {
    extern __shared__ int smem[];
    __shared__ int s_off[2049];
    __shared__ long long s_red[2 * H_THREADS / 32];
    const QM &qm = a.qm;
    const int n_items = (int)(((a.n_sel + a.chunk - 1) / a.chunk) * a.n_groups);
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int g = it % a.n_groups;
        const long long start = (long long)(it / a.n_groups) * a.chunk;
        const int len = (int)min((long long)a.chunk, a.n_sel - start);
        const Group grp = a.groups[g];
        SmemHist h{smem, grp.bin_hi - grp.bin_lo, a.hstride};
        if (a.rows_ctr && g == 0 && threadIdx.x == 0) atomicAdd(a.rows_ctr, (unsigned long long)len);
        smem_zero<WIDE>(h);
        load_group(qm, grp, a.cut_ptr, s_off);
        __syncthreads();
        ByteLane L = BYTE ? byte_lane(qm, grp, s_off, h.nb) : ByteLane{};
        long long tg = 0, th = 0;
        const bool tot = a.totals && g == 0;
        if (a.ridx) {
            const uint32_t *rp = a.ridx + start;
            accumulate<WIDE, BYTE, SENT>(qm, grp, s_off, h, a.qpair, [&](int r) { return __ldg(rp + r); }, len, L,
                                         &tg, &th, tot);
        } else {
            const uint32_t s0 = (uint32_t)start;
            accumulate<WIDE, BYTE, SENT>(qm, grp, s_off, h, a.qpair, [&](int r) { return s0 + (uint32_t)r; }, len, L,
                                         &tg, &th, tot);
        }
        if (tot) block_totals(tg, th, s_red, a.totals);
        __syncthreads();
        smem_flush<WIDE>(h, a.hist + 2ll * grp.bin_lo);
        __syncthreads();
    }
}

// ============================================================== partition helpers
// Row-index entries of the level buffers.  CARRY (grad_bits <= 15): the row's fixed-point
// gradient pair travels with its index through every partition, so no level pass gathers qpair
// (a 64-byte DRAM access per 8-byte pair).  q_g in [-2^15, 2^15] needs 17 bits, q_h in
// [0, 2^15] 16: x = row | (bit 16 of q_g) << 31 (rows < 2^31), y = q_g[15:0] | q_h << 16.
template <bool CARRY> struct EntryOf { using T = uint32_t; };
template <> struct EntryOf<true> { using T = uint2; };
__device__ __forceinline__ uint32_t row_of(uint32_t e) { return e; }
__device__ __forceinline__ uint32_t row_of(uint2 e) { return e.x & 0x7fffffffu; }
template <bool CARRY>
__device__ __forceinline__ typename EntryOf<CARRY>::T make_entry(uint32_t row, const int2 *__restrict__ qpair) {
    if constexpr (CARRY) {
        const int2 q = __ldg(qpair + row);
        const uint32_t g17 = (uint32_t)q.x & 0x1ffffu;
        return make_uint2(row | ((g17 >> 16) << 31), (g17 & 0xffffu) | ((uint32_t)q.y << 16));
    } else {
        return row;
    }
}
__device__ __forceinline__ int2 entry_q(uint2 e, const int2 *) {
    const uint32_t g17 = ((e.x >> 31) << 16) | (e.y & 0xffffu);
    return make_int2(((int)(g17 << 15)) >> 15, (int)(e.y >> 16));
}
__device__ __forceinline__ int2 entry_q(uint32_t e, const int2 *__restrict__ qpair) { return __ldg(qpair + e); }

__device__ __forceinline__ bool goes_left(const QM &qm, const NodeDev &nd, uint32_t row) {
    if (qm.dbits) return (__ldg(qm.dbits + (row >> 5)) >> (row & 31)) & 1u;  // row_decide_kernel
    const uint32_t sym = split_symbol(qm, row, nd.f);
    return (int)sym == qm.B ? (nd.dl != 0) : ((int)sym <= nd.b);
}

// ============================================================== plan (1 block)
// Tile plan of the parents of a level: tile_base[j] (first 2048-row tile of parent j) and
// run_base[j] (first RUN-tile run); n_items = runs x feature groups.  Work item i of the fused
// kernel is run i / G, group i % G, resolved on the fly (find_parent over run_base).
// Works for any block size that is a multiple of 32 (<= 1024).
// run_tiles < 0: sized per level for -run_tiles resident blocks -- about one item per block, or
// the fewest whole waves when MAX_CHUNK caps the item (each item zeroes and flushes a whole shared
// histogram; measured: Higgs levels 0.975 -> 0.870 ms/round, YearMSD 0.300 -> 0.247, Airline
// 11.94 -> 11.56 against ~4 items per block).  The tiles per item go to n_items[2].
__device__ void plan_block(const NodeDev *__restrict__ nodes, int first, int n_par, int n_groups, int run_tiles,
                           int *__restrict__ tile_base, int *__restrict__ run_base, int *__restrict__ n_items,
                           bool split_only = false, long long rows_ub = 0) {
    __shared__ long long sm32[32];
    __shared__ long long carry;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    auto eligible = [&](const NodeDev &nd) {
        return nd.count > 0 && (split_only ? nd.state == GBM_NODE_SPLIT : nd.state != GBM_NODE_ABSENT);
    };
    if (run_tiles < 0) {  // the level's tiles: at most ceil(rows / PT) + n_par (no extra pass)
        const long long T = (rows_ub + PT - 1) / PT + n_par, np = n_par, B = -(long long)run_tiles;
        // the fewest whole waves of items (w x B, at most) whose items fit MAX_CHUNK rows
        long long rt = MAX_CHUNK / PT;
        for (long long w = 1; w <= 64; ++w) {
            const long long slots = w * B - np * n_groups;  // ceil per parent: <= np extra runs
            if (slots <= 0) continue;
            const long long r = (T * n_groups + slots - 1) / slots;
            if (r <= MAX_CHUNK / PT) {
                rt = max(1ll, r);
                break;
            }
        }
        run_tiles = (int)rt;
    }
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int c = 0; c < n_par; c += blockDim.x) {
        const int j = c + threadIdx.x;
        long long nt = 0, nr = 0;
        if (j < n_par) {
            const NodeDev nd = nodes[first + j];
            if (eligible(nd)) {
                nt = (nd.count + PT - 1) / PT;
                nr = (nt + run_tiles - 1) / run_tiles;
            }
        }
        const long long v = (nt << 32) | nr;
        long long x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) sm32[wid] = x;
        __syncthreads();
        if (wid == 0) {
            long long t = lane < nw ? sm32[lane] : 0;
            for (int o = 1; o < 32; o <<= 1) {
                const long long y = __shfl_up_sync(0xffffffffu, t, o);
                if (lane >= o) t += y;
            }
            sm32[lane] = t;
        }
        __syncthreads();
        const long long ex = carry + (wid ? sm32[wid - 1] : 0) + x - v;
        if (j < n_par) {
            tile_base[j] = (int)(ex >> 32);
            run_base[j] = (int)(ex & 0xffffffff);
        }
        __syncthreads();
        if (threadIdx.x == 0) carry += sm32[nw - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        tile_base[n_par] = (int)(carry >> 32);
        run_base[n_par] = (int)(carry & 0xffffffff);
        n_items[0] = (int)(carry & 0xffffffff) * n_groups;
        n_items[1] = 0;  // dynamic work counter of the fused kernel
        n_items[2] = run_tiles;
    }
}

__global__ void __launch_bounds__(1024) plan_kernel(const NodeDev *__restrict__ nodes, int first, int n_par,
                                                    int n_groups, int *__restrict__ tile_base,
                                                    int *__restrict__ run_base, int *__restrict__ n_items) {
    plan_block(nodes, first, n_par, n_groups, 1, tile_base, run_base, n_items);
}

// ============================================================== fused partition + histogram
struct FusedArgs {
    QM qm;
    const NodeDev *nodes;
    int first, n_par;
    const int *tile_base;
    const int *run_base;
    int n_groups, run_tiles;
    const int *n_items;
    const void *ridx_in;      // entries (EntryOf<CARRY>), null = identity (level 1)
    const StepDev *step;      // loss-guided: parent and ridx buffer come from the device
    const void *bufs[2];      // loss-guided: the two ridx buffers
    uint32_t *flags;          // [tiles][PT/32]
    int *tile_left;           // [tiles]
    int32_t *row_leaf;
    const int2 *qpair;
    const Group *groups;
    const int32_t *cut_ptr;
    unsigned long long *hist;  // [n_par][TB][2]
    long long TB;
    int hstride;
    unsigned long long *rows_ctr;  // profiling: algorithmic BITS moved (see below)
    int bits_parent_row;           // split symbol + ridx read, per scanned parent row
    int bits_built_row;            // packed row + qpair, per row of the built child
    int no_hist;                   // partition only (flags + left counts): hist_seg_kernel follows
    int rep_cap;                   // > 0: replicated low-cardinality bins (byte path, REP_CAP words)
};

// Warp-independent: each warp owns 64 rows of every tile of the item (no block barrier
// inside an item).  Per 64-row batch: (A) split symbol of each row -> left flags (ballot), the
// warp's left count into tile_left, the rows of the built child compacted into a warp-private
// list; (B) the listed rows' words accumulated by the warp (lane -> fixed word of the row).
template <bool WIDE, bool BYTE, bool SENT, bool CARRY>
__global__ void __launch_bounds__(H_THREADS, BYTE ? PH_MINB_BYTE : PH_MINB) part_hist_kernel(FusedArgs a) {
    using E = typename EntryOf<CARRY>::T;
    extern __shared__ int smem[];
    __shared__ int s_off[2049];
    __shared__ E s_rows[H_THREADS / 32][WROWS * (BYTE && !CARRY ? GBM_PH_TPS : 1)];
    __shared__ int s_rep[BYTE ? REP_F : 1];
    const E *rin = static_cast<const E *>(a.ridx_in);
    int first = a.first, run_tiles = a.n_items[2];
    if (a.step) {  // loss-guided step (n_par = 1): no items at all when nothing is expanded
        first = a.step->k;
        run_tiles = a.step->run_tiles;
        rin = a.step->in_buf < 0 ? nullptr : static_cast<const E *>(a.bufs[a.step->in_buf]);
    }
    const QM &qm = a.qm;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n_items = *a.n_items;
    E *wrows = s_rows[wid];
    for (int it = claim_item(const_cast<int *>(a.n_items) + 1); it < n_items;
         it = claim_item(const_cast<int *>(a.n_items) + 1)) {
        const int run = it / a.n_groups, g = it - run * a.n_groups;
        const int j = find_parent(a.run_base, a.n_par, run);
        const int k = first + j;
        const NodeDev nd = a.nodes[k];
        const int tb = a.tile_base[j];
        const int t0 = tb + (run - a.run_base[j]) * run_tiles, t1 = min(a.tile_base[j + 1], t0 + run_tiles);
        const long long seg_end = nd.start + nd.count;
        if (nd.state == GBM_NODE_LEAF) {  // rows stay in this leaf
            if (g != 0) continue;
            for (int t = t0; t < t1; ++t) {
                const long long base = nd.start + (long long)(t - tb) * PT;
                for (int i = threadIdx.x; i < PT; i += H_THREADS) {
                    const long long pos = base + i;
                    if (pos < seg_end) a.row_leaf[rin ? row_of(rin[pos]) : (uint32_t)pos] = k;
                }
            }
            continue;
        }
        const Group grp = a.groups[g];
        SmemHist h{smem, grp.bin_hi - grp.bin_lo, a.hstride};
        // lane -> (row slot, unit) of the group; units per row Ug <= 32 (plan_hist)
        const int Ug = grp.u_hi - grp.u_lo;
        const int rpp = 32 / Ug;                       // rows per pass
        const int my_r = lane < rpp * Ug ? lane / Ug : -1;
        const int my_u = grp.u_lo + (lane - (my_r < 0 ? 0 : my_r) * Ug);
        const int f_lo = grp.u_lo * qm.S;
        const int nf = min(grp.u_hi * qm.S, qm.F) - f_lo;
        const bool rep_on = BYTE && a.rep_cap > 0 && !a.no_hist && nf <= REP_F && rpp > 1;
        if (!a.no_hist) {
            smem_zero<WIDE>(h);
            load_group(qm, grp, a.cut_ptr, s_off);
        }
        if (rep_on && wid == 0) {  // the replica plan: s_rep[fl] = (word of copy 1) << 4 | log2 R
            int carry = 0;
            for (int c0 = 0; c0 < nf; c0 += 32) {
                const int fl = c0 + lane;
                int l = 0, nb = 0;
                if (fl < nf) {
                    nb = __ldg(a.cut_ptr + f_lo + fl + 1) - __ldg(a.cut_ptr + f_lo + fl);
                    l = rep_log2(nb, rpp);
                }
                const int w = ((1 << l) - 1) * nb;
                int x = w;
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                const int base = carry + x - w;
                if (base + w > a.rep_cap) l = 0;
                if (fl < nf) s_rep[fl] = ((h.nb + DUMMY_BINS + base) << 4) | l;
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
        }
        __syncthreads();
        // padding slots (symbol 0) add into a scratch bin of their own lane: one shared scratch bin
        // serialised them (Airline, 13 features: 3 of every 16 slots; levels 11.6 -> 9.9 ms/round)
        const int scratch = h.nb + lane;
        int off[4] = {scratch, scratch, scratch, scratch};
        unsigned agg = 0;
        if (BYTE) {
            unsigned lc = 0;
            if (my_r >= 0) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int f = my_u * 4 + jj;
                    if (f < qm.F) {
                        off[jj] = s_off[f - f_lo];
                        if (rep_on) {
                            const int rv = s_rep[f - f_lo], c = my_r & ((1 << (rv & 15)) - 1);
                            if (c) off[jj] = (rv >> 4) + (c - 1) * (s_off[f - f_lo + 1] - s_off[f - f_lo]);
                        }
                        if (s_off[f - f_lo + 1] - s_off[f - f_lo] <= AGG_MAX_BINS) lc |= 1u << jj;
                    }
                }
            }
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
                if (__any_sync(0xffffffffu, (lc >> jj) & 1u)) agg |= 1u << jj;
        }
        const bool build_left = nd.build_left != 0;
        const long long sw = qm.stride >> 5;
        const uint32_t mask = (1u << qm.bits) - 1u;
        unsigned long long bits_acc = 0;
        const bool no_hist = a.no_hist != 0;
        // TPS tiles per step (byte path: 2): the warp decides its 128 rows of each of the step's
        // tiles (8 entry loads, then 8 split-symbol gathers in flight per lane) and accumulates the
        // built rows of all of them as ONE list, so phase (B) runs on fuller batches.
        constexpr int TPS = BYTE && !CARRY ? GBM_PH_TPS : 1;  // (static shared memory budget: plan_hist)
        for (int t = t0; t < t1; t += TPS) {
            E row[TPS][4];
            uint32_t raw[TPS][4];
            int rem[TPS];
#pragma unroll
            for (int tt = 0; tt < TPS; ++tt) {
                const long long base = nd.start + (long long)(t + tt - tb) * PT + wid * WROWS;
                rem[tt] = t + tt < t1 ? (int)max(-1ll, min((long long)WROWS, seg_end - base)) : -1;
#pragma unroll
                for (int s2 = 0; s2 < 4; ++s2) {
                    const int q = s2 * 32 + lane;
                    if (q < rem[tt]) row[tt][s2] = rin ? rin[base + q] : make_entry<CARRY>((uint32_t)(base + q), a.qpair);
                    else row[tt][s2] = E{};
                }
            }
#pragma unroll
            for (int tt = 0; tt < TPS; ++tt)
#pragma unroll
                for (int s2 = 0; s2 < 4; ++s2) {
                    const uint32_t ro = row_of(row[tt][s2]);
                    raw[tt][s2] = s2 * 32 + lane >= rem[tt] ? 0u
                                  : qm.dbits ? __ldg(qm.dbits + (ro >> 5))
                                             : split_symbol(qm, ro, nd.f);
                }
            // (A) partition flags for the warp's 128 rows of each tile (4 per lane)
            int nbuild = 0;
            const uint32_t ltm = (1u << lane) - 1u;
#pragma unroll
            for (int tt = 0; tt < TPS; ++tt) {
                if (rem[tt] < 0 && tt > 0) break;  // warp-uniform
                int nleft = 0;
#pragma unroll
                for (int s2 = 0; s2 < 4; ++s2) {
                    const bool valid = s2 * 32 + lane < rem[tt];
                    const uint32_t ro = row_of(row[tt][s2]);
                    const uint32_t rv = raw[tt][s2];
                    const bool left = valid && (qm.dbits ? ((rv >> (ro & 31)) & 1u) != 0
                                                         : ((int)rv == qm.B ? (nd.dl != 0) : ((int)rv <= nd.b)));
                    const uint32_t lw = __ballot_sync(0xffffffffu, left);
                    const uint32_t bw = __ballot_sync(0xffffffffu, valid && (left == build_left));
                    if (g == 0 && lane == 0) a.flags[(long long)(t + tt) * (PT / 32) + wid * 4 + s2] = lw;
                    nleft += __popc(lw);
                    if ((bw >> lane) & 1u) wrows[nbuild + __popc(bw & ltm)] = row[tt][s2];
                    nbuild += __popc(bw);
                }
                if (g == 0 && lane == 0) {
                    if (nleft) atomicAdd(a.tile_left + t + tt, nleft);
                    if (a.rows_ctr) bits_acc += (unsigned long long)max(0, rem[tt]) * a.bits_parent_row;
                }
            }
            if (g == 0 && lane == 0 && a.rows_ctr && !a.no_hist)
                bits_acc += (unsigned long long)nbuild * a.bits_built_row;
            __syncwarp();
            if (no_hist) continue;  // partition only
            // (B) histogram of the listed rows
            if (BYTE && agg) {  // warp-uniform loop (aggregated slots use warp intrinsics)
                for (int rb = 0; rb < nbuild; rb += 4 * rpp) {
                    uint32_t wd[4];
                    int2 qq[4];
                    bool ok[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int rr = rb + my_r + i * rpp;
                        ok[i] = my_r >= 0 && rr < nbuild;
                        const E ew = wrows[ok[i] ? rr : 0];
                        wd[i] = __ldg(qm.P + row_of(ew) * sw + (ok[i] ? my_u : grp.u_lo));
                        qq[i] = entry_q(ew, a.qpair);
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i) byte_word_add<WIDE, SENT>(h, off, agg, wd[i], qq[i], ok[i], qm.B);
                }
            } else if (BYTE) {
                if (my_r >= 0) {
                    int rr = my_r;
                    for (; rr + (PH_UNR - 1) * rpp < nbuild; rr += PH_UNR * rpp) {
                        E ew[PH_UNR];
                        uint32_t wd[PH_UNR];
                        int2 qq[PH_UNR];
#pragma unroll
                        for (int i = 0; i < PH_UNR; ++i) ew[i] = wrows[rr + i * rpp];
#pragma unroll
                        for (int i = 0; i < PH_UNR; ++i) {
                            wd[i] = __ldg(qm.P + row_of(ew[i]) * sw + my_u);
                            qq[i] = entry_q(ew[i], a.qpair);
                        }
#pragma unroll
                        for (int i = 0; i < PH_UNR; ++i)
#pragma unroll
                            for (int jj = 0; jj < 4; ++jj) {
                                const int sy = (wd[i] >> (8 * jj)) & 255;
                                if (!SENT || sy != qm.B) hist_add<WIDE>(h.base, h.hstride, off[jj] + sy, qq[i]);
                            }
                    }
                    for (; rr < nbuild; rr += rpp) {
                        const E ea = wrows[rr];
                        const uint32_t wa = __ldg(qm.P + row_of(ea) * sw + my_u);
                        const int2 qa = entry_q(ea, a.qpair);
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
                            const int sa = (wa >> (8 * jj)) & 255;
                            if (!SENT || sa != qm.B) hist_add<WIDE>(h.base, h.hstride, off[jj] + sa, qa);
                        }
                    }
                }
            } else if (my_r >= 0) {
                {
                    const int f0 = my_u * qm.S;
                    const int ns = min(qm.S, qm.F - f0);
                    const long long boff = (long long)f0 * qm.bits;
                    int rr = my_r;
                    for (; rr + 3 * rpp < nbuild; rr += 4 * rpp) {  // four rows in flight
                        uint32_t win[4];
                        int2 qq[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const E ea = wrows[rr + i * rpp];
                            qq[i] = entry_q(ea, a.qpair);
                            win[i] = get_bits(qm.P, (long long)row_of(ea) * qm.stride + boff, ns * qm.bits);
                        }
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            for (int jj = 0; jj < ns; ++jj) {
                                const int sy = (int)((win[i] >> (jj * qm.bits)) & mask);
                                if (sy == qm.B) continue;
                                hist_add<WIDE>(h.base, h.hstride, s_off[f0 + jj - f_lo] + sy, qq[i]);
                            }
                    }
                    for (; rr < nbuild; rr += rpp) {
                        const E ea = wrows[rr];
                        const uint32_t ra = row_of(ea);
                        const int2 q = entry_q(ea, a.qpair);
                        const uint32_t win =
                            get_bits(qm.P, (long long)ra * qm.stride + (long long)f0 * qm.bits, ns * qm.bits);
                        for (int jj = 0; jj < ns; ++jj) {
                            const int sy = (int)((win >> (jj * qm.bits)) & mask);
                            if (sy == qm.B) continue;
                            hist_add<WIDE>(h.base, h.hstride, s_off[f0 + jj - f_lo] + sy, q);
                        }
                    }
                }
            }
            __syncwarp();
        }
        if (bits_acc) atomicAdd(a.rows_ctr, bits_acc);
        __syncthreads();
        if (rep_on) {  // fold the copies into copy 0 (a row adds into one copy: same int32 bound)
            for (int fl = 0; fl < nf; ++fl) {
                const int rv = s_rep[fl], l = rv & 15;
                if (!l) continue;
                const int nb = s_off[fl + 1] - s_off[fl];
                for (int b = threadIdx.x; b < nb; b += H_THREADS)
#pragma unroll
                    for (int ch = 0; ch < (WIDE ? 4 : 2); ++ch) {
                        int *hc = smem + ch * h.hstride;
                        int v = hc[s_off[fl] + b];
                        for (int c = 1; c < (1 << l); ++c) v += hc[(rv >> 4) + (c - 1) * nb + b];
                        hc[s_off[fl] + b] = v;
                    }
            }
            __syncthreads();
        }
        if (!no_hist) smem_flush<WIDE>(h, a.hist + ((long long)j * a.TB + grp.bin_lo) * 2);
        __syncthreads();
    }
}

// ============================================================== warp-specialised levels
// GBM_OPT_LEVEL_HIST = 3: the fused level kernel with the partition and the histogram in
// different warps.  ncu on part_hist_kernel (profiles/r02): at the deep levels ~30 % of the stall
// samples wait on the split-symbol gather of the partition phase (ridx -> symbol: two dependent
// DRAM latencies per tile) and ~14 % on the built rows' word gathers, with each warp alternating
// both phases.  Here WS_NP producer warps decide tile t + 1 (16 rows in flight per lane) while the
// consumer warps accumulate tile t from the producers' lists: named barriers full[b] / empty[b]
// hand the double-buffered lists over.  Compact layout, byte symbols, one feature group.
constexpr int WS_NP = 4;               // producer warps
constexpr int WS_NC = H_THREADS / 32 - WS_NP;  // consumer warps
constexpr int WS_PROWS = PT / WS_NP;   // rows per producer warp per tile (512)

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <bool WIDE, bool SENT>
__global__ void __launch_bounds__(H_THREADS, 2) part_hist_ws_kernel(FusedArgs a) {
    extern __shared__ int smem[];
    __shared__ int s_off[2049];
    __shared__ uint32_t s_list[2][WS_NP][WS_PROWS];
    __shared__ int s_cnt[2][WS_NP];
    const QM &qm = a.qm;
    const uint32_t *rin = static_cast<const uint32_t *>(a.ridx_in);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool producer = wid < WS_NP;
    const int n_items = *a.n_items;
    const uint32_t ltm = (1u << lane) - 1u;
    for (int it = claim_item(const_cast<int *>(a.n_items) + 1); it < n_items;
         it = claim_item(const_cast<int *>(a.n_items) + 1)) {
        const int run = it;
        const int j = find_parent(a.run_base, a.n_par, run);
        const int k = a.first + j;
        const NodeDev nd = a.nodes[k];
        const int tb = a.tile_base[j];
        const int rt = a.n_items[2], t0 = tb + (run - a.run_base[j]) * rt, t1 = min(a.tile_base[j + 1], t0 + rt);
        const long long seg_end = nd.start + nd.count;
        if (nd.state == GBM_NODE_LEAF) {  // rows stay in this leaf
            for (int t = t0; t < t1; ++t) {
                const long long base = nd.start + (long long)(t - tb) * PT;
                for (int i = threadIdx.x; i < PT; i += H_THREADS) {
                    const long long pos = base + i;
                    if (pos < seg_end) a.row_leaf[rin ? rin[pos] : (uint32_t)pos] = k;
                }
            }
            continue;
        }
        const Group grp = a.groups[0];
        SmemHist h{smem, grp.bin_hi - grp.bin_lo, a.hstride};
        smem_zero<WIDE>(h);
        load_group(qm, grp, a.cut_ptr, s_off);
        __syncthreads();
        const bool build_left = nd.build_left != 0;
        const int nt = t1 - t0;
        if (producer) {
            unsigned long long bits_acc = 0;
            for (int i = 0; i < nt; ++i) {
                const int t = t0 + i, b = i & 1;
                if (i >= 2) named_sync(3 + b, H_THREADS);  // consumers are done with buffer b
                const long long base = nd.start + (long long)(t - tb) * PT + wid * WS_PROWS;
                uint32_t row[16];
                bool left[16];
#pragma unroll
                for (int s2 = 0; s2 < 16; ++s2) {
                    const long long pos = base + s2 * 32 + lane;
                    row[s2] = pos < seg_end ? (rin ? __ldg(rin + pos) : (uint32_t)pos) : 0u;
                }
#pragma unroll
                for (int s2 = 0; s2 < 16; ++s2) left[s2] = base + s2 * 32 + lane < seg_end && goes_left(qm, nd, row[s2]);
                int nleft = 0, nbuild = 0;
                uint32_t *lst = s_list[b][wid];
#pragma unroll
                for (int s2 = 0; s2 < 16; ++s2) {
                    const bool valid = base + s2 * 32 + lane < seg_end;
                    const uint32_t lw2 = __ballot_sync(0xffffffffu, valid && left[s2]);
                    const uint32_t bw = __ballot_sync(0xffffffffu, valid && (left[s2] == build_left));
                    if (lane == 0) a.flags[(long long)t * (PT / 32) + wid * 16 + s2] = lw2;
                    nleft += __popc(lw2);
                    if ((bw >> lane) & 1u) lst[nbuild + __popc(bw & ltm)] = row[s2];
                    nbuild += __popc(bw);
                }
                if (lane == 0) {
                    s_cnt[b][wid] = nbuild;
                    if (nleft) atomicAdd(a.tile_left + t, nleft);
                    if (a.rows_ctr) bits_acc += (unsigned long long)nbuild * a.bits_built_row;
                }
                __threadfence_block();
                named_arrive(1 + b, H_THREADS);  // list b of tile t is ready
            }
            for (int i = max(0, nt - 2); i < nt; ++i) named_sync(3 + (i & 1), H_THREADS);  // balance the empties
            if (lane == 0 && bits_acc) atomicAdd(a.rows_ctr, bits_acc);
        } else {
            const int cw = wid - WS_NP;
            const int Ug = grp.u_hi - grp.u_lo;
            const int rpp = 32 / Ug;
            const int my_r = lane < rpp * Ug ? lane / Ug : -1;
            const int my_u = grp.u_lo + (lane - (my_r < 0 ? 0 : my_r) * Ug);
            const int f_lo = grp.u_lo * qm.S;
            int off[4] = {h.nb, h.nb, h.nb, h.nb};
            if (my_r >= 0) {
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int f = my_u * 4 + jj;
                    if (f < qm.F) off[jj] = s_off[f - f_lo];
                }
            }
            const long long sw = qm.stride >> 5;
            for (int i = 0; i < nt; ++i) {
                const int b = i & 1;
                named_sync(1 + b, H_THREADS);  // the producers' lists of this tile
                int pre[WS_NP + 1];
                pre[0] = 0;
#pragma unroll
                for (int w = 0; w < WS_NP; ++w) pre[w + 1] = pre[w] + s_cnt[b][w];
                const int N = pre[WS_NP];
                const int k0 = (int)((long long)cw * N / WS_NC), k1 = (int)((long long)(cw + 1) * N / WS_NC);
                auto entry = [&](int kk) -> uint32_t {
                    int w = 0;
#pragma unroll
                    for (int q = 1; q < WS_NP; ++q) w += kk >= pre[q];
                    return s_list[b][w][kk - pre[w]];
                };
                if (my_r >= 0) {
                    int rr = k0 + my_r;
                    for (; rr + (PH_UNR - 1) * rpp < k1; rr += PH_UNR * rpp) {
                        uint32_t wd[PH_UNR];
                        int2 qq[PH_UNR];
#pragma unroll
                        for (int u = 0; u < PH_UNR; ++u) {
                            const uint32_t r = entry(rr + u * rpp);
                            wd[u] = __ldg(qm.P + r * sw + my_u);
                            qq[u] = __ldg(a.qpair + r);
                        }
#pragma unroll
                        for (int u = 0; u < PH_UNR; ++u)
#pragma unroll
                            for (int jj = 0; jj < 4; ++jj) {
                                const int sy = (wd[u] >> (8 * jj)) & 255;
                                if (!SENT || sy != qm.B) hist_add<WIDE>(h.base, h.hstride, off[jj] + sy, qq[u]);
                            }
                    }
                    for (; rr < k1; rr += rpp) {
                        const uint32_t r = entry(rr);
                        const uint32_t wa = __ldg(qm.P + r * sw + my_u);
                        const int2 qa = __ldg(a.qpair + r);
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
                            const int sa = (wa >> (8 * jj)) & 255;
                            if (!SENT || sa != qm.B) hist_add<WIDE>(h.base, h.hstride, off[jj] + sa, qa);
                        }
                    }
                }
                named_arrive(3 + b, H_THREADS);  // buffer b may be refilled
            }
        }
        __syncthreads();
        smem_flush<WIDE>(h, a.hist + ((long long)j * a.TB + grp.bin_lo) * 2);
        __syncthreads();
    }
}

// ============================================================== shuffle-fed bank-column levels
// The fused level kernel for byte symbols with every feature in one group (F <= 32, rows of U
// whole words): the partition phase is part_hist_kernel's; the built rows are fetched exactly as
// there -- lane (row slot r, word w) loads word w of its row, 32 / U rows per load instruction --
// but accumulated into the conflict-free bank-column histogram (word = bin * 32 + lane): lane
// (copy c, feature f) takes its symbol from lane (r, f / 4) with one shuffle and the row's pair
// with two, then adds into its own bank.  The compact layout's random-bank ATOMS cost ~3.4
// wavefronts each (ncu: 70 % of the level kernel's atomic wavefronts were conflict replays);
// these cost one.  The sentinel (B < 256) lands in a bin >= n_bins(f) of its column, never
// flushed (as in the lean root kernel).
template <bool WIDE>
__global__ void __launch_bounds__(H_THREADS, WIDE ? 1 : 2) part_hist_sb_kernel(FusedArgs a) {
    extern __shared__ int smem[];
    __shared__ uint32_t s_rows[H_THREADS / 32][WROWS];
    constexpr int CH = WIDE ? 4 : 2;
    const QM &qm = a.qm;
    const uint32_t *rin = static_cast<const uint32_t *>(a.ridx_in);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n_items = *a.n_items;
    uint32_t *wrows = s_rows[wid];
    const int F = qm.F, U = (F + 3) >> 2;        // words per row (stride == U words)
    const int rpp = 32 / U;                      // rows per load instruction
    const int lr = lane / U, lw = lane - lr * U; // loading role: row slot, word
    const bool load_on = lr < rpp;
    const int R = 32 / F;                        // rows per accumulate step (copies)
    const int cc = lane / F, cf = lane - cc * F; // accumulating role: copy, feature
    const bool acc_on = cc < R;
    const int src_w = cf >> 2, sh = 8 * (cf & 3);
    const unsigned hb = smem_u32(smem) + 4u * lane;
    const ColGroup cg{0, F};
    for (int it = claim_item(const_cast<int *>(a.n_items) + 1); it < n_items;
         it = claim_item(const_cast<int *>(a.n_items) + 1)) {
        const int run = it;
        const int j = find_parent(a.run_base, a.n_par, run);
        const int k = a.first + j;
        const NodeDev nd = a.nodes[k];
        const int tb = a.tile_base[j];
        const int rt = a.n_items[2], t0 = tb + (run - a.run_base[j]) * rt, t1 = min(a.tile_base[j + 1], t0 + rt);
        const long long seg_end = nd.start + nd.count;
        if (nd.state == GBM_NODE_LEAF) {  // rows stay in this leaf
            for (int t = t0; t < t1; ++t) {
                const long long base = nd.start + (long long)(t - tb) * PT;
                for (int i = threadIdx.x; i < PT; i += H_THREADS) {
                    const long long pos = base + i;
                    if (pos < seg_end) a.row_leaf[rin ? rin[pos] : (uint32_t)pos] = k;
                }
            }
            continue;
        }
        for (int i = threadIdx.x; i < CH * COLB_STRIDE; i += H_THREADS) smem[i] = 0;
        __syncthreads();
        const bool build_left = nd.build_left != 0;
        unsigned long long bits_acc = 0;
        for (int t = t0; t < t1; ++t) {
            const long long base = nd.start + (long long)(t - tb) * PT + wid * WROWS;
            // (A) partition flags for the warp's 128 rows (as part_hist_kernel)
            uint32_t row[4], bw[4];
            int nleft = 0;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const long long pos = base + s2 * 32 + lane;
                row[s2] = pos < seg_end ? (rin ? rin[pos] : (uint32_t)pos) : 0u;
            }
            bool left[4];
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) left[s2] = base + s2 * 32 + lane < seg_end && goes_left(qm, nd, row[s2]);
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const bool valid = base + s2 * 32 + lane < seg_end;
                const uint32_t lw2 = __ballot_sync(0xffffffffu, valid && left[s2]);
                bw[s2] = __ballot_sync(0xffffffffu, valid && (left[s2] == build_left));
                if (lane == 0) a.flags[(long long)t * (PT / 32) + wid * 4 + s2] = lw2;
                nleft += __popc(lw2);
            }
            int nbuild = 0;
            const uint32_t ltm = (1u << lane) - 1u;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                if ((bw[s2] >> lane) & 1u) wrows[nbuild + __popc(bw[s2] & ltm)] = row[s2];
                nbuild += __popc(bw[s2]);
            }
            if (lane == 0) {
                if (nleft) atomicAdd(a.tile_left + t, nleft);
                if (a.rows_ctr) {
                    const long long nv = max(0ll, min((long long)WROWS, seg_end - base));
                    bits_acc += (unsigned long long)nv * a.bits_parent_row + (unsigned long long)nbuild * a.bits_built_row;
                }
            }
            __syncwarp();
            // (B) the listed rows: PH_UNR load groups in flight, then shuffle + conflict-free ATOMS
            for (int rb = 0; rb < nbuild; rb += PH_UNR * rpp) {
                uint32_t wd[PH_UNR];
                int2 qq[PH_UNR];
#pragma unroll
                for (int u = 0; u < PH_UNR; ++u) {
                    const int rr = rb + u * rpp + lr;
                    const bool ok = load_on && rr < nbuild;
                    const uint32_t r = ok ? wrows[rr] : 0u;
                    wd[u] = ok ? __ldg(qm.P + (size_t)r * U + lw) : 0u;
                    qq[u] = ok ? __ldg(a.qpair + r) : make_int2(0, 0);
                }
#pragma unroll
                for (int u = 0; u < PH_UNR; ++u) {
                    for (int s0 = 0; s0 < rpp; s0 += R) {  // R rows per step (warp-uniform)
                        const int rs = s0 + (acc_on ? cc : 0);
                        const int src = rs * U;
                        const uint32_t w = __shfl_sync(0xffffffffu, wd[u], src + src_w);
                        const int qx = __shfl_sync(0xffffffffu, qq[u].x, src);
                        const int qy = __shfl_sync(0xffffffffu, qq[u].y, src);
                        if (acc_on && rs < rpp && rb + u * rpp + rs < nbuild) {
                            const unsigned addr = hb + (((w >> sh) & 255u) << 7);
                            if (WIDE) {
                                asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(qx & 0x7fff) : "memory");
                                asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr + 4 * COLB_STRIDE), "r"(qy & 0x7fff) : "memory");
                                asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr + 8 * COLB_STRIDE), "r"(qx >> 15) : "memory");
                                asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr + 12 * COLB_STRIDE), "r"(qy >> 15) : "memory");
                            } else {
                                asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr), "r"(qx) : "memory");
                                asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(addr + 4 * COLB_STRIDE), "r"(qy) : "memory");
                            }
                        }
                    }
                }
            }
            __syncwarp();
        }
        if (bits_acc) atomicAdd(a.rows_ctr, bits_acc);
        __syncthreads();
        col_flush<WIDE>(smem, COLB_STRIDE, cg, a.cut_ptr, a.hist + (long long)j * a.TB * 2);
        __syncthreads();
    }
}

// ============================================================== segment histograms
// With several shared-memory feature groups (wide data: Epsilon 63, Bosch ~40, YearMSD 3) the
// fused kernel would repeat the partition of every parent row once per group.  Instead the level
// is partitioned once (fused kernel with no_hist), scanned and scattered, and the built
// children's contiguous entry segments are then histogrammed group by group.
struct SegArgs {
    QM qm;
    const NodeDev *nodes;
    int first, n_par;
    const void *ridx;         // the level's scattered entries (EntryOf<CARRY>)
    const int2 *qpair;
    const int *seg_base;      // [n_par + 1] first chunk of each parent's built child
    const int *n_items;       // chunks x groups
    int chunk, n_groups;
    const Group *groups;
    const int32_t *cut_ptr;
    unsigned long long *hist;  // [n_par][TB][2]
    long long TB;
    int hstride;
    unsigned long long *rows_ctr;
};

template <bool WIDE, bool BYTE, bool SENT, bool CARRY>
__global__ void __launch_bounds__(H_THREADS, GBM_HR_MINB) hist_seg_kernel(SegArgs a) {
    using E = typename EntryOf<CARRY>::T;
    extern __shared__ int smem[];
    __shared__ int s_off[2049];
    const QM &qm = a.qm;
    const E *rin = static_cast<const E *>(a.ridx);
    const int n_items = *a.n_items;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int ch = it / a.n_groups, g = it - ch * a.n_groups;
        const int j = find_parent(a.seg_base, a.n_par, ch);
        const int k = a.first + j;
        const NodeDev cd = a.nodes[a.nodes[k].build_left ? 2 * k + 1 : 2 * k + 2];
        const long long start = cd.start + (long long)(ch - a.seg_base[j]) * a.chunk;
        const int len = (int)min((long long)a.chunk, cd.start + cd.count - start);
        const Group grp = a.groups[g];
        SmemHist h{smem, grp.bin_hi - grp.bin_lo, a.hstride};
        if (a.rows_ctr && g == 0 && threadIdx.x == 0) atomicAdd(a.rows_ctr, (unsigned long long)len);
        smem_zero<WIDE>(h);
        load_group(qm, grp, a.cut_ptr, s_off);
        __syncthreads();
        ByteLane L = BYTE ? byte_lane(qm, grp, s_off, h.nb) : ByteLane{};
        long long tg = 0, th = 0;
        const E *rp = rin + start;
        accumulate<WIDE, BYTE, SENT>(qm, grp, s_off, h, a.qpair, [&](int r) { return row_of(rp[r]); }, len, L,
                                     &tg, &th, false);
        __syncthreads();
        smem_flush<WIDE>(h, a.hist + ((long long)j * a.TB + grp.bin_lo) * 2);
        __syncthreads();
    }
}

// ============================================================== bank-column histograms
// Feature-per-lane layout (GBM_OPT_HIST_LAYOUT = 2, when every feature's bins fit a column): the
// shared-memory word of (bin b, column c) is b*32 + c, so every update a lane makes falls into
// bank c and no ATOMS can conflict -- with random bins the compact layout costs ~3.7 bank
// wavefronts per 32-lane atomic (ncu: 74.9M wavefronts vs 20.1M ideal on the Higgs root pass).
// Measured: conflict-free, but one row per warp instruction costs ~63 instructions per row
// (696M vs 111M on the Higgs root pass, 1.19 ms vs 0.33 ms), so it is not the default; it needs
// a feature-major source staged by TMA to pay off.
// A group holds Fg <= 32 features; a warp processes R = 32/Fg rows per step: lane = copy*Fg +
// feature, the R copies of a feature live in different columns and are merged by the flush.
// byte symbols: every feature has <= 256 bins, the channel stride is the constant 256*32 words
constexpr int COLB_UR = 4;   // rows in flight per lane in the byte column kernels (16 measured slower)
template <bool WIDE>
__device__ __forceinline__ void col_add(int *hs, int cstride, int word, int2 q) {
    if (WIDE) {
        atomicAdd(hs + word, q.x & 0x7fff);
        atomicAdd(hs + cstride + word, q.y & 0x7fff);
        atomicAdd(hs + 2 * cstride + word, q.x >> 15);
        atomicAdd(hs + 3 * cstride + word, q.y >> 15);
    } else {
        atomicAdd(hs + word, q.x);
        atomicAdd(hs + cstride + word, q.y);
    }
}

struct ColLane {
    int copy, R, Fg;
    bool active;
    long long bitoff;  // f * bits
};

__device__ __forceinline__ ColLane col_lane(const QM &qm, const ColGroup &cg) {
    ColLane L;
    const int lane = threadIdx.x & 31;
    L.Fg = cg.f_hi - cg.f_lo;
    L.R = 32 / L.Fg;
    L.copy = lane / L.Fg;
    L.active = lane < L.R * L.Fg;
    L.bitoff = (long long)(cg.f_lo + (L.active ? lane % L.Fg : 0)) * qm.bits;
    return L;
}

struct ColRangeArgs {
    int tma;  // staged root: TMA bulk copies of whole rows (set by the host when applicable)
    QM qm;
    const int2 *qpair;
    const uint32_t *ridx;        // null = identity rows
    long long n_sel;
    int chunk, n_groups;
    const ColGroup *groups;
    const int32_t *cut_ptr;
    unsigned long long *hist;    // [TB][2]
    unsigned long long *totals;  // [2] or null
    unsigned long long *rows_ctr;
    int cstride;                 // words per channel = rows * 32
};

template <bool WIDE, bool BYTE>
__global__ void __launch_bounds__(H_THREADS) hist_col_range_kernel(ColRangeArgs a) {
    extern __shared__ int smem[];
    __shared__ long long s_red[2 * H_THREADS / 32];
    const QM &qm = a.qm;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = H_THREADS / 32;
    const int n_items = (int)(((a.n_sel + a.chunk - 1) / a.chunk) * a.n_groups);
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int g = it % a.n_groups;
        const long long start = (long long)(it / a.n_groups) * a.chunk;
        const long long end = min(a.n_sel, start + a.chunk);
        const ColGroup cg = a.groups[g];
        for (int i = threadIdx.x; i < (WIDE ? 4 : 2) * a.cstride; i += H_THREADS) smem[i] = 0;
        if (a.rows_ctr && g == 0 && threadIdx.x == 0) atomicAdd(a.rows_ctr, (unsigned long long)(end - start));
        __syncthreads();
        const ColLane L = col_lane(qm, cg);
        const bool tot = a.totals && g == 0 && L.active && (lane % L.Fg) == 0;
        long long tg = 0, th = 0;
        const long long step = (long long)NW * L.R;
        const uint8_t *Pb = reinterpret_cast<const uint8_t *>(qm.P) + (L.bitoff >> 3);
        const unsigned sb = (unsigned)(qm.stride >> 3);  // bytes per row (BYTE)
        const bool chk = qm.B < 256;
        for (long long r0 = start + (long long)wid * L.R + L.copy; r0 < end; r0 += 4 * step) {
            uint32_t sym[4];
            int2 q[4];
            bool ok[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long r = r0 + u * step;
                ok[u] = L.active && r < end;
                const uint32_t row = ok[u] ? (a.ridx ? __ldg(a.ridx + r) : (uint32_t)r) : 0u;
                if (BYTE) sym[u] = ok[u] ? __ldg(Pb + (size_t)row * sb) : 0u;
                else sym[u] = ok[u] ? get_bits(qm.P, (long long)row * qm.stride + L.bitoff, qm.bits) : 0u;
                q[u] = ok[u] ? __ldg(a.qpair + row) : make_int2(0, 0);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (BYTE) {
                    if (ok[u] && (!chk || (int)sym[u] != qm.B)) col_add_b<WIDE>(smem, (int)(sym[u] << 5) + lane, q[u]);
                } else if (ok[u] && (int)sym[u] != qm.B) {
                    col_add<WIDE>(smem, a.cstride, (int)sym[u] * 32 + lane, q[u]);
                }
                if (tot && ok[u]) {
                    tg += q[u].x;
                    th += q[u].y;
                }
            }
        }
        if (a.totals && g == 0) block_totals(tg, th, s_red, a.totals);
        __syncthreads();
        col_flush<WIDE>(smem, a.cstride, cg, a.cut_ptr, a.hist);
        __syncthreads();
    }
}

// Lean byte-symbol column kernel (bits == 8): branch-free inner loop.  Lanes beyond R*Fg write
// into columns the flush never reads, the sentinel symbol (B < 256) lands in a bin >= n_bins(f)
// of its own column (never flushed), and the ragged tail is masked by a zero gradient pair, so
// every ATOMS is unconditional and conflict-free.  Root totals come from sum_qpair_kernel.
template <bool WIDE, bool IDENT>
__global__ void __launch_bounds__(H_THREADS) hist_colb_range_kernel(ColRangeArgs a) {
    extern __shared__ int smem[];
    const QM &qm = a.qm;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = H_THREADS / 32;
    const int n_items = (int)(((a.n_sel + a.chunk - 1) / a.chunk) * a.n_groups);
    const unsigned sb = (unsigned)(qm.stride >> 3);  // bytes per row
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int g = it % a.n_groups;
        const long long start = (long long)(it / a.n_groups) * a.chunk;
        const long long end = min(a.n_sel, start + a.chunk);
        const ColGroup cg = a.groups[g];
        for (int i = threadIdx.x; i < (WIDE ? 4 : 2) * COLB_STRIDE; i += H_THREADS) smem[i] = 0;
        if (a.rows_ctr && g == 0 && threadIdx.x == 0) atomicAdd(a.rows_ctr, (unsigned long long)(end - start));
        __syncthreads();
        const int Fg = cg.f_hi - cg.f_lo, R = 32 / Fg;
        const int copy = min(lane / Fg, R - 1);
        const uint8_t *Pf = reinterpret_cast<const uint8_t *>(qm.P) + (cg.f_lo + lane % Fg);
        const int step = NW * R;
        const long long last = end - 1;
        // COLB_UR rows in flight per lane: each load moves one row's byte, so memory-level
        // parallelism must come from many independent rows (Little's law)
        for (long long r0 = start + (long long)wid * R + copy; r0 < end; r0 += COLB_UR * step) {
            uint32_t row[COLB_UR];
            bool ok[COLB_UR];
#pragma unroll
            for (int u = 0; u < COLB_UR; ++u) {
                const long long r = r0 + u * step;
                ok[u] = r < end;
                const long long rc = ok[u] ? r : last;
                row[u] = IDENT ? (uint32_t)rc : __ldg(a.ridx + rc);
            }
            uint32_t sym[COLB_UR];
            int2 q[COLB_UR];
#pragma unroll
            for (int u = 0; u < COLB_UR; ++u) {
                sym[u] = __ldg(Pf + (size_t)row[u] * sb);
                q[u] = __ldg(a.qpair + row[u]);
            }
#pragma unroll
            for (int u = 0; u < COLB_UR; ++u) {
                const int2 qq = ok[u] ? q[u] : make_int2(0, 0);
                col_add_b<WIDE>(smem, (int)(sym[u] << 5) + lane, qq);
            }
        }
        __syncthreads();
        col_flush<WIDE>(smem, COLB_STRIDE, cg, a.cut_ptr, a.hist);
        __syncthreads();
    }
}

// root totals T = sum over rows of (q_g, q_h) (InitRoot), for the lean byte kernel
__global__ void __launch_bounds__(256) sum_qpair_kernel(const int2 *__restrict__ q, long long n,
                                                        unsigned long long *__restrict__ out) {
    __shared__ long long red[2 * 256 / 32];
    long long tg = 0, th = 0;
    for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
        const int2 v = __ldg(q + i);
        tg += v.x;
        th += v.y;
    }
    block_totals(tg, th, red, out);
}

// ============================================================== staged bank-column histograms
// GBM_OPT_HIST_LAYOUT = 3 (byte symbols, narrow): every warp stages 32 rows at a time into shared
// memory with coalesced 4-byte loads (the group's words of each row) plus the rows' gradient
// pairs, then lane = (copy, feature column) reads its byte with a conflict-free LDS.U8, the pair
// with a broadcast LDS.64, and updates its own bank column with conflict-free ATOMS.
// Per row (Higgs): ~4.6 L1 data-pipe wavefronts vs ~7.8 for the compact layout.
constexpr int CS_WMAX = 8;                     // words per staged row (<= 32 byte features)
struct CsWarp {
    uint32_t w[32 * CS_WMAX];                  // staged rows: [32][Wg] words
    int2 q[32];                                // their gradient pairs
};

// Stage rows row_i (i < 32, valid_i) of group words [u_lo, u_lo+Wg) and their pairs; then add.
// accumulate a staged batch (R rows per warp instruction, lane = copy * Fg + feature)
__device__ __forceinline__ void cs_consume(const CsWarp &st, int *hs, int Wg, int Fg, int R, int copy, int nrows) {
    const int lane = threadIdx.x & 31;
    const uint8_t *sb = reinterpret_cast<const uint8_t *>(st.w);
    const int col = lane % Fg;  // byte of the feature within the staged row
    const int rowbytes = Wg * 4;
#pragma unroll 4
    for (int i0 = 0; i0 < nrows; i0 += R) {
        const int i = min(i0 + copy, 31);
        const int sym = sb[i * rowbytes + col];
        const int2 q = (i0 + copy < nrows) ? st.q[i] : make_int2(0, 0);
        col_add_b<false>(hs, (sym << 5) + lane, q);
    }
}

template <class RowF, class QF>
__device__ __forceinline__ void cs_batch(const QM &qm, CsWarp &st, int *hs, int u_lo, int Wg, int Fg, int R, int copy,
                                         int nrows, RowF rowf, QF qf) {
    const int lane = threadIdx.x & 31;
    const long long sw = qm.stride >> 5;
    // pairs: lane i stages row i
    {
        const bool ok = lane < nrows;
        const int2 q = ok ? qf(lane) : make_int2(0, 0);
        st.q[lane] = q;
    }
    // words: flattened (row, word) over 32*Wg slots, consecutive lanes -> consecutive words
    for (int idx = lane; idx < 32 * Wg; idx += 32) {
        const int i = idx / Wg, w = idx - i * Wg;
        st.w[idx] = i < nrows ? __ldg(qm.P + (long long)rowf(i) * sw + u_lo + w) : 0u;
    }
    __syncwarp();
    cs_consume(st, hs, Wg, Fg, R, copy, nrows);
    __syncwarp();
}

// One feature per lane (groups of 17..32 byte features, WG = 5..8 words): lane f adds byte f of
// each staged row into its own bank column.  Compile-time row pitch, no per-row bounds logic
// (rows past nrows are staged as symbol 0 with a zero pair: adds of 0), the pair broadcast from
// shared memory -- about 5 instructions and 4 conflict-free wavefronts per row.
template <int WG>
__device__ __forceinline__ void cs_consume_r1(const CsWarp &st, int *hs, int Fg) {
    const int lane = threadIdx.x & 31;
    const uint8_t *sb = reinterpret_cast<const uint8_t *>(st.w) + lane;
    int *hg = hs + lane, *hh = hs + COLB_STRIDE + lane;
    if (lane < Fg) {
#pragma unroll 8
        for (int i = 0; i < 32; ++i) {
            const int sym = sb[i * WG * 4];
            const int2 q = st.q[i];
            atomicAdd(hg + (sym << 5), q.x);
            atomicAdd(hh + (sym << 5), q.y);
        }
    }
}

template <int WG, class RowF, class QF>
__device__ __forceinline__ void cs_batch_r1(const QM &qm, CsWarp &st, int *hs, int u_lo, int Fg, int nrows, RowF rowf,
                                            QF qf) {
    const int lane = threadIdx.x & 31;
    const long long sw = qm.stride >> 5;
    st.q[lane] = lane < nrows ? qf(lane) : make_int2(0, 0);
    uint32_t v[WG];
#pragma unroll
    for (int k = 0; k < WG; ++k) {
        const int idx = lane + 32 * k;
        const int i = idx / WG, w = idx - i * WG;
        v[k] = i < nrows ? __ldg(qm.P + (long long)rowf(i) * sw + u_lo + w) : 0u;
    }
#pragma unroll
    for (int k = 0; k < WG; ++k) st.w[lane + 32 * k] = v[k];
    __syncwarp();
    cs_consume_r1<WG>(st, hs, Fg);
    __syncwarp();
}

template <class RowF, class QF>
__device__ __forceinline__ void cs_batch_any(const QM &qm, CsWarp &st, int *hs, int u_lo, int Wg, int Fg, int R,
                                             int copy, int nrows, RowF rowf, QF qf) {
    if (R == 1) {
        switch (Wg) {
            case 5: cs_batch_r1<5>(qm, st, hs, u_lo, Fg, nrows, rowf, qf); return;
            case 6: cs_batch_r1<6>(qm, st, hs, u_lo, Fg, nrows, rowf, qf); return;
            case 7: cs_batch_r1<7>(qm, st, hs, u_lo, Fg, nrows, rowf, qf); return;
            case 8: cs_batch_r1<8>(qm, st, hs, u_lo, Fg, nrows, rowf, qf); return;
            default: break;
        }
    }
    cs_batch(qm, st, hs, u_lo, Wg, Fg, R, copy, nrows, rowf, qf);
}

// R1: every group has more than 16 features (one row per warp instruction, compile-time row
// pitch); a separate instantiation so the other path's code generation is not affected
// (Airline, 13 features: root 2.69 vs 3.13 ms when the R1 variants are not in the same kernel).
template <bool IDENT, bool R1>
__global__ void __launch_bounds__(H_THREADS, 2) hist_cs_range_kernel(ColRangeArgs a) {
    extern __shared__ int smem[];
    __shared__ long long s_red[2 * H_THREADS / 32];
    __shared__ uint64_t s_bar[2 * H_THREADS / 32];  // per warp: one mbarrier per staging buffer
    CsWarp *stage = reinterpret_cast<CsWarp *>(smem + 2 * COLB_STRIDE);
    const QM &qm = a.qm;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = H_THREADS / 32;
    long long tg = 0, th = 0;
    const long long sw_row = qm.stride >> 5;
    // whole contiguous rows (identity rows, one group covering every word): TMA bulk copies of
    // 32-row batches into two staging buffers per warp, the next batch in flight while the
    // current one is accumulated
    const bool tma = IDENT && a.n_groups == 1 && a.tma;
    uint64_t *bar = s_bar + 2 * wid;
    unsigned uses0 = 0, uses1 = 0;  // completed phases per barrier
    if (tma && lane == 0) {
        mbar_init(bar, 1);
        mbar_init(bar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int n_items = (int)(((a.n_sel + a.chunk - 1) / a.chunk) * a.n_groups);
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int g = it % a.n_groups;
        const bool tot = a.totals && g == 0;
        const long long start = (long long)(it / a.n_groups) * a.chunk;
        const long long end = min(a.n_sel, start + a.chunk);
        const ColGroup cg = a.groups[g];
        for (int i = threadIdx.x; i < 2 * COLB_STRIDE; i += H_THREADS) smem[i] = 0;
        if (a.rows_ctr && g == 0 && threadIdx.x == 0) atomicAdd(a.rows_ctr, (unsigned long long)(end - start));
        __syncthreads();
        const int Fg = cg.f_hi - cg.f_lo, R = 32 / Fg;
        const int copy = min(lane / Fg, R - 1);
        const int u_lo = cg.f_lo >> 2, Wg = ((cg.f_hi + 3) >> 2) - u_lo;
        long long b_first = start + (long long)wid * 32;
        if (tma && Wg == sw_row) {
            const long long first_b = b_first;
            const int n_full = first_b + 32 <= end ? (int)((end - first_b - 32) / (NW * 32)) + 1 : 0;
            const unsigned bytes_w = 32u * Wg * 4u;
            auto issue = [&](int i) {  // lane 0: batch i into buffer i & 1
                const long long b0 = first_b + (long long)i * NW * 32;
                CsWarp *buf = stage + (i & 1) * NW + wid;
                uint64_t *br = bar + (i & 1);
                fence_proxy_async();  // the buffer's previous generic reads precede the TMA writes
                mbar_arrive_expect_tx(br, bytes_w + 256u);
                bulk_g2s(buf->w, qm.P + b0 * sw_row, bytes_w, br);
                bulk_g2s(buf->q, a.qpair + b0, 256u, br);
            };
            if (n_full > 0 && lane == 0) issue(0);
            for (int i = 0; i < n_full; ++i) {
                if (i + 1 < n_full && lane == 0) issue(i + 1);
                const unsigned par = (i & 1) ? (uses1++ & 1u) : (uses0++ & 1u);
                mbar_wait(bar + (i & 1), par);
                const CsWarp &st = stage[(i & 1) * NW + wid];
                if (R1) {
                    switch (Wg) {
                        case 5: cs_consume_r1<5>(st, smem, Fg); break;
                        case 6: cs_consume_r1<6>(st, smem, Fg); break;
                        case 7: cs_consume_r1<7>(st, smem, Fg); break;
                        case 8: cs_consume_r1<8>(st, smem, Fg); break;
                        default: cs_consume(st, smem, Wg, Fg, R, copy, 32); break;
                    }
                } else {
                    cs_consume(st, smem, Wg, Fg, R, copy, 32);
                }
                if (tot) {
                    tg += st.q[lane].x;
                    th += st.q[lane].y;
                }
                __syncwarp();
            }
            b_first = first_b + (long long)n_full * NW * 32;  // the partial tail, if any, below
        }
        for (long long b0 = b_first; b0 < end; b0 += NW * 32) {
            const int nrows = (int)min(32ll, end - b0);
            auto rowf = [&](int i) -> uint32_t {
                const long long r = b0 + i;
                return IDENT ? (uint32_t)r : __ldg(a.ridx + r);
            };
            if (R1) cs_batch_any(qm, stage[wid], smem, u_lo, Wg, Fg, R, copy, nrows, rowf,
                                 [&](int i) { return __ldg(a.qpair + rowf(i)); });
            else cs_batch(qm, stage[wid], smem, u_lo, Wg, Fg, R, copy, nrows, rowf,
                          [&](int i) { return __ldg(a.qpair + rowf(i)); });
            if (tot) {  // the node totals from the staged pairs (rows past nrows are staged as 0)
                const int2 q = stage[wid].q[lane];
                tg += q.x;
                th += q.y;
            }
        }
        if (tot) {
            block_totals(tg, th, s_red, a.totals);
            tg = th = 0;
        }
        __syncthreads();
        col_flush<false>(smem, COLB_STRIDE, cg, a.cut_ptr, a.hist);
        __syncthreads();
    }
}

// Generic symbol widths (9..15 bits, e.g. 256 bins + the missing symbol): the same staged
// bank-column root, lane f extracting its symbol from the staged row's words; missing symbols
// are skipped (their mass is total - sum, R7).  Groups of <= 32 features at any bit offset.
constexpr int CSG_WMAX = 16;  // words per staged row: 32 features x 15 bits + misalignment
struct CsgWarp {
    uint32_t w[32 * CSG_WMAX + 1];  // + 1: the last symbol's word pair never reads past the end
    int2 q[32];
};

template <bool IDENT>
__global__ void __launch_bounds__(H_THREADS, 2) hist_csg_range_kernel(ColRangeArgs a) {
    extern __shared__ int smem[];
    CsgWarp *stage = reinterpret_cast<CsgWarp *>(smem + 2 * COLB_STRIDE);
    const QM &qm = a.qm;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    constexpr int NW = H_THREADS / 32;
    CsgWarp &st = stage[wid];
    __shared__ long long s_red[2 * H_THREADS / 32];
    long long tg = 0, th = 0;
    const long long sw = qm.stride >> 5;
    const uint32_t mask = (1u << qm.bits) - 1u;
    const int n_items = (int)(((a.n_sel + a.chunk - 1) / a.chunk) * a.n_groups);
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int g = it % a.n_groups;
        const bool tot = a.totals && g == 0;
        const long long start = (long long)(it / a.n_groups) * a.chunk;
        const long long end = min(a.n_sel, start + a.chunk);
        const ColGroup cg = a.groups[g];
        for (int i = threadIdx.x; i < 2 * COLB_STRIDE; i += H_THREADS) smem[i] = 0;
        if (a.rows_ctr && g == 0 && threadIdx.x == 0) atomicAdd(a.rows_ctr, (unsigned long long)(end - start));
        __syncthreads();
        const int Fg = cg.f_hi - cg.f_lo;
        const long long bit_lo = (long long)cg.f_lo * qm.bits;
        const int w_lo = (int)(bit_lo >> 5);
        const int Wg = (int)((((long long)cg.f_hi * qm.bits + 31) >> 5) - w_lo);
        const int bp = (int)(bit_lo - 32ll * w_lo) + lane * qm.bits;  // my symbol's bit in the staged row
        const int wi = bp >> 5, off = bp & 31;
        int *hg = smem + lane, *hh = smem + COLB_STRIDE + lane;
        for (long long b0 = start + (long long)wid * 32; b0 < end; b0 += NW * 32) {
            const int nrows = (int)min(32ll, end - b0);
            auto rowf = [&](int i) -> uint32_t { return IDENT ? (uint32_t)(b0 + i) : __ldg(a.ridx + b0 + i); };
            st.q[lane] = lane < nrows ? __ldg(a.qpair + rowf(lane)) : make_int2(0, 0);
            if (tot) {
                tg += st.q[lane].x;
                th += st.q[lane].y;
            }
            for (int idx = lane; idx < 32 * Wg; idx += 32) {
                const int i = idx / Wg, w = idx - i * Wg;
                st.w[idx] = i < nrows ? __ldg(qm.P + (long long)rowf(i) * sw + w_lo + w) : 0u;
            }
            __syncwarp();
            if (lane < Fg) {
                for (int i = 0; i < nrows; ++i) {
                    const uint32_t *rw = st.w + i * Wg + wi;
                    const uint64_t v = (uint64_t)rw[0] | ((uint64_t)rw[1] << 32);
                    const int sym = (int)((uint32_t)(v >> off) & mask);
                    if (sym != qm.B) {
                        const int2 q = st.q[i];
                        atomicAdd(hg + (sym << 5), q.x);
                        atomicAdd(hh + (sym << 5), q.y);
                    }
                }
            }
            __syncwarp();
        }
        if (tot) {
            block_totals(tg, th, s_red, a.totals);
            tg = th = 0;
        }
        __syncthreads();
        col_flush<false>(smem, COLB_STRIDE, cg, a.cut_ptr, a.hist);
        __syncthreads();
    }
}

struct ColFusedArgs {
    QM qm;
    const NodeDev *nodes;
    int first, n_par;
    const int *tile_base;
    const int *run_base;
    int n_groups, run_tiles;
    const int *n_items;
    const void *ridx_in;  // entries, null = identity (level 1)
    uint32_t *flags;
    int *tile_left;
    int32_t *row_leaf;
    const int2 *qpair;
    const ColGroup *groups;
    const int32_t *cut_ptr;
    unsigned long long *hist;  // [n_par][TB][2]
    long long TB;
    int cstride;
    unsigned long long *rows_ctr;
    int bits_parent_row, bits_built_row;
};

template <bool WIDE, bool CARRY, bool BYTE>
__global__ void __launch_bounds__(H_THREADS) part_hist_col_kernel(ColFusedArgs a) {
    using E = typename EntryOf<CARRY>::T;
    extern __shared__ int smem[];
    __shared__ E s_rows[H_THREADS / 32][WROWS];
    const QM &qm = a.qm;
    const E *rin = static_cast<const E *>(a.ridx_in);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n_items = *a.n_items;
    E *wrows = s_rows[wid];
    for (int it = claim_item(const_cast<int *>(a.n_items) + 1); it < n_items;
         it = claim_item(const_cast<int *>(a.n_items) + 1)) {
        const int run = it / a.n_groups, g = it - run * a.n_groups;
        const int j = find_parent(a.run_base, a.n_par, run);
        const int k = a.first + j;
        const NodeDev nd = a.nodes[k];
        const int tb = a.tile_base[j];
        const int rt = a.n_items[2], t0 = tb + (run - a.run_base[j]) * rt, t1 = min(a.tile_base[j + 1], t0 + rt);
        const long long seg_end = nd.start + nd.count;
        if (nd.state == GBM_NODE_LEAF) {  // rows stay in this leaf
            if (g != 0) continue;
            for (int t = t0; t < t1; ++t) {
                const long long base = nd.start + (long long)(t - tb) * PT;
                for (int i = threadIdx.x; i < PT; i += H_THREADS) {
                    const long long pos = base + i;
                    if (pos < seg_end) a.row_leaf[rin ? row_of(rin[pos]) : (uint32_t)pos] = k;
                }
            }
            continue;
        }
        const ColGroup cg = a.groups[g];
        for (int i = threadIdx.x; i < (WIDE ? 4 : 2) * a.cstride; i += H_THREADS) smem[i] = 0;
        __syncthreads();
        const ColLane L = col_lane(qm, cg);
        const bool build_left = nd.build_left != 0;
        unsigned long long bits_acc = 0;
        const uint8_t *Pb = reinterpret_cast<const uint8_t *>(qm.P) + (L.bitoff >> 3);
        const unsigned sb = (unsigned)(qm.stride >> 3);
        const bool chk = qm.B < 256;
        for (int t = t0; t < t1; ++t) {
            const long long base = nd.start + (long long)(t - tb) * PT + wid * WROWS;
            // (A) partition flags for the warp's 128 rows (lane = row)
            E row[4];
            uint32_t bw[4];
            int nleft = 0;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const long long pos = base + s2 * 32 + lane;
                if (pos < seg_end) row[s2] = rin ? rin[pos] : make_entry<CARRY>((uint32_t)pos, a.qpair);
                else row[s2] = E{};
            }
            bool left[4];
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2)
                left[s2] = base + s2 * 32 + lane < seg_end && goes_left(qm, nd, row_of(row[s2]));
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const bool valid = base + s2 * 32 + lane < seg_end;
                const uint32_t lw = __ballot_sync(0xffffffffu, valid && left[s2]);
                bw[s2] = __ballot_sync(0xffffffffu, valid && (left[s2] == build_left));
                if (g == 0 && lane == 0) a.flags[(long long)t * (PT / 32) + wid * 4 + s2] = lw;
                nleft += __popc(lw);
            }
            int nbuild = 0;
            const uint32_t ltm = (1u << lane) - 1u;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                if ((bw[s2] >> lane) & 1u) wrows[nbuild + __popc(bw[s2] & ltm)] = row[s2];
                nbuild += __popc(bw[s2]);
            }
            if (g == 0 && lane == 0) {
                if (nleft) atomicAdd(a.tile_left + t, nleft);
                if (a.rows_ctr) {
                    const long long nv = max(0ll, min((long long)WROWS, seg_end - base));
                    bits_acc += (unsigned long long)nv * a.bits_parent_row +
                                (unsigned long long)nbuild * a.bits_built_row;
                }
            }
            __syncwarp();
            // (B) histogram of the listed rows, lane = (copy, feature column)
            if (BYTE) {  // branch-free (see hist_colb_range_kernel)
                const uint8_t *Pf = reinterpret_cast<const uint8_t *>(qm.P) + (cg.f_lo + lane % L.Fg);
                const int cp2 = min(L.copy, L.R - 1);
                for (int i0 = cp2; i0 < nbuild; i0 += COLB_UR * L.R) {
                    uint32_t sym[COLB_UR];
                    int2 q[COLB_UR];
                    bool ok[COLB_UR];
#pragma unroll
                    for (int u = 0; u < COLB_UR; ++u) {
                        const int i = i0 + u * L.R;
                        ok[u] = i < nbuild;
                        const E e = wrows[ok[u] ? i : nbuild - 1];
                        sym[u] = __ldg(Pf + (size_t)row_of(e) * sb);
                        q[u] = entry_q(e, a.qpair);
                    }
#pragma unroll
                    for (int u = 0; u < COLB_UR; ++u)
                        col_add_b<WIDE>(smem, (int)(sym[u] << 5) + lane, ok[u] ? q[u] : make_int2(0, 0));
                }
            } else
            for (int i0 = L.copy; i0 < nbuild; i0 += 4 * L.R) {
                uint32_t sym[4];
                int2 q[4];
                bool ok[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = i0 + u * L.R;
                    ok[u] = L.active && i < nbuild;
                    const E e = ok[u] ? wrows[i] : E{};
                    const uint32_t r = row_of(e);
                    if (BYTE) sym[u] = ok[u] ? __ldg(Pb + (size_t)r * sb) : 0u;
                    else sym[u] = ok[u] ? get_bits(qm.P, (long long)r * qm.stride + L.bitoff, qm.bits) : 0u;
                    q[u] = ok[u] ? entry_q(e, a.qpair) : make_int2(0, 0);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (BYTE) {
                        if (ok[u] && (!chk || (int)sym[u] != qm.B))
                            col_add_b<WIDE>(smem, (int)(sym[u] << 5) + lane, q[u]);
                    } else if (ok[u] && (int)sym[u] != qm.B) {
                        col_add<WIDE>(smem, a.cstride, (int)sym[u] * 32 + lane, q[u]);
                    }
                }
            }
            __syncwarp();
        }
        if (bits_acc) atomicAdd(a.rows_ctr, bits_acc);
        __syncthreads();
        col_flush<WIDE>(smem, a.cstride, cg, a.cut_ptr, a.hist + (long long)j * a.TB * 2);
        __syncthreads();
    }
}

// fused partition + staged bank-column histogram (GBM_OPT_HIST_LAYOUT = 3)
template <bool CARRY, bool R1>
__global__ void __launch_bounds__(H_THREADS, 2) part_hist_cs_kernel(ColFusedArgs a) {
    using E = typename EntryOf<CARRY>::T;
    extern __shared__ int smem[];
    CsWarp *stage = reinterpret_cast<CsWarp *>(smem + 2 * COLB_STRIDE);
    __shared__ E s_rows[H_THREADS / 32][WROWS];
    const QM &qm = a.qm;
    const E *rin = static_cast<const E *>(a.ridx_in);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int n_items = *a.n_items;
    E *wrows = s_rows[wid];
    for (int it = claim_item(const_cast<int *>(a.n_items) + 1); it < n_items;
         it = claim_item(const_cast<int *>(a.n_items) + 1)) {
        const int run = it / a.n_groups, g = it - run * a.n_groups;
        const int j = find_parent(a.run_base, a.n_par, run);
        const int k = a.first + j;
        const NodeDev nd = a.nodes[k];
        const int tb = a.tile_base[j];
        const int rt = a.n_items[2], t0 = tb + (run - a.run_base[j]) * rt, t1 = min(a.tile_base[j + 1], t0 + rt);
        const long long seg_end = nd.start + nd.count;
        if (nd.state == GBM_NODE_LEAF) {
            if (g != 0) continue;
            for (int t = t0; t < t1; ++t) {
                const long long base = nd.start + (long long)(t - tb) * PT;
                for (int i = threadIdx.x; i < PT; i += H_THREADS) {
                    const long long pos = base + i;
                    if (pos < seg_end) a.row_leaf[rin ? row_of(rin[pos]) : (uint32_t)pos] = k;
                }
            }
            continue;
        }
        const ColGroup cg = a.groups[g];
        for (int i = threadIdx.x; i < 2 * COLB_STRIDE; i += H_THREADS) smem[i] = 0;
        __syncthreads();
        const int Fg = cg.f_hi - cg.f_lo, R = 32 / Fg;
        const int copy = min(lane / Fg, R - 1);
        const int u_lo = cg.f_lo >> 2, Wg = ((cg.f_hi + 3) >> 2) - u_lo;
        const bool build_left = nd.build_left != 0;
        unsigned long long bits_acc = 0;
        for (int t = t0; t < t1; ++t) {
            const long long base = nd.start + (long long)(t - tb) * PT + wid * WROWS;
            E row[4];
            uint32_t bw[4];
            int nleft = 0;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const long long pos = base + s2 * 32 + lane;
                if (pos < seg_end) row[s2] = rin ? rin[pos] : make_entry<CARRY>((uint32_t)pos, a.qpair);
                else row[s2] = E{};
            }
            bool left[4];
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2)
                left[s2] = base + s2 * 32 + lane < seg_end && goes_left(qm, nd, row_of(row[s2]));
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const bool valid = base + s2 * 32 + lane < seg_end;
                const uint32_t lw = __ballot_sync(0xffffffffu, valid && left[s2]);
                bw[s2] = __ballot_sync(0xffffffffu, valid && (left[s2] == build_left));
                if (g == 0 && lane == 0) a.flags[(long long)t * (PT / 32) + wid * 4 + s2] = lw;
                nleft += __popc(lw);
            }
            int nbuild = 0;
            const uint32_t ltm = (1u << lane) - 1u;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                if ((bw[s2] >> lane) & 1u) wrows[nbuild + __popc(bw[s2] & ltm)] = row[s2];
                nbuild += __popc(bw[s2]);
            }
            if (g == 0 && lane == 0) {
                if (nleft) atomicAdd(a.tile_left + t, nleft);
                if (a.rows_ctr) {
                    const long long nv = max(0ll, min((long long)WROWS, seg_end - base));
                    bits_acc += (unsigned long long)nv * a.bits_parent_row +
                                (unsigned long long)nbuild * a.bits_built_row;
                }
            }
            __syncwarp();
            for (int b0 = 0; b0 < nbuild; b0 += 32)
                if (R1) cs_batch_any(qm, stage[wid], smem, u_lo, Wg, Fg, R, copy, min(32, nbuild - b0),
                                     [&](int i) { return row_of(wrows[b0 + i]); },
                                     [&](int i) { return entry_q(wrows[b0 + i], a.qpair); });
                else cs_batch(qm, stage[wid], smem, u_lo, Wg, Fg, R, copy, min(32, nbuild - b0),
                              [&](int i) { return row_of(wrows[b0 + i]); },
                              [&](int i) { return entry_q(wrows[b0 + i], a.qpair); });
            __syncwarp();
        }
        if (bits_acc) atomicAdd(a.rows_ctr, bits_acc);
        __syncthreads();
        col_flush<false>(smem, COLB_STRIDE, cg, a.cut_ptr, a.hist + (long long)j * a.TB * 2);
        __syncthreads();
    }
}

// Final level: every row's leaf by walking the tree on its packed symbols, in ROW order
// (coalesced; no ridx, no gather).  Same decision rule as RepartitionInstances, so
// row_leaf equals the partition the levels would have produced.
constexpr int WALK_THREADS = 256;
__global__ void __launch_bounds__(WALK_THREADS) leaf_walk_kernel(QM qm, const int8_t *__restrict__ kind,
                                                                 const int32_t *__restrict__ feature,
                                                                 const int32_t *__restrict__ bin,
                                                                 const int8_t *__restrict__ dl, int n_internal,
                                                                 int depth, long long n,
                                                                 int32_t *__restrict__ row_leaf) {
    extern __shared__ int s_tree[];  // [n_internal] packed: feature | dl << 20 | split << 21, bin
    int *s_f = s_tree, *s_b = s_tree + n_internal;
    for (int k = threadIdx.x; k < n_internal; k += WALK_THREADS) {
        s_f[k] = kind[k] == GBM_NODE_SPLIT ? (feature[k] | ((int)dl[k] << 20) | (1 << 21)) : 0;
        s_b[k] = bin[k];
    }
    __syncthreads();
    const long long stride = (long long)gridDim.x * WALK_THREADS;
    for (long long i0 = blockIdx.x * (long long)WALK_THREADS + threadIdx.x; i0 < n; i0 += 4 * stride) {
        int k[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) k[u] = 0;
        for (int d = 0; d < depth; ++d) {  // four independent walks in lockstep
            uint32_t sym[4];
            int fk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long i = i0 + u * stride;
                fk[u] = (i < n && k[u] < n_internal) ? s_f[k[u]] : 0;
                sym[u] = (fk[u] & (1 << 21)) ? split_symbol(qm, i, fk[u] & 0xfffff) : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (!(fk[u] & (1 << 21))) continue;
                const bool left = (int)sym[u] == qm.B ? ((fk[u] >> 20) & 1) : ((int)sym[u] <= s_b[k[u]]);
                k[u] = left ? 2 * k[u] + 1 : 2 * k[u] + 2;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const long long i = i0 + u * stride;
            if (i < n) row_leaf[i] = k[u];
        }
    }
}

// Staged variant: a warp loads 32 whole rows (W words each, contiguous) with W coalesced loads
// into shared memory (row pitch W|1 words: conflict-free), then each lane walks its row from
// registers.  Moves exactly the packed bytes once, in row order (vs a 32-byte sector per level
// and row for the feature-major gathers of leaf_walk_kernel once the rows' nodes diverge).
// Fused epilogue of gbm_build_tree_fused: with each row's leaf, margin += weight[leaf]
// (gbm_update_margins) and Eq. 1-2 for the new margin (pass 1 of the next gbm_gradients: the
// logistic sigmoid into sig, this rank's max|g|, max|h|), in the same op order as those entries.
struct WalkEpi {
    double *margin;
    const float *label;
    int objective;
    double *sig;
    unsigned long long *maxbits;
    uint32_t *dev_err;
    const double *weight;
};

// BYTE (8-bit symbols, rows of whole words): the symbol of feature f is byte f of the staged row,
// one LDS.U8 per level (the node record holds the byte index); SENT: the sentinel fits in 8 bits.
template <int W, bool EPI, bool BYTE = false, bool SENT = true>
__global__ void __launch_bounds__(WALK_THREADS) leaf_walk_stg_kernel(QM qm, const int8_t *__restrict__ kind,
                                                                     const int32_t *__restrict__ feature,
                                                                     const int32_t *__restrict__ bin,
                                                                     const int8_t *__restrict__ dl, int n_internal,
                                                                     int depth, long long n,
                                                                     int32_t *__restrict__ row_leaf, WalkEpi ep) {
    constexpr int PW = W | 1;
    extern __shared__ int2 s_node[];
    __shared__ uint32_t s_rows[WALK_THREADS / 32][32 * PW];
    // per internal node, one 64-bit shared load per level: x = split (sign bit) | default-left
    // << 30 | symbol crosses a word << 29 | bit offset << 16 | word index; y = split bin
    for (int k = threadIdx.x; k < n_internal; k += WALK_THREADS) {
        int x = 0;
        if (kind[k] == GBM_NODE_SPLIT) {
            if (BYTE) {
                x = (int)(1u << 31) | ((int)dl[k] << 30) | feature[k];
            } else {
                const int bp = feature[k] * qm.bits, wi = bp >> 5, off = bp & 31;
                x = (int)(1u << 31) | ((int)dl[k] << 30) | ((off + qm.bits > 32) << 29) | (off << 16) | wi;
            }
        }
        s_node[k] = make_int2(x, bin[k]);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *sr = s_rows[wid];
    double mg = 0.0, mh = 0.0;  // (EPI)
    bool bad = false;
    const long long n_chunks = (n + 31) / 32;
    const long long cstep = (long long)gridDim.x * (WALK_THREADS / 32);
    uint32_t v[W];
    double m_next = 0.0;  // (EPI) the lane's row of the next chunk: margin and label in flight
    float y_next = 0.0f;
    auto load = [&](long long c) {  // chunk c's words into registers (coalesced)
        const uint32_t *src = qm.P + c * 32 * W;
        if (c + 1 < n_chunks) {  // a full chunk: no per-word bounds
#pragma unroll
            for (int k = 0; k < W; ++k) v[k] = __ldg(src + lane + 32 * k);
        } else {
            const int rows_c = c < n_chunks ? (int)(n - c * 32) : 0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                const int j = lane + 32 * k;
                v[k] = j / W < rows_c ? __ldg(src + j) : 0u;
            }
        }
        if (EPI) {
            const long long r = c * 32 + lane;
            const bool ok = r < n;
            m_next = ok ? ep.margin[r] : 0.0;
            y_next = ok ? __ldg(ep.label + r) : 0.0f;
        }
    };
    long long c = blockIdx.x * (long long)(WALK_THREADS / 32) + wid;
    if (c < n_chunks) load(c);
    for (; c < n_chunks; c += cstep) {
        const long long rows_here = min(32ll, n - c * 32);
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int j = lane + 32 * k;
            sr[(j / W) * PW + j % W] = v[k];
        }
        __syncwarp();
        const double m_cur = m_next;
        const float y_cur = y_next;
        load(c + cstep);  // the next chunk's loads fly during this chunk's walk
        if (lane < rows_here) {  // walk on the staged row: one shared-memory read per level
            const uint32_t *row = sr + lane * PW;
            const uint32_t mask = (1u << qm.bits) - 1u;
            int k = 0;
            if (BYTE) {
                const uint8_t *rb = reinterpret_cast<const uint8_t *>(row);
                for (int d = 0; d < depth; ++d) {
                    const int2 nk = s_node[k];
                    if (nk.x >= 0) break;  // leaf
                    const int sym = rb[nk.x & 0xffff];
                    const bool left = (SENT && sym == qm.B) ? ((nk.x >> 30) & 1) : (sym <= nk.y);
                    k = 2 * k + 2 - (int)left;
                }
            } else {
                for (int d = 0; d < depth; ++d) {
                    const int2 nk = s_node[k];
                    if (nk.x >= 0) break;  // leaf
                    const int wi = nk.x & 0xffff, off = (nk.x >> 16) & 31;
                    uint32_t v = row[wi] >> off;
                    if (nk.x & (1 << 29)) v |= row[wi + 1] << (32 - off);  // off > 0 here
                    const int sym = (int)(v & mask);
                    const bool left = sym == qm.B ? ((nk.x >> 30) & 1) : (sym <= nk.y);
                    k = left ? 2 * k + 1 : 2 * k + 2;
                }
            }
            const long long r = c * 32 + lane;
            row_leaf[r] = k;
            if (EPI) {
                const double m = dadd(m_cur, __ldg(ep.weight + k));
                ep.margin[r] = m;
                const float yl = y_cur;
                double v = m;
                if (ep.objective == GBM_LOGISTIC) {
                    v = sigmoid(m);
                    ep.sig[r] = v;
                    bad |= !(yl == 0.0f || yl == 1.0f);
                }
                double g, hh;
                grad_hess_s(ep.objective, v, yl, g, hh);
                mg = fmax(mg, fabs(g));
                mh = fmax(mh, fabs(hh));
            }
        }
        __syncwarp();
    }
    if (EPI) {
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(ep.dev_err, DERR_LABEL);
        for (int o = 16; o > 0; o >>= 1) {
            mg = fmax(mg, __shfl_xor_sync(0xffffffffu, mg, o));
            mh = fmax(mh, __shfl_xor_sync(0xffffffffu, mh, o));
        }
        if (lane == 0) {  // non-negative doubles order like their bit patterns
            atomicMax(ep.maxbits + 0, (unsigned long long)__double_as_longlong(mg));
            atomicMax(ep.maxbits + 1, (unsigned long long)__double_as_longlong(mh));
        }
    }
}

// Row-order decisions of one depth-wise level (GBM_OPT_ROW_DECIDE): a warp stages 32 whole rows
// (as leaf_walk_stg_kernel), each lane walks its row from the root through the SPLIT nodes of
// depths < par_depth to its parent at depth par_depth and applies that parent's split -- the
// rule of goes_left on the same symbol -- and the warp writes the 32 decisions as one
// word (bit = goes left).  Rows whose walk ends in a leaf get 0 (never read).  Streams the packed
// rows once (coalesced) instead of gathering a 32-byte sector per row for one symbol.
template <int W>
__global__ void __launch_bounds__(WALK_THREADS) row_decide_kernel(QM qm, const NodeDev *__restrict__ nodes,
                                                                  int par_depth, long long n,
                                                                  uint32_t *__restrict__ dbits) {
    constexpr int PW = W | 1;
    extern __shared__ int2 s_dnode[];  // [2^(par_depth+1) - 1] as in leaf_walk_stg_kernel
    __shared__ uint32_t s_rows[WALK_THREADS / 32][32 * PW];
    const int n_nodes = (2 << par_depth) - 1;
    for (int k = threadIdx.x; k < n_nodes; k += WALK_THREADS) {
        const NodeDev nd = nodes[k];
        int x = 0;
        if (nd.state == GBM_NODE_SPLIT) {
            const int bp = nd.f * qm.bits, wi = bp >> 5, off = bp & 31;
            x = (int)(1u << 31) | ((nd.dl != 0) << 30) | ((off + qm.bits > 32) << 29) | (off << 16) | wi;
        }
        s_dnode[k] = make_int2(x, nd.b);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t *sr = s_rows[wid];
    const uint32_t mask = (1u << qm.bits) - 1u;
    const long long n_chunks = (n + 31) / 32;
    const long long cstep = (long long)gridDim.x * (WALK_THREADS / 32);
    uint32_t v[W];
    auto load = [&](long long c) {
        const uint32_t *src = qm.P + c * 32 * W;
        const long long rows_c = c < n_chunks ? min(32ll, n - c * 32) : 0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int j = lane + 32 * k;
            v[k] = j / W < rows_c ? __ldg(src + j) : 0u;
        }
    };
    long long c = blockIdx.x * (long long)(WALK_THREADS / 32) + wid;
    if (c < n_chunks) load(c);
    for (; c < n_chunks; c += cstep) {
        const long long rows_here = min(32ll, n - c * 32);
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int j = lane + 32 * k;
            sr[(j / W) * PW + j % W] = v[k];
        }
        __syncwarp();
        load(c + cstep);
        bool left = false;
        if (lane < rows_here) {
            const uint32_t *row = sr + lane * PW;
            int k = 0;
            for (int d = 0; d <= par_depth; ++d) {
                const int2 nk = s_dnode[k];
                if (nk.x >= 0) break;  // leaf: no parent at par_depth
                const int wi = nk.x & 0xffff, off = (nk.x >> 16) & 31;
                uint32_t x = row[wi] >> off;
                if (nk.x & (1 << 29)) x |= row[wi + 1] << (32 - off);
                const int sym = (int)(x & mask);
                const bool l = sym == qm.B ? ((nk.x >> 30) & 1) : (sym <= nk.y);
                if (d == par_depth) left = l;
                k = l ? 2 * k + 1 : 2 * k + 2;
            }
        }
        const uint32_t word = __ballot_sync(0xffffffffu, left);
        if (lane == 0) dbits[c] = word;
        __syncwarp();
    }
}

// Deep trees (the heap of internal nodes does not fit shared memory): tree read through L1.
__global__ void __launch_bounds__(WALK_THREADS) leaf_walk_global_kernel(QM qm, TreeDev t, int depth, long long n,
                                                                        int32_t *__restrict__ row_leaf) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
         r += (long long)gridDim.x * blockDim.x) {
        int k = 0;
        for (int d = 0; d < depth && __ldg(t.kind + k) == GBM_NODE_SPLIT; ++d) {
            const int sym = (int)split_symbol(qm, r, __ldg(t.feature + k));
            const bool left = sym == qm.B ? __ldg(t.default_left + k) != 0 : sym <= __ldg(t.bin + k);
            k = left ? 2 * k + 1 : 2 * k + 2;
        }
        row_leaf[r] = k;
    }
}

// ============================================================== scan + scatter
__device__ __forceinline__ long long block_exscan(long long v, long long *total, long long *sm32) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm32[wid] = x;
    __syncthreads();
    if (wid == 0) {
        long long s = lane < nw ? sm32[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        sm32[lane] = s;
    }
    __syncthreads();
    long long ex = (wid ? sm32[wid - 1] : 0) + x - v;
    *total = sm32[nw - 1];
    __syncthreads();
    return ex;
}

// one block per parent: exclusive scan of its tiles' left counts; children segments
__global__ void __launch_bounds__(1024) part_scan_kernel(NodeDev *__restrict__ nodes, int first,
                                                         const int *__restrict__ tile_base,
                                                         const int *__restrict__ tile_left, int *__restrict__ tile_off,
                                                         const StepDev *__restrict__ step) {
    __shared__ long long sm32[32];
    const int j = blockIdx.x;
    int k = first + j, c = 2 * k + 1;
    if (step) {  // loss-guided: the step's parent and its children 2j+1, 2j+2
        k = step->k;
        c = step->c;
        if (k < 0) return;
    }
    const NodeDev nd = nodes[k];
    NodeDev *Lc = nodes + c, *Rc = nodes + c + 1;
    if (nd.state != GBM_NODE_SPLIT) {
        if (threadIdx.x == 0) {
            Lc->count = 0; Lc->start = 0; Lc->state = GBM_NODE_ABSENT;
            Rc->count = 0; Rc->start = 0; Rc->state = GBM_NODE_ABSENT;
        }
        return;
    }
    const int t0 = nd.count > 0 ? tile_base[j] : 0, t1 = nd.count > 0 ? tile_base[j + 1] : 0;
    constexpr int PER = 16;  // consecutive tiles per thread
    long long carry = 0;
    for (int c = t0; c < t1; c += 1024 * PER) {
        const int tb = c + threadIdx.x * PER;
        int v[PER];
        long long loc = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            v[i] = tb + i < t1 ? tile_left[tb + i] : 0;
            loc += v[i];
        }
        long long tot;
        long long ex = carry + block_exscan(loc, &tot, sm32);
#pragma unroll
        for (int i = 0; i < PER; ++i)
            if (tb + i < t1) {
                tile_off[tb + i] = (int)ex;
                ex += v[i];
            }
        carry += tot;
    }
    if (threadIdx.x == 0) {
        Lc->start = nd.start;
        Lc->count = carry;
        Rc->start = nd.start + carry;
        Rc->count = nd.count - carry;
    }
}

__global__ void __launch_bounds__(1024) seg_plan_kernel(const NodeDev *__restrict__ nodes, int first, int n_par,
                                                        int chunk, int n_groups, int *__restrict__ seg_base,
                                                        int *__restrict__ n_items) {
    __shared__ long long sm32[32];
    long long carry = 0;
    for (int c = 0; c < n_par; c += blockDim.x) {
        const int j = c + threadIdx.x;
        long long nc = 0;
        if (j < n_par) {
            const int k = first + j;
            const NodeDev nd = nodes[k];
            if (nd.state == GBM_NODE_SPLIT) {
                const long long cnt = nodes[nd.build_left ? 2 * k + 1 : 2 * k + 2].count;
                nc = (cnt + chunk - 1) / chunk;
            }
        }
        long long tot;
        const long long ex = carry + block_exscan(nc, &tot, sm32);
        if (j < n_par) seg_base[j] = (int)ex;
        carry += tot;
    }
    if (threadIdx.x == 0) {
        seg_base[n_par] = (int)carry;
        n_items[0] = (int)carry * n_groups;
    }
}

template <bool CARRY>
__global__ void __launch_bounds__(P_THREADS) part_scatter_kernel(
    const NodeDev *__restrict__ nodes, int first, int n_par, const int *__restrict__ tile_base,
    const uint32_t *__restrict__ flags, const int *__restrict__ tile_off,
    const typename EntryOf<CARRY>::T *__restrict__ ridx_in, typename EntryOf<CARRY>::T *__restrict__ ridx_out,
    const int2 *__restrict__ qpair, unsigned long long *__restrict__ rows_ctr,
    const StepDev *__restrict__ step = nullptr, void *buf0 = nullptr, void *buf1 = nullptr) {
    using E = typename EntryOf<CARRY>::T;
    constexpr int WPW = PT / 32 / (P_THREADS / 32);  // flag words per warp (8)
    if (step) {  // loss-guided: rows move from the parent's buffer to the other one
        const int ib = step->in_buf, ob = step->out_buf;
        ridx_in = ib < 0 ? nullptr : static_cast<const E *>(ib ? buf1 : buf0);
        ridx_out = static_cast<E *>(ob ? buf1 : buf0);
    }
    __shared__ int wpre[PT / 32];
    const int n_tiles = tile_base[n_par];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int j = find_parent(tile_base, n_par, t);
        const int k = step ? step->k : first + j;
        const NodeDev nd = nodes[k];
        if (nd.state != GBM_NODE_SPLIT) continue;  // uniform per block
        // segment-local 32-bit positions (a rank's segment holds < 2^31 rows); one pointer per tile
        const int n_left = (int)nodes[step ? step->c : 2 * k + 1].count;
        const int lt = t - tile_base[j];
        const int tile_rows = (int)min((long long)PT, nd.count - (long long)lt * PT);
        if (rows_ctr && threadIdx.x == 0) atomicAdd(rows_ctr, (unsigned long long)tile_rows);
        // every load of the tile is issued before the block scan (one exposed DRAM latency)
        const int off = tile_off[t];
        const long long tile0 = nd.start + (long long)lt * PT;  // first position of this tile
        const E *src = ridx_in ? ridx_in + tile0 : nullptr;
        E *dst = ridx_out + nd.start;
        const int wbase = wid * (WPW * 32);
        E rows[WPW];
#pragma unroll
        for (int s = 0; s < WPW; ++s) {
            const int q = wbase + s * 32 + lane;  // position within the tile
            if (q < tile_rows) rows[s] = src ? src[q] : make_entry<CARRY>((uint32_t)(tile0 + q), qpair);
            else rows[s] = E{};
        }
        // one flag word per lane (lanes >= WPW idle), warp-scan of the popcounts
        const uint32_t myw = lane < WPW ? __ldg(flags + (long long)t * (PT / 32) + wid * WPW + lane) : 0u;
        if (lane < WPW) wpre[wid * WPW + lane] = __popc(myw);
        __syncthreads();
        static_assert(PT / 32 == 64, "two flag words per lane below");
        if (threadIdx.x < 32) {  // exclusive scan of the 64 word popcounts, two per lane
            const int v0 = wpre[2 * lane], v1 = wpre[2 * lane + 1];
            const int v = v0 + v1;
            int x = v;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            wpre[2 * lane] = x - v;
            wpre[2 * lane + 1] = x - v + v0;
        }
        __syncthreads();
        const uint32_t ltm = (1u << lane) - 1u;
        const int pin0 = lt * PT + wbase + lane;  // segment position of row s = 0 of this lane
#pragma unroll
        for (int s = 0; s < WPW; ++s) {
            const uint32_t w = __shfl_sync(0xffffffffu, myw, s);
            if (wbase + s * 32 + lane >= tile_rows) continue;
            const int lb = off + wpre[wid * WPW + s] + __popc(w & ltm);  // lefts before
            const bool left = (w >> lane) & 1u;
            dst[left ? lb : n_left + (pin0 + s * 32 - lb)] = rows[s];
        }
        __syncthreads();
    }
}

// ============================================================== split evaluation
__device__ __forceinline__ bool better(double ga, long long ia, double gb, long long ib) {
    if (ia == LLONG_MAX) return false;
    if (ib == LLONG_MAX) return true;
    return ga > gb || (ga == gb && ia < ib);
}

// Histogram source of one node: direct, or sibling = parent - build.  Optionally stored.
struct NodeHist {
    const long long *direct, *parent, *build;
    long long *store;
    // (g, h) of one bin as one 16-byte load (histogram slots are 16-byte aligned): half the L1
    // requests of two 8-byte loads (the wide-data evaluation is L1-bound)
    __device__ __forceinline__ void get(int bin, long long &g, long long &h) const {
        if (direct) {
            const longlong2 v = __ldg(reinterpret_cast<const longlong2 *>(direct) + bin);
            g = v.x;
            h = v.y;
        } else {
            const longlong2 pa = __ldg(reinterpret_cast<const longlong2 *>(parent) + bin);
            const longlong2 bu = __ldg(reinterpret_cast<const longlong2 *>(build) + bin);
            g = pa.x - bu.x;
            h = pa.y - bu.y;
        }
    }
    __device__ __forceinline__ void put(int bin, long long g, long long h) const {
        reinterpret_cast<longlong2 *>(store)[bin] = make_longlong2(g, h);
    }
};

// Best candidate of feature f of one node, computed by one warp (valid in every lane).
// Op order of every fp64 step = R8 (oracle_evaluate_split).
// One candidate (R8 op order); updates best.
__device__ __forceinline__ void eval_candidate(long long Pg, long long Ph, long long Mg, long long Mh, long long Tg,
                                               long long Th, int sg, int sh, double e, const EvalParams &p,
                                               long long bin_global, FeatBest &best) {
    // No missing mass: both default directions give the same (L, R), hence the same gain, and
    // the dl = true candidate comes first in the canonical order -- evaluating it alone picks
    // the identical best (R9).
    const int n_dl = (Mg == 0 && Mh == 0) ? 1 : 2;
    for (int dli = 0; dli < n_dl; ++dli) {
        const bool dl = dli == 0;  // true first (R9)
        const long long Lg = Pg + (dl ? Mg : 0), Lh = Ph + (dl ? Mh : 0);
        const double GL = fixed_to_double(Lg, sg), HL = fixed_to_double(Lh, sh);
        const double GR = fixed_to_double(Tg - Lg, sg), HR = fixed_to_double(Th - Lh, sh);
        if (!(HL >= p.mcw && HR >= p.mcw && dadd(HL, p.lambda) > 0.0 && dadd(HR, p.lambda) > 0.0)) continue;
        double aa = dmul(GL, GL);
        aa = ddiv(aa, dadd(HL, p.lambda));
        double cc = dmul(GR, GR);
        cc = ddiv(cc, dadd(HR, p.lambda));
        double d = dadd(aa, cc);
        d = dsub(d, e);
        d = dmul(0.5, d);
        const double gain = dsub(d, p.gamma);
        const long long idx = bin_global * 2 + dli;
        if (better(gain, idx, best.gain, best.idx)) {
            best.gain = gain;
            best.idx = idx;
            best.Lg = Lg;
            best.Lh = Lh;
        }
    }
}

// Exact-preserving screen.  Every candidate's gain is a monotone non-decreasing function of
// s = GL^2/(HL+lambda) + GR^2/(HR+lambda) (R8: d = a + c, d -= e, d *= 0.5, gain = d - gamma, each
// correctly rounded), so the canonical argmax -- and every candidate whose gain can tie with it --
// lies among the candidates whose s is within rounding of the largest s.  s~ below is s computed
// with a Newton-refined hardware reciprocal (relative error < 2^-38 from a >= 2^-10 seed, two
// non-negative terms), and a candidate is evaluated exactly iff s~ >= (1 - 2^-16) max s~: the
// exact best is never screened out, while almost every other candidate skips its two IEEE
// divisions.  Returns -1 for an invalid candidate (same validity test as eval_candidate).
__device__ __forceinline__ double rcp_refined(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double r = fma(-x, y, 1.0);
    return fma(y, r, y);
}
__device__ __forceinline__ double screen_score(long long Pg, long long Ph, long long Mg, long long Mh, long long Tg,
                                               long long Th, int sg, int sh, const EvalParams &p, int dli) {
    const bool dl = dli == 0;
    const long long Lg = Pg + (dl ? Mg : 0), Lh = Ph + (dl ? Mh : 0);
    const double GL = fixed_to_double(Lg, sg), HL = fixed_to_double(Lh, sh);
    const double GR = fixed_to_double(Tg - Lg, sg), HR = fixed_to_double(Th - Lh, sh);
    const double xl = dadd(HL, p.lambda), xr = dadd(HR, p.lambda);
    if (!(HL >= p.mcw && HR >= p.mcw && xl > 0.0 && xr > 0.0)) return -1.0;
    return dadd(dmul(dmul(GL, GL), rcp_refined(xl)), dmul(dmul(GR, GR), rcp_refined(xr)));
}
constexpr double SCREEN_KEEP = 1.0 - 0x1p-16;

// one default direction of one candidate, exactly (R8 op order)
__device__ __forceinline__ void eval_candidate_dl(long long Pg, long long Ph, long long Mg, long long Mh, long long Tg,
                                                  long long Th, int sg, int sh, double e, const EvalParams &p,
                                                  long long bin_global, int dli, FeatBest &best) {
    const bool dl = dli == 0;
    const long long Lg = Pg + (dl ? Mg : 0), Lh = Ph + (dl ? Mh : 0);
    const double GL = fixed_to_double(Lg, sg), HL = fixed_to_double(Lh, sh);
    const double GR = fixed_to_double(Tg - Lg, sg), HR = fixed_to_double(Th - Lh, sh);
    if (!(HL >= p.mcw && HR >= p.mcw && dadd(HL, p.lambda) > 0.0 && dadd(HR, p.lambda) > 0.0)) return;
    double aa = dmul(GL, GL);
    aa = ddiv(aa, dadd(HL, p.lambda));
    double cc = dmul(GR, GR);
    cc = ddiv(cc, dadd(HR, p.lambda));
    double d = dadd(aa, cc);
    d = dsub(d, e);
    d = dmul(0.5, d);
    const double gain = dsub(d, p.gamma);
    const long long idx = bin_global * 2 + dli;
    if (better(gain, idx, best.gain, best.idx)) {
        best.gain = gain;
        best.idx = idx;
        best.Lg = Lg;
        best.Lh = Lh;
    }
}

// Best candidate of feature f of one node, computed by one warp (valid in every lane).
// Register-blocked: lane owns KB consecutive bins of each 32*KB-bin chunk, so all histogram
// loads of a chunk are in flight together; the prefix is a per-lane serial scan plus one warp
// scan of the lane totals.
// warp variant: bins per lane per chunk, and resident blocks it is compiled for.  Measured
// (Epsilon evaluation, ms/round): KB 2 at 4 blocks (64 registers) spills ~1.7 KB per thread, 0.84;
// KB 2 at 2 blocks (no spills) 0.69; KB 4 / 2 blocks 0.77; KB 8 / 2 blocks 0.90; KB 8 / 1 1.18
// (Bosch 0.56 -> 0.48 at KB 2 / 2 blocks)
#ifndef GBM_EVAL_KB
#define GBM_EVAL_KB 2
#endif
#ifndef GBM_EVAL_MINB
#define GBM_EVAL_MINB 2
#endif
constexpr int KB = GBM_EVAL_KB;
__device__ FeatBest eval_feature(const NodeHist &src, int b0, int nbf, long long Tg, long long Th, int sg, int sh,
                                 double e, const EvalParams &p) {
    const int lane = threadIdx.x & 31;
    constexpr int CH = 32 * KB;
    long long Mg, Mh;
    long long vg[KB], vh[KB];
    auto load_chunk = [&](int c) {
#pragma unroll
        for (int i = 0; i < KB; ++i) {
            const int b = c + lane * KB + i;
            vg[i] = vh[i] = 0;
            if (b < nbf) {
                src.get(b0 + b, vg[i], vh[i]);
                if (src.store) src.put(b0 + b, vg[i], vh[i]);
            }
        }
    };
    auto warp_sum = [&](long long x) {
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        return x;
    };
    if (nbf <= CH) {
        load_chunk(0);
    } else {  // wide features: totals first
        long long sg2 = 0, sh2 = 0;
        for (int b = lane; b < nbf; b += 32) {
            long long g, h;
            src.get(b0 + b, g, h);
            sg2 += g;
            sh2 += h;
        }
        Mg = Tg - warp_sum(sg2);
        Mh = Th - warp_sum(sh2);
    }
    FeatBest best;
    best.gain = 0.0;
    best.idx = LLONG_MAX;
    best.Lg = best.Lh = 0;
    long long cg = 0, ch = 0;  // prefix of earlier chunks
    for (int c = 0; c < nbf; c += CH) {
        if (c > 0 || nbf > CH) load_chunk(c);
        long long lg = 0, lh = 0;
#pragma unroll
        for (int i = 0; i < KB; ++i) {
            lg += vg[i];
            lh += vh[i];
        }
        long long xg = lg, xh = lh;  // inclusive warp scan of lane totals
        for (int o = 1; o < 32; o <<= 1) {
            const long long yg = __shfl_up_sync(0xffffffffu, xg, o), yh = __shfl_up_sync(0xffffffffu, xh, o);
            if (lane >= o) {
                xg += yg;
                xh += yh;
            }
        }
        if (nbf <= CH) {  // single chunk: the feature sum is the scan's total
            Mg = Tg - __shfl_sync(0xffffffffu, xg, 31);
            Mh = Th - __shfl_sync(0xffffffffu, xh, 31);
        }
        const long long Pg0 = cg + xg - lg, Ph0 = ch + xh - lh;
        if (p.screen) {
            const int n_dl = (Mg == 0 && Mh == 0) ? 1 : 2;  // (see eval_candidate)
            double sc[KB][2];
            double smax = -1.0;
            long long Pg = Pg0, Ph = Ph0;
#pragma unroll
            for (int i = 0; i < KB; ++i) {
                const int b = c + lane * KB + i;
                Pg += vg[i];
                Ph += vh[i];
#pragma unroll
                for (int dli = 0; dli < 2; ++dli) {
                    sc[i][dli] = (b < nbf && dli < n_dl) ? screen_score(Pg, Ph, Mg, Mh, Tg, Th, sg, sh, p, dli) : -1.0;
                    smax = fmax(smax, sc[i][dli]);
                }
            }
            for (int o = 16; o > 0; o >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
            const double thr = smax * SCREEN_KEEP;
            Pg = Pg0;
            Ph = Ph0;
#pragma unroll
            for (int i = 0; i < KB; ++i) {
                const int b = c + lane * KB + i;
                Pg += vg[i];
                Ph += vh[i];
#pragma unroll
                for (int dli = 0; dli < 2; ++dli)
                    if (sc[i][dli] >= 0.0 && sc[i][dli] >= thr)
                        eval_candidate_dl(Pg, Ph, Mg, Mh, Tg, Th, sg, sh, e, p, (long long)(b0 + b), dli, best);
            }
        } else {
            long long Pg = Pg0, Ph = Ph0;
#pragma unroll
            for (int i = 0; i < KB; ++i) {
                const int b = c + lane * KB + i;
                Pg += vg[i];
                Ph += vh[i];
                if (b < nbf) eval_candidate(Pg, Ph, Mg, Mh, Tg, Th, sg, sh, e, p, (long long)(b0 + b), best);
            }
        }
        cg += __shfl_sync(0xffffffffu, xg, 31);
        ch += __shfl_sync(0xffffffffu, xh, 31);
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double og = __shfl_xor_sync(0xffffffffu, best.gain, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, best.idx, o);
        const long long olg = __shfl_xor_sync(0xffffffffu, best.Lg, o), olh = __shfl_xor_sync(0xffffffffu, best.Lh, o);
        if (better(og, oi, best.gain, best.idx)) {
            best.gain = og;
            best.idx = oi;
            best.Lg = olg;
            best.Lh = olh;
        }
    }
    return best;
}

// Block-per-feature variant: thread t owns bin c+t of each E_THREADS-bin chunk, so one thread
// evaluates one candidate (two with missing mass) -- the latency of a feature is one candidate
// plus a block scan, where the warp variant runs KB candidates back to back per lane.
constexpr int EWPB = E_THREADS / 32;
// block-wide inclusive scan of an int64 pair; also returns the block totals
__device__ __forceinline__ void block_scan2(long long &g, long long &h, long long &tot_g, long long &tot_h) {
    __shared__ long long s_sg[EWPB], s_sh[EWPB];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        const long long yg = __shfl_up_sync(0xffffffffu, g, o), yh = __shfl_up_sync(0xffffffffu, h, o);
        if (lane >= o) {
            g += yg;
            h += yh;
        }
    }
    if (lane == 31) {
        s_sg[w] = g;
        s_sh[w] = h;
    }
    __syncthreads();
    long long pg = 0, ph = 0, tg = 0, th = 0;
#pragma unroll
    for (int i = 0; i < EWPB; ++i) {
        if (i < w) {
            pg += s_sg[i];
            ph += s_sh[i];
        }
        tg += s_sg[i];
        th += s_sh[i];
    }
    g += pg;
    h += ph;
    tot_g = tg;
    tot_h = th;
    __syncthreads();
}

// canonical argmax over the block; the result is valid in thread 0
__device__ __forceinline__ FeatBest block_best(FeatBest b) {
    __shared__ double s_g[EWPB];
    __shared__ long long s_i[EWPB], s_lg[EWPB], s_lh[EWPB];
    for (int o = 16; o > 0; o >>= 1) {
        const double og = __shfl_xor_sync(0xffffffffu, b.gain, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, b.idx, o);
        const long long olg = __shfl_xor_sync(0xffffffffu, b.Lg, o), olh = __shfl_xor_sync(0xffffffffu, b.Lh, o);
        if (better(og, oi, b.gain, b.idx)) {
            b.gain = og; b.idx = oi; b.Lg = olg; b.Lh = olh;
        }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_g[w] = b.gain; s_i[w] = b.idx; s_lg[w] = b.Lg; s_lh[w] = b.Lh;
    }
    __syncthreads();
    FeatBest r;
    r.gain = s_g[0]; r.idx = s_i[0]; r.Lg = s_lg[0]; r.Lh = s_lh[0];
    for (int i = 1; i < EWPB; ++i)
        if (better(s_g[i], s_i[i], r.gain, r.idx)) {
            r.gain = s_g[i]; r.idx = s_i[i]; r.Lg = s_lg[i]; r.Lh = s_lh[i];
        }
    __syncthreads();
    return r;
}

// Best candidate of feature f of one node, computed by the whole block (valid in thread 0).
__device__ FeatBest eval_feature_blk(const NodeHist &src, int b0, int nbf, long long Tg, long long Th, int sg, int sh,
                                     double e, const EvalParams &p) {
    long long Mg = 0, Mh = 0;
    if (nbf > E_THREADS) {  // wide features: totals first
        long long g2 = 0, h2 = 0, tg, th;
        for (int b = threadIdx.x; b < nbf; b += E_THREADS) {
            long long g, h;
            src.get(b0 + b, g, h);
            g2 += g;
            h2 += h;
        }
        block_scan2(g2, h2, tg, th);
        Mg = Tg - tg;
        Mh = Th - th;
    }
    FeatBest best;
    best.gain = 0.0;
    best.idx = LLONG_MAX;
    best.Lg = best.Lh = 0;
    long long cg = 0, ch = 0;  // prefix of earlier chunks
    for (int c = 0; c < nbf; c += E_THREADS) {
        const int b = c + (int)threadIdx.x;
        long long vg = 0, vh = 0;
        if (b < nbf) {
            src.get(b0 + b, vg, vh);
            if (src.store) src.put(b0 + b, vg, vh);
        }
        long long tg, th;
        block_scan2(vg, vh, tg, th);
        if (nbf <= E_THREADS) {  // single chunk: the feature sum is the scan's total
            Mg = Tg - tg;
            Mh = Th - th;
        }
        if (p.screen) {
            __shared__ double s_max[EWPB];
            const int n_dl = (Mg == 0 && Mh == 0) ? 1 : 2;
            double sc[2];
            double smax = -1.0;
#pragma unroll
            for (int dli = 0; dli < 2; ++dli) {
                sc[dli] = (b < nbf && dli < n_dl) ? screen_score(cg + vg, ch + vh, Mg, Mh, Tg, Th, sg, sh, p, dli) : -1.0;
                smax = fmax(smax, sc[dli]);
            }
            for (int o = 16; o > 0; o >>= 1) smax = fmax(smax, __shfl_xor_sync(0xffffffffu, smax, o));
            if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = smax;
            __syncthreads();
#pragma unroll
            for (int i = 0; i < EWPB; ++i) smax = fmax(smax, s_max[i]);
            __syncthreads();
            const double thr = smax * SCREEN_KEEP;
#pragma unroll
            for (int dli = 0; dli < 2; ++dli)
                if (sc[dli] >= 0.0 && sc[dli] >= thr)
                    eval_candidate_dl(cg + vg, ch + vh, Mg, Mh, Tg, Th, sg, sh, e, p, (long long)(b0 + b), dli, best);
        } else if (b < nbf) {
            eval_candidate(cg + vg, ch + vh, Mg, Mh, Tg, Th, sg, sh, e, p, (long long)(b0 + b), best);
        }
        cg += tg;
        ch += th;
    }
    return block_best(best);
}

struct EvalArgs {
    int level, first, F, n_nodes;
    // tree mode: the last eval_final block plans the next level's partition (plan_block)
    unsigned *done;                 // tree mode: completed-node counter (reset by the last block)
    unsigned *node_done;            // tree mode: [n_nodes] finished warps per node (reset by finishers)
    int plan_mode;                  // tree mode, last block: 0 nothing, 1 plan the next level,
                                    // 2 loss-guided pop of step sel_step (R25)
    int sel_step;
    int *tile_left;                 // loss-guided: zeroed for the popped node's tiles
    int plan_groups, plan_run;
    int plan_split_only;            // record level path: items only for split parents
    int plan_run_min;               // loss-guided: smallest work item (tiles)
    long long plan_rows;            // this rank's rows (plan_run < 0: tiles per item sized per level)
    int *tile_base, *run_base, *n_items;
    long long TB;
    const int32_t *cut_ptr;
    const float *cut_values;
    const int32_t *scale;
    EvalParams p;
    NodeDev *nodes;                 // tree mode
    const long long *hist_root;     // tree mode: root hist + totals
    const long long *hist_build;    // tree mode: built children, per parent slot
    const long long *hist_prev;     // tree mode: parent level hists
    long long *hist_store;          // tree mode: this level's hists (or null)
    const long long *hist_direct;   // direct mode: [n_nodes][TB][2]
    const long long *totals_direct; // direct mode: [n_nodes][2]
    FeatBest *fb;                   // [n_nodes][F]
    LgNode *lg;                     // loss-guided mode (null = depth-wise)
    const StepDev *step;            // loss-guided: the current expansion
    StepDev *step_next;             // loss-guided: written by the pop of the next step
    long long *hist_pool;           // loss-guided: [max_leaves][TB][2] by LgNode::hslot
    // reduce-scatter + feature-sliced evaluation (GBM_OPT_EVAL_SLICED): this rank evaluates the
    // features f0 .. f0 + F - 1 into fb (its histograms hold only their bins, slot stride TB =
    // the slice capacity, base pointers shifted by the slice's first bin); the finisher reduces
    // the all-gathered fb_all [nslices][n_nodes][fsmax] of every rank
    int f0;
    int sliced;                     // 1: feature evaluation only (the finisher runs separately)
    const long long *root_tot;      // root totals (null: hist_root[2 TB])
    const FeatBest *fb_all;
    const int *slice_f0, *slice_nf;
    int nslices, fsmax;
};

// Node j's histogram source and totals; false if the node does not exist.
__device__ __forceinline__ bool node_source(const EvalArgs &a, int j, NodeHist &src, long long &Tg, long long &Th) {
    src.direct = src.parent = src.build = nullptr;
    src.store = nullptr;
    if (a.hist_direct) {
        src.direct = a.hist_direct + (long long)j * a.TB * 2;
        Tg = a.totals_direct[2 * j];
        Th = a.totals_direct[2 * j + 1];
        return true;
    }
    const int k = a.first + j;
    if (a.lg && a.level > 0) {  // loss-guided child k of the step's parent
        const int pk = a.step->k;
        if (pk < 0) return false;
        Tg = a.nodes[k].Tg;
        Th = a.nodes[k].Th;
        const bool is_left = k == a.step->c;
        const bool built = a.nodes[pk].build_left ? is_left : !is_left;
        if (built) {
            src.direct = a.hist_build;
        } else {  // in place: the sibling's histogram replaces the parent's in its pool slot
            src.parent = a.hist_pool + (long long)a.lg[pk].hslot * a.TB * 2;
            src.build = a.hist_build;
        }
        if (a.lg[k].depth < a.p.max_depth) src.store = a.hist_pool + (long long)a.lg[k].hslot * a.TB * 2;
        return true;
    }
    if (a.level == 0) {
        src.direct = a.hist_root;
        Tg = a.root_tot ? a.root_tot[0] : a.hist_root[2 * a.TB];
        Th = a.root_tot ? a.root_tot[1] : a.hist_root[2 * a.TB + 1];
    } else {
        const int pk = (k - 1) / 2;
        const int pslot = pk - ((1 << (a.level - 1)) - 1);
        if (a.nodes[pk].state != GBM_NODE_SPLIT) return false;
        Tg = a.nodes[k].Tg;
        Th = a.nodes[k].Th;
        const bool is_left = (k & 1) == 1;
        const bool built = a.nodes[pk].build_left ? is_left : !is_left;
        const long long *bh = a.hist_build + (long long)pslot * a.TB * 2;
        if (built) {
            src.direct = bh;
        } else {
            src.parent = a.level == 1 ? a.hist_root : a.hist_prev + (long long)pslot * a.TB * 2;
            src.build = bh;
        }
    }
    if (a.hist_store) src.store = a.hist_store + (long long)j * a.TB * 2;
    return true;
}

// one warp per (node, feature): the feature's best candidate into fb[gw]
__device__ __forceinline__ void eval_warp(const EvalArgs &a, long long gw) {
    const int j = (int)(gw / a.F), f = (int)(gw - (long long)j * a.F);
    NodeHist src;
    long long Tg, Th;
    if (!node_source(a, j, src, Tg, Th)) return;
    if (a.lg && a.lg[a.first + j].depth >= a.p.max_depth) return;  // a leaf: not evaluated
    const int sg = a.scale[0], sh = a.scale[1];
    const double G = fixed_to_double(Tg, sg), H = fixed_to_double(Th, sh);
    const double e = ddiv(dmul(G, G), dadd(H, a.p.lambda));
    const int fg = a.f0 + f;
    const int b0 = __ldg(a.cut_ptr + fg), nbf = __ldg(a.cut_ptr + fg + 1) - b0;
    const FeatBest b = eval_feature(src, b0, nbf, Tg, Th, sg, sh, e, a.p);
    if ((threadIdx.x & 31) == 0) a.fb[a.sliced ? (long long)j * a.fsmax + f : gw] = b;
}

// one block per (node, feature) = blk: the feature's best candidate into fb[blk]
__device__ __forceinline__ NodeKnown eval_block(const EvalArgs &a, long long blk) {
    const int j = (int)(blk / a.F), f = (int)(blk - (long long)j * a.F);
    NodeHist src;
    long long Tg, Th;
    if (!node_source(a, j, src, Tg, Th)) return NodeKnown{2, 0, 0};               // block-uniform
    if (a.lg && a.lg[a.first + j].depth >= a.p.max_depth) return NodeKnown{1, Tg, Th};  // a leaf
    const int sg = a.scale[0], sh = a.scale[1];
    const double G = fixed_to_double(Tg, sg), H = fixed_to_double(Th, sh);
    const double e = ddiv(dmul(G, G), dadd(H, a.p.lambda));
    const int fg = a.f0 + f;
    const int b0 = __ldg(a.cut_ptr + fg), nbf = __ldg(a.cut_ptr + fg + 1) - b0;
    const FeatBest b = eval_feature_blk(src, b0, nbf, Tg, Th, sg, sh, e, a.p);
    if (threadIdx.x == 0) a.fb[a.sliced ? (long long)j * a.fsmax + f : blk] = b;
    return NodeKnown{1, Tg, Th};
}

__global__ void __launch_bounds__(E_THREADS) eval_feat_kernel(EvalArgs a) {
    const long long gw = ((long long)blockIdx.x * E_THREADS + threadIdx.x) >> 5;
    if (gw < (long long)a.n_nodes * a.F) eval_warp(a, gw);
}

__global__ void __launch_bounds__(E_THREADS) eval_feat_blk_kernel(EvalArgs a) { eval_block(a, blockIdx.x); }

__device__ __forceinline__ double leaf_weight(long long Tg, long long Th, int sg, int sh, double lambda, double eta) {
    const double G = fixed_to_double(Tg, sg), H = fixed_to_double(Th, sh);
    const double t = dadd(H, lambda);
    if (t == 0.0) return 0.0;
    double w = ddiv(G, t);
    w = -w;
    return dmul(w, eta);
}

__device__ __forceinline__ void write_leaf(const TreeDev &t, int k, long long Tg, long long Th, int sg, int sh,
                                           const EvalParams &p) {
    t.kind[k] = GBM_NODE_LEAF;
    t.sum_qg[k] = Tg;
    t.sum_qh[k] = Th;
    t.weight[k] = leaf_weight(Tg, Th, sg, sh, p.lambda, p.eta);
}


// block-wide canonical argmax over the features of node j
__device__ FeatBest reduce_node(const EvalArgs &a, int j, int &feat) {
    __shared__ double s_g[E_THREADS / 32];
    __shared__ long long s_i[E_THREADS / 32], s_lg[E_THREADS / 32], s_lh[E_THREADS / 32];
    __shared__ int s_f[E_THREADS / 32];
    double bg = 0.0;
    long long bi = LLONG_MAX, blg = 0, blh = 0;
    int bf = -1;  // feature of the best candidate (no binary search over cut_ptr afterwards)
    const int nf_all = a.fb_all ? a.nslices * a.fsmax : a.F;
    for (int i = threadIdx.x; i < nf_all; i += E_THREADS) {
        const FeatBest *cp;
        int f;
        if (a.fb_all) {  // sliced: rank r's entries for node j, its features slice_f0[r] + fl
            const int r = i / a.fsmax, fl = i - r * a.fsmax;
            if (fl >= __ldg(a.slice_nf + r)) continue;
            cp = a.fb_all + ((long long)r * a.n_nodes + j) * a.fsmax + fl;
            f = __ldg(a.slice_f0 + r) + fl;
        } else {
            cp = a.fb + (long long)j * a.F + i;
            f = i;
        }
        FeatBest c;
        c.gain = __ldcg(&cp->gain);
        c.idx = __ldcg(&cp->idx);
        c.Lg = __ldcg(&cp->Lg);
        c.Lh = __ldcg(&cp->Lh);
        if (better(c.gain, c.idx, bg, bi)) {
            bg = c.gain; bi = c.idx; blg = c.Lg; blh = c.Lh; bf = f;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double og = __shfl_xor_sync(0xffffffffu, bg, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const long long olg = __shfl_xor_sync(0xffffffffu, blg, o), olh = __shfl_xor_sync(0xffffffffu, blh, o);
        const int of = __shfl_xor_sync(0xffffffffu, bf, o);
        if (better(og, oi, bg, bi)) {
            bg = og; bi = oi; blg = olg; blh = olh; bf = of;
        }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_g[w] = bg; s_i[w] = bi; s_lg[w] = blg; s_lh[w] = blh; s_f[w] = bf;
    }
    __syncthreads();
    FeatBest r;
    r.gain = s_g[0]; r.idx = s_i[0]; r.Lg = s_lg[0]; r.Lh = s_lh[0];
    feat = s_f[0];
    for (int i = 1; i < E_THREADS / 32; ++i)
        if (better(s_g[i], s_i[i], r.gain, r.idx)) {
            r.gain = s_g[i]; r.idx = s_i[i]; r.Lg = s_lg[i]; r.Lh = s_lh[i]; feat = s_f[i];
        }
    return r;
}


__device__ void eval_final_body(const EvalArgs &a, const TreeDev &t, int j, NodeKnown kn);
__device__ void lg_select_block(const EvalArgs &a, const TreeDev &t, int s);

// Tree mode, one launch per level / loss-guided step: warp per (node, feature) evaluation; the
// block that completes a node's last feature reduces that node (eval_final_body); the block that
// completes the last node plans the next level (plan_mode 1) or pops the next loss-guided
// expansion (plan_mode 2).  Threadfence + counter pattern: every fb / node write is fenced
// before the counter it is published by, and the finisher fences before reading.
// nodes fin[0..nfin) were completed by this block: reduce them; count them; the block that
// completes the level plans / pops the next step
__device__ void eval_finish(const EvalArgs &a, const TreeDev &t, const int *fin, int nfin,
                            const NodeKnown *known) {
    __shared__ bool s_last;
    __threadfence();
    for (int i = 0; i < nfin; ++i) {
        const int j = fin[i];
        eval_final_body(a, t, j, known ? known[i] : NodeKnown{0, 0, 0});
        __syncthreads();
        if (threadIdx.x == 0) a.node_done[j] = 0;
    }
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(a.done, (unsigned)nfin) + nfin == (unsigned)a.n_nodes;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (a.plan_mode == 1)  // the children of this level are the next level's parents
        plan_block(a.nodes, a.first, a.n_nodes, a.plan_groups, a.plan_run, a.tile_base, a.run_base, a.n_items,
                   a.plan_split_only != 0, a.plan_rows);
    else if (a.plan_mode == 2)
        lg_select_block(a, t, a.sel_step);
    if (threadIdx.x == 0) *a.done = 0;
}

__global__ void __launch_bounds__(E_THREADS, GBM_EVAL_MINB) eval_tree_kernel(EvalArgs a, TreeDev t) {
    constexpr int WPB = E_THREADS / 32;
    __shared__ int s_fin[WPB + 1];
    __shared__ int s_nfin;
    const long long total = (long long)a.n_nodes * a.F;
    const long long gw = ((long long)blockIdx.x * E_THREADS + threadIdx.x) >> 5;
    if (gw < total) eval_warp(a, gw);
    if (a.sliced) return;  // the finisher runs after the all-gather of fb
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        int nf = 0;
        const long long w1 = min(total, (long long)(blockIdx.x + 1) * WPB);
        for (long long w = (long long)blockIdx.x * WPB; w < w1;) {
            const int j = (int)(w / a.F);
            const long long we = min(w1, (long long)(j + 1) * a.F);
            const unsigned cnt = (unsigned)(we - w);
            if (atomicAdd(a.node_done + j, cnt) + cnt == (unsigned)a.F) s_fin[nf++] = j;
            w = we;
        }
        s_nfin = nf;
    }
    __syncthreads();
    if (s_nfin == 0) return;
    eval_finish(a, t, s_fin, s_nfin, nullptr);
}

// block per (node, feature); the block completing a node's last feature reduces the node
__global__ void __launch_bounds__(E_THREADS) eval_tree_blk_kernel(EvalArgs a, TreeDev t) {
    __shared__ int s_fin[1];
    __shared__ int s_nfin;
    const long long blk = blockIdx.x;
    const NodeKnown kn = eval_block(a, blk);
    if (a.sliced) return;  // the finisher runs after the all-gather of fb
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int j = (int)(blk / a.F);
        s_fin[0] = j;
        s_nfin = atomicAdd(a.node_done + j, 1u) + 1 == (unsigned)a.F ? 1 : 0;
    }
    __syncthreads();
    if (s_nfin == 0) return;
    eval_finish(a, t, s_fin, 1, &kn);
}

// sliced evaluation: one block per node reduces the all-gathered candidates of every rank; the
// block completing the level plans the next one (eval_finish)
__global__ void __launch_bounds__(E_THREADS) eval_final_sliced_kernel(EvalArgs a, TreeDev t) {
    const int fin = blockIdx.x;
    eval_finish(a, t, &fin, 1, nullptr);
}

// send[r][slot][CB][2] = this rank's partial histograms cut into the ranks' feature slices
// (bins bin_lo[r] .. bin_lo[r+1]), zero-padded to the slice capacity CB: the reduce-scatter
// input of the sliced evaluation
__global__ void slice_permute_kernel(const long long *__restrict__ hist, int n_slots, long long TB,
                                     const int *__restrict__ bin_lo, int p, long long CB,
                                     long long *__restrict__ send) {
    const long long total = (long long)p * n_slots * CB;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long b = i % CB, rs = i / CB;
        const int slot = (int)(rs % n_slots), r = (int)(rs / n_slots);
        const long long g = bin_lo[r] + b;
        long long vg = 0, vh = 0;
        if (g < bin_lo[r + 1]) {
            vg = hist[(slot * TB + g) * 2];
            vh = hist[(slot * TB + g) * 2 + 1];
        }
        send[2 * i] = vg;
        send[2 * i + 1] = vh;
    }
}

__device__ void eval_final_body(const EvalArgs &a, const TreeDev &t, int j, NodeKnown kn) {
    const int k = a.first + j;
    NodeHist src;
    long long Tg = kn.Tg, Th = kn.Th;
    const bool exists = kn.state == 0 ? node_source(a, j, src, Tg, Th) : kn.state == 1;
    if (!exists) {
        if (threadIdx.x == 0) a.nodes[k].state = GBM_NODE_ABSENT;
        return;
    }
    const int sg = a.scale[0], sh = a.scale[1];
    const EvalParams &p = a.p;
    if ((a.lg ? a.lg[k].depth : a.level) >= p.max_depth) {  // max_depth == 0: the root is a leaf
        if (threadIdx.x == 0) {
            write_leaf(t, k, Tg, Th, sg, sh, p);
            a.nodes[k].state = GBM_NODE_LEAF;
            a.nodes[k].Tg = Tg;
            a.nodes[k].Th = Th;
        }
        return;
    }
    int f;
    const FeatBest b = reduce_node(a, j, f);
    if (threadIdx.x != 0) return;
    NodeDev &nd = a.nodes[k];
    nd.Tg = Tg;
    nd.Th = Th;
    const bool split = b.idx != LLONG_MAX && b.gain > 0.0;
    t.sum_qg[k] = Tg;
    t.sum_qh[k] = Th;
    t.weight[k] = leaf_weight(Tg, Th, sg, sh, p.lambda, p.eta);
    if (!split) {
        t.kind[k] = GBM_NODE_LEAF;
        nd.state = GBM_NODE_LEAF;
        return;
    }
    const int gbin = (int)(b.idx >> 1), dl = (b.idx & 1) == 0;
    const int bb = gbin - __ldg(a.cut_ptr + f);
    if (a.lg) {  // loss-guided: a leaf until lg_select_kernel pops it (R25)
        t.kind[k] = GBM_NODE_LEAF;
        nd.state = NODE_OPEN;
        nd.f = f;
        nd.b = bb;
        nd.dl = dl;
        nd.build_left = b.Lh <= Th - b.Lh;  // smaller hessian sum; ties -> left (R17)
        a.lg[k].gain = b.gain;
        a.lg[k].Lg = b.Lg;
        a.lg[k].Lh = b.Lh;
        return;
    }
    t.kind[k] = GBM_NODE_SPLIT;
    t.feature[k] = f;
    t.bin[k] = bb;
    t.threshold[k] = __ldg(a.cut_values + gbin);
    t.default_left[k] = (int8_t)dl;
    t.gain[k] = b.gain;
    if (t.left_child) t.left_child[k] = 2 * k + 1;
    nd.state = GBM_NODE_SPLIT;
    nd.f = f;
    nd.b = bb;
    nd.dl = dl;
    const long long Lg = b.Lg, Lh = b.Lh, Rg = Tg - b.Lg, Rh = Th - b.Lh;
    nd.build_left = Lh <= Rh;  // smaller hessian sum; ties -> left (R17)
    a.nodes[2 * k + 1].Tg = Lg;
    a.nodes[2 * k + 1].Th = Lh;
    a.nodes[2 * k + 2].Tg = Rg;
    a.nodes[2 * k + 2].Th = Rh;
    if (a.level + 1 == p.max_depth) {  // children at depth D are leaves
        write_leaf(t, 2 * k + 1, Lg, Lh, sg, sh, p);
        write_leaf(t, 2 * k + 2, Rg, Rh, sg, sh, p);
    }
}

// direct mode (gbm_evaluate_splits)
__global__ void __launch_bounds__(E_THREADS) eval_out_kernel(EvalArgs a, int8_t *split_d, int32_t *feature_d,
                                                             int32_t *bin_d, int8_t *dl_d, double *gain_d,
                                                             long long *child_d) {
    const int j = blockIdx.x;
    int bf;
    const FeatBest b = reduce_node(a, j, bf);
    if (threadIdx.x != 0) return;
    const long long Tg = a.totals_direct[2 * j], Th = a.totals_direct[2 * j + 1];
    const bool found = b.idx != LLONG_MAX;
    split_d[j] = found && b.gain > 0.0;
    gain_d[j] = found ? b.gain : 0.0;
    int f = -1, bb = -1, dl = 0;
    if (found) {
        const int gbin = (int)(b.idx >> 1);
        dl = (b.idx & 1) == 0;
        f = bf;
        bb = gbin - __ldg(a.cut_ptr + f);
    }
    feature_d[j] = f;
    bin_d[j] = bb;
    dl_d[j] = (int8_t)dl;
    child_d[4 * j + 0] = found ? b.Lg : 0;
    child_d[4 * j + 1] = found ? b.Lh : 0;
    child_d[4 * j + 2] = found ? Tg - b.Lg : 0;
    child_d[4 * j + 3] = found ? Th - b.Lh : 0;
}

__global__ void init_tree_kernel(TreeDev t, long long cap, NodeDev *nodes, long long n_rows) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < cap;
         k += (long long)gridDim.x * blockDim.x) {
        t.kind[k] = GBM_NODE_ABSENT;
        t.feature[k] = -1;
        t.bin[k] = -1;
        t.threshold[k] = 0.0f;
        t.default_left[k] = 0;
        t.gain[k] = 0.0;
        t.weight[k] = 0.0;
        t.sum_qg[k] = 0;
        t.sum_qh[k] = 0;
        if (t.left_child) t.left_child[k] = -1;
        NodeDev nd = {};
        nodes[k] = nd;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        nodes[0].start = 0;
        nodes[0].count = n_rows;
    }
}

// ============================================================== loss-guided growth (R25-R27)
__global__ void lg_init_kernel(LgNode *__restrict__ lg, long long cap) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < cap;
         k += (long long)gridDim.x * blockDim.x) {
        LgNode z = {};
        z.buf = k == 0 ? -1 : 0;  // the root's rows are the identity list
        lg[k] = z;
    }
}

// Step s: expand_queue.pop() -- the OPEN node of largest gain, ties to the smaller id (R25) --
// made a split node with children 2s+1, 2s+2 (R27); plans the step's single-parent partition
// and zeroes its tile counters.  With nothing OPEN the step is void: k = -1 and zero work items,
// so every launch of the step returns at once (the host enqueues a fixed max_leaves - 1 steps:
// graph-capturable).  Runs in the last block of the previous evaluation (any block size).
__device__ void lg_select_block(const EvalArgs &a, const TreeDev &t, int s) {
    __shared__ double s_g[32];
    __shared__ int s_k[32];
    __shared__ long long s_tiles;
    NodeDev *nodes = a.nodes;
    LgNode *lg = a.lg;
    const int n_nodes = 2 * s + 1;
    double bg = 0.0;
    int bk = -1;
    auto take = [&](double g, int k) {
        if (k >= 0 && (bk < 0 || g > bg || (g == bg && k < bk))) {
            bg = g;
            bk = k;
        }
    };
    for (int k = threadIdx.x; k < n_nodes; k += blockDim.x)
        if (__ldcg(&nodes[k].state) == NODE_OPEN) take(__ldcg(&lg[k].gain), k);
    for (int o = 16; o > 0; o >>= 1) {
        const double og = __shfl_xor_sync(0xffffffffu, bg, o);
        const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
        take(og, ok);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_g[w] = bg;
        s_k[w] = bk;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) take(s_g[i], s_k[i]);
        const int c = 2 * s + 1;
        StepDev *step = a.step_next;
        s_tiles = 0;
        if (bk < 0) {
            step->k = -1;
            step->c = c;
            step->in_buf = step->out_buf = 0;
            step->run_tiles = 1;
            a.tile_base[0] = a.tile_base[1] = 0;
            a.run_base[0] = a.run_base[1] = 0;
            a.n_items[0] = a.n_items[1] = 0;
            a.n_items[2] = 1;
        } else {
            const int k = bk;
            NodeDev &nd = nodes[k];
            nd.state = GBM_NODE_SPLIT;
            t.kind[k] = GBM_NODE_SPLIT;
            t.feature[k] = nd.f;
            t.bin[k] = nd.b;
            t.threshold[k] = __ldg(a.cut_values + __ldg(a.cut_ptr + nd.f) + nd.b);
            t.default_left[k] = (int8_t)nd.dl;
            t.gain[k] = lg[k].gain;
            t.left_child[k] = c;
            NodeDev L = {}, R = {};
            L.Tg = lg[k].Lg;
            L.Th = lg[k].Lh;
            R.Tg = nd.Tg - lg[k].Lg;
            R.Th = nd.Th - lg[k].Lh;
            L.state = R.state = GBM_NODE_ABSENT;  // set by the children's evaluation
            nodes[c] = L;                        // start / count: part_scan_kernel
            nodes[c + 1] = R;
            const int in = lg[k].buf, out = in < 0 ? 0 : 1 - in;
            const int built = nd.build_left ? c : c + 1;
            for (int i = 0; i < 2; ++i) {
                LgNode z = {};
                z.depth = lg[k].depth + 1;
                z.hslot = (c + i == built) ? s + 1 : lg[k].hslot;  // the sibling takes the parent's slot
                z.buf = out;
                lg[c + i] = z;
            }
            step->k = k;
            step->c = c;
            step->in_buf = in;
            step->out_buf = out;
            const long long tiles = nd.count > 0 ? (nd.count + PT - 1) / PT : 0;
            // about plan_run (4 x resident blocks) items for this parent (the depth-wise rule)
            const long long rt = max((long long)a.plan_run_min,
                                     min((long long)(MAX_CHUNK / PT), (tiles * a.plan_groups + a.plan_run - 1) / a.plan_run));
            const long long runs = (tiles + rt - 1) / rt;
            step->run_tiles = (int)rt;
            a.tile_base[0] = 0;
            a.tile_base[1] = (int)tiles;
            a.run_base[0] = 0;
            a.run_base[1] = (int)runs;
            a.n_items[0] = (int)runs * a.plan_groups;
            a.n_items[1] = 0;
            a.n_items[2] = (int)rt;
            s_tiles = tiles;
        }
    }
    __syncthreads();
    for (long long i = threadIdx.x; i < s_tiles; i += blockDim.x) a.tile_left[i] = 0;
}

// every row's leaf: walk the linked tree from the root in row order (coalesced row_leaf)
__global__ void __launch_bounds__(WALK_THREADS) lg_walk_kernel(QM qm, TreeDev t, long long n,
                                                               int32_t *__restrict__ row_leaf) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
         r += (long long)gridDim.x * blockDim.x) {
        int k = 0;
        while (__ldg(t.kind + k) == GBM_NODE_SPLIT) {
            const int sym = (int)split_symbol(qm, r, __ldg(t.feature + k));
            const bool left = sym == qm.B ? __ldg(t.default_left + k) != 0 : sym <= __ldg(t.bin + k);
            const int c = __ldg(t.left_child + k);
            k = left ? c : c + 1;
        }
        row_leaf[r] = k;
    }
}

// ============================================================== host planning
struct HistPlan {
    std::vector<Group> groups;
    bool wide = false, byte_path = false, sent = false;
    bool carry = false;   // level entries carry the gradient pairs (grad_bits <= 15)
    bool col = false;     // bank-column kernels (every feature has <= rows bins)
    bool staged = false;  // staged bank-column kernels (layout 3: byte symbols, narrow)
    bool cs_r1 = false;   // staged: every group has > 16 features (the one-row-per-instruction kernel)
    std::vector<ColGroup> cgroups;
    int cstride = 0;      // col: words per channel (rows * 32)
    int hstride = 0;      // words per smem channel
    int rep_cap = 0;      // replica words per channel (fused level kernel, byte path)
    int smem_bytes = 0;   // dynamic smem per block
    int blocks_range = 0, blocks_fused = 0;
    int chunk = 0;        // rows per range item
};

template <bool W, bool B, bool S>
static int setup_kernels(gbm_ctx *ctx, HistPlan &hp) {
    GBM_CUDA(cudaFuncSetAttribute(hist_range_kernel<W, B, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
    GBM_CUDA(cudaFuncSetAttribute(part_hist_kernel<W, B, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  hp.smem_bytes));
    if constexpr (!W)
        GBM_CUDA(cudaFuncSetAttribute(part_hist_kernel<W, B, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      hp.smem_bytes));
    GBM_CUDA(cudaFuncSetAttribute(hist_seg_kernel<W, B, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  hp.smem_bytes));
    if constexpr (!W)
        GBM_CUDA(cudaFuncSetAttribute(hist_seg_kernel<W, B, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      hp.smem_bytes));
    int o1 = 0, o2 = 0;
    GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, hist_range_kernel<W, B, S>, H_THREADS, hp.smem_bytes));
    if constexpr (!W)
        GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, part_hist_kernel<W, B, S, true>, H_THREADS,
                                                               hp.smem_bytes));
    else
        GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, part_hist_kernel<W, B, S, false>, H_THREADS,
                                                               hp.smem_bytes));
    if (o1 < 1 || o2 < 1) return fail(GBM_E_ARG, "histogram kernels cannot be resident (shared memory)");
    hp.blocks_range = o1 * ctx->sm_count;
    hp.blocks_fused = o2 * ctx->sm_count;
    return GBM_OK;
}

#define GBM_DISPATCH(hp, F, ...)                                                                  \
    (hp.wide ? (hp.byte_path ? (hp.sent ? F<true, true, true>(__VA_ARGS__) : F<true, true, false>(__VA_ARGS__)) \
                             : F<true, false, false>(__VA_ARGS__))                                 \
             : (hp.byte_path ? (hp.sent ? F<false, true, true>(__VA_ARGS__) : F<false, true, false>(__VA_ARGS__)) \
                             : F<false, false, false>(__VA_ARGS__)))

template <bool W, bool B>
static int setup_col(gbm_ctx *ctx, HistPlan &hp) {
    GBM_CUDA(cudaFuncSetAttribute(hist_col_range_kernel<W, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
    if constexpr (B) {
        GBM_CUDA(cudaFuncSetAttribute(hist_colb_range_kernel<W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      hp.smem_bytes));
        GBM_CUDA(cudaFuncSetAttribute(hist_colb_range_kernel<W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      hp.smem_bytes));
    }
    GBM_CUDA(cudaFuncSetAttribute(part_hist_col_kernel<W, false, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  hp.smem_bytes));
    if constexpr (!W)
        GBM_CUDA(cudaFuncSetAttribute(part_hist_col_kernel<W, true, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      hp.smem_bytes));
    int o1 = 0, o2 = 0;
    GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, hist_col_range_kernel<W, B>, H_THREADS, hp.smem_bytes));
    GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, part_hist_col_kernel<W, !W, B>, H_THREADS, hp.smem_bytes));
    if (o1 < 1 || o2 < 1) return fail(GBM_E_ARG, "column histogram kernels cannot be resident");
    hp.blocks_range = o1 * ctx->sm_count;
    hp.blocks_fused = o2 * ctx->sm_count;
    return GBM_OK;
}

static int plan_hist(gbm_ctx *ctx, const gbm_qmatrix *q, const QM &qm, bool wide, long long rows_hint,
                     HistPlan &hp, int grad_bits = 30, bool allow_col = true, bool staged = false) {
    const int *cp = q->cut_ptr_h;
    hp.wide = wide;
    hp.carry = !wide && grad_bits <= 15 && ctx->carry_gradients;
    // ---- bank-column plan: every feature's bins fit one column of the smem histogram
    {
        const int channels = wide ? 4 : 2;
        const int budget = (int)std::min<size_t>(ctx->smem_optin - 20 * 1024, 200 * 1024);
        int max_nb = 1;
        for (int f = 0; f < qm.F; ++f) max_nb = std::max(max_nb, cp[f + 1] - cp[f]);
        const bool byte_sym = q->bits == 8;
        const int rows = byte_sym ? 256 : (max_nb + 7) / 8 * 8;
        if (staged && byte_sym && !wide && qm.stride % 32 == 0) {  // staged column kernels
            hp.col = hp.staged = true;
            hp.byte_path = true;
            hp.cstride = COLB_STRIDE;
            hp.smem_bytes = 2 * COLB_STRIDE * 4 + (H_THREADS / 32) * (int)sizeof(CsWarp);
            hp.cgroups.clear();
            const int ng = (qm.F + 31) / 32, nu = (qm.F + 3) / 4;
            for (int g = 0; g < ng; ++g) {  // groups of whole 4-feature words, <= 32 features
                ColGroup c;
                c.f_lo = 4 * (int)((long long)nu * g / ng);
                c.f_hi = std::min(qm.F, 4 * (int)((long long)nu * (g + 1) / ng));
                hp.cgroups.push_back(c);
            }
            hp.cs_r1 = true;
            for (auto &c : hp.cgroups) hp.cs_r1 = hp.cs_r1 && c.f_hi - c.f_lo > 16;
            // one group of whole rows: the root may fetch batches by TMA into 2 buffers per warp
            if (hp.cgroups.size() == 1) hp.smem_bytes += (H_THREADS / 32) * (int)sizeof(CsWarp);
            GBM_CUDA(cudaFuncSetAttribute(hist_cs_range_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
            GBM_CUDA(cudaFuncSetAttribute(hist_cs_range_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
            GBM_CUDA(cudaFuncSetAttribute(hist_cs_range_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
            GBM_CUDA(cudaFuncSetAttribute(hist_cs_range_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
            GBM_CUDA(cudaFuncSetAttribute(part_hist_cs_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
            GBM_CUDA(cudaFuncSetAttribute(part_hist_cs_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
            GBM_CUDA(cudaFuncSetAttribute(part_hist_cs_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
            GBM_CUDA(cudaFuncSetAttribute(part_hist_cs_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
            int o1 = 0, o2 = 0;
            GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, hist_cs_range_kernel<true, true>, H_THREADS, hp.smem_bytes));
            GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, part_hist_cs_kernel<false, true>, H_THREADS, hp.smem_bytes));
            if (o1 < 1 || o2 < 1) return fail(GBM_E_ARG, "staged column kernels cannot be resident");
            hp.blocks_range = o1 * ctx->sm_count;
            hp.blocks_fused = o2 * ctx->sm_count;
            const long long G = (long long)hp.cgroups.size();
            long long per = (rows_hint + 2ll * hp.blocks_range - 1) / (2ll * hp.blocks_range) * G;
            hp.chunk = (int)std::max<long long>(256, std::min<long long>(MAX_CHUNK, per)) / 32 * 32;  // 32-row batches (TMA alignment)
            return GBM_OK;
        }
        if (allow_col && channels * rows * 32 * 4 <= budget) {
            hp.col = true;
            hp.byte_path = byte_sym;
            hp.cstride = rows * 32;
            hp.smem_bytes = channels * hp.cstride * 4;
            hp.cgroups.clear();
            const int ng = (qm.F + 31) / 32;
            for (int g = 0; g < ng; ++g) {  // balanced groups of <= 32 features
                ColGroup c;
                c.f_lo = (int)((long long)qm.F * g / ng);
                c.f_hi = (int)((long long)qm.F * (g + 1) / ng);
                hp.cgroups.push_back(c);
            }
            int rc = wide ? (byte_sym ? setup_col<true, true>(ctx, hp) : setup_col<true, false>(ctx, hp))
                          : (byte_sym ? setup_col<false, true>(ctx, hp) : setup_col<false, false>(ctx, hp));
            GBM_TRY(rc);
            const long long G = (long long)hp.cgroups.size();
            long long per = (rows_hint + 2ll * hp.blocks_range - 1) / (2ll * hp.blocks_range) * G;
            hp.chunk = (int)std::max<long long>(256, std::min<long long>(MAX_CHUNK, per));
            return GBM_OK;
        }
    }
    hp.byte_path = q->bits == 8 && (qm.stride % 32) == 0;
    hp.sent = q->max_bins < 256;  // the sentinel symbol fits in 8 bits
    const int channels = wide ? 4 : 2;
    const int static_smem = 26 * 1024;
    const int budget = (int)std::min<size_t>(ctx->smem_optin - static_smem, 200 * 1024);
    const int max_bins_group = budget / (4 * channels) - DUMMY_BINS - 32;
    // Feature groups of <= ucap units.  Auto: the largest power of two (a warp's lanes map to
    // whole rows x units) whose groups still leave two blocks resident per SM -- measured on the
    // wide workloads (Epsilon 8 units: level pass 2.5 vs 3.6 ms at 24; Bosch 16: 1.8 vs 2.7 at 32).
    auto make_groups = [&](int ucap, std::vector<Group> &out) -> int {
        out.clear();
        const int ng = (qm.U + ucap - 1) / ucap;
        const int umax = (qm.U + ng - 1) / ng;  // balanced: the last group is not a sliver
        int u = 0, mx = 1;
        while (u < qm.U) {
            Group g;
            g.u_lo = u;
            g.bin_lo = cp[std::min(u * qm.S, qm.F)];
            int u_end = u;
            while (u_end < qm.U) {
                const int f_hi = std::min((u_end + 1) * qm.S, qm.F);
                const int nb = cp[f_hi] - g.bin_lo;
                const int nf = f_hi - u * qm.S;
                if ((nb > max_bins_group || nf > 2048 || (u_end - u + 1) > umax) && u_end > u) break;
                if (nb > max_bins_group) return -1;
                u_end++;
            }
            g.u_hi = u_end;
            g.bin_hi = cp[std::min(u_end * qm.S, qm.F)];
            mx = std::max(mx, g.bin_hi - g.bin_lo);
            out.push_back(g);
            u = u_end;
        }
        return mx;
    };
    int sm_smem = 0;
    GBM_CUDA(cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, ctx->device));
    if (ctx->group_units > 0) {
        if (make_groups(ctx->group_units, hp.groups) < 0)
            return fail(GBM_E_ARG, "a single feature unit has more bins than fit in shared memory");
    } else {
        for (int ucap = 32;; ucap >>= 1) {
            const int mx = make_groups(ucap, hp.groups);
            if (mx < 0) return fail(GBM_E_ARG, "a single feature unit has more bins than fit in shared memory");
            const int bytes = channels * ((mx + DUMMY_BINS + 31) / 32 * 32) * 4 + static_smem + 1024;
            if (ucap == 1 || 2 * bytes <= sm_smem) break;
        }
    }
    int max_nb = 1;
    for (auto &g : hp.groups) max_nb = std::max(max_nb, g.bin_hi - g.bin_lo);
    // replica words (fused level kernel, byte path): what the groups' low-cardinality features
    // need under the kernel's rule, if two blocks per SM still fit; 0 = none (no overhead)
    int rep_cap = 0;
    if (hp.byte_path && ctx->level_rep) {
        for (auto &g : hp.groups) {
            const int rpp = 32 / (g.u_hi - g.u_lo);
            const int fa = g.u_lo * qm.S, fb = std::min(g.u_hi * qm.S, qm.F);
            if (fb - fa > REP_F || rpp < 2) continue;
            int need = 0;
            for (int f = fa; f < fb; ++f) {
                const int nb = cp[f + 1] - cp[f];
                need += ((1 << rep_log2(nb, rpp)) - 1) * nb;
            }
            rep_cap = std::max(rep_cap, std::min(REP_CAP, (need + 31) / 32 * 32));
        }
        const int bytes = channels * ((max_nb + DUMMY_BINS + rep_cap + 31) / 32 * 32) * 4 + static_smem + 1024;
        if (2 * bytes > sm_smem) rep_cap = 0;
    }
    hp.rep_cap = rep_cap;
    hp.hstride = (max_nb + DUMMY_BINS + rep_cap + 31) / 32 * 32;
    hp.smem_bytes = channels * hp.hstride * 4;
    GBM_TRY(GBM_DISPATCH(hp, setup_kernels, ctx, hp));
    long long per = (rows_hint + 2ll * hp.blocks_range - 1) / (2ll * hp.blocks_range) * (long long)hp.groups.size();
    hp.chunk = (int)std::max<long long>(256, std::min<long long>(MAX_CHUNK, per));
    return GBM_OK;
}

template <bool W, bool B, bool S>
static int launch_range(gbm_ctx *ctx, const HistPlan &hp, RangeArgs a, cudaStream_t s) {
    const long long n_items = (a.n_sel + a.chunk - 1) / a.chunk * (long long)a.n_groups;
    const int grid = (int)std::max<long long>(1, std::min<long long>(n_items, hp.blocks_range));
    hist_range_kernel<W, B, S><<<grid, H_THREADS, hp.smem_bytes, s>>>(a);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

template <bool W, bool B, bool S>
static int launch_fused(gbm_ctx *ctx, const HistPlan &hp, FusedArgs a, cudaStream_t s, bool carry) {
    if constexpr (!W) {
        if (carry) part_hist_kernel<W, B, S, true><<<hp.blocks_fused, H_THREADS, hp.smem_bytes, s>>>(a);
        else part_hist_kernel<W, B, S, false><<<hp.blocks_fused, H_THREADS, hp.smem_bytes, s>>>(a);
    } else {
        part_hist_kernel<W, B, S, false><<<hp.blocks_fused, H_THREADS, hp.smem_bytes, s>>>(a);
    }
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

template <bool W, bool B, bool S>
static int launch_seg(gbm_ctx *ctx, const HistPlan &hp, SegArgs a, cudaStream_t s, bool carry) {
    if constexpr (!W) {
        if (carry) hist_seg_kernel<W, B, S, true><<<hp.blocks_range, H_THREADS, hp.smem_bytes, s>>>(a);
        else hist_seg_kernel<W, B, S, false><<<hp.blocks_range, H_THREADS, hp.smem_bytes, s>>>(a);
    } else {
        hist_seg_kernel<W, B, S, false><<<hp.blocks_range, H_THREADS, hp.smem_bytes, s>>>(a);
    }
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

static void launch_col_range(const HistPlan &hp, const ColRangeArgs &ca, int grid, cudaStream_t s) {
    const int sm = hp.smem_bytes;
    if (hp.staged) {  // (the staged kernels reduce the totals from their staged pairs)
        if (!hp.byte_path) {  // generic symbol widths
            if (ca.ridx) hist_csg_range_kernel<false><<<grid, H_THREADS, sm, s>>>(ca);
            else hist_csg_range_kernel<true><<<grid, H_THREADS, sm, s>>>(ca);
            return;
        }
        if (hp.cs_r1) {
            if (ca.ridx) hist_cs_range_kernel<false, true><<<grid, H_THREADS, sm, s>>>(ca);
            else hist_cs_range_kernel<true, true><<<grid, H_THREADS, sm, s>>>(ca);
        } else {
            if (ca.ridx) hist_cs_range_kernel<false, false><<<grid, H_THREADS, sm, s>>>(ca);
            else hist_cs_range_kernel<true, false><<<grid, H_THREADS, sm, s>>>(ca);
        }
        return;
    }
    if (hp.byte_path) {
        if (ca.totals) sum_qpair_kernel<<<std::min<long long>((ca.n_sel + 255) / 256, 148 * 8), 256, 0, s>>>(
            ca.qpair, ca.n_sel, ca.totals);
        if (hp.wide) {
            if (ca.ridx) hist_colb_range_kernel<true, false><<<grid, H_THREADS, sm, s>>>(ca);
            else hist_colb_range_kernel<true, true><<<grid, H_THREADS, sm, s>>>(ca);
        } else {
            if (ca.ridx) hist_colb_range_kernel<false, false><<<grid, H_THREADS, sm, s>>>(ca);
            else hist_colb_range_kernel<false, true><<<grid, H_THREADS, sm, s>>>(ca);
        }
        return;
    }
    if (hp.wide) {
        if (hp.byte_path) hist_col_range_kernel<true, true><<<grid, H_THREADS, sm, s>>>(ca);
        else hist_col_range_kernel<true, false><<<grid, H_THREADS, sm, s>>>(ca);
    } else {
        if (hp.byte_path) hist_col_range_kernel<false, true><<<grid, H_THREADS, sm, s>>>(ca);
        else hist_col_range_kernel<false, false><<<grid, H_THREADS, sm, s>>>(ca);
    }
}

static void launch_col_fused(const HistPlan &hp, const ColFusedArgs &ca, cudaStream_t s) {
    const int g = hp.blocks_fused, sm = hp.smem_bytes;
    if (hp.staged) {
        if (hp.cs_r1) {
            if (hp.carry) part_hist_cs_kernel<true, true><<<g, H_THREADS, sm, s>>>(ca);
            else part_hist_cs_kernel<false, true><<<g, H_THREADS, sm, s>>>(ca);
        } else {
            if (hp.carry) part_hist_cs_kernel<true, false><<<g, H_THREADS, sm, s>>>(ca);
            else part_hist_cs_kernel<false, false><<<g, H_THREADS, sm, s>>>(ca);
        }
        return;
    }
    if (hp.wide) {
        if (hp.byte_path) part_hist_col_kernel<true, false, true><<<g, H_THREADS, sm, s>>>(ca);
        else part_hist_col_kernel<true, false, false><<<g, H_THREADS, sm, s>>>(ca);
    } else if (hp.carry) {
        if (hp.byte_path) part_hist_col_kernel<false, true, true><<<g, H_THREADS, sm, s>>>(ca);
        else part_hist_col_kernel<false, true, false><<<g, H_THREADS, sm, s>>>(ca);
    } else {
        if (hp.byte_path) part_hist_col_kernel<false, false, true><<<g, H_THREADS, sm, s>>>(ca);
        else part_hist_col_kernel<false, false, false><<<g, H_THREADS, sm, s>>>(ca);
    }
}

template <int W, bool BYTE, bool SENT>
static void launch_walk_t(int grid, size_t sm, cudaStream_t s, const QM &qm, const TreeDev &t, int n_int, int D,
                          long long n, int32_t *rl, const WalkEpi *epi) {
    if (epi) {
        auto k = leaf_walk_stg_kernel<W, true, BYTE, SENT>;
        if (sm > 16 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k<<<grid, WALK_THREADS, sm, s>>>(qm, t.kind, t.feature, t.bin, t.default_left, n_int, D, n, rl, *epi);
    } else {
        auto k = leaf_walk_stg_kernel<W, false, BYTE, SENT>;
        if (sm > 16 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k<<<grid, WALK_THREADS, sm, s>>>(qm, t.kind, t.feature, t.bin, t.default_left, n_int, D, n, rl, WalkEpi{});
    }
}

template <int W>
static void launch_walk_reg(int grid, size_t sm, cudaStream_t s, const QM &qm, const TreeDev &t, int n_int, int D,
                            long long n, int32_t *rl, const WalkEpi *epi) {
    // byte symbols (8-bit, rows of whole words, F <= 4 W): one LDS.U8 per level
    if constexpr (W <= 8) {
        if (qm.bits == 8) {
            if (qm.B < 256) launch_walk_t<W, true, true>(grid, sm, s, qm, t, n_int, D, n, rl, epi);
            else launch_walk_t<W, true, false>(grid, sm, s, qm, t, n_int, D, n, rl, epi);
            return;
        }
    }
    launch_walk_t<W, false, true>(grid, sm, s, qm, t, n_int, D, n, rl, epi);
}

static TreeDev tree_dev(const gbm_tree *t) {
    TreeDev d;
    d.kind = t->kind;
    d.feature = t->feature;
    d.bin = t->bin;
    d.threshold = t->threshold;
    d.default_left = t->default_left;
    d.gain = t->gain;
    d.weight = t->weight;
    d.left_child = t->left_child;
    d.sum_qg = reinterpret_cast<long long *>(t->sum_qg);
    d.sum_qh = reinterpret_cast<long long *>(t->sum_qh);
    return d;
}

static int check_qm(const gbm_qmatrix *qm) {
    GBM_REQUIRE(qm && qm->packed_d && qm->cut_values_d && qm->cut_ptr_d && qm->cut_ptr_h, GBM_E_ARG,
                "qmatrix: null pointer");
    GBM_REQUIRE(qm->n_features > 0 && qm->bits >= 1 && qm->bits <= 16 && qm->max_bins >= 2 &&
                    qm->max_bins <= 65535 && qm->n_rows >= 0 && qm->n_rows < (1ll << 31),
                GBM_E_ARG, "qmatrix: bad sizes");
    GBM_REQUIRE(qm->row_align_bits == 0 || qm->row_align_bits == 32 || qm->row_align_bits == 128 ||
                    qm->row_align_bits == 256, GBM_E_ARG,
                "qmatrix: row_align_bits must be 0, 32, 128 or 256");
    return GBM_OK;
}

static EvalArgs eval_args_base(const gbm_ctx *ctx, const gbm_qmatrix *q, const int32_t *scale_d,
                               const gbm_params *prm) {
    EvalArgs a = {};
    a.F = q->n_features;
    a.TB = q->cut_ptr_h[q->n_features];
    a.cut_ptr = q->cut_ptr_d;
    a.cut_values = q->cut_values_d;
    a.scale = scale_d;
    a.p = EvalParams{prm->eta, prm->lambda, prm->gamma, prm->min_child_weight, prm->max_depth,
                     ctx->eval_screen ? 1 : 0};
    return a;
}

static int launch_eval_tree(gbm_ctx *ctx, const EvalArgs &ea, const TreeDev &t, cudaStream_t s) {
    const long long units = (long long)ea.n_nodes * ea.F;
    // auto: a warp per (node, feature) once there are enough of them to fill the GPU
    // (throughput: Epsilon 5.13 vs 5.32 ms/round) or with many features (YearMSD evaluation 0.151
    // -> 0.143 ms/round, Bosch 0.483 -> 0.455 at >= 64), else a block per (node, feature)
    // (latency: loss-guided Higgs 6.49 vs 7.29 ms/round)
    const bool warp = ctx->eval_warp == 1 ||
                      (ctx->eval_warp == 0 && (units >= 16ll * ctx->sm_count || ea.F >= 64));
    if (warp)
        eval_tree_kernel<<<(int)((units + E_THREADS / 32 - 1) / (E_THREADS / 32)), E_THREADS, 0, s>>>(ea, t);
    else
        eval_tree_blk_kernel<<<(int)units, E_THREADS, 0, s>>>(ea, t);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

// Fork the side stream off s after the work enqueued so far / join it back.
static int fork_side(gbm_ctx *ctx, cudaStream_t s) {
    GBM_CUDA(cudaEventRecord(ctx->ev_fork, s));
    GBM_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    return GBM_OK;
}
static int wait_on(cudaStream_t waiter, cudaEvent_t e, cudaStream_t signaller) {
    GBM_CUDA(cudaEventRecord(e, signaller));
    GBM_CUDA(cudaStreamWaitEvent(waiter, e, 0));
    return GBM_OK;
}

// Upload the feature-group table when it changed (keeps tree builds free of pageable copies so
// a whole round can be captured in a CUDA graph).
static int upload_groups(gbm_ctx *ctx, const HistPlan &hp, Group *groups, ColGroup *cgroups, const Arena &A,
                         cudaStream_t s, const HistPlan *hr = nullptr, ColGroup *cg_root = nullptr) {
    const int G = hp.col ? (int)hp.cgroups.size() : (int)hp.groups.size();
    std::vector<int> key;
    key.push_back(hp.col ? 1 : 0);
    key.push_back((int)(reinterpret_cast<uintptr_t>(hp.col ? (void *)cgroups : (void *)groups) & 0x7fffffff));
    key.push_back((int)A.generation);
    if (hp.col)
        for (auto &g : hp.cgroups) { key.push_back(g.f_lo); key.push_back(g.f_hi); }
    else
        for (auto &g : hp.groups) { key.push_back(g.u_lo); key.push_back(g.u_hi); key.push_back(g.bin_lo); key.push_back(g.bin_hi); }
    if (hr) {  // the root pass's own (staged column) groups
        key.push_back(-1);
        key.push_back((int)(reinterpret_cast<uintptr_t>(cg_root) & 0x7fffffff));
        for (auto &g : hr->cgroups) { key.push_back(g.f_lo); key.push_back(g.f_hi); }
    }
    if (key != ctx->tree_groups_key) {
        if (hp.col) GBM_CUDA(cudaMemcpyAsync(cgroups, hp.cgroups.data(), G * sizeof(ColGroup), cudaMemcpyHostToDevice, s));
        else GBM_CUDA(cudaMemcpyAsync(groups, hp.groups.data(), G * sizeof(Group), cudaMemcpyHostToDevice, s));
        if (hr)
            GBM_CUDA(cudaMemcpyAsync(cg_root, hr->cgroups.data(), hr->cgroups.size() * sizeof(ColGroup),
                                     cudaMemcpyHostToDevice, s));
        ctx->tree_groups_key = key;
    }
    return GBM_OK;
}

// The root pass streams every row: there the staged bank-column kernel (one feature per lane,
// conflict-free atomics) beats the compact layout (Higgs root 0.28 vs 0.33 ms, Epsilon 0.78 vs
// 1.07, Airline 3.09 vs 3.73; rounds -3 %, -6 %, -3 %), while the level passes gather rows and
// stay compact (staged levels: Higgs 1.17 vs 0.92 ms).  Auto layout only; byte symbols, narrow
// fixed point, word-aligned rows, at least 10^8 (row, feature) updates.
// Staged root for generic symbol widths (9..15 bits): groups of <= 32 features, every feature's
// present symbols < 256 (one column of COLB_STRIDE rows), word-aligned rows.
static bool plan_root_staged_generic(gbm_ctx *ctx, const gbm_qmatrix *q, const QM &qm, long long n, HistPlan &hr) {
    if (q->bits < 9 || q->bits > 15 || qm.stride % 32 != 0) return false;
    for (int f = 0; f < q->n_features; ++f)
        if (q->cut_ptr_h[f + 1] - q->cut_ptr_h[f] > 256) return false;
    hr = HistPlan();
    hr.col = hr.staged = true;
    hr.byte_path = false;
    hr.cstride = COLB_STRIDE;
    hr.smem_bytes = 2 * COLB_STRIDE * 4 + (H_THREADS / 32) * (int)sizeof(CsgWarp);
    const int ng = (q->n_features + 31) / 32;
    for (int g = 0; g < ng; ++g) {
        ColGroup c;
        c.f_lo = (int)((long long)q->n_features * g / ng);
        c.f_hi = (int)((long long)q->n_features * (g + 1) / ng);
        hr.cgroups.push_back(c);
    }
    if (cudaFuncSetAttribute(hist_csg_range_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, hr.smem_bytes) !=
            cudaSuccess ||
        cudaFuncSetAttribute(hist_csg_range_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, hr.smem_bytes) !=
            cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    int o1 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, hist_csg_range_kernel<true>, H_THREADS, hr.smem_bytes) !=
            cudaSuccess || o1 < 1) {
        cudaGetLastError();
        return false;
    }
    hr.blocks_range = o1 * ctx->sm_count;
    const long long G = (long long)hr.cgroups.size();
    const long long per = (n + 2ll * hr.blocks_range - 1) / (2ll * hr.blocks_range) * G;
    hr.chunk = (int)std::max<long long>(256, std::min<long long>(MAX_CHUNK, per));
    return true;
}

static bool plan_root_staged(gbm_ctx *ctx, const gbm_qmatrix *q, const QM &qm, const HistPlan &hp, int grad_bits,
                             long long n, HistPlan &hr) {
    if (hp.col || (ctx->hist_layout != 0 && ctx->hist_layout != 4) || grad_bits > 15 || qm.stride % 32 != 0 ||
        n <= 0)
        return false;
    const bool forced = ctx->hist_layout == 4;
    if (q->bits != 8) {
        if (!forced && (double)n * q->n_features < 1e8) return false;
        return plan_root_staged_generic(ctx, q, qm, n, hr);
    }
    // small (L2-resident) matrices keep the compact root: YearMSD 515K x 90 0.565 vs 0.540 ms/round
    if (!forced && (double)n * q->n_features < 1e8) return false;
    if (plan_hist(ctx, q, qm, false, n, hr, grad_bits, true, true) != GBM_OK) return false;  // compact root
    return hr.col && hr.staged;
}

static int launch_root_staged(gbm_ctx *ctx, const HistPlan &hr, const QM &qm, const gbm_qmatrix *q,
                              const int32_t *qpair_d, const ColGroup *cg_root, long long *hist_root,
                              long long *totals, long long n, double row_bytes, cudaStream_t s) {
    ColRangeArgs ca = {};
    ca.qm = qm;
    ca.qpair = reinterpret_cast<const int2 *>(qpair_d);
    ca.ridx = nullptr;
    ca.n_sel = n;
    ca.chunk = hr.chunk;
    // TMA bulk copies need 16-byte aligned sources (row batches are 32 rows: 16-byte multiples)
    ca.tma = (hr.cgroups.size() == 1 && reinterpret_cast<uintptr_t>(q->packed_d) % 16 == 0 &&
              reinterpret_cast<uintptr_t>(qpair_d) % 16 == 0 && ctx->stage_tma) ? 1 : 0;
    ca.n_groups = (int)hr.cgroups.size();
    ca.groups = cg_root;
    ca.cut_ptr = q->cut_ptr_d;
    ca.hist = reinterpret_cast<unsigned long long *>(hist_root);
    ca.totals = reinterpret_cast<unsigned long long *>(totals);
    ca.cstride = hr.cstride;
    int slot = -1;
    ca.rows_ctr = prof_rows_slot(ctx, &slot);
    ProfScope ps(ctx, PC_HIST_ROOT, s, 0.0, slot, row_bytes + 8.0);
    const long long n_it = (n + hr.chunk - 1) / hr.chunk * (long long)ca.n_groups;
    const int grid = (int)std::max<long long>(1, std::min<long long>(n_it, hr.blocks_range));
    launch_col_range(hr, ca, grid, s);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

// the tensor-fed root (root_ct.cu) where it applies: 1 launched, 0 not applicable, < 0 error
static int try_root_tensor(gbm_ctx *ctx, const gbm_qmatrix *q, const QM &qm, const int32_t *qpair_d, int grad_bits,
                           long long *hist, long long *totals, long long n, cudaStream_t s) {
    RootCtLaunch L = {};
    L.colsym = qm.col;
    L.qpair = reinterpret_cast<const int2 *>(qpair_d);
    L.n = n;
    L.F = q->n_features;
    L.bits = q->bits;
    L.wide = grad_bits > 15;
    L.cut_ptr = q->cut_ptr_d;
    L.hist = reinterpret_cast<unsigned long long *>(hist);
    L.totals = reinterpret_cast<unsigned long long *>(totals);
    return root_ct_launch(ctx, L, s);  // profiled as PC_HIST_ROOT when it launches
}

// Loss-guided growth (R25-R27): InitRoot as depth-wise, then max_leaves - 1 device-driven
// expansion steps, each = select (pop) -> fused repartition + smaller-child histogram of the one
// parent -> scan -> scatter -> allreduce -> sibling by subtraction + EvaluateSplit of both
// children.  Open nodes keep their histograms in a pool of max_leaves slots (the sibling
// overwrites its parent's slot, the built child takes slot s+1); a node's rows stay in the
// ridx buffer its parent's step wrote (segments of open nodes are disjoint, so two buffers do).
static int build_tree_lossguide(gbm_ctx *ctx, const gbm_qmatrix *q, const QM &qm, const int32_t *qpair_d,
                                const int32_t *scale_d, const gbm_params *prm, const gbm_tree *tree,
                                int32_t *row_leaf_d, cudaStream_t s) {
    const long long n = q->n_rows;
    const int F = q->n_features, D = prm->max_depth, L = prm->max_leaves;
    const long long TB = q->cut_ptr_h[F];
    const long long cap = 2ll * L - 1;
    HistPlan hp;
    GBM_TRY(plan_hist(ctx, q, qm, prm->grad_bits > 15, std::max<long long>(n, 1), hp, prm->grad_bits, false, false));
    const int G = (int)hp.groups.size();
    HistPlan hr;
    const bool root_staged = plan_root_staged(ctx, q, qm, hp, prm->grad_bits, n, hr);
    const size_t esz = hp.carry ? 8 : 4;
    const long long max_tiles = (n + PT - 1) / PT + 2;
    const size_t hist_unit = (size_t)std::max<long long>(TB, 1) * 2;
    const bool grow = D > 0 && L > 1;
    size_t need = 0;
    need += 2 * (size_t)std::max<long long>(n, 1) * esz + 512;    // ridx buffers
    need += (size_t)max_tiles * (PT / 32) * 4 + 256;              // flags
    need += 2 * (size_t)max_tiles * 4 + 512;                      // tile_left / tile_off
    need += 6 * 64 + 6 * 256;                                     // tile_base, run_base, n_items x2
    need += (size_t)(cap + 2) * (sizeof(NodeDev) + sizeof(LgNode)) + 512;
    need += 2 * (sizeof(StepDev) + 256);
    need += (size_t)G * sizeof(Group) + 256;
    need += (root_staged ? hr.cgroups.size() : 1) * sizeof(ColGroup) + 256;
    need += (2 * hist_unit + 2) * 8 + 512;                        // root (+ totals), build
    need += (grow ? (size_t)L : 1) * hist_unit * 8 + 256;         // pool
    need += 2 * (size_t)F * sizeof(FeatBest) + 256;
    need += 4 * sizeof(unsigned) + 256;                           // eval counters
    Arena &A = ctx->tree_arena;
    GBM_TRY(A.reserve(need));
    char *ridx[2] = {A.take<char>(std::max<long long>(n, 1) * esz), A.take<char>(std::max<long long>(n, 1) * esz)};
    uint32_t *flags = A.take<uint32_t>((size_t)max_tiles * (PT / 32));
    int *tile_left = A.take<int>(max_tiles);
    int *tile_off = A.take<int>(max_tiles);
    // step plans double-buffered by step parity: step st+1 is popped (by step st's evaluation)
    // while step st's scatter still reads step st's plan on the side stream
    int *tile_base_b[2] = {A.take<int>(4), A.take<int>(4)};
    int *run_base_b[2] = {A.take<int>(4), A.take<int>(4)};
    int *n_items_b[2] = {A.take<int>(4), A.take<int>(4)};
    NodeDev *nodes = A.take<NodeDev>(cap + 2);
    LgNode *lg = A.take<LgNode>(cap + 2);
    StepDev *step_b[2] = {A.take<StepDev>(1), A.take<StepDev>(1)};
    Group *groups = A.take<Group>(G);
    ColGroup *cg_root = A.take<ColGroup>(root_staged ? hr.cgroups.size() : 1);
    long long *hist_root = A.take<long long>(hist_unit + 2);
    long long *hist_build = A.take<long long>(hist_unit);
    long long *hist_pool = A.take<long long>((grow ? (size_t)L : 1) * hist_unit);
    FeatBest *fb = A.take<FeatBest>(2 * (size_t)F);
    unsigned *done = A.take<unsigned>(4);  // [0] nodes completed, [1..2] warps per node
    GBM_TRY(upload_groups(ctx, hp, groups, nullptr, A, s, root_staged ? &hr : nullptr, cg_root));
    GBM_CUDA(cudaMemsetAsync(done, 0, 4 * sizeof(unsigned), s));
    const TreeDev t = tree_dev(tree);
    const double row_bytes = (double)F * q->bits / 8.0;
    {
        ProfScope ps(ctx, PC_INIT, s);
        const int g = (int)std::min<long long>((cap + 255) / 256, 1024);
        init_tree_kernel<<<g, 256, 0, s>>>(t, cap, nodes, n);
        lg_init_kernel<<<g, 256, 0, s>>>(lg, cap);
    }
    // ---- InitRoot
    GBM_CUDA(cudaMemsetAsync(hist_root, 0, (hist_unit + 2) * 8, s));
    const int root_ct = (n > 0 && TB > 0) ? try_root_tensor(ctx, q, qm, qpair_d, prm->grad_bits, hist_root,
                                                            hist_root + hist_unit, n, s)
                                          : 0;
    if (root_ct < 0) return root_ct;
    if (root_ct == 1) {
        // the tensor-fed root (root_ct.cu)
    } else if (n > 0 && TB > 0 && root_staged) {
        GBM_TRY(launch_root_staged(ctx, hr, qm, q, qpair_d, cg_root, hist_root, hist_root + hist_unit, n, row_bytes, s));
    } else if (n > 0 && TB > 0) {
        RangeArgs ra = {};
        ra.qm = qm;
        ra.qpair = reinterpret_cast<const int2 *>(qpair_d);
        ra.n_sel = n;
        ra.chunk = hp.chunk;
        ra.n_groups = G;
        ra.groups = groups;
        ra.cut_ptr = q->cut_ptr_d;
        ra.hist = reinterpret_cast<unsigned long long *>(hist_root);
        ra.totals = reinterpret_cast<unsigned long long *>(hist_root + hist_unit);
        ra.hstride = hp.hstride;
        int slot = -1;
        ra.rows_ctr = prof_rows_slot(ctx, &slot);
        ProfScope ps(ctx, PC_HIST_ROOT, s, 0.0, slot, row_bytes + 8.0);
        GBM_TRY(GBM_DISPATCH(hp, launch_range, ctx, hp, ra, s));
    } else if (n > 0) {
        return fail(GBM_E_ARG, "gbm_build_tree: no feature has a cut (all values missing)");
    }
    {
        ProfScope ps(ctx, PC_ALLREDUCE, s, (double)(hist_unit + 2) * 8);
        GBM_TRY(allreduce_i64(ctx, hist_root, hist_unit + 2, s));
    }
    EvalArgs ea = eval_args_base(ctx, q, scale_d, prm);
    ea.nodes = nodes;
    ea.hist_root = hist_root;
    ea.hist_build = hist_build;
    ea.fb = fb;
    ea.lg = lg;
    ea.step = step_b[1];       // (unused at the root)
    ea.step_next = step_b[0];  // the root's evaluation pops step 0
    ea.hist_pool = hist_pool;
    ea.level = 0;
    ea.first = 0;
    ea.n_nodes = 1;
    ea.hist_store = grow ? hist_pool : nullptr;  // the root's histogram -> pool slot 0
    const long long tiles_all = (n + PT - 1) / PT;
#ifndef GBM_LG_ITEMS  // work items per resident block for a large parent (measured, Higgs 64
#define GBM_LG_ITEMS 1  // leaves: 5.93 ms/round at 4, 5.81 at 2, 5.54 at 1 -- fewer flushes)
#endif
    const long long target = (long long)GBM_LG_ITEMS * hp.blocks_fused;
    const int run_tiles = ctx->run_tiles > 0 ? ctx->run_tiles : (int)std::max<long long>(
        1, std::min<long long>(RUN_MAX, (tiles_all * G + target - 1) / target));
    ea.done = done;
    ea.node_done = done + 1;
    ea.plan_groups = G;
    ea.plan_run = (int)target;  // loss-guided: the pop sizes the work items to the parent
    // at least 2 tiles per item: small parents pay one histogram zero + flush per item
    // (loss-guided Higgs, 64 leaves: 4.92 ms/round at 2, 5.14 at 1, 5.35 at 4)
    ea.plan_run_min = ctx->run_tiles > 0 ? ctx->run_tiles : 2;
    ea.tile_base = tile_base_b[0];
    ea.run_base = run_base_b[0];
    ea.n_items = n_items_b[0];
    ea.tile_left = tile_left;
    ea.plan_mode = grow ? 2 : 0;  // the root's evaluation pops the first expansion
    ea.sel_step = 0;
    {
        ProfScope ps(ctx, PC_EVAL, s, (double)TB * 16);
        GBM_TRY(launch_eval_tree(ctx, ea, t, s));
    }
    if (!grow) {  // a single leaf
        GBM_CUDA(cudaMemsetAsync(row_leaf_d, 0, sizeof(int32_t) * (size_t)std::max<long long>(n, 0), s));
        return GBM_OK;
    }
    FusedArgs fa = {};
    fa.qm = qm;
    fa.nodes = nodes;
    fa.first = 0;
    fa.n_par = 1;
    fa.n_groups = G;
    fa.run_tiles = run_tiles;
    fa.ridx_in = nullptr;
    fa.bufs[0] = ridx[0];
    fa.bufs[1] = ridx[1];
    fa.flags = flags;
    fa.tile_left = tile_left;
    fa.row_leaf = row_leaf_d;
    fa.qpair = reinterpret_cast<const int2 *>(qpair_d);
    fa.groups = groups;
    fa.cut_ptr = q->cut_ptr_d;
    fa.hist = reinterpret_cast<unsigned long long *>(hist_build);
    fa.TB = std::max<long long>(TB, 1);
    fa.hstride = hp.hstride;
    fa.rep_cap = hp.rep_cap;
    fa.bits_parent_row = q->bits + 32;  // split symbol + entry (identity at the root: upper bound)
    fa.bits_built_row = F * q->bits + 64;
    const int pgrid = ctx->sm_count * 8;
    ea.level = 1;  // child mode of node_source
    ea.n_nodes = 2;
    ea.hist_store = nullptr;
    for (int st = 0; st < L - 1; ++st) {
        // (the pop of step st ran in the last block of the previous evaluation)
        StepDev *step = step_b[st & 1];
        int *tile_base = tile_base_b[st & 1];
        fa.step = step;
        fa.tile_base = tile_base;
        fa.run_base = run_base_b[st & 1];
        fa.n_items = n_items_b[st & 1];
        GBM_CUDA(cudaMemsetAsync(hist_build, 0, hist_unit * 8, s));
        {
            int slot;
            fa.rows_ctr = prof_rows_slot(ctx, &slot);
            ProfScope ps(ctx, PC_HIST_LEVEL, s, 0.0, slot, 1.0 / 8.0);
            GBM_TRY(GBM_DISPATCH(hp, launch_fused, ctx, hp, fa, s, hp.carry));
        }
        GBM_TRY(fork_side(ctx, s));  // scan + scatter overlap the allreduce / evaluation
        cudaStream_t ss = ctx->side;
        {
            ProfScope ps(ctx, PC_PART_SCAN, ss);
            part_scan_kernel<<<1, 1024, 0, ss>>>(nodes, 0, tile_base, tile_left, tile_off, step);
        }
        GBM_CUDA(cudaEventRecord(ctx->ev_scan, ss));
        {
            int slot;
            unsigned long long *rc = prof_rows_slot(ctx, &slot);
            ProfScope ps(ctx, PC_PART_SCATTER, ss, 0.0, slot, 8.0);
            if (hp.carry)
                part_scatter_kernel<true><<<pgrid, P_THREADS, 0, ss>>>(
                    nodes, 0, 1, tile_base, flags, tile_off, nullptr, nullptr, reinterpret_cast<const int2 *>(qpair_d),
                    rc, step, ridx[0], ridx[1]);
            else
                part_scatter_kernel<false><<<pgrid, P_THREADS, 0, ss>>>(
                    nodes, 0, 1, tile_base, flags, tile_off, nullptr, nullptr, nullptr, rc, step, ridx[0], ridx[1]);
            GBM_CUDA(cudaGetLastError());
        }
        {
            ProfScope ps(ctx, PC_ALLREDUCE, s, (double)hist_unit * 8);
            GBM_TRY(allreduce_i64(ctx, hist_build, hist_unit, s));
        }
        ea.first = 2 * st + 1;
        ea.plan_mode = st + 1 < L - 1 ? 2 : 0;
        ea.sel_step = st + 1;
        ea.step = step;  // this step's parent (node_source) ...
        ea.step_next = step_b[(st + 1) & 1];  // ... and the pop of the next one
        ea.tile_base = tile_base_b[(st + 1) & 1];
        ea.run_base = run_base_b[(st + 1) & 1];
        ea.n_items = n_items_b[(st + 1) & 1];
        GBM_CUDA(cudaStreamWaitEvent(s, ctx->ev_scan, 0));  // the pop reads the children's counts
        {
            ProfScope ps(ctx, PC_EVAL, s, (double)hist_unit * 8 * 4.0);
            GBM_TRY(launch_eval_tree(ctx, ea, t, s));
        }
        GBM_TRY(wait_on(s, ctx->ev_join, ctx->side));
    }
    if (n > 0) {
        ProfScope ps(ctx, PC_PART_FINAL, s, (double)n * 4.0);
        const int grid = (int)std::max<long long>(1, std::min<long long>((n + WALK_THREADS - 1) / WALK_THREADS,
                                                                        (long long)ctx->sm_count * 8));
        // (a staged shared-memory walk, as depth-wise, measured slower here: loss-guided trees are
        // deep and their node ids scatter over shared-memory banks -- 0.36 vs 0.18 ms on Higgs)
        lg_walk_kernel<<<grid, WALK_THREADS, 0, s>>>(qm, t, n, row_leaf_d);
        GBM_CUDA(cudaGetLastError());
    }
    return GBM_OK;
}

}  // namespace gbm

using namespace gbm;

extern "C" {

int gbm_build_histogram(gbm_ctx *ctx, const gbm_qmatrix *q, const int32_t *qpair_d, int32_t grad_bits,
                        const uint32_t *rows_d, int64_t n_sel, int64_t *hist_d, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_TRY(check_qm(q));
    GBM_REQUIRE(qpair_d && hist_d && grad_bits >= 1 && grad_bits <= 30, GBM_E_ARG, "gbm_build_histogram: bad arguments");
    if (!rows_d) n_sel = q->n_rows;
    GBM_REQUIRE(n_sel >= 0, GBM_E_ARG, "gbm_build_histogram: n_sel < 0");
    cudaStream_t s = (cudaStream_t)stream;
    const QM qm = make_qm(q);
    const int TB = q->cut_ptr_h[q->n_features];
    HistPlan hp;
    // layouts 2 / 3 force the column levels; 4 = staged root + compact levels
    GBM_TRY(plan_hist(ctx, q, qm, grad_bits > 15, n_sel, hp, grad_bits,
                      ctx->hist_layout == 2 || ctx->hist_layout == 3, ctx->hist_layout == 3));
    GBM_CUDA(cudaMemsetAsync(hist_d, 0, (size_t)std::max(TB, 1) * 2 * 8, s));
    if (n_sel == 0 || TB == 0) return GBM_OK;
    HistPlan hr;
    if (!rows_d) {  // the tensor-fed root first (as gbm_build_tree's InitRoot)
        GBM_TRY(ctx->arena.reserve(512));
        long long *tot0 = ctx->arena.take<long long>(2);
        GBM_CUDA(cudaMemsetAsync(tot0, 0, 16, s));
        const int ct = try_root_tensor(ctx, q, qm, qpair_d, grad_bits, reinterpret_cast<long long *>(hist_d), tot0, n_sel, s);
        if (ct != 0) return ct < 0 ? ct : GBM_OK;
    }
    if (!rows_d && plan_root_staged(ctx, q, qm, hp, grad_bits, n_sel, hr)) {
        // the staged bank-column root of gbm_build_tree (hist_cs_range / hist_csg_range), so it can
        // be compared bin for bin with the oracle
        GBM_TRY(ctx->arena.reserve(hr.cgroups.size() * sizeof(ColGroup) + 512));
        ColGroup *cgs = ctx->arena.take<ColGroup>(hr.cgroups.size());
        long long *tot = ctx->arena.take<long long>(2);
        GBM_CUDA(cudaMemcpyAsync(cgs, hr.cgroups.data(), hr.cgroups.size() * sizeof(ColGroup), cudaMemcpyHostToDevice, s));
        GBM_CUDA(cudaMemsetAsync(tot, 0, 16, s));
        return launch_root_staged(ctx, hr, qm, q, qpair_d, cgs, reinterpret_cast<long long *>(hist_d), tot, n_sel,
                                  (double)q->n_features * q->bits / 8.0, s);
    }
    if (hp.col) {
        GBM_TRY(ctx->arena.reserve(hp.cgroups.size() * sizeof(ColGroup) + 256));
        ColGroup *cgs = ctx->arena.take<ColGroup>(hp.cgroups.size());
        GBM_CUDA(cudaMemcpyAsync(cgs, hp.cgroups.data(), hp.cgroups.size() * sizeof(ColGroup), cudaMemcpyHostToDevice, s));
        ColRangeArgs ca = {};
        ca.qm = qm;
        ca.qpair = reinterpret_cast<const int2 *>(qpair_d);
        ca.ridx = rows_d;
        ca.n_sel = n_sel;
        ca.chunk = hp.chunk;
        ca.n_groups = (int)hp.cgroups.size();
        ca.groups = cgs;
        ca.cut_ptr = q->cut_ptr_d;
        ca.hist = reinterpret_cast<unsigned long long *>(hist_d);
        ca.cstride = hp.cstride;
        int slot = -1;
        ca.rows_ctr = prof_rows_slot(ctx, &slot);
        ProfScope ps(ctx, PC_HIST_LEVEL, s, 0.0, slot, (double)q->n_features * q->bits / 8.0 + 8.0 + (rows_d ? 4.0 : 0.0));
        const long long n_items = (n_sel + hp.chunk - 1) / hp.chunk * (long long)hp.cgroups.size();
        const int grid = (int)std::max<long long>(1, std::min<long long>(n_items, hp.blocks_range));
        launch_col_range(hp, ca, grid, s);
        GBM_CUDA(cudaGetLastError());
        return GBM_OK;
    }
    GBM_TRY(ctx->arena.reserve(hp.groups.size() * sizeof(Group) + 256));
    Group *groups = ctx->arena.take<Group>(hp.groups.size());
    GBM_CUDA(cudaMemcpyAsync(groups, hp.groups.data(), hp.groups.size() * sizeof(Group), cudaMemcpyHostToDevice, s));
    RangeArgs a = {};
    a.qm = qm;
    a.qpair = reinterpret_cast<const int2 *>(qpair_d);
    a.ridx = rows_d;
    a.n_sel = n_sel;
    a.chunk = hp.chunk;
    a.n_groups = (int)hp.groups.size();
    a.groups = groups;
    a.cut_ptr = q->cut_ptr_d;
    a.hist = reinterpret_cast<unsigned long long *>(hist_d);
    a.hstride = hp.hstride;
    int slot = -1;
    a.rows_ctr = prof_rows_slot(ctx, &slot);
    ProfScope ps(ctx, PC_HIST_LEVEL, s, 0.0, slot, (double)q->n_features * q->bits / 8.0 + 8.0 + (rows_d ? 4.0 : 0.0));
    return GBM_DISPATCH(hp, launch_range, ctx, hp, a, s);
}

int gbm_allreduce_histograms(gbm_ctx *ctx, int64_t *hist_d, int64_t count, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_REQUIRE(hist_d && count >= 0, GBM_E_ARG, "gbm_allreduce_histograms: bad arguments");
    ProfScope ps(ctx, PC_ALLREDUCE, (cudaStream_t)stream, (double)count * 8);
    return allreduce_i64(ctx, reinterpret_cast<long long *>(hist_d), (size_t)count, (cudaStream_t)stream);
}

int gbm_evaluate_splits(gbm_ctx *ctx, const gbm_qmatrix *q, const int64_t *hist_d, const int64_t *totals_d,
                        int32_t n_nodes, const int32_t *scale_d, const gbm_params *prm, int8_t *split_d,
                        int32_t *feature_d, int32_t *bin_d, int8_t *default_left_d, double *gain_d,
                        int64_t *child_d, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_REQUIRE(q && q->cut_ptr_d && q->cut_ptr_h && hist_d && totals_d && scale_d && prm && split_d && feature_d &&
                    bin_d && default_left_d && gain_d && child_d && n_nodes >= 0,
                GBM_E_ARG, "gbm_evaluate_splits: bad arguments");
    if (n_nodes == 0) return GBM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    EvalArgs a = eval_args_base(ctx, q, scale_d, prm);
    a.n_nodes = n_nodes;
    a.hist_direct = reinterpret_cast<const long long *>(hist_d);
    a.totals_direct = reinterpret_cast<const long long *>(totals_d);
    GBM_TRY(ctx->arena.reserve((size_t)n_nodes * a.F * sizeof(FeatBest) + 256));
    a.fb = ctx->arena.take<FeatBest>((size_t)n_nodes * a.F);
    ProfScope ps(ctx, PC_EVAL, s);
    const long long warps = (long long)n_nodes * a.F;
    if (ctx->eval_warp == 1 || (ctx->eval_warp == 0 && warps >= 16ll * ctx->sm_count))
        eval_feat_kernel<<<(int)((warps + E_THREADS / 32 - 1) / (E_THREADS / 32)), E_THREADS, 0, s>>>(a);
    else
        eval_feat_blk_kernel<<<(int)warps, E_THREADS, 0, s>>>(a);
    eval_out_kernel<<<n_nodes, E_THREADS, 0, s>>>(a, split_d, feature_d, bin_d, default_left_d, gain_d,
                                                  reinterpret_cast<long long *>(child_d));
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

int gbm_repartition(gbm_ctx *ctx, const gbm_qmatrix *q, const uint32_t *rows_d, int64_t n_sel, int32_t feature,
                    int32_t bin, int32_t default_left, uint32_t *out_d, int64_t *n_left_d, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_TRY(check_qm(q));
    GBM_REQUIRE(n_left_d && n_sel >= 0 && feature >= 0 && feature < q->n_features && ((rows_d && out_d) || n_sel == 0),
                GBM_E_ARG, "gbm_repartition: bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    if (n_sel == 0) {
        GBM_CUDA(cudaMemsetAsync(n_left_d, 0, sizeof(int64_t), s));
        return GBM_OK;
    }
    const QM qm = make_qm(q);
    HistPlan hp;
    GBM_TRY(plan_hist(ctx, q, qm, false, n_sel, hp, 30, false));
    const int tiles = (int)((n_sel + PT - 1) / PT);

    Arena &A = ctx->arena;
    GBM_TRY(A.reserve(3 * sizeof(NodeDev) + (size_t)tiles * (PT / 32) * 4 + 2 * (size_t)tiles * 4 + 32 * 256 +
                      64 + (size_t)q->cut_ptr_h[q->n_features] * 16 + hp.groups.size() * 16 +
                      1024));
    NodeDev *nodes = A.take<NodeDev>(3);
    int *tile_base = A.take<int>(4);
    uint32_t *flags = A.take<uint32_t>((size_t)tiles * (PT / 32));
    int *tile_left = A.take<int>(tiles);
    int *tile_off = A.take<int>(tiles);
    int *n_items = A.take<int>(4);  // [0] items, [1] work counter, [2] tiles per item
    int *run_base = A.take<int>(4);
    unsigned long long *hist = A.take<unsigned long long>((size_t)std::max(1, q->cut_ptr_h[q->n_features]) * 2);
    Group *groups = A.take<Group>(hp.groups.size());
    NodeDev h[3] = {};
    h[0].start = 0;
    h[0].count = n_sel;
    h[0].state = GBM_NODE_SPLIT;
    h[0].f = feature;
    h[0].b = bin;
    h[0].dl = default_left ? 1 : 0;
    h[0].build_left = 1;
    GBM_CUDA(cudaMemcpyAsync(nodes, h, sizeof(h), cudaMemcpyHostToDevice, s));
    GBM_CUDA(cudaMemcpyAsync(groups, hp.groups.data(), hp.groups.size() * sizeof(Group), cudaMemcpyHostToDevice, s));
    plan_kernel<<<1, 1024, 0, s>>>(nodes, 0, 1, 1, tile_base, run_base, n_items);  // group 0 only: flags
    GBM_CUDA(cudaMemsetAsync(tile_left, 0, sizeof(int) * (size_t)tiles, s));
    FusedArgs fa = {};
    fa.qm = qm;
    fa.nodes = nodes;
    fa.first = 0;
    fa.n_par = 1;
    fa.tile_base = tile_base;
    fa.run_base = run_base;
    fa.n_groups = 1;
    fa.run_tiles = 1;
    fa.n_items = n_items;
    fa.ridx_in = rows_d;
    fa.flags = flags;
    fa.tile_left = tile_left;
    fa.qpair = nullptr;  // histogram of a dummy group is not computed: see n_groups = 1 below
    fa.groups = groups;
    fa.cut_ptr = q->cut_ptr_d;
    fa.hist = hist;
    fa.TB = q->cut_ptr_h[q->n_features];
    fa.hstride = hp.hstride;
    fa.rep_cap = hp.rep_cap;
    // the fused kernel needs a qpair for the build rows: use a zero pair array of the rows
    int2 *zq;
    GBM_CUDA(cudaMallocAsync((void **)&zq, sizeof(int2) * (size_t)q->n_rows, s));
    GBM_CUDA(cudaMemsetAsync(zq, 0, sizeof(int2) * (size_t)q->n_rows, s));
    fa.qpair = zq;
    GBM_TRY(GBM_DISPATCH(hp, launch_fused, ctx, hp, fa, s, false));
    part_scan_kernel<<<1, 1024, 0, s>>>(nodes, 0, tile_base, tile_left, tile_off, nullptr);
    part_scatter_kernel<false><<<std::max(1, std::min(tiles, ctx->sm_count * 8)), P_THREADS, 0, s>>>(
        nodes, 0, 1, tile_base, flags, tile_off, rows_d, out_d, nullptr, nullptr);
    GBM_CUDA(cudaGetLastError());
    GBM_CUDA(cudaFreeAsync(zq, s));
    GBM_CUDA(cudaMemcpyAsync(n_left_d, &nodes[1].count, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    GBM_CUDA(cudaStreamSynchronize(s));  // host staging above must outlive the copies
    return GBM_OK;
}

}  // extern "C"

// gbm_build_tree / gbm_build_tree_fused: ep (nullable) is fused into the final walk when the
// staged walk applies (*ep_done = true); otherwise the caller runs it as separate kernels.
// argument checks of gbm_build_tree (local decision; build_tree_impl makes it collective)
static int validate_tree_args(gbm_ctx *ctx, const gbm_qmatrix *q, const int32_t *qpair_d, const int32_t *scale_d,
                              const gbm_params *prm, const gbm_tree *tree, const int32_t *row_leaf_d) {
    GBM_TRY(check_qm(q));
    GBM_REQUIRE(prm && tree && scale_d && ((row_leaf_d && qpair_d) || q->n_rows == 0), GBM_E_ARG,
                "gbm_build_tree: null argument");
    GBM_REQUIRE(tree->kind && tree->feature && tree->bin && tree->threshold && tree->default_left && tree->gain &&
                    tree->weight && tree->sum_qg && tree->sum_qh,
                GBM_E_ARG, "gbm_build_tree: null tree array");
    GBM_REQUIRE(prm->grow_policy == GBM_GROW_DEPTHWISE || prm->grow_policy == GBM_GROW_LOSSGUIDE, GBM_E_ARG,
                "gbm_build_tree: grow_policy must be GBM_GROW_DEPTHWISE or GBM_GROW_LOSSGUIDE");
    if (prm->grow_policy == GBM_GROW_LOSSGUIDE) {
        GBM_REQUIRE(prm->max_leaves >= 1 && prm->max_leaves <= 65536, GBM_E_ARG,
                    "gbm_build_tree: lossguide max_leaves in 1..65536");
        GBM_REQUIRE(prm->max_depth >= 0, GBM_E_ARG, "gbm_build_tree: max_depth >= 0");
        GBM_REQUIRE(tree->left_child, GBM_E_ARG, "gbm_build_tree: lossguide trees need left_child");
    } else {
        GBM_REQUIRE(prm->max_depth >= 0 && prm->max_depth <= 16, GBM_E_ARG, "gbm_build_tree: max_depth in 0..16");
    }
    GBM_REQUIRE(prm->grad_bits >= 1 && prm->grad_bits <= 30, GBM_E_ARG, "gbm_build_tree: grad_bits in 1..30");
    GBM_REQUIRE(prm->lambda >= 0 && prm->gamma >= 0 && prm->min_child_weight >= 0, GBM_E_ARG,
                "gbm_build_tree: lambda, gamma, min_child_weight must be >= 0");
    const long long n = q->n_rows;
    GBM_REQUIRE(n > 0 || (coll_on(ctx) && ctx->nranks > 1), GBM_E_EMPTY, "gbm_build_tree: zero rows (S:321)");
    return GBM_OK;
}

static int build_tree_impl(gbm_ctx *ctx, const gbm_qmatrix *q, const int32_t *qpair_d, const int32_t *scale_d,
                           const gbm_params *prm, const gbm_tree *tree, int32_t *row_leaf_d, void *stream,
                           const gbm_epilogue *ep, bool *ep_done) {
    GBM_TRY(ctx_enter(ctx));
    // every argument check decides locally; the ranks then agree (one collective) so that all of
    // them return the same error -- or GBM_E_MISMATCH when their shapes differ -- and none enters
    // a histogram allreduce its peers skip
    int rc = validate_tree_args(ctx, q, qpair_d, scale_d, prm, tree, row_leaf_d);
    long long sig[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    if (q && q->cut_ptr_h && prm && q->n_features > 0) {
        const long long v[9] = {q->n_features, q->cut_ptr_h[q->n_features], q->bits, q->row_align_bits,
                                q->max_bins, prm->max_depth, prm->grow_policy, prm->max_leaves, prm->grad_bits};
        std::copy(v, v + 9, sig);
    }
    rc = coll_agree(ctx, rc, sig, 9, (cudaStream_t)stream, "gbm_build_tree");
    if (rc != GBM_OK) return rc;
    const long long n = q->n_rows;

    cudaStream_t s = (cudaStream_t)stream;
    const QM qm = make_qm(q);
    if (prm->grow_policy == GBM_GROW_LOSSGUIDE)
        return build_tree_lossguide(ctx, q, qm, qpair_d, scale_d, prm, tree, row_leaf_d, s);
    const int F = q->n_features, D = prm->max_depth;
    const long long TB = q->cut_ptr_h[F];
    const long long cap = (1ll << (D + 1)) - 1;
    HistPlan hp;
    GBM_TRY(plan_hist(ctx, q, qm, prm->grad_bits > 15, std::max<long long>(n, 1), hp, prm->grad_bits,
                      ctx->hist_layout == 2 || ctx->hist_layout == 3, ctx->hist_layout == 3));
    const int G = hp.col ? (int)hp.cgroups.size() : (int)hp.groups.size();
    const size_t esz = hp.carry ? 8 : 4;  // bytes per level entry
    HistPlan hr;
    const bool root_staged = plan_root_staged(ctx, q, qm, hp, prm->grad_bits, n, hr);

    // ---- scratch (tree arena)
    const int max_par = D >= 1 ? (1 << (D - 1)) : 1;  // parents of one level
    const long long max_tiles = (n + PT - 1) / PT + 2ll * max_par + 2;  // (runs <= tiles)
    const long long slots = std::max(1, D >= 2 ? (1 << (D - 2)) : 1);
    const size_t hist_unit = (size_t)std::max<long long>(TB, 1) * 2;
    size_t need = 0;
    need += 2 * (size_t)std::max<long long>(n, 1) * 8 + 512;          // ridx entries x2
    need += (size_t)max_tiles * (PT / 32) * 4 + 256;                  // flags
    need += 2 * (size_t)max_tiles * 4 + 512;                          // tile_left/off
    need += 2 * ((size_t)(2 * max_par + 2) * 4 + 256);                // tile base x2
    need += (size_t)(2 * cap + 2) * sizeof(NodeDev) + 256;            // nodes
    need += 2 * ((size_t)(2 * max_par + 2) * 4 + 512);                // run base + count x2
    need += G * std::max(sizeof(Group), sizeof(ColGroup)) + 256;
    need += (root_staged ? hr.cgroups.size() : 1) * sizeof(ColGroup) + 256;
    need += (slots * hist_unit + hist_unit + 2) * 8 + 512;            // build + root
    need += 2 * slots * hist_unit * 8 + 512;                          // level hists
    need += (size_t)std::max(1, 1 << std::max(0, D - 1)) * F * sizeof(FeatBest) + 512;
    need += (1 + (size_t)max_par) * sizeof(unsigned) + 256;           // eval counters
    need += ((size_t)max_par + 1) * 4 + 8 + 512;                      // segment plan
    // row-order decisions (GBM_OPT_ROW_DECIDE): rows of whole words, <= 16 words
    const int dW = (qm.stride % 32 == 0) ? (int)(qm.stride / 32) : 0;
    // measured slower end to end (the extra streaming pass costs more than the gathers it
    // removes: Higgs 2.06 vs 1.73, Airline 24.6 vs 19.9 ms/round), so only when forced
    const bool row_decide = D > 1 && D <= 12 && dW >= 1 && dW <= 16 && ctx->row_decide == 2;
    if (row_decide) need += (size_t)((n + 31) / 32) * 4 + 256;
    // records level path (records.cu): 8-bit symbols, <= 32 features, rows of whole words
    const int RW = (qm.stride % 32 == 0) ? (int)(qm.stride / 32) : 0;
    const bool rec_ok = D >= 2 && q->bits == 8 && F <= 32 && RW >= 1 && RW <= 8 && !row_decide;
    // measured slower than the row-index path in the whole round on Higgs (2.17-2.25 vs 1.83 ms/round:
    // twice the DRAM bytes per level, the block-wide reservation), so only when forced
    const bool rec = rec_ok && ctx->level_path == 2;
    const int RWP = rec ? rec_row_words(RW) : 0;
    const size_t rec_rows_bytes = (size_t)std::max<long long>(n, 1) * RWP * 4 + 64;
    const size_t rec_q_bytes = (size_t)std::max<long long>(n, 1) * 8 + 64;
    if (rec) {
        need -= 2 * (size_t)std::max<long long>(n, 1) * 8;                  // no ridx lists
        need += 2 * (rec_rows_bytes + 256) + 2 * (rec_q_bytes + 256);       // two record buffers
        need += (size_t)(2 * cap + 2) * 2 * 8 + 256;                        // cursors
    }
    // reduce-scatter + feature-sliced evaluation (§8(f)#1; GBM_OPT_EVAL_SLICED): rank r owns the
    // contiguous features f0[r] .. f0[r] + nf[r] - 1 (bins balanced), receives only their summed
    // histograms (ncclReduceScatter instead of ncclAllReduce: half the bytes per rank), evaluates
    // them, and the ranks all-gather their best candidates before the replicated node reduction
    const int P = ctx->nranks;
    const bool sliced = ctx->eval_sliced == 1 && coll_on(ctx) && P > 1 && !rec;
    std::vector<int> sl_f0(P + 1, 0), sl_nf(P, 0), sl_bin(P + 1, 0);
    long long CB = 1;
    int fsmax = 1;
    if (sliced) {
        for (int r = 0; r <= P; ++r) {
            const long long target = (long long)TB * r / P;
            int f = 0;
            while (f < F && q->cut_ptr_h[f] < target) ++f;
            sl_f0[r] = r == P ? F : f;
        }
        for (int r = 0; r < P; ++r) {
            sl_nf[r] = sl_f0[r + 1] - sl_f0[r];
            sl_bin[r] = q->cut_ptr_h[sl_f0[r]];
            fsmax = std::max(fsmax, sl_nf[r]);
        }
        sl_bin[P] = (int)TB;
        for (int r = 0; r < P; ++r) CB = std::max<long long>(CB, sl_bin[r + 1] - sl_bin[r]);
        const size_t sunit = (size_t)CB * 2;
        need += (size_t)P * slots * sunit * 8 + 512;            // send
        need += (size_t)slots * sunit * 8 + 512;                // received built slots
        need += 2 * (size_t)slots * sunit * 8 + 512;            // received level slots x2
        need += (sunit + 2) * 8 + 512;                          // received root
        need += (size_t)P * std::max(1, 1 << std::max(0, D - 1)) * 2 * fsmax * sizeof(FeatBest) + 512;
        need += 3 * (size_t)(P + 1) * 4 + 768;                  // slice tables
    }
    Arena &A = ctx->tree_arena;
    GBM_TRY(A.reserve(need));
    char *ridx[2] = {nullptr, nullptr};
    if (!rec) {
        ridx[0] = A.take<char>(std::max<long long>(n, 1) * esz);
        ridx[1] = A.take<char>(std::max<long long>(n, 1) * esz);
    }
    uint32_t *rec_rows[2] = {nullptr, nullptr};
    int2 *rec_q[2] = {nullptr, nullptr};
    unsigned long long *cursor = nullptr;
    if (rec) {
        for (int b = 0; b < 2; ++b) {
            rec_rows[b] = reinterpret_cast<uint32_t *>(A.take<char>(rec_rows_bytes));
            rec_q[b] = reinterpret_cast<int2 *>(A.take<char>(rec_q_bytes));
        }
        cursor = A.take<unsigned long long>((size_t)(2 * cap + 2) * 2);
    }
    uint32_t *flags = A.take<uint32_t>((size_t)max_tiles * (PT / 32));
    int *tile_left = A.take<int>(max_tiles);
    int *tile_off = A.take<int>(max_tiles);
    // plans double-buffered by level parity: level l+1 is planned (by level l's evaluation) while
    // level l's scatter still reads level l's plan on the side stream
    int *tile_base_b[2] = {A.take<int>(2 * max_par + 2), A.take<int>(2 * max_par + 2)};
    NodeDev *nodes = A.take<NodeDev>(2 * cap + 2);
    int *run_base_b[2] = {A.take<int>(2 * max_par + 2), A.take<int>(2 * max_par + 2)};
    int *n_items_b[2] = {A.take<int>(4), A.take<int>(4)};  // [0] items, [1] work counter, [2] tiles per item
    Group *groups = A.take<Group>(hp.col ? 1 : G);
    ColGroup *cgroups = A.take<ColGroup>(hp.col ? G : 1);
    ColGroup *cg_root = A.take<ColGroup>(root_staged ? hr.cgroups.size() : 1);
    long long *hist_root = A.take<long long>(hist_unit + 2);  // root histogram + totals
    long long *hist_build = A.take<long long>(slots * hist_unit);
    long long *hist_lvl[2] = {A.take<long long>(slots * hist_unit), A.take<long long>(slots * hist_unit)};
    FeatBest *fb = A.take<FeatBest>((size_t)std::max(1, 1 << std::max(0, D - 1)) * F);
    unsigned *done = A.take<unsigned>(1 + (size_t)max_par);  // [0] nodes completed, [1..] warps per node
    int *seg_base = A.take<int>((size_t)max_par + 1);
    int *seg_items = A.take<int>(2);
    uint32_t *dbits = row_decide ? A.take<uint32_t>((size_t)((n + 31) / 32)) : nullptr;
    long long *sl_send = nullptr, *sl_build = nullptr, *sl_lvl[2] = {nullptr, nullptr}, *sl_root = nullptr;
    FeatBest *fb_all = nullptr;
    int *sl_f0_d = nullptr, *sl_nf_d = nullptr, *sl_bin_d = nullptr;
    const long long sl_shift = sliced ? 2ll * sl_bin[ctx->rank] : 0;  // slice base -> global bin index
    if (sliced) {
        const size_t sunit = (size_t)CB * 2;
        sl_send = A.take<long long>((size_t)P * slots * sunit);
        sl_build = A.take<long long>((size_t)slots * sunit);
        sl_lvl[0] = A.take<long long>((size_t)slots * sunit);
        sl_lvl[1] = A.take<long long>((size_t)slots * sunit);
        sl_root = A.take<long long>(sunit + 2);
        fb_all = A.take<FeatBest>((size_t)P * std::max(1, 1 << std::max(0, D - 1)) * 2 * fsmax);
        sl_f0_d = A.take<int>(P + 1);
        sl_nf_d = A.take<int>(P + 1);
        sl_bin_d = A.take<int>(P + 1);
        std::vector<int> key = {(int)A.generation, (int)(reinterpret_cast<uintptr_t>(sl_f0_d) & 0x7fffffff), P};
        key.insert(key.end(), sl_f0.begin(), sl_f0.end());
        key.insert(key.end(), sl_bin.begin(), sl_bin.end());
        if (key != ctx->tree_slice_key) {  // uploaded once per shape (never inside a graph capture)
            GBM_CUDA(cudaMemcpyAsync(sl_f0_d, sl_f0.data(), (P + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
            GBM_CUDA(cudaMemcpyAsync(sl_nf_d, sl_nf.data(), P * sizeof(int), cudaMemcpyHostToDevice, s));
            GBM_CUDA(cudaMemcpyAsync(sl_bin_d, sl_bin.data(), (P + 1) * sizeof(int), cudaMemcpyHostToDevice, s));
            GBM_CUDA(cudaStreamSynchronize(s));  // the host vectors go out of scope
            ctx->tree_slice_key = key;
        }
    }
    GBM_TRY(upload_groups(ctx, hp, groups, cgroups, A, s, root_staged ? &hr : nullptr, cg_root));
    const TreeDev t = tree_dev(tree);
    const double row_bytes = (double)F * q->bits / 8.0;  // algorithmic bytes of one packed row
    // C2 of the sliced mode: this rank's partial slots -> the summed slots of its feature slice
    auto slice_reduce = [&](const long long *hist, int n_slots, long long *recv) -> int {
        const long long total = (long long)P * n_slots * CB;
        slice_permute_kernel<<<(int)std::min<long long>((total + 255) / 256, 4096), 256, 0, s>>>(
            hist, n_slots, std::max<long long>(TB, 1), sl_bin_d, P, CB, sl_send);
        GBM_CUDA(cudaGetLastError());
        ++ctx->launches;
        ProfScope ps(ctx, PC_ALLREDUCE, s, (double)n_slots * CB * 16 * P);
        return coll_reduce_scatter_i64(ctx, sl_send, recv, (size_t)n_slots * CB * 2, s);
    };
    // features-only evaluation of this rank's slice, all-gather of the candidates, node reduction
    auto sliced_eval = [&](EvalArgs e, bool wait_scan) -> int {
        e.sliced = 1;
        e.f0 = sl_f0[ctx->rank];
        e.F = sl_nf[ctx->rank];
        e.TB = CB;
        e.fsmax = fsmax;
        const size_t fbb = (size_t)e.n_nodes * fsmax * sizeof(FeatBest);
        if (e.F > 0) {
            ProfScope ps(ctx, PC_EVAL, s, (double)e.n_nodes * CB * 16);
            GBM_TRY(launch_eval_tree(ctx, e, t, s));
        }
        {
            ProfScope ps(ctx, PC_ALLREDUCE, s, (double)fbb * P);
            GBM_TRY(coll_allgather(ctx, fb, fb_all, fbb, s));
        }
        if (wait_scan) GBM_CUDA(cudaStreamWaitEvent(s, ctx->ev_scan, 0));
        e.sliced = 0;
        e.fb_all = fb_all;
        e.slice_f0 = sl_f0_d;
        e.slice_nf = sl_nf_d;
        e.nslices = P;
        ProfScope ps(ctx, PC_EVAL_FINAL, s);
        eval_final_sliced_kernel<<<e.n_nodes, E_THREADS, 0, s>>>(e, t);
        GBM_CUDA(cudaGetLastError());
        return GBM_OK;
    };


    {
        ProfScope ps(ctx, PC_INIT, s);
        init_tree_kernel<<<(int)std::min<long long>((cap + 255) / 256, 1024), 256, 0, s>>>(t, cap, nodes, n);
    }
    if (rec) {
        ProfScope ps(ctx, PC_INIT, s);
        GBM_TRY(rec_root_launch(ctx, cursor, n, s));
    }

    // ---- InitRoot: root histogram + totals, allreduce, evaluate
    GBM_CUDA(cudaMemsetAsync(hist_root, 0, (hist_unit + 2) * 8, s));
    const int root_ct = (n > 0 && TB > 0) ? try_root_tensor(ctx, q, qm, qpair_d, prm->grad_bits, hist_root,
                                                            hist_root + hist_unit, n, s)
                                          : 0;
    if (root_ct < 0) return root_ct;
    if (root_ct == 1) {
        // the tensor-fed root (root_ct.cu)
    } else if (n > 0 && TB > 0 && root_staged) {
        GBM_TRY(launch_root_staged(ctx, hr, qm, q, qpair_d, cg_root, hist_root, hist_root + hist_unit, n, row_bytes, s));
    } else if (n > 0 && TB > 0 && hp.col) {
        ColRangeArgs ca = {};
        ca.qm = qm;
        ca.qpair = reinterpret_cast<const int2 *>(qpair_d);
        ca.ridx = nullptr;
        ca.n_sel = n;
        ca.chunk = hp.chunk;
        ca.n_groups = G;
        ca.groups = cgroups;
        ca.cut_ptr = q->cut_ptr_d;
        ca.hist = reinterpret_cast<unsigned long long *>(hist_root);
        ca.totals = reinterpret_cast<unsigned long long *>(hist_root + hist_unit);
        ca.cstride = hp.cstride;
        int slot = -1;
        ca.rows_ctr = prof_rows_slot(ctx, &slot);
        ProfScope ps(ctx, PC_HIST_ROOT, s, 0.0, slot, row_bytes + 8.0);
        const long long n_it = (n + hp.chunk - 1) / hp.chunk * (long long)G;
        const int grid = (int)std::max<long long>(1, std::min<long long>(n_it, hp.blocks_range));
        launch_col_range(hp, ca, grid, s);
        GBM_CUDA(cudaGetLastError());
    } else if (n > 0 && TB > 0) {
        RangeArgs ra = {};
        ra.qm = qm;
        ra.qpair = reinterpret_cast<const int2 *>(qpair_d);
        ra.ridx = nullptr;
        ra.n_sel = n;
        ra.chunk = hp.chunk;
        ra.n_groups = G;
        ra.groups = groups;
        ra.cut_ptr = q->cut_ptr_d;
        ra.hist = reinterpret_cast<unsigned long long *>(hist_root);
        ra.totals = reinterpret_cast<unsigned long long *>(hist_root + hist_unit);
        ra.hstride = hp.hstride;
        int slot = -1;
        ra.rows_ctr = prof_rows_slot(ctx, &slot);  // device-counted: correct under graph replays too
        ProfScope ps(ctx, PC_HIST_ROOT, s, 0.0, slot, row_bytes + 8.0);
        GBM_TRY(GBM_DISPATCH(hp, launch_range, ctx, hp, ra, s));
    } else if (n > 0) {
        return fail(GBM_E_ARG, "gbm_build_tree: no feature has a cut (all values missing)");
    }
    if (sliced) {  // the root's totals (all ranks), its histogram cut into the feature slices
        {
            ProfScope ps(ctx, PC_ALLREDUCE, s, 16.0);
            GBM_TRY(allreduce_i64(ctx, hist_root + hist_unit, 2, s));
        }
        GBM_TRY(slice_reduce(hist_root, 1, sl_root));
    } else {
        ProfScope ps(ctx, PC_ALLREDUCE, s, (double)(hist_unit + 2) * 8);
        GBM_TRY(allreduce_i64(ctx, hist_root, hist_unit + 2, s));
    }
    GBM_CUDA(cudaMemsetAsync(done, 0, (1 + (size_t)max_par) * sizeof(unsigned), s));
    EvalArgs ea = eval_args_base(ctx, q, scale_d, prm);
    ea.nodes = nodes;
    ea.hist_root = hist_root;
    ea.hist_build = hist_build;
    ea.fb = fb;
    // tiles per fused work item: about 4 items per resident block at the widest level (items are
    // claimed dynamically; measured on Higgs: 4 tiles 0.79 ms, 8 tiles 0.84, 16 tiles 0.99 / round)
    // several feature groups: partition each level once, then histogram the built segments per
    // group (hist_seg_kernel) instead of re-partitioning every parent row in every group.
    // Measured: a gain for the generic (non-byte) symbol path (Bosch 4.00 vs 4.20 ms/round), not
    // for byte symbols (Epsilon 4.71 vs 4.57, YearMSD 0.540 vs 0.533), so auto = generic only.
    const bool seg_mode = !hp.col && G > 1 &&
                          (ctx->seg_hist == 2 || (ctx->seg_hist == 0 && !hp.byte_path));
    const int Gf = seg_mode ? 1 : G;  // groups of the fused launch
    // shuffle-fed bank-column level kernel (part_hist_sb_kernel): byte symbols, one group of
    // every feature (F <= 32), rows of whole words, row-index entries without gradient pairs
    const bool sb_ok = !hp.col && hp.byte_path && G == 1 && F <= 32 && qm.stride == 32ll * ((F + 3) / 4) &&
                       !hp.carry && !seg_mode;
    const bool sb_levels = sb_ok && ctx->level_hist == 2;
    // warp-specialised compact level kernel (part_hist_ws_kernel): byte symbols, one group
    const bool ws_levels = !hp.col && hp.byte_path && G == 1 && !hp.carry && !seg_mode && ctx->level_hist == 3;
    int ws_grid = 1;
    if (ws_levels) {
        int occ = 0;
        auto setk = [&](auto kern) -> int {
            GBM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
            GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, H_THREADS, hp.smem_bytes));
            return GBM_OK;
        };
        if (hp.wide) GBM_TRY(setk(part_hist_ws_kernel<true, false>));
        else if (hp.sent) GBM_TRY(setk(part_hist_ws_kernel<false, true>));
        else GBM_TRY(setk(part_hist_ws_kernel<false, false>));
        GBM_REQUIRE(occ >= 1, GBM_E_ARG, "warp-specialised level kernel cannot be resident");
        ws_grid = occ * ctx->sm_count;
    }
    int sb_grid = 1;
    if (sb_levels) {
        const size_t smb = (size_t)(hp.wide ? 4 : 2) * COLB_STRIDE * 4;
        int occ = 0;
        if (hp.wide) {
            GBM_CUDA(cudaFuncSetAttribute(part_hist_sb_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
            GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, part_hist_sb_kernel<true>, H_THREADS, smb));
        } else {
            GBM_CUDA(cudaFuncSetAttribute(part_hist_sb_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
            GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, part_hist_sb_kernel<false>, H_THREADS, smb));
        }
        GBM_REQUIRE(occ >= 1, GBM_E_ARG, "bank-column level kernel cannot be resident");
        sb_grid = occ * ctx->sm_count;
    }
    const long long tiles_all = (n + PT - 1) / PT;
    const long long target = 4ll * hp.blocks_fused;
    const int run_tiles = ctx->run_tiles > 0 ? ctx->run_tiles : (int)std::max<long long>(
        1, std::min<long long>(RUN_MAX, (tiles_all * Gf + target - 1) / target));
    ea.plan_groups = rec ? 1 : Gf;
    // auto: tiles per item chosen per level by the plan for the level kernel's resident blocks
    const int lvl_blocks = sb_levels ? sb_grid : ws_levels ? ws_grid : hp.blocks_fused;
    ea.plan_run = rec ? 1 : ctx->run_tiles > 0 ? run_tiles : -lvl_blocks;  // records: one-tile items, split parents only
    ea.plan_rows = n;
    ea.plan_split_only = rec ? 1 : 0;
    ea.tile_base = tile_base_b[1];  // the root's evaluation plans level 1
    ea.run_base = run_base_b[1];
    ea.n_items = n_items_b[1];
    ea.level = 0;
    ea.first = 0;
    ea.n_nodes = 1;
    ea.done = done;
    ea.node_done = done + 1;
    ea.plan_mode = (1 < D) ? 1 : 0;
    if (sliced) {
        ea.root_tot = hist_root + hist_unit;
        ea.hist_root = sl_root - sl_shift;
        GBM_TRY(sliced_eval(ea, false));
    } else {
        ProfScope ps(ctx, PC_EVAL, s, (double)TB * 16);
        GBM_TRY(launch_eval_tree(ctx, ea, t, s));
    }
    if (D == 0) {  // every row sits in the root leaf
        GBM_CUDA(cudaMemsetAsync(row_leaf_d, 0, sizeof(int32_t) * (size_t)std::max<long long>(n, 0), s));
        return GBM_OK;
    }

    FusedArgs fa = {};
    fa.qm = qm;
    fa.nodes = nodes;
    fa.n_groups = Gf;
    fa.no_hist = seg_mode ? 1 : 0;
    fa.run_tiles = run_tiles;
    fa.flags = flags;
    fa.tile_left = tile_left;
    fa.row_leaf = row_leaf_d;
    fa.qpair = reinterpret_cast<const int2 *>(qpair_d);
    fa.groups = groups;
    fa.cut_ptr = q->cut_ptr_d;
    fa.hist = reinterpret_cast<unsigned long long *>(hist_build);
    fa.TB = std::max<long long>(TB, 1);
    fa.hstride = hp.hstride;
    fa.rep_cap = hp.rep_cap;
    const int pgrid = ctx->sm_count * 8;
    for (int l = 1; l <= D; ++l) {
        const int first = (1 << (l - 1)) - 1, n_par = 1 << (l - 1);
        const char *rin = l == 1 ? nullptr : ridx[(l - 1) & 1];
        char *rout = ridx[l & 1];
        int *tile_base = tile_base_b[l & 1], *run_base = run_base_b[l & 1], *n_items = n_items_b[l & 1];
        fa.tile_base = tile_base;
        fa.run_base = run_base;
        fa.n_items = n_items;
        const double ridx_b = rin ? 4.0 : 0.0;
        if (l == D) {  // final level: every row's leaf by a row-order walk of the tree
            const int n_internal = (1 << D) - 1;
            const size_t sm = (size_t)n_internal * 8;
            ProfScope ps(ctx, PC_PART_FINAL, s, (double)n * (q->bits * D / 8.0 + 4.0));
            const int grid = (int)std::max<long long>(1, std::min<long long>((n + WALK_THREADS - 1) / WALK_THREADS,
                                                                            (long long)ctx->sm_count * 8));
            // rows of whole words: staged row-order walk (each packed byte read once); else the
            // feature-major copy (one byte per level) or per-level gathers from the packed rows
            const int W = (qm.stride % 32 == 0) ? (int)(qm.stride / 32) : 0;
            if (n > 0 && sm > 64 * 1024) {
                leaf_walk_global_kernel<<<grid, WALK_THREADS, 0, s>>>(qm, t, D, n, row_leaf_d);
            } else if (n > 0 && W >= 1 && W <= 16 && ctx->walk_mode != 1) {
                WalkEpi wepi_v = {};
                const WalkEpi *wepi = nullptr;
                if (ep) {  // margin update + next round's gradient statistics in the same pass
                    GBM_CUDA(cudaMemsetAsync(ep->maxbits_d, 0, 16, s));
                    wepi_v = WalkEpi{ep->margin_d, ep->label_d, ep->objective, ep->sig_d,
                                     reinterpret_cast<unsigned long long *>(ep->maxbits_d), ctx->dev_err, t.weight};
                    wepi = &wepi_v;
                    *ep_done = true;
                }
                switch (W) {
#define GBM_WALK(w) case w: launch_walk_reg<w>(grid, sm, s, qm, t, n_internal, D, n, row_leaf_d, wepi); break;
                    GBM_WALK(1) GBM_WALK(2) GBM_WALK(3) GBM_WALK(4) GBM_WALK(5) GBM_WALK(6) GBM_WALK(7) GBM_WALK(8)
                    GBM_WALK(9) GBM_WALK(10) GBM_WALK(11) GBM_WALK(12) GBM_WALK(13) GBM_WALK(14) GBM_WALK(15)
                    GBM_WALK(16)
#undef GBM_WALK
                }
            } else if (n > 0) {
                if (sm > 48 * 1024)
                    GBM_CUDA(cudaFuncSetAttribute(leaf_walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
                leaf_walk_kernel<<<grid, WALK_THREADS, sm, s>>>(qm, t.kind, t.feature, t.bin, t.default_left,
                                                                n_internal, D, n, row_leaf_d);
            }
            GBM_CUDA(cudaGetLastError());
            break;
        }
        if (rec) {  // records: partition + smaller-child histogram in one streaming pass
            GBM_CUDA(cudaMemsetAsync(hist_build, 0, (size_t)n_par * hist_unit * 8, s));
            RecLaunch L = {};
            L.nodes = nodes;
            L.first = first;
            L.n_par = n_par;
            L.tile_base = tile_base;
            L.items_hint = (int)std::min<long long>(INT_MAX, tiles_all + n_par);
            if (l == 1) {  // the canonical packed matrix and qpair, identity positions
                L.in_rows = q->packed_d;
                L.in_q = reinterpret_cast<const int2 *>(qpair_d);
                L.in_rows_bytes = (unsigned long long)gbm_packed_words(n, F, q->bits, q->row_align_bits) * 4;
                L.in_q_bytes = (unsigned long long)n * 8;
            } else {
                L.in_rows = rec_rows[(l - 1) & 1];
                L.in_q = rec_q[(l - 1) & 1];
                L.in_rows_bytes = rec_rows_bytes;
                L.in_q_bytes = rec_q_bytes;
            }
            const bool out = l < D - 1;  // the last histogram level moves no rows (the walk follows)
            L.out_rows = out ? rec_rows[l & 1] : nullptr;
            L.out_q = out ? rec_q[l & 1] : nullptr;
            L.cursor = cursor;
            L.cut_ptr = q->cut_ptr_d;
            L.F = F;
            L.B = q->max_bins;
            L.RW = RW;
            L.RW_in = l == 1 ? RW : RWP;
            L.wide = prm->grad_bits > 15;
            L.hist = reinterpret_cast<unsigned long long *>(hist_build);
            L.TB = std::max<long long>(TB, 1);
            int slot;
            L.rows_ctr = prof_rows_slot(ctx, &slot);
            // algorithmic bits of the histogram: per row of the built child its packed
            // row + qpair + row index; the partition bytes are §8(d)'s partition term, not counted
            L.bits_parent_row = 0;
            L.bits_built_row = F * q->bits + 96;
            {
                ProfScope ps(ctx, PC_HIST_LEVEL, s, 0.0, slot, 1.0 / 8.0);
                GBM_TRY(rec_level_launch(ctx, L, s));
            }
            if (out) {  // the children's segments (the next level's plan reads their counts)
                ProfScope ps(ctx, PC_PART_SCAN, s);
                GBM_TRY(rec_seg_launch(ctx, nodes, first, n_par, cursor, s));
            }
            {
                ProfScope ps(ctx, PC_ALLREDUCE, s, (double)n_par * hist_unit * 8);
                GBM_TRY(allreduce_i64(ctx, hist_build, (size_t)n_par * hist_unit, s));
            }
            ea.level = l;
            ea.first = (1 << l) - 1;
            ea.n_nodes = 1 << l;
            ea.hist_prev = l == 1 ? nullptr : hist_lvl[(l - 1) & 1];
            ea.hist_store = (l < D - 1) ? hist_lvl[l & 1] : nullptr;
            ea.plan_mode = (l + 1 < D) ? 1 : 0;
            ea.tile_base = tile_base_b[(l + 1) & 1];
            ea.run_base = run_base_b[(l + 1) & 1];
            ea.n_items = n_items_b[(l + 1) & 1];
            {
                ProfScope ps(ctx, PC_EVAL, s, (double)n_par * hist_unit * 8 * (2.0 + (ea.hist_store ? 2.0 : 0.0)));
                GBM_TRY(launch_eval_tree(ctx, ea, t, s));
            }
            continue;
        }
        GBM_CUDA(cudaMemsetAsync(tile_left, 0, sizeof(int) * (size_t)max_tiles, s));
        // RepartitionInstances + BuildPartialHistograms (fused)
        GBM_CUDA(cudaMemsetAsync(hist_build, 0, (size_t)n_par * hist_unit * 8, s));
        if (row_decide && n > 0) {  // every row's go-left bit at its parent (depth l - 1)
            ProfScope ps(ctx, PC_PART_DECIDE, s, (double)n * (qm.stride / 8.0 + 0.125));
            const int grid = (int)std::max<long long>(1, std::min<long long>((n + WALK_THREADS - 1) / WALK_THREADS,
                                                                            (long long)ctx->sm_count * 8));
            const size_t dsm = (size_t)((2 << (l - 1)) - 1) * 8;
            switch (dW) {
#define GBM_DECIDE(w) case w: row_decide_kernel<w><<<grid, WALK_THREADS, dsm, s>>>(qm, nodes, l - 1, n, dbits); break;
                GBM_DECIDE(1) GBM_DECIDE(2) GBM_DECIDE(3) GBM_DECIDE(4) GBM_DECIDE(5) GBM_DECIDE(6) GBM_DECIDE(7)
                GBM_DECIDE(8) GBM_DECIDE(9) GBM_DECIDE(10) GBM_DECIDE(11) GBM_DECIDE(12) GBM_DECIDE(13)
                GBM_DECIDE(14) GBM_DECIDE(15) GBM_DECIDE(16)
#undef GBM_DECIDE
            }
            GBM_CUDA(cudaGetLastError());
        }
        {
            fa.qm.dbits = dbits;
            fa.first = first;
            fa.n_par = n_par;
            fa.ridx_in = rin;
            int slot;
            fa.rows_ctr = prof_rows_slot(ctx, &slot);
            // algorithmic bits of the histogram: per row of the built child its packed
            // row + row index + qpair (F b / 8 + 12 bytes); the partition inputs the fused kernel also
            // reads (split symbol + row index per parent row) are §8(d)'s partition bytes, not counted
            fa.bits_parent_row = 0;
            fa.bits_built_row = F * q->bits + 96;
            ProfScope ps(ctx, PC_HIST_LEVEL, s, 0.0, slot, 1.0 / 8.0);
            if (hp.col) {
                ColFusedArgs ca = {};
                ca.qm = qm;
                ca.qm.dbits = dbits;
                ca.nodes = nodes;
                ca.first = first;
                ca.n_par = n_par;
                ca.tile_base = tile_base;
                ca.run_base = run_base;
                ca.n_groups = G;
                ca.run_tiles = run_tiles;
                ca.n_items = n_items;
                ca.ridx_in = rin;
                ca.flags = flags;
                ca.tile_left = tile_left;
                ca.row_leaf = row_leaf_d;
                ca.qpair = reinterpret_cast<const int2 *>(qpair_d);
                ca.groups = cgroups;
                ca.cut_ptr = q->cut_ptr_d;
                ca.hist = reinterpret_cast<unsigned long long *>(hist_build);
                ca.TB = std::max<long long>(TB, 1);
                ca.cstride = hp.cstride;
                ca.rows_ctr = fa.rows_ctr;
                ca.bits_parent_row = fa.bits_parent_row;
                ca.bits_built_row = fa.bits_built_row;
                launch_col_fused(hp, ca, s);
                GBM_CUDA(cudaGetLastError());
            } else if (ws_levels) {  // warp-specialised levels
                if (hp.wide) part_hist_ws_kernel<true, false><<<ws_grid, H_THREADS, hp.smem_bytes, s>>>(fa);
                else if (hp.sent) part_hist_ws_kernel<false, true><<<ws_grid, H_THREADS, hp.smem_bytes, s>>>(fa);
                else part_hist_ws_kernel<false, false><<<ws_grid, H_THREADS, hp.smem_bytes, s>>>(fa);
                GBM_CUDA(cudaGetLastError());
            } else if (sb_levels) {  // shuffle-fed bank-column levels
                const size_t smb = (size_t)(hp.wide ? 4 : 2) * COLB_STRIDE * 4;
                if (hp.wide) part_hist_sb_kernel<true><<<sb_grid, H_THREADS, smb, s>>>(fa);
                else part_hist_sb_kernel<false><<<sb_grid, H_THREADS, smb, s>>>(fa);
                GBM_CUDA(cudaGetLastError());
            } else {
                GBM_TRY(GBM_DISPATCH(hp, launch_fused, ctx, hp, fa, s, hp.carry));
            }
        }
        // side stream: scan + scatter of this level, concurrent with the allreduce and (after the
        // scan: the plan of level l+1 needs the children's counts) the evaluation.  In segment
        // mode the histograms need the scattered entries: everything stays on s.
        if (!seg_mode) GBM_TRY(fork_side(ctx, s));
        cudaStream_t ss = seg_mode ? s : ctx->side;
        {
            ProfScope ps(ctx, PC_PART_SCAN, ss);
            part_scan_kernel<<<n_par, 1024, 0, ss>>>(nodes, first, tile_base, tile_left, tile_off, nullptr);
        }
        GBM_CUDA(cudaEventRecord(ctx->ev_scan, ss));
        {
            int slot;
            unsigned long long *rc = prof_rows_slot(ctx, &slot);
            ProfScope ps(ctx, PC_PART_SCATTER, ss, 0.0, slot, ridx_b + 4.0);
            if (hp.carry)
                part_scatter_kernel<true><<<pgrid, P_THREADS, 0, ss>>>(
                    nodes, first, n_par, tile_base, flags, tile_off, reinterpret_cast<const uint2 *>(rin),
                    reinterpret_cast<uint2 *>(rout), reinterpret_cast<const int2 *>(qpair_d), rc);
            else
                part_scatter_kernel<false><<<pgrid, P_THREADS, 0, ss>>>(
                    nodes, first, n_par, tile_base, flags, tile_off, reinterpret_cast<const uint32_t *>(rin),
                    reinterpret_cast<uint32_t *>(rout), nullptr, rc);
        }
        GBM_CUDA(cudaGetLastError());
        if (seg_mode) {  // the built children's segments, group by group
            const long long half = (n / 2 + 2ll * hp.blocks_range - 1) / (2ll * hp.blocks_range);
            const int seg_chunk = (int)std::max<long long>(256, std::min<long long>(MAX_CHUNK, half * G));
            seg_plan_kernel<<<1, 1024, 0, s>>>(nodes, first, n_par, seg_chunk, G, seg_base, seg_items);
            SegArgs sa = {};
            sa.qm = qm;
            sa.nodes = nodes;
            sa.first = first;
            sa.n_par = n_par;
            sa.ridx = rout;
            sa.qpair = reinterpret_cast<const int2 *>(qpair_d);
            sa.seg_base = seg_base;
            sa.n_items = seg_items;
            sa.chunk = seg_chunk;
            sa.n_groups = G;
            sa.groups = groups;
            sa.cut_ptr = q->cut_ptr_d;
            sa.hist = reinterpret_cast<unsigned long long *>(hist_build);
            sa.TB = std::max<long long>(TB, 1);
            sa.hstride = hp.hstride;
            int slot;
            sa.rows_ctr = prof_rows_slot(ctx, &slot);
            ProfScope ps(ctx, PC_HIST_LEVEL, s, 0.0, slot, row_bytes + 8.0 + esz);
            GBM_TRY(GBM_DISPATCH(hp, launch_seg, ctx, hp, sa, s, hp.carry));
        }
        if (sliced) {  // reduce-scatter into this rank's feature slice, sliced evaluation
            GBM_TRY(slice_reduce(hist_build, n_par, sl_build));
            ea.level = l;
            ea.first = (1 << l) - 1;
            ea.n_nodes = 1 << l;
            ea.hist_build = sl_build - sl_shift;
            ea.hist_prev = l == 1 ? nullptr : sl_lvl[(l - 1) & 1] - sl_shift;
            ea.hist_store = (l < D - 1) ? sl_lvl[l & 1] - sl_shift : nullptr;
            ea.plan_mode = (l + 1 < D) ? 1 : 0;
            ea.tile_base = tile_base_b[(l + 1) & 1];
            ea.run_base = run_base_b[(l + 1) & 1];
            ea.n_items = n_items_b[(l + 1) & 1];
            GBM_TRY(sliced_eval(ea, !seg_mode));
            if (!seg_mode) GBM_TRY(wait_on(s, ctx->ev_join, ctx->side));
            continue;
        }
        {  // AllReduceHistograms
            ProfScope ps(ctx, PC_ALLREDUCE, s, (double)n_par * hist_unit * 8);
            GBM_TRY(allreduce_i64(ctx, hist_build, (size_t)n_par * hist_unit, s));
        }
        {  // subtraction + EvaluateSplit for every node of level l
            ea.level = l;
            ea.first = (1 << l) - 1;
            ea.n_nodes = 1 << l;
            ea.hist_prev = l == 1 ? nullptr : hist_lvl[(l - 1) & 1];
            ea.hist_store = (l < D - 1) ? hist_lvl[l & 1] : nullptr;
            ea.plan_mode = (l + 1 < D) ? 1 : 0;  // this level's eval plans level l + 1
            ea.tile_base = tile_base_b[(l + 1) & 1];
            ea.run_base = run_base_b[(l + 1) & 1];
            ea.n_items = n_items_b[(l + 1) & 1];
            if (!seg_mode) GBM_CUDA(cudaStreamWaitEvent(s, ctx->ev_scan, 0));
            {
                ProfScope ps(ctx, PC_EVAL, s, (double)n_par * hist_unit * 8 * (2.0 + (ea.hist_store ? 2.0 : 0.0)));
                GBM_TRY(launch_eval_tree(ctx, ea, t, s));
            }
            if (!seg_mode) GBM_TRY(wait_on(s, ctx->ev_join, ctx->side));  // join: the next level reads the scatter
        }
    }
    return GBM_OK;
}

extern "C" {

int gbm_build_tree(gbm_ctx *ctx, const gbm_qmatrix *q, const int32_t *qpair_d, const int32_t *scale_d,
                   const gbm_params *prm, const gbm_tree *tree, int32_t *row_leaf_d, void *stream) {
    bool done = false;
    return build_tree_impl(ctx, q, qpair_d, scale_d, prm, tree, row_leaf_d, stream, nullptr, &done);
}

int gbm_build_tree_fused(gbm_ctx *ctx, const gbm_qmatrix *q, const int32_t *qpair_d, const int32_t *scale_d,
                         const gbm_params *prm, const gbm_tree *tree, int32_t *row_leaf_d,
                         const gbm_epilogue *ep, void *stream) {
    GBM_REQUIRE(ep && (ep->objective == GBM_SQUARED_ERROR || ep->objective == GBM_LOGISTIC), GBM_E_ARG,
                "gbm_build_tree_fused: bad epilogue");
    GBM_REQUIRE(q && ((ep->margin_d && ep->label_d) || q->n_rows == 0) && ep->maxbits_d &&
                    (ep->objective != GBM_LOGISTIC || ep->sig_d || q->n_rows == 0),
                GBM_E_ARG, "gbm_build_tree_fused: null epilogue buffer");
    bool done = false;
    GBM_TRY(build_tree_impl(ctx, q, qpair_d, scale_d, prm, tree, row_leaf_d, stream, ep, &done));
    if (!done) {  // the separate kernels of gbm_update_margins and pass 1 of gbm_gradients
        cudaStream_t s = (cudaStream_t)stream;
        GBM_TRY(update_margins_launch(ctx, tree->weight, row_leaf_d, q->n_rows, ep->margin_d, s));
        GBM_TRY(grad_pass1(ctx, ep->objective, ep->margin_d, ep->label_d, q->n_rows,
                           reinterpret_cast<unsigned long long *>(ep->maxbits_d), ep->sig_d, s));
    }
    return GBM_OK;
}

}  // extern "C"
