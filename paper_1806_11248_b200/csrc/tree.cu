// tree.cu -- §2.3 decision-tree construction (Algorithm 1) on sm_100a.
//
// The tree is grown level-synchronously (R15): every node of a depth is handled by one launch of
// each kernel, and one NCCL allreduce per level carries the histograms of all of that level's
// built children.  Per level l = 1..D:
//
//   part_count   RepartitionInstances, pass 1: per 1024-row tile of every split parent, the
//                split symbol of each row (gathered from the packed matrix), a warp-ballot flag
//                word per 32 rows, the tile's left count.  Leaf parents write row_leaf.
//   part_scan    one block: per parent an exclusive scan of its tiles' left counts (stable
//                order), the children's segments, the histogram work items of the built child,
//                and the next level's tile plan.
//   part_scatter RepartitionInstances, pass 2: stable scatter of row ids to the children.
//   hist         BuildPartialHistograms of the smaller child of every split (R17): privatised
//                shared-memory int32 histograms (32-bit ATOMS are native on sm_100; 64-bit
//                shared atomics compile to a CAS loop), flushed into int64 global histograms.
//   allreduce    AllReduceHistograms: ncclAllReduce(int64, sum) over the level's buffer.
//   eval         one block per node: sibling = parent - built child (exact in int64), per-feature
//                warp prefix scans, XGBoost gain in the exact op order of R8, canonical argmax.
//
// Exactness of the smem accumulators (R14): a work item covers at most 65535 rows.  With
// grad_bits P <= 15 every |q| <= 2^15, so a bin's int32 sum stays below 65535 * 2^15 < 2^31
// ("narrow", 2 ATOMS per update).  With 15 < P <= 30 each q is split as q = hi*2^15 + lo,
// 0 <= lo < 2^15, |hi| <= 2^15, and hi / lo are accumulated separately ("wide", 4 ATOMS).
#include <algorithm>
#include <climits>
#include <vector>

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

struct HistItem {
    int slot, group;
    long long start;
    int len, pad;
};

struct Group {
    int u_lo, u_hi;      // units [u_lo, u_hi) of the row (a unit = S consecutive features)
    int bin_lo, bin_hi;  // global bins of the group's features
};

constexpr int PT = 1024;           // partition tile (rows)
constexpr int P_THREADS = 256;     // partition block: 8 warps x 4 flag words
constexpr int H_THREADS = 512;     // histogram block
constexpr int E_THREADS = 256;     // evaluate block
constexpr int MAX_CHUNK = 65535;   // rows per histogram work item (exactness bound above)

struct EvalParams {
    double eta, lambda, gamma, mcw;
    int max_depth;
};

// ============================================================== partition
__device__ __forceinline__ int find_parent(const int *__restrict__ tile_base, int n_par, int t) {
    int lo = 0, hi = n_par - 1;  // largest j with tile_base[j] <= t
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(tile_base + mid) <= t) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// mode 0: flags + tile_left (and row_leaf for leaf parents); mode 1: final level (row_leaf)
template <bool FINAL>
__global__ void __launch_bounds__(P_THREADS) part_count_kernel(
    QM qm, const NodeDev *__restrict__ nodes, int first, int n_par, const int *__restrict__ tile_base,
    const uint32_t *__restrict__ ridx_in, uint32_t *__restrict__ flags, int *__restrict__ tile_left,
    int32_t *__restrict__ row_leaf) {
    __shared__ int red[P_THREADS / 32];
    const int n_tiles = tile_base[n_par];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int j = find_parent(tile_base, n_par, t);
        const int k = first + j;
        const NodeDev nd = nodes[k];
        const long long base = nd.start + (long long)(t - tile_base[j]) * PT;
        const long long end = nd.start + nd.count;
        int cnt = 0;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const long long pos = base + wid * 128 + s * 32 + lane;
            const bool valid = pos < end;
            uint32_t row = 0;
            if (valid) row = ridx_in ? __ldg(ridx_in + pos) : (uint32_t)pos;
            if (nd.state == GBM_NODE_LEAF) {
                if (valid) row_leaf[row] = k;
                continue;
            }
            bool left = false;
            if (valid) {
                uint32_t sym = symbol_at(qm, row, nd.f);
                left = (int)sym == qm.B ? (nd.dl != 0) : ((int)sym <= nd.b);
            }
            if (FINAL) {
                if (valid) row_leaf[row] = left ? 2 * k + 1 : 2 * k + 2;
                continue;
            }
            uint32_t w = __ballot_sync(0xffffffffu, valid && left);
            if (lane == 0) flags[(long long)t * (PT / 32) + wid * 4 + s] = w;
            cnt += __popc(w);
        }
        if (!FINAL) {
            if (lane == 0) red[wid] = cnt;
            __syncthreads();
            if (threadIdx.x == 0) {
                int sum = 0;
                for (int w = 0; w < P_THREADS / 32; ++w) sum += red[w];
                tile_left[t] = sum;
            }
            __syncthreads();
        }
    }
}

// Block-wide exclusive scan helper (1024 threads) over int values; returns exclusive prefix and
// the chunk total through *total.
__device__ __forceinline__ long long block_exscan_1024(long long v, long long *total, long long *sm32) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long x = v;
    for (int o = 1; o < 32; o <<= 1) {
        long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm32[wid] = x;
    __syncthreads();
    if (wid == 0) {
        long long s = sm32[lane];
        for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        sm32[lane] = s;
    }
    __syncthreads();
    long long ex = (wid ? sm32[wid - 1] : 0) + x - v;
    *total = sm32[31];
    __syncthreads();
    return ex;
}

// single block (1024 threads): children segments, hist items of the built children, next tiles
__global__ void __launch_bounds__(1024) part_scan_kernel(
    NodeDev *__restrict__ nodes, int first, int n_par, const int *__restrict__ tile_base,
    const int *__restrict__ tile_left, int *__restrict__ tile_off, HistItem *__restrict__ items,
    int *__restrict__ n_items, int n_groups, int chunk, int *__restrict__ next_tile_base,
    int make_items) {
    __shared__ long long sm32[32];
    __shared__ long long item_base[1024];
    // 1. per split parent: exclusive scan of its tiles' left counts -> tile_off, n_left
    for (int j = 0; j < n_par; ++j) {
        const int k = first + j;
        NodeDev nd = nodes[k];
        NodeDev *L = nodes + 2 * k + 1, *R = nodes + 2 * k + 2;
        if (nd.state != GBM_NODE_SPLIT) {
            if (threadIdx.x == 0) {
                L->count = 0; L->start = 0; L->state = GBM_NODE_ABSENT;
                R->count = 0; R->start = 0; R->state = GBM_NODE_ABSENT;
            }
            continue;
        }
        const int t0 = tile_base[j], t1 = tile_base[j + 1];
        long long carry = 0;
        for (int c = t0; c < t1; c += 1024) {
            int t = c + threadIdx.x;
            long long v = t < t1 ? tile_left[t] : 0;
            long long tot;
            long long ex = block_exscan_1024(v, &tot, sm32);
            if (t < t1) tile_off[t] = (int)(carry + ex);
            carry += tot;
        }
        if (threadIdx.x == 0) {
            L->start = nd.start; L->count = carry;
            R->start = nd.start + carry; R->count = nd.count - carry;
        }
        __syncthreads();
    }
    __syncthreads();
    // 2. histogram work items of the built child of every split parent
    if (make_items) {
        const int nthr = 1024;
        for (int c = 0; c < n_par; c += nthr) {
            int j = c + threadIdx.x;
            long long cntj = 0;
            if (j < n_par) {
                const int k = first + j;
                if (nodes[k].state == GBM_NODE_SPLIT) {
                    const NodeDev *ch = nodes + 2 * k + (nodes[k].build_left ? 1 : 2);
                    cntj = ((ch->count + chunk - 1) / chunk) * n_groups;
                }
            }
            item_base[threadIdx.x] = cntj;
            __syncthreads();
            if (threadIdx.x == 0) {
                long long run = c == 0 ? 0 : (long long)*n_items;
                for (int i = 0; i < nthr; ++i) {
                    long long x = item_base[i];
                    item_base[i] = run;
                    run += x;
                }
                *n_items = (int)run;
            }
            __syncthreads();
            if (j < n_par && cntj) {
                const int k = first + j;
                const NodeDev *ch = nodes + 2 * k + (nodes[k].build_left ? 1 : 2);
                long long b = item_base[threadIdx.x];
                for (long long q = 0; q < cntj; ++q) {
                    long long chk = q / n_groups;
                    int g = (int)(q - chk * n_groups);
                    HistItem it;
                    it.slot = j;
                    it.group = g;
                    it.start = ch->start + chk * chunk;
                    it.len = (int)min((long long)chunk, ch->count - chk * chunk);
                    it.pad = 0;
                    items[b + q] = it;
                }
            }
            __syncthreads();
        }
        if (n_par == 0 && threadIdx.x == 0) *n_items = 0;
    }
    __syncthreads();
    // 3. tile plan of the children (the next level's parents), in heap order
    {
        const int n_ch = 2 * n_par, cfirst = 2 * first + 1;
        long long carry = 0;
        for (int c = 0; c < n_ch; c += 1024) {
            int j = c + threadIdx.x;
            long long v = 0;
            if (j < n_ch) v = (nodes[cfirst + j].count + PT - 1) / PT;
            long long tot;
            long long ex = block_exscan_1024(v, &tot, sm32);
            if (j < n_ch) next_tile_base[j] = (int)(carry + ex);
            carry += tot;
        }
        if (threadIdx.x == 0) next_tile_base[n_ch] = (int)carry;
    }
}

__global__ void __launch_bounds__(P_THREADS) part_scatter_kernel(
    const NodeDev *__restrict__ nodes, int first, int n_par, const int *__restrict__ tile_base,
    const uint32_t *__restrict__ flags, const int *__restrict__ tile_off,
    const uint32_t *__restrict__ ridx_in, uint32_t *__restrict__ ridx_out) {
    __shared__ int wpre[PT / 32];
    const int n_tiles = tile_base[n_par];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int j = find_parent(tile_base, n_par, t);
        const int k = first + j;
        const NodeDev nd = nodes[k];
        if (nd.state != GBM_NODE_SPLIT) continue;  // uniform per block
        const long long n_left = nodes[2 * k + 1].count;
        const int lt = t - tile_base[j];
        uint32_t w[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) w[s] = __ldg(flags + (long long)t * (PT / 32) + wid * 4 + s);
        if (lane < 4) wpre[wid * 4 + lane] = __popc(w[lane]);
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = 0;
            for (int i = 0; i < PT / 32; ++i) {
                int x = wpre[i];
                wpre[i] = run;
                run += x;
            }
        }
        __syncthreads();
        const long long off = tile_off[t];
        const uint32_t ltm = (1u << lane) - 1u;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int i = wid * 128 + s * 32 + lane;
            const long long pin = (long long)lt * PT + i;  // position within the node
            if (pin >= nd.count) continue;
            const long long pos = nd.start + pin;
            const uint32_t row = ridx_in ? __ldg(ridx_in + pos) : (uint32_t)pos;
            const long long lb = off + wpre[wid * 4 + s] + __popc(w[s] & ltm);  // lefts before
            const bool left = (w[s] >> lane) & 1u;
            const long long dst = left ? nd.start + lb : nd.start + n_left + (pin - lb);
            ridx_out[dst] = row;
        }
        __syncthreads();
    }
}

// ============================================================== histograms
struct HistArgs {
    QM qm;
    const int2 *qpair;
    const uint32_t *ridx;        // null = identity rows
    const HistItem *items;       // null = arithmetic items over [0, n_sel)
    const int *n_items_dev;
    long long n_sel;             // arithmetic mode: rows
    int chunk, n_groups;
    const Group *groups;
    const int32_t *cut_ptr;
    long long *hist;             // [slots][TB][2]
    long long *totals;           // arithmetic mode: root totals [2] (may be null)
    int TB;
};

template <bool WIDE>
__global__ void __launch_bounds__(H_THREADS) hist_kernel(HistArgs a) {
    extern __shared__ int smem[];
    __shared__ int s_off[2049];     // bin offset (relative to the group) per feature of the group
    __shared__ long long s_red[2][H_THREADS / 32];
    const QM &qm = a.qm;
    const int n_items = a.items ? *a.n_items_dev
                                : (int)(((a.n_sel + a.chunk - 1) / a.chunk) * a.n_groups);
    const uint32_t mask = qm.bits == 32 ? 0xffffffffu : ((1u << qm.bits) - 1u);
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        int slot, g, len;
        long long start;
        if (a.items) {
            HistItem hi = a.items[it];
            slot = hi.slot; g = hi.group; start = hi.start; len = hi.len;
        } else {
            slot = 0;
            g = it % a.n_groups;
            long long ch = it / a.n_groups;
            start = ch * a.chunk;
            len = (int)min((long long)a.chunk, a.n_sel - start);
        }
        const Group grp = a.groups[g];
        const int nb = grp.bin_hi - grp.bin_lo;
        const int f_lo = grp.u_lo * qm.S;
        const int f_hi = min(grp.u_hi * qm.S, qm.F);
        int *sg0 = smem, *sh0 = smem + nb;               // narrow: g, h  | wide: g_lo, h_lo
        int *sg1 = smem + 2 * nb, *sh1 = smem + 3 * nb;  // wide: g_hi, h_hi
        for (int i = threadIdx.x; i < (WIDE ? 4 : 2) * nb; i += H_THREADS) smem[i] = 0;
        for (int f = f_lo + threadIdx.x; f <= f_hi; f += H_THREADS)
            s_off[f - f_lo] = __ldg(a.cut_ptr + f) - grp.bin_lo;
        __syncthreads();
        const int Ug = grp.u_hi - grp.u_lo;
        const uint32_t magic = 0xffffffffu / (uint32_t)Ug + 1u;
        const uint32_t total = (uint32_t)len * (uint32_t)Ug;
        long long tg = 0, th = 0;
        for (uint32_t j = threadIdx.x; j < total; j += H_THREADS) {
            const uint32_t r = Ug == 1 ? j : fast_div(j, magic);
            const int u = grp.u_lo + (int)(j - r * (uint32_t)Ug);
            const long long pos = start + r;
            const uint32_t row = a.ridx ? __ldg(a.ridx + pos) : (uint32_t)pos;
            const int2 q = __ldg(a.qpair + row);
            if (a.totals && u == grp.u_lo) {
                tg += q.x;
                th += q.y;
            }
            const int f0 = u * qm.S;
            const int ns = min(qm.S, qm.F - f0);
            const uint32_t win = get_bits(qm.P, (long long)row * qm.stride + (long long)f0 * qm.bits,
                                          ns * qm.bits);
#pragma unroll 4
            for (int jj = 0; jj < ns; ++jj) {
                const int s = (int)((win >> (jj * qm.bits)) & mask);
                if (s == qm.B) continue;  // missing: mass recovered as total - sum (R7)
                const int bin = s_off[f0 + jj - f_lo] + s;
                if (WIDE) {
                    atomicAdd(sg0 + bin, q.x & 0x7fff);
                    atomicAdd(sg1 + bin, q.x >> 15);
                    atomicAdd(sh0 + bin, q.y & 0x7fff);
                    atomicAdd(sh1 + bin, q.y >> 15);
                } else {
                    atomicAdd(sg0 + bin, q.x);
                    atomicAdd(sh0 + bin, q.y);
                }
            }
        }
        if (a.totals && g == 0) {
            for (int o = 16; o > 0; o >>= 1) {
                tg += __shfl_xor_sync(0xffffffffu, tg, o);
                th += __shfl_xor_sync(0xffffffffu, th, o);
            }
            if ((threadIdx.x & 31) == 0) {
                s_red[0][threadIdx.x >> 5] = tg;
                s_red[1][threadIdx.x >> 5] = th;
            }
        }
        __syncthreads();
        if (a.totals && g == 0 && threadIdx.x == 0) {
            long long sgt = 0, sht = 0;
            for (int w = 0; w < H_THREADS / 32; ++w) {
                sgt += s_red[0][w];
                sht += s_red[1][w];
            }
            atomicAdd((unsigned long long *)a.totals + 0, (unsigned long long)sgt);
            atomicAdd((unsigned long long *)a.totals + 1, (unsigned long long)sht);
        }
        // flush into the int64 global histogram of this slot
        unsigned long long *dst = (unsigned long long *)a.hist + ((long long)slot * a.TB + grp.bin_lo) * 2;
        for (int b = threadIdx.x; b < nb; b += H_THREADS) {
            long long G, H;
            if (WIDE) {
                G = (long long)sg1[b] * 32768 + (long long)(unsigned)sg0[b];
                H = (long long)sh1[b] * 32768 + (long long)(unsigned)sh0[b];
            } else {
                G = sg0[b];
                H = sh0[b];
            }
            if (G) atomicAdd(dst + 2 * b, (unsigned long long)G);
            if (H) atomicAdd(dst + 2 * b + 1, (unsigned long long)H);
        }
        __syncthreads();
    }
}

// ============================================================== split evaluation
struct Best {
    double gain;
    long long idx;  // canonical candidate order: (global bin)*2 + (dl ? 0 : 1); LLONG_MAX = none
    long long Lg, Lh;
};

__device__ __forceinline__ bool better(const Best &a, const Best &b) {
    if (a.idx == LLONG_MAX) return false;
    if (b.idx == LLONG_MAX) return true;
    return a.gain > b.gain || (a.gain == b.gain && a.idx < b.idx);
}

__device__ __forceinline__ Best shfl_best(const Best &b, int o) {
    Best r;
    r.gain = __shfl_xor_sync(0xffffffffu, b.gain, o);
    r.idx = __shfl_xor_sync(0xffffffffu, b.idx, o);
    r.Lg = __shfl_xor_sync(0xffffffffu, b.Lg, o);
    r.Lh = __shfl_xor_sync(0xffffffffu, b.Lh, o);
    return r;
}

// Histogram source of one node: direct (hist), or sibling = parent - build.  Optionally stores
// the node's histogram (for the next level's subtraction).
struct NodeHist {
    const long long *direct;  // [TB][2] or null
    const long long *parent;  // [TB][2]
    const long long *build;   // [TB][2]
    long long *store;         // [TB][2] or null
    __device__ __forceinline__ void get(int bin, long long &g, long long &h) const {
        if (direct) {
            g = __ldg(direct + 2 * bin);
            h = __ldg(direct + 2 * bin + 1);
        } else {
            g = __ldg(parent + 2 * bin) - __ldg(build + 2 * bin);
            h = __ldg(parent + 2 * bin + 1) - __ldg(build + 2 * bin + 1);
        }
    }
};

// Evaluate one node with the whole block (E_THREADS).  Returns (in *out, valid on thread 0) the
// best candidate.  Op order of every fp64 step = R8 (oracle_evaluate_split).
__device__ void evaluate_node(const NodeHist &src, int F, const int32_t *__restrict__ cut_ptr,
                              long long Tg, long long Th, int sg, int sh, const EvalParams &p,
                              Best *out) {
    __shared__ Best s_best[E_THREADS / 32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const double G = fixed_to_double(Tg, sg), H = fixed_to_double(Th, sh);
    const double e = ddiv(dmul(G, G), dadd(H, p.lambda));
    Best best;
    best.gain = 0.0;
    best.idx = LLONG_MAX;
    best.Lg = best.Lh = 0;
    for (int f = wid; f < F; f += E_THREADS / 32) {
        const int b0 = __ldg(cut_ptr + f), nbf = __ldg(cut_ptr + f + 1) - b0;
        // pass 1: feature sums (missing mass) and the optional store of the node histogram
        long long sgs = 0, shs = 0;
        for (int b = lane; b < nbf; b += 32) {
            long long g, h;
            src.get(b0 + b, g, h);
            if (src.store) {
                src.store[2 * (b0 + b)] = g;
                src.store[2 * (b0 + b) + 1] = h;
            }
            sgs += g;
            shs += h;
        }
        for (int o = 16; o > 0; o >>= 1) {
            sgs += __shfl_xor_sync(0xffffffffu, sgs, o);
            shs += __shfl_xor_sync(0xffffffffu, shs, o);
        }
        const long long Mg = Tg - sgs, Mh = Th - shs;
        // pass 2: prefix scan in chunks of 32 bins, both default directions
        long long cg = 0, ch = 0;  // carry: prefix of earlier chunks
        for (int c = 0; c < nbf; c += 32) {
            const int b = c + lane;
            long long g = 0, h = 0;
            if (b < nbf) src.get(b0 + b, g, h);
            long long pg = g, ph = h;
            for (int o = 1; o < 32; o <<= 1) {
                long long yg = __shfl_up_sync(0xffffffffu, pg, o);
                long long yh = __shfl_up_sync(0xffffffffu, ph, o);
                if (lane >= o) {
                    pg += yg;
                    ph += yh;
                }
            }
            const long long Pg = cg + pg, Ph = ch + ph;
            cg += __shfl_sync(0xffffffffu, pg, 31);
            ch += __shfl_sync(0xffffffffu, ph, 31);
            if (b < nbf) {
#pragma unroll
                for (int dli = 0; dli < 2; ++dli) {
                    const bool dl = dli == 0;  // true first (R9)
                    const long long Lg = Pg + (dl ? Mg : 0), Lh = Ph + (dl ? Mh : 0);
                    const double GL = fixed_to_double(Lg, sg), HL = fixed_to_double(Lh, sh);
                    const double GR = fixed_to_double(Tg - Lg, sg), HR = fixed_to_double(Th - Lh, sh);
                    if (!(HL >= p.mcw && HR >= p.mcw && dadd(HL, p.lambda) > 0.0 &&
                          dadd(HR, p.lambda) > 0.0))
                        continue;
                    double a = dmul(GL, GL);
                    a = ddiv(a, dadd(HL, p.lambda));
                    double cc = dmul(GR, GR);
                    cc = ddiv(cc, dadd(HR, p.lambda));
                    double d = dadd(a, cc);
                    d = dsub(d, e);
                    d = dmul(0.5, d);
                    Best cand;
                    cand.gain = dsub(d, p.gamma);
                    cand.idx = (long long)(b0 + b) * 2 + dli;
                    cand.Lg = Lg;
                    cand.Lh = Lh;
                    if (better(cand, best)) best = cand;
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        Best other = shfl_best(best, o);
        if (better(other, best)) best = other;
    }
    if (lane == 0) s_best[wid] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        Best b = s_best[0];
        for (int w = 1; w < E_THREADS / 32; ++w)
            if (better(s_best[w], b)) b = s_best[w];
        *out = b;
    }
    __syncthreads();
}

__device__ __forceinline__ double leaf_weight(long long Tg, long long Th, int sg, int sh, double lambda, double eta) {
    const double G = fixed_to_double(Tg, sg), H = fixed_to_double(Th, sh);
    const double t = dadd(H, lambda);
    if (t == 0.0) return 0.0;
    double w = ddiv(G, t);
    w = -w;
    return dmul(w, eta);
}

struct TreeDev {
    int8_t *kind;
    int32_t *feature, *bin;
    float *threshold;
    int8_t *default_left;
    double *gain, *weight;
    long long *sum_qg, *sum_qh;
};

__device__ __forceinline__ void write_leaf(const TreeDev &t, int k, long long Tg, long long Th, int sg, int sh,
                                           const EvalParams &p) {
    t.kind[k] = GBM_NODE_LEAF;
    t.sum_qg[k] = Tg;
    t.sum_qh[k] = Th;
    t.weight[k] = leaf_weight(Tg, Th, sg, sh, p.lambda, p.eta);
}

// Evaluate every node of level l (heap ids first .. first + 2^l - 1).  One block per node.
//   level 0: hist = root buffer (totals at hist_root[2*TB]).
//   level l > 0: node k, parent pk; absent if the parent did not split; otherwise the built
//   child's histogram is hist_build[parent slot], the sibling's = hist_prev[slot] - build.
__global__ void __launch_bounds__(E_THREADS) eval_level_kernel(
    int level, int first, int F, int TB, const int32_t *__restrict__ cut_ptr,
    const float *__restrict__ cut_values, const int32_t *__restrict__ scale, EvalParams p,
    NodeDev *__restrict__ nodes, const long long *__restrict__ hist_root,
    const long long *__restrict__ hist_build, const long long *__restrict__ hist_prev,
    long long *__restrict__ hist_store, TreeDev t) {
    __shared__ Best s_out;
    const int j = blockIdx.x;
    const int k = first + j;
    const int sg = scale[0], sh = scale[1];
    NodeHist src;
    src.direct = nullptr;
    src.parent = src.build = nullptr;
    src.store = nullptr;
    long long Tg, Th;
    if (level == 0) {
        Tg = hist_root[2 * (long long)TB];
        Th = hist_root[2 * (long long)TB + 1];
        src.direct = hist_root;
        if (threadIdx.x == 0) {
            nodes[0].Tg = Tg;
            nodes[0].Th = Th;
        }
    } else {
        const int pk = (k - 1) / 2;
        const int pslot = pk - ((1 << (level - 1)) - 1);
        if (nodes[pk].state != GBM_NODE_SPLIT) {
            if (threadIdx.x == 0) nodes[k].state = GBM_NODE_ABSENT;
            return;
        }
        Tg = nodes[k].Tg;
        Th = nodes[k].Th;
        const bool is_left = (k & 1) == 1;
        const bool built = nodes[pk].build_left ? is_left : !is_left;
        const long long *bh = hist_build + (long long)pslot * TB * 2;
        if (built) {
            src.direct = bh;
        } else {
            src.parent = (level == 1 ? hist_root : hist_prev + (long long)pslot * TB * 2);
            src.build = bh;
        }
    }
    if (hist_store && level < p.max_depth - 1) src.store = hist_store + (long long)j * TB * 2;
    if (level >= p.max_depth) {  // (max_depth == 0) the root is a leaf
        if (threadIdx.x == 0) {
            write_leaf(t, k, Tg, Th, sg, sh, p);
            nodes[k].state = GBM_NODE_LEAF;
        }
        return;
    }
    evaluate_node(src, F, cut_ptr, Tg, Th, sg, sh, p, &s_out);
    if (threadIdx.x == 0) {
        Best b = s_out;
        const bool split = b.idx != LLONG_MAX && b.gain > 0.0;
        t.sum_qg[k] = Tg;
        t.sum_qh[k] = Th;
        t.weight[k] = leaf_weight(Tg, Th, sg, sh, p.lambda, p.eta);
        if (!split) {
            t.kind[k] = GBM_NODE_LEAF;
            nodes[k].state = GBM_NODE_LEAF;
        } else {
            const int gbin = (int)(b.idx >> 1), dl = (b.idx & 1) == 0;
            int f = 0;  // feature owning global bin gbin
            {
                int lo = 0, hi = F - 1;
                while (lo < hi) {
                    int mid = (lo + hi + 1) >> 1;
                    if (__ldg(cut_ptr + mid) <= gbin) lo = mid;
                    else hi = mid - 1;
                }
                f = lo;
            }
            const int bb = gbin - __ldg(cut_ptr + f);
            t.kind[k] = GBM_NODE_SPLIT;
            t.feature[k] = f;
            t.bin[k] = bb;
            t.threshold[k] = __ldg(cut_values + gbin);
            t.default_left[k] = (int8_t)dl;
            t.gain[k] = b.gain;
            NodeDev &nd = nodes[k];
            nd.state = GBM_NODE_SPLIT;
            nd.f = f;
            nd.b = bb;
            nd.dl = dl;
            const long long Lg = b.Lg, Lh = b.Lh, Rg = Tg - b.Lg, Rh = Th - b.Lh;
            nd.build_left = Lh <= Rh;  // smaller hessian sum; ties -> left (R17)
            nodes[2 * k + 1].Tg = Lg;
            nodes[2 * k + 1].Th = Lh;
            nodes[2 * k + 2].Tg = Rg;
            nodes[2 * k + 2].Th = Rh;
            if (level + 1 == p.max_depth) {  // children at depth D are leaves
                write_leaf(t, 2 * k + 1, Lg, Lh, sg, sh, p);
                write_leaf(t, 2 * k + 2, Rg, Rh, sg, sh, p);
            }
        }
    }
}

// standalone EvaluateSplit over n_nodes given histograms (gbm_evaluate_splits)
__global__ void __launch_bounds__(E_THREADS) eval_many_kernel(
    int F, int TB, const int32_t *__restrict__ cut_ptr, const int32_t *__restrict__ scale, EvalParams p,
    const long long *__restrict__ hist, const long long *__restrict__ totals, int8_t *split_d,
    int32_t *feature_d, int32_t *bin_d, int8_t *dl_d, double *gain_d, long long *child_d) {
    __shared__ Best s_out;
    const int j = blockIdx.x;
    NodeHist src;
    src.direct = hist + (long long)j * TB * 2;
    src.parent = src.build = nullptr;
    src.store = nullptr;
    const long long Tg = totals[2 * j], Th = totals[2 * j + 1];
    evaluate_node(src, F, cut_ptr, Tg, Th, scale[0], scale[1], p, &s_out);
    if (threadIdx.x == 0) {
        Best b = s_out;
        const bool found = b.idx != LLONG_MAX;
        split_d[j] = found && b.gain > 0.0;
        gain_d[j] = found ? b.gain : 0.0;
        int f = -1, bb = -1, dl = 0;
        if (found) {
            const int gbin = (int)(b.idx >> 1);
            dl = (b.idx & 1) == 0;
            int lo = 0, hi = F - 1;
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (__ldg(cut_ptr + mid) <= gbin) lo = mid;
                else hi = mid - 1;
            }
            f = lo;
            bb = gbin - __ldg(cut_ptr + f);
        }
        feature_d[j] = f;
        bin_d[j] = bb;
        dl_d[j] = (int8_t)dl;
        child_d[4 * j + 0] = found ? b.Lg : 0;
        child_d[4 * j + 1] = found ? b.Lh : 0;
        child_d[4 * j + 2] = found ? Tg - b.Lg : 0;
        child_d[4 * j + 3] = found ? Th - b.Lh : 0;
    }
}

__global__ void init_tree_kernel(TreeDev t, long long cap, NodeDev *nodes, long long n_rows,
                                 int *tile_base0) {
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
        NodeDev nd = {};
        nodes[k] = nd;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        nodes[0].start = 0;
        nodes[0].count = n_rows;
        tile_base0[0] = 0;
        tile_base0[1] = (int)((n_rows + PT - 1) / PT);
    }
}

// ============================================================== host planning
struct HistPlan {
    std::vector<Group> groups;
    int smem_bytes = 0;   // dynamic smem per block
    int blocks = 0;       // resident grid
    int chunk = 0;        // rows per item
};

static int plan_hist(gbm_ctx *ctx, const QM &qm, const int32_t *cut_ptr_h, bool wide, long long rows_hint,
                     HistPlan &hp) {
    const int bytes_per_bin = wide ? 16 : 8;
    const int budget = (int)std::min<size_t>(ctx->smem_optin - 24 * 1024, 200 * 1024);
    const int max_bins_group = budget / bytes_per_bin;
    hp.groups.clear();
    int u = 0;
    while (u < qm.U) {
        Group g;
        g.u_lo = u;
        g.bin_lo = cut_ptr_h[std::min(u * qm.S, qm.F)];
        int u_end = u;
        while (u_end < qm.U) {
            int f_hi = std::min((u_end + 1) * qm.S, qm.F);
            int nb = cut_ptr_h[f_hi] - g.bin_lo;
            int nf = f_hi - u * qm.S;
            if ((nb > max_bins_group || nf > 2048) && u_end > u) break;
            if (nb > max_bins_group) return fail(GBM_E_ARG, "a single feature unit has more bins than fit in shared memory");
            u_end++;
        }
        g.u_hi = u_end;
        g.bin_hi = cut_ptr_h[std::min(u_end * qm.S, qm.F)];
        hp.groups.push_back(g);
        u = u_end;
    }
    int max_nb = 1;
    for (auto &g : hp.groups) max_nb = std::max(max_nb, g.bin_hi - g.bin_lo);
    hp.smem_bytes = max_nb * bytes_per_bin;
    auto kern = wide ? hist_kernel<true> : hist_kernel<false>;
    GBM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, hp.smem_bytes));
    int occ = 0;
    GBM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, H_THREADS, hp.smem_bytes));
    if (occ < 1) return fail(GBM_E_ARG, "histogram kernel cannot be resident");
    hp.blocks = occ * ctx->sm_count;
    // about two items per resident block per pass over the rows, capped by the exactness bound
    long long per = (rows_hint + 2ll * hp.blocks - 1) / (2ll * hp.blocks) * (long long)hp.groups.size();
    hp.chunk = (int)std::max<long long>(256, std::min<long long>(MAX_CHUNK, per));
    return GBM_OK;
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
    GBM_REQUIRE(qm->row_align_bits == 0 || qm->row_align_bits == 32 || qm->row_align_bits == 128, GBM_E_ARG,
                "qmatrix: row_align_bits must be 0, 32 or 128");
    return GBM_OK;
}

static int launch_hist(gbm_ctx *ctx, bool wide, const HistPlan &hp, const HistArgs &a, int grid, cudaStream_t s) {
    if (wide) hist_kernel<true><<<grid, H_THREADS, hp.smem_bytes, s>>>(a);
    else hist_kernel<false><<<grid, H_THREADS, hp.smem_bytes, s>>>(a);
    GBM_CUDA(cudaGetLastError());
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
    const bool wide = grad_bits > 15;
    HistPlan hp;
    GBM_TRY(plan_hist(ctx, qm, q->cut_ptr_h, wide, n_sel, hp));
    GBM_TRY(ctx->arena.reserve(hp.groups.size() * sizeof(Group) + 256));
    Group *groups = ctx->arena.take<Group>(hp.groups.size());
    GBM_CUDA(cudaMemcpyAsync(groups, hp.groups.data(), hp.groups.size() * sizeof(Group), cudaMemcpyHostToDevice, s));
    GBM_CUDA(cudaMemsetAsync(hist_d, 0, (size_t)TB * 2 * 8, s));
    if (n_sel == 0 || TB == 0) return GBM_OK;
    HistArgs a = {};
    a.qm = qm;
    a.qpair = reinterpret_cast<const int2 *>(qpair_d);
    a.ridx = rows_d;
    a.items = nullptr;
    a.n_sel = n_sel;
    a.chunk = hp.chunk;
    a.n_groups = (int)hp.groups.size();
    a.groups = groups;
    a.cut_ptr = q->cut_ptr_d;
    a.hist = reinterpret_cast<long long *>(hist_d);
    a.totals = nullptr;
    a.TB = TB;
    long long n_items = (n_sel + hp.chunk - 1) / hp.chunk * (long long)hp.groups.size();
    int grid = (int)std::min<long long>(n_items, hp.blocks);
    GBM_TRY(launch_hist(ctx, wide, hp, a, grid, s));
    // the pageable H2D copy of `groups` above completes before this call returns
    return GBM_OK;
}

int gbm_allreduce_histograms(gbm_ctx *ctx, int64_t *hist_d, int64_t count, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_REQUIRE(hist_d && count >= 0, GBM_E_ARG, "gbm_allreduce_histograms: bad arguments");
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
    EvalParams p = {prm->eta, prm->lambda, prm->gamma, prm->min_child_weight, prm->max_depth};
    const int TB = q->cut_ptr_h[q->n_features];
    eval_many_kernel<<<n_nodes, E_THREADS, 0, (cudaStream_t)stream>>>(
        q->n_features, TB, q->cut_ptr_d, scale_d, p, reinterpret_cast<const long long *>(hist_d),
        reinterpret_cast<const long long *>(totals_d), split_d, feature_d, bin_d, default_left_d, gain_d,
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
    const int tiles = (int)((n_sel + PT - 1) / PT);
    Arena &A = ctx->arena;
    GBM_TRY(A.reserve(3 * sizeof(NodeDev) + 64 + (size_t)tiles * (PT / 32) * 4 + 2 * (size_t)tiles * 4 + 16 * 256 +
                      sizeof(HistItem)));
    NodeDev *nodes = A.take<NodeDev>(3);
    int *tile_base = A.take<int>(2);
    int *next_tb = A.take<int>(3);
    uint32_t *flags = A.take<uint32_t>((size_t)std::max(tiles, 1) * (PT / 32));
    int *tile_left = A.take<int>(std::max(tiles, 1));
    int *tile_off = A.take<int>(std::max(tiles, 1));
    int *n_items = A.take<int>(1);
    NodeDev h[3] = {};
    h[0].start = 0;
    h[0].count = n_sel;
    h[0].state = GBM_NODE_SPLIT;
    h[0].f = feature;
    h[0].b = bin;
    h[0].dl = default_left ? 1 : 0;
    h[0].build_left = 1;
    int tb[2] = {0, tiles};
    GBM_CUDA(cudaMemcpyAsync(nodes, h, sizeof(h), cudaMemcpyHostToDevice, s));
    GBM_CUDA(cudaMemcpyAsync(tile_base, tb, sizeof(tb), cudaMemcpyHostToDevice, s));
    const int grid = std::max(1, std::min(tiles, ctx->sm_count * 8));
    part_count_kernel<false><<<grid, P_THREADS, 0, s>>>(qm, nodes, 0, 1, tile_base, rows_d, flags, tile_left, nullptr);
    part_scan_kernel<<<1, 1024, 0, s>>>(nodes, 0, 1, tile_base, tile_left, tile_off, nullptr, n_items, 1, 1, next_tb, 0);
    part_scatter_kernel<<<grid, P_THREADS, 0, s>>>(nodes, 0, 1, tile_base, flags, tile_off, rows_d, out_d);
    GBM_CUDA(cudaGetLastError());
    GBM_CUDA(cudaMemcpyAsync(n_left_d, &nodes[1].count, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    GBM_CUDA(cudaStreamSynchronize(s));  // host staging above must outlive the copies
    return GBM_OK;
}

int gbm_build_tree(gbm_ctx *ctx, const gbm_qmatrix *q, const int32_t *qpair_d, const int32_t *scale_d,
                   const gbm_params *prm, const gbm_tree *tree, int32_t *row_leaf_d, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_TRY(check_qm(q));
    GBM_REQUIRE(prm && tree && scale_d && row_leaf_d && qpair_d, GBM_E_ARG, "gbm_build_tree: null argument");
    GBM_REQUIRE(tree->kind && tree->feature && tree->bin && tree->threshold && tree->default_left && tree->gain &&
                    tree->weight && tree->sum_qg && tree->sum_qh,
                GBM_E_ARG, "gbm_build_tree: null tree array");
    GBM_REQUIRE(prm->max_depth >= 0 && prm->max_depth <= 16, GBM_E_ARG, "gbm_build_tree: max_depth in 0..16");
    GBM_REQUIRE(prm->grad_bits >= 1 && prm->grad_bits <= 30, GBM_E_ARG, "gbm_build_tree: grad_bits in 1..30");
    GBM_REQUIRE(prm->lambda >= 0 && prm->gamma >= 0 && prm->min_child_weight >= 0, GBM_E_ARG,
                "gbm_build_tree: lambda, gamma, min_child_weight must be >= 0");
    const long long n = q->n_rows;
    GBM_REQUIRE(n > 0 || (ctx->comm && ctx->nranks > 1), GBM_E_EMPTY, "gbm_build_tree: zero rows (S:321)");
    cudaStream_t s = (cudaStream_t)stream;
    const QM qm = make_qm(q);
    const int F = q->n_features, D = prm->max_depth;
    const int TB = q->cut_ptr_h[F];
    const bool wide = prm->grad_bits > 15;
    const long long cap = (1ll << (D + 1)) - 1;
    HistPlan hp;
    GBM_TRY(plan_hist(ctx, qm, q->cut_ptr_h, wide, std::max<long long>(n, 1), hp));
    const int G = (int)hp.groups.size();

    // ---- scratch (tree arena)
    const int max_par = D >= 1 ? (1 << (D - 1)) : 1;            // parents partitioned at one level
    const long long max_tiles = (n + PT - 1) / PT + 2ll * max_par + 2;
    const long long max_items = ((n + hp.chunk - 1) / hp.chunk + max_par + 1) * G;
    const long long slots_build = std::max(1, D >= 2 ? (1 << (D - 2)) : 1);
    const long long slots_lvl = std::max(1, D >= 2 ? (1 << (D - 2)) : 1);
    const size_t hist_unit = (size_t)TB * 2;
    size_t need = 0;
    need += 2 * (size_t)std::max<long long>(n, 1) * 4 + 512;                  // ridx x2
    need += (size_t)max_tiles * (PT / 32) * 4 + 256;                          // flags
    need += 2 * (size_t)max_tiles * 4 + 512;                                  // tile_left/off
    need += (size_t)(D + 2) * (2 * max_par + 2) * 4 + 256 * (D + 2);           // tile bases
    need += (size_t)(2 * cap + 2) * sizeof(NodeDev) + 256;                    // nodes
    need += (size_t)max_items * sizeof(HistItem) + 256 + 256;                 // items + count
    need += G * sizeof(Group) + 256;
    need += (slots_build * hist_unit + hist_unit + 2) * 8 + 512;                // build + root
    need += 2 * slots_lvl * hist_unit * 8 + 512;                              // level hists
    Arena &A = ctx->tree_arena;
    GBM_TRY(A.reserve(need));
    uint32_t *ridx[2] = {A.take<uint32_t>(std::max<long long>(n, 1)), A.take<uint32_t>(std::max<long long>(n, 1))};
    uint32_t *flags = A.take<uint32_t>((size_t)max_tiles * (PT / 32));
    int *tile_left = A.take<int>(max_tiles);
    int *tile_off = A.take<int>(max_tiles);
    std::vector<int *> tile_base(D + 2);
    for (int l = 0; l <= D + 1; ++l) tile_base[l] = A.take<int>(2 * max_par + 2);
    NodeDev *nodes = A.take<NodeDev>(2 * cap + 2);
    HistItem *items = A.take<HistItem>(max_items);
    int *n_items = A.take<int>(1);
    Group *groups = A.take<Group>(G);
    long long *hist_root = A.take<long long>(hist_unit + 2);   // root histogram + totals
    long long *hist_build = A.take<long long>(slots_build * hist_unit);
    long long *hist_lvl[2] = {A.take<long long>(slots_lvl * hist_unit), A.take<long long>(slots_lvl * hist_unit)};

    GBM_CUDA(cudaMemcpyAsync(groups, hp.groups.data(), G * sizeof(Group), cudaMemcpyHostToDevice, s));
    const TreeDev t = tree_dev(tree);
    const EvalParams ep = {prm->eta, prm->lambda, prm->gamma, prm->min_child_weight, D};
    init_tree_kernel<<<(int)std::min<long long>((cap + 255) / 256, 1024), 256, 0, s>>>(t, cap, nodes, n, tile_base[0]);
    GBM_CUDA(cudaGetLastError());

    // ---- InitRoot: root histogram + totals, allreduce, evaluate
    GBM_CUDA(cudaMemsetAsync(hist_root, 0, (hist_unit + 2) * 8, s));
    HistArgs a = {};
    a.qm = qm;
    a.qpair = reinterpret_cast<const int2 *>(qpair_d);
    a.n_groups = G;
    a.groups = groups;
    a.cut_ptr = q->cut_ptr_d;
    a.TB = TB;
    if (n > 0) {
        a.ridx = nullptr;
        a.items = nullptr;
        a.n_sel = n;
        a.chunk = hp.chunk;
        a.hist = hist_root;
        a.totals = hist_root + hist_unit;
        long long n_it = (n + hp.chunk - 1) / hp.chunk * (long long)G;
        GBM_TRY(launch_hist(ctx, wide, hp, a, (int)std::min<long long>(n_it, hp.blocks), s));
    }
    GBM_TRY(allreduce_i64(ctx, hist_root, hist_unit + 2, s));
    eval_level_kernel<<<1, E_THREADS, 0, s>>>(0, 0, F, TB, q->cut_ptr_d, q->cut_values_d, scale_d, ep, nodes,
                                              hist_root, nullptr, nullptr, nullptr, t);
    GBM_CUDA(cudaGetLastError());

    const int pgrid = ctx->sm_count * 8;
    for (int l = 1; l <= D; ++l) {
        const int first = (1 << (l - 1)) - 1, n_par = 1 << (l - 1);
        const uint32_t *rin = l == 1 ? nullptr : ridx[(l - 1) & 1];
        uint32_t *rout = ridx[l & 1];
        if (l == D) {  // final partition: rows straight to their leaves
            part_count_kernel<true><<<pgrid, P_THREADS, 0, s>>>(qm, nodes, first, n_par, tile_base[l - 1], rin, flags,
                                                                tile_left, row_leaf_d);
            GBM_CUDA(cudaGetLastError());
            break;
        }
        part_count_kernel<false><<<pgrid, P_THREADS, 0, s>>>(qm, nodes, first, n_par, tile_base[l - 1], rin, flags,
                                                             tile_left, row_leaf_d);
        part_scan_kernel<<<1, 1024, 0, s>>>(nodes, first, n_par, tile_base[l - 1], tile_left, tile_off, items, n_items,
                                            G, hp.chunk, tile_base[l], 1);
        part_scatter_kernel<<<pgrid, P_THREADS, 0, s>>>(nodes, first, n_par, tile_base[l - 1], flags, tile_off, rin,
                                                        rout);
        GBM_CUDA(cudaGetLastError());
        // BuildPartialHistograms of the built children
        GBM_CUDA(cudaMemsetAsync(hist_build, 0, (size_t)n_par * hist_unit * 8, s));
        a.ridx = rout;
        a.items = items;
        a.n_items_dev = n_items;
        a.hist = hist_build;
        a.totals = nullptr;
        GBM_TRY(launch_hist(ctx, wide, hp, a, hp.blocks, s));
        // AllReduceHistograms
        GBM_TRY(allreduce_i64(ctx, hist_build, (size_t)n_par * hist_unit, s));
        // subtraction + EvaluateSplit for every node of level l
        const long long *prev = l == 1 ? nullptr : hist_lvl[(l - 1) & 1];
        long long *store = (l < D - 1) ? hist_lvl[l & 1] : nullptr;
        eval_level_kernel<<<1 << l, E_THREADS, 0, s>>>(l, (1 << l) - 1, F, TB, q->cut_ptr_d, q->cut_values_d, scale_d,
                                                       ep, nodes, hist_root, hist_build, prev, store, t);
        GBM_CUDA(cudaGetLastError());
    }
    if (D == 0) {  // every row sits in the root leaf
        part_count_kernel<false><<<pgrid, P_THREADS, 0, s>>>(qm, nodes, 0, 1, tile_base[0], nullptr, flags, tile_left,
                                                             row_leaf_d);
        GBM_CUDA(cudaGetLastError());
    }
    return GBM_OK;
}

}  // extern "C"
