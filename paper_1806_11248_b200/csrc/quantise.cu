// quantise.cu -- §2.1 feature quantiles and §2.2 compression on sm_100a.
//
//  gbm_cuts           exact global cuts: column transpose to monotone uint32 keys, a per-feature
//                     stable LSD radix sort (4 x 8-bit passes, warp match_any ranking), then the
//                     rank rule / lossless distinct values of R5 selected on the device.
//  gbm_quantise       bin map (lower-bound binary search per element, R6/R7).
//  gbm_compress       bit-pack, one thread per output word (no atomics, each word written once).
//  gbm_quantise_compress  both fused: one thread per output word bins its own elements.
#include <algorithm>
#include <string>
#include <vector>

#include "gbm_internal.cuh"

namespace gbm {

// ------------------------------------------------------------------ shared device helpers
__device__ __forceinline__ uint32_t float_key(float v) {
    // monotone map fp32 -> uint32 (present values); -0.0 canonicalised to +0.0 (R22)
    if (v == 0.0f) v = 0.0f;
    uint32_t b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_float(uint32_t k) {
    uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(b);
}
constexpr uint32_t KEY_MISSING = 0xffffffffu;  // NaN and padding; no finite float maps here

// lower bound: smallest k in [0, nb) with v <= cuts[k], clamped to nb-1
__device__ __forceinline__ int bin_search(const float *__restrict__ cuts, int nb, float v) {
    int lo = 0, hi = nb;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (v <= __ldg(cuts + mid)) hi = mid;
        else lo = mid + 1;
    }
    return lo < nb ? lo : nb - 1;
}

__device__ __forceinline__ int quantise_one(float v, int f, const float *__restrict__ cv,
                                            const int32_t *__restrict__ cp, int B,
                                            uint32_t *dev_err) {
    if (isinf(v)) atomicOr(dev_err, DERR_NONFINITE);
    int lo = __ldg(cp + f), nb = __ldg(cp + f + 1) - lo;
    if (isnan(v) || nb == 0) return B;
    return bin_search(cv + lo, nb, v);
}

// ------------------------------------------------------------------ bin map
__global__ void quantise_kernel(const float *__restrict__ X, long long total, int F,
                                const float *__restrict__ cv, const int32_t *__restrict__ cp,
                                int B, uint16_t *__restrict__ bins, uint32_t *dev_err) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        int f = (int)(e % F);
        bins[e] = (uint16_t)quantise_one(__ldg(X + e), f, cv, cp, B, dev_err);
    }
}

// ------------------------------------------------------------------ bit-pack, one word / thread
// Word w holds stream bits [32w, 32w+32).  The thread walks the elements overlapping them
// (R3 layout; padding between rows and after the last row stays zero).
template <bool FROM_X>
__global__ void pack_kernel(const uint16_t *__restrict__ bins, const float *__restrict__ X,
                            long long n, int F, int bits, long long stride,
                            const float *__restrict__ cv, const int32_t *__restrict__ cp, int B,
                            uint32_t *__restrict__ out, long long n_words, uint32_t *dev_err) {
    const long long row_bits = (long long)F * bits;
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < n_words;
         w += (long long)gridDim.x * blockDim.x) {
        long long p = w * 32, end = p + 32;
        uint32_t word = 0;
        while (p < end) {
            long long row = p / stride;
            if (row >= n) break;
            long long off = p - row * stride;
            if (off >= row_bits) {  // row padding
                p = (row + 1) * stride;
                continue;
            }
            int f = (int)(off / bits);
            long long es = row * stride + (long long)f * bits;
            uint32_t s;
            if (FROM_X) s = (uint32_t)quantise_one(__ldg(X + row * F + f), f, cv, cp, B, dev_err);
            else s = __ldg(bins + row * F + f);
            if (s >> bits) atomicOr(dev_err, DERR_OVERFLOW);
            long long sh = es - w * 32;
            word |= sh >= 0 ? (uint32_t)((uint64_t)s << sh) : (uint32_t)(s >> (-sh));
            p = es + bits;
        }
        out[w] = word;
    }
}

// Byte symbols with rows of whole words (the common layout): word w = (row, unit u) by one 32-bit
// division, its 4 symbols from X[row][4u .. 4u+3] -- the generic walk above spends two 64-bit
// divisions per element (Higgs 11M x 28: 1.35 ms).
__global__ void pack_byte_kernel(const float *__restrict__ X, int F, uint32_t W, const float *__restrict__ cv,
                                 const int32_t *__restrict__ cp, int B, uint32_t *__restrict__ out,
                                 uint32_t n_words, uint32_t *dev_err) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < n_words; w += gridDim.x * blockDim.x) {
        const uint32_t row = w / W, u = w - row * W;
        const float *xr = X + (size_t)row * F;
        uint32_t word = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int f = (int)(4 * u) + j;
            if (f < F) {
                const uint32_t s = (uint32_t)quantise_one(__ldg(xr + f), f, cv, cp, B, dev_err);
                if (s >> 8) atomicOr(dev_err, DERR_OVERFLOW);
                word |= (s & 255u) << (8 * j);
            }
        }
        out[w] = word;
    }
}

// ------------------------------------------------------------------ cuts: radix sort machinery
constexpr int SORT_THREADS = 256;                 // 8 warps
constexpr int SORT_ITEMS = 16;                    // per thread
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;  // 4096 keys per tile

// X [n][F] (row-major, rows of all ranks) -> keys [F][n_pad] column-major
__global__ void keys_kernel(const float *__restrict__ X, long long n, int F, long long n_pad,
                            uint32_t *__restrict__ keys, unsigned long long *__restrict__ present,
                            uint32_t *dev_err) {
    // grid: x strides over row blocks of 32, y over feature blocks of 32; transpose through smem.
    // The present-value counts stay in registers (4 features per thread) and reach `present`
    // once per (block, feature): one atomic per 32-row block serialised on F addresses.
    __shared__ uint32_t t[32][33];
    const int f0 = blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    unsigned cnt[4] = {0u, 0u, 0u, 0u};
    unsigned err = 0;
    for (long long r0 = (long long)blockIdx.x * 32; r0 < n_pad; r0 += (long long)gridDim.x * 32) {
        for (int k = ty; k < 32; k += 8) {
            const long long r = r0 + k;
            const int f = f0 + tx;
            uint32_t key = KEY_MISSING;
            if (r < n && f < F) {
                const float v = __ldg(X + r * F + f);
                if (isinf(v)) err = 1;
                if (!isnan(v)) key = float_key(v);
            }
            t[k][tx] = key;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = ty + 8 * i;
            const int f = f0 + k;
            const long long r = r0 + tx;
            if (f < F && r < n_pad) {
                const uint32_t key = t[tx][k];
                keys[(long long)f * n_pad + r] = key;
                cnt[i] += key != KEY_MISSING;
            }
        }
        __syncthreads();
    }
    if (err) atomicOr(dev_err, DERR_NONFINITE);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        unsigned c = cnt[i];
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        const int f = f0 + ty + 8 * i;
        if (tx == 0 && f < F && c) atomicAdd(present + f, (unsigned long long)c);
    }
}

// digit histogram per (feature, tile): counts[f][digit][tile]
__global__ void __launch_bounds__(SORT_THREADS) sort_count_kernel(const uint32_t *__restrict__ keys,
                                                                  long long n_pad, int tiles,
                                                                  int shift,
                                                                  uint32_t *__restrict__ counts) {
    __shared__ uint32_t h[256];
    int f = blockIdx.y, tile = blockIdx.x;
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint32_t *k = keys + (long long)f * n_pad + (long long)tile * SORT_TILE;
    for (int i = threadIdx.x; i < SORT_TILE; i += SORT_THREADS)
        atomicAdd(&h[(__ldg(k + i) >> shift) & 255u], 1u);
    __syncthreads();
    counts[((long long)f * 256 + threadIdx.x) * tiles + tile] = h[threadIdx.x];
}

// exclusive scan per feature over [256 digits][tiles] (digit-major), in place
__global__ void __launch_bounds__(1024) scan_rows_kernel(uint32_t *__restrict__ data, long long len) {
    // one block per row of `len` entries
    uint32_t *d = data + (long long)blockIdx.x * len;
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (long long base = 0; base < len; base += 1024) {
        long long i = base + threadIdx.x;
        uint32_t v = i < len ? d[i] : 0;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t s = warp_sums[lane];
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        uint32_t excl = carry + (wid ? warp_sums[wid - 1] : 0) + x - v;
        if (i < len) d[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
}

// stable scatter: warp w owns tile keys [w*512, w*512+512) in 16 rounds of 32 consecutive keys
__global__ void __launch_bounds__(SORT_THREADS) sort_scatter_kernel(
    const uint32_t *__restrict__ in, uint32_t *__restrict__ out, long long n_pad, int tiles,
    int shift, const uint32_t *__restrict__ offsets) {
    __shared__ uint32_t wc[SORT_THREADS / 32][256];  // per-warp digit counters
    __shared__ uint32_t base[256];
    const int f = blockIdx.y, tile = blockIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (SORT_THREADS / 32) * 256; i += SORT_THREADS) (&wc[0][0])[i] = 0;
    base[threadIdx.x] = offsets[((long long)f * 256 + threadIdx.x) * tiles + tile];
    __syncthreads();
    const uint32_t *k = in + (long long)f * n_pad + (long long)tile * SORT_TILE + wid * 512;
    uint32_t key[SORT_ITEMS], rank[SORT_ITEMS];
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < SORT_ITEMS; ++j) {
        key[j] = __ldg(k + j * 32 + lane);
        uint32_t d = (key[j] >> shift) & 255u;
        uint32_t peers = __match_any_sync(0xffffffffu, d);
        uint32_t before = wc[wid][d];
        __syncwarp();
        rank[j] = before + __popc(peers & lt);
        if ((peers & lt) == 0) wc[wid][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // exclusive prefix over warps per digit (thread = digit)
    {
        uint32_t run = 0;
        for (int w = 0; w < SORT_THREADS / 32; ++w) {
            uint32_t c = wc[w][threadIdx.x];
            wc[w][threadIdx.x] = run;
            run += c;
        }
    }
    __syncthreads();
    uint32_t *o = out + (long long)f * n_pad;
#pragma unroll
    for (int j = 0; j < SORT_ITEMS; ++j) {
        uint32_t d = (key[j] >> shift) & 255u;
        o[base[d] + wc[wid][d] + rank[j]] = key[j];
    }
}

// run starts (first key of each run of equal present keys) per (feature, tile)
__global__ void __launch_bounds__(SORT_THREADS) runs_count_kernel(const uint32_t *__restrict__ keys,
                                                                  long long n_pad, int tiles,
                                                                  uint32_t *__restrict__ cnt) {
    const int f = blockIdx.y, tile = blockIdx.x;
    const uint32_t *k = keys + (long long)f * n_pad;
    long long i0 = (long long)tile * SORT_TILE;
    uint32_t c = 0;
    for (int i = threadIdx.x; i < SORT_TILE; i += SORT_THREADS) {
        long long i_ = i0 + i;
        uint32_t v = __ldg(k + i_);
        c += (v != KEY_MISSING && (i_ == 0 || __ldg(k + i_ - 1) != v));
    }
    __shared__ uint32_t s[SORT_THREADS];
    s[threadIdx.x] = c;
    __syncthreads();
    for (int o = SORT_THREADS / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] += s[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) cnt[(long long)f * tiles + tile] = s[0];
}

// per feature: distinct count d (from the scanned run counts) and n_bins; for d > B pick the
// rank-rule values and dedup them into tmp [F][B].  One block per feature.
__global__ void __launch_bounds__(1024) select_kernel(const uint32_t *__restrict__ keys, long long n_pad,
                                                      int tiles, const uint32_t *__restrict__ run_off,
                                                      const uint32_t *__restrict__ run_cnt,
                                                      const unsigned long long *__restrict__ present,
                                                      int B, float *__restrict__ tmp,
                                                      int32_t *__restrict__ nbins) {
    const int f = blockIdx.x;
    const long long m = (long long)present[f];
    const uint32_t d = run_off[(long long)f * tiles + tiles - 1] + run_cnt[(long long)f * tiles + tiles - 1];
    if ((long long)d <= B) {
        if (threadIdx.x == 0) nbins[f] = (int32_t)d;
        return;
    }
    const uint32_t *k = keys + (long long)f * n_pad;
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < B; base += 1024) {
        int j = base + threadIdx.x;
        uint32_t keep = 0, v = 0;
        if (j < B) {
            long long idx = ((long long)(j + 1) * m) / B - 1;
            v = __ldg(k + idx);
            keep = (j == 0) || (__ldg(k + ((long long)j * m) / B - 1) != v);
        }
        uint32_t x = keep;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[wid] = x;
        __syncthreads();
        if (wid == 0) {
            uint32_t s = warp_sums[lane];
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        uint32_t pos = carry + (wid ? warp_sums[wid - 1] : 0) + x - keep;
        if (keep) tmp[(long long)f * B + pos] = key_float(v);
        __syncthreads();
        if (threadIdx.x == 1023) carry = pos + keep;
        __syncthreads();
    }
    if (threadIdx.x == 0) nbins[f] = (int32_t)carry;
}

// cut_ptr = exclusive prefix of nbins (single block, F small)
__global__ void cutptr_kernel(const int32_t *__restrict__ nbins, int F, int32_t *__restrict__ cp) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int32_t run = 0;
        for (int f = 0; f < F; ++f) {
            cp[f] = run;
            run += nbins[f];
        }
        cp[F] = run;
    }
}

// write cut values: lossless features from run starts, rank-rule features from tmp
__global__ void __launch_bounds__(SORT_THREADS) write_cuts_kernel(
    const uint32_t *__restrict__ keys, long long n_pad, int tiles, const uint32_t *__restrict__ run_off,
    const int32_t *__restrict__ nbins, const float *__restrict__ tmp, int B,
    const int32_t *__restrict__ cp, float *__restrict__ cv) {
    const int f = blockIdx.y, tile = blockIdx.x;
    const int nb = nbins[f];  // < 0: rank-rule feature, values in tmp (tag_kernel)
    if (nb >= 0) {
        // lossless path: run starts are the cuts
        const uint32_t *k = keys + (long long)f * n_pad;
        long long i0 = (long long)tile * SORT_TILE;
        // block-local exclusive ranks of run starts in this tile, in key order
        __shared__ uint32_t s[SORT_THREADS];
        uint32_t c = 0;
        const int per = SORT_ITEMS;
        long long mine = i0 + (long long)threadIdx.x * per;
        for (int j = 0; j < per; ++j) {
            long long i_ = mine + j;
            uint32_t v = __ldg(k + i_);
            c += (v != KEY_MISSING && (i_ == 0 || __ldg(k + i_ - 1) != v));
        }
        s[threadIdx.x] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t run = 0;
            for (int t = 0; t < SORT_THREADS; ++t) {
                uint32_t x = s[t];
                s[t] = run;
                run += x;
            }
        }
        __syncthreads();
        uint32_t pos = run_off[(long long)f * tiles + tile] + s[threadIdx.x];
        for (int j = 0; j < per; ++j) {
            long long i_ = mine + j;
            uint32_t v = __ldg(k + i_);
            if (v != KEY_MISSING && (i_ == 0 || __ldg(k + i_ - 1) != v)) cv[cp[f] + pos++] = key_float(v);
        }
    } else if (tile == 0) {
        int cnt = -nb - 1;
        for (int j = threadIdx.x; j < cnt; j += SORT_THREADS) cv[cp[f] + j] = tmp[(long long)f * B + j];
    }
}

// n_bins sign-tagging: rank-rule features store -(count)-1 so write_cuts can tell them apart
__global__ void tag_kernel(const uint32_t *__restrict__ run_off, const uint32_t *__restrict__ run_cnt,
                           int tiles, int F, int B, int32_t *__restrict__ nbins,
                           int32_t *__restrict__ nbins_plain) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= F) return;
    uint32_t d = run_off[(long long)f * tiles + tiles - 1] + run_cnt[(long long)f * tiles + tiles - 1];
    int nb = nbins[f];
    nbins_plain[f] = nb;
    if ((long long)d > B) nbins[f] = -nb - 1;
}

// packed (row-major, bits <= 8) -> feature-major uint8 copy; 64 rows x all features per block
constexpr int TR_ROWS = 64;
__global__ void __launch_bounds__(256) transpose_kernel(QM qm, long long n, uint8_t *__restrict__ col) {
    extern __shared__ uint8_t tr[];  // [TR_ROWS][F]
    const long long r0 = (long long)blockIdx.x * TR_ROWS;
    const int rows = (int)min((long long)TR_ROWS, n - r0);
    for (int e = threadIdx.x; e < rows * qm.F; e += blockDim.x) {
        const int r = e / qm.F, f = e - r * qm.F;
        tr[r * qm.F + f] = (uint8_t)symbol_at(qm, r0 + r, f);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * qm.F; e += blockDim.x) {
        const int f = e / rows, r = e - f * rows;
        col[(long long)f * n + r0 + r] = tr[r * qm.F + f];
    }
}

static int grid_for(long long work, int threads, int sm) {
    long long g = (work + threads - 1) / threads;
    long long cap = (long long)sm * 32;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace gbm

using namespace gbm;

extern "C" {

int gbm_quantise(gbm_ctx *ctx, const float *X_d, int64_t n_rows, int32_t F, int32_t max_bins,
                 const float *cv, const int32_t *cp, uint16_t *bins_d, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_REQUIRE(n_rows > 0, GBM_E_EMPTY, "gbm_quantise: zero rows");
    GBM_REQUIRE(X_d && cv && cp && bins_d && F > 0 && max_bins >= 2 && max_bins <= 65535, GBM_E_ARG,
                "gbm_quantise: bad arguments");
    long long total = (long long)n_rows * F;
    quantise_kernel<<<grid_for(total, 256, ctx->sm_count), 256, 0, (cudaStream_t)stream>>>(
        X_d, total, F, cv, cp, max_bins, bins_d, ctx->dev_err);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

int gbm_compress(gbm_ctx *ctx, const uint16_t *bins_d, int64_t n_rows, int32_t F, int32_t bits,
                 int32_t row_align_bits, uint32_t *packed_d, int64_t packed_words, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_REQUIRE(n_rows > 0, GBM_E_EMPTY, "gbm_compress: zero rows");
    int64_t need = gbm_packed_words(n_rows, F, bits, row_align_bits);
    if (need < 0) return (int)need;
    GBM_REQUIRE(bins_d && packed_d && packed_words >= need, GBM_E_ARG,
                "gbm_compress: null pointer or packed buffer too small");
    long long stride = row_stride_bits(F, bits, row_align_bits);
    pack_kernel<false><<<grid_for(packed_words, 256, ctx->sm_count), 256, 0, (cudaStream_t)stream>>>(
        bins_d, nullptr, n_rows, F, bits, stride, nullptr, nullptr, 0, packed_d, packed_words,
        ctx->dev_err);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

int gbm_quantise_compress(gbm_ctx *ctx, const float *X_d, int64_t n_rows, int32_t F,
                          int32_t max_bins, const float *cv, const int32_t *cp, int32_t bits,
                          int32_t row_align_bits, uint32_t *packed_d, int64_t packed_words,
                          void *stream) {
    GBM_TRY(ctx_enter(ctx));
    // a rank of several may hold no rows (its shard of a tiny matrix): only the zero pad words
    const bool empty_rank = n_rows == 0 && coll_on(ctx) && ctx->nranks > 1;
    GBM_REQUIRE(n_rows > 0 || empty_rank, GBM_E_EMPTY, "gbm_quantise_compress: zero rows");
    int64_t need = gbm_packed_words(n_rows, F, bits, row_align_bits);
    if (need < 0) return (int)need;
    GBM_REQUIRE((X_d || empty_rank) && cv && cp && packed_d && packed_words >= need && max_bins >= 2 &&
                    max_bins <= 65535,
                GBM_E_ARG, "gbm_quantise_compress: bad arguments");
    if (empty_rank) {
        GBM_CUDA(cudaMemsetAsync(packed_d, 0, (size_t)packed_words * 4, (cudaStream_t)stream));
        return GBM_OK;
    }
    long long stride = row_stride_bits(F, bits, row_align_bits);
    ProfScope ps(ctx, PC_QUANT, (cudaStream_t)stream, (double)n_rows * F * 4 + (double)packed_words * 4);
    const long long row_words = stride / 32, data_words = (long long)n_rows * row_words;
    if (bits == 8 && stride % 32 == 0 && data_words < (1ll << 32)) {
        // the words past the last row (if any) stay zero
        if (packed_words > data_words)
            GBM_CUDA(cudaMemsetAsync(packed_d + data_words, 0, (size_t)(packed_words - data_words) * 4,
                                     (cudaStream_t)stream));
        pack_byte_kernel<<<grid_for(data_words, 256, ctx->sm_count), 256, 0, (cudaStream_t)stream>>>(
            X_d, F, (uint32_t)row_words, cv, cp, max_bins, packed_d, (uint32_t)data_words, ctx->dev_err);
    } else {
        pack_kernel<true><<<grid_for(packed_words, 256, ctx->sm_count), 256, 0, (cudaStream_t)stream>>>(
            nullptr, X_d, n_rows, F, bits, stride, cv, cp, max_bins, packed_d, packed_words,
            ctx->dev_err);
    }
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

// The exact cuts (R5) of the F columns of Xg ([n_all][F] row-major, NaN = missing, padding rows
// all-NaN) into cut_values_d / cut_ptr_d; on the host: each feature's bin count nb[f] and present
// value count pres[f].  GBM_E_NONFINITE on +-inf.  Synchronises s.
static int cuts_core(gbm_ctx *ctx, const float *Xg, long long n_all, int F, int max_bins, float *cut_values_d,
                     int32_t *cut_ptr_d, std::vector<int32_t> &nb, std::vector<unsigned long long> &pres,
                     cudaStream_t s) {
    ProfScope ps(ctx, PC_CUTS, s, (double)n_all * F * 4);
    const int tiles = (int)((n_all + SORT_TILE - 1) / SORT_TILE);
    const long long n_pad = (long long)tiles * SORT_TILE;
    Arena &A = ctx->arena;
    size_t need = 2 * (size_t)F * n_pad * 4 + (size_t)F * 256 * tiles * 4 + 2 * (size_t)F * tiles * 4 +
                  (size_t)F * 8 + (size_t)F * max_bins * 4 + 3 * (size_t)F * 4 + 16 * 256;
    GBM_TRY(A.reserve(need));
    uint32_t *kA = A.take<uint32_t>((size_t)F * n_pad);
    uint32_t *kB = A.take<uint32_t>((size_t)F * n_pad);
    uint32_t *counts = A.take<uint32_t>((size_t)F * 256 * tiles);
    uint32_t *run_cnt = A.take<uint32_t>((size_t)F * tiles);
    uint32_t *run_off = A.take<uint32_t>((size_t)F * tiles);
    unsigned long long *present = A.take<unsigned long long>(F);
    float *tmp = A.take<float>((size_t)F * max_bins);
    int32_t *nbins = A.take<int32_t>(F);
    int32_t *nbins_plain = A.take<int32_t>(F);
    GBM_CUDA(cudaMemsetAsync(present, 0, (size_t)F * 8, s));
    GBM_CUDA(cudaMemsetAsync(ctx->dev_err, 0, 4, s));
    dim3 tg((unsigned)std::min<long long>((n_pad + 31) / 32, 16ll * ctx->sm_count), (unsigned)((F + 31) / 32));
    keys_kernel<<<tg, 256, 0, s>>>(Xg, n_all, F, n_pad, kA, present, ctx->dev_err);
    GBM_CUDA(cudaGetLastError());
    dim3 sg((unsigned)tiles, (unsigned)F);
    for (int pass = 0; pass < 4; ++pass) {
        int shift = 8 * pass;
        sort_count_kernel<<<sg, SORT_THREADS, 0, s>>>(kA, n_pad, tiles, shift, counts);
        scan_rows_kernel<<<F, 1024, 0, s>>>(counts, 256ll * tiles);
        sort_scatter_kernel<<<sg, SORT_THREADS, 0, s>>>(kA, kB, n_pad, tiles, shift, counts);
        std::swap(kA, kB);
    }
    GBM_CUDA(cudaGetLastError());
    runs_count_kernel<<<sg, SORT_THREADS, 0, s>>>(kA, n_pad, tiles, run_cnt);
    GBM_CUDA(cudaMemcpyAsync(run_off, run_cnt, (size_t)F * tiles * 4, cudaMemcpyDeviceToDevice, s));
    scan_rows_kernel<<<F, 1024, 0, s>>>(run_off, tiles);
    select_kernel<<<F, 1024, 0, s>>>(kA, n_pad, tiles, run_off, run_cnt, present, max_bins, tmp, nbins);
    cutptr_kernel<<<1, 32, 0, s>>>(nbins, F, cut_ptr_d);
    tag_kernel<<<(F + 255) / 256, 256, 0, s>>>(run_off, run_cnt, tiles, F, max_bins, nbins, nbins_plain);
    write_cuts_kernel<<<sg, SORT_THREADS, 0, s>>>(kA, n_pad, tiles, run_off, nbins, tmp, max_bins,
                                                  cut_ptr_d, cut_values_d);
    GBM_CUDA(cudaGetLastError());
    nb.assign(F, 0);
    pres.assign(F, 0);
    uint32_t err = 0;
    GBM_CUDA(cudaMemcpyAsync(nb.data(), nbins_plain, (size_t)F * 4, cudaMemcpyDeviceToHost, s));
    GBM_CUDA(cudaMemcpyAsync(pres.data(), present, (size_t)F * 8, cudaMemcpyDeviceToHost, s));
    GBM_CUDA(cudaMemcpyAsync(&err, ctx->dev_err, 4, cudaMemcpyDeviceToHost, s));
    GBM_CUDA(cudaStreamSynchronize(s));
    if (err & DERR_NONFINITE) {
        cudaMemsetAsync(ctx->dev_err, 0, 4, s);
        return fail(GBM_E_NONFINITE, "gbm_cuts: +-inf feature value (S:32)");
    }
    return GBM_OK;
}

// C3 by per-feature ownership: feature f belongs to rank f mod p; every rank sends
// each owner its shard's columns of the owner's features (all-to-all), the owner computes their
// exact cuts over the global rows, and the ranks all-gather the cuts.  Per-rank memory and traffic
// O(n F / p) instead of the O(n F) of an all-gather of X.
__global__ void owned_columns_kernel(const float *__restrict__ X, long long n, int F, int p,
                                     float *__restrict__ out /* [p][n][F_d] */) {
    // destination d holds features d, d + p, ...; its block starts at n * (features of ranks < d)
    const long long total = n * (long long)F;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / F;
        const int f = (int)(e - i * F);
        const int d = f % p, c = f / p;
        const int Fd = (F - d + p - 1) / p;
        long long before = 0;  // features owned by ranks < d
        for (int q = 0; q < d; ++q) before += (F - q + p - 1) / p;
        out[n * before + i * Fd + c] = X[e];
    }
}

// gathered per-rank results -> the global cut arrays in feature order
__global__ void assemble_cuts_kernel(const float *__restrict__ vals /* [p][Fo][B] */, const int32_t *__restrict__ cnt /* [p][Fo] */,
                                     int F, int p, int Fo, int B, const int32_t *__restrict__ cut_ptr,
                                     float *__restrict__ cut_values) {
    for (int f = blockIdx.x; f < F; f += gridDim.x) {
        const int r = f % p, c = f / p;
        const int nbf = cnt[r * Fo + c];
        const float *src = vals + ((long long)r * Fo + c) * B;
        for (int k = threadIdx.x; k < nbf; k += blockDim.x) cut_values[cut_ptr[f] + k] = src[k];
    }
}

static int cuts_by_ownership(gbm_ctx *ctx, const float *X_d, long long n_rows, int F, int max_bins, float *cut_values_d,
                             int32_t *cut_ptr_d, std::vector<int32_t> &nb, std::vector<unsigned long long> &pres,
                             long long &n_total, cudaStream_t s) {
    const int p = ctx->nranks, r = ctx->rank;
    auto owned = [&](int q) { return q < F ? (F - q + p - 1) / p : 0; };
    const int Fr = owned(r), Fo = std::max(1, owned(0));  // rank 0 owns the most features
    // every rank's row count
    std::vector<long long> ns(p);
    long long *d_n = nullptr;
    GBM_CUDA(cudaMalloc(&d_n, (size_t)(p + 1) * 8));
    struct Free {
        std::vector<void *> v;
        ~Free() { for (void *x : v) cudaFree(x); }
    } fr;
    fr.v.push_back(d_n);
    GBM_CUDA(cudaMemcpyAsync(d_n + p, &n_rows, 8, cudaMemcpyHostToDevice, s));
    GBM_TRY(coll_allgather(ctx, d_n + p, d_n, 8, s));
    GBM_CUDA(cudaMemcpyAsync(ns.data(), d_n, (size_t)p * 8, cudaMemcpyDeviceToHost, s));
    GBM_CUDA(cudaStreamSynchronize(s));
    n_total = 0;
    for (long long v : ns) n_total += v;
    if (n_total <= 0) return fail(GBM_E_EMPTY, "gbm_cuts: zero rows");
    // all-to-all of the owned columns: to rank d, [n_rows][F_d]; from rank q, [ns[q]][F_r]
    std::vector<size_t> soff(p), scnt(p), roff(p), rcnt(p);
    size_t o = 0;
    for (int d = 0; d < p; ++d) {
        soff[d] = o;
        scnt[d] = (size_t)n_rows * owned(d);
        o += scnt[d];
    }
    o = 0;
    for (int q = 0; q < p; ++q) {
        roff[q] = o;
        rcnt[q] = (size_t)ns[q] * Fr;
        o += rcnt[q];
    }
    float *sendb = nullptr, *recvb = nullptr;
    GBM_CUDA(cudaMalloc(&sendb, std::max<size_t>((size_t)n_rows * F, 1) * 4));
    fr.v.push_back(sendb);
    GBM_CUDA(cudaMalloc(&recvb, std::max<size_t>((size_t)n_total * Fr, 1) * 4));
    fr.v.push_back(recvb);
    if (n_rows > 0) {
        owned_columns_kernel<<<grid_for(n_rows * (long long)F, 256, ctx->sm_count), 256, 0, s>>>(X_d, n_rows, F, p, sendb);
        GBM_CUDA(cudaGetLastError());
    }
    GBM_TRY(coll_alltoallv_f32(ctx, sendb, soff.data(), scnt.data(), recvb, roff.data(), rcnt.data(), s));
    // this rank's features over the global rows
    const size_t vbytes = (size_t)Fo * max_bins * 4;
    float *vals = nullptr, *gvals = nullptr;
    int32_t *cnt = nullptr, *gcnt = nullptr, *lptr = nullptr, *gptr = nullptr;
    unsigned long long *pr = nullptr, *gpr = nullptr;
    GBM_CUDA(cudaMalloc(&vals, vbytes));
    fr.v.push_back(vals);
    GBM_CUDA(cudaMalloc(&gvals, vbytes * p));
    fr.v.push_back(gvals);
    GBM_CUDA(cudaMalloc(&cnt, (size_t)Fo * 4));
    fr.v.push_back(cnt);
    GBM_CUDA(cudaMalloc(&gcnt, (size_t)Fo * 4 * p));
    fr.v.push_back(gcnt);
    GBM_CUDA(cudaMalloc(&pr, (size_t)Fo * 8));
    fr.v.push_back(pr);
    GBM_CUDA(cudaMalloc(&gpr, (size_t)Fo * 8 * p));
    fr.v.push_back(gpr);
    GBM_CUDA(cudaMalloc(&lptr, (size_t)(Fo + 1) * 4));
    fr.v.push_back(lptr);
    GBM_CUDA(cudaMalloc(&gptr, (size_t)(F + 1) * 4));
    fr.v.push_back(gptr);
    GBM_CUDA(cudaMemsetAsync(vals, 0, vbytes, s));
    GBM_CUDA(cudaMemsetAsync(cnt, 0, (size_t)Fo * 4, s));
    GBM_CUDA(cudaMemsetAsync(pr, 0, (size_t)Fo * 8, s));
    std::vector<int32_t> lnb;
    std::vector<unsigned long long> lpres;
    int rc = GBM_OK;
    if (Fr > 0) {
        float *lcv = nullptr;
        GBM_CUDA(cudaMalloc(&lcv, (size_t)Fr * max_bins * 4));
        fr.v.push_back(lcv);
        rc = cuts_core(ctx, recvb, n_total, Fr, max_bins, lcv, lptr, lnb, lpres, s);
        if (rc == GBM_OK) {  // to the fixed-stride exchange layout [Fo][max_bins]
            std::vector<int32_t> lp(Fr + 1);
            GBM_CUDA(cudaMemcpy(lp.data(), lptr, (size_t)(Fr + 1) * 4, cudaMemcpyDeviceToHost));
            for (int c = 0; c < Fr; ++c)
                if (lnb[c])
                    GBM_CUDA(cudaMemcpyAsync(vals + (size_t)c * max_bins, lcv + lp[c], (size_t)lnb[c] * 4,
                                             cudaMemcpyDeviceToDevice, s));
            GBM_CUDA(cudaMemcpyAsync(cnt, lnb.data(), (size_t)Fr * 4, cudaMemcpyHostToDevice, s));
            GBM_CUDA(cudaMemcpyAsync(pr, lpres.data(), (size_t)Fr * 8, cudaMemcpyHostToDevice, s));
        }
    }
    // every rank joins the exchange even if its own cuts failed (its code rides along in cnt)
    int32_t my_err = rc == GBM_OK ? 0 : rc;
    int32_t *errb = nullptr;
    GBM_CUDA(cudaMalloc(&errb, (size_t)(p + 1) * 4));
    fr.v.push_back(errb);
    GBM_CUDA(cudaMemcpyAsync(errb + p, &my_err, 4, cudaMemcpyHostToDevice, s));
    GBM_TRY(coll_allgather(ctx, errb + p, errb, 4, s));
    GBM_TRY(coll_allgather(ctx, vals, gvals, vbytes, s));
    GBM_TRY(coll_allgather(ctx, cnt, gcnt, (size_t)Fo * 4, s));
    GBM_TRY(coll_allgather(ctx, pr, gpr, (size_t)Fo * 8, s));
    std::vector<int32_t> errs(p), hc((size_t)Fo * p);
    std::vector<unsigned long long> hp((size_t)Fo * p);
    GBM_CUDA(cudaMemcpyAsync(errs.data(), errb, (size_t)p * 4, cudaMemcpyDeviceToHost, s));
    GBM_CUDA(cudaMemcpyAsync(hc.data(), gcnt, (size_t)Fo * 4 * p, cudaMemcpyDeviceToHost, s));
    GBM_CUDA(cudaMemcpyAsync(hp.data(), gpr, (size_t)Fo * 8 * p, cudaMemcpyDeviceToHost, s));
    GBM_CUDA(cudaStreamSynchronize(s));
    for (int q = 0; q < p; ++q)
        if (errs[q] != 0)
            return rc != GBM_OK ? rc : fail(errs[q], "gbm_cuts: another rank failed (code " + std::to_string(errs[q]) + ")");
    nb.assign(F, 0);
    pres.assign(F, 0);
    std::vector<int32_t> cp(F + 1, 0);
    for (int f = 0; f < F; ++f) {
        const int q = f % p, c = f / p;
        nb[f] = hc[(size_t)q * Fo + c];
        pres[f] = hp[(size_t)q * Fo + c];
        cp[f + 1] = cp[f] + nb[f];
    }
    GBM_CUDA(cudaMemcpyAsync(cut_ptr_d, cp.data(), (size_t)(F + 1) * 4, cudaMemcpyHostToDevice, s));
    GBM_CUDA(cudaMemcpyAsync(gptr, cp.data(), (size_t)(F + 1) * 4, cudaMemcpyHostToDevice, s));
    assemble_cuts_kernel<<<std::min(F, 1024), 256, 0, s>>>(gvals, gcnt, F, p, Fo, max_bins, gptr, cut_values_d);
    GBM_CUDA(cudaGetLastError());
    GBM_CUDA(cudaStreamSynchronize(s));  // the host tables and scratch are released on return
    return GBM_OK;
}

int gbm_cuts(gbm_ctx *ctx, const float *X_d, int64_t n_rows, int32_t F, int32_t max_bins,
             float *cut_values_d, int32_t *cut_ptr_d, int32_t *n_cuts_h, int32_t *max_symbol_h,
             void *stream) {
    GBM_TRY(ctx_enter(ctx));
    cudaStream_t s = (cudaStream_t)stream;
    // local checks, then one collective decision: the same error, or GBM_E_MISMATCH when the ranks
    // disagree on the features, max_bins or the C3 mode
    const int local = (F > 0 && max_bins >= 2 && max_bins <= 65535 && cut_values_d && cut_ptr_d && n_cuts_h &&
                       max_symbol_h && n_rows >= 0 && (X_d || n_rows == 0))
                          ? GBM_OK
                          : fail(GBM_E_ARG, "gbm_cuts: bad arguments");
    const long long sig[3] = {F, max_bins, ctx->cuts_gather};
    GBM_TRY(coll_agree(ctx, local, sig, 3, s, "gbm_cuts"));
    std::vector<int32_t> nb;
    std::vector<unsigned long long> pres;
    long long n_total = n_rows;
    if (coll_on(ctx) && ctx->nranks > 1 && ctx->cuts_gather == 0) {
        GBM_TRY(cuts_by_ownership(ctx, X_d, n_rows, F, max_bins, cut_values_d, cut_ptr_d, nb, pres, n_total, s));
    } else {
        // single rank, or GBM_OPT_CUTS_GATHER: all-gather the shards (C3), padded with NaN rows
        long long n_max = n_rows;
        const float *Xg = X_d;
        float *gathered = nullptr;
        if (coll_on(ctx)) {
            long long *tmp;
            GBM_CUDA(cudaMallocAsync((void **)&tmp, 2 * sizeof(long long), s));
            long long h2[2] = {n_rows, n_rows};
            GBM_CUDA(cudaMemcpyAsync(tmp, h2, sizeof(h2), cudaMemcpyHostToDevice, s));
            int rc = coll_allreduce(ctx, tmp, 1, COLL_SUM_I64, s);
            if (rc == GBM_OK) rc = coll_allreduce(ctx, tmp + 1, 1, COLL_MAX_I64, s);
            if (rc == GBM_OK && cudaMemcpyAsync(h2, tmp, sizeof(h2), cudaMemcpyDeviceToHost, s) != cudaSuccess)
                rc = fail(GBM_E_CUDA, "gbm_cuts: copy of the global row counts");
            if (rc == GBM_OK && cudaStreamSynchronize(s) != cudaSuccess) rc = fail(GBM_E_CUDA, "gbm_cuts: sync");
            cudaFreeAsync(tmp, s);
            if (rc != GBM_OK) return rc;
            n_total = h2[0];
            n_max = h2[1];
            size_t slab = (size_t)n_max * F;
            float *mine = nullptr;
            if (cudaMallocAsync((void **)&gathered, std::max<size_t>(slab, 1) * ctx->nranks * sizeof(float), s) != cudaSuccess ||
                cudaMallocAsync((void **)&mine, std::max<size_t>(slab, 1) * sizeof(float), s) != cudaSuccess) {
                cudaGetLastError();
                if (gathered) cudaFreeAsync(gathered, s);
                return fail(GBM_E_NOMEM, "gbm_cuts: cannot allocate the gathered rows");
            }
            cudaMemsetAsync(mine, 0xff, slab * sizeof(float), s);  // 0xffffffff is a NaN
            if (n_rows) cudaMemcpyAsync(mine, X_d, (size_t)n_rows * F * sizeof(float), cudaMemcpyDeviceToDevice, s);
            rc = coll_allgather(ctx, mine, gathered, slab * sizeof(float), s);  // C3
            cudaFreeAsync(mine, s);
            if (rc != GBM_OK) {
                cudaFreeAsync(gathered, s);
                return rc;
            }
            Xg = gathered;
            n_max = n_max * ctx->nranks;  // rows of the gathered buffer (padding rows are all-NaN)
        }
        if (n_total <= 0) {
            if (gathered) cudaFreeAsync(gathered, s);
            return fail(GBM_E_EMPTY, "gbm_cuts: zero rows");
        }
        const int rc = cuts_core(ctx, Xg, n_max, F, max_bins, cut_values_d, cut_ptr_d, nb, pres, s);
        if (gathered) cudaFreeAsync(gathered, s);
        GBM_TRY(rc);
    }
    long long tb = 0, present_total = 0;
    int max_nb = 0;
    for (int f = 0; f < F; ++f) {
        tb += nb[f];
        present_total += (long long)pres[f];
        max_nb = std::max(max_nb, nb[f]);
    }
    *n_cuts_h = (int32_t)tb;
    bool any_missing = present_total < n_total * (long long)F;
    *max_symbol_h = any_missing ? max_bins : std::max(0, max_nb - 1);
    return GBM_OK;
}

int gbm_transpose_symbols(gbm_ctx *ctx, const gbm_qmatrix *q, uint8_t *colsym_d, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_REQUIRE(q && q->packed_d && colsym_d && q->n_features > 0 && q->n_rows >= 0, GBM_E_ARG,
                "gbm_transpose_symbols: bad arguments");
    GBM_REQUIRE(q->bits >= 1 && q->bits <= 8, GBM_E_ARG, "gbm_transpose_symbols: needs bits <= 8");
    if (q->n_rows == 0) return GBM_OK;
    gbm_qmatrix qq = *q;
    qq.colsym_d = nullptr;
    const QM qm = make_qm(&qq);
    const size_t sm = (size_t)TR_ROWS * q->n_features;
    GBM_REQUIRE(sm <= 200 * 1024, GBM_E_ARG, "gbm_transpose_symbols: too many features");
    if (sm > 48 * 1024) GBM_CUDA(cudaFuncSetAttribute(transpose_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    ProfScope ps(ctx, PC_QUANT, (cudaStream_t)stream, (double)q->n_rows * q->n_features * (q->bits / 8.0 + 1.0));
    transpose_kernel<<<(int)((q->n_rows + TR_ROWS - 1) / TR_ROWS), 256, sm, (cudaStream_t)stream>>>(qm, q->n_rows, colsym_d);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

}  // extern "C"
