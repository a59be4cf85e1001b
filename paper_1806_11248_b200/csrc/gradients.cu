// gradients.cu -- §2.5 gradient evaluation (Eq. 1-2) with the fixed point of R14,
// §2.4 prediction and the margin update on sm_100a.
//
// Bit-exactness (R19-R21): the sigmoid goes through det_exp, which uses only correctly rounded
// IEEE +,-,*,/, fma and an exact power-of-two scale, and every fp64 op is an explicitly rounded
// intrinsic (no contraction).  All three kernels are plain streaming kernels: HBM-bound.
#include <algorithm>

#include "gbm_internal.cuh"

namespace gbm {

constexpr int G_THREADS = 256;
constexpr int GU = 4;  // rows in flight per thread in the streaming kernels

// pass 1: per-row (g, h), the block maxima of |g|, |h|; for the logistic objective the
// sigmoid of each row is kept (sig) so that pass 2 does not evaluate det_exp again
__global__ void __launch_bounds__(G_THREADS) grad_max_kernel(int obj, const double *__restrict__ margin,
                                                             const float *__restrict__ label, long long n,
                                                             unsigned long long *__restrict__ maxbits,
                                                             double *__restrict__ sig, uint32_t *dev_err) {
    double mg = 0.0, mh = 0.0;
    bool bad = false;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n; i0 += GU * stride) {
        float yl[GU];
        double v[GU];
#pragma unroll
        for (int u = 0; u < GU; ++u) {  // GU rows' loads in flight
            const long long i = i0 + u * stride;
            yl[u] = i < n ? __ldg(label + i) : 0.0f;
            v[u] = i < n ? __ldg(margin + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < GU; ++u) {
            const long long i = i0 + u * stride;
            if (i >= n) break;
            if (obj == GBM_LOGISTIC) {
                v[u] = sigmoid(v[u]);
                sig[i] = v[u];
                bad |= !(yl[u] == 0.0f || yl[u] == 1.0f);
            }
            double g, h;
            grad_hess_s(obj, v[u], yl[u], g, h);
            mg = fmax(mg, fabs(g));
            mh = fmax(mh, fabs(h));
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(dev_err, DERR_LABEL);
    for (int o = 16; o > 0; o >>= 1) {
        mg = fmax(mg, __shfl_xor_sync(0xffffffffu, mg, o));
        mh = fmax(mh, __shfl_xor_sync(0xffffffffu, mh, o));
    }
    __shared__ double sg[G_THREADS / 32], sh[G_THREADS / 32];
    if ((threadIdx.x & 31) == 0) {
        sg[threadIdx.x >> 5] = mg;
        sh[threadIdx.x >> 5] = mh;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < G_THREADS / 32; ++w) {
            mg = fmax(mg, sg[w]);
            mh = fmax(mh, sh[w]);
        }
        // non-negative doubles order like their bit patterns
        atomicMax(maxbits + 0, (unsigned long long)__double_as_longlong(mg));
        atomicMax(maxbits + 1, (unsigned long long)__double_as_longlong(mh));
    }
}

__device__ __forceinline__ int scale_of(unsigned long long bits, int P) {
    double M = __longlong_as_double((long long)bits);
    int E = 0;
    if (M > 0.0) frexp(M, &E);
    return P - E;
}

__global__ void __launch_bounds__(G_THREADS) grad_quant_kernel(int obj, int P, const double *__restrict__ margin,
                                                               const float *__restrict__ label, long long n,
                                                               const unsigned long long *__restrict__ maxbits,
                                                               const double *__restrict__ sig,
                                                               int2 *__restrict__ qpair, int32_t *__restrict__ scale) {
    const int sg = scale_of(maxbits[0], P), sh = scale_of(maxbits[1], P);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        scale[0] = sg;
        scale[1] = sh;
    }
    const long long stride = (long long)gridDim.x * blockDim.x;
    const double *src = obj == GBM_LOGISTIC ? sig : margin;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n; i0 += GU * stride) {
        double v[GU];
        float yl[GU];
#pragma unroll
        for (int u = 0; u < GU; ++u) {
            const long long i = i0 + u * stride;
            v[u] = i < n ? __ldg(src + i) : 0.0;
            yl[u] = i < n ? __ldg(label + i) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < GU; ++u) {
            const long long i = i0 + u * stride;
            if (i >= n) break;
            double g, h;
            grad_hess_s(obj, v[u], yl[u], g, h);
            qpair[i] = make_int2(__double2int_rn(ldexp_exact(g, sg)), __double2int_rn(ldexp_exact(h, sh)));
        }
    }
}

__global__ void update_margins_kernel(const double *__restrict__ w, const int32_t *__restrict__ leaf,
                                      long long n, double *__restrict__ margin) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n; i0 += GU * stride) {
        double m[GU];
        int lf[GU];
#pragma unroll
        for (int u = 0; u < GU; ++u) {
            const long long i = i0 + u * stride;
            m[u] = i < n ? margin[i] : 0.0;
            lf[u] = i < n ? __ldg(leaf + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < GU; ++u) {
            const long long i = i0 + u * stride;
            if (i < n) margin[i] = dadd(m[u], __ldg(w + lf[u]));
        }
    }
}

// LINKED: children of k are left_child[k], left_child[k] + 1 (R27); else heap 2k+1, 2k+2
template <bool LINKED>
__global__ void predict_kernel(int n_trees, long long cap, const int8_t *__restrict__ kind,
                               const int32_t *__restrict__ feature, const float *__restrict__ thr,
                               const int8_t *__restrict__ dl, const int32_t *__restrict__ left_child,
                               const double *__restrict__ weight, double base, const float *__restrict__ X,
                               long long n, int F, double *__restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float *x = X + i * F;
        double m = base;
        for (int t = 0; t < n_trees; ++t) {
            long long o = t * cap, k = 0;
            while (__ldg(kind + o + k) == GBM_NODE_SPLIT) {
                int f = __ldg(feature + o + k);
                float v = f < F ? __ldg(x + f) : __int_as_float(0x7fffffff);
                bool left = isnan(v) ? (__ldg(dl + o + k) != 0) : (v <= __ldg(thr + o + k));
                if (LINKED) {
                    const long long c = __ldg(left_child + o + k);
                    k = left ? c : c + 1;
                } else {
                    k = left ? 2 * k + 1 : 2 * k + 2;
                }
            }
            m = dadd(m, __ldg(weight + o + k));
        }
        out[i] = m;
    }
}

// Staged prediction ("one training instance per thread ... iterating through each tree
// sequentially", Q7): a block stages PR_ROWS rows of X with coalesced 16-byte loads into shared
// memory (row pitch F | 1 floats: the per-thread reads of one feature fall into distinct banks) and
// a chunk of trees as packed node records; each thread then walks its row through the chunk's
// trees in order, adding the leaf weights to its fp64 margin in tree order (the oracle's
// operation sequence).  Nodes: meta = (threshold bits, feature | default_left << 16 | split << 17),
// left child (heap 2k+1, or left_child[k] for linked trees), weight.
constexpr int PR_THREADS = 256;
constexpr int PR_ROWS = 256;  // one row per thread
constexpr int PR_FMAX = 64;   // features staged (wider matrices use predict_kernel)
struct PNode {
    uint32_t thr;   // threshold bits
    uint32_t info;  // feature (16 bits) | default_left << 16 | split << 17
};

template <bool LINKED>
__global__ void __launch_bounds__(PR_THREADS) predict_stg_kernel(
    int n_trees, long long cap, int trees_per_chunk, const int8_t *__restrict__ kind,
    const int32_t *__restrict__ feature, const float *__restrict__ thr, const int8_t *__restrict__ dl,
    const int32_t *__restrict__ left_child, const double *__restrict__ weight, double base,
    const float *__restrict__ X, long long n, int F, double *__restrict__ out) {
    extern __shared__ __align__(16) unsigned char psm[];
    const int pitch = F | 1;
    float *xs = reinterpret_cast<float *>(psm);                                   // [PR_ROWS][pitch]
    const size_t xs_bytes = ((size_t)PR_ROWS * pitch * 4 + 15) & ~size_t(15);
    const int chunk_nodes = trees_per_chunk * (int)cap;
    double *ws = reinterpret_cast<double *>(psm + xs_bytes);                      // [chunk_nodes]
    PNode *ns = reinterpret_cast<PNode *>(ws + chunk_nodes);                      // [chunk_nodes]
    int32_t *ls = reinterpret_cast<int32_t *>(ns + chunk_nodes);                  // [chunk_nodes] (LINKED)
    const long long tiles = (n + PR_ROWS - 1) / PR_ROWS;
    const bool vec = (F % 4) == 0;  // rows of whole float4s (16-byte aligned when X is)
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const long long r0 = tile * PR_ROWS;
        const int nr = (int)min((long long)PR_ROWS, n - r0);
        __syncthreads();  // previous tile's readers are done
        if (vec) {
            const float4 *src = reinterpret_cast<const float4 *>(X + r0 * F);
            const int F4 = F / 4;
            for (int i = threadIdx.x; i < nr * F4; i += PR_THREADS) {
                const float4 v = __ldg(src + i);
                const int r = i / F4, c = (i - r * F4) * 4;
                float *d = xs + r * pitch + c;
                d[0] = v.x;
                d[1] = v.y;
                d[2] = v.z;
                d[3] = v.w;
            }
        } else {
            const float *src = X + r0 * F;
            for (int i = threadIdx.x; i < nr * F; i += PR_THREADS) {
                const int r = i / F;
                xs[r * pitch + (i - r * F)] = __ldg(src + i);
            }
        }
        double m = base;
        const int row = threadIdx.x;
        const float *x = xs + row * pitch;
        for (int t0 = 0; t0 < n_trees; t0 += trees_per_chunk) {
            const int nt = min(trees_per_chunk, n_trees - t0);
            if (t0 > 0 || tile == blockIdx.x || n_trees > trees_per_chunk) {
                if (t0 > 0) __syncthreads();  // the previous chunk's walkers are done
                const long long base_node = (long long)t0 * cap;
                for (int i = threadIdx.x; i < nt * (int)cap; i += PR_THREADS) {
                    const long long g = base_node + i;
                    const int k = __ldg(kind + g);
                    const int f = __ldg(feature + g);
                    PNode pn;
                    pn.thr = __float_as_uint(__ldg(thr + g));
                    pn.info = (k == GBM_NODE_SPLIT) ? ((uint32_t)(f & 0xffff) | ((uint32_t)(__ldg(dl + g) != 0) << 16) |
                                                       (1u << 17))
                                                    : 0u;
                    ns[i] = pn;
                    ws[i] = __ldg(weight + g);
                    if (LINKED) ls[i] = __ldg(left_child + g);
                }
            }
            __syncthreads();
            if (row < nr) {
                for (int t = 0; t < nt; ++t) {
                    const int o = t * (int)cap;
                    int k = 0;
                    PNode pn = ns[o];
                    while (pn.info & (1u << 17)) {
                        const int f = pn.info & 0xffff;
                        const float v = f < F ? x[f] : __int_as_float(0x7fffffff);
                        const bool left = isnan(v) ? ((pn.info >> 16) & 1u) : (v <= __uint_as_float(pn.thr));
                        const int c = LINKED ? ls[o + k] : 2 * k + 1;
                        k = left ? c : c + 1;
                        pn = ns[o + k];
                    }
                    m = dadd(m, ws[o + k]);
                }
            }
        }
        if (row < nr) out[r0 + row] = m;
    }
}

// shared bytes of predict_stg_kernel for F features and `trees` trees of capacity cap per chunk
static size_t predict_smem(int F, long long cap, int trees, bool linked) {
    const size_t xs = ((size_t)PR_ROWS * (F | 1) * 4 + 15) & ~size_t(15);
    return xs + (size_t)trees * cap * (8 + sizeof(PNode) + (linked ? 4 : 0));
}

// staged launch when it applies (F <= PR_FMAX, at least one tree fits): 1 on success, 0 to fall
// back to predict_kernel, < 0 on a CUDA error
template <bool LINKED>
static int launch_predict_stg(gbm_ctx *ctx, int n_trees, long long cap, const int8_t *kind, const int32_t *feature,
                              const float *thr, const int8_t *dl, const int32_t *left_child, const double *weight,
                              double base, const float *X, long long n, int F, double *out, cudaStream_t s) {
    if (F > PR_FMAX || F >= 65536 || cap > (1 << 20) || reinterpret_cast<uintptr_t>(X) % 16 != 0) return 0;
    const size_t budget = 96 * 1024;  // two blocks per SM
    const size_t one = predict_smem(F, cap, 1, LINKED);
    if (one > budget) return 0;
    int tpc = (int)std::max<long long>(1, std::min<long long>(std::max(n_trees, 1),
                                                              (long long)((budget - predict_smem(F, cap, 0, LINKED)) /
                                                                          (cap * (8 + sizeof(PNode) + (LINKED ? 4 : 0))))));
    const size_t sm = predict_smem(F, cap, tpc, LINKED);
    if (cudaFuncSetAttribute(predict_stg_kernel<LINKED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
        cudaSuccess)
        return fail(GBM_E_CUDA, "predict: shared memory attribute");
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, predict_stg_kernel<LINKED>, PR_THREADS, sm) != cudaSuccess ||
        occ < 1)
        return 0;
    const long long tiles = (n + PR_ROWS - 1) / PR_ROWS;
    const int grid = (int)std::max<long long>(1, std::min<long long>(tiles, (long long)occ * ctx->sm_count));
    predict_stg_kernel<LINKED><<<grid, PR_THREADS, sm, s>>>(n_trees, cap, tpc, kind, feature, thr, dl, left_child,
                                                            weight, base, X, n, F, out);
    return cudaGetLastError() == cudaSuccess ? 1 : fail(GBM_E_CUDA, "predict_stg_kernel launch");
}

static int grid_for(long long work, int threads, int sm) {
    long long g = (work + threads - 1) / threads;
    long long cap = (long long)sm * 16;
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace gbm

using namespace gbm;

extern "C" {

}  // extern "C"

namespace gbm {
// pass 1 of gbm_gradients into caller-provided statistics (maxbits zeroed here)
int grad_pass1(gbm_ctx *ctx, int objective, const double *margin_d, const float *label_d, long long n_rows,
               unsigned long long *maxbits, double *sig, cudaStream_t s) {
    GBM_CUDA(cudaMemsetAsync(maxbits, 0, 16, s));
    if (n_rows > 0) {
        ProfScope ps(ctx, PC_GRAD_MAX, s, (double)n_rows * 12);
        grad_max_kernel<<<grid_for(n_rows, G_THREADS, ctx->sm_count), G_THREADS, 0, s>>>(
            objective, margin_d, label_d, n_rows, maxbits, sig, ctx->dev_err);
        GBM_CUDA(cudaGetLastError());
    }
    return GBM_OK;
}
// pass 2: C1 (global max over ranks) and the fixed-point quantisation
static int grad_pass2(gbm_ctx *ctx, int objective, int grad_bits, const double *margin_d, const float *label_d,
                      long long n_rows, unsigned long long *maxbits, const double *sig, int32_t *qpair_d,
                      int32_t *scale_d, cudaStream_t s) {
    if (coll_on(ctx)) {  // C1: global max of |g|, |h| (exact, order-free)
        ProfScope ps(ctx, PC_ALLREDUCE, s, 16.0);
        GBM_TRY(coll_allreduce(ctx, maxbits, 2, COLL_MAX_U64, s));
    }
    {
        ProfScope ps(ctx, PC_GRAD_QUANT, s, (double)n_rows * 20);
        grad_quant_kernel<<<grid_for(n_rows, G_THREADS, ctx->sm_count), G_THREADS, 0, s>>>(
            objective, grad_bits, margin_d, label_d, n_rows, maxbits, sig, reinterpret_cast<int2 *>(qpair_d), scale_d);
    }
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}
int update_margins_launch(gbm_ctx *ctx, const double *weight_d, const int32_t *row_leaf_d, long long n_rows,
                          double *margin_d, cudaStream_t s) {
    if (n_rows == 0) return GBM_OK;
    ProfScope ps(ctx, PC_MARGINS, s, (double)n_rows * 20);
    update_margins_kernel<<<grid_for(n_rows, 256, ctx->sm_count), 256, 0, s>>>(weight_d, row_leaf_d, n_rows, margin_d);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}
}  // namespace gbm

extern "C" {

int gbm_gradients_from_stats(gbm_ctx *ctx, int32_t objective, int32_t grad_bits, const double *margin_d,
                             const float *label_d, int64_t n_rows, const double *sig_d, uint64_t *maxbits_d,
                             int32_t *qpair_d, int32_t *scale_d, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    auto check = [&]() -> int {
        GBM_REQUIRE(objective == GBM_SQUARED_ERROR || objective == GBM_LOGISTIC, GBM_E_ARG,
                    "gbm_gradients_from_stats: unknown objective");
        GBM_REQUIRE(grad_bits >= 1 && grad_bits <= 30, GBM_E_ARG, "gbm_gradients_from_stats: grad_bits in 1..30");
        GBM_REQUIRE(n_rows > 0 || (coll_on(ctx) && ctx->nranks > 1), GBM_E_EMPTY,
                    "gbm_gradients_from_stats: zero rows");
        GBM_REQUIRE(((margin_d && label_d && qpair_d) || n_rows == 0) && scale_d && maxbits_d &&
                        (objective != GBM_LOGISTIC || sig_d || n_rows == 0),
                    GBM_E_ARG, "gbm_gradients_from_stats: null pointer");
        return GBM_OK;
    };
    const long long sig[2] = {objective, grad_bits};  // C1 follows: every rank agrees first
    GBM_TRY(coll_agree(ctx, check(), sig, 2, (cudaStream_t)stream, "gbm_gradients_from_stats"));
    return grad_pass2(ctx, objective, grad_bits, margin_d, label_d, n_rows,
                      reinterpret_cast<unsigned long long *>(maxbits_d), sig_d, qpair_d, scale_d, (cudaStream_t)stream);
}

int gbm_gradients(gbm_ctx *ctx, int32_t objective, int32_t grad_bits, const double *margin_d,
                  const float *label_d, int64_t n_rows, int32_t *qpair_d, int32_t *scale_d,
                  void *stream) {
    GBM_TRY(ctx_enter(ctx));
    auto check = [&]() -> int {
        GBM_REQUIRE(objective == GBM_SQUARED_ERROR || objective == GBM_LOGISTIC, GBM_E_ARG,
                    "gbm_gradients: unknown objective");
        GBM_REQUIRE(grad_bits >= 1 && grad_bits <= 30, GBM_E_ARG, "gbm_gradients: grad_bits in 1..30");
        GBM_REQUIRE(n_rows > 0 || (coll_on(ctx) && ctx->nranks > 1), GBM_E_EMPTY, "gbm_gradients: zero rows");
        GBM_REQUIRE((margin_d && label_d && qpair_d) || n_rows == 0, GBM_E_ARG, "gbm_gradients: null pointer");
        GBM_REQUIRE(scale_d, GBM_E_ARG, "gbm_gradients: null scale");
        return GBM_OK;
    };
    const long long sig[2] = {objective, grad_bits};  // C1 follows: every rank agrees first
    GBM_TRY(coll_agree(ctx, check(), sig, 2, (cudaStream_t)stream, "gbm_gradients"));
    cudaStream_t s = (cudaStream_t)stream;
    const bool lg = objective == GBM_LOGISTIC;
    GBM_TRY(ctx->arena.reserve(512 + (lg ? (size_t)n_rows * 8 : 0)));
    unsigned long long *maxbits = ctx->arena.take<unsigned long long>(2);
    double *sig_p = lg ? ctx->arena.take<double>((size_t)std::max<int64_t>(n_rows, 1)) : nullptr;
    GBM_TRY(grad_pass1(ctx, objective, margin_d, label_d, n_rows, maxbits, sig_p, s));
    return grad_pass2(ctx, objective, grad_bits, margin_d, label_d, n_rows, maxbits, sig_p, qpair_d, scale_d, s);
}

int gbm_update_margins(gbm_ctx *ctx, const double *weight_d, const int32_t *row_leaf_d,
                       int64_t n_rows, double *margin_d, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_REQUIRE(n_rows >= 0 && weight_d && row_leaf_d && margin_d, GBM_E_ARG, "gbm_update_margins: bad arguments");
    if (n_rows == 0) return GBM_OK;
    ProfScope ps(ctx, PC_MARGINS, (cudaStream_t)stream, (double)n_rows * 20);
    update_margins_kernel<<<grid_for(n_rows, 256, ctx->sm_count), 256, 0, (cudaStream_t)stream>>>(
        weight_d, row_leaf_d, n_rows, margin_d);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

int gbm_predict(gbm_ctx *ctx, int32_t n_trees, int32_t max_depth, const int8_t *kind_d,
                const int32_t *feature_d, const float *threshold_d, const int8_t *default_left_d,
                const double *weight_d, double base_margin, const float *X_d, int64_t n_rows,
                int32_t n_features, double *margin_d, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_REQUIRE(n_trees >= 0 && max_depth >= 0 && max_depth <= 24 && n_rows >= 0 && n_features > 0,
                GBM_E_ARG, "gbm_predict: bad sizes");
    GBM_REQUIRE(margin_d && (X_d || n_rows == 0) &&
                    (n_trees == 0 || (kind_d && feature_d && threshold_d && default_left_d && weight_d)),
                GBM_E_ARG, "gbm_predict: null pointer");
    if (n_rows == 0) return GBM_OK;
    long long cap = (1ll << (max_depth + 1)) - 1;
    ProfScope ps(ctx, PC_PREDICT, (cudaStream_t)stream, (double)n_rows * (4.0 * n_features + 8.0));
    const int st = launch_predict_stg<false>(ctx, n_trees, cap, kind_d, feature_d, threshold_d, default_left_d, nullptr,
                                             weight_d, base_margin, X_d, n_rows, n_features, margin_d,
                                             (cudaStream_t)stream);
    if (st < 0) return st;
    if (st == 0)  // wide rows: per-thread gathers of the visited features
        predict_kernel<false><<<grid_for(n_rows, 128, ctx->sm_count), 128, 0, (cudaStream_t)stream>>>(
            n_trees, cap, kind_d, feature_d, threshold_d, default_left_d, nullptr, weight_d, base_margin, X_d,
            n_rows, n_features, margin_d);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

int gbm_predict_linked(gbm_ctx *ctx, int32_t n_trees, int64_t cap, const int8_t *kind_d,
                       const int32_t *feature_d, const float *threshold_d, const int8_t *default_left_d,
                       const int32_t *left_child_d, const double *weight_d, double base_margin,
                       const float *X_d, int64_t n_rows, int32_t n_features, double *margin_d, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    GBM_REQUIRE(n_trees >= 0 && cap >= 1 && n_rows >= 0 && n_features > 0, GBM_E_ARG,
                "gbm_predict_linked: bad sizes");
    GBM_REQUIRE(margin_d && (X_d || n_rows == 0) &&
                    (n_trees == 0 || (kind_d && feature_d && threshold_d && default_left_d && left_child_d &&
                                      weight_d)),
                GBM_E_ARG, "gbm_predict_linked: null pointer");
    if (n_rows == 0) return GBM_OK;
    ProfScope ps(ctx, PC_PREDICT, (cudaStream_t)stream, (double)n_rows * (4.0 * n_features + 8.0));
    const int st = launch_predict_stg<true>(ctx, n_trees, cap, kind_d, feature_d, threshold_d, default_left_d,
                                            left_child_d, weight_d, base_margin, X_d, n_rows, n_features, margin_d,
                                            (cudaStream_t)stream);
    if (st < 0) return st;
    if (st == 0)
        predict_kernel<true><<<grid_for(n_rows, 128, ctx->sm_count), 128, 0, (cudaStream_t)stream>>>(
            n_trees, cap, kind_d, feature_d, threshold_d, default_left_d, left_child_d, weight_d, base_margin,
            X_d, n_rows, n_features, margin_d);
    GBM_CUDA(cudaGetLastError());
    return GBM_OK;
}

}  // extern "C"
