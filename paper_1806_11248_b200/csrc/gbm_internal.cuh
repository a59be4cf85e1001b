// gbm_internal.cuh -- shared internals of libgbm.so (device helpers, context, error plumbing).
// Product code: never includes or links anything under oracle/.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/gbm.h"

struct gbm_vcomm;  // comm.cu: in-process communicator of virtual ranks

namespace gbm {

// ------------------------------------------------------------------ error plumbing
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);

#define GBM_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return ::gbm::fail(GBM_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define GBM_NCCL(call)                                                                        \
    do {                                                                                      \
        ncclResult_t r_ = (call);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return ::gbm::fail(GBM_E_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

#define GBM_TRY(expr)                                                                         \
    do {                                                                                      \
        int rc_ = (expr);                                                                     \
        if (rc_ != GBM_OK)                                                                    \
            return rc_;                                                                       \
    } while (0)

#define GBM_REQUIRE(cond, code, msg)                                                          \
    do {                                                                                      \
        if (!(cond))                                                                          \
            return ::gbm::fail((code), (msg));                                                \
    } while (0)

// device-latched error bits (ctx->dev_err), surfaced by gbm_check
enum : uint32_t { DERR_LABEL = 1u, DERR_OVERFLOW = 2u, DERR_NONFINITE = 4u };

// ------------------------------------------------------------------ scratch arena
// A grow-only device buffer carved into named regions per call.  Reallocation synchronises
// the device (cudaFree), which only happens when a call needs more scratch than before.
struct Arena {
    char *base = nullptr;
    size_t cap = 0, used = 0;
    unsigned generation = 0;  // bumped on every reallocation
    int reserve(size_t bytes);
    void reset() { used = 0; }
    template <class T> T *take(size_t count) {
        size_t off = (used + 255) & ~size_t(255);
        used = off + count * sizeof(T);
        return reinterpret_cast<T *>(base + off);
    }
};

// ------------------------------------------------------------------ profiling
// Optional per-launch CUDA-event timing inside the library (bench.py's roofline): every kernel
// launch site is bracketed by a ProfScope; when profiling is on, two events are recorded on the
// launching stream and the launch's algorithmic bytes are kept as  fixed + rows * bytes_per_row,
// where `rows` is counted on the device (rows_slot) when only the device knows it.
enum ProfCat {
    PC_GRAD_MAX = 0, PC_GRAD_QUANT, PC_HIST_ROOT, PC_HIST_LEVEL, PC_PART_COUNT, PC_PART_SCAN,
    PC_PART_SCATTER, PC_PART_FINAL, PC_EVAL, PC_ALLREDUCE, PC_MARGINS, PC_INIT, PC_PREDICT,
    PC_CUTS, PC_QUANT, PC_EVAL_FINAL, PC_PLAN, PC_PART_DECIDE, PC_N
};
extern const char *const PROF_NAMES[PC_N];

struct ProfRec {
    int cat;
    cudaEvent_t a, b;
    int rows_slot;
    double bytes_per_row, fixed_bytes;
};

struct Prof {
    bool on = false;
    unsigned mask = 0xffffffffu;  // categories recorded (bit = ProfCat)
    std::vector<ProfRec> recs;
    std::vector<cudaEvent_t> pool;
    size_t pool_used = 0;
    unsigned long long *rows_dev = nullptr;  // device row counters, one per launch slot
    int rows_cap = 0, rows_used = 0;
};

}  // namespace gbm

struct gbm_ctx {
    int device = 0;
    int sm_count = 148;
    size_t smem_optin = 227 * 1024;
    ncclComm_t comm = nullptr;
    gbm_vcomm *vcomm = nullptr;    // virtual ranks on one device (comm.cu), instead of NCCL
    long long *agree_d = nullptr;  // coll_agree scratch
    int nranks = 1, rank = 0;
    uint32_t *dev_err = nullptr;   // device-latched error bits
    gbm::Arena arena;              // scratch for the current call
    gbm::Arena tree_arena;         // scratch owned by gbm_build_tree
    gbm::Prof prof;                // optional event timing (gbm_profile_*)
    long long launches = 0;        // kernel launches issued by this context
    int hist_layout = 0;           // GBM_OPT_HIST_LAYOUT: 0 auto, 1 compact, 2 bank-column
    int carry_gradients = 0;       // GBM_OPT_CARRY_GRADIENTS
    int run_tiles = 0;             // GBM_OPT_RUN_TILES (0 = auto)
    int group_units = 0;           // GBM_OPT_GROUP_UNITS (0 = auto = 32)
    int eval_warp = 0;             // GBM_OPT_EVAL_WARP (0 auto, 1 warp per feature, 2 block)
    int eval_screen = 0;           // GBM_OPT_EVAL_SCREEN (1 on, 0 every candidate exactly)
    int seg_hist = 0;              // GBM_OPT_SEGMENT_HIST (0 auto, 1 off, 2 on)
    int stage_tma = 1;             // staged root: TMA bulk row copies (GBM_OPT_TMA_ROWS)
    int row_decide = 0;            // GBM_OPT_ROW_DECIDE (2 on; measured slower, off by default)
    int level_path = 0;            // GBM_OPT_LEVEL_PATH (0 auto, 1 row-index lists, 2 records)
    int level_hist = 0;            // GBM_OPT_LEVEL_HIST (0 auto, 1 compact, 2 shuffle-fed, 3 warp-specialised)
    int eval_sliced = 0;           // GBM_OPT_EVAL_SLICED (1: reduce-scatter + feature-sliced evaluation)
    int cuts_gather = 0;           // GBM_OPT_CUTS_GATHER (1: C3 as an all-gather of X)
    int root_ct = 0;               // GBM_OPT_ROOT_TENSOR (0 auto, 1 off, 2-4 tensor-fed root shapes)
    int level_rep = 1;             // GBM_OPT_LEVEL_REPLICAS (1: replicated low-cardinality bins)
    int walk_mode = 0;             // GBM_OPT_LEAF_WALK (0 auto = staged rows, 1 feature-major copy)
    std::vector<int> tree_groups_key;  // group table currently uploaded in tree_arena
    std::vector<int> tree_slice_key;   // feature-slice tables currently uploaded (sliced evaluation)
    // second stream of gbm_build_tree: the partition scatter of a level overlaps the allreduce
    // and evaluation of that level (fork / join by events; captured as graph edges)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_scan = nullptr, ev_join = nullptr;
};

namespace gbm {

int ctx_enter(gbm_ctx *ctx);  // cudaSetDevice + argument check

// gradients.cu helpers used by the tree builder's fused epilogue fallback
int grad_pass1(gbm_ctx *ctx, int objective, const double *margin_d, const float *label_d, long long n_rows,
               unsigned long long *maxbits, double *sig, cudaStream_t s);
int update_margins_launch(gbm_ctx *ctx, const double *weight_d, const int32_t *row_leaf_d, long long n_rows,
                          double *margin_d, cudaStream_t s);

// device row counter for the next profiled launch (nullptr when profiling is off)
unsigned long long *prof_rows_slot(gbm_ctx *ctx, int *slot);

struct ProfScope {
    gbm_ctx *c;
    int cat, slot;
    cudaStream_t s;
    double bpr, fixed;
    cudaEvent_t a = nullptr;
    ProfScope(gbm_ctx *c_, int cat_, cudaStream_t s_, double fixed_ = 0.0, int slot_ = -1, double bpr_ = 0.0);
    ~ProfScope();
};
int allreduce_i64(gbm_ctx *ctx, long long *buf, size_t count, cudaStream_t s);

// ------------------------------------------------------------------ collectives (comm.cu)
enum CollOp { COLL_SUM_I64 = 0, COLL_MAX_U64 = 1, COLL_MAX_I64 = 2 };
bool coll_on(const gbm_ctx *ctx);  // an NCCL or virtual communicator is attached
int coll_allreduce(gbm_ctx *ctx, void *buf, size_t count, CollOp op, cudaStream_t s);
int coll_allgather(gbm_ctx *ctx, const void *send, void *recv, size_t bytes_per_rank, cudaStream_t s);
int coll_alltoallv_f32(gbm_ctx *ctx, const float *send, const size_t *soff, const size_t *scnt, float *recv,
                       const size_t *roff, const size_t *rcnt, cudaStream_t s);
int coll_reduce_scatter_i64(gbm_ctx *ctx, const long long *send, long long *recv, size_t count_per_rank,
                            cudaStream_t s);
int coll_agree(gbm_ctx *ctx, int local_code, const long long *sig, int nsig, cudaStream_t s, const char *where);

// ------------------------------------------------------------------ packed-matrix access
// The layout of gbm_compress (R3): element (r, f) at stream bit r*stride + f*bits.
struct QM {
    const uint32_t *P;
    long long stride;  // bits per row
    int F, bits, B;    // features, symbol width, sentinel (max_bins)
    int S;             // symbols per unit (a unit spans <= 32 bits)
    int U;             // units per row = ceil(F / S)
    const uint8_t *col;  // optional feature-major symbol copy [F][n]
    long long n;         // rows (column stride of col)
    const uint32_t *dbits = nullptr;  // optional go-left bit per row at its parent (ROW_DECIDE)
};

inline long long row_stride_bits(int F, int bits, int row_align_bits) {
    long long rb = (long long)F * bits;
    if (row_align_bits > 0) rb = (rb + row_align_bits - 1) / row_align_bits * row_align_bits;
    return rb;
}

inline QM make_qm(const gbm_qmatrix *q) {
    QM m;
    m.P = q->packed_d;
    m.F = q->n_features;
    m.bits = q->bits;
    m.B = q->max_bins;
    m.stride = row_stride_bits(q->n_features, q->bits, q->row_align_bits);
    m.S = 32 / q->bits;
    m.U = (q->n_features + m.S - 1) / m.S;
    m.col = q->colsym_d;
    m.n = q->n_rows;
    return m;
}

// nbits (<= 32) stream bits starting at bitpos; the buffer's 4 zero pad words make the
// second word always readable.
__device__ __forceinline__ uint32_t get_bits(const uint32_t *__restrict__ P, long long bitpos,
                                             int nbits) {
    long long w = bitpos >> 5;
    int off = (int)(bitpos & 31);
    uint32_t lo = __ldg(P + w);
    uint64_t v = lo;
    if (off + nbits > 32) v |= (uint64_t)__ldg(P + w + 1) << 32;
    v >>= off;
    return nbits == 32 ? (uint32_t)v : (uint32_t)v & ((1u << nbits) - 1u);
}

__device__ __forceinline__ uint32_t symbol_at(const QM &m, long long row, int f) {
    return get_bits(m.P, row * m.stride + (long long)f * m.bits, m.bits);
}
// symbol of (row, f), from the feature-major copy when present
__device__ __forceinline__ uint32_t split_symbol(const QM &m, long long row, int f) {
    if (m.col) return __ldg(m.col + (long long)f * m.n + row);
    return symbol_at(m, row, f);
}

// exact floor(j / d) for j < 2^32 / d via a 32-bit multiply-high (magic = ceil(2^32 / d))
inline uint32_t div_magic(uint32_t d) { return (uint32_t)(((1ull << 32) + d - 1) / d); }
__device__ __forceinline__ uint32_t fast_div(uint32_t j, uint32_t magic) { return __umulhi(j, magic); }

// ------------------------------------------------------------------ fp64 without contraction
// Every parity-relevant fp64 operation goes through an explicitly rounded intrinsic so that no
// FMA contraction can occur (R20) regardless of compiler flags.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
// exact 2^e as a double, -1022 <= e <= 1023
__device__ __forceinline__ double pow2i(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
// x * 2^e with one correct rounding (== ldexp): a multiply by an exact power of two when 2^e is
// a normal double (the product is then exact or rounded once), scalbn otherwise
__device__ __forceinline__ double ldexp_exact(double x, int e) {
    return (e >= -1022 && e <= 1023) ? __dmul_rn(x, pow2i(e)) : scalbn(x, e);
}
// (double)int64 rounded to nearest even, then the power-of-two scale 2^-s
__device__ __forceinline__ double fixed_to_double(long long v, int s) {
    return ldexp_exact(__ll2double_rn(v), -s);
}

__host__ __device__ inline int ceil_div_i(long long a, long long b) { return (int)((a + b - 1) / b); }

// ---- Eq. 1-2 with the canonical sigmoid (R19): shared by gradients.cu and the fused epilogue of
// the tree builder (tree.cu)
static __constant__ double DE_C[14] = {
    0x1p+0, 0x1p+0, 0x1p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,
    0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22,
    0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33};

// det_exp(t), t <= 0
__device__ __forceinline__ double det_exp(double t) {
    if (t < -745.0) return 0.0;
    double k = rint(dmul(t, 0x1.71547652b82fep+0));
    double r = fma(-k, 0x1.62e42feep-1, t);
    r = fma(-k, 0x1.a39ef35793c76p-33, r);
    double p = DE_C[13];
#pragma unroll
    for (int i = 12; i >= 0; --i) p = fma(p, r, DE_C[i]);
    return ldexp_exact(p, (int)k);
}

// Branch-free over the sign of x (one det_exp per lane, no divergent halves in a warp): both
// cases of R19 take e = det_exp(-|x|); the numerator is 1 for x >= 0, e otherwise.
__device__ __forceinline__ double sigmoid(double x) {
    const double e = det_exp(-fabs(x));
    return ddiv(x >= 0.0 ? 1.0 : e, dadd(1.0, e));
}

// Eq. 1-2 (logistic, from s = sigmoid(margin)) / squared error
__device__ __forceinline__ void grad_hess_s(int obj, double m_or_s, float yl, double &g, double &h) {
    const double y = (double)yl;
    if (obj == GBM_SQUARED_ERROR) {
        g = dsub(m_or_s, y);
        h = 1.0;
        return;
    }
    const double s = m_or_s;
    g = dsub(s, y);
    h = dmul(s, dsub(1.0, s));
}


}  // namespace gbm
