// api.cu -- lifecycle, errors, scratch arena and the NCCL communicator of libgbm.so.
#include <cstdio>
#include <cstring>
#include <string>

#include "gbm_internal.cuh"

namespace gbm {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

int Arena::reserve(size_t bytes) {
    bytes = (bytes + 4095) & ~size_t(4095);
    if (bytes <= cap) {
        used = 0;
        return GBM_OK;
    }
    if (base) {
        cudaError_t e = cudaFree(base);  // synchronises the device: only on growth
        if (e != cudaSuccess) return fail(GBM_E_CUDA, std::string("cudaFree: ") + cudaGetErrorString(e));
        base = nullptr;
        cap = 0;
    }
    size_t want = bytes + bytes / 4;  // head room so a slightly larger next call does not regrow
    cudaError_t e = cudaMalloc(&base, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        e = cudaMalloc(&base, bytes);
        want = bytes;
        if (e != cudaSuccess) {
            cudaGetLastError();
            base = nullptr;
            return fail(GBM_E_NOMEM, "scratch arena: cannot allocate " + std::to_string(bytes) + " bytes");
        }
    }
    cap = want;
    used = 0;
    generation++;
    return GBM_OK;
}

const char *const PROF_NAMES[PC_N] = {
    "grad_max", "grad_quant", "hist_root", "hist_level", "part_count", "part_scan",
    "part_scatter", "part_final", "evaluate", "allreduce", "update_margins", "init_tree",
    "predict", "cuts", "quantise_compress", "eval_final", "plan", "part_decide"};

// Under stream capture an event record must be an EXTERNAL event node to be timed after replays.
static void record(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    if (st == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else cudaEventRecord(e, s);
}

static cudaEvent_t pool_event(Prof &p) {
    if (p.pool_used == p.pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        p.pool.push_back(e);
    }
    return p.pool[p.pool_used++];
}

unsigned long long *prof_rows_slot(gbm_ctx *ctx, int *slot) {
    *slot = -1;
    if (!ctx->prof.on || ctx->prof.rows_used >= ctx->prof.rows_cap) return nullptr;
    *slot = ctx->prof.rows_used++;
    return ctx->prof.rows_dev + *slot;
}

ProfScope::ProfScope(gbm_ctx *c_, int cat_, cudaStream_t s_, double fixed_, int slot_, double bpr_)
    : c(c_), cat(cat_), slot(slot_), s(s_), bpr(bpr_), fixed(fixed_) {
    c->launches += (cat_ == PC_ALLREDUCE) ? 0 : 1;
    if (!c->prof.on || !((c->prof.mask >> cat_) & 1u)) return;
    a = pool_event(c->prof);
    if (a) record(a, s);
}

ProfScope::~ProfScope() {
    if (!a) return;
    cudaEvent_t b = pool_event(c->prof);
    if (!b) return;
    record(b, s);
    c->prof.recs.push_back(ProfRec{cat, a, b, slot, bpr, fixed});
}

int ctx_enter(gbm_ctx *ctx) {
    if (!ctx) return fail(GBM_E_ARG, "null context");
    GBM_CUDA(cudaSetDevice(ctx->device));
    return GBM_OK;
}


}  // namespace gbm

using namespace gbm;

extern "C" {

const char *gbm_last_error(void) { return g_last_error.c_str(); }

int gbm_abi_version(void) { return GBM_ABI_VERSION; }

int gbm_ctx_create(int device, gbm_ctx **out) {
    if (!out) return fail(GBM_E_ARG, "gbm_ctx_create: out is null");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(GBM_E_CUDA, "gbm_ctx_create: no CUDA device available (libgbm has no CPU fallback)");
    }
    if (device < 0 || device >= n) return fail(GBM_E_ARG, "gbm_ctx_create: bad device ordinal");
    GBM_CUDA(cudaSetDevice(device));
    gbm_ctx *c = new gbm_ctx();
    c->device = device;
    cudaDeviceProp prop;
    GBM_CUDA(cudaGetDeviceProperties(&prop, device));
    c->sm_count = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    GBM_CUDA(cudaMalloc(&c->dev_err, sizeof(uint32_t)));
    GBM_CUDA(cudaMemset(c->dev_err, 0, sizeof(uint32_t)));
    GBM_CUDA(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    GBM_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    GBM_CUDA(cudaEventCreateWithFlags(&c->ev_scan, cudaEventDisableTiming));
    GBM_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    *out = c;
    return GBM_OK;
}

int gbm_ctx_destroy(gbm_ctx *ctx) {
    if (!ctx) return GBM_OK;
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    if (ctx->arena.base) cudaFree(ctx->arena.base);
    if (ctx->tree_arena.base) cudaFree(ctx->tree_arena.base);
    if (ctx->dev_err) cudaFree(ctx->dev_err);
    if (ctx->agree_d) cudaFree(ctx->agree_d);
    if (ctx->prof.rows_dev) cudaFree(ctx->prof.rows_dev);
    for (auto e : ctx->prof.pool) cudaEventDestroy(e);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    for (cudaEvent_t e : {ctx->ev_fork, ctx->ev_scan, ctx->ev_join})
        if (e) cudaEventDestroy(e);
    delete ctx;
    return GBM_OK;
}

int gbm_check(gbm_ctx *ctx, void *stream) {
    GBM_TRY(ctx_enter(ctx));
    cudaStream_t s = (cudaStream_t)stream;
    GBM_CUDA(cudaStreamSynchronize(s));
    GBM_CUDA(cudaGetLastError());
    uint32_t bits = 0;
    GBM_CUDA(cudaMemcpy(&bits, ctx->dev_err, sizeof(bits), cudaMemcpyDeviceToHost));
    if (bits) {
        GBM_CUDA(cudaMemset(ctx->dev_err, 0, sizeof(uint32_t)));
        if (bits & DERR_LABEL) return fail(GBM_E_LABEL, "label outside {0,1} under binary:logistic (S:246)");
        if (bits & DERR_OVERFLOW) return fail(GBM_E_OVERFLOW, "symbol does not fit the bit width (S:183)");
        if (bits & DERR_NONFINITE) return fail(GBM_E_NONFINITE, "non-finite feature value (S:32)");
    }
    return GBM_OK;
}

int gbm_comm_unique_id(uint8_t id_h[128]) {
    if (!id_h) return fail(GBM_E_ARG, "gbm_comm_unique_id: null buffer");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    GBM_NCCL(ncclGetUniqueId(&id));
    memcpy(id_h, &id, 128);
    return GBM_OK;
}

int gbm_comm_init(gbm_ctx *ctx, const uint8_t id_h[128], int nranks, int rank) {
    GBM_TRY(ctx_enter(ctx));
    if (!id_h || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(GBM_E_ARG, "gbm_comm_init: bad id / nranks / rank");
    if (ctx->comm || ctx->vcomm) return fail(GBM_E_STATE, "gbm_comm_init: communicator already initialised");
    ncclUniqueId id;
    memcpy(&id, id_h, 128);
    GBM_NCCL(ncclCommInitRank(&ctx->comm, nranks, id, rank));
    ctx->nranks = nranks;
    ctx->rank = rank;
    return GBM_OK;
}

int gbm_comm_info(gbm_ctx *ctx, int *nranks_h, int *rank_h) {
    if (!ctx) return fail(GBM_E_ARG, "null context");
    if (nranks_h) *nranks_h = ctx->nranks;
    if (rank_h) *rank_h = ctx->rank;
    return GBM_OK;
}

int gbm_profile_enable(gbm_ctx *ctx, int enable) {
    GBM_TRY(ctx_enter(ctx));
    Prof &p = ctx->prof;
    GBM_CUDA(cudaDeviceSynchronize());
    p.recs.clear();
    p.pool_used = 0;
    p.rows_used = 0;
    if (enable && !p.rows_dev) {
        p.rows_cap = 1 << 16;
        GBM_CUDA(cudaMalloc(&p.rows_dev, sizeof(unsigned long long) * p.rows_cap));
    }
    if (p.rows_dev) GBM_CUDA(cudaMemset(p.rows_dev, 0, sizeof(unsigned long long) * p.rows_cap));
    p.on = enable != 0;
    p.mask = enable == 1 ? 0xffffffffu : (unsigned)enable;
    return GBM_OK;
}

int gbm_profile_read(gbm_ctx *ctx, gbm_prof_entry *out, int32_t cap, int32_t *n_out) {
    GBM_TRY(ctx_enter(ctx));
    GBM_REQUIRE(out && n_out && cap >= PC_N, GBM_E_ARG, "gbm_profile_read: need room for every category");
    Prof &p = ctx->prof;
    GBM_CUDA(cudaDeviceSynchronize());
    std::vector<unsigned long long> rows(p.rows_used > 0 ? p.rows_used : 1, 0);
    if (p.rows_used > 0)
        GBM_CUDA(cudaMemcpy(rows.data(), p.rows_dev, sizeof(unsigned long long) * p.rows_used, cudaMemcpyDeviceToHost));
    for (int c = 0; c < PC_N; ++c) {
        memset(&out[c], 0, sizeof(gbm_prof_entry));
        strncpy(out[c].name, PROF_NAMES[c], sizeof(out[c].name) - 1);
    }
    for (const ProfRec &r : p.recs) {
        float ms = 0.0f;
        GBM_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
        gbm_prof_entry &e = out[r.cat];
        e.launches += 1;
        e.ms += ms;
        double rw = r.rows_slot >= 0 ? (double)rows[r.rows_slot] : 0.0;
        e.bytes += r.fixed_bytes + rw * r.bytes_per_row;
        e.rows += rw;
    }
    *n_out = PC_N;
    // reset for the next window (keeps profiling on)
    p.recs.clear();
    p.pool_used = 0;
    p.rows_used = 0;
    if (p.rows_dev) GBM_CUDA(cudaMemset(p.rows_dev, 0, sizeof(unsigned long long) * p.rows_cap));
    return GBM_OK;
}

int gbm_profile_zero_rows(gbm_ctx *ctx) {
    GBM_TRY(ctx_enter(ctx));
    Prof &p = ctx->prof;
    GBM_CUDA(cudaDeviceSynchronize());
    if (p.rows_dev) GBM_CUDA(cudaMemset(p.rows_dev, 0, sizeof(unsigned long long) * p.rows_cap));
    return GBM_OK;
}

int64_t gbm_launch_count(gbm_ctx *ctx) { return ctx ? ctx->launches : 0; }

int gbm_set_option(gbm_ctx *ctx, int32_t option, int64_t value) {
    if (!ctx) return fail(GBM_E_ARG, "null context");
    if (option == GBM_OPT_HIST_LAYOUT) {
        if (value < 0 || value > 4)
            return fail(GBM_E_ARG, "GBM_OPT_HIST_LAYOUT: 0 auto, 1 compact, 2 column, 3 staged column, "
                                   "4 staged root + compact levels");
        ctx->hist_layout = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_RUN_TILES) {
        // a work item flushes its int32 shared histogram once: <= MAX_CHUNK (65535) rows per item
        // keeps every bin sum exact (tree.cu header), so at most 31 tiles of 2048 rows
        if (value < 0 || value > 31) return fail(GBM_E_ARG, "GBM_OPT_RUN_TILES: 0 (auto) .. 31");
        ctx->run_tiles = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_GROUP_UNITS) {
        if (value < 0 || value > 32) return fail(GBM_E_ARG, "GBM_OPT_GROUP_UNITS: 0 (auto) .. 32");
        ctx->group_units = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_EVAL_WARP) {
        if (value < 0 || value > 2) return fail(GBM_E_ARG, "GBM_OPT_EVAL_WARP: 0 auto, 1 warp, 2 block");
        ctx->eval_warp = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_SEGMENT_HIST) {
        if (value < 0 || value > 2) return fail(GBM_E_ARG, "GBM_OPT_SEGMENT_HIST: 0 auto, 1 off, 2 on");
        ctx->seg_hist = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_TMA_ROWS) {
        ctx->stage_tma = value != 0;
        return GBM_OK;
    }
    if (option == GBM_OPT_EVAL_SCREEN) {
        ctx->eval_screen = value != 0;
        return GBM_OK;
    }
    if (option == GBM_OPT_LEAF_WALK) {
        if (value < 0 || value > 1) return fail(GBM_E_ARG, "GBM_OPT_LEAF_WALK: 0 auto, 1 feature-major copy");
        ctx->walk_mode = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_ROOT_TENSOR) {
        if (value < 0 || value > 7)
            return fail(GBM_E_ARG, "GBM_OPT_ROOT_TENSOR: 0 auto, 1 off, 2-7 always (warps x stages x tile rows: "
                                   "16x2x32, 12x3x32, 8x4x32, 8x2x64, 16x2x64, 16x2x128)");
        ctx->root_ct = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_LEVEL_REPLICAS) {
        if (value < 0 || value > 1) return fail(GBM_E_ARG, "GBM_OPT_LEVEL_REPLICAS: 1 on (default), 0 off");
        ctx->level_rep = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_CUTS_GATHER) {
        if (value < 0 || value > 1) return fail(GBM_E_ARG, "GBM_OPT_CUTS_GATHER: 0 per-feature ownership, 1 all-gather");
        ctx->cuts_gather = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_EVAL_SLICED) {
        if (value < 0 || value > 1) return fail(GBM_E_ARG, "GBM_OPT_EVAL_SLICED: 0 off, 1 on");
        ctx->eval_sliced = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_LEVEL_HIST) {
        if (value < 0 || value > 3)
            return fail(GBM_E_ARG, "GBM_OPT_LEVEL_HIST: 0 auto, 1 compact, 2 bank-column, 3 warp-specialised compact");
        ctx->level_hist = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_LEVEL_PATH) {
        if (value < 0 || value > 2) return fail(GBM_E_ARG, "GBM_OPT_LEVEL_PATH: 0 auto, 1 row-index lists, 2 records");
        ctx->level_path = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_ROW_DECIDE) {
        if (value < 0 || value > 2) return fail(GBM_E_ARG, "GBM_OPT_ROW_DECIDE: 0/1 off (default), 2 on");
        ctx->row_decide = (int)value;
        return GBM_OK;
    }
    if (option == GBM_OPT_CARRY_GRADIENTS) {
        ctx->carry_gradients = value != 0;
        return GBM_OK;
    }
    return fail(GBM_E_ARG, "gbm_set_option: unknown option");
}

int gbm_symbol_bits(int32_t max_symbol) {
    if (max_symbol < 0) return fail(GBM_E_ARG, "gbm_symbol_bits: negative max_symbol");
    int b = 1;
    while (b < 31 && (1ll << b) <= (long long)max_symbol) b++;
    return b;
}

int64_t gbm_packed_words(int64_t n_rows, int32_t n_features, int32_t bits, int32_t row_align_bits) {
    if (n_rows < 0 || n_features <= 0 || bits < 1 || bits > 16)
        return fail(GBM_E_ARG, "gbm_packed_words: bad sizes");
    if (row_align_bits != 0 && row_align_bits != 32 && row_align_bits != 128 && row_align_bits != 256)
        return fail(GBM_E_ARG, "gbm_packed_words: row_align_bits must be 0, 32, 128 or 256");
    long long total = n_rows * row_stride_bits(n_features, bits, row_align_bits);
    long long w = (total + 31) / 32;
    w = (w + 3) / 4 * 4;
    return w + 4;
}

}  // extern "C"
