// comm.cu -- the collectives of libgbm: C1 the global gradient maxima,
// C2 AllReduceHistograms, C3 the global cuts' all-gather, and the collective agreement every
// rank reaches before a tree (GBM_E_MISMATCH).  Two backends behind one interface:
//
//  * NCCL (gbm_comm_init): one process per GPU, the product path.
//  * virtual (gbm_comm_init_virtual): p contexts on ONE device, one host thread per rank, joined
//    by an in-process gbm_vcomm.  Each collective synchronises the callers' streams, meets at a
//    host barrier, and rank 0 reduces / gathers the posted device buffers into shared scratch
//    that every rank then copies back.  It is the test harness that runs libgbm's own multi-rank
//    code -- shard contexts packed from bit 0, per-rank partial histograms summed, global maxima,
//    global cuts over the concatenated shards -- on a single GPU (SURVEY §4 "virtual shards").
//    Not capturable into CUDA graphs (host barriers); correctness only.
#include <climits>
#include <condition_variable>
#include <mutex>
#include <vector>

#include "gbm_internal.cuh"

struct gbm_vcomm {
    int nranks = 1;
    int device = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    std::vector<const void *> posted;
    std::vector<const size_t *> posted_off;  // all-to-all: each rank's per-destination offsets
    void *scratch = nullptr;
    size_t scratch_bytes = 0;
    int err = GBM_OK;  // rank 0's result of the current collective, read by every rank
};

namespace gbm {

constexpr int VC_MAX = 64;

static void vc_barrier(gbm_vcomm *v) {
    std::unique_lock<std::mutex> l(v->mu);
    const unsigned long long g = v->gen;
    if (++v->arrived == v->nranks) {
        v->arrived = 0;
        v->gen++;
        v->cv.notify_all();
    } else {
        v->cv.wait(l, [&] { return v->gen != g; });
    }
}

struct VcPtrs {
    const void *p[VC_MAX];
};

__global__ void vc_reduce_kernel(VcPtrs src, int nranks, size_t count, int op, void *dst) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        if (op == COLL_SUM_I64) {
            long long s = 0;
            for (int r = 0; r < nranks; ++r) s += static_cast<const long long *>(src.p[r])[i];
            static_cast<long long *>(dst)[i] = s;
        } else if (op == COLL_MAX_U64) {
            unsigned long long m = 0;
            for (int r = 0; r < nranks; ++r) m = max(m, static_cast<const unsigned long long *>(src.p[r])[i]);
            static_cast<unsigned long long *>(dst)[i] = m;
        } else {
            long long m = LLONG_MIN;
            for (int r = 0; r < nranks; ++r) m = max(m, static_cast<const long long *>(src.p[r])[i]);
            static_cast<long long *>(dst)[i] = m;
        }
    }
}

static int vc_scratch(gbm_vcomm *v, size_t bytes) {
    if (v->scratch_bytes >= bytes) return GBM_OK;
    if (v->scratch) cudaFree(v->scratch);
    v->scratch = nullptr;
    v->scratch_bytes = 0;
    GBM_CUDA(cudaMalloc(&v->scratch, bytes));
    v->scratch_bytes = bytes;
    return GBM_OK;
}

static bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    return st != cudaStreamCaptureStatusNone;
}

// One virtual collective: every rank posts `send`; rank 0 runs `work` (reduce / gather into the
// scratch); every rank then copies `out_bytes` of scratch into `recv`.  Three barriers: posted,
// scratch ready, copies done (so the next collective may reuse the scratch).
template <class Work>
static int vc_collective(gbm_ctx *ctx, const void *send, void *recv, size_t out_bytes, cudaStream_t s, Work work) {
    gbm_vcomm *v = ctx->vcomm;
    if (capturing(s)) return fail(GBM_E_STATE, "virtual communicator: collectives cannot be graph-captured");
    GBM_CUDA(cudaStreamSynchronize(s));
    v->posted[ctx->rank] = send;
    vc_barrier(v);
    if (ctx->rank == 0) {
        v->err = vc_scratch(v, std::max<size_t>(out_bytes, 16));
        if (v->err == GBM_OK) v->err = work(v);
        if (v->err == GBM_OK && cudaDeviceSynchronize() != cudaSuccess) v->err = GBM_E_CUDA;
    }
    vc_barrier(v);
    const int err = v->err;
    if (err == GBM_OK && out_bytes) {
        GBM_CUDA(cudaMemcpyAsync(recv, v->scratch, out_bytes, cudaMemcpyDeviceToDevice, s));
        GBM_CUDA(cudaStreamSynchronize(s));
    }
    vc_barrier(v);
    return err == GBM_OK ? GBM_OK : fail(err, "virtual collective failed on rank 0");
}

bool coll_on(const gbm_ctx *ctx) { return ctx->comm != nullptr || ctx->vcomm != nullptr; }

int coll_allreduce(gbm_ctx *ctx, void *buf, size_t count, CollOp op, cudaStream_t s) {
    if (!coll_on(ctx) || count == 0) return GBM_OK;
    if (ctx->comm) {
        const ncclDataType_t t = op == COLL_MAX_U64 ? ncclUint64 : ncclInt64;
        const ncclRedOp_t o = op == COLL_SUM_I64 ? ncclSum : ncclMax;
        GBM_NCCL(ncclAllReduce(buf, buf, count, t, o, ctx->comm, s));
        return GBM_OK;
    }
    return vc_collective(ctx, buf, buf, count * 8, s, [&](gbm_vcomm *v) -> int {
        VcPtrs p = {};
        for (int r = 0; r < v->nranks; ++r) p.p[r] = v->posted[r];
        vc_reduce_kernel<<<256, 256>>>(p, v->nranks, count, (int)op, v->scratch);
        return cudaGetLastError() == cudaSuccess ? GBM_OK : GBM_E_CUDA;
    });
}

int coll_allgather(gbm_ctx *ctx, const void *send, void *recv, size_t bytes, cudaStream_t s) {
    if (!coll_on(ctx)) {
        if (bytes) GBM_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
        return GBM_OK;
    }
    if (ctx->comm) {
        GBM_NCCL(ncclAllGather(send, recv, bytes, ncclUint8, ctx->comm, s));
        return GBM_OK;
    }
    return vc_collective(ctx, send, recv, bytes * ctx->nranks, s, [&](gbm_vcomm *v) -> int {
        for (int r = 0; r < v->nranks; ++r)
            if (bytes && cudaMemcpy(static_cast<char *>(v->scratch) + (size_t)r * bytes, v->posted[r], bytes,
                                    cudaMemcpyDeviceToDevice) != cudaSuccess)
                return GBM_E_CUDA;
        return GBM_OK;
    });
}

// All-to-all of float pieces: this rank sends scnt[d] floats at send + soff[d] to rank d and
// receives rcnt[q] floats from rank q at recv + roff[q] (host arrays of p entries; C3 of the
// per-feature cut ownership).  NCCL: grouped ncclSend / ncclRecv.
int coll_alltoallv_f32(gbm_ctx *ctx, const float *send, const size_t *soff, const size_t *scnt, float *recv,
                       const size_t *roff, const size_t *rcnt, cudaStream_t s) {
    const int p = ctx->nranks, me = ctx->rank;
    if (!coll_on(ctx) || p == 1) {
        if (scnt[0]) GBM_CUDA(cudaMemcpyAsync(recv + roff[0], send + soff[0], scnt[0] * 4, cudaMemcpyDeviceToDevice, s));
        return GBM_OK;
    }
    if (ctx->comm) {
        GBM_NCCL(ncclGroupStart());
        for (int q = 0; q < p; ++q) {
            if (scnt[q]) GBM_NCCL(ncclSend(send + soff[q], scnt[q], ncclFloat32, q, ctx->comm, s));
            if (rcnt[q]) GBM_NCCL(ncclRecv(recv + roff[q], rcnt[q], ncclFloat32, q, ctx->comm, s));
        }
        GBM_NCCL(ncclGroupEnd());
        return GBM_OK;
    }
    // virtual: every rank posts its send buffer and offsets, then copies its pieces from the peers'
    gbm_vcomm *v = ctx->vcomm;
    if (capturing(s)) return fail(GBM_E_STATE, "virtual communicator: collectives cannot be graph-captured");
    GBM_CUDA(cudaStreamSynchronize(s));
    v->posted[me] = send;
    v->posted_off[me] = soff;
    vc_barrier(v);
    int err = GBM_OK;
    for (int q = 0; q < p && err == GBM_OK; ++q)
        if (rcnt[q] && cudaMemcpyAsync(recv + roff[q], static_cast<const float *>(v->posted[q]) + v->posted_off[q][me],
                                       rcnt[q] * 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            err = GBM_E_CUDA;
    if (cudaStreamSynchronize(s) != cudaSuccess) err = GBM_E_CUDA;
    vc_barrier(v);  // the peers' buffers may be released after this
    return err == GBM_OK ? GBM_OK : fail(err, "virtual all-to-all failed");
}

// Sum of every rank's send[p][count] (int64) with chunk r delivered to rank r's recv[count]
// (ncclReduceScatter; the reduce-scatter + feature-sliced evaluation variant of C2).
int coll_reduce_scatter_i64(gbm_ctx *ctx, const long long *send, long long *recv, size_t count, cudaStream_t s) {
    if (!coll_on(ctx)) {
        if (count) GBM_CUDA(cudaMemcpyAsync(recv, send, count * 8, cudaMemcpyDeviceToDevice, s));
        return GBM_OK;
    }
    if (ctx->comm) {
        GBM_NCCL(ncclReduceScatter(send, recv, count, ncclInt64, ncclSum, ctx->comm, s));
        return GBM_OK;
    }
    // virtual: rank 0 sums the posted [p][count] buffers into scratch; rank r copies chunk r
    gbm_vcomm *v = ctx->vcomm;
    if (capturing(s)) return fail(GBM_E_STATE, "virtual communicator: collectives cannot be graph-captured");
    GBM_CUDA(cudaStreamSynchronize(s));
    v->posted[ctx->rank] = send;
    vc_barrier(v);
    const size_t total = count * v->nranks;
    if (ctx->rank == 0) {
        v->err = vc_scratch(v, std::max<size_t>(total * 8, 16));
        if (v->err == GBM_OK && total) {
            VcPtrs p = {};
            for (int r = 0; r < v->nranks; ++r) p.p[r] = v->posted[r];
            vc_reduce_kernel<<<256, 256>>>(p, v->nranks, total, (int)COLL_SUM_I64, v->scratch);
            if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) v->err = GBM_E_CUDA;
        }
    }
    vc_barrier(v);
    const int err = v->err;
    if (err == GBM_OK && count) {
        GBM_CUDA(cudaMemcpyAsync(recv, static_cast<const long long *>(v->scratch) + count * ctx->rank, count * 8,
                                 cudaMemcpyDeviceToDevice, s));
        GBM_CUDA(cudaStreamSynchronize(s));
    }
    vc_barrier(v);
    return err == GBM_OK ? GBM_OK : fail(err, "virtual reduce-scatter failed on rank 0");
}

// The decision every rank must share before a collective call sequence: the first
// nonzero local error code of any rank, or GBM_E_MISMATCH when the ranks' signatures (sizes
// that must be equal everywhere, e.g. F, TB, bits) differ, is returned on EVERY rank, so no rank
// enters a collective its peers skip.  One int64 max-allreduce of [error?, -code, sig, -sig];
// skipped inside a graph capture (the eager calls before the capture ran it).
int coll_agree(gbm_ctx *ctx, int local_code, const long long *sig, int nsig, cudaStream_t s, const char *where) {
    if (!coll_on(ctx) || ctx->nranks <= 1 || capturing(s)) return local_code;
    const int n = 2 + 2 * nsig;
    std::vector<long long> h(n);
    h[0] = local_code != GBM_OK ? 1 : 0;
    h[1] = -(long long)local_code;
    for (int i = 0; i < nsig; ++i) {
        h[2 + i] = sig[i];
        h[2 + nsig + i] = -sig[i];
    }
    if (!ctx->agree_d) GBM_CUDA(cudaMalloc(&ctx->agree_d, 64 * sizeof(long long)));
    if (n > 64) return fail(GBM_E_ARG, "coll_agree: signature too long");
    GBM_CUDA(cudaMemcpyAsync(ctx->agree_d, h.data(), n * sizeof(long long), cudaMemcpyHostToDevice, s));
    GBM_TRY(coll_allreduce(ctx, ctx->agree_d, n, COLL_MAX_I64, s));
    GBM_CUDA(cudaMemcpyAsync(h.data(), ctx->agree_d, n * sizeof(long long), cudaMemcpyDeviceToHost, s));
    GBM_CUDA(cudaStreamSynchronize(s));
    if (h[0]) {
        if (local_code != GBM_OK) return local_code;  // this rank's own message is in gbm_last_error
        return fail((int)-h[1], std::string(where) + ": another rank failed (code " + std::to_string(-h[1]) + ")");
    }
    for (int i = 0; i < nsig; ++i)
        if (h[2 + i] != -h[2 + nsig + i])
            return fail(GBM_E_MISMATCH, std::string(where) + ": ranks disagree on argument " + std::to_string(i) +
                                            " (e.g. features, total bins, symbol bits, row alignment; S:348)");
    return GBM_OK;
}

int allreduce_i64(gbm_ctx *ctx, long long *buf, size_t count, cudaStream_t s) {
    return coll_allreduce(ctx, buf, count, COLL_SUM_I64, s);
}

}  // namespace gbm

using namespace gbm;

extern "C" {

int gbm_vcomm_create(int nranks, gbm_vcomm **out) {
    if (!out || nranks < 1 || nranks > VC_MAX) return fail(GBM_E_ARG, "gbm_vcomm_create: nranks in 1..64");
    gbm_vcomm *v = new gbm_vcomm();
    v->nranks = nranks;
    v->posted.assign(nranks, nullptr);
    v->posted_off.assign(nranks, nullptr);
    cudaGetDevice(&v->device);
    *out = v;
    return GBM_OK;
}

int gbm_vcomm_destroy(gbm_vcomm *v) {
    if (!v) return GBM_OK;
    if (v->scratch) cudaFree(v->scratch);
    delete v;
    return GBM_OK;
}

int gbm_comm_init_virtual(gbm_ctx *ctx, gbm_vcomm *v, int rank) {
    GBM_TRY(ctx_enter(ctx));
    if (!v || rank < 0 || rank >= v->nranks) return fail(GBM_E_ARG, "gbm_comm_init_virtual: bad communicator / rank");
    if (ctx->comm || ctx->vcomm) return fail(GBM_E_STATE, "gbm_comm_init_virtual: communicator already initialised");
    ctx->vcomm = v;
    ctx->nranks = v->nranks;
    ctx->rank = rank;
    return GBM_OK;
}

}  // extern "C"
