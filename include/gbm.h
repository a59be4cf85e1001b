/*
 * gbm.h -- C-ABI of libgbm.so, the B200 (sm_100a) hot path of multi-GPU histogram gradient
 * boosting (arXiv 1806.11248, "XGBoost: Scalable GPU Accelerated Learning").
 *
 * Citations: P:nn = PAPER.md line nn (section), S:nn = SPEC.md line nn, R# = reading number in
 * DESIGN.md "Readings of the paper".
 *
 * Conventions (apply to every entry point):
 *  - Pointers suffixed _d are DEVICE pointers on the context's device, _h are HOST pointers.
 *    The caller owns every buffer passed in (allocates, frees, keeps it alive for the call and
 *    for all work the call enqueued); the library never retains a caller pointer after a call
 *    returns.  Device buffers must be 16-byte aligned and contiguous.
 *  - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).  All work is
 *    enqueued on it, asynchronously, unless an entry says it synchronises.
 *  - Every function returns GBM_OK (0) or a negative GBM_E_* code and never throws; the message
 *    of the last failure on the calling thread is gbm_last_error().  Argument checks happen
 *    before anything is enqueued.  Errors detected ON the device (a label outside {0,1} under
 *    the logistic objective) are latched in the context and returned by the next gbm_check.
 *  - A context is bound to one device, owns a scratch arena and (optionally) an NCCL
 *    communicator, and is not thread-safe.  One context per (process, device).
 *  - "Collective": with a communicator of nranks > 1 every rank must make the same call in the
 *    same order (NCCL semantics).  Rank k owns rows [floor(k n/p), floor((k+1) n/p)) (R18).
 *  - No CPU fallback exists: without a CUDA device every compute entry fails with GBM_E_CUDA.
 */
#ifndef GBM_H
#define GBM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GBM_ABI_VERSION 2

#if defined(__GNUC__)
#define GBM_API __attribute__((visibility("default")))
#else
#define GBM_API
#endif

enum {
    GBM_OK = 0,
    GBM_E_ARG = -1,       /* invalid argument (null pointer, size, enum, alignment)         */
    GBM_E_EMPTY = -2,     /* zero rows                                        */
    GBM_E_OVERFLOW = -3,  /* symbol does not fit the bit width                       */
    GBM_E_LABEL = -4,     /* label outside {0,1} under binary:logistic               */
    GBM_E_NONFINITE = -5, /* +-inf feature value                                      */
    GBM_E_MISMATCH = -6,  /* ranks disagree on sizes                                 */
    GBM_E_STATE = -7,     /* call not valid in the context's state (e.g. no communicator)    */
    GBM_E_CUDA = -10,     /* CUDA runtime error or no device                                 */
    GBM_E_NCCL = -11,     /* NCCL error                                                      */
    GBM_E_NOMEM = -12     /* device or host allocation failed                                */
};

enum { GBM_SQUARED_ERROR = 0, GBM_LOGISTIC = 1 };   /* objectives */
enum { GBM_NODE_ABSENT = 0, GBM_NODE_SPLIT = 1, GBM_NODE_LEAF = 2 };
enum { GBM_GROW_DEPTHWISE = 0, GBM_GROW_LOSSGUIDE = 1 };  /* tree growth policies      */

typedef struct gbm_ctx gbm_ctx;

/* ---------------------------------------------------------------- lifecycle, errors */
GBM_API const char *gbm_last_error(void);   /* thread-local; valid until the next gbm_* call     */
GBM_API int gbm_abi_version(void);          /* == GBM_ABI_VERSION                                  */
GBM_API int gbm_ctx_create(int device, gbm_ctx **out);
GBM_API int gbm_ctx_destroy(gbm_ctx *ctx);  /* frees scratch and the communicator; NULL is a no-op */
/* Synchronises `stream` and reports asynchronous failures (CUDA errors and device-detected
 * argument errors such as GBM_E_LABEL) latched since the last gbm_check. */
GBM_API int gbm_check(gbm_ctx *ctx, void *stream);

/* ---------------------------------------------------------------- instrumentation
 * Optional CUDA-event timing of every kernel launch the context issues, grouped by kernel
 * (bench.py's per-kernel roofline).  gbm_profile_enable(1) resets and starts recording every
 * category; any other non-zero value is a bitmask of the categories to record (bit i = entry i
 * of gbm_profile_read); 0 stops.  It synchronises the device.  Launches captured into a CUDA
 * graph record their events as graph nodes: after replays, ms are those of the last replay while
 * the device row counters (hence bytes, rows) accumulate over every replay.
 * gbm_profile_read synchronises, fills one entry per kernel
 * category (cap >= 32) and starts a new window.  bytes = the launches' ALGORITHMIC bytes
 * (DESIGN.md "Algorithmic bytes"), rows = rows they processed, counted on the device.
 * gbm_launch_count: kernel launches issued by the context since creation. */
typedef struct {
    char name[32];
    int64_t launches;
    double ms;
    double bytes;
    double rows;
} gbm_prof_entry;
GBM_API int gbm_profile_enable(gbm_ctx *ctx, int enable);
GBM_API int gbm_profile_read(gbm_ctx *ctx, gbm_prof_entry *out, int32_t cap, int32_t *n_out);
/* Zero the device counters of algorithmic bytes but keep the timing records (e.g. of the event
 * nodes of a captured CUDA graph): start a measurement window after warm-up replays. */
GBM_API int gbm_profile_zero_rows(gbm_ctx *ctx);
GBM_API int64_t gbm_launch_count(gbm_ctx *ctx);

/* Tuning options (do not change results, only which kernels compute them).
 * GBM_OPT_HIST_LAYOUT: shared-memory histogram layout of BuildPartialHistograms --
 *   0 auto (staged bank-column root for large matrices, compact levels), 1 compact (random
 *   bins, bank conflicts), 2 bank-column (feature per lane, conflict-free; falls back to
 *   compact when the bins do not fit), 3 staged bank-column everywhere, 4 staged root whatever
 *   the size + compact levels.
 * GBM_OPT_CARRY_GRADIENTS: 0 (default) level passes gather qpair by row; 1 the row-index
 *   entries of every level carry the row's gradient pair (grad_bits <= 15; 8-byte entries).
 * GBM_OPT_RUN_TILES: 2048-row tiles per work item of the fused level kernel (0 = auto, 1..31:
 *   one int32 shared-memory flush per item must stay within 65535 rows).
 * GBM_OPT_GROUP_UNITS: at most this many packed units (S features each) per shared-memory
 *   feature group of the compact layout (0 = auto = 32; 1..32).  Smaller groups mean less
 *   shared memory per block (more resident blocks) but more passes over the row list.
 * GBM_OPT_EVAL_WARP: EvaluateSplit with one warp per (node, feature), 8 bins per lane (1), or
 *   one block per (node, feature), one bin per thread (2); 0 (default) = warps when there are
 *   at least 16 per SM, else blocks.
 * GBM_OPT_LEAF_WALK: final-level leaf assignment of a depth-wise tree: 0 (default) rows of whole
 *   words staged through shared memory in row order; 1 the feature-major symbol copy.
 * GBM_OPT_EVAL_SCREEN: 1 EvaluateSplit computes the exact gain (two IEEE divisions) only for
 *   candidates that pass an approximate screen proven never to drop the exact argmax or a tie
 *   with it (tree.cu, screen_score); 0 (default: measured faster, the evaluation is bound by
 *   memory and latency, not by the divisions) evaluates every candidate exactly.  Results are
 *   identical either way.
 * GBM_OPT_SEGMENT_HIST: with several shared-memory feature groups (wide data): 2 = each level
 *   is partitioned once and the built children's row segments are histogrammed group by group;
 *   1 = the fused kernel repeats the partition in every group; 0 (default) = 2 for symbols
 *   wider or narrower than a byte, else 1 (measured).
 * GBM_OPT_TMA_ROWS: 1 (default) the staged root kernel fetches whole 32-row batches with TMA bulk
 *   copies (cp.async.bulk + mbarrier, double-buffered) when one group covers every word of a
 *   row; 0 = per-lane loads.
 * GBM_OPT_ROW_DECIDE: depth-wise levels 1..D-1 of RepartitionInstances: 2 = a row-order
 *   pass walks every row's staged packed row down the tree built so far and writes its
 *   go-left decision at its parent as one bit per row (n/8 bytes, L2-resident), which the fused
 *   partition + histogram kernel then reads instead of gathering the split symbol from DRAM;
 *   applies to rows of whole words (<= 16 words) and max_depth <= 12; 0 (default) and 1 = the
 *   split symbol is gathered per row (measured faster: the extra streaming pass costs more than
 *   the gathers it removes).  Same decisions either way.
 * GBM_OPT_LEVEL_PATH: depth-wise levels 1..D-1.  2 = records: every level streams its
 *   parents' rows (packed row words + gradient pair, grouped by node; level 1 reads the packed
 *   matrix and qpair) by TMA bulk copies, decides each row's side from the staged split symbol,
 *   accumulates the smaller child into a conflict-free shared histogram, and moves every row into
 *   its child's segment of a second buffer (2 x n x (row bytes + 8) of scratch); applies to
 *   8-bit symbols, <= 32 features, rows of whole words.  1 = row-index lists (partition flags +
 *   scan + scatter of row ids; packed rows and qpair gathered per level).  0 (default) = 1
 *   (measured faster end to end).  Same trees either way.
 * GBM_OPT_LEVEL_HIST: the shared-memory histogram of the row-index level kernel.  1 = compact
 *   (bins of all features packed; lane = (row, packed word), random-bank atomics); 2 =
 *   bank-column (lane = feature, word = bin * 32 + lane: conflict-free atomics, the row's words
 *   moved to the feature lanes by warp shuffles; byte symbols, <= 32 features, whole-word rows);
 *   0 (default) = 1 (measured faster: the shuffles cost more issue slots than the bank conflicts
 *   they remove).  Same histograms either way.
 * GBM_OPT_EVAL_SLICED: with a communicator of p > 1 ranks, depth-wise trees:
 *   1 = AllReduceHistograms becomes a reduce-scatter: rank r receives only the summed bins of its
 *   contiguous feature slice (features balanced by bins), evaluates those features, and the ranks
 *   all-gather their per-(node, feature) best candidates before the replicated node reduction --
 *   half the collective bytes per rank and 1/p of the evaluation; 0 (default) = allreduce.  Same
 *   trees either way (exact sums, canonical argmax).
 * GBM_OPT_CUTS_GATHER: gbm_cuts with several ranks (C3).  0 (default) = per-feature ownership:
 *   feature f belongs to rank f mod p, the ranks exchange their shards' columns (all-to-all), each
 *   owner cuts its features over the global rows and the cuts are all-gathered -- O(n F / p) per
 *   rank; 1 = all-gather every shard's X to every rank (O(n F) per rank).  Same cuts either way.
 * GBM_OPT_ROOT_TENSOR: the root histogram of byte-symbol matrices with the feature-major copy
 *   (gbm_transpose_symbols) and n a multiple of 16: every warp fetches a [features x TR rows]
 *   tile of that copy with one TMA tensor copy and lane f holds its feature's symbols in
 *   registers (root_ct.cu); 1 = the staged packed rows; 2-7 = the tensor-fed root with (warps x
 *   stages x TR) 16x2x32, 12x3x32, 8x4x32, 8x2x64, 16x2x64, 16x2x128; 0 (default) = 2 with several
 *   feature groups (> 32 features) or <= 16 features, 6 for one group of 17..32 features
 *   (measured).  Same histogram.
 * GBM_OPT_LEVEL_REPLICAS: 1 (default) = the fused level histogram of byte symbols keeps R <= 8
 *   copies of the bins of each feature with few bins (R x bins <= 128), row slot r adding into
 *   copy r mod R, folded before the flush: lanes hitting one bin of a low-cardinality feature no
 *   longer serialise on one shared-memory word; 0 = one copy.  Same histogram. */
enum { GBM_OPT_HIST_LAYOUT = 1, GBM_OPT_CARRY_GRADIENTS = 2, GBM_OPT_RUN_TILES = 3, GBM_OPT_GROUP_UNITS = 4,
       GBM_OPT_EVAL_WARP = 5, GBM_OPT_LEAF_WALK = 6, GBM_OPT_EVAL_SCREEN = 7, GBM_OPT_SEGMENT_HIST = 8,
       GBM_OPT_TMA_ROWS = 10, GBM_OPT_ROW_DECIDE = 11, GBM_OPT_LEVEL_PATH = 12, GBM_OPT_LEVEL_HIST = 13,
       GBM_OPT_EVAL_SLICED = 14, GBM_OPT_CUTS_GATHER = 15, GBM_OPT_ROOT_TENSOR = 16,
       GBM_OPT_LEVEL_REPLICAS = 17 };
GBM_API int gbm_set_option(gbm_ctx *ctx, int32_t option, int64_t value);

/* ---------------------------------------------------------------- communicator
 * Rank 0 calls gbm_comm_unique_id and broadcasts the 128 bytes with its own process group
 * (the Python binding uses torch.distributed); then every rank calls gbm_comm_init
 * (collective; blocks until all ranks joined).  nranks == 1 is allowed.  Without a
 * communicator every entry behaves as a single rank. */
GBM_API int gbm_comm_unique_id(uint8_t id_h[128]);
GBM_API int gbm_comm_init(gbm_ctx *ctx, const uint8_t id_h[128], int nranks, int rank);
GBM_API int gbm_comm_info(gbm_ctx *ctx, int *nranks_h, int *rank_h);

/* Virtual ranks (test harness for the multi-rank path on ONE GPU): a gbm_vcomm joins
 * nranks contexts of one process on one device, each driven by its own host thread and stream.
 * gbm_comm_init_virtual attaches ctx as `rank`; afterwards every collective entry (gbm_cuts C3,
 * gbm_gradients C1, gbm_build_tree C2 and its argument agreement) exchanges through the vcomm
 * exactly where it would call NCCL: the callers' streams are synchronised, the ranks meet at a
 * host barrier, rank 0 sums (int64) / takes the max / gathers the posted device buffers, and
 * every rank copies the result back.  Results equal NCCL's (integer sums and maxima are exact).
 * Not usable inside CUDA graph capture (GBM_E_STATE).  The vcomm is owned by the caller and
 * must outlive its contexts' last collective call.  nranks in 1..64.
 * Errors: GBM_E_ARG (bad nranks / rank), GBM_E_STATE (ctx already has a communicator). */
typedef struct gbm_vcomm gbm_vcomm;
GBM_API int gbm_vcomm_create(int nranks, gbm_vcomm **out);
GBM_API int gbm_vcomm_destroy(gbm_vcomm *vc);
GBM_API int gbm_comm_init_virtual(gbm_ctx *ctx, gbm_vcomm *vc, int rank);

/* ---------------------------------------------------------------- §2.1 quantiles
 * gbm_cuts: exact per-feature cut points over the GLOBAL rows (collective: the ranks'
 * shards are all-gathered).  Rule R5: with V the sorted present values of a
 * feature (m of them, d distinct) the cuts are the distinct values if d <= max_bins, else
 * dedup(V[floor((j+1) m / max_bins) - 1], j = 0..max_bins-1).  NaN = missing; -0.0 counts as
 * +0.0.
 *   X_d          fp32 [n_rows][n_features] row-major, this rank's shard
 *   cut_values_d fp32 [n_features * max_bins] (capacity), written compactly
 *   cut_ptr_d    int32 [n_features + 1], exclusive prefix sum of per-feature bin counts
 *   n_cuts_h     total bins TB = cut_ptr[F]
 *   max_symbol_h the largest symbol gbm_quantise will store for these rows: max_bins if any
 *                value (on any rank) is missing, else max_f(n_bins(f)) - 1 (R4)
 * Synchronises `stream` (the sizes are returned on the host).  Errors: GBM_E_EMPTY (no
 * rows on every rank), GBM_E_NONFINITE (+-inf), GBM_E_ARG (max_bins < 2 or > 65535). */
GBM_API int gbm_cuts(gbm_ctx *ctx, const float *X_d, int64_t n_rows, int32_t n_features,
             int32_t max_bins, float *cut_values_d, int32_t *cut_ptr_d, int32_t *n_cuts_h,
             int32_t *max_symbol_h, void *stream);

/* gbm_quantise: bin map (R6/R7): bins[i][f] = max_bins (the missing sentinel) if
 * X[i][f] is NaN (or the feature has no cuts), else the smallest k with X[i][f] <=
 * cuts_f[k], clamped to n_bins(f)-1.  bins_d uint16 [n_rows][n_features].  Asynchronous. */
GBM_API int gbm_quantise(gbm_ctx *ctx, const float *X_d, int64_t n_rows, int32_t n_features,
                 int32_t max_bins, const float *cut_values_d, const int32_t *cut_ptr_d,
                 uint16_t *bins_d, void *stream);

/* ---------------------------------------------------------------- §2.2 compression
 * symbol width (R1): max(1, ceil(log2(max_symbol + 1))).  Pure, host only. */
GBM_API int gbm_symbol_bits(int32_t max_symbol);
/* packed buffer size in uint32 words for the layout of gbm_compress (R3): element (r, f)
 * starts at bit r*stride + f*bits, stride = n_features*bits rounded up to row_align_bits
 * (0, 32, 128 or 256; 0 = SPEC's continuous stream; 256 = one 32-byte DRAM sector, so a
 * gathered row of <= 32 bytes touches one sector); ceil(n*stride/32) words rounded up to a
 * multiple of 4, plus 4 zero words.  Returns a negative GBM_E_* on bad arguments. */
GBM_API int64_t gbm_packed_words(int64_t n_rows, int32_t n_features, int32_t bits,
                         int32_t row_align_bits);
/* gbm_compress: bit-pack bins into packed_d (uint32 words, little-endian bit order: bit j of
 * a symbol is stream bit start+j, i.e. bit (s mod 32) of word floor(s/32)); every padding
 * bit is zero.  bits in 1..16.  A symbol >= 2^bits is detected on the device and latched as
 * GBM_E_OVERFLOW for the next gbm_check.  packed_words must be >= gbm_packed_words(...). */
GBM_API int gbm_compress(gbm_ctx *ctx, const uint16_t *bins_d, int64_t n_rows, int32_t n_features,
                 int32_t bits, int32_t row_align_bits, uint32_t *packed_d, int64_t packed_words,
                 void *stream);
/* gbm_quantise_compress: the fused a2 step -- bin map and bit-pack in one pass straight from
 * X_d to packed_d, no uint16 intermediate.  Same layout and results as gbm_quantise followed
 * by gbm_compress.  bits must be >= gbm_symbol_bits(max_symbol of these rows). */
GBM_API int gbm_quantise_compress(gbm_ctx *ctx, const float *X_d, int64_t n_rows, int32_t n_features,
                          int32_t max_bins, const float *cut_values_d, const int32_t *cut_ptr_d,
                          int32_t bits, int32_t row_align_bits, uint32_t *packed_d,
                          int64_t packed_words, void *stream);

/* ---------------------------------------------------------------- the quantised matrix
 * A rank's shard as consumed by tree construction.  cut_ptr_h is a HOST copy of cut_ptr_d
 * (the host plans shared-memory feature groups from it without a device sync). */
typedef struct {
    const uint32_t *packed_d;  /* gbm_compress layout                                      */
    int64_t n_rows;            /* rows of this shard                                       */
    int32_t n_features;
    int32_t bits;              /* symbol width                                             */
    int32_t row_align_bits;    /* 0, 32, 128 or 256                                        */
    int32_t max_bins;          /* B; the missing sentinel symbol                           */
    const float *cut_values_d; /* fp32 [TB]                                                */
    const int32_t *cut_ptr_d;  /* int32 [F+1]                                              */
    const int32_t *cut_ptr_h;  /* int32 [F+1], host copy                                   */
    const uint8_t *colsym_d;   /* OPTIONAL feature-major copy of the symbols (bits <= 8):    */
                               /* uint8 [n_features][n_rows], made by gbm_transpose_symbols; */
                               /* NULL = split symbols are gathered from packed_d            */
} gbm_qmatrix;

/* gbm_transpose_symbols: fill colsym_d (uint8 [n_features][n_rows], caller-owned) with the
 * symbols of qm->packed_d in feature-major order.  A time/space trade: RepartitionInstances
 * then reads one byte per row of the split feature instead of a 32-byte sector of the packed
 * row.  Requires qm->bits <= 8.  Asynchronous. */
GBM_API int gbm_transpose_symbols(gbm_ctx *ctx, const gbm_qmatrix *qm, uint8_t *colsym_d,
                                  void *stream);

typedef struct {
    int32_t objective;         /* GBM_SQUARED_ERROR | GBM_LOGISTIC                          */
    int32_t max_depth;         /* D >= 0: root depth 0, no node deeper than D (R23)         */
    int32_t grad_bits;         /* fixed-point precision P of the gradient pairs (R14); 1..30 */
    int32_t grow_policy;       /* GBM_GROW_DEPTHWISE (0, the zero-initialised default) or   */
                               /* GBM_GROW_LOSSGUIDE (R25-R27)                          */
    double eta, lambda, gamma, min_child_weight;   /* S:311-314, defaults 0.3/1/0/1 */
    int32_t max_leaves;        /* lossguide: at most this many leaves, 1..65536      */
    int32_t reserved;          /* 0                                                          */
} gbm_params;

/* ---------------------------------------------------------------- §2.5 gradients
 * gbm_gradients: per row g, h (Eq. 1-2; squared error g = yhat - y, h = 1) in fp64 with the
 * sigmoid through det_exp (R19); then the fixed point (R14): M = max|g| over every rank's
 * rows (collective max), E = frexp exponent of M (0 if M == 0), s = grad_bits - E,
 * q = rint(g * 2^s) (half to even), |q| <= 2^grad_bits.  Same for h.
 *   margin_d  fp64 [n_rows]     label_d fp32 [n_rows]
 *   qpair_d   int32 [n_rows][2] = (q_g, q_h)
 *   scale_d   int32 [2] device  = (s_g, s_h)
 * Asynchronous; label-domain violations (logistic, label not 0/1) latch GBM_E_LABEL. */
GBM_API int gbm_gradients(gbm_ctx *ctx, int32_t objective, int32_t grad_bits, const double *margin_d,
                  const float *label_d, int64_t n_rows, int32_t *qpair_d, int32_t *scale_d,
                  void *stream);

/* ---------------------------------------------------------------- §2.3 trees (Alg. 1)
 * A tree is a set of DEVICE arrays.  Depth-wise: heap order (root 0, children 2k+1 / 2k+2),
 * capacity 2^(max_depth+1) - 1.  Loss-guided (R27): root 0, the j-th expansion (j = 0, 1, ...)
 * creates children 2j+1 (left) and 2j+2 (right), capacity 2*max_leaves - 1.  kind: GBM_NODE_*.
 * For split nodes: feature, bin, threshold = cuts_feature[bin], default_left, gain, and
 * left_child (the right child is left_child + 1).  For every present node: weight (R11:
 * -G/(H+lambda) * eta, the leaf value for leaves), sum_qg / sum_qh (the node's fixed-point
 * totals over all ranks).  Absent slots and leaves: feature/bin/left_child -1, gain 0; absent
 * slots kind 0 and every other field 0.  left_child may be NULL for depth-wise trees (then it
 * is not written); loss-guided trees require it. */
typedef struct {
    int8_t *kind;
    int32_t *feature;
    int32_t *bin;
    float *threshold;
    int8_t *default_left;
    double *gain;
    double *weight;
    int64_t *sum_qg;
    int64_t *sum_qh;
    int32_t *left_child;
} gbm_tree;

/* gbm_build_tree: Algorithm 1.
 * Depth-wise (grow_policy 0), level-synchronously (R15): InitRoot; then per level:
 * RepartitionInstances (stable), BuildPartialHistograms of the smaller child of every split
 * (R17), AllReduceHistograms (collective: one NCCL int64 sum per level), sibling histogram =
 * parent - built child (north star), EvaluateSplit for every node of the level (R8-R10).
 * Loss-guided (grow_policy 1, R25-R27): max_leaves - 1 expansion steps, each: pop the
 * open node of largest gain (selected on the device), repartition its rows, build the smaller
 * child's histogram, one allreduce, sibling by subtraction, evaluate both children.  Uses the
 * compact histogram layout whatever GBM_OPT_HIST_LAYOUT says.
 * row_leaf_d int32 [n_rows] receives the leaf each row ends in.
 * Asynchronous (no host synchronisation inside a tree).
 * Errors: GBM_E_ARG (null pointers, max_depth outside 0..16, grad_bits outside 1..30, negative
 * lambda / gamma / min_child_weight, lossguide max_leaves outside 1..65536), GBM_E_EMPTY (zero
 * rows on a single rank; a rank of several may hold none).  With a communicator of several
 * ranks (outside CUDA-graph capture) the ranks first agree in one small collective: every rank
 * returns the same code when any rank's arguments are bad, and GBM_E_MISMATCH when the
 * ranks' n_features, total bins, symbol bits, row alignment, max_bins, max_depth, grow_policy,
 * max_leaves or grad_bits differ -- so no rank enters a histogram allreduce its peers skip. */
GBM_API int gbm_build_tree(gbm_ctx *ctx, const gbm_qmatrix *qm, const int32_t *qpair_d,
                   const int32_t *scale_d, const gbm_params *params, const gbm_tree *tree,
                   int32_t *row_leaf_d, void *stream);

/* gbm_build_tree_fused: gbm_build_tree followed by gbm_update_margins and by pass 1 of the NEXT
 * round's gbm_gradients (Eq. 1-2 for the updated margins: the per-row sigmoid for the logistic
 * objective and this rank's max|g|, max|h|), fused into the final leaf assignment when the tree
 * is depth-wise and its rows are staged (else run as separate kernels).  Results are identical
 * to gbm_build_tree + gbm_update_margins + gbm_gradients; the next round then calls
 * gbm_gradients_from_stats instead of gbm_gradients.  All buffers are caller-owned:
 *   margin_d  fp64 [n_rows], updated in place     label_d  fp32 [n_rows]
 *   sig_d     fp64 [n_rows] (logistic; unused for squared error)
 *   maxbits_d uint64 [2]: this rank's maxima as bit patterns of non-negative doubles
 * Label-domain violations latch GBM_E_LABEL as in gbm_gradients. */
typedef struct {
    double *margin_d;
    const float *label_d;
    int32_t objective;
    int32_t reserved;
    double *sig_d;
    uint64_t *maxbits_d;
} gbm_epilogue;
GBM_API int gbm_build_tree_fused(gbm_ctx *ctx, const gbm_qmatrix *qm, const int32_t *qpair_d,
                         const int32_t *scale_d, const gbm_params *params, const gbm_tree *tree,
                         int32_t *row_leaf_d, const gbm_epilogue *epilogue, void *stream);
/* gbm_gradients_from_stats: pass 2 of gbm_gradients from the statistics of the previous
 * gbm_build_tree_fused (same margins and labels): the collective max over ranks (C1) and the
 * fixed-point quantisation (R14).  Same outputs as gbm_gradients. */
GBM_API int gbm_gradients_from_stats(gbm_ctx *ctx, int32_t objective, int32_t grad_bits,
                             const double *margin_d, const float *label_d, int64_t n_rows,
                             const double *sig_d, uint64_t *maxbits_d, int32_t *qpair_d,
                             int32_t *scale_d, void *stream);

/* ---- the steps of Algorithm 1, exposed one by one (used by the parity tests) ---------- */
/* BuildPartialHistograms: hist_d int64 [TB][2] (overwritten) = sum over the listed
 * rows of (q_g, q_h) into bin cut_ptr[f] + symbol for every non-missing symbol.  rows_d
 * uint32 [n_sel] row indices of this shard (NULL = all rows, n_sel ignored).  Not collective. */
GBM_API int gbm_build_histogram(gbm_ctx *ctx, const gbm_qmatrix *qm, const int32_t *qpair_d,
                        int32_t grad_bits, const uint32_t *rows_d, int64_t n_sel,
                        int64_t *hist_d, void *stream);
/* AllReduceHistograms: in-place int64 sum over ranks (collective). */
GBM_API int gbm_allreduce_histograms(gbm_ctx *ctx, int64_t *hist_d, int64_t count, void *stream);
/* EvaluateSplit for n_nodes nodes: hist_d int64 [n_nodes][TB][2], totals_d
 * int64 [n_nodes][2].  Outputs per node (device arrays of n_nodes): split_d int8 (1 iff the
 * best valid candidate has gain > 0), feature_d, bin_d, default_left_d int8, gain_d fp64
 * (best valid gain, 0 if none), child_d int64 [n_nodes][4] = (L_g, L_h, R_g, R_h). */
GBM_API int gbm_evaluate_splits(gbm_ctx *ctx, const gbm_qmatrix *qm, const int64_t *hist_d,
                        const int64_t *totals_d, int32_t n_nodes, const int32_t *scale_d,
                        const gbm_params *params, int8_t *split_d, int32_t *feature_d,
                        int32_t *bin_d, int8_t *default_left_d, double *gain_d,
                        int64_t *child_d, void *stream);
/* RepartitionInstances: stable partition of the rows rows_d uint32 [n_sel] of one
 * node by the split (feature, bin, default_left): left rows (symbol <= bin, or missing and
 * default_left) first, then right rows, each in input order, into out_d uint32 [n_sel];
 * the left count is written to n_left_d int64 [1] (device). */
GBM_API int gbm_repartition(gbm_ctx *ctx, const gbm_qmatrix *qm, const uint32_t *rows_d, int64_t n_sel,
                    int32_t feature, int32_t bin, int32_t default_left, uint32_t *out_d,
                    int64_t *n_left_d, void *stream);

/* ---------------------------------------------------------------- margins and prediction
 * gbm_update_margins: margin[i] = margin[i] + weight[row_leaf[i]] (fp64).  */
GBM_API int gbm_update_margins(gbm_ctx *ctx, const double *weight_d, const int32_t *row_leaf_d,
                       int64_t n_rows, double *margin_d, void *stream);
/* gbm_predict (§2.4): one thread per row; for every tree in order walk
 * from the root, left iff (isnan(v) ? default_left : v <= threshold), and add the leaf
 * weight: margin[i] = base_margin + sum_t w_t(i) in tree order.  Trees are concatenated
 * heap arrays (device) of capacity 2^(max_depth+1)-1 each; X_d fp32 [n_rows][n_features]. */
GBM_API int gbm_predict(gbm_ctx *ctx, int32_t n_trees, int32_t max_depth, const int8_t *kind_d,
                const int32_t *feature_d, const float *threshold_d, const int8_t *default_left_d,
                const double *weight_d, double base_margin, const float *X_d, int64_t n_rows,
                int32_t n_features, double *margin_d, void *stream);

/* gbm_predict_linked: as gbm_predict for trees with explicit child links (the loss-guided
 * layout, R27; depth-wise trees written with left_child work too): the children of split node
 * k are left_child[k] and left_child[k] + 1.  Trees are concatenated device arrays of capacity
 * `cap` each. */
GBM_API int gbm_predict_linked(gbm_ctx *ctx, int32_t n_trees, int64_t cap, const int8_t *kind_d,
                       const int32_t *feature_d, const float *threshold_d,
                       const int8_t *default_left_d, const int32_t *left_child_d,
                       const double *weight_d, double base_margin, const float *X_d,
                       int64_t n_rows, int32_t n_features, double *margin_d, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GBM_H */
