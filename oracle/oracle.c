/*
 * oracle/oracle.c -- CPU ORACLE for the gbm hot path (arXiv 1806.11248, multi-GPU XGBoost).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` leg may load, call or link this library.  The product path
 * (paper_1806_11248_b200/, include/gbm.h) never does, and the two share no code, headers,
 * tables or helpers.
 *
 * Plain, slow, obviously correct C99 in fp64, compiled with `gcc -O2 -ffp-contract=off`
 * (no FMA contraction, no fast-math).  Every function cites the passage it follows:
 *   P:nn  = /root/reference/PAPER.md line nn (section given),
 *   S:nn  = /root/reference/SPEC.md line nn,
 *   R#    = the numbered reading in DESIGN.md "Readings of the paper" where the paper is
 *           silent, ambiguous or garbled.
 * Pins (what ties each function to something other than itself) are listed in DESIGN.md
 * "Oracle pins" and implemented in tests/test_oracle_*.py.
 *
 * Error codes mirror the C-ABI's documented values but are defined here independently.
 *
 * Threaded mode (SURVEY.md §8(d) "Oracle timing"): oracle_set_threads(T) runs the row loops over
 * T contiguous row blocks (OpenMP), the per-feature sort of the cuts over features, and each
 * BuildPartialHistograms over T row blocks with private int64 partial histograms summed in block
 * order.  Every result is a selection, an exact integer sum or a per-row value, so T changes no
 * output (pinned by tests/test_oracle_tree.py::test_threaded_oracle_identical).  T = 1 (default)
 * is the plain single-thread program.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_E_ARG (-1)
#define OR_E_EMPTY (-2)
#define OR_E_OVERFLOW (-3)
#define OR_E_LABEL (-4)
#define OR_E_NONFINITE (-5)
#define OR_E_NOMEM (-12)

static int g_threads = 1;

/* Threads of the row loops (>= 1); returns the previous value. */
int oracle_set_threads(int32_t t)
{
    int old = g_threads;
    g_threads = t < 1 ? 1 : t;
    return old;
}

/* ------------------------------------------------------------------------------------------
 * §2.2 Data compression.  "Matrix values are compressed down to log2(max_value)
 * bits" -- read as the fewest bits that hold every symbol 0..max_value (R1).
 * ------------------------------------------------------------------------------------------ */
int oracle_symbol_bits(int32_t max_symbol)
{
    int b = 1;
    while (b < 31 && ((int64_t)1 << b) <= (int64_t)max_symbol)
        b++;
    return b;
}

/* ------------------------------------------------------------------------------------------
 * §2.1 Feature quantile generation.  The paper's sketch is unspecified; the exact
 * rank rule of R5: for feature f let V be its sorted present values (m of them,
 * d distinct).  d <= B: the cuts are the distinct values (lossless).  Otherwise cut j is
 * V[floor((j+1) m / B) - 1], j = 0..B-1, then duplicates dropped.  -0.0 is canonicalised to
 * +0.0 (R22); +-inf is rejected.
 * ------------------------------------------------------------------------------------------ */
static int cmp_float(const void *a, const void *b)
{
    float x = *(const float *)a, y = *(const float *)b;
    return (x > y) - (x < y);
}

int oracle_cuts(const float *X, int64_t n, int32_t F, int32_t B, float *cut_values,
                int32_t *cut_ptr)
{
    if (n <= 0)
        return OR_E_EMPTY;
    if (F <= 0 || B < 2)
        return OR_E_ARG;
    /* every feature's cuts into its own slot of tmp (at most B each), then concatenated */
    float *tmp = (float *)malloc(sizeof(float) * (size_t)F * (size_t)B);
    int32_t *cnt = (int32_t *)calloc((size_t)F, sizeof(int32_t));
    if (!tmp || !cnt) {
        free(tmp);
        free(cnt);
        return OR_E_NOMEM;
    }
    int err = OR_OK;
#pragma omp parallel num_threads(g_threads)
    {
        float *V = (float *)malloc(sizeof(float) * (size_t)n);
#pragma omp for schedule(dynamic, 1)
        for (int32_t f = 0; f < F; f++) {
            if (!V) {
                err = OR_E_NOMEM;
                continue;
            }
            int64_t m = 0;
            int bad = 0;
            for (int64_t i = 0; i < n; i++) {
                float v = X[i * F + f];
                if (isnan(v))
                    continue;
                if (isinf(v)) {
                    bad = 1;
                    break;
                }
                if (v == 0.0f)
                    v = 0.0f; /* -0.0 -> +0.0 */
                V[m++] = v;
            }
            if (bad) {
                err = OR_E_NONFINITE;
                continue;
            }
            qsort(V, (size_t)m, sizeof(float), cmp_float);
            int64_t d = 0;
            for (int64_t i = 0; i < m; i++)
                if (i == 0 || V[i] != V[i - 1])
                    d++;
            float *out = tmp + (size_t)f * B;
            int32_t c = 0;
            if (d <= B) {
                for (int64_t i = 0; i < m; i++)
                    if (i == 0 || V[i] != V[i - 1])
                        out[c++] = V[i];
            } else {
                for (int64_t j = 0; j < B; j++) {
                    int64_t idx = ((j + 1) * m) / B - 1;
                    float v = V[idx];
                    if (c == 0 || out[c - 1] != v)
                        out[c++] = v;
                }
            }
            cnt[f] = c;
        }
        free(V);
    }
    if (err == OR_OK) {
        int32_t total = 0;
        cut_ptr[0] = 0;
        for (int32_t f = 0; f < F; f++) {
            memcpy(cut_values + total, tmp + (size_t)f * B, sizeof(float) * (size_t)cnt[f]);
            total += cnt[f];
            cut_ptr[f + 1] = total;
        }
    }
    free(tmp);
    free(cnt);
    return err;
}

/* Bin of a present value: the smallest k with v <= cuts[k]; values above the last
 * cut clamp to the last bin (prediction-time quantisation).  Lower-bound binary search. */
static int32_t bin_of(float v, const float *cuts, int32_t nb)
{
    int32_t lo = 0, hi = nb; /* answer in [lo, hi] */
    while (lo < hi) {
        int32_t mid = lo + (hi - lo) / 2;
        if (v <= cuts[mid])
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo < nb ? lo : nb - 1;
}

/* Quantise (R6/R7): symbol = bin_of(v) for present v, the sentinel B for NaN (and for
 * a feature with no cuts).  Reports the maximum stored symbol (R4). */
int oracle_symbols(const float *X, int64_t n, int32_t F, const float *cut_values,
                   const int32_t *cut_ptr, int32_t B, uint16_t *sym, int32_t *max_symbol)
{
    if (n <= 0)
        return OR_E_EMPTY;
    int32_t mx = 0;
    int err = OR_OK;
#pragma omp parallel for num_threads(g_threads) schedule(static) reduction(max : mx)
    for (int64_t i = 0; i < n; i++) {
        for (int32_t f = 0; f < F; f++) {
            float v = X[i * F + f];
            int32_t nb = cut_ptr[f + 1] - cut_ptr[f];
            int32_t s;
            if (isinf(v)) {
                err = OR_E_NONFINITE;
                s = B;
            } else if (isnan(v) || nb == 0) {
                s = B;
            } else {
                s = bin_of(v, cut_values + cut_ptr[f], nb);
            }
            sym[i * F + f] = (uint16_t)s;
            if (s > mx)
                mx = s;
        }
    }
    if (err != OR_OK)
        return err;
    *max_symbol = mx;
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------
 * Bit-packing ("packed and unpacked at runtime using bitwise operations"; S:175-192,
 * layout R3/Q3): element e = (r, f) starts at stream bit r*row_stride + f*bits, bit j of the
 * symbol is stream bit start+j, which is bit (s mod 32) of uint32 word floor(s/32).
 * row_stride = F*bits, rounded up to row_align_bits when that is 32 or 128 (0 = SPEC layout).
 * Buffer = ceil(total_bits/32) words rounded up to a multiple of 4, plus 4 zero words.
 * ------------------------------------------------------------------------------------------ */
static int64_t row_stride_bits(int32_t F, int32_t bits, int32_t row_align_bits)
{
    int64_t rb = (int64_t)F * bits;
    if (row_align_bits > 0)
        rb = (rb + row_align_bits - 1) / row_align_bits * row_align_bits;
    return rb;
}

int64_t oracle_packed_words(int64_t n, int32_t F, int32_t bits, int32_t row_align_bits)
{
    if (n < 0 || F <= 0 || bits < 1 || bits > 16)
        return OR_E_ARG;
    if (row_align_bits != 0 && row_align_bits != 32 && row_align_bits != 128 && row_align_bits != 256)
        return OR_E_ARG;
    int64_t total_bits = n * row_stride_bits(F, bits, row_align_bits);
    int64_t w = (total_bits + 31) / 32;
    w = (w + 3) / 4 * 4;
    return w + 4;
}

int oracle_pack(const uint16_t *sym, int64_t n, int32_t F, int32_t bits, int32_t row_align_bits,
                uint32_t *words, int64_t n_words)
{
    int64_t need = oracle_packed_words(n, F, bits, row_align_bits);
    if (need < 0 || n_words < need)
        return OR_E_ARG;
    int64_t stride = row_stride_bits(F, bits, row_align_bits);
    memset(words, 0, sizeof(uint32_t) * (size_t)n_words);
    for (int64_t r = 0; r < n; r++) {
        for (int32_t f = 0; f < F; f++) {
            uint32_t s = sym[r * F + f];
            if (s >= (1u << bits))
                return OR_E_OVERFLOW;
            int64_t start = r * stride + (int64_t)f * bits;
            for (int32_t j = 0; j < bits; j++) {
                if ((s >> j) & 1u) {
                    int64_t p = start + j;
                    words[p / 32] |= 1u << (p % 32);
                }
            }
        }
    }
    return OR_OK;
}

/* read_symbol: pure O(bits) read of one element, bit by bit. */
static uint32_t read_symbol(const uint32_t *words, int64_t stride, int32_t bits, int64_t r,
                            int32_t f)
{
    int64_t start = r * stride + (int64_t)f * bits;
    uint32_t s = 0;
    for (int32_t j = 0; j < bits; j++) {
        int64_t p = start + j;
        s |= ((words[p / 32] >> (p % 32)) & 1u) << j;
    }
    return s;
}

int oracle_unpack(const uint32_t *words, int64_t n, int32_t F, int32_t bits,
                  int32_t row_align_bits, uint16_t *sym)
{
    int64_t stride = row_stride_bits(F, bits, row_align_bits);
    for (int64_t r = 0; r < n; r++)
        for (int32_t f = 0; f < F; f++)
            sym[r * F + f] = (uint16_t)read_symbol(words, stride, bits, r, f);
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------
 * §2.5 Gradient evaluation (Eq. 1-2 at P:73-80).  sigmoid through det_exp (R19,
 * SURVEY.md Appendix A): only IEEE +,-,*,/, fma and ldexp, so any correctly rounded
 * implementation of those gives the same bits.
 * ------------------------------------------------------------------------------------------ */
static const double DE_C[14] = {
    0x1p+0, 0x1p+0, 0x1p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,
    0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
    0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22,
    0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29, 0x1.6124613a86d09p-33};

double oracle_det_exp(double t) /* defined for t <= 0 */
{
    if (t < -745.0)
        return 0.0;
    double k = rint(t * 0x1.71547652b82fep+0);
    double r = fma(-k, 0x1.62e42feep-1, t);
    r = fma(-k, 0x1.a39ef35793c76p-33, r);
    double p = DE_C[13];
    for (int i = 12; i >= 0; i--)
        p = fma(p, r, DE_C[i]);
    return ldexp(p, (int)k);
}

double oracle_sigmoid(double x)
{
    if (x >= 0.0) {
        double e = oracle_det_exp(-x);
        return 1.0 / (1.0 + e);
    }
    double e = oracle_det_exp(x);
    return e / (1.0 + e);
}

/* Per-row (g, h), then fixed point (R14, Q4): with M = max|g| over ALL rows (every shard),
 * E = frexp exponent of M (M < 2^E; E = 0 when M = 0), s = P - E and q = rint(g * 2^s)
 * (round half to even), so |q| <= 2^P.  Same for h.  objective 0 = reg:squarederror
 * (g = yhat - y, h = 1), 1 = binary:logistic (Eq. 1-2; labels must be 0 or 1).
 * qpair is [n][2] = (q_g, q_h); scale = (s_g, s_h).  g, h may be NULL. */
int oracle_gradients(int32_t objective, const double *margin, const float *label, int64_t n,
                     int32_t P, double *g_out, double *h_out, int32_t *qpair, int32_t *scale)
{
    if (n <= 0)
        return OR_E_EMPTY;
    if (P < 1 || P > 30 || (objective != 0 && objective != 1))
        return OR_E_ARG;
    double *g = (double *)malloc(sizeof(double) * (size_t)n);
    double *h = (double *)malloc(sizeof(double) * (size_t)n);
    if (!g || !h) {
        free(g);
        free(h);
        return OR_E_NOMEM;
    }
    int bad_label = 0;
    double Mg = 0.0, Mh = 0.0;
#pragma omp parallel for num_threads(g_threads) schedule(static) reduction(max : Mg, Mh)
    for (int64_t i = 0; i < n; i++) {
        double y = (double)label[i];
        if (objective == 0) {
            g[i] = margin[i] - y;
            h[i] = 1.0;
        } else {
            if (!(label[i] == 0.0f || label[i] == 1.0f)) {
                bad_label = 1;
                g[i] = h[i] = 0.0;
                continue;
            }
            double s = oracle_sigmoid(margin[i]);
            g[i] = s - y;
            h[i] = s * (1.0 - s);
        }
        if (fabs(g[i]) > Mg)
            Mg = fabs(g[i]);
        if (fabs(h[i]) > Mh)
            Mh = fabs(h[i]);
    }
    if (bad_label) {
        free(g);
        free(h);
        return OR_E_LABEL;
    }
    int Eg = 0, Eh = 0;
    if (Mg > 0.0)
        (void)frexp(Mg, &Eg);
    if (Mh > 0.0)
        (void)frexp(Mh, &Eh);
    int sg = P - Eg, sh = P - Eh;
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        qpair[2 * i + 0] = (int32_t)rint(ldexp(g[i], sg));
        qpair[2 * i + 1] = (int32_t)rint(ldexp(h[i], sh));
        if (g_out)
            g_out[i] = g[i];
        if (h_out)
            h_out[i] = h[i];
    }
    scale[0] = sg;
    scale[1] = sh;
    free(g);
    free(h);
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------
 * §2.3 Decision tree construction, Algorithm 1 and its steps.
 * ------------------------------------------------------------------------------------------ */

/* BuildPartialHistograms: H[cut_ptr[f] + s] += (q_g, q_h) as int64 for
 * every listed row and every feature whose symbol s is not the sentinel B.  hist is
 * [TB][2], overwritten. */
int oracle_node_histogram(const uint32_t *words, int32_t F, int32_t bits, int32_t row_align_bits,
                          const int32_t *cut_ptr, int32_t B, const int32_t *qpair,
                          const int64_t *rows, int64_t n_sel, int64_t *hist)
{
    int64_t stride = row_stride_bits(F, bits, row_align_bits);
    int32_t TB = cut_ptr[F];
    memset(hist, 0, sizeof(int64_t) * 2 * (size_t)TB);
    for (int64_t k = 0; k < n_sel; k++) {
        int64_t r = rows[k];
        for (int32_t f = 0; f < F; f++) {
            uint32_t s = read_symbol(words, stride, bits, r, f);
            if ((int32_t)s == B)
                continue; /* missing: mass recovered as total - sum (R7) */
            int64_t bin = cut_ptr[f] + s;
            hist[2 * bin + 0] += qpair[2 * r + 0];
            hist[2 * bin + 1] += qpair[2 * r + 1];
        }
    }
    return OR_OK;
}

/* AllReduceHistograms of the p_workers' partial histograms of node `node` (the rows i
 * with pos[i] == node; worker w owns rows [w n / p, (w + 1) n / p), R18), summed in worker
 * order.  Threaded mode splits each worker's rows over g_threads blocks, each with a private
 * partial (parts: [g_threads][2 TB]); int64 sums are exact, so the block count is invisible.
 * rows: scratch [n]. */
static void reduced_histogram(const uint32_t *words, int64_t n, int32_t F, int32_t bits,
                              int32_t row_align_bits, const int32_t *cut_ptr, int32_t B,
                              const int32_t *qpair, const int32_t *pos, int32_t node,
                              int32_t p_workers, int64_t *rows, int64_t *parts, int64_t *hist)
{
    const int32_t TB = cut_ptr[F];
    const int T = g_threads;
    memset(hist, 0, sizeof(int64_t) * 2 * (size_t)TB);
    for (int32_t w = 0; w < p_workers; w++) {
        const int64_t lo = (w * n) / p_workers, hi = ((w + 1) * n) / p_workers;
#pragma omp parallel for num_threads(T) schedule(static, 1)
        for (int t = 0; t < T; t++) {
            const int64_t b0 = lo + ((hi - lo) * t) / T, b1 = lo + ((hi - lo) * (t + 1)) / T;
            int64_t *rr = rows + b0, m = 0;
            for (int64_t i = b0; i < b1; i++)
                if (pos[i] == node)
                    rr[m++] = i;
            oracle_node_histogram(words, F, bits, row_align_bits, cut_ptr, B, qpair, rr, m,
                                  parts + (size_t)t * 2 * TB);
        }
        for (int t = 0; t < T; t++)
            for (int32_t k = 0; k < 2 * TB; k++)
                hist[k] += parts[(size_t)t * 2 * TB + k];
    }
}

/* RepartitionInstances: a row of node k goes to `left` iff
 * (symbol == sentinel ? default_left : symbol <= bin), else to `right`; rows are independent. */
static void repartition(const uint32_t *words, int64_t n, int64_t stride, int32_t bits, int32_t B,
                        int32_t *pos, int32_t k, const int32_t *si, int32_t left, int32_t right)
{
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        if (pos[i] != k)
            continue;
        uint32_t s = read_symbol(words, stride, bits, i, si[0]);
        int go_left = ((int32_t)s == B) ? si[2] : ((int32_t)s <= si[1]);
        pos[i] = go_left ? left : right;
    }
}

/* EvaluateSplit (R8-R10, Q5).  For every feature f, missing mass
 * M = T - sum_b H[f][b]; for b = 0..n_bins(f)-1 and dl in (true, false) in that order:
 * prefix P = sum_{b'<=b} H[f][b'], L = P + (dl ? M : 0), R = T - L, then the XGBoost gain in
 * the exact op order of R8.  Best = the first valid candidate whose gain is strictly greater
 * than every earlier one.  Returns 1 (split) iff a best exists and its gain > 0, else 0.
 * out_i = (feature, bin, default_left), out_l = (L_g, L_h, R_g, R_h). */
int oracle_evaluate_split(const int64_t *hist, int32_t F, const int32_t *cut_ptr, int64_t Tg,
                          int64_t Th, int32_t sg, int32_t sh, double lambda, double gamma,
                          double mcw, int32_t *out_i, double *out_gain, int64_t *out_l)
{
    double G = ldexp((double)Tg, -sg), H = ldexp((double)Th, -sh);
    double e = G * G;
    e = e / (H + lambda);
    int found = 0;
    double best = 0.0;
    for (int32_t f = 0; f < F; f++) {
        int64_t sumg = 0, sumh = 0;
        for (int32_t b = cut_ptr[f]; b < cut_ptr[f + 1]; b++) {
            sumg += hist[2 * b + 0];
            sumh += hist[2 * b + 1];
        }
        int64_t Mg = Tg - sumg, Mh = Th - sumh;
        int64_t Pg = 0, Ph = 0;
        for (int32_t b = 0; b < cut_ptr[f + 1] - cut_ptr[f]; b++) {
            Pg += hist[2 * (cut_ptr[f] + b) + 0];
            Ph += hist[2 * (cut_ptr[f] + b) + 1];
            for (int dli = 0; dli < 2; dli++) {
                int dl = (dli == 0); /* true first (R9) */
                int64_t Lg = Pg + (dl ? Mg : 0), Lh = Ph + (dl ? Mh : 0);
                int64_t Rg = Tg - Lg, Rh = Th - Lh;
                double GL = ldexp((double)Lg, -sg), HL = ldexp((double)Lh, -sh);
                double GR = ldexp((double)Rg, -sg), HR = ldexp((double)Rh, -sh);
                if (!(HL >= mcw && HR >= mcw && HL + lambda > 0.0 && HR + lambda > 0.0))
                    continue;
                double a = GL * GL;
                a = a / (HL + lambda);
                double c = GR * GR;
                c = c / (HR + lambda);
                double d = a + c;
                d = d - e;
                d = 0.5 * d;
                double gain = d - gamma;
                if (!found || gain > best) {
                    found = 1;
                    best = gain;
                    out_i[0] = f;
                    out_i[1] = b;
                    out_i[2] = dl;
                    out_l[0] = Lg;
                    out_l[1] = Lh;
                    out_l[2] = Rg;
                    out_l[3] = Rh;
                }
            }
        }
    }
    *out_gain = found ? best : 0.0;
    return (found && best > 0.0) ? 1 : 0;
}

/* Leaf weight (R11): t = H + lambda; w = (t == 0) ? 0 : -(G / t) * eta. */
double oracle_leaf_weight(int64_t Tg, int64_t Th, int32_t sg, int32_t sh, double lambda,
                          double eta)
{
    double G = ldexp((double)Tg, -sg), H = ldexp((double)Th, -sh);
    double t = H + lambda;
    if (t == 0.0)
        return 0.0;
    double w = G / t;
    w = -w;
    w = w * eta;
    return w;
}

/* Tree arrays: heap order (root 0, children 2k+1 / 2k+2), capacity 2^(D+1)-1.
 * kind: 0 absent, 1 split, 2 leaf. */
typedef struct {
    int32_t node, depth;
    int64_t Tg, Th;
    int split; /* EvaluateSplit result */
    int32_t si[3];
    double gain;
    int64_t sl[4];
} entry_t;

/* Alg. 1 as written, with the readings R15 (a popped entry becomes a split node iff its
 * EvaluateSplit found gain > 0 and depth < max_depth, otherwise a leaf), R16 (the p workers
 * run the same steps on their shards), R18 (shard k = rows [k n / p, (k+1) n / p)).
 * "AllReduce" = sum of the p partial histograms in ascending worker order.
 * The expand queue is FIFO: depth-wise growth, "nodes closer to the root" first.
 * Both child histograms are built directly (the oracle does not use the subtraction trick).
 * positions[i] = the node row i currently sits in (SPEC's WorkerSet); at the end it
 * is row_leaf.  params = (eta, lambda, gamma, min_child_weight). */
int oracle_build_tree(const uint32_t *words, int64_t n, int32_t F, int32_t bits,
                      int32_t row_align_bits, const float *cut_values, const int32_t *cut_ptr,
                      int32_t B, const int32_t *qpair, const int32_t *scale, int32_t max_depth,
                      const double *params, int32_t p_workers, int8_t *kind, int32_t *feature,
                      int32_t *bin, float *threshold, int8_t *default_left, double *gain,
                      double *weight, int64_t *sum_qg, int64_t *sum_qh, int32_t *row_leaf)
{
    if (n <= 0)
        return OR_E_EMPTY;
    if (max_depth < 0 || max_depth > 20 || p_workers < 1)
        return OR_E_ARG;
    const double eta = params[0], lambda = params[1], gamma = params[2], mcw = params[3];
    const int32_t sg = scale[0], sh = scale[1];
    const int64_t stride = row_stride_bits(F, bits, row_align_bits);
    const int32_t TB = cut_ptr[F];
    const int64_t cap = ((int64_t)1 << (max_depth + 1)) - 1;
    for (int64_t k = 0; k < cap; k++) {
        kind[k] = 0;
        feature[k] = -1;
        bin[k] = -1;
        threshold[k] = 0.0f;
        default_left[k] = 0;
        gain[k] = 0.0;
        weight[k] = 0.0;
        sum_qg[k] = 0;
        sum_qh[k] = 0;
    }
    int64_t *hist = (int64_t *)calloc(2 * (size_t)(TB > 0 ? TB : 1), sizeof(int64_t));
    int64_t *part = (int64_t *)calloc(2 * (size_t)(TB > 0 ? TB : 1) * (size_t)g_threads,
                                      sizeof(int64_t));
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    entry_t *queue = (entry_t *)malloc(sizeof(entry_t) * (size_t)cap);
    if (!hist || !part || !rows || !queue) {
        free(hist);
        free(part);
        free(rows);
        free(queue);
        return OR_E_NOMEM;
    }
    for (int64_t i = 0; i < n; i++)
        row_leaf[i] = 0;

    /* AllReduce of the p partial histograms of node `node` (rows with position == node). */
#define BUILD_REDUCED_HIST(node_id)                                                              \
    reduced_histogram(words, n, F, bits, row_align_bits, cut_ptr, B, qpair, row_leaf, (node_id),   \
                      p_workers, rows, part, hist)

    /* InitRoot: root totals over every worker's rows, root histogram, root split. */
    entry_t root;
    memset(&root, 0, sizeof(root));
    root.node = 0;
    root.depth = 0;
    for (int32_t w = 0; w < p_workers; w++) {
        int64_t lo = (w * n) / p_workers, hi = ((w + 1) * n) / p_workers;
        for (int64_t i = lo; i < hi; i++) {
            root.Tg += qpair[2 * i + 0];
            root.Th += qpair[2 * i + 1];
        }
    }
    if (max_depth > 0) {
        BUILD_REDUCED_HIST(0);
        root.split = oracle_evaluate_split(hist, F, cut_ptr, root.Tg, root.Th, sg, sh, lambda,
                                           gamma, mcw, root.si, &root.gain, root.sl);
    }
    int64_t qhead = 0, qtail = 0;
    queue[qtail++] = root;

    while (qhead < qtail) {                 /* while expand_queue is not empty */
        entry_t e = queue[qhead++];         /*   expand_entry <- expand_queue.pop() */
        int32_t k = e.node;                 /*   tree.insert(expand_entry) */
        sum_qg[k] = e.Tg;
        sum_qh[k] = e.Th;
        weight[k] = oracle_leaf_weight(e.Tg, e.Th, sg, sh, lambda, eta);
        if (!(e.split && e.depth < max_depth)) {
            kind[k] = 2;
            continue;
        }
        kind[k] = 1;
        feature[k] = e.si[0];
        bin[k] = e.si[1];
        default_left[k] = (int8_t)e.si[2];
        threshold[k] = cut_values[cut_ptr[e.si[0]] + e.si[1]];
        gain[k] = e.gain;
        /* RepartitionInstances on every worker: a row of node k goes left
         * iff (symbol == sentinel ? default_left : symbol <= bin).  Rows keep row order. */
        int32_t left = 2 * k + 1, right = 2 * k + 2;
        repartition(words, n, stride, bits, B, row_leaf, k, e.si, left, right);
        entry_t le, re;
        memset(&le, 0, sizeof(le));
        memset(&re, 0, sizeof(re));
        le.node = left;
        re.node = right;
        le.depth = re.depth = e.depth + 1;
        le.Tg = e.sl[0];
        le.Th = e.sl[1];
        re.Tg = e.sl[2];
        re.Th = e.sl[3];
        if (e.depth + 1 < max_depth) {
            /* BuildPartialHistograms + AllReduceHistograms + EvaluateSplit, both children */
            BUILD_REDUCED_HIST(left);
            le.split = oracle_evaluate_split(hist, F, cut_ptr, le.Tg, le.Th, sg, sh, lambda,
                                             gamma, mcw, le.si, &le.gain, le.sl);
            BUILD_REDUCED_HIST(right);
            re.split = oracle_evaluate_split(hist, F, cut_ptr, re.Tg, re.Th, sg, sh, lambda,
                                             gamma, mcw, re.si, &re.gain, re.sl);
        }
        queue[qtail++] = le;                /* expand_queue.push(left_expand_entry) */
        queue[qtail++] = re;                /* expand_queue.push(right_expand_entry) */
    }
#undef BUILD_REDUCED_HIST
    free(hist);
    free(part);
    free(rows);
    free(queue);
    return OR_OK;
}

/* Loss-guided growth (the loop of Alg. 1 "reconfigurable to prioritise expanding nodes
 * with a higher reduction in the objective function").  Readings:
 * R25  expand_queue is a priority queue: pop = the entry of largest priority, priority = the
 *      entry's split gain if it is expandable, else below every gain; ties to the smaller node
 *      id.  (Non-expandable entries become leaves whenever popped, so their order is moot.)
 * R26  an entry is expandable iff its EvaluateSplit found gain > 0, its depth < max_depth and
 *      fewer than max_leaves - 1 expansions were made (at most max_leaves leaves).
 * R27  node ids: root 0; the j-th expansion (j = 0, 1, ...) creates left 2j+1, right 2j+2;
 *      left_child[k] = 2j+1 for a split node, -1 otherwise; capacity 2 max_leaves - 1.
 * Children are evaluated iff depth + 1 < max_depth (as oracle_build_tree).  Everything else --
 * repartition, both child histograms built directly, AllReduce order, EvaluateSplit, leaf
 * weights -- is oracle_build_tree's. */
int oracle_build_tree_lossguide(const uint32_t *words, int64_t n, int32_t F, int32_t bits,
                                int32_t row_align_bits, const float *cut_values,
                                const int32_t *cut_ptr, int32_t B, const int32_t *qpair,
                                const int32_t *scale, int32_t max_depth, int32_t max_leaves,
                                const double *params, int32_t p_workers, int8_t *kind,
                                int32_t *feature, int32_t *bin, float *threshold,
                                int8_t *default_left, double *gain, double *weight,
                                int64_t *sum_qg, int64_t *sum_qh, int32_t *left_child,
                                int32_t *row_leaf)
{
    if (n <= 0)
        return OR_E_EMPTY;
    if (max_depth < 0 || max_leaves < 1 || max_leaves > (1 << 20) || p_workers < 1)
        return OR_E_ARG;
    const double eta = params[0], lambda = params[1], gamma = params[2], mcw = params[3];
    const int32_t sg = scale[0], sh = scale[1];
    const int64_t stride = row_stride_bits(F, bits, row_align_bits);
    const int32_t TB = cut_ptr[F];
    const int64_t cap = 2 * (int64_t)max_leaves - 1;
    for (int64_t k = 0; k < cap; k++) {
        kind[k] = 0;
        feature[k] = -1;
        bin[k] = -1;
        threshold[k] = 0.0f;
        default_left[k] = 0;
        gain[k] = 0.0;
        weight[k] = 0.0;
        sum_qg[k] = 0;
        sum_qh[k] = 0;
        left_child[k] = -1;
    }
    int64_t *hist = (int64_t *)calloc(2 * (size_t)(TB > 0 ? TB : 1), sizeof(int64_t));
    int64_t *part = (int64_t *)calloc(2 * (size_t)(TB > 0 ? TB : 1) * (size_t)g_threads,
                                      sizeof(int64_t));
    int64_t *rows = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    entry_t *queue = (entry_t *)malloc(sizeof(entry_t) * (size_t)cap);
    if (!hist || !part || !rows || !queue) {
        free(hist);
        free(part);
        free(rows);
        free(queue);
        return OR_E_NOMEM;
    }
    for (int64_t i = 0; i < n; i++)
        row_leaf[i] = 0;

#define BUILD_REDUCED_HIST(node_id)                                                              \
    reduced_histogram(words, n, F, bits, row_align_bits, cut_ptr, B, qpair, row_leaf, (node_id),   \
                      p_workers, rows, part, hist)

    entry_t root;
    memset(&root, 0, sizeof(root));
    for (int32_t w = 0; w < p_workers; w++) {
        int64_t lo = (w * n) / p_workers, hi = ((w + 1) * n) / p_workers;
        for (int64_t i = lo; i < hi; i++) {
            root.Tg += qpair[2 * i + 0];
            root.Th += qpair[2 * i + 1];
        }
    }
    if (max_depth > 0) {
        BUILD_REDUCED_HIST(0);
        root.split = oracle_evaluate_split(hist, F, cut_ptr, root.Tg, root.Th, sg, sh, lambda,
                                           gamma, mcw, root.si, &root.gain, root.sl);
    }
    int64_t qn = 0;         /* entries in the queue: queue[0 .. qn) */
    int32_t expansions = 0; /* j */
    queue[qn++] = root;

    while (qn > 0) { /* while expand_queue is not empty */
        /* expand_entry <- expand_queue.pop(): largest priority (R25) */
        int64_t bi = -1;
        for (int64_t q = 0; q < qn; q++) {
            const entry_t *c = &queue[q];
            int c_exp = c->split && c->depth < max_depth && expansions < max_leaves - 1;
            if (!c_exp)
                continue;
            if (bi < 0 || c->gain > queue[bi].gain ||
                (c->gain == queue[bi].gain && c->node < queue[bi].node))
                bi = q;
        }
        if (bi < 0)
            bi = 0; /* only non-expandable entries remain: any of them */
        entry_t e = queue[bi];
        queue[bi] = queue[--qn];
        int32_t k = e.node; /* tree.insert(expand_entry) */
        sum_qg[k] = e.Tg;
        sum_qh[k] = e.Th;
        weight[k] = oracle_leaf_weight(e.Tg, e.Th, sg, sh, lambda, eta);
        if (!(e.split && e.depth < max_depth && expansions < max_leaves - 1)) {
            kind[k] = 2;
            continue;
        }
        int32_t left = 2 * expansions + 1, right = 2 * expansions + 2; /* R27 */
        expansions++;
        kind[k] = 1;
        feature[k] = e.si[0];
        bin[k] = e.si[1];
        default_left[k] = (int8_t)e.si[2];
        threshold[k] = cut_values[cut_ptr[e.si[0]] + e.si[1]];
        gain[k] = e.gain;
        left_child[k] = left;
        repartition(words, n, stride, bits, B, row_leaf, k, e.si, left, right); /* every worker */
        entry_t le, re;
        memset(&le, 0, sizeof(le));
        memset(&re, 0, sizeof(re));
        le.node = left;
        re.node = right;
        le.depth = re.depth = e.depth + 1;
        le.Tg = e.sl[0];
        le.Th = e.sl[1];
        re.Tg = e.sl[2];
        re.Th = e.sl[3];
        if (e.depth + 1 < max_depth) {
            BUILD_REDUCED_HIST(left);
            le.split = oracle_evaluate_split(hist, F, cut_ptr, le.Tg, le.Th, sg, sh, lambda,
                                             gamma, mcw, le.si, &le.gain, le.sl);
            BUILD_REDUCED_HIST(right);
            re.split = oracle_evaluate_split(hist, F, cut_ptr, re.Tg, re.Th, sg, sh, lambda,
                                             gamma, mcw, re.si, &re.gain, re.sl);
        }
        queue[qn++] = le; /* expand_queue.push(left_expand_entry) */
        queue[qn++] = re; /* expand_queue.push(right_expand_entry) */
    }
#undef BUILD_REDUCED_HIST
    free(hist);
    free(part);
    free(rows);
    free(queue);
    return OR_OK;
}

/* Prediction over trees with explicit child links (loss-guided layout, R27): as
 * oracle_predict, but the children of split node k are left_child[k] and left_child[k] + 1;
 * trees are concatenated arrays of capacity cap each. */
int oracle_predict_linked(int32_t n_trees, int64_t cap, const int8_t *kind, const int32_t *feature,
                          const float *threshold, const int8_t *default_left,
                          const int32_t *left_child, const double *weight, double base_margin,
                          const float *X, int64_t n, int32_t F, double *margin)
{
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double m = base_margin;
        for (int32_t t = 0; t < n_trees; t++) {
            int64_t o = t * cap, k = 0;
            while (kind[o + k] == 1) {
                int32_t f = feature[o + k];
                float v = f < F ? X[i * F + f] : NAN;
                int go_left = isnan(v) ? default_left[o + k] : (v <= threshold[o + k]);
                k = go_left ? left_child[o + k] : left_child[o + k] + 1;
            }
            m = m + weight[o + k];
        }
        margin[i] = m;
    }
    return OR_OK;
}

/* Margin update (Q6): margin[i] = margin[i] + w[row_leaf[i]] in fp64. */
int oracle_update_margins(const double *weight, const int32_t *row_leaf, int64_t n,
                          double *margin)
{
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t i = 0; i < n; i++)
        margin[i] = margin[i] + weight[row_leaf[i]];
    return OR_OK;
}

/* §2.4 Prediction (Q7): one row at a time, trees in order; from the root
 * go left iff (isnan(v) ? default_left : v <= threshold) until a leaf, then m = m + w.
 * Trees are concatenated heap arrays of capacity cap = 2^(max_depth+1)-1 each. */
int oracle_predict(int32_t n_trees, int32_t max_depth, const int8_t *kind,
                   const int32_t *feature, const float *threshold, const int8_t *default_left,
                   const double *weight, double base_margin, const float *X, int64_t n,
                   int32_t F, double *margin)
{
    int64_t cap = ((int64_t)1 << (max_depth + 1)) - 1;
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double m = base_margin;
        for (int32_t t = 0; t < n_trees; t++) {
            int64_t o = t * cap, k = 0;
            while (kind[o + k] == 1) {
                int32_t f = feature[o + k];
                float v = f < F ? X[i * F + f] : NAN;
                int go_left = isnan(v) ? default_left[o + k] : (v <= threshold[o + k]);
                k = go_left ? 2 * k + 1 : 2 * k + 2;
            }
            m = m + weight[o + k];
        }
        margin[i] = m;
    }
    return OR_OK;
}
