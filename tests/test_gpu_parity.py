"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Bit-exact on cuts, bin indices, packed words, fixed-point gradients, histograms, row
partitions, split choices and gains; leaf weights / margins / predictions are bit-exact by
construction (identical IEEE op sequences) and asserted within the north star's 1e-6 relative
floor as well.  Sizes span several tiles / work items and ragged tails.
"""
import numpy as np
import pytest
import torch

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    import paper_1806_11248_b200 as G
    return G


@pytest.fixture(scope="module")
def ctx(G):
    c = G.Context(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def _qm_from_oracle(G, X, B, align, cuts=None):
    v, p = O.cuts(X, B) if cuts is None else cuts
    s, mx = O.symbols(X, v, p, B)
    bits = O.symbol_bits(mx)
    words = O.pack(s, bits, align)
    qm = G.QMatrix(dev(words.view(np.int32)), X.shape[0], X.shape[1], bits, align, B,
                   dev(v if v.size else np.zeros(1, np.float32)), dev(p), p.copy())
    return qm, v, p, s, bits, words


# ------------------------------------------------------------------ a1: cuts
CUT_CASES = [("rand", 5000, 6, 16, None, 0.0), ("ties", 9000, 5, 32, 40, 0.1),
             ("lossless", 4097, 3, 256, 200, 0.0), ("wideB", 30000, 2, 1000, None, 0.02),
             ("one_row", 1, 4, 16, None, 0.0), ("allnan", 100, 3, 8, None, 1.0)]


@pytest.mark.parametrize("name,n,F,B,distinct,missing", CUT_CASES)
def test_cuts_parity(ctx, name, n, F, B, distinct, missing):
    X = W.random_matrix(hash(name) % 1000, n, F, distinct=distinct, missing=missing)
    X[0, 0] = -0.0 if n > 1 else X[0, 0]
    v, p = O.cuts(X, B)
    cv, cp, mx = ctx.cuts(dev(X), B)
    np.testing.assert_array_equal(cp.cpu().numpy(), p)
    np.testing.assert_array_equal(cv.cpu().numpy().view(np.uint32), v.view(np.uint32))
    _, omx = O.symbols(X, v, p, B)
    assert mx == omx


@pytest.mark.parametrize("cfg", ["tiny", "yearmsd", "higgs", "airline"])
def test_cuts_parity_workloads(ctx, cfg):
    X, _ = W.generate(cfg, 0, 2000 if cfg == "tiny" else 60_000)
    B = W.CONFIGS[cfg].max_bins
    v, p = O.cuts(X, B)
    cv, cp, mx = ctx.cuts(dev(X), B)
    np.testing.assert_array_equal(cp.cpu().numpy(), p)
    np.testing.assert_array_equal(cv.cpu().numpy(), v)


def test_cuts_reject_inf(ctx, G):
    X = np.ones((10, 2), np.float32)
    X[3, 1] = np.inf
    with pytest.raises(G.GbmError) as e:
        ctx.cuts(dev(X), 8)
    assert e.value.code == -5


# ------------------------------------------------------------------ a2: bin map + pack
@pytest.mark.parametrize("missing", [0.0, 0.05])
def test_quantise_parity(ctx, missing):
    X = W.random_matrix(3, 7001, 9, missing=missing)
    B = 64
    v, p = O.cuts(X, B)
    s, _ = O.symbols(X, v, p, B)
    bins = ctx.quantise(dev(X), B, dev(v), dev(p))
    np.testing.assert_array_equal(bins.cpu().numpy(), s)


@pytest.mark.parametrize("bits", [1, 2, 3, 4, 5, 7, 8, 9, 11, 13, 16])
@pytest.mark.parametrize("align", [0, 32, 128, 256])
def test_compress_parity(ctx, bits, align):
    rng = np.random.default_rng(bits * 7 + align)
    n, F = 3001, 13
    sym = rng.integers(0, 1 << bits, (n, F)).astype(np.uint16)
    words = ctx.compress(dev(sym), bits, align)
    np.testing.assert_array_equal(u32(words), O.pack(sym, bits, align))


@pytest.mark.parametrize("cfg,align,B,missing", [("tiny", 0, None, 0.03), ("higgs", 32, None, 0.0),
                                                 ("airline", 128, None, 0.0), ("yearmsd", 32, None, 0.0),
                                                 ("higgs", 256, 200, 0.05), ("airline", 32, 255, 0.02),
                                                 ("epsilon", 32, None, 0.0)])
def test_quantise_compress_parity(ctx, G, cfg, align, B, missing):
    """The fused bin map + pack: the generic walk and the byte kernel (8-bit symbols, rows of whole
    words: padding slots and words, the missing sentinel inside 8 bits)."""
    X, _ = W.generate(cfg, 0, 2000 if cfg == "tiny" else 3000 if cfg == "epsilon" else 40_000,
                      n_rows=None if cfg != "epsilon" else 3000, missing=missing)
    B = B or W.CONFIGS[cfg].max_bins
    v, p = O.cuts(X, B)
    s, mx = O.symbols(X, v, p, B)
    bits = O.symbol_bits(mx)
    packed = ctx.quantise_compress(dev(X), B, dev(v), dev(p), bits, align)
    np.testing.assert_array_equal(u32(packed), O.pack(s, bits, align))


def test_compress_overflow_latched(ctx, G):
    sym = np.full((4, 3), 9, np.uint16)
    ctx.compress(dev(sym), 3, 0)
    with pytest.raises(G.GbmError) as e:
        ctx.check()
    assert e.value.code == -3


@pytest.mark.parametrize("cfg,align", [("higgs", 32), ("airline", 0), ("tiny", 128)])
def test_transpose_symbols_parity(ctx, G, cfg, align):
    X, _ = W.generate(cfg, 0, 2000 if cfg == "tiny" else 30_001)
    qm, v, p, s, bits, words = _qm_from_oracle(G, X, W.CONFIGS[cfg].max_bins, align)
    ctx.transpose_symbols(qm)
    np.testing.assert_array_equal(qm.colsym.cpu().numpy(), s.T.astype(np.uint8))


# ------------------------------------------------------------------ a3: gradients
@pytest.mark.parametrize("obj", ["reg:squarederror", "binary:logistic"])
@pytest.mark.parametrize("P", [15, 30, 7])
def test_gradients_parity(ctx, obj, P):
    rng = np.random.default_rng(P)
    n = 300_001
    m = rng.standard_normal(n) * (6 if obj == "binary:logistic" else 30)
    m[:5] = [0.0, 40.0, -40.0, 709.0, -745.5]
    y = ((rng.random(n) < 0.5).astype(np.float32) if obj == "binary:logistic"
         else (rng.standard_normal(n) * 20).astype(np.float32))
    _, _, q, sc = O.gradients(obj, m, y, P)
    qg, sg = ctx.gradients(obj, dev(m), dev(y), P)
    np.testing.assert_array_equal(qg.cpu().numpy(), q)
    assert tuple(sg.cpu().tolist()) == sc


def test_gradients_label_error(ctx, G):
    y = np.array([0, 1, 2, 1], np.float32)
    ctx.gradients("binary:logistic", dev(np.zeros(4)), dev(y), 15)
    with pytest.raises(G.GbmError) as e:
        ctx.check()
    assert e.value.code == -4


# ------------------------------------------------------------------ a4/a6: histograms
@pytest.mark.parametrize("layout", [1, 2, 3])
@pytest.mark.parametrize("P", [15, 30])
@pytest.mark.parametrize("cfg,align,missing", [("higgs", 32, 0.0), ("tiny", 0, 0.05),
                                               ("airline", 128, 0.0), ("yearmsd", 32, 0.01)])
def test_histogram_parity(ctx, G, P, cfg, align, missing, layout):
    ctx.set_option(ctx.HIST_LAYOUT, layout)
    n = 2000 if cfg == "tiny" else 150_000
    X, y = W.generate(cfg, 0, n, missing=missing)
    qm, v, p, s, bits, words = _qm_from_oracle(G, X, W.CONFIGS[cfg].max_bins, align)
    rng = np.random.default_rng(1)
    margin = rng.standard_normal(n)
    obj = "reg:squarederror"
    _, _, q, sc = O.gradients(obj, margin, y, P)
    qd = dev(q)
    # all rows (identity) and a sorted random subset (gather)
    for rows in (None, np.sort(rng.choice(n, n // 3, replace=False)).astype(np.uint32)):
        sel = np.arange(n) if rows is None else rows.astype(np.int64)
        ref = O.node_histogram(words, X.shape[1], bits, align, p, qm.max_bins, q, sel)
        got = ctx.build_histogram(qm, qd, P, None if rows is None else dev(rows.view(np.int32)))
        np.testing.assert_array_equal(got.cpu().numpy(), ref)
    ctx.set_option(ctx.HIST_LAYOUT, 0)


# ------------------------------------------------------------------ a9: EvaluateSplit
@pytest.mark.parametrize("eval_warp", [1, 2])
@pytest.mark.parametrize("seed", range(4))
def test_evaluate_parity(ctx, G, seed, eval_warp):
    ctx.set_option(ctx.EVAL_WARP, eval_warp)
    X, y = W.generate("higgs", 0, 20_000, seed_offset=seed)
    qm, v, p, s, bits, words = _qm_from_oracle(G, X, 256, 32)
    rng = np.random.default_rng(seed)
    nodes = []
    _, _, q, sc = O.gradients("binary:logistic", rng.standard_normal(20_000) * 0.3, y, 15)
    for k in range(6):
        rows = np.sort(rng.choice(20_000, 500 * (k + 1), replace=False)).astype(np.int64)
        H = O.node_histogram(words, 28, bits, 32, p, 256, q, rows)
        T = q[rows].astype(np.int64).sum(0)
        nodes.append((H, T))
    lam, gam, mcw = (1.0, 0.0, 1.0) if seed % 2 == 0 else (0.5, 0.1, 3.0)
    hist = dev(np.stack([h for h, _ in nodes]))
    tot = dev(np.stack([t for _, t in nodes]))
    out = ctx.evaluate_splits(qm, hist, tot, dev(np.array(sc, np.int32)), reg_lambda=lam,
                              gamma=gam, min_child_weight=mcw)
    out = {k: v.cpu().numpy() for k, v in out.items()}
    for j, (H, T) in enumerate(nodes):
        r = O.evaluate_split(H, p, T[0], T[1], sc, lam, gam, mcw)
        assert bool(out["split"][j]) == r["split"]
        assert out["gain"][j] == r["gain"]
        if r["feature"] >= 0:
            assert (out["feature"][j], out["bin"][j], bool(out["default_left"][j])) == \
                (r["feature"], r["bin"], r["default_left"])
            assert tuple(out["child"][j]) == r["L"] + r["R"]
    ctx.set_option(ctx.EVAL_WARP, 0)


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("seed", range(6))
def test_evaluate_screen_is_exact_on_near_ties(ctx, G, seed, kernel):
    """The approximate screen (GBM_OPT_EVAL_SCREEN) never changes a result: histograms built to
    have many exact ties and near ties (duplicated features, +-1 perturbations, coarse counts),
    with and without missing mass; screened == unscreened == oracle, bit for bit."""
    rng = np.random.default_rng(500 + seed)
    F, nb = 12, 64
    cut_ptr = np.arange(F + 1, dtype=np.int32) * nb
    base = rng.integers(-40, 41, (nb, 2)) * (1 << 10)
    base[:, 1] = np.abs(base[:, 1]) + (1 << 12)
    nodes = []
    for j in range(5):
        H = np.concatenate([base for _ in range(F)]).astype(np.int64)
        for f in range(F):  # near ties: tiny perturbations of a few bins
            k = rng.integers(0, nb, 3)
            H[f * nb + k, 0] += rng.integers(-1, 2, 3)
        T = H.sum(0)
        if j % 2:  # missing mass
            T = T + np.array([rng.integers(-5000, 5000), rng.integers(0, 5000)])
        nodes.append((H, T))
    hist, tot = dev(np.stack([h for h, _ in nodes])), dev(np.stack([t for _, t in nodes]))
    qm = G.QMatrix(torch.zeros(4, dtype=torch.int32, device="cuda"), 1, F, 8, 32, 256,
                   torch.zeros(F * nb, dtype=torch.float32, device="cuda"), dev(cut_ptr), cut_ptr)
    sc = dev(np.array([20, 20], np.int32))
    ctx.set_option(ctx.EVAL_WARP, kernel)
    outs = []
    for screen in (0, 1):
        ctx.set_option(ctx.EVAL_SCREEN, screen)
        o = ctx.evaluate_splits(qm, hist, tot, sc, reg_lambda=1.0, gamma=0.0, min_child_weight=0.0)
        outs.append({k: v.cpu().numpy() for k, v in o.items()})
    ctx.set_option(ctx.EVAL_SCREEN, 0)
    ctx.set_option(ctx.EVAL_WARP, 0)
    for k in outs[0]:
        np.testing.assert_array_equal(outs[0][k], outs[1][k], err_msg=k)
    for j, (H, T) in enumerate(nodes):
        r = O.evaluate_split(H, cut_ptr, T[0], T[1], [20, 20], 1.0, 0.0, 0.0)
        assert outs[1]["gain"][j] == r["gain"] and bool(outs[1]["split"][j]) == r["split"]
        if r["feature"] >= 0:
            assert (outs[1]["feature"][j], outs[1]["bin"][j]) == (r["feature"], r["bin"])


# ------------------------------------------------------------------ a5: RepartitionInstances
@pytest.mark.parametrize("n_sel", [0, 1, 31, 1024, 1025, 70_001])
def test_repartition_parity(ctx, G, n_sel):
    X, y = W.generate("higgs", 0, 80_000, missing=0.02)
    qm, v, p, s, bits, words = _qm_from_oracle(G, X, 256, 32)
    rng = np.random.default_rng(n_sel)
    rows = np.sort(rng.choice(80_000, n_sel, replace=False)).astype(np.uint32)
    f, b, dl = 3, 100, 1
    sym = s[rows.astype(np.int64), f]
    left = np.where(sym == 256, bool(dl), sym <= b)
    ref = np.concatenate([rows[left], rows[~left]])
    out, nl = ctx.repartition(qm, dev(rows.view(np.int32)), f, b, dl)
    np.testing.assert_array_equal(u32(out), ref)
    assert int(nl.item()) == int(left.sum())


# ------------------------------------------------------------------ whole trees and rounds
def _compare_tree(gt, ot):
    for k in ("kind", "feature", "bin", "default_left", "sum_qg", "sum_qh"):
        np.testing.assert_array_equal(gt[k], ot[k], err_msg=k)
    np.testing.assert_array_equal(gt["threshold"].view(np.uint32), ot["threshold"].view(np.uint32))
    np.testing.assert_array_equal(gt["gain"], ot["gain"])
    # leaf weights: bit-exact by construction; the north-star floor is 1e-6 relative
    np.testing.assert_allclose(gt["weight"], ot["weight"], rtol=1e-6, atol=0)
    np.testing.assert_array_equal(gt["weight"], ot["weight"])


TREE_CASES = [
    # cfg, rows, missing, align, P, rounds, depth override
    ("tiny", 2000, 0.0, 32, 15, 3, None),
    ("tiny", 2000, 0.05, 0, 30, 3, 5),
    ("tiny", 2000, 0.05, 32, 15, 2, 4),
    ("yearmsd", 30_000, 0.0, 32, 15, 3, None),
    ("higgs", 100_000, 0.0, 32, 15, 3, None),
    ("higgs", 100_000, 0.0, 32, 16, 2, None),
    ("higgs", 50_000, 0.02, 128, 30, 2, None),
    ("higgs", 40_000, 0.0, 256, 15, 2, None),   # sector-aligned rows (28 -> 32 bytes)
    ("airline", 120_000, 0.0, 32, 15, 2, None),
    ("airline", 60_000, 0.03, 0, 12, 2, None),
    ("bosch", 12_000, 0.0, 32, 15, 2, None),   # ~81% missing: 9-bit symbols, default directions
]


@pytest.mark.parametrize("layout,colsym,carry", [(0, True, 0), (2, True, 0), (0, False, 1), (2, False, 1),
                                                 (3, True, 0), (3, False, 1)])
@pytest.mark.parametrize("cfg,n,missing,align,P,rounds,depth", TREE_CASES)
def test_training_rounds_parity(ctx, G, cfg, n, missing, align, P, rounds, depth, colsym, layout,
                                carry):
    ctx.set_option(ctx.HIST_LAYOUT, layout)
    ctx.set_option(ctx.CARRY_GRADIENTS, carry)
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n, missing=missing)
    D = c.max_depth if depth is None else depth
    kw = dict(eta=0.3, reg_lambda=1.0, gamma=0.0, mcw=1.0)
    ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=D, grad_bits=P,
                   row_align_bits=align, **kw)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=c.max_bins, objective=c.objective, max_depth=D,
                   grad_bits=P, row_align_bits=align, base_margin=ob.base_margin, eta=0.3,
                   reg_lambda=1.0, gamma=0.0, min_child_weight=1.0, colsym=colsym)
    np.testing.assert_array_equal(u32(gb.qm.packed), ob.words)
    for r in range(rounds):
        ot = ob.round()
        gt = gb.round().to_numpy()
        np.testing.assert_array_equal(gb.qpair.cpu().numpy(), ob.last["qpair"])
        _compare_tree(gt, ot)
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    # prediction (§2.4) on the training rows and on fresh rows
    Xt, _ = W.generate(cfg, n, n + 5000, n_rows=max(n + 5000, c.n_rows))
    np.testing.assert_array_equal(gb.predict(dev(X)).cpu().numpy(), ob.predict())
    np.testing.assert_array_equal(gb.predict(dev(Xt)).cpu().numpy(), ob.predict(Xt))
    ctx.set_option(ctx.HIST_LAYOUT, 0)
    ctx.set_option(ctx.CARRY_GRADIENTS, 0)


REC_CASES = [
    # cfg, rows, missing, align, P, max_bins override, depth override
    ("higgs", 100_000, 0.0, 32, 15, None, None),
    ("higgs", 70_001, 0.0, 32, 30, None, None),       # wide accumulators (4 channels)
    ("higgs", 50_000, 0.02, 32, 15, 200, None),       # 8-bit symbols with the sentinel (200)
    ("higgs", 40_000, 0.0, 256, 15, None, 9),         # 32-byte rows, 256 parents at the last level
    ("airline", 120_000, 0.0, 32, 15, None, None),    # 13 features: two rows per warp step
    ("airline", 30_000, 0.03, 128, 20, None, 4),
    ("tiny", 2000, 0.0, 32, 15, 256, 5),              # 8 features, 8-bit symbols: four rows per step
    ("epsilon", 3000, 0.0, 32, 15, None, 3),          # > 32 features: falls back to row-index lists
]


@pytest.mark.parametrize("path", [1, 2])
@pytest.mark.parametrize("cfg,n,missing,align,P,B,depth", REC_CASES)
def test_record_levels_parity(ctx, G, cfg, n, missing, align, P, B, depth, path):
    """GBM_OPT_LEVEL_PATH 2 (records: rows moved into node-grouped buffers, TMA-staged, bank-column
    histograms) against 1 (row-index lists), both against the oracle, every tree field, the row
    partition and the margins bit for bit."""
    ctx.set_option(ctx.LEVEL_PATH, path)
    c = W.CONFIGS[cfg]
    B = B or c.max_bins
    D = depth or c.max_depth
    X, y = W.generate(cfg, 0, n, n_rows=max(n, c.n_rows), missing=missing)
    ob = O.Booster(X, y, max_bins=B, objective=c.objective, max_depth=D, grad_bits=P, row_align_bits=align,
                   eta=0.3)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=B, objective=c.objective, max_depth=D, grad_bits=P,
                   row_align_bits=align, base_margin=ob.base_margin, eta=0.3)
    for _ in range(3):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    ctx.set_option(ctx.LEVEL_PATH, 0)


@pytest.mark.parametrize("level_hist", [1, 2, 3])
@pytest.mark.parametrize("cfg,n,missing,align,P,B,depth", REC_CASES + [("higgs", 150_000, 0.0, 32, 15, None, 8)])
def test_level_hist_layouts_parity(ctx, G, cfg, n, missing, align, P, B, depth, level_hist):
    """GBM_OPT_LEVEL_HIST 2 (bank-column level histograms fed by warp shuffles) and 1 (compact),
    both against the oracle bit for bit, with multi-tile work items (RUN_TILES 3)."""
    ctx.set_option(ctx.LEVEL_HIST, level_hist)
    ctx.set_option(ctx.RUN_TILES, 3)
    c = W.CONFIGS[cfg]
    B = B or c.max_bins
    D = depth or c.max_depth
    X, y = W.generate(cfg, 0, n, n_rows=max(n, c.n_rows), missing=missing)
    ob = O.Booster(X, y, max_bins=B, objective=c.objective, max_depth=D, grad_bits=P, row_align_bits=align,
                   eta=0.3)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=B, objective=c.objective, max_depth=D, grad_bits=P,
                   row_align_bits=align, base_margin=ob.base_margin, eta=0.3)
    for _ in range(3):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    ctx.set_option(ctx.LEVEL_HIST, 0)
    ctx.set_option(ctx.RUN_TILES, 0)


@pytest.mark.parametrize("rep", [1, 0])
@pytest.mark.parametrize("cfg,n,missing,P,B", [("airline", 250_000, 0.0, 15, None), ("airline", 120_000, 0.1, 30, None),
                                               ("higgs", 200_000, 0.0, 15, None), ("yearmsd", 60_000, 0.0, 15, 16),
                                               ("higgs", 100_000, 0.05, 15, 3), ("epsilon", 20_000, 0.0, 15, 8)])
def test_level_replicas_parity(ctx, G, cfg, n, missing, P, B, rep):
    """GBM_OPT_LEVEL_REPLICAS: copies of the bins of low-cardinality features in the fused level
    kernel (row slot r adds into copy r mod R, folded before the flush) -- Airline's few-level
    columns, Higgs's b-tags, every feature at 16 / 8 / 3 bins (copies capped by REP_CAP), missing
    values (sentinel skipped) and P = 30 (four channels); bit for bit against the oracle."""
    ctx.set_option(ctx.LEVEL_REPLICAS, rep)
    c = W.CONFIGS[cfg]
    B = B or c.max_bins
    X, y = W.generate(cfg, 0, n, n_rows=max(n, c.n_rows), missing=missing)
    ob = O.Booster(X, y, max_bins=B, objective=c.objective, max_depth=c.max_depth, grad_bits=P)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=B, objective=c.objective, max_depth=c.max_depth,
                   grad_bits=P, base_margin=ob.base_margin)
    for _ in range(2):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    ctx.set_option(ctx.LEVEL_REPLICAS, 1)


@pytest.mark.parametrize("run_tiles", [2, 5, 8, 31])
@pytest.mark.parametrize("cfg,n,missing,P", [("higgs", 300_000, 0.0, 15), ("airline", 250_000, 0.0, 15),
                                             ("higgs", 200_000, 0.0, 30), ("bosch", 40_000, 0.0, 15)])
def test_run_tiles_rounds_parity(ctx, G, cfg, n, missing, P, run_tiles):
    """Work items of several 2048-row tiles (the auto value at 11M rows is 5): many items per
    parent, items straddling parents, and the 31-tile maximum (one flush per <= 63488 rows)."""
    ctx.set_option(ctx.RUN_TILES, run_tiles)
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n, missing=missing)
    ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=c.max_depth, grad_bits=P)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=c.max_bins, objective=c.objective, max_depth=c.max_depth,
                   grad_bits=P, base_margin=ob.base_margin)
    for _ in range(2):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    ctx.set_option(ctx.RUN_TILES, 0)


def test_run_tiles_option_bounds(ctx, G):
    with pytest.raises(G.GbmError):
        ctx.set_option(ctx.RUN_TILES, 32)
    ctx.set_option(ctx.RUN_TILES, 31)
    ctx.set_option(ctx.RUN_TILES, 0)


@pytest.mark.parametrize("opt,good,bad,default", [("LEVEL_REPLICAS", (0, 1), (2, -1), 1),
                                                  ("ROOT_TENSOR", (0, 1, 7), (8, -1), 0),
                                                  ("LEVEL_HIST", (0, 3), (4,), 0), ("LEVEL_PATH", (0, 2), (3,), 0),
                                                  ("EVAL_SLICED", (0, 1), (2,), 0), ("CUTS_GATHER", (0, 1), (2,), 0)])
def test_option_bounds(ctx, G, opt, good, bad, default):
    """Every tuning option accepts its documented range and rejects values outside it (GBM_E_ARG)."""
    code = getattr(ctx, opt)
    for v in bad:
        with pytest.raises(G.GbmError) as e:
            ctx.set_option(code, v)
        assert e.value.code == -1
    for v in good:
        ctx.set_option(code, v)
    ctx.set_option(code, default)


@pytest.mark.parametrize("layout", [0, 3])
@pytest.mark.parametrize("cfg,n,missing,align,P,depth", [
    ("tiny", 2000, 0.05, 32, 15, 5),            # 1 word per row, missing (default directions)
    ("higgs", 70_000, 0.0, 32, 15, None),       # 7 words
    ("higgs", 30_000, 0.02, 256, 15, None),     # 8 words (sector-aligned)
    ("airline", 90_000, 0.03, 32, 15, None),    # depth 8, 4 words, missing
    ("yearmsd", 20_000, 0.0, 128, 15, 4),       # 24 words: out of range -> gathered symbols
    ("tiny", 1999, 0.0, 32, 30, 3),             # ragged last 32-row chunk, wide gradients
])
def test_row_decide_rounds_parity(ctx, G, cfg, n, missing, align, P, depth, layout):
    """GBM_OPT_ROW_DECIDE = 2: RepartitionInstances from the row-order decision bits
    equals the oracle (trees, row_leaf, margins) -- and equals the gathered-symbol path."""
    ctx.set_option(ctx.HIST_LAYOUT, layout)
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n, missing=missing)
    D = c.max_depth if depth is None else depth
    ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=D, grad_bits=P,
                   row_align_bits=align, eta=0.3, reg_lambda=1.0, gamma=0.0, mcw=1.0)
    gbs = {}
    for mode in (2, 1):
        ctx.set_option(ctx.ROW_DECIDE, mode)
        gbs[mode] = G.Booster(ctx, dev(X), dev(y), max_bins=c.max_bins, objective=c.objective,
                              max_depth=D, grad_bits=P, row_align_bits=align,
                              base_margin=ob.base_margin, eta=0.3, reg_lambda=1.0, gamma=0.0,
                              min_child_weight=1.0)
    try:
        for r in range(2):
            ot = ob.round()
            for mode in (2, 1):
                ctx.set_option(ctx.ROW_DECIDE, mode)
                gb = gbs[mode]
                gt = gb.round().to_numpy()
                _compare_tree(gt, ot)
                np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
                np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    finally:
        ctx.set_option(ctx.ROW_DECIDE, 0)
        ctx.set_option(ctx.HIST_LAYOUT, 0)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("cfg,n,missing,grow", [("airline", 60_000, 0.03, "depthwise"),
                                                ("bosch", 12_000, 0.0, "depthwise"),
                                                ("tiny", 2000, 0.05, "lossguide")])
def test_eval_variant_rounds_parity(ctx, G, cfg, n, missing, grow, mode):
    """Both evaluation kernels (GBM_OPT_EVAL_WARP 1 = warp, 2 = block per feature) on wide
    features and missing mass."""
    ctx.set_option(ctx.EVAL_WARP, mode)
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n, missing=missing)
    L = 20 if grow == "lossguide" else 0
    D = 10 if grow == "lossguide" else c.max_depth
    ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=D,
                   grow_policy=grow, max_leaves=L)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=c.max_bins, objective=c.objective, max_depth=D,
                   base_margin=ob.base_margin, grow_policy=grow, max_leaves=L)
    for _ in range(2):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    ctx.set_option(ctx.EVAL_WARP, 0)


@pytest.mark.parametrize("walk", [0, 1])
def test_lossguide_leaf_walks(ctx, G, walk):
    """Loss-guided final assignment: staged linked walk (0) and the gather walk (1)."""
    ctx.set_option(ctx.LEAF_WALK, walk)
    X, y = W.generate("higgs", 0, 40_000)
    kw = dict(max_bins=256, objective="binary:logistic", max_depth=12, grow_policy="lossguide",
              max_leaves=40)
    ob = O.Booster(X, y, **kw)
    gb = G.Booster(ctx, dev(X), dev(y), base_margin=ob.base_margin, **kw)
    for _ in range(2):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
    ctx.set_option(ctx.LEAF_WALK, 0)


@pytest.mark.parametrize("walk", [0, 1])
@pytest.mark.parametrize("D", [3, 12, 16])
def test_deep_trees_and_leaf_walks(ctx, G, D, walk):
    """max_depth up to the ABI limit (16: the heap of internal nodes no longer fits shared memory)
    and both final-level walks (staged rows / feature-major copy)."""
    ctx.set_option(ctx.LEAF_WALK, walk)
    X, y = W.generate("tiny", 0, 3000, n_rows=3000, missing=0.05)
    ob = O.Booster(X, y, max_bins=64, objective="reg:squarederror", max_depth=D, mcw=0.0)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=64, objective="reg:squarederror", max_depth=D,
                   base_margin=ob.base_margin, min_child_weight=0.0)
    for _ in range(2):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
    ctx.set_option(ctx.LEAF_WALK, 0)


def _edge_matrix(kind):
    rng = np.random.default_rng(77)
    if kind == "one_row":
        X = np.array([[1.5, -2.0, 0.25]], np.float32)
    elif kind == "ragged_33":
        X = W.random_matrix(5, 33, 4, distinct=7, missing=0.1)
    elif kind == "one_feature":
        X = W.random_matrix(6, 5000, 1)
    elif kind == "constant_and_missing_features":
        X = W.random_matrix(7, 4000, 5, missing=0.05)
        X[:, 1] = 3.0            # one bin
        X[:, 3] = np.nan         # no cuts at all
    elif kind == "many_features_few_rows":
        X = W.random_matrix(8, 64, 300, distinct=5, missing=0.2)
    elif kind == "wide_bins_9bit":
        X = W.random_matrix(9, 20000, 3)
        X[rng.random(X.shape) < 0.01] = np.nan
    else:
        raise KeyError(kind)
    y = (np.nan_to_num(X[:, 0]) + rng.standard_normal(X.shape[0]) > 0).astype(np.float32)
    return X, y


@pytest.mark.parametrize("grow", ["depthwise", "lossguide"])
@pytest.mark.parametrize("kind", ["one_row", "ragged_33", "one_feature", "constant_and_missing_features",
                                  "many_features_few_rows", "wide_bins_9bit"])
def test_edge_shapes_parity(ctx, G, kind, grow):
    """Degenerate shapes: one row, ragged tails, one feature, a constant feature and an
    all-missing feature, more features than rows, 9-bit symbols from 256 bins + missing."""
    X, y = _edge_matrix(kind)
    B = 256 if kind == "wide_bins_9bit" else 16
    L = 7 if grow == "lossguide" else 0
    kw = dict(max_bins=B, objective="binary:logistic", max_depth=4, grow_policy=grow, max_leaves=L)
    ob = O.Booster(X, y, mcw=0.0, **kw)
    gb = G.Booster(ctx, dev(X), dev(y), base_margin=ob.base_margin, min_child_weight=0.0, **kw)
    for _ in range(3):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    np.testing.assert_array_equal(gb.predict(dev(X)).cpu().numpy(), ob.predict())


@pytest.mark.parametrize("cfg,n,missing,align,P", [("higgs", 60_000, 0.0, 32, 15), ("bosch", 12_000, 0.0, 32, 15),
                                                  ("tiny", 3000, 0.05, 32, 15), ("airline", 40_000, 0.03, 32, 12),
                                                  ("epsilon", 4_000, 0.0, 32, 15), ("higgs", 30_000, 0.0, 128, 15),
                                                  ("bosch", 6_000, 0.0, 128, 15), ("tiny", 3000, 0.05, 0, 15)])
def test_staged_root_parity(ctx, G, cfg, n, missing, align, P):
    """The staged bank-column root (byte and generic symbol widths) forced at small sizes
    (GBM_OPT_HIST_LAYOUT 4, the tensor-fed root off), levels compact; and the root histogram
    itself vs the oracle."""
    ctx.set_option(ctx.HIST_LAYOUT, 4)
    ctx.set_option(ctx.ROOT_TENSOR, 1)
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n, n_rows=max(n, c.n_rows) if cfg == "tiny" else None, missing=missing)
    ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=c.max_depth, grad_bits=P,
                   row_align_bits=align)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=c.max_bins, objective=c.objective, max_depth=c.max_depth,
                   grad_bits=P, row_align_bits=align, base_margin=ob.base_margin)
    # word-aligned rows of 8-bit (byte) or 9..15-bit (generic) symbols: the staged kernels apply
    staged = align % 32 == 0 and (gb.qm.bits == 8 or 9 <= gb.qm.bits <= 15)
    for _ in range(2):
        ctx.profile(True, only=("hist_root", "hist_level"))
        _compare_tree(gb.round().to_numpy(), ob.round())
        prof = ctx.profile_read()
        ctx.profile(False)
        if staged:  # the staged root kernel is the one that ran (it books under hist_root)
            assert prof["hist_root"]["launches"] >= 1
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    # the root histogram itself, bin for bin (gbm_build_histogram takes the same staged kernel)
    qm, v, p, s, bits, words = _qm_from_oracle(G, X, c.max_bins, align)
    _, _, q, _ = O.gradients(c.objective, np.zeros(n), y, P)
    ref = O.node_histogram(words, X.shape[1], bits, align, p, qm.max_bins, q, np.arange(n))
    ctx.profile(True, only=("hist_root", "hist_level"))
    got = ctx.build_histogram(qm, dev(q), P)
    prof = ctx.profile_read()
    ctx.profile(False)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)
    if staged:
        assert prof["hist_root"]["launches"] == 1 and prof["hist_level"]["launches"] == 0
    ctx.set_option(ctx.HIST_LAYOUT, 0)
    ctx.set_option(ctx.ROOT_TENSOR, 0)


def test_max_depth_zero_and_one(ctx, G):
    X, y = W.generate("tiny")
    for D in (0, 1):
        ob = O.Booster(X, y, max_bins=16, objective="reg:squarederror", max_depth=D)
        gb = G.Booster(ctx, dev(X), dev(y), max_bins=16, objective="reg:squarederror",
                       max_depth=D, base_margin=ob.base_margin)
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])


# ------------------------------------------------------------------ loss-guided growth
LG_CASES = [
    # cfg, rows, missing, align, P, rounds, max_depth, max_leaves
    ("tiny", 2000, 0.05, 32, 15, 3, 8, 12),
    ("tiny", 2000, 0.0, 0, 30, 2, 3, 64),       # budget not binding
    ("tiny", 2000, 0.0, 32, 15, 2, 6, 1),       # a single leaf
    ("tiny", 2000, 0.0, 32, 15, 2, 0, 8),       # max_depth 0
    ("higgs", 100_000, 0.0, 32, 15, 3, 12, 31),
    ("higgs", 50_000, 0.02, 128, 16, 2, 10, 63),  # wide fixed point
    ("yearmsd", 30_000, 0.0, 32, 15, 2, 8, 20),
    ("airline", 60_000, 0.03, 0, 12, 2, 16, 40),
    ("bosch", 12_000, 0.0, 32, 15, 2, 8, 16),   # 9-bit symbols, ~81% missing
]


@pytest.mark.parametrize("colsym,carry", [(True, 0), (False, 1)])
@pytest.mark.parametrize("cfg,n,missing,align,P,rounds,D,L", LG_CASES)
def test_lossguide_rounds_parity(ctx, G, cfg, n, missing, align, P, rounds, D, L, colsym, carry):
    ctx.set_option(ctx.CARRY_GRADIENTS, carry)
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n, missing=missing)
    kw = dict(eta=0.3, reg_lambda=1.0, gamma=0.0)
    ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=D, grad_bits=P,
                   row_align_bits=align, mcw=1.0, grow_policy="lossguide", max_leaves=L, **kw)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=c.max_bins, objective=c.objective, max_depth=D,
                   grad_bits=P, row_align_bits=align, base_margin=ob.base_margin,
                   min_child_weight=1.0, colsym=colsym, grow_policy="lossguide", max_leaves=L, **kw)
    for r in range(rounds):
        ot = ob.round()
        gt = gb.round().to_numpy()
        _compare_tree(gt, ot)
        np.testing.assert_array_equal(gt["left_child"], ot["left_child"])
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    Xt, _ = W.generate(cfg, n, n + 3000, n_rows=max(n + 3000, c.n_rows))
    np.testing.assert_array_equal(gb.predict(dev(X)).cpu().numpy(), ob.predict())
    np.testing.assert_array_equal(gb.predict(dev(Xt)).cpu().numpy(), ob.predict(Xt))
    ctx.set_option(ctx.CARRY_GRADIENTS, 0)


def test_depthwise_trees_carry_links(ctx, G):
    """Depth-wise trees fill left_child (2k+1) too, so the linked predictor walks them."""
    X, y = W.generate("tiny")
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=16, objective="reg:squarederror", max_depth=4)
    t = gb.round().to_numpy()
    k = np.nonzero(t["kind"] == 1)[0]
    np.testing.assert_array_equal(t["left_child"][k], 2 * k + 1)
    assert np.all(t["left_child"][t["kind"] != 1] == -1)


# ------------------------------------------------------------------ full-size properties
@pytest.mark.parametrize("cfg", ["higgs"])
def test_full_size_round_properties(ctx, G, cfg):
    """BASELINE.json full size, in bench.py's launch configuration: exact gradient parity for
    every row, exact root histogram, exact child totals of every node from row_leaf, and the
    row->leaf map of sampled rows re-derived by the oracle's predictor on the raw values."""
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg)
    n, F = X.shape
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=c.max_bins, objective=c.objective,
                   max_depth=c.max_depth, eta=c.eta)
    # cuts on a sample of columns are checked elsewhere; here: gradients + one round
    gb.ctx.gradients(c.objective, gb.margin, gb.y, gb.grad_bits, out=gb.qpair, scale=gb.scale)
    _, _, q, sc = O.gradients(c.objective, np.zeros(n), y, gb.grad_bits)
    np.testing.assert_array_equal(gb.qpair.cpu().numpy(), q)
    words = u32(gb.qm.packed)
    p = gb.qm.cut_ptr_h
    root = ctx.build_histogram(gb.qm, gb.qpair, gb.grad_bits).cpu().numpy()
    ref = O.node_histogram(words, F, gb.qm.bits, 32, p, c.max_bins, q, np.arange(n))
    np.testing.assert_array_equal(root, ref)
    tree = gb.round().to_numpy()
    rl = gb.row_leaf.cpu().numpy()
    # root split == oracle EvaluateSplit on the full root histogram
    T = q.astype(np.int64).sum(0)
    r = O.evaluate_split(ref, p, T[0], T[1], sc, 1.0, 0.0, 1.0)
    assert (tree["feature"][0], tree["bin"][0], bool(tree["default_left"][0])) == \
        (r["feature"], r["bin"], r["default_left"]) and tree["gain"][0] == r["gain"]
    # every node's totals == sum of qpair over the rows of its subtree (exact, int64)
    cap = tree["kind"].shape[0]
    sums = np.zeros((cap, 2), np.int64)
    np.add.at(sums, rl, q.astype(np.int64))
    for k in range(cap - 1, 0, -1):
        sums[(k - 1) // 2] += sums[k] if tree["kind"][k] else 0
    present = tree["kind"] > 0
    np.testing.assert_array_equal(sums[present, 0], tree["sum_qg"][present])
    np.testing.assert_array_equal(sums[present, 1], tree["sum_qh"][present])
    # sampled rows: the leaf the oracle's predictor reaches on raw values == row_leaf
    idx = np.random.default_rng(0).choice(n, 20_000, replace=False)
    tid = {k: v.copy() for k, v in tree.items()}
    tid["weight"] = np.arange(cap, dtype=np.float64)
    leaf = O.predict([tid], c.max_depth, 0.0, X[idx]).astype(np.int64)
    np.testing.assert_array_equal(leaf, rl[idx])


@pytest.mark.parametrize("cfg,P", [("higgs", 15), ("higgs", 30)])
def test_full_size_training_parity(ctx, G, cfg, P):
    """BASELINE.json's Higgs-shaped 11M x 28 at full size, the headline configuration (auto
    level plan: several 2048-row tiles per work item, several parents per level): GPU cuts,
    packed words, and two boosting rounds -- every tree field, the row -> leaf map and the
    margins -- bit for bit against the oracle (threaded over the host's cores; results do not
    depend on the thread count, tests/test_oracle_tree.py::test_threaded_oracle_identical)."""
    import os
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg)
    old = O.set_threads(len(os.sched_getaffinity(0)))
    try:
        ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=c.max_depth,
                       eta=c.eta, grad_bits=P)
        gb = G.Booster(ctx, dev(X), dev(y), max_bins=c.max_bins, objective=c.objective,
                       max_depth=c.max_depth, eta=c.eta, grad_bits=P, base_margin=ob.base_margin)
        np.testing.assert_array_equal(gb.qm.cut_ptr_h, ob.cut_ptr)
        np.testing.assert_array_equal(gb.qm.cut_values.cpu().numpy().view(np.uint32),
                                      ob.cut_values.view(np.uint32))
        np.testing.assert_array_equal(u32(gb.qm.packed), ob.words)
        for _ in range(2):
            _compare_tree(gb.round().to_numpy(), ob.round())
            np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
            np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    finally:
        O.set_threads(old)


def test_single_rank_communicator_paths(G):
    """A 1-rank NCCL communicator: every collective of the path (C3 all-gather in gbm_cuts, C1
    max in gbm_gradients, C2 histogram sums in gbm_build_tree) runs through NCCL and the model
    is unchanged (integer sums, exact maxima)."""
    X, y = W.generate("tiny", missing=0.05)
    c = G.Context(0)
    c.comm_init(G.Context.comm_unique_id(), 1, 0)
    assert G.lib().gbm_comm_info(c.h, None, None) == 0
    ob = O.Booster(X, y, max_bins=16, objective="reg:squarederror", max_depth=4, eta=0.3)
    gb = G.Booster(c, dev(X), dev(y), max_bins=16, objective="reg:squarederror", max_depth=4,
                   eta=0.3, base_margin=ob.base_margin)
    np.testing.assert_array_equal(u32(gb.qm.packed), ob.words)
    for _ in range(3):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    h = torch.arange(10, dtype=torch.int64, device="cuda")
    c.allreduce_histograms(h)
    assert h.cpu().tolist() == list(range(10))
    c.close()


@pytest.mark.parametrize("grow", ["depthwise", "lossguide"])
def test_graph_captured_rounds_with_communicator(G, grow):
    """bench.py's launch configuration at N > 1: whole rounds captured as CUDA graphs with the
    NCCL collectives (C1 max, C2 histogram sums) and the side-stream scatter inside, here with a
    1-rank communicator.  Every replayed round equals the oracle's."""
    X, y = W.generate("higgs", 0, 60_000)
    c = G.Context(0)
    c.comm_init(G.Context.comm_unique_id(), 1, 0)
    L = 24 if grow == "lossguide" else 0
    kw = dict(max_bins=256, objective="binary:logistic", max_depth=6, eta=0.1, grow_policy=grow,
              max_leaves=L)
    ob = O.Booster(X, y, **kw)
    gb = G.Booster(c, dev(X), dev(y), base_margin=ob.base_margin, **kw)
    _compare_tree(gb.round(keep_tree=False).to_numpy(), ob.round())  # eager round 1
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph):
            tree = gb.round(keep_tree=False)
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(3):
        graph.replay()
        torch.cuda.synchronize()
        _compare_tree(tree.to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    del graph
    c.close()


def test_build_tree_argument_errors(ctx, G):
    """gbm_build_tree's documented argument errors (GBM_E_ARG = -1): bad growth policy, leaf
    budget out of range, loss-guided tree without left_child, depth-wise depth > 16."""
    X, y = W.generate("tiny")
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=16, objective="reg:squarederror", max_depth=3)
    q, sc = ctx.gradients("reg:squarederror", gb.margin, gb.y)
    cases = [dict(grow_policy=7, max_depth=3), dict(grow_policy="lossguide", max_leaves=0, max_depth=3),
             dict(grow_policy="lossguide", max_leaves=70000, max_depth=3), dict(max_depth=17)]
    for kw in cases:
        with pytest.raises(G.GbmError) as e:
            ctx.build_tree(gb.qm, q, sc, objective="reg:squarederror", **kw)
        assert e.value.code == -1, kw
    t = G.Tree(3, "cuda", 4)
    t.arrays["left_child"] = torch.empty(0, dtype=torch.int32, device="cuda")  # null pointer
    with pytest.raises(G.GbmError) as e:
        ctx.build_tree(gb.qm, q, sc, objective="reg:squarederror", max_depth=3,
                       grow_policy="lossguide", max_leaves=4, tree=t)
    assert e.value.code == -1
    ctx.check()


@pytest.mark.parametrize("seg", [1, 2])
@pytest.mark.parametrize("cfg,n,missing,carry", [("yearmsd", 30_000, 0.0, 0), ("bosch", 12_000, 0.0, 1),
                                                 ("epsilon", 6_000, 0.02, 0)])
def test_segment_histogram_modes(ctx, G, cfg, n, missing, carry, seg):
    """Wide data (several shared-memory feature groups): levels partitioned once + per-group
    segment histograms (GBM_OPT_SEGMENT_HIST 2) and the per-group fused kernel (1)."""
    ctx.set_option(ctx.SEGMENT_HIST, seg)
    ctx.set_option(ctx.CARRY_GRADIENTS, carry)
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n, missing=missing)
    ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=c.max_depth)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=c.max_bins, objective=c.objective,
                   max_depth=c.max_depth, base_margin=ob.base_margin)
    for _ in range(2):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.row_leaf.cpu().numpy(), ob.last["row_leaf"])
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    ctx.set_option(ctx.SEGMENT_HIST, 0)
    ctx.set_option(ctx.CARRY_GRADIENTS, 0)


@pytest.mark.parametrize("cfg,obj_override,D", [("higgs", None, 6), ("tiny", None, 3), ("yearmsd", None, 6),
                                                ("tiny", None, 0), ("bosch", None, 4)])
def test_fused_round_equals_separate_calls(ctx, G, cfg, obj_override, D):
    """gbm_build_tree_fused + gbm_gradients_from_stats (the default Booster round) against
    gbm_gradients + gbm_build_tree + gbm_update_margins, and both against the oracle."""
    c = W.CONFIGS[cfg]
    n = min(c.n_rows, 40_000)
    X, y = W.generate(cfg, 0, n, missing=0.02 if cfg == "tiny" else 0.0)
    ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=D)
    kw = dict(max_bins=c.max_bins, objective=c.objective, max_depth=D, base_margin=ob.base_margin)
    gf = G.Booster(ctx, dev(X), dev(y), fused=True, **kw)
    gs = G.Booster(ctx, dev(X), dev(y), fused=False, **kw)
    for _ in range(3):
        ot = ob.round()
        tf, ts = gf.round().to_numpy(), gs.round().to_numpy()
        _compare_tree(tf, ot)
        _compare_tree(ts, ot)
        np.testing.assert_array_equal(gf.qpair.cpu().numpy(), ob.last["qpair"])
        np.testing.assert_array_equal(gf.margin.cpu().numpy(), ob.margin)
        np.testing.assert_array_equal(gs.margin.cpu().numpy(), ob.margin)


@pytest.mark.parametrize("cfg,n,rounds,grow,missing", [
    ("higgs", 5_003, 70, "depthwise", 0.0),      # 70 trees: several tree chunks per row tile
    ("airline", 3_001, 12, "depthwise", 0.03),   # 13 features (not whole float4s), NaNs
    ("tiny", 700, 40, "lossguide", 0.05),        # linked trees, many chunks
    ("epsilon", 1_500, 3, "depthwise", 0.0),     # 2000 features: the gather predictor
])
def test_predict_many_trees_parity(ctx, G, cfg, n, rounds, grow, missing):
    """gbm_predict / gbm_predict_linked (Q7) after many rounds, on the training rows and
    on fresh rows with missing values: the margins equal the oracle's predictor bit for bit (fp64
    adds in tree order) and the staged-consistency identity predict(k trees) == margins."""
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n, n_rows=max(n, c.n_rows), missing=missing)
    kw = dict(max_bins=c.max_bins, objective=c.objective, max_depth=(c.max_depth if grow == "depthwise" else 7),
              eta=0.3)
    L = 10 if grow == "lossguide" else 0
    ob = O.Booster(X, y, grow_policy=grow, max_leaves=L, **kw)
    gb = G.Booster(ctx, dev(X), dev(y), base_margin=ob.base_margin, grow_policy=grow, max_leaves=L, **kw)
    for _ in range(rounds):
        ob.round()
        gb.round()
    np.testing.assert_array_equal(gb.predict(dev(X)).cpu().numpy().view(np.uint64), ob.margin.view(np.uint64))
    Xt, _ = W.generate(cfg, n, n + 2_345, n_rows=max(n + 2_345, c.n_rows), missing=0.1)
    np.testing.assert_array_equal(gb.predict(dev(Xt)).cpu().numpy().view(np.uint64),
                                  ob.predict(Xt).view(np.uint64))


@pytest.mark.parametrize("F,P", [(20, 15), (13, 15), (20, 30)])
def test_root_int32_exactness_bound(ctx, G, F, P):
    """The shared-memory bank columns are int32 and flushed per work item: with every row's pair at
    the extreme (|q| = 2^P) and one feature constant (every row in one bin), the root histogram
    over 10.5M rows must still be exact -- the work items (all root kernels, any shape) stay within
    MAX_CHUNK rows per accumulator copy between flushes.  Closed forms: the constant feature's
    only bin holds n * q, and every feature's bins sum to n * q."""
    n = 10_500_000
    rng = np.random.default_rng(7)
    X = rng.integers(0, 200, (n, F)).astype(np.float32)  # > 128 bins: 8-bit symbols (every root kernel)
    X[:, 0] = 3.0
    Xd = dev(X)
    qm = ctx.make_qmatrix(Xd, 256, 32)
    del Xd
    assert qm.bits == 8
    qg, qh = (1 << P) - 1, 1 << P
    q = torch.empty((n, 2), dtype=torch.int32, device="cuda")
    q[:, 0] = qg
    q[:, 1] = qh
    for shape in (0, 1, 2, 6, 7):
        ctx.set_option(ctx.ROOT_TENSOR, shape)
        h = ctx.build_histogram(qm, q, P).cpu().numpy()
        cp = qm.cut_ptr_h
        assert cp[1] - cp[0] == 1
        np.testing.assert_array_equal(h[cp[0]], [n * qg, n * qh])
        for f in range(F):
            np.testing.assert_array_equal(h[cp[f]:cp[f + 1]].sum(axis=0), [n * qg, n * qh])
    ctx.set_option(ctx.ROOT_TENSOR, 0)


@pytest.mark.parametrize("shape", [2, 5, 7])
@pytest.mark.parametrize("P", [15, 30])
@pytest.mark.parametrize("cfg,n,B", [("higgs", 40_016, None), ("airline", 30_000, None), ("yearmsd", 20_000, None),
                                     ("epsilon", 2_048, None), ("tiny", 2_000, 256), ("higgs", 9_008, 200),
                                     ("higgs", 100_048, None)])
def test_root_tensor_parity(ctx, G, cfg, n, B, P, shape):
    """The tensor-fed root (root_ct.cu: TMA tiles of the feature-major symbols, GBM_OPT_ROOT_TENSOR
    forced on): the root histogram bin for bin and whole rounds bit for bit vs the oracle, with a
    16-row tail batch (n = 16 mod 32), several feature groups, 1 / 2 / 4 rows per step (28, 13, 8
    features), wide accumulators (P = 30) and the 8-bit sentinel (B = 200); tiles of 32 / 64 / 128
    rows (shapes 2, 5, 7: partial tail tiles of 16..112 rows)."""
    ctx.set_option(ctx.ROOT_TENSOR, shape)
    c = W.CONFIGS[cfg]
    B = B or c.max_bins
    X, y = W.generate(cfg, 0, n, n_rows=max(n, c.n_rows), missing=0.02 if B == 200 else 0.0)
    qm, v, p, s, bits, words = _qm_from_oracle(G, X, B, 32)
    assert bits == 8
    ctx.transpose_symbols(qm)
    _, _, q, _ = O.gradients(c.objective, np.zeros(n), y, P)
    ref = O.node_histogram(words, X.shape[1], bits, 32, p, B, q, np.arange(n))
    ctx.profile(True, only=("hist_root", "hist_level"))
    got = ctx.build_histogram(qm, dev(q), P)
    prof = ctx.profile_read()
    ctx.profile(False)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)
    if not (shape == 7 and P == 30):  # 128-row tiles with four wide channels do not fit: other root
        assert prof["hist_root"]["launches"] == 1
    ob = O.Booster(X, y, max_bins=B, objective=c.objective, max_depth=4, grad_bits=P, eta=0.3)
    gb = G.Booster(ctx, dev(X), dev(y), max_bins=B, objective=c.objective, max_depth=4, grad_bits=P,
                   base_margin=ob.base_margin, eta=0.3)
    for _ in range(2):
        _compare_tree(gb.round().to_numpy(), ob.round())
        np.testing.assert_array_equal(gb.margin.cpu().numpy(), ob.margin)
    ctx.set_option(ctx.ROOT_TENSOR, 0)
