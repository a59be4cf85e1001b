"""Oracle pins for §2.3 tree construction (Alg. 1): histograms, EvaluateSplit, the
worked examples, brute-force exact greedy equivalence and worker invariance."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _quantised(X, B, row_align=32):
    v, p = O.cuts(X, B)
    s, mx = O.symbols(X, v, p, B)
    bits = O.symbol_bits(mx)
    return v, p, s, bits, O.pack(s, bits, row_align)


# ------------------------------------------------------------------ histograms
@pytest.mark.parametrize("seed", range(4))
def test_histogram_direct_summation_and_conservation(seed):
    X = W.random_matrix(seed, 700, 6, distinct=11, missing=0.15)
    B = 32
    v, p, s, bits, words = _quantised(X, B)
    rng = np.random.default_rng(seed)
    q = rng.integers(-2 ** 15, 2 ** 15, (700, 2)).astype(np.int32)
    q[:, 1] = np.abs(q[:, 1])
    rows = np.sort(rng.choice(700, 300, replace=False)).astype(np.int64)
    H = O.node_histogram(words, 6, bits, 32, p, B, q, rows)
    # library scatter-add (numpy.add.at) over the unpacked symbols
    ref = np.zeros_like(H)
    for f in range(6):
        sf = s[rows, f].astype(np.int64)
        ok = sf != B
        np.add.at(ref, p[f] + sf[ok], q[rows[ok]].astype(np.int64))
    np.testing.assert_array_equal(H, ref)
    # sum_b H[f][b] + missing mass == node totals, exactly (S:305 superseded, R14)
    T = q[rows].astype(np.int64).sum(0)
    for f in range(6):
        miss = q[rows[s[rows, f] == B]].astype(np.int64).sum(0)
        np.testing.assert_array_equal(H[p[f]:p[f + 1]].sum(0) + miss, T)
    # parent = left + right exactly, for any split of the row set
    left = rows[rng.random(rows.size) < 0.4]
    right = np.setdiff1d(rows, left)
    HL = O.node_histogram(words, 6, bits, 32, p, B, q, left)
    HR = O.node_histogram(words, 6, bits, 32, p, B, q, right)
    np.testing.assert_array_equal(HL + HR, H)
    # empty node -> all-zero histogram
    assert not O.node_histogram(words, 6, bits, 32, p, B, q, np.zeros(0, np.int64)).any()


def test_allreduce_shard_invariance():
    # Sum_k H(shard k) == H(all rows), exactly, for p in {1,2,4,8}
    X = W.random_matrix(9, 1001, 4, distinct=30)
    v, p, s, bits, words = _quantised(X, 16)
    q = np.random.default_rng(1).integers(0, 2 ** 15, (1001, 2)).astype(np.int32)
    full = O.node_histogram(words, 4, bits, 32, p, 16, q, np.arange(1001))
    for P in (1, 2, 4, 8):
        acc = np.zeros_like(full)
        for k in range(P):
            lo, hi = W.shard_range(1001, k, P)
            acc += O.node_histogram(words, 4, bits, 32, p, 16, q, np.arange(lo, hi))
        np.testing.assert_array_equal(acc, full)


# ------------------------------------------------------------------ EvaluateSplit
def test_two_bin_gain_spec():
    e = GOLD["spec_examples"]["two_bin_gain"]
    r = O.evaluate_split(np.array(e["hist"], np.int64), np.array([0, 2], np.int32), *e["totals"],
                         (0, 0), 0.0, 0.0, 0.0)
    assert r["split"] and r["bin"] == e["bin"] and Fraction(r["gain"]) == Fraction(e["gain"])


def test_uniform_histogram_is_leaf():
    hist = np.tile(np.array([[3, 2]], np.int64), (8, 1))
    r = O.evaluate_split(hist, np.array([0, 8], np.int32), 24, 16, (0, 0), 1.0, 0.0, 1.0)
    assert not r["split"] and r["gain"] <= 0


def test_min_child_weight_and_gamma():
    hist = np.array([[-4, 1], [4, 5]], np.int64)
    cp = np.array([0, 2], np.int32)
    assert O.evaluate_split(hist, cp, 0, 6, (0, 0), 0.0, 0.0, 1.0)["split"]
    assert not O.evaluate_split(hist, cp, 0, 6, (0, 0), 0.0, 0.0, 2.0)["split"]   # HL=1 < mcw
    g = O.evaluate_split(hist, cp, 0, 6, (0, 0), 0.0, 0.0, 0.0)["gain"]
    assert not O.evaluate_split(hist, cp, 0, 6, (0, 0), 0.0, g, 0.0)["split"]     # gamma >= gain


def _exact_gain(GL, HL, GR, HR, lam, gam):
    G, H = GL + GR, HL + HR
    return (GL * GL / (HL + lam) + GR * GR / (HR + lam) - G * G / (H + lam)) / 2 - gam


# ------------------------------------------------------------------ brute-force exact greedy
def _fp64_gain(GL, HL, GR, HR, G, H, lam, gam):
    # the R8 operation order, evaluated on directly-summed (not histogram) totals
    e = G * G
    e = e / (H + lam)
    a = GL * GL
    a = a / (HL + lam)
    c = GR * GR
    c = c / (HR + lam)
    d = a + c
    d = d - e
    d = 0.5 * d
    return d - gam


def brute_force_tree(X, q, scale, cut_values, cut_ptr, D, lam, gam, mcw, eta):
    """Exact greedy search over RAW values (no histograms, no prefix scan, no packing):
    every (feature, cut value, default direction) of every node, rows moved by v <= cut."""
    n, F = X.shape
    sg, sh = scale
    cap = (1 << (D + 1)) - 1
    out = {"kind": [0] * cap, "feature": [-1] * cap, "bin": [-1] * cap, "default_left": [0] * cap,
           "gain": [0.0] * cap, "weight": [0.0] * cap, "exact_gain": [None] * cap}
    row_leaf = [0] * n
    frontier = [(0, list(range(n)))]
    for depth in range(D + 1):
        nxt = []
        for k, rows in frontier:
            Tg = sum(int(q[i, 0]) for i in rows)
            Th = sum(int(q[i, 1]) for i in rows)
            G, H = math.ldexp(float(Tg), -sg), math.ldexp(float(Th), -sh)
            t = H + lam
            out["weight"][k] = 0.0 if t == 0 else (-(G / t)) * eta
            best = None
            if depth < D:
                for f in range(F):
                    for b in range(cut_ptr[f + 1] - cut_ptr[f]):
                        c = cut_values[cut_ptr[f] + b]
                        for dl in (True, False):
                            L = [i for i in rows if (dl if np.isnan(X[i, f]) else X[i, f] <= c)]
                            Lg = sum(int(q[i, 0]) for i in L)
                            Lh = sum(int(q[i, 1]) for i in L)
                            GL, HL = math.ldexp(float(Lg), -sg), math.ldexp(float(Lh), -sh)
                            GR = math.ldexp(float(Tg - Lg), -sg)
                            HR = math.ldexp(float(Th - Lh), -sh)
                            if not (HL >= mcw and HR >= mcw and HL + lam > 0 and HR + lam > 0):
                                continue
                            gain = _fp64_gain(GL, HL, GR, HR, G, H, lam, gam)
                            if best is None or gain > best[0]:
                                ex = _exact_gain(Fraction(Lg, 2 ** sg), Fraction(Lh, 2 ** sh),
                                                 Fraction(Tg - Lg, 2 ** sg),
                                                 Fraction(Th - Lh, 2 ** sh), Fraction(lam),
                                                 Fraction(gam))
                                best = (gain, f, b, dl, L, ex)
            if best is not None and best[0] > 0:
                gain, f, b, dl, L, ex = best
                out["kind"][k] = 1
                out["feature"][k], out["bin"][k], out["default_left"][k] = f, b, int(dl)
                out["gain"][k], out["exact_gain"][k] = gain, ex
                Ls = set(L)
                nxt.append((2 * k + 1, [i for i in rows if i in Ls]))
                nxt.append((2 * k + 2, [i for i in rows if i not in Ls]))
            else:
                out["kind"][k] = 2
                for i in rows:
                    row_leaf[i] = k
        frontier = nxt
    return out, np.array(row_leaf, np.int32)


def _random_case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(8, 257))
    F = int(rng.integers(1, 9))
    X = rng.integers(0, int(rng.integers(2, 9)), (n, F)).astype(np.float32)
    if seed % 2:
        X[rng.random((n, F)) < 0.1] = np.nan
    y = (rng.standard_normal(n) * 3 + X[:, 0] * 2).astype(np.float32)
    y = np.nan_to_num(y)
    return X, y


@pytest.mark.parametrize("seed", range(50))
def test_exact_greedy_equivalence(seed):
    # S:375 / S:582: with max_bins >= distinct values the histogram method is lossless, so the
    # oracle's tree equals an exact greedy search over raw values -- same splits, same gains.
    X, y = _random_case(seed)
    obj = "reg:squarederror" if seed % 3 else "binary:logistic"
    if obj == "binary:logistic":
        y = (y > np.median(y)).astype(np.float32)
    D = 3
    lam, gam, mcw, eta = (1.0, 0.0, 1.0, 0.3) if seed % 4 else (0.0, 0.5, 0.0, 1.0)
    v, p, s, bits, words = _quantised(X, 64)
    margin = np.full(X.shape[0], 0.25)
    _, _, q, sc = O.gradients(obj, margin, y, 15 if seed % 2 else 30)
    tree, row_leaf = O.build_tree(words, X.shape[0], X.shape[1], bits, 32, v, p, 64, q, sc, D,
                                  eta, lam, gam, mcw)
    ref, ref_leaf = brute_force_tree(X, q, sc, v, p, D, lam, gam, mcw, eta)
    for k in range(len(ref["kind"])):
        kk = int(tree["kind"][k])
        assert kk == ref["kind"][k], k
        if kk == 1:
            assert (tree["feature"][k], tree["bin"][k], tree["default_left"][k]) == \
                (ref["feature"][k], ref["bin"][k], ref["default_left"][k]), k
            assert tree["gain"][k] == ref["gain"][k]
            ex = ref["exact_gain"][k]
            assert abs(Fraction(tree["gain"][k]) - ex) <= abs(ex) * Fraction(1, 10 ** 12)
        if kk:
            assert tree["weight"][k] == ref["weight"][k]
    np.testing.assert_array_equal(row_leaf, ref_leaf)


@pytest.mark.parametrize("seed", range(10))
def test_worker_invariance(seed):
    # S:373 / S:583: p in {1,2,4,8} logical workers give identical trees and partitions
    X, y = W.generate("tiny", missing=0.05 * (seed % 2), seed_offset=seed)
    v, p, s, bits, words = _quantised(X, 16)
    _, _, q, sc = O.gradients("reg:squarederror", np.full(len(y), float(y.mean())), y, 15)
    ref = None
    for P in (1, 2, 4, 8):
        t, rl = O.build_tree(words, len(y), 8, bits, 32, v, p, 16, q, sc, 4, 0.3, 1.0, 0.0, 1.0, P)
        if ref is None:
            ref = (t, rl)
            continue
        for k in t:
            np.testing.assert_array_equal(t[k], ref[0][k])
        np.testing.assert_array_equal(rl, ref[1])


# ------------------------------------------------------------------ worked examples
def _tree_from_rows(rows, y, beta, lam, gam, mcw, eta, D, B, P=30):
    X = np.array(rows, np.float32)
    v, p, s, bits, words = _quantised(X, B)
    _, _, q, sc = O.gradients("reg:squarederror", np.full(len(y), float(beta)),
                              np.array(y, np.float32), P)
    t, rl = O.build_tree(words, len(y), X.shape[1], bits, 32, v, p, B, q, sc, D, eta, lam, gam, mcw)
    return X, v, p, t, rl


def _check_nodes(t, nodes, rel=Fraction(1, 10 ** 12)):
    for k, spec in nodes.items():
        k = int(k)
        if spec["kind"] == "split":
            assert t["kind"][k] == 1, k
            assert t["feature"][k] == spec["feature"] and t["bin"][k] == spec["bin"], k
            ex = Fraction(spec["gain"])
            assert abs(Fraction(t["gain"][k]) - ex) <= ex * rel, (k, t["gain"][k], ex)
        else:
            assert t["kind"][k] == 2, k
            ex = Fraction(spec["weight"])
            assert abs(Fraction(t["weight"][k]) - ex) <= abs(ex) * rel, (k, t["weight"][k], ex)


def test_worked_example_two_feature_additive():
    e = GOLD["two_feature_additive"]
    y = [1 + x0 + 4 * x1 for x0, x1 in e["rows"]]
    X, v, p, t, rl = _tree_from_rows(e["rows"], y, Fraction(e["base_margin"]), 1.0, 0.0, 1.0,
                                     1.0, e["max_depth"], e["max_bins"])
    _check_nodes(t, e["nodes"])
    assert float(t["threshold"][0]) == float(Fraction(e["nodes"]["0"]["threshold"]))
    m = O.update_margins(t["weight"], rl, np.full(8, 4.5))
    assert [Fraction(x) for x in m] == [Fraction(z) for z in e["predictions"]]
    assert np.array_equal(O.predict([t], 2, 4.5, X), m)


def test_worked_example_unbalanced_xor():
    e = GOLD["unbalanced_xor"]
    rows, y = [], []
    for x0, x1, yy, c in e["cells"]:
        rows += [[x0, x1]] * c
        y += [yy] * c
    X, v, p, t, rl = _tree_from_rows(rows, y, Fraction(1, 2), 0.0, 0.0, 0.0, 1.0, 2, 16)
    _check_nodes(t, e["nodes"])
    m = O.update_margins(t["weight"], rl, np.full(len(y), 0.5))
    assert m.tolist() == [float(v) for v in y]                      # training RMSE exactly 0


@pytest.mark.parametrize("case", [0, 1])
def test_worked_example_missing_default_direction(case):
    e = GOLD["missing_default_direction"]
    c = e["cases"][case]
    X = np.array([[float(x)] for x in e["x"]], np.float32)
    y = np.array([float(v) for v in c["y"]], np.float32)
    beta = float(np.mean(y.astype(np.float64)))
    v, p, s, bits, words = _quantised(X, 4)
    assert bits == e["bits"] and v.tolist() == [1, 2, 3, 4]
    _, _, q, sc = O.gradients("reg:squarederror", np.full(6, beta), y, 30)
    t, rl = O.build_tree(words, 6, 1, bits, 32, v, p, 4, q, sc, 1, 1.0, 1.0, 0.0, 1.0)
    assert t["kind"][0] == 1 and t["bin"][0] == c["bin"]
    assert float(t["threshold"][0]) == float(c["threshold"])
    assert bool(t["default_left"][0]) == c["default_left"]
    # base margin 20/3 is not a binary fraction -> gains/weights exact only to ~2^-26 (P=30)
    assert abs(t["gain"][0] - float(Fraction(c["gain"]))) < 1e-6
    for k, w in c["leaf_weights"].items():
        assert abs(t["weight"][int(k)] - float(Fraction(w))) < 1e-6
    assert rl.tolist() == c["row_leaf"]


def test_single_leaf_closed_form():
    # S:368 / S:477: max_depth = 0 -> one leaf, w = -G/(H+lambda)*eta
    X, y = W.generate("tiny")
    v, p, s, bits, words = _quantised(X, 16)
    _, _, q, sc = O.gradients("reg:squarederror", np.zeros(len(y)), y, 30)
    t, rl = O.build_tree(words, len(y), 8, bits, 32, v, p, 16, q, sc, 0, 0.3, 1.0, 0.0, 1.0)
    G = Fraction(int(q[:, 0].astype(np.int64).sum()), 2 ** sc[0])
    H = Fraction(int(q[:, 1].astype(np.int64).sum()), 2 ** sc[1])
    ex = -G / (H + 1) * Fraction(0.3)
    assert t["kind"][0] == 2 and abs(Fraction(t["weight"][0]) - ex) <= abs(ex) * Fraction(1, 10**12)
    assert not rl.any()


def test_all_gradients_zero_root_is_leaf():
    X = W.random_matrix(1, 50, 3)
    v, p, s, bits, words = _quantised(X, 16)
    q = np.zeros((50, 2), np.int32)
    q[:, 1] = 1
    t, rl = O.build_tree(words, 50, 3, bits, 32, v, p, 16, q, (15, 15), 3, 0.3, 1.0, 0.0, 0.0)
    assert t["kind"][0] == 2


@pytest.mark.parametrize("grow,p", [("depthwise", 1), ("depthwise", 3), ("lossguide", 2)])
def test_threaded_oracle_identical(grow, p):
    """Threaded mode: T row blocks with private int64 partial histograms, summed in
    block order, the cut sort over features, the per-row loops split -- identical cuts, symbols,
    gradients, trees, row partitions and margins for T = 1 and T = 5."""
    import workloads as W
    X, y = W.generate("higgs", 0, 30_011)
    runs = []
    for T in (1, 5):
        old = O.set_threads(T)
        try:
            b = O.Booster(X, y, max_bins=256, objective="binary:logistic",
                          max_depth=6 if grow == "depthwise" else 10, eta=0.3, p_workers=p,
                          grow_policy=grow, max_leaves=20 if grow == "lossguide" else 0)
            trees = [b.round() for _ in range(2)]
            runs.append((b.cut_values.copy(), b.cut_ptr.copy(), b.words.copy(), trees,
                         b.last["row_leaf"].copy(), b.last["qpair"].copy(), b.margin.copy(),
                         b.predict()))
        finally:
            O.set_threads(old)
    a, c = runs
    for i in (0, 1, 2, 4, 5, 6, 7):
        np.testing.assert_array_equal(a[i], c[i])
    for ta, tc in zip(a[3], c[3]):
        for k in ta:
            np.testing.assert_array_equal(ta[k], tc[k])
