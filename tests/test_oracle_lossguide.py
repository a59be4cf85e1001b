"""Oracle pins for loss-guided growth ("prioritise expanding nodes with a higher reduction
in the objective function"; readings R25-R27 in DESIGN.md).

The pins do not retype the loop: (1) with a leaf budget >= 2^D the priority order cannot change
which nodes are split, so the tree equals the (separately pinned) depth-wise tree up to node
numbering; (2) max_leaves = 2 is the depth-1 stump; (3) the greedy prefix property -- the tree
with L leaves is the tree with L-1 leaves plus ONE expansion, of the open leaf whose best split
gain (computed here from numpy histograms of the leaf's rows and the pinned EvaluateSplit) is
the largest, ties to the smaller id; (4) the leaf budget; (5) worker invariance; (6) the
linked-tree prediction reproduces the training margins."""
import numpy as np
import pytest

import oracle as O
import workloads as W


def _case(seed, n=600, F=5, missing=0.1, objective="reg:squarederror"):
    X = W.random_matrix(seed, n, F, distinct=9, missing=missing)
    rng = np.random.default_rng(1000 + seed)
    if objective == "binary:logistic":
        y = (rng.random(n) < 1 / (1 + np.exp(-np.nan_to_num(X[:, 0] - X[:, 1] / 2)))).astype(np.float32)
    else:
        y = (np.nan_to_num(X[:, 0]) * 0.7 - np.nan_to_num(X[:, 2]) ** 2 / 5 +
             rng.standard_normal(n)).astype(np.float32)
    return X, y


def _same_tree_by_path(td, kd, tl, kl, left_of_l):
    """Walk the heap tree td from heap id kd and the linked tree tl from id kl in lockstep."""
    assert td["kind"][kd] == tl["kind"][kl]
    for f in ("feature", "bin", "default_left", "sum_qg", "sum_qh"):
        assert td[f][kd] == tl[f][kl], f
    for f in ("gain", "weight", "threshold"):
        assert td[f][kd] == tl[f][kl], f  # same arithmetic on the same sums: bit-identical
    if td["kind"][kd] == O.KIND_SPLIT:
        c = left_of_l[kl]
        _same_tree_by_path(td, 2 * kd + 1, tl, c, left_of_l)
        _same_tree_by_path(td, 2 * kd + 2, tl, c + 1, left_of_l)
    else:
        assert left_of_l[kl] == -1


@pytest.mark.parametrize("seed,D,objective,p", [(0, 3, "reg:squarederror", 1),
                                                 (1, 4, "binary:logistic", 1),
                                                 (2, 2, "reg:squarederror", 3),
                                                 (3, 5, "binary:logistic", 2)])
def test_unbounded_budget_equals_depthwise(seed, D, objective, p):
    X, y = _case(seed, objective=objective)
    kw = dict(max_bins=8, objective=objective, max_depth=D, p_workers=p)
    bd = O.Booster(X, y, **kw)
    bl = O.Booster(X, y, grow_policy="lossguide", max_leaves=2 ** D + 3, **kw)
    for _ in range(3):
        td, tl = bd.round(), bl.round()
        _same_tree_by_path(td, 0, tl, 0, tl["left_child"])
        assert np.array_equal(bd.margin, bl.margin)
    assert np.array_equal(bd.predict(), bl.predict())


def test_two_leaves_is_the_stump():
    X, y = _case(7)
    bd = O.Booster(X, y, max_bins=16, objective="reg:squarederror", max_depth=1)
    bl = O.Booster(X, y, max_bins=16, objective="reg:squarederror", max_depth=12,
                   grow_policy="lossguide", max_leaves=2)
    td, tl = bd.round(), bl.round()
    _same_tree_by_path(td, 0, tl, 0, tl["left_child"])
    assert np.array_equal(bd.margin, bl.margin)


def test_one_leaf_budget_is_the_root_leaf():
    X, y = _case(8)
    bl = O.Booster(X, y, max_bins=16, objective="reg:squarederror", max_depth=6,
                   grow_policy="lossguide", max_leaves=1)
    t = bl.round()
    assert list(t["kind"]) == [O.KIND_LEAF] and t["left_child"][0] == -1
    Tg, Th = int(bl.last["qpair"][:, 0].sum()), int(bl.last["qpair"][:, 1].sum())
    assert t["sum_qg"][0] == Tg and t["sum_qh"][0] == Th
    assert t["weight"][0] == O.leaf_weight(Tg, Th, bl.last["scale"], 1.0, 0.3)


def _leaf_gain(bl, row_leaf, k, q, sc):
    """Best split of leaf k from scratch: numpy histogram of its rows + the pinned EvaluateSplit."""
    rows = np.nonzero(row_leaf == k)[0]
    H = np.zeros((int(bl.cut_ptr[-1]), 2), np.int64)
    for f in range(bl.F):
        s = bl.sym[rows, f].astype(np.int64)
        ok = s != bl.max_bins
        np.add.at(H, bl.cut_ptr[f] + s[ok], q[rows[ok]].astype(np.int64))
    Tg, Th = int(q[rows, 0].astype(np.int64).sum()), int(q[rows, 1].astype(np.int64).sum())
    r = O.evaluate_split(H, bl.cut_ptr, Tg, Th, sc, 1.0, 0.0, 1.0)
    return r


def _depths(t):
    d = {0: 0}
    for k in range(t["kind"].shape[0]):
        if t["kind"][k] == O.KIND_SPLIT:
            c = int(t["left_child"][k])
            d[c] = d[c + 1] = d[k] + 1
    return d


@pytest.mark.parametrize("seed", range(3))
def test_greedy_prefix_property(seed):
    """tree(L) = tree(L-1) + the expansion of tree(L-1)'s best open leaf (R25, R26)."""
    X, y = _case(20 + seed, n=500, F=4)
    D = 5
    mk = lambda L: O.Booster(X, y, max_bins=8, objective="reg:squarederror", max_depth=D,
                             grow_policy="lossguide", max_leaves=L)
    prev = mk(1)
    tp = prev.round()
    q, sc = prev.last["qpair"], prev.last["scale"]
    for L in range(2, 12):
        cur = mk(L)
        tc = cur.round()
        assert np.array_equal(cur.last["qpair"], q)
        n_leaves = int((tc["kind"] == O.KIND_LEAF).sum())
        assert n_leaves <= L
        # the open leaves of tree(L-1) and their independently computed best splits
        depth = _depths(tp)
        best = None
        for k in np.nonzero(tp["kind"] == O.KIND_LEAF)[0]:
            if depth[int(k)] >= D:
                continue
            r = _leaf_gain(prev, prev.last["row_leaf"], int(k), q, sc)
            if r["split"] and (best is None or r["gain"] > best[1]):
                best = (int(k), r["gain"], r)
        if best is None:  # nothing left to split: the budget is not binding any more
            assert n_leaves == int((tp["kind"] == O.KIND_LEAF).sum())
            break
        k, g, r = best
        assert n_leaves == L
        j = L - 2  # the last expansion creates 2j+1, 2j+2 (R27)
        assert tc["left_child"][k] == 2 * j + 1
        assert tc["kind"][k] == O.KIND_SPLIT and tc["feature"][k] == r["feature"]
        assert tc["bin"][k] == r["bin"] and tc["default_left"][k] == r["default_left"]
        assert tc["gain"][k] == g
        # every other node of tree(L-1) is unchanged
        for kk in range(tp["kind"].shape[0]):
            if kk == k:
                continue
            for f in ("kind", "feature", "bin", "left_child", "sum_qg", "sum_qh", "weight"):
                assert tp[f][kk] == tc[f][kk], (L, kk, f)
        prev, tp = cur, tc


@pytest.mark.parametrize("seed", range(2))
def test_worker_invariance_lossguide(seed):
    X, y = _case(40 + seed, missing=0.2, objective="binary:logistic")
    kw = dict(max_bins=8, objective="binary:logistic", max_depth=8, grow_policy="lossguide",
              max_leaves=9)
    b1, b3 = O.Booster(X, y, p_workers=1, **kw), O.Booster(X, y, p_workers=3, **kw)
    for _ in range(2):
        t1, t3 = b1.round(), b3.round()
        for f in t1:
            assert np.array_equal(t1[f], t3[f]), f
    assert np.array_equal(b1.margin, b3.margin)


def test_budget_binds_and_prediction_matches_training_margins():
    X, y = _case(50, n=900, F=6)
    b = O.Booster(X, y, max_bins=16, objective="reg:squarederror", max_depth=10,
                  grow_policy="lossguide", max_leaves=6)
    for _ in range(4):
        t = b.round()
        assert int((t["kind"] == O.KIND_LEAF).sum()) == 6
        assert int((t["kind"] == O.KIND_SPLIT).sum()) == 5
        # row_leaf points at leaves; conservation at every split node
        assert np.all(t["kind"][b.last["row_leaf"]] == O.KIND_LEAF)
        for k in np.nonzero(t["kind"] == O.KIND_SPLIT)[0]:
            c = t["left_child"][k]
            assert t["sum_qg"][c] + t["sum_qg"][c + 1] == t["sum_qg"][k]
            assert t["sum_qh"][c] + t["sum_qh"][c + 1] == t["sum_qh"][k]
    assert np.array_equal(b.predict(), b.margin)
