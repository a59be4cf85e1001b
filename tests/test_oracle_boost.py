"""Oracle pins for the Fig. 1 pipeline: prediction (§2.4), margin update,
staged consistency, descent and learning sanity."""
import numpy as np
import pytest

import oracle as O
import workloads as W


def _stump(feature, thr, dl, wl, wr, D=1):
    cap = O.tree_capacity(D)
    t = {k: np.zeros(cap, dt) for k, dt in O.TREE_FIELDS}
    t["kind"][:3] = [1, 2, 2]
    t["feature"][0], t["threshold"][0], t["default_left"][0] = feature, thr, dl
    t["weight"][1], t["weight"][2] = wl, wr
    return t


def test_predict_spec_examples():
    X = np.array([[2.0], [2.5], [np.nan]], np.float32)
    assert O.predict([], 1, 0.7, X).tolist() == [0.7] * 3            # S:422 empty ensemble
    t = _stump(0, 2.0, 1, -1.0, 1.0)
    m = O.predict([t], 1, 0.5, X)
    assert m.tolist() == [-0.5, 1.5, -0.5]                            # S:423 boundary goes left
    perm = np.array([2, 0, 1])
    assert O.predict([t], 1, 0.5, X[perm]).tolist() == m[perm].tolist()


def test_update_margins_examples():
    w = np.array([0.0, 0.7, -0.2])
    m = O.update_margins(w, np.array([1], np.int32), np.array([1.0]))
    assert m.tolist() == [1.0 + 0.7]
    m0 = np.array([0.1, 0.2])
    assert O.update_margins(np.zeros(3), np.array([1, 2], np.int32), m0).tolist() == [0.1, 0.2]


@pytest.mark.parametrize("obj,missing", [("reg:squarederror", 0.0), ("binary:logistic", 0.05),
                                         ("reg:squarederror", 0.05)])
def test_staged_consistency_and_partition_equals_predict(obj, missing):
    # predict with the first k trees == cached margins after round k, bitwise, every k;
    # the training partition of every row == the leaf predict() reaches.
    X, y = W.generate("tiny", missing=missing)
    if obj == "binary:logistic":
        y = (y > np.median(y)).astype(np.float32)
    b = O.Booster(X, y, max_bins=16, objective=obj, max_depth=4, eta=0.3)
    for k in range(1, 31):
        t = b.round()
        np.testing.assert_array_equal(b.predict(n_trees=k), b.margin)
        # leaf reached by predict on this tree alone
        only = O.predict([t], 4, 0.0, X)
        np.testing.assert_array_equal(only, t["weight"][b.last["row_leaf"]])
        assert np.all(t["kind"][b.last["row_leaf"]] == O.KIND_LEAF)


def test_squared_error_descent():
    # S:478 / S:501: training RMSE never increases (Newton steps, h=1, eta<=1, gamma=0)
    X, y = W.generate("yearmsd", 0, 4000)
    b = O.Booster(X, y, max_bins=64, objective="reg:squarederror", max_depth=4, eta=0.3)
    rmse = []
    for r in range(40):
        b.round()
        rmse.append(np.sqrt(np.mean((b.margin - y) ** 2)))
    assert all(rmse[i + 1] <= rmse[i] + 1e-12 for i in range(len(rmse) - 1))
    assert rmse[-1] < 0.8 * rmse[0]


def test_separable_classification_accuracy():
    # separable synthetic classification reaches accuracy >= 0.95 within 100 rounds
    rng = np.random.default_rng(1)
    X = rng.standard_normal((10_000, 20)).astype(np.float32)
    y = ((X[:, 0] + 0.5 * X[:, 1] - 0.25 * X[:, 2]) > 0).astype(np.float32)
    b = O.Booster(X, y, max_bins=64, objective="binary:logistic", max_depth=4, eta=0.3)
    acc = 0.0
    for r in range(100):
        b.round()
        acc = np.mean((b.margin >= 0) == (y == 1))
        if acc >= 0.95:
            break
    assert acc >= 0.95


def test_determinism_two_runs_identical():
    X, y = W.generate("tiny", missing=0.05)
    ms = []
    for _ in range(2):
        b = O.Booster(X, y, max_bins=16, objective="reg:squarederror", max_depth=3)
        for _ in range(5):
            b.round()
        ms.append(b.margin.copy())
    np.testing.assert_array_equal(ms[0], ms[1])


def test_fixed_point_precision_quality():
    # R14: the default 15-bit per-row fixed point trains the same model quality as 30 bits
    # (the survey's reading) on a Higgs-shaped sample -- the design choice of DESIGN.md
    # "Gradient precision" is evidenced here.
    X, y = W.generate("higgs", 0, 20_000)
    losses = {}
    for P in (15, 30):
        b = O.Booster(X, y, max_bins=64, objective="binary:logistic", max_depth=5, eta=0.3,
                      grad_bits=P)
        for _ in range(15):
            b.round()
        p = 1 / (1 + np.exp(-b.margin))
        losses[P] = float(-np.mean(y * np.log(p) + (1 - y) * np.log(1 - p)))
    assert abs(losses[15] - losses[30]) <= 1e-5 * losses[30]
