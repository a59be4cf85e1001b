"""Oracle pins for §2.5 gradient evaluation (Eq. 1-2) and the fixed point (R14)."""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def test_spec_gradient_examples():
    ex = GOLD["spec_examples"]["gradients"]
    for cite, e in ex.items():
        obj = "reg:squarederror" if cite == "S:257" else "binary:logistic"
        g, h, _, _ = O.gradients(obj, np.array([e["yhat"]], float), np.array([e["y"]], np.float32),
                                 30)
        assert Fraction(g[0]) == Fraction(e["g"]) and Fraction(h[0]) == Fraction(e["h"]), cite


def test_det_exp_within_one_ulp_of_libm():
    rng = np.random.default_rng(1)
    t = np.concatenate([-rng.random(20000) * 745.0, -rng.random(2000) * 1e-3, [0.0, -1e-300]])
    worst = 0
    for x in t:
        a, b = O.det_exp(x), math.exp(x)
        if b == 0.0:
            assert a == 0.0 or a < 5e-324 * 4
            continue
        worst = max(worst, abs(a - b) / math.ulp(b))
    assert worst <= 1.0
    assert O.det_exp(-746.0) == 0.0 and O.det_exp(0.0) == 1.0


def test_sigmoid_properties():
    assert O.sigmoid(0.0) == 0.5
    assert O.sigmoid(50.0) == 1.0                                  # binary64 saturation (App. C)
    assert O.sigmoid(36.0) < 1.0 and O.sigmoid(37.0) == 1.0        # saturation point ~36.8
    rng = np.random.default_rng(2)
    for x in rng.standard_normal(2000) * 10:
        assert abs(O.sigmoid(-x) - (1.0 - O.sigmoid(x))) <= 1e-15
    for x in np.linspace(-700, 700, 301):
        assert 0.0 <= O.sigmoid(x) <= 1.0


def _logloss(m, y):
    m, y = float(m), float(y)
    p = 1.0 / (1.0 + math.exp(-m))
    return -(y * math.log(p) + (1 - y) * math.log(1 - p))


def test_logistic_finite_differences():
    # S:250 / S:585: g matches d/dm of the log loss within 1e-4, h the 2nd difference within 1e-3
    rng = np.random.default_rng(3)
    m = rng.standard_normal(1000) * 3
    y = (rng.random(1000) < 0.5).astype(np.float32)
    g, h, _, _ = O.gradients("binary:logistic", m, y, 30)
    eps = 1e-4
    for i in range(1000):
        fd1 = (_logloss(m[i] + eps, y[i]) - _logloss(m[i] - eps, y[i])) / (2 * eps)
        fd2 = (_logloss(m[i] + eps, y[i]) - 2 * _logloss(m[i], y[i]) +
               _logloss(m[i] - eps, y[i])) / eps ** 2
        assert abs(g[i] - fd1) < 1e-4 and abs(h[i] - fd2) < 1e-3
        assert 0.0 <= h[i] <= 0.25


def test_squared_error_finite_differences():
    rng = np.random.default_rng(4)
    m = rng.standard_normal(1000) * 10
    y = rng.standard_normal(1000).astype(np.float32) * 10
    g, h, _, _ = O.gradients("reg:squarederror", m, y, 30)
    for i in range(1000):
        f = lambda z: 0.5 * (z - float(y[i])) ** 2  # noqa: E731
        eps = 1e-3
        assert abs(g[i] - (f(m[i] + eps) - f(m[i] - eps)) / (2 * eps)) < 1e-4
        assert h[i] == 1.0


@pytest.mark.parametrize("P", [1, 8, 15, 30])
@pytest.mark.parametrize("obj", ["binary:logistic", "reg:squarederror"])
def test_fixed_point_bounds(P, obj):
    rng = np.random.default_rng(P)
    n = 5000
    m = rng.standard_normal(n) * 4
    y = ((rng.random(n) < 0.4).astype(np.float32) if obj == "binary:logistic"
         else (rng.standard_normal(n) * 50).astype(np.float32))
    g, h, q, (sg, sh) = O.gradients(obj, m, y, P)
    for v, qq, s in ((g, q[:, 0], sg), (h, q[:, 1], sh)):
        M = np.abs(v).max()
        E = math.frexp(M)[1]
        assert s == P - E and M < 2.0 ** E
        # per-row error of round-half-even is at most half a quantum
        err = np.abs(qq.astype(np.float64) * 2.0 ** -s - v)
        assert np.all(err <= 2.0 ** -(s + 1))
        assert np.abs(qq).max() <= 2 ** P and np.abs(qq).max() > 2 ** (P - 2)
        # closed-form bound on sums: |sum q 2^-s - sum v| <= n 2^-(s+1)
        assert abs(qq.astype(np.int64).sum() * 2.0 ** -s - v.sum()) <= n * 2.0 ** -(s + 1) + 1e-9


def test_fixed_point_round_half_even_and_zero():
    # g values on exact half quanta round to even: with P=2, max|g|=3.5 (E=2) -> s=0
    m = np.array([0.0, 0.0, 0.0, 0.0], float)
    y = np.array([-0.5, -1.5, -2.5, -3.5], np.float32)
    g, _, q, (sg, _) = O.gradients("reg:squarederror", m, y, 2)
    assert sg == 0 and q[:, 0].tolist() == [0, 2, 2, 4]
    _, _, q, sc = O.gradients("reg:squarederror", np.ones(3), np.ones(3, np.float32), 15)
    assert q[:, 0].tolist() == [0, 0, 0] and sc[0] == 15


def test_label_domain_error():
    with pytest.raises(O.OracleError) as e:
        O.gradients("binary:logistic", np.zeros(3), np.array([0, 1, 3], np.float32), 15)
    assert e.value.code == -4
