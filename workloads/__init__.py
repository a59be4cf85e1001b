"""Seeded synthetic inputs shaped like the paper's workloads (Table 1).

This module is shared by the CPU oracle's tests and the CUDA path's tests/bench. It holds
NONE of the method's arithmetic: it only draws feature matrices X (fp32, NaN = missing) and
labels y (fp32) with numpy's counter-based Philox generator.  The recipe is documented in
DESIGN.md ("Input recipe"); the shapes are BASELINE.json's configs.

Generation is blocked: rows are produced in fixed blocks of BLOCK rows, block b drawn from
``Philox(key=(seed << 32) + b)``.  Any row range [lo, hi) can therefore be generated on its
own (one shard per rank) and is byte-identical to the same rows of the full
matrix, whatever the number of shards.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

BLOCK = 1 << 16
BASE_SEED = 11248  # seed = 11248 + config index


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    index: int
    n_rows: int
    n_features: int
    max_bins: int
    objective: str  # "reg:squarederror" | "binary:logistic"
    max_depth: int
    n_rounds: int
    gpus: str
    eta: float = 0.1
    reg_lambda: float = 1.0
    gamma: float = 0.0
    min_child_weight: float = 1.0

    @property
    def seed(self) -> int:
        return BASE_SEED + self.index


# BASELINE.json "configs", in order.
CONFIGS = {
    "tiny": Config("tiny", 0, 2_000, 8, 16, "reg:squarederror", 3, 1, "1"),
    "yearmsd": Config("yearmsd", 1, 515_000, 90, 256, "reg:squarederror", 6, 100, "1"),
    "higgs": Config("higgs", 2, 11_000_000, 28, 256, "binary:logistic", 6, 500, "1/2/4/8"),
    "epsilon": Config("epsilon", 3, 500_000, 2000, 256, "binary:logistic", 6, 100, "1/2/4/8"),
    "airline": Config("airline", 4, 115_000_000, 13, 256, "binary:logistic", 8, 500, "1/2/4/8"),
    # SURVEY.md §8(f) NEXT #4 (not a BASELINE.json config): Bosch-shaped sparse matrix
    # (1M x 968 binary) -- ~81% of the values missing, ~0.6% positives
    "bosch": Config("bosch", 5, 1_000_000, 968, 256, "binary:logistic", 6, 100, "1"),
}

# Airline-shaped cardinalities: Year, Month, DayofMonth, DayOfWeek, DepTime,
# ArrTime, UniqueCarrier (Zipf), FlightNum, ActualElapsedTime, Origin (Zipf), Dest (Zipf),
# Distance, Diverted.
AIRLINE_CARD = (22, 12, 31, 7, 1400, 1400, 30, 7500, 700, 350, 350, 1500, 2)


def shard_range(n_rows: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard of rank k: [floor(k n / p), floor((k+1) n / p))."""
    return (rank * n_rows) // world, ((rank + 1) * n_rows) // world


def _rng(seed: int, block: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=(seed << 32) + block))


def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


# --- per-config block generators: return (X float32 [m, F], y float32 [m]) -------------------

def _tiny(rng, m, F):
    X = rng.random((m, F), dtype=np.float64).astype(np.float32)
    w = np.array([1.0, -2.0, 3.0, 0.5, -1.0, 2.0, 0.0, 1.5])[:F]
    t = np.array([0.5, 0.3, 0.7, 0.2, 0.6, 0.4, 0.5, 0.8])[:F]
    y = (X.astype(np.float64) > t).astype(np.float64) @ w + 0.1 * rng.standard_normal(m)
    return X, y.astype(np.float32)


def _yearmsd(rng, m, F):
    lat = rng.standard_normal((m, 16))
    mix = _rng(BASE_SEED + 1, 1 << 30).standard_normal((16, F)) / 4.0
    X = lat @ mix + 0.5 * rng.standard_normal((m, F))
    X[:, 12:] = X[:, 12:] * np.abs(X[:, :1]) * 3.0  # "covariance"-like heavier tails
    X = X.astype(np.float32)
    s = np.tanh(lat[:, 0] + 0.5 * lat[:, 1] * lat[:, 2]) + 0.3 * np.sin(2 * lat[:, 3])
    back = 45.0 * _sigmoid(-2.0 * s) ** 2 + np.abs(rng.standard_normal(m)) * 4.0
    y = np.clip(np.floor(2011.0 - back), 1922, 2011)
    return X, y.astype(np.float32)


def _higgs(rng, m, F):
    X = np.empty((m, F), dtype=np.float64)
    lat = rng.standard_normal(m)  # signal-ish latent
    X[:, 0] = rng.lognormal(0.0 + 0.2 * lat, 0.5, m)        # lepton pT
    X[:, 1] = rng.standard_normal(m) * 1.2                   # lepton eta
    X[:, 2] = rng.uniform(-math.pi, math.pi, m)              # lepton phi
    X[:, 3] = rng.lognormal(0.0 + 0.1 * lat, 0.6, m)        # missing ET
    X[:, 4] = rng.uniform(-math.pi, math.pi, m)              # MET phi
    for j in range(4):                                       # 4 jets x (pT, eta, phi, b-tag)
        c = 5 + 4 * j
        X[:, c] = rng.lognormal(0.1 * lat, 0.55, m)
        X[:, c + 1] = rng.standard_normal(m) * 1.4
        X[:, c + 2] = rng.uniform(-math.pi, math.pi, m)
        p = _sigmoid(0.4 * lat - 0.5)
        u = rng.random(m)
        X[:, c + 3] = np.where(u < p * 0.6, 2.1730, np.where(u < p, 1.0865, 0.0))  # 3 values
    for j in range(7):                                       # high-level: positive skewed
        X[:, 21 + j] = rng.gamma(2.0 + 0.3 * j, 0.5, m) * np.exp(0.15 * lat)
    logit = 0.9 * lat + 0.5 * (X[:, 24] - 1.3) - 0.3 * (X[:, 21] - 1.0) + 0.2
    y = (rng.random(m) < _sigmoid(logit)).astype(np.float32)
    return X.astype(np.float32), y


_EPS_W = None


def _epsilon(rng, m, F):
    global _EPS_W
    if _EPS_W is None or _EPS_W.shape[0] != F:
        _EPS_W = _rng(BASE_SEED + 3, 1 << 30).standard_normal(F)
    X = rng.standard_normal((m, F))
    X /= np.linalg.norm(X, axis=1, keepdims=True)
    z = X @ _EPS_W + 0.3 * rng.standard_normal(m)
    y = (z > 0).astype(np.float32)
    return X.astype(np.float32), y


def _zipf_codes(rng, m, card, a=1.3):
    r = np.arange(1, card + 1, dtype=np.float64)
    p = r ** -a
    p /= p.sum()
    return rng.choice(card, size=m, p=p)


def _airline(rng, m, F):
    X = np.empty((m, F), dtype=np.float64)
    X[:, 0] = 1987 + rng.integers(0, 22, m)
    X[:, 1] = 1 + rng.integers(0, 12, m)
    X[:, 2] = 1 + rng.integers(0, 31, m)
    X[:, 3] = 1 + rng.integers(0, 7, m)
    dep = rng.integers(0, 1400, m)
    X[:, 4] = (dep // 60) * 100 + dep % 60 + 500       # hhmm-like, ~1400 distinct
    arr = (dep + rng.integers(30, 400, m)) % 1400
    X[:, 5] = (arr // 60) * 100 + arr % 60 + 500
    X[:, 6] = _zipf_codes(rng, m, 30)
    X[:, 7] = rng.integers(1, 7501, m)
    X[:, 8] = 20 + rng.integers(0, 700, m)
    X[:, 9] = _zipf_codes(rng, m, 350)
    X[:, 10] = _zipf_codes(rng, m, 350)
    X[:, 11] = 30 + rng.integers(0, 1500, m)
    X[:, 12] = (rng.random(m) < 0.003).astype(np.float64)
    logit = (-0.35 + 0.0012 * (dep - 700) + 0.15 * (X[:, 1] > 10) + 0.08 * (X[:, 6] < 3)
             - 0.05 * (X[:, 3] > 5) + 0.5 * rng.standard_normal(m))
    y = (rng.random(m) < _sigmoid(logit)).astype(np.float32)
    return X.astype(np.float32), y


_BOSCH_W = None


def _bosch(rng, m, F):
    """Production-line measurements: ~81% missing (whole stations absent per part), values with a
    few distinct levels for some features, rare failures (~0.6%) driven by a few measurements."""
    global _BOSCH_W
    if _BOSCH_W is None or _BOSCH_W[0].shape[0] != F:
        r0 = _rng(BASE_SEED + 5, 1 << 30)
        _BOSCH_W = (r0.standard_normal(F) * (r0.random(F) < 0.05), r0.integers(2, 40, F),
                    r0.random(F) < 0.2)
    w, levels, coarse = _BOSCH_W
    X = rng.standard_normal((m, F), dtype=np.float32)
    X[:, coarse] = np.round(X[:, coarse] * levels[coarse] / 4) / (levels[coarse] / 4)
    station = rng.random((m, (F + 47) // 48), dtype=np.float32) < 0.19   # ~19% of stations visited
    present = np.repeat(station, 48, axis=1)[:, :F]
    z = np.where(present, X, 0.0).astype(np.float64) @ w - 7.0 + 0.5 * rng.standard_normal(m)
    X[~present] = np.nan
    y = (rng.random(m) < _sigmoid(z)).astype(np.float32)
    return X, y


_GEN = {"tiny": _tiny, "yearmsd": _yearmsd, "higgs": _higgs, "epsilon": _epsilon,
        "airline": _airline, "bosch": _bosch}


def generate(name: str, lo: int = 0, hi: int | None = None, *, n_rows: int | None = None,
             missing: float = 0.0, seed_offset: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Rows [lo, hi) of config `name` (default: all rows).

    `n_rows` overrides the config's row count (a smaller sample of the same distribution:
    the first n_rows rows of the full matrix).  `missing` > 0 replaces that fraction of
    entries by NaN (the sparse/missing-value variant, SURVEY.md §8(d) tiny row).
    """
    cfg = CONFIGS[name]
    n = cfg.n_rows if n_rows is None else n_rows
    hi = n if hi is None else hi
    if not (0 <= lo <= hi <= n):
        raise ValueError(f"bad row range [{lo}, {hi}) for n={n}")
    F = cfg.n_features
    seed = cfg.seed + 1000 * seed_offset
    X = np.empty((hi - lo, F), dtype=np.float32)
    y = np.empty(hi - lo, dtype=np.float32)
    b0, b1 = lo // BLOCK, (hi + BLOCK - 1) // BLOCK
    for b in range(b0, b1):
        rng = _rng(seed, b)
        Xb, yb = _GEN[name](rng, BLOCK, F)
        if missing > 0.0:
            mrng = _rng(seed + 7, b)
            Xb[mrng.random(Xb.shape) < missing] = np.nan
        s, e = max(lo, b * BLOCK), min(hi, (b + 1) * BLOCK)
        X[s - lo:e - lo] = Xb[s - b * BLOCK:e - b * BLOCK]
        y[s - lo:e - lo] = yb[s - b * BLOCK:e - b * BLOCK]
    return X, y


def base_margin(objective: str, y_full_mean: float | None = None) -> float:
    """Base margin beta (SURVEY.md §8(c) ambiguity 12): 0 for logistic, label mean for
    squared error (the caller computes the mean on the host in row order)."""
    if objective == "binary:logistic":
        return 0.0
    return float(y_full_mean)


def random_matrix(seed: int, n: int, F: int, *, distinct: int | None = None,
                  missing: float = 0.0, dtype=np.float32) -> np.ndarray:
    """Small random matrices for property tests: `distinct` caps the number of distinct
    values per column (integers 0..distinct-1) so ties and lossless binning are exercised."""
    rng = _rng(seed, 0)
    if distinct is None:
        X = rng.standard_normal((n, F)).astype(dtype)
    else:
        X = rng.integers(0, distinct, (n, F)).astype(dtype)
    if missing > 0.0:
        X[rng.random((n, F)) < missing] = np.nan
    return X
