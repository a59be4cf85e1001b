"""CPU oracle for the gbm hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference`` leg may
import this package.  It wraps ``oracle/oracle.c`` (plain C99, fp64, ``-O2 -ffp-contract=off``)
with numpy-friendly functions; the C file cites the PAPER.md / SPEC.md passage each function
follows.  It shares no code with ``paper_1806_11248_b200`` (the CUDA path) and never imports it.

Functions without an independent pin are marked "parity unpinned" in their docstring and in
DESIGN.md; at present every function has at least one pin (tests/test_oracle_*.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

SQUARED_ERROR, LOGISTIC = 0, 1
OBJECTIVES = {"reg:squarederror": SQUARED_ERROR, "binary:logistic": LOGISTIC}
KIND_ABSENT, KIND_SPLIT, KIND_LEAF = 0, 1, 2


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where} failed with code {code}")
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fno-fast-math",
                               "-fopenmp", "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _P(t):
    return C.POINTER(t)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            i32, i64, f64, f32 = C.c_int32, C.c_int64, C.c_double, C.c_float
            sig = {
                "oracle_symbol_bits": (C.c_int, [i32]),
                "oracle_set_threads": (C.c_int, [i32]),
                "oracle_cuts": (C.c_int, [_P(f32), i64, i32, i32, _P(f32), _P(i32)]),
                "oracle_symbols": (C.c_int, [_P(f32), i64, i32, _P(f32), _P(i32), i32,
                                             _P(C.c_uint16), _P(i32)]),
                "oracle_packed_words": (i64, [i64, i32, i32, i32]),
                "oracle_pack": (C.c_int, [_P(C.c_uint16), i64, i32, i32, i32, _P(C.c_uint32),
                                          i64]),
                "oracle_unpack": (C.c_int, [_P(C.c_uint32), i64, i32, i32, i32,
                                            _P(C.c_uint16)]),
                "oracle_det_exp": (f64, [f64]),
                "oracle_sigmoid": (f64, [f64]),
                "oracle_gradients": (C.c_int, [i32, _P(f64), _P(f32), i64, i32, _P(f64),
                                               _P(f64), _P(i32), _P(i32)]),
                "oracle_node_histogram": (C.c_int, [_P(C.c_uint32), i32, i32, i32, _P(i32), i32,
                                                    _P(i32), _P(i64), i64, _P(i64)]),
                "oracle_evaluate_split": (C.c_int, [_P(i64), i32, _P(i32), i64, i64, i32, i32,
                                                    f64, f64, f64, _P(i32), _P(f64), _P(i64)]),
                "oracle_leaf_weight": (f64, [i64, i64, i32, i32, f64, f64]),
                "oracle_build_tree": (C.c_int, [_P(C.c_uint32), i64, i32, i32, i32, _P(f32),
                                                _P(i32), i32, _P(i32), _P(i32), i32, _P(f64),
                                                i32, _P(C.c_int8), _P(i32), _P(i32), _P(f32),
                                                _P(C.c_int8), _P(f64), _P(f64), _P(i64),
                                                _P(i64), _P(i32)]),
                "oracle_build_tree_lossguide": (C.c_int, [_P(C.c_uint32), i64, i32, i32, i32,
                                                          _P(f32), _P(i32), i32, _P(i32), _P(i32),
                                                          i32, i32, _P(f64), i32, _P(C.c_int8),
                                                          _P(i32), _P(i32), _P(f32), _P(C.c_int8),
                                                          _P(f64), _P(f64), _P(i64), _P(i64),
                                                          _P(i32), _P(i32)]),
                "oracle_predict_linked": (C.c_int, [i32, i64, _P(C.c_int8), _P(i32), _P(f32),
                                                    _P(C.c_int8), _P(i32), _P(f64), f64, _P(f32),
                                                    i64, i32, _P(f64)]),
                "oracle_update_margins": (C.c_int, [_P(f64), _P(i32), i64, _P(f64)]),
                "oracle_predict": (C.c_int, [i32, i32, _P(C.c_int8), _P(i32), _P(f32),
                                             _P(C.c_int8), _P(f64), f64, _P(f32), i64, i32,
                                             _P(f64)]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    assert a.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
    return a.ctypes.data_as(_P(ct))


def _check(code: int, where: str):
    if code != 0:
        raise OracleError(code, where)


# ---------------------------------------------------------------------------------------------
def set_threads(t: int) -> int:
    """Threaded mode (T row blocks with private int64 partials); returns the
    previous thread count.  Results do not depend on T (exact sums, per-row values)."""
    return int(lib().oracle_set_threads(int(t)))


def symbol_bits(max_symbol: int) -> int:
    """max(1, ceil(log2(max_symbol + 1))) -- P:30 read as R1."""
    return lib().oracle_symbol_bits(int(max_symbol))


def cuts(X: np.ndarray, max_bins: int) -> tuple[np.ndarray, np.ndarray]:
    """Exact rank-rule cuts (R5).  Returns (cut_values fp32 [TB], cut_ptr int32 [F+1])."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, F = X.shape
    vals = np.zeros(max(1, F * max_bins), dtype=np.float32)
    ptr = np.zeros(F + 1, dtype=np.int32)
    _check(lib().oracle_cuts(_ptr(X, C.c_float), n, F, max_bins, _ptr(vals, C.c_float),
                             _ptr(ptr, C.c_int32)), "oracle_cuts")
    return vals[: ptr[-1]].copy(), ptr


def symbols(X: np.ndarray, cut_values: np.ndarray, cut_ptr: np.ndarray,
            max_bins: int) -> tuple[np.ndarray, int]:
    """Bin map: uint16 [n, F], sentinel = max_bins for NaN; and the max symbol."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, F = X.shape
    cv = np.ascontiguousarray(cut_values, dtype=np.float32)
    if cv.size == 0:
        cv = np.zeros(1, np.float32)
    cp = np.ascontiguousarray(cut_ptr, dtype=np.int32)
    sym = np.zeros((n, F), dtype=np.uint16)
    mx = C.c_int32(0)
    _check(lib().oracle_symbols(_ptr(X, C.c_float), n, F, _ptr(cv, C.c_float),
                                _ptr(cp, C.c_int32), max_bins, _ptr(sym, C.c_uint16),
                                C.byref(mx)), "oracle_symbols")
    return sym, mx.value


def packed_words(n: int, F: int, bits: int, row_align_bits: int = 0) -> int:
    w = lib().oracle_packed_words(n, F, bits, row_align_bits)
    if w < 0:
        raise OracleError(int(w), "oracle_packed_words")
    return int(w)


def pack(sym: np.ndarray, bits: int, row_align_bits: int = 0) -> np.ndarray:
    """Bit-pack (layout R3)."""
    sym = np.ascontiguousarray(sym, dtype=np.uint16)
    n, F = sym.shape
    nw = packed_words(n, F, bits, row_align_bits)
    words = np.zeros(nw, dtype=np.uint32)
    _check(lib().oracle_pack(_ptr(sym, C.c_uint16), n, F, bits, row_align_bits,
                             _ptr(words, C.c_uint32), nw), "oracle_pack")
    return words


def unpack(words: np.ndarray, n: int, F: int, bits: int, row_align_bits: int = 0) -> np.ndarray:
    words = np.ascontiguousarray(words, dtype=np.uint32)
    sym = np.zeros((n, F), dtype=np.uint16)
    _check(lib().oracle_unpack(_ptr(words, C.c_uint32), n, F, bits, row_align_bits,
                               _ptr(sym, C.c_uint16)), "oracle_unpack")
    return sym


def det_exp(t: float) -> float:
    return lib().oracle_det_exp(float(t))


def sigmoid(x: float) -> float:
    return lib().oracle_sigmoid(float(x))


def gradients(objective, margin: np.ndarray, label: np.ndarray, P: int):
    """Eq. 1-2 + fixed point (R14).  Returns (g, h, qpair int32 [n,2], (s_g, s_h))."""
    obj = OBJECTIVES.get(objective, objective)
    margin = np.ascontiguousarray(margin, dtype=np.float64)
    label = np.ascontiguousarray(label, dtype=np.float32)
    n = margin.shape[0]
    g = np.zeros(n, np.float64)
    h = np.zeros(n, np.float64)
    q = np.zeros((n, 2), np.int32)
    sc = np.zeros(2, np.int32)
    _check(lib().oracle_gradients(obj, _ptr(margin, C.c_double), _ptr(label, C.c_float), n, P,
                                  _ptr(g, C.c_double), _ptr(h, C.c_double), _ptr(q, C.c_int32),
                                  _ptr(sc, C.c_int32)), "oracle_gradients")
    return g, h, q, (int(sc[0]), int(sc[1]))


def node_histogram(words, F, bits, row_align_bits, cut_ptr, max_bins, qpair, rows):
    """BuildPartialHistograms: int64 [TB, 2] over the listed rows."""
    cp = np.ascontiguousarray(cut_ptr, dtype=np.int32)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    qpair = np.ascontiguousarray(qpair, dtype=np.int32)
    words = np.ascontiguousarray(words, dtype=np.uint32)
    hist = np.zeros((max(1, int(cp[-1])), 2), np.int64)
    _check(lib().oracle_node_histogram(_ptr(words, C.c_uint32), F, bits, row_align_bits,
                                       _ptr(cp, C.c_int32), max_bins, _ptr(qpair, C.c_int32),
                                       _ptr(rows, C.c_int64), rows.shape[0],
                                       _ptr(hist, C.c_int64)), "oracle_node_histogram")
    return hist[: int(cp[-1])]


def evaluate_split(hist, cut_ptr, Tg, Th, scale, reg_lambda, gamma, mcw):
    """EvaluateSplit.  Returns dict(split, feature, bin, default_left, gain,
    L=(g,h), R=(g,h))."""
    cp = np.ascontiguousarray(cut_ptr, dtype=np.int32)
    F = cp.shape[0] - 1
    hist = np.ascontiguousarray(hist, dtype=np.int64)
    if hist.size == 0:
        hist = np.zeros((1, 2), np.int64)
    oi = np.full(3, -1, np.int32)
    ol = np.zeros(4, np.int64)
    gain = C.c_double(0.0)
    r = lib().oracle_evaluate_split(_ptr(hist, C.c_int64), F, _ptr(cp, C.c_int32), int(Tg),
                                    int(Th), int(scale[0]), int(scale[1]), float(reg_lambda),
                                    float(gamma), float(mcw), _ptr(oi, C.c_int32),
                                    C.byref(gain), _ptr(ol, C.c_int64))
    return dict(split=bool(r), feature=int(oi[0]), bin=int(oi[1]), default_left=bool(oi[2]),
                gain=gain.value, L=(int(ol[0]), int(ol[1])), R=(int(ol[2]), int(ol[3])))


def leaf_weight(Tg, Th, scale, reg_lambda, eta):
    return lib().oracle_leaf_weight(int(Tg), int(Th), int(scale[0]), int(scale[1]),
                                    float(reg_lambda), float(eta))


TREE_FIELDS = (("kind", np.int8), ("feature", np.int32), ("bin", np.int32),
               ("threshold", np.float32), ("default_left", np.int8), ("gain", np.float64),
               ("weight", np.float64), ("sum_qg", np.int64), ("sum_qh", np.int64))


def tree_capacity(max_depth: int) -> int:
    return (1 << (max_depth + 1)) - 1


def build_tree(words, n, F, bits, row_align_bits, cut_values, cut_ptr, max_bins, qpair, scale,
               max_depth, eta=0.3, reg_lambda=1.0, gamma=0.0, mcw=1.0, p_workers=1,
               grow_policy="depthwise", max_leaves=0):
    """Algorithm 1 on p logical workers.  Returns (tree dict, row_leaf int32 [n]).
    depthwise: heap arrays of capacity 2^(D+1)-1 (FIFO queue, "nodes closer to the root").
    lossguide: priority queue on the gain (R25-R27), capacity 2*max_leaves-1, plus the
    array left_child (right child = left + 1)."""
    lossguide = grow_policy == "lossguide"
    cap = 2 * max_leaves - 1 if lossguide else tree_capacity(max_depth)
    t = {k: np.zeros(max(cap, 1), dt) for k, dt in TREE_FIELDS}
    row_leaf = np.zeros(n, np.int32)
    cv = np.ascontiguousarray(cut_values, dtype=np.float32)
    if cv.size == 0:
        cv = np.zeros(1, np.float32)
    cp = np.ascontiguousarray(cut_ptr, dtype=np.int32)
    qpair = np.ascontiguousarray(qpair, dtype=np.int32)
    sc = np.asarray(scale, dtype=np.int32)
    params = np.array([eta, reg_lambda, gamma, mcw], np.float64)
    words = np.ascontiguousarray(words, dtype=np.uint32)
    common = (_ptr(words, C.c_uint32), n, F, bits, row_align_bits, _ptr(cv, C.c_float),
              _ptr(cp, C.c_int32), max_bins, _ptr(qpair, C.c_int32), _ptr(sc, C.c_int32))
    arrays = (_ptr(t["kind"], C.c_int8), _ptr(t["feature"], C.c_int32), _ptr(t["bin"], C.c_int32),
              _ptr(t["threshold"], C.c_float), _ptr(t["default_left"], C.c_int8),
              _ptr(t["gain"], C.c_double), _ptr(t["weight"], C.c_double),
              _ptr(t["sum_qg"], C.c_int64), _ptr(t["sum_qh"], C.c_int64))
    if lossguide:
        t["left_child"] = np.full(max(cap, 1), -1, np.int32)
        _check(lib().oracle_build_tree_lossguide(
            *common, max_depth, max_leaves, _ptr(params, C.c_double), p_workers, *arrays,
            _ptr(t["left_child"], C.c_int32), _ptr(row_leaf, C.c_int32)),
            "oracle_build_tree_lossguide")
    else:
        _check(lib().oracle_build_tree(
            *common, max_depth, _ptr(params, C.c_double), p_workers, *arrays,
            _ptr(row_leaf, C.c_int32)), "oracle_build_tree")
    return t, row_leaf


def update_margins(weight: np.ndarray, row_leaf: np.ndarray, margin: np.ndarray) -> np.ndarray:
    """margin[i] += w[row_leaf[i]]; returns a new array."""
    m = np.array(margin, dtype=np.float64, copy=True)
    w = np.ascontiguousarray(weight, dtype=np.float64)
    rl = np.ascontiguousarray(row_leaf, dtype=np.int32)
    _check(lib().oracle_update_margins(_ptr(w, C.c_double), _ptr(rl, C.c_int32), m.shape[0],
                                       _ptr(m, C.c_double)), "oracle_update_margins")
    return m


def predict(trees: list[dict], max_depth: int, base_margin: float, X: np.ndarray) -> np.ndarray:
    """§2.4 prediction: base + sum over trees of the reached leaf weight.  Trees with
    a "left_child" array (loss-guided, R27) are walked through their links."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    n, F = X.shape
    out = np.zeros(n, np.float64)
    if trees and "left_child" in trees[0]:
        cap = int(trees[0]["kind"].shape[0])
        cat = {k: np.ascontiguousarray(np.concatenate([t[k][:cap] for t in trees]))
               for k in ("kind", "feature", "threshold", "default_left", "left_child", "weight")}
        _check(lib().oracle_predict_linked(len(trees), cap, _ptr(cat["kind"], C.c_int8),
                                           _ptr(cat["feature"], C.c_int32),
                                           _ptr(cat["threshold"], C.c_float),
                                           _ptr(cat["default_left"], C.c_int8),
                                           _ptr(cat["left_child"], C.c_int32),
                                           _ptr(cat["weight"], C.c_double), float(base_margin),
                                           _ptr(X, C.c_float), n, F, _ptr(out, C.c_double)),
               "oracle_predict_linked")
        return out
    cap = tree_capacity(max_depth)
    if trees:
        cat = {k: np.ascontiguousarray(np.concatenate([t[k][:cap] for t in trees]))
               for k in ("kind", "feature", "threshold", "default_left", "weight")}
    else:
        cat = {k: np.zeros(1, dt) for k, dt in TREE_FIELDS}
    _check(lib().oracle_predict(len(trees), max_depth, _ptr(cat["kind"], C.c_int8),
                                _ptr(cat["feature"], C.c_int32),
                                _ptr(cat["threshold"], C.c_float),
                                _ptr(cat["default_left"], C.c_int8),
                                _ptr(cat["weight"], C.c_double), float(base_margin),
                                _ptr(X, C.c_float), n, F, _ptr(out, C.c_double)),
           "oracle_predict")
    return out


# ---------------------------------------------------------------------------------------------
class Booster:
    """Fig. 1 pipeline on the oracle: quantise -> compress -> per round gradients,
    Alg. 1 tree, margin update.  Used by tests and by bench.py's CPU legs."""

    def __init__(self, X, y, *, max_bins, objective, max_depth, eta=0.3, reg_lambda=1.0,
                 gamma=0.0, mcw=1.0, grad_bits=15, p_workers=1, row_align_bits=32,
                 base_margin=None, grow_policy="depthwise", max_leaves=0):
        self.X = np.ascontiguousarray(X, np.float32)
        self.y = np.ascontiguousarray(y, np.float32)
        self.n, self.F = self.X.shape
        self.max_bins, self.objective, self.max_depth = max_bins, objective, max_depth
        self.eta, self.reg_lambda, self.gamma, self.mcw = eta, reg_lambda, gamma, mcw
        self.P, self.p_workers, self.row_align_bits = grad_bits, p_workers, row_align_bits
        self.grow_policy, self.max_leaves = grow_policy, max_leaves
        self.cut_values, self.cut_ptr = cuts(self.X, max_bins)
        self.sym, self.max_symbol = symbols(self.X, self.cut_values, self.cut_ptr, max_bins)
        self.bits = symbol_bits(self.max_symbol)
        self.words = pack(self.sym, self.bits, row_align_bits)
        if base_margin is None:
            base_margin = 0.0 if OBJECTIVES.get(objective, objective) == LOGISTIC else \
                float(np.mean(self.y.astype(np.float64)))
        self.base_margin = float(base_margin)
        self.margin = np.full(self.n, self.base_margin, np.float64)
        self.trees: list[dict] = []
        self.last = None

    def round(self):
        _, _, q, sc = gradients(self.objective, self.margin, self.y, self.P)
        tree, row_leaf = build_tree(self.words, self.n, self.F, self.bits, self.row_align_bits,
                                    self.cut_values, self.cut_ptr, self.max_bins, q, sc,
                                    self.max_depth, self.eta, self.reg_lambda, self.gamma,
                                    self.mcw, self.p_workers, self.grow_policy, self.max_leaves)
        self.margin = update_margins(tree["weight"], row_leaf, self.margin)
        self.trees.append(tree)
        self.last = dict(qpair=q, scale=sc, row_leaf=row_leaf)
        return tree

    def predict(self, X=None, n_trees=None):
        X = self.X if X is None else X
        t = self.trees if n_trees is None else self.trees[:n_trees]
        return predict(t, self.max_depth, self.base_margin, X)
