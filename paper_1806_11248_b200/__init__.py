"""paper_1806_11248_b200 -- B200-native hot path of multi-GPU histogram gradient boosting
(arXiv 1806.11248), behind the C-ABI of ``include/gbm.h`` (``libgbm.so``).

This module is the thin Python binding: argument marshalling only.  torch supplies device
memory (tensors), the current CUDA stream and the process group used to broadcast the NCCL id;
every step of the path runs in the CUDA kernels of ``csrc/``.  There is no CPU fallback: without
the built library or a CUDA device every call raises ``GbmError``.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import threading

import numpy as np
import torch

from . import build_lib

__all__ = ["GbmError", "Context", "QMatrix", "Tree", "Booster", "VirtualComm", "lib", "symbol_bits",
           "packed_words", "SQUARED_ERROR", "LOGISTIC", "OBJECTIVES"]

SQUARED_ERROR, LOGISTIC = 0, 1
OBJECTIVES = {"reg:squarederror": SQUARED_ERROR, "binary:logistic": LOGISTIC}
NODE_ABSENT, NODE_SPLIT, NODE_LEAF = 0, 1, 2
DEFAULT_GRAD_BITS = 15   # R14 / DESIGN.md "Gradient precision"

_lock = threading.Lock()
_lib = None


class GbmError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: {msg} (code {code})")
        self.code = code


class _Params(C.Structure):
    _fields_ = [("objective", C.c_int32), ("max_depth", C.c_int32), ("grad_bits", C.c_int32),
                ("grow_policy", C.c_int32), ("eta", C.c_double), ("reg_lambda", C.c_double),
                ("gamma", C.c_double), ("min_child_weight", C.c_double),
                ("max_leaves", C.c_int32), ("reserved", C.c_int32)]


class _QM(C.Structure):
    _fields_ = [("packed_d", C.c_void_p), ("n_rows", C.c_int64), ("n_features", C.c_int32),
                ("bits", C.c_int32), ("row_align_bits", C.c_int32), ("max_bins", C.c_int32),
                ("cut_values_d", C.c_void_p), ("cut_ptr_d", C.c_void_p),
                ("cut_ptr_h", C.POINTER(C.c_int32)), ("colsym_d", C.c_void_p)]


class _Tree(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("kind", "feature", "bin", "threshold", "default_left",
                                          "gain", "weight", "sum_qg", "sum_qh", "left_child")]


class _Epilogue(C.Structure):
    _fields_ = [("margin_d", C.c_void_p), ("label_d", C.c_void_p), ("objective", C.c_int32),
                ("reserved", C.c_int32), ("sig_d", C.c_void_p), ("maxbits_d", C.c_void_p)]


class _ProfEntry(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("ms", C.c_double),
                ("bytes", C.c_double), ("rows", C.c_double)]


EXPORTS = {
    # name: (restype, argtypes)
    "gbm_last_error": (C.c_char_p, []),
    "gbm_abi_version": (C.c_int, []),
    "gbm_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "gbm_ctx_destroy": (C.c_int, [C.c_void_p]),
    "gbm_check": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gbm_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "gbm_profile_read": (C.c_int, [C.c_void_p, C.POINTER(_ProfEntry), C.c_int32,
                                   C.POINTER(C.c_int32)]),
    "gbm_launch_count": (C.c_int64, [C.c_void_p]),
    "gbm_profile_zero_rows": (C.c_int, [C.c_void_p]),
    "gbm_set_option": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
    "gbm_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8)]),
    "gbm_comm_init": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_int, C.c_int]),
    "gbm_comm_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "gbm_vcomm_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "gbm_vcomm_destroy": (C.c_int, [C.c_void_p]),
    "gbm_comm_init_virtual": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "gbm_cuts": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                           C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_void_p]),
    "gbm_quantise": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gbm_symbol_bits": (C.c_int, [C.c_int32]),
    "gbm_packed_words": (C.c_int64, [C.c_int64, C.c_int32, C.c_int32, C.c_int32]),
    "gbm_compress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                               C.c_void_p, C.c_int64, C.c_void_p]),
    "gbm_quantise_compress": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32,
                                        C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                        C.c_int64, C.c_void_p]),
    "gbm_transpose_symbols": (C.c_int, [C.c_void_p, C.POINTER(_QM), C.c_void_p, C.c_void_p]),
    "gbm_gradients": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gbm_build_tree": (C.c_int, [C.c_void_p, C.POINTER(_QM), C.c_void_p, C.c_void_p,
                                 C.POINTER(_Params), C.POINTER(_Tree), C.c_void_p, C.c_void_p]),
    "gbm_build_tree_fused": (C.c_int, [C.c_void_p, C.POINTER(_QM), C.c_void_p, C.c_void_p,
                                       C.POINTER(_Params), C.POINTER(_Tree), C.c_void_p,
                                       C.POINTER(_Epilogue), C.c_void_p]),
    "gbm_gradients_from_stats": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                           C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.c_void_p]),
    "gbm_build_histogram": (C.c_int, [C.c_void_p, C.POINTER(_QM), C.c_void_p, C.c_int32,
                                      C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "gbm_allreduce_histograms": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "gbm_evaluate_splits": (C.c_int, [C.c_void_p, C.POINTER(_QM), C.c_void_p, C.c_void_p,
                                      C.c_int32, C.c_void_p, C.POINTER(_Params), C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    "gbm_repartition": (C.c_int, [C.c_void_p, C.POINTER(_QM), C.c_void_p, C.c_int64, C.c_int32,
                                  C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "gbm_update_margins": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                     C.c_void_p]),
    "gbm_predict": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_void_p,
                              C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
    "gbm_predict_linked": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                     C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]),
}


def lib():
    """Load (building if stale) the in-tree libgbm.so.  Raises if it cannot be built/loaded."""
    global _lib
    with _lock:
        if _lib is None:
            path = build_lib.LIB
            if build_lib.stale():
                path = build_lib.build()
            L = C.CDLL(path)
            for name, (res, args) in EXPORTS.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().gbm_last_error().decode(errors="replace")
        raise GbmError(rc, name, msg)
    return rc


def _p(t: torch.Tensor | None):
    if t is None:
        return None
    assert t.is_contiguous(), "tensors passed to libgbm must be contiguous"
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def symbol_bits(max_symbol: int) -> int:
    b = lib().gbm_symbol_bits(int(max_symbol))
    if b < 0:
        raise GbmError(b, "gbm_symbol_bits", "bad max_symbol")
    return b


def packed_words(n_rows: int, n_features: int, bits: int, row_align_bits: int = 32) -> int:
    w = lib().gbm_packed_words(n_rows, n_features, bits, row_align_bits)
    if w < 0:
        raise GbmError(int(w), "gbm_packed_words", lib().gbm_last_error().decode())
    return int(w)


GROW_POLICIES = {"depthwise": 0, "lossguide": 1}


def _params(objective, max_depth, eta, reg_lambda, gamma, mcw, grad_bits, grow_policy="depthwise",
            max_leaves=0):
    return _Params(OBJECTIVES.get(objective, objective), max_depth, grad_bits,
                   GROW_POLICIES.get(grow_policy, grow_policy), eta, reg_lambda, gamma, mcw,
                   max_leaves, 0)


@dataclasses.dataclass
class QMatrix:
    """A rank's quantised, bit-packed shard (device tensors) + its cuts."""
    packed: torch.Tensor          # int32 view of the uint32 words
    n_rows: int
    n_features: int
    bits: int
    row_align_bits: int
    max_bins: int
    cut_values: torch.Tensor      # fp32 [TB]
    cut_ptr: torch.Tensor         # int32 [F+1] (device)
    cut_ptr_h: np.ndarray         # int32 [F+1] (host)
    colsym: torch.Tensor | None = None  # optional uint8 [F][n] feature-major symbol copy

    def c(self) -> _QM:
        self._cp = np.ascontiguousarray(self.cut_ptr_h, dtype=np.int32)
        cv = self.cut_values if self.cut_values.numel() else torch.zeros(1, device=self.packed.device)
        self._cv = cv
        return _QM(self.packed.data_ptr(), self.n_rows, self.n_features, self.bits,
                   self.row_align_bits, self.max_bins, cv.data_ptr(), self.cut_ptr.data_ptr(),
                   self._cp.ctypes.data_as(C.POINTER(C.c_int32)),
                   self.colsym.data_ptr() if self.colsym is not None else None)

    @property
    def n_bins_total(self) -> int:
        return int(self.cut_ptr_h[-1])


TREE_FIELDS = (("kind", torch.int8), ("feature", torch.int32), ("bin", torch.int32),
               ("threshold", torch.float32), ("default_left", torch.int8),
               ("gain", torch.float64), ("weight", torch.float64), ("sum_qg", torch.int64),
               ("sum_qh", torch.int64), ("left_child", torch.int32))


class Tree:
    """Device arrays of one tree.  Depth-wise: heap order, capacity 2^(D+1)-1.  Loss-guided
    (max_leaves > 0, R27): children of the j-th expansion at 2j+1 / 2j+2, capacity
    2*max_leaves-1.  left_child links the children in both layouts (-1 for leaves)."""

    def __init__(self, max_depth: int, device, max_leaves: int = 0):
        cap = 2 * max_leaves - 1 if max_leaves > 0 else (1 << (max_depth + 1)) - 1
        self.max_depth, self.max_leaves, self.capacity = max_depth, max_leaves, cap
        self.arrays = {n: torch.empty(cap, dtype=dt, device=device) for n, dt in TREE_FIELDS}

    def c(self) -> _Tree:
        return _Tree(*[self.arrays[n].data_ptr() for n, _ in TREE_FIELDS])

    def __getitem__(self, k):
        return self.arrays[k]

    def to_numpy(self) -> dict:
        return {k: v.cpu().numpy() for k, v in self.arrays.items()}


class Context:
    """One gbm_ctx bound to a CUDA device (and optionally an NCCL communicator)."""

    def __init__(self, device: int | None = None):
        if not torch.cuda.is_available():
            raise GbmError(-10, "Context", "no CUDA device: libgbm has no CPU fallback")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.dev = torch.device("cuda", self.device)
        h = C.c_void_p()
        _call("gbm_ctx_create", self.device, C.byref(h))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            lib().gbm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ communicator
    def comm_init_from_torch(self, group=None):
        """NCCL communicator over the ranks of the torch.distributed (default) process group:
        rank 0 makes the id, torch broadcasts the 128 bytes (plumbing only)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        ids = share_unique_id(Context.comm_unique_id, group, device=self.dev)
        _call("gbm_comm_init", self.h, (C.c_uint8 * 128)(*ids), world, rank)

    def comm_init(self, id_bytes: bytes, nranks: int, rank: int):
        ids = (C.c_uint8 * 128)(*id_bytes)
        _call("gbm_comm_init", self.h, ids, nranks, rank)

    def comm_init_virtual(self, vcomm: "VirtualComm", rank: int):
        """Attach this context as virtual rank `rank` of `vcomm` (p ranks on one device, one
        host thread each; the test harness of the multi-rank path, gbm.h)."""
        _call("gbm_comm_init_virtual", self.h, vcomm.h, int(rank))
        self._vcomm = vcomm  # keep the communicator alive while this context uses it

    @staticmethod
    def comm_unique_id() -> bytes:
        buf = (C.c_uint8 * 128)()
        _call("gbm_comm_unique_id", buf)
        return bytes(buf)

    def check(self):
        _call("gbm_check", self.h, _stream())

    # ------------------------------------------------------------ instrumentation
    PROFILE_CATEGORIES = ("grad_max", "grad_quant", "hist_root", "hist_level", "part_count", "part_scan",
                          "part_scatter", "part_final", "evaluate", "allreduce", "update_margins",
                          "init_tree", "predict", "cuts", "quantise_compress", "eval_final", "plan",
                          "part_decide")

    def profile(self, enable: bool = True, only=None):
        """Start (reset) / stop in-library event timing; `only` = category names to record."""
        v = int(bool(enable))
        if enable and only:
            v = 0
            for name in only:
                v |= 1 << self.PROFILE_CATEGORIES.index(name)
            assert v > 1, "pick at least one category other than grad_max alone"
        _call("gbm_profile_enable", self.h, v)

    def profile_zero_rows(self):
        """Zero the algorithmic-byte counters, keep the timing records (graph event nodes)."""
        _call("gbm_profile_zero_rows", self.h)

    def profile_read(self) -> dict:
        """Per-kernel {launches, ms, bytes, rows} since the last read (synchronises)."""
        arr = (_ProfEntry * 32)()
        n = C.c_int32()
        _call("gbm_profile_read", self.h, arr, 32, C.byref(n))
        return {arr[i].name.decode(): dict(launches=arr[i].launches, ms=arr[i].ms,
                                           bytes=arr[i].bytes, rows=arr[i].rows)
                for i in range(n.value)}

    HIST_LAYOUT = 1
    CARRY_GRADIENTS = 2
    RUN_TILES = 3
    GROUP_UNITS = 4
    EVAL_WARP = 5
    LEAF_WALK = 6
    EVAL_SCREEN = 7
    SEGMENT_HIST = 8
    TMA_ROWS = 10
    ROW_DECIDE = 11
    LEVEL_PATH = 12
    LEVEL_HIST = 13
    EVAL_SLICED = 14
    CUTS_GATHER = 15
    ROOT_TENSOR = 16
    LEVEL_REPLICAS = 17

    def set_option(self, option: int, value: int):
        _call("gbm_set_option", self.h, int(option), int(value))

    def launch_count(self) -> int:
        return int(lib().gbm_launch_count(self.h))

    # ------------------------------------------------------------ §2.1 / §2.2
    def cuts(self, X: torch.Tensor, max_bins: int):
        n, F = X.shape
        cv = torch.empty(max(1, F * max_bins), dtype=torch.float32, device=self.dev)
        cp = torch.empty(F + 1, dtype=torch.int32, device=self.dev)
        ncut, mx = C.c_int32(), C.c_int32()
        _call("gbm_cuts", self.h, _p(X), n, F, max_bins, _p(cv), _p(cp), C.byref(ncut),
              C.byref(mx), _stream())
        return cv[: ncut.value], cp, mx.value

    def quantise(self, X, max_bins, cut_values, cut_ptr):
        n, F = X.shape
        bins = torch.empty((n, F), dtype=torch.uint16, device=self.dev)
        _call("gbm_quantise", self.h, _p(X), n, F, max_bins, _p(_nz(cut_values)), _p(cut_ptr),
              _p(bins), _stream())
        return bins

    def compress(self, bins, bits, row_align_bits=32):
        n, F = bins.shape
        nw = packed_words(n, F, bits, row_align_bits)
        out = torch.empty(nw, dtype=torch.int32, device=self.dev)
        _call("gbm_compress", self.h, _p(bins), n, F, bits, row_align_bits, _p(out), nw,
              _stream())
        return out

    def quantise_compress(self, X, max_bins, cut_values, cut_ptr, bits, row_align_bits=32):
        n, F = X.shape
        nw = packed_words(n, F, bits, row_align_bits)
        out = torch.empty(nw, dtype=torch.int32, device=self.dev)
        _call("gbm_quantise_compress", self.h, _p(X), n, F, max_bins, _p(_nz(cut_values)),
              _p(cut_ptr), bits, row_align_bits, _p(out), nw, _stream())
        return out

    def make_qmatrix(self, X: torch.Tensor, max_bins: int, row_align_bits: int = 32,
                     cuts=None, colsym: bool = True) -> QMatrix:
        """Fig. 1 preprocessing: global cuts (collective), then fused bin map + pack, then
        (bits <= 8, optional) the feature-major symbol copy used by RepartitionInstances."""
        if cuts is None:
            cv, cp, mx = self.cuts(X, max_bins)
        else:
            cv, cp, mx = cuts
        bits = symbol_bits(mx)
        packed = self.quantise_compress(X, max_bins, cv, cp, bits, row_align_bits)
        qm = QMatrix(packed, X.shape[0], X.shape[1], bits, row_align_bits, max_bins, cv, cp,
                     cp.cpu().numpy())
        if colsym and bits <= 8:
            self.transpose_symbols(qm)
        return qm

    def transpose_symbols(self, qm: QMatrix) -> QMatrix:
        qm.colsym = None
        col = torch.empty((qm.n_features, max(qm.n_rows, 1)), dtype=torch.uint8, device=self.dev)
        _call("gbm_transpose_symbols", self.h, C.byref(qm.c()), _p(col), _stream())
        qm.colsym = col
        return qm

    # ------------------------------------------------------------ §2.5
    def gradients(self, objective, margin, label, grad_bits=DEFAULT_GRAD_BITS, out=None,
                  scale=None):
        n = margin.shape[0]
        q = out if out is not None else torch.empty((n, 2), dtype=torch.int32, device=self.dev)
        sc = scale if scale is not None else torch.empty(2, dtype=torch.int32, device=self.dev)
        _call("gbm_gradients", self.h, OBJECTIVES.get(objective, objective), grad_bits,
              _p(margin), _p(label), n, _p(q), _p(sc), _stream())
        return q, sc

    # ------------------------------------------------------------ §2.3
    def build_tree(self, qm: QMatrix, qpair, scale, *, objective, max_depth, eta=0.3,
                   reg_lambda=1.0, gamma=0.0, min_child_weight=1.0,
                   grad_bits=DEFAULT_GRAD_BITS, tree: Tree | None = None, row_leaf=None,
                   grow_policy="depthwise", max_leaves=0, epilogue=None):
        lossguide = GROW_POLICIES.get(grow_policy, grow_policy) == 1
        tree = tree if tree is not None else Tree(max_depth, self.dev,
                                                  max_leaves if lossguide else 0)
        rl = row_leaf if row_leaf is not None else torch.empty(qm.n_rows, dtype=torch.int32,
                                                               device=self.dev)
        prm = _params(objective, max_depth, eta, reg_lambda, gamma, min_child_weight, grad_bits,
                      grow_policy, max_leaves)
        qc, tc = qm.c(), tree.c()
        if epilogue is None:
            _call("gbm_build_tree", self.h, C.byref(qc), _p(qpair), _p(scale), C.byref(prm),
                  C.byref(tc), _p(rl), _stream())
        else:  # fused: margin update + the next round's gradient statistics
            margin, label, sig, maxbits = epilogue
            ep = _Epilogue(margin.data_ptr(), label.data_ptr(), OBJECTIVES.get(objective, objective), 0,
                           sig.data_ptr() if sig is not None else None, maxbits.data_ptr())
            _call("gbm_build_tree_fused", self.h, C.byref(qc), _p(qpair), _p(scale), C.byref(prm),
                  C.byref(tc), _p(rl), C.byref(ep), _stream())
        return tree, rl

    def gradients_from_stats(self, objective, margin, label, sig, maxbits,
                             grad_bits=DEFAULT_GRAD_BITS, out=None, scale=None):
        """Pass 2 of gradients() from the statistics of the previous build_tree(epilogue=...)."""
        n = margin.shape[0]
        q = out if out is not None else torch.empty((n, 2), dtype=torch.int32, device=self.dev)
        sc = scale if scale is not None else torch.empty(2, dtype=torch.int32, device=self.dev)
        _call("gbm_gradients_from_stats", self.h, OBJECTIVES.get(objective, objective), grad_bits,
              _p(margin), _p(label), n, _p(sig), _p(maxbits), _p(q), _p(sc), _stream())
        return q, sc

    def build_histogram(self, qm: QMatrix, qpair, grad_bits, rows=None):
        TB = qm.n_bins_total
        hist = torch.empty((max(TB, 1), 2), dtype=torch.int64, device=self.dev)
        n_sel = qm.n_rows if rows is None else rows.numel()
        _call("gbm_build_histogram", self.h, C.byref(qm.c()), _p(qpair), grad_bits, _p(rows),
              n_sel, _p(hist), _stream())
        return hist[:TB]

    def allreduce_histograms(self, hist: torch.Tensor):
        _call("gbm_allreduce_histograms", self.h, _p(hist), hist.numel(), _stream())

    def evaluate_splits(self, qm: QMatrix, hist, totals, scale, *, eta=0.3, reg_lambda=1.0,
                        gamma=0.0, min_child_weight=1.0, max_depth=1):
        n = totals.shape[0]
        d = self.dev
        out = dict(split=torch.empty(n, dtype=torch.int8, device=d),
                   feature=torch.empty(n, dtype=torch.int32, device=d),
                   bin=torch.empty(n, dtype=torch.int32, device=d),
                   default_left=torch.empty(n, dtype=torch.int8, device=d),
                   gain=torch.empty(n, dtype=torch.float64, device=d),
                   child=torch.empty((n, 4), dtype=torch.int64, device=d))
        prm = _params(0, max_depth, eta, reg_lambda, gamma, min_child_weight, 15)
        _call("gbm_evaluate_splits", self.h, C.byref(qm.c()), _p(hist), _p(totals), n, _p(scale),
              C.byref(prm), _p(out["split"]), _p(out["feature"]), _p(out["bin"]),
              _p(out["default_left"]), _p(out["gain"]), _p(out["child"]), _stream())
        return out

    def repartition(self, qm: QMatrix, rows, feature, bin_, default_left):
        out = torch.empty_like(rows)
        nl = torch.zeros(1, dtype=torch.int64, device=self.dev)
        _call("gbm_repartition", self.h, C.byref(qm.c()), _p(rows), rows.numel(), feature, bin_,
              int(bool(default_left)), _p(out), _p(nl), _stream())
        return out, nl

    # ------------------------------------------------------------ margins / §2.4
    def update_margins(self, weight, row_leaf, margin):
        _call("gbm_update_margins", self.h, _p(weight), _p(row_leaf), margin.shape[0],
              _p(margin), _stream())
        return margin

    def predict(self, trees: list[Tree], max_depth: int, base_margin: float, X: torch.Tensor):
        n, F = X.shape
        out = torch.empty(n, dtype=torch.float64, device=self.dev)
        if trees and trees[0].max_leaves > 0:  # loss-guided layout: follow the links
            names = ("kind", "feature", "threshold", "default_left", "left_child", "weight")
            cat = {k: torch.cat([t[k] for t in trees]) for k in names}
            _call("gbm_predict_linked", self.h, len(trees), trees[0].capacity, _p(cat["kind"]),
                  _p(cat["feature"]), _p(cat["threshold"]), _p(cat["default_left"]),
                  _p(cat["left_child"]), _p(cat["weight"]), float(base_margin), _p(X), n, F,
                  _p(out), _stream())
            return out
        if trees:
            cat = {k: torch.cat([t[k] for t in trees]) for k in
                   ("kind", "feature", "threshold", "default_left", "weight")}
        else:
            cat = {k: None for k in ("kind", "feature", "threshold", "default_left", "weight")}
        _call("gbm_predict", self.h, len(trees), max_depth, _p(cat["kind"]), _p(cat["feature"]),
              _p(cat["threshold"]), _p(cat["default_left"]), _p(cat["weight"]),
              float(base_margin), _p(X), n, F, _p(out), _stream())
        return out


class VirtualComm:
    """An in-process communicator of `nranks` virtual ranks on one device (gbm_vcomm_create)."""

    def __init__(self, nranks: int):
        h = C.c_void_p()
        _call("gbm_vcomm_create", int(nranks), C.byref(h))
        self.h, self.nranks = h, int(nranks)

    def close(self):
        if getattr(self, "h", None):
            lib().gbm_vcomm_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def share_unique_id(make_id, group=None, device=None) -> bytes:
    """Rank 0 calls make_id() (128 bytes); torch.distributed broadcasts them to every rank of
    `group` (gloo: CPU tensor, nccl: tensor on `device`).  Returns the bytes on every rank."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    raw = make_id() if rank == 0 else bytes(128)
    if len(raw) != 128:
        raise GbmError(-1, "share_unique_id", "the NCCL unique id must be 128 bytes")
    t = torch.tensor(list(raw), dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast(t, src, group=group)
    return bytes(t.cpu().tolist())


def _nz(t):
    return t if t.numel() else torch.zeros(1, dtype=t.dtype, device=t.device)


class Booster:
    """The Fig. 1 pipeline on one rank: quantise+compress once, then per boosting
    round gradients (collective max) -> Alg. 1 tree (collective per level) -> margin update.
    X / y are this rank's shard (device tensors)."""

    def __init__(self, ctx: Context, X: torch.Tensor, y: torch.Tensor, *, max_bins: int,
                 objective: str, max_depth: int, eta=0.3, reg_lambda=1.0, gamma=0.0,
                 min_child_weight=1.0, grad_bits=DEFAULT_GRAD_BITS, row_align_bits=32,
                 base_margin=0.0, cuts=None, colsym=True, grow_policy="depthwise", max_leaves=0,
                 fused=True):
        self.ctx, self.y = ctx, y
        self.objective, self.max_depth, self.grad_bits = objective, max_depth, grad_bits
        self.kw = dict(eta=eta, reg_lambda=reg_lambda, gamma=gamma,
                       min_child_weight=min_child_weight, grow_policy=grow_policy,
                       max_leaves=max_leaves)
        self.qm = ctx.make_qmatrix(X, max_bins, row_align_bits, cuts=cuts, colsym=colsym)
        self.base_margin = float(base_margin)
        n = X.shape[0]
        self.margin = torch.full((n,), self.base_margin, dtype=torch.float64, device=ctx.dev)
        self.qpair = torch.empty((n, 2), dtype=torch.int32, device=ctx.dev)
        self.scale = torch.empty(2, dtype=torch.int32, device=ctx.dev)
        self.row_leaf = torch.empty(n, dtype=torch.int32, device=ctx.dev)
        self.trees: list[Tree] = []
        # fused rounds: the tree build also updates the margins and computes the next round's
        # gradient statistics (gbm_build_tree_fused / gbm_gradients_from_stats)
        self.fused = fused
        lg = OBJECTIVES.get(objective, objective) == 1
        self.sig = torch.empty(max(n, 1), dtype=torch.float64, device=ctx.dev) if fused and lg else None
        self.maxbits = torch.zeros(2, dtype=torch.int64, device=ctx.dev) if fused else None
        self.stats_valid = False

    def round(self, keep_tree=True) -> Tree:
        c = self.ctx
        if self.fused and self.stats_valid:
            c.gradients_from_stats(self.objective, self.margin, self.y, self.sig, self.maxbits,
                                   self.grad_bits, out=self.qpair, scale=self.scale)
        else:
            c.gradients(self.objective, self.margin, self.y, self.grad_bits, out=self.qpair,
                        scale=self.scale)
        if self.fused:
            tree, _ = c.build_tree(self.qm, self.qpair, self.scale, objective=self.objective,
                                   max_depth=self.max_depth, grad_bits=self.grad_bits,
                                   row_leaf=self.row_leaf,
                                   epilogue=(self.margin, self.y, self.sig, self.maxbits), **self.kw)
            self.stats_valid = True
        else:
            tree, _ = c.build_tree(self.qm, self.qpair, self.scale, objective=self.objective,
                                   max_depth=self.max_depth, grad_bits=self.grad_bits,
                                   row_leaf=self.row_leaf, **self.kw)
            c.update_margins(tree["weight"], self.row_leaf, self.margin)
        if keep_tree:
            self.trees.append(tree)
        return tree

    def predict(self, X, n_trees=None):
        t = self.trees if n_trees is None else self.trees[:n_trees]
        return self.ctx.predict(t, self.max_depth, self.base_margin, X)
