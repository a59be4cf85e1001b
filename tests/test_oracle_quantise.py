"""Oracle pins for §2.1 quantiles and §2.2 compression.

Each test ties the oracle to something other than its own formula: SPEC examples, library
routines (numpy.unique / searchsorted / packbits), invariants and the paper's 4x claim.
"""
import json
import os

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import oracle as O
import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
SPEC = GOLD["spec_examples"]


def test_symbol_bits_spec_examples():
    for cite, pairs in SPEC["symbol_bits"].items():
        for mx, bits in pairs:
            assert O.symbol_bits(mx) == bits, cite


@pytest.mark.parametrize("mx", list(range(0, 70000, 997)) + [1, 2, 3, 4, 255, 256, 65535])
def test_symbol_bits_is_fewest_bits(mx):
    b = O.symbol_bits(mx)
    assert (1 << b) > mx and (b == 1 or (1 << (b - 1)) <= mx)


def test_cuts_spec_examples():
    c = SPEC["cuts"]
    v, p = O.cuts(np.array(c["S:106"]["values"], np.float32)[:, None], 4)
    assert v.tolist() == c["S:106"]["cuts"] and p.tolist() == [0, 4]
    v, p = O.cuts(np.array(c["S:107"]["values"], np.float32)[:, None], 8)
    assert v.tolist() == c["S:107"]["cuts"]
    x = np.array(c["S:108"]["values"], np.float32)[:, None]
    v, p = O.cuts(x, 2)
    pops = np.bincount(np.searchsorted(v, x[:, 0], side="left"), minlength=len(v))
    assert pops.tolist() == c["S:108"]["populations"]


@pytest.mark.parametrize("seed", range(6))
def test_cuts_lossless_equals_numpy_unique(seed):
    # d <= B: cuts are exactly the distinct values (library routine numpy.unique)
    X = W.random_matrix(seed, 500, 5, distinct=7 + 3 * seed, missing=0.1)
    v, p = O.cuts(X, 64)
    for f in range(X.shape[1]):
        col = X[:, f]
        col = col[~np.isnan(col)]
        np.testing.assert_array_equal(v[p[f]:p[f + 1]], np.unique(col))


@pytest.mark.parametrize("seed,B", [(0, 16), (1, 256), (2, 5), (3, 100)])
def test_cuts_rank_rule_equal_frequency(seed, B):
    # with distinct values, cut j is the value whose empirical CDF count is floor((j+1) m / B)
    # (S:136): checked by counting with numpy.searchsorted, not by re-running the rule.
    X = W.random_matrix(seed, 3000, 3)
    v, p = O.cuts(X, B)
    for f in range(3):
        col = np.sort(X[:, f])
        m = col.size
        c = v[p[f]:p[f + 1]]
        assert len(c) == B and np.all(np.diff(c) > 0) and c[-1] == col[-1]
        counts = np.searchsorted(col, c, side="right")
        assert counts.tolist() == [((j + 1) * m) // B for j in range(B)]


def test_cuts_with_ties_invariants():
    # strictly increasing, 1 <= len <= B, last cut == max, offsets are the prefix sum
    rng = np.random.default_rng(5)
    X = np.concatenate([rng.integers(0, 40, (4000, 2)), rng.standard_normal((4000, 2)) ** 3],
                       axis=1).astype(np.float32)
    X[rng.random(X.shape) < 0.05] = np.nan
    for B in (2, 3, 16, 33, 256):
        v, p = O.cuts(X, B)
        assert p[0] == 0
        for f in range(X.shape[1]):
            c = v[p[f]:p[f + 1]]
            col = X[:, f][~np.isnan(X[:, f])]
            assert 1 <= len(c) <= B and np.all(np.diff(c) > 0) and c[-1] == col.max()
            assert set(c.tolist()) <= set(col.tolist())


def test_cuts_all_missing_feature_and_errors():
    X = np.array([[np.nan, 1.0], [np.nan, 2.0]], np.float32)
    v, p = O.cuts(X, 4)
    assert p.tolist() == [0, 0, 2]
    with pytest.raises(O.OracleError) as e:
        O.cuts(np.array([[np.inf]], np.float32), 4)
    assert e.value.code == -5
    with pytest.raises(O.OracleError):
        O.cuts(np.zeros((0, 2), np.float32), 4)


def test_cuts_negative_zero_canonical():
    v, _ = O.cuts(np.array([[-0.0], [1.0]], np.float32), 4)
    assert np.signbit(v[0]) == False  # noqa: E712


def test_bin_of_spec_examples():
    for cite, (cuts, v, expect) in SPEC["bin_of"].items():
        X = np.array([[v]], np.float32)
        cv = np.array(cuts, np.float32)
        s, _ = O.symbols(X, cv, np.array([0, len(cuts)], np.int32), 256)
        assert int(s[0, 0]) == expect, cite


@pytest.mark.parametrize("seed", range(5))
def test_symbols_equal_searchsorted_and_bracket(seed):
    X = W.random_matrix(seed, 2000, 4, missing=0.07)
    B = 16 + seed * 50
    v, p = O.cuts(X, B)
    s, mx = O.symbols(X, v, p, B)
    for f in range(4):
        c = v[p[f]:p[f + 1]]
        col = X[:, f]
        nan = np.isnan(col)
        ref = np.minimum(np.searchsorted(c, col[~nan], side="left"), len(c) - 1)
        np.testing.assert_array_equal(s[~nan, f], ref)
        assert np.all(s[nan, f] == B)
        k = s[~nan, f].astype(np.int64)
        assert np.all(col[~nan] <= c[k])                     # v <= cuts[bin]
        assert np.all((k == 0) | (col[~nan] > c[np.maximum(k - 1, 0)]))  # cuts[bin-1] < v
    assert mx == (B if np.isnan(X).any() else s.max())


@settings(max_examples=40, deadline=None)
@given(st.lists(st.floats(-1e6, 1e6, width=32), min_size=2, max_size=60),
       st.integers(2, 20))
def test_symbols_monotone(vals, B):
    x = np.array(vals, np.float32)[:, None]
    v, p = O.cuts(x, B)
    probe = np.sort(np.array(vals + [-1e7, 1e7], np.float32))[:, None]
    s, _ = O.symbols(probe, v, p, B)
    assert np.all(np.diff(s[:, 0].astype(int)) >= 0)


def _packbits_reference(sym, bits):
    # library routine: expand each symbol into its `bits` bits (LSB first) and let
    # numpy.packbits(bitorder="little") build the byte stream.
    n, F = sym.shape
    bitmat = ((sym.reshape(-1, 1).astype(np.uint32) >> np.arange(bits, dtype=np.uint32)) & 1)
    stream = np.packbits(bitmat.reshape(-1).astype(np.uint8), bitorder="little")
    return stream


@pytest.mark.parametrize("bits", [1, 2, 3, 4, 5, 7, 8, 9, 12, 13, 16])
def test_pack_equals_numpy_packbits(bits):
    rng = np.random.default_rng(bits)
    sym = rng.integers(0, 1 << bits, (37, 11)).astype(np.uint16)
    words = O.pack(sym, bits, 0)
    ref = _packbits_reference(sym, bits)
    got = words.view(np.uint8)
    np.testing.assert_array_equal(got[:ref.size], ref)
    assert not got[ref.size:].any()                       # zero tail padding
    assert words.size % 4 == 0 and words.size >= (sym.size * bits + 31) // 32 + 4


@pytest.mark.parametrize("align", [32, 128, 256])
def test_pack_row_alignment_is_per_row_packbits(align):
    rng = np.random.default_rng(align)
    bits, F = 9, 5
    sym = rng.integers(0, 1 << bits, (20, F)).astype(np.uint16)
    words = O.pack(sym, bits, align)
    stride_words = -(-F * bits // align) * align // 32
    for r in range(sym.shape[0]):
        ref = _packbits_reference(sym[r:r + 1], bits)
        row = words[r * stride_words:(r + 1) * stride_words].view(np.uint8)
        np.testing.assert_array_equal(row[:ref.size], ref)
        assert not row[ref.size:].any()


def test_pack_roundtrip_all_widths_1e6():
    # S:195 / S:586: unpack(compress(s, b)) == s for widths 1..16 over 10^6 elements
    rng = np.random.default_rng(0)
    for bits in range(1, 17):
        n = 1_000_000 // 8 if bits > 1 else 1_000_000
        sym = rng.integers(0, 1 << bits, (n // 8, 8)).astype(np.uint16)
        for align in (0, 32):
            words = O.pack(sym, bits, align)
            np.testing.assert_array_equal(O.unpack(words, sym.shape[0], 8, bits, align), sym)


def test_pack_overflow_and_spec_roundtrip():
    with pytest.raises(O.OracleError) as e:
        O.pack(np.array([[7]], np.uint16), 2)
    assert e.value.code == -3
    w = O.pack(np.array([[3, 1, 2]], np.uint16), 2)
    assert O.unpack(w, 1, 3, 2).tolist() == [[3, 1, 2]]
    w = O.pack(np.array([[5, 6, 7]], np.uint16), 3)
    assert int(O.unpack(w, 1, 3, 3)[0, 1]) == 6


def test_compression_four_times_or_more():
    # P:30 "reduces GPU memory consumption by four times or more"; 100,000 x 50 dense,
    # 256 bins -> 8-bit symbols -> >= 3.98x after padding.
    X = W.random_matrix(3, 100_000, 50)
    v, p = O.cuts(X, 256)
    s, mx = O.symbols(X, v, p, 256)
    bits = O.symbol_bits(mx)
    assert bits == 8
    words = O.pack(s, bits, 0)
    ratio = X.nbytes / words.nbytes
    assert ratio >= 3.98
    # E4: Airline 115M x 13 on 8 GPUs at 8 bits -> ~187 MB per GPU (paper: 600 MB)
    per_gpu = O.packed_words(115_000_000 // 8, 13, 8, 0) * 4
    assert 180e6 < per_gpu < 190e6
