"""Multi-rank libgbm on ONE GPU through the virtual communicator (gbm_comm_init_virtual; SURVEY
§4 "virtual shards"): p contexts, one host thread and one stream each, every rank holding its
contiguous shard [floor(k n / p), floor((k+1) n / p)) (R18) packed from bit 0.  Global
cuts over the concatenated shards (C3), global gradient maxima (C1), per-level partial histograms
summed (C2) -- libgbm's own multi-rank code, not a model of it -- must give the oracle's
p-worker trees (worker invariance) on every rank, bit for bit, and the argument
agreement must turn mismatched ranks into GBM_E_MISMATCH on every rank, not a hang."""
import threading

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


def run_ranks(G, p, body, timeout=300):
    """Run body(ctx, rank) on p threads, each with its own context and stream; returns the
    per-rank results or raises the first exception.  A thread still running after `timeout`
    seconds fails the test (a collective that never completes)."""
    vc = G.VirtualComm(p)
    out, err = [None] * p, [None] * p

    def work(k):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = G.Context(0)
                ctx.comm_init_virtual(vc, k)
                try:
                    out[k] = body(ctx, k)
                    torch.cuda.synchronize()
                finally:
                    ctx.close()
        except BaseException as e:  # noqa: BLE001
            err[k] = e

    ts = [threading.Thread(target=work, args=(k,), daemon=True) for k in range(p)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert not any(t.is_alive() for t in ts), "a virtual collective did not complete (hang)"
    vc.close()
    return out, err


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


CASES = [  # cfg, rows, missing, grow, p
    ("higgs", 40_000, 0.0, "depthwise", 1),
    ("higgs", 40_000, 0.0, "depthwise", 2),
    ("higgs", 40_001, 0.0, "depthwise", 3),
    ("higgs", 40_000, 0.0, "depthwise", 8),
    ("tiny", 2000, 0.05, "depthwise", 3),
    ("airline", 30_000, 0.02, "depthwise", 4),
    ("bosch", 8_000, 0.0, "depthwise", 2),
    ("higgs", 30_000, 0.0, "lossguide", 3),
    ("tiny", 2000, 0.0, "depthwise", 8),     # 250-row shards
    ("tiny", 5, 0.0, "depthwise", 8),        # ranks with no rows at all
    ("tiny", 3000, 0.0, "depthwise", 12),    # more ranks than features: ranks owning no feature
    ("epsilon", 3000, 0.0, "depthwise", 3),  # 2000 features in three slices
    ("higgs", 1_300_000, 0.0, "depthwise", 2),   # > 296 x 2048 rows per rank: multi-tile work items per level
    ("airline", 1_500_000, 0.01, "depthwise", 2),
]


@pytest.mark.parametrize("sliced", [0, 1])
@pytest.mark.parametrize("cfg,n,missing,grow,p", CASES)
def test_virtual_shards_equal_oracle_workers(G, cfg, n, missing, grow, p, sliced):
    """sliced = 1: the reduce-scatter + feature-sliced evaluation variant of C2 (GBM_OPT_EVAL_SLICED):
    each rank evaluates its feature slice, the candidates are all-gathered -- same trees."""
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n, n_rows=max(n, c.n_rows), missing=missing)
    D = c.max_depth if grow == "depthwise" else 9
    L = 24 if grow == "lossguide" else 0
    ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=D, eta=0.3,
                   p_workers=p, grow_policy=grow, max_leaves=L)
    R = 2
    otrees = []
    oleaf = []
    for _ in range(R):
        otrees.append(ob.round())
        oleaf.append(ob.last["row_leaf"].copy())

    def body(ctx, k):
        ctx.set_option(ctx.EVAL_SLICED, sliced)
        lo, hi = W.shard_range(n, k, p)
        gb = G.Booster(ctx, dev(X[lo:hi]), dev(y[lo:hi]), max_bins=c.max_bins, objective=c.objective,
                       max_depth=D, eta=0.3, base_margin=ob.base_margin, grow_policy=grow, max_leaves=L)
        res = {"cuts": (gb.qm.cut_ptr_h.copy(), gb.qm.cut_values.cpu().numpy().copy()),
               "packed": gb.qm.packed.cpu().numpy().view(np.uint32).copy(), "bits": gb.qm.bits,
               "trees": [], "leaf": []}
        for _ in range(R):
            res["trees"].append(gb.round().to_numpy())
            res["leaf"].append(gb.row_leaf.cpu().numpy().copy())
        res["margin"] = gb.margin.cpu().numpy().copy()
        return res

    out, err = run_ranks(G, p, body)
    for e in err:
        if e is not None:
            raise e
    for k in range(p):
        lo, hi = W.shard_range(n, k, p)
        r = out[k]
        np.testing.assert_array_equal(r["cuts"][0], ob.cut_ptr)
        np.testing.assert_array_equal(r["cuts"][1].view(np.uint32), ob.cut_values.view(np.uint32))
        assert r["bits"] == ob.bits
        if hi > lo:  # each shard packed from bit 0 (R3)
            np.testing.assert_array_equal(r["packed"], O.pack(ob.sym[lo:hi], ob.bits, 32))
        for t in range(R):
            for f in otrees[t]:
                ga, oa = r["trees"][t][f], otrees[t][f]
                if ga.dtype.kind == "f":
                    ga, oa = ga.view(np.uint64 if ga.itemsize == 8 else np.uint32), \
                        oa.view(np.uint64 if oa.itemsize == 8 else np.uint32)
                np.testing.assert_array_equal(ga, oa, err_msg=f"rank {k} round {t} field {f}")
            np.testing.assert_array_equal(r["leaf"][t], oleaf[t][lo:hi])
        np.testing.assert_array_equal(r["margin"].view(np.uint64), ob.margin[lo:hi].view(np.uint64))


@pytest.mark.parametrize("what", ["max_depth", "grad_bits", "max_bins"])
def test_virtual_mismatch_is_collective(G, what):
    """Ranks that disagree on a size every rank must share get GBM_E_MISMATCH (or, for a local
    argument error, the same error code) on every rank, and nobody hangs."""
    X, y = W.generate("higgs", 0, 6000)
    p = 2

    def body(ctx, k):
        lo, hi = W.shard_range(len(y), k, p)
        kw = dict(max_bins=256, objective="binary:logistic", max_depth=4, grad_bits=15)
        if what == "max_bins":  # different cuts -> different TB: caught by the collective cuts? no:
            qm_bins = 256 if k == 0 else 64  # each rank asks for its own max_bins
            kw["max_bins"] = qm_bins
        gb = None
        try:
            gb = G.Booster(ctx, dev(X[lo:hi]), dev(y[lo:hi]), **kw)
            if what == "max_depth":
                gb.max_depth = 4 + k
            if what == "grad_bits":
                gb.grad_bits = 15 + k
            gb.round()
        except G.GbmError as e:
            return e.code
        return 0

    out, err = run_ranks(G, p, body, timeout=120)
    assert err == [None, None]
    expect = -6  # GBM_E_MISMATCH on both ranks
    assert out == [expect, expect], out


def test_virtual_local_argument_error_is_collective(G):
    """One rank passes a bad lambda to gbm_build_tree: both ranks return GBM_E_ARG."""
    X, y = W.generate("higgs", 0, 4000)
    p = 2

    def body(ctx, k):
        lo, hi = W.shard_range(len(y), k, p)
        gb = G.Booster(ctx, dev(X[lo:hi]), dev(y[lo:hi]), max_bins=256, objective="binary:logistic",
                       max_depth=3, reg_lambda=-1.0 if k == 1 else 1.0)
        try:
            gb.round()
        except G.GbmError as e:
            return e.code
        return 0

    out, err = run_ranks(G, p, body, timeout=120)
    assert err == [None, None]
    assert out == [-1, -1], out


@pytest.mark.parametrize("gather", [0, 1])
@pytest.mark.parametrize("cfg,n,missing,p", [("higgs", 20_011, 0.03, 3), ("airline", 30_000, 0.0, 5),
                                             ("tiny", 2000, 0.05, 12), ("yearmsd", 9_000, 0.0, 2),
                                             ("tiny", 3, 0.0, 4)])
def test_virtual_cuts_both_c3_modes(G, cfg, n, missing, p, gather):
    """C3 by per-feature ownership (all-to-all of the owned columns, cuts all-gathered; default) and
    by an all-gather of X (GBM_OPT_CUTS_GATHER=1): every rank's cuts and max symbol equal the
    oracle's global cuts (R5 over the concatenated shards)."""
    c = W.CONFIGS[cfg]
    X, _ = W.generate(cfg, 0, n, n_rows=max(n, c.n_rows), missing=missing)
    v, ptr = O.cuts(X, c.max_bins)
    _, mx = O.symbols(X, v, ptr, c.max_bins)

    def body(ctx, k):
        ctx.set_option(ctx.CUTS_GATHER, gather)
        lo, hi = W.shard_range(n, k, p)
        cv, cp, m = ctx.cuts(dev(X[lo:hi]), c.max_bins)
        return cv.cpu().numpy().copy(), cp.cpu().numpy().copy(), m

    out, err = run_ranks(G, p, body)
    for e in err:
        if e is not None:
            raise e
    for k in range(p):
        np.testing.assert_array_equal(out[k][1], ptr)
        np.testing.assert_array_equal(out[k][0].view(np.uint32), v.view(np.uint32))
        assert out[k][2] == mx
