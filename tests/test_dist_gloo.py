"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 path's host logic.

The GPU path shards rows contiguously (R18), takes the gradient scale from a global max (C1)
and sums per-shard int64 histograms with one allreduce per level (C2); every rank
then evaluates the same splits.  Here two real processes run exactly that exchange protocol
with the oracle doing the per-shard arithmetic and torch.distributed (gloo) doing the
collectives, and the trees must equal the single-process oracle's.  The NCCL-id broadcast used
by Context.comm_init_from_torch is exercised too.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _allgather_rows(a: np.ndarray, world):
    """all-gather a per-rank [n_k, ...] array of varying n_k (padding to the max)."""
    n = torch.tensor([a.shape[0]], dtype=torch.int64)
    ns = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(ns, n)
    m = int(max(x.item() for x in ns))
    pad = np.zeros((m,) + a.shape[1:], a.dtype)
    pad[: a.shape[0]] = a
    outs = [torch.zeros_like(torch.from_numpy(pad)) for _ in range(world)]
    dist.all_gather(outs, torch.from_numpy(pad))
    return np.concatenate([o.numpy()[: int(k.item())] for o, k in zip(outs, ns)])


def _dist_tree_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        from paper_1806_11248_b200 import share_unique_id
        ids = share_unique_id(lambda: bytes(range(128)), None)
        assert ids == bytes(range(128))
        n = 3001
        lo, hi = W.shard_range(n, rank, world)
        Xs, ys = W.generate("tiny", lo, hi, n_rows=n, missing=0.05)
        # C3: global cuts from the all-gathered rows
        Xall = _allgather_rows(Xs, world)
        v, p = O.cuts(Xall, 16)
        s_loc, mx_loc = O.symbols(Xs, v, p, 16)
        mx = torch.tensor([mx_loc])
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        bits = O.symbol_bits(int(mx.item()))
        words = O.pack(s_loc, bits, 32)
        # C1: gradient scale from the global max |g|, |h| -> identical fixed point everywhere
        yall = _allgather_rows(ys, world)
        beta = float(np.mean(yall.astype(np.float64)))
        _, _, q_all, sc = O.gradients("reg:squarederror", np.full(n, beta), yall, 15)
        qloc = np.ascontiguousarray(q_all[lo:hi])
        # level-synchronous Alg. 1 with one int64 allreduce per node histogram (C2)
        D, lam, gam, mcw, eta = 4, 1.0, 0.0, 1.0, 0.3
        cap = (1 << (D + 1)) - 1
        pos = np.zeros(hi - lo, np.int64)
        kind = np.zeros(cap, np.int8)
        feat = np.full(cap, -1, np.int32)
        binv = np.full(cap, -1, np.int32)
        dlv = np.zeros(cap, np.int8)
        tot = torch.from_numpy(qloc.astype(np.int64).sum(0))
        dist.all_reduce(tot)
        totals = {0: (int(tot[0]), int(tot[1]))}
        frontier = [0]
        for depth in range(D):
            nxt = []
            for k in frontier:
                rows = np.nonzero(pos == k)[0].astype(np.int64)
                H = torch.from_numpy(O.node_histogram(words, Xs.shape[1], bits, 32, p, 16, qloc,
                                                      rows))
                dist.all_reduce(H)   # AllReduceHistograms
                Tg, Th = totals[k]
                r = O.evaluate_split(H.numpy(), p, Tg, Th, sc, lam, gam, mcw)
                if not r["split"]:
                    kind[k] = 2
                    continue
                kind[k], feat[k], binv[k], dlv[k] = 1, r["feature"], r["bin"], r["default_left"]
                sym = s_loc[rows, r["feature"]].astype(np.int64)
                left = np.where(sym == 16, r["default_left"], sym <= r["bin"])
                pos[rows[left]] = 2 * k + 1
                pos[rows[~left]] = 2 * k + 2
                totals[2 * k + 1], totals[2 * k + 2] = r["L"], r["R"]
                nxt += [2 * k + 1, 2 * k + 2]
            frontier = nxt
        for k in frontier:
            kind[k] = 2
        leaf = _allgather_rows(pos.astype(np.int32), world)
        if rank == 0:
            q.put((kind, feat, binv, dlv, leaf))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(repr(e))
        raise


def test_two_process_tree_equals_single_process_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_tree_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    res = q.get(timeout=240)
    for p_ in procs:
        p_.join(timeout=60)
    assert not isinstance(res, str), res
    kind, feat, binv, dlv, leaf = res
    # single-process reference on the full matrix
    X, y = W.generate("tiny", 0, 3001, n_rows=3001, missing=0.05)
    b = O.Booster(X, y, max_bins=16, objective="reg:squarederror", max_depth=4, eta=0.3)
    t = b.round()
    np.testing.assert_array_equal(kind, t["kind"])
    np.testing.assert_array_equal(feat[kind == 1], t["feature"][kind == 1])
    np.testing.assert_array_equal(binv[kind == 1], t["bin"][kind == 1])
    np.testing.assert_array_equal(dlv[kind == 1], t["default_left"][kind == 1])
    np.testing.assert_array_equal(leaf, b.last["row_leaf"])


def test_shards_partition_rows_and_regenerate_identically():
    for n in (1, 7, 1000, 70001):
        for p in (1, 2, 3, 8):
            rs = [W.shard_range(n, k, p) for k in range(p)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[k][1] == rs[k + 1][0] for k in range(p - 1))
    X, y = W.generate("higgs", 0, 140_000)
    parts = [W.generate("higgs", *W.shard_range(140_000, k, 3), n_rows=140_000) for k in range(3)]
    np.testing.assert_array_equal(np.concatenate([a for a, _ in parts]), X)
    np.testing.assert_array_equal(np.concatenate([b for _, b in parts]), y)
