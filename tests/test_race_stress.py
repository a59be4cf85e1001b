"""Race / determinism stress (compute-sanitizer is closed on this pool, profiles/r02/
compute_sanitizer_refused.log): the kernels' exact int64 sums make every result independent of
scheduling, so an intermittent race (a missing fence before a finisher's counter, a staging buffer
reused before its readers finish, a work item claimed twice) shows up as a bit difference between
repeated runs.  Each configuration below -- dynamic work claiming, threadfence + last-block
finishers, mbarrier / cp.async.bulk double buffers, warp-private compaction lists, the side-stream
scatter, CUDA-graph replays -- is run repeatedly on the same data and compared bit for bit with the
first run (and the first run with the oracle)."""
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


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


OPTS = [
    {},
    {"RUN_TILES": 1}, {"RUN_TILES": 7},
    {"EVAL_WARP": 1}, {"EVAL_WARP": 2},
    {"LEVEL_HIST": 2}, {"LEVEL_PATH": 2},
    {"HIST_LAYOUT": 3}, {"TMA_ROWS": 0},
]


def snapshot(gb, tree):
    t = tree.to_numpy()
    return [t[k].copy() for k in sorted(t)] + [gb.row_leaf.cpu().numpy().copy(), gb.margin.cpu().numpy().copy()]


@pytest.mark.parametrize("opts", OPTS, ids=lambda o: ",".join(f"{k}={v}" for k, v in o.items()) or "default")
@pytest.mark.parametrize("cfg,n,grow", [("higgs", 200_003, "depthwise"), ("higgs", 100_000, "lossguide")])
def test_repeated_runs_identical(G, cfg, n, grow, opts):
    ctx = G.Context(0)
    for k, v in opts.items():
        ctx.set_option(getattr(G.Context, k), v)
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n)
    Xd, yd = dev(X), dev(y)
    kw = dict(max_bins=c.max_bins, objective=c.objective, max_depth=(c.max_depth if grow == "depthwise" else 12),
              eta=0.3, grow_policy=grow, max_leaves=(40 if grow == "lossguide" else 0))
    runs = []
    for rep in range(4):
        gb = G.Booster(ctx, Xd, yd, **kw)
        snaps = []
        if rep % 2 == 0:  # eager rounds
            for _ in range(3):
                snaps.append(snapshot(gb, gb.round()))
        else:  # one eager round, then two replays of a captured round
            snaps.append(snapshot(gb, gb.round()))
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    t = gb.round(keep_tree=False)
            torch.cuda.current_stream().wait_stream(side)
            for _ in range(2):
                g.replay()
                torch.cuda.synchronize()
                snaps.append(snapshot(gb, t))
            del g
        runs.append(snaps)
    ref = runs[0]
    for rep, snaps in enumerate(runs[1:], 1):
        for r, (a, b) in enumerate(zip(ref, snaps)):
            for i, (u, v) in enumerate(zip(a, b)):
                assert np.array_equal(u.view(np.uint8), v.view(np.uint8)), f"rep {rep} round {r} array {i} differs"
    ctx.check()
    ctx.close()
    if not opts:  # the first run against the oracle (once per case): margins after 3 rounds
        ob = O.Booster(X, y, max_bins=c.max_bins, objective=c.objective, max_depth=kw["max_depth"], eta=0.3,
                       grow_policy=grow, max_leaves=kw["max_leaves"])
        for _ in range(3):
            ob.round()
        np.testing.assert_array_equal(ref[2][-1], ob.margin)
