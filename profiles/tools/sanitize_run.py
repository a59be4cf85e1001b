"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): tiny and 100K-row Higgs,
depth-wise and loss-guided, eager rounds then graph-captured replays, every round checked
against the previous eager tree (no oracle: the parity suite covers results)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1806_11248_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

cases = [("tiny", 2000, "depthwise"), ("tiny", 2000, "lossguide"),
         ("higgs", 100_000, "depthwise"), ("higgs", 100_000, "lossguide"),
         ("bosch", 20_000, "depthwise")]
only = sys.argv[1:] or None
ctx = G.Context(0)
for cfg, n, grow in cases:
    if only and cfg not in only:
        continue
    c = W.CONFIGS[cfg]
    X, y = W.generate(cfg, 0, n, n_rows=max(n, c.n_rows))
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    D = c.max_depth if grow == "depthwise" else 10
    beta = 0.0 if c.objective == "binary:logistic" else float(np.mean(y.astype(np.float64)))
    for P in (15, 30):
        b = G.Booster(ctx, Xd, yd, max_bins=c.max_bins, objective=c.objective, max_depth=D, eta=0.3,
                      grad_bits=P, grow_policy=grow, max_leaves=(24 if grow == "lossguide" else 0),
                      base_margin=beta)
        for _ in range(2):
            b.round(keep_tree=False)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            b.round(keep_tree=False)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            b.round(keep_tree=False)
        for _ in range(2):
            g.replay()
        torch.cuda.synchronize()
        ctx.check()
        del g, b
    print(f"sanitize workload {cfg} n={n} {grow}: ok", flush=True)
ctx.close()
