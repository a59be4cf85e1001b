"""Where the end-to-end train() time goes (bench.py's e2e protocol, host wall clock per phase with
a synchronize after each): H2D, cuts, quantise/compress + feature-major copy + buffers, the first
eager round, the graph capture, K-1 replays with tree read-back.  usage: e2e_breakdown.py [K] [config]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1806_11248_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfg = W.CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "higgs"]
X, y = W.generate(cfg.name)
ctx = G.Context(0)
kw = dict(max_bins=cfg.max_bins, objective=cfg.objective, max_depth=cfg.max_depth, eta=0.1)
# warm everything once (module loading, allocator), as bench.py does before its e2e leg
Xd = torch.from_numpy(X).cuda(); yd = torch.from_numpy(y).cuda()
b = G.Booster(ctx, Xd, yd, **kw); b.round(); del b, Xd, yd
torch.cuda.synchronize()
Xh = torch.from_numpy(X).pin_memory(); yh = torch.from_numpy(y).pin_memory()
for rep in range(2):
    T = {}
    t0 = time.perf_counter()
    def mark(k):
        torch.cuda.synchronize(); T[k] = time.perf_counter()
    Xd = Xh.cuda(non_blocking=True); yd = yh.cuda(non_blocking=True); mark("h2d")
    cuts = ctx.cuts(Xd, cfg.max_bins); mark("cuts")
    b2 = G.Booster(ctx, Xd, yd, cuts=cuts, **kw); mark("booster")
    t = b2.round(keep_tree=False); mark("round0")
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):
        t = b2.round(keep_tree=False)
    mark("capture")
    for i in range(K - 1):
        g2.replay()
    mark("replays")
    prev = t0
    print(f"rep {rep}: " + ", ".join(f"{k} {1e3 * (v - prev):.1f} ms" for k, v in T.items() if not (prev := prev) or True))
    prev = t0
    out = []
    for k, v in T.items():
        out.append(f"{k} {1e3 * (v - prev):.1f}")
        prev = v
    print(f"rep {rep} (ms): " + ", ".join(out) + f"; total {1e3 * (prev - t0):.1f}")
    del b2, Xd, yd, g2
