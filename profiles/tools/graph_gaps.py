"""Per-kernel durations inside a replayed round graph (every launch bracketed by CUDA-event nodes)
against the replay's total: how much of a round is kernel time on each stream and how much is
dependency gaps.  usage: graph_gaps.py [config] [K]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1806_11248_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "higgs"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
X, y = W.generate(cfg.name)
ctx = G.Context(0)
b = G.Booster(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), max_bins=cfg.max_bins,
              objective=cfg.objective, max_depth=cfg.max_depth, eta=0.1)
for _ in range(5):
    b.round(keep_tree=False)
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    b.round(keep_tree=False)
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
for prof_on in (False, True):
    if prof_on:
        ctx.profile(True)  # every category: event nodes around every launch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        b.round(keep_tree=False)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    if prof_on:
        ctx.profile_zero_rows()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    per = e0.elapsed_time(e1) / K
    if not prof_on:
        print(f"replay without event nodes: {per:.4f} ms/round")
        continue
    p = ctx.profile_read()
    ctx.profile(False)
    print(f"replay with event nodes: {per:.4f} ms/round")
    # the graph's event nodes hold the LAST replay's durations
    tot = 0.0
    for k, v in sorted(p.items(), key=lambda kv: -kv[1]["ms"]):
        if v["launches"]:
            print(f"  {k:16s} launches {v['launches']:4d}  ms {v['ms']:.4f}")
            if k not in ("part_scan", "part_scatter"):
                tot += v["ms"]
    print(f"main-stream kernel time (excl. the side stream's scan + scatter): {tot:.4f} ms")
