import sys, torch, time
sys.path.insert(0,'/root/repo')
import paper_1806_11248_b200 as G, workloads as W
X, y = W.generate("higgs")
Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
ctx = G.Context(0)
b = G.Booster(ctx, Xd, yd, max_bins=256, objective="binary:logistic", max_depth=6, eta=0.1)
for _ in range(10): b.round()
for trees in (1, 10):
    for k in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.profile(True, only=("predict",))
        e0.record(); out = b.predict(Xd, n_trees=trees); e1.record(); torch.cuda.synchronize()
        pr = ctx.profile_read(); ctx.profile(False)
        print(trees, "trees: events", e0.elapsed_time(e1), "ms; kernel", pr["predict"]["ms"], "ms")
