"""Per-replay durations of the captured Higgs round: is there a warm-up curve over the first replays?"""
import sys, os, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1806_11248_b200 as G, workloads as W
X, y = W.generate("higgs")
Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
ctx = G.Context(0)
b = G.Booster(ctx, Xd, yd, max_bins=256, objective="binary:logistic", max_depth=6, eta=0.1)
for _ in range(5): b.round(keep_tree=False)
side = torch.cuda.Stream(); side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side): b.round(keep_tree=False)
torch.cuda.current_stream().wait_stream(side); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g): b.round(keep_tree=False)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(301)]
ev[0].record()
for i in range(300):
    g.replay(); ev[i + 1].record()
torch.cuda.synchronize()
t = [ev[i].elapsed_time(ev[i + 1]) for i in range(300)]
print(json.dumps({"first10": [round(x, 3) for x in t[:10]], "mean_0_20": sum(t[:20]) / 20, "mean_20_100": sum(t[20:100]) / 80,
                  "mean_100_300": sum(t[100:]) / 200}))
