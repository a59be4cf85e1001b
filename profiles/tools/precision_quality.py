"""Held-out quality of the per-row fixed-point precision (R14): Higgs-shaped 11M x 28
train rows, 1M held-out rows of the same generator (rows 11M..12M), depth 6, 256 bins, eta 0.1,
R rounds on the GPU at grad_bits 15 and 30; held-out log-loss and accuracy every 50 rounds.
Writes one JSON object (stdout)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1806_11248_b200 as G  # noqa: E402
import workloads as W  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 200
n_tr, n_te = 11_000_000, 1_000_000
X, y = W.generate("higgs", 0, n_tr, n_rows=n_tr + n_te)
Xt, yt = W.generate("higgs", n_tr, n_tr + n_te, n_rows=n_tr + n_te)
dev = torch.device("cuda", 0)
Xd, yd, Xtd = torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), torch.from_numpy(Xt).to(dev)
ctx = G.Context(0)
cfg = W.CONFIGS["higgs"]
out = {"train_rows": n_tr, "heldout_rows": n_te, "rounds": R, "config": "higgs depth 6, 256 bins, eta 0.1",
       "by_grad_bits": {}}
for P in (15, 30):
    b = G.Booster(ctx, Xd, yd, max_bins=256, objective="binary:logistic", max_depth=6, eta=cfg.eta,
                  reg_lambda=cfg.reg_lambda, gamma=cfg.gamma, min_child_weight=cfg.min_child_weight,
                  grad_bits=P)
    curve = []
    t0 = time.time()
    for r in range(1, R + 1):
        b.round()
        if r % 50 == 0 or r == R:
            m = b.predict(Xtd).cpu().numpy()
            p = 1.0 / (1.0 + np.exp(-m))
            eps = 1e-15
            ll = float(-np.mean(yt * np.log(np.clip(p, eps, 1)) + (1 - yt) * np.log(np.clip(1 - p, eps, 1))))
            acc = float(np.mean((p > 0.5) == (yt > 0.5)))
            mt = b.margin.cpu().numpy()
            pt = 1.0 / (1.0 + np.exp(-mt))
            ll_tr = float(-np.mean(y * np.log(np.clip(pt, eps, 1)) + (1 - y) * np.log(np.clip(1 - pt, eps, 1))))
            curve.append({"round": r, "heldout_logloss": ll, "heldout_accuracy": acc, "train_logloss": ll_tr})
    out["by_grad_bits"][str(P)] = {"curve": curve, "wall_s": round(time.time() - t0, 1)}
    del b
    torch.cuda.empty_cache()
a, c = out["by_grad_bits"]["15"]["curve"][-1], out["by_grad_bits"]["30"]["curve"][-1]
out["final_delta"] = {"heldout_logloss_rel": (a["heldout_logloss"] - c["heldout_logloss"]) / c["heldout_logloss"],
                      "heldout_accuracy_abs": a["heldout_accuracy"] - c["heldout_accuracy"]}
print(json.dumps(out))
