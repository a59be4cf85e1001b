#!/usr/bin/env python
"""bench.py -- seconds per boosting round of the B200 hot path (BASELINE.json metric).

A "step" is one boosting round of the Fig. 1 pipeline over the whole configured
workload: gradients (Eq. 1-2, fixed point, collective max) -> Algorithm 1 tree (root histogram,
then per level partition + smaller-child histogram + NCCL allreduce + subtraction + evaluate)
-> margin update.  One-time quantile cuts and quantise+compress are timed separately
("one_time"), prediction too ("predict_ms").

Default workload: the Higgs-shaped config (11M x 28, 256 bins, depth 6, logistic), the
BASELINE.json config the metric "(depth 6, 256 bins) at 1/2/4/8 B200" is quoted on that fits one
GPU.  Inputs (packed matrix 308 MB + per-row state) exceed the 126 MB
L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config higgs]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N   (N > 1)
  python bench.py --impl reference   # the CPU oracle, the reference arm of this tier
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

FALLBACK_HBM_GBS = 6650.0   # /opt/skills/guides/B200_PROFILING.md fallback (of fallback)
METRIC = "sec/boosting round (depth 6, 256 bins) at 1/2/4/8 B200; histogram GB/s vs HBM peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="higgs", choices=sorted(W.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--rows", type=int, default=None, help="override the row count (debug)")
    ap.add_argument("--grad-bits", type=int, default=15)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches, not a CUDA graph")
    ap.add_argument("--cpu-rounds", type=int, default=3,
                    help="oracle rounds of the cpu_baseline / parity leg (full rows, threaded)")
    ap.add_argument("--cpu-threads", type=int, default=0, help="oracle threads (0 = the host's cores)")
    ap.add_argument("--no-parity", action="store_true", help="skip the full-size oracle parity leg")
    ap.add_argument("--no-p30", action="store_true", help="skip the grad_bits = 30 figure")
    ap.add_argument("--no-full-run", action="store_true",
                    help="skip the full-training figure (the config's round count, e.g. 500 for Higgs)")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--row-align-bits", type=int, default=32,
                    help="packed row stride rounded up to this many bits (gbm_compress)")
    ap.add_argument("--grow-policy", default="depthwise", choices=["depthwise", "lossguide"],
                    help="lossguide: priority-queue growth (P:65) with --max-leaves")
    ap.add_argument("--max-leaves", type=int, default=None,
                    help="lossguide leaf budget (default 2^max_depth of the config)")
    ap.add_argument("--comm", action="store_true",
                    help="initialise torch.distributed + the NCCL communicator even for one rank "
                         "(exercises the N > 1 code path on one GPU)")
    ap.add_argument("--opt", action="append", default=[], metavar="NAME=VALUE",
                    help="gbm_set_option before training, e.g. RUN_TILES=4 (GBM_OPT_* of include/gbm.h)")
    ap.add_argument("--max-depth", type=int, default=None,
                    help="depth limit (default: the config's; lossguide default 16)")
    a = ap.parse_args()
    a.warmup = max(3, a.warmup)
    return a


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(config):
    """dram read+write bytes per launch of the histogram kernel from the committed ncu summary
    (profiles/ncu_hist_<config>.json, written from an `ncu --set full` capture), or None."""
    p = os.path.join(ROOT, "profiles", f"ncu_hist_{config}.json")
    try:
        d = json.load(open(p))
        return d.get("dram_bytes_per_launch"), d.get("source"), d.get("l1tex_pct_of_peak_active_mean")
    except Exception:
        return None, None, None


def clocks_max_mhz():
    """Max SM clock (MEASURED_PEAKS.json sm_max_mhz, else nvidia-smi, else 1965)."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        pass
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits", "-i", "0"],
                             capture_output=True, text=True, timeout=10).stdout
        return float(out.split()[0])
    except Exception:
        return 1965.0


class Clocks:
    """nvidia-smi sampler running across the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.p = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(gpu_index)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        load = [s for s, pw in zip(sm, power) if pw > 200.0] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm), "samples_under_load": len(load)}


# ---------------------------------------------------------------------------------------------
def run_ours(a, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_1806_11248_b200 as G

    torch.cuda.set_device(local)
    cfg = W.CONFIGS[a.config]
    n = a.rows or cfg.n_rows
    lo, hi = W.shard_range(n, rank, world)
    t_gen = time.time()
    X, y = W.generate(a.config, lo, hi, n_rows=n)
    t_gen = time.time() - t_gen
    dev = torch.device("cuda", local)
    # base margin: 0 (logistic) / global label mean (squared error), host-side in row order
    if cfg.objective == "binary:logistic":
        beta = 0.0
    else:
        s = torch.tensor([float(np.sum(y.astype(np.float64))), float(len(y))], dtype=torch.float64)
        if a.dist:
            s = s.to(dev)
            dist.all_reduce(s)
        beta = float(s[0] / s[1])
    ctx = G.Context(local)
    for o in a.opt:
        name, val = o.split("=", 1)
        ctx.set_option(getattr(G.Context, name), int(val))
    if a.dist:
        ctx.comm_init_from_torch()
    kw = dict(max_bins=cfg.max_bins, objective=cfg.objective, max_depth=a.depth,
              eta=cfg.eta, reg_lambda=cfg.reg_lambda, gamma=cfg.gamma,
              min_child_weight=cfg.min_child_weight, grad_bits=a.grad_bits, base_margin=beta,
              grow_policy=a.grow_policy, max_leaves=a.leaves, row_align_bits=a.row_align_bits)
    stream = torch.cuda.current_stream()

    def barrier():
        if a.dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if not a.dist:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident run: inputs already in HBM when the timed region starts
    Xd = torch.from_numpy(X).to(dev)
    yd = torch.from_numpy(y).to(dev)
    # warm the one-time kernels (lazy module loading, attributes) on a small slice, then once at
    # full size so that the timed one-time figures are the kernels, not the first cudaMalloc of
    # each buffer (the caching allocator keeps the freed blocks), untimed
    m = min(4096, n)
    ctx.make_qmatrix(Xd[:m].contiguous(), cfg.max_bins, 32, cuts=ctx.cuts(Xd[:m].contiguous(), cfg.max_bins))
    warm = G.Booster(ctx, Xd, yd, cuts=ctx.cuts(Xd, cfg.max_bins), **kw)
    del warm
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    cuts = ctx.cuts(Xd, cfg.max_bins)
    e1.record(stream)
    e2 = torch.cuda.Event(enable_timing=True)
    booster = G.Booster(ctx, Xd, yd, cuts=cuts, **kw)
    e2.record(stream)
    torch.cuda.synchronize()
    booster_bits = booster.qm.bits
    one_time = {"cuts_ms": max_over_ranks(e0.elapsed_time(e1)),
                "quantise_compress_ms": max_over_ranks(e1.elapsed_time(e2)),
                "bits": booster.qm.bits, "n_bins_total": booster.qm.n_bins_total,
                "packed_bytes_per_gpu": booster.qm.packed.numel() * 4,
                "generate_s_host": round(t_gen, 2)}
    for _ in range(a.warmup):
        booster.round(keep_tree=False)
    # ---- one round as a CUDA graph (launch gaps removed); the histogram launches keep CUDA-event
    # nodes so their durations are measured live inside the timed region (last replay), while the
    # device row counters accumulate the algorithmic bytes of every replay
    hist_cats = ("hist_root", "hist_level")
    use_graph = not a.no_graph
    if use_graph:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            booster.round(keep_tree=False)  # warm the capture stream
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        ctx.profile(True, only=hist_cats)
        graph = torch.cuda.CUDAGraph()
        l0 = ctx.launch_count()
        with torch.cuda.graph(graph):
            booster.round(keep_tree=False)
        launches_per_round = ctx.launch_count() - l0
        step = graph.replay
        for _ in range(3):  # graph upload / first-launch costs stay out of the timed region
            graph.replay()
        torch.cuda.synchronize()
        ctx.profile_zero_rows()  # byte counters restart with the timed replays
    else:
        ctx.profile(True, only=hist_cats)
        l0 = ctx.launch_count()
        booster.round(keep_tree=False)
        launches_per_round = ctx.launch_count() - l0
        ctx.profile(True, only=hist_cats)
        step = lambda: booster.round(keep_tree=False)  # noqa: E731
    # L2 rule: the per-round working set (packed matrix, feature-major copy, per-row state) must
    # exceed the 126 MB L2, else L2 is flushed between the timed steps (outside their events)
    qm = booster.qm
    footprint = qm.packed.numel() * 4 + qm.n_rows * 36 + (qm.colsym.numel() if qm.colsym is not None else 0)
    flush = footprint < 2 * 126e6
    l2_note = (f"inputs larger than L2 ({footprint / 1e6:.0f} MB working set > 126 MB L2)" if not flush else
               f"L2 flushed between timed steps ({footprint / 1e6:.0f} MB working set; a 256 MB "
               "buffer is written outside the per-step events)")
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None
    clocks = Clocks(local)
    time.sleep(0.3)
    barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if flush:  # per-step events; the flush between them is not timed
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(a.steps)]
        for i, (e_a, e_b) in enumerate(evs):
            flush_buf.zero_()
            if use_graph and i == a.steps - 1:
                ctx.profile_zero_rows()  # the roofline pairs the last replay's bytes and times
            e_a.record(stream)
            step()
            e_b.record(stream)
        barrier()
        ms_total = sum(e_a.elapsed_time(e_b) for e_a, e_b in evs)
    else:
        t0.record(stream)
        for i in range(a.steps):
            if use_graph and i == a.steps - 1:
                # the event nodes time the last replay: pair them with that replay's bytes (the
                # counters restart here; one host sync inside the K-step window)
                ctx.profile_zero_rows()
            step()
        t1.record(stream)
        barrier()
        ms_total = t0.elapsed_time(t1)
    launches = launches_per_round * a.steps
    prof = ctx.profile_read()
    ctx.profile(False)
    clk = clocks.stop()
    ms_step = max_over_ranks(ms_total / a.steps)

    # ---- dominant kernel: the histogram pass (root + level launches), algorithmic bytes
    ms_div = 1 if use_graph else a.steps          # graph: event nodes hold the last replay
    hist_ms = (prof["hist_root"]["ms"] + prof["hist_level"]["ms"]) / ms_div       # per round
    hist_bytes = (prof["hist_root"]["bytes"] + prof["hist_level"]["bytes"]) / ms_div   # per round
    hist_launches = (prof["hist_root"]["launches"] + prof["hist_level"]["launches"]) // ms_div
    peak, peak_src = measured_peak()
    achieved = hist_bytes / (hist_ms * 1e-3) / 1e9 if hist_ms > 0 else 0.0
    # the committed ncu capture is of the depth-wise bench command: attach it only to that line
    traffic, traffic_src, l1_pct = ncu_traffic(a.config) if a.grow_policy == "depthwise" else (None, None, None)
    roofline = {"bound": "hbm", "kernel": "hist_kernel (root + level launches)",
                "bytes_definition": "SURVEY 8(d): root n (F b/8 + 8); level: each row of the built child "
                                    "F b/8 + 12 (packed row, row index, qpair); the fused level kernel's "
                                    "partition inputs (split symbol + row index per parent row) not counted",
                "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "algorithmic_bytes_per_launch": hist_bytes / max(1, hist_launches),
                "avg_launch_ms": hist_ms / max(1, hist_launches), "launches_per_round": hist_launches,
                "peak_source": peak_src, "traffic_source": traffic_src,
                "timing": ("CUDA-event nodes inside the replayed graph (last replay)" if use_graph
                           else "CUDA events around every launch of the timed region"),
                "share_of_step": round(hist_ms / (ms_total / a.steps), 4) if ms_total else None,
                # what actually binds it: shared-memory atomics on the L1/TEX data
                # pipe -- the committed ncu capture's L1/TEX utilisation of these launches
                "binding_unit": {"unit": "L1/TEX data pipe (shared-memory ATOMS)",
                                 "pct_of_peak": round(l1_pct, 1) if l1_pct else None,
                                 "source": traffic_src}}
    # ---- the unit that binds the histogram kernels: shared-memory atomics.  (g, h) updates per
    # round = rows streamed or built x features (missing symbols included: an upper bound for the
    # sparse sets), against the measured conflict-free rate of 8.65 updates/clk/SM
    # (profiles/microbench_smem_atomics.txt, lane-private copies) x SMs x the max SM clock
    cfg_b = W.CONFIGS[a.config]
    bits_b = booster_bits
    root_rows = prof["hist_root"]["bytes"] / ms_div / (cfg_b.n_features * bits_b / 8.0 + 8.0)
    level_rows = prof["hist_level"]["bytes"] / ms_div / (cfg_b.n_features * bits_b / 8.0 + 12.0)
    updates = (root_rows + level_rows) * cfg_b.n_features
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    sm_hz_max = clocks_max_mhz() * 1e6  # (not `clk`: that name holds the sampled clocks dict)
    atom_peak = 8.65 * sm_count * sm_hz_max
    atom_ach = updates / (hist_ms * 1e-3) if hist_ms > 0 else 0.0
    roofline_atomics = {"bound": "smem_atomics", "kernel": "hist_kernel (root + level launches)",
                        "achieved": atom_ach / 1e9, "peak": atom_peak / 1e9, "unit": "G (g,h) updates/s",
                        "frac": round(atom_ach / atom_peak, 4) if atom_peak else None,
                        "updates_per_round": updates,
                        "peak_source": "8.65 conflict-free (g,h) updates/clk/SM measured "
                                       "(profiles/microbench_smem_atomics.txt) x SMs x max SM clock"}
    # ---- per-stage breakdown: a separate eager window with every launch timed
    ctx.profile(True)
    n_st = min(20, a.steps)
    for _ in range(n_st):
        booster.round(keep_tree=False)
    sprof = ctx.profile_read()
    ctx.profile(False)
    stages = {k: {"ms_per_round": round(v["ms"] / n_st, 4),
                  "GBps": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else None}
              for k, v in sprof.items() if v["launches"]}
    allreduce_ms = sprof["allreduce"]["ms"] / n_st
    if use_graph:
        del graph

    # ---- predict (§2.4) over the training rows with the warm-up+timed trees? -> one tree set
    booster.trees = []
    for _ in range(10):
        booster.round()
    booster.predict(Xd)  # warm: lazy module load and the tree concatenation's allocations
    torch.cuda.synchronize()
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(5):
        booster.predict(Xd)
    p1.record(stream)
    torch.cuda.synchronize()
    predict_ms = max_over_ranks(p0.elapsed_time(p1) / 5)
    Xd_keep, yd_keep = Xd, yd
    del booster, Xd, yd, flush_buf
    torch.cuda.empty_cache()

    # ---- end to end through the public API from pinned host memory: H2D of X, y, global cuts,
    # quantise + compress (+ the feature-major copy), then K rounds (one eager, the rest replays of
    # a captured round), each round's tree copied back into pinned host memory (async D2H)
    e2e = None
    if not a.no_e2e:
        Xh = torch.from_numpy(X).pin_memory()
        yh = torch.from_numpy(y).pin_memory()
        cap = 2 * a.leaves - 1 if a.grow_policy == "lossguide" else (1 << (a.depth + 1)) - 1
        host_trees = {nm: torch.empty((a.steps, cap), dtype=dt, pin_memory=True)
                      for nm, dt in G.TREE_FIELDS}
        # the device copies of X, y reuse cached allocator blocks (a process that has trained
        # before): a first cudaMalloc of 1+ GB inside the region made the figure vary 4-25 ms/round
        # from box to box at K = 20
        warm = (torch.empty(Xh.shape, dtype=Xh.dtype, device=dev), torch.empty(yh.shape, dtype=yh.dtype, device=dev))
        del warm
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        Xd = Xh.to(dev, non_blocking=True)
        yd = yh.to(dev, non_blocking=True)
        b2 = G.Booster(ctx, Xd, yd, **kw)
        g2 = None
        # capturing + instantiating the round's graph costs ~17-50 ms of host time
        # (profiles/tools/e2e_breakdown.py) against ~0.2 ms saved per replay: a short training
        # runs its rounds eagerly, a long one replays a graph
        e2e_graph = not a.no_graph and a.steps >= 100
        for i in range(a.steps):
            if i == 0 or not e2e_graph:
                t = b2.round(keep_tree=False)
            else:
                if g2 is None:
                    g2 = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g2):
                        t = b2.round(keep_tree=False)
                g2.replay()
            for nm, _ in G.TREE_FIELDS:
                host_trees[nm][i].copy_(t.arrays[nm], non_blocking=True)
        s1.record(stream)
        barrier()
        e2e_ms = max_over_ranks(s0.elapsed_time(s1) / a.steps)
        h2d = (X.nbytes + y.nbytes) / a.steps
        d2h = sum(v[0].numel() * v.element_size() for v in host_trees.values())
        e2e = {"value": e2e_ms / 1e3, "unit": "s/round", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h,
               "note": "train() from pinned host X,y: H2D + cuts + quantise/compress + K rounds "
                       "(eager below 100 rounds, else CUDA graph replays), each round's tree read back "
                       "to pinned host memory; amortised per round"}
        del b2, Xd, yd, g2

    # ---- the whole training of the config (e.g. 500 rounds for Higgs) from a fresh booster: the
    # per-round cost falls as training proceeds (later trees split off smaller children, so fewer
    # rows are histogrammed), so a K-step window early in training is not the training's average
    full = None
    if not a.no_full_run and a.grow_policy == "depthwise":
        full = time_full_training(G, ctx, torch, Xd_keep, yd_keep, kw, a, stream, barrier, max_over_ranks,
                                  cfg.n_rounds)
    # ---- grad_bits = 30 (SURVEY §8(c) Q4's s = 30 - E): the same timed graph protocol
    p30 = None
    if not a.no_p30 and a.grad_bits != 30 and a.grow_policy == "depthwise":
        p30 = time_precision(G, ctx, torch, dev, Xd_keep, yd_keep, kw, a, stream, barrier, max_over_ranks, 30)
    del Xd_keep, yd_keep
    torch.cuda.empty_cache()
    # ---- CPU baseline + full-size parity: the oracle (threaded, as it stands) on the full rows
    # of this rank's workload for R rounds, the GPU's first R rounds compared with it (rank 0, N=1)
    cpu = parity = None
    if rank == 0 and world == 1 and not (a.no_cpu_baseline and a.no_parity):
        cpu, parity = cpu_baseline_and_parity(G, ctx, torch, dev, X, y, kw, a)
    return dict(p30=p30, parity=parity, full=full, roofline_atomics=roofline_atomics, ms_step=ms_step, n=n, world=world, roofline=roofline, stages=stages, l2=l2_note,
                one_time=one_time, clocks=clk, launches=launches, e2e=e2e, cpu=cpu,
                predict_ms=predict_ms, allreduce_ms=allreduce_ms, grad_bits=a.grad_bits)


def host_facts():
    """Cores this process may use and the CPU model (record nproc and lscpu)."""
    nproc = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return nproc, model


def time_full_training(G, ctx, torch, Xd, yd, kw, a, stream, barrier, max_over_ranks, rounds):
    """Seconds per round averaged over a whole training of `rounds` rounds: one eager round, then
    rounds - 1 replays of the captured round, all inside one pair of CUDA events."""
    b = G.Booster(ctx, Xd, yd, **kw)
    side = torch.cuda.Stream()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    b.round(keep_tree=False)
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            b.round(keep_tree=False)
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(rounds - 1):
        g.replay()
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    del g, b
    return {"rounds": rounds, "total_s": ms / 1e3, "value": ms / 1e3 / rounds, "unit": "s/round",
            "note": "a fresh booster trained for the config's full round count (BASELINE.json), one "
                    "eager round + graph replays, the capture itself included; total / rounds"}


def time_precision(G, ctx, torch, dev, Xd, yd, kw, a, stream, barrier, max_over_ranks, bits):
    """ms per round at another grad_bits (same data, cuts, graph-replay protocol as the line)."""
    kw2 = dict(kw, grad_bits=bits)
    b = G.Booster(ctx, Xd, yd, **kw2)
    for _ in range(a.warmup):
        b.round(keep_tree=False)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        b.round(keep_tree=False)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        b.round(keep_tree=False)
    for _ in range(3):
        g.replay()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        g.replay()
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / a.steps)
    del g, b
    return {"grad_bits": bits, "ms_per_step": ms, "value": ms / 1e3, "unit": "s/round",
            "note": "same workload, cuts and timed CUDA-graph protocol as the line; "
                    "4 ATOMS per (g,h) update instead of 2 (DESIGN.md R14)"}


def oracle_booster(X, y, cfg, a, threads):
    import oracle as O
    O.set_threads(threads)
    beta = 0.0 if cfg.objective == "binary:logistic" else float(np.mean(y.astype(np.float64)))
    t = time.perf_counter()
    b = O.Booster(X, y, max_bins=cfg.max_bins, objective=cfg.objective, max_depth=a.depth,
                  eta=cfg.eta, reg_lambda=cfg.reg_lambda, gamma=cfg.gamma,
                  mcw=cfg.min_child_weight, grad_bits=a.grad_bits, base_margin=beta,
                  grow_policy=a.grow_policy, max_leaves=a.leaves)
    return b, time.perf_counter() - t, beta


def cpu_baseline_and_parity(G, ctx, torch, dev, X, y, kw, a):
    """The oracle (C, -O2, threaded over the host's cores) on the FULL rows of the workload for
    R rounds: its mean seconds per round is cpu_baseline (measured, not extrapolated), and the
    GPU's first R rounds from the same X, y (cuts and packing on the GPU) are compared with it
    field by field: cuts, packed words, every tree field, the row -> leaf map and the margins."""
    cfg = W.CONFIGS[a.config]
    nproc, model = host_facts()
    T = a.cpu_threads or nproc
    R = max(1, a.cpu_rounds)
    ob, t_prep, beta = oracle_booster(X, y, cfg, a, T)
    times, otrees, oleaf = [], [], []
    for _ in range(R):
        t = time.perf_counter()
        otrees.append(ob.round())
        times.append(time.perf_counter() - t)
        oleaf.append(ob.last["row_leaf"].copy())
    cpu = {"value": float(np.mean(times)), "unit": "s/round", "cores": T, "kind": "oracle",
           "host": {"nproc": nproc, "cpu_model": model},
           "sample": f"{R} oracle rounds on all {len(y)} rows of the {a.config} workload "
                     f"(per round {', '.join(f'{t:.2f}' for t in times)} s; one-time cuts + "
                     f"quantise + pack {t_prep:.1f} s not included), C oracle -O2, {T} threads "
                     "(row blocks with private int64 partial histograms)"}
    parity = None
    if not a.no_parity:
        import oracle as O  # noqa: F401  (the oracle is the checker here)
        Xd = torch.from_numpy(X).to(dev)
        yd = torch.from_numpy(y).to(dev)
        gb = G.Booster(ctx, Xd, yd, **dict(kw, base_margin=beta))
        qm = gb.qm
        res = {"rows": int(len(y)), "rounds": R, "cuts": bool(
            np.array_equal(qm.cut_ptr_h, ob.cut_ptr) and
            np.array_equal(qm.cut_values.cpu().numpy().view(np.uint32), ob.cut_values.view(np.uint32))),
            "packed_words": bool(np.array_equal(qm.packed.cpu().numpy().view(np.uint32), ob.words))}
        fields = ("kind", "feature", "bin", "threshold", "default_left", "gain", "weight", "sum_qg",
                  "sum_qh")
        trees_ok, leaf_ok = True, True
        for r in range(R):
            gt = gb.round().to_numpy()
            for k in fields:
                ga, oa = gt[k], otrees[r][k]
                if ga.dtype.kind == "f":
                    ga, oa = ga.view(np.uint64 if ga.itemsize == 8 else np.uint32), \
                        oa.view(np.uint64 if oa.itemsize == 8 else np.uint32)
                trees_ok = trees_ok and bool(np.array_equal(ga, oa))
            leaf_ok = leaf_ok and bool(np.array_equal(gb.row_leaf.cpu().numpy(), oleaf[r]))
        gm = gb.margin.cpu().numpy()
        res.update({"trees": trees_ok, "row_leaf": leaf_ok,
                    "margins": bool(np.array_equal(gm.view(np.uint64), ob.margin.view(np.uint64))),
                    "margins_max_rel_diff": float(np.max(np.abs(gm - ob.margin) /
                                                         np.maximum(np.abs(ob.margin), 1e-300)))})
        res["identical"] = all(res[k] for k in ("cuts", "packed_words", "trees", "row_leaf", "margins"))
        res["fields"] = list(fields)
        parity = res
        del gb, Xd, yd
        torch.cuda.empty_cache()
    if a.no_cpu_baseline:
        cpu = None
    return cpu, parity


def run_reference(a):
    """Reference arm of this tier: the CPU oracle, as it stands, threaded over the host's cores,
    each step one boosting round on ALL rows of the workload (no sample, no extrapolation)."""
    cfg = W.CONFIGS[a.config]
    n = a.rows or cfg.n_rows
    nproc, model = host_facts()
    T = a.cpu_threads or nproc
    X, y = W.generate(a.config, 0, n, n_rows=max(n, cfg.n_rows))
    b, t_prep, _ = oracle_booster(X, y, cfg, a, T)
    for _ in range(a.warmup):
        b.round()
    t = time.perf_counter()
    for _ in range(a.steps):
        b.round()
    per = (time.perf_counter() - t) / a.steps
    sample = (f"each step = one oracle boosting round on all {n} rows of the {a.config} workload "
              f"(C oracle -O2, {T} threads; one-time cuts + quantise + pack {t_prep:.1f} s untimed)")
    out = {"metric": metric_of(a), "value": per, "unit": "s/round", "n_gpus": 0, "steps": a.steps,
           "warmup": a.warmup, "ms_per_step": per * 1e3, "higher_is_better": False,
           "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": a.config, "rows": n, "features": cfg.n_features,
                      "max_bins": cfg.max_bins, "max_depth": a.depth,
                      "objective": cfg.objective, "grad_bits": a.grad_bits, **policy_keys(a)},
           "cpu_baseline": {"value": per, "unit": "s/round", "cores": T, "kind": "oracle",
                            "host": {"nproc": nproc, "cpu_model": model}, "sample": sample},
           "e2e": {"value": per, "unit": "s/round", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def metric_of(a):
    if a.grow_policy == "lossguide":
        return (f"sec/boosting round (loss-guided, {a.leaves} leaves, depth <= {a.depth}, 256 bins); "
                "histogram GB/s vs HBM peak")
    return METRIC


def policy_keys(a):
    keys = {"grow_policy": "lossguide", "max_leaves": a.leaves} if a.grow_policy == "lossguide" else {}
    if a.opt:
        keys["options"] = dict(o.split("=", 1) for o in a.opt)
    return keys


def main():
    a = parse()
    cfg0 = W.CONFIGS[a.config]
    a.depth = a.max_depth if a.max_depth is not None else (
        16 if a.grow_policy == "lossguide" else cfg0.max_depth)
    a.leaves = a.max_leaves if a.max_leaves is not None else (
        2 ** cfg0.max_depth if a.grow_policy == "lossguide" else 0)
    world, rank, local = dist_env()
    a.dist = world > 1 or (a.comm and a.impl == "ours")
    if a.dist:
        import torch
        import torch.distributed as dist
        if world == 1:  # --comm without torchrun: a one-rank group on the loopback interface
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29561")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if a.impl == "reference":
        rc = 0
        if rank == 0:
            rc = run_reference(a)
        if a.dist:
            import torch.distributed as dist
            dist.destroy_process_group()
        return rc
    r = run_ours(a, world, rank, local)
    if rank == 0:
        cfg = W.CONFIGS[a.config]
        out = {
            "metric": metric_of(a),
            "value": r["ms_step"] / 1e3,
            "unit": "s/round",
            "n_gpus": world,
            "steps": a.steps,
            "warmup": a.warmup,
            "ms_per_step": r["ms_step"],
            "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "int64",
            "data": "synthetic",
            "config": {"workload": a.config, "rows": r["n"], "features": cfg.n_features,
                       "max_bins": cfg.max_bins, "max_depth": a.depth, **policy_keys(a),
                       "objective": cfg.objective, "eta": cfg.eta, "grad_bits": r["grad_bits"],
                       "parallelism": f"dp{world} (rows sharded, NCCL histogram allreduce)",
                       "l2": r["l2"]},
            "roofline": r["roofline"],
            "roofline_atomics": r["roofline_atomics"],
            "cpu_baseline": r["cpu"],
            "parity": r["parity"],
            "grad_bits_30": r["p30"],
            "full_training": r["full"],
            "e2e": r["e2e"],
            "gpu_launches": r["launches"],
            "clocks": r["clocks"],
            "stages_ms_per_round (separate eager profiled window)": r["stages"],
            "cuda_graph": not a.no_graph,
            "allreduce_ms_per_round": r["allreduce_ms"],
            "one_time": r["one_time"],
            "predict_ms_10_trees": r["predict_ms"],
        }
        line = json.dumps(out)
        print(line)
        if a.json_out:
            open(a.json_out, "w").write(line + "\n")
    if a.dist:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
