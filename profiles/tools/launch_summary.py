"""Summarise an `ncu --metrics gpu__time_duration.sum --clock-control none --csv` launch list of
bench.py into a markdown table of per-round kernel time and shares.

usage: python profiles/tools/launch_summary.py LAUNCHES.csv OUT.md "command line" [bench_ms_per_round]
A boosting round is counted by its init_tree_kernel launch (one per tree); one-time kernels
(cuts, packing, transpose, predict, torch copies) are listed separately."""
import collections
import csv
import sys

src, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
bench_ms = float(sys.argv[4]) if len(sys.argv) > 4 else None
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
rounds = max(c for k, (c, _) in agg.items() if "init_tree_kernel" in k)
ONE_TIME = ("keys_kernel", "sort_", "scan_rows", "runs_count", "select", "cutptr", "tag",
            "write_cuts", "quantise", "pack_kernel", "pack_byte", "transpose", "predict", "at::", "init_")
per_round = {k: v for k, v in agg.items() if not any(t in k for t in ONE_TIME) or "init_tree" in k}
one_time = {k: v for k, v in agg.items() if k not in per_round}
tot = sum(v[1] for v in per_round.values()) / rounds
L = [f"# launch list summary (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
     f"Command: `{cmd}` on one B200.  ncu serialises launches and runs them cold-cache (no graph",
     "overlap of the side stream): compare SHARES, not absolute times.  Raw list: the .csv next to",
     f"this file.  {rounds} boosting rounds executed; one-time kernels listed at the end.", "",
     f"Per-round kernel time under ncu: {tot / 1e3:.3f} ms/round" +
     (f" (bench.py without ncu: {bench_ms:.3f} ms/round)." if bench_ms else "."), "",
     "| kernel | launches | us/round | share of round |", "|---|---|---|---|"]
for k, (c, us) in sorted(per_round.items(), key=lambda x: -x[1][1]):
    L.append(f"| {k} | {c} | {us / rounds:.1f} | {100 * us / rounds / tot:.1f}% |")
hist = sum(us for k, (c, us) in per_round.items()
           if "hist_range" in k or "hist_cs_range" in k or "hist_ct_root" in k or "part_hist" in k) / rounds
L += ["", f"Histogram kernels (root + fused level launches): {100 * hist / tot:.1f}% of the round.", "",
      "One-time kernels (cuts, packing, transpose, predict, torch):", "",
      "| kernel | launches | total us |", "|---|---|---|"]
for k, (c, us) in sorted(one_time.items(), key=lambda x: -x[1][1]):
    L.append(f"| {k} | {c} | {us:.1f} |")
open(out, "w").write("\n".join(L) + "\n")
print("\n".join(L[:30]))
