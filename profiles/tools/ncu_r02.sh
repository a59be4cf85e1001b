#!/bin/bash
# r02 ncu evidence for the bench line: (1) the launch list of a short bench run (per-launch times,
# cold, serialised: shares only), (2) ncu --set full of the histogram launches of the LAST timed
# graph replay of `bench.py --steps 20 --warmup 5` (the driver's command): launches matched before
# it = 6 per round x (5 warm-up + 1 side-stream warm + 3 untimed replays + 19 timed replays) = 168,
# (3) the other kernels of one round (walk, evaluation, gradients, scatter) and the predictor.
mkdir -p gpurun_out/n2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/n2/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-p30 --no-full-run > gpurun_out/n2/launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"hist_ct_root|hist_cs_range|part_hist|hist_range" -s 168 -c 6 \
  -o gpurun_out/n2/hist -f python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-parity --no-p30 --no-full-run > gpurun_out/n2/hist.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"leaf_walk|eval_tree|grad_quant|part_scatter|part_scan|predict_stg" -s 40 -c 16 \
  -o gpurun_out/n2/other -f python bench.py --steps 3 --warmup 5 --no-e2e --no-cpu-baseline --no-parity --no-p30 --no-full-run > gpurun_out/n2/other.log 2>&1
echo done
