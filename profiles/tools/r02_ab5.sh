#!/bin/bash
mkdir -p gpurun_out/ab5
for c in epsilon yearmsd bosch; do
for o in "HIST_LAYOUT=0" "HIST_LAYOUT=2" "HIST_LAYOUT=3" "LEVEL_HIST=3"; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --no-full-run --opt $o > gpurun_out/ab5/bench_${c}_$o.log 2>&1
done; done
