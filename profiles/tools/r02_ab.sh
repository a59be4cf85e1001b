#!/bin/bash
# A/B: level paths (records vs row-index lists) in one session + ncu warm-cache capture
mkdir -p gpurun_out/ab
for o in "LEVEL_PATH=1" "LEVEL_PATH=2"; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --opt $o > gpurun_out/ab/bench_$o.log 2>&1
done
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"rec_level|part_hist" -s 5 -c 5 \
  -o gpurun_out/ab/warm -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab/ncu.log 2>&1
