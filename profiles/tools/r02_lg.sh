#!/bin/bash
mkdir -p gpurun_out/lg
for o in "" "--opt GROUP_UNITS=2" "--opt GROUP_UNITS=4" "--opt RUN_TILES=1" "--opt GROUP_UNITS=2 --opt RUN_TILES=1" "--opt EVAL_WARP=1"; do
  n=$(echo "$o" | tr -d ' -=' ); [ -z "$n" ] && n=default
  timeout 600 python bench.py --grow-policy lossguide --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --no-full-run $o > gpurun_out/lg/bench_$n.log 2>&1
done
