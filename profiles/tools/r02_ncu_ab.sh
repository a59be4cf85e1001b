#!/bin/bash
mkdir -p gpurun_out/nab
timeout 900 ncu --set full --clock-control none -k regex:"part_hist" -s 7 -c 2 -o gpurun_out/nab/compact -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-p30 --opt LEVEL_HIST=1 > gpurun_out/nab/c.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"part_hist" -s 7 -c 2 -o gpurun_out/nab/sb -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-p30 --opt LEVEL_HIST=2 > gpurun_out/nab/s.log 2>&1
