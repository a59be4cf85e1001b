#!/bin/bash
mkdir -p gpurun_out/ee
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_tree" -s 12 -c 6 -o gpurun_out/ee/eval -f python bench.py --config epsilon --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-p30 --no-full-run > gpurun_out/ee/ncu.log 2>&1
