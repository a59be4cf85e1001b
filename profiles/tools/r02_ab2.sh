#!/bin/bash
# A/B of level layouts + the one-rank communicator path, one box
mkdir -p gpurun_out/ab2
for o in "HIST_LAYOUT=0" "HIST_LAYOUT=2" "HIST_LAYOUT=3" "HIST_LAYOUT=4"; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --opt $o > gpurun_out/ab2/bench_$o.log 2>&1
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --comm > gpurun_out/ab2/bench_comm.log 2>&1
