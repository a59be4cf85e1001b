#!/bin/bash
mkdir -p gpurun_out/ab3
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "level_hist_layouts" > gpurun_out/ab3/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab3/pytest.log
for o in "LEVEL_HIST=1" "LEVEL_HIST=2"; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --opt $o > gpurun_out/ab3/bench_$o.log 2>&1
done
