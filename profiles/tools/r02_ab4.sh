#!/bin/bash
mkdir -p gpurun_out/ab4
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "level_hist_layouts" > gpurun_out/ab4/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab4/pytest.log
for o in "LEVEL_HIST=1" "LEVEL_HIST=3"; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --no-full-run --opt $o > gpurun_out/ab4/bench_$o.log 2>&1
done
timeout 900 ncu --set full --clock-control none -k regex:"part_hist" -s 7 -c 5 -o gpurun_out/ab4/ws -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-p30 --no-full-run --opt LEVEL_HIST=3 > gpurun_out/ab4/ncu.log 2>&1
