#!/bin/bash
mkdir -p gpurun_out/ab6
timeout 1500 python -m pytest tests -q -m gpu -x -k "evaluate or training_rounds or lossguide or virtual or full_size" > gpurun_out/ab6/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab6/pytest.log
for c in higgs epsilon bosch yearmsd; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --no-full-run > gpurun_out/ab6/bench_$c.log 2>&1
done
