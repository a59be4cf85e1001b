#!/bin/bash
mkdir -p gpurun_out/ct2
timeout 900 python -m pytest tests -q -m gpu -x -k "root_tensor" > gpurun_out/ct2/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ct2/pytest.log
for c in higgs airline epsilon; do
 for o in 1 2 3 4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --no-full-run --opt ROOT_TENSOR=$o > gpurun_out/ct2/bench_${c}_$o.log 2>&1
 done
done
