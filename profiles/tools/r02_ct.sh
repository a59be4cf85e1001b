#!/bin/bash
mkdir -p gpurun_out/ct
timeout 1500 python -m pytest tests -q -m gpu -x -k "staged_root or histogram_parity or training_rounds or full_size or virtual_shards or lossguide_rounds or fused_round" > gpurun_out/ct/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ct/pytest.log
for c in higgs epsilon airline; do
 for o in "ROOT_TENSOR=0" "ROOT_TENSOR=1"; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --no-full-run --opt $o > gpurun_out/ct/bench_${c}_$o.log 2>&1
 done
done
