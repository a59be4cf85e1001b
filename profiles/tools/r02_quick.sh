#!/bin/bash
# quick GPU check: selected parity tests, then a short bench (args: pytest -k expression)
mkdir -p gpurun_out/q
K="${1:-record_levels}"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/q/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/q/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/q/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/q/bench.log
