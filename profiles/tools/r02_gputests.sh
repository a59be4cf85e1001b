#!/bin/bash
# the GPU test suite (optionally a -k expression), log under gpurun_out/gt
mkdir -p gpurun_out/gt
K="${1:-}"
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/gt/pytest.log 2>&1
else
  timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gt/pytest.log 2>&1
fi
echo "rc=$?" >> gpurun_out/gt/pytest.log
