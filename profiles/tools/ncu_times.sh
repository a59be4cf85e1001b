#!/bin/bash
# per-launch durations (one pass, no replay, warm caches) of every kernel of a short bench run
mkdir -p gpurun_out/t
timeout 900 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -c ${COUNT:-400} --csv \
  --log-file gpurun_out/t/launches${TAG}.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/t/ncu${TAG}.log 2>&1
echo rc=$? >> gpurun_out/t/ncu${TAG}.log
