#!/bin/bash
# ncu --set full of one round's histogram launches (root + levels) of the Higgs bench
mkdir -p gpurun_out/ncu
REGEX="${1:-hist_cs_range|rec_level|part_hist}"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$REGEX" -s ${SKIP:-6} -c ${COUNT:-6} \
  -o gpurun_out/ncu/full -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu/full.log 2>&1
echo NCU_EXIT $? >> gpurun_out/ncu/full.log
