#!/bin/bash
# Refresh of the YearMSD and Bosch lines after the evaluation-kernel rule for >= 64 features
mkdir -p gpurun_out/refresh
R=gpurun_out/refresh
run() { name=$1; shift; timeout 1500 python bench.py "$@" --json-out $R/$name.json > $R/$name.log 2>&1; echo "rc=$?" >> $R/$name.log; }
run yearmsd --config yearmsd --steps 200 --warmup 10
run bosch --config bosch --steps 100 --warmup 5 --cpu-rounds 2
echo refresh_done
