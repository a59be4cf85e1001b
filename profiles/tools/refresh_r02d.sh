#!/bin/bash
# Refresh of one line after the evaluation-kernel rule for >= 64 features (YearMSD, Bosch, then Epsilon)
mkdir -p gpurun_out/refresh
R=gpurun_out/refresh
run() { name=$1; shift; timeout 1500 python bench.py "$@" --json-out $R/$name.json > $R/$name.log 2>&1; echo "rc=$?" >> $R/$name.log; }
run epsilon --config epsilon --steps 100 --warmup 5 --cpu-rounds 2

echo refresh_done
