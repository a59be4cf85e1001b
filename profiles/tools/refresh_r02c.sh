#!/bin/bash
# Refresh of the Higgs lines after the 64-row tensor-fed root (one box, one call) + the ncu evidence
mkdir -p gpurun_out/refresh
R=gpurun_out/refresh
run() { name=$1; shift; timeout 1500 python bench.py "$@" --json-out $R/$name.json > $R/$name.log 2>&1; echo "rc=$?" >> $R/$name.log; }
run higgs --steps 200 --warmup 10
run higgs_lossguide --grow-policy lossguide --steps 50 --warmup 5 --cpu-rounds 2
run higgs_comm --comm --steps 200 --warmup 10 --no-cpu-baseline --no-parity
run higgs_k20 --steps 20 --warmup 5 --no-cpu-baseline --no-parity
bash profiles/tools/ncu_r02.sh
echo refresh_done
