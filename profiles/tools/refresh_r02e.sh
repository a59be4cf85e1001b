#!/bin/bash
# Final refresh after the exactness cap of the tensor-fed root's work items (Airline, Higgs lines)
mkdir -p gpurun_out/refresh
R=gpurun_out/refresh
run() { name=$1; shift; timeout 1500 python bench.py "$@" --json-out $R/$name.json > $R/$name.log 2>&1; echo "rc=$?" >> $R/$name.log; }
run higgs --steps 200 --warmup 10
run higgs_k20 --steps 20 --warmup 5 --no-cpu-baseline --no-parity
run airline --config airline --steps 50 --warmup 5 --cpu-rounds 1
run higgs_lossguide --grow-policy lossguide --steps 50 --warmup 5 --cpu-rounds 2
run higgs_comm --comm --steps 200 --warmup 10 --no-cpu-baseline --no-parity
echo refresh_done
