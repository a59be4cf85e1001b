#!/bin/bash
# Round-2 bench refresh: every config with its full-size parity leg and threaded oracle baseline
# (one box, one call); JSON lines under gpurun_out/refresh/.
mkdir -p gpurun_out/refresh
R=gpurun_out/refresh
bash profiles/tools/hostinfo.sh > $R/hostinfo.txt 2>&1
run() { name=$1; shift; timeout 1500 python bench.py "$@" --json-out $R/$name.json > $R/$name.log 2>&1; echo "rc=$?" >> $R/$name.log; }
run higgs --steps 200 --warmup 10
run yearmsd --config yearmsd --steps 200 --warmup 10
run epsilon --config epsilon --steps 100 --warmup 5 --cpu-rounds 2
run bosch --config bosch --steps 100 --warmup 5 --cpu-rounds 2
run airline --config airline --steps 50 --warmup 5 --cpu-rounds 1
run higgs_lossguide --grow-policy lossguide --steps 50 --warmup 5 --cpu-rounds 2
run higgs_comm --comm --steps 200 --warmup 10 --no-cpu-baseline --no-parity
run higgs_ref --impl reference --steps 20 --warmup 5
