#!/bin/bash
mkdir -p gpurun_out/ctn
timeout 900 ncu --set full --clock-control none -k regex:"hist_ct_root|hist_cs_range" -s 3 -c 1 -o gpurun_out/ctn/higgs_ct -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-p30 --no-full-run > gpurun_out/ctn/a.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"hist_ct_root|hist_cs_range" -s 3 -c 1 -o gpurun_out/ctn/higgs_cs -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-p30 --no-full-run --opt ROOT_TENSOR=1 > gpurun_out/ctn/b.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"hist_ct_root|hist_cs_range" -s 3 -c 1 -o gpurun_out/ctn/eps_ct -f python bench.py --config epsilon --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-parity --no-p30 --no-full-run > gpurun_out/ctn/c.log 2>&1
