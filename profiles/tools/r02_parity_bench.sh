#!/bin/bash
# full bench line (parity leg + threaded oracle baseline + P=30 figure), reference arm, precision study
mkdir -p gpurun_out/pb
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/pb/bench.log 2>&1; echo "rc=$?" >> gpurun_out/pb/bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/pb/ref.log 2>&1; echo "rc=$?" >> gpurun_out/pb/ref.log
timeout 900 python profiles/tools/precision_quality.py 200 > gpurun_out/pb/precision.json 2> gpurun_out/pb/precision.err
