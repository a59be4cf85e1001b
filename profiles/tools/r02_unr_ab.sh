#!/bin/bash
# A/B of compile-time tuning defines on the Higgs bench (rebuilds libgbm.so per variant on the box)
mkdir -p gpurun_out/unr
rm -f gpurun_out/unr/summary.txt
if [ $# -eq 0 ]; then set -- "" "-DGBM_PH_UNR=6" "-DGBM_PH_UNR=8"; fi
for v in "$@"; do
  GBM_NVCC_EXTRA="$v" python -c "from paper_1806_11248_b200 import build_lib; build_lib.build(force=True)" > /dev/null 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --no-full-run ${BENCH_ARGS} > gpurun_out/unr/b.log 2>&1
  python - "$v" <<'PY' >> gpurun_out/unr/summary.txt
import json, sys
d = json.loads(open('gpurun_out/unr/b.log').readline())
st = d['stages_ms_per_round (separate eager profiled window)']
print(repr(sys.argv[1]), round(d['value'] * 1e3, 4), {k: st[k]['ms_per_round'] for k in ('hist_root', 'hist_level', 'evaluate', 'part_final')})
PY
done
python -c "from paper_1806_11248_b200 import build_lib; build_lib.build(force=True)" > /dev/null 2>&1
