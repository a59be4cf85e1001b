#!/bin/bash
# A/B of two builds of libgbm.so (libgbm_base.so at the repo root = before, the in-tree build = after)
# over bench configs.  usage: r02_lib_ab.sh "higgs airline ..." [extra bench args]
mkdir -p gpurun_out/libab
rm -f gpurun_out/libab/summary.txt
L=paper_1806_11248_b200/libgbm.so
cp $L libgbm_new.so
for cfg in ${1:-higgs}; do
  for v in base new; do
    cp libgbm_$v.so $L
    timeout 900 python bench.py --config $cfg --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --no-full-run ${@:2} > gpurun_out/libab/b.log 2>&1
    python - "$cfg $v" <<'PY' >> gpurun_out/libab/summary.txt
import json, sys
try:
    d = json.loads(open('gpurun_out/libab/b.log').readline())
except Exception:
    print(sys.argv[1], "FAILED", open('gpurun_out/libab/b.log').read()[-300:]); sys.exit()
st = d['stages_ms_per_round (separate eager profiled window)']
print(sys.argv[1], round(d['ms_per_step'], 4), {k: v['ms_per_round'] for k, v in st.items() if k in ('hist_root', 'hist_level', 'evaluate', 'part_scan', 'part_scatter', 'part_final')})
PY
  done
done
cp libgbm_new.so $L
