#!/bin/bash
# A/B of runtime options on the Higgs bench: each argument is one --opt list ("" = defaults)
mkdir -p gpurun_out/optab
rm -f gpurun_out/optab/summary.txt
if [ $# -eq 0 ]; then set -- ""; fi
for v in "$@"; do
  o=""; for x in $v; do o="$o --opt $x"; done
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-parity --no-p30 --no-full-run $o ${BENCH_ARGS} > gpurun_out/optab/b.log 2>&1
  python - "$v" <<'PY' >> gpurun_out/optab/summary.txt
import json, sys
try:
    d = json.loads(open('gpurun_out/optab/b.log').readline())
except Exception as e:
    print(repr(sys.argv[1]), "FAILED", open('gpurun_out/optab/b.log').read()[-300:]); sys.exit()
st = d['stages_ms_per_round (separate eager profiled window)']
print(repr(sys.argv[1]), round(d['value'] * 1e3, 4), {k: st[k]['ms_per_round'] for k in ('hist_root', 'hist_level', 'evaluate', 'part_scan', 'part_scatter', 'part_final')})
PY
done
