# Option sweep on the Higgs default workload (bench.py --opt NAME=VALUE); one line per setting.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sw_build.log 2>&1
for o in "" "RUN_TILES=1" "RUN_TILES=2" "RUN_TILES=4" "RUN_TILES=8" "GROUP_UNITS=16" "CARRY_GRADIENTS=1" "HIST_LAYOUT=1" "SEGMENT_HIST=2" "EVAL_WARP=1" "EVAL_WARP=2"; do
  arg=""; [ -n "$o" ] && arg="--opt $o"
  timeout 300 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline $arg > gpurun_out/sw.log 2>&1
  echo "$o $(tail -n 1 gpurun_out/sw.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])' 2>&1)" >> gpurun_out/sweep_higgs.txt
done
