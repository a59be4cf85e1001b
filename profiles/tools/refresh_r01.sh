set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1; echo SMOKE_EXIT $? >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo TESTS_EXIT $? >> gpurun_out/gputests.log
timeout 600 python bench.py --json-out gpurun_out/bench_higgs.json > gpurun_out/bench_higgs.log 2>&1
for c in yearmsd epsilon airline bosch tiny; do timeout 600 python bench.py --config $c --json-out gpurun_out/bench_$c.json > gpurun_out/bench_$c.log 2>&1; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo DONE
