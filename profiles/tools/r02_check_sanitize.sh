mkdir -p gpurun_out/r02a
bash profiles/tools/hostinfo.sh > gpurun_out/r02a/hostinfo.txt 2>&1
python -c "import os; print(os.cpu_count(), len(os.sched_getaffinity(0)))" >> gpurun_out/r02a/hostinfo.txt
( time python -m pytest tests -m gpu -x -q ) > gpurun_out/r02a/pytest_gpu.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python profiles/tools/sanitize_run.py tiny higgs bosch > gpurun_out/r02a/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r02a/sanitize_$tool.log
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02a/bench.log 2>&1
