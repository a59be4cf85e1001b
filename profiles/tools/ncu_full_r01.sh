# One ncu --set full capture of the histogram launches of one Higgs round (root + levels).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu_build.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"hist_cs_range|hist_range|part_hist" -s 6 -c 6 \
  -o gpurun_out/hist_full -f python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo NCU_EXIT $? >> gpurun_out/ncu_full.log
