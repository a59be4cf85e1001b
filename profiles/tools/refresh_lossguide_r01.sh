# Loss-guided Higgs bench line + the single-rank communicator path (--comm).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/lg_build.log 2>&1
timeout 600 python bench.py --grow-policy lossguide --max-leaves 64 --steps 50 --warmup 5 --json-out gpurun_out/bench_lossguide.json > gpurun_out/bench_lossguide.log 2>&1
timeout 600 torchrun --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 50 --warmup 5 --comm --no-cpu-baseline --json-out gpurun_out/bench_comm.json > gpurun_out/bench_comm.log 2>&1
echo DONE
