#!/bin/bash
# host facts for the CPU-oracle baselines (SURVEY §8(d) "Record nproc and lscpu model")
echo "nproc: $(nproc)"
lscpu | grep -E 'Model name|Socket|Core|Thread|^CPU\(s\)|NUMA node\(s\)'
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv
free -g | head -2
