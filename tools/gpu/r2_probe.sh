# round-2 first call: box resources, micro layout probe, GPU suite baseline
free -g; nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA"; 
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
./tools/micro/zlayout
./tools/micro/zstride
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
