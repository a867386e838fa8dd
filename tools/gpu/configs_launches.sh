# every config at full size + the ncu launch list of a short C5 bench (our kernels only)
timeout 1200 python tools/gpu/configs_bench.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu --no-solvers > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
