# default bench line + smoke + ncu launch list of a short bench (cold, serialised per-launch times)
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_full.err
cat gpurun_out/bench_full.json
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu --no-solvers > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
