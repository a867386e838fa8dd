# full GPU suite, default bench, smoke, ncu launch list + ncu --set full of the iteration kernels
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_full.err
cat gpurun_out/bench_full.json
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CMD="python bench.py --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu --no-solvers"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_xpass_pipe|k_stile" -s 8 -c 4 -o gpurun_out/prof_iter -f $CMD > gpurun_out/ncu.log 2>&1; echo "ncu full rc=$?"
