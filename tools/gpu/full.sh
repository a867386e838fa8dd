timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_full.err
cat gpurun_out/bench_full.json
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
