# end-of-session check after the LSA-barrier / bench changes: whole GPU suite, smoke, default bench
timeout 1500 python -m pytest tests -m gpu -q --durations=10 2>&1 | tail -18 > gpurun_out/gputest_r02_s4.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r02_s4.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r02_s4.log
python bench.py > gpurun_out/bench_r02_s4.json 2> gpurun_out/bench_r02_s4.err; echo bench_rc=$?
