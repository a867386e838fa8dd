# end-of-round check: whole GPU suite, smoke, default bench
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/gputest_r02_final.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r02.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r02.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref_rc=$?
