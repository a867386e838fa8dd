# re-entry check of HEAD on a fresh box: whole GPU suite (with durations), smoke, default bench, reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=25 2>&1 | tail -40 > gpurun_out/gputest_r02_s7.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02_s7.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r02_s7.log
python bench.py > gpurun_out/bench_r02_s7.json 2> gpurun_out/bench_r02_s7.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_s7.json 2> gpurun_out/bench_ref_s7.err; echo ref_rc=$?
