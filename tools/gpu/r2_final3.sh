# last session of round 2: whole GPU suite (with durations), smoke, default
# bench, reference arm, launch list and a full capture of the iteration kernels
timeout 1500 python -m pytest tests -m gpu -q --durations=25 2>&1 | tail -40 > gpurun_out/gputest_r02_s3.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r02_s3.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_r02_s3.log
python bench.py > gpurun_out/bench_r02_s3.json 2> gpurun_out/bench_r02_s3.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_s3.json 2> gpurun_out/bench_ref_s3.err; echo ref_rc=$?
CMD="python bench.py --steps 1 --warmup 1 --iters 3 --no-e2e --no-cpu --no-solvers --no-variants"
$CMD > gpurun_out/ncu_s3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_s3.csv $CMD > gpurun_out/ncu_s3_launch.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:"k_xpass_pipe|k_stile" -s 14 -c 4 -o gpurun_out/prof_r02_s3_iter $CMD > gpurun_out/ncu_s3_full.log 2>&1; echo ncu2=$?
