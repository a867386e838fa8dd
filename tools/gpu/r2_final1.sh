# GPU suite (all), default bench, launch list and a full capture of the iteration kernels
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/gputest_r02.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench_rc=$?
CMD="python bench.py --steps 1 --warmup 1 --iters 3 --no-e2e --no-cpu --no-solvers --no-variants"
$CMD > gpurun_out/ncu_final_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1=$?
$CMD > gpurun_out/ncu_final_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_xpass_pipe|k_stile" -s 14 -c 4 -o gpurun_out/prof_r02_iter $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
