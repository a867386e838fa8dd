# GPU suite, then the launch list and one ncu --set full capture of an iteration's kernels at 1024^3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
CMD="python bench.py --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_stile|k_xpass_pipe" -s 6 -c 4 \
    -o gpurun_out/prof_iter -f $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu.log
