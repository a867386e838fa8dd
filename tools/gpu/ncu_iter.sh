# ncu --set full (with source) of one C5 iteration's kernels after the store changes
set -e
CMD="python bench.py --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu --no-solvers"
timeout 600 $CMD > gpurun_out/plain.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_xpass_pipe|k_stile" -s 8 -c 4 \
    -o gpurun_out/prof_iter -f $CMD > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
