# ncu --set full of one iteration's strided passes (k_stile) at 1024^3
set -e
CMD="python bench.py --steps 1 --warmup 3 --iters 2 --no-e2e --no-cpu"
$CMD > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stile -s 3 -c 3 \
    -o gpurun_out/prof_stile -f $CMD > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log
